// lorakv/kvcache.hpp -- the scheme-aware cache store of the reference (proj/include/lorakv/kvcache.hpp)
// kept in B200 HBM.  Same class and function names, argument meaning and error text:
//
//   plan_core / PrefillPlan / Interval   kvcache.hpp:79-142   pure integers, via lorakv_plan_core
//   KvStore<T>                           kvcache.hpp:213-420  a lorakv_pool: paged HBM cache + host bookkeeping
//   CacheBytes / bytes()                 kvcache.hpp:144-150, 330-358
//   plan_step                            kvcache.hpp:423-425
//
// What differs, by design:
//   * rows live in pages on the device (page_layout.cuh); append_* copies the caller's rows in (first
//     writer wins, resolved on the host before any launch) and *_view() de-paginates into a host
//     buffer owned by the store, valid until the next append or view of the same buffer;
//   * the store needs the head split and a capacity up front -> DeviceOptions (defaults keep the
//     reference's two-argument constructor source-compatible);
//   * T is float.  HBM storage is fp32 (bit-exact views) or, with DeviceOptions::bf16, bfloat16;
//   * SelectiveRecompute, the hidden-state cache and snapshot files belong to a baseline scheme and
//     to I/O outside the Flash-LoRA-Attention path: constructing that scheme fails, append_hidden /
//     recompute_overwrite throw the reference's own errors for the schemes that exist here.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "lorakv/matrix.hpp"

namespace lorakv {

enum class SchemeKind { NonShared, FullShared, BaseShared, BaseLRShared, SelectiveRecompute };

struct CacheScheme {
  SchemeKind kind = SchemeKind::NonShared;
  std::vector<idx> recompute_layers;   // SelectiveRecompute only; sorted, unique

  std::string name() const {
    static const char* const names[] = {"NonShared", "FullShared", "BaseShared", "BaseLRShared", "SelectiveRecompute"};
    return names[static_cast<int>(kind)];
  }
  static CacheScheme parse(const std::string& s) {
    for (int k = 0; k < 5; ++k) {
      CacheScheme c{static_cast<SchemeKind>(k), {}};
      if (c.name() == s) return c;
    }
    fail("unknown cache scheme '" + s + "'");
  }
  bool is_recompute_layer(idx layer) const {
    return std::binary_search(recompute_layers.begin(), recompute_layers.end(), layer);
  }
  idx first_recompute() const { return recompute_layers.empty() ? 0 : recompute_layers.front(); }
};

// half-open token interval
struct Interval {
  idx begin = 0;
  idx end = 0;
  idx size() const { return end - begin; }
  bool empty() const { return end <= begin; }
  bool operator==(const Interval& o) const { return begin == o.begin && end == o.end; }
};

struct PrefillPlan {
  Interval hidden_pass;
  Interval kv_project;
  Interval lr_project;
  Interval kv_recompute;
  idx skip_layers_below = 0;

  Interval kv_project_at(idx layer, const CacheScheme& scheme) const {
    const bool redo = scheme.kind == SchemeKind::SelectiveRecompute && scheme.is_recompute_layer(layer);
    return redo ? kv_recompute : kv_project;
  }
  Interval lr_project_at(idx layer, const CacheScheme& scheme) const {
    const bool redo = scheme.kind == SchemeKind::SelectiveRecompute && scheme.is_recompute_layer(layer);
    return redo ? kv_recompute : lr_project;
  }
};

// length = trajectory length before the step, seen = how far this agent has processed
inline PrefillPlan plan_core(const CacheScheme& scheme, idx length, idx seen, idx new_tokens) {
  std::int64_t v[9];
  b200::check(lorakv_plan_core(static_cast<int>(scheme.kind), scheme.first_recompute(), length, seen, new_tokens, v));
  PrefillPlan p;
  p.hidden_pass = Interval{v[0], v[1]};
  p.kv_project = Interval{v[2], v[3]};
  p.lr_project = Interval{v[4], v[5]};
  p.kv_recompute = Interval{v[6], v[7]};
  p.skip_layers_below = v[8];
  return p;
}

struct CacheBytes {
  std::uint64_t key = 0;
  std::uint64_t value = 0;
  std::uint64_t lr = 0;
  std::uint64_t hidden = 0;
  std::uint64_t total() const { return key + value + lr + hidden; }
};

struct StoreDims {
  idx n_layers = 0;
  idx d_kv = 0;      // n_kv_heads * d_head
  idx d_model = 0;
  idx rank = 0;
  idx n_agents = 0;
};

// Device-side choices the reference has no counterpart for.
struct DeviceOptions {
  idx n_kv_heads = 1;       // d_head = d_kv / n_kv_heads
  idx max_tokens = 4096;    // capacity of the trajectory (rounded up to whole pages)
  bool bf16 = false;        // bfloat16 pages (the hot-path storage mode) instead of fp32
  idx page_tokens = 0;      // 0 = library default (64)
  idx kv_head_begin = 0;    // this store keeps kv heads [kv_head_begin, kv_head_begin + n_kv_local)
  idx n_kv_local = 0;       // 0 = all of them (single GPU)
};

template <class T>
class KvStore {
  static_assert(std::is_same_v<T, float>, "the HBM cache stores fp32 or bf16 rows: use KvStore<float>");

 public:
  KvStore(CacheScheme scheme, StoreDims dims, DeviceOptions opt = DeviceOptions{})
      : scheme_(std::move(scheme)), dims_(dims), opt_(opt) {
    if (dims.n_layers < 1 || dims.d_kv < 1 || dims.d_model < 1 || dims.n_agents < 1) fail("KvStore: invalid dims");
    if (dims.rank < 0) fail("KvStore: negative rank");
    if (opt.n_kv_heads < 1 || dims.d_kv % opt.n_kv_heads != 0) fail("KvStore: d_kv is not a multiple of n_kv_heads");
    lorakv_pool_dims pd{};
    pd.scheme = static_cast<int>(scheme_.kind);
    pd.dtype = opt.bf16 ? LORAKV_BF16 : LORAKV_F32;
    pd.n_layers = dims.n_layers;
    pd.n_kv_heads = opt.n_kv_heads;
    pd.d_head = dims.d_kv / opt.n_kv_heads;
    pd.d_model = dims.d_model;
    pd.rank = dims.rank;
    pd.n_agents = dims.n_agents;
    pd.page_tokens = opt.page_tokens;
    pd.max_tokens = opt.max_tokens;
    pd.kv_head_begin = opt.kv_head_begin;
    pd.n_kv_local = opt.n_kv_local;
    b200::check(lorakv_pool_create(b200::Runtime::ctx(), &pd, &pool_));
  }
  ~KvStore() { lorakv_pool_destroy(pool_); }
  KvStore(const KvStore&) = delete;
  KvStore& operator=(const KvStore&) = delete;
  KvStore(KvStore&& o) noexcept
      : scheme_(std::move(o.scheme_)), dims_(o.dims_), opt_(o.opt_), pool_(o.pool_), tokens_(std::move(o.tokens_)),
        views_(std::move(o.views_)) {
    o.pool_ = nullptr;
  }

  const CacheScheme& scheme() const { return scheme_; }
  const StoreDims& dims() const { return dims_; }
  const DeviceOptions& device_options() const { return opt_; }
  idx length() const { return lorakv_pool_length(pool_); }
  const std::vector<std::int32_t>& tokens() const { return tokens_; }
  lorakv_pool* handle() const { return pool_; }

  void append_tokens(const std::vector<std::int32_t>& ids) {
    b200::check(lorakv_pool_append_tokens(pool_, static_cast<idx>(ids.size())));
    tokens_.insert(tokens_.end(), ids.begin(), ids.end());
  }

  idx seen(idx agent) const {
    std::int64_t s = 0;
    b200::check(lorakv_pool_seen(pool_, agent, &s));
    return s;
  }
  void mark_seen(idx agent) { b200::check(lorakv_pool_mark_seen(pool_, agent)); }

  // First-writer-wins appends: rows the buffer already holds are skipped, a gap is an error.
  void append_key(idx layer, idx agent, idx row_begin, Span2D<const T> rows) { append(LORAKV_KEY, layer, agent, row_begin, rows); }
  void append_value(idx layer, idx agent, idx row_begin, Span2D<const T> rows) { append(LORAKV_VALUE, layer, agent, row_begin, rows); }
  void append_lr(idx layer, idx agent, idx row_begin, Span2D<const T> rows) { append(LORAKV_LR, layer, agent, row_begin, rows); }

  void append_hidden(idx, Span2D<const T>) { fail("KvStore: scheme " + scheme_.name() + " has no hidden-state cache"); }
  void recompute_overwrite(idx layer, idx, Span2D<const T>, Span2D<const T>) {
    fail("KvStore: overwrite of existing cache rows is forbidden (scheme " + scheme_.name() + ", layer " +
         std::to_string(layer) + ")");
  }

  Span2D<const T> key_view(idx layer, idx agent) const { return view(LORAKV_KEY, layer, agent); }
  Span2D<const T> value_view(idx layer, idx agent) const { return view(LORAKV_VALUE, layer, agent); }
  // zero-column span (L x 0) when the scheme keeps no low-rank cache
  Span2D<const T> lr_view(idx layer, idx agent) const { return view(LORAKV_LR, layer, agent); }

  CacheBytes bytes() const {
    std::uint64_t b[4];
    b200::check(lorakv_pool_bytes(pool_, b));
    return CacheBytes{b[0], b[1], b[2], b[3]};
  }
  std::uint64_t allocated_elements() const { return lorakv_pool_allocated_elements(pool_); }
  // HBM actually reserved for pages (capacity, not occupancy)
  std::uint64_t reserved_bytes() const { return lorakv_pool_reserved_bytes(pool_); }

  // The reference's snapshot container (kvcache.hpp:438-546 of the reference), written from / read into HBM pages.
  // load_snapshot needs the device options a snapshot does not carry (head split, capacity, storage dtype).
  void save_snapshot(const std::string& path) const {
    b200::check(lorakv_pool_save_snapshot(pool_, path.c_str(), tokens_.data(), static_cast<idx>(tokens_.size())));
  }
  static KvStore load_snapshot(const std::string& path, DeviceOptions opt = DeviceOptions{}) {
    lorakv_pool* pool = nullptr;
    std::int64_t n_tokens = 0;
    std::vector<std::int32_t> tokens(static_cast<std::size_t>(1) << 20);
    b200::check(lorakv_pool_load_snapshot(b200::Runtime::ctx(), path.c_str(), opt.bf16 ? LORAKV_BF16 : LORAKV_F32, opt.n_kv_heads,
                                          opt.page_tokens, opt.max_tokens, &pool, tokens.data(), static_cast<idx>(tokens.size()),
                                          &n_tokens));
    tokens.resize(static_cast<std::size_t>(std::min<std::int64_t>(n_tokens, static_cast<std::int64_t>(tokens.size()))));
    lorakv_pool_dims pd{};
    b200::check(lorakv_pool_dims_get(pool, &pd));
    return KvStore(pool, pd, opt, std::move(tokens));
  }

  // logical page -> physical page of the page set (which, agent) resolves to
  std::vector<std::int32_t> page_table(int which, idx agent) const {
    std::int64_t n = 0;
    b200::check(lorakv_pool_page_table(pool_, which, agent, nullptr, 0, &n));
    std::vector<std::int32_t> t(static_cast<std::size_t>(n));
    if (n > 0) b200::check(lorakv_pool_page_table(pool_, which, agent, t.data(), n, &n));
    return t;
  }

 private:
  KvStore(lorakv_pool* pool, const lorakv_pool_dims& pd, DeviceOptions opt, std::vector<std::int32_t> tokens)
      : scheme_{static_cast<SchemeKind>(pd.scheme), {}}, dims_{pd.n_layers, pd.n_kv_heads * pd.d_head, pd.d_model, pd.rank, pd.n_agents},
        opt_(opt), pool_(pool), tokens_(std::move(tokens)) {
    opt_.page_tokens = pd.page_tokens; opt_.max_tokens = pd.max_tokens;
  }

  void append(int which, idx layer, idx agent, idx row_begin, Span2D<const T> rows) {
    const idx want = which == LORAKV_LR ? dims_.rank : dims_.d_kv;
    const bool has_buffer = which != LORAKV_LR || scheme_.kind == SchemeKind::BaseShared || scheme_.kind == SchemeKind::BaseLRShared;
    if (has_buffer && rows.cols != want) fail("GrowMat::append: column mismatch");
    b200::check(lorakv_pool_append(pool_, which, layer, agent, row_begin, rows.data, rows.rows, rows.stride, LORAKV_HOST, nullptr));
  }

  Span2D<const T> view(int which, idx layer, idx agent) const {
    std::int64_t n = 0;
    b200::check(lorakv_pool_rows(pool_, which, layer, agent, &n));
    const bool lr_less = which == LORAKV_LR && scheme_.kind != SchemeKind::BaseShared && scheme_.kind != SchemeKind::BaseLRShared;
    if (lr_less) return Span2D<const T>{nullptr, n, 0, 0};
    const idx local_heads = opt_.n_kv_local > 0 ? opt_.n_kv_local : opt_.n_kv_heads - opt_.kv_head_begin;
    const idx cols = which == LORAKV_LR ? dims_.rank : local_heads * (dims_.d_kv / opt_.n_kv_heads);
    std::vector<T>& buf = views_[std::make_tuple(which, layer, agent)];
    buf.assign(static_cast<std::size_t>(n * cols), T(0));
    if (n * cols > 0) b200::check(lorakv_pool_read(pool_, which, layer, agent, 0, n, buf.data()));
    return Span2D<const T>{buf.data(), n, cols, cols};
  }

  CacheScheme scheme_;
  StoreDims dims_;
  DeviceOptions opt_;
  lorakv_pool* pool_ = nullptr;
  std::vector<std::int32_t> tokens_;
  mutable std::map<std::tuple<int, idx, idx>, std::vector<T>> views_;
};

template <class T>
inline PrefillPlan plan_step(const KvStore<T>& store, idx agent, idx new_tokens) {
  return plan_core(store.scheme(), store.length(), store.seen(agent), new_tokens);
}

}  // namespace lorakv
