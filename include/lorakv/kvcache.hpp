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
//   * KvStore<float>: HBM storage is fp32 (bit-exact views) or, with DeviceOptions::bf16, bfloat16 -- the hot path.
//     KvStore<double>: fp64 pages, exact rows; storage only (the attention kernels read fp32 / bf16 pages), there so that
//     the reference's double-precision callers and tests (tests/test_kvcache.cpp, step<double>) run against this store;
//   * SelectiveRecompute with its hidden-state cache and recompute_overwrite (kvcache.hpp:53-58, 289-305) is a baseline
//     scheme outside the Flash-LoRA-Attention path; the store implements it (shared K / V pages, one hidden cache paged
//     through the same table, overwrite on the recompute layers only) for the same reason.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "lorakv/matrix.hpp"
#include "lorakv/rng.hpp"

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

  // The reference's pseudo-sensitivity pick (kvcache.hpp:56-76): ceil(n / 3) layers, layer 0 always among them, the others
  // the head of a seeded Fisher-Yates shuffle of 1 .. n-1 (stream Rng::mix(seed, 0x5ec7), draws taken modulo the shrinking
  // range from the back).  Pure integers: must reproduce the reference's list exactly.
  static std::vector<idx> default_recompute_layers(idx n_layers, std::uint64_t seed) {
    if (n_layers < 1) fail("default_recompute_layers: n_layers must be >= 1");
    std::vector<idx> upper(static_cast<std::size_t>(n_layers - 1));
    for (std::size_t i = 0; i < upper.size(); ++i) upper[i] = static_cast<idx>(i) + 1;
    Rng rng(Rng::mix(seed, 0x5ec7));
    for (std::size_t hi = upper.size(); hi > 1; --hi) std::swap(upper[hi - 1], upper[rng.next_u64() % hi]);
    const std::size_t extra = std::min<std::size_t>(static_cast<std::size_t>((n_layers + 2) / 3 - 1), upper.size());
    std::vector<idx> picked{0};
    picked.insert(picked.end(), upper.begin(), upper.begin() + static_cast<std::ptrdiff_t>(extra));
    std::sort(picked.begin(), picked.end());
    return picked;
  }
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

namespace detail {
// snapshot dtype tag of an element type (kvcache.hpp:429-435)
template <class T> const char* dtype_name();
template <> inline const char* dtype_name<float>() { return "f32"; }
template <> inline const char* dtype_name<double>() { return "f64"; }
}  // namespace detail

template <class T>
class KvStore {
  static_assert(b200::is_supported<T>, "KvStore exists for float (fp32 / bf16 pages) and double (fp64 pages)");
  static constexpr bool kDouble = std::is_same_v<T, double>;

 public:
  KvStore(CacheScheme scheme, StoreDims dims, DeviceOptions opt = DeviceOptions{})
      : scheme_(std::move(scheme)), dims_(dims), opt_(opt) {
    if (dims.n_layers < 1 || dims.d_kv < 1 || dims.d_model < 1 || dims.n_agents < 1) fail("KvStore: invalid dims");
    if (dims.rank < 0) fail("KvStore: negative rank");
    for (idx l : scheme_.recompute_layers)
      if (l < 0 || l >= dims.n_layers) fail("KvStore: recompute layer " + std::to_string(l) + " out of range");
    if (scheme_.kind == SchemeKind::SelectiveRecompute && scheme_.recompute_layers.empty())
      fail("KvStore: SelectiveRecompute requires a non-empty recompute set");
    if (opt.n_kv_heads < 1 || dims.d_kv % opt.n_kv_heads != 0) fail("KvStore: d_kv is not a multiple of n_kv_heads");
    if (kDouble && opt.bf16) fail("KvStore<double>: fp64 pages; bf16 storage belongs to KvStore<float>");
    lorakv_pool_dims pd{};
    pd.scheme = static_cast<int>(scheme_.kind);
    pd.dtype = kDouble ? LORAKV_F64 : (opt.bf16 ? LORAKV_BF16 : LORAKV_F32);
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
    if (!scheme_.recompute_layers.empty()) {
      std::vector<std::int64_t> rl(scheme_.recompute_layers.begin(), scheme_.recompute_layers.end());
      b200::check(lorakv_pool_set_recompute_layers(pool_, rl.data(), static_cast<idx>(rl.size())));
    }
  }
  ~KvStore() { lorakv_pool_destroy(pool_); }
  // A copy is a second pool with the same contents (the reference's store is a value type; test_engine.cpp:498 keeps a
  // "before" copy): rows travel device -> host -> device, bookkeeping is replayed (tokens, seen_upto in ascending order).
  KvStore(const KvStore& o) : KvStore(o.scheme_, o.dims_, o.opt_) { copy_from(o); }
  KvStore& operator=(const KvStore& o) {
    if (this != &o) { KvStore tmp(o); *this = std::move(tmp); }
    return *this;
  }
  KvStore(KvStore&& o) noexcept
      : scheme_(std::move(o.scheme_)), dims_(o.dims_), opt_(o.opt_), pool_(o.pool_), tokens_(std::move(o.tokens_)),
        views_(std::move(o.views_)) {
    o.pool_ = nullptr;
  }
  KvStore& operator=(KvStore&& o) noexcept {
    if (this != &o) {
      lorakv_pool_destroy(pool_);
      scheme_ = std::move(o.scheme_); dims_ = o.dims_; opt_ = o.opt_; pool_ = o.pool_; tokens_ = std::move(o.tokens_);
      views_ = std::move(o.views_);
      o.pool_ = nullptr;
    }
    return *this;
  }

  const CacheScheme& scheme() const { return scheme_; }
  const StoreDims& dims() const { return dims_; }
  const DeviceOptions& device_options() const { return opt_; }
  idx length() const { return lorakv_pool_length(pool_); }
  const std::vector<std::int32_t>& tokens() const { return tokens_; }
  lorakv_pool* handle() const { return pool_; }

  void append_tokens(const std::vector<std::int32_t>& ids) {
    // the device capacity is a DeviceOptions choice the reference has no counterpart for: grow it with the trajectory
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
  void append_hidden(idx row_begin, Span2D<const T> rows) {
    if (scheme_.kind != SchemeKind::SelectiveRecompute) fail("KvStore: scheme " + scheme_.name() + " has no hidden-state cache");
    append(LORAKV_HIDDEN, 0, 0, row_begin, rows);
  }

  // Overwrite of rows that exist: only the recompute layers of SelectiveRecompute may (kvcache.hpp:298-305).
  void recompute_overwrite(idx layer, idx row_begin, Span2D<const T> k_rows, Span2D<const T> v_rows) {
    if (scheme_.kind != SchemeKind::SelectiveRecompute || !scheme_.is_recompute_layer(layer))
      fail("KvStore: overwrite of existing cache rows is forbidden (scheme " + scheme_.name() + ", layer " + std::to_string(layer) + ")");
    if (layer < 0 || layer >= dims_.n_layers) fail("layer " + std::to_string(layer) + " out of range");
    if (k_rows.cols != dims_.d_kv || v_rows.cols != dims_.d_kv) fail("GrowMat::overwrite: column mismatch");
    overwrite(LORAKV_KEY, layer, row_begin, k_rows);
    overwrite(LORAKV_VALUE, layer, row_begin, v_rows);
  }

  Span2D<const T> key_view(idx layer, idx agent) const { return view(LORAKV_KEY, layer, agent); }
  Span2D<const T> value_view(idx layer, idx agent) const { return view(LORAKV_VALUE, layer, agent); }
  // zero-column span (L x 0) when the scheme keeps no low-rank cache
  Span2D<const T> lr_view(idx layer, idx agent) const { return view(LORAKV_LR, layer, agent); }
  Span2D<const T> hidden_rows(idx begin, idx end) const {
    if (scheme_.kind != SchemeKind::SelectiveRecompute) return Span2D<const T>{nullptr, 0, 0, 0}.row_range(begin, end);
    return view(LORAKV_HIDDEN, 0, 0).row_range(begin, end);
  }
  idx hidden_size() const {
    if (scheme_.kind != SchemeKind::SelectiveRecompute) return 0;
    std::int64_t n = 0;
    b200::check(lorakv_pool_rows(pool_, LORAKV_HIDDEN, 0, 0, &n));
    return n;
  }

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
    std::int64_t n_tokens = 0;
    b200::check(lorakv_snapshot_tokens(path.c_str(), nullptr, 0, &n_tokens));       // size the token list first
    std::vector<std::int32_t> tokens(static_cast<std::size_t>(n_tokens));
    lorakv_pool* pool = nullptr;
    b200::check(lorakv_pool_load_snapshot(b200::Runtime::ctx(), path.c_str(), kDouble ? LORAKV_F64 : (opt.bf16 ? LORAKV_BF16 : LORAKV_F32),
                                          opt.n_kv_heads, opt.page_tokens, opt.max_tokens, &pool, tokens.data(),
                                          static_cast<idx>(tokens.size()), &n_tokens));
    lorakv_pool_dims pd{};
    b200::check(lorakv_pool_dims_get(pool, &pd));
    std::int64_t n_rl = 0;
    b200::check(lorakv_pool_get_recompute_layers(pool, nullptr, 0, &n_rl));
    std::vector<std::int64_t> rl(static_cast<std::size_t>(n_rl));
    if (n_rl > 0) b200::check(lorakv_pool_get_recompute_layers(pool, rl.data(), n_rl, &n_rl));
    KvStore s(pool, pd, opt, std::move(tokens));
    s.scheme_.recompute_layers.assign(rl.begin(), rl.end());
    return s;
  }

  // Same contents (kvcache.hpp:363-390): scheme kind, length, seen_upto, tokens and every buffer's shape and values.
  bool operator==(const KvStore& o) const {
    if (scheme_.kind != o.scheme_.kind || length() != o.length() || tokens_ != o.tokens_) return false;
    if (dims_.n_layers != o.dims_.n_layers || dims_.n_agents != o.dims_.n_agents) return false;
    for (idx a = 0; a < dims_.n_agents; ++a)
      if (seen(a) != o.seen(a)) return false;
    auto same = [](Span2D<const T> x, Span2D<const T> y) {
      if (x.rows != y.rows || x.cols != y.cols) return false;
      for (idx i = 0; i < x.rows; ++i)
        if (x.cols > 0 && !std::equal(x.row(i), x.row(i) + x.cols, y.row(i))) return false;
      return true;
    };
    const bool per_agent_kv = scheme_.kind == SchemeKind::NonShared, per_agent_lr = scheme_.kind == SchemeKind::BaseShared;
    for (idx l = 0; l < dims_.n_layers; ++l) {
      for (idx a = 0; a < (per_agent_kv ? dims_.n_agents : 1); ++a)
        if (!same(key_view(l, a), o.key_view(l, a)) || !same(value_view(l, a), o.value_view(l, a))) return false;
      for (idx a = 0; a < (per_agent_lr ? dims_.n_agents : 1); ++a)
        if (!same(lr_view(l, a), o.lr_view(l, a))) return false;
    }
    if (scheme_.kind == SchemeKind::SelectiveRecompute && !same(hidden_rows(0, hidden_size()), o.hidden_rows(0, o.hidden_size()))) return false;
    return true;
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

  void copy_from(const KvStore& o) {
    std::vector<std::pair<idx, idx>> order;                       // (seen_upto, agent), ascending
    for (idx a = 0; a < dims_.n_agents; ++a) order.emplace_back(o.seen(a), a);
    std::sort(order.begin(), order.end());
    std::size_t fed = 0;
    auto feed = [&](std::size_t upto) {
      if (upto > fed) append_tokens(std::vector<std::int32_t>(o.tokens_.begin() + static_cast<std::ptrdiff_t>(fed),
                                                              o.tokens_.begin() + static_cast<std::ptrdiff_t>(upto)));
      fed = std::max(fed, upto);
    };
    for (const auto& [upto, agent] : order) {
      if (upto == 0) continue;                                    // never marked
      feed(static_cast<std::size_t>(upto));
      mark_seen(agent);
    }
    feed(o.tokens_.size());
    const bool per_agent_kv = scheme_.kind == SchemeKind::NonShared, per_agent_lr = scheme_.kind == SchemeKind::BaseShared;
    const bool has_lr = per_agent_lr || scheme_.kind == SchemeKind::BaseLRShared;
    for (idx l = 0; l < dims_.n_layers; ++l) {
      for (idx a = 0; a < (per_agent_kv ? dims_.n_agents : 1); ++a) {
        append(LORAKV_KEY, l, a, 0, o.key_view(l, a));
        append(LORAKV_VALUE, l, a, 0, o.value_view(l, a));
      }
      if (has_lr)
        for (idx a = 0; a < (per_agent_lr ? dims_.n_agents : 1); ++a) append(LORAKV_LR, l, a, 0, o.lr_view(l, a));
    }
    if (scheme_.kind == SchemeKind::SelectiveRecompute) append(LORAKV_HIDDEN, 0, 0, 0, o.hidden_rows(0, o.hidden_size()));
  }

  static int pool_append(lorakv_pool* p, int which, idx layer, idx agent, idx row_begin, Span2D<const T> rows) {
    if constexpr (kDouble) return lorakv_pool_append_f64(p, which, layer, agent, row_begin, rows.data, rows.rows, rows.stride, LORAKV_HOST, nullptr);
    else return lorakv_pool_append(p, which, layer, agent, row_begin, rows.data, rows.rows, rows.stride, LORAKV_HOST, nullptr);
  }

  void append(int which, idx layer, idx agent, idx row_begin, Span2D<const T> rows) {
    const idx want = which == LORAKV_LR ? dims_.rank : which == LORAKV_HIDDEN ? dims_.d_model : dims_.d_kv;
    const bool has_buffer = which != LORAKV_LR || scheme_.kind == SchemeKind::BaseShared || scheme_.kind == SchemeKind::BaseLRShared;
    if (has_buffer && rows.cols != want) fail("GrowMat::append: column mismatch");
    b200::check(pool_append(pool_, which, layer, agent, row_begin, rows));
  }
  void overwrite(int which, idx layer, idx row_begin, Span2D<const T> rows) {
    if constexpr (kDouble) b200::check(lorakv_pool_overwrite_f64(pool_, which, layer, row_begin, rows.data, rows.rows, rows.stride, LORAKV_HOST));
    else b200::check(lorakv_pool_overwrite(pool_, which, layer, row_begin, rows.data, rows.rows, rows.stride, LORAKV_HOST));
    views_.erase(std::make_tuple(which, layer, idx(0)));     // cached rows of this buffer are stale
  }

  // A view de-paginates into a host buffer the store keeps.  Buffers are append-only (overwrite drops the copy), so a view
  // fetches only the rows that arrived since the last one: polling views costs the new rows, not the whole cache.
  Span2D<const T> view(int which, idx layer, idx agent) const {
    std::int64_t n = 0;
    b200::check(lorakv_pool_rows(pool_, which, layer, agent, &n));
    const bool lr_less = which == LORAKV_LR && scheme_.kind != SchemeKind::BaseShared && scheme_.kind != SchemeKind::BaseLRShared;
    if (lr_less) return Span2D<const T>{nullptr, n, 0, 0};
    const idx local_heads = opt_.n_kv_local > 0 ? opt_.n_kv_local : opt_.n_kv_heads - opt_.kv_head_begin;
    const idx cols = which == LORAKV_LR ? dims_.rank : which == LORAKV_HIDDEN ? dims_.d_model : local_heads * (dims_.d_kv / opt_.n_kv_heads);
    const bool per_agent = (which != LORAKV_LR && scheme_.kind == SchemeKind::NonShared) || (which == LORAKV_LR && scheme_.kind == SchemeKind::BaseShared);
    HostRows& h = views_[std::make_tuple(which, layer, per_agent ? agent : idx(0))];
    if (h.rows > n) h.rows = 0;
    h.data.resize(static_cast<std::size_t>(n * cols));
    if (n > h.rows && cols > 0) {
      T* dst = h.data.data() + h.rows * cols;
      if constexpr (kDouble) b200::check(lorakv_pool_read_f64(pool_, which, layer, agent, h.rows, n - h.rows, dst));
      else b200::check(lorakv_pool_read(pool_, which, layer, agent, h.rows, n - h.rows, dst));
    }
    h.rows = n;
    return Span2D<const T>{h.data.data(), n, cols, cols};
  }

  struct HostRows { std::vector<T> data; idx rows = 0; };

  CacheScheme scheme_;
  StoreDims dims_;
  DeviceOptions opt_;
  lorakv_pool* pool_ = nullptr;
  std::vector<std::int32_t> tokens_;
  mutable std::map<std::tuple<int, idx, idx>, HostRows> views_;
};

template <class T>
inline PrefillPlan plan_step(const KvStore<T>& store, idx agent, idx new_tokens) {
  return plan_core(store.scheme(), store.length(), store.seen(agent), new_tokens);
}

}  // namespace lorakv
