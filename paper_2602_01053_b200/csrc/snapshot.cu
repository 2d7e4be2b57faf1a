// snapshot.cu -- the reference's cache snapshot container (proj/include/lorakv/kvcache.hpp:438-546,
// "lorakv-cache-snapshot" version 1) written from / read into the paged HBM pool, so that the
// reference's tools read GPU state and a GPU pool resumes from a reference dump.
//
// File = u64 header length | JSON header | tensors.  The header is what nlohmann::json::dump() emits for the
// reference's object (std::map order = keys sorted, no whitespace), so a pool holding the same state produces the
// reference's file byte for byte.  Tensors are dense row-major float32 in the order of SnapshotAccess::collect
// (:523-544); pages are de-paginated on save and re-paginated on load (bf16 pools hold every value a float32
// snapshot of a bf16 pool contains, so save -> load -> save is the identity).  Host code only.
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "state.hpp"

namespace lk {

namespace {

const char* kSchemeName[5] = {"NonShared", "FullShared", "BaseShared", "BaseLRShared", "SelectiveRecompute"};

struct TensorRef { std::string name; int which; int64_t layer, agent, cols; };

// SnapshotAccess::collect (kvcache.hpp:523-544)
std::vector<TensorRef> collect(int scheme, int64_t n_layers, int64_t n_agents, int64_t d_kv, int64_t rank, int64_t d_model) {
  std::vector<TensorRef> out;
  for (int64_t l = 0; l < n_layers; ++l) {
    const std::string tag = "layer" + std::to_string(l);
    if (scheme != LORAKV_NONSHARED) {
      out.push_back({tag + ".key", LORAKV_KEY, l, 0, d_kv});
      out.push_back({tag + ".value", LORAKV_VALUE, l, 0, d_kv});
    } else {
      for (int64_t a = 0; a < n_agents; ++a) {
        out.push_back({tag + ".key.agent" + std::to_string(a), LORAKV_KEY, l, a, d_kv});
        out.push_back({tag + ".value.agent" + std::to_string(a), LORAKV_VALUE, l, a, d_kv});
      }
    }
    if (scheme == LORAKV_BASESHARED)
      for (int64_t a = 0; a < n_agents; ++a) out.push_back({tag + ".lr.agent" + std::to_string(a), LORAKV_LR, l, a, rank});
    if (scheme == LORAKV_BASELRSHARED) out.push_back({tag + ".lr", LORAKV_LR, l, 0, rank});
  }
  if (scheme == LORAKV_SELECTIVE) out.push_back({"hidden", LORAKV_HIDDEN, 0, 0, d_model});
  return out;
}

template <class V>
std::string int_array(const V& v, size_t n) {
  std::string s = "[";
  for (size_t i = 0; i < n; ++i) { if (i) s += ','; s += std::to_string((long long)v[i]); }
  return s + "]";
}

// ---- a reader for the header's JSON subset: objects, arrays, strings without escapes worth keeping, integers ----
struct Json {
  enum Kind { Null, Int, Str, Arr, Obj } kind = Null;
  long long i = 0;
  std::string s;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const char* key) const {
    for (const auto& kv : obj) if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const std::string& t;
  size_t p = 0;
  bool ok = true;
  explicit Parser(const std::string& text) : t(text) {}
  void ws() { while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\t' || t[p] == '\r')) ++p; }
  bool eat(char c) { ws(); if (p < t.size() && t[p] == c) { ++p; return true; } return false; }
  std::string str() {
    std::string out;
    if (!eat('"')) { ok = false; return out; }
    while (p < t.size() && t[p] != '"') {
      if (t[p] == '\\' && p + 1 < t.size()) { ++p; }
      out += t[p++];
    }
    if (p >= t.size()) ok = false; else ++p;
    return out;
  }
  Json value() {
    Json j;
    ws();
    if (p >= t.size()) { ok = false; return j; }
    const char c = t[p];
    if (c == '{') {
      ++p; j.kind = Json::Obj;
      if (eat('}')) return j;
      do { std::string k = str(); if (!eat(':')) ok = false; j.obj.emplace_back(std::move(k), value()); } while (ok && eat(','));
      if (!eat('}')) ok = false;
    } else if (c == '[') {
      ++p; j.kind = Json::Arr;
      if (eat(']')) return j;
      do { j.arr.push_back(value()); } while (ok && eat(','));
      if (!eat(']')) ok = false;
    } else if (c == '"') {
      j.kind = Json::Str; j.s = str();
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      size_t q = p; if (t[q] == '-') ++q;
      while (q < t.size() && t[q] >= '0' && t[q] <= '9') ++q;
      j.kind = Json::Int;
      if (q - p > 18 || q == p + (t[p] == '-' ? 1u : 0u)) { ok = false; return j; }   // fits int64 without overflow; at least one digit
      j.i = std::stoll(t.substr(p, q - p)); p = q;
    } else {
      ok = false;
    }
    return j;
  }
};

int need_int(const Json& h, const char* key, int64_t* out, const char* path) {
  const Json* v = h.get(key);
  if (!v || v->kind != Json::Int) return fail("snapshot header has no integer '%s': %s", key, path);
  *out = v->i;
  return LORAKV_OK;
}

}  // namespace
}  // namespace lk

using namespace lk;

extern "C" {

int lorakv_pool_save_snapshot(const lorakv_pool* pool, const char* path, const int32_t* tokens, int64_t n_tokens) {
  if (!pool || !path) return fail("null argument");
  if (n_tokens < 0 || (n_tokens > 0 && !tokens)) return fail("save_snapshot: bad token list");
  if (pool->n_kv_local != pool->dims.n_kv_heads)
    return fail("save_snapshot: a kv-head shard holds %lld of %lld heads; snapshots are written from an unsharded pool",
                (long long)pool->n_kv_local, (long long)pool->dims.n_kv_heads);
  const lorakv_pool_dims& d = pool->dims;
  const int64_t d_kv = d.n_kv_heads * d.d_head;
  const std::vector<TensorRef> tensors = collect(d.scheme, d.n_layers, d.n_agents, d_kv, d.rank, d.d_model);
  const bool f64 = d.dtype == LORAKV_F64;      // KvStore<double>: dtype "f64", float64 payloads (detail::dtype_name, kvcache.hpp:431-435)
  std::vector<int64_t> rows(tensors.size());
  for (size_t i = 0; i < tensors.size(); ++i)
    LK_TRY(lorakv_pool_rows(pool, tensors[i].which, tensors[i].layer, tensors[i].agent, &rows[i]));
  // nlohmann::json::dump(): std::map order (keys sorted), no whitespace
  std::string h = "{";
  h += "\"d_kv\":" + std::to_string((long long)d_kv);
  h += ",\"d_model\":" + std::to_string((long long)d.d_model);
  h += std::string(",\"dtype\":\"") + (f64 ? "f64" : "f32") + "\",\"format\":\"lorakv-cache-snapshot\"";
  h += ",\"length\":" + std::to_string((long long)pool->length);
  h += ",\"n_agents\":" + std::to_string((long long)d.n_agents);
  h += ",\"n_layers\":" + std::to_string((long long)d.n_layers);
  h += ",\"rank\":" + std::to_string((long long)d.rank);
  h += ",\"recompute_layers\":" + int_array(pool->recompute_layers, pool->recompute_layers.size()) + ",\"scheme\":\"" +
       std::string(kSchemeName[d.scheme]) + "\"";
  h += ",\"seen_upto\":" + int_array(pool->seen, pool->seen.size());
  h += ",\"tensors\":[";
  for (size_t i = 0; i < tensors.size(); ++i) {
    if (i) h += ',';
    h += "{\"cols\":" + std::to_string((long long)tensors[i].cols) + ",\"name\":\"" + tensors[i].name + "\",\"rows\":" +
         std::to_string((long long)rows[i]) + "}";
  }
  h += "],\"tokens\":" + int_array(tokens, (size_t)n_tokens) + ",\"version\":1}";

  std::ofstream out(path, std::ios::binary);
  if (!out) return fail("cannot open snapshot file for writing: %s", path);
  const uint64_t hlen = h.size();
  out.write(reinterpret_cast<const char*>(&hlen), sizeof hlen);
  out.write(h.data(), (std::streamsize)h.size());
  std::vector<float> buf;
  std::vector<double> buf64;
  for (size_t i = 0; i < tensors.size(); ++i) {
    const size_t n = (size_t)(rows[i] * tensors[i].cols);
    if (n == 0) continue;
    if (f64) {
      buf64.resize(n);
      LK_TRY(lorakv_pool_read_f64(pool, tensors[i].which, tensors[i].layer, tensors[i].agent, 0, rows[i], buf64.data()));
      out.write(reinterpret_cast<const char*>(buf64.data()), (std::streamsize)(n * sizeof(double)));
    } else {
      buf.resize(n);
      LK_TRY(lorakv_pool_read(pool, tensors[i].which, tensors[i].layer, tensors[i].agent, 0, rows[i], buf.data()));
      out.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(n * sizeof(float)));
    }
  }
  if (!out) return fail("snapshot write failed: %s", path);
  return LORAKV_OK;
}

}  // extern "C"

// header of a snapshot file: length-prefixed JSON; the length is checked against the file size before anything is allocated
static int read_header(std::ifstream& in, const char* path, Json* header) {
  if (!in) return fail("cannot open snapshot file: %s", path);
  in.seekg(0, std::ios::end);
  const std::streamoff file_size = in.tellg();
  in.seekg(0, std::ios::beg);
  uint64_t hlen = 0;
  in.read(reinterpret_cast<char*>(&hlen), sizeof hlen);
  if (!in || file_size < (std::streamoff)sizeof hlen || hlen > (uint64_t)(file_size - (std::streamoff)sizeof hlen))
    return fail("snapshot header truncated: %s", path);
  std::string hs((size_t)hlen, '\0');
  in.read(&hs[0], (std::streamsize)hlen);
  if (!in) return fail("snapshot header truncated: %s", path);
  Parser ps(hs);
  *header = ps.value();
  if (!ps.ok || header->kind != Json::Obj) return fail("snapshot header is not valid JSON: %s", path);
  return LORAKV_OK;
}

static int load_snapshot_impl(lorakv_ctx* ctx, const char* path, int dtype, int64_t n_kv_heads, int64_t page_tokens,
                              int64_t max_tokens, lorakv_pool** out_pool, int32_t* tokens_out, int64_t tokens_cap,
                              int64_t* n_tokens) {
  std::ifstream in(path, std::ios::binary);
  Json header;
  LK_TRY(read_header(in, path, &header));
  const Json* fmt = header.get("format");
  if (!fmt || fmt->s != "lorakv-cache-snapshot") return fail("not a cache snapshot: %s", path);
  const Json* dt = header.get("dtype");
  const bool f64 = dtype == LORAKV_F64;
  const char* want_dt = f64 ? "f64" : "f32";
  if (!dt || dt->s != want_dt) return fail("snapshot dtype %s does not match build dtype %s", dt ? dt->s.c_str() : "?", want_dt);
  const Json* sch = header.get("scheme");
  int scheme = -1;
  for (int k = 0; k < 5; ++k) if (sch && sch->s == kSchemeName[k]) scheme = k;
  if (scheme < 0) return fail("unknown cache scheme '%s'", sch ? sch->s.c_str() : "?");
  lorakv_pool_dims dims{};
  int64_t d_kv = 0, length = 0;
  LK_TRY(need_int(header, "n_layers", &dims.n_layers, path));
  LK_TRY(need_int(header, "d_kv", &d_kv, path));
  LK_TRY(need_int(header, "d_model", &dims.d_model, path));
  LK_TRY(need_int(header, "rank", &dims.rank, path));
  LK_TRY(need_int(header, "n_agents", &dims.n_agents, path));
  LK_TRY(need_int(header, "length", &length, path));
  if (dims.n_layers < 1 || dims.n_layers > 4096 || d_kv < 1 || dims.d_model < 1 || dims.rank < 0 || dims.n_agents < 1 ||
      dims.n_agents > 65536 || length < 0 || length > ((int64_t)1 << 40))
    return fail("snapshot header holds implausible dimensions: %s", path);
  if (n_kv_heads < 1 || d_kv % n_kv_heads != 0)
    return fail("load_snapshot: d_kv %lld is not divisible by n_kv_heads %lld", (long long)d_kv, (long long)n_kv_heads);
  dims.scheme = scheme; dims.dtype = dtype; dims.n_kv_heads = n_kv_heads; dims.d_head = d_kv / n_kv_heads;
  dims.page_tokens = page_tokens; dims.max_tokens = std::max<int64_t>(max_tokens, std::max<int64_t>(length, 1));
  const Json* seen = header.get("seen_upto");
  const Json* toks = header.get("tokens");
  const Json* tj = header.get("tensors");
  if (!seen || seen->kind != Json::Arr || !toks || toks->kind != Json::Arr || !tj || tj->kind != Json::Arr)
    return fail("snapshot header truncated: %s", path);
  lorakv_pool* pool = nullptr;
  LK_TRY(lorakv_pool_create(ctx, &dims, &pool));
  auto bail = [&](int rc) { lorakv_pool_destroy(pool); return rc; };
  if ((int64_t)seen->arr.size() != dims.n_agents) return bail(fail("snapshot seen_upto has %zu entries for %lld agents", seen->arr.size(), (long long)dims.n_agents));
  pool->length = length;
  for (size_t a = 0; a < seen->arr.size(); ++a) pool->seen[a] = seen->arr[a].i;
  if (const Json* rl = header.get("recompute_layers")) {
    std::vector<int64_t> layers;
    if (rl->kind == Json::Arr) for (const Json& x : rl->arr) layers.push_back(x.i);
    const int rc = lorakv_pool_set_recompute_layers(pool, layers.data(), (int64_t)layers.size());
    if (rc != LORAKV_OK) return bail(rc);
  }
  const std::vector<TensorRef> tensors = collect(scheme, dims.n_layers, dims.n_agents, d_kv, dims.rank, dims.d_model);
  if (tj->arr.size() != tensors.size()) return bail(fail("snapshot tensor list mismatch: %s", path));
  std::vector<float> buf;
  std::vector<double> buf64;
  for (size_t i = 0; i < tensors.size(); ++i) {
    const Json& meta = tj->arr[i];
    const Json *nm = meta.get("name"), *rj = meta.get("rows"), *cj = meta.get("cols");
    if (!nm || !rj || !cj || nm->s != tensors[i].name) return bail(fail("snapshot tensor order mismatch at %s", tensors[i].name.c_str()));
    if (cj->i != tensors[i].cols) return bail(fail("snapshot tensor width mismatch at %s", tensors[i].name.c_str()));
    const int64_t rows = rj->i;
    if (rows < 0 || rows > dims.max_tokens)
      return bail(fail("snapshot tensor %s claims %lld rows; the trajectory holds at most %lld", tensors[i].name.c_str(), (long long)rows,
                       (long long)dims.max_tokens));
    const size_t n = (size_t)(rows * tensors[i].cols);
    int64_t added = 0;
    int rc;
    if (f64) {
      buf64.resize(std::max<size_t>(n, 1));
      in.read(reinterpret_cast<char*>(buf64.data()), (std::streamsize)(n * sizeof(double)));
      if (!in) return bail(fail("snapshot payload truncated: %s", path));
      rc = lorakv_pool_append_f64(pool, tensors[i].which, tensors[i].layer, tensors[i].agent, 0, buf64.data(), rows, tensors[i].cols,
                                  LORAKV_HOST, &added);
    } else {
      buf.resize(std::max<size_t>(n, 1));
      in.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)(n * sizeof(float)));
      if (!in) return bail(fail("snapshot payload truncated: %s", path));
      rc = lorakv_pool_append(pool, tensors[i].which, tensors[i].layer, tensors[i].agent, 0, buf.data(), rows, tensors[i].cols,
                              LORAKV_HOST, &added);
    }
    if (rc != LORAKV_OK) return bail(rc);
  }
  if (n_tokens) *n_tokens = (int64_t)toks->arr.size();
  if (tokens_out)
    for (size_t i = 0; i < toks->arr.size() && (int64_t)i < tokens_cap; ++i) tokens_out[i] = (int32_t)toks->arr[i].i;
  *out_pool = pool;
  return LORAKV_OK;
}

extern "C" {

// No C++ exception may cross the C ABI: a malformed file (absurd sizes -> bad_alloc, ...) becomes a status + message.
int lorakv_pool_load_snapshot(lorakv_ctx* ctx, const char* path, int dtype, int64_t n_kv_heads, int64_t page_tokens,
                              int64_t max_tokens, lorakv_pool** out_pool, int32_t* tokens_out, int64_t tokens_cap,
                              int64_t* n_tokens) {
  if (!ctx || !path || !out_pool) return fail("null argument");
  *out_pool = nullptr;
  try {
    return load_snapshot_impl(ctx, path, dtype, n_kv_heads, page_tokens, max_tokens, out_pool, tokens_out, tokens_cap, n_tokens);
  } catch (const std::exception& e) {
    if (*out_pool) { lorakv_pool_destroy(*out_pool); *out_pool = nullptr; }
    return fail("load_snapshot: %s: %s", path, e.what());
  }
}

// Token ids of a snapshot without loading it (header only): writes min(cap, n) ids, *n_tokens = how many the file holds.
int lorakv_snapshot_tokens(const char* path, int32_t* tokens_out, int64_t cap, int64_t* n_tokens) {
  if (!path) return fail("null argument");
  try {
    std::ifstream in(path, std::ios::binary);
    Json header;
    LK_TRY(read_header(in, path, &header));
    const Json* toks = header.get("tokens");
    if (!toks || toks->kind != Json::Arr) return fail("snapshot header truncated: %s", path);
    if (n_tokens) *n_tokens = (int64_t)toks->arr.size();
    if (tokens_out)
      for (size_t i = 0; i < toks->arr.size() && (int64_t)i < cap; ++i) tokens_out[i] = (int32_t)toks->arr[i].i;
    return LORAKV_OK;
  } catch (const std::exception& e) {
    return fail("snapshot_tokens: %s: %s", path, e.what());
  }
}

}  // extern "C"
