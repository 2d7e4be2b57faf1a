/*
 * lorakv_oracle.c -- CPU restatement of the reference's Flash-LoRA-Attention path.
 * TEST INFRASTRUCTURE ONLY (see lorakv_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, as the reference pins in proj/CMakeLists.txt:12-14).
 *
 * Parity: pinned against oracle/_ref (reference headers compiled here) and the
 * fixtures in tests/golden/ -- see tests/test_oracle_golden.py, tests/test_oracle_vs_ref.py.
 */
#define _GNU_SOURCE
#include "lorakv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- errors: the reference throws std::runtime_error (matrix.hpp:17-19); here a status
 * code plus a thread-local message carrying the same text ---------------------------- */
static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int orc_fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return ORC_ERR;
}

/* ---- rng.hpp ------------------------------------------------------------------------ */
typedef struct { uint64_t seed, state; } orc_rng;

static const uint64_t kGolden = 0x9e3779b97f4a7c15ull;

static uint64_t finalize64(uint64_t z) { /* shared tail of next_u64 / mix, rng.hpp:17-19,45-47 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t orc_rng_next(orc_rng* g) { /* rng.hpp:14-20 */
  g->state += kGolden;
  return finalize64(g->state);
}

static double orc_rng_gaussian(orc_rng* g) { /* rng.hpp:23-35: Box-Muller, u1 in (0,1], u2 in [0,1) */
  const double u1 = (double)((orc_rng_next(g) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(orc_rng_next(g) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

uint64_t orc_rng_mix(uint64_t a, uint64_t b) { /* rng.hpp:41-48 */
  uint64_t z = a ^ (b + kGolden + (a << 6) + (a >> 2));
  z += kGolden;
  return finalize64(z);
}

uint64_t orc_rng_child_seed(uint64_t seed, uint64_t key) { return orc_rng_mix(seed, key); }

void orc_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  orc_rng g = {seed, seed};
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_next(&g);
}

/* ---- attention.hpp:35-41 --------------------------------------------------------------- */
void orc_lr_mac_counts(int64_t total_len, int64_t cur_len, int64_t rank, int64_t d_head,
                       uint64_t* no_reorder, uint64_t* reorder) {
  const uint64_t L = (uint64_t)total_len, Lc = (uint64_t)cur_len, r = (uint64_t)rank,
                 d = (uint64_t)d_head;
  *no_reorder = L * r * d + Lc * L * d;
  *reorder = Lc * L * r + Lc * r * d;
}

/* ---- typed kernels ------------------------------------------------------------------- */
#define REAL float
#define SPAN orc_span_f32
#define FN(name) name##_f32
#define R_EXP expf
#define R_SQRT sqrtf
#define R_NEG_INF (-INFINITY)
#include "fla_oracle_impl.inc"
#undef REAL
#undef SPAN
#undef FN
#undef R_EXP
#undef R_SQRT
#undef R_NEG_INF

#define REAL double
#define SPAN orc_span_f64
#define FN(name) name##_f64
#define R_EXP exp
#define R_SQRT sqrt
#define R_NEG_INF (-(double)INFINITY)
#include "fla_oracle_impl.inc"
#undef REAL
#undef SPAN
#undef FN
#undef R_EXP
#undef R_SQRT
#undef R_NEG_INF

/* ---- multi-threaded head loop for the CPU baseline ------------------------------------ */
typedef struct {
  orc_span_f32 q, k, v_base, v_lr, b_up;
  float lr_scale;
  int64_t query_offset, group, d_head, b_r, b_c, n_q;
  float* out;
  int64_t next;          /* shared head counter */
  int failed;
  char err[512];
  pthread_mutex_t mu;
} mt_job;

static void* mt_worker(void* arg) {
  mt_job* job = (mt_job*)arg;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    const int64_t h = job->next++;
    pthread_mutex_unlock(&job->mu);
    if (h >= job->n_q) break;
    if (gqa_head_f32(job->q, job->k, job->v_base, job->v_lr, job->b_up, job->lr_scale,
                     job->query_offset, h, job->group, job->d_head, job->b_r, job->b_c, job->out,
                     NULL)) {
      pthread_mutex_lock(&job->mu);
      job->failed = 1;
      snprintf(job->err, sizeof job->err, "%s", g_err);
      pthread_mutex_unlock(&job->mu);
    }
  }
  return NULL;
}

int orc_gqa_attention_f32_mt(orc_span_f32 q, orc_span_f32 k, orc_span_f32 v_base,
                             orc_span_f32 v_lr, orc_span_f32 b_up, float lr_scale,
                             int64_t query_offset, int64_t n_q, int64_t n_kv, int64_t b_r,
                             int64_t b_c, float* out, int threads) {
  if (gqa_check_f32(q, k, v_base, n_q, n_kv)) return ORC_ERR;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  mt_job job;
  memset(&job, 0, sizeof job);
  job.q = q; job.k = k; job.v_base = v_base; job.v_lr = v_lr; job.b_up = b_up;
  job.lr_scale = lr_scale; job.query_offset = query_offset;
  job.d_head = q.cols / n_q; job.group = n_q / n_kv; job.b_r = b_r; job.b_c = b_c;
  job.n_q = n_q; job.out = out;
  pthread_mutex_init(&job.mu, NULL);
  pthread_t tid[256];
  int started = 0;
  for (int t = 0; t < threads; ++t)
    if (pthread_create(&tid[started], NULL, mt_worker, &job) == 0) ++started;
  if (started == 0) mt_worker(&job);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  pthread_mutex_destroy(&job.mu);
  if (job.failed) return orc_fail("%s", job.err);
  return ORC_OK;
}

/* ---- kvcache.hpp:112-142 -------------------------------------------------------------- */
int orc_plan_core(int scheme, int64_t first_recompute, int64_t length, int64_t seen,
                  int64_t new_tokens, int64_t out[9]) {
  if (new_tokens < 0) return orc_fail("plan_core: new_tokens must be >= 0");
  if (seen < 0 || seen > length) return orc_fail("plan_core: seen out of range");
  const int64_t total = length + new_tokens;
  const int64_t fresh[2] = {length, total}, unseen[2] = {seen, total};
  const int64_t *hidden = fresh, *kv = fresh, *lr = fresh;
  int64_t recompute[2] = {0, 0}, skip = 0;
  switch (scheme) {
    case ORC_NONSHARED: hidden = kv = lr = unseen; break;
    case ORC_FULLSHARED: break;
    case ORC_BASESHARED: hidden = lr = unseen; break;
    case ORC_BASELRSHARED: break;
    case ORC_SELECTIVE:
      hidden = unseen;
      recompute[0] = unseen[0]; recompute[1] = unseen[1];
      skip = first_recompute;
      break;
    default: return orc_fail("plan_core: unknown scheme %d", scheme);
  }
  out[0] = hidden[0]; out[1] = hidden[1];
  out[2] = kv[0]; out[3] = kv[1];
  out[4] = lr[0]; out[5] = lr[1];
  out[6] = recompute[0]; out[7] = recompute[1];
  out[8] = skip;
  return ORC_OK;
}

/* ---- kvcache.hpp:400-407 -------------------------------------------------------------- */
int orc_append_fww(int64_t rows, int64_t row_begin, int64_t n_src, int64_t* skip,
                   int64_t* appended) {
  if (row_begin > rows) return orc_fail("append leaves a gap at row %lld", (long long)rows);
  const int64_t present = rows - row_begin;
  if (present >= n_src) { *skip = n_src; *appended = 0; return ORC_OK; }
  *skip = present;
  *appended = n_src - present;
  return ORC_OK;
}

/* ---- KvStore, kvcache.hpp:161-420 ------------------------------------------------------- */
typedef struct { int64_t cols, rows; uint64_t elements; size_t cap; char* data; } growmat;

struct orc_store {
  int scheme, elem;
  int64_t n_layers, d_kv, d_model, rank, n_agents, length;
  int64_t* seen;
  growmat *key, *value, *shared_lr;          /* [n_layers] or NULL */
  growmat *agent_key, *agent_value, *agent_lr; /* [n_agents * n_layers] or NULL */
};

static growmat* mats_new(int64_t n, int64_t cols) {
  growmat* m = (growmat*)calloc((size_t)n, sizeof(growmat));
  if (m) for (int64_t i = 0; i < n; ++i) m[i].cols = cols;
  return m;
}
static void mats_free(growmat* m, int64_t n) {
  if (!m) return;
  for (int64_t i = 0; i < n; ++i) free(m[i].data);
  free(m);
}

orc_store* orc_store_create(int scheme, int64_t n_layers, int64_t d_kv, int64_t d_model,
                            int64_t rank, int64_t n_agents, int elem_size) {
  if (n_layers < 1 || d_kv < 1 || d_model < 1 || n_agents < 1) { orc_fail("KvStore: invalid dims"); return NULL; }
  if (rank < 0) { orc_fail("KvStore: negative rank"); return NULL; }
  if (scheme < ORC_NONSHARED || scheme > ORC_BASELRSHARED) {
    orc_fail("KvStore: scheme %d is outside the oracle's scope", scheme); /* SelectiveRecompute: out of scope */
    return NULL;
  }
  if (elem_size != 4 && elem_size != 8) { orc_fail("KvStore: elem_size must be 4 or 8"); return NULL; }
  orc_store* s = (orc_store*)calloc(1, sizeof *s);
  if (!s) return NULL;
  s->scheme = scheme; s->elem = elem_size;
  s->n_layers = n_layers; s->d_kv = d_kv; s->d_model = d_model; s->rank = rank; s->n_agents = n_agents;
  s->seen = (int64_t*)calloc((size_t)n_agents, sizeof(int64_t));
  if (scheme == ORC_NONSHARED) {              /* :226-233 */
    s->agent_key = mats_new(n_agents * n_layers, d_kv);
    s->agent_value = mats_new(n_agents * n_layers, d_kv);
  } else {                                    /* :234-237 */
    s->key = mats_new(n_layers, d_kv);
    s->value = mats_new(n_layers, d_kv);
  }
  if (scheme == ORC_BASESHARED) s->agent_lr = mats_new(n_agents * n_layers, rank);   /* :238-242 */
  if (scheme == ORC_BASELRSHARED) s->shared_lr = mats_new(n_layers, rank);           /* :243-244 */
  return s;
}

void orc_store_destroy(orc_store* s) {
  if (!s) return;
  mats_free(s->key, s->n_layers); mats_free(s->value, s->n_layers); mats_free(s->shared_lr, s->n_layers);
  mats_free(s->agent_key, s->n_agents * s->n_layers);
  mats_free(s->agent_value, s->n_agents * s->n_layers);
  mats_free(s->agent_lr, s->n_agents * s->n_layers);
  free(s->seen);
  free(s);
}

int orc_store_append_tokens(orc_store* s, int64_t n) {
  if (n < 0) return orc_fail("append_tokens: negative count");
  s->length += n;
  return ORC_OK;
}
int64_t orc_store_length(const orc_store* s) { return s->length; }

static int check_agent(const orc_store* s, int64_t agent) {
  if (agent < 0 || agent >= s->n_agents) return orc_fail("unknown agent %lld", (long long)agent);
  return ORC_OK;
}
static int check_layer(const orc_store* s, int64_t layer) {
  if (layer < 0 || layer >= s->n_layers) return orc_fail("layer %lld out of range", (long long)layer);
  return ORC_OK;
}

int orc_store_seen(const orc_store* s, int64_t agent, int64_t* out) {
  if (check_agent(s, agent)) return ORC_ERR;
  *out = s->seen[agent];
  return ORC_OK;
}
int orc_store_mark_seen(orc_store* s, int64_t agent) {
  if (check_agent(s, agent)) return ORC_ERR;
  if (s->length < s->seen[agent]) return orc_fail("KvStore: seen_upto may not decrease");
  s->seen[agent] = s->length;
  return ORC_OK;
}

static const char* kWhat[3] = {"key", "value", "lr"};
static const char* kScheme[5] = {"NonShared", "FullShared", "BaseShared", "BaseLRShared",
                                 "SelectiveRecompute"};

/* resolve (which, layer, agent) to a buffer the way append_* / *_view do (:268-288, :307-324);
 * *none is set when the scheme keeps no LR cache */
static int resolve(const orc_store* s, int which, int64_t layer, int64_t agent, growmat** m,
                   int* none) {
  *none = 0; *m = NULL;
  if (which < 0 || which > 2) return orc_fail("bad cache selector %d", which);
  if (which < 2) {
    if (s->scheme == ORC_NONSHARED) {
      if (check_agent(s, agent) || check_layer(s, layer)) return ORC_ERR;
      *m = (which == 0 ? s->agent_key : s->agent_value) + agent * s->n_layers + layer;
    } else {
      if (check_layer(s, layer)) return ORC_ERR;
      *m = (which == 0 ? s->key : s->value) + layer;
    }
    return ORC_OK;
  }
  if (s->scheme == ORC_BASESHARED) {
    if (check_agent(s, agent) || check_layer(s, layer)) return ORC_ERR;
    *m = s->agent_lr + agent * s->n_layers + layer;
  } else if (s->scheme == ORC_BASELRSHARED) {
    if (check_layer(s, layer)) return ORC_ERR;
    *m = s->shared_lr + layer;
  } else {
    *none = 1;
  }
  return ORC_OK;
}

int orc_store_append(orc_store* s, int which, int64_t layer, int64_t agent, int64_t row_begin,
                     const void* rows, int64_t n, int64_t stride) {
  growmat* m; int none;
  if (resolve(s, which, layer, agent, &m, &none)) return ORC_ERR;
  if (none) return orc_fail("KvStore: scheme %s has no LR cache", kScheme[s->scheme]);
  int64_t skip, add;
  if (orc_append_fww(m->rows, row_begin, n, &skip, &add)) {
    char tail[400];
    snprintf(tail, sizeof tail, "%.399s", g_err);
    return orc_fail("KvStore: %s %s", kWhat[which], tail);
  }
  if (add == 0) return ORC_OK;
  if (m->cols == 0) { m->rows += add; return ORC_OK; }   /* GrowMat::append :173-176 */
  const size_t row_bytes = (size_t)m->cols * (size_t)s->elem;
  const size_t need = ((size_t)m->rows + (size_t)add) * row_bytes;
  if (need > m->cap) {
    size_t cap = m->cap ? m->cap : 1024;
    while (cap < need) cap *= 2;
    char* nd = (char*)realloc(m->data, cap);
    if (!nd) return orc_fail("oracle: out of memory");
    m->data = nd; m->cap = cap;
  }
  for (int64_t i = 0; i < add; ++i)
    memcpy(m->data + ((size_t)m->rows + (size_t)i) * row_bytes,
           (const char*)rows + (size_t)(skip + i) * (size_t)stride * (size_t)s->elem, row_bytes);
  m->rows += add;
  m->elements += (uint64_t)add * (uint64_t)m->cols;
  return ORC_OK;
}

int orc_store_view(const orc_store* s, int which, int64_t layer, int64_t agent, const void** data,
                   int64_t* rows, int64_t* cols) {
  growmat* m; int none;
  if (resolve(s, which, layer, agent, &m, &none)) return ORC_ERR;
  if (none) {                       /* lr_view on a scheme without LR: L x 0 (:323) */
    growmat* km;
    if (resolve(s, 0, layer, agent, &km, &none)) return ORC_ERR;
    *data = NULL; *rows = km->rows; *cols = 0;
    return ORC_OK;
  }
  *data = m->data; *rows = m->rows; *cols = m->cols;
  return ORC_OK;
}

static uint64_t sum_elements(const growmat* m, int64_t n) {
  uint64_t t = 0;
  if (m) for (int64_t i = 0; i < n; ++i) t += m[i].elements;
  return t;
}

void orc_store_bytes(const orc_store* s, uint64_t out[4]) {
  const uint64_t sz = (uint64_t)s->elem;
  const int64_t per = s->n_agents * s->n_layers;
  out[0] = (sum_elements(s->key, s->n_layers) + sum_elements(s->agent_key, per)) * sz;
  out[1] = (sum_elements(s->value, s->n_layers) + sum_elements(s->agent_value, per)) * sz;
  out[2] = (sum_elements(s->shared_lr, s->n_layers) + sum_elements(s->agent_lr, per)) * sz;
  out[3] = 0;                       /* hidden-state cache: SelectiveRecompute only, out of scope */
}

uint64_t orc_store_allocated_elements(const orc_store* s) {
  const int64_t per = s->n_agents * s->n_layers;
  return sum_elements(s->key, s->n_layers) + sum_elements(s->value, s->n_layers) +
         sum_elements(s->shared_lr, s->n_layers) + sum_elements(s->agent_key, per) +
         sum_elements(s->agent_value, per) + sum_elements(s->agent_lr, per);
}

/* ---- page model ----------------------------------------------------------------------- */
void orc_page_of(int64_t row, int64_t page_tokens, int64_t* logical_page, int64_t* row_in_page) {
  *logical_page = row / page_tokens;
  *row_in_page = row % page_tokens;
}

/* ---- bf16 ------------------------------------------------------------------------------ */
float orc_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {      /* inf / nan: keep, quieting nan */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);           /* round to nearest even */
    u &= 0xffff0000u;
  }
  float y;
  memcpy(&y, &u, 4);
  return y;
}
void orc_round_bf16_array(const float* in, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_round_bf16(in[i]);
}

/* ---- engine.hpp:225-243  apply_rope: half-dim rotation per head; row i carries position pos_begin + i.
 * freq = 10000^(-2c/d_head) in double, cos / sin in double, cast to T, then x0*c - x1*s and x0*s + x1*c in T
 * (no FMA: the reference build pins -ffp-contract=off). ------------------------------------------------ */
#define ORC_ROPE(SUF, T)                                                                                   \
  int orc_apply_rope_##SUF(T* m, int64_t rows, int64_t stride, int64_t n_heads, int64_t d_head,            \
                           int64_t pos_begin) {                                                            \
    if (!m || rows < 0 || n_heads < 0 || d_head < 0 || stride < n_heads * d_head)                          \
      return orc_fail("apply_rope: bad arguments");                                                        \
    const int64_t half = d_head / 2;                                                                       \
    for (int64_t i = 0; i < rows; ++i) {                                                                   \
      const double pos = (double)(pos_begin + i);                                                          \
      for (int64_t h = 0; h < n_heads; ++h) {                                                              \
        T* base = m + i * stride + h * d_head;                                                             \
        for (int64_t c = 0; c < half; ++c) {                                                               \
          const double freq = pow(10000.0, -2.0 * (double)c / (double)d_head);                             \
          const T cos_t = (T)cos(pos * freq);                                                              \
          const T sin_t = (T)sin(pos * freq);                                                              \
          const T x0 = base[c], x1 = base[c + half];                                                       \
          base[c] = x0 * cos_t - x1 * sin_t;                                                               \
          base[c + half] = x0 * sin_t + x1 * cos_t;                                                        \
        }                                                                                                  \
      }                                                                                                    \
    }                                                                                                      \
    return ORC_OK;                                                                                         \
  }
ORC_ROPE(f32, float)
ORC_ROPE(f64, double)
