/*
 * fedsim_oracle.c -- CPU restatement of the reference federated-round path.
 *
 * TEST INFRASTRUCTURE ONLY (see fedsim_oracle.h).  Plain C99, f64, strict
 * left-to-right loops, compiled with -O2 -ffp-contract=off (no FMA) so that
 * each result is bit-identical to the reference built from its own sources.
 * File:line citations are relative to /root/reference/proj/core.
 */
#include "fedsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------
 * rng.h:14-32  splitmix64 finalizer and seed mixing
 * ------------------------------------------------------------------------- */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t orc_mix_seed(uint64_t seed, uint64_t a) { return orc_mix64(seed ^ orc_mix64(a)); }
uint64_t orc_mix_seed2(uint64_t seed, uint64_t a, uint64_t b) {
  return orc_mix_seed(orc_mix_seed(seed, a), b);
}
uint64_t orc_mix_seed3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return orc_mix_seed(orc_mix_seed2(seed, a, b), c);
}

/* ---------------------------------------------------------------------------
 * rng.h:37-84  Rng = std::mt19937_64 + pinned conversions.  The engine is the
 * standard MT19937-64 (ISO C++ [rand.predef]); restated here.
 * ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
  double spare;
  int have_spare;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t rng_next(rng_t* r) {
  if (r->idx >= MT_N) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
      uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
      uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static uint64_t rng_uniform_u64(rng_t* r, uint64_t n) { return rng_next(r) % n; }

static double rng_normal(rng_t* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  do {
    u1 = rng_uniform(r);
  } while (u1 <= 0.0);
  const double u2 = rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

static void rng_shuffle_u32(rng_t* r, uint32_t* v, uint64_t n) {
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = rng_uniform_u64(r, i);
    uint32_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

void orc_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64_out, double* uniform_out,
                   double* normal_out) {
  rng_t r;
  if (u64_out) {
    rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) u64_out[i] = rng_next(&r);
  }
  if (uniform_out) {
    rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) uniform_out[i] = rng_uniform(&r);
  }
  if (normal_out) {
    rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) normal_out[i] = rng_normal(&r);
  }
}

/* ---------------------------------------------------------------------------
 * model.cpp:10-61  validation, parameter count and canonical layout
 * ------------------------------------------------------------------------- */
int orc_model_validate(const orc_model_cfg* c) {
  if (c->n_blocks == 0 || c->d_model == 0) return ORC_CONFIG;
  if (c->n_heads == 0 || c->d_model % c->n_heads != 0) return ORC_CONFIG;
  if (c->expansion_ratio == 0 || c->vocab_size < 2 || c->seq_len == 0) return ORC_CONFIG;
  return ORC_OK;
}

uint64_t orc_param_count(const orc_model_cfg* c) {
  const uint64_t d = c->d_model, e = c->expansion_ratio;
  const uint64_t per_block = (4 + 2 * e) * d * d + (9 + e) * d;
  return c->vocab_size * d + c->seq_len * d + c->n_blocks * per_block + 2 * d +
         d * c->vocab_size + c->vocab_size;
}

uint64_t orc_layout_size(const orc_model_cfg* c) { return 2 + 16 * c->n_blocks + 4; }

/* per-block entry table: suffix, rows/cols in units of (d, hidden) */
static const char* kBlockNames[16] = {"ln1.gain", "ln1.bias", "attn.wq", "attn.bq",
                                      "attn.wk",  "attn.bk",  "attn.wv", "attn.bv",
                                      "attn.wo",  "attn.bo",  "ln2.gain", "ln2.bias",
                                      "mlp.w1",   "mlp.b1",   "mlp.w2",  "mlp.b2"};

static void block_entry_shape(const orc_model_cfg* c, int j, uint64_t* rows, uint64_t* cols) {
  const uint64_t d = c->d_model, h = c->expansion_ratio * d;
  switch (j) {
    case 2: case 4: case 6: case 8: *rows = d; *cols = d; return;
    case 12: *rows = d; *cols = h; return;
    case 13: *rows = h; *cols = 0; return;
    case 14: *rows = h; *cols = d; return;
    default: *rows = d; *cols = 0; return;
  }
}

int orc_layout_entry(const orc_model_cfg* c, uint64_t i, uint64_t* offset, uint64_t* rows,
                     uint64_t* cols, char* name, int name_cap) {
  const uint64_t n = orc_layout_size(c);
  if (i >= n) return ORC_INDEX;
  uint64_t off = 0;
  for (uint64_t e = 0; e <= i; ++e) {
    uint64_t r = 0, cc = 0;
    char nm[64];
    if (e == 0) { r = c->vocab_size; cc = c->d_model; snprintf(nm, 64, "token_embedding"); }
    else if (e == 1) { r = c->seq_len; cc = c->d_model; snprintf(nm, 64, "position_embedding"); }
    else if (e < 2 + 16 * c->n_blocks) {
      const uint64_t b = (e - 2) / 16;
      const int j = (int)((e - 2) % 16);
      block_entry_shape(c, j, &r, &cc);
      snprintf(nm, 64, "block%llu.%s", (unsigned long long)b, kBlockNames[j]);
    } else {
      const uint64_t j = e - 2 - 16 * c->n_blocks;
      if (j == 0) { r = c->d_model; snprintf(nm, 64, "final_ln.gain"); }
      else if (j == 1) { r = c->d_model; snprintf(nm, 64, "final_ln.bias"); }
      else if (j == 2) { r = c->d_model; cc = c->vocab_size; snprintf(nm, 64, "head.w"); }
      else { r = c->vocab_size; snprintf(nm, 64, "head.b"); }
    }
    if (e == i) {
      *offset = off;
      *rows = r;
      *cols = cc;
      if (name && name_cap > 0) snprintf(name, (size_t)name_cap, "%s", nm);
      return ORC_OK;
    }
    off += cc ? r * cc : r;
  }
  return ORC_INDEX;
}

static int ends_with(const char* s, const char* suf) {
  const size_t a = strlen(s), b = strlen(suf);
  return a >= b && strcmp(s + a - b, suf) == 0;
}

/* model.cpp:72-96 */
int orc_init_params(const orc_model_cfg* c, uint64_t seed, double* out) {
  if (orc_model_validate(c)) return ORC_CONFIG;
  rng_t r;
  rng_init(&r, seed);
  const double base_std = 0.02;
  const double resid_std = base_std / sqrt(2.0 * (double)c->n_blocks);
  const uint64_t n = orc_layout_size(c);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t off, rows, cols;
    char name[64];
    orc_layout_entry(c, i, &off, &rows, &cols, name, 64);
    const uint64_t cnt = cols ? rows * cols : rows;
    double* v = out + off;
    if (ends_with(name, ".gain")) {
      for (uint64_t j = 0; j < cnt; ++j) v[j] = 1.0;
    } else if (ends_with(name, ".bias") || ends_with(name, ".bq") || ends_with(name, ".bk") ||
               ends_with(name, ".bv") || ends_with(name, ".bo") || ends_with(name, ".b1") ||
               ends_with(name, ".b2") || ends_with(name, ".b")) {
      for (uint64_t j = 0; j < cnt; ++j) v[j] = 0.0;
    } else {
      const double sd =
          (ends_with(name, "attn.wo") || ends_with(name, "mlp.w2")) ? resid_std : base_std;
      for (uint64_t j = 0; j < cnt; ++j) v[j] = rng_normal(&r) * sd;
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * data.cpp:24-71  synthetic corpora
 * ------------------------------------------------------------------------- */
static const uint32_t kStyleMult[4] = {1, 3, 5, 7};
static const uint32_t kStyleAdd[4] = {1, 1, 2, 3};

int orc_generate_corpus(int32_t style, uint64_t length, uint64_t seed, uint32_t vocab,
                        uint16_t* out) {
  if (style < 0 || style > 3) return ORC_CONFIG;
  if (vocab < 8 || vocab % 4 != 0) return ORC_CONFIG;
  if (length == 0) return ORC_CONFIG;
  const uint32_t band = vocab / 4;
  const uint32_t base = (uint32_t)style * band;
  rng_t r;
  rng_init(&r, orc_mix_seed2(seed, 0x436f7270ULL, (uint64_t)style));
  uint32_t cur = (uint32_t)rng_uniform_u64(&r, band);
  out[0] = (uint16_t)(base + cur);
  for (uint64_t i = 1; i < length; ++i) {
    if (rng_uniform(&r) < 0.8) {
      cur = (kStyleMult[style] * cur + kStyleAdd[style]) % band;
    } else {
      cur = (uint32_t)rng_uniform_u64(&r, band);
    }
    out[i] = (uint16_t)(base + cur);
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * data.cpp:137-199  shard plans
 * ------------------------------------------------------------------------- */
struct orc_plan {
  uint64_t seq_len;
  uint64_t n_sources;
  uint16_t** corpora;
  uint64_t* corpus_len;
  uint64_t n_clients;
  uint64_t* n_blocks;       /* per client */
  uint32_t** block_source;  /* per client */
  uint64_t** block_offset;  /* per client */
};

static orc_plan* plan_alloc(uint64_t n_sources, uint64_t n_clients, uint64_t seq_len) {
  orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
  p->seq_len = seq_len;
  p->n_sources = n_sources;
  p->corpora = (uint16_t**)calloc(n_sources, sizeof(uint16_t*));
  p->corpus_len = (uint64_t*)calloc(n_sources, sizeof(uint64_t));
  p->n_clients = n_clients;
  p->n_blocks = (uint64_t*)calloc(n_clients, sizeof(uint64_t));
  p->block_source = (uint32_t**)calloc(n_clients, sizeof(uint32_t*));
  p->block_offset = (uint64_t**)calloc(n_clients, sizeof(uint64_t*));
  return p;
}

void orc_plan_free(orc_plan* p) {
  if (!p) return;
  for (uint64_t s = 0; s < p->n_sources; ++s) free(p->corpora[s]);
  for (uint64_t c = 0; c < p->n_clients; ++c) {
    free(p->block_source[c]);
    free(p->block_offset[c]);
  }
  free(p->corpora);
  free(p->corpus_len);
  free(p->n_blocks);
  free(p->block_source);
  free(p->block_offset);
  free(p);
}

orc_plan* orc_plan_iid(const uint16_t* tokens, uint64_t n_tokens, uint64_t n_shards,
                       uint64_t seq_len, uint64_t seed, int* err) {
  *err = ORC_OK;
  if (n_shards == 0 || seq_len == 0) { *err = ORC_CONFIG; return NULL; }
  const uint64_t bl = seq_len + 1;
  const uint64_t n_blocks = n_tokens / bl;
  if (n_blocks < n_shards) { *err = ORC_CONFIG; return NULL; }
  uint32_t* order = (uint32_t*)malloc(n_blocks * sizeof(uint32_t));
  for (uint64_t i = 0; i < n_blocks; ++i) order[i] = (uint32_t)i;
  rng_t r;
  rng_init(&r, orc_mix_seed(seed, 0x53686172ULL));
  rng_shuffle_u32(&r, order, n_blocks);
  orc_plan* p = plan_alloc(1, n_shards, seq_len);
  p->corpora[0] = (uint16_t*)malloc(n_tokens * sizeof(uint16_t));
  memcpy(p->corpora[0], tokens, n_tokens * sizeof(uint16_t));
  p->corpus_len[0] = n_tokens;
  for (uint64_t c = 0; c < n_shards; ++c) {
    const uint64_t cnt = n_blocks / n_shards + (c < n_blocks % n_shards ? 1 : 0);
    p->block_source[c] = (uint32_t*)calloc(cnt ? cnt : 1, sizeof(uint32_t));
    p->block_offset[c] = (uint64_t*)calloc(cnt ? cnt : 1, sizeof(uint64_t));
  }
  for (uint64_t i = 0; i < n_blocks; ++i) {
    const uint64_t c = i % n_shards;
    p->block_offset[c][p->n_blocks[c]] = (uint64_t)order[i] * bl;
    p->n_blocks[c] += 1;
  }
  free(order);
  return p;
}

orc_plan* orc_plan_by_source(const uint16_t* const* corpora, const uint64_t* lens,
                             uint64_t n_sources, uint64_t cps, uint64_t seq_len, int* err) {
  *err = ORC_OK;
  if (n_sources == 0 || cps == 0 || seq_len == 0) { *err = ORC_CONFIG; return NULL; }
  const uint64_t bl = seq_len + 1;
  for (uint64_t s = 0; s < n_sources; ++s) {
    if ((lens[s] / bl) / cps == 0) { *err = ORC_CONFIG; return NULL; }
  }
  orc_plan* p = plan_alloc(n_sources, n_sources * cps, seq_len);
  for (uint64_t s = 0; s < n_sources; ++s) {
    p->corpora[s] = (uint16_t*)malloc(lens[s] * sizeof(uint16_t));
    memcpy(p->corpora[s], corpora[s], lens[s] * sizeof(uint16_t));
    p->corpus_len[s] = lens[s];
    const uint64_t per_client = (lens[s] / bl) / cps;
    for (uint64_t c = 0; c < cps; ++c) {
      const uint64_t id = s * cps + c;
      p->n_blocks[id] = per_client;
      p->block_source[id] = (uint32_t*)malloc(per_client * sizeof(uint32_t));
      p->block_offset[id] = (uint64_t*)malloc(per_client * sizeof(uint64_t));
      for (uint64_t b = 0; b < per_client; ++b) {
        p->block_source[id][b] = (uint32_t)s;
        p->block_offset[id][b] = (c * per_client + b) * bl;
      }
    }
  }
  return p;
}

uint64_t orc_plan_n_clients(const orc_plan* p) { return p->n_clients; }
uint64_t orc_plan_client_blocks(const orc_plan* p, uint64_t client) {
  return client < p->n_clients ? p->n_blocks[client] : 0;
}
void orc_plan_block(const orc_plan* p, uint64_t client, uint64_t b, uint32_t* source,
                    uint64_t* offset) {
  *source = p->block_source[client][b];
  *offset = p->block_offset[client][b];
}

/* data.cpp:201-203 */
uint64_t orc_stream_seed(uint64_t global_seed, uint64_t client) {
  return orc_mix_seed2(global_seed, 0x44617461ULL, client);
}

/* data.cpp:222-253  BatchStream::next; the epoch permutation is recomputed
 * functionally (it depends only on (seed, client, epoch)). */
int orc_stream_next(const orc_plan* p, uint64_t client, uint64_t batch, uint64_t seq_len,
                    uint64_t seed, uint64_t* cursor, int32_t* inputs, int32_t* targets) {
  if (client >= p->n_clients) return ORC_LOOKUP;
  if (batch == 0) return ORC_CONFIG;
  if (seq_len != p->seq_len) return ORC_USAGE;
  const uint64_t n = p->n_blocks[client];
  uint32_t* perm = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint64_t cached_epoch = ~0ULL;
  for (uint64_t r = 0; r < batch; ++r) {
    const uint64_t idx = *cursor + r;
    const uint64_t epoch = idx / n;
    if (epoch != cached_epoch) {
      for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
      rng_t rg;
      rng_init(&rg, orc_mix_seed3(seed, 0x45706f63ULL, client, epoch));
      rng_shuffle_u32(&rg, perm, n);
      cached_epoch = epoch;
    }
    const uint64_t bi = perm[idx % n];
    const uint16_t* tok = p->corpora[p->block_source[client][bi]];
    const uint64_t off = p->block_offset[client][bi];
    for (uint64_t t = 0; t < seq_len; ++t) {
      inputs[r * seq_len + t] = (int32_t)tok[off + t];
      targets[r * seq_len + t] = (int32_t)tok[off + t + 1];
    }
  }
  *cursor += batch;
  free(perm);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * aggregator.cpp:25-41  client sampling
 * ------------------------------------------------------------------------- */
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int orc_sample_clients(uint64_t population, uint64_t k, uint64_t seed, uint64_t round,
                       uint64_t* out) {
  if (k > population || k == 0) return ORC_CONFIG;
  uint64_t* ids = (uint64_t*)malloc(population * sizeof(uint64_t));
  for (uint64_t i = 0; i < population; ++i) ids[i] = i;
  rng_t r;
  rng_init(&r, orc_mix_seed2(seed, 0x53616d70ULL, round));
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t j = i + rng_uniform_u64(&r, population - i);
    const uint64_t t = ids[i];
    ids[i] = ids[j];
    ids[j] = t;
  }
  qsort(ids, k, sizeof(uint64_t), cmp_u64);
  memcpy(out, ids, k * sizeof(uint64_t));
  free(ids);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * optim.cpp:10-27  LR schedule
 * ------------------------------------------------------------------------- */
int orc_lr_at(const orc_train_cfg* s, uint64_t step, double* out) {
  if (!(s->eta_max > 0.0) || s->decay_steps == 0 || s->alpha < 0.0 || s->alpha > 1.0)
    return ORC_CONFIG;
  if (s->warmup_steps > 0 && step < s->warmup_steps) {
    *out = s->eta_max * (double)step / (double)s->warmup_steps;
    return ORC_OK;
  }
  double p = (double)(step - s->warmup_steps) / (double)s->decay_steps;
  if (p > 1.0) p = 1.0;
  const double lo = s->alpha * s->eta_max;
  *out = lo + (s->eta_max - lo) * 0.5 * (1.0 + cos(3.14159265358979323846 * p));
  return ORC_OK;
}

/* param_vector.cpp:105-110 */
double orc_global_norm(const double* x, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += x[i] * x[i];
  return sqrt(acc);
}

/* optim.cpp:50-57 */
static int clip_factor(const double* g, uint64_t n, double clip_norm, double* cf) {
  const double norm = orc_global_norm(g, n);
  if (!isfinite(norm)) return ORC_NUMERIC;
  *cf = (clip_norm > 0.0 && norm > clip_norm) ? clip_norm / norm : 1.0;
  return ORC_OK;
}

/* optim.cpp:61-90 */
int orc_adamw_step(double* p, const double* g, double* m, double* v, uint64_t n,
                   uint64_t* step_count, const orc_train_cfg* t, double lr) {
  if (!(lr >= 0.0) || !isfinite(lr)) return ORC_CONFIG;
  double cf;
  int rc = clip_factor(g, n, t->clip_norm, &cf);
  if (rc) return rc;
  *step_count += 1;
  const double b1 = t->beta1, b2 = t->beta2;
  const double bc1 = 1.0 - pow(b1, (double)*step_count);
  const double bc2 = 1.0 - pow(b2, (double)*step_count);
  for (uint64_t j = 0; j < n; ++j) {
    const double gj = g[j] * cf;
    m[j] = b1 * m[j] + (1.0 - b1) * gj;
    v[j] = b2 * v[j] + (1.0 - b2) * gj * gj;
    const double mhat = m[j] / bc1;
    const double vhat = v[j] / bc2;
    p[j] -= lr * (mhat / (sqrt(vhat) + t->eps) + t->weight_decay * p[j]);
  }
  return ORC_OK;
}

/* optim.cpp:92-103 */
int orc_sgd_step(double* p, const double* g, uint64_t n, double lr, double clip_norm) {
  double cf;
  int rc = clip_factor(g, n, clip_norm, &cf);
  if (rc) return rc;
  for (uint64_t j = 0; j < n; ++j) p[j] -= lr * (g[j] * cf);
  return ORC_OK;
}

/* param_vector.cpp:127-152  anchored mean */
int orc_mean(const double* const* vs, uint64_t k, uint64_t n, double* out) {
  if (k == 0) return ORC_USAGE;
  const double cnt = (double)k;
  for (uint64_t j = 0; j < n; ++j) {
    const double anchor = vs[0][j];
    double corr = 0.0;
    for (uint64_t i = 1; i < k; ++i) corr += vs[i][j] - anchor;
    out[j] = anchor;
    if (corr != 0.0) out[j] = anchor + corr / cnt;
  }
  return ORC_OK;
}

/* param_vector.cpp:120-125  a + (-1.0)*b */
void orc_sub(const double* a, const double* b, uint64_t n, double* out) {
  for (uint64_t j = 0; j < n; ++j) out[j] = a[j] + -1.0 * b[j];
}

/* optim.cpp:105-159 */
int orc_server_step(const orc_server_cfg* s, const double* theta, const double* delta,
                    const double* mean, double* velocity, uint64_t n, double* out) {
  if (!(s->eta > 0.0) || s->momentum < 0.0 || s->momentum >= 1.0) return ORC_CONFIG;
  if (s->kind == 0 && (s->eta != 1.0 || s->momentum != 0.0)) return ORC_CONFIG;
  if (s->kind == 0) {
    memcpy(out, mean, n * sizeof(double));
    return ORC_OK;
  }
  const double mu = s->momentum;
  for (uint64_t j = 0; j < n; ++j) velocity[j] = mu * velocity[j] + delta[j];
  if (s->eta == 1.0 && mu == 0.0) {
    memcpy(out, mean, n * sizeof(double));
    return ORC_OK;
  }
  for (uint64_t j = 0; j < n; ++j) {
    const double dir = s->nesterov ? mu * velocity[j] + delta[j] : velocity[j];
    out[j] = theta[j] - s->eta * dir;
  }
  return ORC_OK;
}

/* client.cpp:96-110 */
int orc_post_process(const double* theta_ref, const double* theta_k, uint64_t n,
                     int32_t kind, double threshold, double* out) {
  if (kind == 0) {
    memcpy(out, theta_k, n * sizeof(double));
    return ORC_OK;
  }
  if (!(threshold > 0.0)) return ORC_CONFIG;
  double* upd = (double*)malloc(n * sizeof(double));
  orc_sub(theta_k, theta_ref, n, upd);
  const double norm = orc_global_norm(upd, n);
  if (norm <= threshold) {
    memcpy(out, theta_k, n * sizeof(double));
  } else {
    const double a = threshold / norm;
    for (uint64_t j = 0; j < n; ++j) out[j] = theta_ref[j] + a * upd[j];
  }
  free(upd);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Model forward / backward.  Restates model.cpp:98-174 through the tensor
 * ops of tensor.cpp, with the backward replaying the reverse topological
 * order the reference's DFS produces (tensor.cpp:605-647): within a block
 * add(x_mid) -> mlp -> LN2 -> add(x) -> attn-out -> attention -> v -> k -> q
 * -> LN1; so LN1's output gradient sums the v, k, q contributions in that
 * order and each residual node sums (residual edge, LN edge).
 * ------------------------------------------------------------------------- */

/* matmul fwd tensor.cpp:160-172: out[m,n] = a[m,k] b[k,n] */
static void mm_fwd(const double* a, const double* b, double* out, uint64_t m, uint64_t k,
                   uint64_t n) {
  memset(out, 0, m * n * sizeof(double));
  for (uint64_t i = 0; i < m; ++i) {
    double* ci = out + i * n;
    for (uint64_t p = 0; p < k; ++p) {
      const double aip = a[i * k + p];
      const double* bp = b + p * n;
      for (uint64_t j = 0; j < n; ++j) ci[j] += aip * bp[j];
    }
  }
}
/* matmul bwd tensor.cpp:181-205: ga += g b^T ; gb += a^T g */
static void mm_bwd(const double* g, const double* a, const double* b, double* ga, double* gb,
                   uint64_t m, uint64_t k, uint64_t n) {
  if (ga) {
    for (uint64_t i = 0; i < m; ++i)
      for (uint64_t p = 0; p < k; ++p) {
        double acc = 0.0;
        const double* gi = g + i * n;
        const double* bp = b + p * n;
        for (uint64_t j = 0; j < n; ++j) acc += gi[j] * bp[j];
        ga[i * k + p] += acc;
      }
  }
  if (gb) {
    for (uint64_t i = 0; i < m; ++i) {
      const double* gi = g + i * n;
      for (uint64_t p = 0; p < k; ++p) {
        const double aip = a[i * k + p];
        double* gbp = gb + p * n;
        for (uint64_t j = 0; j < n; ++j) gbp[j] += aip * gi[j];
      }
    }
  }
}
/* add_bias tensor.cpp:261-288 */
static void bias_fwd(double* x, const double* b, uint64_t m, uint64_t n) {
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < n; ++j) x[i * n + j] = x[i * n + j] + b[j];
}
static void bias_bwd(const double* g, double* gx, double* gb, uint64_t m, uint64_t n) {
  for (uint64_t i = 0; i < m * n; ++i) gx[i] += g[i];
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < n; ++j) gb[j] += g[i * n + j];
}
/* layer_norm tensor.cpp:322-394 */
static void ln_fwd(const double* x, const double* gain, const double* bias, double* out,
                   double* xhat, double* inv_std, uint64_t m, uint64_t n) {
  for (uint64_t i = 0; i < m; ++i) {
    const double* xi = x + i * n;
    double mean = 0.0;
    for (uint64_t j = 0; j < n; ++j) mean += xi[j];
    mean /= (double)n;
    double var = 0.0;
    for (uint64_t j = 0; j < n; ++j) {
      const double dd = xi[j] - mean;
      var += dd * dd;
    }
    var /= (double)n;
    const double inv = 1.0 / sqrt(var + 1e-5);
    inv_std[i] = inv;
    for (uint64_t j = 0; j < n; ++j) {
      const double xh = (xi[j] - mean) * inv;
      xhat[i * n + j] = xh;
      out[i * n + j] = gain[j] * xh + bias[j];
    }
  }
}
static void ln_bwd(const double* g, const double* xhat, const double* inv_std,
                   const double* gain, double* gx, double* ggain, double* gbias, uint64_t m,
                   uint64_t n) {
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < n; ++j) ggain[j] += g[i * n + j] * xhat[i * n + j];
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < n; ++j) gbias[j] += g[i * n + j];
  for (uint64_t i = 0; i < m; ++i) {
    const double* gi = g + i * n;
    const double* xh = xhat + i * n;
    double s1 = 0.0, s2 = 0.0;
    for (uint64_t j = 0; j < n; ++j) {
      const double dxh = gi[j] * gain[j];
      s1 += dxh;
      s2 += dxh * xh[j];
    }
    s1 /= (double)n;
    s2 /= (double)n;
    const double inv = inv_std[i];
    for (uint64_t j = 0; j < n; ++j) {
      const double dxh = gi[j] * gain[j];
      gx[i * n + j] += inv * (dxh - s1 - xh[j] * s2);
    }
  }
}
/* gelu tensor.cpp:396-420 */
static void gelu_fwd(const double* x, double* out, uint64_t n) {
  const double inv_sqrt2 = 0.70710678118654752440;
  for (uint64_t i = 0; i < n; ++i) out[i] = 0.5 * x[i] * (1.0 + erf(x[i] * inv_sqrt2));
}
static void gelu_bwd(const double* g, const double* x, double* gx, uint64_t n) {
  const double inv_sqrt2 = 0.70710678118654752440;
  const double inv_sqrt2pi = 0.39894228040143267794;
  for (uint64_t i = 0; i < n; ++i) {
    const double xv = x[i];
    const double cdf = 0.5 * (1.0 + erf(xv * inv_sqrt2));
    const double pdf = inv_sqrt2pi * exp(-0.5 * xv * xv);
    gx[i] += g[i] * (cdf + xv * pdf);
  }
}
/* causal_attention tensor.cpp:436-542 */
static void attn_fwd(const double* q, const double* k, const double* v, double* out,
                     double* probs, uint64_t B, uint64_t S, uint64_t H, uint64_t d) {
  const uint64_t dh = d / H;
  const double inv_scale = 1.0 / sqrt((double)dh);
  double* scores = (double*)malloc(S * sizeof(double));
  memset(out, 0, B * S * d * sizeof(double));
  memset(probs, 0, B * H * S * S * sizeof(double));
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t h = 0; h < H; ++h) {
      const uint64_t c0 = h * dh;
      double* pr = probs + (b * H + h) * S * S;
      for (uint64_t i = 0; i < S; ++i) {
        const double* qi = q + (b * S + i) * d + c0;
        double row_max = -1e300;
        for (uint64_t j = 0; j <= i; ++j) {
          const double* kj = k + (b * S + j) * d + c0;
          double s = 0.0;
          for (uint64_t c = 0; c < dh; ++c) s += qi[c] * kj[c];
          s *= inv_scale;
          scores[j] = s;
          if (s > row_max) row_max = s;
        }
        double denom = 0.0;
        for (uint64_t j = 0; j <= i; ++j) {
          const double e = exp(scores[j] - row_max);
          scores[j] = e;
          denom += e;
        }
        double* oi = out + (b * S + i) * d + c0;
        for (uint64_t j = 0; j <= i; ++j) {
          const double p = scores[j] / denom;
          pr[i * S + j] = p;
          const double* vj = v + (b * S + j) * d + c0;
          for (uint64_t c = 0; c < dh; ++c) oi[c] += p * vj[c];
        }
      }
    }
  free(scores);
}
static void attn_bwd(const double* g, const double* q, const double* k, const double* v,
                     const double* probs, double* gq, double* gk, double* gv, uint64_t B,
                     uint64_t S, uint64_t H, uint64_t d) {
  const uint64_t dh = d / H;
  const double inv_scale = 1.0 / sqrt((double)dh);
  double* dp = (double*)malloc(S * sizeof(double));
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t h = 0; h < H; ++h) {
      const uint64_t c0 = h * dh;
      const double* pr = probs + (b * H + h) * S * S;
      for (uint64_t i = 0; i < S; ++i) {
        const double* gi = g + (b * S + i) * d + c0;
        double dot = 0.0;
        for (uint64_t j = 0; j <= i; ++j) {
          const double p = pr[i * S + j];
          const double* vj = v + (b * S + j) * d + c0;
          double dpj = 0.0;
          for (uint64_t c = 0; c < dh; ++c) dpj += gi[c] * vj[c];
          dp[j] = dpj;
          dot += p * dpj;
          double* gvj = gv + (b * S + j) * d + c0;
          for (uint64_t c = 0; c < dh; ++c) gvj[c] += p * gi[c];
        }
        for (uint64_t j = 0; j <= i; ++j) {
          const double ds = pr[i * S + j] * (dp[j] - dot) * inv_scale;
          const double* kj = k + (b * S + j) * d + c0;
          const double* qi = q + (b * S + i) * d + c0;
          double* gqi = gq + (b * S + i) * d + c0;
          for (uint64_t c = 0; c < dh; ++c) gqi[c] += ds * kj[c];
          double* gkj = gk + (b * S + j) * d + c0;
          for (uint64_t c = 0; c < dh; ++c) gkj[c] += ds * qi[c];
        }
      }
    }
  free(dp);
}

typedef struct {
  double *x_in, *xhat1, *inv1, *h, *q, *k, *v, *probs, *att, *x_mid, *xhat2, *inv2, *h2,
      *pre, *u;
} layer_acts;

static double* dalloc(uint64_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }

/* entry offsets of block b in the canonical layout */
typedef struct {
  uint64_t ln1g, ln1b, wq, bq, wk, bk, wv, bv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
} block_offs;

static block_offs block_offsets(const orc_model_cfg* c, uint64_t b) {
  uint64_t o[16], rows, cols;
  for (int j = 0; j < 16; ++j) orc_layout_entry(c, 2 + 16 * b + (uint64_t)j, &o[j], &rows, &cols, NULL, 0);
  block_offs r = {o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7],
                  o[8], o[9], o[10], o[11], o[12], o[13], o[14], o[15]};
  return r;
}

/* model.cpp:98-158 + tensor.cpp:544-603 + backward */
int orc_forward_backward(const orc_model_cfg* c, const double* P, const int32_t* inputs,
                         const int32_t* targets, uint64_t B, uint64_t S, double* loss_out,
                         double* G) {
  if (orc_model_validate(c)) return ORC_CONFIG;
  if (B == 0 || S == 0) return ORC_SHAPE;
  if (S > c->seq_len) return ORC_SHAPE;
  const uint64_t d = c->d_model, H = c->n_heads, hid = c->expansion_ratio * d,
                 V = c->vocab_size, L = c->n_blocks, M = B * S;
  for (uint64_t i = 0; i < M; ++i)
    if (inputs[i] < 0 || (uint64_t)inputs[i] >= V) return ORC_INDEX;
  uint64_t count = 0;
  for (uint64_t i = 0; i < M; ++i)
    if (targets[i] >= 0) {
      if ((uint64_t)targets[i] >= V) return ORC_INDEX;
      ++count;
    }
  if (count == 0) return ORC_USAGE;

  uint64_t off_pos, off_fg, off_fb, off_hw, off_hb, rr, cc;
  orc_layout_entry(c, 1, &off_pos, &rr, &cc, NULL, 0);
  orc_layout_entry(c, 2 + 16 * L + 0, &off_fg, &rr, &cc, NULL, 0);
  orc_layout_entry(c, 2 + 16 * L + 1, &off_fb, &rr, &cc, NULL, 0);
  orc_layout_entry(c, 2 + 16 * L + 2, &off_hw, &rr, &cc, NULL, 0);
  orc_layout_entry(c, 2 + 16 * L + 3, &off_hb, &rr, &cc, NULL, 0);

  layer_acts* la = (layer_acts*)calloc(L, sizeof(layer_acts));
  /* embeddings: add(gather(tok, inputs), gather(pos, r % S)) */
  double* x = dalloc(M * d);
  for (uint64_t i = 0; i < M; ++i) {
    const double* te = P + (uint64_t)inputs[i] * d;
    const double* pe = P + off_pos + (i % S) * d;
    for (uint64_t j = 0; j < d; ++j) x[i * d + j] = te[j] + pe[j];
  }
  for (uint64_t b = 0; b < L; ++b) {
    const block_offs o = block_offsets(c, b);
    layer_acts* a = &la[b];
    a->x_in = x;
    a->xhat1 = dalloc(M * d); a->inv1 = dalloc(M); a->h = dalloc(M * d);
    ln_fwd(x, P + o.ln1g, P + o.ln1b, a->h, a->xhat1, a->inv1, M, d);
    a->q = dalloc(M * d); a->k = dalloc(M * d); a->v = dalloc(M * d);
    mm_fwd(a->h, P + o.wq, a->q, M, d, d); bias_fwd(a->q, P + o.bq, M, d);
    mm_fwd(a->h, P + o.wk, a->k, M, d, d); bias_fwd(a->k, P + o.bk, M, d);
    mm_fwd(a->h, P + o.wv, a->v, M, d, d); bias_fwd(a->v, P + o.bv, M, d);
    a->probs = dalloc(B * H * S * S); a->att = dalloc(M * d);
    attn_fwd(a->q, a->k, a->v, a->att, a->probs, B, S, H, d);
    double* proj = dalloc(M * d);
    mm_fwd(a->att, P + o.wo, proj, M, d, d); bias_fwd(proj, P + o.bo, M, d);
    a->x_mid = dalloc(M * d);
    for (uint64_t i = 0; i < M * d; ++i) a->x_mid[i] = x[i] + proj[i];
    free(proj);
    a->xhat2 = dalloc(M * d); a->inv2 = dalloc(M); a->h2 = dalloc(M * d);
    ln_fwd(a->x_mid, P + o.ln2g, P + o.ln2b, a->h2, a->xhat2, a->inv2, M, d);
    a->pre = dalloc(M * hid); a->u = dalloc(M * hid);
    mm_fwd(a->h2, P + o.w1, a->pre, M, d, hid); bias_fwd(a->pre, P + o.b1, M, hid);
    gelu_fwd(a->pre, a->u, M * hid);
    double* mlp = dalloc(M * d);
    mm_fwd(a->u, P + o.w2, mlp, M, hid, d); bias_fwd(mlp, P + o.b2, M, d);
    x = dalloc(M * d);
    for (uint64_t i = 0; i < M * d; ++i) x[i] = a->x_mid[i] + mlp[i];
    free(mlp);
  }
  double* xL = x;
  double* xhatf = dalloc(M * d); double* invf = dalloc(M); double* xf = dalloc(M * d);
  ln_fwd(xL, P + off_fg, P + off_fb, xf, xhatf, invf, M, d);
  double* logits = dalloc(M * V);
  mm_fwd(xf, P + off_hw, logits, M, d, V); bias_fwd(logits, P + off_hb, M, V);

  /* softmax_cross_entropy tensor.cpp:544-603 */
  double* probs = dalloc(M * V);
  double loss = 0.0;
  for (uint64_t i = 0; i < M; ++i) {
    const double* li = logits + i * V;
    double mx = li[0];
    for (uint64_t v = 1; v < V; ++v)
      if (li[v] > mx) mx = li[v];
    double denom = 0.0;
    for (uint64_t v = 0; v < V; ++v) {
      const double e = exp(li[v] - mx);
      probs[i * V + v] = e;
      denom += e;
    }
    for (uint64_t v = 0; v < V; ++v) probs[i * V + v] /= denom;
    if (targets[i] >= 0) loss += log(denom) + mx - li[targets[i]];
  }
  loss /= (double)count;
  *loss_out = loss;

  if (G) {
    const uint64_t Pn = orc_param_count(c);
    memset(G, 0, Pn * sizeof(double));
    /* CE backward */
    double* glog = dalloc(M * V);
    const double g0 = 1.0 / (double)count;
    for (uint64_t i = 0; i < M; ++i) {
      if (targets[i] < 0) continue;
      double* gi = glog + i * V;
      const double* pi = probs + i * V;
      for (uint64_t v = 0; v < V; ++v) gi[v] += g0 * pi[v];
      gi[targets[i]] -= g0;
    }
    /* logits = add_bias(mm_h, bh) */
    double* gmm = dalloc(M * V);
    bias_bwd(glog, gmm, G + off_hb, M, V);
    free(glog);
    double* gxf = dalloc(M * d);
    mm_bwd(gmm, xf, P + off_hw, gxf, G + off_hw, M, d, V);
    free(gmm);
    double* gx = dalloc(M * d); /* grad of the residual stream node */
    ln_bwd(gxf, xhatf, invf, P + off_fg, gx, G + off_fg, G + off_fb, M, d);
    free(gxf);
    for (uint64_t bb = L; bb-- > 0;) {
      const block_offs o = block_offsets(c, bb);
      layer_acts* a = &la[bb];
      /* x_out = add(x_mid, mlp): x_mid.grad += g ; mlp.grad += g */
      double* gxmid = dalloc(M * d);
      for (uint64_t i = 0; i < M * d; ++i) gxmid[i] += gx[i];
      double* gmlp = dalloc(M * d);
      for (uint64_t i = 0; i < M * d; ++i) gmlp[i] += gx[i];
      free(gx);
      double* gmm2 = dalloc(M * d);
      bias_bwd(gmlp, gmm2, G + o.b2, M, d);
      free(gmlp);
      double* gu = dalloc(M * hid);
      mm_bwd(gmm2, a->u, P + o.w2, gu, G + o.w2, M, hid, d);
      free(gmm2);
      double* gpre = dalloc(M * hid);
      gelu_bwd(gu, a->pre, gpre, M * hid);
      free(gu);
      double* gmm1 = dalloc(M * hid);
      bias_bwd(gpre, gmm1, G + o.b1, M, hid);
      free(gpre);
      double* gh2 = dalloc(M * d);
      mm_bwd(gmm1, a->h2, P + o.w1, gh2, G + o.w1, M, d, hid);
      free(gmm1);
      ln_bwd(gh2, a->xhat2, a->inv2, P + o.ln2g, gxmid, G + o.ln2g, G + o.ln2b, M, d);
      free(gh2);
      /* x_mid = add(x_in, attn_out) */
      double* gxin = dalloc(M * d);
      for (uint64_t i = 0; i < M * d; ++i) gxin[i] += gxmid[i];
      double* gproj = dalloc(M * d);
      for (uint64_t i = 0; i < M * d; ++i) gproj[i] += gxmid[i];
      free(gxmid);
      double* gmmo = dalloc(M * d);
      bias_bwd(gproj, gmmo, G + o.bo, M, d);
      free(gproj);
      double* gatt = dalloc(M * d);
      mm_bwd(gmmo, a->att, P + o.wo, gatt, G + o.wo, M, d, d);
      free(gmmo);
      double* gq = dalloc(M * d); double* gk = dalloc(M * d); double* gv = dalloc(M * d);
      attn_bwd(gatt, a->q, a->k, a->v, a->probs, gq, gk, gv, B, S, H, d);
      free(gatt);
      double* gh = dalloc(M * d);
      double* tmp = dalloc(M * d);
      /* v, then k, then q (reverse topological order) */
      bias_bwd(gv, tmp, G + o.bv, M, d);
      mm_bwd(tmp, a->h, P + o.wv, gh, G + o.wv, M, d, d);
      memset(tmp, 0, M * d * sizeof(double));
      bias_bwd(gk, tmp, G + o.bk, M, d);
      mm_bwd(tmp, a->h, P + o.wk, gh, G + o.wk, M, d, d);
      memset(tmp, 0, M * d * sizeof(double));
      bias_bwd(gq, tmp, G + o.bq, M, d);
      mm_bwd(tmp, a->h, P + o.wq, gh, G + o.wq, M, d, d);
      free(tmp); free(gq); free(gk); free(gv);
      ln_bwd(gh, a->xhat1, a->inv1, P + o.ln1g, gxin, G + o.ln1g, G + o.ln1b, M, d);
      free(gh);
      gx = gxin;
    }
    /* x0 = add(gather(tok), gather(pos)); gather bwd ascending rows */
    for (uint64_t i = 0; i < M; ++i) {
      double* dst = G + (uint64_t)inputs[i] * d;
      for (uint64_t j = 0; j < d; ++j) dst[j] += gx[i * d + j];
    }
    for (uint64_t i = 0; i < M; ++i) {
      double* dst = G + off_pos + (i % S) * d;
      for (uint64_t j = 0; j < d; ++j) dst[j] += gx[i * d + j];
    }
    free(gx);
  }

  for (uint64_t b = 0; b < L; ++b) {
    layer_acts* a = &la[b];
    free(a->x_in); free(a->xhat1); free(a->inv1); free(a->h); free(a->q); free(a->k);
    free(a->v); free(a->probs); free(a->att); free(a->xhat2); free(a->inv2); free(a->h2);
    free(a->pre); free(a->u);
    if (b + 1 == L) { /* x_mid of last block is still referenced nowhere */ }
    free(a->x_mid);
  }
  free(la);
  free(xL); free(xhatf); free(invf); free(xf); free(logits); free(probs);
  return ORC_OK;
}

/* model.cpp:176-192 */
int orc_eval_perplexity(const orc_model_cfg* c, const double* params, const int32_t* inputs,
                        const int32_t* targets, uint64_t n_batches, const uint64_t* bsz,
                        uint64_t seq, double* ppl_out) {
  if (n_batches == 0) return ORC_USAGE;
  double total_nll = 0.0;
  uint64_t total_tokens = 0, row = 0;
  for (uint64_t bi = 0; bi < n_batches; ++bi) {
    const int32_t* in = inputs + row * seq;
    const int32_t* tg = targets + row * seq;
    uint64_t valid = 0;
    for (uint64_t i = 0; i < bsz[bi] * seq; ++i)
      if (tg[i] >= 0) ++valid;
    double loss;
    int rc = orc_forward_backward(c, params, in, tg, bsz[bi], seq, &loss, NULL);
    if (rc) return rc;
    total_nll += loss * (double)valid;
    total_tokens += valid;
    row += bsz[bi];
  }
  if (total_tokens == 0) return ORC_USAGE;
  *ppl_out = exp(total_nll / (double)total_tokens);
  return ORC_OK;
}

/* client.cpp:125-158 */
int orc_local_round(const orc_model_cfg* c, const orc_train_cfg* t, const double* theta_in,
                    const orc_plan* plan, uint64_t client, uint64_t stream_seed,
                    uint64_t* cursor, uint64_t round, uint64_t step_base, double* theta_out,
                    double* losses, uint64_t* err_step) {
  (void)round;
  if (orc_model_validate(c)) return ORC_CONFIG;
  if (t->beta1 < 0.0 || t->beta1 >= 1.0 || t->beta2 < 0.0 || t->beta2 >= 1.0 ||
      !(t->eps > 0.0) || t->weight_decay < 0.0)
    return ORC_CONFIG;
  const uint64_t Pn = orc_param_count(c), B = t->batch_size, S = plan->seq_len;
  double* th = dalloc(Pn);
  memcpy(th, theta_in, Pn * sizeof(double));
  double* m = dalloc(Pn);
  double* v = dalloc(Pn);
  double* g = dalloc(Pn);
  int32_t* in = (int32_t*)malloc(B * S * sizeof(int32_t));
  int32_t* tg = (int32_t*)malloc(B * S * sizeof(int32_t));
  uint64_t steps = 0;
  int rc = ORC_OK;
  for (uint64_t i = 0; i < t->local_steps && rc == ORC_OK; ++i) {
    rc = orc_stream_next(plan, client, B, S, stream_seed, cursor, in, tg);
    if (rc) break;
    double loss;
    rc = orc_forward_backward(c, th, in, tg, B, S, &loss, g);
    if (rc) break;
    if (!isfinite(loss)) {
      if (err_step) *err_step = i;
      rc = ORC_DIVERGENCE;
      break;
    }
    double lr;
    rc = orc_lr_at(t, step_base + i, &lr);
    if (rc) break;
    if (t->opt == 0)
      rc = orc_adamw_step(th, g, m, v, Pn, &steps, t, lr);
    else
      rc = orc_sgd_step(th, g, Pn, lr, t->sgd_clip_norm);
    if (losses) losses[i] = loss;
  }
  if (rc == ORC_OK) rc = orc_post_process(theta_in, th, Pn, t->post_kind, t->post_threshold, theta_out);
  free(th); free(m); free(v); free(g); free(in); free(tg);
  return rc;
}

/* aggregator.cpp:93-220 (cost model, eval and checkpoint hooks omitted) */
int orc_run_round(const orc_model_cfg* c, const orc_train_cfg* t, const orc_server_cfg* s,
                  const orc_plan* plan, uint64_t population, uint64_t k, uint64_t seed,
                  uint64_t round, double* theta, double* velocity, uint64_t* cursors,
                  const uint64_t* dropped, uint64_t n_dropped, int32_t ring_topology,
                  uint64_t* sampled_out, double* client_mean_losses) {
  const uint64_t Pn = orc_param_count(c);
  uint64_t* sampled = (uint64_t*)malloc(k * sizeof(uint64_t));
  int rc = orc_sample_clients(population, k, seed, round, sampled);
  if (rc) { free(sampled); return rc; }
  double** models = (double**)calloc(k, sizeof(double*));
  double* losses = dalloc(t->local_steps);
  const double** surv = (const double**)calloc(k, sizeof(double*));
  uint64_t n_surv = 0;
  for (uint64_t si = 0; si < k && rc == ORC_OK; ++si) {
    const uint64_t cl = sampled[si];
    models[si] = dalloc(Pn);
    uint64_t cur = cursors[cl];
    rc = orc_local_round(c, t, theta, plan, cl, orc_stream_seed(seed, cl), &cur, round,
                         round * t->local_steps, models[si], losses, NULL);
    if (rc) break;
    cursors[cl] = cur;
    double acc = 0.0;
    for (uint64_t i = 0; i < t->local_steps; ++i) acc += losses[i];
    if (client_mean_losses)
      client_mean_losses[si] = t->local_steps ? acc / (double)t->local_steps : 0.0;
    int drop = 0;
    for (uint64_t d = 0; d < n_dropped; ++d)
      if (dropped[d] == cl) drop = 1;
    if (!drop) surv[n_surv++] = models[si];
  }
  if (rc == ORC_OK) {
    if (n_surv == 0) rc = ORC_ROUND_FAILURE;
    else if (n_surv < k && ring_topology) rc = ORC_ROUND_FAILURE;
  }
  if (rc == ORC_OK) {
    double* mean = dalloc(Pn);
    double* delta = dalloc(Pn);
    double* next = dalloc(Pn);
    orc_mean(surv, n_surv, Pn, mean);
    orc_sub(theta, mean, Pn, delta);
    rc = orc_server_step(s, theta, delta, mean, velocity, Pn, next);
    if (rc == ORC_OK) memcpy(theta, next, Pn * sizeof(double));
    free(mean); free(delta); free(next);
  }
  if (sampled_out) memcpy(sampled_out, sampled, k * sizeof(uint64_t));
  for (uint64_t si = 0; si < k; ++si) free(models[si]);
  free(models); free(surv); free(losses); free(sampled);
  return rc;
}
