// capi.cpp -- the extern "C" boundary (include/photon.h).  C++ exceptions
// (photon::Error, carrying fedsim/errors.h-equivalent codes) are converted to
// status codes + photon_err here and nowhere else.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "gemm.cuh"
#include "kernels.cuh"
#include "nccl_api.hpp"
#include "runner.hpp"
#include "central.hpp"

struct photon_plan {
  photon::Plan p;
};
struct photon_ctx {
  photon::Ctx c;
  photon_ctx(int dev, const photon_model_cfg& m, int prec, uint64_t mb) : c(dev, m, prec, mb) {}
};
struct photon_runner {
  std::unique_ptr<photon::Runner> r;
};
struct photon_eval_set {
  photon::EvalSet s;
};
struct photon_central {
  std::unique_ptr<photon::Central> c;
};

using namespace photon;

namespace {

void set_err(photon_err* err, int code, const char* msg, uint64_t round = 0, uint64_t client = 0,
             uint64_t step = 0) {
  if (!err) return;
  err->code = code;
  err->round = round;
  err->client = client;
  err->step = step;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

template <typename F>
int guarded(photon_err* err, F&& f) {
  try {
    f();
    if (err) err->code = PHOTON_OK;
    return PHOTON_OK;
  } catch (const Error& e) {
    set_err(err, e.code, e.what(), e.round, e.client, e.step);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err(err, PHOTON_ERR_CAPACITY, "host allocation failed");
    return PHOTON_ERR_CAPACITY;
  } catch (const std::exception& e) {
    set_err(err, PHOTON_ERR_USAGE, e.what());
    return PHOTON_ERR_USAGE;
  }
}

void need(bool ok, int code, const char* msg) {
  if (!ok) throw Error(code, msg);
}

// One batch [B,S] staged as a single-step round.
void stage_single(Ctx& c, RoundBatches& rb, const int32_t* inputs, const int32_t* targets,
                  uint64_t B, uint64_t S) {
  rb.prepare(1, (int)B, (int)S, (int)c.cfg.vocab_size);
  std::memcpy(rb.tokens.ptr, inputs, B * S * 4);
  std::memcpy(rb.targets.ptr, targets, B * S * 4);
  rb.finalize((int)c.cfg.vocab_size);
  c.upload(rb);
}

void load_params(Ctx& c, const double* params) {
  Engine& e = *c.eng;
  c.h2d_f64_to_f32(params, e.master, e.P);
  e.refresh_shadow();
}

void check_batch(const Ctx& c, uint64_t B, uint64_t S) {
  need(B > 0 && S > 0, PHOTON_ERR_SHAPE, "forward: inconsistent batch");
  need(S <= c.cfg.seq_len, PHOTON_ERR_SHAPE, "forward: batch seq_len exceeds model seq_len");
}

}  // namespace

extern "C" {

int photon_abi_version(void) { return PHOTON_ABI_VERSION; }

const char* photon_status_name(int code) {
  switch (code) {
    case PHOTON_OK: return "OK";
    case PHOTON_ERR_CONFIG: return "ConfigError";
    case PHOTON_ERR_CAPACITY: return "CapacityError";
    case PHOTON_ERR_SHAPE: return "ShapeError";
    case PHOTON_ERR_INDEX: return "IndexError";
    case PHOTON_ERR_USAGE: return "UsageError";
    case PHOTON_ERR_LOOKUP: return "LookupError";
    case PHOTON_ERR_NUMERIC: return "NumericError";
    case PHOTON_ERR_DIVERGENCE: return "DivergenceError";
    case PHOTON_ERR_IO: return "IoError";
    case PHOTON_ERR_INTEGRITY: return "IntegrityError";
    case PHOTON_ERR_ROUND_FAILURE: return "RoundFailureError";
    case PHOTON_ERR_PARSE: return "ParseError";
    case PHOTON_ERR_CUDA: return "CudaError";
    case PHOTON_ERR_NCCL: return "NcclError";
  }
  return "Unknown";
}

uint64_t photon_mix64(uint64_t x) { return mix64(x); }
uint64_t photon_stream_seed(uint64_t s, uint64_t client) { return derive(s, kPurposeStream, client); }

int photon_sample_clients(uint64_t population, uint64_t k, uint64_t seed, uint64_t round,
                          uint64_t* out, photon_err* err) {
  return guarded(err, [&] {
    const auto ids = sample_clients(population, k, seed, round);
    std::memcpy(out, ids.data(), ids.size() * 8);
  });
}

int photon_lr_at(const photon_lr_schedule* s, uint64_t step, double* out, photon_err* err) {
  return guarded(err, [&] { *out = lr_at(*s, step); });
}

uint64_t photon_param_count(const photon_model_cfg* m) { return param_count(*m); }
uint64_t photon_layout_size(const photon_model_cfg* m) { return 2 + 16 * m->n_blocks + 4; }

int photon_layout_entry(const photon_model_cfg* m, uint64_t i, uint64_t* offset, uint64_t* rows,
                        uint64_t* cols, char* name, int cap) {
  return guarded(nullptr, [&] {
    const auto lay = layout(*m);
    need(i < lay.size(), PHOTON_ERR_INDEX, "param entry index out of range");
    *offset = lay[i].offset;
    *rows = lay[i].rows;
    *cols = lay[i].cols;
    if (name && cap > 0) std::snprintf(name, (size_t)cap, "%s", lay[i].name.c_str());
  });
}

int photon_init_params(const photon_model_cfg* m, uint64_t seed, double* out, photon_err* err) {
  return guarded(err, [&] {
    const auto v = init_params(*m, seed);
    std::memcpy(out, v.data(), v.size() * 8);
  });
}

int photon_generate_corpus(const char* style, uint64_t length, uint64_t seed, uint32_t vocab,
                           uint16_t* out, photon_err* err) {
  return guarded(err, [&] {
    const auto v = generate_corpus(style_index(style), length, seed, vocab);
    std::memcpy(out, v.data(), v.size() * 2);
  });
}

int photon_plan_iid(const uint16_t* tokens, uint64_t n, uint64_t shards, uint64_t seq_len,
                    uint64_t seed, photon_plan** out, photon_err* err) {
  return guarded(err, [&] {
    *out = new photon_plan{Plan::iid(std::vector<uint16_t>(tokens, tokens + n), shards, seq_len, seed)};
  });
}

int photon_plan_by_source(const uint16_t* const* corpora, const uint64_t* lens, uint64_t n_sources,
                          uint64_t cps, uint64_t seq_len, photon_plan** out, photon_err* err) {
  return guarded(err, [&] {
    std::vector<std::vector<uint16_t>> cs;
    for (uint64_t s = 0; s < n_sources; ++s) cs.emplace_back(corpora[s], corpora[s] + lens[s]);
    *out = new photon_plan{Plan::by_source(std::move(cs), cps, seq_len)};
  });
}

int photon_plan_from_blocks(const uint16_t* const* corpora, const uint64_t* lens,
                            uint64_t n_sources, uint64_t seq_len, const uint64_t* n_blocks,
                            uint64_t n_clients, const uint32_t* sources, const uint64_t* offsets,
                            photon_plan** out, photon_err* err) {
  return guarded(err, [&] {
    need(corpora && lens && n_blocks && sources && offsets && out, PHOTON_ERR_USAGE,
         "plan_from_blocks: null argument");
    need(n_sources >= 1 && n_sources < (1u << 15), PHOTON_ERR_CONFIG,
         "plan_from_blocks: bad source count");
    need(seq_len >= 1 && n_clients >= 1, PHOTON_ERR_CONFIG, "plan_from_blocks: empty plan");
    Plan p;
    p.seq_len = seq_len;
    for (uint64_t s = 0; s < n_sources; ++s) p.corpora.emplace_back(corpora[s], corpora[s] + lens[s]);
    p.blocks.assign(n_clients, {});
    uint64_t j = 0;
    for (uint64_t c = 0; c < n_clients; ++c) {
      for (uint64_t i = 0; i < n_blocks[c]; ++i, ++j) {
        need(sources[j] < n_sources, PHOTON_ERR_INDEX, "plan_from_blocks: source out of range");
        need(offsets[j] + seq_len + 1 <= lens[sources[j]] && offsets[j] < (1ull << 48),
             PHOTON_ERR_INDEX, "plan_from_blocks: block past the end of its corpus");
        p.blocks[c].push_back((uint64_t)sources[j] << 48 | offsets[j]);
      }
    }
    *out = new photon_plan{std::move(p)};
  });
}

void photon_plan_free(photon_plan* p) { delete p; }
uint64_t photon_plan_n_clients(const photon_plan* p) { return p->p.blocks.size(); }
uint64_t photon_plan_client_blocks(const photon_plan* p, uint64_t c) {
  return c < p->p.blocks.size() ? p->p.blocks[c].size() : 0;
}

int photon_stream_next(const photon_plan* p, uint64_t client, uint64_t batch, uint64_t seed,
                       uint64_t* cursor, int32_t* inputs, int32_t* targets, photon_err* err) {
  return guarded(err, [&] {
    stream_rows(p->p, client, seed, *cursor, batch, inputs, targets);
    *cursor += batch;
  });
}

int photon_ctx_create(int device, const photon_model_cfg* m, int precision, uint64_t max_batch,
                      photon_ctx** out, photon_err* err) {
  return guarded(err, [&] { *out = new photon_ctx(device, *m, precision, max_batch); });
}

void photon_ctx_destroy(photon_ctx* ctx) { delete ctx; }
double photon_ctx_last_ms(const photon_ctx* ctx) { return ctx->c.last_ms; }

int photon_forward_backward(photon_ctx* ctx, const double* params, const int32_t* inputs,
                            const int32_t* targets, uint64_t B, uint64_t S, double* loss,
                            double* grads, photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    check_batch(c, B, S);
    RoundBatches rb;
    stage_single(c, rb, inputs, targets, B, S);
    load_params(c, params);
    Engine& e = *c.eng;
    c.d_losses.reserve(1);
    c.begin_timing();
    const DeviceBatches& db = c.dev_batches;
    StepBatch sb{db.tokens.ptr, db.targets.ptr, db.csr_off.ptr, db.csr_rows.ptr,
                 (int)B, (int)S, rb.inv_count[0]};
    e.forward_backward(sb, c.d_losses.ptr, grads != nullptr);
    c.end_timing();
    PH_CUDA(cudaMemcpy(loss, c.d_losses.ptr, 8, cudaMemcpyDeviceToHost));
    if (grads) c.d2h_f32_to_f64(e.grads, grads, e.P);
  });
}

// model.cpp:176-192
int photon_eval_perplexity(photon_ctx* ctx, const double* params, const int32_t* inputs,
                           const int32_t* targets, uint64_t n_batches, const uint64_t* bsz,
                           uint64_t S, double* ppl, photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    need(n_batches > 0, PHOTON_ERR_USAGE, "eval_perplexity: no batches");
    load_params(c, params);
    double nll = 0.0;
    uint64_t tokens = 0, row = 0;
    RoundBatches rb;
    c.d_losses.reserve(1);
    for (uint64_t b = 0; b < n_batches; ++b) {
      check_batch(c, bsz[b], S);
      const int32_t* in = inputs + row * S;
      const int32_t* tg = targets + row * S;
      uint64_t valid = 0;
      for (uint64_t i = 0; i < bsz[b] * S; ++i) valid += tg[i] >= 0;
      stage_single(c, rb, in, tg, bsz[b], S);
      const DeviceBatches& db = c.dev_batches;
      StepBatch sb{db.tokens.ptr, db.targets.ptr, db.csr_off.ptr, db.csr_rows.ptr,
                   (int)bsz[b], (int)S, rb.inv_count[0]};
      c.eng->forward_backward(sb, c.d_losses.ptr, false);
      double loss = 0.0;
      PH_CUDA(cudaMemcpyAsync(&loss, c.d_losses.ptr, 8, cudaMemcpyDeviceToHost, c.stream));
      PH_CUDA(cudaStreamSynchronize(c.stream));
      nll += loss * (double)valid;
      tokens += valid;
      row += bsz[b];
    }
    need(tokens > 0, PHOTON_ERR_USAGE, "eval_perplexity: no target tokens");
    *ppl = std::exp(nll / (double)tokens);
  });
}

int photon_client_round(photon_ctx* ctx, const photon_train_cfg* cfg, const double* theta_in,
                        const int32_t* inputs, const int32_t* targets, uint64_t round,
                        uint64_t client, uint64_t step_base, double* theta_out,
                        photon_step_metric* metrics, photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    check_train_cfg(*cfg);
    need(std::memcmp(&cfg->model, &c.cfg, sizeof(photon_model_cfg)) == 0, PHOTON_ERR_SHAPE,
         "params do not match model layout");
    const uint64_t B = cfg->batch_size, S = c.cfg.seq_len, tau = cfg->local_steps;
    check_batch(c, B, S);
    Engine& e = *c.eng;
    RoundBatches rb;
    rb.prepare((int)tau, (int)B, (int)S, (int)c.cfg.vocab_size);
    std::memcpy(rb.tokens.ptr, inputs, tau * B * S * 4);
    std::memcpy(rb.targets.ptr, targets, tau * B * S * 4);
    rb.finalize((int)c.cfg.vocab_size);
    c.begin_timing();
    c.upload(rb);
    c.d_f32b.reserve(e.P);
    c.h2d_f64_to_f32(theta_in, c.d_f32b.ptr, e.P);
    LocalResult r = c.local_round(*cfg, c.d_f32b.ptr, e.master, step_base);
    if (r.error) {
      Error ex(r.error, r.error == PHOTON_ERR_DIVERGENCE
                            ? "client " + std::to_string(client) + " diverged at round " +
                                  std::to_string(round) + ", step " + std::to_string(r.error_step)
                            : "gradient norm is not finite");
      ex.round = round;
      ex.client = client;
      ex.step = r.error_step;
      throw ex;
    }
    c.d2h_f32_to_f64(e.master, theta_out, e.P);
    c.end_timing();
    if (metrics)
      for (uint64_t i = 0; i < tau; ++i)
        metrics[i] = photon_step_metric{r.losses[i], B * S, 1.0 / cfg->throughput_bps};
  });
}

// ---- f64 aggregation / optimizer entry points --------------------------------------
namespace {
// Upload k host models into d_f64c [k][n]; pointer table into d_ptrs.
const double* const* stage_models(Ctx& c, const double* const* models, uint64_t k, uint64_t n) {
  need(k > 0, PHOTON_ERR_USAGE, "mean of zero param vectors");
  const uint64_t stride = (n + 1) / 2 * 2;  // 16-byte aligned rows for the vector path
  c.d_f64c.reserve(k * stride);
  std::vector<const void*> ptrs(k);
  for (uint64_t i = 0; i < k; ++i) {
    need(models[i] != nullptr, PHOTON_ERR_USAGE, "mean: null param vector");
    PH_CUDA(cudaMemcpyAsync(c.d_f64c.ptr + i * stride, models[i], n * 8, cudaMemcpyHostToDevice, c.stream));
    ptrs[i] = c.d_f64c.ptr + i * stride;
  }
  c.d_ptrs.reserve(k);
  PH_CUDA(cudaMemcpyAsync(c.d_ptrs.ptr, ptrs.data(), k * sizeof(void*), cudaMemcpyHostToDevice, c.stream));
  PH_CUDA(cudaStreamSynchronize(c.stream));  // ptrs vector goes out of scope
  return reinterpret_cast<const double* const*>(c.d_ptrs.ptr);
}
}  // namespace

int photon_mean(photon_ctx* ctx, const double* const* models, uint64_t k, uint64_t n, double* out,
                photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    auto ptrs = stage_models(c, models, k, n);
    c.d_f64a.reserve(n);
    c.begin_timing();
    k::mean_only<double>(ptrs, (int)k, n, c.d_f64a.ptr, c.stream);
    c.end_timing();
    PH_CUDA(cudaMemcpy(out, c.d_f64a.ptr, n * 8, cudaMemcpyDeviceToHost));
  });
}

int photon_sub(photon_ctx* ctx, const double* a, const double* b, uint64_t n, double* out,
               photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    c.d_f64a.reserve(n);
    c.d_f64b.reserve(n);
    PH_CUDA(cudaMemcpyAsync(c.d_f64a.ptr, a, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64b.ptr, b, n * 8, cudaMemcpyHostToDevice, c.stream));
    k::sub_only<double>(c.d_f64a.ptr, c.d_f64b.ptr, n, c.d_f64a.ptr, c.stream);
    PH_CUDA(cudaMemcpyAsync(out, c.d_f64a.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int photon_server_step(photon_ctx* ctx, const photon_server_cfg* cfg, const double* theta,
                       const double* delta, const double* mean, double* velocity, uint64_t n,
                       double* theta_out, photon_err* err) {
  return guarded(err, [&] {
    validate_server(*cfg);
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    c.d_f64a.reserve(n);
    c.d_f64b.reserve(n);
    c.d_f64c.reserve(n);
    c.d_f64d.reserve(2 * n);
    PH_CUDA(cudaMemcpyAsync(c.d_f64a.ptr, theta, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64b.ptr, delta, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64c.ptr, mean, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64d.ptr, velocity, n * 8, cudaMemcpyHostToDevice, c.stream));
    double* out = c.d_f64d.ptr + n;
    k::server_step_only<double>(c.d_f64a.ptr, c.d_f64b.ptr, c.d_f64c.ptr, c.d_f64d.ptr, out, n,
                                cfg->kind, cfg->eta, cfg->momentum, cfg->nesterov, c.stream);
    PH_CUDA(cudaMemcpyAsync(theta_out, out, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaMemcpyAsync(velocity, c.d_f64d.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int photon_aggregate(photon_ctx* ctx, const double* const* models, uint64_t k, uint64_t n,
                     const double* theta, double* velocity, const photon_server_cfg* cfg,
                     double* theta_out, photon_err* err) {
  return guarded(err, [&] {
    validate_server(*cfg);
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    auto ptrs = stage_models(c, models, k, n);
    c.d_f64a.reserve(n);
    c.d_f64b.reserve(n);
    PH_CUDA(cudaMemcpyAsync(c.d_f64a.ptr, theta, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64b.ptr, velocity, n * 8, cudaMemcpyHostToDevice, c.stream));
    c.begin_timing();
    k::aggregate<double>(ptrs, (int)k, n, c.d_f64a.ptr, c.d_f64b.ptr, cfg->kind, cfg->eta,
                         cfg->momentum, cfg->nesterov, c.stream);
    c.end_timing();
    PH_CUDA(cudaMemcpyAsync(theta_out, c.d_f64a.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaMemcpyAsync(velocity, c.d_f64b.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int photon_adamw_step(photon_ctx* ctx, double* params, const double* grads, double* m, double* v,
                      uint64_t n, uint64_t* step_count, const photon_adamw_cfg* cfg, double lr,
                      photon_err* err) {
  return guarded(err, [&] {
    need(cfg->beta1 >= 0.0 && cfg->beta1 < 1.0 && cfg->beta2 >= 0.0 && cfg->beta2 < 1.0,
         PHOTON_ERR_CONFIG, "adamw: betas must be in [0,1)");
    need(cfg->eps > 0.0, PHOTON_ERR_CONFIG, "adamw: eps must be > 0");
    need(lr >= 0.0 && std::isfinite(lr), PHOTON_ERR_CONFIG, "adamw: lr must be finite and >= 0");
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    c.d_f64a.reserve(n);
    c.d_f64b.reserve(n);
    c.d_f64c.reserve(n);
    c.d_f64d.reserve(n + 1);
    PH_CUDA(cudaMemcpyAsync(c.d_f64a.ptr, params, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64b.ptr, grads, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64c.ptr, m, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64d.ptr, v, n * 8, cudaMemcpyHostToDevice, c.stream));
    double* norm = c.d_f64d.ptr + n;
    k::sumsq_sequential_f64(c.d_f64b.ptr, n, norm, c.stream);
    double h_norm = 0.0;
    PH_CUDA(cudaMemcpyAsync(&h_norm, norm, 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
    need(std::isfinite(h_norm), PHOTON_ERR_NUMERIC, "gradient norm is not finite");
    *step_count += 1;
    const double sc = (double)*step_count;
    k::adamw_f64(c.d_f64a.ptr, c.d_f64b.ptr, c.d_f64c.ptr, c.d_f64d.ptr, n, norm, cfg->clip_norm,
                 lr, cfg->beta1, cfg->beta2, 1.0 - std::pow(cfg->beta1, sc),
                 1.0 - std::pow(cfg->beta2, sc), cfg->eps, cfg->weight_decay, c.stream);
    PH_CUDA(cudaMemcpyAsync(params, c.d_f64a.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaMemcpyAsync(m, c.d_f64c.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaMemcpyAsync(v, c.d_f64d.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int photon_sgd_step(photon_ctx* ctx, double* params, const double* grads, uint64_t n, double lr,
                    double clip, photon_err* err) {
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    c.d_f64a.reserve(n);
    c.d_f64b.reserve(n + 1);
    PH_CUDA(cudaMemcpyAsync(c.d_f64a.ptr, params, n * 8, cudaMemcpyHostToDevice, c.stream));
    PH_CUDA(cudaMemcpyAsync(c.d_f64b.ptr, grads, n * 8, cudaMemcpyHostToDevice, c.stream));
    double* norm = c.d_f64b.ptr + n;
    k::sumsq_sequential_f64(c.d_f64b.ptr, n, norm, c.stream);
    double h_norm = 0.0;
    PH_CUDA(cudaMemcpyAsync(&h_norm, norm, 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
    need(std::isfinite(h_norm), PHOTON_ERR_NUMERIC, "gradient norm is not finite");
    k::sgd_f64(c.d_f64a.ptr, c.d_f64b.ptr, n, norm, clip, lr, c.stream);
    PH_CUDA(cudaMemcpyAsync(params, c.d_f64a.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
    PH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int photon_aggregate_device_f32(photon_ctx* ctx, const float* const* d_models, uint64_t k,
                                uint64_t n, float* d_theta, float* d_velocity,
                                const photon_server_cfg* cfg, double* ms, photon_err* err) {
  return guarded(err, [&] {
    validate_server(*cfg);
    Ctx& c = ctx->c;
    PH_CUDA(cudaSetDevice(c.device));
    need(k > 0, PHOTON_ERR_USAGE, "mean of zero param vectors");
    for (uint64_t i = 0; i < k; ++i)
      need((reinterpret_cast<uintptr_t>(d_models[i]) & 15) == 0, PHOTON_ERR_USAGE,
           "aggregate_device_f32: model pointers must be 16-byte aligned");
    need((reinterpret_cast<uintptr_t>(d_theta) & 15) == 0 &&
             (reinterpret_cast<uintptr_t>(d_velocity) & 15) == 0,
         PHOTON_ERR_USAGE, "aggregate_device_f32: theta/velocity must be 16-byte aligned");
    c.d_ptrs.reserve(k);
    PH_CUDA(cudaMemcpyAsync(c.d_ptrs.ptr, d_models, k * sizeof(void*), cudaMemcpyHostToDevice, c.stream));
    c.begin_timing();
    k::aggregate<float>(reinterpret_cast<const float* const*>(c.d_ptrs.ptr), (int)k, n, d_theta,
                        d_velocity, cfg->kind, cfg->eta, cfg->momentum, cfg->nesterov, c.stream);
    const double t = c.end_timing();
    if (ms) *ms = t;
  });
}

// ---- test hooks ---------------------------------------------------------------------------
int photon_debug_gemm(int impl, int M, int N, int K, const void* A, int64_t lda, int a_kmajor,
                      const void* B, int64_t ldb, int b_kmajor, int ab_dtype, void* C,
                      int64_t ldc, int c_dtype, int epi, const float* bias, const float* resid,
                      void* aux, int iters, double* ms, photon_err* err) {
  return guarded(err, [&] {
    GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_kmajor = a_kmajor != 0;
    g.B = B; g.ldb = ldb; g.b_kmajor = b_kmajor != 0;
    g.ab = ab_dtype ? DT::BF16 : DT::F32;
    g.C = C; g.ldc = ldc; g.c = c_dtype ? DT::BF16 : DT::F32;
    g.epi = static_cast<Epi>(epi);
    g.bias = bias; g.resid = resid; g.aux = aux;
    if (const char* ns = std::getenv("PHOTON_DEBUG_NSEG")) {  // timing experiments: A/B repeated
      g.nseg = std::atoi(ns);
      for (int i = 1; i < g.nseg && i < 3; ++i) {
        g.A_seg[i] = A;
        g.B_seg[i] = B;
      }
    }
    cudaStream_t st;
    cudaEvent_t e0, e1;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the inputs come from other streams (torch's): complete them first
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    const int n = std::max(iters, 1);
    PH_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < n; ++i) {
      if (impl == 1) {
        if (!gemm_tc(g, st)) throw Error(PHOTON_ERR_CONFIG, "tcgen05 GEMM: unsupported arguments");
      } else {
        gemm_simt(g, st);
      }
    }
    PH_CUDA(cudaEventRecord(e1, st));
    PH_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PH_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t / n;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

int photon_debug_colsum(const void* x, int x_bf16, int M, int N, float* out, double* ms,
                        photon_err* err) {
  return guarded(err, [&] {
    need(x && out && M > 0 && N > 0, PHOTON_ERR_USAGE, "debug_colsum: bad arguments");
    DevBuf<float> part;
    part.reserve(std::max<size_t>(k::colsum_part_floats(M, N), 1));
    cudaStream_t st;
    cudaEvent_t e0, e1;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the inputs come from other streams (torch's): complete them first
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    PH_CUDA(cudaEventRecord(e0, st));
    if (x_bf16) k::colsum<bf16>(static_cast<const bf16*>(x), M, N, part.ptr, out, st);
    else k::colsum<float>(static_cast<const float*>(x), M, N, part.ptr, out, st);
    PH_CUDA(cudaEventRecord(e1, st));
    PH_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PH_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

// Cross-entropy forward+backward exactly as the engine runs it (tensor.cpp:544-603)
// plus the head-bias gradient (the column sums of dlogits, tensor.cpp:279-285)
// when dbias != NULL: accumulated inside the cross-entropy pass where the
// kernel supports the shape, else the column-sum pass over the written dlogits.
int photon_debug_ce(void* logits, int logits_bf16, const int32_t* targets, int M, int V,
                    float inv_count, double* rowloss, int write_grad, float* dbias, double* ms,
                    photon_err* err) {
  return guarded(err, [&] {
    need(logits && targets && rowloss && M > 0 && V > 1, PHOTON_ERR_USAGE,
         "debug_ce: bad arguments");
    DevBuf<float> part;
    part.reserve(std::max(k::colsum_part_floats(M, V), k::ce_bias_part_floats(V)));
    cudaStream_t st;
    cudaEvent_t e0, e1;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the inputs come from other streams (torch's): complete them first
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    PH_CUDA(cudaEventRecord(e0, st));
    if (logits_bf16) {
      auto* l = static_cast<bf16*>(logits);
      const bool fused = k::ce_fwd_bwd<bf16>(l, targets, M, V, inv_count, rowloss, write_grad != 0,
                                             st, write_grad ? dbias : nullptr, part.ptr);
      if (dbias && write_grad && !fused) k::colsum<bf16>(l, M, V, part.ptr, dbias, st);
    } else {
      auto* l = static_cast<float*>(logits);
      k::ce_fwd_bwd<float>(l, targets, M, V, inv_count, rowloss, write_grad != 0, st);
      if (dbias && write_grad) k::colsum<float>(l, M, V, part.ptr, dbias, st);
    }
    PH_CUDA(cudaEventRecord(e1, st));
    PH_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PH_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

// LayerNorm forward (and, with dy != NULL, backward) exactly as the engine runs
// them (tensor.cpp:322-394): y, dy and dxT in bf16 when y_bf16 else fp32; the backward
// writes dx = dres + LN'(dy) (dres may be NULL), its bf16/fp32 copy dxT, the
// gain / bias gradients and (dsum != NULL) the column sums of dx.
int photon_debug_layernorm(int y_bf16, int M, int d, const float* x, const float* gain,
                           const float* bias, void* y, float* mean, float* rstd, const void* dy,
                           const float* dres, float* dx, void* dxT, float* dgain, float* dbias,
                           float* dsum, double* ms, photon_err* err) {
  return guarded(err, [&] {
    need(x && gain && bias && y && mean && rstd && M > 0 && d > 0, PHOTON_ERR_USAGE,
         "debug_layernorm: bad arguments");
    need(!dy || (dx && dxT && dgain && dbias), PHOTON_ERR_USAGE,
         "debug_layernorm: backward needs dx, dxT, dgain, dbias");
    DevBuf<float> part;
    part.reserve((size_t)k::ln_bwd_parts() * 3 * d);
    cudaStream_t st;
    cudaEvent_t e0, e1;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the inputs come from other streams (torch's): complete them first
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    PH_CUDA(cudaEventRecord(e0, st));
    if (y_bf16) {
      k::ln_fwd<bf16>(x, gain, bias, static_cast<bf16*>(y), mean, rstd, M, d, st);
      if (dy)
        k::ln_bwd<bf16>(static_cast<const bf16*>(dy), x, mean, rstd, gain, dres, dx,
                        static_cast<bf16*>(dxT), part.ptr,
                        dgain, dbias, M, d, st, dsum);
    } else {
      k::ln_fwd<float>(x, gain, bias, static_cast<float*>(y), mean, rstd, M, d, st);
      if (dy)
        k::ln_bwd<float>(static_cast<const float*>(dy), x, mean, rstd, gain, dres, dx,
                         static_cast<float*>(dxT), part.ptr,
                         dgain, dbias, M, d, st, dsum);
    }
    PH_CUDA(cudaEventRecord(e1, st));
    PH_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PH_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

int photon_debug_attention(int impl, int B, int S, int H, int d, const void* q, const void* k,
                           const void* v, void* o, float* lse, const void* dO, float* scratch,
                           void* dq, void* dk, void* dv, double* ms, photon_err* err) {
  return guarded(err, [&] {
    cudaStream_t st;
    cudaEvent_t e0, e1;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the inputs come from other streams (torch's): complete them first
    PH_CUDA(cudaDeviceSynchronize());
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    auto Q = static_cast<const bf16*>(q), K = static_cast<const bf16*>(k),
         Vv = static_cast<const bf16*>(v);
    PH_CUDA(cudaEventRecord(e0, st));
    if (!dO) {
      if (impl == 2) k::attn_fwd_tc(Q, K, Vv, static_cast<bf16*>(o), lse, B, S, H, d, st);
      else if (impl == 1) k::attn_fwd_mma(Q, K, Vv, static_cast<bf16*>(o), lse, B, S, H, d, st);
      else k::attn_fwd_simt<bf16>(Q, K, Vv, static_cast<bf16*>(o), lse, B, S, H, d, st);
    } else {
      auto O = static_cast<const bf16*>(o), DO = static_cast<const bf16*>(dO);
      if (impl == 2)
        k::attn_bwd_tc(Q, K, Vv, O, DO, lse, static_cast<bf16*>(dq), static_cast<bf16*>(dk),
                       static_cast<bf16*>(dv), B, S, H, d, nullptr, st);
      else if (impl == 1)
        k::attn_bwd_mma(Q, K, Vv, O, DO, lse, scratch, static_cast<bf16*>(dq),
                        static_cast<bf16*>(dk), static_cast<bf16*>(dv), B, S, H, d, st);
      else
        k::attn_bwd_simt<bf16>(Q, K, Vv, O, DO, lse, scratch, static_cast<bf16*>(dq),
                               static_cast<bf16*>(dk), static_cast<bf16*>(dv), B, S, H, d, st);
    }
    PH_CUDA(cudaEventRecord(e1, st));
    PH_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PH_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

int photon_ctx_set_timing(photon_ctx* ctx, int on) {
  ctx->c.eng->timing = on != 0;
  ctx->c.eng->times = KernelTimes{};
  return PHOTON_OK;
}

uint64_t photon_launch_count(void) { return launch_counter().load(); }

int photon_ctx_kernel_times(photon_ctx* ctx, double* t) {
  const KernelTimes& k = ctx->c.eng->times;
  t[0] = k.gemm_ms;
  t[1] = k.attn_ms;
  t[2] = k.other_ms + k.optim_ms;
  t[3] = k.gemm_flops;
  t[4] = k.attn_flops;
  t[5] = k.gemm_launches;
  t[6] = k.attn_launches;
  t[7] = k.launches;
  return PHOTON_OK;
}

// ---- the boundary plan (host.hpp) ----------------------------------------------------------
uint64_t photon_shard_len(uint64_t n_params, int world) {
  return world >= 1 ? shard_len(n_params, world) : 0;
}
int photon_slot_owner(uint64_t slot, int world) { return world >= 1 ? slot_owner(slot, world) : -1; }
int photon_boundary_peer(uint64_t n_params, uint64_t k, uint64_t n_survivors, int world) {
  if (world <= 1) return 0;
  return boundary_prefers_peer(shard_len(n_params, world) * (uint64_t)world * 4) &&
                 peer_round_ok(n_survivors, k, world)
             ? 1
             : 0;
}

// ---- runner ------------------------------------------------------------------------------
int photon_nccl_unique_id(uint8_t* out, photon_err* err) {
  return guarded(err, [&] {
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) throw Error(PHOTON_ERR_NCCL, "ncclGetUniqueId failed");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, 128);
  });
}

int photon_runner_create(photon_ctx* ctx, const photon_fed_cfg* fed, const photon_train_cfg* train,
                         const photon_server_cfg* server, const photon_plan* plan,
                         const double* theta0, int rank, int world, const uint8_t* nccl_id,
                         photon_runner** out, photon_err* err) {
  return guarded(err, [&] {
    need(plan != nullptr, PHOTON_ERR_USAGE, "runner: null shard plan");
    auto r = std::make_unique<Runner>(&ctx->c, *fed, *train, *server, &plan->p, theta0, rank,
                                      world, nccl_id);
    *out = new photon_runner{std::move(r)};
  });
}

void photon_runner_destroy(photon_runner* r) { delete r; }

int photon_runner_add_dropout(photon_runner* r, uint64_t round, uint64_t client) {
  r->r->dropouts.insert({round, client});
  return PHOTON_OK;
}

int photon_runner_run_round(photon_runner* r, photon_round_record* rec, photon_err* err) {
  return guarded(err, [&] { r->r->run_round(rec); });
}

uint64_t photon_runner_next_round(const photon_runner* r) { return r->r->next_round; }

int photon_runner_theta(photon_runner* r, double* out, photon_err* err) {
  return guarded(err, [&] { r->r->theta_f64(out); });
}

int photon_runner_velocity(photon_runner* r, double* out, photon_err* err) {
  return guarded(err, [&] { r->r->velocity_f64(out); });
}

uint64_t photon_runner_cursor(const photon_runner* r, uint64_t client) {
  return client < r->r->cursors.size() ? r->r->cursors[client] : 0;
}

int photon_runner_restore(photon_runner* r, const double* theta, const double* velocity,
                          uint64_t next_round, const uint64_t* cursors, uint64_t n,
                          photon_err* err) {
  return guarded(err, [&] { r->r->restore(theta, velocity, next_round, cursors, n); });
}

int photon_debug_boundary(int device, uint64_t n_params, int rank, int world,
                          const uint8_t* nccl_id, const photon_server_cfg* server, int iters,
                          double* ms_out, photon_err* err) {
  return guarded(err, [&] {
    need(world >= 1 && rank >= 0 && rank < world && n_params > 0 && iters > 0, PHOTON_ERR_USAGE,
         "debug_boundary: bad arguments");
    need(world == 1 || nccl_id != nullptr, PHOTON_ERR_USAGE, "debug_boundary: needs an NCCL id");
    validate_server(*server);
    PH_CUDA(cudaSetDevice(device));
    const uint64_t P = n_params;
    const uint64_t shard = shard_len(P, world), Ppad = shard * world;
    cudaStream_t st;
    PH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DevBuf<float> theta, vel, model, recv;
    DevBuf<const float*> ptrs;
    theta.reserve(Ppad);
    vel.reserve(world > 1 ? shard : Ppad);
    model.reserve(Ppad);
    if (world > 1 && !use_peer_boundary(Ppad * 4)) recv.reserve((size_t)world * shard);
    PH_CUDA(cudaMemsetAsync(theta.ptr, 0, Ppad * 4, st));
    PH_CUDA(cudaMemsetAsync(vel.ptr, 0, vel.n * 4, st));
    PH_CUDA(cudaMemsetAsync(model.ptr, 0, Ppad * 4, st));
    ncclComm_t comm = nullptr;
    if (world > 1) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      if (nccl().CommInitRank(&comm, world, id, rank) != ncclSuccess)
        throw Error(PHOTON_ERR_NCCL, "debug_boundary: ncclCommInitRank failed");
    }
    std::vector<int> surv(world);
    for (int s = 0; s < world; ++s) surv[s] = s;  // one client per rank
    const float* local[1] = {model.ptr};
    cudaEvent_t e0, e1;
    PH_CUDA(cudaEventCreate(&e0));
    PH_CUDA(cudaEventCreate(&e1));
    std::unique_ptr<PeerBoundary> p2p;
    try {
      if (world > 1 && use_peer_boundary(Ppad * 4)) {
        p2p = std::make_unique<PeerBoundary>(comm, rank, world, device);
        p2p->publish(local, 1, theta.ptr, st);
      }
      auto once = [&] {
        if (p2p) p2p->run(surv, shard, vel.ptr, *server, st);
        else round_boundary(comm, rank, world, P, shard, surv, local, recv.ptr, ptrs, theta.ptr,
                            vel.ptr, *server, st);
      };
      for (int i = 0; i < 2; ++i) once();  // warm-up (connection setup)
      PH_CUDA(cudaEventRecord(e0, st));
      for (int i = 0; i < iters; ++i) once();
      PH_CUDA(cudaEventRecord(e1, st));
      PH_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      PH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      *ms_out = ms / iters;
      p2p.reset();
    } catch (...) {
      p2p.reset();
      if (comm) nccl().CommDestroy(comm);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaStreamDestroy(st);
      throw;
    }
    if (comm) nccl().CommDestroy(comm);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PH_CUDA(cudaStreamDestroy(st));
  });
}

int photon_central_create(photon_ctx* ctx, const photon_central_cfg* cfg, const photon_plan* plan,
                          uint64_t seed, const double* theta0, int rank, int world,
                          const uint8_t* nccl_id, photon_central** out, photon_err* err) {
  return guarded(err, [&] {
    need(ctx && cfg && out && theta0, PHOTON_ERR_USAGE, "central_create: null argument");
    PH_CUDA(cudaSetDevice(ctx->c.device));
    auto h = std::make_unique<photon_central>();
    h->c = std::make_unique<Central>(&ctx->c, *cfg, plan ? &plan->p : nullptr, seed, theta0, rank,
                                     world, nccl_id);
    *out = h.release();
  });
}

void photon_central_destroy(photon_central* c) { delete c; }

int photon_central_step(photon_central* c, photon_step_metric* metric, photon_err* err) {
  return guarded(err, [&] { c->c->step(metric); });
}

uint64_t photon_central_next_step(const photon_central* c) { return c->c->t; }

uint64_t photon_central_cursor(const photon_central* c, uint64_t worker) {
  return worker < c->c->cursors.size() ? c->c->cursors[worker] : 0;
}

int photon_central_theta(photon_central* c, double* out, photon_err* err) {
  return guarded(err, [&] { c->c->theta_f64(out); });
}

int photon_eval_set_create(const char* const* styles, uint64_t n_styles, uint64_t eval_sequences,
                           uint64_t data_seed, uint64_t vocab, uint64_t seq_len,
                           uint64_t eval_batch, photon_eval_set** out, photon_err* err) {
  return guarded(err, [&] {
    need(out != nullptr && (styles != nullptr || n_styles == 0), PHOTON_ERR_USAGE,
         "eval_set_create: null argument");
    std::vector<std::string> st;
    for (uint64_t i = 0; i < n_styles; ++i) st.emplace_back(styles[i]);
    auto es = std::make_unique<photon_eval_set>();
    es->s = build_eval_set(st, eval_sequences, data_seed, vocab, seq_len, eval_batch);
    *out = es.release();
  });
}

void photon_eval_set_destroy(photon_eval_set* s) { delete s; }

uint64_t photon_eval_set_batches(const photon_eval_set* s) { return s ? s->s.batch_sizes.size() : 0; }

int photon_eval_set_batch(const photon_eval_set* s, uint64_t i, const int32_t** inputs,
                          const int32_t** targets, uint64_t* batch_size, photon_err* err) {
  return guarded(err, [&] {
    need(s != nullptr && i < s->s.batch_sizes.size(), PHOTON_ERR_INDEX, "eval_set_batch: index");
    uint64_t row = 0;
    for (uint64_t b = 0; b < i; ++b) row += s->s.batch_sizes[b];
    *inputs = s->s.inputs.data() + row * s->s.seq_len;
    *targets = s->s.targets.data() + row * s->s.seq_len;
    *batch_size = s->s.batch_sizes[i];
  });
}

int photon_runner_set_eval(photon_runner* r, const photon_eval_set* s, uint64_t eval_every,
                           photon_err* err) {
  return guarded(err, [&] {
    need(s != nullptr, PHOTON_ERR_USAGE, "runner_set_eval: null eval set");
    r->r->set_eval(s->s, eval_every);
  });
}

int photon_runner_eval(photon_runner* r, double* ppl, photon_err* err) {
  return guarded(err, [&] {
    *ppl = r->r->eval_theta();
    r->r->initial_ppl = r->r->next_round == 0 ? *ppl : r->r->initial_ppl;
  });
}

uint64_t photon_crc64(const void* data, uint64_t len) { return crc64(data, len); }

int photon_checkpoint_write(const char* path, const photon_model_cfg* m, const double* params,
                            uint64_t round, photon_err* err) {
  return guarded(err, [&] {
    validate_model(*m);
    write_phck(path, *m, params, round);
  });
}

int photon_checkpoint_read(const char* path, const photon_model_cfg* m, double* params,
                           uint64_t* round, photon_err* err) {
  return guarded(err, [&] {
    validate_model(*m);
    const uint64_t rd = read_phck(path, *m, params);
    if (round) *round = rd;
  });
}

int photon_runner_save(photon_runner* r, const char* dir, photon_err* err) {
  return guarded(err, [&] { r->r->save(dir); });
}

int photon_runner_resume(photon_runner* r, const char* dir, photon_err* err) {
  return guarded(err, [&] { r->r->resume(dir); });
}

}  // extern "C"
