/*
 * photon.h -- C ABI of the B200-native Photon federated-round path.
 *
 * Drop-in boundary for the reference library `fedsim::core`
 * (/root/reference/proj/core).  Every entry point names the reference
 * interface it replaces (file:line).  Plain pointers and sizes only: host
 * buffers are f64 in the reference's canonical flat parameter order
 * (ParamVector::flatten, param_vector.cpp:154-159); device state is owned by
 * opaque handles.  Errors: every call returns a photon status code and fills
 * an optional photon_err; codes map 1:1 onto fedsim/errors.h:9-72, so an
 * adapter can rethrow the matching fedsim:: exception.
 */
#ifndef PHOTON_H
#define PHOTON_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHOTON_ABI_VERSION 2

/* status codes (fedsim/errors.h) */
enum {
  PHOTON_OK = 0,
  PHOTON_ERR_CONFIG = 1,        /* ConfigError */
  PHOTON_ERR_CAPACITY = 2,      /* CapacityError */
  PHOTON_ERR_SHAPE = 3,         /* ShapeError */
  PHOTON_ERR_INDEX = 4,         /* IndexError */
  PHOTON_ERR_USAGE = 5,         /* UsageError */
  PHOTON_ERR_LOOKUP = 6,        /* LookupError */
  PHOTON_ERR_NUMERIC = 7,       /* NumericError */
  PHOTON_ERR_DIVERGENCE = 8,    /* DivergenceError{round,client,step} */
  PHOTON_ERR_IO = 9,            /* IoError */
  PHOTON_ERR_INTEGRITY = 10,    /* IntegrityError */
  PHOTON_ERR_ROUND_FAILURE = 11,/* RoundFailureError */
  PHOTON_ERR_PARSE = 12,        /* ParseError */
  PHOTON_ERR_CUDA = 20,         /* device failure (no reference equivalent) */
  PHOTON_ERR_NCCL = 21
};

/* arithmetic of the client step */
enum {
  PHOTON_PREC_F32 = 0,  /* fp32 storage + fp32 SIMT contractions (parity mode) */
  PHOTON_PREC_BF16 = 1  /* fp32 master/moments, bf16 operands on tcgen05, fp32 accumulate */
};

typedef struct {
  int32_t code;
  uint64_t round, client, step; /* DivergenceError fields (errors.h:45-52) */
  char msg[256];
} photon_err;

/* ModelConfig, model.h:12-25 */
typedef struct {
  uint64_t n_blocks, d_model, n_heads, expansion_ratio, vocab_size, seq_len;
} photon_model_cfg;

/* LrSchedule, optim.h:13-21 */
typedef struct {
  double eta_max;
  uint64_t warmup_steps, decay_steps;
  double alpha;
} photon_lr_schedule;

/* AdamWConfig, optim.h:25-33 */
typedef struct {
  double beta1, beta2, eps, weight_decay, clip_norm;
} photon_adamw_cfg;

/* LocalTrainConfig, client.h:66-76 (+ PostProcessPolicy client.h:58-62) */
typedef struct {
  photon_model_cfg model;
  photon_adamw_cfg adamw;
  photon_lr_schedule schedule;
  int32_t opt;            /* 0 AdamW, 1 SGD (ClientOptKind) */
  double sgd_clip_norm;
  uint64_t local_steps;   /* tau */
  uint64_t batch_size;    /* B */
  double throughput_bps;  /* nu (simulated seconds per step = 1/nu) */
  int32_t post_kind;      /* 0 identity, 1 clip update norm */
  double post_threshold;
} photon_train_cfg;

/* ServerOptConfig, optim.h:54-63 */
typedef struct {
  int32_t kind;           /* 0 FedAvg, 1 FedMomentum */
  double eta, momentum;
  int32_t nesterov;
} photon_server_cfg;

/* FederationConfig, aggregator.h:18-26 */
typedef struct {
  uint64_t population;        /* P */
  uint64_t clients_per_round; /* K */
  uint64_t rounds;            /* T */
  int32_t topology;           /* 0 ps, 1 ar, 2 rar (cost_model.h Topology) */
  uint64_t seed;
} photon_fed_cfg;

/* StepMetric, client.h:78-82 */
typedef struct {
  double loss;
  uint64_t tokens;
  double sim_seconds;
} photon_step_metric;

/* RoundRecord, aggregator.h:38-53 (simulated-cost fields omitted: cost model is
 * out of scope) + measured device time of the round on this rank. */
typedef struct {
  uint64_t round;
  uint64_t n_sampled;
  uint64_t sampled_ids[64];   /* first min(K,64) sampled ids, ascending */
  double mean_client_loss, min_client_loss, max_client_loss;
  double local_ms;            /* device time: first client step -> last client step */
  double aggregate_ms;        /* device time: exchange + fused mean/outer update + gather */
  double round_ms;            /* device time of the whole round on this rank */
  uint64_t tokens;            /* tokens trained on this rank this round */
  double host_ms;             /* host batch staging (BatchStream x tau) + H2D issue */
  uint64_t h2d_bytes;         /* inputs copied host->device this round on this rank */
  uint64_t d2h_bytes;         /* results read back device->host this round */
  double eval_ppl;            /* RoundRecord::eval_ppl: perplexity of theta_{t+1} on the
                                 held-out set when the eval cadence fires, else NaN */
  double boundary_ms;         /* device ms of the boundary's data movement + update alone
                                 (peer-memory path: the fused kernel, after the slowest
                                 rank arrived; NCCL path / one GPU: the whole boundary) */
} photon_round_record;

typedef struct photon_ctx photon_ctx;       /* one GPU: device state of one client slot */
typedef struct photon_plan photon_plan;     /* ShardPlan (data.h:33-62), host */
typedef struct photon_runner photon_runner; /* FederationRunner (aggregator.h:70-102) */
typedef struct photon_eval_set photon_eval_set; /* held-out batches (harness.cpp:440-472) */
typedef struct photon_central photon_central;   /* run_centralized (baselines.cpp:25-127) */

/* CentralizedConfig, baselines.h:19-35 */
typedef struct {
  photon_model_cfg model;
  photon_adamw_cfg adamw;
  photon_lr_schedule schedule;
  int32_t opt;                 /* 0 AdamW, 1 SGD */
  double sgd_clip_norm;
  uint64_t n_workers;
  uint64_t global_batch;       /* divisible by n_workers */
  uint64_t total_steps;
  uint64_t opt_reset_interval; /* fresh AdamW state every N steps, 0 = never */
  double throughput_bps;
} photon_central_cfg;

int photon_abi_version(void);
const char* photon_status_name(int code);

/* ---- host: determinism primitives (bit-exact ports) ------------------------ */
uint64_t photon_mix64(uint64_t x);                                 /* rng.h:14-19 */
uint64_t photon_stream_seed(uint64_t global_seed, uint64_t client); /* data.cpp:201-203 */
int photon_sample_clients(uint64_t population, uint64_t k, uint64_t seed, uint64_t round,
                          uint64_t* out_ids, photon_err* err);     /* aggregator.cpp:25-41 */
int photon_lr_at(const photon_lr_schedule* s, uint64_t step, double* out,
                 photon_err* err);                                 /* optim.cpp:16-27 */

/* ---- host: model layout + init ---------------------------------------------- */
uint64_t photon_param_count(const photon_model_cfg* m);            /* model.cpp:21-26 */
uint64_t photon_layout_size(const photon_model_cfg* m);            /* model.cpp:32-61 */
int photon_layout_entry(const photon_model_cfg* m, uint64_t i, uint64_t* offset,
                        uint64_t* rows, uint64_t* cols, char* name, int name_cap);
int photon_init_params(const photon_model_cfg* m, uint64_t seed, double* out,
                       photon_err* err);                           /* model.cpp:72-96 */

/* ---- host: data (data.cpp) ---------------------------------------------------- */
int photon_generate_corpus(const char* style, uint64_t length, uint64_t seed, uint32_t vocab,
                           uint16_t* out, photon_err* err);        /* data.cpp:44-71 */
int photon_plan_iid(const uint16_t* tokens, uint64_t n_tokens, uint64_t n_shards,
                    uint64_t seq_len, uint64_t seed, photon_plan** out,
                    photon_err* err);                              /* data.cpp:137-164 */
int photon_plan_by_source(const uint16_t* const* corpora, const uint64_t* lens,
                          uint64_t n_sources, uint64_t clients_per_source, uint64_t seq_len,
                          photon_plan** out, photon_err* err);     /* data.cpp:166-199 */
/* ShardPlan import (data.h:33-62): an existing plan's corpora and per-client
 * block lists -- e.g. a fedsim::ShardPlan handed over by the C++ adapter.
 * Client c owns n_blocks[c] blocks of seq_len + 1 tokens; its i-th block is
 * (sources[j], offsets[j]) with j = n_blocks[0] + ... + n_blocks[c-1] + i. */
int photon_plan_from_blocks(const uint16_t* const* corpora, const uint64_t* lens,
                            uint64_t n_sources, uint64_t seq_len, const uint64_t* n_blocks,
                            uint64_t n_clients, const uint32_t* sources, const uint64_t* offsets,
                            photon_plan** out, photon_err* err);
void photon_plan_free(photon_plan* p);
uint64_t photon_plan_n_clients(const photon_plan* p);
uint64_t photon_plan_client_blocks(const photon_plan* p, uint64_t client);
/* BatchStream::next, data.cpp:231-253: batch rows from cursor; advances cursor */
int photon_stream_next(const photon_plan* p, uint64_t client, uint64_t batch_size,
                       uint64_t seed, uint64_t* cursor, int32_t* inputs, int32_t* targets,
                       photon_err* err);

/* ---- device context ------------------------------------------------------------ */
/* One GPU's client engine for `model` at `precision`, activations sized for
 * max_batch rows of model->seq_len tokens.  A larger batch (a client's local
 * batch, an eval batch) runs as micro-batches of max_batch rows whose
 * gradients and losses accumulate into the step's (the loss stays the mean
 * over all of the batch's targets, client.cpp:135-154). */
int photon_ctx_create(int device, const photon_model_cfg* model, int precision,
                      uint64_t max_batch, photon_ctx** out, photon_err* err);
void photon_ctx_destroy(photon_ctx* ctx);
/* ms of device time of the last call that ran kernels on this ctx */
double photon_ctx_last_ms(const photon_ctx* ctx);

/* TransformerModel::forward_loss + backward + collect_grads (model.cpp:98-174):
 * params/grads f64 host, canonical order; grads may be NULL (forward only). */
int photon_forward_backward(photon_ctx* ctx, const double* params, const int32_t* inputs,
                            const int32_t* targets, uint64_t batch, uint64_t seq,
                            double* loss, double* grads, photon_err* err);

/* eval_perplexity (model.cpp:176-192): n_batches batches of batch_sizes[i] rows */
int photon_eval_perplexity(photon_ctx* ctx, const double* params, const int32_t* inputs,
                           const int32_t* targets, uint64_t n_batches,
                           const uint64_t* batch_sizes, uint64_t seq, double* ppl,
                           photon_err* err);

/* run_local_round (client.cpp:125-158 / client.h:97-99): tau local steps from
 * theta_in with fresh optimizer state; inputs/targets hold the tau batches the
 * client's BatchStream yields ([tau][B][S] int32, from photon_stream_next).
 * Non-finite loss -> PHOTON_ERR_DIVERGENCE with (round, client, step). */
int photon_client_round(photon_ctx* ctx, const photon_train_cfg* cfg, const double* theta_in,
                        const int32_t* inputs, const int32_t* targets, uint64_t round,
                        uint64_t client, uint64_t step_base, double* theta_out,
                        photon_step_metric* metrics, photon_err* err);

/* ---- aggregation + outer optimizer, f64, bit-exact vs the reference ------------- */
/* ParamVector::mean (param_vector.cpp:127-152), anchored, ascending order */
int photon_mean(photon_ctx* ctx, const double* const* models, uint64_t k, uint64_t n,
                double* out, photon_err* err);
/* ParamVector::sub (param_vector.cpp:120-125) */
int photon_sub(photon_ctx* ctx, const double* a, const double* b, uint64_t n, double* out,
               photon_err* err);
/* server_step (optim.cpp:124-159); velocity updated in place */
int photon_server_step(photon_ctx* ctx, const photon_server_cfg* cfg, const double* theta,
                       const double* delta, const double* mean, double* velocity, uint64_t n,
                       double* theta_out, photon_err* err);
/* fused mean -> pseudo-gradient -> outer step (aggregator.cpp:177-179) */
int photon_aggregate(photon_ctx* ctx, const double* const* models, uint64_t k, uint64_t n,
                     const double* theta, double* velocity, const photon_server_cfg* cfg,
                     double* theta_out, photon_err* err);
/* adamw_step / sgd_step (optim.cpp:61-103) on f64 host buffers, bit-exact */
int photon_adamw_step(photon_ctx* ctx, double* params, const double* grads, double* m,
                      double* v, uint64_t n, uint64_t* step_count,
                      const photon_adamw_cfg* cfg, double lr, photon_err* err);
int photon_sgd_step(photon_ctx* ctx, double* params, const double* grads, uint64_t n,
                    double lr, double clip_norm, photon_err* err);

/* fp32 device-resident fused aggregation over device pointers (the fast path):
 * models[k] -> theta (in/out) and velocity (in/out); returns device ms. */
int photon_aggregate_device_f32(photon_ctx* ctx, const float* const* d_models, uint64_t k,
                                uint64_t n, float* d_theta, float* d_velocity,
                                const photon_server_cfg* cfg, double* ms, photon_err* err);

/* ---- test / benchmark hooks ------------------------------------------------------- */
/* One contraction of the client step on device pointers: impl 0 = SIMT,
 * 1 = tcgen05; dtypes 0 f32 / 1 bf16; epi as gemm.cuh (0 store, 1 accum,
 * 2 bias, 3 resid+bias, 4 gelu+bias, 5 gelu backward).  Runs `iters` times
 * on an internal stream; *ms = mean device time per launch. */
int photon_debug_gemm(int impl, int M, int N, int K, const void* A, int64_t lda, int a_kmajor,
                      const void* B, int64_t ldb, int b_kmajor, int ab_dtype, void* C,
                      int64_t ldc, int c_dtype, int epi, const float* bias, const float* resid,
                      void* aux, int iters, double* ms, photon_err* err);

/* Bias-gradient column sums out[N] = sum_i x[i][:] of a device matrix x [M, N]
 * (bf16 when x_bf16, else fp32), as the engine computes them (add_bias
 * backward, tensor.cpp:279-285).  *ms = device time of the call. */
int photon_debug_colsum(const void* x, int x_bf16, int M, int N, float* out, double* ms,
                        photon_err* err);

/* Softmax cross-entropy forward + backward on a device logits matrix [M, V]
 * (bf16 when logits_bf16, else fp32), as the engine runs it
 * (tensor.cpp:544-603): rowloss[M] (f64) = logsumexp - logit[target]; with
 * write_grad the logits are overwritten by (softmax - onehot) * inv_count and,
 * when dbias != NULL, dbias[V] receives their column sums (the head-bias
 * gradient, tensor.cpp:279-285) exactly as the engine produces them.  *ms =
 * device time of the call. */
int photon_debug_ce(void* logits, int logits_bf16, const int32_t* targets, int M, int V,
                    float inv_count, double* rowloss, int write_grad, float* dbias, double* ms,
                    photon_err* err);

/* LayerNorm forward (+ backward when dy != NULL) on device pointers, as the
 * engine runs them (tensor.cpp:322-394): x, gain, bias, dres fp32; y, dy and
 * dxT bf16 when y_bf16 else fp32; mean / rstd fp32 [M]; dx = dres + LN'(dy);
 * dgain / dbias [d]; dsum (optional) = column sums of dx. */
int photon_debug_layernorm(int y_bf16, int M, int d, const float* x, const float* gain,
                           const float* bias, void* y, float* mean, float* rstd, const void* dy,
                           const float* dres, float* dx, void* dxT, float* dgain, float* dbias,
                           float* dsum, double* ms, photon_err* err);

/* Causal attention on device pointers (bf16 q,k,v,o,dO,dq,dk,dv as [B*S, d]
 * with head h in columns [h*dh,(h+1)*dh); lse, scratch fp32 [B*H*S]):
 * impl 0 = SIMT, 1 = mma.sync tensor core, 2 = tcgen05 (dh = 64 or 128).
 * dO == NULL: forward only.  *ms = device
 * time of the call. */
int photon_debug_attention(int impl, int B, int S, int H, int d, const void* q, const void* k,
                           const void* v, void* o, float* lse, const void* dO, float* scratch,
                           void* dq, void* dk, void* dv, double* ms, photon_err* err);

/* Per-kernel-class device timing of the client step (CUDA events around each
 * launch; adds overhead, for profiling rounds only).  times[8] = {gemm_ms,
 * attn_ms, other_ms, gemm_flops, attn_flops, gemm_launches, attn_launches,
 * launches}, accumulated since the last reset (set_timing resets). */
int photon_ctx_set_timing(photon_ctx* ctx, int on);
int photon_ctx_kernel_times(photon_ctx* ctx, double* times8);
/* Kernels this library has launched in this process (every launch site, plus
 * the kernel nodes of each CUDA-graph replay of a local round). */
uint64_t photon_launch_count(void);

/* ---- the multi-GPU round boundary's plan (host logic, no GPU) -------------------
 * What every rank of the runner derives identically: the flat parameter
 * vector is cut into `world` shards of photon_shard_len elements (a multiple
 * of 4; world * shard_len >= n_params); sampled slot si (ascending client ids;
 * worker w of the centralized baseline) trains on rank photon_slot_owner(si);
 * photon_boundary_peer says whether a round with n_survivors of k sampled
 * clients runs on the NVLink peer-memory kernel (1) or the NCCL send/recv +
 * all-gather path (0), honouring PHOTON_BOUNDARY.  The runner uses the same
 * functions; tests drive them over gloo. */
uint64_t photon_shard_len(uint64_t n_params, int world);
int photon_slot_owner(uint64_t slot, int world);
int photon_boundary_peer(uint64_t n_params, uint64_t k, uint64_t n_survivors, int world);

/* ---- federated round runner (FederationRunner, aggregator.h:70-102) ------------ */
/* Device-resident: theta_t, velocity and client state live in HBM.  With
 * world > 1 each rank runs the sampled clients with slot % world == rank and
 * the round boundary exchanges parameter shards over NCCL (nccl_id: 128-byte
 * ncclUniqueId from rank 0; NULL when world == 1). */
int photon_runner_create(photon_ctx* ctx, const photon_fed_cfg* fed,
                         const photon_train_cfg* train, const photon_server_cfg* server,
                         const photon_plan* plan, const double* theta0, int rank, int world,
                         const uint8_t* nccl_id, photon_runner** out, photon_err* err);
void photon_runner_destroy(photon_runner* r);
int photon_nccl_unique_id(uint8_t* out128, photon_err* err);
/* simulated dropouts (RunnerOptions::dropouts, aggregator.h:59-61) */
int photon_runner_add_dropout(photon_runner* r, uint64_t round, uint64_t client);
int photon_runner_run_round(photon_runner* r, photon_round_record* rec, photon_err* err);
uint64_t photon_runner_next_round(const photon_runner* r);
int photon_runner_theta(photon_runner* r, double* out, photon_err* err);
int photon_runner_velocity(photon_runner* r, double* out, photon_err* err);
uint64_t photon_runner_cursor(const photon_runner* r, uint64_t client);
/* FederationRunner::restore (aggregator.cpp:78-91) */
int photon_runner_restore(photon_runner* r, const double* theta, const double* velocity,
                          uint64_t next_round, const uint64_t* cursors, uint64_t n_cursors,
                          photon_err* err);


/* Round boundary alone: n_params fp32 parameters, one
 * synthetic client model per rank, `iters` timed rounds of exchange -> fused
 * anchored-mean + outer update (server kind/eta/momentum) -> all-gather on
 * `device`.  *ms_out: mean device ms per boundary on this rank.  Collective
 * across `world` ranks (nccl_id from rank 0; NULL when world == 1). */
int photon_debug_boundary(int device, uint64_t n_params, int rank, int world,
                          const uint8_t* nccl_id, const photon_server_cfg* server, int iters,
                          double* ms_out, photon_err* err);

/* ---- centralized / DDP baseline (baselines.cpp:25-127) ---------
 * n_workers data-parallel workers (worker w: shard w, stream_seed(seed, w), on
 * rank w % world); per step: each worker's gradient, the ascending-worker
 * anchored mean (NCCL shard exchange + all-gather for world > 1), one shared
 * AdamW / SGD update.  Non-finite mean loss -> PHOTON_ERR_DIVERGENCE (step). */
int photon_central_create(photon_ctx* ctx, const photon_central_cfg* cfg, const photon_plan* plan,
                          uint64_t seed, const double* theta0, int rank, int world,
                          const uint8_t* nccl_id, photon_central** out, photon_err* err);
void photon_central_destroy(photon_central* c);
int photon_central_step(photon_central* c, photon_step_metric* metric, photon_err* err);
uint64_t photon_central_next_step(const photon_central* c);
uint64_t photon_central_cursor(const photon_central* c, uint64_t worker);
int photon_central_theta(photon_central* c, double* out, photon_err* err);

/* ---- evaluation and checkpoints -------------------------- */
/* build_eval_batches (harness.cpp:440-472): per style a held-out corpus from
 * mix_seed(data_seed, "Eval"), eval_sequences / n_styles sequences each, batches
 * of eval_batch rows (the last may be short).  Host only. */
int photon_eval_set_create(const char* const* styles, uint64_t n_styles, uint64_t eval_sequences,
                           uint64_t data_seed, uint64_t vocab, uint64_t seq_len,
                           uint64_t eval_batch, photon_eval_set** out, photon_err* err);
void photon_eval_set_destroy(photon_eval_set* s);
uint64_t photon_eval_set_batches(const photon_eval_set* s);
int photon_eval_set_batch(const photon_eval_set* s, uint64_t i, const int32_t** inputs,
                          const int32_t** targets, uint64_t* batch_size, photon_err* err);
/* RunnerOptions::eval_every + eval_fn (aggregator.cpp:207-212): theta_{t+1} is
 * evaluated after round t when t % every == every - 1 or t is the last round;
 * the eval batches stay resident in HBM (batch i on rank i % world). */
int photon_runner_set_eval(photon_runner* r, const photon_eval_set* s, uint64_t eval_every,
                           photon_err* err);
/* eval_fn(theta) now (e.g. the initial perplexity); collective for world > 1 */
int photon_runner_eval(photon_runner* r, double* ppl, photon_err* err);

/* PHCK snapshot (checkpoint.h:17-45): byte-identical to the reference writer.
 * Integrity failures -> PHOTON_ERR_INTEGRITY, layout mismatch -> PHOTON_ERR_SHAPE. */
uint64_t photon_crc64(const void* data, uint64_t len); /* CRC-64/XZ, checkpoint.h:14-16 */
int photon_checkpoint_write(const char* path, const photon_model_cfg* m, const double* params,
                            uint64_t round, photon_err* err);
int photon_checkpoint_read(const char* path, const photon_model_cfg* m, double* params,
                           uint64_t* round, photon_err* err);
/* Resume directory (harness.cpp:802-905): checkpoint.phck (theta, round = next
 * round), velocity.phck (momentum server), state.json (next_round, cursors,
 * initial_ppl, sync_events).  Collective for world > 1; rank 0 writes. */
int photon_runner_save(photon_runner* r, const char* dir, photon_err* err);
int photon_runner_resume(photon_runner* r, const char* dir, photon_err* err);

#ifdef __cplusplus
}
#endif
#endif
