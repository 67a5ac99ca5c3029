/*
 * fedsim_oracle.h -- CPU restatement of the reference's federated-round path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity oracle: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker (or the timed CPU baseline).  The
 * product (paper_2411_02908_b200/) never links or calls it.
 *
 * Every function restates, in plain C99 with the reference's loop order and
 * left-to-right f64 summation (built with -ffp-contract=off, no FMA), the
 * function cited next to it in /root/reference/proj/core.  It is pinned
 * bit-for-bit against the reference compiled from its own sources
 * (oracle/_ref, see oracle/Makefile) and against the golden vectors of the
 * reference's unit tests (tests/test_oracle_golden.py).
 */
#ifndef FEDSIM_ORACLE_H
#define FEDSIM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes mirror fedsim/errors.h:9-72 */
enum {
  ORC_OK = 0,
  ORC_CONFIG = 1,
  ORC_CAPACITY = 2,
  ORC_SHAPE = 3,
  ORC_INDEX = 4,
  ORC_USAGE = 5,
  ORC_LOOKUP = 6,
  ORC_NUMERIC = 7,
  ORC_DIVERGENCE = 8,
  ORC_ROUND_FAILURE = 11
};

/* ModelConfig, model.h:12-25 */
typedef struct {
  uint64_t n_blocks, d_model, n_heads, expansion_ratio, vocab_size, seq_len;
} orc_model_cfg;

/* LrSchedule optim.h:13-21 + AdamWConfig optim.h:25-33 + LocalTrainConfig client.h:66-76 */
typedef struct {
  double eta_max;
  uint64_t warmup_steps, decay_steps;
  double alpha;
  double beta1, beta2, eps, weight_decay, clip_norm;
  int32_t opt;            /* 0 = AdamW, 1 = SGD (ClientOptKind) */
  double sgd_clip_norm;
  uint64_t local_steps, batch_size;
  int32_t post_kind;      /* 0 identity, 1 clip update norm (client.h:58-62) */
  double post_threshold;
} orc_train_cfg;

/* ServerOptConfig optim.h:54-63 */
typedef struct {
  int32_t kind;           /* 0 FedAvg, 1 FedMomentum */
  double eta, momentum;
  int32_t nesterov;
} orc_server_cfg;

/* --- rng.h:14-84 --------------------------------------------------------- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_mix_seed(uint64_t seed, uint64_t a);
uint64_t orc_mix_seed2(uint64_t seed, uint64_t a, uint64_t b);
uint64_t orc_mix_seed3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
/* first n draws of Rng(seed): u64, uniform, normal */
void orc_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64_out, double* uniform_out,
                   double* normal_out);

/* --- model layout / init (model.cpp:21-96) ------------------------------- */
int orc_model_validate(const orc_model_cfg* c);
uint64_t orc_param_count(const orc_model_cfg* c);
uint64_t orc_layout_size(const orc_model_cfg* c);
/* entry i: flat offset, rows, cols (cols==0 for rank-1), name */
int orc_layout_entry(const orc_model_cfg* c, uint64_t i, uint64_t* offset, uint64_t* rows,
                     uint64_t* cols, char* name, int name_cap);
int orc_init_params(const orc_model_cfg* c, uint64_t seed, double* out);

/* --- data (data.cpp) ------------------------------------------------------ */
int orc_generate_corpus(int32_t style, uint64_t length, uint64_t seed, uint32_t vocab,
                        uint16_t* out);
typedef struct orc_plan orc_plan;
orc_plan* orc_plan_iid(const uint16_t* tokens, uint64_t n_tokens, uint64_t n_shards,
                       uint64_t seq_len, uint64_t seed, int* err);
orc_plan* orc_plan_by_source(const uint16_t* const* corpora, const uint64_t* lens,
                             uint64_t n_sources, uint64_t clients_per_source,
                             uint64_t seq_len, int* err);
void orc_plan_free(orc_plan* p);
uint64_t orc_plan_n_clients(const orc_plan* p);
uint64_t orc_plan_client_blocks(const orc_plan* p, uint64_t client);
/* block b of client: (source, offset) */
void orc_plan_block(const orc_plan* p, uint64_t client, uint64_t b, uint32_t* source,
                    uint64_t* offset);
uint64_t orc_stream_seed(uint64_t global_seed, uint64_t client);
int orc_stream_next(const orc_plan* p, uint64_t client, uint64_t batch, uint64_t seq_len,
                    uint64_t seed, uint64_t* cursor, int32_t* inputs, int32_t* targets);

/* --- aggregator / optim --------------------------------------------------- */
int orc_sample_clients(uint64_t population, uint64_t k, uint64_t seed, uint64_t round,
                       uint64_t* out);
int orc_lr_at(const orc_train_cfg* t, uint64_t step, double* out);
double orc_global_norm(const double* x, uint64_t n);
int orc_adamw_step(double* p, const double* g, double* m, double* v, uint64_t n,
                   uint64_t* step_count, const orc_train_cfg* t, double lr);
int orc_sgd_step(double* p, const double* g, uint64_t n, double lr, double clip_norm);
int orc_mean(const double* const* vs, uint64_t k, uint64_t n, double* out);
void orc_sub(const double* a, const double* b, uint64_t n, double* out);
int orc_server_step(const orc_server_cfg* s, const double* theta, const double* delta,
                    const double* mean, double* velocity, uint64_t n, double* out);
int orc_post_process(const double* theta_ref, const double* theta_k, uint64_t n,
                     int32_t kind, double threshold, double* out);

/* --- model forward / backward (model.cpp:98-174, tensor.cpp) -------------- */
/* loss over one batch; grads (canonical order, length P) when non-NULL */
int orc_forward_backward(const orc_model_cfg* c, const double* params, const int32_t* inputs,
                         const int32_t* targets, uint64_t batch, uint64_t seq,
                         double* loss_out, double* grads);
int orc_eval_perplexity(const orc_model_cfg* c, const double* params, const int32_t* inputs,
                        const int32_t* targets, uint64_t n_batches, const uint64_t* batch_sizes,
                        uint64_t seq, double* ppl_out);

/* --- client update (client.cpp:125-158) ----------------------------------- */
int orc_local_round(const orc_model_cfg* c, const orc_train_cfg* t, const double* theta_in,
                    const orc_plan* plan, uint64_t client, uint64_t stream_seed,
                    uint64_t* cursor, uint64_t round, uint64_t step_base, double* theta_out,
                    double* losses, uint64_t* err_step);

/* --- one federated round (aggregator.cpp:93-220) --------------------------- */
/* theta / velocity are updated in place; cursors has one entry per population
 * client; sampled_out (K) and client_losses (K mean losses) are optional. */
int orc_run_round(const orc_model_cfg* c, const orc_train_cfg* t, const orc_server_cfg* s,
                  const orc_plan* plan, uint64_t population, uint64_t k, uint64_t seed,
                  uint64_t round, double* theta, double* velocity, uint64_t* cursors,
                  const uint64_t* dropped_clients, uint64_t n_dropped, int32_t ring_topology,
                  uint64_t* sampled_out, double* client_mean_losses);

#ifdef __cplusplus
}
#endif
#endif
