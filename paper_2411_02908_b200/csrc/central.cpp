// central.cpp -- run_centralized (baselines.cpp:25-127), the paper's
// centralized / DDP comparison baseline, on B200s.
//
// n_workers data-parallel workers draw per-worker batches from their own
// streams (worker w: shard w, stream_seed(seed, w)); worker w runs on rank
// w % world.  Each step: every local worker's forward + backward into its own
// gradient buffer; the gradients are averaged in ascending worker order with
// the anchored mean of ParamVector::mean (param_vector.cpp:127-152) -- across
// ranks the shards of every worker's gradient go to their owners over NCCL,
// the owner averages its shard, an all-gather rebuilds the mean -- and every
// rank applies the same AdamW / SGD update to its replica.  Results do not
// depend on the GPU count.
#include <cmath>
#include <cstring>
#include <limits>

#include "central.hpp"
#include "kernels.cuh"
#include "nccl_api.hpp"

namespace photon {

#define PH_NCCL(call)                                                                    \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw Error(PHOTON_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

// CentralizedConfig::validate (baselines.cpp:13-23)
void validate_central(const photon_central_cfg& c) {
  photon_train_cfg t{};
  t.model = c.model;
  t.adamw = c.adamw;
  t.schedule = c.schedule;
  t.opt = c.opt;
  t.batch_size = 1;
  check_train_cfg(t);
  if (c.n_workers < 1) throw Error(PHOTON_ERR_CONFIG, "centralized: n_workers must be >= 1");
  if (c.global_batch < 1 || c.global_batch % c.n_workers != 0)
    throw Error(PHOTON_ERR_CONFIG, "centralized: global batch must divide by n_workers");
  if (c.total_steps < 1) throw Error(PHOTON_ERR_CONFIG, "centralized: total_steps must be >= 1");
  if (!(c.throughput_bps > 0.0)) throw Error(PHOTON_ERR_CONFIG, "centralized: nu must be > 0");
}

Central::Central(Ctx* c, const photon_central_cfg& cf, const Plan* p, uint64_t sd,
                 const double* theta0, int rk, int ws, const uint8_t* nccl_id)
    : ctx(c), cfg(cf), plan(p), seed(sd), rank(rk), world(ws) {
  validate_central(cf);
  if (!p) throw Error(PHOTON_ERR_USAGE, "centralized: null shard plan");
  if (p->blocks.size() < cf.n_workers)
    throw Error(PHOTON_ERR_CONFIG, "shard plan covers " + std::to_string(p->blocks.size()) +
                                       " shards, run needs " + std::to_string(cf.n_workers));
  if (std::memcmp(&cf.model, &c->cfg, sizeof(photon_model_cfg)) != 0)
    throw Error(PHOTON_ERR_CONFIG, "centralized: model differs from the context's model");
  if (p->seq_len != cf.model.seq_len)
    throw Error(PHOTON_ERR_USAGE, "stream: seq_len does not match the plan's block size");
  if (ws < 1 || rk < 0 || rk >= ws) throw Error(PHOTON_ERR_USAGE, "centralized: bad rank/world");
  per_worker = cf.global_batch / cf.n_workers;
  P = c->eng->P;
  shard = shard_len(P, ws);
  Ppad = shard * ws;
  cursors.assign(cf.n_workers, 0);
  for (uint64_t w = 0; w < cf.n_workers; ++w)
    if ((int)(w % ws) == rk) mine.push_back((int)w);
  PH_CUDA(cudaSetDevice(c->device));
  d_grads.reserve(std::max<size_t>(mine.size(), 1) * Ppad);
  PH_CUDA(cudaMemsetAsync(d_grads.ptr, 0, d_grads.n * 4, c->stream));
  if (ws > 1) {
    d_recv.reserve((size_t)cf.n_workers * shard);
    d_mean.reserve(Ppad);
  }
  d_loss.reserve(cf.n_workers);
  h_loss.reserve(cf.n_workers);
  h_flag.reserve(1);
  batches.resize(mine.size());
  dev.resize(mine.size());
  Engine& e = *c->eng;
  c->h2d_f64_to_f32(theta0, e.master, P);
  e.refresh_shadow();
  PH_CUDA(cudaMemsetAsync(e.mom, 0, P * 4, c->stream));
  PH_CUDA(cudaMemsetAsync(e.vel2, 0, P * 4, c->stream));
  if (ws > 1) {
    if (!nccl_id) throw Error(PHOTON_ERR_USAGE, "centralized: world > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    PH_NCCL(nccl().CommInitRank(&comm, ws, id, rk));
  }
  PH_CUDA(cudaStreamSynchronize(c->stream));
}

Central::~Central() {
  if (comm) nccl().CommDestroy(comm);
}

void Central::step(photon_step_metric* out) {
  if (t >= cfg.total_steps) throw Error(PHOTON_ERR_USAGE, "centralized: all steps already taken");
  PH_CUDA(cudaSetDevice(ctx->device));
  Engine& e = *ctx->eng;
  cudaStream_t st = ctx->stream;
  const int S = (int)plan->seq_len, V = (int)cfg.model.vocab_size, B = (int)per_worker;
  const int nw = (int)cfg.n_workers;
  if (cfg.opt_reset_interval > 0 && t % cfg.opt_reset_interval == 0) {  // fresh AdamW state
    PH_CUDA(cudaMemsetAsync(e.mom, 0, P * 4, st));
    PH_CUDA(cudaMemsetAsync(e.vel2, 0, P * 4, st));
    since_reset = 0;
  }
  // batches are drawn per worker from its own stream (baselines.cpp:63-69)
  for (size_t j = 0; j < mine.size(); ++j) {
    const uint64_t w = (uint64_t)mine[j];
    RoundBatches& hb = batches[j];
    hb.prepare(1, B, S, V);
    stream_rows(*plan, w, derive(seed, kPurposeStream, w), cursors[w], per_worker, hb.tokens.ptr,
                hb.targets.ptr);
    hb.finalize(V);
    dev[j].upload(hb, V, st);
  }
  PH_CUDA(cudaMemsetAsync(d_loss.ptr, 0, nw * sizeof(double), st));
  for (size_t j = 0; j < mine.size(); ++j) {
    const DeviceBatches& db = dev[j];
    StepBatch sb{db.tokens.ptr, db.targets.ptr, db.csr_off.ptr, db.csr_rows.ptr, db.B, db.S,
                 db.inv_count[0]};
    e.forward_backward(sb, d_loss.ptr + mine[j], true);
    PH_CUDA(cudaMemcpyAsync(d_grads.ptr + j * Ppad, e.grads, P * 4, cudaMemcpyDeviceToDevice, st));
  }
  // every worker's loss sits on exactly one rank: a sum reassembles them exactly
  if (world > 1) PH_NCCL(nccl().AllReduce(d_loss.ptr, d_loss.ptr, nw, ncclDouble, ncclSum, comm, st));
  PH_CUDA(cudaMemcpyAsync(h_loss.ptr, d_loss.ptr, nw * sizeof(double), cudaMemcpyDeviceToHost, st));

  // ascending-worker anchored mean of the gradients into e.grads
  std::vector<const float*> ptrs(nw);
  if (world == 1) {
    for (int w = 0; w < nw; ++w) ptrs[w] = d_grads.ptr + (size_t)w * Ppad;
    d_ptrs.reserve(nw);
    PH_CUDA(cudaMemcpyAsync(d_ptrs.ptr, ptrs.data(), nw * sizeof(float*), cudaMemcpyHostToDevice, st));
    k::mean_only<float>(d_ptrs.ptr, nw, P, e.grads, st);
  } else {
    PH_NCCL(nccl().GroupStart());
    for (int w = 0; w < nw; ++w) {
      const int owner = slot_owner(w, world);
      if (owner == rank) {
        const float* g = d_grads.ptr + (size_t)(w / world) * Ppad;
        for (int q = 0; q < world; ++q)
          PH_NCCL(nccl().Send(g + (size_t)q * shard, shard, ncclFloat, q, comm, st));
      }
      PH_NCCL(nccl().Recv(d_recv.ptr + (size_t)w * shard, shard, ncclFloat, owner, comm, st));
    }
    PH_NCCL(nccl().GroupEnd());
    for (int w = 0; w < nw; ++w) ptrs[w] = d_recv.ptr + (size_t)w * shard;
    d_ptrs.reserve(nw);
    PH_CUDA(cudaMemcpyAsync(d_ptrs.ptr, ptrs.data(), nw * sizeof(float*), cudaMemcpyHostToDevice, st));
    k::mean_only<float>(d_ptrs.ptr, nw, shard, d_mean.ptr + (size_t)rank * shard, st);
    PH_NCCL(nccl().AllGather(d_mean.ptr + (size_t)rank * shard, d_mean.ptr, shard, ncclFloat, comm, st));
    PH_CUDA(cudaMemcpyAsync(e.grads, d_mean.ptr, P * 4, cudaMemcpyDeviceToDevice, st));
  }
  PH_CUDA(cudaStreamSynchronize(st));
  double loss = 0.0;
  for (int w = 0; w < nw; ++w) loss += h_loss.ptr[w];
  loss /= (double)nw;
  if (!std::isfinite(loss)) {
    Error ex(PHOTON_ERR_DIVERGENCE, "centralized run diverged at step " + std::to_string(t));
    ex.round = 0;
    ex.client = 0;
    ex.step = t;
    throw ex;
  }
  // one shared update (baselines.cpp:114-120)
  PH_CUDA(cudaMemsetAsync(e.bad_step, 0, sizeof(int), st));
  const double lr = lr_at(cfg.schedule, t);
  if (cfg.opt == 0) {
    const double sc = (double)(since_reset + 1), b1 = cfg.adamw.beta1, b2 = cfg.adamw.beta2;
    e.adamw(cfg.adamw.clip_norm, lr, b1, b2, 1.0 - std::pow(b1, sc), 1.0 - std::pow(b2, sc),
            cfg.adamw.eps, cfg.adamw.weight_decay, 0);
  } else {
    e.sgd(cfg.sgd_clip_norm, lr, 0);
  }
  PH_CUDA(cudaMemcpyAsync(h_flag.ptr, e.bad_step, sizeof(int), cudaMemcpyDeviceToHost, st));
  PH_CUDA(cudaStreamSynchronize(st));
  if (h_flag.ptr[0]) throw Error(PHOTON_ERR_NUMERIC, "gradient norm is not finite");
  for (auto& c : cursors) c += per_worker;
  ++t;
  ++since_reset;
  if (out) *out = photon_step_metric{loss, cfg.global_batch * plan->seq_len, 1.0 / cfg.throughput_bps};
}

void Central::theta_f64(double* out) {
  PH_CUDA(cudaSetDevice(ctx->device));
  ctx->d2h_f32_to_f64(ctx->eng->master, out, P);
}

}  // namespace photon
