// central.hpp -- device-resident run_centralized (baselines.h:19-51): the
// centralized / DDP baseline with a per-step gradient all-reduce.
#pragma once

#include <nccl.h>

#include <vector>

#include "ctx.hpp"

namespace photon {

void validate_central(const photon_central_cfg& c);

struct Central {
  Ctx* ctx;
  photon_central_cfg cfg;
  const Plan* plan;
  uint64_t seed;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;

  uint64_t P = 0, shard = 0, Ppad = 0, per_worker = 0;
  uint64_t t = 0, since_reset = 0;  // next step; steps since the last optimizer reset
  std::vector<uint64_t> cursors;    // per worker (every rank tracks all)
  std::vector<int> mine;            // workers on this rank (w % world == rank)

  DevBuf<float> d_grads;  // [mine][Ppad] per-worker gradients
  DevBuf<float> d_recv;   // [n_workers][shard] exchanged gradient shards
  DevBuf<float> d_mean;   // [Ppad] all-gathered mean gradient
  DevBuf<const float*> d_ptrs;
  DevBuf<double> d_loss;
  PinnedBuf<double> h_loss;
  PinnedBuf<int> h_flag;
  std::vector<RoundBatches> batches;
  std::vector<DeviceBatches> dev;

  Central(Ctx* c, const photon_central_cfg& cfg, const Plan* p, uint64_t seed,
          const double* theta0, int rank, int world, const uint8_t* nccl_id);
  ~Central();
  void step(photon_step_metric* out);
  void theta_f64(double* out);
};

}  // namespace photon
