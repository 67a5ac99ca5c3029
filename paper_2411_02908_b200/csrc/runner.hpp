// runner.hpp -- device-resident FederationRunner (aggregator.h:70-102) with a
// sharded, NCCL-backed round boundary across ranks.
#pragma once

#include <nccl.h>

#include <memory>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "ctx.hpp"
#include "p2p.hpp"

namespace photon {

struct Runner {
  Ctx* ctx;
  photon_fed_cfg fed;
  photon_train_cfg train;
  photon_server_cfg server;
  const Plan* plan;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  // world > 1: the boundary over NVLink peer memory (PHOTON_BOUNDARY=nccl selects
  // the NCCL send/recv + all-gather path instead; both are bit-identical)
  std::unique_ptr<PeerBoundary> p2p;

  uint64_t P = 0, shard = 0, Ppad = 0;
  uint64_t next_round = 0;
  std::vector<uint64_t> cursors;
  std::set<std::pair<uint64_t, uint64_t>> dropouts;

  DevBuf<float> d_theta;     // [Ppad] theta_t (replicated)
  DevBuf<float> d_vel;       // [Ppad] outer velocity (this rank's shard is authoritative)
  DevBuf<float> d_models;    // [slots_local][Ppad] client results on this rank
  DevBuf<float> d_recv;      // [K][shard] exchanged shards
  DevBuf<const float*> d_model_ptrs;
  DevBuf<double> d_stats;    // [2K] loss stats / error exchange
  PinnedBuf<double> h_stats;
  // token pipeline: two host/device batch sets alternate by
  // round; round t+1's tau batches are staged and copied (copy_stream) while the
  // GPU trains round t
  std::vector<RoundBatches> host_batches[2];  // per local slot (pinned)
  std::vector<DeviceBatches> dev_batches[2];  // per local slot
  int buf = 0;                                // set holding the next round to run
  uint64_t staged_round = ~0ULL;              // round whose batches sit in set `buf`
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr};
  double stage(uint64_t round, int set, const std::vector<uint64_t>& cur);
  DevBuf<double> d_loss;
  DevBuf<int> d_flag;
  PinnedBuf<double> h_loss;
  PinnedBuf<int> h_flag;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_b2 = nullptr;

  // per-round evaluation (RunnerOptions::eval_every / eval_fn, aggregator.cpp:207-212):
  // batch i of the eval set lives on rank i % world, resident in HBM
  uint64_t eval_every = 0, eval_n = 0;
  std::vector<DeviceBatches> eval_dev;
  std::vector<uint64_t> eval_ids, eval_valid;
  DevBuf<double> d_eval;
  PinnedBuf<double> h_eval;
  // harness bookkeeping persisted in state.json (harness.cpp:527-535)
  double initial_ppl = 0.0;
  uint64_t sync_events = 0;

  Runner(Ctx* c, const photon_fed_cfg& f, const photon_train_cfg& t, const photon_server_cfg& s,
         const Plan* p, const double* theta0, int rank, int world, const uint8_t* nccl_id);
  ~Runner();

  void run_round(photon_round_record* rec);
  void theta_f64(double* out);
  void velocity_f64(double* out);
  void restore(const double* theta, const double* velocity, uint64_t next_round,
               const uint64_t* cursors, uint64_t n);
  void set_eval(const EvalSet& es, uint64_t every);
  double eval_theta();  // perplexity of the replicated theta (collective for world > 1)
  // checkpoint.phck + velocity.phck + state.json under dir (collective; rank 0 writes)
  void save(const std::string& dir);
  void resume(const std::string& dir);
};

void validate_server(const photon_server_cfg& s);
// world > 1: NVLink peer memory for replicas up to PeerBoundary::fits, else NCCL;
// PHOTON_BOUNDARY=nccl|p2p forces either path
bool use_peer_boundary(uint64_t replica_bytes);

// The round boundary (aggregator.cpp:177-179) over NCCL: every surviving
// slot's model goes in 1/world shards to the shard owners in ascending slot
// order (slot si lives on rank si % world), the owner runs the fused
// anchored-mean -> pseudo-gradient -> outer update on its shard of theta
// (d_vel holds that shard), and an all-gather rebuilds theta on every rank.
// world == 1: the fused update over the local models, no communication.
// Per-GPU wire bytes 2 (world-1)/world * P * 4.
void round_boundary(ncclComm_t comm, int rank, int world, uint64_t P, uint64_t shard,
                    const std::vector<int>& surv, const float* const* local_models,
                    float* recv, DevBuf<const float*>& d_ptrs, float* d_theta, float* d_vel,
                    const photon_server_cfg& server, cudaStream_t st);

}  // namespace photon
