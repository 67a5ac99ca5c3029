// p2p.hpp -- the round boundary over NVLink peer memory (one process per GPU).
//
// Every rank exports, through CUDA IPC, the device buffers the boundary touches:
// its local client models, its theta replica and a small flag array.  The
// tables are exchanged with one NCCL all-gather (control plane only); peers'
// buffers are opened once and cached.  The boundary itself is
//   barrier -> boundary_p2p_kernel (read all models' shard, anchored mean,
//   outer step, write theta_{t+1} into every replica) -> barrier
// with the barriers done by a one-block kernel over the peers' flag arrays
// (release/acquire at system scope).  No NCCL call sits on the data path.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "kernels.cuh"

namespace photon {

struct PeerBoundary {
  PeerBoundary(ncclComm_t comm, int rank, int world, int device);
  ~PeerBoundary();
  PeerBoundary(const PeerBoundary&) = delete;
  PeerBoundary& operator=(const PeerBoundary&) = delete;

  // Collective: publish this rank's local client models (slot order) and its
  // theta replica; map every peer's.  Cheap when nothing changed (cached opens).
  void publish(const float* const* local_models, int n_local, float* theta, cudaStream_t st);
  // Collective: survivors are slot ids (ascending); slot si lives on rank
  // si % world at local index si / world.  vel = this rank's velocity shard.
  void run(const std::vector<int>& surv, uint64_t shard, float* vel,
           const photon_server_cfg& server, cudaStream_t st);
  static bool supported(int n_survivors, int world) {
    return n_survivors <= kMaxPeerModels && world <= kMaxPeerWorld;
  }
  // device ms of the last run()'s fused kernel (after the opening barrier)
  float last_kernel_ms() const;
  // after run() has completed on the stream: throws if a peer never arrived
  // (the barrier timed out; the boundary kernel was skipped)
  void check();

 private:
  struct Region {  // one exported pointer
    cudaIpcMemHandle_t handle;
    uint64_t offset;  // from the allocation base
    uint64_t raw;     // the pointer in the owner's address space
    int32_t pid, valid;
  };
  static constexpr int kMaxLocal = k::kMaxPeerModels;
  struct Table {
    Region models[kMaxLocal];
    Region theta, flags;
    int32_t n_local, pad;
  };
  Region export_ptr(const void* p) const;
  void* import(int peer, const Region& r);
  void barrier(cudaStream_t st);

  ncclComm_t comm_;
  int rank_, world_, device_;
  DevBuf<uint64_t> flags_;  // [world]: flags_[j] = last epoch rank j signalled to us
  DevBuf<int> abort_;       // 0, or 1 + the rank a barrier gave up on
  DevBuf<uint8_t> tab_dev_;
  uint64_t epoch_ = 0;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  std::vector<std::vector<const float*>> models_;  // [rank][local idx] in this address space
  std::vector<float*> thetas_;
  std::vector<uint64_t*> peer_flags_;
  std::map<std::string, void*> opened_;  // handle bytes -> mapped allocation base
};

}  // namespace photon
