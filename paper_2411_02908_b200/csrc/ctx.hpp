// ctx.hpp -- photon_ctx: one GPU's engine plus the per-round device buffers,
// and the device-resident client update (run_local_round, client.cpp:125-158).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "engine.cuh"

namespace photon {

template <typename U>
struct DevBuf {
  U* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n) {
    o.ptr = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(n, o.n);
    return *this;
  }
  void reserve(size_t want) {
    if (want <= n) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
    PH_CUDA(cudaMalloc(&ptr, want * sizeof(U)));
    n = want;
  }
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
};

template <typename U>
struct PinnedBuf {
  U* ptr = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  PinnedBuf(PinnedBuf&& o) noexcept : ptr(o.ptr), n(o.n) {
    o.ptr = nullptr;
    o.n = 0;
  }
  PinnedBuf& operator=(PinnedBuf&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(n, o.n);
    return *this;
  }
  void reserve(size_t want) {
    if (want <= n) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    n = 0;
    PH_CUDA(cudaMallocHost(&ptr, want * sizeof(U)));
    n = want;
  }
  ~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
};

// The tau batches of one client round, staged on the host.
struct RoundBatches {
  int tau = 0, B = 0, S = 0;
  PinnedBuf<int32_t> tokens, targets, csr_off, csr_rows;  // [tau][...]
  std::vector<float> inv_count;                            // [tau]
  void prepare(int tau_, int B_, int S_, int V);           // sizes pinned buffers
  void finalize(int V);                                    // CSR + counts from tokens/targets
};

// A staged round's batches on the device.
struct DeviceBatches {
  DevBuf<int32_t> tokens, targets, csr_off, csr_rows;
  std::vector<float> inv_count;
  DevBuf<float> inv_dev;  // inv_count on the device (read by graph-captured rounds)
  int tau = 0, B = 0, S = 0;
  void upload(const RoundBatches& rb, int V, cudaStream_t st);
};

struct LocalResult {
  std::vector<double> losses;  // tau
  int error = PHOTON_OK;
  uint64_t error_step = 0;
};

struct Ctx {
  int device = 0;
  photon_model_cfg cfg{};
  int precision = 0;
  uint64_t max_batch = 0;
  cudaStream_t stream = nullptr;
  std::unique_ptr<Engine> eng;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;

  // device copies of the current call's batches (C-ABI single-client path)
  DeviceBatches dev_batches;
  DevBuf<double> d_losses;
  PinnedBuf<double> h_losses;
  DevBuf<int> d_flags;
  PinnedBuf<int> h_flag;
  // generic scratch
  DevBuf<double> d_f64a, d_f64b, d_f64c, d_f64d;
  DevBuf<float> d_f32a, d_f32b;
  DevBuf<const void*> d_ptrs;
  // CUDA graphs of the local round (launch-bound small models): one executable
  // graph per (buffers, shapes, hyper-parameters) key, captured on the second
  // launch with that key (the first runs eagerly: lazy allocations and kernel
  // attributes happen outside capture); lr per step comes from d_lr
  struct RoundGraph {
    cudaGraphExec_t exec = nullptr;
    int seen = 0;
    uint64_t kernels = 0;  // kernel nodes (added to launch_counter per replay)
  };
  std::map<std::string, RoundGraph> graphs;
  bool graphs_on = true;
  DevBuf<double> d_lr;

  Ctx(int dev, const photon_model_cfg& m, int prec, uint64_t mb);
  ~Ctx();

  // f64 host <-> fp32 device through a bounded staging chunk (d_f64a holds one
  // chunk, not P doubles: 7B-scale parameter vectors are 55 GB in f64)
  void h2d_f64_to_f32(const double* host, float* dev, uint64_t n);
  void d2h_f32_to_f64(const float* dev, double* host, uint64_t n);  // synchronous

  void begin_timing();
  double end_timing();  // syncs, returns ms since begin_timing

  // H2D of a staged round (async on stream) into dev_batches
  void upload(const RoundBatches& rb);
  // Enqueue tau local steps from d_theta_in (fp32 device) into d_theta_out (may
  // equal engine master): per-step losses -> d_loss[0..tau), first bad-norm
  // step (1-based, 0 = none) -> *d_flag.  Asynchronous.
  void launch_local_round(const photon_train_cfg& cfg, const DeviceBatches& db,
                          const float* d_theta_in, float* d_theta_out, uint64_t step_base,
                          double* d_loss, int* d_flag);
  // Synchronous convenience over dev_batches: launch, read back, classify.
  LocalResult local_round(const photon_train_cfg& cfg, const float* d_theta_in,
                          float* d_theta_out, uint64_t step_base);
};

void check_train_cfg(const photon_train_cfg& t);
// First failure in step order (DivergenceError before the same step's NumericError).
LocalResult classify(const double* losses, int tau, int bad_step);

}  // namespace photon
