// p2p.cpp -- round boundary over NVLink peer memory (see p2p.hpp).
#include "p2p.hpp"

#include <cuda.h>
#include <unistd.h>

#include <cstring>

#include "nccl_api.hpp"

namespace photon {

namespace {

#define PH_NCCL_P2P(call)                                                                    \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      throw Error(PHOTON_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_));   \
  } while (0)

struct FlagArgs {
  uint64_t* peer[k::kMaxPeerWorld];  // rank j's flag array, mapped here
  uint64_t* mine;
  int* abort;  // this rank's abort word (device), checked by the host after the boundary
  uint64_t epoch;
  int rank, world;
};

// Thread j signals rank j (writes epoch into rank j's flags[rank]) and waits
// for rank j's signal in our flags[j].  A peer that never arrives (dead rank)
// sets the abort word after ~20 s and the wait ends: the boundary kernel then
// does nothing and PeerBoundary::check() raises a host error -- no sticky
// device fault, no hang.
__global__ void peer_barrier_kernel(const __grid_constant__ FlagArgs a) {
  const int j = threadIdx.x;
  if (j >= a.world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.peer[j] + a.rank), "l"(a.epoch)
               : "memory");
  const long long t0 = clock64();
  for (;;) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.mine + j) : "memory");
    if (v >= a.epoch) break;
    if (*(volatile int*)a.abort) break;  // another lane already gave up
    if (clock64() - t0 > (1ll << 35)) {
      atomicMax(a.abort, j + 1);  // 1 + the rank that did not arrive
      break;
    }
    __nanosleep(64);
  }
}

}  // namespace

PeerBoundary::PeerBoundary(ncclComm_t comm, int rank, int world, int device)
    : comm_(comm), rank_(rank), world_(world), device_(device) {
  if (world > k::kMaxPeerWorld) throw Error(PHOTON_ERR_CONFIG, "peer boundary: world too large");
  flags_.reserve(world);
  PH_CUDA(cudaMemset(flags_.ptr, 0, world * sizeof(uint64_t)));
  abort_.reserve(1);
  PH_CUDA(cudaMemset(abort_.ptr, 0, sizeof(int)));
  tab_dev_.reserve((size_t)world * sizeof(Table));
  models_.assign(world, {});
  thetas_.assign(world, nullptr);
  peer_flags_.assign(world, nullptr);
  PH_CUDA(cudaEventCreate(&ev0_));
  PH_CUDA(cudaEventCreate(&ev1_));
}

float PeerBoundary::last_kernel_ms() const {
  float ms = 0.f;
  PH_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  return ms;
}

PeerBoundary::~PeerBoundary() {
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  for (auto& kv : opened_) cudaIpcCloseMemHandle(kv.second);
}

PeerBoundary::Region PeerBoundary::export_ptr(const void* p) const {
  Region r;
  std::memset(&r, 0, sizeof(r));
  // driver entry point resolved at run time: libphoton.so must load on hosts
  // without libcuda.so (the CPU test suite)
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRange>(f);
  }();
  if (!get_range) throw Error(PHOTON_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    throw Error(PHOTON_ERR_CUDA, "peer boundary: pointer is not a device allocation");
  PH_CUDA(cudaIpcGetMemHandle(&r.handle, reinterpret_cast<void*>(base)));
  r.offset = reinterpret_cast<uint64_t>(p) - (uint64_t)base;
  r.raw = reinterpret_cast<uint64_t>(p);
  r.pid = (int32_t)getpid();
  r.valid = device_ + 1;
  return r;
}

void* PeerBoundary::import(int peer, const Region& r) {
  if (!r.valid) throw Error(PHOTON_ERR_USAGE, "peer boundary: missing region");
  if (peer == rank_) return reinterpret_cast<void*>(r.raw);
  if (r.pid == (int32_t)getpid()) {  // ranks sharing a process: plain peer access
    const cudaError_t e = cudaDeviceEnablePeerAccess(r.valid - 1, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) PH_CUDA(e);
    cudaGetLastError();
    return reinterpret_cast<void*>(r.raw);
  }
  const std::string key(reinterpret_cast<const char*>(&r.handle), sizeof(r.handle));
  auto it = opened_.find(key);
  if (it == opened_.end()) {
    void* base = nullptr;
    PH_CUDA(cudaIpcOpenMemHandle(&base, r.handle, cudaIpcMemLazyEnablePeerAccess));
    it = opened_.emplace(key, base).first;
  }
  return static_cast<uint8_t*>(it->second) + r.offset;
}

void PeerBoundary::publish(const float* const* local_models, int n_local, float* theta,
                           cudaStream_t st) {
  if (n_local > kMaxLocal) throw Error(PHOTON_ERR_CONFIG, "peer boundary: too many local clients");
  PH_CUDA(cudaSetDevice(device_));
  Table t;
  std::memset(&t, 0, sizeof(t));
  for (int j = 0; j < n_local; ++j) t.models[j] = export_ptr(local_models[j]);
  t.theta = export_ptr(theta);
  t.flags = export_ptr(flags_.ptr);
  t.n_local = n_local;
  uint8_t* mine = tab_dev_.ptr + (size_t)rank_ * sizeof(Table);
  PH_CUDA(cudaMemcpyAsync(mine, &t, sizeof(Table), cudaMemcpyHostToDevice, st));
  PH_NCCL_P2P(nccl().AllGather(mine, tab_dev_.ptr, sizeof(Table), ncclUint8, comm_, st));
  std::vector<Table> all(world_);
  PH_CUDA(cudaMemcpyAsync(all.data(), tab_dev_.ptr, (size_t)world_ * sizeof(Table),
                          cudaMemcpyDeviceToHost, st));
  PH_CUDA(cudaStreamSynchronize(st));
  for (int q = 0; q < world_; ++q) {
    models_[q].assign(all[q].n_local, nullptr);
    for (int j = 0; j < all[q].n_local; ++j)
      models_[q][j] = static_cast<const float*>(import(q, all[q].models[j]));
    thetas_[q] = static_cast<float*>(import(q, all[q].theta));
    peer_flags_[q] = static_cast<uint64_t*>(import(q, all[q].flags));
  }
}

void PeerBoundary::barrier(cudaStream_t st) {
  FlagArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int q = 0; q < world_; ++q) a.peer[q] = peer_flags_[q];
  a.mine = flags_.ptr;
  a.abort = abort_.ptr;
  a.epoch = ++epoch_;
  a.rank = rank_;
  a.world = world_;
  peer_barrier_kernel<<<1, 32, 0, st>>>(a);
  PH_LAUNCH_CHECK();
}

void PeerBoundary::run(const std::vector<int>& surv, uint64_t shard, float* vel,
                       const photon_server_cfg& server, cudaStream_t st) {
  const int n = (int)surv.size();
  if (!supported(n, world_)) throw Error(PHOTON_ERR_USAGE, "peer boundary: too many clients");
  k::PeerBoundaryArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int r = 0; r < n; ++r) {
    const int si = surv[r], owner = slot_owner(si, world_), j = si / world_;
    if (j >= (int)models_[owner].size())
      throw Error(PHOTON_ERR_USAGE, "peer boundary: slot not published by its rank");
    a.models[r] = models_[owner][j];
  }
  for (int q = 0; q < world_; ++q) a.replicas[q] = thetas_[q];
  a.vel = vel;
  a.off = (uint64_t)rank_ * shard;
  a.len = shard;
  a.n = n;
  a.world = world_;
  a.rank = rank_;
  a.kind = server.kind;
  a.nesterov = server.nesterov;
  a.eta = (float)server.eta;
  a.mu = (float)server.momentum;
  a.abort = abort_.ptr;
  barrier(st);  // every rank's client models are final
  PH_CUDA(cudaEventRecord(ev0_, st));
  k::boundary_p2p(a, st);
  PH_CUDA(cudaEventRecord(ev1_, st));
  barrier(st);  // every replica holds theta_{t+1}; nobody reads our models any more
}

void PeerBoundary::check() {
  int h = 0;
  PH_CUDA(cudaMemcpy(&h, abort_.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  if (h)
    throw Error(PHOTON_ERR_NCCL, "peer boundary: rank " + std::to_string(h - 1) +
                                     " did not reach the round boundary within ~20 s");
}

}  // namespace photon
