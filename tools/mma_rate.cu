// mma_rate.cu -- tcgen05.mma.cta_group::1.kind::f16 (bf16 -> f32) issue-to-completion
// rate for M=128 and N in {64,128,256}: SS with K-major B, SS with MN-major B, and
// A-from-TMEM (TS).  Operand contents are irrelevant (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate tools/mma_rate.cu && /tmp/mma_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, int FORM, int NACC = 1>  // FORM 0: SS K-major B, 1: SS MN-major B, 2: TS (A in TMEM), MN-major B
// NACC: independent accumulators issued round-robin (1 = one dependent chain)
__global__ void mma_kernel(int n_mma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((FORM >= 1 ? 1u : 0u) << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int kk = i & 3;
      const uint64_t bd = FORM >= 1 ? sw128(b + kk * 2048, 8192, 1024) : sw128(b + kk * 32, 16, 1024);
      if (FORM == 2) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256),
            "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1));
      } else {
        const uint64_t ad = sw128(a + kk * 32, 16, 1024);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (i % NACC) * N),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    const unsigned long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    const unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int FORM, int NACC = 1>
void run(const char* name) {
  unsigned long long* d;
  unsigned long long h[2];
  cudaMalloc(&d, 16);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mma_kernel<N, FORM, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (NACC > 1) printf("(%d independent accumulators)\n", NACC);
  for (int n : {8, 64, 512}) {
    mma_kernel<N, FORM, NACC><<<148, 128, smem>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-16s N=%3d  %4d MMAs: issue %7llu cyc, done %7llu cyc -> %6.1f cyc/MMA (floor %d)\n",
           name, N, n, h[0], h[1], (double)h[1] / n, 128 * N / 256);
  }
  cudaFree(d);
}

// 2-CTA pair: leader issues M=256 x N MMAs (cta_group::2), both CTAs hold operands.
template <int N, int TS = 0>  // TS: A from TMEM (the attention backward's dV / dK form)
__global__ void __cluster_dims__(2, 1, 1) mma_pair_kernel(int n_mma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int kk = i & 3;
      const uint64_t ad = sw128(a + kk * 32, 16, 1024), bd = sw128(b + kk * 32, 16, 1024);
      if (TS) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256),
            "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1));
      } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    const unsigned long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)1) : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    const unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int TS = 0>
void run_pair() {
  unsigned long long* d;
  unsigned long long h[2];
  cudaMalloc(&d, 16);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mma_pair_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int n : {8, 64, 512}) {
    mma_pair_kernel<N, TS><<<148, 128, smem>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("pair: %s\n", cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("PAIR M=256 %s   N=%3d  %4d MMAs: issue %7llu cyc, done %7llu cyc -> %6.1f cyc/MMA (1-CTA M128 equiv %d)\n",
           TS ? "TS" : "SS", N, n, h[0], h[1], (double)h[1] / n, 128 * N / 256);
  }
  cudaFree(d);
}

int main() {
  run_pair<256>();
  run_pair<128>();
  run_pair<64>();
  run_pair<128, 1>();
  run_pair<64, 1>();
  run<64, 0>("SS Kmaj");
  run<64, 1>("SS MNmaj");
  run<64, 2>("TS MNmaj");
  run<128, 0>("SS Kmaj");
  run<128, 2>("TS MNmaj");
  run<256, 0>("SS Kmaj");
  run<64, 0, 2>("SS Kmaj");
  run<64, 0, 4>("SS Kmaj");
  run<64, 1, 2>("SS MNmaj");
  run<128, 0, 2>("SS Kmaj");
  return 0;
}
