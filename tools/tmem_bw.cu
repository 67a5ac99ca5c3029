// tmem_bw.cu -- measure tcgen05.ld (TMEM -> registers) throughput per SM for
// 4..16 warps and with/without interleaved MUFU work.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MUFU>
__global__ void tmem_read_kernel(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + (it & 1) * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x = __uint_as_float(r[i]);
      if (MUFU) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x + acc));
        acc += y;
      } else {
        acc += x;
      }
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int MUFU>
__global__ void mufu_only_kernel(int iters, unsigned long long* cycles, float* sink) {
  float acc = threadIdx.x * 1e-3f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(acc * 1e-3f + i));
      acc += y * 1e-9f;
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int iters = 4096, blocks = 148;
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, blocks * sizeof(unsigned long long));
  cudaMalloc(&sink, blocks * 1024 * sizeof(float));
  unsigned long long h[148];
  for (int warps : {4, 8, 16}) {
    for (int mufu : {0, 1}) {
      if (mufu) tmem_read_kernel<1><<<blocks, warps * 32>>>(iters, cyc, sink);
      else tmem_read_kernel<0><<<blocks, warps * 32>>>(iters, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * 32 * 32 * 4 * iters;  // per SM
      printf("warps=%2d mufu=%d: %.1f cycles/iter/warp, TMEM read %.1f B/clk/SM%s\n", warps, mufu,
             (double)h[0] / iters, bytes / (double)h[0],
             mufu ? " (with 32 ex2 per ld per lane)" : "");
    }
  }
  for (int warps : {4, 8, 16}) {
    mufu_only_kernel<1><<<blocks, warps * 32>>>(iters, cyc, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double ops = (double)warps * 32 * 32 * iters;
    printf("mufu only warps=%2d: %.1f ex2/clk/SM\n", warps, ops / (double)h[0]);
  }
  return 0;
}
