// mufu_bw.cu -- MUFU.EX2 / FFMA issue throughput per SM with independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_bw tools/mufu_bw.cu && /tmp/mufu_bw
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(int iters, unsigned long long* cycles, float* sink) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -1.0f - 1e-3f * (threadIdx.x + i);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (OP == 1) {
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0fBC000000;" : "+f"(a[i]));
      } else if (OP == 2) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(*reinterpret_cast<unsigned*>(&a[i])));
      } else if (OP == 3) {  // F2FP pack: two fp32 -> bf16x2
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(a[i]));
        a[i] = __uint_as_float(r);
      } else {  // one ex2 + one pack per element (the softmax mix)
        unsigned r;
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(a[i]));
        a[i] = __uint_as_float(r);
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  unsigned long long h;
  const int iters = 2048;
  const char* names[5] = {"ex2.f32", "ffma", "ex2.bf16x2", "cvt.bf16x2", "ex2+cvt"};
  for (int op = 0; op < 5; ++op)
    for (int warps : {4, 8, 16, 32}) {
      if (op == 0) kern<0><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 1) kern<1><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 2) kern<2><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 3) kern<3><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 4) kern<4><<<148, warps * 32>>>(iters, cyc, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-11s warps=%2d: %6.1f warp-instr... lane-ops/clk/SM = %.1f\n", names[op], warps,
             0.0, (double)warps * 32 * 8 * iters / (double)h);
    }
  return 0;
}
