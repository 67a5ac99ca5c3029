// gemm_simt.cu -- CUDA-core fp32-accumulate GEMM with fused epilogues.  The
// parity path (PHOTON_PREC_F32) and the reference for the tcgen05 kernel's
// tests.  64x64 output tile, BK = 16, 256 threads, 4x4 micro-tile with a
// 16-stride thread mapping (conflict-free shared-memory reads).
#include "gemm.cuh"

namespace photon {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename TA, typename TC>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const TA* A = static_cast<const TA*>(g.A);
  const TA* B = static_cast<const TA*>(g.B);
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < (BM * BK) / 256; ++r) {
      const int idx = t + 256 * r;
      int i, kk;
      if (g.a_kmajor) { i = idx / BK; kk = idx % BK; }
      else { i = idx % BM; kk = idx / BM; }
      const int gi = m0 + i, gk = k0 + kk;
      float v = 0.f;
      if (gi < g.M && gk < g.K)
        v = to_f<TA>(g.a_kmajor ? A[(int64_t)gi * g.lda + gk] : A[(int64_t)gk * g.lda + gi]);
      As[kk][i] = v;
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / 256; ++r) {
      const int idx = t + 256 * r;
      int j, kk;
      if (g.b_kmajor) { j = idx / BK; kk = idx % BK; }
      else { j = idx % BN; kk = idx / BN; }
      const int gj = n0 + j, gk = k0 + kk;
      float v = 0.f;
      if (gj < g.N && gk < g.K)
        v = to_f<TA>(g.b_kmajor ? B[(int64_t)gj * g.ldb + gk] : B[(int64_t)gk * g.ldb + gj]);
      Bs[kk][j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[kk][ty + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = Bs[kk][tx + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] += a[x] * b[y];
    }
    __syncthreads();
  }
  TC* C = static_cast<TC*>(g.C);
  TA* aux = static_cast<TA*>(g.aux);
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int r = m0 + ty + 16 * x;
    if (r >= g.M) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int c = n0 + tx + 16 * y;
      if (c >= g.N) continue;
      const int64_t o = (int64_t)r * g.ldc + c;
      const float v = acc[x][y];
      switch (g.epi) {
        case Epi::Store: C[o] = from_f<TC>(v); break;
        case Epi::Accum: C[o] = from_f<TC>(to_f<TC>(C[o]) + v); break;
        case Epi::Bias: C[o] = from_f<TC>(v + g.bias[c]); break;
        case Epi::ResidBias: C[o] = from_f<TC>(g.resid[o] + (v + g.bias[c])); break;
        case Epi::GeluBias: {
          const float pre = v + g.bias[c];
          aux[o] = from_f<TA>(gelu_grad_f(pre));
          C[o] = from_f<TC>(gelu_f(pre));
          break;
        }
        case Epi::GeluBwd: C[o] = from_f<TC>(v * to_f<TA>(aux[o])); break;
      }
    }
  }
}

}  // namespace

void gemm_simt(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  dim3 grid(cdiv(g.N, BN), cdiv(g.M, BM));
  if (grid.y > 65535) throw Error(PHOTON_ERR_CONFIG, "gemm_simt: M too large");
  if (g.ab == DT::F32 && g.c == DT::F32) gemm_simt_kernel<float, float><<<grid, 256, 0, st>>>(g);
  else if (g.ab == DT::BF16 && g.c == DT::F32) gemm_simt_kernel<bf16, float><<<grid, 256, 0, st>>>(g);
  else if (g.ab == DT::BF16 && g.c == DT::BF16) gemm_simt_kernel<bf16, bf16><<<grid, 256, 0, st>>>(g);
  else throw Error(PHOTON_ERR_CONFIG, "gemm_simt: unsupported dtype combination");
  PH_LAUNCH_CHECK();
}

}  // namespace photon
