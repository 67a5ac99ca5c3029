// gemm.cuh -- contraction interface of the client step.
//
// C[M,N] = epi( sum_k A(i,k) B(k,j) ) covering the three matmul layouts of
// tensor.cpp:152-207 on the reference's canonical [in,out] row-major weights:
//   forward  Y  = X  W     A = X  (K-major), B = W  ([K,N], N-major)
//   backward dX = dY W^T   A = dY (K-major), B = W  viewed K-major
//   backward dW = X^T dY   A = X  (M-major), B = dY (N-major)
// with the add_bias / residual add / GELU (tensor.cpp:209-288, 396-420)
// forward and backward fused into the epilogue.
#pragma once

#include "common.cuh"

namespace photon {

enum class DT : int { F32 = 0, BF16 = 1 };

enum class Epi : int {
  Store = 0,      // C = acc
  Accum = 1,      // C += acc
  Bias = 2,       // C = acc + bias
  ResidBias = 3,  // C(f32) = resid + (acc + bias)
  GeluBias = 4,   // u = acc + bias ; C = gelu(u), aux = gelu'(u)  (the backward's factor)
  GeluBwd = 5,    // C = acc * aux  (aux = gelu'(u) from the forward)
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr;
  int64_t lda = 0;
  bool a_kmajor = true;  // A(i,k) = kmajor ? A[i*lda + k] : A[k*lda + i]
  const void* B = nullptr;
  int64_t ldb = 0;
  bool b_kmajor = false;  // B(k,j) = kmajor ? B[j*ldb + k] : B[k*ldb + j]
  DT ab = DT::F32;        // operand element type
  void* C = nullptr;
  int64_t ldc = 0;
  DT c = DT::F32;
  Epi epi = Epi::Store;
  const float* bias = nullptr;   // [N]
  const float* resid = nullptr;  // fp32, leading dim ldc
  void* aux = nullptr;           // operand type, leading dim ldc
  // K concatenation: C = epi(sum_s A_s B_s) over nseg operand pairs of the same
  // shape / layout (segment 0 is A, B); one accumulator, one output pass --
  // e.g. dX of LayerNorm-1 = dv Wv^T + dk Wk^T + dq Wq^T (tcgen05 path only)
  int nseg = 1;
  const void* A_seg[3] = {nullptr, nullptr, nullptr};
  const void* B_seg[3] = {nullptr, nullptr, nullptr};
  // split-K partials: caller-owned (engines pass their own, so engines sharing a
  // device never share partials); nullptr = a per-device scratch (debug / tests)
  float* ws = nullptr;
  size_t ws_floats = 0;
  // GeluBwd without split-K, M % 32 == 0: the epilogue also writes the column
  // sums of each 32-row block of the fp32 result (before the bf16 rounding) to
  // colsum_part[M / 32][N] -- the bias gradient's partials, read by colsum_parts
  float* colsum_part = nullptr;
};
// split-K partial floats any tcgen05 GEMM can need: splits * M * N <= the
// concurrent tile slots times one (pair) tile
constexpr size_t kGemmWsFloats = (size_t)148 * 128 * 256;

void gemm_simt(const GemmArgs& g, cudaStream_t st);
// true when gemm_tc runs g in one pass (no split-K), e.g. for colsum_part
bool gemm_tc_single_pass(const GemmArgs& g);
// tcgen05 + TMA path (bf16 operands); returns false when the shape/layout is
// outside what the kernel supports (caller falls back to gemm_simt only in
// tests -- the engine treats that as a configuration error).
bool gemm_tc(const GemmArgs& g, cudaStream_t st);
bool gemm_tc_supported(const GemmArgs& g);

}  // namespace photon
