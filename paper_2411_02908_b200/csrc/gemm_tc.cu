// gemm_tc.cu -- tcgen05 / TMA / TMEM GEMM for sm_100a.
//
// bf16 operands, fp32 accumulation in tensor memory, fused epilogues
// (gemm.cuh).  One CTA per SM, persistent over (tile, k-split) work units:
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a STAGES-deep ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128,
//               N=BN, K=16) into one of two TMEM accumulators
//   warps 2..5  epilogue: tcgen05.ld accumulator rows -> registers -> fused
//               bias / residual / GELU -> global, overlapped with the next
//               tile's main loop through the second accumulator
// Operands may be K-major or MN-major (the three layouts of tensor.cpp:152-207
// on canonical [in,out] weights); both are legal UMMA smem layouts, so no
// transposes are materialised.  Small-tile GEMMs with a long contraction
// (weight gradients, K = B*S) are split along K into an fp32 workspace and
// reduced in a fixed order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm.cuh"

namespace photon {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 192;
constexpr int kSmemBudget = 196608;  // operand ring bytes

struct TcParams {
  int M, N, K;
  int num_m, num_n, splits, kb_total, kb_per_split, units;
  int epi;     // Epi
  int c_bf16;  // output dtype
  void* C;
  int64_t ldc;
  const float* bias;
  const float* resid;
  void* aux;
  float* ws;  // split-K partials [splits][M][N]
};

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version bits.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ---- epilogue -------------------------------------------------------------------
__device__ __forceinline__ void store_vals(const TcParams& p, int row, int col0, const float* v,
                                           int n) {
  // v[0..n) -> columns [col0, col0+n) of row, applying p.epi
  const int64_t o = (int64_t)row * p.ldc + col0;
  const bool vec = (n == 32) && ((p.ldc & 7) == 0) && ((col0 & 7) == 0);
  const Epi epi = static_cast<Epi>(p.epi);
  float r[32];
  switch (epi) {
    case Epi::Store:
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = v[i];
      break;
    case Epi::Accum:
      for (int i = 0; i < n; ++i) r[i] = static_cast<float*>(p.C)[o + i] + v[i];
      break;
    case Epi::Bias:
      for (int i = 0; i < n; ++i) r[i] = v[i] + p.bias[col0 + i];
      break;
    case Epi::ResidBias:
      for (int i = 0; i < n; ++i) r[i] = p.resid[o + i] + (v[i] + p.bias[col0 + i]);
      break;
    case Epi::GeluBias: {
      bf16* aux = static_cast<bf16*>(p.aux);
      for (int i = 0; i < n; ++i) {
        const float pre = v[i] + p.bias[col0 + i];
        aux[o + i] = __float2bfloat16_rn(pre);
        r[i] = gelu_f(pre);
      }
      break;
    }
    case Epi::GeluBwd: {
      const bf16* aux = static_cast<const bf16*>(p.aux);
      for (int i = 0; i < n; ++i) r[i] = v[i] * gelu_grad_f(__bfloat162float(aux[o + i]));
      break;
    }
  }
  if (p.c_bf16) {
    bf16* C = static_cast<bf16*>(p.C) + o;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 pk;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(r[i], r[i + 1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(r[i + 2], r[i + 3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(r[i + 4], r[i + 5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(r[i + 6], r[i + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&t0);
        pk.y = *reinterpret_cast<uint32_t*>(&t1);
        pk.z = *reinterpret_cast<uint32_t*>(&t2);
        pk.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(C + i) = pk;
      }
    } else {
      for (int i = 0; i < n; ++i) C[i] = __float2bfloat16_rn(r[i]);
    }
  } else {
    float* C = static_cast<float*>(p.C) + o;
    if (vec && ((p.ldc & 3) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(C + i) = make_float4(r[i], r[i + 1], r[i + 2], r[i + 3]);
    } else {
      for (int i = 0; i < n; ++i) C[i] = r[i];
    }
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const TcParams p) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int STAGES = kSmemBudget / STAGE_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulators
  // instruction descriptor: D f32, A/B bf16, majors, N, M = 128
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int tile = u / p.splits, split = u % p.splits;
        const int m0 = (tile % p.num_m) * BM, n0 = (tile / p.num_m) * BN;
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          // MN-major 64-wide boxes lying wholly past M / N are skipped: their
          // smem is stale but only feeds accumulator rows/cols never stored.
          const int a_boxes = A_MN ? min(BM / 64, (p.M - m0 + 63) / 64) : 1;
          const int b_boxes = B_MN ? min(BN / 64, (p.N - n0 + 63) / 64) : 1;
          mbar_expect_tx(&full[stage], (A_MN ? a_boxes * 8192 : A_BYTES) +
                                           (B_MN ? b_boxes * 8192 : B_BYTES));
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          } else {
            for (int c = 0; c < a_boxes; ++c) tma_load_2d(sa + c * 8192, &tmA, &full[stage], m0 + 64 * c, k0);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          } else {
            for (int c = 0; c < b_boxes; ++c) tma_load_2d(sb + c * 8192, &tmB, &full[stage], n0 + 64 * c, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer =================
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int split = u % p.splits;
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = su32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = A_MN ? sw128_desc(sa + kk * 2048, 8192, 1024)
                                     : sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? sw128_desc(sb + kk * 2048, 8192, 1024)
                                     : sw128_desc(sb + kk * 32, 16, 1024);
            tc_mma(d, da, db, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);  // accumulator ready
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue (warps 2..5) =================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int tile = u / p.splits, split = u % p.splits;
      const int m0 = (tile % p.num_m) * BM, n0 = (tile / p.num_m) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(taddr + c0, v);
        const int col0 = n0 + c0;
        if (row < p.M && col0 < p.N) {
          const int n = min(32, p.N - col0);
          if (p.splits > 1) {
            float* w = p.ws + ((int64_t)split * p.M + row) * p.N + col0;
            if (n == 32 && (p.N & 3) == 0) {
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(w + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
              for (int i = 0; i < n; ++i) w[i] = v[i];
            }
          } else {
            store_vals(p, row, col0, v, n);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// split-K: out = epi(sum_s ws[s]) in fixed order
__global__ void splitk_reduce_kernel(const TcParams p) {
  const int64_t total = (int64_t)p.M * p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s) acc += p.ws[s * total + i];
    const int row = (int)(i / p.N), col = (int)(i % p.N);
    float v[32];
    v[0] = acc;
    store_vals(p, row, col, v, 1);
  }
}

// ---- host side ----------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw Error(PHOTON_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D bf16 tensor [outer][inner] (inner contiguous, row stride ld elements),
// box {64, box_outer}, 128B swizzle, zero fill out of bounds.
CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, int64_t ld,
                     uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(PHOTON_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int BN, bool A_MN, bool B_MN>
void launch(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, int grid,
            cudaStream_t st) {
  constexpr int STAGE_BYTES = (BM + BN) * BK * 2;
  constexpr int STAGES = kSmemBudget / STAGE_BYTES;
  constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  static bool configured = false;
  if (!configured) {
    PH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    configured = true;
  }
  kern<<<grid, kThreads, SMEM, st>>>(a, b, p);
  PH_LAUNCH_CHECK();
}

struct Workspace {
  float* ptr = nullptr;
  size_t n = 0;
  std::mutex mu;
};
Workspace g_ws;

float* workspace(size_t n) {
  std::lock_guard<std::mutex> lk(g_ws.mu);
  if (n > g_ws.n) {
    if (g_ws.ptr) cudaFree(g_ws.ptr);
    g_ws.ptr = nullptr;
    PH_CUDA(cudaMalloc(&g_ws.ptr, n * sizeof(float)));
    g_ws.n = n;
  }
  return g_ws.ptr;
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.ab != DT::BF16) return false;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return false;
  if ((g.lda & 7) || (g.ldb & 7)) return false;  // TMA: 16-byte row strides
  if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15))
    return false;
  if ((g.epi == Epi::GeluBias || g.epi == Epi::GeluBwd) && g.c != DT::BF16) return false;
  return true;
}

bool gemm_tc(const GemmArgs& g, cudaStream_t st) {
  if (!gemm_tc_supported(g)) return false;
  const int BN = g.N <= 128 ? 128 : 256;
  TcParams p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.num_m = (g.M + BM - 1) / BM;
  p.num_n = (g.N + BN - 1) / BN;
  p.kb_total = (g.K + BK - 1) / BK;
  const int tiles = p.num_m * p.num_n;
  // split-K when the tile grid cannot fill the chip and the contraction is long
  int splits = 1;
  if (tiles < kNumSMs && p.kb_total >= 16) {
    splits = std::min(kNumSMs / tiles, p.kb_total / 8);
    splits = std::max(1, std::min(splits, 16));
  }
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.units = tiles * p.splits;
  p.epi = static_cast<int>(g.epi);
  p.c_bf16 = g.c == DT::BF16;
  p.C = g.C;
  p.ldc = g.ldc;
  p.bias = g.bias;
  p.resid = g.resid;
  p.aux = g.aux;
  if (p.splits > 1) p.ws = workspace((size_t)p.splits * g.M * g.N);

  // A(i,k): K-major -> [M][K] rows; MN-major -> [K][M] rows
  const CUtensorMap ta = g.a_kmajor ? make_map(g.A, g.K, g.M, g.lda, BM)
                                    : make_map(g.A, g.M, g.K, g.lda, 64);
  // B(k,j): K-major -> [N][K] rows; N-major -> [K][N] rows
  const CUtensorMap tb = g.b_kmajor ? make_map(g.B, g.K, g.N, g.ldb, BN)
                                    : make_map(g.B, g.N, g.K, g.ldb, 64);
  const int grid = std::min(p.units, kNumSMs);
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  if (BN == 128) {
    if (!amn && !bmn) launch<128, false, false>(ta, tb, p, grid, st);
    else if (!amn && bmn) launch<128, false, true>(ta, tb, p, grid, st);
    else if (amn && !bmn) launch<128, true, false>(ta, tb, p, grid, st);
    else launch<128, true, true>(ta, tb, p, grid, st);
  } else {
    if (!amn && !bmn) launch<256, false, false>(ta, tb, p, grid, st);
    else if (!amn && bmn) launch<256, false, true>(ta, tb, p, grid, st);
    else if (amn && !bmn) launch<256, true, false>(ta, tb, p, grid, st);
    else launch<256, true, true>(ta, tb, p, grid, st);
  }
  if (p.splits > 1) {
    splitk_reduce_kernel<<<kNumSMs * 4, 256, 0, st>>>(p);
    PH_LAUNCH_CHECK();
  }
  return true;
}

}  // namespace photon
