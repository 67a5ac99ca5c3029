// gemm_tc.cu -- tcgen05 / TMA / TMEM GEMM for sm_100a.
//
// bf16 operands, fp32 accumulation in tensor memory, fused epilogues
// (gemm.cuh).  One CTA per SM, persistent over (tile, k-split) work units:
//   warp 0      TMA producer: 128B-swizzled A/B k-blocks into a STAGES-deep ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128,
//               N=BN, K=16) into one of two TMEM accumulators
//   warps 2..9  epilogue, two per TMEM lane quarter: tcgen05.ld 32x32 chunks,
//               fused bias / residual / GELU math in registers, st.shared into
//               a staging box and one TMA store per chunk; per-element inputs
//               (residual, GELU pre-activation, accumulate target) arrive by
//               TMA one chunk ahead.  The second accumulator lets the epilogue
//               of tile i overlap the main loop of tile i+1.
// Pair mode (NCTA = 2, cta_group::2): a 2-CTA cluster on one TPC computes a
// 256 x 256 tile; each CTA stages its own 128 rows of A and half of B, the
// leader issues M=256 MMAs that write each CTA's 128 accumulator rows into that
// CTA's TMEM, and completions are multicast to both CTAs.  Per-SM operand
// traffic through shared memory halves and the ring gets 5 stages.
// Operands may be K-major or MN-major (the three layouts of tensor.cpp:152-207
// on canonical [in,out] weights); both are legal UMMA smem layouts, so no
// transposes are materialised.  Small-tile GEMMs with a long contraction
// (weight gradients, K = B*S) are split along K into an fp32 workspace and
// reduced in a fixed order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <atomic>
#include <mutex>

#include "gemm.cuh"

#ifndef PHOTON_GELU_AS
#define PHOTON_GELU_AS 1  // 0: gelu_pair2_poly (one MUFU op per element; measured 0.7 % slower in the step)
#endif
namespace photon {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter, alternating 32-column chunks
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiBytesPerWarp = 8192;  // out 4 KB + in 4 KB
constexpr int kRingBudget = 232448 - kEpiWarps * kEpiBytesPerWarp - 2048;

struct OperandMaps {  // per K segment: A and B tensor maps
  CUtensorMap a[3];
  CUtensorMap b[3];
};

struct TcParams {
  int M, N, K;
  int num_m, num_n, splits, kb_total, kb_per_split, units;
  int kb_seg;  // k-blocks per operand segment (kb_total = nseg * kb_seg)
  int group_m;  // raster: bands of group_m M-tiles, N-tiles swept inside a band
  int epi;     // Epi
  int c_bf16;  // output dtype
  const float* bias;
  float* colsum_part;  // GeluBwd: per-32-row column sums [M / 32][N] (or nullptr)
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
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(su32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
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

// ---- cluster / CTA-pair wrappers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of `local` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(local)), "r"(rank));
  return r;
}
// Relaxed remote arrive: used only after this CTA's tcgen05.ld of the
// accumulator completed (wait::ld), so nothing the leader's next MMA
// overwrites is still being read; a release would cost a GPU-scope fence.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA load into this CTA's smem, completing on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on both CTAs' copy
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
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

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Grouped raster: the tiles in flight share a band of group_m row tiles of A
// (L2-resident) and sweep N inside it, so A streams from HBM about once.
__device__ __forceinline__ void tile_coords(const TcParams& p, int tile, int bm, int bn, int& m0,
                                            int& n0) {
  const int per_group = p.group_m * p.num_n;
  const int g = tile / per_group;
  const int first_m = g * p.group_m;
  const int gsz = min(p.group_m, p.num_m - first_m);
  const int r = tile - g * per_group;
  m0 = (first_m + r % gsz) * bm;
  n0 = (r / gsz) * bn;
}

// Staging offsets of 16-byte column chunk j of row `lane` in a TMA box of 32
// rows: bf16 rows are 64 B (SWIZZLE_64B), fp32 rows 128 B (SWIZZLE_128B);
// the XOR spreads the 32 lanes over all banks.
__device__ __forceinline__ uint32_t sw64_off(int lane, int j) {
  return lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
}
__device__ __forceinline__ uint32_t sw128_off(int lane, int j) {
  return lane * 128 + ((j ^ (lane & 7)) << 4);
}

// Epilogue tensor maps (row-major [M][N] boxes of 32 rows x 32 cols).
struct EpiMaps {
  CUtensorMap C;    // output (or split-K workspace, 3D [splits][M][N])
  CUtensorMap aux;  // gelu'(u) (bf16): stored by GeluBias, loaded by GeluBwd
  CUtensorMap in;   // fp32 residual (ResidBias) or C itself (Accum)
};

template <int BN, bool A_MN, bool B_MN, int NCTA>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ OperandMaps om,
                   const __grid_constant__ EpiMaps em, const TcParams p) {
  pdl_launch_dependents();
  constexpr int BNL = BN / NCTA;  // B rows (N) staged by this CTA
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BNL * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int STAGES = kRingBudget / STAGE_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulators
  // instruction descriptor: D f32, A/B bf16, majors, N, M = 128 * NCTA
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((BM * NCTA) >> 4) << 24);
  const uint32_t rank = NCTA == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int cid = blockIdx.x / NCTA, ncl = gridDim.x / NCTA;  // cluster id / count

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* epi_buf = smem + STAGES * STAGE_BYTES;  // [kEpiWarps][out in] x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_buf + kEpiWarps * kEpiBytesPerWarp);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;  // [kEpiWarps]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inbar + kEpiWarps);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const Epi epi = static_cast<Epi>(p.epi);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // pair: only the leader arrives (expecting both CTAs' bytes); the peer's
      // bytes complete on the leader's copy.  The peer refills a stage only
      // after the MMA consumed it, so its bytes never leak into an older phase.
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * NCTA);
    }
    for (int i = 0; i < kEpiWarps; ++i) mbar_init(&inbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&om.a[0])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&om.b[0])) : "memory");
  }
  if (warp == 1) {
    if (NCTA == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if (NCTA == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel visible from here

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      int stage = 0;
      uint32_t phase = 0;
      // bytes one CTA of the pair lands per k-block (MN-major 64-wide boxes
      // lying wholly past M / N are skipped: their smem is stale but only feeds
      // accumulator rows/cols that are never stored)
      auto stage_tx = [&](int mr, int nr) -> uint32_t {
        const int ab = A_MN ? max(0, min(BM / 64, (p.M - mr + 63) / 64)) : 1;
        const int bb = B_MN ? max(0, min(BNL / 64, (p.N - nr + 63) / 64)) : 1;
        return (A_MN ? ab * 8192 : A_BYTES) + (B_MN ? bb * 8192 : B_BYTES);
      };
      const uint32_t leader_full0 = NCTA == 2 ? mapa_rank(&full[0], 0) : 0;
      for (int u = cid; u < p.units; u += ncl) {
        const int tile = u / p.splits, split = u % p.splits;
        int m0, n0;
        tile_coords(p, tile, BM * NCTA, BN, m0, n0);
        const int mr = m0 + (int)rank * BM, nr = n0 + (int)rank * BNL;  // this CTA's slices
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        const int a_boxes = A_MN ? max(0, min(BM / 64, (p.M - mr + 63) / 64)) : 1;
        const int b_boxes = B_MN ? max(0, min(BNL / 64, (p.N - nr + 63) / 64)) : 1;
        const uint32_t tx = NCTA == 2 ? stage_tx(m0, n0) + stage_tx(m0 + BM, n0 + BNL)
                                      : stage_tx(mr, nr);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const int seg = kb / p.kb_seg;  // K-concatenated operand pair
          const int k0 = (kb - seg * p.kb_seg) * BK;
          const CUtensorMap* tmA = &om.a[seg];
          const CUtensorMap* tmB = &om.b[seg];
          if (NCTA == 1) {
            mbar_expect_tx(&full[stage], tx);
            if (!A_MN) {
              tma_load_2d(sa, tmA, &full[stage], k0, mr);
            } else {
              for (int c = 0; c < a_boxes; ++c) tma_load_2d(sa + c * 8192, tmA, &full[stage], mr + 64 * c, k0);
            }
            if (!B_MN) {
              tma_load_2d(sb, tmB, &full[stage], k0, nr);
            } else {
              for (int c = 0; c < b_boxes; ++c) tma_load_2d(sb + c * 8192, tmB, &full[stage], nr + 64 * c, k0);
            }
          } else {
            const uint32_t lbar = leader_full0 + stage * 8;  // leader's full[stage]
            if (leader) mbar_expect_tx(&full[stage], tx);   // its arrive + both CTAs' bytes
            if (!A_MN) {
              tma_load_2d_pair(sa, tmA, lbar, k0, mr);
            } else {
              for (int c = 0; c < a_boxes; ++c) tma_load_2d_pair(sa + c * 8192, tmA, lbar, mr + 64 * c, k0);
            }
            if (!B_MN) {
              tma_load_2d_pair(sb, tmB, lbar, k0, nr);
            } else {
              for (int c = 0; c < b_boxes; ++c) tma_load_2d_pair(sb + c * 8192, tmB, lbar, nr + 64 * c, k0);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ================= MMA issuer (pair leader) =================
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cid; u < p.units; u += ncl) {
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
            if (NCTA == 1) tc_mma(d, da, db, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
            else tc_mma_pair(d, da, db, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          // smem slot free once these MMAs retire
          if (NCTA == 1) tc_commit(&empty[stage]);
          else tc_commit_pair(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (NCTA == 1) tc_commit(&tfull[acc]);  // accumulator ready
        else tc_commit_pair(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue (warps 2..9) =================
    const int ew = warp - 2;
    const int q = warp & 3;     // TMEM lane quarter this warp may access
    const int sub = ew >> 2;    // this warp takes chunks c = sub, sub + 2, ...
    uint8_t* obuf = epi_buf + ew * kEpiBytesPerWarp;
    uint8_t* ibuf = obuf + 4096;
    uint64_t* ibar = inbar + ew;
    uint32_t in_phase = 0;
    const bool splitk = p.splits > 1;
    const bool need_in = !splitk && (epi == Epi::ResidBias || epi == Epi::Accum || epi == Epi::GeluBwd);
    const bool in_bf16 = epi == Epi::GeluBwd;
    const uint32_t in_bytes = in_bf16 ? 2048 : 4096;
    const CUtensorMap* in_map = in_bf16 ? &em.aux : &em.in;
    const bool out_bf16 = !splitk && p.c_bf16;
    int acc = 0;
    uint32_t acc_phase = 0;
    int stage_i = 0;  // epilogues without an input alternate two staging buffers (across tiles)
    const uint32_t leader_tempty0 = NCTA == 2 ? mapa_rank(&tempty[0], 0) : 0;
    for (int u = cid; u < p.units; u += ncl) {
      const int tile = u / p.splits, split = u % p.splits;
      int m0, n0;
      tile_coords(p, tile, BM * NCTA, BN, m0, n0);
      const int row0 = m0 + (int)rank * BM + q * 32;
      const bool rows_live = row0 < p.M;
      const int nchunks = min(BN / 32, (p.N - n0 + 31) / 32);
      if (need_in && rows_live && sub < nchunks && lane == 0) {  // overlaps the main loop
        mbar_expect_tx(ibar, in_bytes);
        tma_load_2d(ibuf, in_map, ibar, n0 + 32 * sub, row0);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      // bias of a chunk, loaded one chunk ahead: its global-load latency overlaps
      // the previous chunk instead of following the TMEM load
      const bool has_bias =
          !splitk && (epi == Epi::Bias || epi == Epi::ResidBias || epi == Epi::GeluBias);
      float4 bb[8];
      auto load_bias = [&](int col0) {
        if (col0 + 32 <= p.N) {
          const float4* b4 = reinterpret_cast<const float4*>(p.bias + col0);
#pragma unroll
          for (int j = 0; j < 8; ++j) bb[j] = b4[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            bb[j] = make_float4(col0 + 4 * j < p.N ? p.bias[col0 + 4 * j] : 0.f,
                                col0 + 4 * j + 1 < p.N ? p.bias[col0 + 4 * j + 1] : 0.f,
                                col0 + 4 * j + 2 < p.N ? p.bias[col0 + 4 * j + 2] : 0.f,
                                col0 + 4 * j + 3 < p.N ? p.bias[col0 + 4 * j + 3] : 0.f);
        }
      };
      if (has_bias && rows_live && sub < nchunks) load_bias(n0 + sub * 32);
      if (rows_live) {
#pragma unroll 1
        for (int c = sub; c < nchunks; c += 2, ++stage_i) {
          const int col0 = n0 + c * 32;
          float v[32];
          tmem_ld32(taddr + c * 32, v);  // v[j] = acc[row0 + lane][col0 + j]
          if (has_bias) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // packed adds (FADD2), same rounding
              const float2 lo = __fadd2_rn(make_float2(v[4 * j], v[4 * j + 1]), make_float2(bb[j].x, bb[j].y));
              const float2 hi =
                  __fadd2_rn(make_float2(v[4 * j + 2], v[4 * j + 3]), make_float2(bb[j].z, bb[j].w));
              v[4 * j] = lo.x;
              v[4 * j + 1] = lo.y;
              v[4 * j + 2] = hi.x;
              v[4 * j + 3] = hi.y;
            }
            if (c + 2 < nchunks) load_bias(col0 + 64);
          }
          if (need_in) {
            mbar_wait(ibar, in_phase);
            in_phase ^= 1;
            const uint32_t ia = su32(ibuf);
            if (in_bf16) {  // GeluBwd: v *= gelu'(u), stored by the forward
              uint32_t w[16];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 t = lds128(ia + sw64_off(lane, j));
                w[4 * j] = t.x;
                w[4 * j + 1] = t.y;
                w[4 * j + 2] = t.z;
                w[4 * j + 3] = t.w;
              }
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                v[2 * e] *= bf_lo(w[e]);
                v[2 * e + 1] *= bf_hi(w[e]);
              }
              // the shared loads are consumed (values used) before the async
              // proxy may overwrite the buffer
              __syncwarp();
              if (lane == 0 && c + 2 < nchunks) {
                mbar_expect_tx(ibar, in_bytes);
                tma_load_2d(ibuf, in_map, ibar, col0 + 64, row0);
              }
            } else {  // ResidBias: resid + (acc + bias);  Accum: C + acc
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint4 t = lds128(ia + sw128_off(lane, j));
                v[4 * j] += __uint_as_float(t.x);
                v[4 * j + 1] += __uint_as_float(t.y);
                v[4 * j + 2] += __uint_as_float(t.z);
                v[4 * j + 3] += __uint_as_float(t.w);
              }
              __syncwarp();
              if (lane == 0 && c + 2 < nchunks) {
                mbar_expect_tx(ibar, in_bytes);
                tma_load_2d(ibuf, in_map, ibar, col0 + 64, row0);
              }
            }
          }
          // stage the chunk once the previous store from this buffer has read it
          // (with two buffers the store of the previous chunk may still be reading)
          // GeluBwd (bf16 in, bf16 out: 2 KB chunks) alternates the two halves of obuf
          const bool two_bufs = !need_in || (in_bf16 && out_bf16);
          uint8_t* sbuf = (two_bufs && (stage_i & 1)) ? (need_in ? obuf + 2048 : ibuf) : obuf;
          if (lane == 0) {
            if (two_bufs) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          const uint32_t oa = su32(sbuf);
          if (epi == Epi::GeluBias && !splitk) {
            // one Phi / phi evaluation per element (one MUFU op): gelu'(u) = Phi + u phi -> aux box
            // (second 2 KB, the backward's factor), v <- gelu(u) = u Phi
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float gp[8];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                float2 g2, gp2;
#if PHOTON_GELU_AS
                gelu_pair2(make_float2(v[8 * j + e], v[8 * j + e + 1]), g2, gp2);
#else
                gelu_pair2_poly(make_float2(v[8 * j + e], v[8 * j + e + 1]), g2, gp2);
#endif
                v[8 * j + e] = g2.x;
                v[8 * j + e + 1] = g2.y;
                gp[e] = gp2.x;
                gp[e + 1] = gp2.y;
              }
              sts128(oa + 2048 + sw64_off(lane, j), pack2(gp[0], gp[1]), pack2(gp[2], gp[3]),
                     pack2(gp[4], gp[5]), pack2(gp[6], gp[7]));
            }
          }
          if (out_bf16) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              sts128(oa + sw64_off(lane, j), pack2(v[8 * j], v[8 * j + 1]),
                     pack2(v[8 * j + 2], v[8 * j + 3]), pack2(v[8 * j + 4], v[8 * j + 5]),
                     pack2(v[8 * j + 6], v[8 * j + 7]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              sts128(oa + sw128_off(lane, j), __float_as_uint(v[4 * j]),
                     __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                     __float_as_uint(v[4 * j + 3]));
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (splitk) {
              tma_store_3d(&em.C, sbuf, col0, row0, split);
            } else {
              tma_store_2d(&em.C, sbuf, col0, row0);
              if (epi == Epi::GeluBias) tma_store_2d(&em.aux, sbuf + 2048, col0, row0);
            }
            bulk_commit();
          }
          if (epi == Epi::GeluBwd && p.colsum_part) {
            // column sums of this warp's 32 rows: a butterfly reduce-scatter
            // leaves column (col0 + lane) in v[0] of lane `lane`
#pragma unroll
            for (int w = 16; w >= 1; w >>= 1) {
              const bool up = lane & w;
#pragma unroll
              for (int i = 0; i < w; ++i) {
                const float send = up ? v[i] : v[i + w];
                const float keep = up ? v[i + w] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
              }
            }
            if (col0 + lane < p.N) p.colsum_part[(size_t)(row0 >> 5) * p.N + col0 + lane] = v[0];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // this CTA's accumulator rows are drained
        if (NCTA == 1 || leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_remote(leader_tempty0 + acc * 8);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  if (NCTA == 2) cluster_sync_all();  // no remote arrive / multicast still in flight
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (NCTA == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
  }
}

// split-K: out = epi(sum_s ws[s]) in fixed order (ws[s] is [M][N] fp32)
struct ReduceArgs {
  int M, N, splits, epi, c_bf16;
  int64_t ldc;
  const float* ws;
  void* C;
  const float* bias;
  const float* resid;
  void* aux;
};
__global__ void splitk_reduce_kernel(const ReduceArgs r) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t total = (int64_t)r.M * r.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < r.splits; ++s) acc += r.ws[s * total + i];
    const int row = (int)(i / r.N), col = (int)(i % r.N);
    const int64_t o = (int64_t)row * r.ldc + col;
    const float b = r.bias ? r.bias[col] : 0.f;
    float out;
    switch (static_cast<Epi>(r.epi)) {
      case Epi::Store: out = acc; break;
      case Epi::Accum: out = static_cast<const float*>(r.C)[o] + acc; break;
      case Epi::Bias: out = acc + b; break;
      case Epi::ResidBias: out = r.resid[o] + (acc + b); break;
      case Epi::GeluBias:
        static_cast<bf16*>(r.aux)[o] = __float2bfloat16_rn(gelu_grad_f(acc + b));
        out = gelu_f(acc + b);
        break;
      default:
        out = acc * __bfloat162float(static_cast<const bf16*>(r.aux)[o]);
        break;
    }
    if (r.c_bf16) static_cast<bf16*>(r.C)[o] = __float2bfloat16_rn(out);
    else static_cast<float*>(r.C)[o] = out;
  }
}

// The weight-gradient case (Store into fp32, N % 4 == 0): 16-byte accesses, the
// split partials of a float4 loaded together and added in split order (the
// same order as splitk_reduce_kernel, so the result is unchanged).
__global__ void splitk_reduce_store4_kernel(const float* __restrict__ ws, int M, int N, int splits,
                                            float* __restrict__ C, int64_t ldc) {
  pdl_launch_dependents();
  pdl_wait();
  const int n4 = N / 4;
  const int64_t total4 = (int64_t)M * n4, total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(ws)[i];
    int s = 1;
    for (; s + 3 < splits; s += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = reinterpret_cast<const float4*>(ws + (s + u) * total)[i];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(ws + s * total)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const int64_t row = i / n4, c4 = i - row * n4;
    *reinterpret_cast<float4*>(C + row * ldc + 4 * c4) = acc;
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

CUtensorMap encode(CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                   const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, dt, rank, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(PHOTON_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// operand: 2D bf16 [outer][inner] (row stride ld), box {64, box_outer}, 128B swizzle
CUtensorMap operand_map(const void* base, uint64_t inner, uint64_t outer, int64_t ld,
                        uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  return encode(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B);
}

// epilogue tile: row-major [M][N] (row stride ld), box {32 cols, 32 rows},
// swizzled to match sw64_off / sw128_off
CUtensorMap epi_map(const void* base, bool bf, uint64_t N, uint64_t M, int64_t ld) {
  cuuint64_t dims[2] = {N, M};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (bf ? 2 : 4)};
  cuuint32_t box[2] = {32, 32};
  return encode(bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base,
                dims, strides, box, bf ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, bool A_MN, bool B_MN, int NCTA>
void launch(const OperandMaps& om, const EpiMaps& em, const TcParams& p, int grid, cudaStream_t st) {
  constexpr int STAGE_BYTES = (BM + BN / NCTA) * BK * 2;
  constexpr int STAGES = kRingBudget / STAGE_BYTES;
  static_assert(STAGES >= 3, "operand ring too shallow");
  constexpr int SMEM = STAGES * STAGE_BYTES + kEpiWarps * kEpiBytesPerWarp + 1024 + 512;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, NCTA>;
  static std::atomic<uint64_t> configured{0};  // per device
  int dev = 0;
  PH_CUDA(cudaGetDevice(&dev));
  if (!(configured.load() & (1ull << (dev & 63)))) {
    PH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    configured.fetch_or(1ull << (dev & 63));
  }
  if (NCTA == 1) {
    launch_pdl_cls(kPdlGemm, kern, grid, kThreads, SMEM, st, om, em, p);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see launch_pdl
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_class_on(kPdlGemm) ? 2 : 1;
    PH_CUDA(cudaLaunchKernelEx(&cfg, kern, om, em, p));
  }
  PH_LAUNCH_CHECK();
}

// split-K partials, per device (launches on one device are stream-ordered by
// their engine; the buffer only grows)
float* workspace(size_t n) {
  static std::mutex mu;
  static float* ptr[64] = {};
  static size_t cap[64] = {};
  int dev = 0;
  PH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (n > cap[dev]) {
    if (ptr[dev]) cudaFree(ptr[dev]);
    ptr[dev] = nullptr;
    PH_CUDA(cudaMalloc(&ptr[dev], n * sizeof(float)));
    cap[dev] = n;
  }
  return ptr[dev];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.ab != DT::BF16) return false;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return false;
  if ((g.lda & 7) || (g.ldb & 7)) return false;  // TMA: 16-byte row strides
  if (!aligned16(g.A) || !aligned16(g.B) || !aligned16(g.C)) return false;
  for (int s = 1; s < g.nseg; ++s)
    if (!aligned16(g.A_seg[s]) || !aligned16(g.B_seg[s])) return false;
  if ((g.ldc * (g.c == DT::BF16 ? 2 : 4)) & 15) return false;
  if ((g.epi == Epi::GeluBias || g.epi == Epi::GeluBwd) && (g.c != DT::BF16 || !aligned16(g.aux)))
    return false;
  if (g.epi == Epi::ResidBias && (g.c != DT::F32 || !aligned16(g.resid))) return false;
  if (g.epi == Epi::Accum && g.c != DT::F32) return false;
  if ((g.epi == Epi::Bias || g.epi == Epi::ResidBias || g.epi == Epi::GeluBias) &&
      (!g.bias || !aligned16(g.bias)))
    return false;
  return true;
}

namespace {
int pair_env() {
  static const int v = [] {
    const char* e = std::getenv("PHOTON_GEMM_PAIR");  // 0 never, 1 by shape, 2 always
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
// split-K factor of a shape (1 = single pass): the tile grid cannot fill the
// chip and the contraction is long
int split_count(int M, int N, int K, int nseg, int ncta, int BN) {
  const int slots = kNumSMs / ncta;
  const int tiles = ((M + BM * ncta - 1) / (BM * ncta)) * ((N + BN - 1) / BN);
  const int kb_total = ((K + BK - 1) / BK) * nseg;
  int splits = 1;
  if (tiles < slots && kb_total >= 16) {
    splits = std::min(slots / tiles, kb_total / 8);
    splits = std::max(1, std::min(splits, 16));
  }
  const int per = (kb_total + splits - 1) / splits;
  return (kb_total + per - 1) / per;
}
int cta_count(const GemmArgs& g, int BN) {
  const bool pair_ok = BN == 256 && g.M > BM;
  return (pair_env() == 2 || (pair_env() == 1 && pair_ok)) && BN == 256 && g.M > BM ? 2 : 1;
}
}  // namespace

bool gemm_tc_single_pass(const GemmArgs& g) {
  const int BN = g.N <= 128 ? 128 : 256;
  return gemm_tc_supported(g) && split_count(g.M, g.N, g.K, g.nseg, cta_count(g, BN), BN) == 1;
}

bool gemm_tc(const GemmArgs& g, cudaStream_t st) {
  if (!gemm_tc_supported(g)) return false;
  const int BN = g.N <= 128 ? 128 : 256;
  // CTA pairs (256 x 256 tiles) wherever N is a 256 multiple-ish and M spans
  // more than one 128-row tile: wide tiles without split-K, and the split-K
  // weight gradients (d x d, d x 4d, 4d x d: 25-30% faster than single-CTA
  // 128 x 256 tiles in tools/gemm_bench.py).
  const int ncta = cta_count(g, BN);
  const int slots = kNumSMs / ncta;  // concurrent tile workers
  TcParams p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.num_m = (g.M + BM * ncta - 1) / (BM * ncta);
  p.num_n = (g.N + BN - 1) / BN;
  if (g.nseg < 1 || g.nseg > 3 || (g.nseg > 1 && g.K % BK))
    throw Error(PHOTON_ERR_USAGE, "gemm_tc: K segments need 1..3 segments of whole k-blocks");
  p.kb_seg = (g.K + BK - 1) / BK;
  p.kb_total = p.kb_seg * g.nseg;
  const int tiles = p.num_m * p.num_n;
  const int splits = split_count(g.M, g.N, g.K, g.nseg, ncta, BN);
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.units = tiles * p.splits;
  static const int group_env = [] {
    const char* e = std::getenv("PHOTON_GEMM_GROUP");
    return e ? std::atoi(e) : -1;
  }();
  // measured on the 125M shapes: bands of 8 row tiles, 32 for very wide N
  const int group = group_env >= 0 ? group_env : (p.num_n >= 64 ? 32 : 8);
  p.group_m = std::max(1, std::min(group > 0 ? group : p.num_m, p.num_m));
  p.epi = static_cast<int>(g.epi);
  p.c_bf16 = g.c == DT::BF16;
  p.bias = g.bias;
  p.colsum_part = g.colsum_part;
  if (g.colsum_part && (g.epi != Epi::GeluBwd || p.splits > 1 || g.M % 32))
    throw Error(PHOTON_ERR_USAGE, "gemm_tc: fused column sums need GeluBwd, no split-K, M % 32 == 0");

  EpiMaps em{};
  float* ws = nullptr;
  if (p.splits > 1) {
    const size_t need = (size_t)p.splits * g.M * g.N;
    ws = g.ws && g.ws_floats >= need ? g.ws : workspace(need);
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)p.splits};
    cuuint64_t strides[2] = {(cuuint64_t)g.N * 4, (cuuint64_t)g.N * g.M * 4};
    cuuint32_t box[3] = {32, 32, 1};
    em.C = encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ws, dims, strides, box,
                  CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    em.C = epi_map(g.C, g.c == DT::BF16, g.N, g.M, g.ldc);
    if (g.epi == Epi::GeluBias || g.epi == Epi::GeluBwd) em.aux = epi_map(g.aux, true, g.N, g.M, g.ldc);
    if (g.epi == Epi::ResidBias) em.in = epi_map(g.resid, false, g.N, g.M, g.ldc);
    if (g.epi == Epi::Accum) em.in = epi_map(g.C, false, g.N, g.M, g.ldc);
  }

  OperandMaps om;
  for (int sgi = 0; sgi < g.nseg; ++sgi) {
    const void* A = sgi == 0 ? g.A : g.A_seg[sgi];
    const void* B = sgi == 0 ? g.B : g.B_seg[sgi];
    // A(i,k): K-major -> [M][K] rows; MN-major -> [K][M] rows
    om.a[sgi] = g.a_kmajor ? operand_map(A, g.K, g.M, g.lda, BM) : operand_map(A, g.M, g.K, g.lda, 64);
    // B(k,j): K-major -> [N][K] rows; N-major -> [K][N] rows
    om.b[sgi] = g.b_kmajor ? operand_map(B, g.K, g.N, g.ldb, BN / ncta)
                           : operand_map(B, g.N, g.K, g.ldb, 64);
  }
  const int grid = std::min(p.units, slots) * ncta;
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  if (BN == 128) {
    if (!amn && !bmn) launch<128, false, false, 1>(om, em, p, grid, st);
    else if (!amn && bmn) launch<128, false, true, 1>(om, em, p, grid, st);
    else if (amn && !bmn) launch<128, true, false, 1>(om, em, p, grid, st);
    else launch<128, true, true, 1>(om, em, p, grid, st);
  } else if (ncta == 1) {
    if (!amn && !bmn) launch<256, false, false, 1>(om, em, p, grid, st);
    else if (!amn && bmn) launch<256, false, true, 1>(om, em, p, grid, st);
    else if (amn && !bmn) launch<256, true, false, 1>(om, em, p, grid, st);
    else launch<256, true, true, 1>(om, em, p, grid, st);
  } else {
    if (!amn && !bmn) launch<256, false, false, 2>(om, em, p, grid, st);
    else if (!amn && bmn) launch<256, false, true, 2>(om, em, p, grid, st);
    else if (amn && !bmn) launch<256, true, false, 2>(om, em, p, grid, st);
    else launch<256, true, true, 2>(om, em, p, grid, st);
  }
  if (p.splits > 1) {
    if (g.epi == Epi::Store && !p.c_bf16 && g.N % 4 == 0 && g.ldc % 4 == 0 && aligned16(g.C)) {
      launch_pdl(splitk_reduce_store4_kernel, kNumSMs * 4, 256, 0, st, ws, g.M, g.N, p.splits,
                                                               static_cast<float*>(g.C), g.ldc);
    } else {
      ReduceArgs r{g.M, g.N, p.splits, p.epi, p.c_bf16, g.ldc, ws, g.C, g.bias, g.resid, g.aux};
      launch_pdl(splitk_reduce_kernel, kNumSMs * 4, 256, 0, st, r);
    }
    PH_LAUNCH_CHECK();
  }
  return true;
}

}  // namespace photon
