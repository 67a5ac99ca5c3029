// attn_tc.cu -- causal attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// One CTA per (128-query tile, batch*head), two CTAs per SM (80 KB smem,
// 256 TMEM columns each) so one CTA's softmax overlaps the other's MMAs; 6 warps:
//   warp 0     TMA producer: Q once, K/V 128-key tiles into a 2-stage ring
//   warp 1     MMA issuer (one thread): S_j = Q K_j^T (M128 N128 K64) into
//              TMEM, then O += P_{j-1} V_{j-1} (M128 N64 K128) with P read
//              from TMEM (tcgen05.mma A-from-TMEM form)
//   warps 2-5  softmax, thread = query row (its TMEM lane): tcgen05.ld the
//              score row, causal mask, online max/sum in the exp2 domain
//              (one FFMA + EX2 per score), P as packed bf16 via tcgen05.st;
//              O is rescaled in TMEM only when the running max grows by more
//              than 2^8 (lazy rescale), final O / l and the log-sum-exp out.
// Semantics are those of tensor.cpp:436-542 (scale 1/sqrt(dh) before the max,
// keys j <= i); the lse feeds the (deterministic) backward in attn_mma.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kernels.cuh"

namespace photon {
namespace k {

namespace {

constexpr int TQ = 128, TK = 128;  // query / key tile (head dims 64 and 128 are templates)

// Opt-in timeline instrumentation (PHOTON_BUILD_TRACE=1): clock64 stamps of one
// mid-grid CTA, event e of iteration it at g_attn_trace[e * 64 + it].
#ifdef PHOTON_ATTN_TRACE
__device__ unsigned long long g_attn_trace[64 * 64];
#define ATTN_TRACE(e, it)                                                             \
  do {                                                                                \
    if (blockIdx.x == 0 && blockIdx.y == 200 && (it) < 64)                            \
      g_attn_trace[(e) * 64 + (it)] = clock64();                                      \
  } while (0)
// persistent kernels: CTA 0, global pair index g
#define ATTN_TRACE_P(e, g)                                                            \
  do {                                                                                \
    if (blockIdx.x == 0 && (g) < 64) g_attn_trace[(e) * 64 + (g)] = clock64();        \
  } while (0)
// the latest of all callers (e.g. every softmax warp's lane 0)
#define ATTN_TRACE_MAX(e, g)                                                          \
  do {                                                                                \
    if (blockIdx.x == 0 && (g) < 64)                                                  \
      atomicMax(&g_attn_trace[(e) * 64 + (g)], (unsigned long long)clock64());        \
  } while (0)
#else
#define ATTN_TRACE_P(e, g) \
  do {                     \
  } while (0)
#define ATTN_TRACE_MAX(e, g) \
  do {                       \
  } while (0)
#define ATTN_TRACE(e, it) \
  do {                    \
  } while (0)
#endif
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThresh = 8.0f;  // log2 units

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
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
      "{\n.reg .pred p;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n}\n" ::"r"(su32(b)),
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
// L2 eviction-priority policies for TMA loads / stores (createpolicy)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void st_hint_u4(void* p, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint64_t sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
#define TMEM_LD32(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),             \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),          \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),          \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),          \
        "=r"(r[31])                                                                             \
      : "r"(taddr))
#define TMEM_ST32(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"   \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"( \
          taddr),                                                                               \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),        \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),      \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),      \
      "r"(r[29]), "r"(r[30]), "r"(r[31])                                                        \
      : "memory")
#define TMEM_LD8(taddr, r)                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"          \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),         \
                 "=r"(r[6]), "=r"(r[7])                                                          \
               : "r"(taddr))
#define TMEM_ST8(taddr, r)                                                                      \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(   \
                   taddr),                                                                       \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),      \
               "r"(r[7])                                                                         \
               : "memory")
#define TMEM_LD16(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
      "%14,%15}, [%16];"                                                                        \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),             \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                   \
      : "r"(taddr))
#define TMEM_ST16(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"   \
      "%13,%14,%15,%16};" ::"r"(taddr),                                                         \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),        \
      "r"(r[15])                                                                                \
      : "memory")
// CPT consecutive fp32 columns of this thread's lane
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int c = 0; c < N / 32; ++c) TMEM_LD32(taddr + c * 32, (r + c * 32));
  if constexpr (N % 32 == 16) TMEM_LD16(taddr + (N / 32) * 32, (r + (N / 32) * 32));
}
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* r) {
#pragma unroll
  for (int c = 0; c < N / 32; ++c) TMEM_ST32(taddr + c * 32, (r + c * 32));
  if constexpr (N % 32 >= 16) TMEM_ST16(taddr + (N / 32) * 32, (r + (N / 32) * 32));
  if constexpr (N % 16 == 8) TMEM_ST8(taddr + (N / 16) * 16, (r + (N / 16) * 16));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {  // FMNMX3 (sm_100)
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2 without range fix-up
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifndef PHOTON_FWD_FMA_PRE
#define PHOTON_FWD_FMA_PRE 0  // the same for the pre-wait chunk (0: none)
#endif
#ifndef PHOTON_FWD_FMA_EXP
#define PHOTON_FWD_FMA_EXP 8  // every 8th pair of the P loops on the FMA pipe (0: none)
#endif
// (measured at the 125M shape: 1/8 of the main loop's pairs 0.357-0.367 ms vs
// 0.365-0.381 with none, 1/4 0.359, 1/2 0.372, 1/16 0.369; also in the pre-wait
// chunk: no better)
constexpr int kFmaExp = PHOTON_FWD_FMA_EXP, kFmaExpMod = kFmaExp > 0 ? kFmaExp : 1;
constexpr int kFmaPre = PHOTON_FWD_FMA_PRE, kFmaPreMod = kFmaPre > 0 ? kFmaPre : 1;
__device__ __forceinline__ float4 lds_f4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(su32(p)));
  return v;
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

struct FwdArgs {
  int S, H, d;
  float sl2;  // scale * log2(e)
  bf16* o;
  float* lse;
};

// A from TMEM ("TS" form): D[tmem] += A[tmem] * B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// TMEM columns per CTA: S [0,128) fp32 scores, P [128,192) bf16x2, O [192,256).
constexpr uint32_t kColS = 0, kColP = 128, kColO = 192;
// forward K ring depth: a TMA load under the forward's traffic takes up to ~5k
// cycles (clock64 trace), more than two tiles of softmax (last session: 2 stages
// 0.353-0.361 ms, 3 0.351-0.355, 4 0.564 -- one CTA per SM at head dim 64)
#ifndef PHOTON_FWD_NKF
#define PHOTON_FWD_NKF 3
#endif
constexpr int NKF = PHOTON_FWD_NKF;
#ifndef PHOTON_FWD_PRE
#define PHOTON_FWD_PRE 1
#endif
constexpr int kFwdPre = PHOTON_FWD_PRE;  // 32-score chunks of P computed before the PV wait

#ifndef PHOTON_FWD_CHUNK_MB
#define PHOTON_FWD_CHUNK_MB 64
#endif
constexpr int64_t kFwdChunkBytes = (int64_t)PHOTON_FWD_CHUNK_MB << 20;

template <int HD>
__global__ void __launch_bounds__(kThreads, HD == 64 ? 2 : 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const FwdArgs a) {
  pdl_launch_dependents();
  // smem: Q | K[2] | V[2] | barriers; 16 KB tiles at HD = 64 (two CTAs per SM),
  // 32 KB at HD = 128 (one CTA per SM, 512 TMEM columns)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  constexpr int NA = HD / 64, TB = 16384 * NA;  // 64-column swizzle atoms per row, tile bytes
  constexpr uint32_t kColO_ = HD == 64 ? kColO : 256, kCols = HD == 64 ? 256 : 512;
  uint8_t* sQ = sm;
  uint8_t* sK = sm + TB;         // [NKF]
  uint8_t* sV = sK + NKF * TB;   // [2]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * TB);
  // K and V have separate rings: a K stage is free once S_j retires, a V stage
  // once PV_j retires, so K_{j+2} streams in while PV_j is still running
  uint64_t* q_full = bar;
  uint64_t* s_full = bar + 1;
  uint64_t* s_empty = bar + 2;
  uint64_t* p_full = bar + 3;
  uint64_t* o_done = bar + 4;    // one completion per PV_j
  uint64_t* v_full = bar + 5;    // [2]
  uint64_t* v_empty = bar + 7;   // [2]
  uint64_t* k_full = bar + 9;    // [NKF]
  uint64_t* k_empty = k_full + NKF;  // [NKF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(k_empty + NKF);

  const int nqt = (a.S + TQ - 1) / TQ;
  // dispatch order (x fastest): chunks of heads whose K / V total kFwdChunkBytes,
  // in a chunk the heaviest query tile of every head first, then the next
  // heaviest, ... -- the grid's last CTAs are light ones (no long tail), and a
  // chunk's K / V stay in L2 while its tiles run (125M shape: 128 heads per
  // chunk, 0.376 -> 0.350 ms; 1.3B heads: 64)
  int qt, bh;
  {
    const int chunk = max(1, (int)(kFwdChunkBytes / ((int64_t)a.S * HD * 4)));
    const int L = blockIdx.x + blockIdx.y * nqt, per = chunk * nqt;
    const int c0 = L / per * chunk, r = L % per, cg = min(chunk, (int)gridDim.y - c0);
    qt = nqt - 1 - r / cg;
    bh = c0 + r % cg;
  }
  const int b = bh / a.H, h = bh % a.H;
  const int q0 = qt * TQ;
  const int row_base = b * a.S;
  const int n_kt = (q0 + TQ - 1) / TK + 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NKF; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        su32(tmem_slot)), "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel visible from here

  if (warp == 0) {
    if (lane == 0) {  // ===== producer: Q, then the K ring =====
      mbar_expect_tx(q_full, TB);
      for (int t = 0; t < NA; ++t)
        tma_load_2d(sQ + t * 16384, &tq, q_full, h * HD + 64 * t, row_base + q0);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % NKF;
        mbar_wait(&k_empty[st], ((j / NKF) & 1) ^ 1);
        ATTN_TRACE(0, j);
        mbar_expect_tx(&k_full[st], TB);
        for (int t = 0; t < NA; ++t)
          tma_load_2d(sK + st * TB + t * 16384, &tk, &k_full[st], h * HD + 64 * t, row_base + j * TK);
      }
    } else if (lane == 1) {  // ===== producer: the V ring =====
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], TB);
        for (int t = 0; t < NA; ++t)
          tma_load_2d(sV + st * TB + t * 16384, &tv, &v_full[st], h * HD + 64 * t, row_base + j * TK);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      constexpr uint32_t IDS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TK >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      constexpr uint32_t IDO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TQ >> 4) << 24);
      mbar_wait(q_full, 0);
      const uint32_t aq = su32(sQ);
      auto issue_pv = [&](int j) {
        const int st = j & 1;
        mbar_wait(&v_full[st], (j >> 1) & 1);
        mbar_wait(p_full, j & 1);
        ATTN_TRACE(2, j);
        fence_after();
        const uint32_t bv = su32(sV + st * TB);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)  // 16 keys = 8 packed bf16x2 TMEM columns
          mma_ts(tmem + kColO_, tmem + kColP + kk * 8, sw128(bv + kk * 2048, 16384, 1024), IDO,
                 (j > 0 || kk > 0) ? 1u : 0u);
        commit(o_done);
        commit(&v_empty[st]);
      };
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % NKF;
        mbar_wait(&k_full[st], (j / NKF) & 1);
        mbar_wait(s_empty, (j & 1) ^ 1);  // softmax holds S_{j-1} in registers
        ATTN_TRACE(1, j);
        fence_after();
        const uint32_t bk = su32(sK + st * TB);  // st: K stage
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma(tmem + kColS, sw128(aq + off, 16, 1024), sw128(bk + off, 16, 1024), IDS,
              kk > 0 ? 1u : 0u);
        }
        commit(s_full);
        commit(&k_empty[st]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kt - 1);
    }
  } else {
    // ===== softmax: thread = query row r (its TMEM lane) =====
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int qrow = q0 + r;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = a.sl2;
    float m = -INFINITY, l = 0.f;  // m in log2 units
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(s_full, j & 1);
      if (warp == 2 && lane == 0) ATTN_TRACE(5, j);
      fence_after();
      uint32_t s[TK];
#pragma unroll
      for (int c = 0; c < TK / 32; ++c) TMEM_LD32(tmem + lane_off + kColS + c * 32, (s + c * 32));
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      const int k0 = j * TK;
      if (k0 + TK > q0) {  // diagonal / tail tile: causal and length mask
#pragma unroll
        for (int i = 0; i < TK; ++i)
          if (k0 + i > qrow || k0 + i >= a.S) s[i] = __float_as_uint(-INFINITY);
      }
      // raw-score max (scale > 0 keeps the order): eight independent chains
      // instead of one 128-deep dependent chain on the softmax's critical path
      // (three-input FMNMX3: two new scores per instruction)
      float mxs[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mxs[u] = __uint_as_float(s[u]);
#pragma unroll
      for (int i = 8; i < TK; i += 2)
        mxs[(i >> 1) & 7] = fmax3(mxs[(i >> 1) & 7], __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
      float mx = fmax3(fmax3(mxs[0], mxs[1], mxs[2]), fmax3(mxs[3], mxs[4], mxs[5]),
                       fmaxf(mxs[6], mxs[7]));
      mx *= sl2;
      // lazy rescale: keep the stale max unless it grew by > 2^8
      float scale = 1.f;
      bool rescale = false;
      if (mx > m + kRescaleThresh || m == -INFINITY) {
        if (m != -INFINITY) {
          scale = exp2f(m - mx);
          rescale = true;
        }
        m = mx;
      }
      if (warp == 2 && lane == 0) ATTN_TRACE(6, j);
      // the first kFwdPre 32-score chunks of P are computed before waiting for
      // PV_{j-1}, so their exponentials overlap that product
      float2 rs2 = make_float2(0.f, 0.f);
      uint32_t pre[kFwdPre * 16 + 1];
#pragma unroll
      for (int c = 0; c < kFwdPre; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // packed FFMA2 / FADD2: half the issue slots of the scale and the sum
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[c * 32 + 2 * i]),
                                                  __uint_as_float(s[c * 32 + 2 * i + 1])),
                                      make_float2(sl2, sl2), make_float2(-m, -m));
          float2 e2;
          if (kFmaPre > 0 && i % kFmaPreMod == kFmaPreMod - 1)
            e2 = ex2_fma2(x);
          else
            e2 = make_float2(ex2(x.x), ex2(x.y));
          rs2 = __fadd2_rn(rs2, e2);
          pre[c * 16 + i] = pk(e2.x, e2.y);
        }
      // P and O are free once PV_{j-1} retired
      if (j >= 1) mbar_wait(o_done, (j - 1) & 1);
      if (warp == 2 && lane == 0) ATTN_TRACE(7, j);
      fence_after();
      if (__any_sync(0xffffffffu, rescale)) {  // 8 columns at a time: s[] stays in registers
#pragma unroll 1
        for (int c = 0; c < HD / 8; ++c) {
          uint32_t u[8];
          TMEM_LD8(tmem + lane_off + kColO_ + c * 8, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * scale);
          TMEM_ST8(tmem + lane_off + kColO_ + c * 8, u);
        }
      }
      l *= scale;
      // P = exp2(s*sl2 - m) -> bf16 pairs into TMEM columns [128, 192)
#pragma unroll
      for (int c = 0; c < kFwdPre; ++c) TMEM_ST16(tmem + lane_off + kColP + c * 16, (pre + c * 16));
#pragma unroll
      for (int c = kFwdPre; c < 4; ++c) {
        uint32_t pp[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // packed FFMA2 / FADD2: half the issue slots of the scale and the sum
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[c * 32 + 2 * i]),
                                                  __uint_as_float(s[c * 32 + 2 * i + 1])),
                                      make_float2(sl2, sl2), make_float2(-m, -m));
          float2 e2;
          if (kFmaExp > 0 && i % kFmaExpMod == kFmaExpMod - 1)
            e2 = ex2_fma2(x);  // part of the exponentials off the MUFU pipe
          else
            e2 = make_float2(ex2(x.x), ex2(x.y));
          rs2 = __fadd2_rn(rs2, e2);
          pp[i] = pk(e2.x, e2.y);
        }
        TMEM_ST16(tmem + lane_off + kColP + c * 16, pp);
      }
      l += rs2.x + rs2.y;
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (warp == 2 && lane == 0) ATTN_TRACE(8, j);
    }
    // final: O / l, log-sum-exp
    mbar_wait(o_done, (n_kt - 1) & 1);
    fence_after();
    const float inv = 1.f / l;
    bf16* orow = a.o + (int64_t)(row_base + qrow) * a.d + h * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t u[32];
      TMEM_LD32(tmem + lane_off + kColO_ + c * 32, u);
      tmem_wait_ld();
      if (qrow < a.S) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(orow + c * 32 + i) =
              make_uint4(pk(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv),
                         pk(__uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv),
                         pk(__uint_as_float(u[i + 4]) * inv, __uint_as_float(u[i + 5]) * inv),
                         pk(__uint_as_float(u[i + 6]) * inv, __uint_as_float(u[i + 7]) * inv));
      }
    }
    if (qrow < a.S) a.lse[(int64_t)bh * a.S + qrow] = m * kLn2 + logf(l);
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

// ============================================================================
// Backward.  prep: D = rowsum(dO * O) and lse in log2 units into padded
// [B*H][Spad] arrays (pad: lse = +inf -> P = 0, D = 0), so every 128-query
// slice is an in-bounds 512-byte bulk copy.
// ============================================================================
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}

// D = dO . O per (row, head).  A warp takes RPW rows of one head at a time
// (lane = row within the group x 16-byte vector of the head's columns, so each
// load instruction reads whole 128-byte lines), four groups per iteration with
// all loads issued before the first product; the VPH lanes of a row sum their
// partial dot products with butterfly shuffles and the row's first lane writes
// D and lse (log2 units) -- consecutive rows of one head, so the writes into the
// [B*H][Spad] arrays and the lse reads are contiguous.
template <int HD>
__global__ void attn_bwd_prep_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dO,
                                     const float* __restrict__ lse, float* __restrict__ Lp,
                                     float* __restrict__ Dp, int B, int S, int H, int d, int Spad,
                                     uint32_t* __restrict__ sync, int nsync) {
  pdl_launch_dependents();
  pdl_wait();
  if (sync && blockIdx.x == 0)
    for (int i = threadIdx.x; i < nsync; i += blockDim.x) sync[i] = 0u;
  constexpr int VPH = HD / 8;     // 16-byte vectors per head row
  constexpr int RPW = 32 / VPH;   // rows per warp instruction
  constexpr int U = 4;            // row groups in flight per lane
  const int lane = threadIdx.x & 31, vec = lane % VPH, rsub = lane / VPH;
  const int warps = blockDim.x / 32;
  const int groups = (S + RPW * U - 1) / (RPW * U);  // per head
  const int64_t items = (int64_t)B * H * groups;
  for (int64_t it = (int64_t)blockIdx.x * warps + threadIdx.x / 32; it < items;
       it += (int64_t)gridDim.x * warps) {
    const int bh = (int)(it / groups), g = (int)(it % groups);
    const int b = bh / H, h = bh % H;
    uint4 xs[U], ys[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = (g * U + u) * RPW + rsub;
      if (i < S) {
        const int64_t off = ((int64_t)(b * S + i) * d + h * HD) / 8 + vec;
        xs[u] = reinterpret_cast<const uint4*>(o)[off];
        ys[u] = reinterpret_cast<const uint4*>(dO)[off];
      } else {
        xs[u] = ys[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t xw[4] = {xs[u].x, xs[u].y, xs[u].z, xs[u].w};
      const uint32_t yw[4] = {ys[u].x, ys[u].y, ys[u].z, ys[u].w};
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc = fmaf(__uint_as_float(xw[e] << 16), __uint_as_float(yw[e] << 16), acc);
        acc = fmaf(__uint_as_float(xw[e] & 0xffff0000u), __uint_as_float(yw[e] & 0xffff0000u), acc);
      }
#pragma unroll
      for (int off = 1; off < VPH; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      const int i = (g * U + u) * RPW + rsub;
      if (vec == 0 && i < S) {
        Dp[(int64_t)bh * Spad + i] = acc;
        Lp[(int64_t)bh * Spad + i] = lse[(int64_t)bh * S + i] * kLog2e;
      }
    }
  }
  // padded query slots: P = 0 (lse = +inf) and D = 0
  const int64_t npad = (int64_t)B * H * (Spad - S);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < npad; t += stride) {
    const int64_t bh = t / (Spad - S), i = S + t % (Spad - S);
    Lp[bh * Spad + i] = INFINITY;
    Dp[bh * Spad + i] = 0.f;
  }
}

struct BwdArgs {
  int S, H, d, Spad, BH;
  float sl2, scale;
  const float* Lp;
  const float* Dp;
  bf16* g0;  // dk (dkdv kernel) or dq (dq kernel)
  bf16* g1;  // dv
  // optional column sums (the q / k / v bias gradients' partials): per
  // 32-row block of a sequence, [B * nblk][d] for g0 and g1 (nullptr = none)
  float* s0;
  float* s1;
  int nblk;
  // fused backward: g0 = dq, g1 = dk, g2 = dv (sums s0 / s1 / s2), and the fp32
  // dQ accumulator [BH][ntq][HD/4][128] float4
  bf16* g2;
  float* s2;
  float* dqa;
  // fused backward's cross-CTA schedule words (zeroed by the prep kernel):
  // sync[0] = CTA ticket, sync[1 + bh] = "head bh's first part done" flag
  uint32_t* sync;
};

// producer, MMA, SWB softmax warps: SWB/4 warps per TMEM lane quarter, each on
// CPT = 128 / (SWB/4) columns of the score tile
#ifndef PHOTON_ATTN_SWB
#define PHOTON_ATTN_SWB 16
#endif
constexpr int SWB = PHOTON_ATTN_SWB;
constexpr int NCG = SWB / 4;       // column groups
constexpr int CPT = 128 / NCG;     // score columns per thread
constexpr int kBwdThreads = 64 + SWB * 32;
// Ring depth of the streamed operand (Q/dO/L/D in dK/dV, K/V in dQ).  A stage is
// held until the tile's gradient MMAs retire, and a TMA load under the full
// backward's memory traffic takes ~2.5-3.6k cycles (clock64 traces): two stages
// left the MMA issuer waiting on loads; four cover the latency.
#ifndef PHOTON_ATTN_NR
#define PHOTON_ATTN_NR 4
#endif
constexpr int NR = PHOTON_ATTN_NR;
// dQ pass (HD = 64): K/V ring depth (32 KB stages; up to 5 fit).  clock64
// traces show a K/V load taking ~4.5 k cycles under the backward's L2 traffic,
// but 5 stages (and, in dK/dV, one K/V buffer with 5 Q/dO stages) measured the
// same as 4 -- the loads are not what paces the passes.
#ifndef PHOTON_ATTN_NRQ
#define PHOTON_ATTN_NRQ 4
#endif
constexpr int NRQ64 = PHOTON_ATTN_NRQ;
// dK/dV pass (HD = 64): K/V buffers (2 = the next key tile prefetched) and the
// Q/dO ring depth that fits beside them
#ifndef PHOTON_ATTN_NKV
#define PHOTON_ATTN_NKV 2
#endif
constexpr int NKV64 = PHOTON_ATTN_NKV;
#ifndef PHOTON_ATTN_NR64
#define PHOTON_ATTN_NR64 NR
#endif
constexpr int NR64 = PHOTON_ATTN_NR64;

// Store N columns of a row of a 64-column fp32 TMEM accumulator (thread = row)
// as bf16 into the head slice.
// Store N columns of a row of an fp32 TMEM accumulator (thread = row), scaled
// by `mul`, as bf16 into the head slice; f keeps the scaled fp32 values (0 for
// a dead row) for warp_colsum.
template <int N>
__device__ __forceinline__ void store_acc_rows(uint32_t taddr, bf16* row_ptr, float mul, bool live,
                                               float (&f)[N], uint64_t policy = 0) {
  uint32_t u[N];
  if constexpr (N == 32) TMEM_LD32(taddr, u);
  else TMEM_LD16(taddr, u);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < N; ++i) f[i] = live ? __uint_as_float(u[i]) * mul : 0.f;
  if (live) {
#pragma unroll
    for (int i = 0; i < N; i += 8) {
      const uint4 w = make_uint4(pk(f[i], f[i + 1]), pk(f[i + 2], f[i + 3]), pk(f[i + 4], f[i + 5]),
                                 pk(f[i + 6], f[i + 7]));
      if (policy) st_hint_u4(row_ptr + i, w, policy);
      else *reinterpret_cast<uint4*>(row_ptr + i) = w;
    }
  }
}
// Column sums of the warp's 32 rows of f (the bias gradients' partials): a
// butterfly reduce-scatter leaves column `lane` in f[0] of lanes < N, which
// write part[lane].  Runs after the accumulator is released to the MMA warp.
template <int N>
__device__ __forceinline__ void warp_colsum(float (&f)[N], float* part) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = N / 2; w >= 1; w >>= 1) {
    const bool up = lane & w;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? f[i] : f[i + w];
      const float keep = up ? f[i + w] : f[i];
      f[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
#pragma unroll
  for (int w = N; w < 32; w <<= 1) f[0] += __shfl_xor_sync(0xffffffffu, f[0], w);
  if (lane < N) part[lane] = f[0];
}

// Both backward kernels are persistent (one CTA per SM): a CTA walks a static
// list of units, each unit = the tile pair (p, n-1-p) of one head, whose costs
// (number of 128 x 128 tile pairs) add up to the same n+1 -- so a round-robin
// over units balances to ~1 %, and the units of a head are adjacent, so the
// CTAs running concurrently share their heads' Q/dO/K/V in L2.  Tile i+1's K/V
// (resp. Q/dO) stream in while tile i finishes; the accumulators are drained by
// the softmax warps while the MMA issuer already computes the next tile's S.
#define PH_FOR_TILES(ntile)                                                    \
  for (int u = blockIdx.x; u < a.BH * (((ntile) + 1) / 2); u += gridDim.x)     \
    for (int hf = 0; hf < 2; ++hf)                                             \
      if (const int npair_ = ((ntile) + 1) / 2, p_ = u % npair_,               \
          tile = hf ? (ntile) - 1 - p_ : p_, bh = u / npair_;                  \
          !(hf && tile == p_))

// ---- dK, dV: 128-key tiles; keys are the TMEM lanes -------------------------------
// TMEM at HD = 64 (128-query tiles):
//   S^T [0,128)  dP^T [128,256)  P^T [256,320)  dS^T [320,384)  dV [384,448)  dK [448,512)
// at HD = 128 (64-query tiles):
//   S^T [0,64)   dP^T [64,128)   P^T [128,160)  dS^T [160,192)  dV [256,384)  dK [384,512)
template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                            const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                            const BwdArgs a) {
  pdl_launch_dependents();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  // HD = 128: 64-query tiles so that S^T, dP^T, P^T, dS^T, dV and dK all fit in TMEM
  constexpr int NA = HD / 64, KB = 16384 * NA;  // swizzle atoms per row, K/V tile bytes
  constexpr int TQB = HD == 64 ? 128 : 64, QB = TQB * 128 * NA, QA = TQB * 128;  // Q tile, atom
  constexpr int CPQ = TQB / NCG, GPH = HD / NCG;  // score / accumulator columns per thread
  constexpr int NKV = HD == 64 ? NKV64 : 1;       // K/V buffers (the next tile's prefetch)
  constexpr int NRK = HD == 64 ? NR64 : NR;       // Q/dO/L/D ring depth
  constexpr uint32_t colDP = TQB, colP = 2 * TQB, colDS = colP + TQB / 2, colDV = 512 - 2 * HD,
                     colDK = 512 - HD;
  uint8_t* sK = sm;               // [NKV]
  uint8_t* sV = sK + NKV * KB;    // [NKV]
  uint8_t* sQ = sV + NKV * KB;    // [NRK]
  uint8_t* sO = sQ + NRK * QB;     // [NRK] dO
  float* sL = reinterpret_cast<float*>(sO + NRK * QB);  // [NRK][TQB]
  float* sD = sL + NRK * TQB;                           // [NRK][TQB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + NRK * TQB);
  uint64_t* kv_full = bar;                 // [NKV]
  uint64_t* kv_empty = bar + NKV;          // [NKV]
  uint64_t* q_full = bar + 2 * NKV;        // [NRK]
  uint64_t* q_empty = q_full + NRK;         // [NRK]
  uint64_t* s_full = q_empty + NRK;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_full + 2;
  uint64_t* g_done = s_full + 3;
  uint64_t* acc_empty = s_full + 4;        // dK/dV drained by the softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

  const int nkt = (a.S + TK - 1) / TK, ntq = (a.S + TQB - 1) / TQB;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NKV; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < NRK; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, SWB);
    mbar_init(p_full, SWB);
    mbar_init(g_done, 1);
    mbar_init(acc_empty, SWB);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel visible from here

  if (warp == 0) {
    if (lane == 0) {
      int ti = 0, gi = 0;
      PH_FOR_TILES(nkt) {
        const int kt = tile, b = bh / a.H, h = bh % a.H, row_base = b * a.S;
        const int qt0 = kt * (TK / TQB), n_it = ntq - qt0;
        const int kb = ti % NKV;
        mbar_wait(&kv_empty[kb], ((ti / NKV) & 1) ^ 1);
        mbar_expect_tx(&kv_full[kb], 2 * KB);
        for (int t = 0; t < NA; ++t) {
          tma_load_2d(sK + kb * KB + t * 16384, &tk, &kv_full[kb], h * HD + 64 * t, row_base + kt * TK);
          tma_load_2d(sV + kb * KB + t * 16384, &tv, &kv_full[kb], h * HD + 64 * t, row_base + kt * TK);
        }
        for (int it = 0; it < n_it; ++it, ++gi) {
          const int st = gi % NRK, qt = qt0 + it;
          mbar_wait(&q_empty[st], ((gi / NRK) & 1) ^ 1);
          ATTN_TRACE_P(0, gi);
          mbar_expect_tx(&q_full[st], 2 * QB + 8 * TQB);
          for (int t = 0; t < NA; ++t) {
            tma_load_2d(sQ + st * QB + t * QA, &tq, &q_full[st], h * HD + 64 * t, row_base + qt * TQB);
            tma_load_2d(sO + st * QB + t * QA, &tdo, &q_full[st], h * HD + 64 * t, row_base + qt * TQB);
          }
          bulk_load(sL + st * TQB, a.Lp + (int64_t)bh * a.Spad + qt * TQB, 4 * TQB, &q_full[st]);
          bulk_load(sD + st * TQB, a.Dp + (int64_t)bh * a.Spad + qt * TQB, 4 * TQB, &q_full[st]);
        }
        ++ti;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TQB >> 3) << 17) |
                               ((uint32_t)(TK >> 4) << 24);
      constexpr uint32_t IDG = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TK >> 4) << 24);
      // gradients of pair g (its ring stage, whether it opens its tile, the tile index)
      auto issue_grads = [&](int g, int st, bool first, int t) {
        mbar_wait(p_full, g & 1);
        ATTN_TRACE_P(3, g);
        if (first && t > 0) mbar_wait(acc_empty, (t - 1) & 1);  // previous dK/dV drained
        fence_after();
        const uint32_t bo = su32(sO + st * QB), bq = su32(sQ + st * QB);
#pragma unroll
        for (int kk = 0; kk < TQB / 16; ++kk)  // dV += P^T dO (dO MN-major, QA-byte panels)
          mma_ts(tmem + colDV, tmem + colP + kk * 8, sw128(bo + kk * 2048, QA, 1024), IDG,
                 (!first || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < TQB / 16; ++kk)  // dK += dS^T Q
          mma_ts(tmem + colDK, tmem + colDS + kk * 8, sw128(bq + kk * 2048, QA, 1024), IDG,
                 (!first || kk > 0) ? 1u : 0u);
        commit(g_done);
        commit(&q_empty[st]);
      };
      int ti = 0, gi = 0;
      int pend = -1, pend_st = 0, pend_t = 0;
      bool pend_first = false;
      PH_FOR_TILES(nkt) {
        (void)bh;
        const int kt = tile, qt0 = kt * (TK / TQB), n_it = ntq - qt0;
        const int kb = ti % NKV;
        mbar_wait(&kv_full[kb], (ti / NKV) & 1);
        const uint32_t ak = su32(sK + kb * KB), av = su32(sV + kb * KB);
        for (int it = 0; it < n_it; ++it, ++gi) {
          const int st = gi % NRK;
          mbar_wait(&q_full[st], (gi / NRK) & 1);
          ATTN_TRACE_P(1, gi);
          mbar_wait(s_empty, (gi & 1) ^ 1);
          ATTN_TRACE_P(2, gi);
          fence_after();
          const uint32_t bq = su32(sQ + st * QB), bo = su32(sO + st * QB);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // S^T = K Q^T
            const uint32_t oa = (kk >> 2) * 16384 + (kk & 3) * 32, ob = (kk >> 2) * QA + (kk & 3) * 32;
            mma(tmem + 0, sw128(ak + oa, 16, 1024), sw128(bq + ob, 16, 1024), IDS, kk > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // dP^T = V dO^T
            const uint32_t oa = (kk >> 2) * 16384 + (kk & 3) * 32, ob = (kk >> 2) * QA + (kk & 3) * 32;
            mma(tmem + colDP, sw128(av + oa, 16, 1024), sw128(bo + ob, 16, 1024), IDS,
                kk > 0 ? 1u : 0u);
          }
          commit(s_full);
          if (it == n_it - 1) commit(&kv_empty[kb]);  // this tile's K/V no longer read
          if (pend >= 0) issue_grads(pend, pend_st, pend_first, pend_t);
          pend = gi;
          pend_st = st;
          pend_first = it == 0;
          pend_t = ti;
        }
        ++ti;
      }
      if (pend >= 0) issue_grads(pend, pend_st, pend_first, pend_t);
    }
  } else {
    const int q = warp & 3, cg = (warp - 2) >> 2;  // lane quarter, query-column group
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int gi = 0;
    PH_FOR_TILES(nkt) {
      const int kt = tile, b = bh / a.H, h = bh % a.H, row_base = b * a.S;
      const int qt0 = kt * (TK / TQB), n_it = ntq - qt0;
      const int key = kt * TK + r;
      const bool key_live = key < a.S;
      for (int it = 0; it < n_it; ++it, ++gi) {
        const int st = gi % NRK, q0 = (qt0 + it) * TQB;
        mbar_wait(&q_full[st], (gi / NRK) & 1);  // L, D of this query tile visible
        mbar_wait(s_full, gi & 1);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(5, gi);
        fence_after();
        uint32_t s[CPQ], dp[CPQ];
        tmem_ld_cols<CPQ>(tmem + lane_off + cg * CPQ, s);
        tmem_ld_cols<CPQ>(tmem + lane_off + colDP + cg * CPQ, dp);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(6, gi);
        if (lane == 0) ATTN_TRACE_MAX(4, gi);
        const float* L = sL + st * TQB + cg * CPQ;
        const float* D = sD + st * TQB + cg * CPQ;
        // masking only where this key tile meets the diagonal or the sequence end
        const bool masked = (kt * TK + TK > q0) || (kt * TK + TK > a.S);
        uint32_t pp[CPQ / 2], dd[CPQ / 2];
        // dS^T is kept unscaled (the softmax scale is applied to dK at the store)
#pragma unroll
        for (int i = 0; i < CPQ / 4; ++i) {
          const float4 l4 = lds_f4(L + 4 * i), d4 = lds_f4(D + 4 * i);
          float p0 = ex2(fmaf(__uint_as_float(s[4 * i]), a.sl2, -l4.x));
          float p1 = ex2(fmaf(__uint_as_float(s[4 * i + 1]), a.sl2, -l4.y));
          float p2 = ex2(fmaf(__uint_as_float(s[4 * i + 2]), a.sl2, -l4.z));
          float p3 = ex2(fmaf(__uint_as_float(s[4 * i + 3]), a.sl2, -l4.w));
          if (masked) {
            const int qc = q0 + cg * CPQ + 4 * i;
            p0 = (key_live && key <= qc) ? p0 : 0.f;
            p1 = (key_live && key <= qc + 1) ? p1 : 0.f;
            p2 = (key_live && key <= qc + 2) ? p2 : 0.f;
            p3 = (key_live && key <= qc + 3) ? p3 : 0.f;
          }
          pp[2 * i] = pk(p0, p1);
          pp[2 * i + 1] = pk(p2, p3);
          dd[2 * i] = pk(p0 * (__uint_as_float(dp[4 * i]) - d4.x),
                         p1 * (__uint_as_float(dp[4 * i + 1]) - d4.y));
          dd[2 * i + 1] = pk(p2 * (__uint_as_float(dp[4 * i + 2]) - d4.z),
                             p3 * (__uint_as_float(dp[4 * i + 3]) - d4.w));
        }
        if (warp == 2 && lane == 0) ATTN_TRACE_P(7, gi);
        if (gi >= 1) mbar_wait(g_done, (gi - 1) & 1);  // P^T / dS^T columns free
        if (warp == 2 && lane == 0) ATTN_TRACE_P(8, gi);
        fence_after();
        tmem_st_cols<CPQ / 2>(tmem + lane_off + colP + cg * (CPQ / 2), pp);
        tmem_st_cols<CPQ / 2>(tmem + lane_off + colDS + cg * (CPQ / 2), dd);
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(9, gi);
      }
      // the tile's dK / dV are complete once its last gradient MMAs retire
      mbar_wait(g_done, (gi - 1) & 1);
      fence_after();
      const int64_t row = (int64_t)(row_base + key) * a.d + h * HD + cg * GPH;
      // the warp's 32 keys are one column-sum block (if any of them is live)
      const bool sums = a.s0 && kt * TK + q * 32 < a.S;
      const int64_t prow = ((int64_t)b * a.nblk + kt * (TK / 32) + q) * a.d + h * HD + cg * GPH;
      float fk[GPH], fv[GPH];
      store_acc_rows<GPH>(tmem + lane_off + colDK + cg * GPH, a.g0 + row, a.scale, key_live, fk);  // dK
      store_acc_rows<GPH>(tmem + lane_off + colDV + cg * GPH, a.g1 + row, 1.f, key_live, fv);      // dV
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (sums) {
        warp_colsum<GPH>(fk, a.s0 + prow);
        warp_colsum<GPH>(fv, a.s1 + prow);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---- dQ: 128-query tiles; queries are the TMEM lanes --------------------------------
// TMEM: S [0,128)  dP [128,256)  dS [256,320)  dQ [320,320+HD)
template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                          const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                          const BwdArgs a) {
  pdl_launch_dependents();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  constexpr int NA = HD / 64, KB = 16384 * NA;  // swizzle atoms per row, tile bytes
  constexpr int NRQ = HD == 64 ? NRQ64 : 2;      // K/V ring depth within 227 KB
  constexpr int NQO = HD == 64 ? 2 : 1;          // Q/dO buffers (the next tile's prefetch)
  constexpr int GPH = HD / NCG;
  uint8_t* sQ = sm;                // [NQO]
  uint8_t* sO = sQ + NQO * KB;     // [NQO]
  uint8_t* sK = sO + NQO * KB;     // [NRQ]
  uint8_t* sV = sK + NRQ * KB;     // [NRQ]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + NRQ * KB);
  uint64_t* qo_full = bar;                 // [NQO]
  uint64_t* qo_empty = bar + NQO;          // [NQO]
  uint64_t* kv_full = bar + 2 * NQO;       // [NRQ]
  uint64_t* kv_empty = kv_full + NRQ;      // [NRQ]
  uint64_t* s_full = kv_empty + NRQ;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_full + 2;
  uint64_t* g_done = s_full + 3;
  uint64_t* acc_empty = s_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

  const int nqt = (a.S + TQ - 1) / TQ;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NQO; ++i) {
      mbar_init(&qo_full[i], 1);
      mbar_init(&qo_empty[i], 1);
    }
    for (int i = 0; i < NRQ; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, SWB);
    mbar_init(p_full, SWB);
    mbar_init(g_done, 1);
    mbar_init(acc_empty, SWB);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel visible from here

  if (warp == 0) {
    if (lane == 0) {
      int ti = 0, gj = 0;
      PH_FOR_TILES(nqt) {
        const int qt = tile, b = bh / a.H, h = bh % a.H, row_base = b * a.S;
        const int qb = ti % NQO;
        mbar_wait(&qo_empty[qb], ((ti / NQO) & 1) ^ 1);
        mbar_expect_tx(&qo_full[qb], 2 * KB);
        for (int t = 0; t < NA; ++t) {
          tma_load_2d(sQ + qb * KB + t * 16384, &tq, &qo_full[qb], h * HD + 64 * t, row_base + qt * TQ);
          tma_load_2d(sO + qb * KB + t * 16384, &tdo, &qo_full[qb], h * HD + 64 * t, row_base + qt * TQ);
        }
        for (int j = 0; j <= qt; ++j, ++gj) {
          const int st = gj % NRQ;
          mbar_wait(&kv_empty[st], ((gj / NRQ) & 1) ^ 1);
          ATTN_TRACE_P(10, gj);
          mbar_expect_tx(&kv_full[st], 2 * KB);
          for (int t = 0; t < NA; ++t) {
            tma_load_2d(sK + st * KB + t * 16384, &tk, &kv_full[st], h * HD + 64 * t, row_base + j * TK);
            tma_load_2d(sV + st * KB + t * 16384, &tv, &kv_full[st], h * HD + 64 * t, row_base + j * TK);
          }
        }
        ++ti;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TK >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      constexpr uint32_t IDG = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TQ >> 4) << 24);
      auto issue_dq = [&](int g, int st, bool first, int t) {
        mbar_wait(p_full, g & 1);
        ATTN_TRACE_P(13, g);
        if (first && t > 0) mbar_wait(acc_empty, (t - 1) & 1);  // previous dQ drained
        fence_after();
        const uint32_t bk = su32(sK + st * KB);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)  // dQ += dS K (K MN-major, 16 KB panels)
          mma_ts(tmem + 320, tmem + 256 + kk * 8, sw128(bk + kk * 2048, 16384, 1024), IDG,
                 (!first || kk > 0) ? 1u : 0u);
        commit(g_done);
        commit(&kv_empty[st]);
      };
      int ti = 0, gj = 0;
      int pend = -1, pend_st = 0, pend_t = 0;
      bool pend_first = false;
      PH_FOR_TILES(nqt) {
        (void)bh;
        const int qt = tile, qb = ti % NQO;
        mbar_wait(&qo_full[qb], (ti / NQO) & 1);
        const uint32_t aq = su32(sQ + qb * KB), ao = su32(sO + qb * KB);
        for (int j = 0; j <= qt; ++j, ++gj) {
          const int st = gj % NRQ;
          mbar_wait(&kv_full[st], (gj / NRQ) & 1);
          ATTN_TRACE_P(11, gj);
          mbar_wait(s_empty, (gj & 1) ^ 1);
          ATTN_TRACE_P(12, gj);
          fence_after();
          const uint32_t bk = su32(sK + st * KB), bv = su32(sV + st * KB);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // S = Q K^T
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma(tmem + 0, sw128(aq + off, 16, 1024), sw128(bk + off, 16, 1024), IDS, kk > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // dP = dO V^T
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma(tmem + 128, sw128(ao + off, 16, 1024), sw128(bv + off, 16, 1024), IDS,
                kk > 0 ? 1u : 0u);
          }
          commit(s_full);
          if (j == qt) commit(&qo_empty[qb]);  // this tile's Q/dO no longer read
          if (pend >= 0) issue_dq(pend, pend_st, pend_first, pend_t);
          pend = gj;
          pend_st = st;
          pend_first = j == 0;
          pend_t = ti;
        }
        ++ti;
      }
      if (pend >= 0) issue_dq(pend, pend_st, pend_first, pend_t);
    }
  } else {
    const int q = warp & 3, cg = (warp - 2) >> 2;  // lane quarter, key-column group
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int gj = 0;
    PH_FOR_TILES(nqt) {
      const int qt = tile, b = bh / a.H, h = bh % a.H, row_base = b * a.S;
      const int q0 = qt * TQ, qrow = q0 + r;
      const float L = a.Lp[(int64_t)bh * a.Spad + qrow];
      const float D = a.Dp[(int64_t)bh * a.Spad + qrow];
      for (int j = 0; j <= qt; ++j, ++gj) {
        mbar_wait(s_full, gj & 1);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(15, gj);
        fence_after();
        uint32_t s[CPT], dp[CPT];
        tmem_ld_cols<CPT>(tmem + lane_off + cg * CPT, s);
        tmem_ld_cols<CPT>(tmem + lane_off + 128 + cg * CPT, dp);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(16, gj);
        if (lane == 0) ATTN_TRACE_MAX(14, gj);
        const int k0 = j * TK + cg * CPT;
        const bool masked = (j * TK + TK > q0) || (j * TK + TK > a.S);
        uint32_t dd[CPT / 2];  // dS unscaled (the softmax scale is applied to dQ at the store)
#pragma unroll
        for (int i = 0; i < CPT / 2; ++i) {
          float p0 = ex2(fmaf(__uint_as_float(s[2 * i]), a.sl2, -L));
          float p1 = ex2(fmaf(__uint_as_float(s[2 * i + 1]), a.sl2, -L));
          if (masked) {
            p0 = (k0 + 2 * i <= qrow && k0 + 2 * i < a.S) ? p0 : 0.f;
            p1 = (k0 + 2 * i + 1 <= qrow && k0 + 2 * i + 1 < a.S) ? p1 : 0.f;
          }
          dd[i] = pk(p0 * (__uint_as_float(dp[2 * i]) - D), p1 * (__uint_as_float(dp[2 * i + 1]) - D));
        }
        if (warp == 2 && lane == 0) ATTN_TRACE_P(17, gj);
        if (gj >= 1) mbar_wait(g_done, (gj - 1) & 1);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(18, gj);
        fence_after();
        tmem_st_cols<CPT / 2>(tmem + lane_off + 256 + cg * (CPT / 2), dd);
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (warp == 2 && lane == 0) ATTN_TRACE_P(19, gj);
      }
      mbar_wait(g_done, (gj - 1) & 1);
      fence_after();
      const bool sums = a.s0 && q0 + q * 32 < a.S;
      float fq[GPH];
      store_acc_rows<GPH>(tmem + lane_off + 320 + cg * GPH,
                          a.g0 + (int64_t)(row_base + qrow) * a.d + h * HD + cg * GPH, a.scale,
                          qrow < a.S, fq);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (sums) warp_colsum<GPH>(fq, a.s0 + ((int64_t)b * a.nblk + qt * (TQ / 32) + q) * a.d + h * HD + cg * GPH);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
#undef PH_FOR_TILES

// ---- fused backward at HD = 64: dK, dV and dQ in one pass -------------------------
// The two-pass backward computes every P tile twice (once per pass): 2 x 1,024
// MUFU cycles and 2,196 MMA cycles per 128 x 128 tile pair, against 1,024 and
// 1,685 for one pass.  One pass needs dQ_i = sum_j dS_ij K_j summed across the
// key tiles j, which the two-pass design got from a query-major second pass.
// Here a CTA owns a whole (batch, head): key tiles j ascending (outer), query
// tiles i = j..n-1 (inner), and dQ_i's per-tile partials (an M = 128-query MMA
// with A = dS read from shared memory) are drained by the softmax warps into an
// fp32 accumulator in global memory, each (row, column) always by the same
// thread, in the order j = 0, 1, ..., i: j = 0 stores, 0 < j < i adds
// (red.add), j = i reads back, adds, scales and writes the bf16 dq row and the
// bias partials.  Same-thread same-address operations are ordered, and no other
// CTA touches the head: deterministic, no atomics across CTAs.
// dS^T goes to shared memory only (a 32 KB buffer, NDS below, [2 query halves][128 keys]
// [64 queries] with the 128B swizzle), read as the K-major A of dK = dS^T Q and
// as the MN-major A of dQ = dS K.  The gradient products of a tile are split
// over two completions (pv_done: dV, which frees P^T; gq_done: dK and dQ), so
// the next tile's P^T store waits only for the dV product.  Clock64 timelines
// (tools/attn_trace_fused.py) and ncu (L2 hit rate 44 %) show the pass paced by
// the per-tile hand-offs and by L2 misses on the re-streamed Q/dO (a head's
// Q/dO and dQ accumulator are ~1 MB, 128 heads in flight): odd CTAs walk the
// key tiles in descending order to halve that footprint, and the grid keeps the
// waves of heads even (384 heads: 128 CTAs x 3).
// TMEM: S^T [0,128) dP^T [128,256) P^T [256,320) dV [320,384) dK [384,448) dQ [448,512)
#ifndef PHOTON_ATTN_FUSED
#define PHOTON_ATTN_FUSED 1
#endif
// Q/dO/L/D ring depth and K buffers (2: the next key tile's K streams in while
// the last tile's dQ product still reads K; V is read by dP^T only, one buffer)
#ifndef PHOTON_ATTN_NRF
#define PHOTON_ATTN_NRF 3
#endif
#ifndef PHOTON_ATTN_NKF
#define PHOTON_ATTN_NKF 2
#endif
constexpr int NRF = PHOTON_ATTN_NRF, NKF2 = PHOTON_ATTN_NKF;
#ifndef PHOTON_FUSED_ALT
#define PHOTON_FUSED_ALT 1
#endif
#ifndef PHOTON_FUSED_HINTS
#define PHOTON_FUSED_HINTS 1
#endif
#ifndef PHOTON_FUSED_EARLY_Q
#define PHOTON_FUSED_EARLY_Q 1
#endif
#ifndef PHOTON_FUSED_GRID
#define PHOTON_FUSED_GRID 2
#endif
// dS^T buffers: 2 (the next tile's dS^T is stored while the previous tile's dK /
// dQ products may still read theirs) or 1 (the store waits for them; they have
// retired by then in the steady state).  Measured at the 125M shape: one buffer
// 0.983-0.987 ms, two 0.995-0.996, one + a fourth Q/dO stage 0.996-0.998 (the
// smaller shared-memory carve-out leaves more L1)
#ifndef PHOTON_ATTN_NDS
#define PHOTON_ATTN_NDS 1
#endif
constexpr int NDS = PHOTON_ATTN_NDS;
constexpr int kFusedSmem = 1024 + NDS * 32768 + (NKF2 + 1) * 16384 + NRF * (2 * 16384 + 8 * 128) + 512;
static_assert(kFusedSmem <= 232448, "fused attention backward: shared memory");

__device__ __forceinline__ void st_relaxed_f4(float* p, float4 v) {
  asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red_add_f4(float* p, float4 v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 ld_relaxed_f4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// barrier among the fused pass's 16 softmax warps (hardware barrier 1)
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, %0;" ::"n"(SWB * 32) : "memory"); }

// The fused pass's work split.  A unit is one key tile of one head; its cost is
// its number of query tiles (nt - kt).  Units are ordered head-major, each
// head's key tiles in its walking order (odd heads descending, see desc()), and
// logical CTA c owns the contiguous units whose cost midpoints fall in
// [c C / G, (c+1) C / G) -- every CTA within half a unit of the mean, so all
// SMs finish together (384 heads: 353 +- 8 tile pairs per CTA on 148 SMs instead
// of 408 on 128).  A head cut between CTAs c and c+1 keeps one dQ summation
// order: c walks the head's first key tiles FIRST and then raises the head's
// flag; c+1 walks the rest LAST, after acquiring the flag, so the dQ partials
// still arrive key tile by key tile in the head's order (bitwise the same as an
// uncut head).  Logical ids come from a ticket taken at start, so CTA c-1 is
// resident (or done) whenever c waits, and c-1 raises the flag before it
// waits on anything -- no dependence on the hardware's CTA dispatch order.
struct FusedSched {
  int G, BH, nt;
  int64_t Hc, C;
  __device__ FusedSched(int g, int bh, int n)
      : G(g), BH(bh), nt(n), Hc((int64_t)n * (n + 1) / 2), C((int64_t)bh * n * (n + 1) / 2) {}
  // odd heads walk their key tiles in descending order: the live set of an
  // ascending head (Q/dO tiles j..n-1 and the accumulators of dQ_{j+1..n-1})
  // shrinks while a descending one's grows, so the L2 footprint of all heads in
  // flight stays near half of its peak
  __device__ bool desc(int bh) const { return PHOTON_FUSED_ALT && (bh & 1); }
  __device__ int kt_of(int bh, int kk) const { return desc(bh) ? nt - 1 - kk : kk; }
  __device__ int owner(int bh, int kk) const {
    const int64_t pre = desc(bh) ? (int64_t)kk * (kk + 1) / 2 : (int64_t)kk * nt - (int64_t)kk * (kk - 1) / 2;
    const int64_t m2 = 2 * ((int64_t)bh * Hc + pre) + (nt - kt_of(bh, kk));
    return (int)(m2 * G / (2 * C));
  }
  // first global unit (bh * nt + kk) owned by CTA >= c: the unit holding cost
  // position c C / G lies in head floor(c BH / G), so it or the next one is it
  __device__ int64_t first_unit(int c) const {
    if (c >= G) return (int64_t)BH * nt;
    const int bh0 = (int)((int64_t)c * BH / G);
    for (int bh = bh0; bh < BH && bh <= bh0 + 1; ++bh)
      for (int kk = 0; kk < nt; ++kk)
        if (owner(bh, kk) >= c) return (int64_t)bh * nt + kk;
    return (int64_t)BH * nt;
  }
};

// The segments CTA c walks, in order: the first part of its last head (if cut:
// raises the flag), its whole heads, the rest of its first head (if cut: waits
// for the flag).  A range inside a single head is one segment doing both.
struct FusedSegs {
  int hf, kf, hl, kle, n;
  __device__ FusedSegs(const FusedSched& f, int c) {
    const int64_t u0 = f.first_unit(c), u1 = f.first_unit(c + 1);
    if (u1 <= u0) {
      n = 0;
      hf = kf = hl = kle = 0;
      return;
    }
    hf = (int)(u0 / f.nt);
    kf = (int)(u0 % f.nt);
    hl = (int)((u1 - 1) / f.nt);
    kle = (int)((u1 - 1) % f.nt) + 1;
    if (hf == hl) n = 1;
    else n = (kle < f.nt) + (kf > 0) + ((kle < f.nt ? hl : hl + 1) - (kf > 0 ? hf + 1 : hf));
  }
  // segment s: head bh, key-tile positions [k0, k1), wait / signal the flag
  __device__ void get(int s, int nt, int& bh, int& k0, int& k1, bool& wait, bool& sig) const {
    if (hf == hl) {
      bh = hf, k0 = kf, k1 = kle, wait = kf > 0, sig = kle < nt;
      return;
    }
    wait = sig = false;
    const bool cut_last = kle < nt;
    if (cut_last && s == 0) {
      bh = hl, k0 = 0, k1 = kle, sig = true;
      return;
    }
    if (kf > 0 && s == n - 1) {
      bh = hf, k0 = kf, k1 = nt, wait = true;
      return;
    }
    bh = (kf > 0 ? hf + 1 : hf) + s - (cut_last ? 1 : 0);
    k0 = 0, k1 = nt;
  }
};

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_fused64_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                               const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                               const BwdArgs a) {
  pdl_launch_dependents();
  static_assert(SWB == 16, "fused backward: 16 softmax warps (4 column groups of 32 queries)");
  constexpr int HD = 64, KB = 16384, QB = 16384, T = 128;  // tiles: 128 rows x 64 bf16
  constexpr int CPQ = 32, GPH = 16;                          // per-thread score / accumulator columns
  constexpr uint32_t colDP = 128, colP = 256, colDV = 320, colDK = 384, colDQ = 448;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sDS = sm;                    // dS^T [NDS], 32 KB each
  uint8_t* sK = sDS + NDS * 32768;      // [NKF2]
  uint8_t* sV = sK + NKF2 * KB;         // [1]
  uint8_t* sQ = sV + KB;                // [NRF]
  uint8_t* sO = sQ + NRF * QB;          // [NRF] dO
  float* sL = reinterpret_cast<float*>(sO + NRF * QB);  // [NRF][128]
  float* sD = sL + NRF * T;                             // [NRF][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + NRF * T);
  uint64_t* k_full = bar;                   // [NKF2]
  uint64_t* k_empty = bar + NKF2;           // [NKF2]
  uint64_t* v_full = bar + 2 * NKF2;
  uint64_t* v_empty = v_full + 1;
  uint64_t* q_full = v_full + 2;            // [NRF]
  uint64_t* q_empty = q_full + NRF;         // [NRF]
  uint64_t* s_full = q_empty + NRF;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_full + 2;            // P^T and dS^T of the tile stored
  uint64_t* pv_done = s_full + 3;           // dV product retired (P^T free)
  uint64_t* gq_done = s_full + 4;           // dK, dQ products retired (dS^T buffer free, dQ ready)
  uint64_t* dq_free = s_full + 5;           // dQ drained from TMEM by the softmax warps
  uint64_t* acc_empty = s_full + 6;         // dK / dV drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 7);
  uint32_t* cta_slot = tmem_slot + 1;

  const int nt = (a.S + T - 1) / T;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const FusedSched fs(gridDim.x, a.BH, nt);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NKF2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    for (int i = 0; i < NRF; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, SWB);
    mbar_init(p_full, SWB);
    mbar_init(pv_done, 1);
    mbar_init(gq_done, 1);
    mbar_init(dq_free, SWB);
    mbar_init(acc_empty, SWB);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel visible from here (and the zeroed sync words)
  if (threadIdx.x == 0) *cta_slot = atomicAdd(a.sync, 1u);
  __syncthreads();
  const FusedSegs segs(fs, (int)*cta_slot);

  if (warp == 0) {
    if (lane == 0) {  // ===== producer: K, V per key tile, the Q / dO / L / D ring =====
      // K / V are read once per head (evict first); a head's Q / dO are re-read
      // by every key tile (evict last)
      const uint64_t pol_once = PHOTON_FUSED_HINTS ? policy_evict_first() : 0;
      const uint64_t pol_keep = PHOTON_FUSED_HINTS ? policy_evict_last() : 0;
      int ti = 0, gi = 0;
      for (int sg = 0; sg < segs.n; ++sg) {
        int bh, k0, k1;
        bool sw, ss;
        segs.get(sg, nt, bh, k0, k1, sw, ss);
        const int b = bh / a.H, h = bh % a.H, row_base = b * a.S;
        for (int kk = k0; kk < k1; ++kk, ++ti) {
          const int kt = fs.kt_of(bh, kk);
          const int kb = ti % NKF2;
          mbar_wait(&k_empty[kb], ((ti / NKF2) & 1) ^ 1);
          mbar_expect_tx(&k_full[kb], KB);
          if (PHOTON_FUSED_HINTS)
            tma_load_2d_hint(sK + kb * KB, &tk, &k_full[kb], h * HD, row_base + kt * T, pol_once);
          else
            tma_load_2d(sK + kb * KB, &tk, &k_full[kb], h * HD, row_base + kt * T);
          mbar_wait(v_empty, (ti & 1) ^ 1);
          mbar_expect_tx(v_full, KB);
          if (PHOTON_FUSED_HINTS)
            tma_load_2d_hint(sV, &tv, v_full, h * HD, row_base + kt * T, pol_once);
          else
            tma_load_2d(sV, &tv, v_full, h * HD, row_base + kt * T);
          for (int qt = kt; qt < nt; ++qt, ++gi) {
            const int st = gi % NRF;
            mbar_wait(&q_empty[st], ((gi / NRF) & 1) ^ 1);
            ATTN_TRACE_P(20, gi);
            mbar_expect_tx(&q_full[st], 2 * QB + 8 * T);
            if (PHOTON_FUSED_HINTS) {
              tma_load_2d_hint(sQ + st * QB, &tq, &q_full[st], h * HD, row_base + qt * T, pol_keep);
              tma_load_2d_hint(sO + st * QB, &tdo, &q_full[st], h * HD, row_base + qt * T, pol_keep);
            } else {
              tma_load_2d(sQ + st * QB, &tq, &q_full[st], h * HD, row_base + qt * T);
              tma_load_2d(sO + st * QB, &tdo, &q_full[st], h * HD, row_base + qt * T);
            }
            bulk_load(sL + st * T, a.Lp + (int64_t)bh * a.Spad + qt * T, 4 * T, &q_full[st]);
            bulk_load(sD + st * T, a.Dp + (int64_t)bh * a.Spad + qt * T, 4 * T, &q_full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      // S^T, dP^T: M = 128 keys, N = 128 queries, both operands K-major
      constexpr uint32_t IDS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T >> 3) << 17) |
                               ((uint32_t)(T >> 4) << 24);
      // dV, dK: M = 128 keys, N = 64, B (dO / Q) MN-major
      constexpr uint32_t IDG = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                               ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(T >> 4) << 24);
      // dQ: M = 128 queries, N = 64, A (dS) and B (K) MN-major
      constexpr uint32_t IDQ = IDG | (1u << 15);
      auto issue_grads = [&](int g, int st, bool first, int t, int kb, bool last) {
        mbar_wait(p_full, g & 1);
        if (first && t > 0) mbar_wait(acc_empty, (t - 1) & 1);  // previous dK/dV drained
        ATTN_TRACE_P(23, g);
        fence_after();
        const uint32_t bo = su32(sO + st * QB), bq = su32(sQ + st * QB), bk = su32(sK + kb * KB);
        const uint32_t ads = su32(sDS + (NDS == 2 ? (g & 1) * 32768 : 0));
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dV += P^T dO (P^T from TMEM)
          mma_ts(tmem + colDV, tmem + colP + kk * 8, sw128(bo + kk * 2048, QB, 1024), IDG,
                 (!first || kk > 0) ? 1u : 0u);
        commit(pv_done);
#if PHOTON_FUSED_EARLY_Q
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dK += dS^T Q (dS^T K-major in smem)
          mma(tmem + colDK, sw128(ads + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
              sw128(bq + kk * 2048, QB, 1024), IDG, (!first || kk > 0) ? 1u : 0u);
        // the stage's Q / dO / L / D are read by nothing after dK: free it before
        // the dQ product (a stage lives ~3 tile periods; its reload is on the
        // critical path)
        commit(&q_empty[st]);
        if (g > 0) mbar_wait(dq_free, (g - 1) & 1);  // the previous tile's dQ drained
        fence_after();
#else
        if (g > 0) mbar_wait(dq_free, (g - 1) & 1);  // the previous tile's dQ drained
        fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dK += dS^T Q (dS^T K-major in smem)
          mma(tmem + colDK, sw128(ads + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
              sw128(bq + kk * 2048, QB, 1024), IDG, (!first || kk > 0) ? 1u : 0u);
#endif
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dQ_tile = dS K (dS MN-major in smem, K MN-major)
          mma(tmem + colDQ, sw128(ads + kk * 2048, 16384, 1024), sw128(bk + kk * 2048, KB, 1024),
              IDQ, kk > 0 ? 1u : 0u);
        commit(gq_done);
#if !PHOTON_FUSED_EARLY_Q
        commit(&q_empty[st]);
#endif
        if (last) commit(&k_empty[kb]);  // this key tile's K no longer read
      };
      int ti = 0, gi = 0;
      int pend = -1, pend_st = 0, pend_t = 0, pend_kb = 0;
      bool pend_first = false, pend_last = false;
      for (int sg = 0; sg < segs.n; ++sg) {
        int bh, k0, k1;
        bool sw, ss;
        segs.get(sg, nt, bh, k0, k1, sw, ss);
        for (int kk = k0; kk < k1; ++kk, ++ti) {
          const int kt = fs.kt_of(bh, kk);
          const int kb = ti % NKF2;
          mbar_wait(&k_full[kb], (ti / NKF2) & 1);
          mbar_wait(v_full, ti & 1);
          const uint32_t ak = su32(sK + kb * KB), av = su32(sV);
          for (int qt = kt; qt < nt; ++qt, ++gi) {
            const int st = gi % NRF;
            mbar_wait(&q_full[st], (gi / NRF) & 1);
            ATTN_TRACE_P(21, gi);
            mbar_wait(s_empty, (gi & 1) ^ 1);
            ATTN_TRACE_P(22, gi);
            fence_after();
            const uint32_t bq = su32(sQ + st * QB), bo = su32(sO + st * QB);
#pragma unroll
            for (int k4 = 0; k4 < HD / 16; ++k4)  // S^T = K Q^T
              mma(tmem + 0, sw128(ak + k4 * 32, 16, 1024), sw128(bq + k4 * 32, 16, 1024), IDS,
                  k4 > 0 ? 1u : 0u);
#pragma unroll
            for (int k4 = 0; k4 < HD / 16; ++k4)  // dP^T = V dO^T
              mma(tmem + colDP, sw128(av + k4 * 32, 16, 1024), sw128(bo + k4 * 32, 16, 1024), IDS,
                  k4 > 0 ? 1u : 0u);
            commit(s_full);
            if (qt == nt - 1) commit(v_empty);  // the key tile's V no longer read
            if (pend >= 0) issue_grads(pend, pend_st, pend_first, pend_t, pend_kb, pend_last);
            pend = gi;
            pend_st = st;
            pend_first = qt == kt;
            pend_t = ti;
            pend_kb = kb;
            pend_last = qt == nt - 1;
          }
        }
      }
      if (pend >= 0) issue_grads(pend, pend_st, pend_first, pend_t, pend_kb, pend_last);
    }
  } else {
    // ===== softmax: thread = key row r (TMEM lane) x 32 query columns (group cg) =====
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint64_t pol_out = PHOTON_FUSED_HINTS ? policy_evict_first() : 0;  // dq / dk / dv rows
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // this thread's 16-byte chunks of the dS^T row r (queries cg*32 + 8t .. +7)
    const uint32_t ds_row = su32(sDS) + (cg >> 1) * 16384 + r * 128;
    // dQ of the previous tile (drained one tile late: its MMA runs under this
    // tile's softmax) and where it goes
    auto emit_dq = [&](const uint32_t (&u)[GPH], int p_bh, int p_qt, int p_kt) {
      float* acc = a.dqa + (((int64_t)p_bh * nt + p_qt) * (HD / 4) + cg * (GPH / 4)) * (4 * T) + 4 * r;
      const bool desc = fs.desc(p_bh);
      const bool first = desc ? p_kt == p_qt : p_kt == 0, fin = desc ? p_kt == 0 : p_kt == p_qt;
      if (!fin) {
#pragma unroll
        for (int c = 0; c < GPH / 4; ++c) {
          const float4 v = make_float4(__uint_as_float(u[4 * c]), __uint_as_float(u[4 * c + 1]),
                                       __uint_as_float(u[4 * c + 2]), __uint_as_float(u[4 * c + 3]));
          if (first) st_relaxed_f4(acc + c * 4 * T, v);
          else red_add_f4(acc + c * 4 * T, v);
        }
        return;
      }
      // dQ_i's last contribution: finish the row
      const int b = p_bh / a.H, h = p_bh % a.H, qrow = p_qt * T + r;
      const bool live = qrow < a.S;
      float f[GPH];
#pragma unroll
      for (int c = 0; c < GPH / 4; ++c) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!first) s = ld_relaxed_f4(acc + c * 4 * T);
        f[4 * c] = live ? (s.x + __uint_as_float(u[4 * c])) * a.scale : 0.f;
        f[4 * c + 1] = live ? (s.y + __uint_as_float(u[4 * c + 1])) * a.scale : 0.f;
        f[4 * c + 2] = live ? (s.z + __uint_as_float(u[4 * c + 2])) * a.scale : 0.f;
        f[4 * c + 3] = live ? (s.w + __uint_as_float(u[4 * c + 3])) * a.scale : 0.f;
      }
      if (live) {
        bf16* row = a.g0 + (int64_t)(b * a.S + qrow) * a.d + h * HD + cg * GPH;
#pragma unroll
        for (int i = 0; i < GPH; i += 8) {
          const uint4 w = make_uint4(pk(f[i], f[i + 1]), pk(f[i + 2], f[i + 3]), pk(f[i + 4], f[i + 5]),
                                     pk(f[i + 6], f[i + 7]));
          if (pol_out) st_hint_u4(row + i, w, pol_out);
          else *reinterpret_cast<uint4*>(row + i) = w;
        }
      }
      if (a.s0 && p_qt * T + q * 32 < a.S)
        warp_colsum<GPH>(f, a.s0 + ((int64_t)b * a.nblk + p_qt * (T / 32) + q) * a.d + h * HD + cg * GPH);
    };
    // drain the dQ of tile g (its products retired) and let the issuer reuse it
    auto drain_dq = [&](int g, uint32_t (&u)[GPH]) {
      mbar_wait(gq_done, g & 1);
      fence_after();
      TMEM_LD16(tmem + lane_off + colDQ + cg * GPH, u);
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
    };
    int gi = 0;
    int p_bh = 0, p_qt = 0, p_kt = 0;
    bool pend = false;  // tile gi-1's dQ not drained yet
    for (int sg = 0; sg < segs.n; ++sg) {
      int bh, k0, k1;
      bool sw, ss;
      segs.get(sg, nt, bh, k0, k1, sw, ss);
      const int b = bh / a.H, h = bh % a.H, row_base = b * a.S;
      if (sw) {  // the rest of a cut head: its first part's dQ partials are in
        if (threadIdx.x == 64) {
          const uint32_t* f = a.sync + 1 + bh;
          uint32_t v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          } while (v == 0u);
          __threadfence();
        }
        softmax_bar();
      }
      for (int kk = k0; kk < k1; ++kk) {
        const int kt = fs.kt_of(bh, kk);
        const int key = kt * T + r;
        const bool key_live = key < a.S;
        for (int qt = kt; qt < nt; ++qt, ++gi) {
          const int st = gi % NRF, q0 = qt * T;
          mbar_wait(&q_full[st], (gi / NRF) & 1);  // L, D of this query tile visible
          mbar_wait(s_full, gi & 1);
          if (warp == 2 && lane == 0) ATTN_TRACE_P(25, gi);
          fence_after();
          const float* L = sL + st * T + cg * CPQ;
          const float* D = sD + st * T + cg * CPQ;
          const bool masked = (kt * T + T > q0) || (kt * T + T > a.S);
          uint32_t pp[CPQ / 2], dd[CPQ / 2];
          // two halves of 16 columns (96 registers at 576 threads): the second
          // half's scores are loaded after the first half's exponentials
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t s[CPQ / 2], dp[CPQ / 2];
            TMEM_LD16(tmem + lane_off + cg * CPQ + hf * 16, s);
            TMEM_LD16(tmem + lane_off + colDP + cg * CPQ + hf * 16, dp);
            tmem_wait_ld();
            if (hf == 1) {
              fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(s_empty);
              if (lane == 0) ATTN_TRACE_MAX(24, gi);
            }
#pragma unroll
            for (int i4 = 0; i4 < CPQ / 8; ++i4) {
              const int i = hf * (CPQ / 8) + i4;
              const float4 l4 = lds_f4(L + 4 * i), d4 = lds_f4(D + 4 * i);
              float p0 = ex2(fmaf(__uint_as_float(s[4 * i4]), a.sl2, -l4.x));
              float p1 = ex2(fmaf(__uint_as_float(s[4 * i4 + 1]), a.sl2, -l4.y));
              float p2 = ex2(fmaf(__uint_as_float(s[4 * i4 + 2]), a.sl2, -l4.z));
              float p3 = ex2(fmaf(__uint_as_float(s[4 * i4 + 3]), a.sl2, -l4.w));
              if (masked) {
                const int qc = q0 + cg * CPQ + 4 * i;
                p0 = (key_live && key <= qc) ? p0 : 0.f;
                p1 = (key_live && key <= qc + 1) ? p1 : 0.f;
                p2 = (key_live && key <= qc + 2) ? p2 : 0.f;
                p3 = (key_live && key <= qc + 3) ? p3 : 0.f;
              }
              pp[2 * i] = pk(p0, p1);
              pp[2 * i + 1] = pk(p2, p3);
              dd[2 * i] = pk(p0 * (__uint_as_float(dp[4 * i4]) - d4.x),
                             p1 * (__uint_as_float(dp[4 * i4 + 1]) - d4.y));
              dd[2 * i + 1] = pk(p2 * (__uint_as_float(dp[4 * i4 + 2]) - d4.z),
                                 p3 * (__uint_as_float(dp[4 * i4 + 3]) - d4.w));
            }
          }
          if (warp == 2 && lane == 0) ATTN_TRACE_P(26, gi);
          if (lane == 0) ATTN_TRACE_MAX(30, gi);
          // dS^T into buffer gi & 1 (its last readers, tile gi-2's dK / dQ
          // products, retired before tile gi-1 drained their dQ)
          if (NDS == 1 && gi >= 1) {  // one buffer: the previous tile's dK / dQ products read it
            mbar_wait(gq_done, (gi - 1) & 1);
            fence_after();
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
            sts128(ds_row + (NDS == 2 ? (gi & 1) * 32768 : 0) + ((((cg & 1) * 4 + t) ^ (r & 7)) << 4), dd[4 * t],
                   dd[4 * t + 1], dd[4 * t + 2], dd[4 * t + 3]);
          // P^T is free once the previous tile's dV product retired
          if (gi >= 1) mbar_wait(pv_done, (gi - 1) & 1);
          if (warp == 2 && lane == 0) ATTN_TRACE_P(27, gi);
          fence_after();
          tmem_st_cols<CPQ / 2>(tmem + lane_off + colP + cg * (CPQ / 2), pp);
          tmem_wait_st();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full);
          if (warp == 2 && lane == 0) ATTN_TRACE_P(28, gi);
          if (pend) {
            uint32_t dqv[GPH];
            drain_dq(gi - 1, dqv);
            emit_dq(dqv, p_bh, p_qt, p_kt);
          }
          pend = true;
          if (warp == 2 && lane == 0) ATTN_TRACE_P(29, gi);
          if (lane == 0) ATTN_TRACE_MAX(31, gi);
          p_bh = bh;
          p_qt = qt;
          p_kt = kt;
        }
        // the key tile's dK / dV are complete once its last products retire
        mbar_wait(pv_done, (gi - 1) & 1);
        mbar_wait(gq_done, (gi - 1) & 1);
        fence_after();
        const int64_t row = (int64_t)(row_base + key) * a.d + h * HD + cg * GPH;
        const bool sums = a.s1 && kt * T + q * 32 < a.S;
        const int64_t prow = ((int64_t)b * a.nblk + kt * (T / 32) + q) * a.d + h * HD + cg * GPH;
        float fk[GPH], fv[GPH];
        store_acc_rows<GPH>(tmem + lane_off + colDK + cg * GPH, a.g1 + row, a.scale, key_live, fk, pol_out);
        store_acc_rows<GPH>(tmem + lane_off + colDV + cg * GPH, a.g2 + row, 1.f, key_live, fv, pol_out);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        if (sums) {
          warp_colsum<GPH>(fk, a.s1 + prow);
          warp_colsum<GPH>(fv, a.s2 + prow);
        }
      }
      if (ss) {  // first part of a cut head: drain its last dQ now, then raise the flag
        if (pend) {
          uint32_t dqv[GPH];
          drain_dq(gi - 1, dqv);
          emit_dq(dqv, p_bh, p_qt, p_kt);
          pend = false;
        }
        __threadfence();
        softmax_bar();
        if (threadIdx.x == 64) {
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.sync + 1 + bh), "r"(1u) : "memory");
        }
      }
    }
    if (pend) {  // the last tile's dQ
      uint32_t dqv[GPH];
      drain_dq(gi - 1, dqv);
      emit_dq(dqv, p_bh, p_qt, p_kt);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qr;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw Error(PHOTON_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// [rows][d] bf16, box {64 cols of one head, box_rows rows}, 128B swizzle
CUtensorMap head_map(const void* base, int rows, int d, int box_rows = 128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(PHOTON_ERR_CUDA, "attention tensor map failed");
  return m;
}

// per-device scratch for the debug entry point (engines pass their own workspace)
float* scratch(size_t n) {
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

// cudaFuncSetAttribute is per device: set once for each device that launches
template <typename F>
void set_smem_once(std::atomic<uint64_t>& done, F kern, int bytes) {
  int dev = 0;
  PH_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load() & bit) return;
  PH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.fetch_or(bit);
}

}  // namespace

#ifdef PHOTON_ATTN_TRACE
extern "C" int photon_debug_attn_trace(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(unsigned long long) * n);
}
#endif

bool attn_tc_supported(int dh, int d) { return (dh == 64 || dh == 128) && (d % 8) == 0; }

size_t attn_bwd_tc_ws_floats(int B, int S, int H, int d) {
  const size_t Spad = (size_t)(S + TQ - 1) / TQ * TQ;
  // L, D; at head dim 64 the fused pass's fp32 dQ accumulator
  // (plus the schedule words: a ticket and one flag per head, 16-byte aligned)
  return (size_t)2 * B * H * Spad +
         (PHOTON_ATTN_FUSED && d == 64 * H ? (size_t)B * H * Spad * 64 + ((size_t)B * H + 4 + 3) / 4 * 4 : 0);
}

namespace {

template <int HD>
void attn_bwd_hd(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                 const float* lse, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H, int d,
                 float* ws, float* sums, cudaStream_t st) {
  const int nt = (S + TQ - 1) / TQ, Spad = nt * TQ, rows = B * S;
  if (!ws) ws = scratch(attn_bwd_tc_ws_floats(B, S, H, d));
  float* Lp = ws;
  float* Dp = Lp + (size_t)B * H * Spad;
  const bool fused = HD == 64 && PHOTON_ATTN_FUSED;
  uint32_t* sync = fused ? reinterpret_cast<uint32_t*>(Dp + (size_t)B * H * Spad + (size_t)B * H * Spad * 64)
                         : nullptr;
  const int nsync = B * H + 1;
  launch_pdl_cls(kPdlAttn, attn_bwd_prep_kernel<HD>, std::min<int64_t>(((int64_t)B * S + 7) / 8, kNumSMs * 16), 256, 0, st, o, dO, lse, Lp, Dp, B, S, H, d, Spad, sync, nsync);
  PH_LAUNCH_CHECK();
  constexpr int TQB = HD == 64 ? 128 : 64;  // dK/dV kernel's query tile
  const CUtensorMap mq = head_map(q, rows, d), mk = head_map(k, rows, d), mv = head_map(v, rows, d),
                    mo = head_map(dO, rows, d);
  const CUtensorMap mqb = TQB == 128 ? mq : head_map(q, rows, d, TQB),
                    mob = TQB == 128 ? mo : head_map(dO, rows, d, TQB);
  const int nblk = (S + 31) / 32;
  const size_t P = (size_t)B * nblk * d;  // sums: dq, dk, dv partials
  BwdArgs a{S,  H,  d,  Spad, B * H, rsqrtf((float)HD) * kLog2e, rsqrtf((float)HD), Lp, Dp, dk, dv,
            sums ? sums + P : nullptr, sums ? sums + 2 * P : nullptr, nblk};
  if constexpr (HD == 64 && PHOTON_ATTN_FUSED) {
    a.g0 = dq;
    a.g1 = dk;
    a.g2 = dv;
    a.s0 = sums;
    a.s1 = sums ? sums + P : nullptr;
    a.s2 = sums ? sums + 2 * P : nullptr;
    a.dqa = Dp + (size_t)B * H * Spad;
    a.sync = sync;
    static std::atomic<uint64_t> cfgf{0};
    set_smem_once(cfgf, attn_bwd_fused64_tc_kernel, kFusedSmem);
    // PHOTON_FUSED_GRID 2: every SM, heads split between neighbouring CTAs at
    // key-tile boundaries (FusedSched); 1: as many CTAs as keep whole heads in
    // even waves (e.g. 384 heads: 128 x 3)
    const int waves = (B * H + kNumSMs - 1) / kNumSMs;
    static const int ctas_env = [] {  // experiments: PHOTON_FUSED_CTAS caps the grid
      const char* e = std::getenv("PHOTON_FUSED_CTAS");
      return e ? std::atoi(e) : 0;
    }();
    int grid = PHOTON_FUSED_GRID == 1 ? std::min(kNumSMs, (B * H + waves - 1) / waves)
                                      : std::min(kNumSMs, B * H);
    if (ctas_env > 0) grid = std::min(grid, ctas_env);
    launch_pdl_cls(kPdlAttn, attn_bwd_fused64_tc_kernel, grid, kBwdThreads, kFusedSmem, st, mq, mk, mv, mo, a);
    PH_LAUNCH_CHECK();
    return;
  }
  constexpr int NA = HD / 64;
  constexpr int NKV = HD == 64 ? NKV64 : 1, NRQ = HD == 64 ? NRQ64 : 2, NQO = HD == 64 ? 2 : 1;
  constexpr int NRK = HD == 64 ? NR64 : NR;
  constexpr int SMEM1 = 1024 + 2 * NKV * 16384 * NA + NRK * 2 * TQB * 128 * NA + NRK * 8 * TQB + 512;
  constexpr int SMEM2 = 1024 + (2 * NQO + 2 * NRQ) * 16384 * NA + 512;
  static_assert(SMEM1 <= 232448 && SMEM2 <= 232448, "attention backward: shared memory");
  static std::atomic<uint64_t> cfg1{0}, cfg2{0};
  set_smem_once(cfg1, attn_bwd_dkdv_tc_kernel<HD>, SMEM1);
  set_smem_once(cfg2, attn_bwd_dq_tc_kernel<HD>, SMEM2);
  // persistent: one CTA per SM over the units (tile pairs) of both kernels
  const int grid = std::min(kNumSMs, B * H * ((nt + 1) / 2));
  launch_pdl_cls(kPdlAttn, attn_bwd_dkdv_tc_kernel<HD>, grid, kBwdThreads, SMEM1, st, mqb, mk, mv, mob, a);
  PH_LAUNCH_CHECK();
  a.g0 = dq;
  a.g1 = nullptr;
  a.s0 = sums;
  a.s1 = nullptr;
  launch_pdl_cls(kPdlAttn, attn_bwd_dq_tc_kernel<HD>, grid, kBwdThreads, SMEM2, st, mq, mk, mv, mo, a);
  PH_LAUNCH_CHECK();
}

template <int HD>
void attn_fwd_hd(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                 int H, int d, cudaStream_t st) {
  const int rows = B * S;
  const CUtensorMap mq = head_map(q, rows, d), mk = head_map(k, rows, d), mv = head_map(v, rows, d);
  const FwdArgs a{S, H, d, rsqrtf((float)HD) * kLog2e, o, lse};
  constexpr int SMEM = 1024 + 16384 * (3 + NKF) * (HD / 64) + 256;
  static std::atomic<uint64_t> cfg{0};
  set_smem_once(cfg, attn_fwd_tc_kernel<HD>, SMEM);
  dim3 grid((S + TQ - 1) / TQ, B * H);
  launch_pdl_cls(kPdlAttn, attn_fwd_tc_kernel<HD>, grid, kThreads, SMEM, st, mq, mk, mv, a);
  PH_LAUNCH_CHECK();
}

}  // namespace

void attn_bwd_tc(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                 const float* lse, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H, int d,
                 float* ws, cudaStream_t st, float* sums) {
  if (d / H == 64) attn_bwd_hd<64>(q, k, v, o, dO, lse, dq, dk, dv, B, S, H, d, ws, sums, st);
  else if (d / H == 128) attn_bwd_hd<128>(q, k, v, o, dO, lse, dq, dk, dv, B, S, H, d, ws, sums, st);
  else throw Error(PHOTON_ERR_CONFIG, "attn_bwd_tc: head dim must be 64 or 128");
}

void attn_fwd_tc(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                 int H, int d, cudaStream_t st) {
  if (d / H == 64) attn_fwd_hd<64>(q, k, v, o, lse, B, S, H, d, st);
  else if (d / H == 128) attn_fwd_hd<128>(q, k, v, o, lse, B, S, H, d, st);
  else throw Error(PHOTON_ERR_CONFIG, "attn_fwd_tc: head dim must be 64 or 128");
}

}  // namespace k
}  // namespace photon
