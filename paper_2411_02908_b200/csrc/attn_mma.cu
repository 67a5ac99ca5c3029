// attn_mma.cu -- fused causal attention on tensor cores (bf16 in, fp32 math).
//
// Flash-style: the B*H*S*S probability tensor the reference stores
// (tensor.cpp:449-450) is never materialised.  Forward keeps an online
// softmax per query row and writes O and the log-sum-exp; the backward
// recomputes P from (Q, K, lse) in two passes -- dK/dV per key tile and dQ per
// query tile -- so there are no atomics and the result is deterministic.
// Semantics follow tensor.cpp:436-542: scores scaled by 1/sqrt(dh) before
// the max, keys j <= i only, dS = P * (dP - rowsum(P*dP)) * scale with
// rowsum(P*dP) = dO . O.
//
// Tiles: 64 queries x 64 keys per step, 4 warps x 16 rows, mma.sync
// m16n8k16 bf16 with fp32 accumulators, cp.async double-buffered K/V (or Q/dO)
// tiles in padded shared memory (conflict-free ldmatrix).
#include "kernels.cuh"

namespace photon {
namespace k {

namespace {

constexpr int BT = 64;        // rows per tile (queries or keys)
constexpr int kWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t sptr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill rows past S
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sptr(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(sptr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                          const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(sptr(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

// Tile of BT rows x DH bf16 in smem, row stride DH+8 (16B pad).
template <int DH>
struct Tile {
  static constexpr int LD = DH + 8;
  bf16 v[BT * LD];
  // async load rows [r0, r0+BT) of a head slice; rows >= S are zero-filled
  __device__ __forceinline__ void load(const bf16* base, int64_t ld, int r0, int S) {
    constexpr int CH = DH / 8;  // 16-byte chunks per row
    for (int i = threadIdx.x; i < BT * CH; i += kWarps * 32) {
      const int r = i / CH, c = i % CH;
      const bool ok = r0 + r < S;
      const bf16* src = base + (int64_t)(ok ? r0 + r : 0) * ld + c * 8;
      cp_async16(&v[r * LD + c * 8], src, ok);
    }
  }
  // A fragment (rows r0..r0+15, k cols 16kk..16kk+15), non-transposed
  __device__ __forceinline__ void a_frag(uint32_t* a, int r0, int kk) const {
    const int l = threadIdx.x & 31, mi = l >> 3, ri = l & 7;
    ldsm_x4(a[0], a[1], a[2], a[3], &v[(r0 + (mi & 1) * 8 + ri) * LD + kk * 16 + (mi >> 1) * 8]);
  }
  // B fragments for n-tiles n8, n8+1 (rows of the tile are the n dim), k = cols 16kk..
  __device__ __forceinline__ void b_frag_rows(uint32_t* b, int n8, int kk) const {
    const int l = threadIdx.x & 31, mi = l >> 3, ri = l & 7;
    ldsm_x4(b[0], b[1], b[2], b[3], &v[((n8 + (mi >> 1)) * 8 + ri) * LD + kk * 16 + (mi & 1) * 8]);
  }
  // B fragments for n-tiles n8, n8+1 over the cols, k = rows 16kk.. (transposed)
  __device__ __forceinline__ void b_frag_cols(uint32_t* b, int n8, int kk) const {
    const int l = threadIdx.x & 31, mi = l >> 3, ri = l & 7;
    ldsm_x4_t(b[0], b[1], b[2], b[3], &v[(kk * 16 + (mi & 1) * 8 + ri) * LD + (n8 + (mi >> 1)) * 8]);
  }
};

// ============================================================================
// forward
// ============================================================================
template <int DH>
__global__ void __launch_bounds__(kWarps * 32)
attn_fwd_mma_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                    const bf16* __restrict__ v, bf16* __restrict__ o, float* __restrict__ lse,
                    int S, int H, int d, float scale) {
  extern __shared__ __align__(16) uint8_t sm[];
  Tile<DH>& sQ = *reinterpret_cast<Tile<DH>*>(sm);
  Tile<DH>* sK = reinterpret_cast<Tile<DH>*>(sm + sizeof(Tile<DH>));
  Tile<DH>* sV = sK + 2;
  const int nqt = (S + BT - 1) / BT;
  const int qt = nqt - 1 - blockIdx.x;  // heavy (late) tiles first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int q0 = qt * BT;
  const int64_t rowbase = (int64_t)b * S * d + (int64_t)h * DH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const float sl2 = scale * kLog2e;

  sQ.load(q + rowbase, d, q0, S);
  sK[0].load(k + rowbase, d, 0, S);
  sV[0].load(v + rowbase, d, 0, S);
  cp_commit();

  uint32_t qa[DH / 16][4];
  float acc[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int r_lo = q0 + warp * 16 + (lane >> 2);  // this thread's rows: r_lo, r_lo + 8

  const int nkt = qt + 1;  // causal: key tiles 0..qt
  for (int kt = 0; kt < nkt; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nkt) {
      sK[cur ^ 1].load(k + rowbase, d, (kt + 1) * BT, S);
      sV[cur ^ 1].load(v + rowbase, d, (kt + 1) * BT, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) sQ.a_frag(qa[kk], warp * 16, kk);
    }
    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int n8 = 0; n8 < 8; n8 += 2) {
        uint32_t bf[4];
        sK[cur].b_frag_rows(bf, n8, kk);
        mma16816(s[n8], qa[kk], bf[0], bf[1]);
        mma16816(s[n8 + 1], qa[kk], bf[2], bf[3]);
      }
    }
    // scale, causal / length mask, online softmax (log2 domain)
    const int k0 = kt * BT;
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n8 = 0; n8 < 8; ++n8)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + n8 * 8 + (lane & 3) * 2 + (e & 1);
        const int row = r_lo + (e >> 1) * 8;
        float x = s[n8][e] * sl2;
        if (key > row || key >= S) x = -INFINITY;
        s[n8][e] = x;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], x);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float corr[2], rsum[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = mnew[r] == -INFINITY ? 1.f : exp2f(mrow[r] - mnew[r]);
#pragma unroll
    for (int n8 = 0; n8 < 8; ++n8)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = mnew[e >> 1];
        const float p = m == -INFINITY ? 0.f : exp2f(s[n8][e] - m);
        s[n8][e] = p;
        rsum[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rsum[r] += __shfl_xor_sync(0xffffffffu, rsum[r], 1);
      rsum[r] += __shfl_xor_sync(0xffffffffu, rsum[r], 2);
      lrow[r] = lrow[r] * corr[r] + rsum[r];
      mrow[r] = mnew[r];
    }
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      acc[i][0] *= corr[0];
      acc[i][1] *= corr[0];
      acc[i][2] *= corr[1];
      acc[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                        pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                        pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int n8 = 0; n8 < DH / 8; n8 += 2) {
        uint32_t bf[4];
        sV[cur].b_frag_cols(bf, n8, kk);
        mma16816(acc[n8], pa, bf[0], bf[1]);
        mma16816(acc[n8 + 1], pa, bf[2], bf[3]);
      }
    }
    __syncthreads();
  }
  // normalise and store
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = r_lo + r * 8;
    if (row >= S) continue;
    const float inv = 1.f / lrow[r];
    bf16* orow = o + rowbase + (int64_t)row * d;
#pragma unroll
    for (int n8 = 0; n8 < DH / 8; ++n8) {
      const int c = n8 * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + c) = pack_bf16(acc[n8][2 * r] * inv, acc[n8][2 * r + 1] * inv);
    }
    if ((lane & 3) == 0) lse[(int64_t)bh * S + row] = mrow[r] * kLn2 + logf(lrow[r]);
  }
}

// ============================================================================
// backward: dK, dV per key tile (keys are the warp rows)
// ============================================================================
template <int DH>
__global__ void __launch_bounds__(kWarps * 32)
attn_bwd_dkdv_mma_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                         const bf16* __restrict__ v, const bf16* __restrict__ dO,
                         const float* __restrict__ lse, const float* __restrict__ Dv,
                         bf16* __restrict__ dk, bf16* __restrict__ dv, int S, int H, int d,
                         float scale) {
  extern __shared__ __align__(16) uint8_t sm[];
  Tile<DH>& sK = *reinterpret_cast<Tile<DH>*>(sm);
  Tile<DH>& sV = *(reinterpret_cast<Tile<DH>*>(sm) + 1);
  Tile<DH>* sQ = reinterpret_cast<Tile<DH>*>(sm) + 2;
  Tile<DH>* sdO = sQ + 2;
  float* sL = reinterpret_cast<float*>(sdO + 2);  // [2][BT] lse (log2 units)
  float* sD = sL + 2 * BT;                          // [2][BT]
  const int nt = (S + BT - 1) / BT;
  const int kt = blockIdx.x;  // key tile: queries kt..nt-1 contribute
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int k0 = kt * BT;
  const int64_t rowbase = (int64_t)b * S * d + (int64_t)h * DH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const float sl2 = scale * kLog2e;

  auto load_q = [&](int buf, int qt) {
    sQ[buf].load(q + rowbase, d, qt * BT, S);
    sdO[buf].load(dO + rowbase, d, qt * BT, S);
    for (int i = threadIdx.x; i < BT; i += kWarps * 32) {
      const int row = qt * BT + i;
      sL[buf * BT + i] = row < S ? lse[(int64_t)bh * S + row] * kLog2e : INFINITY;
      sD[buf * BT + i] = row < S ? Dv[(int64_t)bh * S + row] : 0.f;
    }
  };
  sK.load(k + rowbase, d, k0, S);
  sV.load(v + rowbase, d, k0, S);
  load_q(0, kt);
  cp_commit();

  uint32_t ka[DH / 16][4], va[DH / 16][4];
  float dka[DH / 8][4], dva[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dka[i][e] = dva[i][e] = 0.f;
  const int key_lo = k0 + warp * 16 + (lane >> 2);  // this thread's keys: key_lo, key_lo + 8

  for (int qt = kt; qt < nt; ++qt) {
    const int cur = (qt - kt) & 1;
    if (qt + 1 < nt) load_q(cur ^ 1, qt + 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (qt == kt) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        sK.a_frag(ka[kk], warp * 16, kk);
        sV.a_frag(va[kk], warp * 16, kk);
      }
    }
    // S^T = K Q^T and dP^T = V dO^T (16 keys x 64 queries per warp)
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int n8 = 0; n8 < 8; n8 += 2) {
        uint32_t bq[4], bo[4];
        sQ[cur].b_frag_rows(bq, n8, kk);
        sdO[cur].b_frag_rows(bo, n8, kk);
        mma16816(st[n8], ka[kk], bq[0], bq[1]);
        mma16816(st[n8 + 1], ka[kk], bq[2], bq[3]);
        mma16816(dpt[n8], va[kk], bo[0], bo[1]);
        mma16816(dpt[n8 + 1], va[kk], bo[2], bo[3]);
      }
    }
    // P^T = exp(S^T scale - lse);  dS^T = P^T (dP^T - D) scale
    const int qbase = qt * BT;
#pragma unroll
    for (int n8 = 0; n8 < 8; ++n8)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = n8 * 8 + (lane & 3) * 2 + (e & 1);
        const int query = qbase + qi;
        const int key = key_lo + (e >> 1) * 8;
        float p = exp2f(st[n8][e] * sl2 - sL[cur * BT + qi]);
        if (key > query || query >= S || key >= S) p = 0.f;
        st[n8][e] = p;
        dpt[n8][e] = p * (dpt[n8][e] - sD[cur * BT + qi]) * scale;
      }
    // dV += P^T dO ;  dK += dS^T Q    (k = queries)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pack_bf16(st[2 * kk][0], st[2 * kk][1]), pack_bf16(st[2 * kk][2], st[2 * kk][3]),
                        pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]),
                        pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3])};
      uint32_t da[4] = {pack_bf16(dpt[2 * kk][0], dpt[2 * kk][1]),
                        pack_bf16(dpt[2 * kk][2], dpt[2 * kk][3]),
                        pack_bf16(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]),
                        pack_bf16(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3])};
#pragma unroll
      for (int n8 = 0; n8 < DH / 8; n8 += 2) {
        uint32_t bo[4], bq[4];
        sdO[cur].b_frag_cols(bo, n8, kk);
        sQ[cur].b_frag_cols(bq, n8, kk);
        mma16816(dva[n8], pa, bo[0], bo[1]);
        mma16816(dva[n8 + 1], pa, bo[2], bo[3]);
        mma16816(dka[n8], da, bq[0], bq[1]);
        mma16816(dka[n8 + 1], da, bq[2], bq[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key_lo + r * 8;
    if (key >= S) continue;
    bf16* kr = dk + rowbase + (int64_t)key * d;
    bf16* vr = dv + rowbase + (int64_t)key * d;
#pragma unroll
    for (int n8 = 0; n8 < DH / 8; ++n8) {
      const int c = n8 * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(kr + c) = pack_bf16(dka[n8][2 * r], dka[n8][2 * r + 1]);
      *reinterpret_cast<uint32_t*>(vr + c) = pack_bf16(dva[n8][2 * r], dva[n8][2 * r + 1]);
    }
  }
}

// ============================================================================
// backward: dQ per query tile
// ============================================================================
template <int DH>
__global__ void __launch_bounds__(kWarps * 32)
attn_bwd_dq_mma_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                       const bf16* __restrict__ v, const bf16* __restrict__ dO,
                       const float* __restrict__ lse, const float* __restrict__ Dv,
                       bf16* __restrict__ dq, int S, int H, int d, float scale) {
  extern __shared__ __align__(16) uint8_t sm[];
  Tile<DH>& sQ = *reinterpret_cast<Tile<DH>*>(sm);
  Tile<DH>& sdO = *(reinterpret_cast<Tile<DH>*>(sm) + 1);
  Tile<DH>* sK = reinterpret_cast<Tile<DH>*>(sm) + 2;
  Tile<DH>* sV = sK + 2;
  const int nqt = (S + BT - 1) / BT;
  const int qt = nqt - 1 - blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int q0 = qt * BT;
  const int64_t rowbase = (int64_t)b * S * d + (int64_t)h * DH;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const float sl2 = scale * kLog2e;

  sQ.load(q + rowbase, d, q0, S);
  sdO.load(dO + rowbase, d, q0, S);
  sK[0].load(k + rowbase, d, 0, S);
  sV[0].load(v + rowbase, d, 0, S);
  cp_commit();

  const int r_lo = q0 + warp * 16 + (lane >> 2);
  float Lr[2], Dr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = r_lo + r * 8;
    Lr[r] = row < S ? lse[(int64_t)bh * S + row] * kLog2e : INFINITY;
    Dr[r] = row < S ? Dv[(int64_t)bh * S + row] : 0.f;
  }
  uint32_t qa[DH / 16][4], oa[DH / 16][4];
  float dqa[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) dqa[i][0] = dqa[i][1] = dqa[i][2] = dqa[i][3] = 0.f;

  const int nkt = qt + 1;
  for (int kt = 0; kt < nkt; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nkt) {
      sK[cur ^ 1].load(k + rowbase, d, (kt + 1) * BT, S);
      sV[cur ^ 1].load(v + rowbase, d, (kt + 1) * BT, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        sQ.a_frag(qa[kk], warp * 16, kk);
        sdO.a_frag(oa[kk], warp * 16, kk);
      }
    }
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int n8 = 0; n8 < 8; n8 += 2) {
        uint32_t bk[4], bv[4];
        sK[cur].b_frag_rows(bk, n8, kk);
        sV[cur].b_frag_rows(bv, n8, kk);
        mma16816(s[n8], qa[kk], bk[0], bk[1]);
        mma16816(s[n8 + 1], qa[kk], bk[2], bk[3]);
        mma16816(dp[n8], oa[kk], bv[0], bv[1]);
        mma16816(dp[n8 + 1], oa[kk], bv[2], bv[3]);
      }
    }
    const int k0 = kt * BT;
#pragma unroll
    for (int n8 = 0; n8 < 8; ++n8)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + n8 * 8 + (lane & 3) * 2 + (e & 1);
        const int row = r_lo + (e >> 1) * 8;
        float p = exp2f(s[n8][e] * sl2 - Lr[e >> 1]);
        if (key > row || key >= S || row >= S) p = 0.f;
        dp[n8][e] = p * (dp[n8][e] - Dr[e >> 1]) * scale;
      }
    // dQ += dS K   (k = keys)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t da[4] = {pack_bf16(dp[2 * kk][0], dp[2 * kk][1]), pack_bf16(dp[2 * kk][2], dp[2 * kk][3]),
                        pack_bf16(dp[2 * kk + 1][0], dp[2 * kk + 1][1]),
                        pack_bf16(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
      for (int n8 = 0; n8 < DH / 8; n8 += 2) {
        uint32_t bk[4];
        sK[cur].b_frag_cols(bk, n8, kk);
        mma16816(dqa[n8], da, bk[0], bk[1]);
        mma16816(dqa[n8 + 1], da, bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = r_lo + r * 8;
    if (row >= S) continue;
    bf16* qr = dq + rowbase + (int64_t)row * d;
#pragma unroll
    for (int n8 = 0; n8 < DH / 8; ++n8) {
      const int c = n8 * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(qr + c) = pack_bf16(dqa[n8][2 * r], dqa[n8][2 * r + 1]);
    }
  }
}

// D[row] = dO_row . O_row  (bf16 inputs, fp32 accumulate), one warp per row
__global__ void attn_dot_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dO,
                                float* __restrict__ Dv, int B, int S, int H, int d) {
  const int dh = d / H, lane = threadIdx.x & 31, warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  if (row >= B * H * S) return;
  const int i = row % S, bh = row / S, h = bh % H, b = bh / H;
  const int64_t off = ((int64_t)(b * S + i)) * d + h * dh;
  float acc = 0.f;
  for (int c = lane * 2; c < dh; c += 64) {
    const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(o + off + c);
    const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(dO + off + c);
    acc += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
  }
  acc = warp_sum(acc);
  if (lane == 0) Dv[row] = acc;
}

template <int DH>
size_t fwd_smem() { return sizeof(Tile<DH>) * 5; }
template <int DH>
size_t bwd_smem_dkdv() { return sizeof(Tile<DH>) * 6 + 4 * BT * sizeof(float); }
template <int DH>
size_t bwd_smem_dq() { return sizeof(Tile<DH>) * 6; }

template <int DH>
void launch_fwd(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                int H, int d, cudaStream_t st) {
  const size_t smem = fwd_smem<DH>();
  static std::atomic<uint64_t> cfg{0};
  set_max_smem_once(cfg, attn_fwd_mma_kernel<DH>, (int)smem);
  dim3 grid((S + BT - 1) / BT, B * H);
  attn_fwd_mma_kernel<DH><<<grid, kWarps * 32, smem, st>>>(q, k, v, o, lse, S, H, d,
                                                           rsqrtf((float)DH));
  PH_LAUNCH_CHECK();
}

template <int DH>
void launch_bwd(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                const float* lse, float* Dv, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H,
                int d, cudaStream_t st) {
  const int rows = B * H * S;
  attn_dot_kernel<<<(rows + 7) / 8, 256, 0, st>>>(o, dO, Dv, B, S, H, d);
  PH_LAUNCH_CHECK();
  static std::atomic<uint64_t> cfg1{0}, cfg2{0};
  set_max_smem_once(cfg1, attn_bwd_dkdv_mma_kernel<DH>, (int)bwd_smem_dkdv<DH>());
  set_max_smem_once(cfg2, attn_bwd_dq_mma_kernel<DH>, (int)bwd_smem_dq<DH>());
  dim3 grid((S + BT - 1) / BT, B * H);
  const float scale = rsqrtf((float)DH);
  attn_bwd_dkdv_mma_kernel<DH><<<grid, kWarps * 32, bwd_smem_dkdv<DH>(), st>>>(
      q, k, v, dO, lse, Dv, dk, dv, S, H, d, scale);
  PH_LAUNCH_CHECK();
  attn_bwd_dq_mma_kernel<DH><<<grid, kWarps * 32, bwd_smem_dq<DH>(), st>>>(q, k, v, dO, lse, Dv,
                                                                           dq, S, H, d, scale);
  PH_LAUNCH_CHECK();
}

}  // namespace

bool attn_mma_supported(int dh) { return dh == 16 || dh == 32 || dh == 64 || dh == 128; }

void attn_fwd_mma(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                  int H, int d, cudaStream_t st) {
  switch (d / H) {
    case 16: launch_fwd<16>(q, k, v, o, lse, B, S, H, d, st); break;
    case 32: launch_fwd<32>(q, k, v, o, lse, B, S, H, d, st); break;
    case 64: launch_fwd<64>(q, k, v, o, lse, B, S, H, d, st); break;
    case 128: launch_fwd<128>(q, k, v, o, lse, B, S, H, d, st); break;
    default: throw Error(PHOTON_ERR_CONFIG, "attention: head dim must be 16/32/64/128 for bf16");
  }
}

void attn_bwd_mma(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                  const float* lse, float* Dv, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H,
                  int d, cudaStream_t st) {
  switch (d / H) {
    case 16: launch_bwd<16>(q, k, v, o, dO, lse, Dv, dq, dk, dv, B, S, H, d, st); break;
    case 32: launch_bwd<32>(q, k, v, o, dO, lse, Dv, dq, dk, dv, B, S, H, d, st); break;
    case 64: launch_bwd<64>(q, k, v, o, dO, lse, Dv, dq, dk, dv, B, S, H, d, st); break;
    case 128: launch_bwd<128>(q, k, v, o, dO, lse, Dv, dq, dk, dv, B, S, H, d, st); break;
    default: throw Error(PHOTON_ERR_CONFIG, "attention: head dim must be 16/32/64/128 for bf16");
  }
}

}  // namespace k
}  // namespace photon
