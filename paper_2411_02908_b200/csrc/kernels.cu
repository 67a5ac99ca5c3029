// kernels.cu -- embedding, layer norm, bias-gradient column sums, fused
// softmax cross-entropy and the SIMT attention path of the client step.
// Citations: /root/reference/proj/core/src/tensor.cpp.
#include <atomic>
#include "kernels.cuh"
#include "sm100.cuh"

namespace photon {
namespace k {

// ============================================================================
// Embedding: x[m] = tok[tokens[m]] + pos[m % S]   (model.cpp:140-141)
// ============================================================================
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tokens, const float* __restrict__ tok,
                                 const float* __restrict__ pos, float* __restrict__ x, int M,
                                 int S, int d) {
  pdl_launch_dependents();
  pdl_wait();
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int m = blockIdx.x * warps + threadIdx.x / 32; m < M; m += gridDim.x * warps) {
    const float* te = tok + (size_t)tokens[m] * d;
    const float* pe = pos + (size_t)(m % S) * d;
    float* xo = x + (size_t)m * d;
    if ((d & 3) == 0) {
      for (int j = lane * 4; j < d; j += 128) {
        const float4 a = *reinterpret_cast<const float4*>(te + j);
        const float4 b = *reinterpret_cast<const float4*>(pe + j);
        *reinterpret_cast<float4*>(xo + j) = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      }
    } else {
      for (int j = lane; j < d; j += 32) xo[j] = te[j] + pe[j];
    }
  }
}

void embed_fwd(const int32_t* tokens, const float* tok, const float* pos, float* x, int M, int S,
               int d, cudaStream_t st) {
  const int blocks = std::min<int>(cdiv(M, 8), kNumSMs * 16);
  launch_pdl(embed_fwd_kernel, blocks, 256, 0, st, tokens, tok, pos, x, M, S, d);
  PH_LAUNCH_CHECK();
}

// gather_rows backward (tensor.cpp:305-318): duplicates accumulate in ascending
// row order.  One warp per vocab row walks that token's rows (CSR sorted by
// row), so the sum order is fixed and no atomics are needed.  With d % 128 == 0
// each lane keeps its d / 128 float4 columns in registers and issues all of a
// row's loads at once (the generic loop below is the fallback).
template <int NV4>
__global__ void embed_bwd_tok_vec_kernel(const float* __restrict__ dx, const int32_t* __restrict__ off,
                                         const int32_t* __restrict__ rows, float* __restrict__ dtok,
                                         int V, int d, int row0, int M, int acc) {
  pdl_launch_dependents();
  pdl_wait();
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int v = blockIdx.x * warps + threadIdx.x / 32; v < V; v += gridDim.x * warps) {
    const int b = off[v], e = off[v + 1];
    float4 a[NV4];
#pragma unroll
    for (int c = 0; c < NV4; ++c) a[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = b; r < e; ++r) {
      const int m = rows[r] - row0;  // this micro-batch's rows only
      if ((unsigned)m >= (unsigned)M) continue;
      const float4* src = reinterpret_cast<const float4*>(dx + (size_t)m * d);
      float4 t[NV4];
#pragma unroll
      for (int c = 0; c < NV4; ++c) t[c] = src[lane + 32 * c];
#pragma unroll
      for (int c = 0; c < NV4; ++c) {
        a[c].x += t[c].x;
        a[c].y += t[c].y;
        a[c].z += t[c].z;
        a[c].w += t[c].w;
      }
    }
    float4* out = reinterpret_cast<float4*>(dtok + (size_t)v * d);
#pragma unroll
    for (int c = 0; c < NV4; ++c) {
      float4 o = a[c];
      if (acc) {
        const float4 p = out[lane + 32 * c];
        o = make_float4(p.x + o.x, p.y + o.y, p.z + o.z, p.w + o.w);
      }
      out[lane + 32 * c] = o;
    }
  }
}
__global__ void embed_bwd_tok_kernel(const float* __restrict__ dx, const int32_t* __restrict__ off,
                                     const int32_t* __restrict__ rows, float* __restrict__ dtok,
                                     int V, int d, int row0, int M, int acc) {
  pdl_launch_dependents();
  pdl_wait();
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int v = blockIdx.x * warps + threadIdx.x / 32; v < V; v += gridDim.x * warps) {
    const int b = off[v], e = off[v + 1];
    float* out = dtok + (size_t)v * d;
    for (int j = lane; j < d; j += 32) {
      float a = 0.f;
      for (int r = b; r < e; ++r) {
        const int m = rows[r] - row0;  // this micro-batch's rows only
        if ((unsigned)m < (unsigned)M) a += dx[(size_t)m * d + j];
      }
      out[j] = acc ? out[j] + a : a;
    }
  }
}
// dpos[s] = sum over the batch's rows m = s, s + S, ... in ascending m; with
// d % 4 == 0 a thread owns a float4 of a position and has four rows' loads in
// flight (the per-element sum order is unchanged)
__global__ void embed_bwd_pos_kernel(const float* __restrict__ dx, float* __restrict__ dpos,
                                     int M, int S, int d, int acc) {
  pdl_launch_dependents();
  pdl_wait();
  if (d % 4 == 0) {
    const int d4 = d / 4;
    const size_t total4 = (size_t)S * d4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total4;
         i += (size_t)gridDim.x * blockDim.x) {
      const int s = (int)(i / d4), j4 = (int)(i % d4);
      const float4* src = reinterpret_cast<const float4*>(dx) + j4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      int m = s;
      for (; m + 3 * S < M; m += 4 * S) {
        const float4 t0 = src[(size_t)m * d4], t1 = src[(size_t)(m + S) * d4];
        const float4 t2 = src[(size_t)(m + 2 * S) * d4], t3 = src[(size_t)(m + 3 * S) * d4];
        a.x = (((a.x + t0.x) + t1.x) + t2.x) + t3.x;
        a.y = (((a.y + t0.y) + t1.y) + t2.y) + t3.y;
        a.z = (((a.z + t0.z) + t1.z) + t2.z) + t3.z;
        a.w = (((a.w + t0.w) + t1.w) + t2.w) + t3.w;
      }
      for (; m < M; m += S) {
        const float4 t = src[(size_t)m * d4];
        a.x += t.x;
        a.y += t.y;
        a.z += t.z;
        a.w += t.w;
      }
      float4* o = reinterpret_cast<float4*>(dpos) + i;
      if (acc) {
        const float4 p = *o;
        a = make_float4(p.x + a.x, p.y + a.y, p.z + a.z, p.w + a.w);
      }
      *o = a;
    }
    return;
  }
  const size_t total = (size_t)S * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / d), j = (int)(i % d);
    float a = 0.f;
    for (int m = s; m < M; m += S) a += dx[(size_t)m * d + j];
    dpos[i] = acc ? dpos[i] + a : a;
  }
}

void embed_bwd(const float* dx, const int32_t* csr_off, const int32_t* csr_rows, float* dtok,
               float* dpos, int V, int M, int S, int d, cudaStream_t st, int row0, bool acc) {
  const int tok_grid = std::min<int>(cdiv(V, 8), kNumSMs * 16);
  const bool al = (reinterpret_cast<uintptr_t>(dx) & 15) == 0 && (reinterpret_cast<uintptr_t>(dtok) & 15) == 0;
  if (al && d == 768)
    launch_pdl(embed_bwd_tok_vec_kernel<6>, tok_grid, 256, 0, st, dx, csr_off, csr_rows, dtok, V, d,
               row0, M, acc ? 1 : 0);
  else if (al && d == 2048)
    launch_pdl(embed_bwd_tok_vec_kernel<16>, tok_grid, 256, 0, st, dx, csr_off, csr_rows, dtok, V, d,
               row0, M, acc ? 1 : 0);
  else if (al && d == 4096)
    launch_pdl(embed_bwd_tok_vec_kernel<32>, tok_grid, 256, 0, st, dx, csr_off, csr_rows, dtok, V, d,
               row0, M, acc ? 1 : 0);
  else
    launch_pdl(embed_bwd_tok_kernel, tok_grid, 256, 0, st, dx, csr_off, csr_rows, dtok, V, d, row0, M,
               acc ? 1 : 0);
  PH_LAUNCH_CHECK();
  launch_pdl(embed_bwd_pos_kernel, std::min<int>(cdiv((uint64_t)S * d, 256), kNumSMs * 8), 256, 0, st, 
      dx, dpos, M, S, d, acc ? 1 : 0);
  PH_LAUNCH_CHECK();
}

// ============================================================================
// LayerNorm forward: two-pass mean / biased variance, eps 1e-5 (tensor.cpp:336-357)
// One warp per row; fp32 statistics.
// ============================================================================
template <typename T>
__global__ void ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                              const float* __restrict__ bias, T* __restrict__ y,
                              float* __restrict__ mean_out, float* __restrict__ rstd_out, int M,
                              int d) {
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  const float inv_d = 1.0f / (float)d;
  for (int m = blockIdx.x * warps + threadIdx.x / 32; m < M; m += gridDim.x * warps) {
    const float* xr = x + (size_t)m * d;
    float s = 0.f;
    for (int j = lane; j < d; j += 32) s += xr[j];
    const float mean = warp_sum(s) * inv_d;
    float v = 0.f;
    for (int j = lane; j < d; j += 32) {
      const float t = xr[j] - mean;
      v += t * t;
    }
    const float rstd = rsqrtf(warp_sum(v) * inv_d + 1e-5f);
    T* yr = y + (size_t)m * d;
    for (int j = lane; j < d; j += 32) yr[j] = from_f<T>(gain[j] * ((xr[j] - mean) * rstd) + bias[j]);
    if (lane == 0) {
      mean_out[m] = mean;
      rstd_out[m] = rstd;
    }
  }
}

// Register-resident variant for d = 128 * NV: each lane holds NV float4 of the
// row (16-byte coalesced loads), so x is read from HBM exactly once.
__device__ __forceinline__ void store4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store4(bf16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = u;
}

template <typename T, int NV>
__global__ void __launch_bounds__(256) ln_fwd_vec_kernel(const float* __restrict__ x,
                                                         const float* __restrict__ gain,
                                                         const float* __restrict__ bias,
                                                         T* __restrict__ y,
                                                         float* __restrict__ mean_out,
                                                         float* __restrict__ rstd_out, int M) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int D = NV * 128;
  const int lane = threadIdx.x & 31;
  const float inv_d = 1.0f / (float)D;
  const int step = gridDim.x * 8;
  // the next row's loads are issued before this row's reductions and stores, so
  // every warp keeps a row in flight through its arithmetic
  float4 nx[NV];
  int m = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (m < M) {
#pragma unroll
    for (int i = 0; i < NV; ++i) nx[i] = reinterpret_cast<const float4*>(x + (size_t)m * D)[lane + 32 * i];
  }
  for (; m < M; m += step) {
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = nx[i];
    if (m + step < M) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        nx[i] = reinterpret_cast<const float4*>(x + (size_t)(m + step) * D)[lane + 32 * i];
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += ((v[i].x + v[i].y) + v[i].z) + v[i].w;
    const float mean = warp_sum(s) * inv_d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, e = v[i].w - mean;
      q += ((a * a + b * b) + cc * cc) + e * e;
    }
    const float rstd = rsqrtf(warp_sum(q) * inv_d + 1e-5f);
    T* yr = y + (size_t)m * D;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 g = reinterpret_cast<const float4*>(gain)[c4];
      const float4 b = reinterpret_cast<const float4*>(bias)[c4];
      store4(yr + 4 * c4, g.x * ((v[i].x - mean) * rstd) + b.x, g.y * ((v[i].y - mean) * rstd) + b.y,
             g.z * ((v[i].z - mean) * rstd) + b.z, g.w * ((v[i].w - mean) * rstd) + b.w);
    }
    if (lane == 0) {
      mean_out[m] = mean;
      rstd_out[m] = rstd;
    }
  }
}

// Wide rows (d = 512 * WPR: 1,024 .. 4,096, the 1.3B / 7B widths): WPR warps of
// a CTA share a row, each holding its 512-column slice in registers (4 float4
// per lane); the two row sums cross warps through shared memory (double-
// buffered by row parity, partials added in warp order), one named barrier per
// sum.  8 / WPR rows in flight per CTA.
template <typename T, int WPR>
__global__ void __launch_bounds__(256) ln_fwd_split_kernel(const float* __restrict__ x,
                                                           const float* __restrict__ gain,
                                                           const float* __restrict__ bias,
                                                           T* __restrict__ y,
                                                           float* __restrict__ mean_out,
                                                           float* __restrict__ rstd_out, int M) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int NV = 4, D = NV * 128 * WPR, G = 8 / WPR;
  __shared__ float red[2][2][8];  // [row parity][sum][warp]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = warp / WPR, wi = warp % WPR;
  const int c4base = wi * NV * 32;  // float4 index of this warp's slice
  const float inv_d = 1.0f / (float)D;
  int it = 0;
  for (int m = blockIdx.x * G + grp; m < M; m += gridDim.x * G, ++it) {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)m * D) + c4base;
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = xr[lane + 32 * i];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += ((v[i].x + v[i].y) + v[i].z) + v[i].w;
    s = warp_sum(s);
    float* rs = red[it & 1][0];
    if (lane == 0) rs[warp] = s;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) tot += rs[grp * WPR + w];
    const float mean = tot * inv_d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, e = v[i].w - mean;
      q += ((a * a + b * b) + cc * cc) + e * e;
    }
    q = warp_sum(q);
    float* rq = red[it & 1][1];
    if (lane == 0) rq[warp] = q;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
    float qt = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) qt += rq[grp * WPR + w];
    const float rstd = rsqrtf(qt * inv_d + 1e-5f);
    T* yr = y + (size_t)m * D;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = c4base + lane + 32 * i;
      const float4 g = reinterpret_cast<const float4*>(gain)[c4];
      const float4 b = reinterpret_cast<const float4*>(bias)[c4];
      store4(yr + 4 * c4, g.x * ((v[i].x - mean) * rstd) + b.x, g.y * ((v[i].y - mean) * rstd) + b.y,
             g.z * ((v[i].z - mean) * rstd) + b.z, g.w * ((v[i].w - mean) * rstd) + b.w);
    }
    if (wi == 0 && lane == 0) {
      mean_out[m] = mean;
      rstd_out[m] = rstd;
    }
  }
}

template <typename T>
void ln_fwd(const float* x, const float* gain, const float* bias, T* y, float* mean, float* rstd,
            int M, int d, cudaStream_t st) {
  const int grid = std::min<int>(cdiv(M, 8), kNumSMs * 8);
  switch (d) {
#define PH_LNF(NV)                                                                       \
  case NV * 128:                                                                         \
    launch_pdl(ln_fwd_vec_kernel<T, NV>, grid, 256, 0, st, x, gain, bias, y, mean, rstd, M);      \
    break;
    PH_LNF(1) PH_LNF(2) PH_LNF(3) PH_LNF(4) PH_LNF(5) PH_LNF(6)
#undef PH_LNF
#define PH_LNFS(WPR)                                                                      \
  case 512 * WPR:                                                                          \
    launch_pdl(ln_fwd_split_kernel<T, WPR>, std::min<int>(cdiv(M, 8 / WPR), kNumSMs * 8), 256, 0, st,  \
        x, gain, bias, y, mean, rstd, M);                                                  \
    break;
    PH_LNFS(2) PH_LNFS(4) PH_LNFS(8)
#undef PH_LNFS
    default:
      ln_fwd_kernel<T><<<std::min<int>(cdiv(M, 8), kNumSMs * 16), 256, 0, st>>>(x, gain, bias, y,
                                                                                mean, rstd, M, d);
  }
  PH_LAUNCH_CHECK();
}

// LayerNorm backward (tensor.cpp:370-392):
//   dx = rstd * (dxh - mean(dxh) - xhat * mean(dxh * xhat)),  dxh = dy * gain
// plus dgain = sum dy*xhat, dbias = sum dy over rows (per-block partials).
constexpr int kLnBwdBlocks = kNumSMs * 2;
constexpr int kLnBwdWarps = 8;
int ln_bwd_parts() { return kLnBwdBlocks; }

template <typename T>
__global__ void __launch_bounds__(kLnBwdWarps * 32)
ln_bwd_kernel(const T* __restrict__ dy, const float* __restrict__ x,
              const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
              const float* __restrict__ gain, const float* dres, float* dx_out,
              T* __restrict__ dx_T, float* __restrict__ part, int M, int d, int nsum) {
  extern __shared__ float sm[];  // [warps][nsum][d]: dgain | dbias (| column sums of dx_out)
  const int warps = blockDim.x / 32;  // sized by the launcher to the shared-memory budget
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  float* my = sm + (size_t)warp * nsum * d;
  for (int j = lane; j < nsum * d; j += 32) my[j] = 0.f;
  const float inv_d = 1.0f / (float)d;
  for (int m = blockIdx.x * warps + warp; m < M; m += gridDim.x * warps) {
    const T* dyr = dy + (size_t)m * d;
    const float* xr = x + (size_t)m * d;
    const float mean = mean_in[m], rstd = rstd_in[m];
    float s1 = 0.f, s2 = 0.f;
    for (int j = lane; j < d; j += 32) {
      const float xh = (xr[j] - mean) * rstd;
      const float g = to_f<T>(dyr[j]);
      const float dxh = g * gain[j];
      s1 += dxh;
      s2 += dxh * xh;
      my[j] += g * xh;
      my[d + j] += g;
    }
    s1 = warp_sum(s1) * inv_d;
    s2 = warp_sum(s2) * inv_d;
    float* out = dx_out + (size_t)m * d;
    const float* rr = dres ? dres + (size_t)m * d : nullptr;
    T* outT = dx_T ? dx_T + (size_t)m * d : nullptr;
    for (int j = lane; j < d; j += 32) {
      const float xh = (xr[j] - mean) * rstd;
      float g = rstd * (to_f<T>(dyr[j]) * gain[j] - s1 - xh * s2);
      if (rr) g += rr[j];
      out[j] = g;
      if (outT) outT[j] = from_f<T>(g);
      if (nsum == 3) my[2 * d + j] += g;
    }
  }
  __syncthreads();
  // reduce warps -> block partial
  for (int j = threadIdx.x; j < nsum * d; j += blockDim.x) {
    float acc = 0.f;
    for (int w = 0; w < warps; ++w) acc += sm[(size_t)w * nsum * d + j];
    part[(size_t)blockIdx.x * 3 * d + j] = acc;
  }
}

// out[j] = sum_p part[p*stride + j] for j < n, with columns j >= split going to
// out1[j - split].  Fixed order: slice s of 32 sums parts p = s (mod 32) in
// ascending p, then the 32 slices are added in ascending s.  32 columns per
// CTA of 1024 threads, so each thread has only ~nparts/32 partials to read,
// all issued before the first add (the partials were just written: L2 hits;
// the kernel is latency-, not bandwidth-bound).
__device__ __forceinline__ void colreduce_body(const float* __restrict__ part, int nparts, int n,
                                               int stride, float* __restrict__ out, int split,
                                               float* __restrict__ out1, int acc_out, int split2,
                                               float* __restrict__ out2, int bx) {
  __shared__ float red[32][33];
  const int cl = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int j = bx * 32 + cl;
  float acc = 0.f;
  if (j < n) {
    int p = s;
    for (; p + 96 < nparts; p += 128) {  // four independent loads in flight
      const float a = part[(size_t)p * stride + j], b = part[(size_t)(p + 32) * stride + j];
      const float c2 = part[(size_t)(p + 64) * stride + j], d2 = part[(size_t)(p + 96) * stride + j];
      acc = (((acc + a) + b) + c2) + d2;
    }
    for (; p < nparts; p += 32) acc += part[(size_t)p * stride + j];
  }
  red[s][cl] = acc;
  __syncthreads();
  if (s == 0 && j < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 32; ++w) t += red[w][cl];
    float* o = j < split ? out + j : j < split2 ? out1 + (j - split) : out2 + (j - split2);
    *o = acc_out ? *o + t : t;  // micro-batches after the first add onto the gradient
  }
}
__global__ void __launch_bounds__(1024) colreduce_kernel(const float* __restrict__ part, int nparts,
                                                         int n, int stride, float* __restrict__ out,
                                                         int split, float* __restrict__ out1,
                                                         int acc_out, int split2,
                                                         float* __restrict__ out2) {
  colreduce_body(part, nparts, n, stride, out, split, out1, acc_out, split2, out2, blockIdx.x);
}
// columns [0, split) -> out, [split, split2) -> out1, [split2, n) -> out2
static void colreduce(const float* part, int nparts, int n, int stride, float* out, int split,
                      float* out1, cudaStream_t st, bool acc = false, int split2 = -1,
                      float* out2 = nullptr, ReduceJobs* defer = nullptr) {
  if (defer) {
    defer->cols.push_back(ColJob{part, nparts, n, stride, split, split2 < 0 ? n : split2, out, out1,
                                 out2, acc ? 1 : 0});
    return;
  }
  colreduce_kernel<<<cdiv(n, 32), 1024, 0, st>>>(part, nparts, n, stride, out, split, out1,
                                                 acc ? 1 : 0, split2 < 0 ? n : split2, out2);
  PH_LAUNCH_CHECK();
}

// First level of a many-part column reduction: CTA (x, y) sums parts
// [y * per, (y + 1) * per) of 32 columns in the colreduce order and writes
// row y of `out` ([gridDim.y][n]).
// Several same-shaped partial arrays at once: column J of the combined
// [nseg * n] row is column J % n of segment J / n (segments seg_stride apart).
__device__ __forceinline__ void colreduce_rows_body(const float* __restrict__ part, int nparts,
                                                    int per, int n, float* __restrict__ out,
                                                    int nseg, size_t seg_stride, int bx, int by) {
  __shared__ float red[8][33];
  const int cl = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int J = bx * 32 + cl, nn = n * nseg;
  const int seg = J / n, j = J - seg * n;
  const float* ps = part + (size_t)seg * seg_stride;
  const int p0 = by * per, p1 = min(nparts, p0 + per);
  float acc = 0.f;
  if (J < nn) {
    int p = p0 + s;
    for (; p + 8 < p1; p += 16) {
      const float a = ps[(size_t)p * n + j], b = ps[(size_t)(p + 8) * n + j];
      acc = (acc + a) + b;
    }
    for (; p < p1; p += 8) acc += ps[(size_t)p * n + j];
  }
  red[s][cl] = acc;
  __syncthreads();
  if (s == 0 && J < nn) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][cl];
    out[(size_t)by * nn + J] = t;
  }
}
__global__ void __launch_bounds__(256) colreduce_rows_kernel(const float* __restrict__ part, int nparts,
                                                             int per, int n, float* __restrict__ out,
                                                             int nseg, size_t seg_stride) {
  colreduce_rows_body(part, nparts, per, n, out, nseg, seg_stride, blockIdx.x, blockIdx.y);
}

// ---- deferred column reductions, batched ------------------------------------------
// A job table travels as a kernel parameter; CTA b runs the job whose CTA range
// holds b, with exactly the body (and so the summation order) of the one-job
// kernels above.
constexpr int kReduceBatch = 160;
struct RowTable {
  int njobs;
  int start[kReduceBatch + 1];
  RowJob job[kReduceBatch];
};
struct ColTable {
  int njobs;
  int start[kReduceBatch + 1];
  ColJob job[kReduceBatch];
};
__device__ __forceinline__ int find_job(const int* start, int njobs, int b) {
  int lo = 0, hi = njobs - 1;  // largest j with start[j] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__global__ void __launch_bounds__(256) reduce_rows_batch_kernel(const __grid_constant__ RowTable t) {
  pdl_launch_dependents();
  pdl_wait();
  const int j = find_job(t.start, t.njobs, blockIdx.x);
  const RowJob& r = t.job[j];
  const int local = blockIdx.x - t.start[j], nx = (r.n * r.nseg + 31) / 32;
  colreduce_rows_body(r.part, r.nparts, r.per, r.n, r.out, r.nseg, r.seg_stride, local % nx,
                      local / nx);
}
__global__ void __launch_bounds__(1024) reduce_cols_batch_kernel(const __grid_constant__ ColTable t) {
  pdl_launch_dependents();
  pdl_wait();
  const int j = find_job(t.start, t.njobs, blockIdx.x);
  const ColJob& c = t.job[j];
  colreduce_body(c.part, c.nparts, c.n, c.stride, c.out, c.split, c.out1, c.acc, c.split2, c.out2,
                 blockIdx.x - t.start[j]);
}
void run_reduce_jobs(ReduceJobs& jobs, cudaStream_t st) {
  for (size_t b = 0; b < jobs.rows.size(); b += kReduceBatch) {
    RowTable t{};
    t.njobs = (int)std::min<size_t>(kReduceBatch, jobs.rows.size() - b);
    int n = 0;
    for (int i = 0; i < t.njobs; ++i) {
      t.job[i] = jobs.rows[b + i];
      t.start[i] = n;
      n += cdiv(t.job[i].n * t.job[i].nseg, 32) * t.job[i].used;
    }
    t.start[t.njobs] = n;
    launch_pdl(reduce_rows_batch_kernel, n, 256, 0, st, t);
    PH_LAUNCH_CHECK();
  }
  for (size_t b = 0; b < jobs.cols.size(); b += kReduceBatch) {
    ColTable t{};
    t.njobs = (int)std::min<size_t>(kReduceBatch, jobs.cols.size() - b);
    int n = 0;
    for (int i = 0; i < t.njobs; ++i) {
      t.job[i] = jobs.cols[b + i];
      t.start[i] = n;
      n += cdiv(t.job[i].n, 32);
    }
    t.start[t.njobs] = n;
    launch_pdl(reduce_cols_batch_kernel, n, 1024, 0, st, t);
    PH_LAUNCH_CHECK();
  }
  jobs.rows.clear();
  jobs.cols.clear();
}

size_t colsum_parts_scratch_floats(int N) { return (size_t)kColsumPartGroups * N; }

void colsum_parts(const float* part, int nparts, int N, float* scratch, float* out, cudaStream_t st,
                  bool acc, ReduceJobs* defer) {
  const int groups = std::min(kColsumPartGroups, nparts);
  const int per = cdiv(nparts, groups);
  const int used = cdiv(nparts, per);
  if (defer) {
    defer->rows.push_back(RowJob{part, nparts, per, N, 1, 0, scratch, used});
  } else {
    colreduce_rows_kernel<<<dim3(cdiv(N, 32), used), 256, 0, st>>>(part, nparts, per, N, scratch, 1, 0);
    PH_LAUNCH_CHECK();
  }
  colreduce(scratch, used, N, N, out, N, nullptr, st, acc, -1, nullptr, defer);
}

void colsum_parts3(const float* part, size_t seg_stride, int nparts, int N, float* scratch,
                   float* out0, float* out1, float* out2, cudaStream_t st, bool acc,
                   ReduceJobs* defer) {
  const int groups = std::min(kColsumPartGroups, nparts);
  const int per = cdiv(nparts, groups);
  const int used = cdiv(nparts, per);
  if (defer) {
    defer->rows.push_back(RowJob{part, nparts, per, N, 3, seg_stride, scratch, used});
  } else {
    colreduce_rows_kernel<<<dim3(cdiv(3 * N, 32), used), 256, 0, st>>>(part, nparts, per, N, scratch,
                                                                        3, seg_stride);
    PH_LAUNCH_CHECK();
  }
  colreduce(scratch, used, 3 * N, 3 * N, out0, N, out1, st, acc, 2 * N, out2, defer);
}

// Register-resident variant for d = 128 * NV: one warp per row, x, dy and the
// residual gradient of a row all requested before any arithmetic (one DRAM
// latency per row instead of two), each read once as float4.  The column
// accumulators -- dgain, dbias and the column sums of the output -- live in
// shared memory per warp (each lane owns fixed columns: no conflicts), which
// keeps the registers for the loads in flight; warps are reduced in a fixed
// order at the end.  dres may alias dx_out (in-place residual accumulation),
// so neither is restrict.
constexpr int kLnBwdVecSmem(int D) { return (D / 4) * 16 + 3 * kLnBwdWarps * D * 4; }

template <typename T, int NV>
__global__ void __launch_bounds__(256, 2)
ln_bwd_vec_kernel(const T* __restrict__ dy, const float* __restrict__ x,
                  const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                  const float* __restrict__ gain, const float* dres, float* dx_out,
                  T* __restrict__ dx_T, float* __restrict__ part, int M, int osum) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int D = NV * 128;
  extern __shared__ float4 lnb_sm[];
  float4* gs = lnb_sm;                                      // [D/4] gain
  float* red = reinterpret_cast<float*>(lnb_sm + D / 4);    // [3][warps][D]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* ag = reinterpret_cast<float4*>(red + (size_t)(0 * kLnBwdWarps + warp) * D);
  float4* ab = reinterpret_cast<float4*>(red + (size_t)(1 * kLnBwdWarps + warp) * D);
  float4* ao = reinterpret_cast<float4*>(red + (size_t)(2 * kLnBwdWarps + warp) * D);
  for (int j = threadIdx.x; j < D / 4; j += blockDim.x) gs[j] = reinterpret_cast<const float4*>(gain)[j];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    ag[lane + 32 * i] = z;
    ab[lane + 32 * i] = z;
    ao[lane + 32 * i] = z;
  }
  __syncthreads();
  const float inv_d = 1.0f / (float)D;
  for (int m = blockIdx.x * kLnBwdWarps + warp; m < M; m += gridDim.x * kLnBwdWarps) {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)m * D);
    const T* gr = dy + (size_t)m * D;
    const float4* rr = dres ? reinterpret_cast<const float4*>(dres + (size_t)m * D) : nullptr;
    float4 xv[NV], gv[NV], rv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xv[i] = xr[lane + 32 * i];
      gv[i] = ld4f(gr + 4 * (lane + 32 * i));
      rv[i] = rr ? rr[lane + 32 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float mean = mean_in[m], rstd = rstd_in[m];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 gg = gs[c4];
      float4 a = ag[c4], b = ab[c4];
#define PH_LNB_ACC(c)                                 \
  {                                                   \
    const float xh = (xv[i].c - mean) * rstd;         \
    const float dxh = gv[i].c * gg.c;                 \
    s1 += dxh;                                        \
    s2 += dxh * xh;                                   \
    a.c += gv[i].c * xh;                              \
    b.c += gv[i].c;                                   \
  }
      PH_LNB_ACC(x) PH_LNB_ACC(y) PH_LNB_ACC(z) PH_LNB_ACC(w)
#undef PH_LNB_ACC
      ag[c4] = a;
      ab[c4] = b;
    }
    s1 = warp_sum(s1) * inv_d;
    s2 = warp_sum(s2) * inv_d;
    float* out = dx_out + (size_t)m * D;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 gg = gs[c4];
      float4 r = rv[i];
      r.x += rstd * (gv[i].x * gg.x - s1 - ((xv[i].x - mean) * rstd) * s2);
      r.y += rstd * (gv[i].y * gg.y - s1 - ((xv[i].y - mean) * rstd) * s2);
      r.z += rstd * (gv[i].z * gg.z - s1 - ((xv[i].z - mean) * rstd) * s2);
      r.w += rstd * (gv[i].w * gg.w - s1 - ((xv[i].w - mean) * rstd) * s2);
      reinterpret_cast<float4*>(out)[c4] = r;
      if (dx_T) store4(dx_T + (size_t)m * D + 4 * c4, r.x, r.y, r.z, r.w);
      if (osum) {
        float4 o = ao[c4];
        o.x += r.x;
        o.y += r.y;
        o.z += r.z;
        o.w += r.w;
        ao[c4] = o;
      }
    }
  }
  // block partials: [dgain | dbias | dsum], warps summed in ascending order
  __syncthreads();
  const int nsum = osum ? 3 : 2;
  for (int j = threadIdx.x; j < nsum * D; j += blockDim.x) {
    const int a = j / D, c = j % D;
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kLnBwdWarps; ++w) acc += red[(size_t)(a * kLnBwdWarps + w) * D + c];
    part[(size_t)blockIdx.x * 3 * D + j] = acc;
  }
}

// Wide rows (d = 512 * WPR): WPR warps share a row as in ln_fwd_split_kernel;
// x, dy and the residual gradient of the row slice are requested up front,
// the two row sums cross warps through shared memory, and each lane keeps the
// dgain / dbias / output-column-sum accumulators of its fixed 16 columns in
// registers; row groups are reduced through shared memory in a fixed order.
template <typename T, int WPR>
__global__ void __launch_bounds__(256, 1)
ln_bwd_split_kernel(const T* __restrict__ dy, const float* __restrict__ x,
                    const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                    const float* __restrict__ gain, const float* dres, float* dx_out,
                    T* __restrict__ dx_T, float* __restrict__ part, int M, int osum) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int NV = 4, D = NV * 128 * WPR, G = 8 / WPR;
  extern __shared__ float lnbs_sm[];          // [G][D] final reduction
  __shared__ float red[2][2][8];              // [row parity][sum][warp]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = warp / WPR, wi = warp % WPR;
  const int c4base = wi * NV * 32;
  const float inv_d = 1.0f / (float)D;
  float4 ag[NV], ab[NV], ao[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) ag[i] = ab[i] = ao[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  int it = 0;
  for (int m = blockIdx.x * G + grp; m < M; m += gridDim.x * G, ++it) {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)m * D) + c4base;
    const T* gr = dy + (size_t)m * D + 4 * c4base;
    const float4* rr = dres ? reinterpret_cast<const float4*>(dres + (size_t)m * D) + c4base : nullptr;
    float4 xv[NV], gv[NV], rv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xv[i] = xr[lane + 32 * i];
      gv[i] = ld4f(gr + 4 * (lane + 32 * i));
      rv[i] = rr ? rr[lane + 32 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float mean = mean_in[m], rstd = rstd_in[m];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float4 gg = reinterpret_cast<const float4*>(gain)[c4base + lane + 32 * i];
#define PH_LNB_ACC(c)                                 \
  {                                                   \
    const float xh = (xv[i].c - mean) * rstd;         \
    const float dxh = gv[i].c * gg.c;                 \
    s1 += dxh;                                        \
    s2 += dxh * xh;                                   \
    ag[i].c += gv[i].c * xh;                          \
    ab[i].c += gv[i].c;                               \
  }
      PH_LNB_ACC(x) PH_LNB_ACC(y) PH_LNB_ACC(z) PH_LNB_ACC(w)
#undef PH_LNB_ACC
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float* r1 = red[it & 1][0];
    float* r2 = red[it & 1][1];
    if (lane == 0) {
      r1[warp] = s1;
      r2[warp] = s2;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) {
      t1 += r1[grp * WPR + w];
      t2 += r2[grp * WPR + w];
    }
    t1 *= inv_d;
    t2 *= inv_d;
    float* out = dx_out + (size_t)m * D;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = c4base + lane + 32 * i;
      const float4 gg = reinterpret_cast<const float4*>(gain)[c4];
      float4 r = rv[i];
      r.x += rstd * (gv[i].x * gg.x - t1 - ((xv[i].x - mean) * rstd) * t2);
      r.y += rstd * (gv[i].y * gg.y - t1 - ((xv[i].y - mean) * rstd) * t2);
      r.z += rstd * (gv[i].z * gg.z - t1 - ((xv[i].z - mean) * rstd) * t2);
      r.w += rstd * (gv[i].w * gg.w - t1 - ((xv[i].w - mean) * rstd) * t2);
      reinterpret_cast<float4*>(out)[c4] = r;
      if (dx_T) store4(dx_T + (size_t)m * D + 4 * c4, r.x, r.y, r.z, r.w);
      ao[i].x += r.x;
      ao[i].y += r.y;
      ao[i].z += r.z;
      ao[i].w += r.w;
    }
  }
  // block partials [dgain | dbias | dsum]: the G row groups summed in order
  const int nsum = osum ? 3 : 2;
  for (int a = 0; a < nsum; ++a) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i)
      reinterpret_cast<float4*>(lnbs_sm + (size_t)grp * D)[c4base + lane + 32 * i] =
          a == 0 ? ag[i] : a == 1 ? ab[i] : ao[i];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
      float acc = 0.f;
#pragma unroll
      for (int g = 0; g < G; ++g) acc += lnbs_sm[(size_t)g * D + j];
      part[(size_t)blockIdx.x * 3 * D + a * D + j] = acc;
    }
  }
}

template <typename T>
void ln_bwd(const T* dy, const float* x, const float* mean, const float* rstd,
            const float* gain, const float* dres, float* dx_out, T* dx_T, float* part,
            float* dgain, float* dbias, int M, int d, cudaStream_t st, float* dsum, bool acc,
            ReduceJobs* defer) {
  const int nsum = dsum ? 3 : 2;
  switch (d) {
#define PH_LNB(NV)                                                                         \
  case NV * 128: {                                                                         \
    static std::atomic<uint64_t> attr{0};                                                  \
    int dev = 0;                                                                           \
    PH_CUDA(cudaGetDevice(&dev));                                                          \
    if (!(attr.load() & (1ull << (dev & 63)))) {                                           \
      PH_CUDA(cudaFuncSetAttribute(ln_bwd_vec_kernel<T, NV>,                               \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                                   kLnBwdVecSmem(NV * 128)));                              \
      attr.fetch_or(1ull << (dev & 63));                                                   \
    }                                                                                      \
    launch_pdl(ln_bwd_vec_kernel<T, NV>, kLnBwdBlocks, kLnBwdWarps * 32, kLnBwdVecSmem(NV * 128), st,  \
        dy, x, mean, rstd, gain, dres, dx_out, dx_T, part, M, dsum ? 1 : 0);               \
    break;                                                                                 \
  }
    PH_LNB(1) PH_LNB(2) PH_LNB(3) PH_LNB(4) PH_LNB(5) PH_LNB(6)
#undef PH_LNB
#define PH_LNBS(WPR)                                                                       \
  case 512 * WPR: {                                                                        \
    constexpr int smem = (8 / WPR) * 512 * WPR * 4;                                        \
    launch_pdl(ln_bwd_split_kernel<T, WPR>, kLnBwdBlocks, 256, smem, st,                           \
        dy, x, mean, rstd, gain, dres, dx_out, dx_T, part, M, dsum ? 1 : 0);               \
    break;                                                                                 \
  }
    PH_LNBS(2) PH_LNBS(4) PH_LNBS(8)
#undef PH_LNBS
    default: {
      // as many warps (<= 8) as [warps][nsum][d] fp32 partials fit in shared memory
      const int warps = (int)std::max<size_t>(
          1, std::min<size_t>(kLnBwdWarps, (size_t)(224 * 1024) / ((size_t)nsum * d * sizeof(float))));
      const size_t smem = (size_t)warps * nsum * d * sizeof(float);
      if (smem > 224 * 1024) throw Error(PHOTON_ERR_CONFIG, "layer_norm backward: d_model too large");
      if (smem > 48 * 1024)
        PH_CUDA(cudaFuncSetAttribute(ln_bwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
      ln_bwd_kernel<T><<<kLnBwdBlocks, warps * 32, smem, st>>>(dy, x, mean, rstd, gain, dres,
                                                               dx_out, dx_T, part, M, d, nsum);
    }
  }
  PH_LAUNCH_CHECK();
  // gain, bias and (optionally) the output's column sums in one launch
  colreduce(part, kLnBwdBlocks, dsum ? 3 * d : 2 * d, 3 * d, dgain, d, dbias, st, acc, 2 * d,
            dsum, defer);
}

// ============================================================================
// Column sums for bias gradients (add_bias backward, tensor.cpp:279-285).
// Pass 1: CTA (column strip, row chunk); each lane owns VEC consecutive columns
// (16-byte loads), the 8 warps of a CTA interleave rows, 4 rows in flight per
// lane; warps are reduced in smem in a fixed order.  Pass 2: fixed-order sum
// over row chunks.  Deterministic; reads the matrix once at HBM speed.
// ============================================================================
// Row chunks are sized so the grid holds about 8 CTAs per SM (at least 64 rows
// per chunk); the partial count depends only on (M, N, strip width).
static int colsum_chunks(int M, int N, int strip) {
  const int strips = (N + strip - 1) / strip;
  const int want = std::max(1, (kNumSMs * 8 + strips - 1) / strips);
  return std::max(1, std::min(want, (M + 63) / 64));
}
// Very wide rows (the vocabulary-wide head bias, N = V): one persistent CTA per
// SM streams whole rows (contiguous 100 KB at V = 50,368) into a shared-memory
// fp32 accumulator [N]; thread t owns the 8-column chunks t, t + 1024, ... so the
// accumulation needs no atomics.  Row chunk per CTA is contiguous; partials are
// reduced in CTA order (deterministic).  The strip kernel below reads 512-byte
// pieces of rows 100 KB apart and reached ~4.2 TB/s on this shape.
constexpr int kColsumWideThreads = 1024;
static bool colsum_wide_ok(int N, size_t elem) {
  return elem == 2 && N >= 8192 && (N % 8) == 0 && (size_t)N * 4 <= 220 * 1024;
}
size_t colsum_part_floats(int M, int N) {  // upper bound over element types (bf16 strips are widest)
  size_t n = (size_t)colsum_chunks(M, N, 256) * N;
  if (colsum_wide_ok(N, 2)) n = std::max(n, (size_t)kNumSMs * N);
  if (N % 8 == 0 && N / 8 <= 1024) n = std::max(n, (size_t)kNumSMs * 2 * N);  // colsum_rows
  return n;
}

__global__ void __launch_bounds__(kColsumWideThreads, 1)
    colsum_wide_kernel(const bf16* __restrict__ x, int M, int N, float* __restrict__ part) {
  extern __shared__ float4 acc4[];  // [N / 4]
  const int nvec = N / 8;
  for (int i = threadIdx.x; i < N / 4; i += blockDim.x) acc4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(M, r0 + per);
  // eight rows per pass (eight 16-byte loads in flight per thread before the
  // first add): acc += ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), fixed order
  for (int r = r0; r < r1; r += 8) {
    const uint4* a = reinterpret_cast<const uint4*>(x + (size_t)r * N);
    for (int c = threadIdx.x; c < nvec; c += blockDim.x) {
      uint4 u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        u[k] = r + k < r1 ? a[(size_t)k * nvec + c] : make_uint4(0u, 0u, 0u, 0u);
      float f[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float lo8[8], hi8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t w = (&u[k].x)[j];
          lo8[k] = __uint_as_float(w << 16);
          hi8[k] = __uint_as_float(w & 0xffff0000u);
        }
        f[2 * j] = ((lo8[0] + lo8[1]) + (lo8[2] + lo8[3])) + ((lo8[4] + lo8[5]) + (lo8[6] + lo8[7]));
        f[2 * j + 1] =
            ((hi8[0] + hi8[1]) + (hi8[2] + hi8[3])) + ((hi8[4] + hi8[5]) + (hi8[6] + hi8[7]));
      }
      float4 lo = acc4[2 * c], hi = acc4[2 * c + 1];
      lo.x += f[0];
      lo.y += f[1];
      lo.z += f[2];
      lo.w += f[3];
      hi.x += f[4];
      hi.y += f[5];
      hi.z += f[6];
      hi.w += f[7];
      acc4[2 * c] = lo;
      acc4[2 * c + 1] = hi;
    }
  }
  __syncthreads();
  float4* out = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * N);
  for (int i = threadIdx.x; i < N / 4; i += blockDim.x) out[i] = acc4[i];
}

template <typename T>
__global__ void __launch_bounds__(256) colsum_part_kernel(const T* __restrict__ x, int M, int N,
                                                          int rows_per_chunk,
                                                          float* __restrict__ part) {
  constexpr int VEC = 16 / sizeof(T);  // columns per lane
  constexpr int STRIP = 32 * VEC;      // columns per CTA
  constexpr int U = 8;                 // rows in flight per lane
  __shared__ float red[8][STRIP];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * STRIP + lane * VEC;
  const int r0 = blockIdx.y * rows_per_chunk, r1 = min(M, r0 + rows_per_chunk);
  float acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
  const bool full = c0 + VEC <= N && (N % VEC) == 0;
  for (int r = r0 + warp; r < r1; r += 8 * U) {
    T buf[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rr = r + 8 * u;
      if (rr < r1 && full) {
        *reinterpret_cast<uint4*>(buf[u]) = *reinterpret_cast<const uint4*>(x + (size_t)rr * N + c0);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          buf[u][e] = (rr < r1 && c0 + e < N) ? x[(size_t)rr * N + c0 + e] : from_f<T>(0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] += to_f<T>(buf[u][e]);
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) red[warp][lane * VEC + e] = acc[e];
  __syncthreads();
  for (int j = threadIdx.x; j < STRIP; j += blockDim.x) {
    const int c = blockIdx.x * STRIP + j;
    if (c >= N) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][j];
    part[(size_t)blockIdx.y * N + c] = s;
  }
}

// Moderate rows (N / 8 <= 1024 bf16 columns-of-8: the b1 / q / k / v biases):
// thread = (row slot, 8-column chunk); a CTA reads `slots` whole rows per step
// (contiguous), four steps in flight, sums in registers; slots reduced in a
// fixed order through shared memory at the end.  Row ranges are contiguous per
// CTA, partials reduced in CTA order.
constexpr int kColsumRowsCtas = kNumSMs * 2;
static int colsum_rows_slots(int N) { return std::max(1, 1024 / (N / 8)); }
static bool colsum_rows_ok(int N, size_t elem) {
  return elem == 2 && (N % 8) == 0 && N / 8 <= 1024 && N >= 256;
}

__global__ void __launch_bounds__(1024, 2)
    colsum_rows_kernel(const bf16* __restrict__ x, int M, int N, int slots, float* __restrict__ part) {
  extern __shared__ float red[];  // [slots][N]
  const int nch = N / 8;
  const int slot = threadIdx.x / nch, ch = threadIdx.x % nch;
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(M, r0 + per);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (slot < slots) {
    constexpr int U = 4;
    for (int r = r0 + slot; r < r1; r += U * slots) {
      uint4 u[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int rr = r + k * slots;
        u[k] = rr < r1 ? reinterpret_cast<const uint4*>(x + (size_t)rr * N)[ch] : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[2 * e] += __uint_as_float(w[e] << 16);
          acc[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[(size_t)slot * N + ch * 8 + e] = acc[e];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    float t = 0.f;
    for (int s2 = 0; s2 < slots; ++s2) t += red[(size_t)s2 * N + j];
    part[(size_t)blockIdx.x * N + j] = t;
  }
}

template <typename T>
void colsum(const T* x, int M, int N, float* part, float* out, cudaStream_t st, bool acc) {
  if constexpr (sizeof(T) == 2) {
    if (colsum_wide_ok(N, sizeof(T)) && M >= 4 * kNumSMs &&
        (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      const int smem = N * 4;
      static std::atomic<uint64_t> attr{0};  // per device
      int dev = 0;
      PH_CUDA(cudaGetDevice(&dev));
      if (!(attr.load() & (1ull << (dev & 63)))) {
        PH_CUDA(cudaFuncSetAttribute(colsum_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     220 * 1024));
        attr.fetch_or(1ull << (dev & 63));
      }
      colsum_wide_kernel<<<kNumSMs, kColsumWideThreads, smem, st>>>(
          reinterpret_cast<const bf16*>(x), M, N, part);
      PH_LAUNCH_CHECK();
      colreduce(part, kNumSMs, N, N, out, N, nullptr, st, acc);
      return;
    }
    if (colsum_rows_ok(N, sizeof(T)) && M >= 4 * kColsumRowsCtas &&
        (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      const int slots = colsum_rows_slots(N);
      const int smem = slots * N * 4;
      if (smem > 48 * 1024) {
        static std::atomic<uint64_t> attr{0};
        int dev = 0;
        PH_CUDA(cudaGetDevice(&dev));
        if (!(attr.load() & (1ull << (dev & 63)))) {
          PH_CUDA(cudaFuncSetAttribute(colsum_rows_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
          attr.fetch_or(1ull << (dev & 63));
        }
      }
      colsum_rows_kernel<<<kColsumRowsCtas, 1024, smem, st>>>(reinterpret_cast<const bf16*>(x), M, N,
                                                              slots, part);
      PH_LAUNCH_CHECK();
      colreduce(part, kColsumRowsCtas, N, N, out, N, nullptr, st, acc);
      return;
    }
  }
  constexpr int STRIP = 32 * (16 / sizeof(T));
  const int chunks = colsum_chunks(M, N, STRIP);
  const int rows = (M + chunks - 1) / chunks;
  const int used = (M + rows - 1) / rows;
  colsum_part_kernel<T><<<dim3(cdiv(N, STRIP), used), 256, 0, st>>>(x, M, N, rows, part);
  PH_LAUNCH_CHECK();
  colreduce(part, used, N, N, out, N, nullptr, st, acc);
}

// ============================================================================
// Softmax cross-entropy, fused forward + backward, one CTA per row.
// loss_row = log(sum exp(l - max)) + max - l[t]      (tensor.cpp:569-582)
// dl = (softmax - onehot(t)) / count                   (tensor.cpp:590-600)
// ============================================================================
template <typename T>
__global__ void __launch_bounds__(512) ce_kernel(T* __restrict__ logits,
                                                 const int32_t* __restrict__ targets, int V,
                                                 float inv_v, double* __restrict__ rowloss,
                                                 int write_grad, const float* inv_dev) {
  const float inv_count = inv_dev ? *inv_dev : inv_v;
  __shared__ float red_m[16], red_s[16];
  const int row = blockIdx.x;
  T* l = logits + (size_t)row * V;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  float m = -INFINITY, s = 0.f;
  int bad = 0;  // NaN / +inf logit: the reference's loss is NaN (tensor.cpp:569-582)
  for (int j = tid; j < V; j += blockDim.x) {
    const float v = to_f<T>(l[j]);
    bad |= !(v < INFINITY);
    if (v > m) {
      s = s * __expf(m - v) + 1.f;
      m = v;
    } else {
      s += __expf(v - m);
    }
  }
  // warp combine (max, sum)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  if (lane == 0) {
    red_m[warp] = m;
    red_s[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < nw ? red_m[lane] : -INFINITY;
    s = lane < nw ? red_s[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      red_m[0] = m;
      red_s[0] = s;
    }
  }
  bad = __syncthreads_or(bad);
  m = red_m[0];
  s = red_s[0];
  const int t = targets[row];
  if (tid == 0) {
    rowloss[row] = t < 0 ? 0.0
                   : bad ? (double)NAN
                         : (double)logf(s) + (double)m - (double)to_f<T>(l[t]);
  }
  if (!write_grad) return;
  __syncthreads();  // everyone has read l[t] before it is overwritten
  const float inv_s = 1.f / s;
  const float g = t >= 0 ? inv_count : 0.f;
  for (int j = tid; j < V; j += blockDim.x) {
    const float p = __expf(to_f<T>(l[j]) - m) * inv_s;
    l[j] = from_f<T>(g * (p - (j == t ? 1.f : 0.f)));
  }
}

// bf16 rows up to kCeRegChunks*8*256 wide stay in registers: one HBM read and
// one write per logit.
constexpr int kCeThreads = 256, kCeRegChunks = 26;  // V <= 53248
__global__ void __launch_bounds__(kCeThreads) ce_reg_kernel(bf16* __restrict__ logits,
                                                            const int32_t* __restrict__ targets,
                                                            int V, float inv_v,
                                                            double* __restrict__ rowloss,
                                                            int write_grad, const float* inv_dev) {
  const float inv_count = inv_dev ? *inv_dev : inv_v;
  __shared__ float red[kCeThreads / 32];
  __shared__ float bcast;
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  bf16* l = logits + (size_t)row * V;
  const int nvec = V / 8;  // V % 8 == 0 (checked by the launcher)
  uint4 x[kCeRegChunks];
  float m = -INFINITY;
  int bad = 0;
#pragma unroll
  for (int c = 0; c < kCeRegChunks; ++c) {
    const int i = tid + c * kCeThreads;
    if (i < nvec) {
      x[c] = reinterpret_cast<const uint4*>(l)[i];
      const uint32_t w[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float a = __uint_as_float(w[e] << 16), b = __uint_as_float(w[e] & 0xffff0000u);
        bad |= !(a < INFINITY) | !(b < INFINITY);
        m = fmaxf(m, fmaxf(a, b));
      }
    }
  }
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (tid < 32) {
    float t = tid < kCeThreads / 32 ? red[tid] : -INFINITY;
    t = warp_max(t);
    if (tid == 0) bcast = t;
  }
  __syncthreads();
  m = bcast;
  const float ml2 = m * 1.4426950408889634f;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kCeRegChunks; ++c) {
    const int i = tid + c * kCeThreads;
    if (i < nvec) {
      const uint32_t w[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s += exp2f(fmaf(__uint_as_float(w[e] << 16), 1.4426950408889634f, -ml2));
        s += exp2f(fmaf(__uint_as_float(w[e] & 0xffff0000u), 1.4426950408889634f, -ml2));
      }
    }
  }
  s = warp_sum(s);
  __syncthreads();
  if (lane == 0) red[warp] = s;
  bad = __syncthreads_or(bad);
  if (tid < 32) {
    float t = tid < kCeThreads / 32 ? red[tid] : 0.f;
    t = warp_sum(t);
    if (tid == 0) bcast = t;
  }
  __syncthreads();
  s = bcast;
  const int t = targets[row];
  if (tid == 0)
    rowloss[row] = t < 0 ? 0.0
                   : bad ? (double)NAN
                         : (double)logf(s) + (double)m - (double)__bfloat162float(l[t]);
  if (!write_grad) return;
  __syncthreads();  // l[t] read before it is overwritten
  const float g = t >= 0 ? inv_count : 0.f;
  const float gs = g / s;
#pragma unroll
  for (int c = 0; c < kCeRegChunks; ++c) {
    const int i = tid + c * kCeThreads;
    if (i < nvec) {
      const uint32_t w[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = i * 8 + 2 * e;
        float a = gs * exp2f(fmaf(__uint_as_float(w[e] << 16), 1.4426950408889634f, -ml2));
        float b = gs * exp2f(fmaf(__uint_as_float(w[e] & 0xffff0000u), 1.4426950408889634f, -ml2));
        if (j == t) a -= g;
        if (j + 1 == t) b -= g;
        const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
        o[e] = *reinterpret_cast<const uint32_t*>(&p);
      }
      reinterpret_cast<uint4*>(l)[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// Persistent, smem-pipelined variant (one CTA per SM).  Rows r = blockIdx.x +
// i*gridDim.x alternate between two shared-memory row buffers.  A producer warp
// bulk-copies row i+2 into a buffer once the gradient of row i has been
// bulk-stored out of it, so HBM reads and writes overlap the exp work of the
// 16 compute warps.  One online (max, sum) pass plus one gradient pass, both
// over shared memory; every (max, sum) combine runs in a fixed order.
constexpr int kCePipeWarps = 16, kCePipeThreads = kCePipeWarps * 32;
constexpr int kCePipeMaxSmem = 232448 - 2048;  // opt-in limit minus the static reduction arrays
__host__ __device__ inline uint32_t ce_pipe_buf_stride(int V) { return ((uint32_t)V * 2 + 127) & ~127u; }
static size_t ce_pipe_smem(int V) { return 2 * (size_t)ce_pipe_buf_stride(V) + 64; }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&p);
}
__device__ __forceinline__ void ce_unpack8(const uint4 x, float* v) {
  const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[2 * e] = __uint_as_float(w[e] << 16);
    v[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
  }
}
__device__ __forceinline__ float ex2_approx(float x) {  // one MUFU.EX2, no range fix-up
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (m, s) ⊕ (m2, s2) with s measured relative to m
__device__ __forceinline__ void ce_combine(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  if (mm == -INFINITY) return;
  s = s * ex2_approx((m - mm) * 1.4426950408889634f) + s2 * ex2_approx((m2 - mm) * 1.4426950408889634f);
  m = mm;
}

// bias_part != nullptr (backward): the head-bias gradient -- the column sums of
// dlogits (add_bias backward, tensor.cpp:279-285) -- accumulates in TENSOR
// memory, the one on-chip store this kernel leaves free (shared memory holds
// the two row buffers): thread t owns the 8-column chunks t + 512 j of every
// row, kept in its own TMEM lane (lane quarter w % 4 of warp w, columns
// 128 (w / 4) + 8 j), so the sums need no atomics and no second pass over the
// 6.6 GB of bf16 dlogits.  Summed in fp32 before the bf16 rounding, rows in a
// fixed order per CTA; bias_part[blockIdx.x][V] is reduced in CTA order.
constexpr int kCeBiasMaxChunks = 16;  // per thread: V <= 512 * 16 * 8
__global__ void __launch_bounds__(kCePipeThreads + 32, 1)
    ce_pipe_kernel(bf16* __restrict__ logits, const int32_t* __restrict__ targets, int M, int V,
                   float inv_v, double* __restrict__ rowloss, int write_grad,
                   float* __restrict__ bias_part, const float* inv_dev) {
  pdl_launch_dependents();
  pdl_wait();
  const float inv_count = inv_dev ? *inv_dev : inv_v;
  using namespace sm100;
  extern __shared__ __align__(128) uint8_t ce_sm[];
  __shared__ float red_m[kCePipeWarps], red_s[kCePipeWarps];
  __shared__ uint32_t tmem_slot;
  const uint32_t row_bytes = (uint32_t)V * 2, stride = ce_pipe_buf_stride(V);
  uint64_t* full = reinterpret_cast<uint64_t*>(ce_sm + 2 * stride);
  uint64_t* done = full + 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&done[0], kCePipeWarps);
    mbar_init(&done[1], kCePipeWarps);
    mbar_init_fence();
  }
  const bool bias = bias_part != nullptr;
  if (bias && warp == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int nvec = V / 8;
  // this thread's TMEM accumulator columns (chunk j at tacc + 8 j); the chunk
  // loops are warp-uniform because tcgen05.ld / st are .sync.aligned
  const uint32_t tacc = bias ? tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2) : 0;
  const int warp_chunks = (nvec - warp * 32 + kCePipeThreads - 1) / kCePipeThreads;  // j range
  if (bias && warp < kCePipeWarps) {
    const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < warp_chunks; ++j) tmem_st8(tacc + 8 * j, z);
    tmem_wait_st();
  }

  if (warp == kCePipeWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      for (int k = 0; k < 2; ++k) {
        const int r = blockIdx.x + k * G;
        if (r < M) {
          mbar_expect_tx(&full[k], row_bytes);
          bulk_load(ce_sm + k * stride, logits + (size_t)r * V, row_bytes, &full[k]);
        }
      }
      for (int i = 0;; ++i) {
        const int r = blockIdx.x + i * G;
        if (r >= M) break;
        const int b = i & 1;
        mbar_wait(&done[b], (i >> 1) & 1);
        if (write_grad) {
          bulk_store(logits + (size_t)r * V, ce_sm + b * stride, row_bytes);
          bulk_commit();
        }
        const int r2 = r + 2 * G;
        if (r2 < M) {
          if (write_grad) bulk_wait_read<0>();  // buffer read out before it is refilled
          mbar_expect_tx(&full[b], row_bytes);
          bulk_load(ce_sm + b * stride, logits + (size_t)r2 * V, row_bytes, &full[b]);
        }
      }
      bulk_wait_all();
    }
    if (!bias) return;
    __syncwarp();
  } else {
  // ---------------- compute warps ----------------
  constexpr float kL2e = 1.4426950408889634f;
  for (int i = 0;; ++i) {
    const int r = blockIdx.x + i * G;
    if (r >= M) break;
    const int b = i & 1;
    uint8_t* buf = ce_sm + b * stride;
    const uint32_t base = su32(buf);
    mbar_wait(&full[b], (i >> 1) & 1);
    // Three passes over the row in shared memory with ONE exponential per logit
    // (MUFU was the limit with two): (1) row max; (2) e = exp(l - m), row sum,
    // e written back in place as bf16 when the gradient is wanted (l[t] is read
    // first); (3) dl = e * g / s - g * onehot(t), the target column recomputed
    // from l[t] in fp32 (p - 1 cancels; the bf16 copy of e would not do).  A NaN
    // logit makes s NaN and a +inf logit m = +inf and s NaN, so the reference's
    // NaN loss (tensor.cpp:569-582) is detected from (m, s).
    // (1) on the packed bf16 pairs (HMNMX2: the max of bf16 values is one of
    // them, so the same m as in fp32; like fmaxf it passes over NaNs)
    __nv_bfloat162 m2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    for (int c = tid; c < nvec; c += kCePipeThreads) {
      const uint4 x = lds128(base + c * 16);
      const __nv_bfloat162 a = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&x.x),
                                       *reinterpret_cast<const __nv_bfloat162*>(&x.y));
      const __nv_bfloat162 b = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&x.z),
                                       *reinterpret_cast<const __nv_bfloat162*>(&x.w));
      m2 = __hmax2(m2, __hmax2(a, b));
    }
    float m = fmaxf(__low2float(m2), __high2float(m2));
    m = warp_max(m);
    if (lane == 0) red_m[warp] = m;
    named_bar_sync(1, kCePipeThreads);
    m = red_m[0];
#pragma unroll
    for (int w = 1; w < kCePipeWarps; ++w) m = fmaxf(m, red_m[w]);
    const int t = targets[r];
    const float lt = t >= 0 ? __bfloat162float(reinterpret_cast<const bf16*>(buf)[t]) : 0.f;
    named_bar_sync(1, kCePipeThreads);  // red_* and l[t] read before reuse / overwrite
    const float ml2 = m * kL2e;
    float s = 0.f;
    for (int c = tid; c < nvec; c += kCePipeThreads) {
      float v[8];
      ce_unpack8(lds128(base + c * 16), v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] = ex2_approx(fmaf(v[e], kL2e, -ml2));
        s += v[e];
      }
      if (write_grad) {
        uint4 o;
        o.x = pack_bf16x2(v[0], v[1]);
        o.y = pack_bf16x2(v[2], v[3]);
        o.z = pack_bf16x2(v[4], v[5]);
        o.w = pack_bf16x2(v[6], v[7]);
        sts128(base + c * 16, o);
      }
    }
    s = warp_sum(s);
    if (lane == 0) red_s[warp] = s;
    named_bar_sync(1, kCePipeThreads);
    s = red_s[0];
#pragma unroll
    for (int w = 1; w < kCePipeWarps; ++w) s += red_s[w];
    const bool bad = !(s == s) || m == INFINITY;
    if (tid == 0)
      rowloss[r] = t < 0 ? 0.0 : bad ? (double)NAN : (double)logf(s) + (double)m - (double)lt;
    if (write_grad) {
      const float g = t >= 0 ? inv_count : 0.f;
      const float gs = g / s;
      for (int j = 0; j < warp_chunks; ++j) {
        const int c = tid + j * kCePipeThreads;
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (c < nvec) {
          ce_unpack8(lds128(base + c * 16), v);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] *= gs;
          const int te = t - c * 8;  // target column within this chunk (if any)
          if ((unsigned)te < 8u) {
            const float pt = gs * ex2_approx(fmaf(lt, kL2e, -ml2)) - g;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e == te) v[e] = pt;
          }
          uint4 o;
          o.x = pack_bf16x2(v[0], v[1]);
          o.y = pack_bf16x2(v[2], v[3]);
          o.z = pack_bf16x2(v[4], v[5]);
          o.w = pack_bf16x2(v[6], v[7]);
          sts128(base + c * 16, o);
        }
        if (bias) {  // column sums in fp32, before the bf16 rounding
          float a[8];
          tmem_ld8_wait(tacc + 8 * j, a);
#pragma unroll
          for (int e = 0; e < 8; ++e) a[e] += v[e];
          tmem_st8(tacc + 8 * j, a);
        }
      }
      if (bias) tmem_wait_st();  // this row's sums land before the next row reads them
      fence_async_smem();
    }
    named_bar_sync(1, kCePipeThreads);  // red_s read by every thread before the next row
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[b]);
  }
  if (bias) {  // this CTA's column partial
    for (int j = 0; j < warp_chunks; ++j) {
      const int c = tid + j * kCePipeThreads;
      float a[8];
      tmem_ld8_wait(tacc + 8 * j, a);
      if (c < nvec) {
        float4* o = reinterpret_cast<float4*>(bias_part + (size_t)blockIdx.x * V + (size_t)c * 8);
        o[0] = make_float4(a[0], a[1], a[2], a[3]);
        o[1] = make_float4(a[4], a[5], a[6], a[7]);
      }
    }
  }
  }  // compute warps
  if (bias) {
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc(tmem_slot, 512);
    }
  }
}

size_t ce_bias_part_floats(int V) { return (size_t)kNumSMs * V; }

template <typename T>
bool ce_fwd_bwd(T* logits, const int32_t* targets, int M, int V, float inv_count, double* rowloss,
                bool write_grad, cudaStream_t st, float* dbias, float* part, bool acc,
                const float* inv_dev, ReduceJobs* defer) {
  if constexpr (sizeof(T) == 2) {
    const bool aligned = (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
    if (V % 8 == 0 && ce_pipe_smem(V) <= (size_t)kCePipeMaxSmem && M > 0 && aligned) {
      static std::atomic<uint64_t> attr{0};  // per device
      int dev = 0;
      PH_CUDA(cudaGetDevice(&dev));
      if (!(attr.load() & (1ull << (dev & 63)))) {
        PH_CUDA(cudaFuncSetAttribute(ce_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kCePipeMaxSmem));
        attr.fetch_or(1ull << (dev & 63));
      }
      const bool fuse = write_grad && dbias && part && V / 8 <= kCePipeThreads * kCeBiasMaxChunks;
      const int grid = std::min(M, kNumSMs);
      launch_pdl(ce_pipe_kernel, grid, kCePipeThreads + 32, ce_pipe_smem(V), st, 
          logits, targets, M, V, inv_count, rowloss, write_grad ? 1 : 0, fuse ? part : nullptr,
          inv_dev);
      PH_LAUNCH_CHECK();
      if (fuse) colreduce(part, grid, V, V, dbias, V, nullptr, st, acc, -1, nullptr, defer);
      return fuse;
    }
    if (V % 8 == 0 && V <= kCeRegChunks * 8 * kCeThreads && aligned) {
      ce_reg_kernel<<<M, kCeThreads, 0, st>>>(logits, targets, V, inv_count, rowloss,
                                              write_grad ? 1 : 0, inv_dev);
      PH_LAUNCH_CHECK();
      return false;
    }
  }
  ce_kernel<T><<<M, 512, 0, st>>>(logits, targets, V, inv_count, rowloss, write_grad ? 1 : 0,
                                  inv_dev);
  PH_LAUNCH_CHECK();
  return false;
}

__global__ void sum_scaled_kernel(const double* __restrict__ x, int n, double scale_v,
                                  double* __restrict__ out, int acc_out, const float* scale_dev) {
  pdl_launch_dependents();
  pdl_wait();
  const double scale = scale_dev ? (double)*scale_dev : scale_v;
  __shared__ double sm[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    acc = warp_sum(acc);
    if (threadIdx.x == 0) *out = acc_out ? *out + acc * scale : acc * scale;
  }
}

void sum_scaled(const double* x, int n, double scale, double* out, cudaStream_t st, bool acc,
                const float* scale_dev) {
  launch_pdl(sum_scaled_kernel, 1, 1024, 0, st, x, n, scale, out, acc ? 1 : 0, scale_dev);
  PH_LAUNCH_CHECK();
}

// ============================================================================
// SIMT causal attention (parity path, any head dim).  One warp per query row
// (forward, dQ) or key row (dK, dV); lanes split the head dim.  Matches the
// reference's masking j <= i and scale-before-max (tensor.cpp:455-483).
// ============================================================================
constexpr int kMaxDhPerLane = 8;  // head dim <= 256

template <typename T>
__global__ void attn_fwd_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                     const T* __restrict__ v, T* __restrict__ o,
                                     float* __restrict__ lse, int B, int S, int H, int d) {
  const int dh = d / H, lane = threadIdx.x & 31;
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;  // (b, h, i) flattened as ((b*H+h)*S+i)
  if (row >= B * H * S) return;
  const int i = row % S, bh = row / S, h = bh % H, b = bh / H;
  const float scale = rsqrtf((float)dh);
  float qr[kMaxDhPerLane], acc[kMaxDhPerLane];
  const size_t qoff = ((size_t)(b * S + i)) * d + h * dh;
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    qr[c] = col < dh ? to_f<T>(q[qoff + col]) : 0.f;
    acc[c] = 0.f;
  }
  float mrun = -INFINITY, lrun = 0.f;
  for (int j = 0; j <= i; ++j) {
    const size_t koff = ((size_t)(b * S + j)) * d + h * dh;
    float part = 0.f;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) part += qr[c] * to_f<T>(k[koff + col]);
    }
    const float sc = warp_sum(part) * scale;
    const float mnew = fmaxf(mrun, sc);
    const float corr = __expf(mrun - mnew);
    const float p = __expf(sc - mnew);
    lrun = lrun * corr + p;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) acc[c] = acc[c] * corr + p * to_f<T>(v[koff + col]);
    }
    mrun = mnew;
  }
  const float inv = 1.f / lrun;
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    if (col < dh) o[qoff + col] = from_f<T>(acc[c] * inv);
  }
  if (lane == 0) lse[row] = mrun + logf(lrun);
}

// D[row] = dO_i . O_i
template <typename T>
__global__ void attn_bwd_dot_kernel(const T* __restrict__ o, const T* __restrict__ dO,
                                    float* __restrict__ Dvec, int B, int S, int H, int d) {
  const int dh = d / H, lane = threadIdx.x & 31, warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  if (row >= B * H * S) return;
  const int i = row % S, bh = row / S, h = bh % H, b = bh / H;
  const size_t off = ((size_t)(b * S + i)) * d + h * dh;
  float acc = 0.f;
  for (int c = lane; c < dh; c += 32) acc += to_f<T>(o[off + c]) * to_f<T>(dO[off + c]);
  acc = warp_sum(acc);
  if (lane == 0) Dvec[row] = acc;
}

template <typename T>
__global__ void attn_bwd_dq_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                   const T* __restrict__ v, const T* __restrict__ dO,
                                   const float* __restrict__ lse, const float* __restrict__ Dvec,
                                   T* __restrict__ dq, int B, int S, int H, int d) {
  const int dh = d / H, lane = threadIdx.x & 31, warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  if (row >= B * H * S) return;
  const int i = row % S, bh = row / S, h = bh % H, b = bh / H;
  const float scale = rsqrtf((float)dh);
  const size_t qoff = ((size_t)(b * S + i)) * d + h * dh;
  float qr[kMaxDhPerLane], dor[kMaxDhPerLane], acc[kMaxDhPerLane];
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    qr[c] = col < dh ? to_f<T>(q[qoff + col]) : 0.f;
    dor[c] = col < dh ? to_f<T>(dO[qoff + col]) : 0.f;
    acc[c] = 0.f;
  }
  const float L = lse[row], D = Dvec[row];
  for (int j = 0; j <= i; ++j) {
    const size_t koff = ((size_t)(b * S + j)) * d + h * dh;
    float ps = 0.f, pd = 0.f;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) {
        ps += qr[c] * to_f<T>(k[koff + col]);
        pd += dor[c] * to_f<T>(v[koff + col]);
      }
    }
    const float s = warp_sum(ps) * scale;
    const float dp = warp_sum(pd);
    const float p = __expf(s - L);
    const float ds = p * (dp - D) * scale;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) acc[c] += ds * to_f<T>(k[koff + col]);
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    if (col < dh) dq[qoff + col] = from_f<T>(acc[c]);
  }
}

template <typename T>
__global__ void attn_bwd_dkdv_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                     const T* __restrict__ v, const T* __restrict__ dO,
                                     const float* __restrict__ lse,
                                     const float* __restrict__ Dvec, T* __restrict__ dk,
                                     T* __restrict__ dv, int B, int S, int H, int d) {
  const int dh = d / H, lane = threadIdx.x & 31, warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;  // key row
  if (row >= B * H * S) return;
  const int j = row % S, bh = row / S, h = bh % H, b = bh / H;
  const float scale = rsqrtf((float)dh);
  const size_t koff = ((size_t)(b * S + j)) * d + h * dh;
  float kr[kMaxDhPerLane], vr[kMaxDhPerLane], ak[kMaxDhPerLane], av[kMaxDhPerLane];
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    kr[c] = col < dh ? to_f<T>(k[koff + col]) : 0.f;
    vr[c] = col < dh ? to_f<T>(v[koff + col]) : 0.f;
    ak[c] = 0.f;
    av[c] = 0.f;
  }
  for (int i = j; i < S; ++i) {
    const size_t qoff = ((size_t)(b * S + i)) * d + h * dh;
    const int qrow = bh * S + i;
    float ps = 0.f, pd = 0.f;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) {
        ps += to_f<T>(q[qoff + col]) * kr[c];
        pd += to_f<T>(dO[qoff + col]) * vr[c];
      }
    }
    const float s = warp_sum(ps) * scale;
    const float dp = warp_sum(pd);
    const float p = __expf(s - lse[qrow]);
    const float ds = p * (dp - Dvec[qrow]) * scale;
#pragma unroll
    for (int c = 0; c < kMaxDhPerLane; ++c) {
      const int col = lane + 32 * c;
      if (col < dh) {
        av[c] += p * to_f<T>(dO[qoff + col]);
        ak[c] += ds * to_f<T>(q[qoff + col]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxDhPerLane; ++c) {
    const int col = lane + 32 * c;
    if (col < dh) {
      dk[koff + col] = from_f<T>(ak[c]);
      dv[koff + col] = from_f<T>(av[c]);
    }
  }
}

template <typename T>
void attn_fwd_simt(const T* q, const T* k, const T* v, T* o, float* lse, int B, int S, int H,
                   int d, cudaStream_t st) {
  if (d / H > 32 * kMaxDhPerLane) throw Error(PHOTON_ERR_CONFIG, "attention: head dim > 256");
  const int rows = B * H * S;
  attn_fwd_simt_kernel<T><<<cdiv(rows, 4), 128, 0, st>>>(q, k, v, o, lse, B, S, H, d);
  PH_LAUNCH_CHECK();
}

template <typename T>
void attn_bwd_simt(const T* q, const T* k, const T* v, const T* o, const T* dO, const float* lse,
                   float* Dvec, T* dq, T* dk, T* dv, int B, int S, int H, int d, cudaStream_t st) {
  const int rows = B * H * S;
  attn_bwd_dot_kernel<T><<<cdiv(rows, 4), 128, 0, st>>>(o, dO, Dvec, B, S, H, d);
  PH_LAUNCH_CHECK();
  attn_bwd_dq_kernel<T><<<cdiv(rows, 4), 128, 0, st>>>(q, k, v, dO, lse, Dvec, dq, B, S, H, d);
  PH_LAUNCH_CHECK();
  attn_bwd_dkdv_kernel<T><<<cdiv(rows, 4), 128, 0, st>>>(q, k, v, dO, lse, Dvec, dk, dv, B, S, H,
                                                         d);
  PH_LAUNCH_CHECK();
}

// ============================================================================
// casts
// ============================================================================
__global__ void f64_to_f32_kernel(const double* __restrict__ in, float* __restrict__ out,
                                  uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ in, double* __restrict__ out,
                                  uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}
__global__ void f32_to_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out,
                                   uint64_t n) {
  pdl_launch_dependents();
  pdl_wait();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}
void f64_to_f32(const double* in, float* out, uint64_t n, cudaStream_t st) {
  f64_to_f32_kernel<<<std::min<unsigned>(cdiv(n, 256), kNumSMs * 8), 256, 0, st>>>(in, out, n);
  PH_LAUNCH_CHECK();
}
void f32_to_f64(const float* in, double* out, uint64_t n, cudaStream_t st) {
  f32_to_f64_kernel<<<std::min<unsigned>(cdiv(n, 256), kNumSMs * 8), 256, 0, st>>>(in, out, n);
  PH_LAUNCH_CHECK();
}
void f32_to_bf16(const float* in, bf16* out, uint64_t n, cudaStream_t st) {
  launch_pdl(f32_to_bf16_kernel, std::min<unsigned>(cdiv(n, 256), kNumSMs * 8), 256, 0, st, in, out, n);
  PH_LAUNCH_CHECK();
}

// out[c][r] = in[r][c] for a [rows][cols] bf16 matrix: 64 x 64 tiles through
// shared memory, 16-byte loads of 8 columns and 16-byte stores of 8 rows (a
// warp writes four output rows' 128-byte segments).  Gives the head weight
// gradient a K-major A operand (tokens contiguous): 4.3 -> 3.6 ms for the
// 768 x 50,368 x 65,536 contraction, against ~35 us for this pass.
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const bf16* __restrict__ in, int rows,
                                                             int cols, bf16* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ uint16_t tile[64][66];
  const int tcols = (cols + 63) / 64;
  const int r0 = (blockIdx.x / tcols) * 64, c0 = (blockIdx.x % tcols) * 64;
  const uint16_t* src = reinterpret_cast<const uint16_t*>(in);
  uint16_t* dst = reinterpret_cast<uint16_t*>(out);
  const bool full = r0 + 64 <= rows && c0 + 64 <= cols && (cols & 7) == 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // 512 vectors of 8 columns
    const int v = threadIdx.x + 256 * i, r = v >> 3, c = (v & 7) * 8;
    if (full) {
      const uint4 x = *reinterpret_cast<const uint4*>(src + (int64_t)(r0 + r) * cols + c0 + c);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        tile[r][c + 2 * j] = (uint16_t)(w[j] & 0xffffu);
        tile[r][c + 2 * j + 1] = (uint16_t)(w[j] >> 16);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        tile[r][c + j] = (r0 + r < rows && c0 + c + j < cols) ? src[(int64_t)(r0 + r) * cols + c0 + c + j] : 0;
    }
  }
  __syncthreads();
  const bool full_out = full && (rows & 7) == 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // output row c0 + c, rows r0 + g * 8 .. + 7
    const int v = threadIdx.x + 256 * i, c = v >> 3, g = (v & 7) * 8;
    if (full_out) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = (uint32_t)tile[g + 2 * j][c] | ((uint32_t)tile[g + 2 * j + 1][c] << 16);
      *reinterpret_cast<uint4*>(dst + (int64_t)(c0 + c) * rows + r0 + g) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + c < cols && r0 + g + j < rows) dst[(int64_t)(c0 + c) * rows + r0 + g + j] = tile[g + j][c];
    }
  }
}
void transpose_bf16(const bf16* in, int rows, int cols, bf16* out, cudaStream_t st) {
  const unsigned blocks = (unsigned)(((rows + 63) / 64) * ((cols + 63) / 64));
  launch_pdl(transpose_bf16_kernel, blocks, 256, 0, st, in, rows, cols, out);
  PH_LAUNCH_CHECK();
}

// ---- instantiations ----------------------------------------------------------
#define INST(T)                                                                                 \
  template void ln_fwd<T>(const float*, const float*, const float*, T*, float*, float*, int, int, \
                          cudaStream_t);                                                        \
  template void ln_bwd<T>(const T*, const float*, const float*, const float*, const float*,       \
                          const float*, float*, T*, float*, float*, float*, int, int,            \
                          cudaStream_t, float*, bool, ReduceJobs*);                             \
  template void colsum<T>(const T*, int, int, float*, float*, cudaStream_t, bool);              \
  template bool ce_fwd_bwd<T>(T*, const int32_t*, int, int, float, double*, bool, cudaStream_t, \
                               float*, float*, bool, const float*, ReduceJobs*);              \
  template void attn_fwd_simt<T>(const T*, const T*, const T*, T*, float*, int, int, int, int,    \
                                 cudaStream_t);                                                 \
  template void attn_bwd_simt<T>(const T*, const T*, const T*, const T*, const T*, const float*,  \
                                 float*, T*, T*, T*, int, int, int, int, cudaStream_t);
INST(float)
INST(bf16)
#undef INST

}  // namespace k
}  // namespace photon
