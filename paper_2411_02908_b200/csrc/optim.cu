// optim.cu -- global-norm clip, AdamW / SGD, and the fused anchored-mean ->
// pseudo-gradient -> outer-optimizer aggregation kernel.
//
// Compiled with -fmad=false: every multiply and add rounds separately, as in
// the reference's FMA-free x86-64 build, so the f64 instantiations reproduce
// ParamVector::mean / sub / server_step / adamw_step / sgd_step bit for bit.
// Citations: /root/reference/proj/core/src/{param_vector,optim}.cpp.
#include <cstdlib>
#include "kernels.cuh"

namespace photon {
namespace k {

constexpr int kRedBlocks = kNumSMs * 4;
int sumsq_nparts() { return kRedBlocks; }

template <typename T>
__device__ __forceinline__ double block_sum(double v, T* /*tag*/) {
  __shared__ double sm[32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// ---- global norm (param_vector.cpp:105-110), fast path: fixed-shape tree ------
__global__ void sumsq_kernel(const float* __restrict__ g, uint64_t n, double* __restrict__ part) {
  pdl_launch_dependents();
  pdl_wait();
  double acc = 0.0;
  const uint64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float4 x = g4[i];
    acc += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
  }
  for (uint64_t i = n4 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += (double)g[i] * g[i];
  const double s = block_sum(acc, (float*)nullptr);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void sumsq_parts(const float* g, uint64_t n, double* part, cudaStream_t st) {
  launch_pdl(sumsq_kernel, kRedBlocks, 256, 0, st, g, n, part);
  PH_LAUNCH_CHECK();
}

// optim.cpp:50-57: cf = clip/norm when norm > clip > 0 else 1; non-finite
// norm is recorded (NumericError surfaces at the round boundary).
__global__ void clip_finalize_kernel(const double* __restrict__ part, int nparts, double clip,
                                     double* norm_out, float* cf_out, int* bad_step, int step) {
  pdl_launch_dependents();
  pdl_wait();
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[i];
  const double s = block_sum(acc, (float*)nullptr);
  if (threadIdx.x == 0) {
    const double norm = sqrt(s);
    if (norm_out) *norm_out = norm;
    const bool finite = isfinite(norm);
    if (!finite && bad_step && *bad_step == 0) *bad_step = step + 1;
    // a non-finite norm poisons cf with NaN: the optimizer kernels then leave
    // params and moments untouched, as optim.cpp:52-54 throws before mutating
    *cf_out = !finite ? __int_as_float(0x7fffffff)
                      : (clip > 0.0 && norm > clip) ? (float)(clip / norm) : 1.0f;
  }
}

void clip_finalize(const double* part, double clip, double* norm_out, float* cf_out,
                   int* bad_step, int step, cudaStream_t st) {
  launch_pdl(clip_finalize_kernel, 1, 1024, 0, st, part, kRedBlocks, clip, norm_out, cf_out, bad_step,
                                          step);
  PH_LAUNCH_CHECK();
}

// ---- AdamW (optim.cpp:61-90) over fp32 storage -------------------------------------
// The device engine's optimizer: fp32 arithmetic with the step constants folded
// on the host (1/bc1, 1/bc2), two MUFU-free IEEE operations per element (sqrt,
// division) -- HBM-bound at 30 B/param.  The exact f64 form of the reference
// (bit-exact for the f64 C ABI) is adamw_f64_kernel below.
__device__ __forceinline__ void adamw_elem(float& p, float g, float& m, float& v, float cf,
                                           float lr, float b1, float b2, float ib1, float ib2,
                                           float eps, float wd) {
  const float gj = g * cf;
  const float mm = b1 * m + (1.0f - b1) * gj;
  const float vv = b2 * v + ((1.0f - b2) * gj) * gj;
  p = p - lr * ((mm * ib1) / (sqrtf(vv * ib2) + eps) + wd * p);
  m = mm;
  v = vv;
}

__global__ void __launch_bounds__(256) adamw_f32_kernel(
    float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
    bf16* __restrict__ shadow, uint64_t n, const float* cfp, float lr_v, const double* lr_dev,
    float b1, float b2, float ib1, float ib2, float eps, float wd) {
  pdl_launch_dependents();
  pdl_wait();
  const float cf = *cfp;
  if (cf != cf) return;  // NumericError step: no update (clip_finalize_kernel)
  const float lr = lr_dev ? (float)*lr_dev : lr_v;  // device lr: graph-captured rounds
  const uint64_t n4 = n / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float4 P = reinterpret_cast<float4*>(p)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float4 Mm = reinterpret_cast<float4*>(m)[i];
    float4 Vv = reinterpret_cast<float4*>(v)[i];
    adamw_elem(P.x, G.x, Mm.x, Vv.x, cf, lr, b1, b2, ib1, ib2, eps, wd);
    adamw_elem(P.y, G.y, Mm.y, Vv.y, cf, lr, b1, b2, ib1, ib2, eps, wd);
    adamw_elem(P.z, G.z, Mm.z, Vv.z, cf, lr, b1, b2, ib1, ib2, eps, wd);
    adamw_elem(P.w, G.w, Mm.w, Vv.w, cf, lr, b1, b2, ib1, ib2, eps, wd);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = Mm;
    reinterpret_cast<float4*>(v)[i] = Vv;
    if (shadow) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(shadow)[i] = pk;
    }
  }
  for (uint64_t i = n4 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    adamw_elem(p[i], g[i], m[i], v[i], cf, lr, b1, b2, ib1, ib2, eps, wd);
    if (shadow) shadow[i] = __float2bfloat16_rn(p[i]);
  }
}

void adamw_f32(float* p, const float* g, float* m, float* v, bf16* shadow, uint64_t n,
               const float* cf, double lr, double b1, double b2, double bc1, double bc2,
               double eps, double wd, cudaStream_t st, const double* lr_dev) {
  launch_pdl(adamw_f32_kernel, kNumSMs * 8, 256, 0, st, p, g, m, v, shadow, n, cf, (float)lr, lr_dev, (float)b1,
                                                (float)b2, (float)(1.0 / bc1), (float)(1.0 / bc2),
                                                (float)eps, (float)wd);
  PH_LAUNCH_CHECK();
}

// optim.cpp:92-103: p -= lr * (g * cf)
__global__ void sgd_f32_kernel(float* __restrict__ p, const float* __restrict__ g,
                               bf16* __restrict__ shadow, uint64_t n, const float* cfp,
                               double lr_v, const double* lr_dev) {
  pdl_launch_dependents();
  pdl_wait();
  const double cf = (double)*cfp;
  if (cf != cf) return;  // NumericError step: no update (clip_finalize_kernel)
  const double lr = lr_dev ? *lr_dev : lr_v;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float np = (float)((double)p[i] - lr * ((double)g[i] * cf));
    p[i] = np;
    if (shadow) shadow[i] = __float2bfloat16_rn(np);
  }
}

void sgd_f32(float* p, const float* g, bf16* shadow, uint64_t n, const float* cf, double lr,
             cudaStream_t st, const double* lr_dev) {
  launch_pdl(sgd_f32_kernel, kNumSMs * 8, 256, 0, st, p, g, shadow, n, cf, lr, lr_dev);
  PH_LAUNCH_CHECK();
}

// ---- exact f64 variants (the f64 C-ABI) -----------------------------------------
// Strict left-to-right sum of squares: one thread, as param_vector.cpp:105-110.
__global__ void sumsq_seq_kernel(const double* __restrict__ g, uint64_t n, double* out) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(g[i], g[i]));
  *out = sqrt(acc);
}
void sumsq_sequential_f64(const double* g, uint64_t n, double* out, cudaStream_t st) {
  sumsq_seq_kernel<<<1, 1, 0, st>>>(g, n, out);
  PH_LAUNCH_CHECK();
}

__device__ __forceinline__ double clip_cf(double norm, double clip) {
  return (clip > 0.0 && norm > clip) ? clip / norm : 1.0;
}

__global__ void adamw_f64_kernel(double* __restrict__ p, const double* __restrict__ g,
                                 double* __restrict__ m, double* __restrict__ v, uint64_t n,
                                 const double* norm, double clip, double lr, double b1, double b2,
                                 double bc1, double bc2, double eps, double wd) {
  const double cf = clip_cf(*norm, clip);
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double gj = g[j] * cf;
    m[j] = b1 * m[j] + (1.0 - b1) * gj;
    v[j] = b2 * v[j] + (1.0 - b2) * gj * gj;
    const double mhat = m[j] / bc1;
    const double vhat = v[j] / bc2;
    p[j] -= lr * (mhat / (sqrt(vhat) + eps) + wd * p[j]);
  }
}
void adamw_f64(double* p, const double* g, double* m, double* v, uint64_t n, const double* norm,
               double clip, double lr, double b1, double b2, double bc1, double bc2, double eps,
               double wd, cudaStream_t st) {
  adamw_f64_kernel<<<kNumSMs * 4, 256, 0, st>>>(p, g, m, v, n, norm, clip, lr, b1, b2, bc1, bc2,
                                                eps, wd);
  PH_LAUNCH_CHECK();
}

__global__ void sgd_f64_kernel(double* __restrict__ p, const double* __restrict__ g, uint64_t n,
                               const double* norm, double clip, double lr) {
  const double cf = clip_cf(*norm, clip);
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    p[j] -= lr * (g[j] * cf);
}
void sgd_f64(double* p, const double* g, uint64_t n, const double* norm, double clip, double lr,
             cudaStream_t st) {
  sgd_f64_kernel<<<kNumSMs * 4, 256, 0, st>>>(p, g, n, norm, clip, lr);
  PH_LAUNCH_CHECK();
}

// ---- aggregation ------------------------------------------------------------------
// Per element, in the reference's exact operation order:
//   mean  = corr != 0 ? v0 + corr / n : v0,  corr = sum_{i>=1} (v_i - v0)  (param_vector.cpp:140-150)
//   FedAvg: theta' = mean                                                  (optim.cpp:129-133)
//   momentum: delta = theta + (-1)*mean; v = mu*v + delta;
//             theta' = (eta == 1 && mu == 0) ? mean
//                      : theta - eta * (nesterov ? mu*v + delta : v)       (optim.cpp:136-158)
constexpr int kMaxModelsSmem = 256;

template <typename T>
__device__ __forceinline__ T anchored_mean(const T* const* models, int k, uint64_t j, T nk) {
  const T anchor = models[0][j];
  T corr = T(0);
  for (int i = 1; i < k; ++i) corr += models[i][j] - anchor;
  return corr != T(0) ? anchor + corr / nk : anchor;
}

template <typename T>
__device__ __forceinline__ void outer_update(T& theta, T& vel, T mean, int kind, T eta, T mu,
                                             int nesterov) {
  if (kind == 0) {
    theta = mean;
    return;
  }
  const T delta = theta + T(-1) * mean;
  vel = mu * vel + delta;
  if (eta == T(1) && mu == T(0)) {
    theta = mean;
    return;
  }
  const T dir = nesterov ? mu * vel + delta : vel;
  theta = theta - eta * dir;
}

template <typename T>
__global__ void __launch_bounds__(256) aggregate_kernel(const T* const* __restrict__ models_g,
                                                        int k, uint64_t n, T* __restrict__ theta,
                                                        T* __restrict__ vel, int kind, T eta,
                                                        T mu, int nesterov) {
  // the pointer table is staged in shared memory when it fits; more models
  // (ParamVector::mean has no limit) are read straight from the global table
  __shared__ const T* models_s[kMaxModelsSmem];
  const bool in_smem = k <= kMaxModelsSmem;
  if (in_smem)
    for (int i = threadIdx.x; i < k; i += blockDim.x) models_s[i] = models_g[i];
  __syncthreads();
  const T* const* models = in_smem ? models_s : models_g;
  const T nk = (T)k;
  constexpr int V = 16 / sizeof(T);  // elements per 128-bit access
  using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const uint64_t nv = n / V;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Vec a = reinterpret_cast<const Vec*>(models[0])[i];
    T anchor[V], corr[V];
    memcpy(anchor, &a, sizeof(Vec));
#pragma unroll
    for (int e = 0; e < V; ++e) corr[e] = T(0);
    for (int c = 1; c < k; ++c) {
      Vec b = reinterpret_cast<const Vec*>(models[c])[i];
      T bv[V];
      memcpy(bv, &b, sizeof(Vec));
#pragma unroll
      for (int e = 0; e < V; ++e) corr[e] += bv[e] - anchor[e];
    }
    Vec tv, vv;
    T th[V], ve[V];
    if (kind != 0) {  // FedAvg never reads theta (optim.cpp:129-133)
      tv = reinterpret_cast<Vec*>(theta)[i];
      vv = reinterpret_cast<Vec*>(vel)[i];
      memcpy(th, &tv, sizeof(Vec));
      memcpy(ve, &vv, sizeof(Vec));
    }
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const T mean = corr[e] != T(0) ? anchor[e] + corr[e] / nk : anchor[e];
      outer_update(th[e], ve[e], mean, kind, eta, mu, nesterov);
    }
    memcpy(&tv, th, sizeof(Vec));
    reinterpret_cast<Vec*>(theta)[i] = tv;
    if (kind != 0) {
      memcpy(&vv, ve, sizeof(Vec));
      reinterpret_cast<Vec*>(vel)[i] = vv;
    }
  }
  for (uint64_t j = nv * V + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const T mean = anchored_mean(models, k, j, nk);
    T th = kind != 0 ? theta[j] : T(0), ve = kind != 0 ? vel[j] : T(0);
    outer_update(th, ve, mean, kind, eta, mu, nesterov);
    theta[j] = th;
    if (kind != 0) vel[j] = ve;
  }
}

// ---- round boundary over peer memory ---------------------------------------------
// One kernel per rank does the reduce-scatter, the update and the all-gather:
// for its shard [off, off+len) it loads every surviving client's model straight
// from the owning GPU's HBM over NVLink (IPC-mapped pointers), forms the
// anchored mean in ascending client order, applies the outer step with the
// resident theta_t / velocity shards, and stores theta_{t+1} into EVERY rank's
// replica.  Same per-element arithmetic as aggregate_kernel (bit-identical for
// any world size); wire bytes per GPU = 2 (G-1)/G * P * 4 as for ring all-reduce.
template <int KM>  // KM >= a.n: registers sized to the client count
__global__ void __launch_bounds__(256) boundary_p2p_kernel(const __grid_constant__ PeerBoundaryArgs a) {
  if (a.abort && *a.abort) return;  // a peer never arrived: PeerBoundary::check() reports it
  const int k = a.n;
  const float nk = (float)k;
  const float* const* models = a.models;
  const uint64_t nv = a.len / 4, base = a.off / 4;
  float* mine = a.replicas[a.rank];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv;
       i += (uint64_t)gridDim.x * blockDim.x) {
    // issue every client's load before the first use (NVLink latency ~1-2k cycles)
    float4 m[KM];
#pragma unroll
    for (int c = 0; c < KM; ++c)
      if (c < k) m[c] = reinterpret_cast<const float4*>(models[c])[base + i];
    float4 th = make_float4(0.f, 0.f, 0.f, 0.f), ve = th;
    if (a.kind != 0) {
      th = reinterpret_cast<const float4*>(mine)[base + i];
      ve = reinterpret_cast<const float4*>(a.vel)[i];
    }
    float anchor[4] = {m[0].x, m[0].y, m[0].z, m[0].w};
    float corr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 1; c < KM; ++c) {
      if (c < k) {
        corr[0] += m[c].x - anchor[0];
        corr[1] += m[c].y - anchor[1];
        corr[2] += m[c].z - anchor[2];
        corr[3] += m[c].w - anchor[3];
      }
    }
    float t4[4] = {th.x, th.y, th.z, th.w}, v4[4] = {ve.x, ve.y, ve.z, ve.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float mean = corr[e] != 0.f ? anchor[e] + corr[e] / nk : anchor[e];
      outer_update(t4[e], v4[e], mean, a.kind, a.eta, a.mu, a.nesterov);
    }
    const float4 out = make_float4(t4[0], t4[1], t4[2], t4[3]);
    for (int g = 0; g < a.world; ++g) reinterpret_cast<float4*>(a.replicas[g])[base + i] = out;
    if (a.kind != 0) reinterpret_cast<float4*>(a.vel)[i] = make_float4(v4[0], v4[1], v4[2], v4[3]);
  }
  __threadfence_system();  // the peers' copies are complete before the closing barrier
}

void boundary_p2p(const PeerBoundaryArgs& a, cudaStream_t st) {
  if (a.n < 1 || a.n > kMaxPeerModels || a.world < 1 || a.world > kMaxPeerWorld || a.len % 4 ||
      a.off % 4)
    throw Error(PHOTON_ERR_USAGE, "boundary_p2p: bad arguments");
  // 8 CTAs per SM: twice the resident count (62-106 registers), more remote
  // loads in flight than 2 or 4 per SM (measured)
  const int grid = kNumSMs * 8;
  if (a.n <= 2) boundary_p2p_kernel<2><<<grid, 256, 0, st>>>(a);
  else if (a.n <= 4) boundary_p2p_kernel<4><<<grid, 256, 0, st>>>(a);
  else if (a.n <= 8) boundary_p2p_kernel<8><<<grid, 256, 0, st>>>(a);
  else boundary_p2p_kernel<kMaxPeerModels><<<grid, 256, 0, st>>>(a);
  PH_LAUNCH_CHECK();
}

template <typename T>
void aggregate(const T* const* models, int k, uint64_t n, T* theta, T* velocity, int kind,
               double eta, double mu, int nesterov, cudaStream_t st) {
  if (k < 1) throw Error(PHOTON_ERR_USAGE, "aggregate: bad model count");
  aggregate_kernel<T><<<kNumSMs * 4, 256, 0, st>>>(models, k, n, theta, velocity, kind, (T)eta,
                                                   (T)mu, nesterov);
  PH_LAUNCH_CHECK();
}

template <typename T>
__global__ void mean_kernel(const T* const* __restrict__ models_g, int k, uint64_t n,
                            T* __restrict__ out) {
  __shared__ const T* models_s[kMaxModelsSmem];
  const bool in_smem = k <= kMaxModelsSmem;
  if (in_smem)
    for (int i = threadIdx.x; i < k; i += blockDim.x) models_s[i] = models_g[i];
  __syncthreads();
  const T* const* models = in_smem ? models_s : models_g;
  const T nk = (T)k;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = anchored_mean(models, k, j, nk);
}
template <typename T>
void mean_only(const T* const* models, int k, uint64_t n, T* out, cudaStream_t st) {
  if (k < 1) throw Error(PHOTON_ERR_USAGE, "mean: bad model count");
  mean_kernel<T><<<kNumSMs * 4, 256, 0, st>>>(models, k, n, out);
  PH_LAUNCH_CHECK();
}

template <typename T>
__global__ void sub_kernel(const T* __restrict__ a, const T* __restrict__ b, uint64_t n,
                           T* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = a[j] + T(-1) * b[j];
}
template <typename T>
void sub_only(const T* a, const T* b, uint64_t n, T* out, cudaStream_t st) {
  sub_kernel<T><<<kNumSMs * 4, 256, 0, st>>>(a, b, n, out);
  PH_LAUNCH_CHECK();
}

// server_step with an explicit delta (optim.cpp:124-159)
template <typename T>
__global__ void server_step_kernel(const T* __restrict__ theta, const T* __restrict__ delta,
                                   const T* __restrict__ mean, T* __restrict__ vel,
                                   T* __restrict__ out, uint64_t n, int kind, T eta, T mu,
                                   int nesterov) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (kind == 0) {
      out[j] = mean[j];
      continue;
    }
    const T v = mu * vel[j] + delta[j];
    vel[j] = v;
    if (eta == T(1) && mu == T(0)) {
      out[j] = mean[j];
      continue;
    }
    const T dir = nesterov ? mu * v + delta[j] : v;
    out[j] = theta[j] - eta * dir;
  }
}
template <typename T>
void server_step_only(const T* theta, const T* delta, const T* mean, T* velocity, T* out,
                      uint64_t n, int kind, double eta, double mu, int nesterov,
                      cudaStream_t st) {
  server_step_kernel<T><<<kNumSMs * 4, 256, 0, st>>>(theta, delta, mean, velocity, out, n, kind,
                                                     (T)eta, (T)mu, nesterov);
  PH_LAUNCH_CHECK();
}

// ---- post_process clip (client.cpp:96-110) -----------------------------------------
__global__ void diff_sumsq_kernel(const float* __restrict__ ref, const float* __restrict__ th,
                                  uint64_t n, double* __restrict__ part) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = (double)th[i] - (double)ref[i];
    acc += u * u;
  }
  const double s = block_sum(acc, (float*)nullptr);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void clip_apply_kernel(const float* __restrict__ ref, float* __restrict__ th,
                                  uint64_t n, const double* __restrict__ part, int nparts,
                                  double thr) {
  __shared__ double scale;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < nparts; ++i) acc += part[i];
    const double norm = sqrt(acc);
    scale = norm <= thr ? -1.0 : thr / norm;
  }
  __syncthreads();
  if (scale < 0.0) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = (double)th[i] - (double)ref[i];
    th[i] = (float)((double)ref[i] + scale * u);
  }
}
void clip_update_f32(const float* ref, float* theta_k, uint64_t n, double threshold,
                     double* part, cudaStream_t st) {
  diff_sumsq_kernel<<<kRedBlocks, 256, 0, st>>>(ref, theta_k, n, part);
  PH_LAUNCH_CHECK();
  clip_apply_kernel<<<kRedBlocks, 256, 0, st>>>(ref, theta_k, n, part, kRedBlocks, threshold);
  PH_LAUNCH_CHECK();
}

#define INST(T)                                                                               \
  template void aggregate<T>(const T* const*, int, uint64_t, T*, T*, int, double, double, int, \
                             cudaStream_t);                                                   \
  template void mean_only<T>(const T* const*, int, uint64_t, T*, cudaStream_t);               \
  template void sub_only<T>(const T*, const T*, uint64_t, T*, cudaStream_t);                  \
  template void server_step_only<T>(const T*, const T*, const T*, T*, T*, uint64_t, int,      \
                                    double, double, int, cudaStream_t);
INST(float)
INST(double)
#undef INST

}  // namespace k
}  // namespace photon
