// common.cuh -- shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <utility>
#include <string>

#include "host.hpp"

namespace photon {

#define PH_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::photon::Error(PHOTON_ERR_CUDA, std::string(#call) + ": " +               \
                                                 cudaGetErrorString(e_) + " @" +       \
                                                 __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Every kernel launch site is followed by exactly one PH_LAUNCH_CHECK, which
// also counts the launch (photon_launch_count; a CUDA graph replay adds the
// kernel nodes it holds, see Ctx::launch_local_round).
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}
#define PH_LAUNCH_CHECK()                                                  \
  do {                                                                     \
    PH_CUDA(cudaGetLastError());                                           \
    ::photon::launch_counter().fetch_add(1, std::memory_order_relaxed);    \
  } while (0)

using bf16 = __nv_bfloat16;

// Programmatic dependent launch (PDL): the step's hot kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, start with
// pdl_launch_dependents() (the next kernel's CTAs may be scheduled once every
// CTA of this one has started) and pdl_wait() before their first access to
// global memory another kernel wrote or reads (it returns once the previous
// kernel has completed and its writes are visible) -- so a kernel's launch and
// its prologue (barriers, TMEM allocation, descriptor prefetch) overlap the
// tail of the one before it.  Measured: +9 % tokens/s on the launch-bound
// hetero4 model, but 3-8 % slower on the 125M step (graph replays of large
// persistent kernels), so it is on by default only while a small model
// (d_model <= 512) enqueues its step (PdlScope); PHOTON_PDL=0 / 1 forces it off /
// on everywhere (the two instructions are no-ops without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline int& pdl_thread_flag() {
  static thread_local int on = 0;
  return on;
}
inline bool pdl_on() {
  static const int forced = [] {
    const char* e = std::getenv("PHOTON_PDL");
    return e ? (std::string(e) != "0" ? 1 : 0) : -1;
  }();
  return forced >= 0 ? forced == 1 : pdl_thread_flag() != 0;
}
// PDL for the launches made while it lives on this thread (nests)
struct PdlScope {
  int saved;
  explicit PdlScope(bool on) : saved(pdl_thread_flag()) { pdl_thread_flag() = on ? 1 : saved; }
  ~PdlScope() { pdl_thread_flag() = saved; }
  PdlScope(const PdlScope&) = delete;
  PdlScope& operator=(const PdlScope&) = delete;
};
constexpr uint64_t kPdlMaxWidth = 512;
// kernel classes for PHOTON_PDL_MASK (experiments): 1 GEMM, 2 attention, 4 the rest.
// On the 125M step (PHOTON_PDL=1), per MHz: off 537.6, GEMM only 532, attention
// only 538, the rest only 513-519, all 519 tokens/s/MHz.
enum PdlClass : int { kPdlGemm = 1, kPdlAttn = 2, kPdlOther = 4 };
inline bool pdl_class_on(int cls) {
  static const int mask = [] {
    const char* e = std::getenv("PHOTON_PDL_MASK");
    return e ? std::atoi(e) : 7;
  }();
  return pdl_on() && (mask & cls);
}
template <typename... KArgs, typename... Args>
inline void launch_pdl_cls(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_class_on(cls) ? 1 : 0;
  PH_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_class_on(kPdlOther) ? 1 : 0;
  PH_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: set it
// once for every device that launches the kernel (bit per device in `done`).
template <typename K>
inline void set_max_smem_once(std::atomic<uint64_t>& done, K kern, int bytes) {
  int dev = 0;
  PH_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load() & bit) return;
  PH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.fetch_or(bit);
}

constexpr int kNumSMs = 148;

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// four consecutive values as float4 (16-byte fp32 or 8-byte bf16 load)
__device__ __forceinline__ float4 ld4f(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4f(const bf16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}

// 2^x for a pair on the FMA / ALU pipes (no MUFU): round-to-nearest split via
// the 1.5 * 2^23 magic constant, degree-3 minimax polynomial of 2^f on
// [-1/2, 1/2] (relative error 1.9e-4, far below the bf16 rounding of P), the
// exponent added to the bits; x <= -126 gives 0.
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  constexpr float M = 12582912.0f;
  const float2 j = __fadd2_rn(make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f)), make_float2(M, M));
  const float2 r = __fadd2_rn(j, make_float2(-M, -M));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = __ffma2_rn(make_float2(0.054898735135793686f, 0.054898735135793686f), f,
                        make_float2(0.24193310737609863f, 0.24193310737609863f));
  p = __ffma2_rn(p, f, make_float2(0.6932485103607178f, 0.6932485103607178f));
  p = __ffma2_rn(p, f, make_float2(0.9999765157699585f, 0.9999765157699585f));
  const int ex = __float_as_int(j.x) - __float_as_int(M), ey = __float_as_int(j.y) - __float_as_int(M);
  return make_float2(x.x > -126.f ? __int_as_float(__float_as_int(p.x) + (ex << 23)) : 0.f,
                     x.y > -126.f ? __int_as_float(__float_as_int(p.y) + (ey << 23)) : 0.f);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline unsigned cdiv(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// exact-erf GELU (tensor.cpp:396-420)
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752440f));
  const float pdf = 0.39894228040143267794f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}

// Fast exact-erf GELU for bf16 epilogues: Phi(x) from Abramowitz & Stegun
// 7.1.26 (|erf error| <= 1.5e-7) sharing one exp(-x^2/2) with phi(x).
__device__ __forceinline__ void phi_Phi(float x, float& Phi, float& phi) {
  const float z = fabsf(x) * 0.70710678118654752440f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
  const float e = __expf(-0.5f * x * x);  // = exp(-z^2)
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  const float erf_abs = 1.0f - poly * t * e;
  const float erf_x = copysignf(erf_abs, x);
  Phi = 0.5f * (1.0f + erf_x);
  phi = 0.39894228040143267794f * e;
}
// GELU(x) = x Phi(x) and GELU'(x) = Phi(x) + x phi(x) together, for the GEMM
// epilogue: the same A&S 7.1.26 erf, with the 1/2 of Phi folded into the
// coefficients so that w = Phi(-|x|) = t (b1 + t (b2 + ...)) exp(-x^2/2) and
// Phi = x >= 0 ? 1 - w : w -- 16 FP ops + 2 MUFU per element.
__device__ __forceinline__ void gelu_pair(float x, float& g, float& gp) {
  const float z = fabsf(x) * 0.70710678118654752440f;
  float t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * (x * -0.72134752044448170f)));  // exp(-x^2/2)
  float p = fmaf(0.5307027145f, t, -0.7265760135f);
  p = fmaf(p, t, 0.7107068705f);
  p = fmaf(p, t, -0.142248368f);
  p = fmaf(p, t, 0.127414796f);
  const float w = p * t * e;
  const float Phi = x >= 0.f ? 1.0f - w : w;
  g = x * Phi;
  gp = fmaf(x * 0.39894228040143267794f, e, Phi);
}
// gelu_pair on two elements with sm_100's packed fp32 FMA / MUL / ADD (one
// issue slot per pair): the GeluBias epilogue is issue-bound, not MUFU-bound.
// Same A&S 7.1.26 evaluation; Phi = 1/2 + sign(x) (1/2 - w) and the 1/sqrt(2)
// folded into the first coefficient (ulp-level differences from gelu_pair).
__device__ __forceinline__ void gelu_pair2(float2 x, float2& g, float2& gp) {
  constexpr float c0 = 0.3275911f * 0.70710678118654752440f;
  float2 t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(fmaf(c0, fabsf(x.x), 1.0f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(fmaf(c0, fabsf(x.y), 1.0f)));
  const float2 q = __fmul2_rn(x, __fmul2_rn(x, make_float2(-0.72134752044448170f, -0.72134752044448170f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(q.x));  // exp(-x^2/2)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(q.y));
  float2 p = __ffma2_rn(make_float2(0.5307027145f, 0.5307027145f), t,
                        make_float2(-0.7265760135f, -0.7265760135f));
  p = __ffma2_rn(p, t, make_float2(0.7107068705f, 0.7107068705f));
  p = __ffma2_rn(p, t, make_float2(-0.142248368f, -0.142248368f));
  p = __ffma2_rn(p, t, make_float2(0.127414796f, 0.127414796f));
  const float2 w = __fmul2_rn(__fmul2_rn(p, t), e);  // Phi(-|x|), in (0, 1/2]
  float2 h = __ffma2_rn(w, make_float2(-1.0f, -1.0f), make_float2(0.5f, 0.5f));
  h.x = copysignf(h.x, x.x);
  h.y = copysignf(h.y, x.y);
  const float2 Phi = __fadd2_rn(h, make_float2(0.5f, 0.5f));
  g = __fmul2_rn(x, Phi);
  gp = __ffma2_rn(__fmul2_rn(x, make_float2(0.39894228040143267794f, 0.39894228040143267794f)), e,
                  Phi);
}
// The same pair with one MUFU operation per element (ex2) instead of two: the
// tail of the normal distribution as 0.5 * exp(-x^2/2) * R(|x| / 6.5), R a
// degree-10 polynomial fit of erfcx(|x| / sqrt 2) weighted by exp(-x^2/2)
// (|Phi - Phi_exact| <= 3.1e-7 in fp32, far below the bf16 rounding of the
// epilogue's outputs; |x| > 6.5 clamps, where Phi is 0 or 1 in fp32).  The
// tensor-core GEMM measured it slower in the step than the A&S form (its FMA
// work costs more than the MUFU op it saves), so it is off by default.
__device__ __forceinline__ void gelu_pair2_poly(float2 x, float2& g, float2& gp) {
  constexpr float c[11] = {0.999999463558197f,  -5.186119079589844f, 21.11585235595703f,
                           -72.7467269897461f,  217.98768615722656f, -562.3059692382812f,
                           1190.892822265625f,  -1921.429443359375f, 2145.36767578125f,
                           -1443.036376953125f, 433.9256286621094f};
  const float2 t = make_float2(fminf(fabsf(x.x) * (1.0f / 6.5f), 1.0f), fminf(fabsf(x.y) * (1.0f / 6.5f), 1.0f));
  float2 p = make_float2(c[10], c[10]);
#pragma unroll
  for (int k = 9; k >= 0; --k) p = __ffma2_rn(p, t, make_float2(c[k], c[k]));
  const float2 q = __fmul2_rn(x, __fmul2_rn(x, make_float2(-0.72134752044448170f, -0.72134752044448170f)));
  float2 e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(q.x));  // exp(-x^2/2)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(q.y));
  const float2 w = __fmul2_rn(__fmul2_rn(p, e), make_float2(0.5f, 0.5f));  // Phi(-|x|)
  float2 h = __ffma2_rn(w, make_float2(-1.0f, -1.0f), make_float2(0.5f, 0.5f));
  h.x = copysignf(h.x, x.x);
  h.y = copysignf(h.y, x.y);
  const float2 Phi = __fadd2_rn(h, make_float2(0.5f, 0.5f));
  g = __fmul2_rn(x, Phi);
  gp = __ffma2_rn(__fmul2_rn(x, make_float2(0.39894228040143267794f, 0.39894228040143267794f)), e,
                  Phi);
}
__device__ __forceinline__ float gelu_fast(float x) {
  float Phi, phi;
  phi_Phi(x, Phi, phi);
  return x * Phi;
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  float Phi, phi;
  phi_Phi(x, Phi, phi);
  return fmaf(x, phi, Phi);
}

}  // namespace photon
