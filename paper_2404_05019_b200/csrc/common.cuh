// Shared helpers for the sm_100a ScMoE kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/scmoe.h"

namespace scmoe {

// Records a message for scmoe_last_error(); defined in capi.cu.
void set_error(const char* fmt, ...);

#define SCMOE_CHECK_ARG(cond, ...)            \
  do {                                        \
    if (!(cond)) {                            \
      ::scmoe::set_error(__VA_ARGS__);        \
      return SCMOE_ERR_ARG;                   \
    }                                         \
  } while (0)

#define SCMOE_CUDA_TRY(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::scmoe::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                         __FILE__, __LINE__);                                  \
      return SCMOE_ERR_CUDA;                                                   \
    }                                                                          \
  } while (0)

#define SCMOE_LAUNCH_CHECK()                                                   \
  do {                                                                         \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::scmoe::set_error("kernel launch failed: %s (%s:%d)",                  \
                         cudaGetErrorString(_e), __FILE__, __LINE__);          \
      return SCMOE_ERR_CUDA;                                                   \
    }                                                                          \
  } while (0)

int num_sms();

// Fused ScMoE combine in the shared expert's GEMM2 epilogue (direct add):
// y is the routed experts' (E, capacity, d) output.
struct CombineSpec {
  const void* y;
  const int32_t* indices;
  const int32_t* slots;
  const float* weights;
  int capacity, k;
};

// ---- element access ---------------------------------------------------------

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// 16-byte vector of T: 8 x bf16 or 4 x f32.
template <typename T> struct Vec16;
template <> struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  uint4 raw;
  __device__ __forceinline__ void to_float(float* f) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 p = __bfloat1622float2(h[i]);
      f[2 * i] = p.x;
      f[2 * i + 1] = p.y;
    }
  }
  __device__ __forceinline__ void from_float(const float* f) {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  }
};
template <> struct Vec16<float> {
  static constexpr int N = 4;
  uint4 raw;
  __device__ __forceinline__ void to_float(float* f) const {
    const float* s = reinterpret_cast<const float*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = s[i];
  }
  __device__ __forceinline__ void from_float(const float* f) {
    float* s = reinterpret_cast<float*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = f[i];
  }
};

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// Exact (erf) GELU, the reference's numkit.gelu (numkit.py:96-99).
__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}

// Branch-free erf GELU for bf16 epilogues: Abramowitz & Stegun 7.1.26
// (|erf error| < 1.5e-7, far below bf16 resolution), one RCP + one EX2 on the
// MUFU pipe and ~12 FMA-pipe instructions; erff() diverges between two
// polynomial branches and costs ~3x more issue slots in a tcgen05 epilogue.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float gelu_erf_fast(float x) {
  // gelu(x) = x/2 (1 + erf(x/sqrt2)) = x/2 + |x|/2 erf(|x|/sqrt2); erf by
  // A&S 7.1.26 in t = 1/(1 + p|x|/sqrt2) (the 1/sqrt2 folded into p and into
  // the exponent: exp(-x^2/2) = 2^(-x^2 log2(e)/2)); 12 FP ops + 2 MUFU
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752440f, fabsf(x), 1.0f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float e = ex2_approx((x * x) * -0.72134752044448170368f);   // exp(-x^2/2)
  const float erf_abs = fmaf(-p, e, 1.0f);
  const float hx = 0.5f * x;
  return fmaf(fabsf(hx), erf_abs, hx);
}

// d/dz gelu(z) = Phi(z) + z * phi(z), same erf approximation (shares exp(-z^2/2))
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752440f, fabsf(x), 1.0f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float e = ex2_approx((x * x) * -0.72134752044448170368f);   // exp(-x^2/2)
  const float erf_v = copysignf(fmaf(-p, e, 1.0f), x);
  return fmaf(0.5f, erf_v, 0.5f) + x * e * 0.39894228040143267794f;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace scmoe
