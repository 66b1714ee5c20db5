// K7 elementwise GELU passes of the training FFN (tape.py:137-142, exact-erf
// GELU of numkit.py:96-99 via the A&S erf of common.cuh, |erf err| < 1.5e-7).
//
// Why not in the GEMM epilogue: at configs[1] (d = 384) a tcgen05 tile of the
// FFN GEMMs has K = 384, so its MMAs take ~2.7 us while an epilogue that
// evaluates erf for 32K outputs with the GEMM's 8-16 epilogue warps runs at
// IPC ~0.5 per scheduler (measured, ncu: stall_wait / short_sb) — the fused
// GELU / GELU-backward epilogues made those GEMMs 2-3.5x slower than the
// plain ones.  Here the same math runs at full occupancy as an HBM-bound pass,
// and the backward pass also produces the bias gradient (column sums of dZ)
// from the registers it already holds.
//
//   gelu_fwd:  h = gelu(z) on rows < rows(g), 0 on [rows(g), rows_pad(g))
//   gelu_bwd:  dz = dh * gelu'(z) on rows < rows(g), 0 on [rows(g), rows_pad(g))
//              db_part[g][stripe][c] = sum over the stripe's valid rows of dz
// rows(g) = min(group_rows[g], rows_clip) (all `cap` rows without
// group_rows); rows_pad(g) = min(cap, roundup(rows(g), 64)) keeps the
// zero-padded 64-row blocks the weight-gradient GEMM sums.
#include "common.cuh"

namespace scmoe {
namespace {

constexpr int GT = 256;                  // threads per block
constexpr int PAD = 64;                  // weight-gradient k-block

__device__ __forceinline__ int rows_valid(const int32_t* gr, int g, int clip, int cap) {
  return gr ? max(0, min(gr[g], clip)) : cap;
}
__device__ __forceinline__ int rows_padded(int rows, int cap) {
  return min(cap, (rows + PAD - 1) / PAD * PAD);
}

// one 16-byte vector (8 bf16) per thread per step, 4 steps in flight; rows
// in [rows(g), rows_pad(g)) are written as zeros (the zero-padded blocks the
// weight gradient reads; z there is never initialised)
__device__ __forceinline__ uint4 gelu_vec(uint4 raw) {
  Vec16<__nv_bfloat16> a;
  a.raw = raw;
  float f[8];
  a.to_float(f);
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = gelu_erf_fast(f[e]);
  a.from_float(f);
  return a.raw;
}

// gelu(x) and gelu'(x) sharing the reciprocal and the exponential: the same
// operation sequences as gelu_erf_fast / gelu_grad_fast, so both values are
// bit-identical to the separate evaluations
__device__ __forceinline__ void gelu_both(float x, float& g, float& dg) {
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752440f, fabsf(x), 1.0f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float e = ex2_approx((x * x) * -0.72134752044448170368f);   // exp(-x^2/2)
  const float erf_abs = fmaf(-p, e, 1.0f);
  const float hx = 0.5f * x;
  g = fmaf(fabsf(hx), erf_abs, hx);
  const float erf_v = copysignf(erf_abs, x);
  dg = fmaf(0.5f, erf_v, 0.5f) + x * e * 0.39894228040143267794f;
}

__device__ __forceinline__ void gelu_vec2(uint4 raw, uint4& h, uint4& dh) {
  Vec16<__nv_bfloat16> a;
  a.raw = raw;
  float f[8], g[8], d[8];
  a.to_float(f);
#pragma unroll
  for (int e = 0; e < 8; ++e) gelu_both(f[e], g[e], d[e]);
  a.from_float(g);
  h = a.raw;
  a.from_float(d);
  dh = a.raw;
}

// h = gelu(z) and, with GRAD, dg = gelu'(z) (the backward then multiplies
// in the data-gradient GEMM's epilogue instead of re-evaluating erf)
template <bool GRAD>
__global__ void __launch_bounds__(GT)
gelu_fwd_kernel(const uint4* __restrict__ z, uint4* __restrict__ h, uint4* __restrict__ dg,
                int cap, int vecs_per_row, const int32_t* __restrict__ gr, int clip) {
  const int g = blockIdx.y;
  const int rows = rows_valid(gr, g, clip, cap);
  const int rows_pad = gr ? rows_padded(rows, cap) : cap;
  const long long n = (long long)rows * vecs_per_row;
  const long long n_pad = (long long)rows_pad * vecs_per_row;
  const long long base = (long long)g * cap * vecs_per_row;
  const long long stride = (long long)gridDim.x * GT;
  long long i = blockIdx.x * (long long)GT + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)      // z is dead after this pass: evict-first (GRAD)
      v[u] = GRAD ? __ldcs(z + base + i + u * stride) : ld_nc_v4(z + base + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (GRAD) {
        // gelu'(z) is read only by the backward: a streaming (evict-first)
        // store keeps h — read by the next GEMM right away — in L2
        uint4 hv, dv;
        gelu_vec2(v[u], hv, dv);
        h[base + i + u * stride] = hv;
        __stcs(dg + base + i + u * stride, dv);
      }
      else h[base + i + u * stride] = gelu_vec(v[u]);
    }
  }
  for (; i < n_pad; i += stride) {
    if (GRAD) {
      uint4 a = make_uint4(0, 0, 0, 0), b = a;
      if (i < n) gelu_vec2(ld_nc_v4(z + base + i), a, b);
      h[base + i] = a;
      __stcs(dg + base + i, b);
    } else {
      h[base + i] = i < n ? gelu_vec(ld_nc_v4(z + base + i)) : make_uint4(0, 0, 0, 0);
    }
  }
}

// block (column tile of up to GT vectors, row stripe, group); thread (v, lane)
// owns column vector v and rows lane, lane + lanes, ... of the stripe
__global__ void __launch_bounds__(GT)
gelu_bwd_kernel(const __nv_bfloat16* __restrict__ dh, const __nv_bfloat16* __restrict__ z,
                __nv_bfloat16* __restrict__ dz, int cap, int cols, const int32_t* __restrict__ gr,
                int clip, int stripe_rows, int n_stripes, float* __restrict__ part) {
  constexpr int U = 4;
  __shared__ float red[GT][9];
  const int vecs = cols / 8;
  const int vpb = min(vecs, GT);
  const int lanes = GT / vpb;
  const int v = threadIdx.x % vpb, lane = threadIdx.x / vpb;
  const int g = blockIdx.z, stripe = blockIdx.y;
  const int cv = blockIdx.x * vpb + v;
  const bool active = lane < lanes && cv < vecs;
  const int rows = rows_valid(gr, g, clip, cap);
  const int rows_pad = gr ? rows_padded(rows, cap) : cap;
  const int r0 = stripe * stripe_rows, r1 = min(rows_pad, r0 + stripe_rows);
  float s[8] = {};
  if (active) {
    const long long off0 = ((long long)g * cap) * cols + (long long)cv * 8;
    int r = r0 + lane;
    for (; r + (U - 1) * lanes < r1; r += U * lanes) {
      uint4 a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long o = off0 + (long long)(r + u * lanes) * cols;
        a[u] = ld_nc_v4(dh + o);
        b[u] = ld_nc_v4(z + o);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = r + u * lanes;
        Vec16<__nv_bfloat16> va, vb;
        va.raw = a[u];
        vb.raw = b[u];
        float fa[8], fb[8];
        va.to_float(fa);
        vb.to_float(fb);
        const bool ok = rr < rows;
#pragma unroll
        for (int e = 0; e < 8; ++e) fa[e] = ok ? fa[e] * gelu_grad_fast(fb[e]) : 0.f;
        va.from_float(fa);
        st_v4(dz + off0 + (long long)rr * cols, va.raw);
        // the bias gradient sums the stored (bf16-rounded) dz, as the weight
        // gradient GEMM reads it
        va.to_float(fa);
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] += fa[e];
      }
    }
    for (; r < r1; r += lanes) {
      const long long o = off0 + (long long)r * cols;
      Vec16<__nv_bfloat16> va, vb;
      va.raw = ld_nc_v4(dh + o);
      vb.raw = ld_nc_v4(z + o);
      float fa[8], fb[8];
      va.to_float(fa);
      vb.to_float(fb);
      const bool ok = r < rows;
#pragma unroll
      for (int e = 0; e < 8; ++e) fa[e] = ok ? fa[e] * gelu_grad_fast(fb[e]) : 0.f;
      va.from_float(fa);
      st_v4(dz + o, va.raw);
      va.to_float(fa);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] += fa[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.x][e] = s[e];
  __syncthreads();
  if (part && lane == 0 && cv < vecs) {
    float o[8] = {};
    for (int l = 0; l < lanes; ++l)
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += red[l * vpb + v][e];
    float* q = part + ((long long)g * n_stripes + stripe) * cols + (long long)cv * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = o[e];
  }
}

// out[g][c] = sum_stripe part[g][stripe][c]: block (32 columns x 32 lanes)
__global__ void stripe_sum_kernel(const float* __restrict__ part, int n_stripes, int cols,
                                  float* __restrict__ out) {
  __shared__ float red[32][33];
  const int g = blockIdx.y;
  const int c = blockIdx.x * 32 + threadIdx.x;
  float a0 = 0.f, a1 = 0.f;
  if (c < cols) {
    const float* p = part + (long long)g * n_stripes * cols + c;
    int k = threadIdx.y;
    for (; k + 32 < n_stripes; k += 64) {
      a0 += p[(long long)k * cols];
      a1 += p[(long long)(k + 32) * cols];
    }
    for (; k < n_stripes; k += 32) a0 += p[(long long)k * cols];
  }
  red[threadIdx.y][threadIdx.x] = a0 + a1;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float t = 0.f;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) t += red[y][threadIdx.x];
    out[(long long)g * cols + c] = t;
  }
}

int bwd_stripes(int num_groups, int cap, int cols) {
  const int vecs = cols / 8;
  const int col_tiles = (vecs + GT - 1) / GT;
  // ~6 blocks' worth of stripes per SM: short per-thread row loops (the
  // loads of a stripe are latency-bound), partials stay small
  int st = (6 * num_sms() + col_tiles * num_groups - 1) / (col_tiles * num_groups);
  return max(1, min(st, (cap + 7) / 8));
}

}  // namespace
}  // namespace scmoe

using namespace scmoe;

extern "C" int scmoe_gelu_fwd(const void* z, void* h, int num_groups, int group_cap, int cols,
                              const int32_t* group_rows, int rows_clip, void* stream) {
  SCMOE_CHECK_ARG(z && h && num_groups >= 1 && group_cap >= 1 && cols >= 8 && cols % 8 == 0,
                  "gelu_fwd: bad arguments");
  SCMOE_CHECK_ARG(((uintptr_t)z & 15) == 0 && ((uintptr_t)h & 15) == 0,
                  "gelu_fwd: 16-byte aligned bf16 rows needed");
  if (rows_clip <= 0) rows_clip = group_cap;
  const long long per_group = (long long)group_cap * cols / 8;
  long long bx = (per_group + GT * 4 - 1) / (GT * 4);
  const long long cap_bx = 8ll * num_sms() / num_groups;
  if (bx > cap_bx) bx = cap_bx;
  gelu_fwd_kernel<false><<<dim3((unsigned)(bx < 1 ? 1 : bx), num_groups), GT, 0,
                           (cudaStream_t)stream>>>((const uint4*)z, (uint4*)h, nullptr, group_cap,
                                                   cols / 8, group_rows, rows_clip);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_gelu_fwd_grad(const void* z, void* h, void* dgelu, int num_groups,
                                   int group_cap, int cols, const int32_t* group_rows,
                                   int rows_clip, void* stream) {
  SCMOE_CHECK_ARG(z && h && dgelu && num_groups >= 1 && group_cap >= 1 && cols >= 8 &&
                      cols % 8 == 0,
                  "gelu_fwd_grad: bad arguments");
  SCMOE_CHECK_ARG(((uintptr_t)z & 15) == 0 && ((uintptr_t)h & 15) == 0 &&
                      ((uintptr_t)dgelu & 15) == 0,
                  "gelu_fwd_grad: 16-byte aligned bf16 rows needed");
  if (rows_clip <= 0) rows_clip = group_cap;
  const long long per_group = (long long)group_cap * cols / 8;
  long long bx = (per_group + GT * 4 - 1) / (GT * 4);
  const long long cap_bx = 8ll * num_sms() / num_groups;
  if (bx > cap_bx) bx = cap_bx;
  gelu_fwd_kernel<true><<<dim3((unsigned)(bx < 1 ? 1 : bx), num_groups), GT, 0,
                          (cudaStream_t)stream>>>((const uint4*)z, (uint4*)h, (uint4*)dgelu,
                                                  group_cap, cols / 8, group_rows, rows_clip);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" size_t scmoe_gelu_bwd_workspace_bytes(int num_groups, int group_cap, int cols) {
  if (num_groups < 1 || group_cap < 1 || cols < 8) return 0;
  return (size_t)bwd_stripes(num_groups, group_cap, cols) * num_groups * cols * sizeof(float);
}

extern "C" int scmoe_gelu_bwd(const void* dh, const void* z, void* dz, float* bias_grad,
                              int num_groups, int group_cap, int cols, const int32_t* group_rows,
                              int rows_clip, void* workspace, size_t workspace_bytes,
                              void* stream) {
  SCMOE_CHECK_ARG(dh && z && dz && num_groups >= 1 && group_cap >= 1 && cols >= 8 &&
                      cols % 8 == 0,
                  "gelu_bwd: bad arguments");
  SCMOE_CHECK_ARG(((uintptr_t)dh & 15) == 0 && ((uintptr_t)z & 15) == 0 &&
                      ((uintptr_t)dz & 15) == 0,
                  "gelu_bwd: 16-byte aligned bf16 rows needed");
  const int n_stripes = bwd_stripes(num_groups, group_cap, cols);
  SCMOE_CHECK_ARG(!bias_grad || (workspace && workspace_bytes >= scmoe_gelu_bwd_workspace_bytes(
                                                                     num_groups, group_cap, cols)),
                  "gelu_bwd: workspace too small");
  if (rows_clip <= 0) rows_clip = group_cap;
  cudaStream_t st = (cudaStream_t)stream;
  const int vecs = cols / 8;
  const int vpb = min(vecs, GT);
  const int stripe_rows = (group_cap + n_stripes - 1) / n_stripes;
  dim3 grid((vecs + vpb - 1) / vpb, n_stripes, num_groups);
  gelu_bwd_kernel<<<grid, GT, 0, st>>>((const __nv_bfloat16*)dh, (const __nv_bfloat16*)z,
                                       (__nv_bfloat16*)dz, group_cap, cols, group_rows, rows_clip,
                                       stripe_rows, n_stripes,
                                       bias_grad ? (float*)workspace : nullptr);
  SCMOE_LAUNCH_CHECK();
  if (bias_grad) {
    stripe_sum_kernel<<<dim3((cols + 31) / 32, num_groups), dim3(32, 32), 0, st>>>(
        (const float*)workspace, n_stripes, cols, bias_grad);
    SCMOE_LAUNCH_CHECK();
  }
  return SCMOE_OK;
}
