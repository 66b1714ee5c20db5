// K2 dispatch ("encode") and K5 combine ("decode"), the HBM-bound halves of
// the routed path.  One warp per token, 16-byte vector accesses, every row
// streamed exactly once.
//
// Reference semantics (relative to /root/reference/pkg/src/scmoelab/):
//   the reference evaluates experts densely and never permutes
//   (arch.py:418-433); dispatch is the sparse equivalent of "expert i sees the
//   rows whose kept weight is non-zero".  combine reproduces
//   routed = sum_j w_j * keep_j * E_{e_j}(x) (arch.py:481-483, 418-433),
//   combine(se, routed, x) (arch.py:380-392) and the block residual add
//   (arch.py:616).
#include "common.cuh"

namespace scmoe {
namespace {

constexpr int WARPS = 8;

template <typename T, int KMAX>
__global__ void __launch_bounds__(WARPS * 32) dispatch_kernel(
    const T* __restrict__ x, long long ld_x, int n_tok, int d, int k,
    const int32_t* __restrict__ indices, const int32_t* __restrict__ slots, int cap,
    const float* __restrict__ row_scale, T* __restrict__ buf) {
  constexpr int VEC = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= n_tok) return;
  // per-selection destinations in registers (KMAX-unrolled; a dropped
  // selection keeps dst = -1)
  long long dst[KMAX];
  float scl[KMAX];
  bool any = false;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    dst[j] = -1;
    scl[j] = 1.f;
    if (j < k) {
      const int s = slots[t * k + j];
      if (s < cap) {
        dst[j] = ((long long)indices[t * k + j] * cap + s) * d;
        if (row_scale) scl[j] = row_scale[t * k + j];
        any = true;
      }
    }
  }
  if (!any) return;
  const T* src = x + t * ld_x;
  // U x 16B loads in flight per lane before the stores
  constexpr int U = 8;
  for (int c = lane * VEC; c < d; c += 32 * VEC * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cc = c + u * 32 * VEC;
      if (cc < d) v[u] = ld_nc_v4(src + cc);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cc = c + u * 32 * VEC;
      if (cc < d) {
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
          if (dst[q] < 0) continue;
          if (row_scale) {
            // combine backward: d expert_out[e, slot] = w * d_out[t]
            Vec16<T> iv, ov;
            iv.raw = v[u];
            float f[VEC];
            iv.to_float(f);
#pragma unroll
            for (int i = 0; i < VEC; ++i) f[i] *= scl[q];
            ov.from_float(f);
            st_v4(buf + dst[q] + cc, ov.raw);
          } else {
            st_v4(buf + dst[q] + cc, v[u]);
          }
        }
      }
    }
  }
}

template <typename T, int MODE, bool HAS_SE, bool HAS_RES, int KMAX>
__global__ void __launch_bounds__(WARPS * 32) combine_kernel(
    const T* __restrict__ se, const T* __restrict__ y, const T* __restrict__ xcur,
    const float* __restrict__ wcg, const T* __restrict__ res,
    const int32_t* __restrict__ indices, const int32_t* __restrict__ slots,
    const float* __restrict__ weights, int cap, int n_tok, int d, int k, T* __restrict__ out) {
  constexpr int VEC = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= n_tok) return;

  // combination coefficients from x_cur (CG-1 sigmoid / CG-2 softmax)
  float c_se = 1.f, c_rt = 1.f;
  if (MODE != SCMOE_COMBINE_DIRECT_ADD) {
    float z0 = 0.f, z1 = 0.f;
    const T* xr = xcur + t * d;
    for (int c = lane * VEC; c < d; c += 32 * VEC) {
      Vec16<T> v;
      v.raw = ld_nc_v4(xr + c);
      float f[VEC];
      v.to_float(f);
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        z0 = fmaf(f[i], wcg[c + i], z0);
        if (MODE == SCMOE_COMBINE_CG2) z1 = fmaf(f[i], wcg[d + c + i], z1);
      }
    }
    z0 = warp_sum(z0);
    if (MODE == SCMOE_COMBINE_CG1) {
      c_se = z0 >= 0.f ? 1.f / (1.f + expf(-z0)) : expf(z0) / (1.f + expf(z0));
    } else {
      z1 = warp_sum(z1);
      const float m = fmaxf(z0, z1);
      const float e0 = expf(z0 - m), e1 = expf(z1 - m);
      c_se = e0 / (e0 + e1);
      c_rt = e1 / (e0 + e1);
    }
  }

  // kept selections in registers (KMAX-unrolled; dropped -> src = -1)
  long long src[KMAX];
  float wt[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    src[j] = -1;
    wt[j] = 0.f;
    if (j < k) {
      const int s = slots[t * k + j];
      if (s < cap) {
        src[j] = ((long long)indices[t * k + j] * cap + s) * d;
        wt[j] = weights[t * k + j];
      }
    }
  }
  // two column chunks per lane at a time: every row's loads of both chunks
  // are issued before any math
  constexpr int U = 2;
  for (int c0 = lane * VEC; c0 < d; c0 += 32 * VEC * U) {
    uint4 yv[U][KMAX], sev[U], rsv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 32 * VEC;
      const bool in = c < d;
#pragma unroll
      for (int q = 0; q < KMAX; ++q)
        yv[u][q] = (in && src[q] >= 0) ? ld_nc_v4(y + src[q] + c) : make_uint4(0, 0, 0, 0);
      if (HAS_SE) sev[u] = in ? ld_nc_v4(se + t * d + c) : make_uint4(0, 0, 0, 0);
      if (HAS_RES) rsv[u] = in ? ld_nc_v4(res + t * d + c) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
    const int c = c0 + u * 32 * VEC;
    if (c >= d) break;
    float r[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) r[i] = 0.f;
#pragma unroll
    for (int q = 0; q < KMAX; ++q) {
      Vec16<T> v;
      v.raw = yv[u][q];
      float f[VEC];
      v.to_float(f);
#pragma unroll
      for (int i = 0; i < VEC; ++i) r[i] = fmaf(wt[q], f[i], r[i]);
    }
    float o[VEC];
    if (HAS_SE) {
      Vec16<T> v;
      v.raw = sev[u];
      float f[VEC];
      v.to_float(f);
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] = c_se * f[i] + c_rt * r[i];
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] = r[i];
    }
    if (HAS_RES) {
      Vec16<T> v;
      v.raw = rsv[u];
      float f[VEC];
      v.to_float(f);
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] += f[i];
    }
    Vec16<T> ov;
    ov.from_float(o);
    st_v4(out + t * d + c, ov.raw);
    }
  }
}

template <typename T, int MODE, int KMAX>
void launch_combine_k(const T* se, const T* y, const T* xc, const float* wcg, const T* res,
                      const int32_t* idx, const int32_t* sl, const float* w, int cap, int n, int d,
                      int k, T* out, cudaStream_t st) {
  const int grid = (n + WARPS - 1) / WARPS;
  if (se && res)
    combine_kernel<T, MODE, true, true, KMAX><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else if (se)
    combine_kernel<T, MODE, true, false, KMAX><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else if (res)
    combine_kernel<T, MODE, false, true, KMAX><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else
    combine_kernel<T, MODE, false, false, KMAX><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
}

template <typename T, int MODE>
void launch_combine_mode(const T* se, const T* y, const T* xc, const float* wcg, const T* res,
                         const int32_t* idx, const int32_t* sl, const float* w, int cap, int n,
                         int d, int k, T* out, cudaStream_t st) {
  if (k == 1)
    launch_combine_k<T, MODE, 1>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
  else if (k == 2)
    launch_combine_k<T, MODE, 2>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
  else
    launch_combine_k<T, MODE, SCMOE_MAX_K>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
}

template <typename T>
void launch_combine(int mode, const void* se, const void* y, const void* xc, const float* wcg,
                    const void* res, const int32_t* idx, const int32_t* sl, const float* w,
                    int cap, int n, int d, int k, void* out, cudaStream_t st) {
  const T *se_ = (const T*)se, *y_ = (const T*)y, *xc_ = (const T*)xc, *res_ = (const T*)res;
  if (mode == SCMOE_COMBINE_CG1)
    launch_combine_mode<T, SCMOE_COMBINE_CG1>(se_, y_, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
  else if (mode == SCMOE_COMBINE_CG2)
    launch_combine_mode<T, SCMOE_COMBINE_CG2>(se_, y_, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
  else
    launch_combine_mode<T, SCMOE_COMBINE_DIRECT_ADD>(se_, y_, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace
}  // namespace scmoe

extern "C" int scmoe_dispatch_scaled(const void* x, int dtype, long long ld_x, int n_tokens,
                                     int d_model, int k, const int32_t* indices,
                                     const int32_t* slots, int capacity, const float* row_scale,
                                     void* dispatch_buf, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(k >= 1 && k <= SCMOE_MAX_K, "k=%d out of range", k);
  SCMOE_CHECK_ARG(capacity >= 1, "capacity must be >= 1");
  const int vec = dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0 && ld_x % vec == 0, "d_model/ld_x must be multiples of %d", vec);
  SCMOE_CHECK_ARG(aligned16(x) && aligned16(dispatch_buf), "buffers must be 16-byte aligned");
  if (n_tokens <= 0) return SCMOE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (n_tokens + WARPS - 1) / WARPS;
#define SCMOE_DISPATCH(T, KM)                                                                  \
  dispatch_kernel<T, KM><<<grid, WARPS * 32, 0, st>>>((const T*)x, ld_x, n_tokens, d_model, k,    \
                                                      indices, slots, capacity, row_scale,      \
                                                      (T*)dispatch_buf)
  if (dtype == SCMOE_BF16) {
    if (k == 1) SCMOE_DISPATCH(__nv_bfloat16, 1);
    else if (k == 2) SCMOE_DISPATCH(__nv_bfloat16, 2);
    else SCMOE_DISPATCH(__nv_bfloat16, SCMOE_MAX_K);
  } else {
    if (k == 1) SCMOE_DISPATCH(float, 1);
    else if (k == 2) SCMOE_DISPATCH(float, 2);
    else SCMOE_DISPATCH(float, SCMOE_MAX_K);
  }
#undef SCMOE_DISPATCH
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_dispatch(const void* x, int dtype, long long ld_x, int n_tokens,
                              int d_model, int k, const int32_t* indices, const int32_t* slots,
                              int capacity, void* dispatch_buf, void* stream) {
  return scmoe_dispatch_scaled(x, dtype, ld_x, n_tokens, d_model, k, indices, slots, capacity,
                               nullptr, dispatch_buf, stream);
}

extern "C" int scmoe_combine(const void* se_out, const void* expert_out, const void* x_cur,
                             const float* w_cg, int mode, const void* residual,
                             const int32_t* indices, const int32_t* slots, const float* weights,
                             int capacity, int n_tokens, int d_model, int k, int dtype, void* out,
                             void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(mode >= 0 && mode <= 2, "bad combine mode %d", mode);
  SCMOE_CHECK_ARG(mode == SCMOE_COMBINE_DIRECT_ADD || (w_cg && x_cur && se_out),
                  "CG modes need w_cg, x_cur and se_out");
  SCMOE_CHECK_ARG(k >= 1 && k <= SCMOE_MAX_K, "k=%d out of range", k);
  const int vec = dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0, "d_model must be a multiple of %d", vec);
  SCMOE_CHECK_ARG(aligned16(expert_out) && aligned16(out) && (!se_out || aligned16(se_out)) &&
                      (!residual || aligned16(residual)) && (!x_cur || aligned16(x_cur)),
                  "buffers must be 16-byte aligned");
  if (n_tokens <= 0) return SCMOE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SCMOE_BF16)
    launch_combine<__nv_bfloat16>(mode, se_out, expert_out, x_cur, w_cg, residual, indices, slots,
                                  weights, capacity, n_tokens, d_model, k, out, st);
  else
    launch_combine<float>(mode, se_out, expert_out, x_cur, w_cg, residual, indices, slots, weights,
                          capacity, n_tokens, d_model, k, out, st);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}
