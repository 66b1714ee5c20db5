// K8 — fp32 grouped GEMM on the FFMA pipe, the parity path for fp32 layers
// (BASELINE configs[0]; tolerance rtol 1e-4 vs the float64 reference).
// Single-pass TF32 tensor cores (10-bit mantissa) cannot meet 1e-4, so this
// path stays on CUDA cores.  Same grouped semantics as the tcgen05 kernel:
//   out[g, r, :] = epi(a[g, r, :] . wt[g % n_wgroups]^T + bias[g % n_wgroups])
// for r < rows(g); expert_forward = arch.py:349-351.
#include "common.cuh"

namespace scmoe {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256;

template <int EPI>
__global__ void __launch_bounds__(THREADS) gemm_f32_kernel(
    const float* __restrict__ a, const float* __restrict__ wt, const float* __restrict__ bias,
    const float* __restrict__ residual, float* __restrict__ out, int n_wgroups, int cap, const int32_t* __restrict__ group_rows,
    int rows_clip, int N, int K) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int g = blockIdx.z;
  const int rows = group_rows ? min(group_rows[g], rows_clip) : cap;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= rows) return;
  const int wg = g % n_wgroups;
  const float* A = a + (long long)g * cap * K;
  const float* B = wt + (long long)wg * N * K;
  const int tid = threadIdx.x;
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  const int ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    {
      const int m = m0 + lr, kk = k0 + lk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < rows) {
        if (kk + 3 < K) v = *reinterpret_cast<const float4*>(A + (long long)m * K + kk);
        else {
          float t[4] = {0.f, 0.f, 0.f, 0.f};
          for (int i = 0; i < 4; ++i) if (kk + i < K) t[i] = A[(long long)m * K + kk + i];
          v = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      As[lk + 0][lr] = v.x; As[lk + 1][lr] = v.y; As[lk + 2][lr] = v.z; As[lk + 3][lr] = v.w;
    }
    {
      const int n = n0 + lr, kk = k0 + lk;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < N) {
        if (kk + 3 < K) v = *reinterpret_cast<const float4*>(B + (long long)n * K + kk);
        else {
          float t[4] = {0.f, 0.f, 0.f, 0.f};
          for (int i = 0; i < 4; ++i) if (kk + i < K) t[i] = B[(long long)n * K + kk + i];
          v = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      Bs[lk + 0][lr] = v.x; Bs[lk + 1][lr] = v.y; Bs[lk + 2][lr] = v.z; Bs[lk + 3][lr] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? bias[(long long)wg * N + n] : 0.f);
      if (EPI == SCMOE_EPI_BIAS_GELU) v = gelu_erf(v);
      const long long o = ((long long)g * cap + m) * N + n;
      if (residual) v += residual[o];
      out[o] = v;
    }
  }
}
}  // namespace

int grouped_gemm_f32(const float* a, const float* wt, const float* bias, const float* residual,
                     float* out,
                     int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                     int rows_clip, int N, int K, int epi, cudaStream_t st) {
  dim3 grid((N + BN - 1) / BN, (cap + BM - 1) / BM, num_groups);
  if (epi == SCMOE_EPI_BIAS_GELU)
    gemm_f32_kernel<SCMOE_EPI_BIAS_GELU><<<grid, THREADS, 0, st>>>(a, wt, bias, residual, out, n_wgroups, cap,
                                                                   group_rows, rows_clip, N, K);
  else
    gemm_f32_kernel<SCMOE_EPI_BIAS><<<grid, THREADS, 0, st>>>(a, wt, bias, residual, out, n_wgroups, cap,
                                                              group_rows, rows_clip, N, K);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

}  // namespace scmoe
