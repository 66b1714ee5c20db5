// K7 gate backward: the VJP of the gate's differentiable outputs (the
// kept-selection weights and the balance loss) with respect to the routed
// source rows and the gate / noise weights, in one pass over the tokens.
//
// Reference semantics (scmoelab):
//   H   = src W_gate (+ eps * softplus(src W_noise))           arch.py:405-415
//   aux = N * sum_j f_j P_j, f_j = counts_j / (T k) (constant),
//         P_j = mean_t softmax(H)_tj                            arch.py:436-439
//   w   = masked softmax of H over the k selections (k > 1)   arch.py:481-482
// VJPs (tape.py:161-176 masked_row_softmax, 121-127 mm, softplus' = sigmoid):
//   dH_tj  = (d_aux N / T) p_tj (f_j - <f, p_t>)
//          + [k > 1] sum_i [idx_ti = j] w_ti (dw_ti - <w_t, dw_t>)
//   dHn_tj = dH_tj eps_tj sigmoid((src W_noise)_tj)
//   d_src  = dH W_gate^T + dHn W_noise^T   (row-wise, written in src's dtype)
//   dW_gate = src^T dH, dW_noise = src^T dHn   (fp32, deterministic)
//
// Layout: block (column chunk of 256, token range).  Phase 1 computes dH (and
// dHn) for 32 tokens into shared memory (one thread per token); phase 2 has
// every thread own two adjacent columns: it streams the 32 src rows
// (coalesced bf16x2 / float2), writes d_src for them and accumulates the
// per-expert column partials of dW in registers.  Partials of every token
// range go to a workspace and a second kernel sums them in a fixed order.
#include "common.cuh"

namespace scmoe {
namespace {

constexpr int GB_THREADS = 128;          // 2 columns each: 256 columns per block
constexpr int GB_TOK = 32;               // tokens per phase-1 batch

struct GateBwdArgs {
  const void* src;
  int T, d, N, k;
  const float* logits;
  const int32_t* indices;
  const float* weights;
  const float* d_weights;
  const int32_t* counts;
  const float* d_aux;
  const float* w_gate_t;      // (N, d)
  const float* w_noise_t;     // (N, d) or null
  const float* eps;           // (T, N) or null
  const float* noise_pre;     // (T, N) = src W_noise, or null
  void* d_src;
  float* part;                // (n_tok_blocks, 2 if noise else 1, N, d)
  int tok_per_block;
};

template <typename T> struct Pair;
template <> struct Pair<__nv_bfloat16> {
  static __device__ __forceinline__ float2 load(const void* p, long long i) {
    return __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(p)[i >> 1]);
  }
  static __device__ __forceinline__ void store(void* p, long long i, float a, float b) {
    reinterpret_cast<__nv_bfloat162*>(p)[i >> 1] = __floats2bfloat162_rn(a, b);
  }
};
template <> struct Pair<float> {
  static __device__ __forceinline__ float2 load(const void* p, long long i) {
    return reinterpret_cast<const float2*>(p)[i >> 1];
  }
  static __device__ __forceinline__ void store(void* p, long long i, float a, float b) {
    reinterpret_cast<float2*>(p)[i >> 1] = make_float2(a, b);
  }
};

template <typename T, int NMAX, bool NOISE>
__global__ void __launch_bounds__(GB_THREADS)
gate_bwd_kernel(GateBwdArgs a) {
  __shared__ float s_dh[GB_TOK][NMAX];
  __shared__ float s_dhn[NOISE ? GB_TOK : 1][NOISE ? NMAX : 1];
  __shared__ float s_f[NMAX];
  const int N = a.N, d = a.d;
  const int c = (blockIdx.x * GB_THREADS + threadIdx.x) * 2;     // first of my two columns
  const bool col_ok = c < d;
  const int t_begin = blockIdx.y * a.tok_per_block;
  const int t_end = min(a.T, t_begin + a.tok_per_block);
  const float inv_tk = 1.0f / ((float)a.T * (float)a.k);
  for (int j = threadIdx.x; j < NMAX; j += GB_THREADS) s_f[j] = j < N ? a.counts[j] * inv_tk : 0.f;
  const float c_aux = a.d_aux ? (*a.d_aux) * (float)N / (float)a.T : 0.f;

  float wg[NMAX][2], wn[NOISE ? NMAX : 1][2];
  float acc[NMAX][2], accn[NOISE ? NMAX : 1][2];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    wg[j][0] = wg[j][1] = 0.f;
    acc[j][0] = acc[j][1] = 0.f;
    if (j < N && col_ok) {
      const float2 v = *reinterpret_cast<const float2*>(a.w_gate_t + (long long)j * d + c);
      wg[j][0] = v.x;
      wg[j][1] = v.y;
    }
    if constexpr (NOISE) {
      wn[j][0] = wn[j][1] = 0.f;
      accn[j][0] = accn[j][1] = 0.f;
      if (j < N && col_ok) {
        const float2 v = *reinterpret_cast<const float2*>(a.w_noise_t + (long long)j * d + c);
        wn[j][0] = v.x;
        wn[j][1] = v.y;
      }
    }
  }
  __syncthreads();

  for (int t0 = t_begin; t0 < t_end; t0 += GB_TOK) {
    const int nt = min(GB_TOK, t_end - t0);
    // the batch's rows of my two columns: all loads in flight before phase 1
    float2 xv[GB_TOK];
#pragma unroll
    for (int i = 0; i < GB_TOK; ++i)
      xv[i] = (col_ok && i < nt) ? Pair<T>::load(a.src, (long long)(t0 + i) * d + c)
                                 : make_float2(0.f, 0.f);
    // ---- phase 1: dH rows of this batch (one thread per token) ----
    if (threadIdx.x < nt) {
      const int t = t0 + threadIdx.x;
      const float* h = a.logits + (long long)t * N;
      float p[NMAX];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) {
        p[j] = j < N ? h[j] : -INFINITY;
        mx = fmaxf(mx, p[j]);
      }
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) {
        p[j] = j < N ? __expf(p[j] - mx) : 0.f;
        s += p[j];
      }
      const float inv = 1.0f / s;
      float fp = 0.f;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) {
        p[j] *= inv;
        fp = fmaf(s_f[j], p[j], fp);
      }
      float dh[NMAX];
#pragma unroll
      for (int j = 0; j < NMAX; ++j) dh[j] = c_aux * p[j] * (s_f[j] - fp);
      if (a.d_weights && a.k > 1) {
        const float* w = a.weights + (long long)t * a.k;
        const float* dw = a.d_weights + (long long)t * a.k;
        const int32_t* ix = a.indices + (long long)t * a.k;
        float sw = 0.f;
        for (int i = 0; i < a.k; ++i) sw = fmaf(w[i], dw[i], sw);
        for (int i = 0; i < a.k; ++i) {
          const float g = w[i] * (dw[i] - sw);
          const int e = ix[i];
#pragma unroll
          for (int j = 0; j < NMAX; ++j)
            if (j == e) dh[j] += g;
        }
      }
#pragma unroll
      for (int j = 0; j < NMAX; ++j) s_dh[threadIdx.x][j] = dh[j];
      if constexpr (NOISE) {
        const float* ep = a.eps + (long long)t * N;
        const float* np = a.noise_pre + (long long)t * N;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
          float v = 0.f;
          if (j < N) v = dh[j] * ep[j] / (1.0f + __expf(-np[j]));   // softplus' = sigmoid
          s_dhn[threadIdx.x][j] = v;
        }
      }
    }
    __syncthreads();
    // ---- phase 2: my two columns of the batch's rows ----
    if (col_ok) {
#pragma unroll
      for (int i = 0; i < GB_TOK; ++i) {
        if (i >= nt) break;
        const long long off = (long long)(t0 + i) * d + c;
        const float2 x = xv[i];
        float o0 = 0.f, o1 = 0.f;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
          const float g = s_dh[i][j];
          o0 = fmaf(g, wg[j][0], o0);
          o1 = fmaf(g, wg[j][1], o1);
          acc[j][0] = fmaf(g, x.x, acc[j][0]);
          acc[j][1] = fmaf(g, x.y, acc[j][1]);
          if constexpr (NOISE) {
            const float gn = s_dhn[i][j];
            o0 = fmaf(gn, wn[j][0], o0);
            o1 = fmaf(gn, wn[j][1], o1);
            accn[j][0] = fmaf(gn, x.x, accn[j][0]);
            accn[j][1] = fmaf(gn, x.y, accn[j][1]);
          }
        }
        if (a.d_src) Pair<T>::store(a.d_src, off, o0, o1);
      }
    }
    __syncthreads();
  }
  if (!col_ok) return;
  const int planes = NOISE ? 2 : 1;
  float* o = a.part + (long long)blockIdx.y * planes * N * d;
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j < N) {
      *reinterpret_cast<float2*>(o + (long long)j * d + c) = make_float2(acc[j][0], acc[j][1]);
      if constexpr (NOISE)
        *reinterpret_cast<float2*>(o + (long long)(N + j) * d + c) =
            make_float2(accn[j][0], accn[j][1]);
    }
  }
}

// out[p][j][c] = sum_b part[b][p][j][c]: block (32 outputs x 32 lanes), lane
// y sums blocks y, y+32, ..., then the lane sums are added in a fixed order
__global__ void gate_bwd_reduce_kernel(const float* __restrict__ part, int n_blocks, long long n,
                                       float* __restrict__ d_wg, float* __restrict__ d_wn,
                                       long long per_plane) {
  __shared__ float red[32][33];
  const long long i = blockIdx.x * 32ll + threadIdx.x;
  float s0 = 0.f, s1 = 0.f;
  if (i < n) {
    int b = threadIdx.y;
    for (; b + 32 < n_blocks; b += 64) {
      s0 += part[(long long)b * n + i];
      s1 += part[(long long)(b + 32) * n + i];
    }
    for (; b < n_blocks; b += 32) s0 += part[(long long)b * n + i];
  }
  red[threadIdx.y][threadIdx.x] = s0 + s1;
  __syncthreads();
  if (threadIdx.y == 0 && i < n) {
    float s = 0.f;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) s += red[y][threadIdx.x];
    if (i < per_plane) d_wg[i] = s;
    else d_wn[i - per_plane] = s;
  }
}

template <typename T, int NMAX>
void launch_gate_bwd(const GateBwdArgs& a, bool noise, dim3 grid, cudaStream_t st) {
  if (noise) gate_bwd_kernel<T, NMAX, true><<<grid, GB_THREADS, 0, st>>>(a);
  else gate_bwd_kernel<T, NMAX, false><<<grid, GB_THREADS, 0, st>>>(a);
}

int gate_bwd_token_blocks(int T, int d) {
  const int col_blocks = (d + 2 * GB_THREADS - 1) / (2 * GB_THREADS);
  int tb = (4 * num_sms() + col_blocks - 1) / col_blocks;        // ~4 blocks per SM
  tb = max(1, min(tb, (T + GB_TOK - 1) / GB_TOK));
  return tb;
}

}  // namespace
}  // namespace scmoe

using namespace scmoe;

extern "C" size_t scmoe_gate_backward_workspace_bytes(int T, int d, int N, int noise) {
  if (T <= 0 || d <= 0 || N <= 0) return 0;
  return (size_t)gate_bwd_token_blocks(T, d) * (noise ? 2 : 1) * N * d * sizeof(float);
}

extern "C" int scmoe_gate_backward(const void* src, int dtype, int T, int d, int N, int k,
                                   const float* logits, const int32_t* indices,
                                   const float* weights, const float* d_weights,
                                   const int32_t* counts, const float* d_aux,
                                   const float* w_gate_t, const float* w_noise_t,
                                   const float* eps, const float* noise_pre, void* d_src,
                                   float* d_w_gate, float* d_w_noise, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  SCMOE_CHECK_ARG(src && logits && counts && w_gate_t && d_w_gate, "gate_backward: null pointer");
  SCMOE_CHECK_ARG(T > 0 && d > 0 && N >= 1 && N <= SCMOE_MAX_EXPERTS && k >= 1 &&
                  k <= SCMOE_MAX_K, "gate_backward: bad shape T=%d d=%d N=%d k=%d", T, d, N, k);
  SCMOE_CHECK_ARG(d % 2 == 0, "gate_backward: d must be even");
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16 || dtype == SCMOE_F32, "gate_backward: bad dtype");
  const bool noise = w_noise_t != nullptr;
  SCMOE_CHECK_ARG(!noise || (eps && noise_pre && d_w_noise),
                  "gate_backward: noise needs eps, noise_pre and d_w_noise");
  SCMOE_CHECK_ARG(!(d_weights && k > 1) || (weights && indices),
                  "gate_backward: d_weights needs weights and indices");
  const size_t need = scmoe_gate_backward_workspace_bytes(T, d, N, noise);
  SCMOE_CHECK_ARG(workspace && workspace_bytes >= need,
                  "gate_backward: workspace %zu < %zu bytes", workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int col_blocks = (d + 2 * GB_THREADS - 1) / (2 * GB_THREADS);
  const int tb = gate_bwd_token_blocks(T, d);
  int per = (T + tb - 1) / tb;
  per = (per + GB_TOK - 1) / GB_TOK * GB_TOK;
  const int tb_used = (T + per - 1) / per;
  GateBwdArgs a{src, T, d, N, k, logits, indices, weights, d_weights, counts, d_aux, w_gate_t,
                w_noise_t, eps, noise_pre, d_src, (float*)workspace, per};
  const dim3 grid(col_blocks, tb_used);
  const bool bf = dtype == SCMOE_BF16;
#define SCMOE_GB(NM)                                                              \
  (bf ? launch_gate_bwd<__nv_bfloat16, NM>(a, noise, grid, st)                   \
      : launch_gate_bwd<float, NM>(a, noise, grid, st))
  if (N <= 8) SCMOE_GB(8);
  else if (N <= 16) SCMOE_GB(16);
  else SCMOE_GB(64);
#undef SCMOE_GB
  SCMOE_LAUNCH_CHECK();
  const long long per_plane = (long long)N * d;
  const long long n = per_plane * (noise ? 2 : 1);
  gate_bwd_reduce_kernel<<<(unsigned)((n + 31) / 32), dim3(32, 32), 0, st>>>(
      (const float*)workspace, tb_used, n, d_w_gate, d_w_noise, per_plane);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}
