// K1 / K1b: gate logits + top-k + capacity slots, one pass over x_src.
//
// Reference semantics (relative to /root/reference/pkg/src/scmoelab/):
//   logits        gating.py:93-107, arch.py:405-415 (noise: eps*softplus(x W_noise))
//   top-k order   gating.py:110-116 (stable argsort of -h: ties -> lowest index)
//   weights       gating.py:119-131 (softmax over the k kept logits)
//   quota/drops   gating.py:134-156 (token-major order; counter advances on keeps)
//   aux stats     gating.py:159-170, arch.py:436-439 (pre-drop counts, mean softmax)
//
// Layout: one CTA handles a tile of TOK tokens.  Phase 1 computes the N logits
// with TPT threads per token (16-byte vector loads, gate-weight chunks staged
// in shared memory and read as broadcasts).  Phase 2 runs the routing with one
// thread per token: per-expert ballots give ranks inside a warp, a shared
// prefix gives ranks inside the tile, and a decoupled look-back over per-tile
// (flag | count) words gives the exclusive count of every earlier tile.  Tile
// ids come from an atomic counter, so a tile only ever waits on tiles that
// were scheduled before it.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace scmoe {
namespace {

constexpr int TOK = 64;        // tokens per CTA
constexpr int TPT = 4;         // threads per token in phase 1
constexpr int THREADS = TOK * TPT;
constexpr int ROUTE_WARPS = TOK / 32;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;
constexpr size_t CTR_BYTES = 256;

__device__ __forceinline__ bool gt_nan_last(float a, float b) {
  // a ranks above b: larger value; NaN ranks below everything (numpy sorts
  // NaN last, so -h NaN entries come after all numbers in the stable argsort).
  return (a > b) || (isnan(b) && !isnan(a));
}

__device__ __forceinline__ float softplus_f(float v) {
  return v > 30.f ? v : log1pf(expf(fminf(v, 30.f)));
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T, int NMAX, bool NOISE>
__global__ void __launch_bounds__(THREADS) gate_topk_kernel(
    const T* __restrict__ x, long long ld_x, const float* __restrict__ wg_t,
    const float* __restrict__ wn_t, const float* __restrict__ eps,
    const int32_t* __restrict__ exclude, int n_tok, int d,
    int N, int k, int quota, int dc_max, float* __restrict__ logits,
    int32_t* __restrict__ indices, float* __restrict__ weights, int32_t* __restrict__ slots,
    uint8_t* __restrict__ dropped, int32_t* __restrict__ counts, float* __restrict__ prob_sum,
    uint32_t* __restrict__ ctrs, uint32_t* __restrict__ status, float* __restrict__ psum,
    int num_tiles) {
  extern __shared__ float4 dyn_smem4[];
  float* wsm = reinterpret_cast<float*>(dyn_smem4);  // [(1+NOISE)][N][dc_max]
  __shared__ float s_logit[TOK][NMAX + 1];
  __shared__ int s_wcnt[ROUTE_WARPS][NMAX];
  __shared__ float s_wprob[ROUTE_WARPS][NMAX];
  __shared__ uint32_t s_excl[NMAX];
  __shared__ uint32_t s_tile;
  __shared__ int s_last;

  constexpr int VEC = Vec16<T>::N;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(&ctrs[0], 1u);
  __syncthreads();
  const int tile = (int)s_tile;

  // ---------------- phase 1: logits --------------------------------------
  const int tok_local = tid / TPT;
  const int sub = tid % TPT;
  const int t1 = tile * TOK + tok_local;
  const bool valid1 = t1 < n_tok;
  const T* xrow = x + (long long)(valid1 ? t1 : 0) * ld_x;
  float acc[NMAX];
  float accn[NOISE ? NMAX : 1];
#pragma unroll
  for (int e = 0; e < NMAX; ++e) acc[e] = 0.f;
#pragma unroll
  for (int e = 0; e < (NOISE ? NMAX : 1); ++e) accn[e] = 0.f;

  // Load blocks of LB columns; each thread keeps MAXV 16-byte loads in flight
  // and prefetches block b+1 while it multiplies block b.  Gate weights are
  // staged in shared memory chunks of dc_max (a multiple of LB) columns.
  constexpr int STEP = VEC * TPT;
  constexpr int MAXV = (NMAX * (NOISE ? 2 : 1) >= 64) ? 4 : 8;  // bounded registers
  constexpr int LB = MAXV * STEP;
  const int nlb = (d + LB - 1) / LB;
  uint4 cur[MAXV], nxt[MAXV];
#pragma unroll
  for (int u = 0; u < MAXV; ++u) {
    const int c = sub * VEC + u * STEP;
    cur[u] = (valid1 && c < d) ? ld_nc_v4(xrow + c) : make_uint4(0, 0, 0, 0);
  }
  int chunk0 = 0;
  for (int lb = 0; lb < nlb; ++lb) {
    const int cb = lb * LB;
    if (cb % dc_max == 0) {
      chunk0 = cb;
      const int dc = min(dc_max, d - cb);
      __syncthreads();
      for (int i = tid * 4; i < N * dc; i += THREADS * 4) {
        // dc is a multiple of 4: a float4 never straddles two experts
        const int e = i / dc, c = i - e * dc;
        *reinterpret_cast<float4*>(wsm + e * dc_max + c) =
            __ldg(reinterpret_cast<const float4*>(wg_t + (long long)e * d + cb + c));
        if (NOISE)
          *reinterpret_cast<float4*>(wsm + (N + e) * dc_max + c) =
              __ldg(reinterpret_cast<const float4*>(wn_t + (long long)e * d + cb + c));
      }
      __syncthreads();
    }
    if (lb + 1 < nlb) {
#pragma unroll
      for (int u = 0; u < MAXV; ++u) {
        const int c = cb + LB + sub * VEC + u * STEP;
        nxt[u] = (valid1 && c < d) ? ld_nc_v4(xrow + c) : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < MAXV; ++u) {
      const int c = cb + sub * VEC + u * STEP;
      if (c < d) {
        Vec16<T> v;
        v.raw = cur[u];
        float xf[VEC];
        v.to_float(xf);
        const int cw = c - chunk0;
#pragma unroll
        for (int e = 0; e < NMAX; ++e) {
          if (e < N) {
            const float4* w4 = reinterpret_cast<const float4*>(wsm + e * dc_max + cw);
#pragma unroll
            for (int q = 0; q < VEC / 4; ++q) {
              const float4 w = w4[q];
              acc[e] = fmaf(xf[4 * q + 0], w.x, acc[e]);
              acc[e] = fmaf(xf[4 * q + 1], w.y, acc[e]);
              acc[e] = fmaf(xf[4 * q + 2], w.z, acc[e]);
              acc[e] = fmaf(xf[4 * q + 3], w.w, acc[e]);
            }
            if (NOISE) {
              const float4* n4 = reinterpret_cast<const float4*>(wsm + (N + e) * dc_max + cw);
#pragma unroll
              for (int q = 0; q < VEC / 4; ++q) {
                const float4 w = n4[q];
                accn[e] = fmaf(xf[4 * q + 0], w.x, accn[e]);
                accn[e] = fmaf(xf[4 * q + 1], w.y, accn[e]);
                accn[e] = fmaf(xf[4 * q + 2], w.z, accn[e]);
                accn[e] = fmaf(xf[4 * q + 3], w.w, accn[e]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < MAXV; ++u) cur[u] = nxt[u];
  }
  // reduce the TPT partial sums of a token (adjacent lanes)
#pragma unroll
  for (int e = 0; e < NMAX; ++e) {
#pragma unroll
    for (int o = 1; o < TPT; o <<= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (NOISE) {
#pragma unroll
      for (int o = 1; o < TPT; o <<= 1) accn[e] += __shfl_xor_sync(0xffffffffu, accn[e], o);
    }
  }
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      if (e < N) {
        float hv = acc[e];
        if (NOISE && valid1) hv += eps[(long long)t1 * N + e] * softplus_f(accn[NOISE ? e : 0]);
        s_logit[tok_local][e] = hv;
      }
    }
  }
  __syncthreads();

  // ---------------- phase 2: routing, one thread per token -----------------
  const int warp = tid >> 5, lane = tid & 31;
  int sel[SCMOE_MAX_K];
  float selv[SCMOE_MAX_K];
  int rank[SCMOE_MAX_K];
  const int t = tile * TOK + tid;
  const bool valid = (tid < TOK) && (t < n_tok);
  if (tid < TOK) {
    float h[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) h[e] = (e < N) ? s_logit[tid][e] : 0.f;
    if (valid) {
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < N) logits[(long long)t * N + e] = h[e];
    }
    // top-k: repeated argmax with strict '>' (lowest index wins ties).  An
    // excluded expert (DGMoE distinct-expert constraint, arch.py:453-457) is
    // skipped, so the pick becomes the runner-up exactly when it would clash.
    uint64_t blocked = 0;
    if (exclude && valid) {
      const int ex = exclude[t];
      if (ex >= 0 && ex < N) blocked = 1ull << ex;
    }
    uint64_t selmask = 0;
#pragma unroll
    for (int j = 0; j < SCMOE_MAX_K; ++j) {
      sel[j] = 0;
      selv[j] = 0.f;
      rank[j] = 0;
      if (j < k) {
        int bi = -1;
        float bv = 0.f;
#pragma unroll
        for (int e = 0; e < NMAX; ++e) {
          if (e < N && !(((selmask | blocked) >> e) & 1ull)) {
            if (bi < 0 || gt_nan_last(h[e], bv)) {
              bi = e;
              bv = h[e];
            }
          }
        }
        sel[j] = bi;
        selv[j] = bv;
        selmask |= 1ull << bi;
      }
    }
    // full-softmax probabilities for the balance-loss mean (arch.py:484-485)
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < NMAX; ++e)
      if (e < N) mx = fmaxf(mx, h[e]);
    float ex[NMAX];
    float den = 0.f;
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      ex[e] = (e < N) ? expf(h[e] - mx) : 0.f;
      den += ex[e];
    }
    const float inv = 1.f / den;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int e = 0; e < NMAX; ++e) {
      if (e < N) {
        const bool mine = valid && ((selmask >> e) & 1ull);
        const unsigned b = __ballot_sync(0xffffffffu, mine);
        const float p = warp_sum(valid ? ex[e] * inv : 0.f);
        if (lane == 0) {
          s_wcnt[warp][e] = __popc(b);
          s_wprob[warp][e] = p;
        }
        if (mine) {
#pragma unroll
          for (int j = 0; j < SCMOE_MAX_K; ++j)
            if (j < k && sel[j] == e) rank[j] = __popc(b & lt);
        }
      }
    }
  }
  __syncthreads();

  // per-expert tile aggregate and within-tile warp offsets; publish the
  // aggregate at once so later tiles can make progress
  if (tid < N) {
    const int e = tid;
    uint32_t run = 0;
    float psum_tile = 0.f;
#pragma unroll
    for (int w = 0; w < ROUTE_WARPS; ++w) {
      const int c = s_wcnt[w][e];
      s_wcnt[w][e] = (int)run;
      run += (uint32_t)c;
      psum_tile += s_wprob[w][e];
    }
    s_excl[e] = run;  // temporarily: this tile's aggregate
    st_volatile_u32(status + (size_t)tile * N + e, (tile == 0 ? FLAG_INC : FLAG_AGG) | run);
    if (run) atomicAdd(&counts[e], (int)run);
    psum[(size_t)tile * N + e] = psum_tile;
    __threadfence();
  }
  __syncthreads();
  // decoupled look-back, one warp per expert, 32 predecessor tiles per step:
  // lane l reads tile (j - l); the nearest INCLUSIVE word ends the walk, every
  // word before it must at least carry its AGGREGATE.  Tiles finish phase 1 at
  // about the same time, so a one-tile-per-step walk would serialise ~T/TOK
  // dependent loads.
  for (int e = warp; e < N; e += THREADS / 32) {
    const uint32_t agg = s_excl[e];
    uint32_t excl = 0;
    if (tile > 0) {
      int j = tile - 1;
      while (true) {
        const int jj = j - lane;
        const uint32_t v = jj >= 0 ? ld_volatile_u32(status + (size_t)jj * N + e) : FLAG_INC;
        const uint32_t f = v & ~VAL_MASK;
        const unsigned inc = __ballot_sync(0xffffffffu, f == FLAG_INC);
        const unsigned not_ready = __ballot_sync(0xffffffffu, f == 0);
        const int first = inc ? __ffs(inc) - 1 : 31;              // last lane that counts
        const unsigned span = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if (not_ready & span) continue;                          // retry the same window
        uint32_t part = (lane <= first) ? (v & VAL_MASK) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (inc) break;
        j -= 32;
      }
      if (lane == 0) st_volatile_u32(status + (size_t)tile * N + e, FLAG_INC | (excl + agg));
    }
    __syncwarp();
    if (lane == 0) s_excl[e] = excl;
  }
  __syncthreads();

  if (valid) {
#pragma unroll
    for (int j = 0; j < SCMOE_MAX_K; ++j) {
      if (j < k) {
        const int e = sel[j];
        const int slot = (int)s_excl[e] + s_wcnt[warp][e] + rank[j];
        const long long o = (long long)t * k + j;
        indices[o] = e;
        slots[o] = slot;
        dropped[o] = slot >= quota ? 1 : 0;
        // softmax over the kept logits, stabilised by the top logit
        float den = 0.f;
#pragma unroll
        for (int q = 0; q < SCMOE_MAX_K; ++q)
          if (q < k) den += expf(selv[q] - selv[0]);
        weights[o] = (k == 1) ? 1.0f : expf(selv[j] - selv[0]) / den;
      }
    }
  }

  // the last tile to finish reduces the per-tile probability sums in order
  if (tid == 0) {
    const uint32_t prev = atomicAdd(&ctrs[1], 1u);
    s_last = (prev == (uint32_t)num_tiles - 1u);
  }
  __syncthreads();
  if (s_last && tid < N) {
    __threadfence();
    float s = 0.f;
    for (int j = 0; j < num_tiles; ++j) s += __ldcg(psum + (size_t)j * N + tid);
    prob_sum[tid] = s;
  }
}

template <typename T, int NMAX>
int launch_gate(const void* x, long long ld_x, const float* wg, const float* wn,
                const float* eps, const int32_t* excl, int T_, int d, int N, int k, int quota,
                float* logits,
                int32_t* idx, float* w, int32_t* slots, uint8_t* drop, int32_t* counts,
                float* prob_sum, uint8_t* ws, cudaStream_t st) {
  const int tiles = (T_ + TOK - 1) / TOK;
  uint32_t* ctrs = reinterpret_cast<uint32_t*>(ws);
  uint32_t* status = reinterpret_cast<uint32_t*>(ws + CTR_BYTES);
  float* psum = reinterpret_cast<float*>(ws + CTR_BYTES + (size_t)tiles * N * 4);
  SCMOE_CUDA_TRY(cudaMemsetAsync(ws, 0, CTR_BYTES + (size_t)tiles * N * 4, st));
  SCMOE_CUDA_TRY(cudaMemsetAsync(counts, 0, (size_t)N * sizeof(int32_t), st));
  const bool noise = wn != nullptr;
  // gate-weight chunk: a multiple of the (largest) load block, the whole row when it
  // fits in 64 KB of shared memory
  constexpr int LB = 8 * Vec16<T>::N * TPT;
  const size_t per_col = (size_t)(noise ? 2 : 1) * N * 4;
  int dc = ((d + LB - 1) / LB) * LB;
  while (dc > LB && per_col * dc > 65536) dc -= LB;
  const size_t smem = per_col * dc;
  // raise the dynamic-smem limit once per instantiation (never inside a
  // CUDA-graph capture of a later call)
  static size_t smem_set[2] = {0, 0};
  if (smem > smem_set[noise ? 1 : 0]) {
    if (noise)
      SCMOE_CUDA_TRY(cudaFuncSetAttribute(gate_topk_kernel<T, NMAX, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    else
      SCMOE_CUDA_TRY(cudaFuncSetAttribute(gate_topk_kernel<T, NMAX, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    smem_set[noise ? 1 : 0] = 160 * 1024;
  }
  if (noise) {
    auto kern = gate_topk_kernel<T, NMAX, true>;
    kern<<<tiles, THREADS, smem, st>>>((const T*)x, ld_x, wg, wn, eps, excl, T_, d, N, k, quota, dc,
                                       logits, idx, w, slots, drop, counts, prob_sum, ctrs,
                                       status, psum, tiles);
  } else {
    auto kern = gate_topk_kernel<T, NMAX, false>;
    kern<<<tiles, THREADS, smem, st>>>((const T*)x, ld_x, wg, wn, eps, excl, T_, d, N, k, quota, dc,
                                       logits, idx, w, slots, drop, counts, prob_sum, ctrs,
                                       status, psum, tiles);
  }
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

template <typename T>
int dispatch_nmax(const void* x, long long ld_x, const float* wg, const float* wn,
                  const float* eps, const int32_t* excl, int T_, int d, int N, int k, int quota,
                  float* logits, int32_t* idx, float* w, int32_t* slots, uint8_t* drop,
                  int32_t* counts, float* prob_sum, uint8_t* ws, cudaStream_t st) {
#define SCMOE_GATE_CASE(NM)                                                                    \
  if (N <= NM)                                                                                 \
    return launch_gate<T, NM>(x, ld_x, wg, wn, eps, excl, T_, d, N, k, quota, logits, idx, w,  \
                              slots, drop, counts, prob_sum, ws, st);
  SCMOE_GATE_CASE(4)
  SCMOE_GATE_CASE(8)
  SCMOE_GATE_CASE(16)
  SCMOE_GATE_CASE(32)
  SCMOE_GATE_CASE(64)
#undef SCMOE_GATE_CASE
  set_error("n_experts=%d exceeds %d", N, SCMOE_MAX_EXPERTS);
  return SCMOE_ERR_ARG;
}

}  // namespace
}  // namespace scmoe

extern "C" size_t scmoe_gate_workspace_bytes(int n_tokens, int n_experts) {
  const size_t tiles = (size_t)((n_tokens + scmoe::TOK - 1) / scmoe::TOK);
  return scmoe::CTR_BYTES + 2 * tiles * (size_t)n_experts * 4;
}

extern "C" int scmoe_gate_topk(const void* x, int x_dtype, long long ld_x,
                               const float* w_gate_t, const float* w_noise_t, const float* eps,
                               const int32_t* exclude,
                               int n_tokens, int d_model, int n_experts, int k, int quota,
                               float* logits, int32_t* indices, float* weights, int32_t* slots,
                               uint8_t* dropped, int32_t* counts, float* prob_sum,
                               void* workspace, size_t workspace_bytes, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(n_tokens >= 1, "n_tokens must be >= 1 (got %d)", n_tokens);
  SCMOE_CHECK_ARG(n_experts >= 1 && n_experts <= SCMOE_MAX_EXPERTS, "n_experts=%d out of [1,%d]",
                  n_experts, SCMOE_MAX_EXPERTS);
  SCMOE_CHECK_ARG(k >= 1 && k <= n_experts && k <= SCMOE_MAX_K, "k=%d out of range for N=%d", k,
                  n_experts);
  SCMOE_CHECK_ARG(quota >= 1, "quota must be >= 1");
  SCMOE_CHECK_ARG(x_dtype == SCMOE_F32 || x_dtype == SCMOE_BF16, "bad dtype %d", x_dtype);
  const int vec = x_dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0 && ld_x % vec == 0,
                  "d_model and ld_x must be multiples of %d", vec);
  SCMOE_CHECK_ARG(((uintptr_t)x & 15) == 0, "x must be 16-byte aligned");
  SCMOE_CHECK_ARG((w_noise_t == nullptr) == (eps == nullptr), "w_noise and eps go together");
  SCMOE_CHECK_ARG(!exclude || k < n_experts, "an excluded expert needs k < n_experts");
  SCMOE_CHECK_ARG(workspace_bytes >= scmoe_gate_workspace_bytes(n_tokens, n_experts),
                  "gate workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  if (x_dtype == SCMOE_BF16)
    return dispatch_nmax<__nv_bfloat16>(x, ld_x, w_gate_t, w_noise_t, eps, exclude, n_tokens,
                                        d_model, n_experts, k, quota, logits, indices, weights,
                                        slots, dropped, counts, prob_sum, ws, st);
  return dispatch_nmax<float>(x, ld_x, w_gate_t, w_noise_t, eps, exclude, n_tokens, d_model,
                              n_experts, k, quota, logits, indices, weights, slots, dropped,
                              counts, prob_sum, ws, st);
}
