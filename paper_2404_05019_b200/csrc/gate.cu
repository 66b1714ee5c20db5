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

#include <cuda.h>

#include "common.cuh"

namespace scmoe {

int make_map_2d(CUtensorMap* map, const void* base, int inner, int outer,
                long long row_stride_bytes, int box_outer);   // gemm_sm100.cu

namespace {

constexpr int TOK = 64;        // tokens per CTA
constexpr int TPT = 4;         // threads per token in phase 1
constexpr int THREADS = TOK * TPT;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;
constexpr size_t CTR_BYTES = 256;

// workspace = [counters | per-tile status (or tile counts) | per-tile prob partials]
// (per-tile rows for the FMA kernel's 64-token tiles; per-CTA rows for the
// tensor-core kernel, at most one per 16 tokens and at most 1024 CTAs)
__host__ __device__ inline size_t gate_ws_bytes(int n_tok, int n_exp) {
  const size_t t64 = (size_t)((n_tok + 63) / 64), t16 = (size_t)((n_tok + 15) / 16);
  const size_t tiles = t64 > (t16 < 1024 ? t16 : 1024) ? t64 : (t16 < 1024 ? t16 : 1024);
  return (CTR_BYTES + 2 * tiles * (size_t)n_exp * 4 + 15) & ~(size_t)15;
}

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

// Barrier over the first NTHR threads of the CTA (the routing threads; the
// tensor-core kernel's producer warp does not take part).
template <int NTHR, int BAR = 1>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTHR) : "memory");
}

// Debug timeline (build with -DSCMOE_GATE_TRACE): %globaltimer per CTA at
// entry, first stage landed, last tile published, grid-wide wait done, exit.
#ifdef SCMOE_GATE_TRACE
__device__ unsigned long long g_gate_trace[1024][20];
__device__ unsigned long long g_gate_stages[1024][32];   // stage it landed (consumer warp 0)
__device__ __forceinline__ void gate_trace_stage(uint32_t it) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 1024 && it < 32) g_gate_stages[blockIdx.x][it] = t;
}
__device__ __forceinline__ void gate_trace(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 1024) g_gate_trace[blockIdx.x][i] = t;   // last write wins (last tile)
}
#else
__device__ __forceinline__ void gate_trace(int) {}
__device__ __forceinline__ void gate_trace_stage(uint32_t) {}
#endif

// Phase 2, shared by both logit kernels, in two halves so the tensor-core
// kernel can run the look-back of tile i after the logits of tile i+1:
//   route_publish — one thread per token: top-k (strict '>', lowest index
//     wins ties), weights, full-softmax partials, per-expert ballots -> ranks
//     inside the tile; publishes the tile's per-expert AGGREGATE at once;
//   route_finish  — decoupled look-back over the (flag | count) words of the
//     earlier tiles -> exclusive count = capacity slot base; slots / drops;
//     the last tile reduces the per-tile probability partials in a fixed order.
template <int NMAX, int TOK_>
struct RouteState {            // survives between publish and finish (shared memory)
  int tile;
  uint32_t agg[NMAX];
  int8_t sel[TOK_][SCMOE_MAX_K];
  int32_t lr[TOK_][SCMOE_MAX_K];   // rank of the selection inside its tile
};

// LOCAL = true (tensor-core gate): a sub-tile of `nv` tokens from t0 inside
// the CTA's contiguous token range, no look-back at all — every selection's
// rank relative to the CTA's first token (the CTA's running per-expert count
// `cta_run` + the rank inside the sub-tile) goes to lcache[(lc_off + i) * k
// + j] (or to `slots` when lcache is null); the softmax partials accumulate
// into cta_ps; the kernel's tail adds the prefix over earlier CTAs.
template <int NMAX, int TOK_, int THREADS_, int BASE = 0, int BAR = 1, bool LOCAL = false>
__device__ __forceinline__ void route_publish(
    const float (*s_logit)[NMAX + 1], RouteState<NMAX, TOK_>& rs, int tile,
    const int32_t* __restrict__ exclude, int n_tok, int N, int k, float* __restrict__ logits,
    int32_t* __restrict__ indices, float* __restrict__ weights, int32_t* __restrict__ counts,
    uint32_t* __restrict__ status, float* __restrict__ psum, int32_t* __restrict__ slots = nullptr,
    uint32_t* lcache = nullptr, long long t0 = 0, int nv = 0, uint32_t* cta_run = nullptr,
    float* cta_ps = nullptr, int lc_off = 0) {
  constexpr int RW = TOK_ / 32;
  __shared__ int s_wcnt[RW][NMAX];
  __shared__ float s_wprob[RW][NMAX];
  const int tid = (int)threadIdx.x - BASE;
  const int warp = tid >> 5, lane = tid & 31;
  int sel[SCMOE_MAX_K];
  int rank[SCMOE_MAX_K];
  const long long t = LOCAL ? t0 + tid : (long long)tile * TOK_ + tid;
  const bool valid = (tid < TOK_) && (LOCAL ? tid < nv : t < n_tok);
  // SPLIT (tensor-core gate, <= 16 experts, >= 2 threads per token): a
  // second thread per token (tid - TOK_) writes the logits and computes the
  // full-softmax probability sums while the first runs top-k, ballots and
  // ranks — the per-token routing of a CTA's last tile is exposed latency
  // (gate trace).  Same arithmetic and summation order: bit-identical.
  constexpr bool SPLIT = LOCAL && NMAX <= 16 && THREADS_ >= 2 * TOK_;
  if (SPLIT && tid >= TOK_ && tid < 2 * TOK_) {
    const int tok = tid - TOK_;
    const long long tb = t0 + tok;
    const bool vb = tok < nv;
    float h[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) h[e] = (e < N) ? s_logit[tok][e] : 0.f;
    if (vb) {
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < N) logits[(long long)tb * N + e] = h[e];
    }
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
    float pv[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) pv[e] = (vb && e < N) ? ex[e] * inv : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int e = 0; e < NMAX; ++e) pv[e] += __shfl_xor_sync(0xffffffffu, pv[e], o);
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < N) s_wprob[tok >> 5][e] = pv[e];
    }
  }
  if (tid < TOK_) {
    float h[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) h[e] = (e < N) ? s_logit[tid][e] : 0.f;
    if (LOCAL && tid == 0) gate_trace(14);
    if (!SPLIT && valid) {
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < N) logits[(long long)t * N + e] = h[e];
    }
    if (LOCAL && tid == 0) gate_trace(15);
    // top-k: repeated argmax with strict '>' (lowest index wins ties).  An
    // excluded expert (DGMoE distinct-expert constraint, arch.py:453-457) is
    // skipped, so the pick becomes the runner-up exactly when it would clash.
    uint64_t blocked = 0;
    if (exclude && valid) {
      const int ex = exclude[t];
      if (ex >= 0 && ex < N) blocked = 1ull << ex;
    }
    uint64_t selmask = 0;
    float selv[SCMOE_MAX_K];
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
    if (valid && k == 1) {          // top-1: the kept-logit softmax is exactly 1
      indices[t] = sel[0];
      weights[t] = 1.0f;
    } else if (valid) {
#pragma unroll
      for (int j = 0; j < SCMOE_MAX_K; ++j) {
        if (j < k) {
          const long long o = (long long)t * k + j;
          indices[o] = sel[j];
          // softmax over the kept logits, stabilised by the top logit
          float den = 0.f;
#pragma unroll
          for (int q = 0; q < SCMOE_MAX_K; ++q)
            if (q < k) den += expf(selv[q] - selv[0]);
          weights[o] = (k == 1) ? 1.0f : expf(selv[j] - selv[0]) / den;
        }
      }
    }
    if (LOCAL && tid == 0) gate_trace(16);
    // full-softmax probabilities for the balance-loss mean (arch.py:484-485)
    // (SPLIT: computed by the token's second thread above)
    float mx = -INFINITY;
    float ex[NMAX];
    float den = 0.f;
    if constexpr (!SPLIT) {
#pragma unroll
      for (int e = 0; e < NMAX; ++e)
        if (e < N) mx = fmaxf(mx, h[e]);
#pragma unroll
      for (int e = 0; e < NMAX; ++e) {
        ex[e] = (e < N) ? expf(h[e] - mx) : 0.f;
        den += ex[e];
      }
    }
    const float inv = SPLIT ? 0.f : 1.f / den;
    if (LOCAL && tid == 0) gate_trace(17);
    const unsigned lt = (1u << lane) - 1u;
    if constexpr (NMAX <= 16) {
      // all experts' ballots first, then their warp sums as one interleaved
      // butterfly (same xor order as warp_sum: bit-identical) — one expert at
      // a time was ~1.4 us of dependent shuffles per tile (gate trace)
      unsigned bal[NMAX];
      float pv[NMAX];
#pragma unroll
      for (int e = 0; e < NMAX; ++e) {
        bal[e] = __ballot_sync(0xffffffffu, valid && e < N && ((selmask >> e) & 1ull));
        if constexpr (!SPLIT) pv[e] = (valid && e < N) ? ex[e] * inv : 0.f;
      }
      if constexpr (!SPLIT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int e = 0; e < NMAX; ++e) pv[e] += __shfl_xor_sync(0xffffffffu, pv[e], o);
      }
#pragma unroll
      for (int e = 0; e < NMAX; ++e) {
        if (e < N) {
          if (lane == 0) {
            s_wcnt[warp][e] = __popc(bal[e]);
            if constexpr (!SPLIT) s_wprob[warp][e] = pv[e];
          }
          if (valid && ((selmask >> e) & 1ull)) {
#pragma unroll
            for (int j = 0; j < SCMOE_MAX_K; ++j)
              if (j < k && sel[j] == e) rank[j] = __popc(bal[e] & lt);
          }
        }
      }
    } else {
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
  }
  if (LOCAL && tid == 0) gate_trace(10);
  consumer_sync<THREADS_, BAR>();
  if (LOCAL && tid == 0) gate_trace(11);

  // per-expert tile aggregate and within-tile warp offsets; publish the
  // aggregate at once so later tiles can make progress
  if (tid < N) {
    const int e = tid;
    uint32_t run = LOCAL ? cta_run[e] : 0u;
    float psum_tile = 0.f;
#pragma unroll
    for (int w = 0; w < RW; ++w) {
      const int c = s_wcnt[w][e];
      s_wcnt[w][e] = (int)run;
      run += (uint32_t)c;
      psum_tile += s_wprob[w][e];
    }
    if (LOCAL) {
      cta_run[e] = run;
      cta_ps[e] += psum_tile;
    } else {
      psum[(size_t)tile * N + e] = psum_tile;
      rs.agg[e] = run;
      st_volatile_u32(status + (size_t)tile * N + e, (tile == 0 ? FLAG_INC : FLAG_AGG) | run);
      if (run) atomicAdd(&counts[e], (int)run);
      __threadfence();
    }
  }
  if (!LOCAL && tid == 0) rs.tile = tile;
  if (LOCAL && tid == 0) gate_trace(12);
  consumer_sync<THREADS_, BAR>();
  if (LOCAL && tid == 0) gate_trace(13);
  if (valid) {
#pragma unroll
    for (int j = 0; j < SCMOE_MAX_K; ++j) {
      if (j < k) {
        const int lr = s_wcnt[warp][sel[j]] + rank[j];
        if (LOCAL) {
          if (lcache) lcache[(lc_off + tid) * k + j] = ((uint32_t)sel[j] << 16) | (uint32_t)lr;
          else slots[t * k + j] = lr;
        } else {
          rs.sel[tid][j] = (int8_t)sel[j];
          rs.lr[tid][j] = lr;
        }
      }
    }
  }
}

template <int NMAX, int TOK_, int THREADS_, int BASE = 0, int BAR = 1>
__device__ __forceinline__ void route_finish(
    RouteState<NMAX, TOK_>& rs, int n_tok, int N, int k, int quota, int32_t* __restrict__ slots,
    uint8_t* __restrict__ dropped, float* __restrict__ prob_sum, uint32_t* __restrict__ ctrs,
    uint32_t* __restrict__ status, const float* __restrict__ psum, int num_tiles) {
  __shared__ uint32_t s_excl[NMAX];
  __shared__ int s_last;
  const int tid = (int)threadIdx.x - BASE;
  const int warp = tid >> 5, lane = tid & 31;
  consumer_sync<THREADS_, BAR>();     // publish's shared state is complete
  const int tile = rs.tile;
  // decoupled look-back, one warp per expert, 32 predecessor tiles per step:
  // lane l reads tile (j - l); the nearest INCLUSIVE word ends the walk, every
  // word before it must at least carry its AGGREGATE.  Tiles finish phase 1 at
  // about the same time, so a one-tile-per-step walk would serialise ~T/TOK
  // dependent loads.
  for (int e = warp; e < N; e += THREADS_ / 32) {
    const uint32_t agg = rs.agg[e];
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
  consumer_sync<THREADS_, BAR>();

  const int t = tile * TOK_ + tid;
  if (tid < TOK_ && t < n_tok) {
#pragma unroll
    for (int j = 0; j < SCMOE_MAX_K; ++j) {
      if (j < k) {
        const int slot = (int)s_excl[rs.sel[tid][j]] + rs.lr[tid][j];
        const long long o = (long long)t * k + j;
        slots[o] = slot;
        dropped[o] = slot >= quota ? 1 : 0;
      }
    }
  }

  // the last tile to finish reduces the per-tile probability sums
  if (tid == 0) {
    const uint32_t prev = atomicAdd(&ctrs[1], 1u);
    s_last = (prev == (uint32_t)num_tiles - 1u);
  }
  consumer_sync<THREADS_, BAR>();
  if (s_last) {
    // all THREADS_ threads: thread (e, p) sums tiles p, p + P, ... (independent
    // loads in flight), then the P partials are added in order — a fixed
    // summation order, so prob_sum is deterministic
    constexpr int P = THREADS_ / NMAX;
    __shared__ float s_red[P][NMAX];
    __threadfence();
    const int e = tid % NMAX, p = tid / NMAX;
    if (p < P) {
      float s = 0.f;
      if (e < N)
        for (int j = p; j < num_tiles; j += P) s += __ldcg(psum + (size_t)j * N + e);
      s_red[p][e] = s;
    }
    consumer_sync<THREADS_, BAR>();
    if (tid < N) {
      float s = 0.f;
#pragma unroll 1
      for (int q = 0; q < P; ++q) s += s_red[q][tid];
      prob_sum[tid] = s;
    }
  }
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
  __shared__ uint32_t s_tile;

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

  __shared__ RouteState<NMAX, TOK> rs;
  route_publish<NMAX, TOK, THREADS>(s_logit, rs, tile, exclude, n_tok, N, k, logits, indices,
                                    weights, counts, status, psum);
  route_finish<NMAX, TOK, THREADS>(rs, n_tok, N, k, quota, slots, dropped, prob_sum, ctrs, status,
                                   psum, num_tiles);
}

// ---------------------------------------------------------------------------
// K1 tensor-core variant (bf16 tokens, no noise, N <= 16, d >= 64).
//
// Logits run on mma.sync.m16n8k16 (bf16 x bf16 -> fp32).  The fp32 gate
// weights are split into three bf16 parts w = w0 + w1 + w2 (8 + 8 +
// 8 mantissa bits: the whole fp32 mantissa), each multiplied exactly, so the
// logits keep fp32-level accuracy while the FMA pipe no longer bounds the pass
// over x.
//
// Persistent and warp-specialised, one CTA per SM.  CTA c owns a contiguous,
// balanced range of 16-token row tiles (ceil(T/16) split over the grid to
// within one row tile; whole 64-token tiles left 40 of 148 SMs idle for the
// second half of the stream at configs[2]), walked in sub-tiles of <= 4 row
// tiles.  No cross-CTA dependency while streaming; the tail adds the
// capacity-slot prefix over the earlier CTAs.
//   producer warp  — per stage and sub-tile, (KC/64) x (row tiles) TMA boxes of
//                    16 rows x 64 columns (cp.async.bulk.tensor.2d, 128B
//                    swizzle, OOB rows/columns zero-filled; a 2 KB box is the
//                    same swizzle image as a slice of a 64-row box), plus the
//                    matching slice of the split-weight blob
//                    (gate_split_weights_kernel; one 1-D bulk copy), completion
//                    on the stage's "full" mbarrier.  Per-row 1-D copies of x
//                    were measured issue-bound (~1.8 TB/s at 512 B per copy);
//                    boxes are not.  (A shared-memory-resident blob with one
//                    stage fewer was measured slower: the stream is bound by
//                    bytes in flight, not by the blob's L2 reads);
//   8 MMA warps    — warp w takes m16 tile w%4 and half w/4 of the stage's k16
//                    steps: ldmatrix.x4 A fragments, B fragments as 8-byte
//                    shared loads, one accumulator chain per weight part; the two
//                    halves' partial logits are summed in a fixed order into a
//                    double-buffered logits tile;
//   4 routing warps — route_publish(LOCAL) per sub-tile (top-k, weights,
//                    CTA-local ranks, CTA per-expert counts, softmax partials),
//                    off the MMA warps' critical path; after the last sub-tile
//                    one (N-word) table row per CTA, a grid-wide count of
//                    published rows, and the prefix over earlier CTAs' rows.
constexpr int GT_KC = 256;                       // columns per stage (4 TMA boxes)
constexpr int GT_BOXB = TOK * 128;               // one 64-col x TOK-row box, 128B swizzle
constexpr int GT_XB = (GT_KC / 64) * GT_BOXB;    // x part of a stage
constexpr int GT_GROUP_B = 3072;                 // split-weight blob bytes per 64 columns per n8 tile
constexpr int GT_CONSUMERS = 8;                  // MMA warps 0..7
constexpr int GT_PRODUCER = GT_CONSUMERS;        // warp 8
constexpr int GT_ROUTERS = 4;                    // routing warps 9..12
constexpr int GT_ROUTE_BASE = (GT_CONSUMERS + 1) * 32;
constexpr int GT_THREADS = (GT_CONSUMERS + 1 + GT_ROUTERS) * 32;

template <int NT> struct GateTC {
  static constexpr int STAGES = NT == 1 ? 4 : 3;
  static constexpr int BLOBB = (GT_KC / 64) * GT_GROUP_B * NT;
  static constexpr int STAGEB = GT_XB + BLOBB;
  static constexpr int SMEM = STAGES * STAGEB + 1024;   // + alignment slack (swizzle atoms)
  static_assert(STAGEB % 1024 == 0, "stages must stay 1024-byte aligned");
};

__device__ __forceinline__ void mma_bf16_16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}

// Split fp32 gate weights (N, d) into the blob the tensor-core kernel stages:
// per 64-column group [nt][part 3][k16 step 4][lane 32] x uint2, lane
// (g = lane/4, c = lane%4) of step s holding the mma B fragment
//   (w[n][k0+2c], w[n][k0+2c+1]), (w[n][k0+2c+8], w[n][k0+2c+9]),
// n = nt*8 + g, k0 = 64*group + 16*s.  Experts >= N and columns >= d are zero.
// (Splitting on the fly inside the MMA warps was measured ~1.5x slower.)
template <int NT>
__global__ void gate_split_weights_kernel(const float* __restrict__ wg_t, int d, int N, int ngrp,
                                          uint2* __restrict__ blob) {
  const int total = ngrp * NT * 4 * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ln = i & 31, st = (i >> 5) & 3, rest = i >> 7;
    const int nt = rest % NT, gg = rest / NT;
    const int n = nt * 8 + (ln >> 2);
    const int k0 = gg * 64 + st * 16 + 2 * (ln & 3);
    float w[4] = {0.f, 0.f, 0.f, 0.f};
    if (n < N) {     // d % 8 == 0: pairs (k0, k0+1) and (k0+8, k0+9) are all-in or all-out
      const float* row = wg_t + (long long)n * d;
      if (k0 < d) {
        w[0] = row[k0];
        w[1] = row[k0 + 1];
      }
      if (k0 + 8 < d) {
        w[2] = row[k0 + 8];
        w[3] = row[k0 + 9];
      }
    }
    __nv_bfloat16 p[3][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      p[0][q] = __float2bfloat16_rn(w[q]);
      const float r1 = w[q] - __bfloat162float(p[0][q]);
      p[1][q] = __float2bfloat16_rn(r1);
      p[2][q] = __float2bfloat16_rn(r1 - __bfloat162float(p[1][q]));
    }
#pragma unroll
    for (int part = 0; part < 3; ++part)
      blob[(((size_t)(gg * NT + nt) * 3 + part) * 4 + st) * 32 + ln] =
          make_uint2(pack_bf16(p[part][0], p[part][1]), pack_bf16(p[part][2], p[part][3]));
  }
}


template <int NT>
__global__ void __launch_bounds__(GT_THREADS, 1) gate_topk_tc_kernel(
    const __grid_constant__ CUtensorMap xmap, const uint8_t* __restrict__ blob,
    const int32_t* __restrict__ exclude, int n_tok, int d, int N, int k, int quota,
    float* __restrict__ logits, int32_t* __restrict__ indices, float* __restrict__ weights,
    int32_t* __restrict__ slots, uint8_t* __restrict__ dropped, int32_t* __restrict__ counts,
    float* __restrict__ prob_sum, uint32_t* __restrict__ ctrs, uint32_t* __restrict__ cta_cnt,
    float* __restrict__ cta_psum, int n16) {
  using C = GateTC<NT>;
  constexpr int NMAX = NT * 8;
  constexpr int S = C::STAGES;
  extern __shared__ __align__(128) uint8_t gsm_raw[];
  uint8_t* gsm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
  __shared__ float s_logit[2][TOK][NMAX + 1];     // MMA warps -> routing warps
  __shared__ float s_part[2][TOK][NMAX + 1];
  __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S], lfull_bar[2], lempty_bar[2];
  __shared__ int s_stage_row[S], s_stage_m16[S], s_logit_row[2], s_logit_nv[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = (d + GT_KC - 1) / GT_KC;
  // this CTA's contiguous range of 16-token row tiles (balanced to within one
  // tile: whole 64-token tiles left 40 of 148 SMs idle for the second half of
  // the stream at configs[2])
  const int m16_lo = (int)((long long)blockIdx.x * n16 / gridDim.x);
  const int m16_hi = (int)((long long)(blockIdx.x + 1) * n16 / gridDim.x);
  const int cta_t0 = m16_lo * 16;
  if (tid == 0) {
    gate_trace(0);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], GT_CONSUMERS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&lfull_bar[i], GT_CONSUMERS);
      mbar_init(&lempty_bar[i], GT_ROUTERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp > GT_PRODUCER) {
    // ---------------- routing warps ----------------
    // per sub-tile: top-k, weights, ranks relative to the CTA's first token
    // (CTA running counts, no cross-CTA dependency); after the CTA's last
    // sub-tile it publishes its per-expert totals, waits for every CTA's
    // (safe: the grid is persistent and resident, and no CTA waits on the
    // one waiting), and adds the prefix over the earlier CTAs — no second
    // launch, one (N-word) table row per CTA
    __shared__ RouteState<NMAX, TOK> rs;
    constexpr int RT = GT_ROUTERS * 32;
    constexpr int LCACHE = 2048;           // (expert, CTA-local rank) words
    __shared__ uint32_t s_lcache[LCACHE];
    __shared__ uint32_t s_run[NMAX];
    __shared__ float s_ps[NMAX];
    const int rtid = tid - GT_ROUTE_BASE;
    const int cta_tok = min(m16_hi * 16, n_tok) - cta_t0;
    const bool cached = (long long)cta_tok * k <= LCACHE;
    if (rtid < NMAX) {
      s_run[rtid] = 0;
      s_ps[rtid] = 0.f;
    }
    consumer_sync<RT, 2>();
    for (uint32_t n = 0;; ++n) {
      const int b = n & 1;
      mbar_wait(&lfull_bar[b], (n >> 1) & 1);
      const int row0 = s_logit_row[b];
      if (row0 < 0) break;
      const int nv = s_logit_nv[b];
      if (rtid == 0) gate_trace(5);
      route_publish<NMAX, TOK, RT, GT_ROUTE_BASE, 2, true>(
          s_logit[b], rs, 0, exclude, n_tok, N, k, logits, indices, weights, counts, nullptr,
          nullptr, slots, cached ? s_lcache : nullptr, row0, nv, s_run, s_ps, row0 - cta_t0);
      __syncwarp();
      if (rtid == 0) gate_trace(6);
      if (lane == 0) mbar_arrive(&lempty_bar[b]);   // publish read s_logit[b] before its barrier
      consumer_sync<RT, 2>();
    }
    // this CTA's totals -> its table row; every router thread's writes ->
    // CTA barrier -> one release add (cumulative): no per-thread fence
    if (rtid < N) {
      cta_cnt[(size_t)blockIdx.x * N + rtid] = s_run[rtid];
      cta_psum[(size_t)blockIdx.x * N + rtid] = s_ps[rtid];
    }
    consumer_sync<RT, 2>();
    if (rtid == 0) {
      gate_trace(2);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctrs + 2) : "memory");
      const long long t0 = clock64();
      while (ld_acquire_gpu(ctrs + 2) < gridDim.x) {
        __nanosleep(64);
        if (clock64() - t0 > (40LL << 30)) __trap();   // ~20 s: never hang the GPU
      }
      // the last CTA past the wait leaves both words zero for the next launch
      // (a caller-kept sync state then needs no memset node per launch)
      if (atomicAdd(ctrs + 3, 1u) == gridDim.x - 1) {
        atomicExch(ctrs + 2, 0u);
        atomicExch(ctrs + 3, 0u);
      }
      gate_trace(3);
    }
    consumer_sync<RT, 2>();
    // exclusive prefix over the earlier CTAs: thread (e, p) sums CTAs p, p+P,
    // ... (independent loads in flight), the P partials added in order; the
    // last CTA also forms the totals and the softmax mean (fixed order:
    // deterministic)
    constexpr int P = RT / NMAX;
    __shared__ uint32_t s_red[P][NMAX];
    __shared__ float s_fred[P][NMAX];
    __shared__ uint32_t s_base[NMAX];
    const bool last = blockIdx.x == gridDim.x - 1;
    const int e = rtid % NMAX, p = rtid / NMAX;
    {
      uint32_t acc = 0;
      float ps = 0.f;
      if (e < N) {
        const int lim = last ? (int)gridDim.x : (int)blockIdx.x;
        // every row of a batch loaded before any is added: one round trip per
        // 16 rows (148 CTAs: one batch at N <= 8, two at N <= 16) instead of
        // one per 4; the additions keep the rows' order (deterministic)
        constexpr int BATCH = 16;
        for (int c0 = p; c0 < lim; c0 += BATCH * P) {
          uint32_t v[BATCH];
          float f[BATCH];
#pragma unroll
          for (int i = 0; i < BATCH; ++i) {
            const int c2 = c0 + i * P;
            v[i] = (c2 < lim && c2 < (int)blockIdx.x) ? __ldcg(cta_cnt + (size_t)c2 * N + e) : 0u;
            f[i] = (last && c2 < lim) ? __ldcg(cta_psum + (size_t)c2 * N + e) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < BATCH; ++i) {
            acc += v[i];
            if (last && c0 + i * P < lim) ps += f[i];
          }
        }
      }
      s_red[p][e] = acc;
      s_fred[p][e] = ps;
    }
    consumer_sync<RT, 2>();
    if (rtid < NMAX) {
      uint32_t base = 0;
      float fs = 0.f;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        base += s_red[q][rtid];
        fs += s_fred[q][rtid];
      }
      s_base[rtid] = base;
      if (last && rtid < N) {
        counts[rtid] = (int)(base + s_run[rtid]);
        prob_sum[rtid] = fs;
      }
    }
    consumer_sync<RT, 2>();
    for (int i = rtid; i < cta_tok * k; i += RT) {
      const long long o = (long long)cta_t0 * k + i;
      int slot;
      if (cached) {
        const uint32_t v = s_lcache[i];
        slot = (int)s_base[v >> 16] + (int)(v & 0xffffu);
      } else {
        slot = (int)s_base[indices[o]] + slots[o];
      }
      slots[o] = slot;
      dropped[o] = slot >= quota ? 1 : 0;
    }
    if (rtid == 0) gate_trace(4);
    return;
  }

  if (warp == GT_PRODUCER) {
    // ---------------- producer warp ----------------
    // sub-tiles of up to 4 row tiles (64 tokens) of this CTA's range; per
    // stage 16-row x 64-column boxes (2 KB, 1024-aligned: the same 128B-swizzle
    // image as one 64-row box)
    uint32_t it = 0;
    for (int m = m16_lo;; m += 4) {
      const bool live = m < m16_hi;
      const int m16 = live ? min(4, m16_hi - m) : 0;
      for (int kc = 0; kc < (live ? nkc : 1); ++kc, ++it) {
        const int s = it % S;
        mbar_wait(&empty_bar[s], ((it / S) & 1) ^ 1);
        if (!live) {
          if (lane == 0) {
            s_stage_row[s] = -1;
            mbar_arrive(&full_bar[s]);
          }
          break;
        }
        const int c0 = kc * GT_KC;
        const int nbox = (min(GT_KC, d - c0) + 63) / 64;
        const uint32_t blobb = (uint32_t)nbox * GT_GROUP_B * NT;
        uint8_t* st = gsm + (size_t)s * C::STAGEB;
        if (lane == 0) {
          s_stage_row[s] = m * 16;
          s_stage_m16[s] = m16;
          mbar_expect_tx(&full_bar[s], (uint32_t)(nbox * m16) * 2048u + blobb);
          bulk_g2s(st + GT_XB, blob + (size_t)(c0 / 64) * GT_GROUP_B * NT, blobb, &full_bar[s]);
        }
        __syncwarp();
        // one box per lane: lane = b * 4 + r (b < nbox, r < m16)
        if (lane < nbox * 4 && (lane & 3) < m16) {
          const int bx = lane >> 2, r = lane & 3;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
              "[%0], [%1, {%2, %3}], [%4];"
              ::"r"(smem_u32(st + bx * GT_BOXB + r * 2048)), "l"(&xmap), "r"(c0 + 64 * bx),
                "r"(m * 16 + 16 * r), "r"(smem_u32(&full_bar[s]))
              : "memory");
        }
        __syncwarp();
      }
      if (!live) break;
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int mt = warp & 3, kh = warp >> 2;
  const int g = lane >> 2, c = lane & 3;
  // ldmatrix.x4 lane address: matrices (rows 0-7 | 8-15) x (k 0-7 | 8-15);
  // 128B swizzle: 16-byte chunk q of box row r sits at chunk q ^ (r % 8)
  const int lrow = mt * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
  const int lhi = lane >> 4;
  uint32_t it = 0;
  for (uint32_t n = 0;; ++n) {
    float acc[3][NT][4];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][nt][q] = 0.f;
    int row0 = -1, m16 = 0;
    for (int kc = 0; kc < nkc; ++kc, ++it) {
      const int s = it % S;
      mbar_wait(&full_bar[s], (it / S) & 1);
      if (it == 0 && tid == 0) gate_trace(1);
      if (tid == 0) gate_trace_stage(it);
      row0 = s_stage_row[s];
      if (row0 < 0) break;
      m16 = s_stage_m16[s];
      if (mt < m16) {
        const uint8_t* st = gsm + (size_t)s * C::STAGEB;
        const int nsteps = (min(GT_KC, d - kc * GT_KC) + 63) / 64 * 4;
        const int half = nsteps / 2;                       // whole boxes: a multiple of 4
        const uint32_t abase = smem_u32(st) + lrow * 128;
        const uint2* bl = reinterpret_cast<const uint2*>(st + GT_XB);
        for (int j = kh * half; j < (kh + 1) * half; ++j) {
          uint32_t a[4];
          const int q = ((j & 3) * 2 + lhi) ^ (lrow & 7);
          ldmatrix_x4(a, abase + (j >> 2) * GT_BOXB + q * 16);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const uint2 b = bl[((((j >> 2) * NT + nt) * 3 + p) * 4 + (j & 3)) * 32 + lane];
              mma_bf16_16816(acc[p][nt], a[0], a[1], a[2], a[3], b.x, b.y);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    const int b = n & 1;
    if (tid == 0 && row0 >= 0) gate_trace(7);
    mbar_wait(&lempty_bar[b], ((n >> 1) & 1) ^ 1);      // routing done with buffer b
    if (tid == 0 && row0 >= 0) gate_trace(8);
    if (row0 >= 0) {
      // partial logits, smallest weight part first; C fragment rows g / g+8,
      // experts nt*8 + 2c + {0,1}
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int e = nt * 8 + 2 * c;
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (acc[2][nt][q] + acc[1][nt][q]) + acc[0][nt][q];
        s_part[kh][mt * 16 + g][e] = v[0];
        s_part[kh][mt * 16 + g][e + 1] = v[1];
        s_part[kh][mt * 16 + g + 8][e] = v[2];
        s_part[kh][mt * 16 + g + 8][e + 1] = v[3];
      }
      consumer_sync<GT_CONSUMERS * 32>();
      for (int i = tid; i < m16 * 16 * NMAX; i += GT_CONSUMERS * 32) {
        const int t = i / NMAX, e = i % NMAX;
        s_logit[b][t][e] = s_part[0][t][e] + s_part[1][t][e];
      }
    }
    if (tid == 0) {
      s_logit_row[b] = row0;
      s_logit_nv[b] = row0 >= 0 ? min(m16 * 16, n_tok - row0) : 0;
    }
    consumer_sync<GT_CONSUMERS * 32>();   // s_part reads done before the next tile's writes
    if (tid == 0 && row0 >= 0) gate_trace(9);
    if (lane == 0) mbar_arrive(&lfull_bar[b]);
    if (row0 < 0) break;
  }
}



template <int NT>
int launch_gate_tc(const void* x, long long ld_x, const float* wg, const void* presplit,
                   const int32_t* excl, int T_, int d, int N, int k, int quota, float* logits,
                   int32_t* idx, float* w, int32_t* slots, uint8_t* drop, int32_t* counts,
                   float* prob_sum, uint8_t* ws, uint32_t* sync, cudaStream_t st) {
  using C = GateTC<NT>;
  const int n16 = (T_ + 15) / 16;
  const int ngrp = (d + 63) / 64;
  // persistent and fully resident (one CTA per SM): the in-kernel wait for
  // every CTA's counts cannot deadlock
  const int grid = min(min(n16, num_sms()), 1024);
  // sync: caller-kept words (zero before the first launch, left zero by
  // every launch); else the workspace's, zeroed here (a memset node)
  uint32_t* ctrs = sync ? sync - 2 : reinterpret_cast<uint32_t*>(ws);
  uint32_t* cta_cnt = reinterpret_cast<uint32_t*>(ws + CTR_BYTES);
  float* cta_psum = reinterpret_cast<float*>(ws + CTR_BYTES + (size_t)grid * N * 4);
  const uint8_t* blob = (const uint8_t*)presplit;
  if (!blob) {      // split the weights now (inference callers pass a cached blob)
    uint8_t* b = ws + gate_ws_bytes(T_, N);
    const int total = ngrp * NT * 128;
    gate_split_weights_kernel<NT><<<(total + 255) / 256, 256, 0, st>>>(wg, d, N, ngrp, (uint2*)b);
    SCMOE_LAUNCH_CHECK();
    blob = b;
  }
  // publish counter of the in-kernel prefix (a memset node in a graph:
  // ~8 us of idle GPU around it in a replay)
  if (!sync) SCMOE_CUDA_TRY(cudaMemsetAsync(ctrs, 0, 16, st));
  static bool attr_set = false;   // once per instantiation, never inside a graph capture
  if (!attr_set) {
    SCMOE_CUDA_TRY(cudaFuncSetAttribute(gate_topk_tc_kernel<NT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  CUtensorMap xmap;
  const int rc = make_map_2d(&xmap, x, d, T_, ld_x * 2, 16);
  if (rc != SCMOE_OK) return rc;
  gate_topk_tc_kernel<NT><<<grid, GT_THREADS, C::SMEM, st>>>(
      xmap, blob, excl, T_, d, N, k, quota, logits, idx, w, slots, drop, counts, prob_sum, ctrs,
      cta_cnt, cta_psum, n16);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
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

// Testing hook: 1 routes bf16 gates through the FMA kernel (A/B of the two
// logit paths).  Not part of the public header.
extern "C" int scmoe_gate_force_fma = 0;

extern "C" size_t scmoe_gate_workspace_bytes(int n_tokens, int n_experts, int d_model) {
  // + the split-weight blob of the tensor-core path
  return scmoe::gate_ws_bytes(n_tokens, n_experts) +
         (size_t)((d_model + 63) / 64) * ((n_experts + 7) / 8) * scmoe::GT_GROUP_B;
}

namespace scmoe {
namespace {
int gate_topk_impl(const void* x, int x_dtype, long long ld_x, const float* w_gate_t,
                   const void* w_split, const float* w_noise_t, const float* eps,
                   const int32_t* exclude, int n_tokens, int d_model, int n_experts, int k,
                   int quota, float* logits, int32_t* indices, float* weights, int32_t* slots,
                   uint8_t* dropped, int32_t* counts, float* prob_sum, void* workspace,
                   size_t workspace_bytes, uint32_t* sync, void* stream) {
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
  SCMOE_CHECK_ARG(workspace_bytes >= scmoe_gate_workspace_bytes(n_tokens, n_experts, d_model),
                  "gate workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  const bool tc = x_dtype == SCMOE_BF16 && w_noise_t == nullptr && n_experts <= 16 &&
                  d_model >= 64 && !scmoe_gate_force_fma;
  SCMOE_CHECK_ARG(!w_split || tc, "a pre-split weight blob needs the tensor-core gate "
                                  "(bf16 tokens, no noise, N <= 16, d >= 64)");
  if (tc) {
    const int rc =
        n_experts <= 8
            ? launch_gate_tc<1>(x, ld_x, w_gate_t, w_split, exclude, n_tokens, d_model, n_experts,
                                k, quota, logits, indices, weights, slots, dropped, counts,
                                prob_sum, ws, sync, st)
            : launch_gate_tc<2>(x, ld_x, w_gate_t, w_split, exclude, n_tokens, d_model, n_experts,
                                k, quota, logits, indices, weights, slots, dropped, counts,
                                prob_sum, ws, sync, st);
    if (rc != SCMOE_ERR_UNSUPPORTED) return rc;   // very large T: the FMA kernel below
  }
  if (x_dtype == SCMOE_BF16)
    return dispatch_nmax<__nv_bfloat16>(x, ld_x, w_gate_t, w_noise_t, eps, exclude, n_tokens,
                                        d_model, n_experts, k, quota, logits, indices, weights,
                                        slots, dropped, counts, prob_sum, ws, st);
  return dispatch_nmax<float>(x, ld_x, w_gate_t, w_noise_t, eps, exclude, n_tokens, d_model,
                              n_experts, k, quota, logits, indices, weights, slots, dropped,
                              counts, prob_sum, ws, st);
}
}  // namespace
}  // namespace scmoe

extern "C" int scmoe_gate_topk(const void* x, int x_dtype, long long ld_x,
                               const float* w_gate_t, const float* w_noise_t, const float* eps,
                               const int32_t* exclude,
                               int n_tokens, int d_model, int n_experts, int k, int quota,
                               float* logits, int32_t* indices, float* weights, int32_t* slots,
                               uint8_t* dropped, int32_t* counts, float* prob_sum,
                               void* workspace, size_t workspace_bytes, void* stream) {
  return scmoe::gate_topk_impl(x, x_dtype, ld_x, w_gate_t, nullptr, w_noise_t, eps, exclude,
                               n_tokens, d_model, n_experts, k, quota, logits, indices, weights,
                               slots, dropped, counts, prob_sum, workspace, workspace_bytes,
                               nullptr, stream);
}

extern "C" int scmoe_gate_topk_ex(const void* x, int x_dtype, long long ld_x,
                                  const float* w_gate_t, const void* w_split,
                                  const float* w_noise_t, const float* eps,
                                  const int32_t* exclude, int n_tokens, int d_model,
                                  int n_experts, int k, int quota, float* logits,
                                  int32_t* indices, float* weights, int32_t* slots,
                                  uint8_t* dropped, int32_t* counts, float* prob_sum,
                                  void* workspace, size_t workspace_bytes, uint32_t* sync,
                                  void* stream) {
  return scmoe::gate_topk_impl(x, x_dtype, ld_x, w_gate_t, w_split, w_noise_t, eps, exclude,
                               n_tokens, d_model, n_experts, k, quota, logits, indices, weights,
                               slots, dropped, counts, prob_sum, workspace, workspace_bytes, sync,
                               stream);
}

extern "C" size_t scmoe_gate_split_bytes(int n_experts, int d_model) {
  if (n_experts < 1 || n_experts > 16 || d_model < 64) return 0;
  return (size_t)((d_model + 63) / 64) * ((n_experts + 7) / 8) * scmoe::GT_GROUP_B;
}

extern "C" int scmoe_gate_split_weights(const float* w_gate_t, int n_experts, int d_model,
                                        void* blob, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(scmoe_gate_split_bytes(n_experts, d_model) > 0,
                  "the tensor-core gate needs N <= 16 and d >= 64");
  SCMOE_CHECK_ARG(d_model % 8 == 0 && w_gate_t && blob && ((uintptr_t)blob & 15) == 0,
                  "bad arguments");
  const int ngrp = (d_model + 63) / 64;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_experts <= 8) {
    const int total = ngrp * 128;
    gate_split_weights_kernel<1><<<(total + 255) / 256, 256, 0, st>>>(w_gate_t, d_model,
                                                                      n_experts, ngrp,
                                                                      (uint2*)blob);
  } else {
    const int total = ngrp * 2 * 128;
    gate_split_weights_kernel<2><<<(total + 255) / 256, 256, 0, st>>>(w_gate_t, d_model,
                                                                      n_experts, ngrp,
                                                                      (uint2*)blob);
  }
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_gate_topk_presplit(const void* x, int x_dtype, long long ld_x,
                                        const float* w_gate_t, const void* w_split,
                                        const int32_t* exclude, int n_tokens, int d_model,
                                        int n_experts, int k, int quota, float* logits,
                                        int32_t* indices, float* weights, int32_t* slots,
                                        uint8_t* dropped, int32_t* counts, float* prob_sum,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  return scmoe::gate_topk_impl(x, x_dtype, ld_x, w_gate_t, w_split, nullptr, nullptr, exclude,
                               n_tokens, d_model, n_experts, k, quota, logits, indices, weights,
                               slots, dropped, counts, prob_sum, workspace, workspace_bytes,
                               nullptr, stream);
}

#ifdef SCMOE_GATE_TRACE
extern "C" int scmoe_debug_gate_trace(unsigned long long* host, int n_ctas) {
  return cudaMemcpyFromSymbol(host, scmoe::g_gate_trace, (size_t)n_ctas * 20 * 8) == cudaSuccess
             ? 0
             : 1;
}
extern "C" int scmoe_debug_gate_stages(unsigned long long* host, int n_ctas) {
  return cudaMemcpyFromSymbol(host, scmoe::g_gate_stages, (size_t)n_ctas * 32 * 8) == cudaSuccess
             ? 0
             : 1;
}
#endif
