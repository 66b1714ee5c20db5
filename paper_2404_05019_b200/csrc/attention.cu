// Windowed multi-head attention for the backbone of the configs[1] block
// (SwinV2-MoE-S stage 3: 12x12 = 144-token windows, 12 heads of 32), forward
// and backward, reading the packed QKV projection (T, 3d) directly and
// writing O as (T, d) rows / dQKV in the packed layout — no head
// permutes or layout copies around the core.
//
// Semantics: per window of S rows and head h, O = softmax(Q K^T * scale) V
// (arch.py:354-358 generalised the way block.Attention does: heads, windows,
// optional causal mask).  Backward (FA2 form, with the forward's row
// log-sum-exp): P = exp(S*scale - lse), dV = P^T dO, dP = dO V^T,
// D = rowsum(dO o O), dS = P o (dP - D), dQ = dS K * scale,
// dK = dS^T Q * scale.
//
// One CTA per (window, head), one warp per 16 rows, everything in shared
// memory (S <= 192, hd in {32, 64}).  Tensor-core work is mma.sync
// m16n8k16 bf16 -> fp32 with ldmatrix operand loads: at S = 144 one window
// head is 16 KB of operands, far below a tcgen05 tile, and the kernel is
// HBM-bound (the packed QKV read + O write) rather than MMA-bound.
// Shared rows are padded by 16 bytes (pitch = 2*hd + 16), which makes every
// 8-row ldmatrix phase hit 8 distinct 16-byte bank groups.
#include "common.cuh"

namespace scmoe {
namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// shared tile of R rows x HD bf16, row pitch HD*2 + 16 bytes
template <int HD> struct Tile {
  static constexpr int PITCH = HD + 8;       // in bf16 elements
  bf16* p;
  __device__ __forceinline__ bf16* at(int r, int c) const { return p + r * PITCH + c; }
};

// rows [0, S) of one head's columns [col0, col0 + HD) of a (T, ld) bf16
// matrix starting at row `row0` into a padded shared tile (16 B per thread)
template <int HD>
__device__ __forceinline__ void load_tile(Tile<HD> t, const bf16* g, long long ld, long long row0,
                                          int col0, int S) {
  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < S * CH; i += blockDim.x) {
    const int r = i / CH, c = (i % CH) * 8;
    cp_async16(t.at(r, c), g + (row0 + r) * ld + col0 + c);
  }
}
// the same with the window length and the block size (2 SF threads) known at
// compile time: a fixed, fully unrolled trip count
template <int HD, int SF>
__device__ __forceinline__ void load_tile_c(Tile<HD> t, const bf16* g, long long ld,
                                            long long row0, int col0) {
  constexpr int CH = HD / 8, NT = 2 * SF, N = SF * CH;
  const bf16* base = g + row0 * ld + col0;
#pragma unroll
  for (int k = 0; k < (N + NT - 1) / NT; ++k) {
    const int i = threadIdx.x + k * NT;
    if (N % NT == 0 || i < N) {
      const int r = i / CH, c = (i % CH) * 8;
      cp_async16(t.at(r, c), base + r * ld + c);
    }
  }
}

// A fragment (16 x 16 at rows r0, cols c0) of a row-major shared tile
template <int HD>
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], Tile<HD> t, int r0, int c0, int lane) {
  ldsm_x4(a, t.at(r0 + (lane & 15), c0 + (lane >> 4) * 8));
}
// B fragments of two n8 tiles (n0, n0 + 8) for k16 step c0 when B(k, n) =
// t[n][k] (the tile's rows are the n index): {b0, b1} of n0, {b0, b1} of n0+8
template <int HD>
__device__ __forceinline__ void frag_b_rows(uint32_t (&b)[4], Tile<HD> t, int n0, int c0,
                                            int lane) {
  ldsm_x4(b, t.at(n0 + (lane & 7) + ((lane >> 4) << 3), c0 + ((lane >> 3) & 1) * 8));
}
// B fragments of two n8 tiles (n0, n0 + 8) for k16 step k0 when B(k, n) =
// t[k][n] (the tile's rows are the k index): transposed ldmatrix
template <int HD>
__device__ __forceinline__ void frag_b_cols(uint32_t (&b)[4], Tile<HD> t, int k0, int n0,
                                            int lane) {
  ldsm_x4_t(b, t.at(k0 + (lane & 7) + ((lane >> 3) & 1) * 8, n0 + (lane >> 4) * 8));
}

// ---------------------------------------------------------------------------
// forward

// 16 rows x HD columns of one warp, staged in shared memory (rows r0 .. r0+15
// of tile t), written to global rows as whole 16-byte vectors: every row's
// HD*2 bytes are contiguous, so each store covers whole 32-byte sectors
// (lane-scattered 4-byte fragment stores cover half sectors)
template <int HD>
__device__ __forceinline__ void store_rows16(Tile<HD> t, int r0, bf16* g, long long ld, int lane) {
  constexpr int CH = HD / 8;              // 16-byte vectors per row
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16 * CH / 32; ++i) {
    const int q = lane + 32 * i;
    const int r = q / CH, c = (q % CH) * 8;
    *reinterpret_cast<uint4*>(g + (long long)r * ld + c) =
        *reinterpret_cast<const uint4*>(t.at(r0 + r, c));
  }
}
// the accumulator fragments of a 16 x HD warp tile (rows g / g+8, columns
// n*8 + 2*t4) into shared rows r0 .. r0+15, scaled, as bf16
template <int HD>
__device__ __forceinline__ void stage_frag(Tile<HD> t, int r0, const float (&acc)[HD / 8][4],
                                           float s_lo, float s_hi, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    *reinterpret_cast<uint32_t*>(t.at(r0 + g, n * 8 + 2 * t4)) =
        pack_bf16(acc[n][0] * s_lo, acc[n][1] * s_lo);
    *reinterpret_cast<uint32_t*>(t.at(r0 + g + 8, n * 8 + 2 * t4)) =
        pack_bf16(acc[n][2] * s_hi, acc[n][3] * s_hi);
  }
}

// One (window, head) item of the forward on tiles already in (or, before
// `before_pv()`, still landing in) shared memory: scores, softmax, O = P V,
// staged whole-row store of O, base-2 log-sum-exp.  SF: the window length as
// a compile-time constant (0: runtime S) — with it every key-tile loop is
// fully unrolled without bounds predicates.  `before_pv` runs on every
// thread (it may hold a barrier) between the softmax and P V.
template <int HD, int NT, int SF, typename BeforePV>
__device__ __forceinline__ void fwd_item(Tile<HD> Qs, Tile<HD> Ks, Tile<HD> Vs, int S, int H,
                                         int h, long long row0, float scale_log2, bool causal,
                                         bf16* __restrict__ out, float* __restrict__ lse,
                                         BeforePV&& before_pv) {
  const int d = H * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int m0 = warp * 16;
  const bool active = m0 < S;                  // blockDim = 2 S: always, kept for safety
  uint32_t qa[HD / 16][4];
  float sc[NT][4];
  const int nt = S / 8;
  float b0 = 0.f, b1 = 0.f, s0 = 1.f, s1 = 1.f;
  if (active) {
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) frag_a<HD>(qa[kk], Qs, m0, kk * 16, lane);
#pragma unroll
    for (int j = 0; j < NT; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < NT; j += 2) {
      if (SF || j < nt) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          uint32_t b[4];
          frag_b_rows<HD>(b, Ks, j * 8, kk * 16, lane);
          mma16816(sc[j], qa[kk], b[0], b[1]);
          mma16816(sc[j + 1], qa[kk], b[2], b[3]);
        }
      }
    }
    // softmax over keys (rows g and g + 8 of the warp's tile)
    const int r_lo = m0 + g, r_hi = r_lo + 8;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (SF || j < nt) {
        const int c = j * 8 + 2 * t4;
        if (causal) {
          if (c > r_lo) sc[j][0] = -INFINITY;
          if (c + 1 > r_lo) sc[j][1] = -INFINITY;
          if (c > r_hi) sc[j][2] = -INFINITY;
          if (c + 1 > r_hi) sc[j][3] = -INFINITY;
        }
        mx0 = fmaxf(mx0, fmaxf(sc[j][0], sc[j][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[j][2], sc[j][3]));
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    b0 = mx0 * scale_log2;
    b1 = mx1 * scale_log2;
    s0 = 0.f;
    s1 = 0.f;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (SF || j < nt) {
        sc[j][0] = ex2(fmaf(sc[j][0], scale_log2, -b0));
        sc[j][1] = ex2(fmaf(sc[j][1], scale_log2, -b0));
        sc[j][2] = ex2(fmaf(sc[j][2], scale_log2, -b1));
        sc[j][3] = ex2(fmaf(sc[j][3], scale_log2, -b1));
        s0 += sc[j][0] + sc[j][1];
        s1 += sc[j][2] + sc[j][3];
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
  }
  before_pv();
  if (!active) return;
  // O = P V (P as bf16 A fragments straight from the score registers)
  float oc[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) oc[n][0] = oc[n][1] = oc[n][2] = oc[n][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < NT / 2; ++kk) {
    if (SF || 2 * kk < nt) {
      uint32_t pa[4] = {pack_bf16(sc[2 * kk][0], sc[2 * kk][1]),
                        pack_bf16(sc[2 * kk][2], sc[2 * kk][3]),
                        pack_bf16(sc[2 * kk + 1][0], sc[2 * kk + 1][1]),
                        pack_bf16(sc[2 * kk + 1][2], sc[2 * kk + 1][3])};
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b[4];
        frag_b_cols<HD>(b, Vs, kk * 16, n * 8, lane);
        mma16816(oc[n], pa, b[0], b[1]);
        mma16816(oc[n + 1], pa, b[2], b[3]);
      }
    }
  }
  // the warp's own Q rows are free (its Q fragments are in registers): stage
  // O there and store whole rows
  stage_frag<HD>(Qs, m0, oc, 1.0f / s0, 1.0f / s1, lane);
  store_rows16<HD>(Qs, m0, out + (row0 + m0) * d + h * HD, d, lane);
  if (lse != nullptr && t4 == 0) {     // base-2 log-sum-exp of the scaled scores
    lse[(row0 + m0 + g) * H + h] = b0 + __log2f(s0);
    lse[(row0 + m0 + g + 8) * H + h] = b1 + __log2f(s1);
  }
}

// one CTA per (window, head), runtime window length
template <int HD, int SMAX>
__global__ void __launch_bounds__(SMAX * 2, SMAX <= 144 ? 2 : 1)
win_attn_fwd_kernel(const bf16* __restrict__ qkv, int H, int S, float scale_log2, bool causal,
                    bf16* __restrict__ out, float* __restrict__ lse) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = H * HD;
  const long long ld = 3ll * d;
  const int w = blockIdx.x, h = blockIdx.y;
  const long long row0 = (long long)w * S;
  Tile<HD> Qs{(bf16*)smem}, Ks{Qs.p + S * Tile<HD>::PITCH}, Vs{Ks.p + S * Tile<HD>::PITCH};
  // Q and K first (one cp.async group), V behind them: the scores start
  // while V is still in flight
  load_tile<HD>(Qs, qkv, ld, row0, h * HD, S);
  load_tile<HD>(Ks, qkv, ld, row0, d + h * HD, S);
  asm volatile("cp.async.commit_group;" ::: "memory");
  load_tile<HD>(Vs, qkv, ld, row0, 2 * d + h * HD, S);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
  __syncthreads();
  fwd_item<HD, SMAX / 8, 0>(Qs, Ks, Vs, S, H, h, row0, scale_log2, causal, out, lse, [] {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                           // V landed
  });
}

// Persistent form for a compile-time window length SF: each CTA walks items
// (window, head) = blockIdx.x, + gridDim.x, ... with two shared-memory tile
// sets — item i+1's Q / K / V stream in (cp.async) while item i computes, so
// the loads no longer sit between the compute phases of the two resident CTAs
template <int HD, int SF>
__global__ void __launch_bounds__(SF * 2, 2)
win_attn_fwd_persistent(const bf16* __restrict__ qkv, int H, int n_items, float scale_log2,
                        bool causal, bf16* __restrict__ out, float* __restrict__ lse) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int TILE = SF * Tile<HD>::PITCH;   // elements per tile
  const int d = H * HD;
  const long long ld = 3ll * d;
  bf16* base = (bf16*)smem;
  auto issue = [&](int item, int b) {
    const int w = item / H, h = item - w * H;
    const long long row0 = (long long)w * SF;
    bf16* p = base + b * 3 * TILE;
    load_tile_c<HD, SF>(Tile<HD>{p}, qkv, ld, row0, h * HD);
    load_tile_c<HD, SF>(Tile<HD>{p + TILE}, qkv, ld, row0, d + h * HD);
    load_tile_c<HD, SF>(Tile<HD>{p + 2 * TILE}, qkv, ld, row0, 2 * d + h * HD);
  };
  int item = blockIdx.x;
  if (item < n_items) issue(item, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int it = 0; item < n_items; ++it, item += gridDim.x) {
    const int nxt = item + gridDim.x;
    if (nxt < n_items) issue(nxt, (it + 1) & 1);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
    __syncthreads();                           // this item's tiles landed
    bf16* p = base + (it & 1) * 3 * TILE;
    const int w = item / H, h = item - w * H;
    fwd_item<HD, SF / 8, SF>(Tile<HD>{p}, Tile<HD>{p + TILE}, Tile<HD>{p + 2 * TILE}, SF, H, h,
                             (long long)w * SF, scale_log2, causal, out, lse, [] {});
    __syncthreads();                           // every warp is done with this tile set
  }
}

// ---------------------------------------------------------------------------
// backward

template <int HD, int SMAX, int SF>
__global__ void __launch_bounds__(SMAX * 2)
win_attn_bwd_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ o,
                    const bf16* __restrict__ dout, const float* __restrict__ lse, int H, int s_rt,
                    float scale, float scale_log2, bool causal, bf16* __restrict__ dqkv) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int P = Tile<HD>::PITCH;
  const int S = SF ? SF : s_rt;
  const int DSP = S + 8;                      // dS^T row pitch (bf16 elements)
  const int d = H * HD;
  const long long ld = 3ll * d;
  const int w = blockIdx.x, h = blockIdx.y;
  const long long row0 = (long long)w * S;
  Tile<HD> Qs{(bf16*)smem}, Ks{Qs.p + S * P}, Vs{Ks.p + S * P}, Gs{Vs.p + S * P},
      Os{Gs.p + S * P};                       // Gs = dO, Os = O
  bf16* dst = Os.p + S * P;                   // dS^T [key][query]
  float* Dq = (float*)(dst + S * DSP);        // D = rowsum(dO o O) per query
  float* Lq = Dq + S;                         // base-2 lse per query
  auto load = [&](Tile<HD> t, const bf16* g, long long ldg, int col0) {
    if (SF) load_tile_c<HD, SF ? SF : 16>(t, g, ldg, row0, col0);
    else load_tile<HD>(t, g, ldg, row0, col0, S);
  };
  load(Gs, dout, d, h * HD);
  load(Os, o, d, h * HD);
  asm volatile("cp.async.commit_group;" ::: "memory");
  load(Qs, qkv, ld, h * HD);
  load(Ks, qkv, ld, d + h * HD);
  load(Vs, qkv, ld, 2 * d + h * HD);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int i = threadIdx.x; i < S; i += blockDim.x) Lq[i] = lse[(row0 + i) * H + h];
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  __syncthreads();                            // dO and O landed: D while Q / K / V load
  // D = rowsum(dO o O): two threads per row (blockDim = 2 S), HD / 2 columns
  // each, partner sum by shuffle
  {
    const int i = threadIdx.x >> 1, half = threadIdx.x & 1;
    float acc = 0.f;
    if (i < S) {
#pragma unroll
      for (int c = half * (HD / 2); c < (half + 1) * (HD / 2); c += 8) {
        Vec16<bf16> a, b;
        a.raw = *reinterpret_cast<const uint4*>(Os.at(i, c));
        b.raw = *reinterpret_cast<const uint4*>(Gs.at(i, c));
        float fa[8], fb[8];
        a.to_float(fa);
        b.to_float(fb);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(fa[e], fb[e], acc);
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (i < S && half == 0) Dq[i] = acc;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int m0 = warp * 16;
  const bool active = m0 < S;
  const int nq = S / 16;
  // dK / dV of the warp's keys, packed bf16, kept until the final staged store
  uint32_t dk_p[HD / 8][2], dv_p[HD / 8][2];
  // ---- phase A: warp owns keys [m0, m0 + 16); loop over query blocks of 16
  if (active) {
    uint32_t ka[HD / 16][4], va[HD / 16][4];
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      frag_a<HD>(ka[kk], Ks, m0, kk * 16, lane);
      frag_a<HD>(va[kk], Vs, m0, kk * 16, lane);
    }
    float dv[HD / 8][4], dk[HD / 8][4];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) dv[n][e] = dk[n][e] = 0.f;
    const int key_lo = m0 + g, key_hi = key_lo + 8;
#pragma unroll 3
    for (int qb = 0; qb < nq; ++qb) {
      const int q0 = qb * 16;
      if (causal && q0 + 15 < m0) {          // every key of mine is after these queries
        for (int e = 0; e < 2; ++e) {
          const int q = q0 + e * 8 + 2 * t4;
          *reinterpret_cast<uint32_t*>(dst + key_lo * DSP + q) = 0u;
          *reinterpret_cast<uint32_t*>(dst + key_hi * DSP + q) = 0u;
        }
        continue;
      }
      // S^T block (16 keys x 16 queries) = K_w Q_b^T
      float st[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t b[4];
        frag_b_rows<HD>(b, Qs, q0, kk * 16, lane);
        mma16816(st[0], ka[kk], b[0], b[1]);
        mma16816(st[1], ka[kk], b[2], b[3]);
      }
      // dP^T block = V_w dO_b^T (independent of P: issued before the exps)
      float dpt[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t b[4];
        frag_b_rows<HD>(b, Gs, q0, kk * 16, lane);
        mma16816(dpt[0], va[kk], b[0], b[1]);
        mma16816(dpt[1], va[kk], b[2], b[3]);
      }
      // P^T = exp2(S^T * scale_log2 - lse[q])
      float pt[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = q0 + j * 8 + 2 * t4;
        const float2 l = *reinterpret_cast<const float2*>(Lq + q);
        pt[j][0] = ex2(fmaf(st[j][0], scale_log2, -l.x));
        pt[j][1] = ex2(fmaf(st[j][1], scale_log2, -l.y));
        pt[j][2] = ex2(fmaf(st[j][2], scale_log2, -l.x));
        pt[j][3] = ex2(fmaf(st[j][3], scale_log2, -l.y));
        if (causal) {
          if (key_lo > q) pt[j][0] = 0.f;
          if (key_lo > q + 1) pt[j][1] = 0.f;
          if (key_hi > q) pt[j][2] = 0.f;
          if (key_hi > q + 1) pt[j][3] = 0.f;
        }
      }
      const uint32_t pa[4] = {pack_bf16(pt[0][0], pt[0][1]), pack_bf16(pt[0][2], pt[0][3]),
                              pack_bf16(pt[1][0], pt[1][1]), pack_bf16(pt[1][2], pt[1][3])};
      // dV_w += P^T dO_b
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b[4];
        frag_b_cols<HD>(b, Gs, q0, n * 8, lane);
        mma16816(dv[n], pa, b[0], b[1]);
        mma16816(dv[n + 1], pa, b[2], b[3]);
      }
      // dS^T = P^T o (dP^T - D[q])
      float ds[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = q0 + j * 8 + 2 * t4;
        const float2 D = *reinterpret_cast<const float2*>(Dq + q);
        ds[j][0] = pt[j][0] * (dpt[j][0] - D.x);
        ds[j][1] = pt[j][1] * (dpt[j][1] - D.y);
        ds[j][2] = pt[j][2] * (dpt[j][2] - D.x);
        ds[j][3] = pt[j][3] * (dpt[j][3] - D.y);
      }
      const uint32_t da[4] = {pack_bf16(ds[0][0], ds[0][1]), pack_bf16(ds[0][2], ds[0][3]),
                              pack_bf16(ds[1][0], ds[1][1]), pack_bf16(ds[1][2], ds[1][3])};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = q0 + j * 8 + 2 * t4;
        *reinterpret_cast<uint32_t*>(dst + key_lo * DSP + q) = da[2 * j];
        *reinterpret_cast<uint32_t*>(dst + key_hi * DSP + q) = da[2 * j + 1];
      }
      // dK_w += dS^T Q_b
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b[4];
        frag_b_cols<HD>(b, Qs, q0, n * 8, lane);
        mma16816(dk[n], da, b[0], b[1]);
        mma16816(dk[n + 1], da, b[2], b[3]);
      }
    }
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      dk_p[n][0] = pack_bf16(dk[n][0] * scale, dk[n][1] * scale);
      dk_p[n][1] = pack_bf16(dk[n][2] * scale, dk[n][3] * scale);
      dv_p[n][0] = pack_bf16(dv[n][0], dv[n][1]);
      dv_p[n][1] = pack_bf16(dv[n][2], dv[n][3]);
    }
  }
  __syncthreads();
  // ---- phase B: warp owns queries [m0, m0 + 16): dQ = dS K * scale
  float dq[HD / 8][4];
  if (active) {
    // two accumulator sets (even / odd key blocks): the chained MMAs of one
    // set alternate with the other's instead of waiting on each other
    float dq2[HD / 8][4];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) dq[n][e] = dq2[n][e] = 0.f;
    auto kblock = [&](int kb, float (&acc)[HD / 8][4]) __attribute__((always_inline)) {
      const int k0 = kb * 16;
      uint32_t a[4];                            // dS (16 queries x 16 keys) from dS^T
      ldsm_x4_t(a, dst + (k0 + (lane & 7) + (lane >> 4) * 8) * DSP + m0 + ((lane >> 3) & 1) * 8);
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b[4];
        frag_b_cols<HD>(b, Ks, k0, n * 8, lane);
        mma16816(acc[n], a, b[0], b[1]);
        mma16816(acc[n + 1], a, b[2], b[3]);
      }
    };
    // keys after every query of mine contribute nothing (causal)
    const int kb_end = causal ? min(nq, (m0 + 15) / 16 + 1) : nq;
    int kb = 0;
#pragma unroll 2
    for (; kb + 1 < kb_end; kb += 2) {
      kblock(kb, dq);
      kblock(kb + 1, dq2);
    }
    if (kb < kb_end) kblock(kb, dq);
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) dq[n][e] += dq2[n][e];
  }
  __syncthreads();                             // every read of Q / K / V / dS^T is done
  if (!active) return;
  // staged whole-row stores: dQ through the warp's Q rows, dK through its K
  // rows, dV through its V rows
  stage_frag<HD>(Qs, m0, dq, scale, scale, lane);
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    *reinterpret_cast<uint32_t*>(Ks.at(m0 + g, n * 8 + 2 * t4)) = dk_p[n][0];
    *reinterpret_cast<uint32_t*>(Ks.at(m0 + g + 8, n * 8 + 2 * t4)) = dk_p[n][1];
    *reinterpret_cast<uint32_t*>(Vs.at(m0 + g, n * 8 + 2 * t4)) = dv_p[n][0];
    *reinterpret_cast<uint32_t*>(Vs.at(m0 + g + 8, n * 8 + 2 * t4)) = dv_p[n][1];
  }
  bf16* base = dqkv + (row0 + m0) * ld + h * HD;
  store_rows16<HD>(Qs, m0, base, ld, lane);
  store_rows16<HD>(Ks, m0, base + d, ld, lane);
  store_rows16<HD>(Vs, m0, base + 2 * d, ld, lane);
}

constexpr int WIN_SMAX = 192;

// shared bytes for windows of S rows (S % 16 == 0 keeps every region 16-byte
// aligned: pitches are multiples of 16 bytes)
template <int HD>
size_t fwd_smem(int S) { return 3ull * S * Tile<HD>::PITCH * sizeof(bf16); }
template <int HD>
size_t bwd_smem(int S) {
  return 5ull * S * Tile<HD>::PITCH * sizeof(bf16) + (size_t)S * (S + 8) * sizeof(bf16) +
         2ull * S * sizeof(float);
}

template <int HD, int SMAX>
int launch_fwd_s(const bf16* qkv, int n_windows, int H, int S, float scale, int causal, bf16* out,
                 float* lse, cudaStream_t st) {
  auto k = win_attn_fwd_kernel<HD, SMAX>;
  SCMOE_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)fwd_smem<HD>(SMAX)));
  k<<<dim3(n_windows, H), 2 * S, fwd_smem<HD>(S), st>>>(qkv, H, S, scale * 1.4426950408889634f,
                                                      causal != 0, out, lse);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

template <int HD, int SF>
int launch_fwd_p(const bf16* qkv, int n_windows, int H, float scale, int causal, bf16* out,
                 float* lse, cudaStream_t st) {
  auto k = win_attn_fwd_persistent<HD, SF>;
  const int smem = (int)(2 * fwd_smem<HD>(SF));
  SCMOE_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int items = n_windows * H;
  int grid = 2 * num_sms();
  if (grid > items) grid = items;
  k<<<grid, 2 * SF, smem, st>>>(qkv, H, items, scale * 1.4426950408889634f, causal != 0, out, lse);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

// the score registers scale with the longest window a build handles: pick
// the smallest instantiation that covers S (S = 144 -> 18 key tiles, 2 CTAs
// per SM instead of 1); the configs[1] window (144) and 64 run persistent
// with a compile-time S
template <int HD>
int launch_fwd(const bf16* qkv, int n_windows, int H, int S, float scale, int causal, bf16* out,
               float* lse, cudaStream_t st) {
  if (HD == 32 && S == 144) return launch_fwd_p<HD, 144>(qkv, n_windows, H, scale, causal, out, lse, st);
  if (S == 64) return launch_fwd_p<HD, 64>(qkv, n_windows, H, scale, causal, out, lse, st);
  if (S <= 64) return launch_fwd_s<HD, 64>(qkv, n_windows, H, S, scale, causal, out, lse, st);
  if (S <= 128) return launch_fwd_s<HD, 128>(qkv, n_windows, H, S, scale, causal, out, lse, st);
  if (S <= 144) return launch_fwd_s<HD, 144>(qkv, n_windows, H, S, scale, causal, out, lse, st);
  return launch_fwd_s<HD, WIN_SMAX>(qkv, n_windows, H, S, scale, causal, out, lse, st);
}

template <int HD, int SMAX, int SF>
int launch_bwd_s(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse,
                 int n_windows, int H, int S, float scale, int causal, bf16* dqkv,
                 cudaStream_t st) {
  auto k = win_attn_bwd_kernel<HD, SMAX, SF>;
  SCMOE_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)bwd_smem<HD>(SMAX)));
  k<<<dim3(n_windows, H), 2 * S, bwd_smem<HD>(S), st>>>(qkv, o, dout, lse, H, S, scale,
                                                      scale * 1.4426950408889634f, causal != 0,
                                                      dqkv);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

template <int HD>
int launch_bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, int n_windows,
               int H, int S, float scale, int causal, bf16* dqkv, cudaStream_t st) {
  if (S == 144)
    return launch_bwd_s<HD, 144, 144>(qkv, o, dout, lse, n_windows, H, S, scale, causal, dqkv, st);
  return launch_bwd_s<HD, WIN_SMAX, 0>(qkv, o, dout, lse, n_windows, H, S, scale, causal, dqkv, st);
}

}  // namespace
}  // namespace scmoe

using namespace scmoe;

extern "C" int scmoe_window_attention_supported(int seq_len, int head_dim) {
  return seq_len >= 16 && seq_len <= WIN_SMAX && seq_len % 16 == 0 &&
         (head_dim == 32 || head_dim == 64);
}

extern "C" int scmoe_window_attention_fwd(const void* qkv, int n_tokens, int n_heads, int head_dim,
                                          int seq_len, float scale, int causal, void* out,
                                          float* lse, void* stream) {
  SCMOE_CHECK_ARG(qkv && out, "window_attention_fwd: null pointer");
  SCMOE_CHECK_ARG(scmoe_window_attention_supported(seq_len, head_dim),
                  "window_attention_fwd: seq_len %d / head_dim %d unsupported", seq_len, head_dim);
  SCMOE_CHECK_ARG(n_heads >= 1 && n_tokens > 0 && n_tokens % seq_len == 0,
                  "window_attention_fwd: %d tokens do not split into windows of %d", n_tokens,
                  seq_len);
  SCMOE_CHECK_ARG(((uintptr_t)qkv & 15) == 0, "window_attention_fwd: qkv must be 16-byte aligned");
  const int nw = n_tokens / seq_len;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 32)
    return launch_fwd<32>((const bf16*)qkv, nw, n_heads, seq_len, scale, causal, (bf16*)out, lse,
                          st);
  return launch_fwd<64>((const bf16*)qkv, nw, n_heads, seq_len, scale, causal, (bf16*)out, lse, st);
}

extern "C" int scmoe_window_attention_bwd(const void* qkv, const void* out, const void* dout,
                                          const float* lse, int n_tokens, int n_heads,
                                          int head_dim, int seq_len, float scale, int causal,
                                          void* dqkv, void* stream) {
  SCMOE_CHECK_ARG(qkv && out && dout && lse && dqkv, "window_attention_bwd: null pointer");
  SCMOE_CHECK_ARG(scmoe_window_attention_supported(seq_len, head_dim),
                  "window_attention_bwd: seq_len %d / head_dim %d unsupported", seq_len, head_dim);
  SCMOE_CHECK_ARG(n_heads >= 1 && n_tokens > 0 && n_tokens % seq_len == 0,
                  "window_attention_bwd: %d tokens do not split into windows of %d", n_tokens,
                  seq_len);
  const int nw = n_tokens / seq_len;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 32)
    return launch_bwd<32>((const bf16*)qkv, (const bf16*)out, (const bf16*)dout, lse, nw, n_heads,
                          seq_len, scale, causal, (bf16*)dqkv, st);
  return launch_bwd<64>((const bf16*)qkv, (const bf16*)out, (const bf16*)dout, lse, nw, n_heads,
                        seq_len, scale, causal, (bf16*)dqkv, st);
}
