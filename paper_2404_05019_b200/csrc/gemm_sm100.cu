// K3 / K4 / K7 — grouped bf16 GEMMs on 5th-generation tensor cores (tcgen05).
//
// Forward / dgrad ("rows" mode):
//   out[g, r, :] = epi( a[g, r, :] . B(g % W)^T ) for r < rows(g)
// with rows(g) = min(group_rows[g], rows_clip).  B is read K-major from
// (W, n_out, k_in) weights (forward), or MN-major from (W, k_in, n_out) — the
// same stored weights used transposed (dgrad, K7).  Epilogues: expert_forward's
// bias (+ exact-erf GELU, optionally storing the pre-activation) (arch.py:349-351),
// the GELU backward dZ = acc * gelu'(z), an optional fused residual add
// (arch.py:542, 587-588) and zero padding of rows past rows(g) ("zero_tail").
// The routed experts read the capacity-slotted dispatch buffer (group =
// expert, rows = kept tokens known only on the device); dense layers are one
// group.
//
// Weight gradient ("wgrad" mode, K7):
//   out[w] = sum_{g = w mod W} sum_{r < rows(g)} a[g, r, :]^T (x) b[g, r, :]
// both operands MN-major (the token dimension is the reduction), split-K over
// the concatenated k-blocks of the groups feeding weight group w, fp32
// partials reduced by a second kernel.
//
// Structure (persistent, 384 threads per CTA, one CTA per SM):
//   warp 0      TMA producer: 128B-swizzled tiles into a shared-memory ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma kind::f16 (fp32 TMEM
//               accumulators); tcgen05.commit frees ring stages / signals the
//               epilogue
//   warp 2      TMEM allocator (512 columns = two 256-column accumulators)
//   warps 4-11  epilogue: tcgen05.ld 32x32b (next chunk in flight) -> math ->
//               global, double-buffered against the next tile's MMAs
// Two shapes: 1SM 128x256 tile (cta_group::1, 4 stages x 48 KB) and 2SM 256x256
// per CTA pair (cluster of 2, cta_group::2: each CTA loads its half of A and of
// B, the leader's M=256 MMAs read both CTAs' smem and write both TMEMs; 6
// stages x 32 KB).
#include <cuda.h>
#include <type_traits>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace scmoe {
namespace sm100 {

constexpr int BK = 64;
// epilogue warps: 8 (the default: large-K tiles are MMA-bound) or 16 (small-K
// tiles with elementwise-heavy epilogues — GELU, GELU backward, the
// pre-activation store, residuals — where the epilogue's issue rate, not the
// MMA, paces the tile; twice the warps hide twice the latency)
constexpr int EPI_WARPS = 8;
template <int E> struct Threads { static constexpr int value = 128 + E * 32; };
constexpr int THREADS = Threads<EPI_WARPS>::value;
constexpr int TMEM_COLS = 512;                   // 512 / BN accumulator stages
constexpr int MAX_GROUPS = 1024;
// groups up to which the forward / dgrad schedule packs whole groups into
// waves (see the virtual tile starts in gemm_kernel)
constexpr int MAX_PACK = 64;
constexpr int MN_BOX = 64;                       // MN-major TMA box: 64 (mn) x 64 (k)
constexpr int MN_BOX_BYTES = MN_BOX * BK * 2;    // 8 KB

// BN_ = 256 (default) or 128: the narrow tile for n_out = 384-style widths
// (configs[1]) that would leave half a 256-column tile idle; it also doubles
// the accumulator stages (4 x 128 TMEM columns) for small-K tiles.
template <bool TWO_SM, int BN_ = 256, int E_ = 8>
struct Cfg {
  static constexpr int E = E_;                            // epilogue warps
  static constexpr int BN = BN_;
  static constexpr int ACC_STAGES = TMEM_COLS / BN;
  static constexpr int CTA_M = 128;                       // rows of A per CTA
  static constexpr int TILE_M = TWO_SM ? 256 : 128;       // rows per (cluster) tile
  static constexpr int B_ROWS = TWO_SM ? BN / 2 : BN;     // rows of B per CTA
  static constexpr int A_BYTES = CTA_M * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RING_BYTES = E_ == 8 ? 192 * 1024 : 176 * 1024;
  static constexpr int STAGES = (RING_BYTES / STAGE_BYTES) < 8 ? (RING_BYTES / STAGE_BYTES) : 8;
  // + per-epilogue-warp bias slice (E warps x 128 fp32), staged once per tile
  static constexpr size_t MISC =
      256 + ((MAX_GROUPS + 1) * 4 + 15) / 16 * 16 + ((MAX_PACK + 1) * 4 + 15) / 16 * 16;
  // + per-epilogue-warp 2 KB store-transpose staging
  static constexpr size_t SMEM =
      1024 + (size_t)STAGES * STAGE_BYTES + MISC + E_ * 128 * 4 + E_ * 2048;
};

// instruction descriptor: D fp32, A/B bf16, M = TILE_M, N = 256, operand majors
template <bool TWO_SM, bool A_MN, bool B_MN, int BN>
struct Idesc {
  static constexpr uint32_t value = (1u << 4) | (1u << 7) | (1u << 10) |
                                    ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
                                    ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(Cfg<TWO_SM, BN>::TILE_M >> 4) << 24);
};

enum Epi { EPI_BIAS = 0, EPI_BIAS_GELU = 1, EPI_GELU_BWD = 2, EPI_MUL_AUX = 3 };

struct Params {
  int num_groups, n_wgroups, cap, rows_clip, N, K, epi, zero_tail;
  int m_out, splits;                       // wgrad only
  const int32_t* group_rows;
  const float* bias;
  const __nv_bfloat16* residual;
  const __nv_bfloat16* aux_in;             // GELU backward: pre-activation z
  __nv_bfloat16* aux_out;                  // forward: store the pre-activation
  __nv_bfloat16* out;
  float* out_f32;                          // wgrad partials [splits][W][m_out][N]
  // fused ScMoE combine (direct add) in the shared expert's GEMM2 epilogue:
  // out[t] = bf16(acc + b2) + sum_j w_j * cy[c_idx[t,j], c_slot[t,j]] (+ residual)
  const __nv_bfloat16* cy;
  const int32_t* c_idx;
  const int32_t* c_slot;
  const float* c_w;
  int c_cap, c_k;                          // c_k = 0: off
  // per-group output base (expert-parallel return fused into GEMM2): group g's
  // rows go to out_groups[g] + row * N (peer memory), nullptr: out + g*cap*N
  __nv_bfloat16* const* out_groups;
  // 1 when the epilogue reads a row-major operand (residual or the GELU
  // pre-activation): the ring runs one stage short and that stage's A slot
  // (16 KB) holds the per-warp coalesced load buffers
  int ld_buf;
  int dbg;                                 // experiment flags (g_gemm_flags)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the same-offset barrier of CTA `rank` in the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// Accumulator release from the epilogue: the TMEM reads are ordered by
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync; the arrive itself needs
// no cluster-scope release of the epilogue's global stores (that compiled to a
// MEMBAR.ALL.GPU per warp per tile, draining every output store before the
// MMA warp could reuse the accumulator — the small-K limiter).
__device__ __forceinline__ void mbar_arrive_cluster_tmem(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA tile load; in 2-SM mode the bytes land in this CTA's shared memory and
// completion is counted on the leader CTA's barrier (peer bit cleared).
template <bool TWO_SM>
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  if (TWO_SM) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
        "r"(c2)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  }
}
// One operand tile of `ROWS` (M or N) x 64 (K): K-major = one box (64 k, ROWS),
// MN-major = ROWS/64 boxes of (64 mn, 64 k), 8 KB apart.
template <bool TWO_SM, bool MN, int ROWS>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, uint64_t* bar, uint8_t* dst,
                                             int k0, int mn0, int g) {
  if (MN) {
#pragma unroll
    for (int i = 0; i < ROWS / MN_BOX; ++i)
      tma_load_3d<TWO_SM>(map, bar, dst + i * MN_BOX_BYTES, mn0 + i * MN_BOX, k0, g);
  } else {
    tma_load_3d<TWO_SM>(map, bar, dst, k0, mn0, g);
  }
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
template <bool TWO_SM>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if (TWO_SM) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
  }
}
template <bool TWO_SM>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if (TWO_SM) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// Shared-memory matrix descriptors, 128-byte swizzle, sm_100 version bits.
// K-major: rows of 64 bf16 (128 B) along K, 8-row groups 1024 B apart (SBO).
// MN-major: rows of 64 bf16 along MN, one per k; 8-k groups 1024 B apart (SBO),
// 64-element MN blocks one TMA box (8 KB) apart (LBO).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kk) {
  // advance by one UMMA K-step (16 bf16): 32 B inside a K-major row, 16 rows
  // of 128 B in an MN-major tile
  return MN ? sw128_desc(base + kk * 16 * 128, MN_BOX_BYTES) : sw128_desc(base + kk * 32, 16);
}

#define SCMOE_TMEM_LD32(taddr, r)                                                              \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),            \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),         \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),         \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),         \
        "=r"(r[31])                                                                            \
      : "r"(taddr))

__device__ __forceinline__ int group_rows_of(const Params& p, int g) {
  return p.group_rows ? max(0, min(__ldg(p.group_rows + g), p.rows_clip)) : p.cap;
}

// One output tile: (group or weight group, row offset, column offset) and,
// in wgrad mode, the split's k-block range.
struct Tile {
  int g, m0, n0, s, kb_lo, kb_hi;
  bool idle;   // a packing gap of the virtual schedule: no work
};

template <int TILE_M, int BN, bool WGRAD>
__device__ __forceinline__ Tile decode_tile(const Params& p, int t, int n_tiles_n,
                                            const int* prefix, const int* vstart) {
  Tile c;
  c.idle = false;
  if (!WGRAD && p.num_groups <= MAX_PACK) {
    // packed schedule: group g owns virtual slots [vstart[g], vstart[g] +
    // tiles(g)); slots past a group's tiles are gaps
    int lo = 0, hi = p.num_groups - 1;         // largest g with vstart[g] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (vstart[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const int local = t - vstart[lo];
    c.g = lo;
    c.idle = local >= (prefix[lo + 1] - prefix[lo]) * n_tiles_n;
    c.m0 = (local / n_tiles_n) * TILE_M;
    c.n0 = (local % n_tiles_n) * BN;
    c.s = 0;
    c.kb_lo = 0;
    c.kb_hi = c.idle ? 0 : (p.K + BK - 1) / BK;
    return c;
  }
  const int nt = t % n_tiles_n;
  int r = t / n_tiles_n;
  c.n0 = nt * BN;
  if (WGRAD) {
    const int m_tiles = (p.m_out + TILE_M - 1) / TILE_M;
    c.m0 = (r % m_tiles) * TILE_M;
    r /= m_tiles;
    c.g = r % p.n_wgroups;                     // weight group
    c.s = r / p.n_wgroups;                     // split
    const int tot = prefix[c.g];               // k-blocks feeding weight group g
    c.kb_lo = (int)((long long)c.s * tot / p.splits);
    c.kb_hi = (int)((long long)(c.s + 1) * tot / p.splits);
  } else {
    int lo = 0, hi = p.num_groups - 1;         // largest g with prefix[g] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= r) lo = mid;
      else hi = mid - 1;
    }
    c.g = lo;
    c.m0 = (r - prefix[lo]) * TILE_M;
    c.s = 0;
    c.kb_lo = 0;
    c.kb_hi = (p.K + BK - 1) / BK;
  }
  return c;
}

// Walk the k-blocks of a tile: in rows mode kb over K for group tc.g; in wgrad
// mode the concatenation over source groups g = w, w+W, ... of
// ceil(rows(g)/64) blocks each, restricted to [kb_lo, kb_hi).
template <bool WGRAD, typename F>
__device__ __forceinline__ void for_each_kblock(const Params& p, const Tile& tc, F&& body) {
  if (!WGRAD) {
    for (int kb = tc.kb_lo; kb < tc.kb_hi; ++kb) body(tc.g, kb);
    return;
  }
  int c = 0;
  for (int g = tc.g; g < p.num_groups && c < tc.kb_hi; g += p.n_wgroups) {
    const int nkb = (group_rows_of(p, g) + BK - 1) / BK;
    const int a = max(0, tc.kb_lo - c), b = min(nkb, tc.kb_hi - c);
    for (int kb = a; kb < b; ++kb) body(g, kb);
    c += nkb;
  }
}

// Row-per-thread results (lane = row, 4 x 16 B = 32 bf16 columns) to global
// memory through a 2 KB per-warp staging buffer: the warp transposes its
// 32 rows x 64 B so each store instruction writes 8 rows x 64 B (whole 32 B
// sectors) instead of 32 rows x 16 B (half sectors, 32 lines per
// instruction — the small-K limiter).  16-B slot u of row r sits at
// r * 4 + (u ^ ((r >> 1) & 3)): conflict-free both ways.  Rows whose bit is
// clear in `row_mask` and 8-column groups at or past `ncols` are not written.
// explicit shared-window accesses (a generic pointer here compiled to
// generic LD.E / ST.E with address-space resolution on every access)
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void stage_put(uint4* __restrict__ stg, int lane, int u, uint4 v) {
  sts128(smem_u32(stg + lane * 4 + (u ^ ((lane >> 1) & 3))), v);
}
__device__ __forceinline__ void stage_flush(const uint4* __restrict__ stg, int lane,
                                            __nv_bfloat16* row0, long long ld, uint32_t row_mask,
                                            int ncols) {
  __syncwarp();                       // every lane's row is staged
  const int j = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = (lane >> 2) + 8 * i;
    const uint4 v = lds128(smem_u32(stg + rr * 4 + (j ^ ((rr >> 1) & 3))));
    if (((row_mask >> rr) & 1u) && j * 8 < ncols) st_v4(row0 + rr * ld + j * 8, v);
  }
}
// the packed row (16-B slot u = r[4u .. 4u+3]) through the staging buffer
__device__ __forceinline__ void store_rows_staged(const uint32_t (&r)[32], uint4* __restrict__ stg,
                                                  int lane, __nv_bfloat16* row0, long long ld,
                                                  uint32_t row_mask, int ncols) {
  __syncwarp();                       // the previous flush's reads are done
#pragma unroll
  for (int u = 0; u < 4; ++u) stage_put(stg, lane, u, make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]));
  stage_flush(stg, lane, row0, ld, row_mask, ncols);
}

// bias / GELU / GELU-backward / residual -> bf16 for 32 columns of one row,
// zeros for padding rows.  The packed result replaces the accumulator in
// place (16-B slot u = r[4u .. 4u+3], already consumed); the pre-activation
// (aux_out) goes straight into this lane's staging slots `zs`.
// LEAN: no fused combine and no residual (compiled out): the training
// FFN epilogues (GELU + pre-activation store, GELU backward, zero tails)
template <bool LEAN>
__device__ __forceinline__ void epilogue_chunk(const Params& p, uint32_t (&r)[32],
                                               bool row_ok, bool pad_row, int n, const float* sb,
                                               uint4* zs, int lane, const uint4 (&pre)[4],
                                               const __nv_bfloat16* cy0 = nullptr, float cw0 = 0.f,
                                               const __nv_bfloat16* cy1 = nullptr, float cw1 = 0.f) {
  if (n >= p.N || !(row_ok || pad_row)) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int nn = n + u * 8;
    if (nn < p.N) {
      if (!row_ok) {
        r[4 * u] = r[4 * u + 1] = r[4 * u + 2] = r[4 * u + 3] = 0u;
        if (zs) stage_put(zs, lane, u, make_uint4(0, 0, 0, 0));
        continue;
      }
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[u * 8 + i]);
      if (sb) {   // this chunk's bias, staged in shared memory (warp broadcast)
        const uint4 b0u = lds128(smem_u32(sb + u * 8)), b1u = lds128(smem_u32(sb + u * 8 + 4));
        const float4 b0 = make_float4(__uint_as_float(b0u.x), __uint_as_float(b0u.y),
                                      __uint_as_float(b0u.z), __uint_as_float(b0u.w));
        const float4 b1 = make_float4(__uint_as_float(b1u.x), __uint_as_float(b1u.y),
                                      __uint_as_float(b1u.z), __uint_as_float(b1u.w));
        v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
        v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
      }
      if (p.epi == EPI_BIAS_GELU) {
        if (zs) {
          Vec16<__nv_bfloat16> z;
          z.from_float(v);
          stage_put(zs, lane, u, z.raw);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gelu_erf_fast(v[i]);
      } else if (p.epi == EPI_GELU_BWD) {
        Vec16<__nv_bfloat16> zv;
        zv.raw = pre[u];                       // pre-activation, staged load
        float z[8];
        zv.to_float(z);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_fast(z[i]);
      } else if (p.epi == EPI_MUL_AUX) {
        Vec16<__nv_bfloat16> zv;
        zv.raw = pre[u];                       // gelu'(z) saved by the forward
        float z[8];
        zv.to_float(z);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= z[i];
      }
      if (!LEAN && p.c_k) {
        // the ScMoE combine, same fp32 sequence as combine_kernel: shared
        // expert row rounded to bf16, routed rows fmaf-accumulated in
        // selection order, then se + routed, then + residual
        Vec16<__nv_bfloat16> sev;
        sev.from_float(v);
        float se[8], rt[8];
        sev.to_float(se);
#pragma unroll
        for (int i = 0; i < 8; ++i) rt[i] = 0.f;
        if (cy0) {
          Vec16<__nv_bfloat16> yv;
          yv.raw = ld_nc_v4(cy0 + nn);
          float f[8];
          yv.to_float(f);
#pragma unroll
          for (int i = 0; i < 8; ++i) rt[i] = fmaf(cw0, f[i], rt[i]);
        }
        if (cy1) {
          Vec16<__nv_bfloat16> yv;
          yv.raw = ld_nc_v4(cy1 + nn);
          float f[8];
          yv.to_float(f);
#pragma unroll
          for (int i = 0; i < 8; ++i) rt[i] = fmaf(cw1, f[i], rt[i]);
        }
        const float one = 1.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = one * se[i] + one * rt[i];
      }
      if (!LEAN && p.residual) {
        Vec16<__nv_bfloat16> rv;
        rv.raw = pre[u];                       // residual, staged load
        float rf[8];
        rv.to_float(rf);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += rf[i];
      }
      Vec16<__nv_bfloat16> ov;
      ov.from_float(v);
      r[4 * u] = ov.raw.x;
      r[4 * u + 1] = ov.raw.y;
      r[4 * u + 2] = ov.raw.z;
      r[4 * u + 3] = ov.raw.w;
    }
  }
}

// Fast epilogue for the common forward cases (no residual / aux / fused
// combine): bias and GELU are compile-time, the chunk is known to be in range,
// so the 32 values run as straight-line code — the general epilogue_chunk is
// latency-bound on per-element checks with only 8 epilogue warps per SM.
template <bool BIAS, bool GELU, bool AUX = false>
__device__ __forceinline__ void epilogue_chunk_fast(uint32_t (&r)[32],
                                                    const float* __restrict__ sb,
                                                    uint4* zs = nullptr, int lane = 0) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[u * 8 + i]);
    if (BIAS) {
      const uint4 b0u = lds128(smem_u32(sb + u * 8)), b1u = lds128(smem_u32(sb + u * 8 + 4));
      const float4 b0 = make_float4(__uint_as_float(b0u.x), __uint_as_float(b0u.y),
                                    __uint_as_float(b0u.z), __uint_as_float(b0u.w));
      const float4 b1 = make_float4(__uint_as_float(b1u.x), __uint_as_float(b1u.y),
                                    __uint_as_float(b1u.z), __uint_as_float(b1u.w));
      v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
      v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
    }
    if (GELU) {
      if (AUX) {                   // pre-activation (training), into the staging slots
        Vec16<__nv_bfloat16> z;
        z.from_float(v);
        stage_put(zs, lane, u, z.raw);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = gelu_erf_fast(v[i]);
    }
    Vec16<__nv_bfloat16> w;
    w.from_float(v);
    r[4 * u] = w.raw.x;            // in place: slots 4u..4u+3 are consumed
    r[4 * u + 1] = w.raw.y;
    r[4 * u + 2] = w.raw.z;
    r[4 * u + 3] = w.raw.w;
  }
}

// GELU backward, every column in range, no bias / residual: dZ = acc *
// gelu'(z) with z from the staged load (MUL: the staged operand already is
// gelu'(z), saved by the forward); padding rows (zero tails) get zeros
template <bool MUL>
__device__ __forceinline__ void epilogue_chunk_gelu_bwd(uint32_t (&r)[32], const uint4 (&pre)[4],
                                                        bool row_ok) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    Vec16<__nv_bfloat16> zv;
    zv.raw = pre[u];
    float z[8], v[8];
    zv.to_float(z);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = row_ok ? __uint_as_float(r[u * 8 + i]) * (MUL ? z[i] : gelu_grad_fast(z[i])) : 0.f;
    Vec16<__nv_bfloat16> w;
    w.from_float(v);
    r[4 * u] = w.raw.x;
    r[4 * u + 1] = w.raw.y;
    r[4 * u + 2] = w.raw.z;
    r[4 * u + 3] = w.raw.w;
  }
}

// residual (+ bias), every column in range: out = acc (+ b) + res, straight
// line (the general epilogue_chunk is instruction-cache bound here: the
// residual GEMMs of the training step ran ~10 us per tile slower through it)
template <bool BIAS>
__device__ __forceinline__ void epilogue_chunk_res(uint32_t (&r)[32], const float* __restrict__ sb,
                                                   const uint4 (&pre)[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[u * 8 + i]);
    if (BIAS) {
      const uint4 b0u = lds128(smem_u32(sb + u * 8)), b1u = lds128(smem_u32(sb + u * 8 + 4));
      v[0] += __uint_as_float(b0u.x); v[1] += __uint_as_float(b0u.y);
      v[2] += __uint_as_float(b0u.z); v[3] += __uint_as_float(b0u.w);
      v[4] += __uint_as_float(b1u.x); v[5] += __uint_as_float(b1u.y);
      v[6] += __uint_as_float(b1u.z); v[7] += __uint_as_float(b1u.w);
    }
    Vec16<__nv_bfloat16> rv;
    rv.raw = pre[u];
    float rf[8];
    rv.to_float(rf);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += rf[i];
    Vec16<__nv_bfloat16> w;
    w.from_float(v);
    r[4 * u] = w.raw.x;
    r[4 * u + 1] = w.raw.y;
    r[4 * u + 2] = w.raw.z;
    r[4 * u + 3] = w.raw.w;
  }
}

// fp32 wgrad partial: 32 columns of one output row
// fp32 split-K partials of 32 columns through the warp's staging buffer in
// two 16-column halves: every store instruction writes 8 rows x 64 B (whole
// sectors) instead of 32 rows x 16 B — row-per-thread stores left the
// 1-tile-per-CTA weight gradients epilogue-bound (ncu: tensor pipe 33-42%
// with the mainloop at full MMA rate)
__device__ __forceinline__ void stage_flush_f32(const uint4* __restrict__ stg, int lane,
                                                float* row0, long long ld, uint32_t row_mask,
                                                int ncols) {
  __syncwarp();                       // every lane's row is staged
  const int j = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = (lane >> 2) + 8 * i;
    const uint4 v = lds128(smem_u32(stg + rr * 4 + (j ^ ((rr >> 1) & 3))));
    if (((row_mask >> rr) & 1u) && j * 4 < ncols) st_v4(row0 + rr * ld + j * 4, v);
  }
}
__device__ __forceinline__ void epilogue_chunk_f32_staged(const uint32_t (&r)[32], bool zero,
                                                          uint4* __restrict__ stg, int lane,
                                                          float* row0, long long ld,
                                                          uint32_t row_mask, int ncols) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    __syncwarp();                     // the previous flush's reads are done
#pragma unroll
    for (int u = 0; u < 4; ++u)
      stage_put(stg, lane, u,
                zero ? make_uint4(0, 0, 0, 0)
                     : make_uint4(r[16 * h + 4 * u], r[16 * h + 4 * u + 1], r[16 * h + 4 * u + 2],
                                  r[16 * h + 4 * u + 3]));
    stage_flush_f32(stg, lane, row0 + 16 * h, ld, row_mask, ncols - 16 * h);
  }
}
__device__ __forceinline__ void epilogue_chunk_f32(const Params& p, const uint32_t (&r)[32],
                                                   bool row_ok, bool zero, long long row_off,
                                                   int n) {
  if (!row_ok || n >= p.N) return;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int nn = n + u * 4;
    if (nn < p.N) {
      uint4 v = zero ? make_uint4(0, 0, 0, 0)
                     : make_uint4(r[u * 4], r[u * 4 + 1], r[u * 4 + 2], r[u * 4 + 3]);
      st_v4(p.out_f32 + row_off + nn, v);
    }
  }
}

template <bool TWO_SM, bool B_MN, bool WGRAD, int BN, int E = EPI_WARPS>
__global__ void __launch_bounds__(Threads<E>::value, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const Params p) {
  using C = Cfg<TWO_SM, BN, E>;
  constexpr int ACC_STAGES = C::ACC_STAGES;
  constexpr int PARTS = E / 4;          // epilogue warps per TMEM lane quadrant
  constexpr int COLS_W = BN / PARTS;    // accumulator columns per epilogue warp
  constexpr int NCH = COLS_W / 32;      // 32-column chunks per epilogue warp
  // 8 warps: chunk c+1's tcgen05.ld in flight while chunk c is processed;
  // 16 warps (register cap 102): one chunk in registers, the other warps
  // hide the load latency
  constexpr bool PREFETCH = E == 8;
  constexpr bool A_MN = WGRAD;
  constexpr uint32_t IDESC = Idesc<TWO_SM, A_MN, B_MN, BN>::value;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_b + C::STAGES * C::B_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + C::STAGES;
  uint64_t* tfull_bar = bars + 2 * C::STAGES;
  uint64_t* tempty_bar = bars + 2 * C::STAGES + ACC_STAGES;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 2 * ACC_STAGES);
  int* s_prefix = reinterpret_cast<int*>(smem_b + C::STAGES * C::B_BYTES + 256);
  int* s_vstart = s_prefix + ((MAX_GROUPS + 1) * 4 + 15) / 16 * 4;
  float* s_bias = reinterpret_cast<float*>(smem_b + C::STAGES * C::B_BYTES + C::MISC);
  uint4* s_stage = reinterpret_cast<uint4*>(s_bias + E * 128);   // 2 KB per epilogue warp
  const int ring = C::STAGES - p.ld_buf;                                   // mainloop stages
  // if ld_buf (= 2): the last two ring stages are lent to the epilogue: their
  // A slots (32 KB) and B slots hold one 2 KB load buffer per (epilogue warp,
  // chunk), so a tile's whole row-major operand (residual / saved gelu') is
  // requested at the tile start, before the accumulator wait
  constexpr int LB_A = 2 * C::A_BYTES / 2048;              // buffers in the A slots
  static_assert(E * NCH <= LB_A + 2 * C::B_BYTES / 2048, "epilogue load buffers do not fit");
  uint4* s_load0 = reinterpret_cast<uint4*>(smem_a + (C::STAGES - 2) * C::A_BYTES);
  uint4* s_load1 = reinterpret_cast<uint4*>(smem_b + (C::STAGES - 2) * C::B_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = TWO_SM ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int unit = TWO_SM ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // cluster / CTA id
  const int n_units = TWO_SM ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < ACC_STAGES; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], (TWO_SM ? 2 : 1) * E);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if (TWO_SM) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, tensor-map prefetch) overlapped the previous kernel's tail;
  // no global memory is touched before the previous grid completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 3) {
    if (WGRAD) {
      // k-blocks feeding each weight group
      for (int w = lane; w < p.n_wgroups; w += 32) {
        int tot = 0;
        for (int g = w; g < p.num_groups; g += p.n_wgroups) tot += (group_rows_of(p, g) + BK - 1) / BK;
        s_prefix[w] = tot;
      }
    } else {
      // exclusive prefix of m-tiles per group (warp scan, 32 groups at a time)
      int carry = 0;
      if (lane == 0) s_prefix[0] = 0;
      for (int base = 0; base < p.num_groups; base += 32) {
        const int g = base + lane;
        int v = 0;
        if (g < p.num_groups) v = (group_rows_of(p, g) + C::TILE_M - 1) / C::TILE_M;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (g < p.num_groups) s_prefix[g + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
      // Group-aligned waves.  The persistent units take virtual slots t =
      // unit, unit + n_units, ..., so slots [w * n_units, (w+1) * n_units)
      // run together ("wave" w).  A group that fits in one wave but would
      // straddle two is moved to the next wave's start while the gaps fit in
      // the slack of the minimal wave count: its weights are then streamed
      // by one wave instead of two (the K = 8192 routed GEMM2 re-read each
      // expert's W2 in both waves it straddled: 1.42x DRAM traffic).  The
      // tile -> unit assignment never changes a tile's result.
      __syncwarp();
      if (p.num_groups <= MAX_PACK && lane == 0) {
        const int ntn = (p.N + BN - 1) / BN;
        const int units = TWO_SM ? (int)(gridDim.x >> 1) : (int)gridDim.x;
        const int total = s_prefix[p.num_groups] * ntn;
        int slack = (total + units - 1) / units * units - total;
        int v = 0;
        for (int g = 0; g < p.num_groups; ++g) {
          const int c = (s_prefix[g + 1] - s_prefix[g]) * ntn;
          const int f = v % units, gap = units - f;
          if (c > 0 && c <= units && f > 0 && c > gap && gap <= slack) {
            slack -= gap;
            v += gap;
          }
          s_vstart[g] = v;
          v += c;
        }
        s_vstart[p.num_groups] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (TWO_SM) cluster_sync();  // peer barriers initialised before any multicast arrive
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int n_tiles_n = (p.N + BN - 1) / BN;
  const int total_tiles =
      WGRAD ? p.splits * p.n_wgroups * ((p.m_out + C::TILE_M - 1) / C::TILE_M) * n_tiles_n
            : (p.num_groups <= MAX_PACK ? s_vstart[p.num_groups] : s_prefix[p.num_groups] * n_tiles_n);

  if (warp == 0) {
    // ===== TMA producer (both CTAs load their own halves) =====
    int stage = 0;
    uint32_t phase = 0;
    for (int t = unit; t < total_tiles; t += n_units) {
      const Tile tc = decode_tile<C::TILE_M, BN, WGRAD>(p, t, n_tiles_n, s_prefix, s_vstart);
      if (tc.idle) continue;
      const int am = tc.m0 + (int)rank * C::CTA_M;
      const int bn = tc.n0 + (int)rank * C::B_ROWS;
      for_each_kblock<WGRAD>(p, tc, [&](int g, int kb) {
        if (lane == 0) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full_bar[stage], (TWO_SM ? 2 : 1) * C::STAGE_BYTES);
          load_operand<TWO_SM, A_MN, C::CTA_M>(&map_a, &full_bar[stage], smem_a + stage * C::A_BYTES,
                                                kb * BK, am, g);
          load_operand<TWO_SM, B_MN, C::B_ROWS>(&map_b, &full_bar[stage],
                                                 smem_b + stage * C::B_BYTES, kb * BK, bn,
                                                 WGRAD ? g : g % p.n_wgroups);
        }
        __syncwarp();
        if (++stage == ring) {
          stage = 0;
          phase ^= 1;
        }
      });
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA only in 2SM mode) =====
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = unit; t < total_tiles; t += n_units) {
        const Tile tc = decode_tile<C::TILE_M, BN, WGRAD>(p, t, n_tiles_n, s_prefix, s_vstart);
        if (tc.idle) continue;
        const int acc = it % ACC_STAGES;
        const uint32_t acc_phase = (it / ACC_STAGES) & 1;
        const uint32_t d_tmem = tmem_base + acc * BN;
        if (lane == 0) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        __syncwarp();
        bool first = true;
        for_each_kblock<WGRAD>(p, tc, [&](int, int) {
          if (lane == 0) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem_a + stage * C::A_BYTES);
            const uint32_t b0 = smem_u32(smem_b + stage * C::B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              tc_mma<TWO_SM>(d_tmem, operand_desc<A_MN>(a0, kk), operand_desc<B_MN>(b0, kk), IDESC,
                             (first && kk == 0) ? 0u : 1u);
            }
            tc_commit<TWO_SM>(&empty_bar[stage]);
          }
          first = false;
          __syncwarp();
          if (++stage == ring) {
            stage = 0;
            phase ^= 1;
          }
        });
        if (lane == 0) tc_commit<TWO_SM>(&tfull_bar[acc]);
        __syncwarp();
        ++it;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs, each on its own 128 TMEM lanes) =====
    const int ew = warp - 4;
    const int quad = warp & 3;   // TMEM lanes [32*quad, 32*quad+32)
    const int part = ew >> 2;    // accumulator columns [COLS_W*part, COLS_W*(part+1))
    // the fast epilogue covers bias / bias+GELU stores without residual,
    // pre-activation / GELU-backward operands, zero tails or the fused combine
    const bool fast = !WGRAD && !p.residual && (!p.aux_out || p.epi == EPI_BIAS_GELU) &&
                      !p.aux_in && !p.c_k && !p.zero_tail &&
                      (p.epi == EPI_BIAS || p.epi == EPI_BIAS_GELU);
    const bool fast_gelu = p.epi == EPI_BIAS_GELU;
    const bool lean = !p.c_k && !p.residual;   // epilogue_chunk<true>: combine / residual out
    // GELU backward with the pre-activation staged through the load buffer
    const bool fast_bwd = !WGRAD && (p.epi == EPI_GELU_BWD || p.epi == EPI_MUL_AUX) && p.ld_buf &&
                          !p.bias && !p.residual && !p.aux_out && !p.c_k;
    const bool mul_aux = p.epi == EPI_MUL_AUX;
    // residual (+ bias) with the residual staged through the load buffer
    const bool fast_res = !WGRAD && p.epi == EPI_BIAS && p.residual && p.ld_buf && !p.aux_out &&
                          !p.aux_in && !p.c_k && !p.zero_tail && !(p.dbg & 4);
    int it = 0;
    for (int t = unit; t < total_tiles; t += n_units) {
      // this CTA's last tile: let the next kernel start launching (it waits in
      // griddepcontrol.wait for this grid's completion; triggering only here
      // keeps every CTA of this grid resident before any dependent CTA can be)
      if (t + n_units >= total_tiles && ew == 0 && lane == 0)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      const Tile tc = decode_tile<C::TILE_M, BN, WGRAD>(p, t, n_tiles_n, s_prefix, s_vstart);
      if (tc.idle) continue;
      const int acc = it % ACC_STAGES;
      const uint32_t acc_phase = (it / ACC_STAGES) & 1;
      ++it;
      const int row_w0 = tc.m0 + (int)rank * C::CTA_M + quad * 32;   // this warp's first row
      const int row = row_w0 + lane;
      bool row_ok, pad_row = false;
      long long row_off;
      __nv_bfloat16* orow0 = nullptr;      // row row_w0 of the output / aux
      float* frow0 = nullptr;              // wgrad: row row_w0 of this split's partial
      __nv_bfloat16* arow0 = nullptr;
      const float* brow = nullptr;
      if (WGRAD) {
        row_ok = row < p.m_out;
        row_off = (((long long)tc.s * p.n_wgroups + tc.g) * p.m_out + row) * p.N;
        frow0 = p.out_f32 + (((long long)tc.s * p.n_wgroups + tc.g) * p.m_out + row_w0) * p.N;
      } else {
        const int rows = group_rows_of(p, tc.g);
        row_ok = row < rows;
        pad_row = p.zero_tail && row < p.cap;
        row_off = ((long long)tc.g * p.cap + row) * p.N;
        const long long off0 = ((long long)tc.g * p.cap + row_w0) * p.N;
        orow0 = p.out_groups ? p.out_groups[tc.g] + (long long)row_w0 * p.N : p.out + off0;
        if (p.aux_out) arow0 = p.aux_out + off0;
        brow = p.bias ? p.bias + (long long)(tc.g % p.n_wgroups) * p.N : nullptr;
      }
      const bool empty = WGRAD && tc.kb_lo >= tc.kb_hi;   // no MMA ran: write zeros
      // stage this warp's BN/2 bias columns before waiting for the accumulator
      // (the loads overlap the MMAs; the chunk loop reads smem broadcasts)
      float* sbw = s_bias + ew * 128;
      if (!WGRAD && (brow || fast_gelu)) {   // the GELU path adds staged zeros when bias-free
        const int nb = tc.n0 + part * COLS_W + 4 * lane;
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (brow) {
          if (nb + 3 < p.N) b = *reinterpret_cast<const float4*>(brow + nb);
          else
            for (int i = 0; i < 4 && nb + i < p.N; ++i) (&b.x)[i] = brow[nb + i];
        }
        __syncwarp();        // previous tile's reads of sbw are done
        if (4 * lane < COLS_W)
          sts128(smem_u32(sbw + 4 * lane), make_uint4(__float_as_uint(b.x), __float_as_uint(b.y),
                                                      __float_as_uint(b.z), __float_as_uint(b.w)));
        __syncwarp();
      }
      // fused combine: this row's (token's) routed rows, before the wait
      const __nv_bfloat16* cy0 = nullptr;
      const __nv_bfloat16* cy1 = nullptr;
      float cw0 = 0.f, cw1 = 0.f;
      if (!WGRAD && p.c_k && row_ok) {
        const long long o = (long long)row * p.c_k;
        const int s0 = p.c_slot[o];
        if (s0 < p.c_cap) {
          cy0 = p.cy + ((long long)p.c_idx[o] * p.c_cap + s0) * p.N;
          cw0 = p.c_w[o];
        }
        if (p.c_k > 1) {
          const int s1 = p.c_slot[o + 1];
          if (s1 < p.c_cap) {
            cy1 = p.cy + ((long long)p.c_idx[o + 1] * p.c_cap + s1) * p.N;
            cw1 = p.c_w[o + 1];
          }
        }
      }
      const uint32_t wmask = __ballot_sync(0xffffffffu, row_ok || pad_row);
      uint4* stg = s_stage + ew * 128;
      // the row-major epilogue operand (residual / pre-activation / gelu'),
      // 32 rows x 64 B per chunk: coalesced cp.async into this warp's load
      // buffers (same swizzle as the store staging), every chunk of the tile
      // issued (one commit group each) before the accumulator wait, so the
      // epilogue never waits on a load issued while it was running
      const __nv_bfloat16* lsrc =
          WGRAD ? nullptr
                : (p.residual ? p.residual
                              : ((p.epi == EPI_GELU_BWD || p.epi == EPI_MUL_AUX) ? p.aux_in : nullptr));
      const uint32_t lmask = __ballot_sync(0xffffffffu, row_ok);
      auto lbuf = [&](int c) {
        const int q = ew * NCH + c;
        return q < LB_A ? s_load0 + q * 128 : s_load1 + (q - LB_A) * 128;
      };
      const long long lrow0 = ((long long)tc.g * p.cap + row_w0) * p.N;
      auto issue_load = [&](int c) __attribute__((always_inline)) {
        const int n = tc.n0 + part * COLS_W + c * 32;
        const int j = lane & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = (lane >> 2) + 8 * i;
          if (((lmask >> rr) & 1u) && n + j * 8 < p.N) {
            const uint32_t dst = smem_u32(lbuf(c) + rr * 4 + (j ^ ((rr >> 1) & 3)));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(lsrc + lrow0 + (long long)rr * p.N + n + j * 8)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      // chunk c's operand row for this lane: wait until groups 0..c landed
      // (NCH - 1 - c newer groups may still be in flight)
      auto take_load = [&](int c, uint4(&pre)[4]) __attribute__((always_inline)) {
        switch (NCH - 1 - c) {
          case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
          case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
          case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
          default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u)
          pre[u] = lds128(smem_u32(lbuf(c) + lane * 4 + (u ^ ((lane >> 1) & 3))));
      };
      if (lsrc && p.ld_buf && !(p.dbg & 2)) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");   // nothing left from the last tile
        __syncwarp();                  // the previous tile's reads of the buffers are done
#pragma unroll
        for (int c = 0; c < NCH; ++c) issue_load(c);
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      // TMEM -> registers in NCH chunks of 32 columns, chunk c+1's tcgen05.ld in
      // flight while chunk c is processed
      const uint32_t tbase =
          tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + part * COLS_W;
      uint32_t ra[32], rb[32];
      auto release_acc = [&]() __attribute__((always_inline)) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (TWO_SM) mbar_arrive_cluster_tmem(&tempty_bar[acc], 0);
          else mbar_arrive(&tempty_bar[acc]);
        }
      };
      SCMOE_TMEM_LD32(tbase, ra);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (NCH == 1) release_acc();   // the whole accumulator slice is in registers
      // one chunk: cur holds its accumulator columns, nxt receives chunk c+1's
      auto chunk = [&](auto lean_tag, int c, uint32_t(&cur)[32], uint32_t(&nxt)[32])
                       __attribute__((always_inline)) {
        if (PREFETCH) {
          if (c < NCH - 1) SCMOE_TMEM_LD32(tbase + (c + 1) * 32, nxt);
        } else if (c > 0) {
          SCMOE_TMEM_LD32(tbase + c * 32, cur);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c == NCH - 1) release_acc();
        }
        const int n = tc.n0 + part * COLS_W + c * 32;
        if (WGRAD) {
          if (n < p.N && !(p.dbg & 16))
            epilogue_chunk_f32_staged(cur, empty, stg, lane, frow0 + n, p.N, wmask, p.N - n);
          else if (p.dbg & 16)
            epilogue_chunk_f32(p, cur, row_ok, empty, row_off, n);
        } else if (fast && fast_gelu && n + 32 <= p.N) {
          // bias + GELU (+ the pre-activation store in training); plain bias
          // chunks of a partial tile take the general path below
          if (arow0) {
            __syncwarp();              // the previous flush's reads are done before z is staged
            epilogue_chunk_fast<true, true, true>(cur, sbw + c * 32, stg, lane);
            stage_flush(stg, lane, arow0 + n, p.N, wmask, 32);
          } else {
            epilogue_chunk_fast<true, true>(cur, sbw + c * 32);
          }
          store_rows_staged(cur, stg, lane, orow0 + n, p.N, wmask, 32);
        } else if (fast_bwd && n + 32 <= p.N) {
          uint4 pre[4];
          take_load(c, pre);
          if (mul_aux) epilogue_chunk_gelu_bwd<true>(cur, pre, row_ok);
          else epilogue_chunk_gelu_bwd<false>(cur, pre, row_ok);
          store_rows_staged(cur, stg, lane, orow0 + n, p.N, wmask, 32);
        } else if (fast_res && n + 32 <= p.N) {
          uint4 pre[4];
          take_load(c, pre);
          if (brow) epilogue_chunk_res<true>(cur, sbw + c * 32, pre);
          else epilogue_chunk_res<false>(cur, nullptr, pre);
          store_rows_staged(cur, stg, lane, orow0 + n, p.N, wmask, 32);
        } else if (n < p.N && wmask) {
          uint4 pre[4];
          if (p.dbg & 2) {
#pragma unroll
            for (int u = 0; u < 4; ++u) pre[u] = make_uint4(0, 0, 0, 0);
          } else if (lsrc && p.ld_buf) {
            take_load(c, pre);
          } else if (lsrc) {           // no load buffer (not expected): row-per-thread loads
#pragma unroll
            for (int u = 0; u < 4; ++u)
              pre[u] = (row_ok && n + u * 8 < p.N) ? ld_nc_v4(lsrc + row_off + n + u * 8)
                                                  : make_uint4(0, 0, 0, 0);
          }
          if (arow0) __syncwarp();   // the previous flush's reads are done before z is staged
          if (lean)
            epilogue_chunk<true>(p, cur, row_ok, pad_row, n, brow ? sbw + c * 32 : nullptr,
                                 arow0 ? stg : nullptr, lane, pre);
          else
            epilogue_chunk<false>(p, cur, row_ok, pad_row, n, brow ? sbw + c * 32 : nullptr,
                                  arow0 ? stg : nullptr, lane, pre, cy0, cw0, cy1, cw1);
          if (arow0) stage_flush(stg, lane, arow0 + n, p.N, wmask, p.N - n);
          store_rows_staged(cur, stg, lane, orow0 + n, p.N, wmask, p.N - n);
        }
        if (PREFETCH && c < NCH - 1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the whole accumulator is in registers: hand TMEM back to the MMA warp
        if (PREFETCH && c == NCH - 2) release_acc();
      };
      // Plain / bias stores with every chunk in range: straight-line code.
      // Everything else (GELU, residual, pre-activation, combine, tails):
      // chunk pairs in a rolled loop (ra / rb alternate statically) — fully
      // unrolled it overflowed the instruction cache (ncu: stall_no_inst 38%
      // of the GELU epilogue's samples).
      const bool plain = !WGRAD && fast && !fast_gelu && tc.n0 + (part + 1) * COLS_W <= p.N;
      if (plain) {
        auto plain_chunk = [&](auto bias_tag, int c, uint32_t(&cur)[32], uint32_t(&nxt)[32])
                               __attribute__((always_inline)) {
          if (PREFETCH) {
            if (c < NCH - 1) SCMOE_TMEM_LD32(tbase + (c + 1) * 32, nxt);
          } else if (c > 0) {
            SCMOE_TMEM_LD32(tbase + c * 32, cur);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (c == NCH - 1) release_acc();
          }
          const int n = tc.n0 + part * COLS_W + c * 32;
          epilogue_chunk_fast<decltype(bias_tag)::value, false>(cur, sbw + c * 32);
          store_rows_staged(cur, stg, lane, orow0 + n, p.N, wmask, 32);
          if (PREFETCH && c < NCH - 1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (PREFETCH && c == NCH - 2) release_acc();
        };
        if (brow) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (PREFETCH && (c & 1)) plain_chunk(std::true_type{}, c, rb, ra);
            else plain_chunk(std::true_type{}, c, ra, rb);
          }
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (PREFETCH && (c & 1)) plain_chunk(std::false_type{}, c, rb, ra);
            else plain_chunk(std::false_type{}, c, ra, rb);
          }
        }
      } else {
        if (PREFETCH) {
#pragma unroll 1
          for (int c = 0; c < NCH; c += 2) {
            chunk(std::true_type{}, c, ra, rb);
            if (c + 1 < NCH) chunk(std::true_type{}, c + 1, rb, ra);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < NCH; ++c) chunk(std::true_type{}, c, ra, ra);
        }
      }
    }
  }

  // rows stored into peer memory (fused expert-parallel return): each writing
  // thread fences at system scope before the kernel completes; the following
  // signal kernel then releases the ready flags
  if (!WGRAD && warp >= 4 && p.out_groups) __threadfence_system();
  tc_fence_before();
  __syncthreads();
  if (TWO_SM) cluster_sync();  // the leader's MMAs write the peer's TMEM
  if (warp == 2) {
    tc_fence_after();
    if (TWO_SM)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
  }
}

// sum of split-K partials: out[i] = sum_s part[s][i] (fp32), n multiple of 4
// (bf16 output: the parameter-dtype gradient directly, no conversion pass)
template <bool BF16OUT>
__global__ void reduce_splits_kernel(const float4* __restrict__ part, int splits, long long n4,
                                     void* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 a = part[i];
    for (int s = 1; s < splits; ++s) {
      const float4 b = part[s * n4 + i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    if (BF16OUT) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 v;
      v.x = *reinterpret_cast<const uint32_t*>(&lo);
      v.y = *reinterpret_cast<const uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[i] = v;
    } else {
      reinterpret_cast<float4*>(out)[i] = a;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D bf16 map over (inner, outer, groups) with box (64, box_outer, 1), 128B swizzle.
// K-major operands: inner = k, outer = rows (box_outer = tile rows);
// MN-major operands: inner = mn, outer = k (box_outer = 64).
int make_map(CUtensorMap* map, const void* base, int inner, int outer, int groups, int box_outer) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return SCMOE_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)groups};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)inner * 2 * (cuuint64_t)outer};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%d outer=%d groups=%d", (int)r, inner,
              outer, groups);
    return SCMOE_ERR_CUDA;
  }
  return SCMOE_OK;
}

// programmatic dependent launch of the GEMMs (1 = on; scmoe_set_gemm_flags bit 3 turns it off)
static int g_gemm_pdl = 1;

template <bool TWO_SM, bool B_MN, bool WGRAD, int BN, int E = EPI_WARPS>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, int grid,
           cudaStream_t st) {
  using C = Cfg<TWO_SM, BN, E>;
  static bool attr_set = false;
  auto kern = gemm_kernel<TWO_SM, B_MN, WGRAD, BN, E>;
  if (!attr_set) {
    SCMOE_CUDA_TRY(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Threads<E>::value);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TWO_SM ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch (the kernel waits in griddepcontrol.wait
  // before its first global access)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = g_gemm_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  SCMOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, p));
  return SCMOE_OK;
}

}  // namespace sm100

// mode: 0 auto, 1 force 1-SM, 2 force 2-SM (tests / tuning)
static int g_gemm_mode = 0;
// SMs the persistent forward / dgrad GEMMs may occupy (0 = all): while a
// peer-memory exchange kernel is in flight on the side stream, the window
// GEMMs leave its CTAs room to run concurrently instead of queueing behind
// a grid that holds every SM (one CTA per SM, 384-640 threads, ~220 KB smem)
static int g_gemm_sm_budget = 0;
static int gemm_sms() {
  const int all = num_sms();
  if (g_gemm_sm_budget <= 0 || g_gemm_sm_budget >= all) return all;
  return g_gemm_sm_budget < 2 ? 2 : (g_gemm_sm_budget & ~1);   // CTA pairs for cta_group::2
}
// tile width: 0 auto, 128 or 256 forced (tests / tuning)
static int g_gemm_bn = 0;
// tuning / experiment flags: bit 0 = no staged (cp.async) epilogue operand
// loads (row-per-thread loads instead)
static int g_gemm_flags = 0;

// Forward / dgrad tile width.  Measured on the configs[1] shapes
// (scripts/ab_gemm_cublas.py train): BN = 128 loses even where it removes a
// half-empty 256-column tile (n_out = 384: 729 vs 908 TFLOP/s) — the narrower
// MMA re-reads A from shared memory per 128 columns.  BN = 192 (K-major
// weights only) covers n_out = 384 / 1152 exactly where 256 leaves a half /
// a fifth of the last column tile idle.
static int pick_bn(int n_out, bool b_mn) {
  if (g_gemm_bn) return (g_gemm_bn == 192 && b_mn) ? 256 : g_gemm_bn;
  if (!b_mn) {
    const int w256 = (n_out + 255) / 256 * 256 - n_out, w192 = (n_out + 191) / 192 * 192 - n_out;
    if (w192 < w256) return 192;
  }
  return 256;
}

template <bool TWO_SM, bool B_MN, bool WGRAD>
static int launch_bn(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const sm100::Params& p,
                     int grid, cudaStream_t st, bool wide_epi = false) {
  if constexpr (!WGRAD) {
    if (wide_epi && bn == 256) return sm100::launch<TWO_SM, B_MN, WGRAD, 256, 16>(ma, mb, p, grid, st);
    if constexpr (!B_MN) {
      if (bn == 192) return sm100::launch<TWO_SM, B_MN, WGRAD, 192>(ma, mb, p, grid, st);
    }
  }
  return bn == 128 ? sm100::launch<TWO_SM, B_MN, WGRAD, 128>(ma, mb, p, grid, st)
                   : sm100::launch<TWO_SM, B_MN, WGRAD, 256>(ma, mb, p, grid, st);
}

// 16 epilogue warps: small-K forward / dgrad tiles (the MMA of a K <= 1024
// tile is shorter than an 8-warp epilogue of 128 x BN outputs) whose
// epilogue does elementwise work or reads a row-major operand.  Tuning hook
// g_gemm_epi: 0 auto, 8 or 16 forced.
static int g_gemm_epi = 0;
static bool wide_epilogue(int K, int epi, bool aux_out, bool residual) {
  if (g_gemm_epi) return g_gemm_epi == 16;
  return K <= 1024 && (epi != 0 || aux_out || residual);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

int grouped_gemm_bf16(const void* a, const void* wt, int b_mn, const float* bias,
                      const void* residual, const void* aux_in, void* aux_out, void* out,
                      int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                      int rows_clip, int N, int K, int epi, int zero_tail, cudaStream_t st,
                      const CombineSpec* cs, void* const* out_groups) {
  using namespace sm100;
  SCMOE_CHECK_ARG(num_groups <= MAX_GROUPS, "num_groups=%d exceeds %d", num_groups, MAX_GROUPS);
  SCMOE_CHECK_ARG(K % 8 == 0 && N % 8 == 0, "bf16 GEMM needs k_in and n_out multiples of 8");
  SCMOE_CHECK_ARG(aligned16(a) && aligned16(wt) && aligned16(out) && aligned16(bias) &&
                      aligned16(residual) && aligned16(aux_in) && aligned16(aux_out),
                  "GEMM operands must be 16-byte aligned");
  SCMOE_CHECK_ARG((epi != EPI_GELU_BWD && epi != EPI_MUL_AUX) || aux_in,
                  "GELU backward needs the pre-activation / the saved gelu'");
  Params p = {};
  p.num_groups = num_groups;
  p.n_wgroups = n_wgroups;
  p.cap = cap;
  p.rows_clip = rows_clip;
  p.N = N;
  p.K = K;
  p.epi = epi;
  p.zero_tail = zero_tail;
  p.group_rows = group_rows;
  p.bias = bias;
  p.residual = (const __nv_bfloat16*)residual;
  p.aux_in = (const __nv_bfloat16*)aux_in;
  p.aux_out = (__nv_bfloat16*)aux_out;
  p.out = (__nv_bfloat16*)out;
  p.out_groups = (__nv_bfloat16* const*)out_groups;
  p.ld_buf = (residual || ((epi == EPI_GELU_BWD || epi == EPI_MUL_AUX) && aux_in)) &&
                     !(g_gemm_flags & 1) ? 2 : 0;
  p.dbg = g_gemm_flags;
  if (cs) {
    SCMOE_CHECK_ARG(num_groups == 1 && epi == EPI_BIAS && cs->k >= 1 && cs->k <= 2 && cs->y &&
                        cs->indices && cs->slots && cs->weights && cs->capacity >= 1 &&
                        aligned16(cs->y),
                    "fused combine: one group, bias epilogue, k <= 2");
    p.cy = (const __nv_bfloat16*)cs->y;
    p.c_idx = cs->indices;
    p.c_slot = cs->slots;
    p.c_w = cs->weights;
    p.c_cap = cs->capacity;
    p.c_k = cs->k;
  }
  const int sms = gemm_sms();
  auto tiles_of = [&](int tile_m, int bn) {
    return (long long)num_groups * ((cap + tile_m - 1) / tile_m) * ((N + bn - 1) / bn);
  };
  const bool two = g_gemm_mode == 2 || (g_gemm_mode == 0 && tiles_of(256, 256) >= sms / 2);
  const int tile_m = two ? 256 : 128;
  const long long max_units = two ? sms / 2 : sms;
  const int bn = pick_bn(N, b_mn != 0);
  const long long tiles = tiles_of(tile_m, bn);
  const long long units = tiles < max_units ? tiles : max_units;
  if (units <= 0) return SCMOE_OK;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, a, K, cap, num_groups, Cfg<true>::CTA_M);
  if (rc) return rc;
  const int b_rows = two ? bn / 2 : bn;
  rc = b_mn ? make_map(&mb, wt, N, K, n_wgroups, BK) : make_map(&mb, wt, K, N, n_wgroups, b_rows);
  if (rc) return rc;
  // 16 epilogue warps split a 256-column tile in 64-column parts; the
  // 192-column tile stays on 8 (96 columns each)
  const bool wide = !cs && !out_groups && bn == 256 &&
                    wide_epilogue(K, epi, aux_out != nullptr, residual != nullptr);
  if (two)
    rc = b_mn ? launch_bn<true, true, false>(bn, ma, mb, p, (int)units * 2, st, wide)
              : launch_bn<true, false, false>(bn, ma, mb, p, (int)units * 2, st, wide);
  else
    rc = b_mn ? launch_bn<false, true, false>(bn, ma, mb, p, (int)units, st, wide)
              : launch_bn<false, false, false>(bn, ma, mb, p, (int)units, st, wide);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

size_t wgrad_workspace_bytes(int n_wgroups, int m_out, int n_out, int splits) {
  return splits > 1 ? (size_t)splits * n_wgroups * m_out * n_out * sizeof(float) : 0;
}

// out is fp32, or bf16 when out_bf16 (then the fp32 result always goes
// through the workspace: at least one split's worth)
int grouped_wgrad_bf16(const void* a, const void* b, void* out, void* ws, size_t ws_bytes,
                       int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                       int rows_clip, int m_out, int n_out, int splits, cudaStream_t st,
                       bool out_bf16) {
  using namespace sm100;
  SCMOE_CHECK_ARG(num_groups <= MAX_GROUPS, "num_groups=%d exceeds %d", num_groups, MAX_GROUPS);
  SCMOE_CHECK_ARG(m_out % 8 == 0 && n_out % 8 == 0, "wgrad needs m_out, n_out multiples of 8");
  SCMOE_CHECK_ARG(aligned16(a) && aligned16(b) && aligned16(out) && aligned16(ws),
                  "wgrad operands must be 16-byte aligned");
  const int sms = gemm_sms();          // honours the SM budget (concurrent backward GEMMs)
  // Tile shape: 2-SM 256x256 when the outputs alone fill the CTA pairs
  // (configs[2]-size weights); small weights (configs[1]: 384 / 1152 / 1536
  // wide) run split-K on 1-SM 128x128 tiles with 4 accumulator stages — the
  // fastest of the four shapes on every configs[1] weight (scripts/ab_wgrad.py:
  // 546-610 TFLOP/s vs 458-591).
  // (2-SM 256x256 for the configs[1] weights too: within +-3% of 1-SM
  // 128x128 in interleaved A/B, scripts/ab_wgrad.py — not adopted)
  const long long tiles_big = (long long)n_wgroups * ((m_out + 255) / 256) * ((n_out + 255) / 256);
  const bool two = g_gemm_mode == 2 || (g_gemm_mode == 0 && tiles_big >= sms / 2);
  const int tile_m = two ? 256 : 128;
  const int bn = g_gemm_bn ? g_gemm_bn : (two ? 256 : 128);
  const long long max_units = two ? sms / 2 : sms;
  const long long tiles1 =
      (long long)n_wgroups * ((m_out + tile_m - 1) / tile_m) * ((n_out + bn - 1) / bn);
  if (splits <= 0) {
    // fill the persistent units in ONE wave: floor(units / tiles) splits of
    // the token reduction (rounding up left a second wave of a few tiles)
    const long long kb_guess = ((long long)num_groups / n_wgroups) * ((cap + BK - 1) / BK);
    long long s = max_units / tiles1;
    if (s > kb_guess / 4) s = kb_guess / 4;
    splits = (int)(s < 1 ? 1 : (s > 64 ? 64 : s));
  }
  const size_t one_split = (size_t)n_wgroups * m_out * n_out * sizeof(float);
  SCMOE_CHECK_ARG(ws_bytes >= ((splits > 1 || out_bf16) ? (size_t)splits * one_split : 0),
                  "wgrad workspace too small for %d splits", splits);
  Params p = {};
  p.num_groups = num_groups;
  p.n_wgroups = n_wgroups;
  p.cap = cap;
  p.rows_clip = rows_clip;
  p.N = n_out;
  p.m_out = m_out;
  p.splits = splits;
  p.group_rows = group_rows;
  p.out_f32 = (splits > 1 || out_bf16) ? (float*)ws : (float*)out;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, a, m_out, cap, num_groups, BK);
  if (rc) return rc;
  rc = make_map(&mb, b, n_out, cap, num_groups, BK);
  if (rc) return rc;
  const long long units_all = tiles1 * splits;
  const long long units = units_all < max_units ? units_all : max_units;
  rc = two ? launch_bn<true, true, true>(bn, ma, mb, p, (int)units * 2, st)
           : launch_bn<false, true, true>(bn, ma, mb, p, (int)units, st);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  if (splits > 1 || out_bf16) {
    const long long n4 = (long long)n_wgroups * m_out * n_out / 4;
    if (out_bf16)
      reduce_splits_kernel<true><<<sms * 4, 256, 0, st>>>((const float4*)ws, splits, n4, out);
    else
      reduce_splits_kernel<false><<<sms * 4, 256, 0, st>>>((const float4*)ws, splits, n4, out);
    SCMOE_LAUNCH_CHECK();
  }
  return SCMOE_OK;
}

// 2-D bf16 map over a row-major (outer, inner) matrix with row stride
// row_stride_bytes, box (64, box_outer), 128B swizzle, OOB zero fill (used by
// the tensor-core gate's token stages).
int make_map_2d(CUtensorMap* map, const void* base, int inner, int outer,
                long long row_stride_bytes, int box_outer) {
  auto fn = sm100::encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return SCMOE_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%d outer=%d", (int)r, inner, outer);
    return SCMOE_ERR_CUDA;
  }
  return SCMOE_OK;
}

}  // namespace scmoe

extern "C" int scmoe_set_gemm_flags(int flags) {
  scmoe::g_gemm_flags = flags;
  scmoe::sm100::g_gemm_pdl = (flags & 8) ? 0 : 1;
  return SCMOE_OK;
}

extern "C" int scmoe_set_gemm_mode(int mode) {
  if (mode < 0 || mode > 2) {
    scmoe::set_error("gemm mode must be 0 (auto), 1 (1-SM) or 2 (2-SM)");
    return SCMOE_ERR_ARG;
  }
  scmoe::g_gemm_mode = mode;
  return SCMOE_OK;
}

extern "C" int scmoe_set_gemm_sm_budget(int sms) {
  if (sms < 0) {
    scmoe::set_error("gemm SM budget must be >= 0 (0 = all SMs)");
    return SCMOE_ERR_ARG;
  }
  scmoe::g_gemm_sm_budget = sms;
  return SCMOE_OK;
}

extern "C" int scmoe_set_gemm_epilogue_warps(int e) {
  if (e != 0 && e != 8 && e != 16) {
    scmoe::set_error("gemm epilogue warps must be 0 (auto), 8 or 16");
    return SCMOE_ERR_ARG;
  }
  scmoe::g_gemm_epi = e;
  return SCMOE_OK;
}

extern "C" int scmoe_set_gemm_tile_n(int bn) {
  if (bn != 0 && bn != 128 && bn != 192 && bn != 256) {
    scmoe::set_error("gemm tile width must be 0 (auto), 128, 192 or 256");
    return SCMOE_ERR_ARG;
  }
  scmoe::g_gemm_bn = bn;
  return SCMOE_OK;
}
