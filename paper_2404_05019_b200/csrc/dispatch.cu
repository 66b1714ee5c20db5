// K2 dispatch ("encode") and K5 combine ("decode"), the HBM-bound halves of
// the routed path, and their expert-parallel forms over peer memory (K9/K10).
// One warp per token, 16-byte vector accesses, every row streamed once.
//
// Reference semantics (relative to /root/reference/pkg/src/scmoelab/):
//   the reference evaluates experts densely and never permutes
//   (arch.py:418-433); dispatch is the sparse equivalent of "expert i sees the
//   rows whose kept weight is non-zero".  combine reproduces
//   routed = sum_j w_j * keep_j * E_{e_j}(x) (arch.py:481-483, 418-433),
//   combine(se, routed, x) (arch.py:380-392) and the block residual add
//   (arch.py:616).
//
// Expert parallelism over NVLink / NVSwitch peer memory: the
// rows of global expert e = r*E_l + el live on rank r.  Every rank owns a
// receive buffer recv (G_src, E_l, C, d) and an output buffer y (same layout)
// that every peer can address (symmetric memory).  The P2P dispatch writes
// each kept row of source rank `rank` straight into
//   recv_r[(rank*E_l + el)*C + slot]
// on the owner (NVLink stores from the SMs — no staging buffer, no padded
// equal-split all-to-all: only kept rows move), publishes the kept counts into
// the owner's recv_counts[rank*E_l + el], then releases an epoch flag in every
// peer.  The owner's grouped FFN waits for all source flags, runs, and
// releases a y-ready flag; the P2P combine gathers each token's expert rows
// straight from y_r on the owner (NVLink loads) fused with the shared expert,
// combination gate and residual.  Flags carry a per-rank epoch counter kept in
// device memory, so the sequence is CUDA-graph safe.
#include "common.cuh"

namespace scmoe {
namespace {

constexpr int WARPS = 8;

// Row addressing of the capacity-slotted (expert, slot) space.
template <typename T>
struct LocalRows {        // one (E, C, d) buffer on this GPU
  T* base;
  int cap, d;
  __device__ __forceinline__ T* row(int e, int s) const {
    return base + ((long long)e * cap + s) * d;
  }
};
template <typename T>
struct PeerRows {         // per-rank (G_src, E_l, C, d) buffers, this rank's block
  T* const* peers;        // device array [world] of peer base pointers
  int rank, e_local, cap, d;
  __device__ __forceinline__ T* row(int e, int s) const {
    const int r = e / e_local, el = e - r * e_local;
    return peers[r] + ((long long)(rank * e_local + el) * cap + s) * d;
  }
};

// Copy token rows to every kept (expert, slot) row of `dst` (optionally scaled
// — the combine backward).  Grid-stride over tokens, warp per token.
template <typename T, int KMAX, class Dst>
__device__ __forceinline__ void dispatch_rows(const T* __restrict__ x, long long ld_x, int n_tok,
                                              int d, int k, const int32_t* __restrict__ indices,
                                              const int32_t* __restrict__ slots, int cap,
                                              const float* __restrict__ row_scale, const Dst& dst) {
  constexpr int VEC = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  for (long long t = (long long)blockIdx.x * WARPS + (threadIdx.x >> 5); t < n_tok;
       t += (long long)gridDim.x * WARPS) {
    // per-selection destinations in registers (KMAX-unrolled; dropped -> null)
    T* dp[KMAX];
    float scl[KMAX];
    bool any = false;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      dp[j] = nullptr;
      scl[j] = 1.f;
      if (j < k) {
        const int s = slots[t * k + j];
        if (s < cap) {
          dp[j] = dst.row(indices[t * k + j], s);
          if (row_scale) scl[j] = row_scale[t * k + j];
          any = true;
        }
      }
    }
    if (!any) continue;
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
            if (!dp[q]) continue;
            if (row_scale) {
              // combine backward: d expert_out[e, slot] = w * d_out[t]
              Vec16<T> iv, ov;
              iv.raw = v[u];
              float f[VEC];
              iv.to_float(f);
#pragma unroll
              for (int i = 0; i < VEC; ++i) f[i] *= scl[q];
              ov.from_float(f);
              st_v4(dp[q] + cc, ov.raw);
            } else {
              st_v4(dp[q] + cc, v[u]);
            }
          }
        }
      }
    }
  }
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(WARPS * 32) dispatch_kernel(
    const T* __restrict__ x, long long ld_x, int n_tok, int d, int k,
    const int32_t* __restrict__ indices, const int32_t* __restrict__ slots, int cap,
    const float* __restrict__ row_scale, T* __restrict__ buf) {
  dispatch_rows<T, KMAX>(x, ld_x, n_tok, d, k, indices, slots, cap, row_scale,
                         LocalRows<T>{buf, cap, d});
}

// ---- K2 via the TMA bulk-copy engine ------------------------------------------
// The permutation is pure data movement of whole rows (d*s bytes, contiguous
// at both ends), so the copy engine does it: one elected thread per CTA pulls
// token rows into a shared-memory ring with cp.async.bulk (global -> shared,
// mbarrier completion) and pushes each row to every kept (expert, slot) row
// with cp.async.bulk (shared -> global, bulk groups).  No register staging;
// CTA c streams a contiguous range of tokens.

__device__ __forceinline__ uint32_t bk_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bk_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nBK_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra BK_WAIT_%=;\n}\n" ::"r"(bk_smem(bar)), "r"(parity) : "memory");
}

constexpr int BK_SLOTS = 8;      // rows in flight per CTA
constexpr int BK_LAG = 4;        // store groups allowed in flight before a slot is reused

template <int KMAX>
__global__ void __launch_bounds__(32) dispatch_bulk_kernel(
    const uint8_t* __restrict__ x, long long ld_bytes, int n_tok, int row_bytes, int k,
    const int32_t* __restrict__ indices, const int32_t* __restrict__ slots, int cap,
    uint8_t* __restrict__ buf) {
  extern __shared__ __align__(128) uint8_t bk_ring[];
  __shared__ __align__(8) uint64_t bars[BK_SLOTS];
  if (threadIdx.x != 0) return;
  const int per = (n_tok + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(n_tok, t0 + per);
  if (t0 >= t1) return;
  for (int i = 0; i < BK_SLOTS; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bk_smem(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto kept = [&](long long t) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k) any |= slots[t * k + j] < cap;
    return any;
  };
  auto load = [&](int t, int slot) {
    if (!kept(t)) return;
    uint64_t* bar = &bars[slot];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(bk_smem(bar)), "r"(row_bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(bk_smem(bk_ring + (size_t)slot * row_bytes)), "l"(x + (long long)t * ld_bytes),
          "r"(row_bytes), "r"(bk_smem(bar))
        : "memory");
  };
  const int n = t1 - t0;
  uint32_t phase_bits = 0;                 // parity per slot
  for (int i = 0; i < min(n, BK_SLOTS); ++i) load(t0 + i, i);
  for (int i = 0; i < n; ++i) {
    const int t = t0 + i, slot = i % BK_SLOTS;
    if (kept(t)) {
      bk_wait(&bars[slot], (phase_bits >> slot) & 1u);
      phase_bits ^= 1u << slot;
      const uint8_t* row = bk_ring + (size_t)slot * row_bytes;
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < k) {
          const int s = slots[(long long)t * k + j];
          if (s < cap) {
            uint8_t* dst = buf + ((long long)indices[(long long)t * k + j] * cap + s) * row_bytes;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst), "r"(bk_smem(row)), "r"(row_bytes) : "memory");
          }
        }
      }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // reuse the slot of token i - BK_LAG once its stores have read shared memory
    const int r = i - BK_LAG;
    if (r >= 0 && r + BK_SLOTS < n) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(BK_LAG) : "memory");
      load(t0 + r + BK_SLOTS, r % BK_SLOTS);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- peer-memory signalling -------------------------------------------------
// flags (per rank, symmetric): [0][src] = dispatch epoch received from src,
// [1][owner] = y-ready / rows-returned epoch received from owner.  epoch_ctr
// (per rank, local): [0] = epoch of the last completed dispatch, [1] / [2] =
// CTA arrival counters of the dispatch / return kernels.

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr long long SPIN_LIMIT_CYCLES = 40LL * 1000 * 1000 * 1000;   // ~20 s, then trap

template <typename T, int KMAX>
__global__ void __launch_bounds__(WARPS * 32) ep_dispatch_p2p_kernel(
    const T* __restrict__ x, long long ld_x, int n_tok, int d, int k,
    const int32_t* __restrict__ indices, const int32_t* __restrict__ slots,
    const int32_t* __restrict__ counts, int cap, int world, int rank, int e_local,
    T* const* __restrict__ peer_recv, int32_t* const* __restrict__ peer_counts,
    uint32_t* const* __restrict__ peer_flags, uint32_t* __restrict__ epoch_ctr) {
  __shared__ bool s_last;
  const uint32_t epoch = epoch_ctr[0] + 1u;   // read before this CTA's arrival below
  dispatch_rows<T, KMAX>(x, ld_x, n_tok, d, k, indices, slots, cap, nullptr,
                         PeerRows<T>{peer_recv, rank, e_local, cap, d});
  if (blockIdx.x == 0) {
    // kept rows of every global expert -> owner's recv_counts[rank*E_l + el]
    for (int e = threadIdx.x; e < world * e_local; e += blockDim.x) {
      const int r = e / e_local, el = e - r * e_local;
      peer_counts[r][rank * e_local + el] = min(counts[e], cap);
    }
  }
  __threadfence_system();          // this CTA's peer stores before its arrival
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&epoch_ctr[1], 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    for (int r = threadIdx.x; r < world; r += blockDim.x) st_release_sys(peer_flags[r] + rank, epoch);
    if (threadIdx.x == 0) {
      epoch_ctr[1] = 0;
      epoch_ctr[0] = epoch;
    }
  }
}

// Wait until every peer's flag `which` (0 dispatch, 1 y-ready) reached this
// rank's current epoch.  Traps after ~20 s instead of hanging the GPU.
__global__ void ep_wait_kernel(const uint32_t* __restrict__ flags, int which, int world,
                               const uint32_t* __restrict__ epoch_ctr) {
  const uint32_t epoch = epoch_ctr[0];
  for (int s = threadIdx.x; s < world; s += blockDim.x) {
    const long long t0 = clock64();
    while (ld_acquire_sys(flags + which * world + s) < epoch) {
      __nanosleep(128);
      if (clock64() - t0 > SPIN_LIMIT_CYCLES) __trap();
    }
  }
  __syncthreads();
}

// Release this rank's flag `which` in every peer (1: after the grouped FFN).
__global__ void ep_signal_kernel(uint32_t* const* __restrict__ peer_flags, int which, int world,
                                 int rank, const uint32_t* __restrict__ epoch_ctr) {
  __threadfence_system();
  const uint32_t epoch = epoch_ctr[0];
  for (int r = threadIdx.x; r < world; r += blockDim.x)
    st_release_sys(peer_flags[r] + which * world + rank, epoch);
}

// Return trip, push form: the owner stores the valid rows of y (rows <
// recv_counts[g] of every group g = (src, el)) straight into
//   back_src[(rank*E_l + el)*C + row]
// on the source rank, then releases flags_src[1][rank].  back has the layout
// of the local dispatch buffer (E, C, d), so the source runs the plain combine.
// Launched on a side stream it overlaps the window ops after the expert slot.
template <typename T>
__global__ void __launch_bounds__(WARPS * 32) ep_return_p2p_kernel(
    const T* __restrict__ y, const int32_t* __restrict__ recv_counts, int cap, int d, int world,
    int rank, int e_local, T* const* __restrict__ peer_back,
    uint32_t* const* __restrict__ peer_flags, uint32_t* __restrict__ epoch_ctr) {
  constexpr int VEC = Vec16<T>::N;
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)world * e_local * cap;
  for (long long i = (long long)blockIdx.x * WARPS + (threadIdx.x >> 5); i < rows;
       i += (long long)gridDim.x * WARPS) {
    const int g = (int)(i / cap), row = (int)(i - (long long)g * cap);
    if (row >= min(recv_counts[g], cap)) continue;
    const int src = g / e_local, el = g - src * e_local;
    const T* from = y + i * d;
    T* to = peer_back[src] + ((long long)(rank * e_local + el) * cap + row) * d;
    constexpr int U = 8;
    for (int c = lane * VEC; c < d; c += 32 * VEC * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + u * 32 * VEC;
        if (cc < d) v[u] = ld_nc_v4(from + cc);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + u * 32 * VEC;
        if (cc < d) st_v4(to + cc, v[u]);
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&epoch_ctr[2], 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    const uint32_t epoch = epoch_ctr[0];
    for (int r = threadIdx.x; r < world; r += blockDim.x)
      st_release_sys(peer_flags[r] + world + rank, epoch);
    if (threadIdx.x == 0) epoch_ctr[2] = 0;
  }
}

// ---- combine ----------------------------------------------------------------

template <typename T, int MODE, bool HAS_SE, bool HAS_RES, int KMAX, class Src>
__global__ void __launch_bounds__(WARPS * 32) combine_kernel(
    const T* __restrict__ se, const Src ysrc, const T* __restrict__ xcur,
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

  // kept selections in registers (KMAX-unrolled; dropped -> null)
  const T* yp[KMAX];
  float wt[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    yp[j] = nullptr;
    wt[j] = 0.f;
    if (j < k) {
      const int s = slots[t * k + j];
      if (s < cap) {
        yp[j] = ysrc.row(indices[t * k + j], s);
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
        yv[u][q] = (in && yp[q]) ? ld_nc_v4(yp[q] + c) : make_uint4(0, 0, 0, 0);
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

template <typename T, int MODE, int KMAX, class Src>
void launch_combine_k(const T* se, const Src& y, const T* xc, const float* wcg, const T* res,
                      const int32_t* idx, const int32_t* sl, const float* w, int cap, int n, int d,
                      int k, T* out, cudaStream_t st) {
  const int grid = (n + WARPS - 1) / WARPS;
  if (se && res)
    combine_kernel<T, MODE, true, true, KMAX, Src><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else if (se)
    combine_kernel<T, MODE, true, false, KMAX, Src><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else if (res)
    combine_kernel<T, MODE, false, true, KMAX, Src><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
  else
    combine_kernel<T, MODE, false, false, KMAX, Src><<<grid, WARPS * 32, 0, st>>>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out);
}

template <typename T, int MODE, class Src>
void launch_combine_mode(const T* se, const Src& y, const T* xc, const float* wcg, const T* res,
                         const int32_t* idx, const int32_t* sl, const float* w, int cap, int n,
                         int d, int k, T* out, cudaStream_t st) {
  if (k == 1)
    launch_combine_k<T, MODE, 1>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
  else if (k == 2)
    launch_combine_k<T, MODE, 2>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
  else
    launch_combine_k<T, MODE, SCMOE_MAX_K>(se, y, xc, wcg, res, idx, sl, w, cap, n, d, k, out, st);
}

template <typename T, class Src>
void launch_combine(int mode, const void* se, const Src& y, const void* xc, const float* wcg,
                    const void* res, const int32_t* idx, const int32_t* sl, const float* w,
                    int cap, int n, int d, int k, void* out, cudaStream_t st) {
  const T *se_ = (const T*)se, *xc_ = (const T*)xc, *res_ = (const T*)res;
  if (mode == SCMOE_COMBINE_CG1)
    launch_combine_mode<T, SCMOE_COMBINE_CG1>(se_, y, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
  else if (mode == SCMOE_COMBINE_CG2)
    launch_combine_mode<T, SCMOE_COMBINE_CG2>(se_, y, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
  else
    launch_combine_mode<T, SCMOE_COMBINE_DIRECT_ADD>(se_, y, xc_, wcg, res_, idx, sl, w, cap, n, d, k, (T*)out, st);
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

// Testing hooks: 1 routes scmoe_dispatch through the register-staged kernel;
// CTAs per SM of the bulk-copy kernel.
extern "C" int scmoe_dispatch_force_ldst = 0;
extern "C" int scmoe_dispatch_bulk_ctas_per_sm = 16;   // measured: 1x 45, 4x 31, 16x 28.7 us (= ldst)

extern "C" int scmoe_dispatch(const void* x, int dtype, long long ld_x, int n_tokens,
                              int d_model, int k, const int32_t* indices, const int32_t* slots,
                              int capacity, void* dispatch_buf, void* stream) {
  using namespace scmoe;
  const int esz = dtype == SCMOE_BF16 ? 2 : 4;
  const long long row_bytes = (long long)d_model * esz;
  if (scmoe_dispatch_force_ldst || n_tokens <= 0 || (dtype != SCMOE_BF16 && dtype != SCMOE_F32) ||
      k < 1 || k > SCMOE_MAX_K || capacity < 1 || row_bytes % 16 || (ld_x * esz) % 16 ||
      row_bytes * BK_SLOTS > 96 * 1024 || !aligned16(x) || !aligned16(dispatch_buf))
    return scmoe_dispatch_scaled(x, dtype, ld_x, n_tokens, d_model, k, indices, slots, capacity,
                                 nullptr, dispatch_buf, stream);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = (size_t)row_bytes * BK_SLOTS;
  static size_t smem_set[3] = {0, 0, 0};
  const int kk = k == 1 ? 0 : (k == 2 ? 1 : 2);
  if (smem > 48 * 1024 && smem > smem_set[kk]) {
    if (k == 1) SCMOE_CUDA_TRY(cudaFuncSetAttribute(dispatch_bulk_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    else if (k == 2) SCMOE_CUDA_TRY(cudaFuncSetAttribute(dispatch_bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    else SCMOE_CUDA_TRY(cudaFuncSetAttribute(dispatch_bulk_kernel<SCMOE_MAX_K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    smem_set[kk] = 96 * 1024;
  }
  // enough CTAs for the copy engines of every SM, few enough that each CTA
  // streams a long contiguous token range
  const int grid = min(n_tokens, num_sms() * max(1, scmoe_dispatch_bulk_ctas_per_sm));
#define SCMOE_BULK(KM)                                                                          \
  dispatch_bulk_kernel<KM><<<grid, 32, smem, st>>>((const uint8_t*)x, ld_x * esz, n_tokens,      \
                                                   (int)row_bytes, k, indices, slots, capacity, \
                                                   (uint8_t*)dispatch_buf)
  if (k == 1) SCMOE_BULK(1);
  else if (k == 2) SCMOE_BULK(2);
  else SCMOE_BULK(SCMOE_MAX_K);
#undef SCMOE_BULK
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
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
    launch_combine<__nv_bfloat16>(
        mode, se_out, LocalRows<const __nv_bfloat16>{(const __nv_bfloat16*)expert_out, capacity, d_model},
        x_cur, w_cg, residual, indices, slots, weights, capacity, n_tokens, d_model, k, out, st);
  else
    launch_combine<float>(mode, se_out, LocalRows<const float>{(const float*)expert_out, capacity, d_model},
                          x_cur, w_cg, residual, indices, slots, weights, capacity, n_tokens,
                          d_model, k, out, st);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

// ---- K9 / K10: expert parallelism over peer memory -----------------------------

extern "C" int scmoe_ep_dispatch_p2p(const void* x, int dtype, long long ld_x, int n_tokens,
                                     int d_model, int k, const int32_t* indices,
                                     const int32_t* slots, const int32_t* counts, int capacity,
                                     int world, int rank, int experts_per_rank,
                                     void* const* peer_recv, int32_t* const* peer_recv_counts,
                                     uint32_t* const* peer_flags, uint32_t* epoch_ctr,
                                     int max_ctas, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16 || dtype == SCMOE_F32, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(k >= 1 && k <= SCMOE_MAX_K, "k=%d out of range", k);
  SCMOE_CHECK_ARG(capacity >= 1, "capacity must be >= 1");
  SCMOE_CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "rank %d / world %d", rank, world);
  SCMOE_CHECK_ARG(experts_per_rank >= 1 && world * experts_per_rank <= SCMOE_MAX_EXPERTS,
                  "experts_per_rank=%d", experts_per_rank);
  SCMOE_CHECK_ARG(peer_recv && peer_recv_counts && peer_flags && epoch_ctr && counts,
                  "null peer table / counter");
  const int vec = dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0 && ld_x % vec == 0, "d_model/ld_x must be multiples of %d", vec);
  SCMOE_CHECK_ARG(aligned16(x), "x must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  int grid = (max(n_tokens, 1) + WARPS - 1) / WARPS;
  if (max_ctas > 0) grid = min(grid, max_ctas);
#define SCMOE_EPD(T, KM)                                                                           \
  ep_dispatch_p2p_kernel<T, KM><<<grid, WARPS * 32, 0, st>>>(                                     \
      (const T*)x, ld_x, n_tokens, d_model, k, indices, slots, counts, capacity, world, rank,     \
      experts_per_rank, (T* const*)peer_recv, peer_recv_counts, peer_flags, epoch_ctr)
  if (dtype == SCMOE_BF16) {
    if (k == 1) SCMOE_EPD(__nv_bfloat16, 1);
    else if (k == 2) SCMOE_EPD(__nv_bfloat16, 2);
    else SCMOE_EPD(__nv_bfloat16, SCMOE_MAX_K);
  } else {
    if (k == 1) SCMOE_EPD(float, 1);
    else if (k == 2) SCMOE_EPD(float, 2);
    else SCMOE_EPD(float, SCMOE_MAX_K);
  }
#undef SCMOE_EPD
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_ep_wait(const uint32_t* flags, int which, int world,
                             const uint32_t* epoch_ctr, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(which == 0 || which == 1, "which must be 0 (dispatch) or 1 (y ready)");
  SCMOE_CHECK_ARG(world >= 1 && flags && epoch_ctr, "bad flags / world");
  ep_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flags, which, world, epoch_ctr);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_ep_signal(uint32_t* const* peer_flags, int which, int world, int rank,
                               const uint32_t* epoch_ctr, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(which == 0 || which == 1, "which must be 0 (dispatch) or 1 (y ready)");
  SCMOE_CHECK_ARG(world >= 1 && rank >= 0 && rank < world && peer_flags && epoch_ctr,
                  "bad flags / rank");
  ep_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(peer_flags, which, world, rank, epoch_ctr);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_ep_combine_p2p(const void* se_out, const void* const* peer_y,
                                    const void* x_cur, const float* w_cg, int mode,
                                    const void* residual, const int32_t* indices,
                                    const int32_t* slots, const float* weights, int capacity,
                                    int n_tokens, int d_model, int k, int dtype, int world,
                                    int rank, int experts_per_rank, void* out, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(mode >= 0 && mode <= 2, "bad combine mode %d", mode);
  SCMOE_CHECK_ARG(mode == SCMOE_COMBINE_DIRECT_ADD || (w_cg && x_cur && se_out),
                  "CG modes need w_cg, x_cur and se_out");
  SCMOE_CHECK_ARG(k >= 1 && k <= SCMOE_MAX_K, "k=%d out of range", k);
  SCMOE_CHECK_ARG(world >= 1 && rank >= 0 && rank < world && experts_per_rank >= 1 && peer_y,
                  "bad peer table / rank");
  const int vec = dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0, "d_model must be a multiple of %d", vec);
  SCMOE_CHECK_ARG(aligned16(out) && (!se_out || aligned16(se_out)) &&
                      (!residual || aligned16(residual)) && (!x_cur || aligned16(x_cur)),
                  "buffers must be 16-byte aligned");
  if (n_tokens <= 0) return SCMOE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SCMOE_BF16)
    launch_combine<__nv_bfloat16>(
        mode, se_out,
        PeerRows<const __nv_bfloat16>{(const __nv_bfloat16* const*)peer_y, rank, experts_per_rank,
                                      capacity, d_model},
        x_cur, w_cg, residual, indices, slots, weights, capacity, n_tokens, d_model, k, out, st);
  else
    launch_combine<float>(mode, se_out,
                          PeerRows<const float>{(const float* const*)peer_y, rank,
                                                experts_per_rank, capacity, d_model},
                          x_cur, w_cg, residual, indices, slots, weights, capacity, n_tokens,
                          d_model, k, out, st);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_ep_return_p2p(const void* y, int dtype, const int32_t* recv_counts,
                                   int capacity, int d_model, int world, int rank,
                                   int experts_per_rank, void* const* peer_back,
                                   uint32_t* const* peer_flags, uint32_t* epoch_ctr, int max_ctas,
                                   void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16 || dtype == SCMOE_F32, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(capacity >= 1 && world >= 1 && rank >= 0 && rank < world &&
                      experts_per_rank >= 1,
                  "bad capacity / rank / world");
  SCMOE_CHECK_ARG(y && recv_counts && peer_back && peer_flags && epoch_ctr, "null argument");
  const int vec = dtype == SCMOE_BF16 ? 8 : 4;
  SCMOE_CHECK_ARG(d_model % vec == 0, "d_model must be a multiple of %d", vec);
  const long long rows = (long long)world * experts_per_rank * capacity;
  long long g64 = (rows + WARPS - 1) / WARPS;
  int grid = (int)(g64 < (1 << 20) ? g64 : (1 << 20));
  if (max_ctas > 0) grid = min(grid, max_ctas);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SCMOE_BF16)
    ep_return_p2p_kernel<__nv_bfloat16><<<grid, WARPS * 32, 0, st>>>(
        (const __nv_bfloat16*)y, recv_counts, capacity, d_model, world, rank, experts_per_rank,
        (__nv_bfloat16* const*)peer_back, peer_flags, epoch_ctr);
  else
    ep_return_p2p_kernel<float><<<grid, WARPS * 32, 0, st>>>(
        (const float*)y, recv_counts, capacity, d_model, world, rank, experts_per_rank,
        (float* const*)peer_back, peer_flags, epoch_ctr);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}
