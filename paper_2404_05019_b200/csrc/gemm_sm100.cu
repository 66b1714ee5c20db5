// K3 / K4 — grouped bf16 GEMM on 5th-generation tensor cores (tcgen05).
//
//   out[g, r, :] = epi( a[g, r, :] . wt[g % n_wgroups, :, :]^T + bias )
//
// for r < rows(g) = min(group_rows[g], rows_clip): the routed experts read the
// capacity-slotted dispatch buffer (group = expert, rows = kept tokens, known
// only on the device), the shared expert / Block-MLP is a single group.  The
// epilogue is expert_forward's bias (+ exact-erf GELU) (arch.py:349-351).
//
// Structure (persistent, one CTA per SM, 384 threads):
//   warp 0      TMA producer: A (128x64) and B (256x64) bf16 tiles, 128B
//               swizzle, into a 4-stage shared-memory ring (full/empty mbarriers)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16
//               128x256x16, accumulating in TMEM; tcgen05.commit frees smem
//               stages and signals the epilogue
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4-11  epilogue: tcgen05.ld 32x32b -> bias/GELU -> bf16 -> global,
//               double-buffered against the MMA of the next tile
// Tiles are walked in (group, m-tile, n-tile) order with n fastest, skipping
// the m-tiles past each group's device-side row count.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace scmoe {
namespace sm100 {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int STAGES = 4;
constexpr int ACC_STAGES = 2;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + EPI_WARPS * 32;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int TMEM_COLS = ACC_STAGES * BN;
constexpr int MAX_GROUPS = 1024;
constexpr size_t SMEM_BYTES = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + 256 + (MAX_GROUPS + 1) * 4;

// instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

struct Params {
  int num_groups, n_wgroups, cap, rows_clip, N, K, epi;
  const int32_t* group_rows;
  const float* bias;
  __nv_bfloat16* out;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
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
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
// K-major operand, 128-byte swizzle: rows of 64 bf16 (128 B), 8-row groups
// 1024 B apart (SBO), version 1 (sm_100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
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

struct TileCoord {
  int g, m0, n0;
};

__device__ __forceinline__ TileCoord decode_tile(int t, int n_tiles_n, const int* prefix,
                                                 int num_groups) {
  const int mlin = t / n_tiles_n;
  const int nt = t - mlin * n_tiles_n;
  int lo = 0, hi = num_groups - 1;  // largest g with prefix[g] <= mlin
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= mlin) lo = mid;
    else hi = mid - 1;
  }
  TileCoord c;
  c.g = lo;
  c.m0 = (mlin - prefix[lo]) * BM;
  c.n0 = nt * BN;
  return c;
}

__device__ __forceinline__ int group_rows_of(const Params& p, int g) {
  return p.group_rows ? min(__ldg(p.group_rows + g), p.rows_clip) : p.cap;
}

__global__ void __launch_bounds__(THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_b + STAGES * B_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + ACC_STAGES;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * ACC_STAGES);
  int* s_prefix = reinterpret_cast<int*>(smem_b + STAGES * B_BYTES + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < ACC_STAGES; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 3) {
    // exclusive prefix of m-tiles per group (warp scan, 32 groups at a time)
    int carry = 0;
    if (lane == 0) s_prefix[0] = 0;
    for (int base = 0; base < p.num_groups; base += 32) {
      const int g = base + lane;
      int v = 0;
      if (g < p.num_groups) v = (group_rows_of(p, g) + BM - 1) / BM;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (g < p.num_groups) s_prefix[g + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int n_tiles_n = (p.N + BN - 1) / BN;
  const int total_tiles = s_prefix[p.num_groups] * n_tiles_n;
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == 0) {
    // ===== TMA producer =====
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const TileCoord tc = decode_tile(t, n_tiles_n, s_prefix, p.num_groups);
      const int wg = tc.g % p.n_wgroups;
      for (int kb = 0; kb < num_kb; ++kb) {
        if (lane == 0) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_expect_tx(&full_bar[stage], A_BYTES + B_BYTES);
          tma_load_3d(&map_a, &full_bar[stage], smem_a + stage * A_BYTES, kb * BK, tc.m0, tc.g);
          tma_load_3d(&map_b, &full_bar[stage], smem_b + stage * B_BYTES, kb * BK, tc.n0, wg);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const uint32_t d_tmem = tmem_base + acc * BN;
      if (lane == 0) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
      }
      __syncwarp();
      for (int kb = 0; kb < num_kb; ++kb) {
        if (lane == 0) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem_a + stage * A_BYTES);
          const uint32_t b0 = smem_u32(smem_b + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            tc_mma(d_tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32),
                   (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tc_commit(&tfull_bar[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===== epilogue =====
    const int ew = warp - 4;
    const int quad = warp & 3;       // TMEM lanes [32*quad, 32*quad+32)
    const int half = ew >> 2;        // accumulator columns [128*half, 128*half+128)
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const TileCoord tc = decode_tile(t, n_tiles_n, s_prefix, p.num_groups);
      const int wg = tc.g % p.n_wgroups;
      const int rows = group_rows_of(p, tc.g);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = tc.m0 + quad * 32 + lane;
      __nv_bfloat16* orow = p.out + ((long long)tc.g * p.cap + row) * p.N;
      const float* brow = p.bias ? p.bias + (long long)wg * p.N : nullptr;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col = half * 128 + c * 32;
        uint32_t r[32];
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + col;
        SCMOE_TMEM_LD32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int n = tc.n0 + col;
        if (row < rows && n < p.N) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int nn = n + u * 8;
            if (nn < p.N) {
              float v[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[u * 8 + i]);
              if (brow) {
                const float4 b0 = *reinterpret_cast<const float4*>(brow + nn);
                const float4 b1 = *reinterpret_cast<const float4*>(brow + nn + 4);
                v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
                v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
              }
              if (p.epi == SCMOE_EPI_BIAS_GELU) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = gelu_erf(v[i]);
              }
              Vec16<__nv_bfloat16> o;
              o.from_float(v);
              st_v4(orow + nn, o.raw);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
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

// 3-D bf16 map over (k_in, rows, groups), box (64, box_rows, 1), 128B swizzle.
int make_map(CUtensorMap* map, const void* base, int k_in, int rows, int groups, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return SCMOE_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)k_in, (cuuint64_t)rows, (cuuint64_t)groups};
  cuuint64_t strides[2] = {(cuuint64_t)k_in * 2, (cuuint64_t)k_in * 2 * (cuuint64_t)rows};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): k=%d rows=%d groups=%d", (int)r, k_in, rows,
              groups);
    return SCMOE_ERR_CUDA;
  }
  return SCMOE_OK;
}

}  // namespace sm100

int grouped_gemm_bf16(const void* a, const void* wt, const float* bias, void* out, int num_groups,
                      int n_wgroups, int cap, const int32_t* group_rows, int rows_clip, int N,
                      int K, int epi, cudaStream_t st) {
  using namespace sm100;
  SCMOE_CHECK_ARG(num_groups <= MAX_GROUPS, "num_groups=%d exceeds %d", num_groups, MAX_GROUPS);
  SCMOE_CHECK_ARG(K % 8 == 0 && N % 8 == 0, "bf16 GEMM needs k_in and n_out multiples of 8");
  SCMOE_CHECK_ARG(((uintptr_t)a & 15) == 0 && ((uintptr_t)wt & 15) == 0 &&
                      ((uintptr_t)out & 15) == 0 && ((uintptr_t)bias & 15) == 0,
                  "GEMM operands must be 16-byte aligned");
  CUtensorMap ma, mb;
  int rc = make_map(&ma, a, K, cap, num_groups, BM);
  if (rc) return rc;
  rc = make_map(&mb, wt, K, N, n_wgroups, BN);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    SCMOE_CUDA_TRY(cudaFuncSetAttribute(grouped_gemm_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)SMEM_BYTES));
    attr_set = true;
  }
  Params p;
  p.num_groups = num_groups;
  p.n_wgroups = n_wgroups;
  p.cap = cap;
  p.rows_clip = rows_clip;
  p.N = N;
  p.K = K;
  p.epi = epi;
  p.group_rows = group_rows;
  p.bias = bias;
  p.out = (__nv_bfloat16*)out;
  const long long max_tiles =
      (long long)num_groups * ((cap + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = (int)(max_tiles < num_sms() ? max_tiles : num_sms());
  if (grid <= 0) return SCMOE_OK;
  grouped_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(ma, mb, p);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

}  // namespace scmoe
