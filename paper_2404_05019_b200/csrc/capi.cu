// C ABI glue: error reporting, device checks, the GEMM / FFN entries and the
// small training helpers (tail zeroing, grouped column sums).
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace scmoe {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int grouped_gemm_bf16(const void* a, const void* wt, int b_mn, const float* bias,
                      const void* residual, const void* aux_in, void* aux_out, void* out,
                      int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                      int rows_clip, int N, int K, int epi, int zero_tail, cudaStream_t st,
                      const CombineSpec* cs = nullptr, void* const* out_groups = nullptr);
int grouped_gemm_f32(const float* a, const float* wt, const float* bias, const float* residual,
                     float* out, int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                     int rows_clip, int N, int K, int epi, cudaStream_t st);
size_t wgrad_workspace_bytes(int n_wgroups, int m_out, int n_out, int splits);
int grouped_wgrad_bf16(const void* a, const void* b, void* out, void* ws, size_t ws_bytes,
                       int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                       int rows_clip, int m_out, int n_out, int splits, cudaStream_t st,
                       bool out_bf16);

namespace {

// rows [rows(g), min(cap, roundup(rows(g), align))) of group g set to zero
__global__ void zero_tails_kernel(uint4* __restrict__ buf, int cap, int row_vecs,
                                  const int32_t* __restrict__ group_rows, int rows_clip,
                                  int align) {
  const int g = blockIdx.y;
  const int r0 = group_rows ? min(group_rows[g], rows_clip) : cap;
  const int r1 = min(cap, ((r0 + align - 1) / align) * align);
  const long long n = (long long)(r1 - r0) * row_vecs;
  uint4* base = buf + ((long long)g * cap + r0) * row_vecs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    base[i] = make_uint4(0, 0, 0, 0);
}

// Column sums over the valid rows of each group (bias gradients), two
// deterministic passes:
// pass 1: block (256-vector column tile, row stripe, group).  Thread (v, lane)
//         owns 16-byte column vector v and rows lane, lane + lanes, ... of the
//         stripe with 8 loads in flight; the lanes' sums are added in a fixed
//         order through shared memory -> one partial row per stripe.  Stripes
//         are sized for ~6 blocks per SM: short, latency-bound row loops.
// pass 2: block (32 columns x 32 stripe lanes), fixed-order sum of the
//         stripes' partials.
constexpr int COLSUM_THREADS = 256;      // column vectors per block (max)
constexpr int COLSUM_BLOCK = 256;        // threads per block: vectors x row lanes

int colsum_vec(int dtype) { return dtype == SCMOE_BF16 ? 8 : 4; }

// Up to two matrices with the same group structure (an FFN's two bias
// gradients) in one launch per pass: tensor i covers column tiles
// [tile0[i], tile0[i+1]) of blockIdx.x (pass 1) / column blocks (pass 2).
struct ColsumSet {
  const void* x[2];
  int cols[2];
  int vpb[2];          // column vectors per pass-1 tile
  int tiles[2];        // pass-1 column tiles
  int stripes[2];      // row stripes (per group), sized for equal bytes per block
  int stripe_rows[2];
  int pblk0[3];        // pass-1 block ranges (tiles x stripes per tensor)
  int blk0[3];         // pass-2 32-column block ranges
  float* part[2];      // [G][stripes][cols]
  float* out[2];       // [G][cols]
};

template <typename T>
__global__ void __launch_bounds__(COLSUM_BLOCK)
colsum_partial_kernel(ColsumSet cs, int cap, const int32_t* __restrict__ group_rows, int rows_clip) {
  constexpr int VEC = Vec16<T>::N;
  constexpr int U = 8;
  __shared__ float red[COLSUM_BLOCK][VEC + 1];
  // programmatic dependent launch: nothing global is read before the
  // producer of x completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int ti = (int)blockIdx.x >= cs.pblk0[1] ? 1 : 0;
  const T* x = (const T*)cs.x[ti];
  const int cols = cs.cols[ti];
  const int vecs = cols / VEC;
  const int vpb = cs.vpb[ti];                              // vectors per column tile
  const int lanes = blockDim.x / vpb;
  const int v = threadIdx.x % vpb, lane = threadIdx.x / vpb;
  const int local = blockIdx.x - cs.pblk0[ti];
  const int g = blockIdx.z, stripe = local / cs.tiles[ti];
  const int n_stripes = cs.stripes[ti], stripe_rows = cs.stripe_rows[ti];
  const int cv = (local % cs.tiles[ti]) * vpb + v;         // my column vector
  const bool active = lane < lanes && cv < vecs;
  const int rows = group_rows ? max(0, min(group_rows[g], rows_clip)) : cap;
  const int r0 = stripe * stripe_rows, r1 = min(rows, r0 + stripe_rows);
  float s[VEC] = {};
  if (active) {
    const T* p = x + ((long long)g * cap) * cols + (long long)cv * VEC;
    int r = r0 + lane;
    for (; r + (U - 1) * lanes < r1; r += U * lanes) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = ld_nc_v4(p + (long long)(r + u * lanes) * cols);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        Vec16<T> t;
        t.raw = w[u];
        float f[VEC];
        t.to_float(f);
#pragma unroll
        for (int i = 0; i < VEC; ++i) s[i] += f[i];
      }
    }
    for (; r < r1; r += lanes) {
      Vec16<T> t;
      t.raw = ld_nc_v4(p + (long long)r * cols);
      float f[VEC];
      t.to_float(f);
#pragma unroll
      for (int i = 0; i < VEC; ++i) s[i] += f[i];
    }
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) red[threadIdx.x][i] = s[i];
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (lane == 0 && cv < vecs) {
    float o[VEC] = {};
    for (int l = 0; l < lanes; ++l)
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] += red[l * vpb + v][i];
    float* q = cs.part[ti] + ((long long)g * n_stripes + stripe) * cols + (long long)cv * VEC;
#pragma unroll
    for (int i = 0; i < VEC; ++i) q[i] = o[i];
  }
}

// block (32 columns x 32 stripe lanes): lane y sums stripes y, y+32, ...,
// then the 32 lane sums are added in a fixed order
__global__ void colsum_final_kernel(ColsumSet cs) {
  __shared__ float red[32][33];
  asm volatile("griddepcontrol.wait;" ::: "memory");     // pass 1 complete
  const int ti = (int)blockIdx.x >= cs.blk0[1] ? 1 : 0;
  const int n_stripes = cs.stripes[ti];
  const int cols = cs.cols[ti];
  const int g = blockIdx.y;
  const int c = (blockIdx.x - cs.blk0[ti]) * 32 + threadIdx.x;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  if (c < cols) {
    const float* p = cs.part[ti] + (long long)g * n_stripes * cols + c;
    int k = threadIdx.y;
    for (; k + 96 < n_stripes; k += 128) {     // four independent loads in flight
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] += p[(long long)(k + 32 * u) * cols];
    }
    for (; k < n_stripes; k += 32) a[0] += p[(long long)k * cols];
  }
  red[threadIdx.y][threadIdx.x] = (a[0] + a[1]) + (a[2] + a[3]);
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float t = 0.f;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) t += red[y][threadIdx.x];
    cs.out[ti][(long long)g * cols + c] = t;
  }
}

// aux = N / (T * T * k) * sum_e counts[e] * prob_sum[e] in fp32, experts in
// order (arch.py:436-439: N * sum_e f_e P_e with f_e = counts[e] / (T k),
// P_e = prob_sum[e] / T): one warp instead of five tensor ops
__global__ void gate_aux_kernel(const int32_t* __restrict__ counts,
                                const float* __restrict__ prob_sum, int n_experts, float scale,
                                float* __restrict__ aux) {
  if (threadIdx.x != 0) return;
  float s = 0.f;
  for (int e = 0; e < n_experts; ++e) s += (float)counts[e] * prob_sum[e];
  *aux = s * scale;
}

// out[i] = dtype(src[0] * (1 / div)) for i < n: the constant gradient of a mean
// (grad.py:52-67) straight from the device scalar, 16-byte stores
template <typename T>
__global__ void fill_div_kernel(T* __restrict__ out, long long n, const float* __restrict__ src,
                                float div) {
  // torch's tensor / python-scalar multiplies by the fp32 reciprocal:
  // bit-identical to (g / n).to(dtype)
  const float v = __ldg(src) * (1.0f / div);
  T t;
  if constexpr (std::is_same<T, float>::value) t = v;
  else t = __float2bfloat16_rn(v);
  constexpr int V = 16 / sizeof(T);
  T pack[V];
#pragma unroll
  for (int i = 0; i < V; ++i) pack[i] = t;
  const uint4 w = *reinterpret_cast<const uint4*>(pack);
  const long long n_vec = n / V;
  const long long stride = (long long)gridDim.x * blockDim.x;
  uint4* o = reinterpret_cast<uint4*>(out);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_vec; i += stride)
    o[i] = w;
  for (long long i = n_vec * V + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = t;
}

// mean of n elements in fp32, deterministic: pass 1 = MEAN_BLOCKS blocks,
// each a fixed contiguous range (16-byte loads, 4 in flight per thread, a
// fixed-order block tree) -> one partial per block; pass 2 = one block,
// fixed-order tree over the partials, / n.  No memset (a torch reduction
// zeroes its semaphores with a memset node: ~8 us of idle GPU in a graph).
constexpr int MEAN_BLOCKS = 296;
template <typename T>
__global__ void __launch_bounds__(256) mean_partial_kernel(const T* __restrict__ x, long long n,
                                                           float* __restrict__ part) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float red[256];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long per = (n + MEAN_BLOCKS - 1) / MEAN_BLOCKS;
  const long long per_v = (per + V - 1) / V * V;                // whole 16-byte vectors
  const long long lo = min(n, (long long)blockIdx.x * per_v), hi = min(n, lo + per_v);
  float acc = 0.f;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(x + lo) & 15) == 0);
  long long i = lo;
  if (vec_ok) {
    const long long nv = (hi - lo) / V;
    const uint4* xv = reinterpret_cast<const uint4*>(x + lo);
    long long j = threadIdx.x;
    for (; j + 768 < nv; j += 1024) {
      uint4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = ld_nc_v4(xv + j + 256 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Vec16<T> t;
        t.raw = w[u];
        float f[V];
        t.to_float(f);
#pragma unroll
        for (int q = 0; q < V; ++q) acc += f[q];
      }
    }
    for (; j < nv; j += 256) {
      Vec16<T> t;
      t.raw = ld_nc_v4(xv + j);
      float f[V];
      t.to_float(f);
#pragma unroll
      for (int q = 0; q < V; ++q) acc += f[q];
    }
    i = lo + nv * V;
  }
  for (long long r = i + threadIdx.x; r < hi; r += 256) acc += (float)x[r];
  red[threadIdx.x] = acc;
  __syncthreads();
#pragma unroll
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(512) mean_final_kernel(const float* __restrict__ part,
                                                         long long n, float* __restrict__ out) {
  __shared__ float red[512];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  red[threadIdx.x] = threadIdx.x < MEAN_BLOCKS ? part[threadIdx.x] : 0.f;
  __syncthreads();
#pragma unroll
  for (int o = 256; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0] / (float)n;
}

template <typename K, typename... Args>
int launch_pdl(K kern, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SCMOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return SCMOE_OK;
}

int colsum_tiles(int cols, int vec) {
  const int vecs = (cols + vec - 1) / vec;
  return (vecs + COLSUM_THREADS - 1) / COLSUM_THREADS;
}

// Row stripes per group for each matrix: ~6 pass-1 blocks per SM in total,
// shared out in proportion to each matrix's bytes so every block reads about
// the same amount (short, latency-bound row loops with many blocks in
// flight; fewer, longer stripes measured slower; one stripe count for both
// starved the wide matrix)
void colsum_set_stripes(int num_groups, int group_cap, const int* cols, int n, int vec,
                        int* stripes) {
  long long tot = 0;
  for (int i = 0; i < n; ++i) tot += cols[i];
  const double target = 6.0 * num_sms();
  for (int i = 0; i < n; ++i) {
    const double share = target * (double)cols[i] / (double)tot;
    int st = (int)(share / ((double)colsum_tiles(cols[i], vec) * num_groups) + 0.5);
    stripes[i] = max(1, min(st, (group_cap + 7) / 8));
  }
}

size_t colsum2_ws_bytes(int num_groups, int group_cap, int cols0, int cols1) {
  if (num_groups < 1 || group_cap < 1 || cols0 < 1 || cols1 < 0) return 0;
  // large enough for either vector width (bf16 8, fp32 4 per 16 bytes)
  const int cl[2] = {cols0, cols1};
  const int n = cols1 ? 2 : 1;
  size_t best = 0;
  for (int vec : {8, 4}) {
    int st[2] = {0, 0};
    colsum_set_stripes(num_groups, group_cap, cl, n, vec, st);
    size_t b = 0;
    for (int i = 0; i < n; ++i) b += (size_t)st[i] * num_groups * cl[i] * sizeof(float);
    best = std::max(best, b);
  }
  return best;
}

int colsum2_impl(const void* x0, const void* x1, int dtype, int num_groups, int group_cap,
                 int cols0, int cols1, const int32_t* group_rows, int rows_clip, float* out0,
                 float* out1, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(num_groups >= 1 && cols0 >= 1 && cols1 >= 0 && group_cap >= 1,
                  "bad colsum shape");
  SCMOE_CHECK_ARG(workspace_bytes >= colsum2_ws_bytes(num_groups, group_cap, cols0, cols1),
                  "colsum workspace too small");
  if (rows_clip <= 0) rows_clip = group_cap;
  const int vec = colsum_vec(dtype);
  SCMOE_CHECK_ARG(cols0 % vec == 0 && cols1 % vec == 0 && ((uintptr_t)x0 & 15) == 0 &&
                      ((uintptr_t)x1 & 15) == 0,
                  "colsum needs 16-byte aligned rows (cols multiple of %d)", vec);
  ColsumSet cs = {};
  const int n = cols1 ? 2 : 1;
  const void* xs[2] = {x0, x1};
  const int cl[2] = {cols0, cols1};
  float* outs[2] = {out0, out1};
  colsum_set_stripes(num_groups, group_cap, cl, n, vec, cs.stripes);
  cs.pblk0[0] = cs.blk0[0] = 0;
  float* part = (float*)workspace;
  for (int i = 0; i < 2; ++i) {
    cs.x[i] = xs[i];
    cs.cols[i] = cl[i];
    cs.out[i] = outs[i];
    const int vecs = cl[i] / vec;
    cs.vpb[i] = std::max(1, std::min(vecs, COLSUM_THREADS));
    cs.tiles[i] = i < n ? (vecs + cs.vpb[i] - 1) / cs.vpb[i] : 0;
    if (i >= n) cs.stripes[i] = 1;
    cs.stripe_rows[i] = (group_cap + cs.stripes[i] - 1) / cs.stripes[i];
    cs.pblk0[i + 1] = cs.pblk0[i] + cs.tiles[i] * cs.stripes[i];
    cs.blk0[i + 1] = cs.blk0[i] + (i < n ? (cl[i] + 31) / 32 : 0);
    cs.part[i] = part;
    if (i < n) part += (size_t)num_groups * cs.stripes[i] * cl[i];
  }
  dim3 grid(cs.pblk0[2], 1, num_groups);
  int rc = dtype == SCMOE_BF16
               ? launch_pdl(colsum_partial_kernel<__nv_bfloat16>, grid, dim3(COLSUM_BLOCK), st, cs,
                            group_cap, group_rows, rows_clip)
               : launch_pdl(colsum_partial_kernel<float>, grid, dim3(COLSUM_BLOCK), st, cs,
                            group_cap, group_rows, rows_clip);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  rc = launch_pdl(colsum_final_kernel, dim3(cs.blk0[2], num_groups), dim3(32, 32), st, cs);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

// dst[j] = src[ids[j]] for j < min(*n_rows, max_rows); rows of row_bytes
// (multiple of 16).  src may be pinned host memory (UVA-mapped): this is the
// expert-migration copy, 8 x 16-byte loads in flight per thread over PCIe.
__global__ void gather_rows_kernel(const uint4* __restrict__ src, long long row_vecs,
                                   const int32_t* __restrict__ ids,
                                   const int32_t* __restrict__ n_rows, int max_rows,
                                   uint4* __restrict__ dst) {
  const int j = blockIdx.y;
  if (j >= max_rows || j >= *n_rows) return;
  const uint4* s = src + (long long)ids[j] * row_vecs;
  uint4* d = dst + (long long)j * row_vecs;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < row_vecs; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = s[i + u * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) d[i + u * stride] = v[u];
  }
  for (; i < row_vecs; i += stride) d[i] = s[i];
}

}  // namespace
}  // namespace scmoe

using namespace scmoe;

extern "C" int scmoe_version(void) { return 2; }

extern "C" const char* scmoe_last_error(void) { return g_err; }

extern "C" int scmoe_device_check(int device) {
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) {
    set_error("no CUDA device %d: %s", device, cudaGetErrorString(e));
    return SCMOE_ERR_UNSUPPORTED;
  }
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) {
    set_error("libscmoe is built for sm_100a; device %d is sm_%d%d", device, major, minor);
    return SCMOE_ERR_UNSUPPORTED;
  }
  return SCMOE_OK;
}

extern "C" int scmoe_grouped_gemm_ex(const void* a, int dtype, const void* w, int w_layout,
                                     const float* bias, const void* residual, const void* aux_in,
                                     void* aux_out, void* out, int num_groups, int n_wgroups,
                                     int group_cap, const int32_t* group_rows, int rows_clip,
                                     int n_out, int k_in, int epilogue, int zero_tail,
                                     void* stream) {
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(num_groups >= 1 && n_wgroups >= 1, "num_groups/n_wgroups must be >= 1");
  SCMOE_CHECK_ARG(group_cap >= 0 && n_out >= 1 && k_in >= 1, "bad GEMM shape");
  SCMOE_CHECK_ARG(epilogue >= SCMOE_EPI_BIAS && epilogue <= SCMOE_EPI_MUL_AUX, "bad epilogue %d",
                  epilogue);
  SCMOE_CHECK_ARG(w_layout == SCMOE_W_NK || w_layout == SCMOE_W_KN, "bad weight layout %d",
                  w_layout);
  if (group_cap == 0) return SCMOE_OK;
  if (rows_clip <= 0) rows_clip = group_cap;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SCMOE_BF16)
    return grouped_gemm_bf16(a, w, w_layout == SCMOE_W_KN, bias, residual, aux_in, aux_out, out,
                             num_groups, n_wgroups, group_cap, group_rows, rows_clip, n_out, k_in,
                             epilogue, zero_tail, st);
  SCMOE_CHECK_ARG(w_layout == SCMOE_W_NK && epilogue <= SCMOE_EPI_BIAS_GELU && !aux_out &&
                      !zero_tail,
                  "the fp32 parity GEMM supports the forward epilogues only");
  return grouped_gemm_f32((const float*)a, (const float*)w, bias, (const float*)residual,
                          (float*)out, num_groups, n_wgroups, group_cap, group_rows, rows_clip,
                          n_out, k_in, epilogue, st);
}

extern "C" int scmoe_grouped_gemm(const void* a, int dtype, const void* wt, const float* bias,
                                  const void* residual, void* out, int num_groups, int n_wgroups,
                                  int group_cap, const int32_t* group_rows, int rows_clip,
                                  int n_out, int k_in, int epilogue, void* stream) {
  SCMOE_CHECK_ARG(epilogue == SCMOE_EPI_BIAS || epilogue == SCMOE_EPI_BIAS_GELU,
                  "bad epilogue %d", epilogue);
  return scmoe_grouped_gemm_ex(a, dtype, wt, SCMOE_W_NK, bias, residual, nullptr, nullptr, out,
                               num_groups, n_wgroups, group_cap, group_rows, rows_clip, n_out,
                               k_in, epilogue, 0, stream);
}

extern "C" int scmoe_expert_ffn(const void* x, int dtype, const void* w1t, const float* b1,
                                const void* w2t, const float* b2, const void* residual,
                                void* hidden, void* out, int num_groups, int n_wgroups,
                                int group_cap, const int32_t* group_rows, int rows_clip,
                                int d_model, int d_hidden, void* stream) {
  int rc = scmoe_grouped_gemm(x, dtype, w1t, b1, nullptr, hidden, num_groups, n_wgroups,
                              group_cap, group_rows, rows_clip, d_hidden, d_model,
                              SCMOE_EPI_BIAS_GELU, stream);
  if (rc) return rc;
  return scmoe_grouped_gemm(hidden, dtype, w2t, b2, residual, out, num_groups, n_wgroups,
                            group_cap, group_rows, rows_clip, d_model, d_hidden, SCMOE_EPI_BIAS,
                            stream);
}

extern "C" int scmoe_shared_ffn_combine(const void* x, int dtype, const void* w1t,
                                        const float* b1, const void* w2t, const float* b2,
                                        const void* residual, const void* expert_out,
                                        const int32_t* indices, const int32_t* slots,
                                        const float* weights, int capacity, int k, void* hidden,
                                        void* out, int n_tokens, int d_model, int d_hidden,
                                        void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16, "the fused combine runs on bf16");
  SCMOE_CHECK_ARG(k >= 1 && k <= 2 && capacity >= 1, "fused combine: k <= 2");
  int rc = scmoe_grouped_gemm(x, dtype, w1t, b1, nullptr, hidden, 1, 1, n_tokens, nullptr,
                              n_tokens, d_hidden, d_model, SCMOE_EPI_BIAS_GELU, stream);
  if (rc) return rc;
  return scmoe_ffn2_combine(hidden, dtype, w2t, b2, residual, expert_out, indices, slots, weights,
                            capacity, k, out, n_tokens, d_model, d_hidden, stream);
}

extern "C" int scmoe_ffn2_combine(const void* hidden, int dtype, const void* w2t, const float* b2,
                                  const void* residual, const void* expert_out,
                                  const int32_t* indices, const int32_t* slots,
                                  const float* weights, int capacity, int k, void* out,
                                  int n_tokens, int d_model, int d_hidden, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16, "the fused combine runs on bf16");
  SCMOE_CHECK_ARG(k >= 1 && k <= 2 && capacity >= 1, "fused combine: k <= 2");
  const CombineSpec cs{expert_out, indices, slots, weights, capacity, k};
  return grouped_gemm_bf16(hidden, w2t, 0, b2, residual, nullptr, nullptr, out, 1, 1, n_tokens,
                           nullptr, n_tokens, d_model, d_hidden, SCMOE_EPI_BIAS, 0,
                           (cudaStream_t)stream, &cs);
}

extern "C" int scmoe_expert_ffn_to_peers(const void* x, int dtype, const void* w1t,
                                         const float* b1, const void* w2t, const float* b2,
                                         void* hidden, void* const* out_group_ptrs,
                                         int num_groups, int n_wgroups, int group_cap,
                                         const int32_t* group_rows, int rows_clip, int d_model,
                                         int d_hidden, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16 && out_group_ptrs, "bf16 with an output-group table");
  if (rows_clip <= 0) rows_clip = group_cap;
  int rc = scmoe_grouped_gemm(x, dtype, w1t, b1, nullptr, hidden, num_groups, n_wgroups,
                              group_cap, group_rows, rows_clip, d_hidden, d_model,
                              SCMOE_EPI_BIAS_GELU, stream);
  if (rc) return rc;
  // out is only the shape reference; every row goes through out_group_ptrs
  return grouped_gemm_bf16(hidden, w2t, 0, b2, nullptr, nullptr, nullptr, hidden, num_groups,
                           n_wgroups, group_cap, group_rows, rows_clip, d_model, d_hidden,
                           SCMOE_EPI_BIAS, 0, (cudaStream_t)stream, nullptr, out_group_ptrs);
}

extern "C" size_t scmoe_grouped_wgrad_workspace_bytes(int n_wgroups, int m_out, int n_out,
                                                      int splits) {
  if (splits <= 0) splits = 64;  // the automatic choice never exceeds 64
  return wgrad_workspace_bytes(n_wgroups, m_out, n_out, splits);
}

extern "C" int scmoe_grouped_wgrad_ex(const void* a, const void* b, int dtype, void* out,
                                      int out_dtype, void* workspace, size_t workspace_bytes,
                                      int num_groups, int n_wgroups, int group_cap,
                                      const int32_t* group_rows, int rows_clip, int m_out,
                                      int n_out, int splits, void* stream) {
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16, "wgrad runs on bf16 operands");
  SCMOE_CHECK_ARG(out_dtype == SCMOE_F32 || out_dtype == SCMOE_BF16, "wgrad out is fp32 or bf16");
  SCMOE_CHECK_ARG(num_groups >= 1 && n_wgroups >= 1 && num_groups % n_wgroups == 0,
                  "num_groups must be a positive multiple of n_wgroups");
  SCMOE_CHECK_ARG(group_cap >= 1 && m_out >= 1 && n_out >= 1, "bad wgrad shape");
  if (rows_clip <= 0) rows_clip = group_cap;
  return grouped_wgrad_bf16(a, b, out, workspace, workspace_bytes, num_groups, n_wgroups,
                            group_cap, group_rows, rows_clip, m_out, n_out, splits,
                            (cudaStream_t)stream, out_dtype == SCMOE_BF16);
}

extern "C" int scmoe_grouped_wgrad(const void* a, const void* b, int dtype, float* out,
                                   void* workspace, size_t workspace_bytes, int num_groups,
                                   int n_wgroups, int group_cap, const int32_t* group_rows,
                                   int rows_clip, int m_out, int n_out, int splits, void* stream) {
  return scmoe_grouped_wgrad_ex(a, b, dtype, out, SCMOE_F32, workspace, workspace_bytes,
                                num_groups, n_wgroups, group_cap, group_rows, rows_clip, m_out,
                                n_out, splits, stream);
}

extern "C" int scmoe_zero_tails(void* buf, int dtype, int num_groups, int group_cap, int cols,
                                const int32_t* group_rows, int rows_clip, int align,
                                void* stream) {
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  const int esz = dtype == SCMOE_BF16 ? 2 : 4;
  SCMOE_CHECK_ARG((cols * esz) % 16 == 0 && ((uintptr_t)buf & 15) == 0,
                  "rows must be 16-byte multiples and aligned");
  SCMOE_CHECK_ARG(align >= 1 && num_groups >= 1, "bad zero_tails arguments");
  if (group_cap <= 0 || !group_rows) return SCMOE_OK;
  if (rows_clip <= 0) rows_clip = group_cap;
  dim3 grid(32, num_groups);
  zero_tails_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((uint4*)buf, group_cap,
                                                            cols * esz / 16, group_rows,
                                                            rows_clip, align);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" size_t scmoe_grouped_colsum_workspace_bytes(int num_groups, int group_cap, int cols) {
  return colsum2_ws_bytes(num_groups, group_cap, cols, 0);
}

extern "C" int scmoe_grouped_colsum(const void* x, int dtype, int num_groups, int group_cap,
                                    int cols, const int32_t* group_rows, int rows_clip,
                                    float* out, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  return colsum2_impl(x, x, dtype, num_groups, group_cap, cols, 0, group_rows, rows_clip, out,
                      nullptr, workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" size_t scmoe_grouped_colsum2_workspace_bytes(int num_groups, int group_cap, int cols0,
                                                        int cols1) {
  return cols1 >= 1 ? colsum2_ws_bytes(num_groups, group_cap, cols0, cols1) : 0;
}

extern "C" int scmoe_grouped_colsum2(const void* x0, const void* x1, int dtype, int num_groups,
                                     int group_cap, int cols0, int cols1,
                                     const int32_t* group_rows, int rows_clip, float* out0,
                                     float* out1, void* workspace, size_t workspace_bytes,
                                     void* stream) {
  SCMOE_CHECK_ARG(cols1 >= 1 && x1 && out1, "colsum2 needs a second matrix");
  return colsum2_impl(x0, x1, dtype, num_groups, group_cap, cols0, cols1, group_rows, rows_clip,
                      out0, out1, workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" int scmoe_gate_aux_loss(const int32_t* counts, const float* prob_sum, int n_tokens,
                                   int n_experts, int k, float* aux, void* stream) {
  SCMOE_CHECK_ARG(n_tokens >= 1 && n_experts >= 1 && k >= 1 && counts && prob_sum && aux,
                  "bad aux-loss arguments");
  const float scale = (float)((double)n_experts / ((double)n_tokens * (double)n_tokens * k));
  gate_aux_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(counts, prob_sum, n_experts, scale, aux);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_fill_div(void* out, int dtype, long long n, const float* src, float div,
                              void* stream) {
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(n >= 0 && src && (n == 0 || out) && ((uintptr_t)out & 15) == 0,
                  "fill needs a 16-byte aligned output");
  if (n == 0) return SCMOE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)std::min<long long>((n / 8 + 255) / 256 + 1, (long long)num_sms() * 8);
  if (dtype == SCMOE_BF16)
    fill_div_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((__nv_bfloat16*)out, n, src, div);
  else
    fill_div_kernel<float><<<grid, 256, 0, st>>>((float*)out, n, src, div);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" size_t scmoe_mean_workspace_bytes(void) { return MEAN_BLOCKS * sizeof(float); }

extern "C" int scmoe_mean(const void* x, int dtype, long long n, float* out, void* workspace,
                          size_t workspace_bytes, void* stream) {
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(n >= 1 && x && out, "mean needs n >= 1");
  SCMOE_CHECK_ARG(workspace && workspace_bytes >= MEAN_BLOCKS * sizeof(float),
                  "mean workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  float* part = (float*)workspace;
  int rc = dtype == SCMOE_BF16
               ? launch_pdl(mean_partial_kernel<__nv_bfloat16>, dim3(MEAN_BLOCKS), dim3(256), st,
                            (const __nv_bfloat16*)x, n, part)
               : launch_pdl(mean_partial_kernel<float>, dim3(MEAN_BLOCKS), dim3(256), st,
                            (const float*)x, n, part);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  rc = launch_pdl(mean_final_kernel, dim3(1), dim3(512), st, (const float*)part, n, out);
  if (rc) return rc;
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

extern "C" int scmoe_gather_rows(const void* src, size_t row_bytes, const int32_t* ids,
                                 const int32_t* n_rows, int max_rows, void* dst, void* stream) {
  SCMOE_CHECK_ARG(row_bytes % 16 == 0 && ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0,
                  "gather rows must be 16-byte multiples and aligned");
  SCMOE_CHECK_ARG(max_rows >= 0 && ids && n_rows, "bad gather arguments");
  if (max_rows == 0 || row_bytes == 0) return SCMOE_OK;
  const long long vecs = (long long)(row_bytes / 16);
  long long per_row = (vecs + 256 * 8 - 1) / (256 * 8);
  if (per_row > 64) per_row = 64;   // ~64 CTAs per row saturate the host link
  dim3 grid((unsigned)per_row, (unsigned)max_rows);
  gather_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, vecs, ids, n_rows,
                                                            max_rows, (uint4*)dst);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}

// ---------------------------------------------------------------------------
// In-place SGD over a list of tensors in ONE launch (grad.py:330-331,
// p -= lr * g, fp32 arithmetic, rounded to the parameter dtype — the same
// values as torch._foreach_add_(p, g, alpha=-lr)).  The tensor table travels
// as a kernel parameter (no host->device copy, CUDA-graph capturable); 16-byte
// vectors over the concatenated vector index space, grid-stride.
namespace scmoe {
namespace sgd_detail {
constexpr int MAXT = 64;
struct Table {
  void* p[MAXT];
  const void* g[MAXT];
  long long vec_end[MAXT];      // inclusive prefix of 16-byte vectors
  int bf16[MAXT];
  int n;
};

__global__ void __launch_bounds__(256) sgd_kernel(const __grid_constant__ Table t, float lr,
                                                  long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (t.vec_end[k] <= i) ++k;            // <= 64 tensors, warp-uniform mostly
    const long long v = i - (k ? t.vec_end[k - 1] : 0);
    uint4* pp = reinterpret_cast<uint4*>(t.p[k]) + v;
    const uint4 gv = ld_nc_v4(reinterpret_cast<const uint4*>(t.g[k]) + v);
    uint4 pv = *pp;
    if (t.bf16[k]) {
      Vec16<__nv_bfloat16> a, b;
      a.raw = pv;
      b.raw = gv;
      float fa[8], fb[8];
      a.to_float(fa);
      b.to_float(fb);
#pragma unroll
      for (int e = 0; e < 8; ++e) fa[e] = fmaf(-lr, fb[e], fa[e]);
      a.from_float(fa);
      pv = a.raw;
    } else {
      float* fa = reinterpret_cast<float*>(&pv);
      const float* fb = reinterpret_cast<const float*>(&gv);
#pragma unroll
      for (int e = 0; e < 4; ++e) fa[e] = fmaf(-lr, fb[e], fa[e]);
    }
    *pp = pv;
  }
}
}  // namespace sgd_detail
}  // namespace scmoe

extern "C" int scmoe_sgd_update(void* const* params, const void* const* grads,
                                const long long* numels, const int* dtypes, int n, float lr,
                                void* stream) {
  using namespace scmoe::sgd_detail;
  SCMOE_CHECK_ARG(n >= 0 && (n == 0 || (params && grads && numels && dtypes)),
                  "sgd_update: bad arguments");
  for (int base = 0; base < n; base += MAXT) {
    Table t = {};
    long long tot = 0;
    t.n = n - base < MAXT ? n - base : MAXT;
    for (int j = 0; j < t.n; ++j) {
      const int i = base + j;
      SCMOE_CHECK_ARG(dtypes[i] == SCMOE_BF16 || dtypes[i] == SCMOE_F32, "sgd_update: dtype");
      const int vec = dtypes[i] == SCMOE_BF16 ? 8 : 4;
      SCMOE_CHECK_ARG(numels[i] % vec == 0 && ((uintptr_t)params[i] & 15) == 0 &&
                          ((uintptr_t)grads[i] & 15) == 0,
                      "sgd_update: tensor %d needs 16-byte aligned storage of whole vectors", i);
      t.p[j] = params[i];
      t.g[j] = grads[i];
      t.bf16[j] = dtypes[i] == SCMOE_BF16;
      tot += numels[i] / vec;
      t.vec_end[j] = tot;
    }
    if (tot == 0) continue;
    long long blocks = (tot + 255) / 256;
    const long long cap = 4ll * scmoe::num_sms();
    if (blocks > cap) blocks = cap;
    sgd_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(t, lr, tot);
    SCMOE_LAUNCH_CHECK();
  }
  return SCMOE_OK;
}

extern "C" int scmoe_copy_rows(const void* src, size_t row_bytes, const int32_t* ids,
                               int n_rows, void* dst, void* stream) {
  SCMOE_CHECK_ARG(src && dst && (ids || n_rows == 0) && n_rows >= 0, "bad copy_rows arguments");
  const char* s = (const char*)src;
  char* d = (char*)dst;
  for (int j = 0; j < n_rows;) {
    SCMOE_CHECK_ARG(ids[j] >= 0, "copy_rows: negative row id %d", ids[j]);
    int run = 1;                    // consecutive source rows -> one transfer
    while (j + run < n_rows && ids[j + run] == ids[j] + run) ++run;
    SCMOE_CUDA_TRY(cudaMemcpyAsync(d + (size_t)j * row_bytes, s + (size_t)ids[j] * row_bytes,
                                   (size_t)run * row_bytes, cudaMemcpyDefault,
                                   (cudaStream_t)stream));
    j += run;
  }
  return SCMOE_OK;
}

// ---------------------------------------------------------------------------
// Attention layout glue for training (block.py _CudnnPackedAttention): up to
// three (B, H, S, hd) tensors with arbitrary strides (hd contiguous) packed
// into one (B, S, n, H, hd) tensor — dq/dk/dv into the packed QKV gradient,
// or the SDPA output into (T, d) rows.  One thread per 16-byte vector,
// consecutive threads write consecutive destination bytes.
namespace scmoe {
namespace pack_detail {
struct PackSrc {
  const uint4* p[3];
  long long sb[3], sh[3], ss[3];   // element strides of (B, H, S)
};

__global__ void pack_heads_kernel(PackSrc src, int n, int B, int H, int S, int hd,
                                  uint4* __restrict__ dst) {
  const int v_per_head = hd / 8;                        // bf16: 8 per 16 bytes
  const long long total = (long long)B * S * n * H * v_per_head;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i;
    const int e = (int)(r % v_per_head); r /= v_per_head;
    const int h = (int)(r % H); r /= H;
    const int c = (int)(r % n); r /= n;
    const int s = (int)(r % S); r /= S;
    const int b = (int)r;
    const long long off = b * src.sb[c] + h * src.sh[c] + s * src.ss[c];   // elements
    dst[i] = __ldg(src.p[c] + off / 8 + e);
  }
}
}  // namespace pack_detail
}  // namespace scmoe

extern "C" int scmoe_pack_heads(const void* const* srcs, const long long* strides, int n_src,
                                int B, int H, int S, int hd, int dtype, void* dst, void* stream) {
  using namespace scmoe;
  using namespace scmoe::pack_detail;
  SCMOE_CHECK_ARG(dtype == SCMOE_BF16, "pack_heads supports bf16");
  SCMOE_CHECK_ARG(n_src >= 1 && n_src <= 3 && srcs && strides && dst, "bad arguments");
  SCMOE_CHECK_ARG(hd % 8 == 0 && B > 0 && H > 0 && S > 0, "hd must be a multiple of 8");
  PackSrc ps{};
  for (int i = 0; i < n_src; ++i) {
    ps.p[i] = (const uint4*)srcs[i];
    ps.sb[i] = strides[3 * i];
    ps.sh[i] = strides[3 * i + 1];
    ps.ss[i] = strides[3 * i + 2];
    SCMOE_CHECK_ARG(((uintptr_t)srcs[i] & 15) == 0 && ps.sb[i] % 8 == 0 && ps.sh[i] % 8 == 0 &&
                        ps.ss[i] % 8 == 0,
                    "source %d must be 16-byte aligned with strides multiple of 8", i);
  }
  SCMOE_CHECK_ARG(((uintptr_t)dst & 15) == 0, "dst must be 16-byte aligned");
  const long long total = (long long)B * S * n_src * H * (hd / 8);
  const int grid = (int)std::min<long long>((total + 255) / 256, (long long)num_sms() * 16);
  pack_heads_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ps, n_src, B, H, S, hd, (uint4*)dst);
  SCMOE_LAUNCH_CHECK();
  return SCMOE_OK;
}
