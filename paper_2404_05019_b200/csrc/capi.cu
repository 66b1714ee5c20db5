// C ABI glue: error reporting, device checks and the GEMM / FFN entries.
#include <stdarg.h>
#include <stdio.h>

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

int grouped_gemm_bf16(const void* a, const void* wt, const float* bias, const void* residual,
                      void* out, int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                      int rows_clip, int N, int K, int epi, cudaStream_t st);
int grouped_gemm_f32(const float* a, const float* wt, const float* bias, const float* residual,
                     float* out, int num_groups, int n_wgroups, int cap, const int32_t* group_rows,
                     int rows_clip, int N, int K, int epi, cudaStream_t st);

}  // namespace scmoe

extern "C" int scmoe_version(void) { return 1; }

extern "C" const char* scmoe_last_error(void) { return scmoe::g_err; }

extern "C" int scmoe_device_check(int device) {
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) {
    scmoe::set_error("no CUDA device %d: %s", device, cudaGetErrorString(e));
    return SCMOE_ERR_UNSUPPORTED;
  }
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) {
    scmoe::set_error("libscmoe is built for sm_100a; device %d is sm_%d%d", device, major, minor);
    return SCMOE_ERR_UNSUPPORTED;
  }
  return SCMOE_OK;
}

extern "C" int scmoe_grouped_gemm(const void* a, int dtype, const void* wt, const float* bias,
                                  const void* residual, void* out, int num_groups, int n_wgroups, int group_cap,
                                  const int32_t* group_rows, int rows_clip, int n_out, int k_in,
                                  int epilogue, void* stream) {
  using namespace scmoe;
  SCMOE_CHECK_ARG(dtype == SCMOE_F32 || dtype == SCMOE_BF16, "bad dtype %d", dtype);
  SCMOE_CHECK_ARG(num_groups >= 1 && n_wgroups >= 1, "num_groups/n_wgroups must be >= 1");
  SCMOE_CHECK_ARG(group_cap >= 0 && n_out >= 1 && k_in >= 1, "bad GEMM shape");
  SCMOE_CHECK_ARG(epilogue == SCMOE_EPI_BIAS || epilogue == SCMOE_EPI_BIAS_GELU,
                  "bad epilogue %d", epilogue);
  if (group_cap == 0) return SCMOE_OK;
  if (rows_clip <= 0) rows_clip = group_cap;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SCMOE_BF16)
    return grouped_gemm_bf16(a, wt, bias, residual, out, num_groups, n_wgroups, group_cap, group_rows,
                             rows_clip, n_out, k_in, epilogue, st);
  return grouped_gemm_f32((const float*)a, (const float*)wt, bias, (const float*)residual,
                          (float*)out, num_groups,
                          n_wgroups, group_cap, group_rows, rows_clip, n_out, k_in, epilogue, st);
}

extern "C" int scmoe_expert_ffn(const void* x, int dtype, const void* w1t, const float* b1,
                                const void* w2t, const float* b2, const void* residual,
                                void* hidden, void* out,
                                int num_groups, int n_wgroups, int group_cap,
                                const int32_t* group_rows, int rows_clip, int d_model,
                                int d_hidden, void* stream) {
  int rc = scmoe_grouped_gemm(x, dtype, w1t, b1, nullptr, hidden, num_groups, n_wgroups, group_cap,
                              group_rows, rows_clip, d_hidden, d_model, SCMOE_EPI_BIAS_GELU,
                              stream);
  if (rc) return rc;
  return scmoe_grouped_gemm(hidden, dtype, w2t, b2, residual, out, num_groups, n_wgroups, group_cap,
                            group_rows, rows_clip, d_model, d_hidden, SCMOE_EPI_BIAS, stream);
}
