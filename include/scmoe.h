/*
 * scmoe.h — C ABI of libscmoe.so, the B200 (sm_100a) kernels behind the
 * ScMoE layer of arXiv 2404.05019.
 *
 * Conventions:
 *  - every pointer is a DEVICE pointer unless stated; every call is
 *    asynchronous on `stream` (a cudaStream_t passed as void*); no call
 *    synchronises the host or allocates memory (workspaces are caller-owned);
 *  - row-major matrices; weights are stored K-major ("transposed"):
 *    w1t[e] is (d_hidden, d_model), w2t[e] is (d_model, d_hidden), so that
 *    both tcgen05 operands are K-major 128B-swizzled TMA tiles;
 *  - return 0 (SCMOE_OK) on success, otherwise an error code with a message
 *    available from scmoe_last_error() (thread-local).
 *
 * Each entry point cites the reference function (file:line, relative to
 * /root/reference/pkg/src/scmoelab/) whose semantics it reproduces.  The
 * reference is a numpy library; its "binding" to these entries is the ctypes
 * layer in paper_2404_05019_b200/_lib.py.
 */
#ifndef SCMOE_H_
#define SCMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCMOE_OK 0
#define SCMOE_ERR_ARG 1          /* invalid argument (reference: ValueError / ShapeError) */
#define SCMOE_ERR_CUDA 2         /* CUDA runtime / driver error */
#define SCMOE_ERR_UNSUPPORTED 3  /* no sm_100 device or unsupported shape */

#define SCMOE_F32 0
#define SCMOE_BF16 1

/* combine modes, arch.py:380-392 (COMBINE_MODES arch.py:27) */
#define SCMOE_COMBINE_DIRECT_ADD 0
#define SCMOE_COMBINE_CG1 1
#define SCMOE_COMBINE_CG2 2

/* GEMM epilogues: expert_forward (arch.py:349-351) and its backward */
#define SCMOE_EPI_BIAS 0
#define SCMOE_EPI_BIAS_GELU 1
#define SCMOE_EPI_GELU_BWD 2     /* out = acc * gelu'(aux_in)  (tape.py:137-142) */
#define SCMOE_EPI_MUL_AUX 3      /* out = acc * aux_in (aux_in = gelu'(z) saved by the forward) */

/* weight operand layouts of scmoe_grouped_gemm_ex */
#define SCMOE_W_NK 0             /* (W, n_out, k_in): the stored K-major weights */
#define SCMOE_W_KN 1             /* (W, k_in, n_out): stored weights used transposed (dgrad) */

#define SCMOE_MAX_EXPERTS 64
#define SCMOE_MAX_K 8

int scmoe_version(void);
const char* scmoe_last_error(void);
/* 0 when device `device` is an sm_100 part this library can run on. */
int scmoe_device_check(int device);

/*
 * K1 / K1b — gate + top-k + capacity slots in one pass.
 * Replaces gating.gate_logits (gating.py:93-107) / arch._gate_logits_node
 * (arch.py:405-415), gating.topk_indices + select_topk (gating.py:110-131),
 * gating.expert_quota + apply_capacity (gating.py:134-156) and the
 * count / mean-probability half of load_balance_loss (gating.py:159-170).
 *
 *   logits[t,e]  = x[t,:] . w_gate[:,e]  (+ eps[t,e]*softplus(x[t,:].w_noise[:,e]))  fp32
 *   indices[t,j] = j-th largest logit, ties -> lowest expert index (strict >)
 *   weights[t,j] = softmax over the k selected logits (top-1: exactly 1.0)
 *   slots[t,j]   = #earlier selections of the same expert in token-major order
 *   dropped[t,j] = slots[t,j] >= quota   (quota = ceil(cf*T*k/N), host-computed)
 *   counts[e]    = pre-drop selections of expert e   (int32, overwritten)
 *   prob_sum[e]  = sum_t softmax(logits[t,:])[e]     (fp32, overwritten)
 * w_gate_t / w_noise_t are (N, d) fp32 (transposed gate weights); w_noise_t
 * and eps are NULL when noise is disabled.  exclude (T,) int32 or NULL: an
 * expert per token that must not be selected — DGMoE's distinct-expert
 * constraint (arch.py:447-460): the top-1 over the remaining experts is the
 * runner-up exactly when the best expert clashes.  x is (T, d) with row stride
 * ld_x elements, dtype SCMOE_F32 or SCMOE_BF16.  N <= 64, 1 <= k <= min(N, 8).
 * bf16 tokens without noise and N <= 16 take the tensor-core logit path
 * (mma.sync on a 3-part bf16 split of the fp32 weights, fp32 accumulate).
 * The workspace (size from scmoe_gate_workspace_bytes) holds the tile
 * counters, per-tile status words and the split-weight blob.
 */
size_t scmoe_gate_workspace_bytes(int n_tokens, int n_experts, int d_model);
int scmoe_gate_topk(const void* x, int x_dtype, long long ld_x,
                    const float* w_gate_t, const float* w_noise_t, const float* eps,
                    const int32_t* exclude,
                    int n_tokens, int d_model, int n_experts, int k, int quota,
                    float* logits, int32_t* indices, float* weights, int32_t* slots,
                    uint8_t* dropped, int32_t* counts, float* prob_sum,
                    void* workspace, size_t workspace_bytes, void* stream);

/* The tensor-core gate (bf16 tokens, no noise, N <= 16, d >= 64) multiplies a
 * 3-part bf16 split of the fp32 gate weights.  scmoe_gate_topk splits them on
 * every call; an inference caller with fixed weights splits once
 * (scmoe_gate_split_weights into scmoe_gate_split_bytes of 16-byte aligned
 * device memory) and calls scmoe_gate_topk_presplit — same outputs, one
 * kernel launch less.  split_bytes is 0 when the tensor-core path does not
 * apply. */
size_t scmoe_gate_split_bytes(int n_experts, int d_model);
int scmoe_gate_split_weights(const float* w_gate_t, int n_experts, int d_model, void* blob,
                             void* stream);
int scmoe_gate_topk_presplit(const void* x, int x_dtype, long long ld_x, const float* w_gate_t,
                             const void* w_split, const int32_t* exclude, int n_tokens,
                             int d_model, int n_experts, int k, int quota, float* logits,
                             int32_t* indices, float* weights, int32_t* slots, uint8_t* dropped,
                             int32_t* counts, float* prob_sum, void* workspace,
                             size_t workspace_bytes, void* stream);
/* Both of the above in one entry (w_split may be null; noise as in
 * scmoe_gate_topk), plus `sync`: two uint32 words the caller zeroes ONCE
 * and keeps for the gate's lifetime.  Every launch leaves them zero, so the
 * tensor-core path issues no per-call memset of its cross-CTA counter (in a
 * CUDA graph a memset node costs ~8 us of idle GPU).  Launches sharing one
 * `sync` must not overlap in time (one stream per gate).  Null = the
 * workspace's counter, zeroed per call. */
int scmoe_gate_topk_ex(const void* x, int x_dtype, long long ld_x, const float* w_gate_t,
                       const void* w_split, const float* w_noise_t, const float* eps,
                       const int32_t* exclude, int n_tokens, int d_model, int n_experts, int k,
                       int quota, float* logits, int32_t* indices, float* weights,
                       int32_t* slots, uint8_t* dropped, int32_t* counts, float* prob_sum,
                       void* workspace, size_t workspace_bytes, uint32_t* sync, void* stream);

/*
 * K2 — dispatch ("encode"): copy each kept selection's row
 * of x_src into the capacity-slotted buffer
 *   dispatch_buf[(e * capacity + slots[t,j]) * d_model + :] = x[t,:]
 * for slots[t,j] < capacity.  Rows past an expert's fill are left untouched.
 * The reference never permutes (it evaluates experts densely,
 * arch.py:418-433); this is the sparse equivalent.
 */
int scmoe_dispatch(const void* x, int dtype, long long ld_x, int n_tokens, int d_model,
                   int k, const int32_t* indices, const int32_t* slots, int capacity,
                   void* dispatch_buf, void* stream);

/* K7 — combine backward: like scmoe_dispatch with every copied row scaled by
 * row_scale[t, j] (fp32, (T, k)): d expert_out[e, slot] = w[t, j] * d_out[t]
 * (the VJP of routed = sum_j w_j E_{e_j}, arch.py:418-433). */
int scmoe_dispatch_scaled(const void* x, int dtype, long long ld_x, int n_tokens, int d_model,
                          int k, const int32_t* indices, const int32_t* slots, int capacity,
                          const float* row_scale, void* dispatch_buf, void* stream);

/*
 * K3 / K4 / K8 — one grouped GEMM of expert_forward (arch.py:349-351):
 *   out[g, r, :] = epi( a[g, r, :] . wt[g % n_wgroups, :, :]^T + bias[g % n_wgroups, :] )
 * for r < rows(g), rows(g) = min(group_rows[g], rows_clip) (group_rows NULL:
 * rows(g) = group_cap).  a is (num_groups, group_cap, k_in), wt is
 * (n_wgroups, n_out, k_in), bias (n_wgroups, n_out) fp32 or NULL, out is
 * (num_groups, group_cap, n_out); epi = bias (+ exact-erf GELU), then
 * + residual[g, r, :] when `residual` (same layout as out) is not NULL — the
 * block's residual add (arch.py:542, 587-588) fused into the epilogue.
 * SCMOE_BF16 runs the tcgen05/TMEM/TMA kernel (fp32 accumulate);
 * SCMOE_F32 runs the fp32 FFMA parity kernel.
 */
int scmoe_grouped_gemm(const void* a, int dtype, const void* wt, const float* bias,
                       const void* residual, void* out,
                       int num_groups, int n_wgroups, int group_cap,
                       const int32_t* group_rows, int rows_clip,
                       int n_out, int k_in, int epilogue, void* stream);

/*
 * K3 / K7 — general form of scmoe_grouped_gemm (bf16):
 *   out[g, r, :] = epi( a[g, r, :] . Wg + bias )  (+ residual), r < rows(g)
 * with Wg = w[g % W]^T for w_layout SCMOE_W_NK (w is (W, n_out, k_in)) or
 * Wg = w[g % W] for SCMOE_W_KN (w is (W, k_in, n_out)), i.e. the same stored
 * weights read transposed for the data gradient.  Epilogues:
 *   SCMOE_EPI_BIAS / SCMOE_EPI_BIAS_GELU (aux_out, if not NULL, receives the
 *   pre-activation acc + bias as bf16), SCMOE_EPI_GELU_BWD (out = acc *
 *   gelu'(aux_in), aux_in laid out like out).
 * zero_tail != 0 writes zeros to rows [rows(g), min(cap, tile end)) — the
 * padding the weight-gradient GEMM relies on.
 */
int scmoe_grouped_gemm_ex(const void* a, int dtype, const void* w, int w_layout,
                          const float* bias, const void* residual, const void* aux_in,
                          void* aux_out, void* out, int num_groups, int n_wgroups,
                          int group_cap, const int32_t* group_rows, int rows_clip,
                          int n_out, int k_in, int epilogue, int zero_tail, void* stream);

/*
 * K7 — grouped weight gradient (tape.mm VJP, tape.py:121-127):
 *   out[w] (m_out, n_out) fp32 = sum_{g = w mod W} sum_{r < rows(g)} a[g, r, :m_out]^T b[g, r, :n_out]
 * a is (num_groups, group_cap, m_out), b is (num_groups, group_cap, n_out),
 * bf16.  Rows [rows(g), roundup(rows(g), 64)) of a and b must be zero (the
 * producers' zero_tail / scmoe_zero_tails guarantee it).  splits <= 0 picks a
 * split-K factor that fills the GPU; splits > 1 needs
 * scmoe_grouped_wgrad_workspace_bytes() of workspace.
 */
size_t scmoe_grouped_wgrad_workspace_bytes(int n_wgroups, int m_out, int n_out, int splits);
int scmoe_grouped_wgrad(const void* a, const void* b, int dtype, float* out, void* workspace,
                        size_t workspace_bytes, int num_groups, int n_wgroups, int group_cap,
                        const int32_t* group_rows, int rows_clip, int m_out, int n_out,
                        int splits, void* stream);

/* scmoe_grouped_wgrad with the output in the parameter dtype: out_dtype
 * SCMOE_F32 or SCMOE_BF16 (the split reduction rounds once to bf16, no
 * separate conversion pass).  A bf16 out always needs max(splits, 1) splits
 * of workspace (W x m_out x n_out fp32 each). */
int scmoe_grouped_wgrad_ex(const void* a, const void* b, int dtype, void* out, int out_dtype,
                           void* workspace, size_t workspace_bytes, int num_groups, int n_wgroups,
                           int group_cap, const int32_t* group_rows, int rows_clip, int m_out,
                           int n_out, int splits, void* stream);

/* rows [rows(g), min(cap, roundup(rows(g), align))) of every group set to 0 */
int scmoe_zero_tails(void* buf, int dtype, int num_groups, int group_cap, int cols,
                     const int32_t* group_rows, int rows_clip, int align, void* stream);

/* out[g, c] = sum_{r < rows(g)} x[g, r, c] in fp32 (bias gradients), two
 * deterministic passes through a caller-owned workspace */
size_t scmoe_grouped_colsum_workspace_bytes(int num_groups, int group_cap, int cols);
int scmoe_grouped_colsum(const void* x, int dtype, int num_groups, int group_cap, int cols,
                         const int32_t* group_rows, int rows_clip, float* out,
                         void* workspace, size_t workspace_bytes, void* stream);
/* Two matrices with the same groups (x0: (G, cap, cols0), x1: (G, cap,
 * cols1), e.g. an FFN's two bias gradients dy and dz) in one launch per
 * pass: out0 (G, cols0), out1 (G, cols1), same arithmetic as two
 * scmoe_grouped_colsum calls.  The passes are programmatic dependent
 * launches. */
size_t scmoe_grouped_colsum2_workspace_bytes(int num_groups, int group_cap, int cols0,
                                             int cols1);
int scmoe_grouped_colsum2(const void* x0, const void* x1, int dtype, int num_groups,
                          int group_cap, int cols0, int cols1, const int32_t* group_rows,
                          int rows_clip, float* out0, float* out1, void* workspace,
                          size_t workspace_bytes, void* stream);

/* Balance loss from the gate's statistics (arch.py:436-439, gating.py:
 * 159-170): *aux = N * sum_e (counts[e] / (T k)) (prob_sum[e] / T), fp32,
 * experts summed in order. */
int scmoe_gate_aux_loss(const int32_t* counts, const float* prob_sum, int n_tokens,
                        int n_experts, int k, float* aux, void* stream);

/* out[i] = dtype(src[0] / div), i < n: the constant gradient of a mean loss
 * (grad.py:52-67) from a device scalar without a host sync; 16-byte aligned
 * out. */
int scmoe_fill_div(void* out, int dtype, long long n, const float* src, float div, void* stream);

/* *out = mean(x[0..n)) accumulated in fp32, deterministic two-pass (the
 * "mean" LossSpec, grad.py:52-67); workspace of scmoe_mean_workspace_bytes()
 * bytes; no memset. */
size_t scmoe_mean_workspace_bytes(void);
int scmoe_mean(const void* x, int dtype, long long n, float* out, void* workspace,
               size_t workspace_bytes, void* stream);

/* Expert migration (offload.py:109-182 made real): dst[j] = src[ids[j]] for
 * j < min(*n_rows, max_rows), rows of row_bytes.  src may be pinned host
 * memory (read over the host link by the kernel, no host synchronisation:
 * the activated-expert list and its length stay on the device). */
int scmoe_gather_rows(const void* src, size_t row_bytes, const int32_t* ids,
                      const int32_t* n_rows, int max_rows, void* dst, void* stream);

/* In-place SGD over n tensors in one launch (grad.py:330-331): p[i] -= lr *
 * g[i] in fp32, rounded to the parameter dtype (SCMOE_BF16 / SCMOE_F32,
 * gradient in the same dtype).  Host arrays of device pointers; numels a
 * multiple of the 16-byte vector width, storage 16-byte aligned. */
int scmoe_sgd_update(void* const* params, const void* const* grads, const long long* numels,
                     const int* dtypes, int n, float lr, void* stream);

/* Expert migration on the COPY ENGINE (offload.py:109-182, the H2D transfer
 * of the activated experts): dst[j] = src[ids[j]] for j < n_rows, rows of
 * row_bytes, as cudaMemcpyAsync on `stream` (runs of consecutive ids merged
 * into one copy).  ids is a HOST array (the caller read the activated-expert
 * list back); no SM time is spent, so the copies overlap persistent GEMMs
 * that hold every SM.  src: pinned host (or device) memory. */
int scmoe_copy_rows(const void* src, size_t row_bytes, const int32_t* ids, int n_rows, void* dst,
                    void* stream);

/* Attention layout glue (training): n_src (<= 3) bf16 tensors (B, H, S, hd),
 * element strides[3*i .. 3*i+2] = (b, h, s) of source i, hd contiguous, packed
 * into dst (B, S, n_src, H, hd) contiguous — dq/dk/dv into the packed QKV
 * gradient, the SDPA output into (T, d) rows.  srcs / strides are host arrays. */
int scmoe_pack_heads(const void* const* srcs, const long long* strides, int n_src, int B, int H,
                     int S, int hd, int dtype, void* dst, void* stream);

/* Experiment hook: bit 0 = epilogue operands (residual / pre-activation)
 * read row-per-thread instead of staged through cp.async buffers. */
int scmoe_set_gemm_flags(int flags);

/* Tuning / test hook: 0 = pick the tcgen05 variant by problem size, 1 = force
 * the 1-SM 128x256 kernel, 2 = force the 2-SM (cta_group::2) 256x256 kernel. */
int scmoe_set_gemm_mode(int mode);

/* SMs the persistent forward / dgrad GEMMs may occupy, 0 = all (default).
 * The ScMoE block lowers it to (SMs - p2p_ctas) for the window operators
 * that run while a peer-memory exchange kernel is in flight on the side
 * stream, so the exchange executes concurrently (distsim.py:330-387 overlap
 * made real on one device).  Host-side state read at launch (captured into
 * CUDA graphs as launched). */
int scmoe_set_gemm_sm_budget(int sms);

/* Tuning / test hook: epilogue warps of the forward / dgrad tcgen05 GEMM,
 * 0 = auto (16 for K <= 1024 tiles with an elementwise epilogue, else 8),
 * 8 or 16 forced. */
int scmoe_set_gemm_epilogue_warps(int warps);

/* Tuning / test hook: tcgen05 tile width, 0 = auto (128 when n_out is an odd
 * multiple of 128 and the narrow tile needs fewer column-waves), 128 or 256. */
int scmoe_set_gemm_tile_n(int bn);

/*
 * Full expert_forward (arch.py:349-351) over groups: GEMM1 (bias+GELU) into
 * `hidden` (num_groups, group_cap, d_hidden), then GEMM2 (bias, + residual
 * when not NULL) into `out`.
 * The dense shared expert / Block-MLP is num_groups = n_wgroups = 1,
 * group_rows = NULL, group_cap = T.
 */
int scmoe_expert_ffn(const void* x, int dtype, const void* w1t, const float* b1,
                     const void* w2t, const float* b2, const void* residual,
                     void* hidden, void* out,
                     int num_groups, int n_wgroups, int group_cap,
                     const int32_t* group_rows, int rows_clip,
                     int d_model, int d_hidden, void* stream);

/*
 * K4+K5 fused (inference, direct-add combine): the shared expert on x_cur
 * whose GEMM2 epilogue also gathers the routed rows and the residual:
 *   out[t] = bf16(SE(x_cur)[t]) + sum_j w[t,j] * expert_out[idx[t,j], slot[t,j]]
 *            (+ residual[t]),   selections with slot >= capacity skipped,
 * bit-identical to scmoe_expert_ffn followed by scmoe_combine (same fp32
 * operation order) without the SE output round trip or the combine launch.
 * bf16, one group of n_tokens rows, k <= 2.  hidden: (n_tokens, d_hidden).
 */
int scmoe_shared_ffn_combine(const void* x, int dtype, const void* w1t, const float* b1,
                             const void* w2t, const float* b2, const void* residual,
                             const void* expert_out, const int32_t* indices,
                             const int32_t* slots, const float* weights, int capacity, int k,
                             void* hidden, void* out, int n_tokens, int d_model, int d_hidden,
                             void* stream);
/* Its second half alone: out = the fused-combine GEMM2 over an already
 * computed hidden = gelu(x_cur W1 + b1) (a caller that runs GEMM1 while the
 * routed rows are still being produced on another stream). */
int scmoe_ffn2_combine(const void* hidden, int dtype, const void* w2t, const float* b2,
                       const void* residual, const void* expert_out, const int32_t* indices,
                       const int32_t* slots, const float* weights, int capacity, int k, void* out,
                       int n_tokens, int d_model, int d_hidden, void* stream);

/*
 * K5 — combine ("decode") + combination gate + optional residual:
 *   routed[t] = sum_j (slots[t,j] < capacity) * weights[t,j] * expert_out[indices[t,j], slots[t,j], :]
 *   direct_add: f = se + routed; cg1: f = sigmoid(x_cur.w_cg[0]) * se + routed;
 *   cg2: c = softmax(x_cur.w_cg^T); f = c0 * se + c1 * routed
 *   out[t] = f (+ residual[t] when residual != NULL)
 * (arch.py:380-392 combine, arch.py:481-483 weights*keep, arch.py:616
 * residual add).  w_cg is (1|2, d) fp32; x_cur only read for CG modes;
 * se_out NULL means "no shared expert" (moe_standard, arch.py:489-493).
 */
int scmoe_combine(const void* se_out, const void* expert_out, const void* x_cur,
                  const float* w_cg, int mode, const void* residual,
                  const int32_t* indices, const int32_t* slots, const float* weights,
                  int capacity, int n_tokens, int d_model, int k, int dtype,
                  void* out, void* stream);

/*
 * K9 / K10 — expert parallelism over NVLink / NVSwitch peer memory (SURVEY
 * §8(e); replaces the two all-to-alls around the routed experts).  Global
 * expert e = r * experts_per_rank + el lives on rank r.  Every rank owns, in
 * memory every peer can address (symmetric memory), a receive buffer
 * recv (world, E_l, C, d), an output buffer y (same layout), recv_counts
 * (world * E_l) int32 and flags (2 * world) uint32; epoch_ctr (2) uint32 is
 * local, zero-initialised.  The peer tables are DEVICE arrays of `world`
 * pointers (entry r = rank r's buffer).
 *
 * scmoe_ep_dispatch_p2p: every kept selection (t, j) of this rank's tokens is
 *   stored straight into recv_r[(rank*E_l + el)*C + slot] on its owner r (only
 *   kept rows move); recv_counts_r[rank*E_l + el] = min(counts[e], C); then the
 *   epoch flag flags_r[0][rank] is released on every peer.  counts = pre-drop
 *   per global expert (the gate's counts).  max_ctas > 0 bounds the grid so
 *   the copy can run beside compute on a side stream.
 * scmoe_ep_wait(which): spin until flags[which][s] >= this rank's epoch for
 *   every s (which 0: all dispatches into my recv landed; 1: every owner's y
 *   is ready).  Traps after ~20 s instead of hanging.
 * scmoe_ep_signal(which): release flags_r[which][rank] = epoch on every peer
 *   (which 1 after the grouped FFN wrote y).
 * scmoe_ep_combine_p2p: scmoe_combine with each expert row read from
 *   y_r[(rank*E_l + el)*C + slot] on its owner r (return trip fused into the
 *   combine's loads).
 * scmoe_ep_return_p2p: return trip as a push (side stream, overlaps the window
 *   ops after the expert): rows < recv_counts[g] of y group g = (src, el) are
 *   stored into back_src[(rank*E_l + el)*C + row], then flags_src[1][rank] is
 *   released; the source waits (which 1) and runs scmoe_combine on back.
 *   epoch_ctr needs 3 words for this entry.
 */
int scmoe_ep_dispatch_p2p(const void* x, int dtype, long long ld_x, int n_tokens, int d_model,
                          int k, const int32_t* indices, const int32_t* slots,
                          const int32_t* counts, int capacity, int world, int rank,
                          int experts_per_rank, void* const* peer_recv,
                          int32_t* const* peer_recv_counts, uint32_t* const* peer_flags,
                          uint32_t* epoch_ctr, int max_ctas, void* stream);
int scmoe_ep_wait(const uint32_t* flags, int which, int world, const uint32_t* epoch_ctr,
                  void* stream);
int scmoe_ep_signal(uint32_t* const* peer_flags, int which, int world, int rank,
                    const uint32_t* epoch_ctr, void* stream);
int scmoe_ep_combine_p2p(const void* se_out, const void* const* peer_y, const void* x_cur,
                         const float* w_cg, int mode, const void* residual,
                         const int32_t* indices, const int32_t* slots, const float* weights,
                         int capacity, int n_tokens, int d_model, int k, int dtype, int world,
                         int rank, int experts_per_rank, void* out, void* stream);
/* Expert-parallel return fused into the expert FFN (one kernel does the
 * GEMM and the transfer): scmoe_expert_ffn whose GEMM2 epilogue stores the
 * rows of group g to out_group_ptrs[g] + row * d_model (a DEVICE array of
 * num_groups pointers — on the owner rank, group (src, el) points into the
 * source's back buffer over peer memory), tile by tile, then fences at
 * system scope; follow with scmoe_ep_signal(which 1). */
int scmoe_expert_ffn_to_peers(const void* x, int dtype, const void* w1t, const float* b1,
                              const void* w2t, const float* b2, void* hidden,
                              void* const* out_group_ptrs, int num_groups, int n_wgroups,
                              int group_cap, const int32_t* group_rows, int rows_clip,
                              int d_model, int d_hidden, void* stream);
int scmoe_ep_return_p2p(const void* y, int dtype, const int32_t* recv_counts, int capacity,
                        int d_model, int world, int rank, int experts_per_rank,
                        void* const* peer_back, uint32_t* const* peer_flags, uint32_t* epoch_ctr,
                        int max_ctas, void* stream);

/* Gate backward (K7): VJP of the kept-selection weights (k > 1, masked
 * softmax, tape.py:161-176) and of the balance loss (arch.py:436-439, d_aux a
 * DEVICE scalar, may be null) through H = src W_gate (+ eps softplus(src
 * W_noise), arch.py:405-415).  Writes d_src (T, d) in src's dtype (may be
 * null), d_w_gate (N, d) fp32 and, with noise (w_noise_t, eps, noise_pre =
 * src W_noise all non-null), d_w_noise (N, d) fp32; weight gradients are
 * summed in a fixed order through the workspace (deterministic). */
size_t scmoe_gate_backward_workspace_bytes(int n_tokens, int d_model, int n_experts, int noise);
int scmoe_gate_backward(const void* src, int dtype, int n_tokens, int d_model, int n_experts,
                        int k, const float* logits, const int32_t* indices, const float* weights,
                        const float* d_weights, const int32_t* counts, const float* d_aux,
                        const float* w_gate_t, const float* w_noise_t, const float* eps,
                        const float* noise_pre, void* d_src, float* d_w_gate, float* d_w_noise,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Windowed multi-head attention (the configs[1] backbone: 144-token windows,
 * 12 heads of 32), forward and backward on the packed QKV projection:
 * qkv (T, 3*H*hd) bf16 rows [q | k | v], heads contiguous hd-wide slices;
 * windows of seq_len consecutive rows (T % seq_len == 0), O = softmax(Q K^T
 * scale (+ causal mask)) V per window and head (arch.py:354-358 generalised
 * to heads / windows), out (T, H*hd) bf16, lse (T, H) fp32 base-2 row
 * log-sum-exp of the scaled scores (may be null in the forward).  The
 * backward writes dqkv (T, 3*H*hd) in the packed layout from qkv, out, dout
 * and lse.  Supported: seq_len % 16 == 0, 16 <= seq_len <= 192, hd 32 or 64
 * (scmoe_window_attention_supported). */
int scmoe_window_attention_supported(int seq_len, int head_dim);
int scmoe_window_attention_fwd(const void* qkv, int n_tokens, int n_heads, int head_dim,
                               int seq_len, float scale, int causal, void* out, float* lse,
                               void* stream);
int scmoe_window_attention_bwd(const void* qkv, const void* out, const void* dout,
                               const float* lse, int n_tokens, int n_heads, int head_dim,
                               int seq_len, float scale, int causal, void* dqkv, void* stream);

/* Training FFN elementwise GELU passes (exact-erf GELU, numkit.py:96-99;
 * tape.py:137-142), bf16 (num_groups, group_cap, cols) buffers, rows(g) =
 * min(group_rows[g], rows_clip) (all rows when group_rows is null), rows_pad(g)
 * = min(group_cap, roundup(rows(g), 64)):
 *   scmoe_gelu_fwd: h = gelu(z) on rows < rows(g), zeros up to rows_pad(g);
 *   scmoe_gelu_bwd: dz = dh * gelu'(z) on rows < rows(g), zeros up to
 *     rows_pad(g), and (bias_grad non-null) bias_grad[g][c] = sum of dz over
 *     the valid rows, fixed-order (deterministic) through the workspace. */
int scmoe_gelu_fwd(const void* z, void* h, int num_groups, int group_cap, int cols,
                   const int32_t* group_rows, int rows_clip, void* stream);

/* Training forward GELU that also saves the derivative: h = gelu(z) and
 * dgelu = gelu'(z) (tape.py:137-142), both bf16, rows past rows(g) zero up to
 * the 64-row block.  The backward then forms dz = (dy W2) * dgelu in the
 * data-gradient GEMM's epilogue (SCMOE_EPI_MUL_AUX): no erf in the backward,
 * no separate elementwise pass. */
int scmoe_gelu_fwd_grad(const void* z, void* h, void* dgelu, int num_groups, int group_cap,
                        int cols, const int32_t* group_rows, int rows_clip, void* stream);
size_t scmoe_gelu_bwd_workspace_bytes(int num_groups, int group_cap, int cols);
int scmoe_gelu_bwd(const void* dh, const void* z, void* dz, float* bias_grad, int num_groups,
                   int group_cap, int cols, const int32_t* group_rows, int rows_clip,
                   void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SCMOE_H_ */
