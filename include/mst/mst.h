/*
 * mst.h — C ABI of the B200-native Mini-Sequence Transformer (MsT) hot path.
 *
 * The reference (arxiv 2407.15892, mounted at /root/reference) specifies the
 * operator API of module `miniseq` in prose and ships no
 * implementation.  Each entry point below replaces one SPEC operation; the
 * citation is given per function.  All compute runs on sm_100a kernels from
 * libmst.so; there is no CPU fallback.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are CUDA device memory;
 *    `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Activations/weights are bf16 (uint16 storage), row-major, in the SPEC
 *    orientation: X[N,H]; W_gate, W_up [H,I]; W_down [I,H]; W_out [H,V]
 *    (SPEC.md:179-185).  Weight gradients are fp32 row-major, same shapes.
 *    Labels are int32 [N] with ignore value -100.
 *  - The caller owns every buffer, including the scratch `workspace`
 *    (size from the matching *_workspace query).  Calls are asynchronous on
 *    `stream`; results are valid after the stream is synchronised.
 *  - Errors: every function returns an mst_status; mst_last_error() gives a
 *    thread-local message.  Codes map 1:1 onto the reference's error
 *    taxonomy (proj/include/minitrain/error.hpp:14-20).
 */
#ifndef MST_MST_H_
#define MST_MST_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MST_ABI_VERSION 1

#if defined(__GNUC__)
#define MST_API __attribute__((visibility("default")))
#else
#define MST_API
#endif

typedef enum mst_status {
  MST_OK = 0,
  MST_ERR_SHAPE = 1,     /* minitrain::ShapeError      error.hpp:14 */
  MST_ERR_BOUNDS = 2,    /* minitrain::BoundsError     error.hpp:15 */
  MST_ERR_DTYPE = 3,     /* minitrain::DtypeError      error.hpp:16 */
  MST_ERR_CONFIG = 4,    /* minitrain::ConfigError     error.hpp:17 */
  MST_ERR_DATA = 5,      /* minitrain::DataError       error.hpp:18 */
  MST_ERR_STATE = 6,     /* minitrain::StateError      error.hpp:19 */
  MST_ERR_NONFINITE = 7, /* minitrain::NonFiniteError  error.hpp:20 */
  MST_ERR_CUDA = 8,      /* CUDA runtime / driver failure (no reference analogue) */
  MST_ERR_INTERNAL = 9
} mst_status;

/* Loss reduction over mini-sequences. */
typedef enum mst_loss_mode {
  MST_LOSS_TOKEN_WEIGHTED = 0, /* sum(loss_sum_i) / sum(valid_i)  (default) */
  MST_LOSS_PAPER_MEAN = 1      /* (sum_i mean_i) / M  (Alg. 2 line 8 literal) */
} mst_loss_mode;

typedef struct mst_ctx mst_ctx;

/* Layout of the device `stats` buffer written by mst_lmhead_forward.
 * MST_STATS_LEN(M) floats: [0] loss_sum, [1] valid count, [2] loss,
 * [3] invalid-label count, [4..4+M) per-chunk loss sums,
 * [4+M..4+2M) per-chunk valid counts.  Entries 0..1 are additive across
 * sequence shards (all-reduce SUM them for the global token-weighted loss). */
#define MST_STATS_LEN(M) (4 + 2 * (M))

/* Saved state between forward and backward.
 * Filled by the forward call; the backward call checks the fingerprint and
 * raises MST_ERR_STATE on a stale or mismatched record. */
typedef struct mst_mlp_saved {
  const void* x;
  const void* w_gate;
  const void* w_up;
  const void* w_down;
  int64_t n, h, i, m;
  uint64_t fingerprint;
} mst_mlp_saved;

typedef struct mst_lmhead_saved {
  const void* x;
  const int32_t* labels;
  const void* w_out;
  float* lse;   /* device [n] fp32: log-sum-exp per row (the only saved activation) */
  float* stats; /* device MST_STATS_LEN(m) */
  int64_t n, h, v, m;
  int32_t loss_mode;
  int32_t _pad;
  uint64_t fingerprint;
} mst_lmhead_saved;

MST_API int mst_abi_version(void);
MST_API const char* mst_last_error(void);

/* Context: one per host thread per device (SPEC.md:99 threading contract).
 * Calls on one context are serialised by a context lock, and a call on a
 * different stream than the previous call first waits (device-side event)
 * for the previous call's work: the context's device scratch (tile counter,
 * valid-count scratch) is shared by its calls, the stream is per call.  For
 * concurrent work on several streams use one context per stream.
 *
 * Deferred errors: data errors that only the device can see -- every label
 * ignored (DataError), labels outside [0, V) other than -100
 * (DataError), a non-finite loss (NonFiniteError) -- are raised
 * into the context's sticky error word by the kernel that computes the loss.
 * The first call that starts after that kernel has completed returns the
 * error (and clears it) without doing any work; mst_ctx_check synchronises
 * `stream` and returns it at once. */
MST_API int mst_ctx_create(int device, mst_ctx** out);
MST_API void mst_ctx_destroy(mst_ctx* ctx);
MST_API int mst_ctx_check(mst_ctx* ctx, void* stream);
/* Number of CTA pairs a grouped launch uses (diagnostics / tests). */
MST_API int mst_ctx_num_pairs(const mst_ctx* ctx);
/* Kernel launches issued by this context since creation (bench evidence). */
MST_API int64_t mst_ctx_launch_count(const mst_ctx* ctx);

/* Per-launch device timing of the grouped tcgen05 GEMM kernel (the
 * dominant kernel): when enabled, CUDA events are recorded on the launch
 * stream around every launch.  mst_ctx_take_timing() synchronises on them
 * and returns, for the launches since the previous call, the summed device
 * time (ms), their algorithmic FLOPs (2*M*N*K of the valid extents) and the
 * launch count, then resets. */
MST_API int mst_ctx_set_timing(mst_ctx* ctx, int enable);
MST_API int mst_ctx_take_timing(mst_ctx* ctx, double* gemm_ms, double* gemm_flops, int64_t* gemm_launches);
/* Same, per launch: fills up to `cap` (ms, flops) records, returns the count
 * in *n and resets. */
MST_API int mst_ctx_take_timing_records(mst_ctx* ctx, int64_t cap, double* ms, double* flops, int64_t* n);

/* Tuning builds (-DMST_PROFILE) only: device buffer of 64 x 8 uint64 counters;
 * grouped-GEMM launch k (counted from this call) accumulates per-role
 * barrier-wait cycles into slot k % 64 (layout in csrc/gemm.cuh).  NULL
 * disables.  No effect in product builds. */
MST_API int mst_ctx_set_profile_buffer(mst_ctx* ctx, void* dev_counters);

/* Tuning knobs (benchmark / A-B use; defaults are the tuned values; the
 * measured effect of each is in DESIGN.md 4.2):
 *   "dynamic": 1 (default) CTA pairs pull tiles from the global LPT order
 *              through an atomic counter (a scheduler thread per pair claims
 *              up to 8 tiles ahead); 0 static per-pair LPT lists;
 *   "tma3d":   MN-major operands as 3-D tensor maps (default 1);
 *   "fused_head": 1 (default) block_step runs mst_lmhead_fused, 0 runs the
 *              separate forward + backward (logits recomputed);
 *   "chunked_block": 1 (default) block_step with M_mlp == M_head runs the
 *              chunk-wise MLP -> head -> MLP-backward schedule (no G,U
 *              recompute; bitwise-equal results), 0 the op-by-op schedule;
 *   "fuse_swiglu_bwd": 1 = SwiGLU backward in the dh GEMM epilogue (default 0);
 *   "wide", "wide_mask": wide tiles (two N blocks per CTA-pair tile) per GEMM
 *              of the chunk-wise block (default off); "debug_nblk" for
 *              mst_debug_gemm / mst_gemm;
 *   "pairs":   run the GEMMs on fewer CTA pairs (diagnostics);
 *   "pair_dw", "dl_rowscale", "k9_in_k1": chunk-wise schedule variants
 *              (defaults 1, 1, 0);
 *   "attn_fwd", "attn_bwd": attention kernel versions (default 2, 2);
 *   "attn_bwd_order": backward issue orders, bit 0 dK/dV, bit 1 dQ (default 3);
 *   "attn_inorder": 1 = no completion wait between dependent MMAs (default 0);
 *   "attn_poly": forward exp2 pairs (of 4) on the FMA pipe, 0..3 (default 0).
 * Every knob belongs to the context.  Unknown keys are MST_ERR_CONFIG.
 * Changing a knob clears the schedule cache. */
MST_API int mst_ctx_set_tuning(mst_ctx* ctx, const char* key, int value);

/* ---------------------------------------------------------------- memtrack
 * The library's side of the reference's MemTracker (memtrack.hpp:138-228):
 *
 *  * Counters follow the fixed counting conventions of memtrack.hpp:19-35
 *    for the logical operations a call executes (every GEMM as
 *    count_matmul(N, K, P) with operands that are weight tensors added to
 *    weight_read_elements; SiLU / Hadamard / cross-entropy as count_op).
 *    Fused epilogues are counted as the ops they implement; zero-copy chunk
 *    slices count nothing (the reference's slice_rows copies 2*n*H).
 *    Accumulated per context at enqueue time, read with
 *    mst_ctx_get_counters, zeroed with mst_ctx_reset_counters.
 *  * Memory events: the chunk buffers a call carves from its workspace are
 *    reported with their logical lifetime (alloc when a chunk's buffer comes
 *    into use, free when it is dead) and the reference's label classes:
 *    "inter.mlp.*", "inter.head.*" (the [S/M, I] / [S/M, V] intermediates),
 *    "act.*" (activations the block step keeps: O, dO, lse, operand
 *    transposes).  Install a hook with mst_ctx_set_mem_hook; kind 0 = alloc
 *    (MemTracker::on_alloc), 1 = free (on_free).  The count hook, when set,
 *    receives every counted op as it is counted (kind 0: count_matmul(a, b,
 *    c, w); kind 1: count_op(flops = a, hbm = b)), so a C++ caller can
 *    forward both into minitrain::MemTracker::current(). */
typedef struct mst_counters {
  uint64_t flops, matmul_flops, hbm_elements, weight_read_elements;
} mst_counters;
typedef void (*mst_mem_hook)(void* user, int kind, uint64_t bytes, const char* label);
typedef void (*mst_count_hook)(void* user, int kind, int64_t a, int64_t b, int64_t c, uint64_t w);
MST_API int mst_ctx_get_counters(const mst_ctx* ctx, mst_counters* out);
MST_API int mst_ctx_reset_counters(mst_ctx* ctx);
MST_API int mst_ctx_set_mem_hook(mst_ctx* ctx, mst_mem_hook fn, void* user);
MST_API int mst_ctx_set_count_hook(mst_ctx* ctx, mst_count_hook fn, void* user);

/* ---------------------------------------------------------------- optimizer
 * The reference's `optim` module on the device: fp32
 * master weights, fp32 moments, fp32 gradients (the dW accumulators), and
 * the bf16 copy the GEMMs read.  All asynchronous on `stream`.
 *
 * mst_adamw_step       adamw_step: w -= lr*wd*w, then the
 *                      Adam moment update with bias correction for `step`
 *                      (>= 1); the gradient is multiplied by *grad_scale when
 *                      non-NULL (device scalar: clip factor / accumulation
 *                      steps); zero_grad != 0 clears the gradient after use.
 * mst_grad_sumsq       squared L2 norm of one gradient into the device fp64
 *                      *sumsq (accumulate != 0 adds to it; call once per
 *                      tensor for a global norm), deterministic fixed-grid
 *                      reduction through partial_ws (mst_grad_sumsq_workspace()
 *                      doubles).  When scale_out != NULL it also writes
 *                      clip_global_norm's factor times
 *                      inv_steps: max_norm/||g|| if ||g|| > max_norm else 1
 *                      (NaN when ||g|| is non-finite), and ||g|| to norm_out.
 * mst_grad_accumulate  accumulate: into += from; the
 *                      division by the step count is the 1/steps folded into
 *                      grad_scale at flush. */
typedef struct mst_adamw_config { /* doubles: 1 - beta2 must not round through fp32 */
  double lr, weight_decay, beta1, beta2, eps;
} mst_adamw_config;
MST_API int mst_adamw_step(mst_ctx* ctx, void* stream, int64_t n, float* w, void* w_bf16, float* grad, float* m,
                           float* v, const mst_adamw_config* cfg, int64_t step, const float* grad_scale,
                           int zero_grad);
MST_API int mst_grad_sumsq_workspace(void);
MST_API int mst_grad_sumsq(mst_ctx* ctx, void* stream, const float* grad, int64_t n, double* partial_ws,
                           double* sumsq, int accumulate, float max_norm, float inv_steps, float* scale_out,
                           float* norm_out);
MST_API int mst_grad_accumulate(mst_ctx* ctx, void* stream, float* into, const float* from, int64_t n);

/* Gradient-ready hook (optimizer-in-backward): during
 * mst_block_step the library calls fn(user, which, stream) at enqueue time
 * right after the launch that makes a weight gradient final in stream order
 * (which: 0 W_gate, 1 W_up, 2 W_down, 3 W_out), so the caller can enqueue
 * that parameter's optimizer step on the same stream and release its
 * gradient while the rest of the backward is still queued.  NULL disables. */
typedef void (*mst_grad_ready_hook)(void* user, int which, void* stream);
MST_API int mst_ctx_set_grad_ready_hook(mst_ctx* ctx, mst_grad_ready_hook fn, void* user);

/* Gradient-slab hook (sequence-parallel overlap): during
 * mst_block_step[_sp|_host] the library calls fn(user, which, row0, row1,
 * stream) at enqueue time right after the launch that makes rows
 * [row0, row1) of weight gradient `which` (numbering as above; rows of the
 * row-major fp32 gradient, so every slab is one contiguous buffer) final in
 * stream order.  Every row of every gradient is reported exactly once per
 * call.  With `slabs` > 1 the chunk-wise schedule cuts the launches that
 * finalise dW_out (the last head chunk's dW_out GEMM) and dW_gate / dW_up
 * (the last MLP chunk's dW GEMM) into `slabs` row slabs of H, one launch
 * each, so a caller that all-reduces each slab as it is reported overlaps
 * most of the communication with the remaining launches (dW_down is one
 * slab).  slabs = 1: one report per gradient.  NULL disables. */
typedef void (*mst_grad_slab_hook)(void* user, int which, int64_t row0, int64_t row1, void* stream);
MST_API int mst_ctx_set_grad_slab_hook(mst_ctx* ctx, mst_grad_slab_hook fn, void* user, int slabs);

/* make_chunk_plan(N, M) — SPEC.md:286-294.  Writes min(M,N)+1 row bounds
 * into `bounds` (capacity >= min(M,N)+1): chunk c is [bounds[c], bounds[c+1]).
 * Balanced rule: the first N mod M chunks hold ceil(N/M) rows. */
MST_API int mst_make_chunk_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* num_chunks);

/* Scratch sizes (bytes) for each operation. */
MST_API int mst_mlp_workspace(int64_t n, int64_t h, int64_t i, int64_t m, size_t* bytes);
MST_API int mst_lmhead_workspace(int64_t n, int64_t h, int64_t v, int64_t m, size_t* bytes);
MST_API int mst_block_workspace(int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp, int64_t m_head, size_t* bytes);
/* Workspace of mst_block_step / mst_block_step_sp under this context's
 * schedule knobs (mst_block_workspace is the maximum over all schedules).
 * The chunk-wise schedule (default when m_mlp == m_head) keeps only one O
 * chunk and two dO chunks: 4 bytes of lse per token plus chunk buffers. */
MST_API int mst_ctx_block_workspace(const mst_ctx* ctx, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp,
                                    int64_t m_head, size_t* bytes);

/* mst_block_step with host-resident X, labels and dX (pinned host memory for
 * asynchronous copies): X_j is copied in chunk by chunk on the context's copy
 * stream while earlier chunks compute, dX_j is copied out as soon as it is
 * final, so the copies overlap the GEMMs and the device holds only chunk
 * buffers of X / dX (the sequence is bounded by host memory).  Chunk-wise
 * schedule only (M_mlp == M_head == m); results are bitwise those of
 * mst_block_step.  Everything is ordered on `stream` (the copy stream is
 * joined back before the call's work ends).  Workspace from
 * mst_ctx_block_host_workspace (the block workspace: the two X and two dX
 * chunk buffers and the labels are owned by the context, allocated on first
 * use and grown when a larger shape needs them; consecutive calls on one
 * context overlap a step's first X copy with the previous step's tail). */
MST_API int mst_ctx_block_host_workspace(const mst_ctx* ctx, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m,
                                         size_t* bytes);
MST_API int mst_block_step_host(mst_ctx* ctx, void* stream, const void* x_host, const int32_t* labels_host,
                                const void* w_gate, const void* w_up, const void* w_down, const void* w_out, int64_t n,
                                int64_t h, int64_t i, int64_t v, int64_t m, int loss_mode, float grad_loss, float* stats,
                                void* grad_x_host, float* grad_w_gate, float* grad_w_up, float* grad_w_down,
                                float* grad_w_out, int accumulate, void* workspace, size_t workspace_bytes);

/* miniseq_mlp_forward(X, w, plan) -> (O, saved) — SPEC.md:295-303, Alg. 1.
 * O = (silu(X W_gate) * (X W_up)) W_down per chunk; only X is retained. */
MST_API int mst_mlp_forward(mst_ctx* ctx, void* stream, const void* x, const void* w_gate, const void* w_up,
                    const void* w_down, void* out, int64_t n, int64_t h, int64_t i, int64_t m,
                    void* workspace, size_t workspace_bytes, mst_mlp_saved* saved);

/* miniseq_mlp_backward(dO, saved, w, plan) -> (dX, dW) — SPEC.md:304-312, Alg. 3.
 * Per chunk: recompute G,U,h; dX concatenated; dW accumulated in fp32 in
 * ascending chunk order.  accumulate=0 overwrites dW, 1 adds onto it. */
MST_API int mst_mlp_backward(mst_ctx* ctx, void* stream, const void* grad_out, const mst_mlp_saved* saved,
                     const void* w_gate, const void* w_up, const void* w_down, void* grad_x,
                     float* grad_w_gate, float* grad_w_up, float* grad_w_down, int accumulate,
                     void* workspace, size_t workspace_bytes);

/* miniseq_lmhead_forward(X, L, w, plan, mode) -> (loss, saved) — SPEC.md:313-321, Alg. 2.
 * Logits are never written to HBM: the GEMM epilogue keeps an online
 * softmax.  `stats` receives the loss (see MST_STATS_LEN); `lse` [n]. */
MST_API int mst_lmhead_forward(mst_ctx* ctx, void* stream, const void* x, const int32_t* labels, const void* w_out,
                       int64_t n, int64_t h, int64_t v, int64_t m, int loss_mode, float* stats, float* lse,
                       void* workspace, size_t workspace_bytes, mst_lmhead_saved* saved);

/* miniseq_lmhead_backward(saved, w, plan, mode) -> (dX, dW_out) — SPEC.md:322-330, Alg. 4.
 * `global_stats` may be the forward's stats or an all-reduced copy (sequence
 * sharding); token-weighted scaling uses global_stats[1] as the count.
 * grad_loss is the scalar upstream gradient. */
MST_API int mst_lmhead_backward(mst_ctx* ctx, void* stream, const mst_lmhead_saved* saved, const void* w_out,
                        const float* global_stats, float grad_loss, void* grad_x, float* grad_w_out,
                        int accumulate, void* workspace, size_t workspace_bytes);

/* Single-pass LM-Head forward + backward (forward and backward of SPEC.md
 * 313-330 in one chunk loop, for callers that run them back to back): one
 * logits GEMM per chunk whose epilogue keeps the online-softmax partials and
 * writes the unnormalised softmax numerators in-tile; an in-place pass turns
 * them into dlogits once the row LSE is known.  Logits are never stored and
 * the only [n/M, V] buffer is the dlogits chunk.  `global_valid` (device
 * fp64 integer count, nullable) overrides the local valid-token count for token-weighted
 * scaling under sequence sharding.  Writes stats (loss in [2]), lse, dX and
 * dW_out (accumulate as in mst_lmhead_backward). */
MST_API int mst_lmhead_fused(mst_ctx* ctx, void* stream, const void* x, const int32_t* labels, const void* w_out,
                             int64_t n, int64_t h, int64_t v, int64_t m, int loss_mode, float grad_loss,
                             const double* global_valid, float* stats, float* lse, void* grad_x, float* grad_w_out,
                             int accumulate, void* workspace, size_t workspace_bytes);

/* Number of labels in [0, V) among the n labels, written to *out (device
 * fp64, an exact integer below 2^53) — the local count a sequence shard all-reduces before
 * mst_lmhead_fused. */
MST_API int mst_count_valid(mst_ctx* ctx, void* stream, const int32_t* labels, int64_t n, int64_t v, double* out);

/* Non-finite scan ("all elements finite after any op in this
 * module (NaN/Inf is an error surfaced, not propagated)"): writes the number
 * of NaN/Inf elements of a device buffer (bf16 or fp32, any element offset) to
 * the device counter `count`, asynchronously on `stream`.  Callers that want
 * the SPEC's NonFiniteError read it after the op and a stream sync (the
 * Python mirror's `check_finite` / `block_step(check=True)` do exactly that). */
enum { MST_DTYPE_BF16 = 0, MST_DTYPE_F32 = 1 };
MST_API int mst_count_nonfinite(mst_ctx* ctx, void* stream, const void* data, int64_t n, int dtype,
                                unsigned int* count);

/* One fused MLP -> LM-Head block, forward + backward (the bench unit):
 * O = mlp(X); loss = CE(O W_out, L); then dW_out, dO, dX, dW_{gate,up,down}.
 * `stats` as in mst_lmhead_forward (device, MST_STATS_LEN(m_head) floats). */
MST_API int mst_block_step(mst_ctx* ctx, void* stream, const void* x, const int32_t* labels, const void* w_gate,
                   const void* w_up, const void* w_down, const void* w_out, int64_t n, int64_t h, int64_t i,
                   int64_t v, int64_t m_mlp, int64_t m_head, int loss_mode, float grad_loss, float* stats,
                   void* grad_x, float* grad_w_gate, float* grad_w_up, float* grad_w_down, float* grad_w_out,
                   int accumulate, void* workspace, size_t workspace_bytes);

/* Sequence-parallel variant: identical, except that the
 * token-weighted dlogits scale uses the device fp64 scalar *global_valid (the
 * valid-label count all-reduced over the ranks, mst_count_valid + SUM) so
 * the per-rank weight gradients sum to the single-device gradient.  `stats`
 * keeps the rank-local loss sum / count (entries 0..1, additive).  NULL
 * global_valid == mst_block_step.  Paper-mean mode ignores it. */
MST_API int mst_block_step_sp(mst_ctx* ctx, void* stream, const void* x, const int32_t* labels, const void* w_gate,
                   const void* w_up, const void* w_down, const void* w_out, int64_t n, int64_t h, int64_t i,
                   int64_t v, int64_t m_mlp, int64_t m_head, int loss_mode, float grad_loss, float* stats,
                   void* grad_x, float* grad_w_gate, float* grad_w_up, float* grad_w_down, float* grad_w_out,
                   int accumulate, void* workspace, size_t workspace_bytes, const double* global_valid);

/* ---------------------------------------------------------------- decoder layer
 * The plumbing around the MsT blocks in the reference's Llama-style decoder
 * (model module SPEC.md:410-469, blocks-std rmsnorm SPEC.md:242-250):
 *
 * mst_gemm             C[M,N] = A[M,K] B[K,N] (+ C) on the tcgen05 engine,
 *                      any operand majorness (semantics of mst_debug_gemm below)
 * mst_rmsnorm_forward  s = x + residual (bf16, written to sum_out; residual may
 *                      be NULL: s = x), y = s * gain / sqrt(mean(s^2) + eps),
 *                      rstd[n] fp32 saved for the backward.  bf16 x/y, fp32 gain.
 * mst_rmsnorm_backward dx = d(rmsnorm)/ds * dy (+ dres, the residual branch's
 *                      gradient), dgain (+)= sum over rows (fp32, fixed-order
 *                      block partials: deterministic); workspace from
 *                      mst_rmsnorm_workspace.
 * mst_embedding_forward  out[t] = table[tokens[t]]; tokens outside [0, vocab)
 *                      are counted into the device int *bad_count (the caller
 *                      raises DataError, "token out of range").
 * mst_embedding_backward dtable[v] (+)= sum of dx rows of the positions holding
 *                      token v, positions grouped by token (order = positions
 *                      stably sorted by token, seg = nseg+1 group starts, uniq =
 *                      the token of each group): fixed summation order. */
MST_API int mst_gemm(mst_ctx* ctx, void* stream, const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k,
                     int a_mn, int b_mn, int out_f32, int beta);
MST_API int mst_rmsnorm_forward(mst_ctx* ctx, void* stream, const void* x, const void* residual, const float* gain,
                                void* y, void* sum_out, float* rstd, int64_t n, int64_t d, float eps);
MST_API int mst_rmsnorm_workspace(const mst_ctx* ctx, int64_t n, int64_t d, size_t* bytes);
MST_API int mst_rmsnorm_backward(mst_ctx* ctx, void* stream, const void* s, const float* gain, const float* rstd,
                                 const void* dy, const void* dres, void* dx, float* dgain, int accumulate, int64_t n,
                                 int64_t d, void* workspace, size_t workspace_bytes);
MST_API int mst_embedding_forward(mst_ctx* ctx, void* stream, const void* table, const int32_t* tokens, void* out,
                                  int64_t n, int64_t d, int64_t vocab, int* bad_count);
MST_API int mst_embedding_backward(mst_ctx* ctx, void* stream, const int32_t* order, const int32_t* seg,
                                   const int32_t* uniq, int64_t nseg, const void* dx, float* dtable, int64_t d,
                                   int64_t vocab, int accumulate);

/* Causal grouped-query attention (attn_forward / attn_backward, SPEC.md:233-241;
 * the decoder's attention around the MsT blocks) on tcgen05 kernels: exact
 * softmax attention tile by tile, the [S, S] scores never reach HBM.
 * Token-major bf16 tensors: q element (b, t, head h, e) at
 * q[(b*seq + t)*ldq + h*head_dim + e]; k, v with kv_heads heads (query head h
 * reads kv head h / (heads / kv_heads)); o, dq, dk, dv the same way (the
 * decoder passes column slices of its fused [N, d + 2d/G] qkv buffer).
 * head_dim a multiple of 8 up to 128; scale 1/sqrt(head_dim); causal = 1.
 * lse: device fp32 [batch, heads, seq] log-sum-exp of the scaled scores
 * (natural log), written by the forward, read by the backward.  The
 * backward's workspace (mst_attention_workspace) holds rowsum(dO * O).
 * Deterministic: no atomics; dq, dk, dv are overwritten. */
MST_API int mst_attention_forward(mst_ctx* ctx, void* stream, const void* q, int64_t ldq, const void* k, int64_t ldk,
                                  const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, int64_t batch,
                                  int64_t seq, int64_t heads, int64_t kv_heads, int64_t head_dim, int causal);
MST_API int mst_attention_workspace(int64_t batch, int64_t seq, int64_t heads, size_t* bytes);
MST_API int mst_attention_backward(mst_ctx* ctx, void* stream, const void* q, int64_t ldq, const void* k, int64_t ldk,
                                   const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout,
                                   int64_t lddo, const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk,
                                   void* dv, int64_t lddv, int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads,
                                   int64_t head_dim, int causal, void* workspace, size_t workspace_bytes);

/* Diagnostic single GEMM through the same engine: C[M,N] = A[M,K] B[K,N].
 * a_mn=0: A row-major [M,K]; a_mn=1: A given as row-major [K,M] (A^T).
 * b_mn=1: B row-major [K,N]; b_mn=0: B given as row-major [N,K] (B^T).
 * out_f32=0: C bf16; 1: C fp32 with C = beta*C + A B (beta in {0,1});
 * beta = 1 with the bf16 output is MST_ERR_CONFIG. */
MST_API int mst_debug_gemm(mst_ctx* ctx, void* stream, const void* a, const void* b, void* c, int64_t m, int64_t n,
                   int64_t k, int a_mn, int b_mn, int out_f32, int beta);

#ifdef __cplusplus
}
#endif

#endif /* MST_MST_H_ */
