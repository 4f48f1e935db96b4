// miniseq.hpp — C++ operator API of the reference's `miniseq` module
// implemented on the libmst C ABI (mst.h).
//
// This is the binding a maintainer of the reference (a C++20 project,
// proj/CMakeLists.txt) adds to route its mini-sequence ops to the B200
// kernels: same op names, same argument meaning, errors thrown as the
// reference's exception types (proj/include/minitrain/error.hpp:10-25).
// Tensors are device pointers (bf16 activations/weights, fp32 gradients,
// int32 labels) — the reference's host `Tensor` is replaced by a view.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mst/mst.h"

#if defined(__has_include)
#if __has_include("minitrain/memtrack.hpp") && !defined(MST_STANDALONE_ERRORS)
#include "minitrain/memtrack.hpp"
#define MST_HAVE_MINITRAIN_MEMTRACK 1
#endif
#if __has_include("minitrain/error.hpp") && !defined(MST_STANDALONE_ERRORS)
#include "minitrain/error.hpp"
#define MST_HAVE_MINITRAIN_ERRORS 1
#endif
#endif

namespace mst {

#ifdef MST_HAVE_MINITRAIN_ERRORS
using Error = minitrain::Error;
using ShapeError = minitrain::ShapeError;
using BoundsError = minitrain::BoundsError;
using DtypeError = minitrain::DtypeError;
using ConfigError = minitrain::ConfigError;
using DataError = minitrain::DataError;
using StateError = minitrain::StateError;
using NonFiniteError = minitrain::NonFiniteError;
#else
// Same hierarchy shape as the reference when its header is not on the path.
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define MST_ERR_TYPE(name) \
  struct name : Error {    \
    using Error::Error;    \
  }
MST_ERR_TYPE(ShapeError);
MST_ERR_TYPE(BoundsError);
MST_ERR_TYPE(DtypeError);
MST_ERR_TYPE(ConfigError);
MST_ERR_TYPE(DataError);
MST_ERR_TYPE(StateError);
MST_ERR_TYPE(NonFiniteError);
#undef MST_ERR_TYPE
#endif

// Status code -> the reference's exception type.  No exception crosses the C ABI.
inline void throw_on(int status) {
  if (status == MST_OK) return;
  const std::string msg = mst_last_error();
  switch (status) {
    case MST_ERR_SHAPE: throw ShapeError(msg);
    case MST_ERR_BOUNDS: throw BoundsError(msg);
    case MST_ERR_DTYPE: throw DtypeError(msg);
    case MST_ERR_CONFIG: throw ConfigError(msg);
    case MST_ERR_DATA: throw DataError(msg);
    case MST_ERR_STATE: throw StateError(msg);
    case MST_ERR_NONFINITE: throw NonFiniteError(msg);
    default: throw Error("libmst: " + msg);
  }
}

enum class LossMode : int { TokenWeighted = MST_LOSS_TOKEN_WEIGHTED, PaperMean = MST_LOSS_PAPER_MEAN };

// SPEC.md:276-279
struct ChunkPlan {
  int64_t M = 0, N = 0;
  std::vector<std::pair<int64_t, int64_t>> ranges;
};

// SPEC.md:286-294
inline ChunkPlan make_chunk_plan(int64_t N, int64_t M) {
  std::vector<int64_t> b(static_cast<size_t>(std::max<int64_t>(1, std::min(N, M)) + 1));
  int64_t c = 0;
  throw_on(mst_make_chunk_plan(N, M, b.data(), &c));
  ChunkPlan p;
  p.M = M;
  p.N = N;
  for (int64_t i = 0; i < c; ++i) p.ranges.emplace_back(b[i], b[i + 1]);
  return p;
}

// Device views (row-major, SPEC orientation).
struct MlpWeights {
  const void* W_gate;  // [d, I] bf16
  const void* W_up;    // [d, I] bf16
  const void* W_down;  // [I, d] bf16
  int64_t d, I;
};
struct MlpGrads {
  float *W_gate, *W_up, *W_down;  // fp32, same shapes
};
struct LmHeadWeights {
  const void* W_out;  // [d, V] bf16
  int64_t d, V;
};

// One context per host thread per device.  The caller provides
// the device workspace (bytes from the *_workspace_bytes helpers).
class Context {
 public:
  explicit Context(int device = 0) { throw_on(mst_ctx_create(device, &ctx_)); }
  ~Context() { mst_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mst_ctx* get() const { return ctx_; }

 private:
  mst_ctx* ctx_ = nullptr;
};

struct Workspace {
  void* data;
  size_t bytes;
};

inline size_t mlp_workspace_bytes(int64_t N, const MlpWeights& w, const ChunkPlan& plan) {
  size_t b = 0;
  throw_on(mst_mlp_workspace(N, w.d, w.I, plan.M, &b));
  return b;
}
inline size_t lmhead_workspace_bytes(int64_t N, const LmHeadWeights& w, const ChunkPlan& plan) {
  size_t b = 0;
  throw_on(mst_lmhead_workspace(N, w.d, w.V, plan.M, &b));
  return b;
}

// miniseq_mlp_forward(X, w, plan) -> (O, saved)
inline mst_mlp_saved miniseq_mlp_forward(Context& ctx, void* stream, const void* X, int64_t N, const MlpWeights& w,
                                         const ChunkPlan& plan, void* O, Workspace ws) {
  if (plan.N != N) throw ConfigError("plan covers a different N (SPEC.md:297)");
  mst_mlp_saved s{};
  throw_on(mst_mlp_forward(ctx.get(), stream, X, w.W_gate, w.W_up, w.W_down, O, N, w.d, w.I, plan.M, ws.data,
                           ws.bytes, &s));
  return s;
}

// miniseq_mlp_backward(dO, saved, w, plan) -> (dX, dw)
inline void miniseq_mlp_backward(Context& ctx, void* stream, const void* dO, const mst_mlp_saved& saved,
                                 const MlpWeights& w, const ChunkPlan& plan, void* dX, MlpGrads g, bool accumulate,
                                 Workspace ws) {
  if (plan.M != saved.m || plan.N != saved.n) throw StateError("saved state from a different plan (SPEC.md:308)");
  throw_on(mst_mlp_backward(ctx.get(), stream, dO, &saved, w.W_gate, w.W_up, w.W_down, dX, g.W_gate, g.W_up,
                            g.W_down, accumulate ? 1 : 0, ws.data, ws.bytes));
}

// miniseq_lmhead_forward(X, L, w, plan, mode) -> (loss, saved)
// `stats` (device, MST_STATS_LEN(#chunks) floats) receives the loss in [2].
inline mst_lmhead_saved miniseq_lmhead_forward(Context& ctx, void* stream, const void* X, const int32_t* L,
                                               int64_t N, const LmHeadWeights& w, const ChunkPlan& plan,
                                               LossMode mode, float* stats, float* lse, Workspace ws) {
  if (plan.N != N) throw ConfigError("plan covers a different N (SPEC.md:316)");
  mst_lmhead_saved s{};
  throw_on(mst_lmhead_forward(ctx.get(), stream, X, L, w.W_out, N, w.d, w.V, plan.M, static_cast<int>(mode), stats,
                              lse, ws.data, ws.bytes, &s));
  return s;
}

// miniseq_lmhead_backward(saved, w, plan, mode) -> (dX, dW_out)
inline void miniseq_lmhead_backward(Context& ctx, void* stream, const mst_lmhead_saved& saved,
                                    const LmHeadWeights& w, const ChunkPlan& plan, LossMode mode, float grad_loss,
                                    void* dX, float* dW_out, bool accumulate, Workspace ws,
                                    const float* global_stats = nullptr) {
  if (plan.M != saved.m || plan.N != saved.n) throw StateError("saved state from a different plan (SPEC.md:326)");
  if (static_cast<int>(mode) != saved.loss_mode) throw StateError("loss mode differs from the forward's");
  throw_on(mst_lmhead_backward(ctx.get(), stream, &saved, w.W_out, global_stats, grad_loss, dX, dW_out,
                               accumulate ? 1 : 0, ws.data, ws.bytes));
}

// The MLP -> LM-Head block, forward + backward in one call (the unit the
// paper times; cmd_sweep_m / cmd_max_seq SPEC.md:728-754).
// Device tensors; `stats` receives the loss in [2].  M_mlp == M_head runs
// the chunk-wise schedule (one O chunk, two dO chunks on the device).
struct BlockGrads {
  void* dX;  // [N, d] bf16
  float *W_gate, *W_up, *W_down, *W_out;
};
inline size_t block_workspace_bytes(const Context& ctx, int64_t N, const MlpWeights& m, const LmHeadWeights& h,
                                    int64_t M_mlp, int64_t M_head) {
  size_t b = 0;
  throw_on(mst_ctx_block_workspace(ctx.get(), N, m.d, m.I, h.V, M_mlp, M_head, &b));
  return b;
}
inline void block_step(Context& ctx, void* stream, const void* X, const int32_t* L, int64_t N, const MlpWeights& m,
                       const LmHeadWeights& h, int64_t M_mlp, int64_t M_head, LossMode mode, float grad_loss,
                       float* stats, BlockGrads g, bool accumulate, Workspace ws) {
  throw_on(mst_block_step(ctx.get(), stream, X, L, m.W_gate, m.W_up, m.W_down, h.W_out, N, m.d, m.I, h.V, M_mlp,
                          M_head, static_cast<int>(mode), grad_loss, stats, g.dX, g.W_gate, g.W_up, g.W_down, g.W_out,
                          accumulate ? 1 : 0, ws.data, ws.bytes));
}
// Same with X, L and dX in (pinned) host memory, streamed per chunk under the
// GEMMs (mst_block_step_host): the sequence lives in host memory.
inline size_t block_host_workspace_bytes(const Context& ctx, int64_t N, const MlpWeights& m, const LmHeadWeights& h,
                                         int64_t M) {
  size_t b = 0;
  throw_on(mst_ctx_block_host_workspace(ctx.get(), N, m.d, m.I, h.V, M, &b));
  return b;
}
inline void block_step_host(Context& ctx, void* stream, const void* X_host, const int32_t* L_host, int64_t N,
                            const MlpWeights& m, const LmHeadWeights& h, int64_t M, LossMode mode, float grad_loss,
                            float* stats, BlockGrads g_dX_host, bool accumulate, Workspace ws) {
  throw_on(mst_block_step_host(ctx.get(), stream, X_host, L_host, m.W_gate, m.W_up, m.W_down, h.W_out, N, m.d, m.I,
                               h.V, M, static_cast<int>(mode), grad_loss, stats, g_dX_host.dX, g_dX_host.W_gate,
                               g_dX_host.W_up, g_dX_host.W_down, g_dX_host.W_out, accumulate ? 1 : 0, ws.data,
                               ws.bytes));
}

// Deferred device-side errors (mst.h "Deferred errors"): synchronise `stream`
// and throw DataError / NonFiniteError if an earlier call on the context hit
// an all-ignored batch, invalid labels or a non-finite loss.
inline void check(Context& ctx, void* stream) { throw_on(mst_ctx_check(ctx.get(), stream)); }

// Causal grouped-query attention (attn_forward / attn_backward)
// on the tcgen05 kernels: token-major bf16 tensors with row strides (ld) in
// elements; lse fp32 [batch, heads, seq].
struct AttnShape {
  int64_t batch, seq, heads, kv_heads, head_dim;
};
inline void attention_forward(Context& ctx, void* stream, const AttnShape& s, const void* q, int64_t ldq,
                              const void* k, int64_t ldk, const void* v, int64_t ldv, void* o, int64_t ldo,
                              float* lse) {
  throw_on(mst_attention_forward(ctx.get(), stream, q, ldq, k, ldk, v, ldv, o, ldo, lse, s.batch, s.seq, s.heads,
                                 s.kv_heads, s.head_dim, 1));
}
inline size_t attention_workspace_bytes(const AttnShape& s) {
  size_t b = 0;
  throw_on(mst_attention_workspace(s.batch, s.seq, s.heads, &b));
  return b;
}
inline void attention_backward(Context& ctx, void* stream, const AttnShape& s, const void* q, int64_t ldq,
                               const void* k, int64_t ldk, const void* v, int64_t ldv, const void* o, int64_t ldo,
                               const void* dout, int64_t lddo, const float* lse, void* dq, int64_t lddq, void* dk,
                               int64_t lddk, void* dv, int64_t lddv, Workspace ws) {
  throw_on(mst_attention_backward(ctx.get(), stream, q, ldq, k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk,
                                  lddk, dv, lddv, s.batch, s.seq, s.heads, s.kv_heads, s.head_dim, 1, ws.data,
                                  ws.bytes));
}

// Op counters of the context (memtrack.hpp:19-35 conventions; mst.h "memtrack").
inline mst_counters counters(const Context& ctx) {
  mst_counters c{};
  throw_on(mst_ctx_get_counters(ctx.get(), &c));
  return c;
}

#ifdef MST_HAVE_MINITRAIN_MEMTRACK
namespace detail {
inline void mem_to_minitrain(void*, int kind, uint64_t bytes, const char* label) {
  minitrain::MemTracker& t = minitrain::MemTracker::current();
  if (kind == 0)
    t.on_alloc(bytes, label);
  else
    t.on_free(bytes, label);
}
inline void count_to_minitrain(void*, int kind, int64_t a, int64_t b, int64_t c, uint64_t w) {
  minitrain::MemTracker& t = minitrain::MemTracker::current();
  if (kind == 0)
    t.count_matmul(a, b, c, w);
  else
    t.count_op(static_cast<uint64_t>(a), static_cast<uint64_t>(b));
}
}  // namespace detail

// Route the library's chunk-buffer events and op counts into the calling
// thread's current minitrain::MemTracker (memtrack.hpp:143-151), so
// TrackedRegion / export_timeline work unchanged on the GPU path.
inline void attach_current_tracker(Context& ctx) {
  throw_on(mst_ctx_set_mem_hook(ctx.get(), &detail::mem_to_minitrain, nullptr));
  throw_on(mst_ctx_set_count_hook(ctx.get(), &detail::count_to_minitrain, nullptr));
}
inline void detach_tracker(Context& ctx) {
  throw_on(mst_ctx_set_mem_hook(ctx.get(), nullptr, nullptr));
  throw_on(mst_ctx_set_count_hook(ctx.get(), nullptr, nullptr));
}
#endif

// mask_labels_for_chunk(L, range) — SPEC.md:331-339: a pointer offset.
inline const int32_t* mask_labels_for_chunk(const int32_t* L, int64_t N, std::pair<int64_t, int64_t> r) {
  if (r.first < 0 || r.first > r.second || r.second > N) throw BoundsError("chunk range outside [0, N)");
  return L + r.first;
}

}  // namespace mst
