// C-ABI implementation of the MsT hot path (include/mst/mst.h).
//
// Host responsibilities: argument validation with the reference's error
// taxonomy, TMA tensor-map encoding, the mini-sequence chunk loop
// (SPEC.md:271-361), grouping independent GEMMs of a chunk into one
// persistent launch, and an LPT (longest-processing-time-first) tile
// schedule per launch so CTA pairs finish together.  All arithmetic runs in
// the sm_100a kernels of gemm.cuh and the small kernels below.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "mst/mst.h"
#include "attention.cuh"
#include "layers.cuh"
#include "optim.cuh"

using mst::GemmParams;
using mst::PhaseDesc;
using mst::ProblemDesc;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define MST_CUDA(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(MST_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define MST_TRY(expr)              \
  do {                             \
    int s_ = (expr);               \
    if (s_ != MST_OK) return s_;   \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

uint64_t fnv1a(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t k = 0; k < n; ++k) {
    h ^= p[k];
    h *= 0x100000001b3ull;
  }
  return h;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Sequential bump allocator over the caller's workspace.
struct Carve {
  char* base;
  size_t cap;
  size_t used = 0;
  bool dry;  // size query only
  void* take(size_t bytes) {
    used = align_up(used, 256);
    void* p = dry ? nullptr : base + used;
    used += bytes;
    return p;
  }
};

}  // namespace

struct SchedEntry {
  int32_t* dev = nullptr;  // [off (pairs+1) | per-pair tiles | global LPT order]
  int32_t num_pairs = 0;
  int32_t total = 0;
};

struct mst_ctx {
  int device = 0;
  int num_sms = 0;
  int num_pairs = 0;
  int max_pairs = 0;
  EncodeTiledFn encode = nullptr;
  std::map<std::string, SchedEntry> sched_cache;
  int64_t launches = 0;
  float* scratch_dev = nullptr;  // small persistent device scratch
  // per-launch event timing (mst_ctx_set_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pairs: start, end
  std::vector<double> ev_flops;
  size_t ev_used = 0;
  unsigned long long* prof = nullptr;
  int64_t prof_slot = 0;
  int dynamic = 1;     // MST_DYNAMIC: pairs pull tiles from the global LPT order (atomic counter)
  int fused_head = 1;  // block_step: single-pass LM-Head forward+backward (mst_lmhead_fused)
  int chunked_block = 1;  // block_step with M_mlp == M_head: chunk-wise MLP -> head -> MLP-backward schedule
  int wide = 1;           // allow wide tiles (two N blocks per scheduled tile) where a builder asks for them
  // Which GEMMs of the chunk-wise block use wide tiles (bit mask, tuning key
  // "wide_mask"): 1 K3', 2 K5, 4 K2, 8 K9, 16 K7a, 32 K1.
  int wide_mask = 0;
  mst_attn::AttnTuning attn;  // attention kernel knobs ("attn_*" tuning keys)
  // Chunk-wise block: K8 / K10 of chunks (2k, 2k+1) as one K = 2n accumulation
  // (one fp32 dW read-modify-write per two chunks; a second dG / dU / h^T /
  // X^T chunk set stays live through the next chunk's head), and K9(j) in
  // K1(j+1)'s launch instead of K2(j+1)'s (tuning "pair_dw", "k9_in_k1").
  // Row-scaled LM-Head (tuning "dl_rowscale"): numerators relative to one
  // reference per row, the softmax normalisation applied as a per-row factor
  // by K5's epilogue and K6's transposed operand, no normalize pass.
  int dl_rowscale = 1;
  int pair_dw = 1;   // measured +1.6..1.9% at M = 4 / 8 / 16 (config 2)
  int k9_in_k1 = 0;  // measured -0.5%: off
  int fuse_swiglu_bwd = 0;  // 1: chunk-wise block runs the SwiGLU backward in the dh GEMM epilogue (measured -0.7%: off)
  int debug_nblk = 1;     // N blocks per tile of mst_debug_gemm
  // mst_block_step_host: copy stream and chunk events (created on first use)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t io_ev[10] = {};
  // Device chunk buffers of mst_block_step_host (2 X, 2 dX, labels): owned by
  // the context, so only this entry point's own chunk events order them and
  // a step's first X copy can run under the previous step's tail.
  void* io_dev = nullptr;
  size_t io_bytes = 0;
  // memtrack side (mst.h): counters per memtrack.hpp:19-35, event hooks
  mst_counters ctr{};
  mst_mem_hook mem_fn = nullptr;
  void* mem_user = nullptr;
  mst_count_hook cnt_fn = nullptr;
  void* cnt_user = nullptr;
  const void* weights[4] = {nullptr, nullptr, nullptr, nullptr};  // weight tensors of the current call
  mst_grad_ready_hook ready_fn = nullptr;  // optimizer-in-backward hook (mst.h)
  void* ready_user = nullptr;
  mst_grad_slab_hook slab_fn = nullptr;    // sequence-parallel gradient slabs (mst.h)
  void* slab_user = nullptr;
  int slabs = 1;
  int tma3d = 1;  // MN-major operands as 3-D tensor maps (tuning "tma3d")
  // Deferred (sticky) data errors raised by the device (mst.h): host-mapped word
  unsigned int* err_host = nullptr;
  unsigned int* err_dev = nullptr;
  // Cross-stream ordering of the context's device scratch (tile counter,
  // global-valid / count scratch): calls are serialised by `mu`, and a call
  // on a different stream than the previous one waits for `tail_ev`, which
  // every call records on its stream when it returns (mst.h "Threading").
  std::recursive_mutex mu;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  cudaEvent_t tail_ev = nullptr;
};

namespace {

// Deferred data errors (mst.h): a kernel of an earlier call flagged the
// context's host-mapped error word; the next call reports and clears it.
int take_sticky(mst_ctx* c) {
  if (!c->err_host) return MST_OK;
  const unsigned int f = __atomic_exchange_n(c->err_host, 0u, __ATOMIC_ACQ_REL);
  if (f & 1u) return fail(MST_ERR_DATA, "deferred error from an earlier call: all labels ignored, loss undefined (SPEC.md:219)");
  if (f & 2u) return fail(MST_ERR_DATA, "deferred error from an earlier call: labels outside [0, V) and != -100");
  if (f & 4u) return fail(MST_ERR_NONFINITE, "deferred error from an earlier call: non-finite loss (SPEC.md:26)");
  return MST_OK;
}

// One public call on a context: holds the context lock for the call and
// orders the call after the previous call's work when the stream changes
// (the scratch is per context, the stream per call).
struct CtxCall {
  mst_ctx* c;
  cudaStream_t st;
  std::lock_guard<std::recursive_mutex> lk;
  int status = MST_OK;
  CtxCall(mst_ctx* ctx, void* stream) : c(ctx), st(static_cast<cudaStream_t>(stream)), lk(ctx->mu) {
    if (c->has_last && c->last_stream != st && c->tail_ev) {
      if (cudaStreamWaitEvent(st, c->tail_ev, 0) != cudaSuccess)
        status = fail(MST_ERR_CUDA, "cross-stream ordering: cudaStreamWaitEvent failed");
    }
    if (status == MST_OK) status = take_sticky(c);
  }
  ~CtxCall() {
    if (!c->tail_ev) cudaEventCreateWithFlags(&c->tail_ev, cudaEventDisableTiming);
    if (c->tail_ev) cudaEventRecord(c->tail_ev, st);
    c->last_stream = st;
    c->has_last = true;
  }
};
#define MST_CALL(ctx, stream)                                                              \
  if (!(ctx)) return fail(MST_ERR_STATE, "NULL context");                                 \
  CtxCall call_guard_(ctx, stream);                                                        \
  if (call_guard_.status != MST_OK) return call_guard_.status

// ------------------------------------------------------------ memtrack side
// count_matmul / count_op of memtrack.hpp:163-175 (conventions at :19-35).
void cnt_mm(mst_ctx* c, int64_t n, int64_t k, int64_t p, uint64_t weight_elems) {
  const uint64_t f = 2ull * (uint64_t)n * (uint64_t)k * (uint64_t)p;
  c->ctr.flops += f;
  c->ctr.matmul_flops += f;
  c->ctr.hbm_elements += (uint64_t)n * k + (uint64_t)k * p + (uint64_t)n * p;
  c->ctr.weight_read_elements += weight_elems;
  if (c->cnt_fn) c->cnt_fn(c->cnt_user, 0, n, k, p, weight_elems);
}
void cnt_op(mst_ctx* c, uint64_t flops, uint64_t hbm) {
  c->ctr.flops += flops;
  c->ctr.hbm_elements += hbm;
  if (c->cnt_fn) c->cnt_fn(c->cnt_user, 1, (int64_t)flops, (int64_t)hbm, 0, 0);
}
bool is_weight(const mst_ctx* c, const void* p) {
  for (const void* w : c->weights)
    if (w && w == p) return true;
  return false;
}
// MemTracker::on_alloc / on_free (memtrack.hpp:153-167) for a chunk buffer.
void mem_alloc(mst_ctx* c, uint64_t bytes, const char* label) {
  if (c->mem_fn) c->mem_fn(c->mem_user, 0, bytes, label);
}
void mem_free(mst_ctx* c, uint64_t bytes, const char* label) {
  if (c->mem_fn) c->mem_fn(c->mem_user, 1, bytes, label);
}
// Weight tensors of the current call (operands equal to one of them count
// as weight reads, memtrack.hpp:25-26).
struct WeightScope {
  mst_ctx* c;
  WeightScope(mst_ctx* ctx, const void* a, const void* b = nullptr, const void* d = nullptr, const void* e = nullptr)
      : c(ctx) {
    c->weights[0] = a;
    c->weights[1] = b;
    c->weights[2] = d;
    c->weights[3] = e;
  }
  ~WeightScope() { c->weights[0] = c->weights[1] = c->weights[2] = c->weights[3] = nullptr; }
};

// Weight-gradient lifetimes for the tracker: "grad.*" is allocated when a
// block step first writes the gradient; when an optimizer-in-backward hook
// consumes it (grad_ready below) the library also records its release,
// otherwise the caller frees it after its optimizer step.
const char* const kGradLabel[4] = {"grad.W_gate", "grad.W_up", "grad.W_down", "grad.W_out"};
void grad_alloc(mst_ctx* c, int which, uint64_t bytes) { mem_alloc(c, bytes, kGradLabel[which]); }

// Rows [r0, r1) of a weight gradient are final in stream order
// (mst_ctx_set_grad_slab_hook).
void grad_slab(mst_ctx* c, int which, int64_t r0, int64_t r1, cudaStream_t st) {
  if (c->slab_fn && r1 > r0) c->slab_fn(c->slab_user, which, r0, r1, st);
}

// A weight gradient is final in stream order (mst_ctx_set_grad_ready_hook).
void grad_ready(mst_ctx* c, int which, cudaStream_t st, uint64_t bytes) {
  if (!c->ready_fn) return;
  c->ready_fn(c->ready_user, which, st);
  mem_free(c, bytes, kGradLabel[which]);
}

// ------------------------------------------------------------ tensor maps
int tmap_2d(mst_ctx* c, CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_elems,
            uint32_t box_inner, uint32_t box_outer, bool f32 = false) {
  const uint64_t esz = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(MST_ERR_CONFIG, "tensor base %p is not 16-byte aligned", base);
  if ((ld_elems * esz) % 16 != 0)
    return fail(MST_ERR_CONFIG, "row stride %llu elems is not 16-byte aligned", (unsigned long long)ld_elems);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = c->encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                         const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(MST_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) dims=%llu x %llu box=%u x %u", (int)r,
                (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer);
  return MST_OK;
}

// MN-major operand as a 3-D map {64, K, MN/64} with strides {ld, 64 elements}:
// one box {64, 64, nblk} fetches a 64*nblk-wide slab in the [block][k][64]
// order the UMMA MN-major SW128 descriptor expects (LBO = 8 KB).
int tmap_3d_mn(mst_ctx* c, CUtensorMap* m, const void* base, uint64_t mn, uint64_t k, uint64_t ld_elems,
               uint32_t nblk) {
  cuuint64_t dims[3] = {64, k, mn / 64};
  cuuint64_t strides[2] = {ld_elems * 2, 128};
  cuuint32_t box[3] = {64, 64, nblk};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = c->encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(MST_ERR_CUDA, "cuTensorMapEncodeTiled(3d) failed (%d) mn=%llu k=%llu", (int)r,
                (unsigned long long)mn, (unsigned long long)k);
  return MST_OK;
}

// Operand of a GEMM, as stored in global memory (row-major, ld elements).
//   K-major : element (row, k) at base[row*ld + k]      -> map dims {K, rows}
//   MN-major: element (k, mn)  at base[k*ld + mn]       -> map dims {MN, K}
struct Operand {
  const void* base;
  int64_t mn;  // rows (M for A, N for B)
  int64_t k;
  int64_t ld;
  bool mn_major;
};

// Builder for one launch: collects tensor maps and problems.
struct Launch {
  GemmParams p;
  int nmaps = 0;
  int acc_cols = 0;
  double flops = 0;  // algorithmic 2*M*N*K over the valid extents
  Launch() { std::memset(&p, 0, sizeof(p)); }
};

bool use_3d(const mst_ctx* c, const Operand& o, int box_mn) {
  return o.mn_major && c->tma3d && o.mn % 64 == 0 && box_mn % 64 == 0 && (reinterpret_cast<uintptr_t>(o.base) & 127) == 0;
}

int add_map(mst_ctx* c, Launch& L, const Operand& o, int box_mn) {
  if (L.nmaps >= mst::kMaxMaps) return fail(MST_ERR_INTERNAL, "too many tensor maps in one launch");
  CUtensorMap* m = &L.p.maps[L.nmaps];
  int s = !o.mn_major      ? tmap_2d(c, m, o.base, o.k, o.mn, o.ld, 64, box_mn)
          : use_3d(c, o, box_mn) ? tmap_3d_mn(c, m, o.base, o.mn, o.k, o.ld, box_mn / 64)
                              : tmap_2d(c, m, o.base, o.mn, o.k, o.ld, 64, 64);
  if (s != MST_OK) return s;
  return -(L.nmaps++) - 100;  // encoded index (negative to distinguish from status)
}

int map_index(int encoded) { return -(encoded + 100); }

// Output tensor map for the epilogue's TMA stores: 32-row x 128-byte boxes
// (64 bf16 or 32 fp32 columns), SWIZZLE_128B.  Returns the map index via *idx.
int add_out_map(mst_ctx* c, Launch& L, void* base, int64_t cols, int64_t rows, int64_t ld, bool f32, int32_t* idx,
                bool team = true) {
  if (L.nmaps >= mst::kMaxMaps) return fail(MST_ERR_INTERNAL, "too many tensor maps in one launch");
  // fp32 weight-gradient tiles are staged by the 4 epilogue warps together:
  // one box per 128-row CTA slice; everything else: one 32-row box per warp.
  const uint32_t box_rows = (f32 && team) ? 128 : 32;
  MST_TRY(tmap_2d(c, &L.p.maps[L.nmaps], base, (uint64_t)cols, (uint64_t)rows, (uint64_t)ld, f32 ? 32 : 64, box_rows,
                  f32));
  *idx = L.nmaps++;
  return MST_OK;
}

struct PhaseSpec {
  Operand a;
  Operand b0, b1;  // B source for CTA rank 0 / 1
  int umma_n;
  int tmem_col;
  int b_off0, b_off1;
  bool acc_continue;
  int k_start = 0;   // first K block (split-K slice)
  int k_blocks = 0;  // 0: the whole K extent
};

int add_phase(mst_ctx* c, Launch& L, ProblemDesc& P, const PhaseSpec& s) {
  PhaseDesc& d = P.ph[P.num_phases++];
  int ea = add_map(c, L, s.a, 128);
  if (ea >= 0) return ea;
  const int nh = s.umma_n / 2;
  int eb0 = add_map(c, L, s.b0, nh);
  if (eb0 >= 0) return eb0;
  int eb1 = eb0;
  if (s.b1.base != s.b0.base || s.b1.mn != s.b0.mn) {
    eb1 = add_map(c, L, s.b1, nh);
    if (eb1 >= 0) return eb1;
  }
  d.map_a = map_index(ea);
  d.map_b0 = map_index(eb0);
  d.map_b1 = map_index(eb1);
  d.a_mn = s.a.mn_major ? 1 : 0;
  d.b_mn = s.b0.mn_major ? 1 : 0;
  d.a_3d = use_3d(c, s.a, 128) ? 1 : 0;
  d.b_3d = (use_3d(c, s.b0, nh) && use_3d(c, s.b1, nh)) ? 1 : 0;
  d.umma_n = s.umma_n;
  d.tmem_col = s.tmem_col;
  d.k_start = s.k_start;
  d.k_blocks = s.k_blocks ? s.k_blocks : static_cast<int32_t>(cdiv(s.a.k, mst::kBK) - s.k_start);
  d.b_off0 = s.b_off0;
  d.b_off1 = s.b_off1;
  d.acc_continue = s.acc_continue ? 1 : 0;
  // L2 policy: an operand small enough to stay resident while every tile of
  // the problem re-reads it (an activation chunk) is kept (evict_last); weights
  // and large streams use the normal policy so the CTA pairs that share a
  // B tile at the same time still hit in L2.
  auto pol = [](const Operand& o) { return (o.mn * o.k * 2 <= (int64_t(48) << 20)) ? 1 : 0; };
  d.a_pol = pol(s.a);
  d.b_pol = pol(s.b0);
  L.acc_cols = std::max(L.acc_cols, s.tmem_col + s.umma_n);
  return MST_OK;
}

// Estimated tile cost in SM cycles (for LPT scheduling only).
double tile_cost(const ProblemDesc& P) {
  double mma = 0;
  for (int i = 0; i < P.num_phases; ++i) mma += double(P.ph[i].k_blocks) * P.ph[i].umma_n * 2.0 * P.nblk;
  double bytes = 0;
  switch (P.epi) {
    case mst::kEpiStoreBf16: bytes = 256.0 * P.ph[0].umma_n * 2; break;
    case mst::kEpiAccF32: bytes = 256.0 * P.ph[0].umma_n * 4 * (P.beta ? 2 : 1); break;
    case mst::kEpiSwiglu: bytes = 256.0 * 128 * 2; break;
    case mst::kEpiSwigluBwd: bytes = 3 * 256.0 * 128 * 2 + 256.0 * 128 * 4; break;
    case mst::kEpiCeFwd: bytes = 256.0 * 16; break;
    case mst::kEpiCeBwd: bytes = 256.0 * 256 * 2; break;
    case mst::kEpiCeFwdNum: bytes = 256.0 * 256 * 2 + 256.0 * 12; break;
    case mst::kEpiSwigluSave: bytes = 256.0 * 128 * (2 + 4 + 4); break;
    case mst::kEpiDhSwigluBwd: bytes = 256.0 * 256 * (4 + 4 + 2 + 2); break;
  }
  const double epi = bytes * P.nblk / 46.0;
  return std::max(mma, epi) + 800.0;
}

int get_schedule(mst_ctx* c, const GemmParams& p, const int32_t** sched, const int32_t** off, const int32_t** order,
                 int32_t* total) {
  std::string key;
  for (int i = 0; i < p.num_problems; ++i) {
    const ProblemDesc& P = p.prob[i];
    char buf[160];
    snprintf(buf, sizeof(buf), "%d:%d/%d:%d:%d:%d:%d:%d|", P.m_tiles, P.n_tiles, P.nblk, P.epi, P.beta, P.num_phases,
             P.ph[0].k_blocks * 1000 + P.ph[0].umma_n, P.num_phases > 1 ? P.ph[1].k_blocks * 1000 + P.ph[1].umma_n : 0);
    key += buf;
  }
  auto it = c->sched_cache.find(key);
  if (it == c->sched_cache.end()) {
    struct T {
      double cost;
      int32_t code;
      int order;
    };
    std::vector<T> tiles;
    for (int i = 0; i < p.num_problems; ++i) {
      const ProblemDesc& P = p.prob[i];
      const double cst = tile_cost(P);
      const int nt = P.m_tiles * P.n_wide;
      for (int t = 0; t < nt; ++t) tiles.push_back({cst, (i << 24) | t, (int)tiles.size()});
    }
    std::stable_sort(tiles.begin(), tiles.end(), [](const T& a, const T& b) { return a.cost > b.cost; });
    const int np = c->num_pairs;
    using Q = std::pair<double, int>;
    std::priority_queue<Q, std::vector<Q>, std::greater<Q>> heap;
    for (int q = 0; q < np; ++q) heap.push({0.0, q});
    std::vector<std::vector<int32_t>> per(np);
    for (const T& t : tiles) {
      Q top = heap.top();
      heap.pop();
      per[top.second].push_back(t.code);
      heap.push({top.first + t.cost, top.second});
    }
    std::vector<int32_t> host(np + 1 + 2 * tiles.size());
    int32_t acc = 0;
    for (int q = 0; q < np; ++q) {
      host[q] = acc;
      acc += (int32_t)per[q].size();
    }
    host[np] = acc;
    size_t w = np + 1;
    for (int q = 0; q < np; ++q)
      for (int32_t code : per[q]) host[w++] = code;
    for (const T& t : tiles) host[w++] = t.code;  // global LPT order (dynamic mode)
    SchedEntry e;
    e.num_pairs = np;
    e.total = (int32_t)tiles.size();
    MST_CUDA(cudaMalloc(&e.dev, host.size() * sizeof(int32_t)));
    MST_CUDA(cudaMemcpy(e.dev, host.data(), host.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    it = c->sched_cache.emplace(key, e).first;
  }
  *off = it->second.dev;
  *sched = it->second.dev + c->num_pairs + 1;
  *order = *sched + it->second.total;
  *total = it->second.total;
  return MST_OK;
}

int launch(mst_ctx* c, cudaStream_t st, Launch& L) {
  GemmParams& p = L.p;
  if (L.acc_cols > mst::kTmemCols) return fail(MST_ERR_INTERNAL, "accumulator needs %d TMEM columns", L.acc_cols);
  int tiles = 0;
  if (L.acc_cols <= 256) {
    p.acc_stages = 2;
    p.acc_stride = 256;
  } else {
    p.acc_stages = 1;
    p.acc_stride = 0;
  }
  for (int i = 0; i < p.num_problems; ++i) {
    ProblemDesc& P = p.prob[i];
    if (P.nblk <= 0 || c->wide == 0) P.nblk = 1;
    if (P.nblk > mst::kMaxNBlk || P.nblk > p.acc_stages)
      return fail(MST_ERR_INTERNAL, "problem %d: %d N blocks per tile with %d accumulator stages", i, P.nblk,
                  p.acc_stages);
    P.n_wide = (int)cdiv(P.n_tiles, P.nblk);
    tiles += P.m_tiles * P.n_wide;
    p.stage_slots = std::max(p.stage_slots, 1 + P.nblk);
  }
  p.num_stages = mst::kSlots / p.stage_slots;
  if (tiles == 0) return MST_OK;
  MST_TRY(get_schedule(c, p, &p.sched, &p.sched_off, &p.order, &p.total_tiles));
  p.dynamic = c->dynamic;
  p.tile_counter = reinterpret_cast<int32_t*>(c->scratch_dev);
  // p.tile_counter[0..1] are zero here: zeroed at context creation, and every
  // dynamic launch re-zeroes them on exit (gemm.cuh TileFeed::produce).
  // profile slots: 8 counters per launch, 64 slots round robin
  p.prof = c->prof ? c->prof + 8 * (c->prof_slot++ % 64) : nullptr;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(2 * c->num_pairs);
  cfg.blockDim = dim3(mst::kThreads);
  cfg.dynamicSmemBytes = mst::kSmemBytes;
  cfg.stream = st;
  if (c->timing) {
    if (c->ev_used + 2 > c->ev.size()) {
      for (int k = 0; k < 64; ++k) {
        cudaEvent_t e;
        MST_CUDA(cudaEventCreate(&e));
        c->ev.push_back(e);
      }
    }
    MST_CUDA(cudaEventRecord(c->ev[c->ev_used], st));
  }
  MST_CUDA(cudaLaunchKernelEx(&cfg, mst::mst_grouped_gemm_kernel, p));
  if (c->timing) {
    MST_CUDA(cudaEventRecord(c->ev[c->ev_used + 1], st));
    c->ev_used += 2;
    c->ev_flops.push_back(L.flops);
  }
  c->launches++;
  return MST_OK;
}

// ------------------------------------------------------------ small kernels
// Combine the per-128-column softmax partials of one row into lse and the
// row loss (loss = lse - z_label for non-ignored rows).
__global__ void ce_combine_kernel(const float2* __restrict__ part, int nparts, const float* __restrict__ ztarget,
                                  const int32_t* __restrict__ labels, int rows, int vocab, float* __restrict__ lse,
                                  float* __restrict__ loss_row, float* __restrict__ bad) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float2* pr = part + static_cast<int64_t>(warp) * nparts;
  float m = -INFINITY;
  for (int j = lane; j < nparts; j += 32) m = fmaxf(m, pr[j].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
  float s = 0.f;
  for (int j = lane; j < nparts; j += 32) s += pr[j].y * exp2f(pr[j].x - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (lane == 0) {
    const float l2 = m + log2f(s);
    lse[warp] = l2 * 0.69314718055994531f;
    const int lab = labels[warp];
    const bool valid = lab >= 0 && lab < vocab;
    if (lab != -100 && !valid) atomicAdd(bad, 1.0f);
    loss_row[warp] = valid ? l2 * 0.69314718055994531f - ztarget[warp] : 0.0f;
  }
}

// Row-scaled LM-Head (block_step / mst_lmhead_fused default):
// the K3' epilogue stored each vocabulary tile's numerators relative to 2^0
// (or, outside the +-kCeRefWindow window, to the tile maximum recorded in
// part[].x).  Per row (one warp): the LSE and the row loss as in
// ce_combine_kernel, then
//   R* = 0, unless some tile used its own maximum and |lse2| is outside the
//        window (then R* = rint(lse2)); tiles stored relative to another
//        reference are rescaled to R* in place (never taken for logits
//        within +-44 nats);
//   the label column becomes e'_label = (p_label - 1) 2^(lse2 - R*) from the
//        fp32 target logit (confident rows keep the precision of 1 - p_label);
//   rowf[r] = scale 2^(R* - lse2) (0 for ignored rows),
// so that dlogits[r, :] = rowf[r] * e'[r, :]: K5 applies rowf in its epilogue,
// K6 reads (rowf * X)^T.  rowf overwrites ztarget (read first, same warp).
__global__ void ce_combine_rowscale_kernel(const float2* __restrict__ part, int nparts, float* ztarget_rowf,
                                           const int32_t* __restrict__ labels, int rows, int vocab,
                                           float* __restrict__ lse, float* __restrict__ loss_row,
                                           float* __restrict__ bad, uint16_t* __restrict__ e, int64_t ld,
                                           const float* __restrict__ scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float2* pr = part + static_cast<int64_t>(warp) * nparts;
  float m = -INFINITY;
  bool special = false;
  for (int j = lane; j < nparts; j += 32) {
    const float x = pr[j].x;
    m = fmaxf(m, x);
    special |= x != 0.0f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
  special = __any_sync(0xffffffff, special);
  float s = 0.f;
  for (int j = lane; j < nparts; j += 32) s += pr[j].y * exp2f(pr[j].x - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float l2 = m + log2f(s);
  const float rs = (!special || fabsf(l2) <= mst::kCeRefWindow) ? 0.0f : rintf(l2);
  uint16_t* er = e + static_cast<int64_t>(warp) * ld;
  if (special) {  // rare: rescale the tiles stored relative to another reference
    for (int j = 0; j < nparts; ++j) {
      const float ref = pr[j].x;
      if (ref == rs) continue;
      const float f = exp2f(ref - rs);
      const int c0 = j * 256, c1 = min(vocab, c0 + 256);
      for (int c = c0 + lane; c < c1; c += 32) {
        const float x = __bfloat162float(__ushort_as_bfloat16(er[c])) * f;
        er[c] = __bfloat16_as_ushort(__float2bfloat16_rn(x));
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    const float lse_r = l2 * 0.69314718055994531f;
    lse[warp] = lse_r;
    const int lab = labels[warp];
    const bool valid = lab >= 0 && lab < vocab;
    if (lab != -100 && !valid) atomicAdd(bad, 1.0f);
    const float zt = ztarget_rowf[warp];
    loss_row[warp] = valid ? lse_r - zt : 0.0f;
    float f = 0.0f;
    if (valid) {
      const float p = exp2f((zt - lse_r) * 1.4426950408889634f);
      er[lab] = __bfloat16_as_ushort(__float2bfloat16_rn((p - 1.0f) * exp2f(l2 - rs)));
      f = *scale * exp2f(rs - l2);
    }
    ztarget_rowf[warp] = f;
  }
}

// Per-chunk (loss_sum, valid) with a fixed-order block reduction
// (deterministic; SPEC.md:90 bitwise reruns).
__global__ void chunk_reduce_kernel(const float* __restrict__ loss_row, const int32_t* __restrict__ labels, int rows,
                                    int vocab, float* __restrict__ out_sum, float* __restrict__ out_valid) {
  __shared__ float ss[32], sv[32];
  float s = 0.f, v = 0.f;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    s += loss_row[r];
    const int lab = labels[r];
    v += (lab >= 0 && lab < vocab) ? 1.f : 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffff, s, o);
    v += __shfl_xor_sync(0xffffffff, v, o);
  }
  if ((threadIdx.x & 31) == 0) {
    ss[threadIdx.x >> 5] = s;
    sv[threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += ss[w];
      b += sv[w];
    }
    *out_sum = a;
    *out_valid = b;
  }
}

// stats[0..3] from the per-chunk entries (SPEC.md:316-317 loss modes).  The
// SPEC's data errors are also raised into the context's sticky error word
// (host-mapped; mst.h "Deferred errors"): 1 = every label ignored
// (SPEC.md:219), 2 = labels outside [0, V) other than -100, 4 = non-finite loss.
__global__ void finalize_loss_kernel(float* stats, int m, int mode, unsigned int* err, const double* gvalid) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0, v = 0, pm = 0;
  int nonempty = 0;
  for (int c = 0; c < m; ++c) {
    const double cs = stats[4 + c], cv = stats[4 + m + c];
    s += cs;
    v += cv;
    if (cv > 0) {
      pm += cs / cv;
      ++nonempty;
    }
  }
  stats[0] = (float)s;
  stats[1] = (float)v;
  stats[2] = mode == MST_LOSS_PAPER_MEAN ? (float)(pm / m) : (float)(s / v);
  if (err) {
    // a sequence shard with no valid label is fine when the global count is not 0
    const double vall = gvalid ? *gvalid : v;
    const unsigned int f =
        (vall == 0 ? 1u : 0u) | (stats[3] > 0.f ? 2u : 0u) | ((v > 0 && !isfinite(stats[2])) ? 4u : 0u);
    if (f) {
      atomicOr_system(err, f);
      __threadfence_system();
    }
  }
}

// Per-chunk dlogits scale: grad_loss / valid_global (token-weighted) or
// grad_loss / (M * valid_chunk) (paper-mean).
// The global count is exact: a device fp64 integer (`gvalid`: the caller's
// all-reduced count, or this call's total from
// sum_valid_kernel / valid_total_kernel), else the SPEC-op stats pair
// `gstats[1]` of mst_lmhead_backward.
__global__ void grad_scale_kernel(const double* gvalid, const float* gstats, const float* local_stats, int m,
                                  int mode, float grad_loss, float* scales) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  float sc;
  if (mode == MST_LOSS_PAPER_MEAN) {
    const float cv = local_stats[4 + m + c];
    sc = cv > 0 ? grad_loss / (float(m) * cv) : 0.f;
  } else {
    const double gv = gvalid ? *gvalid : static_cast<double>(gstats[1]);
    sc = gv > 0 ? (float)((double)grad_loss / gv) : 0.f;
  }
  scales[c] = sc;
}

// Total of the per-chunk valid counts (exact fp32 integers, < 2^24 rows per
// chunk) summed in fp64: one thread, O(M).
__global__ void valid_total_kernel(const float* __restrict__ stats, int m, double* __restrict__ tot) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t = 0;
  for (int c = 0; c < m; ++c) t += stats[4 + m + c];
  *tot = t;
}

// dst[c, r] = src[r, c] for a rows x cols bf16 block (row strides ld_src /
// ld_dst elements).  Feeds the dW GEMMs a K-major A operand (X^T, O^T, h^T):
// MN-major A costs ~25% tensor throughput on sm_100a, a transpose of the
// chunk costs ~0.1% of the step.  64x64 tiles, 16-byte global accesses.
// Optional rowscale: source row r is multiplied by rowscale[r] (fp32, then
// rounded to bf16) on the way: the row-scaled head's K6 operand (rowf * X)^T.
__device__ __forceinline__ uint32_t scale_bf16x2(uint32_t w, float f) {
  const float lo = __uint_as_float(w << 16) * f, hi = __uint_as_float(w & 0xffff0000u) * f;
  return mst::ptx::pack_bf16(lo, hi);
}
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const uint16_t* __restrict__ src, int64_t ld_src,
                                                              uint16_t* __restrict__ dst, int64_t ld_dst, int rows,
                                                              int cols, const float* __restrict__ rowscale) {
  __shared__ uint16_t tile[64][72];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int r = i >> 3, cc = (i & 7) * 8;
    const int gr = r0 + r, gc = c0 + cc;
    if (gr < rows) {
      const uint16_t* p = src + static_cast<int64_t>(gr) * ld_src + gc;
      const float f = rowscale ? rowscale[gr] : 1.0f;
      if (gc + 8 <= cols) {
        uint4 v = *reinterpret_cast<const uint4*>(p);
        if (rowscale) v = make_uint4(scale_bf16x2(v.x, f), scale_bf16x2(v.y, f), scale_bf16x2(v.z, f), scale_bf16x2(v.w, f));
        const uint16_t* e = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int k = 0; k < 8; ++k) tile[r][cc + k] = e[k];
      } else {
        for (int k = 0; k < 8; ++k) {
          uint16_t x = gc + k < cols ? p[k] : 0;
          if (rowscale) x = __bfloat16_as_ushort(__float2bfloat16_rn(__bfloat162float(__ushort_as_bfloat16(x)) * f));
          tile[r][cc + k] = x;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int c = i >> 3, rr = (i & 7) * 8;
    const int gc = c0 + c, gr = r0 + rr;
    if (gc >= cols || gr >= rows) continue;
    uint16_t* p = dst + static_cast<int64_t>(gc) * ld_dst + gr;
    if (gr + 8 <= rows) {
      uint4 v;
      uint16_t* e = reinterpret_cast<uint16_t*>(&v);
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = tile[rr + k][c];
      *reinterpret_cast<uint4*>(p) = v;
    } else {
      for (int k = 0; k < 8 && gr + k < rows; ++k) p[k] = tile[rr + k][c];
    }
  }
}

// Register-only transpose: each thread moves one 8 x 8 block (8 coalesced
// 16-byte row loads, 32 byte permutes, 8 16-byte stores); a warp covers 32
// rows x 64 columns, a 256-thread block 256 rows x 64 columns.  cols % 8 == 0;
// ragged rows are zero-filled into the destination's padding (ld_dst >= rows
// rounded up to 8), which the consumers' tensor maps never read.
__global__ void __launch_bounds__(256) transpose8_bf16_kernel(const uint16_t* __restrict__ src, int64_t ld_src,
                                                               uint16_t* __restrict__ dst, int64_t ld_dst, int rows,
                                                               int cols, const float* __restrict__ rowscale) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = blockIdx.y * 256 + warp * 32 + (lane >> 3) * 8;  // this thread's 8 source rows
  const int c0 = blockIdx.x * 64 + (lane & 7) * 8;                 // and 8 source columns
  if (r0 >= rows || c0 >= cols) return;
  uint32_t in[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + k < rows) {
      v = __ldcs(reinterpret_cast<const uint4*>(src + static_cast<int64_t>(r0 + k) * ld_src + c0));
      if (rowscale) {
        const float f = rowscale[r0 + k];
        v = make_uint4(scale_bf16x2(v.x, f), scale_bf16x2(v.y, f), scale_bf16x2(v.z, f), scale_bf16x2(v.w, f));
      }
    }
    in[k][0] = v.x, in[k][1] = v.y, in[k][2] = v.z, in[k][3] = v.w;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // output row c0 + j holds source column c0 + j of rows r0..r0+7
    uint32_t o[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) o[w] = __byte_perm(in[2 * w][j >> 1], in[2 * w + 1][j >> 1], (j & 1) ? 0x7632 : 0x5410);
    *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(c0 + j) * ld_dst + r0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

int transpose_bf16(mst_ctx* c, cudaStream_t st, const void* src, int64_t ld_src, void* dst, int64_t ld_dst,
                   int64_t rows, int64_t cols, const float* rowscale = nullptr) {
  if (cols % 8 == 0 && ld_dst % 8 == 0 && ld_dst >= (rows + 7) / 8 * 8 && ld_src % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    dim3 grid((unsigned)cdiv(cols, 64), (unsigned)cdiv(rows, 256));
    transpose8_bf16_kernel<<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(src), ld_src,
                                                  static_cast<uint16_t*>(dst), ld_dst, (int)rows, (int)cols, rowscale);
    c->launches++;
    MST_CUDA(cudaGetLastError());
    return MST_OK;
  }
  dim3 grid((unsigned)cdiv(cols, 64), (unsigned)cdiv(rows, 64));
  transpose_bf16_kernel<<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(src), ld_src, static_cast<uint16_t*>(dst),
                                               ld_dst, (int)rows, (int)cols, rowscale);
  c->launches++;
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

// Per-chunk valid-label counts straight from the labels (balanced chunk
// plan recomputed in-kernel), so the single-pass head knows every dlogits
// scale before its first chunk: stats[4+M+c] and stats[1] (total).
__global__ void chunk_valid_kernel(const int32_t* __restrict__ labels, int64_t n, int m, int vocab, float* stats) {
  __shared__ int sv[32];
  const int c = blockIdx.x;
  const int64_t q = n / m, r = n % m;
  const int64_t s0 = c * q + (c < r ? c : r), s1 = s0 + q + (c < r ? 1 : 0);
  int v = 0;  // integer count: exact; stored as an fp32 integer (< 2^24 rows per chunk)
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    const int lab = labels[i];
    v += (lab >= 0 && lab < vocab) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sv[w];
    stats[4 + m + c] = (float)t;
  }
}

// Exact valid-label count of a whole label vector as an fp64 integer
// (mst_count_valid: the per-rank term of the sequence-parallel all-reduce).
__global__ void count_valid_kernel(const int32_t* __restrict__ labels, int64_t n, int vocab, double* out) {
  __shared__ long long sv[32];
  long long v = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int lab = labels[i];
    v += (lab >= 0 && lab < vocab) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sv[w];
    *out = (double)t;
  }
}

// stats[1] (the reported count) and the exact fp64 total in *tot.
__global__ void sum_valid_kernel(float* stats, int m, double* tot) {
  if (threadIdx.x != 0) return;
  double t = 0;
  for (int c = 0; c < m; ++c) t += stats[4 + m + c];
  stats[1] = (float)t;
  *tot = t;
}

// In place: e (bf16 softmax numerator, tile max m_tile in part[].x) ->
// dlogits = (e * 2^(m_tile - lse*log2e) - [v == label]) * scale, bf16.
// The label column is recomputed from the fp32 target logit instead:
// (exp(z_label - lse) - 1) * scale, so a confident row (p_label -> 1) keeps
// the relative precision of 1 - p_label (e's bf16 rounding would leave an
// absolute error of ~2^-9 on a value that can be far smaller).
__global__ void normalize_dlogits_kernel(uint16_t* __restrict__ dl, int64_t ld, int rows, int cols,
                                         const float2* __restrict__ part, int nparts, const float* __restrict__ lse,
                                         const int32_t* __restrict__ labels, const float* __restrict__ scale,
                                         const float* __restrict__ ztarget) {
  const int64_t per_row = cols / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = idx / per_row;
  if (r >= rows) return;
  const int c = static_cast<int>(idx - r * per_row) * 8;
  const int lab = labels[r];
  const float sc = (lab >= 0 && lab < cols) ? *scale : 0.f;
  const float f = exp2f(part[r * nparts + (c >> 8)].x - lse[r] * 1.4426950408889634f);
  uint4* p = reinterpret_cast<uint4*>(dl + r * ld + c);
  uint4 w = *p;
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float e0 = __uint_as_float(u[k] << 16), e1 = __uint_as_float(u[k] & 0xffff0000u);
    const float d0 = (e0 * f - (c + 2 * k == lab ? 1.f : 0.f)) * sc;
    const float d1 = (e1 * f - (c + 2 * k + 1 == lab ? 1.f : 0.f)) * sc;
    u[k] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d0)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d1)) << 16);
  }
  if (lab >= c && lab < c + 8) {
    const float d = (exp2f((ztarget[r] - lse[r]) * 1.4426950408889634f) - 1.f) * sc;
    const int k = lab - c;
    const uint32_t b = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d));
    u[k >> 1] = (k & 1) ? ((u[k >> 1] & 0x0000ffffu) | (b << 16)) : ((u[k >> 1] & 0xffff0000u) | b);
  }
  *p = w;
}

// SwiGLU backward from the saved fp32 accumulators (chunk-wise block):
// same arithmetic as the kEpiSwigluBwd epilogue, so results are bitwise
// those of the recompute path.  dG, dU bf16.
__device__ __forceinline__ float sig_rn(float x) { return __frcp_rn(1.0f + __expf(-x)); }
__global__ void swiglu_bwd_kernel(const float* __restrict__ G, const float* __restrict__ U,
                                  const float* __restrict__ dh, uint16_t* __restrict__ dG, uint16_t* __restrict__ dU,
                                  int64_t n4) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 g = reinterpret_cast<const float4*>(G)[i];
  const float4 u = reinterpret_cast<const float4*>(U)[i];
  const float4 d = reinterpret_cast<const float4*>(dh)[i];
  const float gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w}, dv[4] = {d.x, d.y, d.z, d.w};
  uint16_t og[4], ou[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float s_ = sig_rn(gv[k]);
    const float act = gv[k] * s_;
    const float dgv = dv[k] * uv[k] * (s_ * (1.0f + gv[k] * (1.0f - s_)));
    const float duv = dv[k] * act;
    og[k] = __bfloat16_as_ushort(__float2bfloat16_rn(dgv));
    ou[k] = __bfloat16_as_ushort(__float2bfloat16_rn(duv));
  }
  reinterpret_cast<uint2*>(dG)[i] = make_uint2(og[0] | ((uint32_t)og[1] << 16), og[2] | ((uint32_t)og[3] << 16));
  reinterpret_cast<uint2*>(dU)[i] = make_uint2(ou[0] | ((uint32_t)ou[1] << 16), ou[2] | ((uint32_t)ou[3] << 16));
}

// ------------------------------------------------------------ validation
int check_dims(int64_t n, int64_t h, int64_t x, int64_t m, const char* xname) {
  if (n <= 0) return fail(MST_ERR_DATA, "N must be >= 1 (SPEC.md:290), got %lld", (long long)n);
  if (m <= 0) return fail(MST_ERR_CONFIG, "M must be >= 1, got %lld", (long long)m);
  if (h <= 0 || x <= 0) return fail(MST_ERR_SHAPE, "extents must be positive (H=%lld %s=%lld)", (long long)h, xname, (long long)x);
  if (h % 8 || x % 8)
    return fail(MST_ERR_SHAPE, "H and %s must be multiples of 8 for 16-byte TMA rows (H=%lld %s=%lld)", xname,
                (long long)h, xname, (long long)x);
  if (n > (int64_t(1) << 30) || h > 65536 * 4 || x > (int64_t(1) << 24))
    return fail(MST_ERR_BOUNDS, "extent too large");
  return MST_OK;
}

std::vector<int64_t> plan_bounds(int64_t n, int64_t m) {
  const int64_t c = std::min(n, m);
  std::vector<int64_t> b(c + 1);
  const int64_t q = n / c, r = n % c;
  b[0] = 0;
  for (int64_t i = 0; i < c; ++i) b[i + 1] = b[i] + q + (i < r ? 1 : 0);
  return b;
}

int64_t max_chunk(int64_t n, int64_t m) { return cdiv(n, std::min(n, m)); }

const char* bptr(const void* p, int64_t off_elems) { return static_cast<const char*>(p) + off_elems * 2; }

// ------------------------------------------------------------ problem builders
// K1: h = silu(X W_g) * (X W_u) for one chunk.
int build_k1(mst_ctx* c, Launch& L, const void* x, const void* wg, const void* wu, void* h, int64_t rows, int64_t H,
             int64_t I) {
  ProblemDesc& P = L.p.prob[L.p.num_problems++];
  PhaseSpec s{};
  s.a = {x, rows, H, H, false};
  s.b0 = {wg, I, H, I, true};
  s.b1 = {wu, I, H, I, true};
  s.umma_n = 256;
  s.tmem_col = 0;
  MST_TRY(add_phase(c, L, P, s));
  P.m_tiles = (int)cdiv(rows, 256);
  P.tile_n = 128;
  P.n_tiles = (int)cdiv(I, 128);
  P.rows = (int)rows;
  P.cols = (int)I;
  P.epi = mst::kEpiSwiglu;
  MST_TRY(add_out_map(c, L, h, I, rows, I, false, &P.map_out0));
  L.flops += 2.0 * rows * (2.0 * I) * H;
  cnt_mm(c, rows, H, I, (uint64_t)(H * I));  // G = X W_g
  cnt_mm(c, rows, H, I, (uint64_t)(H * I));  // U = X W_u
  return MST_OK;
}

// Plain C[rows, cols] = A B with B split {0,128} over the pair; STORE_BF16 or ACC_F32.
int build_plain(mst_ctx* c, Launch& L, const Operand& a, const Operand& b, void* out, int64_t ld_out, int epi,
                int beta, int nblk = 1) {
  ProblemDesc& P = L.p.prob[L.p.num_problems++];
  P.nblk = nblk;
  PhaseSpec s{};
  s.a = a;
  s.b0 = b;
  s.b1 = b;
  s.umma_n = 256;
  s.b_off0 = 0;
  s.b_off1 = 128;
  MST_TRY(add_phase(c, L, P, s));
  P.m_tiles = (int)cdiv(a.mn, 256);
  P.tile_n = 256;
  P.n_tiles = (int)cdiv(b.mn, 256);
  P.rows = (int)a.mn;
  P.cols = (int)b.mn;
  P.epi = epi;
  P.beta = beta;
  if (epi == mst::kEpiStoreBf16 || epi == mst::kEpiAccF32 || epi == mst::kEpiCeBwd || epi == mst::kEpiCeFwdNum) {
    MST_TRY(add_out_map(c, L, out, b.mn, a.mn, ld_out, epi == mst::kEpiAccF32, &P.map_out0));
    P.map_out1 = P.map_out0;
  }
  P.col_off0 = 0;
  P.col_off1 = 128;
  L.flops += 2.0 * a.mn * b.mn * a.k;
  cnt_mm(c, a.mn, a.k, b.mn,
         (is_weight(c, a.base) ? (uint64_t)(a.mn * a.k) : 0) + (is_weight(c, b.base) ? (uint64_t)(b.mn * b.k) : 0));
  return MST_OK;
}

// K9 (dX_j = dG W_g^T + dU W_u^T), K8 (dW_d += h^T dO_j) and K10
// ([dW_g | dW_u] += X_j^T [dG | dU]) of one chunk: mutually independent,
// added to one grouped launch (Alg. 3 lines 5-7).
// parts: bit 1 K9, bit 2 K8, bit 4 K10 restricted to the dW rows [k10_r0, k10_r1)
// of H (row slabs of the final chunk, mst_ctx_set_grad_slab_hook).
enum { kGradK9 = 1, kGradK8 = 2, kGradK10 = 4, kGradAll = 7, kGradDW = 6 };
// A second chunk's dW operands (chunk-wise block, tuning "pair_dw"): K8 and
// K10 then run over both chunks as one accumulation (two phases, K = the two
// chunk lengths) and read-modify-write the fp32 gradients once per pair.
struct DwChunk {
  const void* dg;
  const void* du;
  const void* ht;
  const void* xt;
  const void* doj;
  int64_t rows;
};
int add_mlp_grads(mst_ctx* c, Launch& L, const void* dg, const void* du, const void* ht, const void* xt,
                  const void* doj, const void* wg, const void* wu, void* dxj, float* dwg, float* dwu, float* dwd,
                  int64_t rows, int64_t h, int64_t i, int64_t ldt, int beta, int parts = kGradAll,
                  int64_t k10_r0 = 0, int64_t k10_r1 = -1, const DwChunk* second = nullptr) {
  if (k10_r1 < 0) k10_r1 = h;
  if (parts & kGradK9) {  // K9: one accumulator over both phases (B K-major)
    ProblemDesc& P = L.p.prob[L.p.num_problems++];
    P.nblk = (c->wide_mask & 8) ? 2 : 1;
    PhaseSpec q0{};
    q0.a = {dg, rows, i, i, false};
    q0.b0 = {wg, h, i, i, false};
    q0.b1 = q0.b0;
    q0.umma_n = 256;
    q0.b_off1 = 128;
    MST_TRY(add_phase(c, L, P, q0));
    PhaseSpec q1 = q0;
    q1.a = {du, rows, i, i, false};
    q1.b0 = {wu, h, i, i, false};
    q1.b1 = q1.b0;
    q1.acc_continue = true;
    MST_TRY(add_phase(c, L, P, q1));
    P.m_tiles = (int)cdiv(rows, 256);
    P.tile_n = 256;
    P.n_tiles = (int)cdiv(h, 256);
    P.rows = (int)rows;
    P.cols = (int)h;
    P.epi = mst::kEpiStoreBf16;
    MST_TRY(add_out_map(c, L, dxj, h, rows, h, false, &P.map_out0));
    P.map_out1 = P.map_out0;
    P.col_off0 = 0;
    P.col_off1 = 128;
    L.flops += 2.0 * 2.0 * rows * h * i;
    cnt_mm(c, rows, i, h, (uint64_t)(h * i));  // dG W_g^T
    cnt_mm(c, rows, i, h, (uint64_t)(h * i));  // dU W_u^T
  }
  if (parts & kGradK9) cnt_op(c, (uint64_t)(rows * h), 3ull * rows * h);  // dX' + dX'' (fused: one K = 2I accumulation)
  // K8: dW_d[I,H] += h^T dO_j (A = h^T, K-major)
  if (parts & kGradK8) {
    MST_TRY(build_plain(c, L, Operand{ht, i, rows, ldt, false}, Operand{doj, h, rows, h, true}, dwd, h,
                        mst::kEpiAccF32, beta));
    if (second) {  // + h'^T dO' of the second chunk, same accumulator
      ProblemDesc& P = L.p.prob[L.p.num_problems - 1];
      PhaseSpec s{};
      s.a = {second->ht, i, second->rows, ldt, false};
      s.b0 = {second->doj, h, second->rows, h, true};
      s.b1 = s.b0;
      s.umma_n = 256;
      s.b_off1 = 128;
      s.acc_continue = true;
      MST_TRY(add_phase(c, L, P, s));
      L.flops += 2.0 * i * h * second->rows;
      cnt_mm(c, i, second->rows, h, 0);
    }
  }
  if ((parts & kGradK10) && k10_r1 > k10_r0) {  // K10: [dW_g | dW_u][H, I] += X_j^T [dG | dU]  (A = X_j^T, K-major)
    const int64_t hs = k10_r1 - k10_r0;
    xt = bptr(xt, k10_r0 * ldt);
    dwg += k10_r0 * i;
    dwu += k10_r0 * i;
    ProblemDesc& P = L.p.prob[L.p.num_problems++];
    PhaseSpec q{};
    q.a = {xt, hs, rows, ldt, false};
    q.b0 = {dg, i, rows, i, true};
    q.b1 = {du, i, rows, i, true};
    q.umma_n = 256;
    MST_TRY(add_phase(c, L, P, q));
    if (second) {  // + X'^T [dG' | dU'] of the second chunk
      PhaseSpec q2 = q;
      q2.a = {bptr(second->xt, k10_r0 * ldt), hs, second->rows, ldt, false};
      q2.b0 = {second->dg, i, second->rows, i, true};
      q2.b1 = {second->du, i, second->rows, i, true};
      q2.acc_continue = true;
      MST_TRY(add_phase(c, L, P, q2));
      L.flops += 2.0 * hs * (2.0 * i) * second->rows;
      cnt_mm(c, hs, second->rows, i, 0);
      cnt_mm(c, hs, second->rows, i, 0);
    }
    P.m_tiles = (int)cdiv(hs, 256);
    P.tile_n = 128;
    P.n_tiles = (int)cdiv(i, 128);
    P.rows = (int)hs;
    P.cols = (int)i;
    P.epi = mst::kEpiAccF32;
    P.beta = beta;
    MST_TRY(add_out_map(c, L, dwg, i, hs, i, true, &P.map_out0));
    MST_TRY(add_out_map(c, L, dwu, i, hs, i, true, &P.map_out1));
    P.col_off0 = P.col_off1 = 0;
    L.flops += 2.0 * hs * (2.0 * i) * rows;
    cnt_mm(c, hs, rows, i, 0);  // dW_g += X^T dG
    cnt_mm(c, hs, rows, i, 0);  // dW_u += X^T dU
  }
  return MST_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int mst_abi_version(void) { return MST_ABI_VERSION; }
const char* mst_last_error(void) { return g_last_error.c_str(); }

int mst_ctx_create(int device, mst_ctx** out) {
  if (!out) return fail(MST_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  MST_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MST_ERR_CONFIG, "device %d out of range (%d devices)", device, ndev);
  MST_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  MST_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(MST_ERR_CONFIG, "libmst is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major,
                prop.minor);
  mst_ctx* c = new mst_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) {
    delete c;
    return fail(MST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  }
  c->encode = reinterpret_cast<EncodeTiledFn>(fn);
  if (const char* dy = getenv("MST_DYNAMIC")) c->dynamic = atoi(dy) != 0;
  e = cudaFuncSetAttribute(mst::mst_grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           mst::kSmemBytes);
  if (e == cudaSuccess) e = mst_attn::init_device();
  if (e != cudaSuccess) {
    delete c;
    return fail(MST_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  // Co-resident CTA pairs (persistent grid size).
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(2 * (c->num_sms / 2));
  cfg.blockDim = dim3(mst::kThreads);
  cfg.dynamicSmemBytes = mst::kSmemBytes;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&clusters, mst::mst_grouped_gemm_kernel, &cfg);
  if (e != cudaSuccess || clusters <= 0) clusters = c->num_sms / 2;
  c->num_pairs = std::min(clusters, c->num_sms / 2);
  c->max_pairs = c->num_pairs;
  e = cudaMalloc(&c->scratch_dev, 4096);
  if (e == cudaSuccess) e = cudaMemset(c->scratch_dev, 0, 4096);
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), 64, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *c->err_host = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
  }
  if (e != cudaSuccess) {
    delete c;
    return fail(MST_ERR_CUDA, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  *out = c;
  return MST_OK;
}

void mst_ctx_destroy(mst_ctx* c) {
  if (!c) return;
  for (auto& kv : c->sched_cache) cudaFree(kv.second.dev);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  cudaFree(c->scratch_dev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->io_dev) cudaFree(c->io_dev);
  for (cudaEvent_t e : c->io_ev)
    if (e) cudaEventDestroy(e);
  if (c->tail_ev) cudaEventDestroy(c->tail_ev);
  if (c->err_host) cudaFreeHost(c->err_host);
  delete c;
}

int mst_ctx_set_timing(mst_ctx* c, int enable) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->timing = enable != 0;
  return MST_OK;
}

int mst_ctx_take_timing(mst_ctx* c, double* ms_out, double* flops_out, int64_t* n_out) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  double ms = 0, fl = 0;
  const int64_t n = (int64_t)(c->ev_used / 2);
  for (int64_t k = 0; k < n; ++k) {
    MST_CUDA(cudaEventSynchronize(c->ev[2 * k + 1]));
    float t = 0;
    MST_CUDA(cudaEventElapsedTime(&t, c->ev[2 * k], c->ev[2 * k + 1]));
    ms += t;
    fl += c->ev_flops[k];
  }
  c->ev_used = 0;
  c->ev_flops.clear();
  if (ms_out) *ms_out = ms;
  if (flops_out) *flops_out = fl;
  if (n_out) *n_out = n;
  return MST_OK;
}

int mst_ctx_take_timing_records(mst_ctx* c, int64_t cap, double* ms, double* flops, int64_t* n_out) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  const int64_t n = (int64_t)(c->ev_used / 2);
  int64_t w = 0;
  for (int64_t k = 0; k < n; ++k) {
    MST_CUDA(cudaEventSynchronize(c->ev[2 * k + 1]));
    float t = 0;
    MST_CUDA(cudaEventElapsedTime(&t, c->ev[2 * k], c->ev[2 * k + 1]));
    if (w < cap) {
      ms[w] = t;
      flops[w] = c->ev_flops[k];
      ++w;
    }
  }
  c->ev_used = 0;
  c->ev_flops.clear();
  if (n_out) *n_out = w;
  return MST_OK;
}

int mst_ctx_set_profile_buffer(mst_ctx* c, void* dev_counters) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->prof = static_cast<unsigned long long*>(dev_counters);
  c->prof_slot = 0;
  return MST_OK;
}

int mst_ctx_set_tuning(mst_ctx* c, const char* key, int value) {
  if (!c || !key) return fail(MST_ERR_STATE, "NULL context or key");
  if (std::strcmp(key, "dynamic") == 0) {
    c->dynamic = value != 0;
  } else if (std::strcmp(key, "fused_head") == 0) {
    c->fused_head = value != 0;
  } else if (std::strcmp(key, "chunked_block") == 0) {
    c->chunked_block = value != 0;
  } else if (std::strcmp(key, "wide") == 0) {
    c->wide = value != 0;
  } else if (std::strcmp(key, "dl_rowscale") == 0) {
    c->dl_rowscale = value != 0;
  } else if (std::strcmp(key, "pair_dw") == 0) {
    c->pair_dw = value != 0;
  } else if (std::strcmp(key, "k9_in_k1") == 0) {
    c->k9_in_k1 = value != 0;
  } else if (std::strcmp(key, "fuse_swiglu_bwd") == 0) {
    c->fuse_swiglu_bwd = value != 0;
  } else if (std::strcmp(key, "wide_mask") == 0) {
    c->wide_mask = value;
  } else if (std::strcmp(key, "debug_nblk") == 0) {
    if (value < 1 || value > mst::kMaxNBlk) return fail(MST_ERR_CONFIG, "debug_nblk must be 1..%d", mst::kMaxNBlk);
    c->debug_nblk = value;
  } else if (std::strcmp(key, "pairs") == 0) {  // diagnostics: run GEMMs on fewer CTA pairs
    if (value < 1 || value > c->max_pairs) return fail(MST_ERR_CONFIG, "pairs must be 1..%d", c->max_pairs);
    c->num_pairs = value;
  } else if (std::strcmp(key, "attn_fwd") == 0) {  // attention forward kernel version (per context)
    if (value != 1 && value != 2) return fail(MST_ERR_CONFIG, "attn_fwd must be 1 or 2");
    c->attn.fwd_version = value;
  } else if (std::strcmp(key, "attn_poly") == 0) {  // forward softmax exp2 pairs of 4 on the FMA pipe (per context)
    if (value < 0 || value > 3) return fail(MST_ERR_CONFIG, "attn_poly must be 0..3");
    c->attn.poly_exp = value;
  } else if (std::strcmp(key, "attn_bwd_order") == 0) {  // dK/dV GEMM issue order (per context)
    if (value < 0 || value > 3) return fail(MST_ERR_CONFIG, "attn_bwd_order must be 0..3 (bit 0 dK/dV, bit 1 dQ)");
    c->attn.bwd_order = value;
  } else if (std::strcmp(key, "attn_inorder") == 0) {
    c->attn.mma_inorder = value != 0;
  } else if (std::strcmp(key, "attn_bwd") == 0) {  // attention backward kernel version (per context)
    if (value != 1 && value != 2) return fail(MST_ERR_CONFIG, "attn_bwd must be 1 or 2");
    c->attn.bwd_version = value;
  } else if (std::strcmp(key, "tma3d") == 0) {
    c->tma3d = value != 0;
  } else {
    return fail(MST_ERR_CONFIG, "unknown tuning key '%s'", key);
  }
  for (auto& kv : c->sched_cache) cudaFree(kv.second.dev);
  c->sched_cache.clear();
  return MST_OK;
}

int mst_ctx_num_pairs(const mst_ctx* c) { return c ? c->num_pairs : 0; }

int mst_ctx_get_counters(const mst_ctx* c, mst_counters* out) {
  if (!c || !out) return fail(MST_ERR_STATE, "NULL context or output");
  *out = c->ctr;
  return MST_OK;
}
int mst_ctx_reset_counters(mst_ctx* c) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->ctr = mst_counters{};
  return MST_OK;
}
int mst_ctx_set_mem_hook(mst_ctx* c, mst_mem_hook fn, void* user) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->mem_fn = fn;
  c->mem_user = user;
  return MST_OK;
}
int mst_ctx_check(mst_ctx* c, void* stream) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  MST_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return take_sticky(c);
}

int mst_ctx_set_grad_slab_hook(mst_ctx* c, mst_grad_slab_hook fn, void* user, int slabs) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  if (slabs < 1 || slabs > 64) return fail(MST_ERR_CONFIG, "slabs must be 1..64, got %d", slabs);
  c->slab_fn = fn;
  c->slab_user = user;
  c->slabs = fn ? slabs : 1;
  return MST_OK;
}

int mst_ctx_set_grad_ready_hook(mst_ctx* c, mst_grad_ready_hook fn, void* user) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->ready_fn = fn;
  c->ready_user = user;
  return MST_OK;
}

// ------------------------------------------------------------ optimizer (optim.cu)
int mst_adamw_step(mst_ctx* c, void* stream, int64_t n, float* w, void* w_bf16, float* grad, float* m, float* v,
                   const mst_adamw_config* cfg, int64_t step, const float* grad_scale, int zero_grad) {
  MST_CALL(c, stream);
  if (!cfg) return fail(MST_ERR_CONFIG, "NULL AdamW config");
  if (n < 0) return fail(MST_ERR_SHAPE, "negative parameter count");
  if (!w || !w_bf16 || !grad || !m || !v) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  if (step < 1) return fail(MST_ERR_CONFIG, "step must be >= 1 (bias correction), got %lld", (long long)step);
  if (!(cfg->lr > 0.0) || !(cfg->beta1 > 0.0 && cfg->beta1 < 1.0) || !(cfg->beta2 > 0.0 && cfg->beta2 < 1.0) ||
      !(cfg->eps > 0.0) || !(cfg->weight_decay >= 0.0))
    return fail(MST_ERR_CONFIG, "invalid AdamW config (SPEC.md:477: lr > 0, 0 < betas < 1, eps > 0, wd >= 0)");
  if (!mst_optim::aligned16(w) || !mst_optim::aligned16(grad) || !mst_optim::aligned16(m) ||
      !mst_optim::aligned16(v) || (reinterpret_cast<uintptr_t>(w_bf16) & 7) != 0)
    return fail(MST_ERR_CONFIG, "optimizer tensors must be 16-byte aligned (bf16 copy: 8-byte)");
  if (n == 0) return MST_OK;
  MST_CUDA(mst_optim::launch_adamw(static_cast<cudaStream_t>(stream), c->num_sms, n, w, w_bf16, grad, m, v, *cfg, step,
                                   grad_scale, zero_grad));
  c->launches++;
  return MST_OK;
}

int mst_grad_sumsq_workspace(void) { return mst_optim::kSumsqBlocks; }

int mst_grad_sumsq(mst_ctx* c, void* stream, const float* grad, int64_t n, double* partial_ws, double* sumsq,
                   int accumulate, float max_norm, float inv_steps, float* scale_out, float* norm_out) {
  MST_CALL(c, stream);
  if (!grad || !partial_ws || !sumsq) return fail(MST_ERR_CONFIG, "NULL pointer");
  if (n < 0) return fail(MST_ERR_SHAPE, "negative element count");
  if (!mst_optim::aligned16(grad)) return fail(MST_ERR_CONFIG, "gradient must be 16-byte aligned");
  if (scale_out && !(max_norm > 0.f)) return fail(MST_ERR_CONFIG, "clip norm must be > 0 (SPEC.md:477)");
  MST_CUDA(mst_optim::launch_sumsq(static_cast<cudaStream_t>(stream), grad, n, partial_ws, sumsq, accumulate, max_norm,
                                   inv_steps, scale_out, norm_out));
  c->launches += 2;
  return MST_OK;
}

int mst_grad_accumulate(mst_ctx* c, void* stream, float* into, const float* from, int64_t n) {
  MST_CALL(c, stream);
  if (!into || !from) return fail(MST_ERR_CONFIG, "NULL pointer");
  if (n < 0) return fail(MST_ERR_SHAPE, "negative element count");
  if (!mst_optim::aligned16(into) || !mst_optim::aligned16(from))
    return fail(MST_ERR_CONFIG, "gradients must be 16-byte aligned");
  if (n == 0) return MST_OK;
  MST_CUDA(mst_optim::launch_accumulate(static_cast<cudaStream_t>(stream), c->num_sms, into, from, n));
  c->launches++;
  return MST_OK;
}

int mst_ctx_set_count_hook(mst_ctx* c, mst_count_hook fn, void* user) {
  if (!c) return fail(MST_ERR_STATE, "NULL context");
  c->cnt_fn = fn;
  c->cnt_user = user;
  return MST_OK;
}
int64_t mst_ctx_launch_count(const mst_ctx* c) { return c ? c->launches : 0; }

int mst_make_chunk_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* num_chunks) {
  if (n <= 0) return fail(MST_ERR_DATA, "make_chunk_plan: N must be >= 1 (SPEC.md:290)");
  if (m <= 0) return fail(MST_ERR_CONFIG, "make_chunk_plan: M must be >= 1");
  std::vector<int64_t> b = plan_bounds(n, m);
  if (num_chunks) *num_chunks = (int64_t)b.size() - 1;
  if (bounds) std::memcpy(bounds, b.data(), b.size() * sizeof(int64_t));
  return MST_OK;
}

// ---- workspace layouts (shared by size query and execution)
// Row stride (elements) of the transposed chunk buffers [feature, token]:
// the chunk's token count rounded up to 16-byte rows.
static int64_t ld_t(int64_t n, int64_t m) { return (max_chunk(n, m) + 7) / 8 * 8; }

static int carve_mlp(Carve& cv, int64_t n, int64_t h, int64_t i, int64_t m, void** hbuf, void** dg, void** du,
                     float** dh = nullptr, void** xt = nullptr, void** ht = nullptr) {
  const int64_t nc = max_chunk(n, m);
  const size_t hb = size_t(nc) * i * 2;
  // forward uses two h buffers (ping-pong across chunks); backward h, dG,
  // dU (bf16) and dh (fp32, exactly the accumulator values).
  *hbuf = cv.take(hb);
  *dg = cv.take(hb);
  *du = cv.take(hb);
  float* d = static_cast<float*>(cv.take(size_t(nc) * i * 4));
  if (dh) *dh = d;
  // X_j^T and h^T (K-major A operands of the dW GEMMs K10 / K8)
  void* x = cv.take(size_t(h) * ld_t(n, m) * 2);
  void* t = cv.take(size_t(i) * ld_t(n, m) * 2);
  if (xt) *xt = x;
  if (ht) *ht = t;
  return MST_OK;
}

static void carve_head(Carve& cv, int64_t n, int64_t h, int64_t v, int64_t m, float2** part, float** zt,
                       float** lrow, void** dl, float** scales, void** ot = nullptr) {
  const int64_t nc = max_chunk(n, m);
  const int64_t nparts = cdiv(v, 256);
  *part = static_cast<float2*>(cv.take(size_t(nc) * nparts * sizeof(float2)));
  *zt = static_cast<float*>(cv.take(size_t(nc) * 4));
  *lrow = static_cast<float*>(cv.take(size_t(nc) * 4));
  *dl = cv.take(size_t(nc) * v * 2);
  *scales = static_cast<float*>(cv.take(size_t(std::min(n, m)) * 4 + 64));
  void* o = cv.take(size_t(h) * ld_t(n, m) * 2);  // X_j^T: K-major A operand of K6
  if (ot) *ot = o;
}

int mst_mlp_workspace(int64_t n, int64_t h, int64_t i, int64_t m, size_t* bytes) {
  MST_TRY(check_dims(n, h, i, m, "I"));
  Carve cv{nullptr, 0, 0, true};
  void *a, *b, *d;
  carve_mlp(cv, n, h, i, m, &a, &b, &d);
  *bytes = align_up(cv.used, 256);
  return MST_OK;
}

int mst_lmhead_workspace(int64_t n, int64_t h, int64_t v, int64_t m, size_t* bytes) {
  MST_TRY(check_dims(n, h, v, m, "V"));
  Carve cv{nullptr, 0, 0, true};
  float2* part;
  float *zt, *lr, *sc;
  void* dl;
  carve_head(cv, n, h, v, m, &part, &zt, &lr, &dl, &sc);
  *bytes = align_up(cv.used, 256);
  return MST_OK;
}

static size_t block_fixed_bytes(int64_t n, int64_t h) { return align_up(size_t(n) * h * 2, 256) * 2 + align_up(size_t(n) * 4, 256); }
// Chunk-wise block: O_j lives only within chunk j, dO_j until chunk j+1's
// dW_down GEMM (double buffer); lse stays sequence-sized (4 bytes / token).
static size_t chunked_fixed_bytes(int64_t n, int64_t h, int64_t m) {
  return align_up(size_t(max_chunk(n, m)) * h * 2, 256) * 3 + align_up(size_t(n) * 4, 256);
}

// Chunk-wise block (M_mlp == M_head): MLP and head chunk buffers coexist,
// plus the forward's fp32 G, U accumulators of one chunk.
static size_t chunked_extra_bytes(int64_t n, int64_t h, int64_t i, int64_t m, bool pair) {
  const size_t g = 2 * align_up(size_t(max_chunk(n, m)) * i * 4, 256) + 512;
  if (!pair || std::min(n, m) < 2) return g;
  // second dW operand set {dG, dU, h^T, X^T} (tuning "pair_dw")
  const int64_t nc = max_chunk(n, m), ldt = (nc + 7) / 8 * 8;
  return g + 2 * align_up(size_t(nc) * i * 2, 256) + align_up(size_t(i) * ldt * 2, 256) +
         align_up(size_t(h) * ldt * 2, 256) + 256;
}

// The head plan refines the MLP plan: every MLP chunk boundary is also a
// head chunk boundary, so each MLP chunk holds whole head chunks (always
// true for M_mlp == M_head; for the paper's M_mlp=4 / M_head=16 when 16 | S,
// and in general when the balanced plans happen to nest).
static bool plans_nest(int64_t n, int64_t m_mlp, int64_t m_head) {
  if (n <= 0 || m_mlp <= 0 || m_head <= 0) return false;
  if (m_mlp == m_head) return true;
  const std::vector<int64_t> bm = plan_bounds(n, m_mlp), bh = plan_bounds(n, m_head);
  size_t k = 0;
  for (int64_t x : bm) {
    while (k < bh.size() && bh[k] < x) ++k;
    if (k == bh.size() || bh[k] != x) return false;
  }
  return true;
}

int mst_block_workspace(int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp, int64_t m_head, size_t* bytes) {
  size_t a = 0, b = 0;
  MST_TRY(mst_mlp_workspace(n, h, i, m_mlp, &a));
  MST_TRY(mst_lmhead_workspace(n, h, v, m_head, &b));
  const size_t two_pass = block_fixed_bytes(n, h) + 256 + std::max(a, b);
  const size_t chunked = plans_nest(n, m_mlp, m_head)
                             ? chunked_fixed_bytes(n, h, m_mlp) + 256 + a + b + chunked_extra_bytes(n, h, i, m_mlp, true)
                             : 0;
  *bytes = std::max(two_pass, chunked);
  return MST_OK;
}

static bool uses_chunked_block(const mst_ctx* c, int64_t n, int64_t m_mlp, int64_t m_head) {
  return c->chunked_block && c->fused_head && plans_nest(n, m_mlp, m_head);
}

int mst_ctx_block_workspace(const mst_ctx* c, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp,
                            int64_t m_head, size_t* bytes) {
  if (!c || !bytes) return fail(MST_ERR_STATE, "NULL context or output");
  size_t a = 0, b = 0;
  MST_TRY(mst_mlp_workspace(n, h, i, m_mlp, &a));
  MST_TRY(mst_lmhead_workspace(n, h, v, m_head, &b));
  *bytes = uses_chunked_block(c, n, m_mlp, m_head)
               ? chunked_fixed_bytes(n, h, m_mlp) + 256 + a + b + chunked_extra_bytes(n, h, i, m_mlp, c->pair_dw != 0)
               : block_fixed_bytes(n, h) + 256 + std::max(a, b);
  return MST_OK;
}

static uint64_t mlp_fp(const mst_mlp_saved* s) { return fnv1a(s, offsetof(mst_mlp_saved, fingerprint)) ^ 0x4d4c50ull; }
static uint64_t head_fp(const mst_lmhead_saved* s) {
  return fnv1a(s, offsetof(mst_lmhead_saved, fingerprint)) ^ 0x48454144ull;
}

int mst_mlp_forward(mst_ctx* c, void* stream, const void* x, const void* wg, const void* wu, const void* wd, void* out,
                    int64_t n, int64_t h, int64_t i, int64_t m, void* ws, size_t ws_bytes, mst_mlp_saved* saved) {
  MST_CALL(c, stream);
  MST_TRY(check_dims(n, h, i, m, "I"));
  if (!x || !wg || !wu || !wd || !out) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  size_t need = 0;
  MST_TRY(mst_mlp_workspace(n, h, i, m, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carve cv{static_cast<char*>(ws), ws_bytes, 0, false};
  void *hb[2], *unused;
  carve_mlp(cv, n, h, i, m, &hb[0], &hb[1], &unused);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  WeightScope ws_(c, wg, wu, wd);
  // Software pipeline over chunks: launch j runs K2(j-1) and K1(j) together
  // (independent: different h buffers), so the long-K down GEMM of one chunk
  // fills the tail of the next chunk's gate/up GEMM (Alg. 1 loop).
  // Two h chunk buffers are live across that launch.
  for (int j = 0; j <= nch; ++j) {
    Launch L;
    if (j >= 1) {
      const int64_t r0 = b[j - 1], rows = b[j] - b[j - 1];
      Operand a{hb[(j - 1) & 1], rows, i, i, false};
      Operand bw{wd, h, i, h, true};
      MST_TRY(build_plain(c, L, a, bw, const_cast<char*>(bptr(out, r0 * h)), h, mst::kEpiStoreBf16, 0));
    }
    if (j < nch) {
      const int64_t r0 = b[j], rows = b[j + 1] - b[j];
      mem_alloc(c, (uint64_t)rows * i * 2, "inter.mlp.h");
      MST_TRY(build_k1(c, L, bptr(x, r0 * h), wg, wu, hb[j & 1], rows, h, i));
      cnt_op(c, 4ull * rows * i, 2ull * rows * i);  // silu (fused into the K1 epilogue)
      cnt_op(c, 1ull * rows * i, 3ull * rows * i);  // hadamard
    }
    MST_TRY(launch(c, st, L));
    if (j >= 1) mem_free(c, (uint64_t)(b[j] - b[j - 1]) * i * 2, "inter.mlp.h");
  }
  MST_CUDA(cudaGetLastError());
  if (saved) {
    saved->x = x;
    saved->w_gate = wg;
    saved->w_up = wu;
    saved->w_down = wd;
    saved->n = n;
    saved->h = h;
    saved->i = i;
    saved->m = m;
    saved->fingerprint = mlp_fp(saved);
  }
  return MST_OK;
}

int mst_mlp_backward(mst_ctx* c, void* stream, const void* dout, const mst_mlp_saved* s, const void* wg, const void* wu,
                     const void* wd, void* dx, float* dwg, float* dwu, float* dwd, int accumulate, void* ws,
                     size_t ws_bytes) {
  MST_CALL(c, stream);
  if (!s || s->fingerprint != mlp_fp(s)) return fail(MST_ERR_STATE, "stale or corrupted MLP saved state (SPEC.md:308)");
  if (s->w_gate != wg || s->w_up != wu || s->w_down != wd)
    return fail(MST_ERR_STATE, "MLP saved state was produced with different weights");
  if (!dout || !dx || !dwg || !dwu || !dwd) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  const int64_t n = s->n, h = s->h, i = s->i, m = s->m;
  size_t need = 0;
  MST_TRY(mst_mlp_workspace(n, h, i, m, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carve cv{static_cast<char*>(ws), ws_bytes, 0, false};
  void *hb, *dg, *du, *xt, *ht;
  float* dhb;
  carve_mlp(cv, n, h, i, m, &hb, &dg, &du, &dhb, &xt, &ht);
  const int64_t ldt = ld_t(n, m);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  WeightScope ws_(c, wg, wu, wd);
  // K7a(j): dh = dO_j W_d^T, fp32 (B[k=h, n=i] = W_d[i, h]: K-major).
  auto add_k7a = [&](Launch& L, int j) -> int {
    const int64_t r0 = b[j], rows = b[j + 1] - b[j];
    mem_alloc(c, (uint64_t)rows * i * 4, "inter.mlp.dh");
    return build_plain(c, L, Operand{bptr(dout, r0 * h), rows, h, h, false}, Operand{wd, i, h, h, false}, dhb, i,
                       mst::kEpiAccF32, 0);
  };
  {
    Launch L;
    MST_TRY(add_k7a(L, 0));
    MST_TRY(launch(c, st, L));
  }
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = b[j], rows = b[j + 1] - b[j];
    const int beta = (j > 0 || accumulate) ? 1 : 0;
    const void* xj = bptr(s->x, r0 * h);
    const void* doj = bptr(dout, r0 * h);
    {  // K7b: recompute G,U; epilogue combines with dh -> h, dG, dU (Alg. 3 lines 2-4).
      Launch L;
      ProblemDesc& P = L.p.prob[L.p.num_problems++];
      PhaseSpec p0{};
      p0.a = {xj, rows, h, h, false};
      p0.b0 = {wg, i, h, i, true};
      p0.b1 = {wu, i, h, i, true};
      p0.umma_n = 256;
      MST_TRY(add_phase(c, L, P, p0));
      P.m_tiles = (int)cdiv(rows, 256);
      P.tile_n = 128;
      P.n_tiles = (int)cdiv(i, 128);
      P.rows = (int)rows;
      P.cols = (int)i;
      P.epi = mst::kEpiSwigluBwd;
      P.aux = dhb;
      P.ld_aux = i;
      MST_TRY(add_out_map(c, L, hb, i, rows, i, false, &P.map_out0));
      MST_TRY(add_out_map(c, L, dg, i, rows, i, false, &P.map_out1));
      MST_TRY(add_out_map(c, L, du, i, rows, i, false, &P.map_out2));
      L.flops += 2.0 * rows * (2.0 * i) * h;
      mem_alloc(c, (uint64_t)rows * i * 2, "inter.mlp.h");
      mem_alloc(c, (uint64_t)rows * i * 2, "inter.mlp.dG");
      mem_alloc(c, (uint64_t)rows * i * 2, "inter.mlp.dU");
      cnt_mm(c, rows, h, i, (uint64_t)(h * i));      // G recompute
      cnt_mm(c, rows, h, i, (uint64_t)(h * i));      // U recompute
      cnt_op(c, 4ull * rows * i, 3ull * rows * i);   // silu + silu_backward (fused epilogue)
      cnt_op(c, 2ull * rows * i, 6ull * rows * i);   // dG, dU products
      MST_TRY(launch(c, st, L));
      mem_free(c, (uint64_t)rows * i * 4, "inter.mlp.dh");
    }
    // K-major A operands for the dW GEMMs: h^T (K8) and X_j^T (K10).
    mem_alloc(c, (uint64_t)rows * i * 2, "inter.mlp.hT");
    mem_alloc(c, (uint64_t)rows * h * 2, "act.xT");
    MST_TRY(transpose_bf16(c, st, hb, i, ht, ldt, rows, i));
    MST_TRY(transpose_bf16(c, st, xj, h, xt, ldt, rows, h));
    {  // K9 + K8 + K10 (mutually independent) + K7a of the next chunk, one launch.
      Launch L;
      MST_TRY(add_mlp_grads(c, L, dg, du, ht, xt, doj, wg, wu, const_cast<char*>(bptr(dx, r0 * h)), dwg, dwu, dwd,
                            rows, h, i, ldt, beta));
      if (j + 1 < nch) MST_TRY(add_k7a(L, j + 1));
      MST_TRY(launch(c, st, L));
    }
    mem_free(c, (uint64_t)rows * h * 2, "act.xT");
    mem_free(c, (uint64_t)rows * i * 2, "inter.mlp.hT");
    mem_free(c, (uint64_t)rows * i * 2, "inter.mlp.dU");
    mem_free(c, (uint64_t)rows * i * 2, "inter.mlp.dG");
    mem_free(c, (uint64_t)rows * i * 2, "inter.mlp.h");
  }
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

int mst_lmhead_forward(mst_ctx* c, void* stream, const void* x, const int32_t* labels, const void* wout, int64_t n,
                       int64_t h, int64_t v, int64_t m, int loss_mode, float* stats, float* lse, void* ws,
                       size_t ws_bytes, mst_lmhead_saved* saved) {
  MST_CALL(c, stream);
  MST_TRY(check_dims(n, h, v, m, "V"));
  if (loss_mode != MST_LOSS_TOKEN_WEIGHTED && loss_mode != MST_LOSS_PAPER_MEAN)
    return fail(MST_ERR_CONFIG, "unknown loss mode %d", loss_mode);
  if (!x || !labels || !wout || !stats || !lse) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  size_t need = 0;
  MST_TRY(mst_lmhead_workspace(n, h, v, m, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carve cv{static_cast<char*>(ws), ws_bytes, 0, false};
  float2* part;
  float *zt, *lrow, *scales;
  void* dl;
  carve_head(cv, n, h, v, m, &part, &zt, &lrow, &dl, &scales);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  const int nparts = (int)cdiv(v, 256);
  MST_CUDA(cudaMemsetAsync(stats, 0, sizeof(float) * MST_STATS_LEN(nch), st));
  WeightScope ws_(c, wout);
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = b[j], rows = b[j + 1] - b[j];
    const uint64_t part_bytes = (uint64_t)rows * nparts * 8 + (uint64_t)rows * 8;  // partials + z_target + row loss
    mem_alloc(c, part_bytes, "inter.head.partials");
    cnt_op(c, 5ull * rows * v, (uint64_t)(rows * v + 2 * rows));  // cross-entropy forward (fused epilogue)
    Launch L;  // K3: logits GEMM + online-softmax partials
    MST_TRY(build_plain(c, L, Operand{bptr(x, r0 * h), rows, h, h, false}, Operand{wout, v, h, v, true}, nullptr, 0,
                        mst::kEpiCeFwd, 0));
    ProblemDesc& P = L.p.prob[0];
    P.labels = labels + r0;
    P.part = part;
    P.ztarget = zt;
    P.nparts = nparts;
    MST_TRY(launch(c, st, L));
    const int threads = 256;
    const int blocks = (int)cdiv(rows * 32, threads);
    ce_combine_kernel<<<blocks, threads, 0, st>>>(part, nparts, zt, labels + r0, (int)rows, (int)v, lse + r0, lrow,
                                                   stats + 3);
    chunk_reduce_kernel<<<1, 1024, 0, st>>>(lrow, labels + r0, (int)rows, (int)v, stats + 4 + j, stats + 4 + nch + j);
    c->launches += 2;
    mem_free(c, part_bytes, "inter.head.partials");
  }
  finalize_loss_kernel<<<1, 32, 0, st>>>(stats, nch, loss_mode, c->err_dev, nullptr);
  c->launches += 1;
  MST_CUDA(cudaGetLastError());
  if (saved) {
    saved->x = x;
    saved->labels = labels;
    saved->w_out = wout;
    saved->lse = lse;
    saved->stats = stats;
    saved->n = n;
    saved->h = h;
    saved->v = v;
    saved->m = m;
    saved->loss_mode = loss_mode;
    saved->_pad = 0;
    saved->fingerprint = head_fp(saved);
  }
  return MST_OK;
}

int mst_lmhead_backward(mst_ctx* c, void* stream, const mst_lmhead_saved* s, const void* wout,
                        const float* global_stats, float grad_loss, void* dx, float* dwout, int accumulate, void* ws,
                        size_t ws_bytes) {
  MST_CALL(c, stream);
  if (!s || s->fingerprint != head_fp(s)) return fail(MST_ERR_STATE, "stale or corrupted LM-Head saved state (SPEC.md:308)");
  if (s->w_out != wout) return fail(MST_ERR_STATE, "LM-Head saved state was produced with different weights");
  if (!dx || !dwout) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  const int64_t n = s->n, h = s->h, v = s->v, m = s->m;
  size_t need = 0;
  MST_TRY(mst_lmhead_workspace(n, h, v, m, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carve cv{static_cast<char*>(ws), ws_bytes, 0, false};
  float2* part;
  float *zt, *lrow, *scales;
  void *dl, *ot;
  carve_head(cv, n, h, v, m, &part, &zt, &lrow, &dl, &scales, &ot);
  const int64_t ldt = ld_t(n, m);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  double* tot = reinterpret_cast<double*>(c->scratch_dev + 64);  // context scratch (calls are serialised)
  if (!global_stats) valid_total_kernel<<<1, 32, 0, st>>>(s->stats, nch, tot);
  grad_scale_kernel<<<(nch + 255) / 256, 256, 0, st>>>(global_stats ? nullptr : tot, global_stats, s->stats, nch,
                                                           s->loss_mode, grad_loss, scales);
  c->launches += global_stats ? 1 : 2;
  WeightScope ws_(c, wout);
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = b[j], rows = b[j + 1] - b[j];
    const int beta = (j > 0 || accumulate) ? 1 : 0;
    const void* xj = bptr(s->x, r0 * h);
    mem_alloc(c, (uint64_t)rows * h * 2, "act.xT");
    mem_alloc(c, (uint64_t)rows * v * 2, "inter.head.dlogits");
    cnt_op(c, 5ull * rows * v, (uint64_t)(2 * rows * v + 2 * rows));  // cross-entropy backward (fused epilogue)
    MST_TRY(transpose_bf16(c, st, xj, h, ot, ldt, rows, h));  // (head input)_j^T: K-major A of K6
    {  // K4: recompute logits, dlogits = (softmax - onehot) * scale -> bf16
      Launch L;
      MST_TRY(build_plain(c, L, Operand{xj, rows, h, h, false}, Operand{wout, v, h, v, true}, dl, v,
                          mst::kEpiCeBwd, 0));
      ProblemDesc& P = L.p.prob[0];
      P.labels = s->labels + r0;
      P.lse = s->lse + r0;
      P.scale = scales + j;
      MST_TRY(launch(c, st, L));
    }
    {  // K5 (dX = dl W_out^T) + K6 (dW_out += X^T dl), grouped.
      Launch L;
      MST_TRY(build_plain(c, L, Operand{dl, rows, v, v, false}, Operand{wout, h, v, v, false},
                          const_cast<char*>(bptr(dx, r0 * h)), h, mst::kEpiStoreBf16, 0));
      MST_TRY(build_plain(c, L, Operand{ot, h, rows, ldt, false}, Operand{dl, v, rows, v, true}, dwout, v,
                          mst::kEpiAccF32, beta));
      MST_TRY(launch(c, st, L));
    }
    mem_free(c, (uint64_t)rows * v * 2, "inter.head.dlogits");
    mem_free(c, (uint64_t)rows * h * 2, "act.xT");
  }
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

int mst_lmhead_fused(mst_ctx* c, void* stream, const void* x, const int32_t* labels, const void* wout, int64_t n,
                     int64_t h, int64_t v, int64_t m, int loss_mode, float grad_loss, const double* global_valid,
                     float* stats, float* lse, void* dx, float* dwout, int accumulate, void* ws, size_t ws_bytes) {
  MST_CALL(c, stream);
  MST_TRY(check_dims(n, h, v, m, "V"));
  if (loss_mode != MST_LOSS_TOKEN_WEIGHTED && loss_mode != MST_LOSS_PAPER_MEAN)
    return fail(MST_ERR_CONFIG, "unknown loss mode %d", loss_mode);
  if (!x || !labels || !wout || !stats || !lse || !dx || !dwout) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  size_t need = 0;
  MST_TRY(mst_lmhead_workspace(n, h, v, m, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carve cv{static_cast<char*>(ws), ws_bytes, 0, false};
  float2* part;
  float *zt, *lrow, *scales;
  void *dl, *ot;
  carve_head(cv, n, h, v, m, &part, &zt, &lrow, &dl, &scales, &ot);
  const int64_t ldt = ld_t(n, m);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  const int nparts = (int)cdiv(v, 256);
  // Scales first (they only depend on the labels): per-chunk valid counts,
  // total (or the caller's global count), dlogits scale per chunk.
  MST_CUDA(cudaMemsetAsync(stats, 0, sizeof(float) * MST_STATS_LEN(nch), st));
  chunk_valid_kernel<<<nch, 256, 0, st>>>(labels, n, nch, (int)v, stats);
  double* tot = reinterpret_cast<double*>(c->scratch_dev + 64);  // context scratch (calls are serialised)
  sum_valid_kernel<<<1, 32, 0, st>>>(stats, nch, tot);
  grad_scale_kernel<<<(nch + 255) / 256, 256, 0, st>>>(global_valid ? global_valid : tot, nullptr, stats, nch,
                                                      loss_mode, grad_loss, scales);
  c->launches += 3;
  WeightScope ws_(c, wout);
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = b[j], rows = b[j + 1] - b[j];
    const int beta = (j > 0 || accumulate) ? 1 : 0;
    const void* xj = bptr(x, r0 * h);
    const uint64_t part_bytes = (uint64_t)rows * nparts * 8 + (uint64_t)rows * 8;
    mem_alloc(c, (uint64_t)rows * h * 2, "act.xT");
    mem_alloc(c, part_bytes, "inter.head.partials");
    mem_alloc(c, (uint64_t)rows * v * 2, "inter.head.dlogits");
    cnt_op(c, 5ull * rows * v, (uint64_t)(rows * v + 2 * rows));      // cross-entropy forward
    cnt_op(c, 5ull * rows * v, (uint64_t)(2 * rows * v + 2 * rows));  // cross-entropy backward
    const bool rs = c->dl_rowscale != 0;
    if (!rs) MST_TRY(transpose_bf16(c, st, xj, h, ot, ldt, rows, h));  // (head input)_j^T: K-major A of K6
    {  // K3': logits GEMM; epilogue = online-softmax partials + softmax numerators (bf16)
      Launch L;
      MST_TRY(build_plain(c, L, Operand{xj, rows, h, h, false}, Operand{wout, v, h, v, true}, dl, v,
                          mst::kEpiCeFwdNum, 0));
      ProblemDesc& P = L.p.prob[0];
      P.labels = labels + r0;
      P.part = part;
      P.ztarget = zt;
      P.nparts = nparts;
      P.ce_ref0 = rs ? 1 : 0;
      MST_TRY(launch(c, st, L));
    }
    const int threads = 256;
    if (rs) {  // row-scaled head: rowf (into zt) and the label column; K6 reads (rowf * X_j)^T
      ce_combine_rowscale_kernel<<<(unsigned)cdiv(rows * 32, threads), threads, 0, st>>>(
          part, nparts, zt, labels + r0, (int)rows, (int)v, lse + r0, lrow, stats + 3, static_cast<uint16_t*>(dl), v,
          scales + j);
      chunk_reduce_kernel<<<1, 1024, 0, st>>>(lrow, labels + r0, (int)rows, (int)v, stats + 4 + j,
                                              stats + 4 + nch + j);
      c->launches += 2;
      MST_TRY(transpose_bf16(c, st, xj, h, ot, ldt, rows, h, zt));
    } else {
      ce_combine_kernel<<<(unsigned)cdiv(rows * 32, threads), threads, 0, st>>>(part, nparts, zt, labels + r0,
                                                                                 (int)rows, (int)v, lse + r0, lrow,
                                                                                 stats + 3);
      chunk_reduce_kernel<<<1, 1024, 0, st>>>(lrow, labels + r0, (int)rows, (int)v, stats + 4 + j,
                                              stats + 4 + nch + j);
      normalize_dlogits_kernel<<<(unsigned)cdiv(rows * (v / 8), 256), 256, 0, st>>>(
          static_cast<uint16_t*>(dl), v, (int)rows, (int)v, part, nparts, lse + r0, labels + r0, scales + j, zt);
      c->launches += 3;
    }
    {  // K5 (dX = dl W_out^T) + K6 (dW_out += X^T dl), grouped.
      Launch L;
      MST_TRY(build_plain(c, L, Operand{dl, rows, v, v, false}, Operand{wout, h, v, v, false},
                          const_cast<char*>(bptr(dx, r0 * h)), h, mst::kEpiStoreBf16, 0));
      if (rs) L.p.prob[0].rowscale = zt;
      MST_TRY(build_plain(c, L, Operand{ot, h, rows, ldt, false}, Operand{dl, v, rows, v, true}, dwout, v,
                          mst::kEpiAccF32, beta));
      MST_TRY(launch(c, st, L));
    }
    mem_free(c, (uint64_t)rows * v * 2, "inter.head.dlogits");
    mem_free(c, part_bytes, "inter.head.partials");
    mem_free(c, (uint64_t)rows * h * 2, "act.xT");
  }
  finalize_loss_kernel<<<1, 32, 0, st>>>(stats, nch, loss_mode, c->err_dev, global_valid);
  c->launches += 1;
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

// Non-finite scan (NaN/Inf is an error surfaced, not propagated):
// counts elements whose exponent field is all ones, 16 bytes per thread and
// iteration, grid-stride over the whole buffer; HBM-bound.
__global__ void __launch_bounds__(256) nonfinite_count_kernel(const uint8_t* head, int head_bytes,
                                                              const uint4* __restrict__ p, int64_t n16, const uint8_t* tail,
                                                              int tail_bytes, int f32, unsigned int* __restrict__ out) {
  unsigned int bad = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n16; k += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = __ldcs(p + k);
    const uint32_t q[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (f32) {
        bad += (q[j] & 0x7f800000u) == 0x7f800000u;
      } else {
        bad += (q[j] & 0x7f80u) == 0x7f80u;
        bad += (q[j] & 0x7f800000u) == 0x7f800000u;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 2) {  // unaligned leading / trailing bytes (< 16 each)
    const uint8_t* q = threadIdx.x ? tail : head;
    const int nb = threadIdx.x ? tail_bytes : head_bytes;
    for (int b = 0; b + (f32 ? 4 : 2) <= nb; b += f32 ? 4 : 2) {
      uint32_t v = f32 ? *reinterpret_cast<const uint32_t*>(q + b) : *reinterpret_cast<const uint16_t*>(q + b);
      bad += f32 ? ((v & 0x7f800000u) == 0x7f800000u) : ((v & 0x7f80u) == 0x7f80u);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, bad);
}

int mst_count_nonfinite(mst_ctx* c, void* stream, const void* data, int64_t n, int dtype, unsigned int* count) {
  MST_CALL(c, stream);
  if (!data || !count) return fail(MST_ERR_CONFIG, "NULL pointer");
  if (n < 0) return fail(MST_ERR_SHAPE, "negative element count");
  if (dtype != MST_DTYPE_BF16 && dtype != MST_DTYPE_F32) return fail(MST_ERR_DTYPE, "dtype must be bf16 or f32");
  const int esz = dtype == MST_DTYPE_F32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(data) & (esz - 1)) != 0) return fail(MST_ERR_CONFIG, "misaligned element buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MST_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned int), st));
  const uint8_t* base = static_cast<const uint8_t*>(data);
  const int64_t bytes = n * esz;
  const int64_t head = std::min<int64_t>(bytes, (16 - (reinterpret_cast<uintptr_t>(base) & 15)) & 15);
  const int64_t n16 = (bytes - head) / 16;
  const int64_t tail = bytes - head - n16 * 16;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n16, 256), 4LL * c->num_sms));
  nonfinite_count_kernel<<<blocks, 256, 0, st>>>(base, (int)head, reinterpret_cast<const uint4*>(base + head), n16,
                                                   base + head + n16 * 16, (int)tail, dtype == MST_DTYPE_F32, count);
  c->launches++;
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

int mst_count_valid(mst_ctx* c, void* stream, const int32_t* labels, int64_t n, int64_t v, double* out) {
  MST_CALL(c, stream);
  if (!labels || !out) return fail(MST_ERR_CONFIG, "NULL pointer");
  if (n <= 0) return fail(MST_ERR_DATA, "N must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  count_valid_kernel<<<1, 1024, 0, st>>>(labels, n, (int)v, out);
  c->launches += 1;
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

// Chunk-wise block schedule (block_step when M_mlp == M_head).  With the
// single-pass head, chunk j of the LM-Head needs only O_j, so each chunk
// runs MLP forward -> head forward+backward -> MLP backward.  The forward's
// fp32 G, U accumulators are kept for the chunk's backward, so the
// backward's G,U recompute GEMM becomes an elementwise pass (bitwise the
// same values: same tiles, same K order).  K8/K9/K10 of chunk j-1 share a
// launch with K2 of chunk j.  Chunk buffers of both blocks coexist (peak
// intermediate = one MLP chunk + one head chunk).
// Host-resident X / dX for the chunk-wise block (mst_block_step_host): X_j is
// copied in on the context's copy stream into one of two device chunk
// buffers while earlier chunks compute, dX_j is copied out as soon as its
// GEMM (K9, in chunk j+1's K2 launch) has run.  Events: x_ready / x_free /
// dx_ready / dx_free per buffer, plus `done` joining the copies back into
// the compute stream.
struct HostIO {
  const char* x_host;
  char* dx_host;
  void* xbuf[2];
  void* dxbuf[2];
  cudaStream_t cs;
  cudaEvent_t x_ready[2], x_free[2], dx_ready[2], dx_free[2], done;
};

static size_t host_io_bytes(int64_t n, int64_t h, int64_t m) {  // 2 X + 2 dX chunk buffers, labels, alignment
  return 4 * align_up(size_t(max_chunk(n, m)) * h * 2, 256) + align_up(size_t(n) * 4, 256) + 2048;
}

static int block_step_chunked(mst_ctx* c, cudaStream_t st, const void* x, const int32_t* labels, const void* wg,
                              const void* wu, const void* wd, const void* wout, int64_t n, int64_t h, int64_t i,
                              int64_t v, int64_t m, int64_t mh, int loss_mode, float grad_loss, float* stats, void* dx, float* dwg,
                              float* dwu, float* dwd, float* dwout, int accumulate, void* ws, size_t ws_bytes,
                              const double* global_valid, const HostIO* io = nullptr) {
  char* base = static_cast<char*>(ws);
  // O_j is consumed within chunk j; dO_j also by chunk j's dW_down GEMM,
  // which runs in chunk j+1's K2 launch: one O chunk, two dO chunks.
  const size_t ocb = align_up(size_t(max_chunk(n, m)) * h * 2, 256);
  void* o = base;
  void* dO[2] = {base + ocb, base + 2 * ocb};
  float* lse = reinterpret_cast<float*>(base + 3 * ocb);
  Carve cv{base + chunked_fixed_bytes(n, h, m) + 256, ws_bytes, 0, false};
  void *hb, *dg, *du, *xt, *ht, *dl, *ot;
  float *dhb, *zt, *lrow, *scales;
  float2* part;
  carve_mlp(cv, n, h, i, m, &hb, &dg, &du, &dhb, &xt, &ht);
  carve_head(cv, n, h, v, mh, &part, &zt, &lrow, &dl, &scales, &ot);
  float* g32 = static_cast<float*>(cv.take(size_t(max_chunk(n, m)) * i * 4));
  float* u32 = static_cast<float*>(cv.take(size_t(max_chunk(n, m)) * i * 4));
  const int64_t ldt = ld_t(n, m), ldt_h = ld_t(n, mh);
  const std::vector<int64_t> b = plan_bounds(n, m);
  const int nch = (int)b.size() - 1;
  // dW operand sets {dG, dU, h^T, X^T}: chunk j uses set j & 1 when K8 / K10
  // run per chunk pair (pair_dw), else set 0.
  const bool pair = c->pair_dw != 0 && nch > 1;
  const bool k9k1 = c->k9_in_k1 != 0;
  void *dgS[2] = {dg, dg}, *duS[2] = {du, du}, *htS[2] = {ht, ht}, *xtS[2] = {xt, xt};
  if (pair) {
    const int64_t nc = max_chunk(n, m);
    dgS[1] = cv.take(size_t(nc) * i * 2);
    duS[1] = cv.take(size_t(nc) * i * 2);
    htS[1] = cv.take(size_t(i) * ldt * 2);
    xtS[1] = cv.take(size_t(h) * ldt * 2);
  }
  auto set_of = [&](int j) { return pair ? (j & 1) : 0; };
  // Head plan: refines the MLP plan (plans_nest), head chunks hc0[j] ..
  // hc0[j+1]-1 lie inside MLP chunk j.
  const std::vector<int64_t> bh = plan_bounds(n, mh);
  const int nch_h = (int)bh.size() - 1;
  std::vector<int> hc0(nch + 1, 0);
  for (int j = 0, k = 0; j <= nch; ++j) {
    while (k < nch_h && bh[k] < b[j]) ++k;
    hc0[j] = k;
  }
  hc0[nch] = nch_h;
  const int nparts = (int)cdiv(v, 256);
  // dlogits scales depend only on the labels: compute them up front.
  MST_CUDA(cudaMemsetAsync(stats, 0, sizeof(float) * MST_STATS_LEN(nch_h), st));
  chunk_valid_kernel<<<nch_h, 256, 0, st>>>(labels, n, nch_h, (int)v, stats);
  double* tot = reinterpret_cast<double*>(c->scratch_dev + 64);  // context scratch (calls are serialised)
  sum_valid_kernel<<<1, 32, 0, st>>>(stats, nch_h, tot);
  // a sequence-parallel caller's global_valid is the all-reduced token count
  grad_scale_kernel<<<(nch_h + 255) / 256, 256, 0, st>>>(global_valid ? global_valid : tot, nullptr, stats, nch_h,
                                                        loss_mode, grad_loss, scales);
  c->launches += 3;
  WeightScope ws_(c, wg, wu, wd, wout);
  const uint64_t act_bytes = (uint64_t)max_chunk(n, m) * h * 2;  // one chunk of O, two of dO
  mem_alloc(c, act_bytes, "act.O");
  mem_alloc(c, 2 * act_bytes, "act.dO");
  mem_alloc(c, (uint64_t)n * 4, "act.lse");
  auto rows_of = [&](int j) { return b[j + 1] - b[j]; };
  // Logical lifetimes of the chunk buffers (MemTracker events, mst.h).
  auto mlp_fwd_live = [&](int j, bool on) {  // h (bf16), G and U (fp32) of chunk j
    const uint64_t r = (uint64_t)rows_of(j);
    auto f = on ? mem_alloc : mem_free;
    f(c, r * i * 2, "inter.mlp.h");
    f(c, r * i * 4, "inter.mlp.G");
    f(c, r * i * 4, "inter.mlp.U");
  };
  auto grads_live = [&](int j, bool on) {  // dG, dU, h^T, X^T of chunk j (until K8-K10 ran)
    const uint64_t r = (uint64_t)rows_of(j);
    auto f = on ? mem_alloc : mem_free;
    f(c, r * i * 2, "inter.mlp.dG");
    f(c, r * i * 2, "inter.mlp.dU");
    f(c, r * i * 2, "inter.mlp.hT");
    f(c, r * h * 2, "act.xT");
  };
  // X_j / dX_j: rows of the caller's device tensors, or the streamed chunk buffers
  auto xdev = [&](int j) -> const void* { return io ? io->xbuf[j & 1] : bptr(x, b[j] * h); };
  auto dxdev = [&](int j) -> void* { return io ? io->dxbuf[j & 1] : const_cast<char*>(bptr(dx, b[j] * h)); };
  auto h2d = [&](int j) -> int {  // X_j into buffer j & 1 once chunk j-2 has released it
    MST_CUDA(cudaStreamWaitEvent(io->cs, io->x_free[j & 1], 0));
    MST_CUDA(cudaMemcpyAsync(io->xbuf[j & 1], io->x_host + b[j] * h * 2, size_t(rows_of(j)) * h * 2,
                             cudaMemcpyHostToDevice, io->cs));
    MST_CUDA(cudaEventRecord(io->x_ready[j & 1], io->cs));
    return MST_OK;
  };
  auto d2h = [&](int j) -> int {  // dX_j out once its GEMM has run
    MST_CUDA(cudaEventRecord(io->dx_ready[j & 1], st));
    MST_CUDA(cudaStreamWaitEvent(io->cs, io->dx_ready[j & 1], 0));
    MST_CUDA(cudaMemcpyAsync(io->dx_host + b[j] * h * 2, io->dxbuf[j & 1], size_t(rows_of(j)) * h * 2,
                             cudaMemcpyDeviceToHost, io->cs));
    MST_CUDA(cudaEventRecord(io->dx_free[j & 1], io->cs));
    return MST_OK;
  };
  if (io) {
    MST_TRY(h2d(0));
    if (nch > 1) MST_TRY(h2d(1));
  }
  auto add_k1s = [&](Launch& L, int j) -> int {  // K1 saving G, U (fp32) and h (bf16)
    const int64_t rows = rows_of(j);
    if (io) MST_CUDA(cudaStreamWaitEvent(st, io->x_ready[j & 1], 0));
    ProblemDesc& P = L.p.prob[L.p.num_problems++];
    P.nblk = (c->wide_mask & 32) ? 2 : 1;
    PhaseSpec s{};
    s.a = {xdev(j), rows, h, h, false};
    s.b0 = {wg, i, h, i, true};
    s.b1 = {wu, i, h, i, true};
    s.umma_n = 256;
    MST_TRY(add_phase(c, L, P, s));
    mlp_fwd_live(j, true);
    cnt_mm(c, rows, h, i, (uint64_t)(h * i));     // G = X_j W_g
    cnt_mm(c, rows, h, i, (uint64_t)(h * i));     // U = X_j W_u
    cnt_op(c, 4ull * rows * i, 2ull * rows * i);  // silu
    cnt_op(c, 1ull * rows * i, 3ull * rows * i);  // hadamard
    P.m_tiles = (int)cdiv(rows, 256);
    P.tile_n = 128;
    P.n_tiles = (int)cdiv(i, 128);
    P.rows = (int)rows;
    P.cols = (int)i;
    P.epi = mst::kEpiSwigluSave;
    MST_TRY(add_out_map(c, L, hb, i, rows, i, false, &P.map_out0));
    MST_TRY(add_out_map(c, L, g32, i, rows, i, true, &P.map_out1, false));
    MST_TRY(add_out_map(c, L, u32, i, rows, i, true, &P.map_out2, false));
    L.flops += 2.0 * rows * (2.0 * i) * h;
    return MST_OK;
  };
  bool mlp_grads_alloced = false;
  auto alloc_mlp_grads = [&]() {
    if (mlp_grads_alloced) return;
    mlp_grads_alloced = true;
    for (int wi = 0; wi < 3; ++wi) grad_alloc(c, wi, (uint64_t)h * i * 4);
  };
  // K9 (dX_j) of chunk j
  auto add_k9 = [&](Launch& L, int j) -> int {
    alloc_mlp_grads();
    const int s = set_of(j);
    if (io) MST_CUDA(cudaStreamWaitEvent(st, io->dx_free[j & 1], 0));  // dX of chunk j-2 out
    return add_mlp_grads(c, L, dgS[s], duS[s], htS[s], xtS[s], dO[j & 1], wg, wu, dxdev(j), dwg, dwu, dwd,
                         rows_of(j), h, i, ldt, 0, kGradK9);
  };
  // K8 / K10 of chunk j, or of chunks j and j + 1 as one accumulation
  auto add_dw = [&](Launch& L, int j, bool paired, int parts = kGradDW, int64_t k10_r0 = 0,
                    int64_t k10_r1 = -1) -> int {
    alloc_mlp_grads();
    const int s = set_of(j);
    const int beta = (j > 0 || accumulate) ? 1 : 0;
    DwChunk second{};
    if (paired) {
      const int s2 = set_of(j + 1);
      second = DwChunk{dgS[s2], duS[s2], htS[s2], xtS[s2], dO[(j + 1) & 1], rows_of(j + 1)};
    }
    return add_mlp_grads(c, L, dgS[s], duS[s], htS[s], xtS[s], dO[j & 1], wg, wu, nullptr, dwg, dwu, dwd,
                         rows_of(j), h, i, ldt, beta, parts, k10_r0, k10_r1, paired ? &second : nullptr);
  };
  {
    Launch L;
    MST_TRY(add_k1s(L, 0));
    MST_TRY(launch(c, st, L));
  }
  for (int j = 0; j < nch; ++j) {
    const int64_t r0 = b[j], rows = rows_of(j);
    void* oj = o;
    void* doj = dO[j & 1];
    {  // K2(j) + the weight/input gradients of chunk j-1 (or of chunks j-2, j-1)
      Launch L;
      MST_TRY(build_plain(c, L, Operand{hb, rows, i, i, false}, Operand{wd, h, i, h, true}, oj, h, mst::kEpiStoreBf16,
                          0, (c->wide_mask & 4) ? 2 : 1));
      int freed0 = -1, freed1 = -1;
      if (j > 0) {
        if (!k9k1) MST_TRY(add_k9(L, j - 1));
        if (!pair) {
          MST_TRY(add_dw(L, j - 1, false));
          freed0 = j - 1;
        } else if ((j - 1) & 1) {  // chunk j-1 closes the pair (j-2, j-1)
          MST_TRY(add_dw(L, j - 2, true));
          freed0 = j - 2;
          freed1 = j - 1;
        }
      }
      MST_TRY(launch(c, st, L));
      if (freed0 >= 0) grads_live(freed0, false);
      if (freed1 >= 0) grads_live(freed1, false);
      if (io && j > 0 && !k9k1) MST_TRY(d2h(j - 1));
    }
    if (j == 0) grad_alloc(c, 3, (uint64_t)h * v * 4);
    for (int k = hc0[j]; k < hc0[j + 1]; ++k) {  // the head chunks of MLP chunk j
      const int64_t hr0 = bh[k], hrows = bh[k + 1] - bh[k];
      const int hbeta = (k > 0 || accumulate) ? 1 : 0;
      void* ok = const_cast<char*>(bptr(oj, (hr0 - r0) * h));
      void* dok = const_cast<char*>(bptr(doj, (hr0 - r0) * h));
      const uint64_t part_bytes = (uint64_t)hrows * nparts * 8 + (uint64_t)hrows * 8;
      mem_alloc(c, (uint64_t)hrows * h * 2, "act.oT");
      mem_alloc(c, part_bytes, "inter.head.partials");
      mem_alloc(c, (uint64_t)hrows * v * 2, "inter.head.dlogits");
      cnt_op(c, 5ull * hrows * v, (uint64_t)(hrows * v + 2 * hrows));      // cross-entropy forward
      cnt_op(c, 5ull * hrows * v, (uint64_t)(2 * hrows * v + 2 * hrows));  // cross-entropy backward
      const bool rs = c->dl_rowscale != 0;
      if (!rs) MST_TRY(transpose_bf16(c, st, ok, h, ot, ldt_h, hrows, h));
      {  // K3': logits GEMM, partials + softmax numerators
        Launch L;
        MST_TRY(build_plain(c, L, Operand{ok, hrows, h, h, false}, Operand{wout, v, h, v, true}, dl, v,
                            mst::kEpiCeFwdNum, 0, (c->wide_mask & 1) ? 2 : 1));
        ProblemDesc& P = L.p.prob[0];
        P.labels = labels + hr0;
        P.part = part;
        P.ztarget = zt;
        P.nparts = nparts;
        P.ce_ref0 = rs ? 1 : 0;
        MST_TRY(launch(c, st, L));
      }
      if (rs) {  // LSE + per-row factor rowf (into zt) + label column; then (rowf * O_k)^T for K6
        ce_combine_rowscale_kernel<<<(unsigned)cdiv(hrows * 32, 256), 256, 0, st>>>(
            part, nparts, zt, labels + hr0, (int)hrows, (int)v, lse + hr0, lrow, stats + 3,
            static_cast<uint16_t*>(dl), v, scales + k);
        chunk_reduce_kernel<<<1, 1024, 0, st>>>(lrow, labels + hr0, (int)hrows, (int)v, stats + 4 + k,
                                                stats + 4 + nch_h + k);
        c->launches += 2;
        MST_TRY(transpose_bf16(c, st, ok, h, ot, ldt_h, hrows, h, zt));
      } else {
        ce_combine_kernel<<<(unsigned)cdiv(hrows * 32, 256), 256, 0, st>>>(part, nparts, zt, labels + hr0, (int)hrows,
                                                                          (int)v, lse + hr0, lrow, stats + 3);
        chunk_reduce_kernel<<<1, 1024, 0, st>>>(lrow, labels + hr0, (int)hrows, (int)v, stats + 4 + k,
                                                stats + 4 + nch_h + k);
        normalize_dlogits_kernel<<<(unsigned)cdiv(hrows * (v / 8), 256), 256, 0, st>>>(
            static_cast<uint16_t*>(dl), v, (int)hrows, (int)v, part, nparts, lse + hr0, labels + hr0, scales + k, zt);
        c->launches += 3;
      }
      // K5 + K6.  The last head chunk's K6 finalises dW_out: with a slab hook
      // it is cut into row slabs of H, one launch each (K5 rides in the
      // first), and each slab is handed to the hook as soon as it is enqueued.
      const bool last_head = k == nch_h - 1;
      const int64_t per = (last_head && c->slab_fn && c->slabs > 1) ? cdiv(cdiv(h, 256), c->slabs) * 256 : h;
      for (int64_t s0 = 0; s0 < h; s0 += per) {
        const int64_t s1 = std::min(h, s0 + per);
        Launch L;
        if (s0 == 0) {
          MST_TRY(build_plain(c, L, Operand{dl, hrows, v, v, false}, Operand{wout, h, v, v, false}, dok, h,
                              mst::kEpiStoreBf16, 0, (c->wide_mask & 2) ? 2 : 1));
          if (rs) L.p.prob[0].rowscale = zt;
        }
        MST_TRY(build_plain(c, L, Operand{bptr(ot, s0 * ldt_h), s1 - s0, hrows, ldt_h, false},
                            Operand{dl, v, hrows, v, true}, dwout + s0 * v, v, mst::kEpiAccF32, hbeta));
        MST_TRY(launch(c, st, L));
        if (last_head) grad_slab(c, 3, s0, s1, st);
      }
      if (last_head) grad_ready(c, 3, st, (uint64_t)h * v * 4);  // dW_out complete
      mem_free(c, (uint64_t)hrows * v * 2, "inter.head.dlogits");
      mem_free(c, part_bytes, "inter.head.partials");
      mem_free(c, (uint64_t)hrows * h * 2, "act.oT");
    }
    if (c->fuse_swiglu_bwd) {
      // K7a with the SwiGLU backward in its epilogue: dh = dO_j W_d^T stays in
      // TMEM; dG, dU come out directly (no dh round trip through HBM).
      grads_live(j, true);
      Launch L;
      MST_TRY(build_plain(c, L, Operand{doj, rows, h, h, false}, Operand{wd, i, h, h, false}, dgS[set_of(j)], i,
                          mst::kEpiStoreBf16, 0, (c->wide_mask & 16) ? 2 : 1));
      ProblemDesc& P = L.p.prob[0];
      P.epi = mst::kEpiDhSwigluBwd;
      P.aux = g32;
      P.aux2 = u32;
      P.ld_aux = i;
      MST_TRY(add_out_map(c, L, duS[set_of(j)], i, rows, i, false, &P.map_out1));
      MST_TRY(launch(c, st, L));
      cnt_op(c, 4ull * rows * i, 3ull * rows * i);  // silu_backward (fused epilogue)
      cnt_op(c, 2ull * rows * i, 6ull * rows * i);  // dG, dU products
    } else {
      mem_alloc(c, (uint64_t)rows * i * 4, "inter.mlp.dh");
      {  // K7a: dh = dO_j W_d^T (fp32)
        Launch L;
        MST_TRY(build_plain(c, L, Operand{doj, rows, h, h, false}, Operand{wd, i, h, h, false}, dhb, i,
                            mst::kEpiAccF32, 0, (c->wide_mask & 16) ? 2 : 1));
        MST_TRY(launch(c, st, L));
      }
      {  // SwiGLU backward from the saved accumulators
        const int64_t n4 = rows * i / 4;
        swiglu_bwd_kernel<<<(unsigned)cdiv(n4, 256), 256, 0, st>>>(
            g32, u32, dhb, static_cast<uint16_t*>(dgS[set_of(j)]), static_cast<uint16_t*>(duS[set_of(j)]), n4);
        c->launches += 1;
        cnt_op(c, 4ull * rows * i, 3ull * rows * i);  // silu_backward
        cnt_op(c, 2ull * rows * i, 6ull * rows * i);  // dG, dU products
      }
      grads_live(j, true);
      mem_free(c, (uint64_t)rows * i * 4, "inter.mlp.dh");
    }
    MST_TRY(transpose_bf16(c, st, hb, i, htS[set_of(j)], ldt, rows, i));
    MST_TRY(transpose_bf16(c, st, xdev(j), h, xtS[set_of(j)], ldt, rows, h));
    if (io) {  // last read of X_j: its buffer takes X_{j+2}
      MST_CUDA(cudaEventRecord(io->x_free[j & 1], st));
      if (j + 2 < nch) MST_TRY(h2d(j + 2));
    }
    mlp_fwd_live(j, false);
    if (j + 1 < nch) {  // K1(j+1) (+ K9(j))
      Launch L;
      MST_TRY(add_k1s(L, j + 1));
      if (k9k1) MST_TRY(add_k9(L, j));
      MST_TRY(launch(c, st, L));
      if (io && k9k1) MST_TRY(d2h(j));
    }
  }
  {  // the last chunk's K9 / K8 / K10 finalise dX and dW_{down,gate,up}; with a
     // slab hook K10 is cut into row slabs of H (K9 and K8 ride in the first)
    const int64_t per = (c->slab_fn && c->slabs > 1) ? cdiv(cdiv(h, 256), c->slabs) * 256 : h;
    const int last = nch - 1;
    const bool last_paired = pair && (last & 1);  // the pair (last-1, last)
    const int dw0 = last_paired ? last - 1 : last;
    if (io && per == h) {
      // Host-resident dX: K9 + K8 first, then K10 alone, so the last dX
      // chunk's D2H copy runs under the K10 launch instead of after the step.
      {
        Launch L;
        MST_TRY(add_k9(L, last));
        MST_TRY(add_dw(L, dw0, last_paired, kGradK8));
        MST_TRY(launch(c, st, L));
        grad_slab(c, 2, 0, i, st);
        MST_TRY(d2h(nch - 1));
      }
      Launch L;
      MST_TRY(add_dw(L, dw0, last_paired, kGradK10, 0, h));
      MST_TRY(launch(c, st, L));
      grad_slab(c, 0, 0, h, st);
      grad_slab(c, 1, 0, h, st);
    }
    for (int64_t s0 = 0; s0 < (io && per == h ? 0 : h); s0 += per) {
      const int64_t s1 = std::min(h, s0 + per);
      Launch L;
      if (s0 == 0) MST_TRY(add_k9(L, last));
      MST_TRY(add_dw(L, dw0, last_paired, s0 == 0 ? kGradDW : kGradK10, s0, s1));
      MST_TRY(launch(c, st, L));
      if (s0 == 0) {
        grad_slab(c, 2, 0, i, st);
        if (io) MST_TRY(d2h(nch - 1));  // the last dX chunk out
      }
      grad_slab(c, 0, s0, s1, st);
      grad_slab(c, 1, s0, s1, st);
    }
    if (last_paired) grads_live(last - 1, false);
    grads_live(last, false);
    if (io) {  // the compute stream joins the copies
      MST_CUDA(cudaEventRecord(io->done, io->cs));
      MST_CUDA(cudaStreamWaitEvent(st, io->done, 0));
    }
  }
  for (int wi = 0; wi < 3; ++wi) grad_ready(c, wi, st, (uint64_t)h * i * 4);  // dW_gate, dW_up, dW_down complete
  mem_free(c, (uint64_t)n * 4, "act.lse");
  mem_free(c, 2 * act_bytes, "act.dO");
  mem_free(c, act_bytes, "act.O");
  finalize_loss_kernel<<<1, 32, 0, st>>>(stats, nch_h, loss_mode, c->err_dev, global_valid);
  c->launches += 1;
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

int mst_ctx_block_host_workspace(const mst_ctx* c, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m,
                                 size_t* bytes) {
  if (!c || !bytes) return fail(MST_ERR_STATE, "NULL context or output");
  if (!uses_chunked_block(c, n, m, m))
    return fail(MST_ERR_CONFIG, "host-resident X / dX need the chunk-wise schedule (tuning chunked_block=1, fused_head=1)");
  MST_TRY(mst_ctx_block_workspace(c, n, h, i, v, m, m, bytes));  // the chunk IO buffers are the context's own
  return MST_OK;
}

int mst_block_step_host(mst_ctx* c, void* stream, const void* x_host, const int32_t* labels_host, const void* wg,
                        const void* wu, const void* wd, const void* wout, int64_t n, int64_t h, int64_t i, int64_t v,
                        int64_t m, int loss_mode, float grad_loss, float* stats, void* dx_host, float* dwg, float* dwu,
                        float* dwd, float* dwout, int accumulate, void* ws, size_t ws_bytes) {
  MST_CALL(c, stream);
  size_t need = 0, dev_need = 0;
  MST_TRY(mst_ctx_block_host_workspace(c, n, h, i, v, m, &need));
  MST_TRY(mst_ctx_block_workspace(c, n, h, i, v, m, m, &dev_need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  if (loss_mode != MST_LOSS_TOKEN_WEIGHTED && loss_mode != MST_LOSS_PAPER_MEAN)
    return fail(MST_ERR_CONFIG, "unknown loss mode %d", loss_mode);
  if (!x_host || !labels_host || !wg || !wu || !wd || !wout || !stats || !dx_host || !dwg || !dwu || !dwd || !dwout)
    return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  MST_TRY(check_dims(n, h, i, m, "I"));
  MST_TRY(check_dims(n, h, v, m, "V"));
  if (!c->copy_stream) {
    MST_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : c->io_ev) MST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t io_need = host_io_bytes(n, h, m);
  if (c->io_bytes < io_need) {  // grow (rare): everything that used the old buffers has finished
    MST_CUDA(cudaDeviceSynchronize());
    if (c->io_dev) MST_CUDA(cudaFree(c->io_dev));
    c->io_dev = nullptr;
    c->io_bytes = 0;
    if (cudaMalloc(&c->io_dev, io_need) != cudaSuccess) {
      cudaGetLastError();
      return fail(MST_ERR_CONFIG, "cannot allocate %zu bytes of host-streaming chunk buffers", io_need);
    }
    c->io_bytes = io_need;
  }
  char* io_base = static_cast<char*>(c->io_dev);
  const size_t xcb = align_up(size_t(max_chunk(n, m)) * h * 2, 256);
  HostIO io{static_cast<const char*>(x_host), static_cast<char*>(dx_host),
            {io_base, io_base + xcb}, {io_base + 2 * xcb, io_base + 3 * xcb}, c->copy_stream,
            {c->io_ev[0], c->io_ev[1]}, {c->io_ev[2], c->io_ev[3]}, {c->io_ev[4], c->io_ev[5]},
            {c->io_ev[6], c->io_ev[7]}, c->io_ev[8]};
  int32_t* labels_dev = reinterpret_cast<int32_t*>(io_base + 4 * xcb);
  // The copy stream only writes the context's own X / dX chunk buffers, whose
  // previous uses are ordered by the chunk events of the previous call
  // (x_free, dx_ready / dx_free): no wait for the whole compute stream, so
  // X_0 of this step is copied while the previous step still runs.  The
  // labels go in order on the compute stream.
  MST_CUDA(cudaMemcpyAsync(labels_dev, labels_host, size_t(n) * 4, cudaMemcpyHostToDevice, st));
  return block_step_chunked(c, st, nullptr, labels_dev, wg, wu, wd, wout, n, h, i, v, m, m, loss_mode, grad_loss, stats,
                            nullptr, dwg, dwu, dwd, dwout, accumulate, ws, dev_need, nullptr, &io);
}

int mst_block_step(mst_ctx* c, void* stream, const void* x, const int32_t* labels, const void* wg, const void* wu,
                   const void* wd, const void* wout, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp,
                   int64_t m_head, int loss_mode, float grad_loss, float* stats, void* dx, float* dwg, float* dwu,
                   float* dwd, float* dwout, int accumulate, void* ws, size_t ws_bytes) {
  return mst_block_step_sp(c, stream, x, labels, wg, wu, wd, wout, n, h, i, v, m_mlp, m_head, loss_mode, grad_loss,
                           stats, dx, dwg, dwu, dwd, dwout, accumulate, ws, ws_bytes, nullptr);
}

int mst_block_step_sp(mst_ctx* c, void* stream, const void* x, const int32_t* labels, const void* wg, const void* wu,
                      const void* wd, const void* wout, int64_t n, int64_t h, int64_t i, int64_t v, int64_t m_mlp,
                      int64_t m_head, int loss_mode, float grad_loss, float* stats, void* dx, float* dwg, float* dwu,
                      float* dwd, float* dwout, int accumulate, void* ws, size_t ws_bytes, const double* global_valid) {
  MST_CALL(c, stream);
  size_t need = 0;
  MST_TRY(mst_ctx_block_workspace(c, n, h, i, v, m_mlp, m_head, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  if (loss_mode != MST_LOSS_TOKEN_WEIGHTED && loss_mode != MST_LOSS_PAPER_MEAN)
    return fail(MST_ERR_CONFIG, "unknown loss mode %d", loss_mode);
  if (!x || !labels || !wg || !wu || !wd || !wout || !stats || !dx || !dwg || !dwu || !dwd || !dwout)
    return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  if (uses_chunked_block(c, n, m_mlp, m_head))
    return block_step_chunked(c, static_cast<cudaStream_t>(stream), x, labels, wg, wu, wd, wout, n, h, i, v, m_mlp,
                              m_head, loss_mode, grad_loss, stats, dx, dwg, dwu, dwd, dwout, accumulate, ws, ws_bytes,
                              global_valid);
  char* base = static_cast<char*>(ws);
  const size_t ob = align_up(size_t(n) * h * 2, 256);
  void* o = base;
  void* dO = base + ob;
  float* lse = reinterpret_cast<float*>(base + 2 * ob);
  const size_t fixed = block_fixed_bytes(n, h) + 256;
  void* rest = base + fixed;
  const size_t rest_bytes = ws_bytes - fixed;
  mst_mlp_saved ms;
  mst_lmhead_saved hs;
  MST_TRY(mst_mlp_forward(c, stream, x, wg, wu, wd, o, n, h, i, m_mlp, rest, rest_bytes, &ms));
  grad_alloc(c, 3, (uint64_t)h * v * 4);
  if (c->fused_head) {
    MST_TRY(mst_lmhead_fused(c, stream, o, labels, wout, n, h, v, m_head, loss_mode, grad_loss, global_valid, stats, lse,
                             dO, dwout, accumulate, rest, rest_bytes));
  } else {
    if (global_valid) return fail(MST_ERR_CONFIG, "global_valid needs the fused LM-Head (tuning fused_head=1)");
    MST_TRY(mst_lmhead_forward(c, stream, o, labels, wout, n, h, v, m_head, loss_mode, stats, lse, rest, rest_bytes,
                               &hs));
    MST_TRY(mst_lmhead_backward(c, stream, &hs, wout, stats, grad_loss, dO, dwout, accumulate, rest, rest_bytes));
  }
  grad_slab(c, 3, 0, h, static_cast<cudaStream_t>(stream));
  grad_ready(c, 3, static_cast<cudaStream_t>(stream), (uint64_t)h * v * 4);
  for (int wi = 0; wi < 3; ++wi) grad_alloc(c, wi, (uint64_t)h * i * 4);
  MST_TRY(mst_mlp_backward(c, stream, dO, &ms, wg, wu, wd, dx, dwg, dwu, dwd, accumulate, rest, rest_bytes));
  grad_slab(c, 2, 0, i, static_cast<cudaStream_t>(stream));
  grad_slab(c, 0, 0, h, static_cast<cudaStream_t>(stream));
  grad_slab(c, 1, 0, h, static_cast<cudaStream_t>(stream));
  for (int wi = 0; wi < 3; ++wi) grad_ready(c, wi, static_cast<cudaStream_t>(stream), (uint64_t)h * i * 4);
  return MST_OK;
}

// ------------------------------------------------------------ decoder-layer ops (layers.cu)
int mst_gemm(mst_ctx* c, void* stream, const void* a, const void* b, void* out, int64_t m, int64_t n, int64_t k,
             int a_mn, int b_mn, int out_f32, int beta) {
  return mst_debug_gemm(c, stream, a, b, out, m, n, k, a_mn, b_mn, out_f32, beta);
}

static int check_rows(int64_t n, int64_t d) {
  if (n <= 0 || d <= 0) return fail(MST_ERR_SHAPE, "extents must be positive (n=%lld d=%lld)", (long long)n, (long long)d);
  if (d % 8) return fail(MST_ERR_SHAPE, "hidden size must be a multiple of 8 (d=%lld)", (long long)d);
  if (d > 16384) return fail(MST_ERR_BOUNDS, "hidden size %lld > 16384", (long long)d);
  return MST_OK;
}

int mst_rmsnorm_forward(mst_ctx* c, void* stream, const void* x, const void* residual, const float* gain, void* y,
                        void* sum_out, float* rstd, int64_t n, int64_t d, float eps) {
  MST_CALL(c, stream);
  MST_TRY(check_rows(n, d));
  if (!x || !gain || !y || !rstd || (residual && !sum_out)) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  if (!(eps > 0.f)) return fail(MST_ERR_CONFIG, "eps must be > 0");
  MST_CUDA(mst_layers::rmsnorm_fwd(static_cast<cudaStream_t>(stream), c->num_sms, x, residual, gain, y, sum_out, rstd, n,
                                   (int)d, eps));
  c->launches++;
  cnt_op(c, 4ull * n * d, 2ull * n * d);  // rmsnorm fwd (memtrack.hpp:30)
  if (residual) cnt_op(c, 1ull * n * d, 3ull * n * d);
  return MST_OK;
}

int mst_rmsnorm_workspace(const mst_ctx* c, int64_t n, int64_t d, size_t* bytes) {
  if (!c || !bytes) return fail(MST_ERR_STATE, "NULL context or output");
  MST_TRY(check_rows(n, d));
  *bytes = sizeof(float) * (size_t)mst_layers::rmsnorm_bwd_parts(n, c->num_sms) * (size_t)d;
  return MST_OK;
}

int mst_rmsnorm_backward(mst_ctx* c, void* stream, const void* s, const float* gain, const float* rstd, const void* dy,
                         const void* dres, void* dx, float* dgain, int accumulate, int64_t n, int64_t d, void* ws,
                         size_t ws_bytes) {
  MST_CALL(c, stream);
  MST_TRY(check_rows(n, d));
  if (!s || !gain || !rstd || !dy || !dx || !dgain) return fail(MST_ERR_CONFIG, "NULL tensor pointer");
  if (d > 6144) return fail(MST_ERR_BOUNDS, "rmsnorm backward supports d <= 6144 (per-warp dgain rows in smem)");
  size_t need = 0;
  MST_TRY(mst_rmsnorm_workspace(c, n, d, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  MST_CUDA(mst_layers::rmsnorm_bwd(static_cast<cudaStream_t>(stream), c->num_sms, s, gain, rstd, dy, dres, dx,
                                   static_cast<float*>(ws), dgain, accumulate, n, (int)d));
  c->launches += 2;
  cnt_op(c, 8ull * n * d, 4ull * n * d);  // rmsnorm bwd (memtrack.hpp:30)
  return MST_OK;
}

int mst_embedding_forward(mst_ctx* c, void* stream, const void* table, const int32_t* tokens, void* out, int64_t n,
                          int64_t d, int64_t vocab, int* bad_count) {
  MST_CALL(c, stream);
  MST_TRY(check_rows(n, d));
  if (vocab <= 0) return fail(MST_ERR_SHAPE, "vocabulary must be >= 1");
  if (!table || !tokens || !out || !bad_count) return fail(MST_ERR_CONFIG, "NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MST_CUDA(cudaMemsetAsync(bad_count, 0, sizeof(int), st));
  MST_CUDA(mst_layers::embed_fwd(st, c->num_sms, table, tokens, out, n, (int)d, vocab, bad_count));
  c->launches++;
  cnt_op(c, 0, 2ull * n * d);
  return MST_OK;
}

int mst_embedding_backward(mst_ctx* c, void* stream, const int32_t* order, const int32_t* seg, const int32_t* uniq,
                           int64_t nseg, const void* dx, float* dtable, int64_t d, int64_t vocab, int accumulate) {
  MST_CALL(c, stream);
  if (d <= 0 || d % 8 || vocab <= 0 || nseg < 0) return fail(MST_ERR_SHAPE, "bad embedding extents");
  if (nseg > 0 && (!order || !seg || !uniq || !dx)) return fail(MST_ERR_CONFIG, "NULL pointer");
  if (!dtable) return fail(MST_ERR_CONFIG, "NULL gradient table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!accumulate) MST_CUDA(cudaMemsetAsync(dtable, 0, sizeof(float) * (size_t)vocab * (size_t)d, st));
  MST_CUDA(mst_layers::embed_bwd(st, c->num_sms, order, seg, uniq, (int)nseg, dx, dtable, (int)d, 1));
  c->launches++;
  return MST_OK;
}

// ------------------------------------------------------------ attention (attention.cu)
static int check_attn(const void* const* ptrs, const int64_t* lds, int n, int64_t batch, int64_t seq, int64_t heads,
                      int64_t kvh, int64_t hd, int causal) {
  if (batch < 1 || seq < 1 || heads < 1 || kvh < 1) return fail(MST_ERR_SHAPE, "attention extents must be >= 1");
  if (heads % kvh) return fail(MST_ERR_CONFIG, "heads (%lld) must be a multiple of kv_heads (%lld)", (long long)heads,
                               (long long)kvh);
  if (hd < 8 || hd > 128 || hd % 8)
    return fail(MST_ERR_SHAPE, "head_dim must be a multiple of 8 in [8, 128], got %lld", (long long)hd);
  if (!causal) return fail(MST_ERR_CONFIG, "only causal attention is implemented (SPEC.md:235)");
  if (batch * seq > (int64_t(1) << 31) || batch * heads * seq > (int64_t(1) << 40))
    return fail(MST_ERR_BOUNDS, "attention problem too large");
  for (int i = 0; i < n; ++i) {
    if (!ptrs[i]) return fail(MST_ERR_CONFIG, "NULL attention tensor");
    if ((reinterpret_cast<uintptr_t>(ptrs[i]) & 15) || lds[i] % 8)
      return fail(MST_ERR_CONFIG, "attention tensors need 16-byte aligned rows (ld %% 8 == 0)");
  }
  return MST_OK;
}

int mst_attention_forward(mst_ctx* c, void* stream, const void* q, int64_t ldq, const void* k, int64_t ldk,
                          const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, int64_t batch, int64_t seq,
                          int64_t heads, int64_t kv_heads, int64_t head_dim, int causal) {
  MST_CALL(c, stream);
  const void* ptrs[4] = {q, k, v, o};
  const int64_t lds[4] = {ldq, ldk, ldv, ldo};
  MST_TRY(check_attn(ptrs, lds, 4, batch, seq, heads, kv_heads, head_dim, causal));
  if (!lse) return fail(MST_ERR_CONFIG, "NULL lse");
  if (ldq < heads * head_dim || ldo < heads * head_dim || ldk < kv_heads * head_dim || ldv < kv_heads * head_dim)
    return fail(MST_ERR_SHAPE, "row stride smaller than heads * head_dim");
  const mst_attn::AttnShape sh{(int)batch, (int)seq, (int)heads, (int)kv_heads, (int)head_dim};
  const char* err = "";
  const int r = mst_attn::forward(reinterpret_cast<void*>(c->encode), static_cast<cudaStream_t>(stream), c->attn, sh, q, ldq, k,
                                  ldk, v, ldv, o, ldo, lse, &err);
  if (r) return fail(r == 1 ? MST_ERR_CUDA : MST_ERR_CUDA, "attention forward: %s", err);
  c->launches++;
  // 2 GEMMs of the causal half: 2 * 2 * S^2/2 * hd per (batch, head)
  cnt_op(c, (uint64_t)(2.0 * batch * heads * (double)seq * seq * head_dim), (uint64_t)(batch * seq * 4 * heads * head_dim));
  return MST_OK;
}

int mst_attention_workspace(int64_t batch, int64_t seq, int64_t heads, size_t* bytes) {
  if (!bytes) return fail(MST_ERR_CONFIG, "NULL output");
  if (batch < 1 || seq < 1 || heads < 1) return fail(MST_ERR_SHAPE, "attention extents must be >= 1");
  // D = rowsum(dO * O) [B, heads, S] fp32, then the 128-padded lse (log2 units) and D rows
  const size_t spad = size_t((seq + 127) / 128) * 128;
  *bytes = align_up((size_t(batch) * heads * seq + 63) / 64 * 64 * 4 + 2 * size_t(batch) * heads * spad * 4, 256);
  return MST_OK;
}

int mst_attention_backward(mst_ctx* c, void* stream, const void* q, int64_t ldq, const void* k, int64_t ldk,
                           const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                           const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                           int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads, int64_t head_dim, int causal,
                           void* ws, size_t ws_bytes) {
  MST_CALL(c, stream);
  const void* ptrs[8] = {q, k, v, o, dout, dq, dk, dv};
  const int64_t lds[8] = {ldq, ldk, ldv, ldo, lddo, lddq, lddk, lddv};
  MST_TRY(check_attn(ptrs, lds, 8, batch, seq, heads, kv_heads, head_dim, causal));
  if (!lse) return fail(MST_ERR_CONFIG, "NULL lse");
  size_t need = 0;
  MST_TRY(mst_attention_workspace(batch, seq, heads, &need));
  if (!ws || ws_bytes < need) return fail(MST_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  const mst_attn::AttnShape sh{(int)batch, (int)seq, (int)heads, (int)kv_heads, (int)head_dim};
  const char* err = "";
  const int r = mst_attn::backward(reinterpret_cast<void*>(c->encode), static_cast<cudaStream_t>(stream), c->attn, sh, q, ldq,
                                   k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk, lddk, dv, lddv,
                                   static_cast<float*>(ws), &err);
  if (r) return fail(MST_ERR_CUDA, "attention backward: %s", err);
  c->launches += 3;
  cnt_op(c, (uint64_t)(5.0 * batch * heads * (double)seq * seq * head_dim), (uint64_t)(batch * seq * 8 * heads * head_dim));
  return MST_OK;
}

int mst_debug_gemm(mst_ctx* c, void* stream, const void* a, const void* b, void* out, int64_t m, int64_t n, int64_t k,
                   int a_mn, int b_mn, int out_f32, int beta) {
  MST_CALL(c, stream);
  if (m <= 0 || n <= 0 || k <= 0) return fail(MST_ERR_SHAPE, "extents must be positive");
  if (m % 8 || n % 8 || k % 8) return fail(MST_ERR_SHAPE, "extents must be multiples of 8");
  if (beta && !out_f32) return fail(MST_ERR_CONFIG, "accumulation (beta = 1) needs the fp32 output");
  Launch L;
  Operand oa = a_mn ? Operand{a, m, k, m, true} : Operand{a, m, k, k, false};
  Operand ob = b_mn ? Operand{b, n, k, n, true} : Operand{b, n, k, k, false};
  MST_TRY(build_plain(c, L, oa, ob, out, n, out_f32 ? mst::kEpiAccF32 : mst::kEpiStoreBf16, beta));
  L.p.prob[0].nblk = c->debug_nblk;
  MST_TRY(launch(c, static_cast<cudaStream_t>(stream), L));
  MST_CUDA(cudaGetLastError());
  return MST_OK;
}

}  // extern "C"
