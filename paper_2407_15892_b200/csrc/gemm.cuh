// Persistent, warp-specialised, CTA-pair (cta_group::2) tcgen05 GEMM that
// executes a *group* of independent GEMM problems in one launch, each with a
// fused epilogue.  This is the single compute engine behind every MsT
// kernel:
//
//   K1  gate+up GEMM, SiLU(G)*U epilogue            (Alg. 1)
//   K2  down GEMM, bf16 store                        (Alg. 1)
//   K3  LM-Head GEMM, online-softmax CE partials     (Alg. 2)
//   K4  LM-Head GEMM recompute, dlogits epilogue     (Alg. 4)
//   K5  dX = dlogits * W_out^T                       (Alg. 4)
//   K6  dW_out += X^T dlogits (fp32, TMA reduce-add) (Alg. 4)
//   K7a dh = dO W_down^T (fp32 store)                (Alg. 3)
//   K7b G,U recompute, SwiGLU-backward epilogue      (Alg. 3)
//   K8  dW_down += h^T dO                            (Alg. 3)
//   K9  dX = dG W_g^T + dU W_u^T (two-phase K loop)  (Alg. 3)
//   K10 dW_gate|up += X^T [dG|dU]                    (Alg. 3)
//
// Tile geometry: a CTA pair owns a 256-row output tile (128 rows per CTA,
// UMMA M=256) and up to 256 fp32 accumulator columns.  Operands are staged
// by TMA with 128-byte swizzle, one 64-deep K block per stage.  Each CTA of
// the pair loads its own 128 rows of A and its half of B; the leader CTA
// issues tcgen05.mma for both.  Accumulators live in TMEM (512 columns,
// double-buffered) so the epilogue of tile i overlaps the main loop of tile
// i+1.  Epilogues go TMEM -> registers -> swizzled smem -> TMA store (bf16 /
// fp32) or TMA reduce-add (fp32 weight-gradient accumulation in L2), so no
// epilogue thread ever waits on a global store.
//
// Warp roles (256 threads): w0 TMA producer for A, w3 TMA producer for B,
// w1 MMA issuer (leader CTA only), w2 TMEM allocator + tile scheduler (leader CTA,
// dynamic mode), w4..w7 epilogue (warp w owns TMEM lanes
// 32*(w%4) .. +31, i.e. 32 output rows, and all accumulator columns).
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"

namespace mst {

#ifndef MST_SLOTS
#define MST_SLOTS 12
#endif
#ifndef MST_EPI_BUFS
#define MST_EPI_BUFS 2
#endif
#ifndef MST_SPLIT_PRODUCER
#define MST_SPLIT_PRODUCER 1  // warp 0 issues A loads, warp 3 issues B loads (0: one producer)
#endif
// Diagnostic builds only (tools/pipe_limits.py): MST_DIAG_NO_MMA skips the
// tcgen05.mma issue (commits still arrive), MST_DIAG_NO_TMA replaces the
// operand loads with plain barrier arrivals.  Results are garbage.
#ifndef MST_DIAG_NO_MMA
#define MST_DIAG_NO_MMA 0
#endif
#ifndef MST_DIAG_NO_TMA
#define MST_DIAG_NO_TMA 0
#endif
#ifndef MST_DW_EVICT_FIRST
#define MST_DW_EVICT_FIRST 1  // fp32 dW stores / reduce-adds stream through L2 with evict_first
#endif
// Operand staging: 12 slots of 16 KB grouped into pipeline stages of
// 1 + nblk slots (per launch): one A slot (128 rows x 64 K per CTA) and one
// B slot per N block b (up to 128 columns x 64 K per CTA).  A slots of all
// stages come first, then the B slots (stage-major).  Launches of normal tiles run 6 stages of 2 slots; launches with wide
// tiles (two N blocks sharing the A slot, 256 x 512 per pair: 25% fewer
// operand bytes per FLOP) run 4 stages of 3 slots.  One full and one empty
// barrier per stage (a tcgen05.commit per extra slot measurably slows the
// pipeline).
constexpr int kSlots = MST_SLOTS;
constexpr int kBK = 64;                      // K elements per K block (128 B rows)
constexpr int kSlotBytes = 128 * kBK * 2;    // 16 KB
constexpr int kABytes = kSlotBytes;          // per-CTA A tile
constexpr int kMaxNBlk = 2;                  // N blocks per tile (wide tiles)
constexpr int kNumEpiWarps = 4;
constexpr int kThreads = 128 + 32 * kNumEpiWarps;
constexpr int kEpiBufBytes = 4096;           // one 32-row x 128-byte TMA box
constexpr int kEpiBufs = MST_EPI_BUFS;       // per epilogue warp (>= 2)
constexpr int kEpiBytes = kNumEpiWarps * kEpiBufs * kEpiBufBytes;
constexpr int kMaxProblems = 8;
constexpr int kMaxMaps = 24;
constexpr int kTmemCols = 512;
// Row-scaled LM-Head (ce_ref0): a vocabulary tile whose maximum z*log2e lies
// within +-kCeRefWindow stores its softmax numerators relative to 2^0, so all
// tiles of a row share one reference and the softmax normalisation becomes a
// per-row factor applied by the consumers.
constexpr float kCeRefWindow = 64.0f;
constexpr int kSmemBytes = kSlots * kSlotBytes + kEpiBytes + 1024 /*align*/ + 512 /*barriers, tile ring*/;

enum EpiKind : int32_t {
  kEpiStoreBf16 = 0,  // out{g}[row, col] = bf16(acc)                     (TMA store)
  kEpiSwiglu = 1,     // h = silu(G) * U                                   (TMA store)
  kEpiSwigluBwd = 2,  // h, dG, dU from G, U (TMEM) and dh (global fp32)   (3 TMA stores)
  kEpiAccF32 = 3,     // out{g}[row, col] (+)= acc  fp32                   (TMA store / reduce-add)
  kEpiCeFwd = 4,      // per-row (max, sumexp) partial + target logit
  kEpiCeBwd = 5,      // dlogits = (softmax - onehot) * scale              (TMA store)
  kEpiCeFwdNum = 6,   // kEpiCeFwd + softmax numerator 2^(z log2e - m_tile) (TMA store, bf16)
  kEpiSwigluSave = 7, // kEpiSwiglu + G, U saved in fp32 (chunk-wise block: no backward recompute)
  kEpiDhSwigluBwd = 8,// acc = dh; G, U (fp32, global: aux / aux2) -> dG, dU bf16 (TMA stores)
};

struct PhaseDesc {
  int32_t map_a, map_b0, map_b1;  // tensor-map indices; B map per CTA rank
  int32_t a_mn, b_mn;             // 1 = MN-major operand in smem
  int32_t umma_n;                 // MMA N across the pair (128 or 256)
  int32_t tmem_col;               // accumulator column offset for this phase
  int32_t k_blocks;               // number of 64-deep K blocks
  int32_t b_off0, b_off1;         // per-rank B column offset (added to tn*tile_n)
  int32_t acc_continue;           // 1: keep accumulating onto the previous phase
  int32_t a_pol, b_pol;           // L2 policy of the operand loads: 0 normal, 1 evict_last, 2 evict_first
  int32_t a_3d, b_3d;             // MN-major operand described by a 3-D map: one TMA per slab
  int32_t k_start;                // first K block (split-K problems)
  int32_t _pad;
};

struct ProblemDesc {
  int32_t num_phases;
  PhaseDesc ph[2];
  int32_t m_tiles, n_tiles, tile_n;  // n_tiles counts logical N tiles of tile_n columns
  int32_t nblk;        // logical N tiles per scheduled tile (1, or 2 = wide tile sharing the A slot)
  int32_t n_wide;      // scheduled tiles along N = ceil(n_tiles / nblk)
  int32_t rows, cols;  // valid output rows / columns
  int32_t epi;
  int32_t beta;        // kEpiAccF32: 1 = reduce-add onto the existing value
  int32_t col_off0, col_off1;
  int32_t nparts;      // kEpiCeFwd: partials per row
  int32_t map_out0, map_out1, map_out2;  // output tensor maps (TMA store boxes)
  int32_t ce_ref0;     // kEpiCeFwdNum: numerators relative to 2^0 unless |tile max| > kCeRefWindow (row-scaled head)
  int64_t ld_aux;
  const float* aux;    // kEpiSwigluBwd: dh [rows, ld_aux] fp32; kEpiDhSwigluBwd: G
  const float* aux2;   // kEpiDhSwigluBwd: U [rows, ld_aux] fp32
  const int32_t* labels;
  const float* lse;    // kEpiCeBwd: log-sum-exp per row (natural log)
  const float* scale;  // kEpiCeBwd: device scalar gradient scale
  float2* part;        // kEpiCeFwd: [rows, nparts] (max*log2e, sum 2^(z*log2e - max))
  float* ztarget;      // kEpiCeFwd: [rows] target logit
  const float* rowscale;  // kEpiStoreBf16: per output row factor applied before the bf16 store (or null)
};

struct GemmParams {
  CUtensorMap maps[kMaxMaps];
  ProblemDesc prob[kMaxProblems];
  int32_t num_problems;
  int32_t acc_stages;  // 1 or 2 TMEM accumulator buffers
  int32_t acc_stride;  // TMEM column distance between accumulator buffers
  int32_t stage_slots; // 1 + max nblk over the launch's problems
  int32_t num_stages;  // kSlots / stage_slots
  const int32_t* sched;      // encoded tiles (problem << 24 | tile), grouped per pair
  const int32_t* sched_off;  // [num_pairs + 1]
  unsigned long long* prof;  // MST_PROFILE builds: per-role wait-cycle counters (else unused)
  // Dynamic scheduling (dynamic != 0): CTA pairs pull tiles from `order`
  // (all tiles, longest first) through the atomic `tile_counter` (zeroed
  // before the launch) instead of walking their static `sched` lists.
  int32_t dynamic;
  int32_t total_tiles;
  const int32_t* order;
  int32_t* tile_counter;
};

#ifndef MST_TEMPTY_RELAXED
#define MST_TEMPTY_RELAXED 1
#endif
#ifndef MST_FEED_RELAXED
#define MST_FEED_RELAXED 1
#endif
#ifndef MST_TILE_SLOTS
#define MST_TILE_SLOTS 8
#endif
constexpr int kTileSlots = MST_TILE_SLOTS;  // tile-code ring between the scheduler and all roles
// both A producers, leader MMA, 4 + 4 epilogue warps (+ both B producers)
constexpr int kTileConsumers = 11 + 2 * MST_SPLIT_PRODUCER;

// Per-role iterator over this pair's tiles.  Static mode walks the host LPT
// list.  Dynamic mode: a scheduler (lane 0 of the leader's otherwise idle
// warp 2) claims the next tile of the global order with an atomic and
// publishes its code into a kTileSlots ring in both CTAs (st.shared::cluster
// + release.cluster arrive), up to kTileSlots tiles ahead of the slowest role;
// every other role reads the ring and releases the slot back to the leader.
// A claim costs two dependent global round trips (atomicAdd on the counter,
// then the order list); off the producer's issue path they no longer stall
// the first K block of every tile (measured: 770 -> 650 cycles per K block on
// K = 1024 tiles, where the producer used to claim).
struct TileFeed {
  const int32_t* list;
  int n, it;
  int32_t* codes;      // smem ring [kTileSlots]
  uint64_t* full;      // [kTileSlots] per CTA, count 1
  uint64_t* empty;     // [kTileSlots] leader's, count kTileConsumers
  int slot;
  uint32_t phase;
  uint32_t rank;       // CTA rank in the pair: the leader's codes are written locally

  // Consumer (warp-wide: all lanes wait, lane 0 releases the slot).  The
  // code is reduced across the warp before the release, so the slot is handed
  // back only after its value has been consumed; a relaxed arrive then
  // suffices (a release arrive costs an ERRBAR + MEMBAR per tile and role).
  __device__ __forceinline__ int32_t consume(const GemmParams& p, int lane) {
    if (!p.dynamic) return uniform(it < n ? list[it++] : -1);
    if (rank == 0)  // scheduler in this CTA: CTA-scope acquire (no L1 invalidation)
      ptx::mbar_wait(ptx::smem_u32(&full[slot]), phase);
    else
      ptx::mbar_wait_cluster(ptx::smem_u32(&full[slot]), phase);
    const int32_t code = uniform(*reinterpret_cast<volatile int32_t*>(&codes[slot]));
#if MST_FEED_RELAXED
    if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&empty[slot]), 0));
#else
    if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&empty[slot]), 0));
#endif
    advance();
    return code;
  }
  // Scheduler (one thread).  tile_counter[0] is the claim counter, [1] counts
  // pairs that are done claiming; the last such pair re-zeroes both for the
  // next launch on the stream (no memset).
  __device__ __forceinline__ int32_t claim_publish(const GemmParams& p) {
    ptx::mbar_wait(ptx::smem_u32(&empty[slot]), phase ^ 1);
    const int32_t t = atomicAdd(p.tile_counter, 1);
    const int32_t code = t < p.total_tiles ? __ldg(p.order + t) : -1;
    if (code < 0 && atomicAdd(p.tile_counter + 1, 1) == static_cast<int32_t>(gridDim.x / 2) - 1) {
      atomicExch(p.tile_counter, 0);
      atomicExch(p.tile_counter + 1, 0);
    }
    codes[slot] = code;
    ptx::st_shared_cluster_u32(ptx::mapa(ptx::smem_u32(&codes[slot]), 1), static_cast<uint32_t>(code));
    ptx::mbar_arrive_local(ptx::smem_u32(&full[slot]));
    ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&full[slot]), 1));
    advance();
    return code;
  }
  // The code is broadcast through a warp reduction so everything the role
  // derives from it stays warp-uniform (uniform-datapath registers, no
  // per-instruction ELECT/R2UR loops around the TMA and MMA issues).
  __device__ __forceinline__ int32_t consume_warp(const GemmParams& p, int lane) { return consume(p, lane); }
  // A warp-wide reduction of identical values: REDUX writes a uniform
  // register, so ptxas treats everything derived from it as warp-uniform.
  __device__ __forceinline__ static int32_t uniform(int32_t v) {
    return static_cast<int32_t>(__reduce_min_sync(0xffffffffu, static_cast<uint32_t>(v)));
  }
  __device__ __forceinline__ void advance() {
    if (++slot == kTileSlots) {
      slot = 0;
      phase ^= 1;
    }
  }
};

// Instrumentation (tuning builds only, -DMST_PROFILE): clock64 spent in
// barrier waits, summed per role into p.prof:
//  [0] producer waiting for free smem stages   [1] producer total cycles
//  [2] MMA waiting for TMA data (full)          [3] MMA waiting for TMEM (tempty)
//  [4] MMA total cycles                         [5] epilogue waiting for tfull
//  [6] epilogue busy cycles                     [7] epilogue total cycles
#ifdef MST_PROFILE
#define MST_PROF_DECL unsigned long long prof_t0 = clock64(), prof_acc[3] = {0, 0, 0};
#define MST_PROF_WAIT(idx, expr)              \
  do {                                         \
    const unsigned long long t_ = clock64();  \
    expr;                                      \
    prof_acc[idx] += clock64() - t_;           \
  } while (0)
#define MST_PROF_FLUSH(base, n)                                                     \
  do {                                                                             \
    if (p.prof) {                                                                  \
      for (int i_ = 0; i_ < (n); ++i_) atomicAdd(p.prof + (base) + i_, prof_acc[i_]); \
      atomicAdd(p.prof + (base) + (n), clock64() - prof_t0);                        \
    }                                                                              \
  } while (0)
#else
#define MST_PROF_DECL
#define MST_PROF_WAIT(idx, expr) expr
#define MST_PROF_FLUSH(base, n)
#endif

// Scheduled tile -> (problem, m tile, first logical n tile, number of logical n tiles).
__device__ __forceinline__ void decode_tile(const GemmParams& p, int32_t code, int& prob, int& tm, int& tn0,
                                            int& nb) {
  prob = code >> 24;
  const int t = code & 0xFFFFFF;
  const ProblemDesc& P = p.prob[prob];
  tm = t % P.m_tiles;
  tn0 = (t / P.m_tiles) * P.nblk;
  nb = min(P.nblk, P.n_tiles - tn0);
}

// Position in a ring of `n` barrier-guarded entries; the phase flips on wrap.
struct RingPos {
  int idx;
  uint32_t phase;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      phase ^= 1;
    }
  }
  // The entry j positions further on (j < n), without moving.
  __device__ __forceinline__ RingPos at(int j, int n) const {
    const int i = idx + j;
    return i >= n ? RingPos{i - n, phase ^ 1u} : RingPos{i, phase};
  }
  __device__ __forceinline__ void advance(int j, int n) { *this = at(j, n); }
};

// ------------------------------------------------------------ epilogues
namespace epi {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float sigmoid(float x) { return __frcp_rn(1.0f + __expf(-x)); }

__device__ __forceinline__ void load32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld_32x32b_x32(taddr, r);
  ptx::tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Staging buffers for the TMA-store epilogues: rows of 128 B in SWIZZLE_128B
// layout (16-byte chunk j of row r lives at chunk j ^ (r & 7)), matching the
// output tensor maps, so one thread per row writes conflict-free.  Buffer b
// is a 128-row box; epilogue warp q owns rows [32q, 32q+32) of it.
//  * per-warp mode (bf16 outputs): each warp issues its own 32-row box;
//  * team mode (fp32 weight-gradient tiles, measured +1.8%): named barrier 1
//    hands the box between the 4 epilogue warps and warp 0 issues one
//    128-row TMA store / reduce-add (4x fewer, 4x larger bulk operations).
// Modes switch only between tiles, after draining all outstanding reads.
struct Stager {
  uint8_t* base;  // shared staging area (kEpiBufs x 16 KB)
  int lane;
  int next;       // round-robin buffer index
  int q;          // epilogue warp index 0..3
  bool team;

  __device__ __forceinline__ uint8_t* buf(int b) const { return base + b * (4 * kEpiBufBytes) + q * kEpiBufBytes; }
  __device__ __forceinline__ bool issuer() const { return team ? (q == 0 && lane == 0) : lane == 0; }
  __device__ __forceinline__ void sync() const {
    if (team)
      asm volatile("bar.sync 1, 128;" ::: "memory");
    else
      __syncwarp();
  }
  __device__ __forceinline__ void set_mode(bool want_team) {
    if (want_team == team) return;
    if (lane == 0) ptx::bulk_wait_read<0>();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    team = want_team;
    next = 0;
  }

  // Claim the next buffer: the group that last read it was issued kEpiBufs
  // groups ago, so at most kEpiBufs-1 may still be pending.
  __device__ __forceinline__ int acquire() {
    if (issuer()) ptx::bulk_wait_read<kEpiBufs - 1>();
    sync();
    const int b = next;
    next = next + 1 == kEpiBufs ? 0 : next + 1;
    return b;
  }
  // Claim the next buffer while one claimed buffer is not yet issued: one
  // group fewer may be pending.
  __device__ __forceinline__ int acquire_second() {
    if (issuer()) ptx::bulk_wait_read<kEpiBufs - 2>();
    sync();
    const int b = next;
    next = next + 1 == kEpiBufs ? 0 : next + 1;
    return b;
  }
  // 8 x 16-byte chunks of this thread's row, chunk j at logical column 16*j bytes.
  __device__ __forceinline__ void put_chunk(int b, int j, uint4 w) const {
    *reinterpret_cast<uint4*>(buf(b) + lane * 128 + ((j ^ (lane & 7)) << 4)) = w;
  }
  __device__ __forceinline__ void put_f32x32(int b, const float* v) const {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      put_chunk(b, j,
                make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                           __float_as_uint(v[4 * j + 3])));
  }
  // 32 bf16 values into chunks [4*half, 4*half + 4) of the 128-byte row.
  __device__ __forceinline__ void put_bf16x32(int b, int half, const float* v) const {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      put_chunk(b, 4 * half + j,
                make_uint4(ptx::pack_bf16(v[8 * j], v[8 * j + 1]), ptx::pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                           ptx::pack_bf16(v[8 * j + 4], v[8 * j + 5]), ptx::pack_bf16(v[8 * j + 6], v[8 * j + 7])));
  }
  // Publish buffer b to the async proxy and store (or reduce-add) it at
  // tensor coordinates (col, this warp's first row).  One bulk group per
  // issue.  `dw`: fp32 weight-gradient tile (evict_first hint).
  __device__ __forceinline__ void issue(int b, const CUtensorMap* m, int col, int row, bool reduce,
                                        bool dw = false) const {
    ptx::fence_proxy_async_smem();
    sync();
    if (issuer()) {
      uint32_t src = ptx::smem_u32(buf(b));
      if (team) {
        src = ptx::smem_u32(base + b * (4 * kEpiBufBytes));
        row -= q * 32;
      }
#if MST_DW_EVICT_FIRST
      if (dw) {
        const uint64_t pol = ptx::policy_evict_first();
        if (reduce)
          ptx::tma_reduce_add_2d_hint(m, src, col, row, pol);
        else
          ptx::tma_store_2d_hint(m, src, col, row, pol);
      } else
#endif
      {
        if (reduce)
          ptx::tma_reduce_add_2d(m, src, col, row);
        else
          ptx::tma_store_2d(m, src, col, row);
      }
      ptx::bulk_commit();
    }
  }
  __device__ __forceinline__ void issue_dw(int b, const CUtensorMap* m, int col, int row, bool reduce) const {
    issue(b, m, col, row, reduce, true);
  }
  // All bulk groups issued by this thread have completed.
  __device__ __forceinline__ void drain() const {
    if (lane == 0) ptx::bulk_wait_all();
    __syncwarp();
  }
};

}  // namespace epi

// Runs the epilogue of one tile for the 32 rows of this warp.
//   taddr : TMEM address of this warp's lane quadrant at accumulator column 0
//   row0  : first output row of the warp (tile-relative rows are row0 + lane)
__device__ __forceinline__ void run_epilogue(const GemmParams& p, const ProblemDesc& P, int tn, int row0,
                                             uint32_t taddr, epi::Stager& st) {
  const int lane = st.lane;
  const int row = row0 + lane;
  const bool row_ok = row < P.rows;
  st.set_mode(P.epi == kEpiAccF32);  // fp32 dW tiles: one 128-row box per slice
  switch (P.epi) {
    case kEpiStoreBf16: {
      const int half = P.ph[0].umma_n >> 1;
      const bool scaled = P.rowscale != nullptr;
      const float rs = (scaled && row_ok) ? P.rowscale[row] : 1.0f;
      for (int g = 0; g < 2; ++g) {
        const CUtensorMap* m = &p.maps[g ? P.map_out1 : P.map_out0];
        const int col0 = tn * P.tile_n + (g ? P.col_off1 : P.col_off0);
        for (int c = 0; c < half; c += 64) {
          const int b = st.acquire();
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            float v[32];
            epi::load32(taddr + g * half + c + 32 * s, v);
            if (scaled) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= rs;
            }
            st.put_bf16x32(b, s, v);
          }
          st.issue(b, m, col0 + c, row0, false);
        }
      }
      break;
    }
    case kEpiAccF32: {
      const int half = P.ph[0].umma_n >> 1;
      for (int g = 0; g < 2; ++g) {
        const CUtensorMap* m = &p.maps[g ? P.map_out1 : P.map_out0];
        const int col0 = tn * P.tile_n + (g ? P.col_off1 : P.col_off0);
        for (int c = 0; c < half; c += 32) {
          const int b = st.acquire();
          float v[32];
          epi::load32(taddr + g * half + c, v);
          st.put_f32x32(b, v);
          st.issue_dw(b, m, col0 + c, row0, P.beta != 0);
        }
      }
      break;
    }
    case kEpiSwiglu: {
      // D = [G (128) | U (128)] -> h (128 columns)
      const CUtensorMap* m = &p.maps[P.map_out0];
      for (int c = 0; c < 128; c += 64) {
        const int b = st.acquire();
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          float gv[32], uv[32];
          epi::load32(taddr + c + 32 * s, gv);
          epi::load32(taddr + 128 + c + 32 * s, uv);
#pragma unroll
          for (int j = 0; j < 32; ++j) gv[j] = (gv[j] * epi::sigmoid(gv[j])) * uv[j];
          st.put_bf16x32(b, s, gv);
        }
        st.issue(b, m, tn * 128 + c, row0, false);
      }
      break;
    }
    case kEpiSwigluSave: {
      // D = [G (128) | U (128)] -> h (bf16) and the accumulators G, U (fp32,
      // exactly what the backward recompute would produce).
      for (int c = 0; c < 128; c += 64) {
        float hk[2][32];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          float gv[32], uv[32];
          epi::load32(taddr + c + 32 * s, gv);
          epi::load32(taddr + 128 + c + 32 * s, uv);
          const int col = tn * 128 + c + 32 * s;
          int b = st.acquire();
          st.put_f32x32(b, gv);
          st.issue(b, &p.maps[P.map_out1], col, row0, false);
          b = st.acquire();
          st.put_f32x32(b, uv);
          st.issue(b, &p.maps[P.map_out2], col, row0, false);
#pragma unroll
          for (int j = 0; j < 32; ++j) hk[s][j] = (gv[j] * epi::sigmoid(gv[j])) * uv[j];
        }
        const int b = st.acquire();
        st.put_bf16x32(b, 0, hk[0]);
        st.put_bf16x32(b, 1, hk[1]);
        st.issue(b, &p.maps[P.map_out0], tn * 128 + c, row0, false);
      }
      break;
    }
    case kEpiSwigluBwd: {
      // D = [G (128) | U (128)], dh from global -> h, dG, dU (128 columns).
      // h and dG are staged per 64-column slice while dU waits in registers
      // for the next free buffer (two staging buffers suffice).
      for (int c = 0; c < 128; c += 64) {
        float du_keep[2][32];
        const int bh = st.acquire();
        const int bg = st.acquire_second();
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          float gv[32], uv[32], dh[32];
          epi::load32(taddr + c + 32 * s, gv);
          epi::load32(taddr + 128 + c + 32 * s, uv);
          const int col = tn * 128 + c + 32 * s;
          if (row_ok && col + 32 <= P.cols) {
            const float4* src = reinterpret_cast<const float4*>(P.aux + static_cast<int64_t>(row) * P.ld_aux + col);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 w = __ldg(src + q);
              dh[4 * q] = w.x;
              dh[4 * q + 1] = w.y;
              dh[4 * q + 2] = w.z;
              dh[4 * q + 3] = w.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              dh[j] = (row_ok && col + j < P.cols) ? P.aux[static_cast<int64_t>(row) * P.ld_aux + col + j] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s_ = epi::sigmoid(gv[j]);
            const float act = gv[j] * s_;
            const float h = act * uv[j];
            const float dgv = dh[j] * uv[j] * (s_ * (1.0f + gv[j] * (1.0f - s_)));
            du_keep[s][j] = dh[j] * act;
            gv[j] = h;
            uv[j] = dgv;
          }
          st.put_bf16x32(bh, s, gv);
          st.put_bf16x32(bg, s, uv);
        }
        st.issue(bh, &p.maps[P.map_out0], tn * 128 + c, row0, false);
        st.issue(bg, &p.maps[P.map_out1], tn * 128 + c, row0, false);
        const int bu = st.acquire();
        st.put_bf16x32(bu, 0, du_keep[0]);
        st.put_bf16x32(bu, 1, du_keep[1]);
        st.issue(bu, &p.maps[P.map_out2], tn * 128 + c, row0, false);
      }
      break;
    }
    case kEpiDhSwigluBwd: {
      // D = dh (256 columns of I per CTA row block); the forward's fp32 G, U of
      // the same elements come from global memory (one 128-byte line per
      // thread and 32 columns).  Same arithmetic as the stand-alone SwiGLU
      // backward, so the result is bitwise that of the unfused schedule.
      const int half = P.ph[0].umma_n >> 1;
      for (int g = 0; g < 2; ++g) {
        const int colb = tn * P.tile_n + (g ? P.col_off1 : P.col_off0);
        for (int c = 0; c < half; c += 64) {
          const int bg = st.acquire();
          const int bu = st.acquire_second();
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            float dh[32], gv[32], uv[32];
            epi::load32(taddr + g * half + c + 32 * s2, dh);
            const int col = colb + c + 32 * s2;
            if (row_ok && col + 32 <= P.cols) {
              const float4* sg = reinterpret_cast<const float4*>(P.aux + static_cast<int64_t>(row) * P.ld_aux + col);
              const float4* su = reinterpret_cast<const float4*>(P.aux2 + static_cast<int64_t>(row) * P.ld_aux + col);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 a = __ldcs(sg + q4), b = __ldcs(su + q4);
                gv[4 * q4] = a.x, gv[4 * q4 + 1] = a.y, gv[4 * q4 + 2] = a.z, gv[4 * q4 + 3] = a.w;
                uv[4 * q4] = b.x, uv[4 * q4 + 1] = b.y, uv[4 * q4 + 2] = b.z, uv[4 * q4 + 3] = b.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const bool ok = row_ok && col + j < P.cols;
                gv[j] = ok ? P.aux[static_cast<int64_t>(row) * P.ld_aux + col + j] : 0.f;
                uv[j] = ok ? P.aux2[static_cast<int64_t>(row) * P.ld_aux + col + j] : 0.f;
              }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float s_ = epi::sigmoid(gv[j]);
              const float act = gv[j] * s_;
              const float dgv = dh[j] * uv[j] * (s_ * (1.0f + gv[j] * (1.0f - s_)));
              uv[j] = dh[j] * act;
              gv[j] = dgv;
            }
            st.put_bf16x32(bg, s2, gv);
            st.put_bf16x32(bu, s2, uv);
          }
          st.issue(bg, &p.maps[P.map_out0], colb + c, row0, false);
          st.issue(bu, &p.maps[P.map_out1], colb + c, row0, false);
        }
      }
      break;
    }
    case kEpiCeFwd: {
      // 256 logits columns -> one (max, sumexp) partial per row and tile.
      const int v0 = tn * 256;
      const int lab = row_ok ? P.labels[row] : -1;
      float m = -INFINITY, s = 0.0f, zt = 0.0f;
      for (int c = 0; c < 256; c += 32) {
        float z[32];
        epi::load32(taddr + c, z);
        const int vb = v0 + c;
        const int valid = P.cols - vb;
        float cmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          z[j] *= epi::kLog2e;
          if (j < valid) cmax = fmaxf(cmax, z[j]);
        }
        if (cmax > m) {
          s *= ptx::ex2(m - cmax);
          m = cmax;
        }
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < valid) acc += ptx::ex2(z[j] - m);
        s += acc;
        if (lab >= vb && lab < vb + 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (lab == vb + j) zt = z[j];
        }
      }
      if (row_ok) {
        P.part[static_cast<int64_t>(row) * P.nparts + tn] = make_float2(m, s);
        if (lab >= v0 && lab < v0 + 256) P.ztarget[row] = zt * 0.69314718055994531f;  // natural units
      }
      break;
    }
    case kEpiCeFwdNum: {
      // Single-pass LM-Head forward+backward: per (row, 256-column tile)
      // pass 1 finds m = max z*log2e over the tile, pass 2 writes the
      // unnormalised softmax numerator e = 2^(z*log2e - m) (bf16, in (0,1])
      // into the dlogits buffer and accumulates s = sum e (fp32).  Logits
      // themselves are never stored.  Row-scaled head (ce_ref0): tiles
      // whose maximum lies within +-kCeRefWindow use reference 2^0 instead of
      // m, so dlogits = f_row * e' with one factor per row (applied by the K5
      // epilogue and folded into K6's A operand, ce_combine_rowscale_kernel);
      // otherwise normalize_dlogits turns e into (e 2^(m - lse2) - onehot) * scale.
      const int v0 = tn * 256;
      const int lab = row_ok ? P.labels[row] : -1;
      float m = -INFINITY, zt = 0.0f;
      for (int c = 0; c < 256; c += 32) {
        float z[32];
        epi::load32(taddr + c, z);
        const int vb = v0 + c;
        const int valid = P.cols - vb;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < valid) m = fmaxf(m, z[j] * epi::kLog2e);
        if (lab >= vb && lab < vb + 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (lab == vb + j) zt = z[j];
        }
      }
      float s = 0.0f;
      // Reference of this tile's numerators: its maximum, or 2^0 (row-scaled
      // head) when the maximum lies within the window; the partial records it.
      if (P.ce_ref0 && fabsf(m) <= kCeRefWindow) m = 0.0f;
      const CUtensorMap* mo = &p.maps[P.map_out0];
      for (int c = 0; c < 256; c += 64) {
        const int b = st.acquire();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float z[32];
          epi::load32(taddr + c + 32 * h, z);
          const int vb = v0 + c + 32 * h;
          const int valid = P.cols - vb;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float e = j < valid ? ptx::ex2(z[j] * epi::kLog2e - m) : 0.0f;
            s += e;
            z[j] = e;
          }
          st.put_bf16x32(b, h, z);
        }
        st.issue(b, mo, v0 + c, row0, false);
      }
      if (row_ok) {
        P.part[static_cast<int64_t>(row) * P.nparts + tn] = make_float2(m, s);
        if (lab >= v0 && lab < v0 + 256) P.ztarget[row] = zt;
      }
      break;
    }
    case kEpiCeBwd: {
      const int v0 = tn * 256;
      const int lab = row_ok ? P.labels[row] : -1;
      const float l2 = row_ok ? P.lse[row] * epi::kLog2e : 0.0f;
      const float sc = (row_ok && lab >= 0) ? *P.scale : 0.0f;
      const CUtensorMap* m = &p.maps[P.map_out0];
      for (int c = 0; c < 256; c += 64) {
        const int b = st.acquire();
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          float z[32];
          epi::load32(taddr + c + 32 * s, z);
          const int vb = v0 + c + 32 * s;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float pr = ptx::ex2(z[j] * epi::kLog2e - l2);
            z[j] = (pr - (vb + j == lab ? 1.0f : 0.0f)) * sc;
          }
          st.put_bf16x32(b, s, z);
        }
        st.issue(b, m, v0 + c, row0, false);
      }
      break;
    }
    default:
      break;
  }
}

// ---------------------------------------------------------------- kernel
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    mst_grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_slots = smem;
  uint8_t* smem_epi = smem + kSlots * kSlotBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_epi + kEpiBytes);
  uint64_t* full = bars;                      // [kSlots]   (leader's are used)
  uint64_t* empty = bars + kSlots;            // [kSlots]
  uint64_t* tfull = bars + 2 * kSlots;        // [2]
  uint64_t* tempty = bars + 2 * kSlots + 2;   // [2]         (leader's are used)
  uint64_t* tile_full = bars + 2 * kSlots + 4;                 // [kTileSlots]
  uint64_t* tile_empty = tile_full + kTileSlots;               // [kTileSlots] (leader's are used)
  int32_t* tile_codes = reinterpret_cast<int32_t*>(tile_empty + kTileSlots);  // [kTileSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_codes + kTileSlots);

  const uint32_t rank = ptx::cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kMaxMaps; ++i) ptx::prefetch_tmap(&p.maps[i]);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kSlots; ++s) {
      ptx::mbar_init(ptx::smem_u32(&full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(ptx::smem_u32(&tfull[a]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[a]), 2 * kNumEpiWarps);
    }
    for (int k = 0; k < kTileSlots; ++k) {
      ptx::mbar_init(ptx::smem_u32(&tile_full[k]), 1);
      ptx::mbar_init(ptx::smem_u32(&tile_empty[k]), kTileConsumers);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2(ptx::smem_u32(tmem_slot), kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = __reduce_min_sync(0xffffffffu, *tmem_slot);  // uniform register

  TileFeed feed{p.sched + p.sched_off[pair], p.sched_off[pair + 1] - p.sched_off[pair], 0, tile_codes,
                tile_full, tile_empty, 0, 0, rank};

  if (warp == 0 || (MST_SPLIT_PRODUCER && warp == 3)) {
    // ===================== TMA producer(s) =====================
    // With MST_SPLIT_PRODUCER warp 0 issues the A loads (and the expect_tx),
    // warp 3 the B loads; both walk the same stage ring.  Everything the
    // K-block loop needs is kept in registers: the loop sits on the critical
    // path whenever the MMA waits for operands.
    const bool do_a = warp == 0;
    const bool do_b = !MST_SPLIT_PRODUCER || warp == 3;
    {  // the whole warp walks the loop; lane 0 issues the barrier arrivals and TMA loads
      const bool issuer = lane == 0;
      // Values produced by inline asm (policies, mapa) are opaque to ptxas's
      // uniformity analysis: pass them through a warp reduction once so the
      // TMA issue below takes uniform-register operands directly.
      auto uni64 = [](uint64_t v) {
        return (static_cast<uint64_t>(TileFeed::uniform(static_cast<int32_t>(v >> 32))) << 32) |
               static_cast<uint32_t>(TileFeed::uniform(static_cast<int32_t>(v & 0xffffffffu)));
      };
      uint64_t pols[3];
      pols[0] = uni64(ptx::policy_evict_normal());
      pols[1] = uni64(ptx::policy_evict_last());
      pols[2] = uni64(ptx::policy_evict_first());
      const int nst = p.num_stages;
      const uint32_t slots_u32 = static_cast<uint32_t>(TileFeed::uniform(static_cast<int32_t>(ptx::smem_u32(smem_slots))));
      const uint32_t b_region = slots_u32 + nst * kSlotBytes;
      const uint32_t b_stride = (p.stage_slots - 1) * kSlotBytes;
      const uint32_t empty_u32 = static_cast<uint32_t>(TileFeed::uniform(static_cast<int32_t>(ptx::smem_u32(empty))));
      const uint32_t full_u32 = static_cast<uint32_t>(TileFeed::uniform(static_cast<int32_t>(ptx::smem_u32(full))));
      const uint32_t full_leader =
          static_cast<uint32_t>(TileFeed::uniform(static_cast<int32_t>(ptx::mapa(full_u32, 0))));
      const bool arm = rank == 0 && do_a;
      int sidx = 0;
      uint32_t sphase = 0, sa = slots_u32, sb = b_region;
      MST_PROF_DECL
      for (;;) {
        const int32_t code = feed.consume_warp(p, lane);
        if (code < 0) break;
        int prob, tm, tn0, nb;
        decode_tile(p, code, prob, tm, tn0, nb);
        const ProblemDesc& P = p.prob[prob];
        const int arow = tm * 256 + static_cast<int>(rank) * 128;
        for (int ph = 0; ph < P.num_phases; ++ph) {
          const PhaseDesc& d = P.ph[ph];
          const int nh = d.umma_n >> 1;  // B columns this CTA supplies per N block
          const uint32_t kblock_tx = 2u * (kABytes + nb * nh * kBK * 2);
          const CUtensorMap* ma = &p.maps[d.map_a];
          const CUtensorMap* mb = &p.maps[rank ? d.map_b1 : d.map_b0];
          const int ncol0 = tn0 * P.tile_n + (rank ? d.b_off1 : d.b_off0);
          const int ncol1 = ncol0 + P.tile_n;
          const uint64_t pa = pols[d.a_pol], pb = pols[d.b_pol];
          const int amode = !d.a_mn ? 0 : (d.a_3d ? 1 : 2);
          const int bmode = !d.b_mn ? 0 : (d.b_3d ? 1 : 2);
          const int kbs = d.k_blocks;
          int k0 = d.k_start * kBK;
          for (int kb = 0; kb < kbs; ++kb, k0 += kBK) {
            MST_PROF_WAIT(0, ptx::mbar_wait(empty_u32 + 8 * sidx, sphase ^ 1));
            if (arm && issuer) {
#if MST_DIAG_NO_TMA
              ptx::mbar_arrive_local(full_u32 + 8 * sidx);
              (void)kblock_tx;
#else
              ptx::mbar_arrive_expect_tx(full_u32 + 8 * sidx, kblock_tx);
#endif
            }
#if !MST_DIAG_NO_TMA
            const uint32_t fbar = full_leader + 8 * sidx;
            if (do_a && issuer) {
              if (amode == 0) {
                ptx::tma_load_2d_cg2(ma, sa, fbar, k0, arow, pa);
              } else if (amode == 1) {
                ptx::tma_load_3d_cg2(ma, sa, fbar, 0, k0, arow >> 6, pa);
              } else {
                ptx::tma_load_2d_cg2(ma, sa, fbar, arow, k0, pa);
                ptx::tma_load_2d_cg2(ma, sa + 8192, fbar, arow + 64, k0, pa);
              }
            }
            if (do_b && issuer) {
#pragma unroll
              for (int j = 0; j < kMaxNBlk; ++j) {
                if (j < nb) {
                  const uint32_t sbj = sb + j * kSlotBytes;
                  const int ncol = j ? ncol1 : ncol0;
                  if (bmode == 0) {
                    ptx::tma_load_2d_cg2(mb, sbj, fbar, k0, ncol, pb);
                  } else if (bmode == 1) {
                    ptx::tma_load_3d_cg2(mb, sbj, fbar, 0, k0, ncol >> 6, pb);
                  } else {
                    for (int c = 0; c < nh; c += 64) ptx::tma_load_2d_cg2(mb, sbj + c * 128, fbar, ncol + c, k0, pb);
                  }
                }
              }
            }
#endif
            if (++sidx == nst) {
              sidx = 0;
              sphase ^= 1;
              sa = slots_u32;
              sb = b_region;
            } else {
              sa += kSlotBytes;
              sb += b_stride;
            }
          }
        }
      }
#if defined(MST_PROFILE) && MST_PROFILE == 2
      if (false)
#endif
      if (issuer) MST_PROF_FLUSH(0, 1);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (rank == 0) {  // the whole warp walks the loop; lane 0 issues the MMAs and their commits
      const bool issuer = lane == 0;
      const int nst = p.num_stages;
      const uint32_t slots_u32 = ptx::smem_u32(smem_slots);
      const uint32_t b_region = slots_u32 + nst * kSlotBytes;
      const uint32_t b_stride = (p.stage_slots - 1) * kSlotBytes;
      const uint32_t empty_u32 = ptx::smem_u32(empty);
      const uint32_t full_u32 = ptx::smem_u32(full);
      const int acc_stages = p.acc_stages;
      const uint32_t acc_stride = p.acc_stride;
      int sidx = 0;
      uint32_t sphase = 0, sa = slots_u32, sb = b_region;
      RingPos ap{0, 0};  // TMEM accumulator ring (acc_stages entries of acc_stride columns)
      MST_PROF_DECL
      for (;;) {
#if defined(MST_PROFILE) && MST_PROFILE == 2  // diagnostic: MMA tile-feed waits, reported in slot 1
        int32_t code;
        MST_PROF_WAIT(2, code = feed.consume_warp(p, lane));
#else
        const int32_t code = feed.consume_warp(p, lane);
#endif
        if (code < 0) break;
        int prob, tm, tn0, nb;
        decode_tile(p, code, prob, tm, tn0, nb);
        const ProblemDesc& P = p.prob[prob];
        const RingPos acc0 = ap;  // N block b accumulates in ring entry acc0 + b
        const int acc1 = acc0.at(1 % acc_stages, acc_stages).idx;
        for (int b = 0; b < nb; ++b) {
          const RingPos e = ap.at(b, acc_stages);
          MST_PROF_WAIT(1, ptx::mbar_wait(ptx::smem_u32(&tempty[e.idx]), e.phase ^ 1));
        }
        ap.advance(nb, acc_stages);
        ptx::tc_fence_after();
        for (int ph = 0; ph < P.num_phases; ++ph) {
          const PhaseDesc& d = P.ph[ph];
          const uint32_t idesc = ptx::idesc_bf16(256, d.umma_n, d.a_mn, d.b_mn);
          // Descriptor constant parts; the start-address field (bits 0-13,
          // address >> 4) is added per MMA.  K-major: +32 B per 16-deep step
          // inside the swizzled row; MN-major: +2048 B (2 atoms of 8 k-rows).
          const uint64_t a_hi = d.a_mn ? ptx::sdesc_sw128(0, 8192, 1024) : ptx::sdesc_sw128(0, 16, 1024);
          const uint64_t b_hi = d.b_mn ? ptx::sdesc_sw128(0, 8192, 1024) : ptx::sdesc_sw128(0, 16, 1024);
          const uint32_t a_step = d.a_mn ? (2048 >> 4) : (32 >> 4);
          const uint32_t b_step = d.b_mn ? (2048 >> 4) : (32 >> 4);
          const uint32_t dt0 = tmem_base + acc0.idx * acc_stride + d.tmem_col;
          const uint32_t dt1 = tmem_base + acc1 * acc_stride + d.tmem_col;
          uint32_t accum0 = d.acc_continue ? 1u : 0u;
          const int kbs = d.k_blocks;
          for (int kb = 0; kb < kbs; ++kb) {
            MST_PROF_WAIT(0, ptx::mbar_wait(full_u32 + 8 * sidx, sphase));
            ptx::tc_fence_after();
            const uint32_t a4 = sa >> 4, b4 = sb >> 4;
#pragma unroll
            for (int b = 0; b < kMaxNBlk; ++b) {
              if (b < nb && issuer) {
                const uint32_t dt = b ? dt1 : dt0;
                const uint32_t bb4 = b4 + b * (kSlotBytes >> 4);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                  const uint64_t adesc = a_hi | (a4 + k * a_step);
                  const uint64_t bdesc = b_hi | (bb4 + k * b_step);
                  if (!MST_DIAG_NO_MMA) ptx::umma_bf16_cg2(dt, adesc, bdesc, idesc, k ? 1u : accum0);
                }
              }
            }
            accum0 = 1u;
            if (issuer) ptx::umma_commit_cg2_mc(empty_u32 + 8 * sidx, 0x3);
            if (++sidx == nst) {
              sidx = 0;
              sphase ^= 1;
              sa = slots_u32;
              sb = b_region;
            } else {
              sa += kSlotBytes;
              sb += b_stride;
            }
          }
        }
        if (issuer) {
          ptx::umma_commit_cg2_mc(ptx::smem_u32(&tfull[acc0.idx]), 0x3);
          if (nb > 1) ptx::umma_commit_cg2_mc(ptx::smem_u32(&tfull[acc1]), 0x3);
        }
        __syncwarp();
      }
      if (issuer) MST_PROF_FLUSH(2, 2);
#if defined(MST_PROFILE) && MST_PROFILE == 2
      if (issuer && p.prof) atomicAdd(p.prof + 1, prof_acc[2]);
#endif
    }
  } else if (warp == 2) {
    // ===================== tile scheduler (dynamic mode, leader CTA) =====================
    if (p.dynamic && rank == 0) {
      if (lane == 0)
        while (feed.claim_publish(p) >= 0) {
        }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    RingPos ap{0, 0};
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = ptx::mapa(ptx::smem_u32(&tempty[1]), 0);
    epi::Stager st{smem_epi, lane, 0, q, false};
    MST_PROF_DECL
    for (;;) {
      const int32_t code = feed.consume_warp(p, lane);
      if (code < 0) break;
      int prob, tm, tn0, nb;
      decode_tile(p, code, prob, tm, tn0, nb);
      const ProblemDesc& P = p.prob[prob];
      const int row0 = tm * 256 + static_cast<int>(rank) * 128 + q * 32;
      for (int b = 0; b < nb; ++b) {
        MST_PROF_WAIT(0, ptx::mbar_wait(ptx::smem_u32(&tfull[ap.idx]), ap.phase));
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + ap.idx * p.acc_stride;
#ifndef MST_DIAG_NO_EPI
        MST_PROF_WAIT(1, run_epilogue(p, P, tn0 + b, row0, taddr, st));
#else  // diagnostic builds: epilogue cost removed (results are garbage); =2 keeps all but the CE-forward one
        if (MST_DIAG_NO_EPI == 2 && P.epi != kEpiCeFwdNum) MST_PROF_WAIT(1, run_epilogue(p, P, tn0 + b, row0, taddr, st));
#endif
        // All TMEM reads of this N block are complete (tcgen05.wait::ld);
        // release the accumulator to the MMA warp of the pair leader.
        ptx::tc_fence_before();
        __syncwarp();
        // tcgen05.wait::ld has returned, so the accumulator is already read:
        // a relaxed arrive avoids the MEMBAR.ALL.GPU + ERRBAR a release.cluster
        // arrive compiles to (the fence::before_thread_sync above orders the
        // tcgen05 reads before it).
#if MST_TEMPTY_RELAXED
        if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ap.idx ? tempty_leader1 : tempty_leader0);
#else
        if (lane == 0) ptx::mbar_arrive_cluster(ap.idx ? tempty_leader1 : tempty_leader0);
#endif
        ap.next(p.acc_stages);
      }
    }
    st.drain();
    if (lane == 0) MST_PROF_FLUSH(5, 2);
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(tmem_base, kTmemCols);
  }
}

}  // namespace mst
