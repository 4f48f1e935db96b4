// Persistent, warp-specialised, CTA-pair (cta_group::2) tcgen05 GEMM that
// executes a *group* of independent GEMM problems in one launch, each with a
// fused epilogue.  This is the single compute engine behind every MsT
// kernel K1..K10:
//
//   K1  gate+up GEMM, SiLU(G)*U epilogue            (Alg. 1)
//   K2  down GEMM, bf16 store                        (Alg. 1)
//   K3  LM-Head GEMM, online-softmax CE partials     (Alg. 2)
//   K4  LM-Head GEMM recompute, dlogits epilogue     (Alg. 4)
//   K5  dX = dlogits * W_out^T                       (Alg. 4)
//   K6  dW_out += X^T dlogits (fp32 accumulate)      (Alg. 4)
//   K7  G,U,dh recompute, SwiGLU-backward epilogue   (Alg. 3)
//   K8  dW_down += h^T dO                            (Alg. 3)
//   K9  dX = dG W_g^T + dU W_u^T (two-phase K loop)  (Alg. 3)
//   K10 dW_gate|up += X^T [dG|dU]                    (Alg. 3)
//
// Tile geometry: a CTA pair owns a 256-row output tile (128 rows per CTA,
// UMMA M=256) and an N extent of up to 256 accumulator columns.  Operands
// are staged by TMA with 128-byte swizzle, one 64-deep K block per stage.
// Each CTA of the pair loads its own 128 rows of A and its half of B; the
// leader CTA issues tcgen05.mma for both.  Accumulators live in TMEM
// (512 columns, double-buffered when a tile needs <= 256 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer (leader only),
// w2 TMEM allocator, w3 idle, w4..w11 epilogue (two column groups of four
// warps; warp w reads TMEM lanes 32*(w%4) .. +31).
#pragma once

#include "ptx.cuh"

namespace mst {

constexpr int kStages = 6;
constexpr int kBK = 64;                      // K elements per stage (128 B rows)
constexpr int kABytes = 128 * kBK * 2;       // per-CTA A tile (16 KB)
constexpr int kBBytes = 128 * kBK * 2;       // per-CTA B tile, max (16 KB)
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kNumEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kNumEpiWarps;
constexpr int kMaxProblems = 4;
constexpr int kMaxMaps = 16;
constexpr int kTmemCols = 512;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

enum EpiKind : int32_t {
  kEpiStoreBf16 = 0,  // out{g}[row, col] = bf16(acc)
  kEpiSwiglu = 1,     // h = silu(G) * U
  kEpiMlpBwd = 2,     // h, dG, dU from G, U, dh
  kEpiAccF32 = 3,     // out{g}[row, col] (+)= acc  (fp32)
  kEpiCeFwd = 4,      // per-row (max, sumexp) partials + target logit
  kEpiCeBwd = 5,      // dlogits = (softmax - onehot) * scale
};

struct PhaseDesc {
  int32_t map_a, map_b0, map_b1;  // tensor-map indices; B map per CTA rank
  int32_t a_mn, b_mn;             // 1 = MN-major operand in smem
  int32_t umma_n;                 // MMA N across the pair (64..256, %32 == 0)
  int32_t tmem_col;               // accumulator column offset for this phase
  int32_t k_blocks;               // number of 64-deep K blocks
  int32_t b_off0, b_off1;         // per-rank B column offset (added to tn*tile_n)
  int32_t acc_continue;           // 1: keep accumulating onto the previous phase
};

struct ProblemDesc {
  int32_t num_phases;
  PhaseDesc ph[2];
  int32_t m_tiles, n_tiles, tile_n;
  int32_t rows, cols;  // valid output rows / columns (masking)
  int32_t epi;
  int32_t beta;        // kEpiAccF32: 1 = accumulate onto the existing value
  int32_t col_off0, col_off1;
  int32_t nparts;      // kEpiCeFwd: partials per row
  int32_t _pad;
  void* out0;
  void* out1;
  void* out2;
  int64_t ld0, ld1, ld2;
  const int32_t* labels;
  const float* lse;    // kEpiCeBwd: log-sum-exp per row (natural log)
  const float* scale;  // kEpiCeBwd: device scalar gradient scale
  float2* part;        // kEpiCeFwd: [rows, nparts] (max*log2e, sum 2^(z*log2e - max))
  float* ztarget;      // kEpiCeFwd: [rows] target logit
};

struct GemmParams {
  CUtensorMap maps[kMaxMaps];
  ProblemDesc prob[kMaxProblems];
  int32_t num_problems;
  int32_t acc_stages;  // 1 or 2 TMEM accumulator buffers
  int32_t acc_stride;  // TMEM column distance between accumulator buffers
  int32_t _pad;
  const int32_t* sched;      // encoded tiles (problem << 24 | tile), grouped per pair
  const int32_t* sched_off;  // [num_pairs + 1]
};

__device__ __forceinline__ void decode_tile(const GemmParams& p, int32_t code, int& prob, int& tm, int& tn) {
  prob = code >> 24;
  const int t = code & 0xFFFFFF;
  const int mt = p.prob[prob].m_tiles;
  tm = t % mt;
  tn = t / mt;
}

// ------------------------------------------------------------ epilogues
namespace epi {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float sigmoid(float x) { return __frcp_rn(1.0f + __expf(-x)); }

__device__ __forceinline__ void store_bf16_row32(__nv_bfloat16* dst, const float* v, int valid) {
  if (valid >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = ptx::pack_bf16(v[8 * q + 0], v[8 * q + 1]);
      w.y = ptx::pack_bf16(v[8 * q + 2], v[8 * q + 3]);
      w.z = ptx::pack_bf16(v[8 * q + 4], v[8 * q + 5]);
      w.w = ptx::pack_bf16(v[8 * q + 6], v[8 * q + 7]);
      d4[q] = w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < valid) dst[j] = __float2bfloat16_rn(v[j]);
  }
}

__device__ __forceinline__ void acc_f32_row32(float* dst, const float* v, int valid, int beta) {
  if (valid >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    float4* d4 = reinterpret_cast<float4*>(dst);
    if (beta) {
      float4 old[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) old[q] = d4[q];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        d4[q] = make_float4(old[q].x + v[4 * q], old[q].y + v[4 * q + 1], old[q].z + v[4 * q + 2],
                            old[q].w + v[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < valid) dst[j] = beta ? dst[j] + v[j] : v[j];
  }
}

__device__ __forceinline__ void load32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld_32x32b_x32(taddr, r);
  ptx::tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

}  // namespace epi

// Runs the epilogue of one tile for this thread's row.
//   taddr : TMEM address of this warp's lane quadrant at accumulator column 0
//   g     : column group (0/1) of this epilogue warp
__device__ __forceinline__ void run_epilogue(const ProblemDesc& P, int tm, int tn, int row, uint32_t taddr,
                                             int g) {
  const bool row_ok = row < P.rows;
  switch (P.epi) {
    case kEpiStoreBf16:
    case kEpiAccF32: {
      const int half = P.ph[0].umma_n >> 1;  // D columns per group
      void* out = g ? P.out1 : P.out0;
      const int64_t ld = g ? P.ld1 : P.ld0;
      const int col0 = tn * P.tile_n + (g ? P.col_off1 : P.col_off0);
      for (int c = 0; c < half; c += 32) {
        float v[32];
        epi::load32(taddr + g * half + c, v);
        const int col = col0 + c;
        const int valid = P.cols - col;
        if (row_ok && valid > 0) {
          if (P.epi == kEpiStoreBf16)
            epi::store_bf16_row32(static_cast<__nv_bfloat16*>(out) + row * ld + col, v, valid);
          else
            epi::acc_f32_row32(static_cast<float*>(out) + row * ld + col, v, valid, P.beta);
        }
      }
      break;
    }
    case kEpiSwiglu: {
      // D = [G (128) | U (128)], output 128 columns; group g owns 64.
      for (int c = 0; c < 64; c += 32) {
        float gv[32], uv[32];
        epi::load32(taddr + 64 * g + c, gv);
        epi::load32(taddr + 128 + 64 * g + c, uv);
        const int col = tn * 128 + 64 * g + c;
        const int valid = P.cols - col;
        if (row_ok && valid > 0) {
          float h[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s = epi::sigmoid(gv[j]);
            h[j] = (gv[j] * s) * uv[j];
          }
          epi::store_bf16_row32(static_cast<__nv_bfloat16*>(P.out0) + row * P.ld0 + col, h, valid);
        }
      }
      break;
    }
    case kEpiMlpBwd: {
      // D = [G (128) | U (128) | dh (128)] -> h, dG, dU (128 columns).
      for (int c = 0; c < 64; c += 32) {
        float gv[32], uv[32], dh[32];
        epi::load32(taddr + 64 * g + c, gv);
        epi::load32(taddr + 128 + 64 * g + c, uv);
        epi::load32(taddr + 256 + 64 * g + c, dh);
        const int col = tn * 128 + 64 * g + c;
        const int valid = P.cols - col;
        if (row_ok && valid > 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s = epi::sigmoid(gv[j]);
            const float act = gv[j] * s;
            const float h = act * uv[j];
            const float dgv = dh[j] * uv[j] * (s * (1.0f + gv[j] * (1.0f - s)));
            const float duv = dh[j] * act;
            gv[j] = h;
            uv[j] = dgv;
            dh[j] = duv;
          }
          epi::store_bf16_row32(static_cast<__nv_bfloat16*>(P.out0) + row * P.ld0 + col, gv, valid);
          epi::store_bf16_row32(static_cast<__nv_bfloat16*>(P.out1) + row * P.ld1 + col, uv, valid);
          epi::store_bf16_row32(static_cast<__nv_bfloat16*>(P.out2) + row * P.ld2 + col, dh, valid);
        }
      }
      break;
    }
    case kEpiCeFwd: {
      // 256 logits columns; group g reduces 128 of them to one partial.
      const int v0 = tn * 256 + 128 * g;
      const int lab = row_ok ? P.labels[row] : -1;
      float m = -INFINITY, s = 0.0f, zt = 0.0f;
      for (int c = 0; c < 128; c += 32) {
        float z[32];
        epi::load32(taddr + 128 * g + c, z);
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
        P.part[static_cast<int64_t>(row) * P.nparts + tn * 2 + g] = make_float2(m, s);
        if (lab >= v0 && lab < v0 + 128) P.ztarget[row] = zt * 0.69314718055994531f;  // back to natural units
      }
      break;
    }
    case kEpiCeBwd: {
      const int v0 = tn * 256 + 128 * g;
      const int lab = row_ok ? P.labels[row] : -1;
      const float l2 = row_ok ? P.lse[row] * epi::kLog2e : 0.0f;
      const float sc = (row_ok && lab >= 0) ? *P.scale : 0.0f;
      for (int c = 0; c < 128; c += 32) {
        float z[32];
        epi::load32(taddr + 128 * g + c, z);
        const int vb = v0 + c;
        const int valid = P.cols - vb;
        if (row_ok && valid > 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float p = ptx::ex2(z[j] * epi::kLog2e - l2);
            z[j] = (p - (vb + j == lab ? 1.0f : 0.0f)) * sc;
          }
          epi::store_bf16_row32(static_cast<__nv_bfloat16*>(P.out0) + row * P.ld0 + vb, z, valid);
        }
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
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* full = bars;                     // [kStages]   (leader's are used)
  uint64_t* empty = bars + kStages;          // [kStages]
  uint64_t* tfull = bars + 2 * kStages;      // [2]
  uint64_t* tempty = bars + 2 * kStages + 2; // [2]         (leader's are used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const uint32_t rank = ptx::cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kMaxMaps; ++i) ptx::prefetch_tmap(&p.maps[i]);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(ptx::smem_u32(&full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(ptx::smem_u32(&tfull[a]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[a]), 2 * kNumEpiWarps);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2(ptx::smem_u32(tmem_slot), kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int32_t* tiles = p.sched + p.sched_off[pair];
  const int ntiles = p.sched_off[pair + 1] - p.sched_off[pair];

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_first = ptx::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0; it < ntiles; ++it) {
        int prob, tm, tn;
        decode_tile(p, tiles[it], prob, tm, tn);
        const ProblemDesc& P = p.prob[prob];
        const int arow = tm * 256 + static_cast<int>(rank) * 128;
        for (int ph = 0; ph < P.num_phases; ++ph) {
          const PhaseDesc& d = P.ph[ph];
          const int nh = d.umma_n >> 1;  // B columns this CTA supplies
          const uint32_t stage_tx = 2u * (kABytes + nh * kBK * 2);
          const CUtensorMap* ma = &p.maps[d.map_a];
          const CUtensorMap* mb = &p.maps[rank ? d.map_b1 : d.map_b0];
          const int nb = tn * P.tile_n + (rank ? d.b_off1 : d.b_off0);
          for (int kb = 0; kb < d.k_blocks; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&empty[stage]), phase ^ 1);
            const uint32_t fbar_local = ptx::smem_u32(&full[stage]);
            if (rank == 0) ptx::mbar_arrive_expect_tx(fbar_local, stage_tx);
            const uint32_t fbar = ptx::mapa(fbar_local, 0);
            const uint32_t sa = ptx::smem_u32(smem_a + stage * kABytes);
            const uint32_t sb = ptx::smem_u32(smem_b + stage * kBBytes);
            const int k0 = kb * kBK;
            if (!d.a_mn) {
              ptx::tma_load_2d_cg2(ma, sa, fbar, k0, arow, pol_first);
            } else {
              ptx::tma_load_2d_cg2(ma, sa, fbar, arow, k0, pol_first);
              ptx::tma_load_2d_cg2(ma, sa + 8192, fbar, arow + 64, k0, pol_first);
            }
            if (!d.b_mn) {
              ptx::tma_load_2d_cg2(mb, sb, fbar, k0, nb, pol_first);
            } else {
              for (int j = 0; j < nh; j += 64) ptx::tma_load_2d_cg2(mb, sb + j * 128, fbar, nb + j, k0, pol_first);
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (rank == 0 && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = 0; it < ntiles; ++it) {
        int prob, tm, tn;
        decode_tile(p, tiles[it], prob, tm, tn);
        const ProblemDesc& P = p.prob[prob];
        ptx::mbar_wait(ptx::smem_u32(&tempty[acc]), acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + acc * p.acc_stride;
        for (int ph = 0; ph < P.num_phases; ++ph) {
          const PhaseDesc& d = P.ph[ph];
          const int nh = d.umma_n >> 1;
          const uint32_t idesc = ptx::idesc_bf16(256, d.umma_n, d.a_mn, d.b_mn);
          const uint32_t d_tmem = d_base + d.tmem_col;
          for (int kb = 0; kb < d.k_blocks; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&full[stage]), phase);
            ptx::tc_fence_after();
            const uint32_t sa = ptx::smem_u32(smem_a + stage * kABytes);
            const uint32_t sb = ptx::smem_u32(smem_b + stage * kBBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // K-major: advance 16 elements (32 B) inside the swizzled row.
              // MN-major: advance 16 k-rows (2 atoms of 8 rows = 2048 B).
              const uint64_t adesc =
                  d.a_mn ? ptx::sdesc_sw128(sa + k * 2048, 8192, 1024) : ptx::sdesc_sw128(sa + k * 32, 16, 1024);
              const uint64_t bdesc = d.b_mn ? ptx::sdesc_sw128(sb + k * 2048, (uint32_t)nh * 0 + 8192, 1024)
                                            : ptx::sdesc_sw128(sb + k * 32, 16, 1024);
              const uint32_t accum = (kb > 0 || k > 0 || d.acc_continue) ? 1u : 0u;
              ptx::umma_bf16_cg2(d_tmem, adesc, bdesc, idesc, accum);
            }
            ptx::umma_commit_cg2_mc(ptx::smem_u32(&empty[stage]), 0x3);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          (void)nh;
        }
        ptx::umma_commit_cg2_mc(ptx::smem_u32(&tfull[acc]), 0x3);
        if (++acc == p.acc_stages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    const int g = (warp - 4) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = ptx::mapa(ptx::smem_u32(&tempty[1]), 0);
    for (int it = 0; it < ntiles; ++it) {
      int prob, tm, tn;
      decode_tile(p, tiles[it], prob, tm, tn);
      const ProblemDesc& P = p.prob[prob];
      ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), acc_phase);
      ptx::tc_fence_after();
      const int row = tm * 256 + static_cast<int>(rank) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * p.acc_stride;
      run_epilogue(P, tm, tn, row, taddr, g);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      if (++acc == p.acc_stages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(tmem_base, kTmemCols);
  }
}

}  // namespace mst
