// Causal grouped-query attention, forward and backward, on tcgen05 (sm_100a)
// -- the attention of the Llama-style decoder around the MsT blocks
// (reference: SPEC.md:233-241 attn_forward / attn_backward, PAPER.md:128
// "FlashAttention2").  Exact softmax attention computed
// tile by tile (FlashAttention-style online softmax): the [S, S] scores never
// reach HBM, the forward saves one fp32 log-sum-exp per (row, head).
//
// Layout: token-major, q element (b, t, head h, e) at q[(b*S + t)*ldq + h*hd + e]
// (k, v likewise with kv_heads heads; o, dq, dk, dv likewise), so the
// decoder's fused [N, d + 2d/G] qkv buffer and the Ulysses head-sharded
// tensors are both read in place.  Each operand is a 3-D tensor map
// {hd, heads, rows} with a {64, 1, 128} box: one 128-token x 64-feature
// SWIZZLE_128B tile per load; head dims below 64 are zero-padded by the TMA
// (out-of-bounds fill), 64 < hd <= 128 takes two loads.
//
// Kernels (one CTA per 128-row tile, single-CTA UMMA M=128, fp32 TMEM
// accumulators, warp roles: w0 TMA, w1 MMA, w2 TMEM allocator, w4-w7 softmax /
// gradient math with one row per thread):
//   attn_fwd_kernel   per (q tile, head): S = Q K^T -> online softmax -> O += P V
//   attn_dkv_kernel   per (kv tile, kv head): over the q heads of its group and the
//                     q tiles at or after it: S^T = K Q^T, dP^T = V dO^T,
//                     dV += P^T dO, dK += dS^T Q
//   attn_dq_kernel    per (q tile, head): over the kv tiles at or before it:
//                     S, dP, dQ += dS K
//   attn_delta_kernel D = rowsum(dO * O) per (row, head)
// No atomics anywhere: dQ, dK, dV are each produced by exactly one CTA, so
// results are bitwise reproducible.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "attention.cuh"
#include "ptx.cuh"

namespace mst_attn {

using namespace mst;

constexpr int kBM = 128;           // rows per tile (q or kv tokens)
constexpr int kTile = 16384;       // one 128 x 64 bf16 SW128 tile
constexpr int kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;

struct Maps {
  CUtensorMap q, k, v, o, dout;
};

struct Args {
  Maps m;
  uint16_t* o;         // forward output (bf16)
  float* lse;          // [B, heads, S] natural-log units
  const float* delta;  // [B, heads, S] rowsum(dO * O)
  const float* lse2p;  // [B, heads, nqb * 128] log2-units lse, +inf padded (backward v2)
  const float* deltap; // [B, heads, nqb * 128] D, zero padded
  uint16_t *dq, *dk, *dv;
  int64_t ldo, lddq, lddk, lddv;
  int B, S, heads, kvh, hd;
  float scale2;        // softmax scale * log2(e)
  float scale;         // softmax scale
  int nqb;             // q (= kv) tiles per sequence
  int inorder;         // AttnTuning::mma_inorder
  int poly;            // AttnTuning::poly_exp: exp2 pairs (of every 4) on the FMA pipe in the forward softmax
  int bwd_order;       // AttnTuning::bwd_order: backward GEMM issue orders (bit 0 dK/dV, bit 1 dQ)
};

// 2^x on the FMA / integer pipes (FlashAttention-4's split of the softmax
// exponentials between MUFU and the FMA units): round-to-nearest through the
// 1.5 * 2^23 magic constant, a degree-3 polynomial for 2^f on [-0.5, 0.5]
// (relative error 7.5e-5 with fp32 coefficients, below bf16's 2^-9 P
// rounding), the integer part added to the exponent field.  x is clamped at
// -126 (the result is then ~1e-38, not 0: used only where no score is masked).
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.0f);
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  const float p = fmaf(fmaf(fmaf(0.05517084f, f, 0.24260935f), f, 0.69326097f), f, 0.99992818f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) { return ptx::sdesc_sw128(saddr, 16, 1024); }
// MN-major operand: 64-wide N blocks one 16 KB tile apart.
__device__ __forceinline__ uint64_t mdesc(uint32_t saddr) { return ptx::sdesc_sw128(saddr, kTile, 1024); }

// One 128 x (64 * nblk) operand tile: nblk loads of a 128-row x 64-feature box.
template <int NB>
__device__ __forceinline__ void load_tile(const CUtensorMap* m, uint32_t dst, uint32_t bar, int head, int row) {
#pragma unroll
  for (int c = 0; c < NB; ++c) ptx::tma_load_3d(m, dst + c * kTile, bar, c * 64, head, row);
}

// D[128 x N] (+)= A[128 x K] B: A K-major in 64-deep sub-tiles (kTile apart),
// B K-major (b_mn = 0: 64-deep sub-tiles kTile apart) or MN-major (b_mn = 1:
// K rows of 128 B, 64-wide N blocks kTile apart); K = 64 * ksub.
__device__ __forceinline__ void mma_tile(uint32_t d, uint32_t a, uint32_t b, int ksub, int n, bool b_mn,
                                         bool accumulate) {
  const uint32_t idesc = ptx::idesc_bf16(128, n, 0, b_mn ? 1 : 0);
  for (int c = 0; c < ksub; ++c) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = kdesc(a + c * kTile + k * 32);
      const uint64_t bd = b_mn ? mdesc(b + c * 8192 + k * 2048) : kdesc(b + c * kTile + k * 32);
      ptx::umma_bf16_cg1(d, ad, bd, idesc, (accumulate || c || k) ? 1u : 0u);
    }
  }
}

// This thread's 128-value row r of a K-major [128 x 128] bf16 operand made of
// two 64-column SW128 sub-tiles; v[c] for column c.
__device__ __forceinline__ void store_row_bf16(uint8_t* base, int r, const float* v) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int sub = j >> 3, ch = j & 7;
    const uint4 w = make_uint4(ptx::pack_bf16(v[8 * j], v[8 * j + 1]), ptx::pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                               ptx::pack_bf16(v[8 * j + 4], v[8 * j + 5]), ptx::pack_bf16(v[8 * j + 6], v[8 * j + 7]));
    *reinterpret_cast<uint4*>(base + sub * kTile + r * 128 + ((ch ^ (r & 7)) << 4)) = w;
  }
}

__device__ __forceinline__ void load_row(uint32_t taddr, float (&v)[128]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(taddr + 32 * c, r);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[32 * c + j] = __uint_as_float(r[j]);
  }
  ptx::tmem_ld_wait();
}

// Writes columns [0, hd) of this thread's accumulator row (TMEM, nsub * 64
// columns) times `mul` as bf16 to dst (16-byte stores; hd % 8 == 0).
__device__ __forceinline__ void store_acc_row(uint32_t taddr, int nsub, float mul, uint16_t* dst, int hd, bool ok) {
  for (int c = 0; c < nsub * 2; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(taddr + 32 * c, r);
    ptx::tmem_ld_wait();
    if (!ok) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = 32 * c + 8 * j;
      if (e < hd) {
        const uint4 w = make_uint4(ptx::pack_bf16(__uint_as_float(r[8 * j]) * mul, __uint_as_float(r[8 * j + 1]) * mul),
                                   ptx::pack_bf16(__uint_as_float(r[8 * j + 2]) * mul, __uint_as_float(r[8 * j + 3]) * mul),
                                   ptx::pack_bf16(__uint_as_float(r[8 * j + 4]) * mul, __uint_as_float(r[8 * j + 5]) * mul),
                                   ptx::pack_bf16(__uint_as_float(r[8 * j + 6]) * mul, __uint_as_float(r[8 * j + 7]) * mul));
        *reinterpret_cast<uint4*>(dst + e) = w;
      }
    }
  }
}

// ------------------------------------------------------------------ forward
template <int NSUB>  // head-dim tiles of 64 (hd <= 64 * NSUB)
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ Args a) {
  constexpr int kST = NSUB == 1 ? 3 : 2;  // K/V stages
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = sm;
  uint8_t* k_s = q_s + NSUB * kTile;              // [kST] K tiles
  uint8_t* v_s = k_s + kST * NSUB * kTile;        // [kST] V tiles
  uint8_t* p_s = v_s + kST * NSUB * kTile;        // P: 2 sub-tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_s + 2 * kTile);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + kST;
  uint64_t* kv_empty = v_full + kST;
  uint64_t* s_full = kv_empty + kST;  // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = a.heads * a.B;
  const int qblk = a.nqb - 1 - static_cast<int>(blockIdx.x) / hb;  // longest (last) q tiles first
  const int h = static_cast<int>(blockIdx.x) % a.heads;
  const int b = (static_cast<int>(blockIdx.x) % hb) / a.heads;
  const int g = h / (a.heads / a.kvh);
  const int q0 = qblk * kBM;
  const int nblk = qblk + 1;  // causal: kv tiles 0 .. qblk
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(ptx::smem_u32(q_full), 1);
    for (int s = 0; s < kST; ++s) {
      ptx::mbar_init(ptx::smem_u32(&k_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&v_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&kv_empty[s]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(&s_full[0]), 1);
    ptx::mbar_init(ptx::smem_u32(&s_full[1]), 1);
    ptx::mbar_init(ptx::smem_u32(p_full), 4);
    ptx::mbar_init(ptx::smem_u32(pv_done), 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      ptx::prefetch_tmap(&a.m.q);
      ptx::prefetch_tmap(&a.m.k);
      ptx::prefetch_tmap(&a.m.v);
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(q_full), NSUB * kTile);
      load_tile<NSUB>(&a.m.q, ptx::smem_u32(q_s), ptx::smem_u32(q_full), h, row0 + q0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&kv_empty[s]), ((j / kST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&k_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.k, ptx::smem_u32(k_s + s * NSUB * kTile), ptx::smem_u32(&k_full[s]), g, row0 + j * kBM);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&v_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.v, ptx::smem_u32(v_s + s * NSUB * kTile), ptx::smem_u32(&v_full[s]), g, row0 + j * kBM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      auto pv = [&](int i) {
        const int s = i % kST;
        ptx::mbar_wait(ptx::smem_u32(p_full), i & 1);
        ptx::mbar_wait(ptx::smem_u32(&v_full[s]), (i / kST) & 1);
        ptx::tc_fence_after();
        // O[128 x 64*NSUB] (+)= P[128 x 128] V[128 x 64*NSUB]  (V MN-major)
        mma_tile(tO, ptx::smem_u32(p_s), ptx::smem_u32(v_s + s * NSUB * kTile), 2, 64 * NSUB, true, i > 0);
        ptx::umma_commit_cg1(ptx::smem_u32(pv_done));
        ptx::umma_commit_cg1(ptx::smem_u32(&kv_empty[s]));
      };
      ptx::mbar_wait(ptx::smem_u32(q_full), 0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&k_full[s]), (j / kST) & 1);
        ptx::tc_fence_after();
        mma_tile(tS[j & 1], ptx::smem_u32(q_s), ptx::smem_u32(k_s + s * NSUB * kTile), NSUB, 128, false, false);
        ptx::umma_commit_cg1(ptx::smem_u32(&s_full[j & 1]));
        if (j >= 1) pv(j - 1);
      }
      pv(nblk - 1);
    }
  } else if (warp >= 4) {  // ---- online softmax, one q row per thread
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int q = q0 + r;
    float m2 = -INFINITY, l = 0.f;
    float v[128];
    for (int j = 0; j < nblk; ++j) {
      ptx::mbar_wait(ptx::smem_u32(&s_full[j & 1]), (j >> 1) & 1);
      ptx::tc_fence_after();
      load_row(tS[j & 1] + lane_off, v);
      const int kv0 = j * kBM;
      float mx = -INFINITY;
      if (kv0 + kBM - 1 > q0) {  // the diagonal tile: mask kv > q
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          v[c] = (kv0 + c <= q) ? v[c] * a.scale2 : -INFINITY;
          mx = fmaxf(mx, v[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          v[c] *= a.scale2;
          mx = fmaxf(mx, v[c]);
        }
      }
      const float mn = fmaxf(m2, mx);
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        v[c] = ptx::ex2(v[c] - mn);
        rs += v[c];
      }
      const float alpha = ptx::ex2(m2 - mn);  // 0 on the first tile
      if (j >= 1) {
        ptx::mbar_wait(ptx::smem_u32(pv_done), (j - 1) & 1);  // PV_{j-1} done: O current, P buffer free
        ptx::tc_fence_after();
        if (!__all_sync(0xffffffffu, alpha == 1.f)) {
          for (int c = 0; c < 2 * NSUB; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(tO + lane_off + 32 * c, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_32x32b_x32(tO + lane_off + 32 * c, o);
          }
          ptx::tmem_st_wait();
        }
      }
      l = l * alpha + rs;
      m2 = mn;
      store_row_bf16(p_s, r, v);
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(p_full));
    }
    ptx::mbar_wait(ptx::smem_u32(pv_done), (nblk - 1) & 1);
    ptx::tc_fence_after();
    const bool ok = q < a.S;
    store_acc_row(tO + lane_off, NSUB, 1.f / l, a.o + (static_cast<int64_t>(row0) + q) * a.ldo + h * a.hd, a.hd, ok);
    if (ok) a.lse[(static_cast<int64_t>(b) * a.heads + h) * a.S + q] = (m2 + __log2f(l)) * 0.69314718055994531f;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// ------------------------------------------------------------------ forward, two q tiles per CTA
// Ping-pong over two adjacent q tiles (A = 2p, B = 2p + 1) that share every
// K / V tile: while the math warps of one tile run its online softmax, the
// tensor core works on the other tile's GEMMs.  TMEM: per tile S (128 fp32
// columns) and O (128); P is written back over the first 64 columns of S as
// packed bf16 and read by the PV GEMM straight from TMEM (no shared-memory
// round trip), so shared memory holds only Q (two tiles) and a 2-stage K/V
// ring.  Softmax in two passes over TMEM (max, then exp / sum / pack), one
// FFMA + one ex2 per element, ~70 registers per thread.
template <int NSUB>
__global__ void __launch_bounds__(384, 1) attn_fwd2_kernel(const __grid_constant__ Args a) {
  constexpr int kST = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = sm;                            // [2 tiles]
  uint8_t* k_s = q_s + 2 * NSUB * kTile;        // [kST]
  uint8_t* v_s = k_s + kST * NSUB * kTile;      // [kST]
  uint64_t* bars = reinterpret_cast<uint64_t*>(v_s + kST * NSUB * kTile);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;                  // [kST]
  uint64_t* v_full = k_full + kST;              // [kST]
  uint64_t* kv_empty = v_full + kST;            // [kST]
  uint64_t* s_full = kv_empty + kST;            // [2 tiles]
  uint64_t* p_full = s_full + 2;                // [2 tiles]
  uint64_t* pv_done = p_full + 2;               // [2 tiles]
  uint64_t* o_done = pv_done + 2;               // [2 tiles] the tile's last PV has completed (one phase)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = a.heads * a.B;
  const int npair = (a.nqb + 1) / 2;
  const int pr = npair - 1 - static_cast<int>(blockIdx.x) / hb;  // heaviest pairs first
  const int h = static_cast<int>(blockIdx.x) % a.heads;
  const int b = (static_cast<int>(blockIdx.x) % hb) / a.heads;
  const int g = h / (a.heads / a.kvh);
  const int tq[2] = {2 * pr, 2 * pr + 1};
  const int nt[2] = {tq[0] + 1, tq[1] < a.nqb ? tq[1] + 1 : 0};  // kv tiles per q tile (causal)
  const int ntiles = nt[1] ? 2 : 1;
  const int nkv = nt[1] ? nt[1] : nt[0];
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(ptx::smem_u32(q_full), 1);
    for (int s = 0; s < kST; ++s) {
      ptx::mbar_init(ptx::smem_u32(&k_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&v_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&kv_empty[s]), 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(ptx::smem_u32(&s_full[t]), 1);
      ptx::mbar_init(ptx::smem_u32(&p_full[t]), 4);
      ptx::mbar_init(ptx::smem_u32(&pv_done[t]), 1);
      ptx::mbar_init(ptx::smem_u32(&o_done[t]), 1);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {  // warpgroup 0: TMA (w0) and MMA (w1) need few registers; the math warpgroups take them
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      ptx::prefetch_tmap(&a.m.q);
      ptx::prefetch_tmap(&a.m.k);
      ptx::prefetch_tmap(&a.m.v);
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(q_full), ntiles * NSUB * kTile);
      for (int t = 0; t < ntiles; ++t)
        load_tile<NSUB>(&a.m.q, ptx::smem_u32(q_s + t * NSUB * kTile), ptx::smem_u32(q_full), h, row0 + tq[t] * kBM);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&kv_empty[s]), ((j / kST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&k_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.k, ptx::smem_u32(k_s + s * NSUB * kTile), ptx::smem_u32(&k_full[s]), g, row0 + j * kBM);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&v_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.v, ptx::smem_u32(v_s + s * NSUB * kTile), ptx::smem_u32(&v_full[s]), g, row0 + j * kBM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t pv_idesc = ptx::idesc_bf16(128, 64 * NSUB, 0, 1);
      auto qk = [&](int t, int j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&k_full[s]), (j / kST) & 1);
        ptx::tc_fence_after();
        mma_tile(tmem + 256 * t, ptx::smem_u32(q_s + t * NSUB * kTile), ptx::smem_u32(k_s + s * NSUB * kTile), NSUB,
                 128, false, false);
        ptx::umma_commit_cg1(ptx::smem_u32(&s_full[t]));
      };
      ptx::mbar_wait(ptx::smem_u32(q_full), 0);
      for (int t = 0; t < ntiles; ++t) qk(t, 0);
      // Ping-pong: as soon as tile t's softmax of step j is done, its PV(j)
      // and its next scores QK(j+1) are issued back to back, so the tensor
      // core works on tile t while the other tile's softmax runs (issuing all
      // PVs of step j before any QK(j+1) would make each tile's next softmax
      // wait for the other tile's current one: the two softmaxes then run at
      // the same time and compete for MUFU instead of alternating; measured
      // 846 -> 1001 TFLOP/s at S=8192, hd=128).  Blocking waits: a polling
      // issuer that serves whichever tile is ready first steals issue slots
      // from the softmax warps of its SM sub-partition (measured 800).
      for (int j = 0; j < nkv; ++j) {
        const int s = j % kST;
        for (int t = 0; t < ntiles; ++t) {
          if (j >= nt[t]) continue;
          ptx::mbar_wait(ptx::smem_u32(&p_full[t]), j & 1);
          ptx::mbar_wait(ptx::smem_u32(&v_full[s]), (j / kST) & 1);
          ptx::tc_fence_after();
          // O_t += P_t V_j: P (bf16, 64 packed columns over S_t) from TMEM, V MN-major
          const uint32_t vb = ptx::smem_u32(v_s + s * NSUB * kTile);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::umma_bf16_tmem_a_cg1(tmem + 256 * t + 128, tmem + 256 * t + 8 * k, mdesc(vb + k * 2048), pv_idesc,
                                      (j > 0 || k) ? 1u : 0u);
          // pv_done phases only where the issuer waits for them (every phase
          // observed before the next completes); o_done ends the tile
          if (j + 1 < nt[t] && !a.inorder) ptx::umma_commit_cg1(ptx::smem_u32(&pv_done[t]));
          if (j + 1 == nt[t]) ptx::umma_commit_cg1(ptx::smem_u32(&o_done[t]));
          if (j + 1 < nt[t]) {
            if (!a.inorder) ptx::mbar_wait(ptx::smem_u32(&pv_done[t]), j & 1);  // P_t consumed before S_t is overwritten
            qk(t, j + 1);
          }
        }
        ptx::umma_commit_cg1(ptx::smem_u32(&kv_empty[s]));
      }
    }
  }
  } else {  // ---- online softmax: warps 4-7 tile A, 8-11 tile B, one q row per thread
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
    const int t = (warp - 4) >> 2;
    if (t < ntiles) {
      const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const uint32_t tS = tmem + 256 * t + lane_off, tO = tS + 128;
      const int q0 = tq[t] * kBM;
      const int q = q0 + ((warp & 3) * 32 + lane);
      // Lazy rescaling: P is formed against a reference maximum `ref` (log2
      // units) that moves only when a row's maximum exceeds it by more than 8
      // (exact either way: P and l share the reference; p <= 2^8), so the O
      // accumulator is rescaled only when the running maximum really jumps.
      // The row's 128 scores come from TMEM in one batch (one load latency
      // per tile) and stay in registers for the max and the exp passes; P is
      // packed and written over S columns 0..63 chunk by chunk.
      float m2 = -INFINITY, l = 0.f;
      for (int j = 0; j < nt[t]; ++j) {
        ptx::mbar_wait(ptx::smem_u32(&s_full[t]), j & 1);
        ptx::tc_fence_after();
        const int kv0 = j * kBM;
        const int nvalid = kv0 + kBM - 1 > q0 ? q - kv0 + 1 : kBM;  // columns kv0 .. q are visible
        float x[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x32(tS + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(x + 32 * c));
        ptx::tmem_ld_wait();
        if (kv0 + kBM - 1 > q0) {  // the diagonal tile (warp-uniform): mask kv > q
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= nvalid) x[e] = -INFINITY;
        }
        // 8 independent partial maxima / sums: no 128-long dependency chains
        float m8[8], s8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = x[k];
#pragma unroll
        for (int e = 8; e < 128; ++e) m8[e & 7] = fmaxf(m8[e & 7], x[e]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float mx2 = mx * a.scale2;
        const float ref = (j == 0 || mx2 > m2 + 8.f) ? mx2 : m2;
#pragma unroll
        for (int k = 0; k < 8; ++k) s8[k] = 0.f;
        // P = 2^(s * scale2 - ref); `np` of every 4 column pairs on the FMA
        // pipe (exp2_poly), the rest on MUFU; the diagonal tile (masked
        // scores) stays on MUFU so masked entries are exactly 0.
        auto exp_pass = [&](auto np_tag) {
          constexpr int NP = decltype(np_tag)::value;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const bool fma_pipe = ((e >> 1) & 3) >= 4 - NP;
              const float y0 = fmaf(x[32 * c + e], a.scale2, -ref);
              const float y1 = fmaf(x[32 * c + e + 1], a.scale2, -ref);
              const float p0 = fma_pipe ? exp2_poly(y0) : ptx::ex2(y0);
              const float p1 = fma_pipe ? exp2_poly(y1) : ptx::ex2(y1);
              s8[e & 7] += p0;
              s8[(e + 1) & 7] += p1;
              pk[e >> 1] = ptx::pack_bf16(p0, p1);
            }
            ptx::tmem_st_32x32b_x16(tS + 16 * c, pk);  // P over already-read S columns
          }
        };
        const int np = kv0 + kBM - 1 > q0 ? 0 : a.poly;  // warp-uniform
        if (np == 0)
          exp_pass(std::integral_constant<int, 0>{});
        else if (np == 1)
          exp_pass(std::integral_constant<int, 1>{});
        else if (np == 2)
          exp_pass(std::integral_constant<int, 2>{});
        else
          exp_pass(std::integral_constant<int, 3>{});
        const float rs = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
        const float alpha = ptx::ex2(m2 - ref);  // 0 on the first tile, 1 when the reference stayed
        // S_t(j) was issued after PV_t(j-1) completed: O_t is current here
        if (j > 0 && !__all_sync(0xffffffffu, alpha == 1.f)) {
          for (int c = 0; c < 2 * NSUB; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(tO + 32 * c, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
        l = l * alpha + rs;
        m2 = ref;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(&p_full[t]));
      }
      ptx::mbar_wait(ptx::smem_u32(&o_done[t]), 0);
      ptx::tc_fence_after();
      const bool ok = q < a.S;
      store_acc_row(tO, NSUB, 1.f / l, a.o + (static_cast<int64_t>(row0) + q) * a.ldo + h * a.hd, a.hd, ok);
      if (ok) a.lse[(static_cast<int64_t>(b) * a.heads + h) * a.S + q] = (m2 + __log2f(l)) * 0.69314718055994531f;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// ------------------------------------------------------------------ D = rowsum(dO * O)
__global__ void attn_delta_kernel(const uint16_t* __restrict__ o, int64_t ldo, const uint16_t* __restrict__ dout,
                                  int64_t lddo, float* __restrict__ delta, int B, int S, int heads, int hd) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (b, h, t)
  if (idx >= static_cast<int64_t>(B) * heads * S) return;
  const int t = static_cast<int>(idx % S);
  const int h = static_cast<int>((idx / S) % heads);
  const int b = static_cast<int>(idx / (static_cast<int64_t>(S) * heads));
  const int64_t row = static_cast<int64_t>(b) * S + t;
  const uint16_t* po = o + row * ldo + h * hd;
  const uint16_t* pd = dout + row * lddo + h * hd;
  float acc = 0.f;
  for (int e = 0; e < hd; e += 8) {
    const uint4 x = *reinterpret_cast<const uint4*>(po + e);
    const uint4 y = *reinterpret_cast<const uint4*>(pd + e);
    const uint32_t xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc += __uint_as_float(xa[k] << 16) * __uint_as_float(ya[k] << 16);
      acc += __uint_as_float(xa[k] & 0xffff0000u) * __uint_as_float(ya[k] & 0xffff0000u);
    }
  }
  delta[idx] = acc;
}

// ------------------------------------------------------------------ dK, dV
template <int NSUB>
__global__ void __launch_bounds__(kThreads, 1) attn_dkv_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* k_s = sm;
  uint8_t* v_s = k_s + NSUB * kTile;
  uint8_t* q_s = v_s + NSUB * kTile;
  uint8_t* do_s = q_s + NSUB * kTile;
  uint8_t* pt_s = do_s + NSUB * kTile;  // P^T  [kv][q], 2 sub-tiles
  uint8_t* dst_s = pt_s + 2 * kTile;    // dS^T [kv][q]
  float* vec = reinterpret_cast<float*>(dst_s + 2 * kTile);  // [2][2][128]: lse2, delta per buffer
  uint64_t* bars = reinterpret_cast<uint64_t*>(vec + 512);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* dp_full = bars + 4;
  uint64_t* ps_full = bars + 5;
  uint64_t* ps_free = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gb = a.kvh * a.B;
  const int kblk = static_cast<int>(blockIdx.x) / gb;  // the first kv tiles have the most q tiles: first
  const int g = static_cast<int>(blockIdx.x) % a.kvh;
  const int b = (static_cast<int>(blockIdx.x) % gb) / a.kvh;
  const int grp = a.heads / a.kvh;
  const int k0 = kblk * kBM;
  const int nq = a.nqb - kblk;  // q tiles kblk .. nqb-1
  const int iters = grp * nq;
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 7; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), i == 5 ? 4 : 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(kv_full), 2 * NSUB * kTile);
      load_tile<NSUB>(&a.m.k, ptx::smem_u32(k_s), ptx::smem_u32(kv_full), g, row0 + k0);
      load_tile<NSUB>(&a.m.v, ptx::smem_u32(v_s), ptx::smem_u32(kv_full), g, row0 + k0);
      for (int t = 0; t < iters; ++t) {
        const int hq = g * grp + t / nq, i = kblk + t % nq;
        ptx::mbar_wait(ptx::smem_u32(qdo_empty), (t & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(qdo_full), 2 * NSUB * kTile);
        load_tile<NSUB>(&a.m.q, ptx::smem_u32(q_s), ptx::smem_u32(qdo_full), hq, row0 + i * kBM);
        load_tile<NSUB>(&a.m.dout, ptx::smem_u32(do_s), ptx::smem_u32(qdo_full), hq, row0 + i * kBM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      ptx::mbar_wait(ptx::smem_u32(kv_full), 0);
      for (int t = 0; t < iters; ++t) {
        ptx::mbar_wait(ptx::smem_u32(qdo_full), t & 1);
        ptx::tc_fence_after();
        mma_tile(tS, ptx::smem_u32(k_s), ptx::smem_u32(q_s), NSUB, 128, false, false);    // S^T = K Q^T
        ptx::umma_commit_cg1(ptx::smem_u32(s_full));
        mma_tile(tDP, ptx::smem_u32(v_s), ptx::smem_u32(do_s), NSUB, 128, false, false);  // dP^T = V dO^T
        ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
        ptx::mbar_wait(ptx::smem_u32(ps_full), t & 1);
        ptx::tc_fence_after();
        mma_tile(tDV, ptx::smem_u32(pt_s), ptx::smem_u32(do_s), 2, 64 * NSUB, true, t > 0);   // dV += P^T dO
        mma_tile(tDK, ptx::smem_u32(dst_s), ptx::smem_u32(q_s), 2, 64 * NSUB, true, t > 0);   // dK += dS^T Q
        ptx::umma_commit_cg1(ptx::smem_u32(qdo_empty));
        ptx::umma_commit_cg1(ptx::smem_u32(ps_free));
      }
    }
  } else if (warp >= 4) {  // one kv row per thread
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int kv = k0 + r;
    float p[128], ds[128];
    for (int t = 0; t < iters; ++t) {
      const int hq = g * grp + t / nq, i = kblk + t % nq;
      const int q0 = i * kBM;
      float* lse2 = vec + (t & 1) * 256;
      float* dl = lse2 + 128;
      {  // this q tile's lse (log2 units) and D into shared memory
        const int q = q0 + r;
        const int64_t o = (static_cast<int64_t>(b) * a.heads + hq) * a.S + q;
        lse2[r] = q < a.S ? a.lse[o] * kLog2e : INFINITY;  // rows past the sequence: P = 0
        dl[r] = q < a.S ? a.delta[o] : 0.f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      ptx::mbar_wait(ptx::smem_u32(s_full), t & 1);
      ptx::tc_fence_after();
      load_row(tS + lane_off, p);
      const bool diag = q0 == k0;  // the diagonal tile holds the q < kv entries
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        const float x = ptx::ex2(p[c] * a.scale2 - lse2[c]);
        p[c] = (diag && q0 + c < kv) ? 0.f : x;
      }
      ptx::mbar_wait(ptx::smem_u32(dp_full), t & 1);
      ptx::tc_fence_after();
      load_row(tDP + lane_off, ds);
#pragma unroll
      for (int c = 0; c < 128; ++c) ds[c] = p[c] * (ds[c] - dl[c]);
      if (t >= 1) ptx::mbar_wait(ptx::smem_u32(ps_free), (t - 1) & 1);
      store_row_bf16(pt_s, r, p);
      store_row_bf16(dst_s, r, ds);
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(ps_full));
    }
    ptx::mbar_wait(ptx::smem_u32(ps_free), (iters - 1) & 1);
    ptx::tc_fence_after();
    const bool ok = kv < a.S;
    const int64_t row = static_cast<int64_t>(row0) + kv;
    store_acc_row(tDV + lane_off, NSUB, 1.f, a.dv + row * a.lddv + g * a.hd, a.hd, ok);
    store_acc_row(tDK + lane_off, NSUB, a.scale, a.dk + row * a.lddk + g * a.hd, a.hd, ok);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// ------------------------------------------------------------------ dQ
template <int NSUB>
__global__ void __launch_bounds__(kThreads, 1) attn_dq_kernel(const __grid_constant__ Args a) {
  constexpr int kST = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = sm;
  uint8_t* do_s = q_s + NSUB * kTile;
  uint8_t* k_s = do_s + NSUB * kTile;        // [kST]
  uint8_t* v_s = k_s + kST * NSUB * kTile;   // [kST]
  uint8_t* ds_s = v_s + kST * NSUB * kTile;  // dS [q][kv], 2 sub-tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(ds_s + 2 * kTile);
  uint64_t* qdo_full = bars;
  uint64_t* kv_full = bars + 1;        // [kST]
  uint64_t* kv_empty = kv_full + kST;  // [kST]
  uint64_t* s_full = kv_empty + kST;
  uint64_t* dp_full = s_full + 1;
  uint64_t* ds_full = dp_full + 1;
  uint64_t* ds_free = ds_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ds_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = a.heads * a.B;
  const int qblk = a.nqb - 1 - static_cast<int>(blockIdx.x) / hb;
  const int h = static_cast<int>(blockIdx.x) % a.heads;
  const int b = (static_cast<int>(blockIdx.x) % hb) / a.heads;
  const int g = h / (a.heads / a.kvh);
  const int q0 = qblk * kBM;
  const int nblk = qblk + 1;
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(ptx::smem_u32(qdo_full), 1);
    for (int s = 0; s < kST; ++s) {
      ptx::mbar_init(ptx::smem_u32(&kv_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&kv_empty[s]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(s_full), 1);
    ptx::mbar_init(ptx::smem_u32(dp_full), 1);
    ptx::mbar_init(ptx::smem_u32(ds_full), 4);
    ptx::mbar_init(ptx::smem_u32(ds_free), 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tDP = tmem + 128, tDQ = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(qdo_full), 2 * NSUB * kTile);
      load_tile<NSUB>(&a.m.q, ptx::smem_u32(q_s), ptx::smem_u32(qdo_full), h, row0 + q0);
      load_tile<NSUB>(&a.m.dout, ptx::smem_u32(do_s), ptx::smem_u32(qdo_full), h, row0 + q0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&kv_empty[s]), ((j / kST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&kv_full[s]), 2 * NSUB * kTile);
        load_tile<NSUB>(&a.m.k, ptx::smem_u32(k_s + s * NSUB * kTile), ptx::smem_u32(&kv_full[s]), g, row0 + j * kBM);
        load_tile<NSUB>(&a.m.v, ptx::smem_u32(v_s + s * NSUB * kTile), ptx::smem_u32(&kv_full[s]), g, row0 + j * kBM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      ptx::mbar_wait(ptx::smem_u32(qdo_full), 0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kST;
        ptx::mbar_wait(ptx::smem_u32(&kv_full[s]), (j / kST) & 1);
        ptx::tc_fence_after();
        mma_tile(tS, ptx::smem_u32(q_s), ptx::smem_u32(k_s + s * NSUB * kTile), NSUB, 128, false, false);   // S
        ptx::umma_commit_cg1(ptx::smem_u32(s_full));
        mma_tile(tDP, ptx::smem_u32(do_s), ptx::smem_u32(v_s + s * NSUB * kTile), NSUB, 128, false, false);  // dP
        ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
        ptx::mbar_wait(ptx::smem_u32(ds_full), j & 1);
        ptx::tc_fence_after();
        mma_tile(tDQ, ptx::smem_u32(ds_s), ptx::smem_u32(k_s + s * NSUB * kTile), 2, 64 * NSUB, true, j > 0);  // dQ += dS K
        ptx::umma_commit_cg1(ptx::smem_u32(&kv_empty[s]));
        ptx::umma_commit_cg1(ptx::smem_u32(ds_free));
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int q = q0 + r;
    const bool ok = q < a.S;
    const int64_t o = (static_cast<int64_t>(b) * a.heads + h) * a.S + q;
    const float lse2 = ok ? a.lse[o] * kLog2e : INFINITY;
    const float dd = ok ? a.delta[o] : 0.f;
    float p[128], ds[128];
    for (int j = 0; j < nblk; ++j) {
      const int kv0 = j * kBM;
      ptx::mbar_wait(ptx::smem_u32(s_full), j & 1);
      ptx::tc_fence_after();
      load_row(tS + lane_off, p);
      const bool diag = kv0 + kBM - 1 > q0;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        const float x = ptx::ex2(p[c] * a.scale2 - lse2);
        p[c] = (diag && kv0 + c > q) ? 0.f : x;
      }
      ptx::mbar_wait(ptx::smem_u32(dp_full), j & 1);
      ptx::tc_fence_after();
      load_row(tDP + lane_off, ds);
#pragma unroll
      for (int c = 0; c < 128; ++c) ds[c] = p[c] * (ds[c] - dd);
      if (j >= 1) ptx::mbar_wait(ptx::smem_u32(ds_free), (j - 1) & 1);
      store_row_bf16(ds_s, r, ds);
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(ds_full));
    }
    ptx::mbar_wait(ptx::smem_u32(ds_free), (nblk - 1) & 1);
    ptx::tc_fence_after();
    store_acc_row(tDQ + lane_off, NSUB, a.scale, a.dq + (static_cast<int64_t>(row0) + q) * a.lddq + h * a.hd, a.hd,
                  ok);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// ------------------------------------------------------------------ backward v2
// Padded per-(b, head) rows of the log-sum-exp in log2 units (+inf past the
// sequence: P = 0 there) and of D = rowsum(dO * O), nqb * 128 entries each,
// so the dK/dV kernel's producer fetches a q tile's 128 values with one 512 B
// bulk copy next to its Q / dO tiles.
__global__ void attn_prep_kernel(const uint16_t* __restrict__ o, int64_t ldo, const uint16_t* __restrict__ dout,
                                 int64_t lddo, const float* __restrict__ lse, float* __restrict__ lse2p,
                                 float* __restrict__ deltap, int B, int S, int heads, int hd, int spad) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (b, h, t < spad)
  if (idx >= static_cast<int64_t>(B) * heads * spad) return;
  const int t = static_cast<int>(idx % spad);
  const int64_t bh = idx / spad;
  const int h = static_cast<int>(bh % heads);
  const int b = static_cast<int>(bh / heads);
  if (t >= S) {
    lse2p[idx] = INFINITY;
    deltap[idx] = 0.f;
    return;
  }
  const int64_t row = static_cast<int64_t>(b) * S + t;
  const uint16_t* po = o + row * ldo + h * hd;
  const uint16_t* pd = dout + row * lddo + h * hd;
  float acc = 0.f;
  for (int e = 0; e < hd; e += 8) {
    const uint4 x = *reinterpret_cast<const uint4*>(po + e);
    const uint4 y = *reinterpret_cast<const uint4*>(pd + e);
    const uint32_t xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc += __uint_as_float(xa[k] << 16) * __uint_as_float(ya[k] << 16);
      acc += __uint_as_float(xa[k] & 0xffff0000u) * __uint_as_float(ya[k] & 0xffff0000u);
    }
  }
  lse2p[idx] = lse[bh * S + t] * kLog2e;
  deltap[idx] = acc;
}

constexpr int kThreads2 = 384;  // backward v2: TMA / MMA / TMEM warpgroup + 8 math warps

// TMEM column of the k-th 16-deep K chunk of a packed bf16 A operand written
// by two math warps per row: q (or kv) columns 0..63 packed at base + 0..31,
// columns 64..127 at base + 64..95 (each half over its own fp32 columns).
__device__ __forceinline__ uint32_t pk(uint32_t base, int k) { return base + 8 * k + (k >= 4 ? 32 : 0); }

// Reads 64 columns (2 x 32) of this thread's TMEM row into v.
__device__ __forceinline__ void load64(uint32_t taddr, float (&v)[64]) {
  ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
  ptx::tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
}

// dK / dV, v2: P^T and dS^T go back into TMEM over the S^T / dP^T columns
// they came from (packed bf16) and feed the dV / dK GEMMs as TMEM A operands,
// so shared memory holds K, V and a 2-stage ring of {Q, dO, lse2, D} per q
// tile: the next tile's loads overlap the current tile's math.
template <int NSUB>
__global__ void __launch_bounds__(kThreads2, 1) attn_dkv2_kernel(const __grid_constant__ Args a) {
  constexpr int kVec = 1024;  // lse2[128] + D[128]
  constexpr int kStage = 2 * NSUB * kTile + kVec;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned by offsetting smem_raw itself (not through an integer cast), so
  // the compiler keeps the shared address space: LDS, not generic LD.E.
  uint8_t* sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* k_s = sm;
  uint8_t* v_s = k_s + NSUB * kTile;
  uint8_t* ring = v_s + NSUB * kTile;  // [2] {Q, dO, vec}
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + 2 * kStage);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;   // [2]
  uint64_t* qdo_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;   // S^T in TMEM
  uint64_t* ps_full = bars + 6;  // dS^T written (math -> MMA)
  uint64_t* ps_free = bars + 7;  // dV / dK of the tile done
  uint64_t* dp_full = bars + 8;  // dP^T in TMEM
  uint64_t* p_full = bars + 9;   // P^T written (math -> MMA)
  uint64_t* dv_done = bars + 10; // dV(t) has read P^T(t) (bwd_order 1)
  uint64_t* acc_done = bars + 11; // the last dK / dV MMA has completed (one phase)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gb = a.kvh * a.B;
  const int kblk = static_cast<int>(blockIdx.x) / gb;
  const int g = static_cast<int>(blockIdx.x) % a.kvh;
  const int b = (static_cast<int>(blockIdx.x) % gb) / a.kvh;
  const int grp = a.heads / a.kvh;
  const int k0 = kblk * kBM;
  const int nq = a.nqb - kblk;
  const int iters = grp * nq;
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(ptx::smem_u32(kv_full), 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&qdo_full[i]), 1);
      // the MMA commit after dK(t) + the 8 math warps once they are done with
      // the stage's lse2 / D (the bulk copy of t+2 overwrites them)
      ptx::mbar_init(ptx::smem_u32(&qdo_empty[i]), 9);
    }
    ptx::mbar_init(ptx::smem_u32(s_full), 1);
    ptx::mbar_init(ptx::smem_u32(ps_full), 8);
    ptx::mbar_init(ptx::smem_u32(ps_free), 1);
    ptx::mbar_init(ptx::smem_u32(dp_full), 1);
    ptx::mbar_init(ptx::smem_u32(p_full), 8);
    ptx::mbar_init(ptx::smem_u32(dv_done), 1);
    ptx::mbar_init(ptx::smem_u32(acc_done), 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  // Register pool (launched at 168 per thread): warpgroup 0 (TMA, MMA, TMEM
  // allocator) gives up 128 x (168 - 96) = 9216, the two math warpgroups take
  // 256 x (200 - 168) = 8192 of them (an .inc the pool cannot cover blocks forever).
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(kv_full), 2 * NSUB * kTile);
      load_tile<NSUB>(&a.m.k, ptx::smem_u32(k_s), ptx::smem_u32(kv_full), g, row0 + k0);
      load_tile<NSUB>(&a.m.v, ptx::smem_u32(v_s), ptx::smem_u32(kv_full), g, row0 + k0);
      for (int t = 0; t < iters; ++t) {
        const int hq = g * grp + t / nq, i = kblk + t % nq;
        const int st = t & 1;
        uint8_t* stage = ring + st * kStage;
        ptx::mbar_wait(ptx::smem_u32(&qdo_empty[st]), ((t >> 1) & 1) ^ 1);
        const uint32_t fb = ptx::smem_u32(&qdo_full[st]);
        ptx::mbar_arrive_expect_tx(fb, 2 * NSUB * kTile + kVec);
        load_tile<NSUB>(&a.m.q, ptx::smem_u32(stage), fb, hq, row0 + i * kBM);
        load_tile<NSUB>(&a.m.dout, ptx::smem_u32(stage + NSUB * kTile), fb, hq, row0 + i * kBM);
        const int64_t vo = ((static_cast<int64_t>(b) * a.heads + hq) * a.nqb + i) * kBM;
        ptx::bulk_load_1d(ptx::smem_u32(stage + 2 * NSUB * kTile), a.lse2p + vo, 512, fb);
        ptx::bulk_load_1d(ptx::smem_u32(stage + 2 * NSUB * kTile + 512), a.deltap + vo, 512, fb);
      }
    }
  } else if (warp == 1 && (a.bwd_order & 1)) {
    // Issue order with the next tile's scores under this tile's dS pass:
    //   S^T(0) dP^T(0) | per t: [P^T(t)] dV(t), S^T(t+1) | [dS^T(t)] dK(t), dP^T(t+1)
    // S^T(t+1) overwrites the P^T(t) columns once dV(t) has read them and
    // dP^T(t+1) the dS^T(t) columns once dK(t) has; the math warps run the
    // dS pass of t while the tensor core runs dV(t) + S^T(t+1), and the exp
    // pass of t+1 while it runs dK(t) + dP^T(t+1).  (Order 0 issues S^T(t+1)
    // only after dK(t) completes: the exp pass of t+1 then waits for dK(t)
    // and S^T(t+1) in series.)
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, 64 * NSUB, 0, 1);
      ptx::mbar_wait(ptx::smem_u32(kv_full), 0);
      ptx::mbar_wait(ptx::smem_u32(&qdo_full[0]), 0);
      ptx::tc_fence_after();
      {
        const uint32_t qs = ptx::smem_u32(ring), dos = qs + NSUB * kTile;
        mma_tile(tS, ptx::smem_u32(k_s), qs, NSUB, 128, false, false);    // S^T = K Q^T
        ptx::umma_commit_cg1(ptx::smem_u32(s_full));
        mma_tile(tDP, ptx::smem_u32(v_s), dos, NSUB, 128, false, false);  // dP^T = V dO^T
        ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
      }
      for (int t = 0; t < iters; ++t) {
        const int st = t & 1;
        const uint32_t qs = ptx::smem_u32(ring + st * kStage), dos = qs + NSUB * kTile;
        const bool more = t + 1 < iters;
        const uint32_t qn = ptx::smem_u32(ring + (st ^ 1) * kStage), don = qn + NSUB * kTile;
        ptx::mbar_wait(ptx::smem_u32(p_full), t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // dV += P^T dO (under the dS pass)
          ptx::umma_bf16_tmem_a_cg1(tDV, pk(tS, k), mdesc(dos + k * 2048), idesc, (t > 0 || k) ? 1u : 0u);
        if (more) {
          ptx::mbar_wait(ptx::smem_u32(&qdo_full[st ^ 1]), ((t + 1) >> 1) & 1);
          if (!a.inorder) {
            ptx::umma_commit_cg1(ptx::smem_u32(dv_done));
            ptx::mbar_wait(ptx::smem_u32(dv_done), t & 1);
          }
          ptx::tc_fence_after();
          mma_tile(tS, ptx::smem_u32(k_s), qn, NSUB, 128, false, false);  // S^T(t+1) (under the dS pass)
          ptx::umma_commit_cg1(ptx::smem_u32(s_full));
        }
        ptx::mbar_wait(ptx::smem_u32(ps_full), t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // dK += dS^T Q (under the next exp pass)
          ptx::umma_bf16_tmem_a_cg1(tDK, pk(tDP, k), mdesc(qs + k * 2048), idesc, (t > 0 || k) ? 1u : 0u);
        ptx::umma_commit_cg1(ptx::smem_u32(&qdo_empty[st]));
        // ps_free phases are committed only where they are waited for (each
        // phase observed before the next completes); acc_done ends the tile
        if (more && !a.inorder) ptx::umma_commit_cg1(ptx::smem_u32(ps_free));
        if (!more) ptx::umma_commit_cg1(ptx::smem_u32(acc_done));
        if (more) {
          if (!a.inorder) ptx::mbar_wait(ptx::smem_u32(ps_free), t & 1);  // dK(t) read dS^T(t)
          ptx::tc_fence_after();
          mma_tile(tDP, ptx::smem_u32(v_s), don, NSUB, 128, false, false);  // dP^T(t+1)
          ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, 64 * NSUB, 0, 1);
      ptx::mbar_wait(ptx::smem_u32(kv_full), 0);
      for (int t = 0; t < iters; ++t) {
        const int st = t & 1;
        const uint32_t qs = ptx::smem_u32(ring + st * kStage), dos = qs + NSUB * kTile;
        ptx::mbar_wait(ptx::smem_u32(&qdo_full[st]), (t >> 1) & 1);
        if (t > 0 && !a.inorder) ptx::mbar_wait(ptx::smem_u32(ps_free), (t - 1) & 1);  // dV/dK(t-1) read P^T/dS^T
        ptx::tc_fence_after();
        mma_tile(tS, ptx::smem_u32(k_s), qs, NSUB, 128, false, false);    // S^T = K Q^T
        ptx::umma_commit_cg1(ptx::smem_u32(s_full));
        mma_tile(tDP, ptx::smem_u32(v_s), dos, NSUB, 128, false, false);  // dP^T = V dO^T (under the exp pass)
        ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
        ptx::mbar_wait(ptx::smem_u32(p_full), t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // dV += P^T dO (under the dS pass)
          ptx::umma_bf16_tmem_a_cg1(tDV, pk(tS, k), mdesc(dos + k * 2048), idesc, (t > 0 || k) ? 1u : 0u);
        ptx::mbar_wait(ptx::smem_u32(ps_full), t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // dK += dS^T Q
          ptx::umma_bf16_tmem_a_cg1(tDK, pk(tDP, k), mdesc(qs + k * 2048), idesc, (t > 0 || k) ? 1u : 0u);
        ptx::umma_commit_cg1(ptx::smem_u32(&qdo_empty[st]));
        if (t + 1 < iters && !a.inorder) ptx::umma_commit_cg1(ptx::smem_u32(ps_free));
        if (t + 1 == iters) ptx::umma_commit_cg1(ptx::smem_u32(acc_done));
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    // 8 math warps: kv row (warp & 3) * 32 + lane (the TMEM lane quadrant of
    // the warp), q columns [64 hf, 64 hf + 64): two warps per SM sub-partition
    // interleave their dependency chains.  Each half packs its bf16 P^T / dS^T
    // over its OWN fp32 columns (cb .. cb + 31), so the halves never overwrite
    // columns the other still reads; the GEMMs read the two packed halves
    // through pk().
    const int hf = (warp - 4) >> 2, cb = 64 * hf;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int r = (warp & 3) * 32 + lane;
    const int kv = k0 + r;
    for (int t = 0; t < iters; ++t) {
      const int i = kblk + t % nq;
      const int q0 = i * kBM;
      const int st = t & 1;
      const float* vec = reinterpret_cast<const float*>(ring + st * kStage + 2 * NSUB * kTile) + cb;
      ptx::mbar_wait(ptx::smem_u32(&qdo_full[st]), (t >> 1) & 1);  // lse2 / D visible
      ptx::mbar_wait(ptx::smem_u32(s_full), t & 1);
      ptx::tc_fence_after();
      const int nmask = (q0 == k0 ? r : 0) - cb;  // diagonal tile: columns q < kv are masked
      float p[64];
      load64(tS + lane_off + cb, p);
      ptx::tmem_ld_wait();
      uint32_t pp[32];
      if (nmask > 0) {
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          float p0 = ptx::ex2(fmaf(p[e], a.scale2, -vec[e]));
          float p1 = ptx::ex2(fmaf(p[e + 1], a.scale2, -vec[e + 1]));
          if (e < nmask) p0 = 0.f;
          if (e + 1 < nmask) p1 = 0.f;
          p[e] = p0;
          p[e + 1] = p1;
          pp[e >> 1] = ptx::pack_bf16(p0, p1);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          p[e] = ptx::ex2(fmaf(p[e], a.scale2, -vec[e]));
          p[e + 1] = ptx::ex2(fmaf(p[e + 1], a.scale2, -vec[e + 1]));
          pp[e >> 1] = ptx::pack_bf16(p[e], p[e + 1]);
        }
      }
      ptx::tmem_st_32x32b_x32(tS + lane_off + cb, pp);  // P^T half, packed over its own columns
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(p_full));  // dV GEMM may start
      ptx::mbar_wait(ptx::smem_u32(dp_full), t & 1);
      ptx::tc_fence_after();
      {  // dS^T = P^T (dP^T - D): one TMEM load of the 64 columns (one exposed load latency)
        float y[64];
        load64(tDP + lane_off + cb, y);
        ptx::tmem_ld_wait();
        uint32_t dd[32];
#pragma unroll
        for (int e = 0; e < 64; e += 2)
          dd[e >> 1] = ptx::pack_bf16(p[e] * (y[e] - vec[128 + e]), p[e + 1] * (y[e + 1] - vec[128 + e + 1]));
        ptx::tmem_st_32x32b_x32(tDP + lane_off + cb, dd);  // packed over its own columns
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_local(ptx::smem_u32(ps_full));
        // lse2 / D of this stage read (generic proxy) before the producer's
        // bulk copy (async proxy) of t + 2 overwrites them
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive_local(ptx::smem_u32(&qdo_empty[st]));
      }
    }
    ptx::mbar_wait(ptx::smem_u32(acc_done), 0);
    ptx::tc_fence_after();
    const bool ok = kv < a.S;
    const int64_t row = static_cast<int64_t>(row0) + kv;
    if (hf == 0)
      store_acc_row(tDV + lane_off, NSUB, 1.f, a.dv + row * a.lddv + g * a.hd, a.hd, ok);
    else
      store_acc_row(tDK + lane_off, NSUB, a.scale, a.dk + row * a.lddk + g * a.hd, a.hd, ok);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// dQ, v2: dS goes back into TMEM (over S, order bit 1, or over dP) and feeds
// dQ += dS K as the TMEM A operand; shared memory holds Q, dO, a 3-stage K
// ring and a 2-stage V ring (K(j) is held until dQ(j), V(j) only until dP(j),
// so with three K stages the scores two tiles ahead never wait for a K load
// that could only start after dQ(j)).
template <int NSUB>
__global__ void __launch_bounds__(kThreads2, 1) attn_dq2_kernel(const __grid_constant__ Args a) {
  constexpr int kKS = 3, kVS = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned by offsetting smem_raw itself (not through an integer cast), so
  // the compiler keeps the shared address space: LDS, not generic LD.E.
  uint8_t* sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* q_s = sm;
  uint8_t* do_s = q_s + NSUB * kTile;
  uint8_t* k_s = do_s + NSUB * kTile;        // [kKS]
  uint8_t* v_s = k_s + kKS * NSUB * kTile;   // [kVS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(v_s + kVS * NSUB * kTile);
  uint64_t* qdo_full = bars;
  uint64_t* k_full = bars + 1;        // [kKS]
  uint64_t* k_empty = k_full + kKS;   // [kKS]
  uint64_t* v_full = k_empty + kKS;   // [kVS]
  uint64_t* v_empty = v_full + kVS;   // [kVS]
  uint64_t* s_full = v_empty + kVS;   // [2]: S double-buffered in TMEM
  uint64_t* ds_full = s_full + 2;
  uint64_t* ds_free = ds_full + 1;
  uint64_t* dp_full = ds_free + 1;
  uint64_t* acc_done = dp_full + 1;  // the last dQ MMA has completed (one phase)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = a.heads * a.B;
  const int qblk = a.nqb - 1 - static_cast<int>(blockIdx.x) / hb;
  const int h = static_cast<int>(blockIdx.x) % a.heads;
  const int b = (static_cast<int>(blockIdx.x) % hb) / a.heads;
  const int g = h / (a.heads / a.kvh);
  const int q0 = qblk * kBM;
  const int nblk = qblk + 1;
  const int row0 = b * a.S;

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(ptx::smem_u32(qdo_full), 1);
    for (int s = 0; s < kKS; ++s) {
      ptx::mbar_init(ptx::smem_u32(&k_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&k_empty[s]), 1);
    }
    for (int s = 0; s < kVS; ++s) {
      ptx::mbar_init(ptx::smem_u32(&v_full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&v_empty[s]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(&s_full[0]), 1);
    ptx::mbar_init(ptx::smem_u32(&s_full[1]), 1);
    ptx::mbar_init(ptx::smem_u32(ds_full), 8);
    ptx::mbar_init(ptx::smem_u32(ds_free), 1);
    ptx::mbar_init(ptx::smem_u32(dp_full), 1);
    ptx::mbar_init(ptx::smem_u32(acc_done), 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS2[2] = {tmem, tmem + 128}, tDP = tmem + 256, tDQ = tmem + 384;
  auto kst = [&](int j) { return ptx::smem_u32(k_s + (j % kKS) * NSUB * kTile); };
  auto vst = [&](int j) { return ptx::smem_u32(v_s + (j % kVS) * NSUB * kTile); };

  // Register pool (launched at 168 per thread): warpgroup 0 (TMA, MMA, TMEM
  // allocator) gives up 128 x (168 - 96) = 9216, the two math warpgroups take
  // 256 x (200 - 168) = 8192 of them (an .inc the pool cannot cover blocks forever).
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
  if (warp == 0) {  // Q, dO, then the K ring
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(qdo_full), 2 * NSUB * kTile);
      load_tile<NSUB>(&a.m.q, ptx::smem_u32(q_s), ptx::smem_u32(qdo_full), h, row0 + q0);
      load_tile<NSUB>(&a.m.dout, ptx::smem_u32(do_s), ptx::smem_u32(qdo_full), h, row0 + q0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kKS;
        ptx::mbar_wait(ptx::smem_u32(&k_empty[s]), ((j / kKS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&k_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.k, kst(j), ptx::smem_u32(&k_full[s]), g, row0 + j * kBM);
      }
    }
  } else if (warp == 3) {  // the V ring
    if (lane == 0) {
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kVS;
        ptx::mbar_wait(ptx::smem_u32(&v_empty[s]), ((j / kVS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&v_full[s]), NSUB * kTile);
        load_tile<NSUB>(&a.m.v, vst(j), ptx::smem_u32(&v_full[s]), g, row0 + j * kBM);
      }
    }
  } else if (warp == 1) {
    // order bit 1: dS(j) goes over S(j)'s buffer (the exp pass has read it into
    // registers), so dP(j+1) needs only the dS pass of j to be done, not dQ(j):
    //   S(0) dP(0) S(1) | per j: [dS(j)] dQ(j), dP(j+1), S(j+2) once dQ(j) has read dS(j)
    // otherwise dS(j) goes over dP(j):
    //   S(0) | per j: dP(j) once dQ(j-1) has read dS(j-1), S(j+1) | [dS(j)] dQ(j)
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, 64 * NSUB, 0, 1);
      const bool ds_over_s = (a.bwd_order & 2) != 0;
      ptx::mbar_wait(ptx::smem_u32(qdo_full), 0);
      auto s_mma = [&](int j) {  // S(j) = Q K_j^T into buffer j & 1
        ptx::mbar_wait(ptx::smem_u32(&k_full[j % kKS]), (j / kKS) & 1);
        ptx::tc_fence_after();
        mma_tile(tS2[j & 1], ptx::smem_u32(q_s), kst(j), NSUB, 128, false, false);
        ptx::umma_commit_cg1(ptx::smem_u32(&s_full[j & 1]));
      };
      auto dp_mma = [&](int j) {  // dP(j) = dO V_j^T
        ptx::mbar_wait(ptx::smem_u32(&v_full[j % kVS]), (j / kVS) & 1);
        ptx::tc_fence_after();
        mma_tile(tDP, ptx::smem_u32(do_s), vst(j), NSUB, 128, false, false);
        ptx::umma_commit_cg1(ptx::smem_u32(dp_full));
        ptx::umma_commit_cg1(ptx::smem_u32(&v_empty[j % kVS]));
      };
      // dQ += dS K (dS from TMEM, K MN-major).  ds_free phases are committed
      // only where the issuer waits for them (`free_waited`), so every phase
      // is observed before the next completes; acc_done ends the tile.
      auto dq_mma = [&](int j, uint32_t ds, bool free_waited) {
        ptx::mbar_wait(ptx::smem_u32(ds_full), j & 1);
        ptx::tc_fence_after();
        const uint32_t ks = kst(j);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::umma_bf16_tmem_a_cg1(tDQ, pk(ds, k), mdesc(ks + k * 2048), idesc, (j > 0 || k) ? 1u : 0u);
        ptx::umma_commit_cg1(ptx::smem_u32(&k_empty[j % kKS]));
        if (free_waited && !a.inorder) ptx::umma_commit_cg1(ptx::smem_u32(ds_free));
        if (j + 1 == nblk) ptx::umma_commit_cg1(ptx::smem_u32(acc_done));
      };
      if (ds_over_s) {
        s_mma(0);
        dp_mma(0);
        if (nblk > 1) s_mma(1);
        for (int j = 0; j < nblk; ++j) {
          dq_mma(j, tS2[j & 1], j + 2 < nblk);
          if (j + 1 < nblk) dp_mma(j + 1);  // the dS pass of j has read dP(j)
          if (j + 2 < nblk) {
            if (!a.inorder) ptx::mbar_wait(ptx::smem_u32(ds_free), j & 1);  // dQ(j) read dS(j)
            s_mma(j + 2);
          }
        }
      } else {
        s_mma(0);
        for (int j = 0; j < nblk; ++j) {
          if (j > 0 && !a.inorder) ptx::mbar_wait(ptx::smem_u32(ds_free), (j - 1) & 1);  // dQ(j-1) read dS
          dp_mma(j);
          if (j + 1 < nblk) s_mma(j + 1);  // the next scores under this tile's dS pass
          dq_mma(j, tDP, j + 1 < nblk);
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    // 8 math warps: q row (warp & 3) * 32 + lane, kv columns [64 hf, 64 hf + 64)
    // (two warps per sub-partition; each half packs dS over its own columns, pk()).
    const int hf = (warp - 4) >> 2, cb = 64 * hf;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int r = (warp & 3) * 32 + lane;
    const int q = q0 + r;
    const bool ok = q < a.S;
    const int64_t o = (static_cast<int64_t>(b) * a.heads + h) * (a.nqb * kBM) + q;  // padded rows
    const float lse2 = a.lse2p[o];
    const float dd = a.deltap[o];
    for (int j = 0; j < nblk; ++j) {
      const int kv0 = j * kBM;
      ptx::mbar_wait(ptx::smem_u32(&s_full[j & 1]), (j >> 1) & 1);
      ptx::tc_fence_after();
      const int nvalid = (kv0 + kBM - 1 > q0 ? q - kv0 + 1 : kBM) - cb;  // kv columns <= q
      float p[64];
      load64(tS2[j & 1] + lane_off + cb, p);
      ptx::tmem_ld_wait();
      if (nvalid < 64) {
#pragma unroll
        for (int e = 0; e < 64; ++e) {  // P (the exp pass runs under the dP GEMM)
          const float x = ptx::ex2(fmaf(p[e], a.scale2, -lse2));
          p[e] = e < nvalid ? x : 0.f;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 64; ++e) p[e] = ptx::ex2(fmaf(p[e], a.scale2, -lse2));
      }
      ptx::mbar_wait(ptx::smem_u32(dp_full), j & 1);
      ptx::tc_fence_after();
      const uint32_t tDS = (a.bwd_order & 2) ? tS2[j & 1] : tDP;
      {  // one TMEM load of the 64 columns (one exposed load latency)
        float y[64];
        load64(tDP + lane_off + cb, y);
        ptx::tmem_ld_wait();
        uint32_t d2[32];
#pragma unroll
        for (int e = 0; e < 64; e += 2) d2[e >> 1] = ptx::pack_bf16(p[e] * (y[e] - dd), p[e + 1] * (y[e + 1] - dd));
        ptx::tmem_st_32x32b_x32(tDS + lane_off + cb, d2);  // dS over read S (order bit 1) or dP columns
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(ptx::smem_u32(ds_full));
    }
    ptx::mbar_wait(ptx::smem_u32(acc_done), 0);
    ptx::tc_fence_after();
    // dQ columns [64 hf, 64 hf + 64) of this row
    if (cb < a.hd)
      store_acc_row(tDQ + lane_off + cb, 1, a.scale,
                    a.dq + (static_cast<int64_t>(row0) + q) * a.lddq + h * a.hd + cb, a.hd - cb, ok);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
template <int NSUB>
constexpr int fwd_smem() {
  return 1024 + NSUB * kTile + 2 * (NSUB == 1 ? 3 : 2) * NSUB * kTile + 2 * kTile + 256;
}
template <int NSUB>
constexpr int fwd2_smem() {
  return 1024 + 2 * NSUB * kTile + 4 * NSUB * kTile + 256;
}
template <int NSUB>
constexpr int dkv2_smem() {
  return 1024 + 2 * NSUB * kTile + 2 * (2 * NSUB * kTile + 1024) + 256;  // bars: 12 x 8 B + TMEM slot
}
template <int NSUB>
constexpr int dq2_smem() {  // Q, dO, 3 K stages, 2 V stages, bars
  return 1024 + 2 * NSUB * kTile + 5 * NSUB * kTile + 256;
}
template <int NSUB>
constexpr int dkv_smem() {
  return 1024 + 4 * NSUB * kTile + 4 * kTile + 2048 + 256;
}
template <int NSUB>
constexpr int dq_smem() {
  return 1024 + 2 * NSUB * kTile + 4 * NSUB * kTile + 2 * kTile + 256;
}
static_assert(fwd_smem<2>() <= 232448 && fwd2_smem<2>() <= 232448 && dkv_smem<2>() <= 232448 &&
                  dq_smem<2>() <= 232448,
              "shared memory");

static_assert(dkv2_smem<2>() <= 232448 && dq2_smem<2>() <= 232448, "shared memory");

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int encode(void* enc, CUtensorMap* m, const void* base, int64_t ld, int64_t rows, int heads, int hd) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeFn>(enc)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                                               strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : static_cast<int>(r);
}

template <int NSUB>
static cudaError_t set_attrs() {
  cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem<NSUB>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_fwd2_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd2_smem<NSUB>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_dkv_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, dkv_smem<NSUB>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_dq_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, dq_smem<NSUB>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_dkv2_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, dkv2_smem<NSUB>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_dq2_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, dq2_smem<NSUB>());
  return e;
}

// Shared-memory limits of every attention kernel on the current device: once
// per context (mst_ctx_create), like the GEMM engine's, since a function
// attribute is per device.
cudaError_t init_device() {
  cudaError_t e = set_attrs<1>();
  return e == cudaSuccess ? set_attrs<2>() : e;
}

int forward(void* enc, cudaStream_t st, const AttnTuning& tune, const AttnShape& s, const void* q, int64_t ldq, const void* k, int64_t ldk,
            const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, const char** err) {
  Args a;
  std::memset(&a, 0, sizeof(a));
  const int64_t rows = static_cast<int64_t>(s.B) * s.S;
  if (encode(enc, &a.m.q, q, ldq, rows, s.heads, s.hd) || encode(enc, &a.m.k, k, ldk, rows, s.kvh, s.hd) ||
      encode(enc, &a.m.v, v, ldv, rows, s.kvh, s.hd)) {
    *err = "cuTensorMapEncodeTiled failed for an attention operand";
    return 1;
  }
  a.o = static_cast<uint16_t*>(o);
  a.ldo = ldo;
  a.lse = lse;
  a.B = s.B;
  a.S = s.S;
  a.heads = s.heads;
  a.kvh = s.kvh;
  a.hd = s.hd;
  a.scale = 1.f / sqrtf(static_cast<float>(s.hd));
  a.scale2 = a.scale * kLog2e;
  a.nqb = (s.S + kBM - 1) / kBM;
  a.inorder = tune.mma_inorder;
  a.poly = tune.poly_exp;
  const dim3 grid(static_cast<unsigned>(a.nqb * s.heads * s.B));
  const dim3 grid2(static_cast<unsigned>((a.nqb + 1) / 2 * s.heads * s.B));
  cudaError_t e;
  thread_local char msg[256];
  if (s.hd <= 64) {
    if (tune.fwd_version == 2)
      attn_fwd2_kernel<1><<<grid2, 384, fwd2_smem<1>(), st>>>(a);
    else
      attn_fwd_kernel<1><<<grid, kThreads, fwd_smem<1>(), st>>>(a);
  } else {
    if (tune.fwd_version == 2)
      attn_fwd2_kernel<2><<<grid2, 384, fwd2_smem<2>(), st>>>(a);
    else
      attn_fwd_kernel<2><<<grid, kThreads, fwd_smem<2>(), st>>>(a);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, s.hd <= 64 ? (const void*)attn_fwd2_kernel<1> : (const void*)attn_fwd2_kernel<2>);
    snprintf(msg, sizeof(msg), "%s (fwd v%d: %d regs, max %d threads, %zu B static smem, %zu B local)",
             cudaGetErrorString(e), tune.fwd_version, fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
             fa.localSizeBytes);
    *err = msg;
    return 2;
  }
  return 0;
}

int backward(void* enc, cudaStream_t st, const AttnTuning& tune, const AttnShape& s, const void* q, int64_t ldq, const void* k, int64_t ldk,
             const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo, const float* lse,
             void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv, float* delta, const char** err) {
  Args a;
  std::memset(&a, 0, sizeof(a));
  const int64_t rows = static_cast<int64_t>(s.B) * s.S;
  if (encode(enc, &a.m.q, q, ldq, rows, s.heads, s.hd) || encode(enc, &a.m.k, k, ldk, rows, s.kvh, s.hd) ||
      encode(enc, &a.m.v, v, ldv, rows, s.kvh, s.hd) || encode(enc, &a.m.dout, dout, lddo, rows, s.heads, s.hd)) {
    *err = "cuTensorMapEncodeTiled failed for an attention operand";
    return 1;
  }
  a.lse = const_cast<float*>(lse);
  a.delta = delta;
  a.dq = static_cast<uint16_t*>(dq);
  a.dk = static_cast<uint16_t*>(dk);
  a.dv = static_cast<uint16_t*>(dv);
  a.lddq = lddq;
  a.lddk = lddk;
  a.lddv = lddv;
  a.B = s.B;
  a.S = s.S;
  a.heads = s.heads;
  a.kvh = s.kvh;
  a.hd = s.hd;
  a.scale = 1.f / sqrtf(static_cast<float>(s.hd));
  a.scale2 = a.scale * kLog2e;
  a.nqb = (s.S + kBM - 1) / kBM;
  a.inorder = tune.mma_inorder;
  a.bwd_order = tune.bwd_order;
  const int64_t nrow = static_cast<int64_t>(s.B) * s.heads * s.S;
  const dim3 gkv(static_cast<unsigned>(a.nqb * s.kvh * s.B)), gq(static_cast<unsigned>(a.nqb * s.heads * s.B));
  cudaError_t e;
  if (tune.bwd_version == 2) {
    // workspace: delta [B*heads*S] | lse2p [B*heads*spad] | deltap [B*heads*spad]
    const int spad = a.nqb * kBM;
    float* lse2p = delta + ((nrow + 63) / 64) * 64;
    float* deltap = lse2p + static_cast<int64_t>(s.B) * s.heads * spad;
    a.lse2p = lse2p;
    a.deltap = deltap;
    const int64_t np = static_cast<int64_t>(s.B) * s.heads * spad;
    attn_prep_kernel<<<static_cast<unsigned>((np + 255) / 256), 256, 0, st>>>(
        static_cast<const uint16_t*>(o), ldo, static_cast<const uint16_t*>(dout), lddo, lse, lse2p, deltap, s.B, s.S,
        s.heads, s.hd, spad);
    if (s.hd <= 64) {
      attn_dkv2_kernel<1><<<gkv, kThreads2, dkv2_smem<1>(), st>>>(a);
      attn_dq2_kernel<1><<<gq, kThreads2, dq2_smem<1>(), st>>>(a);
    } else {
      attn_dkv2_kernel<2><<<gkv, kThreads2, dkv2_smem<2>(), st>>>(a);
      attn_dq2_kernel<2><<<gq, kThreads2, dq2_smem<2>(), st>>>(a);
    }
  } else {
    attn_delta_kernel<<<static_cast<unsigned>((nrow + 255) / 256), 256, 0, st>>>(
        static_cast<const uint16_t*>(o), ldo, static_cast<const uint16_t*>(dout), lddo, delta, s.B, s.S, s.heads, s.hd);
    if (s.hd <= 64) {
      attn_dkv_kernel<1><<<gkv, kThreads, dkv_smem<1>(), st>>>(a);
      attn_dq_kernel<1><<<gq, kThreads, dq_smem<1>(), st>>>(a);
    } else {
      attn_dkv_kernel<2><<<gkv, kThreads, dkv_smem<2>(), st>>>(a);
      attn_dq_kernel<2><<<gq, kThreads, dq_smem<2>(), st>>>(a);
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return *err = cudaGetErrorString(e), 2;
  return 0;
}

}  // namespace mst_attn
