// Decoder-layer plumbing around the MsT blocks (the
// reference's blocks-std rmsnorm / embedding, SPEC.md:242-250 and the model
// module SPEC.md:410-469): HBM-bound sm_100a kernels.
//
//   rmsnorm_fwd_kernel  s = x (+ r); y = s * g * rstd, rstd = 1/sqrt(mean(s^2) + eps)
//                       (residual add fused: the residual stream s is written once)
//   rmsnorm_bwd_kernel  dx = rstd * (g*dy - s * rstd^2 * mean(g*dy*s)) (+ d_res),
//                       per-block fp32 partials of dgain = sum_rows dy * s * rstd
//   rmsnorm_dgain_kernel  fixed-order sum of the partials (+= dgain)
//   embed_fwd_kernel    out[t] = E[token[t]]
//   embed_bwd_kernel    dE[v] (+)= sum of dX rows of the positions holding v, in
//                       position order (positions pre-grouped by token: deterministic)
//
// One warp per row (d <= 8192, 16-byte vector accesses), rows grid-strided.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layers.cuh"

namespace mst_layers {

constexpr int kWarps = 8;  // rows in flight per 256-thread block

__device__ __forceinline__ float bf(uint16_t v) { return __uint_as_float(static_cast<uint32_t>(v) << 16); }
__device__ __forceinline__ uint16_t tobf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 8 bf16 <-> float helpers on one 16-byte vector
__device__ __forceinline__ void unpack8(uint4 w, float* f) {
  const uint32_t q[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = __uint_as_float(q[j] << 16);
    f[2 * j + 1] = __uint_as_float(q[j] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint32_t q[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) q[j] = static_cast<uint32_t>(tobf(f[2 * j])) | (static_cast<uint32_t>(tobf(f[2 * j + 1])) << 16);
  return make_uint4(q[0], q[1], q[2], q[3]);
}

// d % 8 == 0; each lane owns columns [8*(lane + 32*c), +8) for c < d/256 (ceil).
__global__ void __launch_bounds__(256) rmsnorm_fwd_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ r,
                                                          const float* __restrict__ g, uint16_t* __restrict__ y,
                                                          uint16_t* __restrict__ s_out, float* __restrict__ rstd,
                                                          int64_t n, int d, float eps) {
  const int lane = threadIdx.x & 31;
  const int nvec = d / 8;
  for (int64_t row = blockIdx.x * (int64_t)kWarps + (threadIdx.x >> 5); row < n; row += (int64_t)gridDim.x * kWarps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * d);
    const uint4* rr = r ? reinterpret_cast<const uint4*>(r + row * d) : nullptr;
    float ss = 0.f;
    for (int v = lane; v < nvec; v += 32) {
      float a[8];
      unpack8(xr[v], a);
      if (rr) {
        float b[8];
        unpack8(rr[v], b);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += b[j];
        // the residual stream is stored in bf16; normalise the stored value
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = bf(tobf(a[j]));
        reinterpret_cast<uint4*>(s_out + row * d)[v] = pack8(a);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += a[j] * a[j];
    }
    ss = warp_sum(ss);
    const float rs = rsqrtf(ss / (float)d + eps);
    if (lane == 0) rstd[row] = rs;
    const uint4* sr = rr ? reinterpret_cast<const uint4*>(s_out + row * d) : xr;
    for (int v = lane; v < nvec; v += 32) {
      float a[8];
      unpack8(sr[v], a);
      const float4 g0 = reinterpret_cast<const float4*>(g)[2 * v], g1 = reinterpret_cast<const float4*>(g)[2 * v + 1];
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = a[j] * rs * gg[j];
      reinterpret_cast<uint4*>(y + row * d)[v] = pack8(a);
    }
  }
}

// One block = kWarps rows at a time; per-block dgain partials [gridDim.x, d] fp32.
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const uint16_t* __restrict__ s, const float* __restrict__ g,
                                                          const float* __restrict__ rstd, const uint16_t* __restrict__ dy,
                                                          const uint16_t* __restrict__ dres, uint16_t* __restrict__ dx,
                                                          float* __restrict__ part, int64_t n, int d) {
  extern __shared__ float sm[];  // [kWarps][d] dgain accumulators of this block's warps
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nvec = d / 8;
  float* acc = sm + w * d;
  for (int c = lane; c < d; c += 32) acc[c] = 0.f;
  __syncwarp();
  for (int64_t row = blockIdx.x * (int64_t)kWarps + w; row < n; row += (int64_t)gridDim.x * kWarps) {
    const uint4* sr = reinterpret_cast<const uint4*>(s + row * d);
    const uint4* dr = reinterpret_cast<const uint4*>(dy + row * d);
    const float rs = rstd[row];
    float dot = 0.f;
    for (int v = lane; v < nvec; v += 32) {
      float a[8], b[8];
      unpack8(sr[v], a);
      unpack8(dr[v], b);
      const float4 g0 = reinterpret_cast<const float4*>(g)[2 * v], g1 = reinterpret_cast<const float4*>(g)[2 * v + 1];
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dot += gg[j] * b[j] * a[j];
        acc[8 * v + j] += b[j] * a[j] * rs;
      }
    }
    dot = warp_sum(dot);
    const float k = dot * rs * rs / (float)d;
    for (int v = lane; v < nvec; v += 32) {
      float a[8], b[8], o[8];
      unpack8(sr[v], a);
      unpack8(dr[v], b);
      const float4 g0 = reinterpret_cast<const float4*>(g)[2 * v], g1 = reinterpret_cast<const float4*>(g)[2 * v + 1];
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      float rr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (dres) unpack8(reinterpret_cast<const uint4*>(dres + row * d)[v], rr);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rs * (gg[j] * b[j] - a[j] * k) + rr[j];
      reinterpret_cast<uint4*>(dx + row * d)[v] = pack8(o);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float t = 0.f;
    for (int ww = 0; ww < kWarps; ++ww) t += sm[ww * d + c];
    part[(int64_t)blockIdx.x * d + c] = t;
  }
}

__global__ void rmsnorm_dgain_kernel(const float* __restrict__ part, int nparts, int d, float* __restrict__ dgain,
                                     int accumulate) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float t = accumulate ? dgain[c] : 0.f;
  for (int b = 0; b < nparts; ++b) t += part[(int64_t)b * d + c];
  dgain[c] = t;
}

__global__ void __launch_bounds__(256) embed_fwd_kernel(const uint16_t* __restrict__ E, const int32_t* __restrict__ tok,
                                                        uint16_t* __restrict__ out, int64_t n, int d, int64_t vocab,
                                                        int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int nvec = d / 8;
  for (int64_t row = blockIdx.x * (int64_t)kWarps + (threadIdx.x >> 5); row < n; row += (int64_t)gridDim.x * kWarps) {
    const int32_t t = tok[row];
    if (t < 0 || t >= vocab) {
      if (lane == 0) atomicAdd(bad, 1);
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(E + (int64_t)t * d);
    uint4* dst = reinterpret_cast<uint4*>(out + row * d);
    for (int v = lane; v < nvec; v += 32) dst[v] = src[v];
  }
}

// order: positions sorted (stably) by token; seg: [vocab_used + 1] segment starts
// into `order`, uniq: the token of each segment.  One warp per segment.
__global__ void __launch_bounds__(256) embed_bwd_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ seg,
                                                        const int32_t* __restrict__ uniq, int nseg,
                                                        const uint16_t* __restrict__ dX, float* __restrict__ dE, int d,
                                                        int accumulate) {
  const int lane = threadIdx.x & 31;
  for (int sgi = blockIdx.x * kWarps + (threadIdx.x >> 5); sgi < nseg; sgi += gridDim.x * kWarps) {
    const int b = seg[sgi], e = seg[sgi + 1];
    float* dst = dE + (int64_t)uniq[sgi] * d;
    for (int c0 = lane * 8; c0 < d; c0 += 256) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = accumulate ? dst[c0 + j] : 0.f;
      for (int k = b; k < e; ++k) {
        float a[8];
        unpack8(*reinterpret_cast<const uint4*>(dX + (int64_t)order[k] * d + c0), a);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += a[j];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[c0 + j] = acc[j];
    }
  }
}

int grid_rows(int64_t n, int sms) {
  const int64_t want = (n + kWarps - 1) / kWarps;
  const int64_t cap = 16LL * sms;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

cudaError_t rmsnorm_fwd(cudaStream_t st, int sms, const void* x, const void* r, const float* g, void* y, void* s_out,
                        float* rstd, int64_t n, int d, float eps) {
  rmsnorm_fwd_kernel<<<grid_rows(n, sms), 256, 0, st>>>(static_cast<const uint16_t*>(x),
                                                        static_cast<const uint16_t*>(r), g, static_cast<uint16_t*>(y),
                                                        static_cast<uint16_t*>(s_out), rstd, n, d, eps);
  return cudaGetLastError();
}

int rmsnorm_bwd_parts(int64_t n, int sms) { return grid_rows(n, sms); }

cudaError_t rmsnorm_bwd(cudaStream_t st, int sms, const void* s, const float* g, const float* rstd, const void* dy,
                        const void* dres, void* dx, float* part, float* dgain, int accumulate, int64_t n, int d) {
  const int blocks = grid_rows(n, sms);
  const size_t smem = sizeof(float) * kWarps * d;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rmsnorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  rmsnorm_bwd_kernel<<<blocks, 256, smem, st>>>(static_cast<const uint16_t*>(s), g, rstd,
                                                static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(dres),
                                                static_cast<uint16_t*>(dx), part, n, d);
  rmsnorm_dgain_kernel<<<(d + 255) / 256, 256, 0, st>>>(part, blocks, d, dgain, accumulate);
  return cudaGetLastError();
}

cudaError_t embed_fwd(cudaStream_t st, int sms, const void* E, const int32_t* tok, void* out, int64_t n, int d,
                      int64_t vocab, int* bad) {
  embed_fwd_kernel<<<grid_rows(n, sms), 256, 0, st>>>(static_cast<const uint16_t*>(E), tok, static_cast<uint16_t*>(out),
                                                      n, d, vocab, bad);
  return cudaGetLastError();
}

cudaError_t embed_bwd(cudaStream_t st, int sms, const int32_t* order, const int32_t* seg, const int32_t* uniq, int nseg,
                      const void* dX, float* dE, int d, int accumulate) {
  if (nseg <= 0) return cudaSuccess;
  embed_bwd_kernel<<<grid_rows(nseg, sms), 256, 0, st>>>(order, seg, uniq, nseg, static_cast<const uint16_t*>(dX), dE,
                                                         d, accumulate);
  return cudaGetLastError();
}

}  // namespace mst_layers
