// AdamW with global-norm clipping and micro-batch gradient accumulation
// (the reference's `optim` module), as HBM-bound sm_100a
// kernels behind the C ABI (include/mst/mst.h "optimizer").
//
// Layout: fp32 master weights, fp32 moments m / v, fp32 gradients (the MsT
// dW accumulators, consumed in place), and the bf16 model copy the GEMMs
// read.  One AdamW pass moves 30 bytes per parameter (read w, g, m, v;
// write w, m, v, bf16 w): at the Llama3-8B block (701M parameters) that is
// 21 GB, ~3.3 ms at the measured 6.5 TB/s copy bandwidth.
//
// Determinism: the squared-norm reduction writes one fp64 partial per block
// (fixed grid) and sums them in index order; no float atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "optim.cuh"

namespace mst_optim {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}

struct AdamCoef {
  float lr, wd_lr, b1, b2, one_m_b1, one_m_b2, inv_bc1, inv_bc2, eps;
};

// adamw_step: decoupled weight decay, then the Adam update
// with bias correction; g is scaled by *gscale (clip factor / accumulation
// steps) when gscale != nullptr.
__device__ __forceinline__ float adam1(float& w, float g, float& m, float& v, const AdamCoef& c) {
  w = w - c.wd_lr * w;
  m = c.b1 * m + c.one_m_b1 * g;
  v = c.b2 * v + c.one_m_b2 * g * g;
  const float mh = m * c.inv_bc1, vh = v * c.inv_bc2;
  w = w - c.lr * mh / (sqrtf(vh) + c.eps);
  return w;
}

__global__ void __launch_bounds__(kThreads) adamw_kernel(float* __restrict__ w, uint16_t* __restrict__ wb,
                                                         float* __restrict__ g, float* __restrict__ m,
                                                         float* __restrict__ v, int64_t n, AdamCoef c,
                                                         const float* __restrict__ gscale, int zero_grad) {
  const float s = gscale ? __ldg(gscale) : 1.0f;
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
    float4 W = __ldcs(reinterpret_cast<const float4*>(w) + k);
    const float4 G = __ldcs(reinterpret_cast<const float4*>(g) + k);
    float4 Mv = __ldcs(reinterpret_cast<const float4*>(m) + k);
    float4 Vv = __ldcs(reinterpret_cast<const float4*>(v) + k);
    adam1(W.x, G.x * s, Mv.x, Vv.x, c);
    adam1(W.y, G.y * s, Mv.y, Vv.y, c);
    adam1(W.z, G.z * s, Mv.z, Vv.z, c);
    adam1(W.w, G.w * s, Mv.w, Vv.w, c);
    __stcs(reinterpret_cast<float4*>(w) + k, W);
    __stcs(reinterpret_cast<float4*>(m) + k, Mv);
    __stcs(reinterpret_cast<float4*>(v) + k, Vv);
    __stcs(reinterpret_cast<uint2*>(wb) + k, make_uint2(pack2(W.x, W.y), pack2(W.z, W.w)));
    if (zero_grad) __stcs(reinterpret_cast<float4*>(g) + k, make_float4(0.f, 0.f, 0.f, 0.f));
  }
  for (int64_t e = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
    float W = w[e], Mv = m[e], Vv = v[e];
    adam1(W, g[e] * s, Mv, Vv, c);
    w[e] = W;
    m[e] = Mv;
    v[e] = Vv;
    wb[e] = __bfloat16_as_ushort(__float2bfloat16_rn(W));
    if (zero_grad) g[e] = 0.f;
  }
}

// Per-block fp64 partial sums of g^2 (block b of a fixed grid), in a fixed order.
__global__ void __launch_bounds__(kThreads) sumsq_kernel(const float* __restrict__ g, int64_t n,
                                                         double* __restrict__ partial) {
  double acc = 0.0;
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n4; k += 4 * stride) {  // 4 independent 16-byte loads in flight per thread
    float4 G[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) G[u] = __ldcs(g4 + k + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      acc += (double)G[u].x * G[u].x + (double)G[u].y * G[u].y + (double)G[u].z * G[u].z + (double)G[u].w * G[u].w;
  }
  for (; k < n4; k += stride) {
    const float4 G = __ldcs(g4 + k);
    acc += (double)G.x * G.x + (double)G.y * G.y + (double)G.z * G.z + (double)G.w * G.w;
  }
  for (int64_t e = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride)
    acc += (double)g[e] * g[e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double warp_sum[kThreads / 32];
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += warp_sum[i];
    partial[blockIdx.x] = s;
  }
}

// Fixed-order sum of the partials into *sumsq (accumulate != 0 adds to it),
// then the clip factor of the averaged gradient g/steps:
// scale = max_norm / ||g/steps|| if that norm exceeds max_norm, else 1;
// times 1 / accumulation steps (the average itself).  A
// non-finite norm propagates NaN into the scale (the host raises
// NonFiniteError when it checks).
__global__ void sumsq_finish_kernel(const double* __restrict__ partial, int nparts, double* sumsq, int accumulate,
                                    float max_norm, float inv_steps, float* scale_out, float* norm_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = accumulate ? *sumsq : 0.0;
  for (int i = 0; i < nparts; ++i) s += partial[i];
  *sumsq = s;
  if (scale_out) {
    // SPEC.md:500-506 then 486-491: the accumulated sum is divided by the
    // step count first, and the clip applies to the norm of that average.
    const double norm = sqrt(s) * (double)inv_steps;
    if (norm_out) *norm_out = (float)norm;
    double sc = (max_norm > 0.f && norm > (double)max_norm) ? (double)max_norm / norm : 1.0;
    if (!isfinite(norm)) sc = NAN;
    *scale_out = (float)(sc * inv_steps);
  }
}

__global__ void __launch_bounds__(kThreads) accumulate_kernel(float* __restrict__ into, const float* __restrict__ from,
                                                              int64_t n) {
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
    float4 a = reinterpret_cast<float4*>(into)[k];
    const float4 b = __ldcs(reinterpret_cast<const float4*>(from) + k);
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    reinterpret_cast<float4*>(into)[k] = a;
  }
  for (int64_t e = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) into[e] += from[e];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int grid_for(int64_t n, int sms) {
  const int64_t want = (n / 4 + kThreads - 1) / kThreads;
  const int64_t cap = 8LL * sms;  // 8 resident 256-thread CTAs per SM: enough bytes in flight for HBM
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_adamw(cudaStream_t st, int sms, int64_t n, float* w, void* w_bf16, float* grad, float* m, float* v,
                         const mst_adamw_config& cfg, int64_t step, const float* grad_scale, int zero_grad) {
  AdamCoef c;  // coefficients formed in double, rounded once to fp32
  c.lr = (float)cfg.lr;
  c.wd_lr = (float)(cfg.lr * cfg.weight_decay);
  c.b1 = (float)cfg.beta1;
  c.b2 = (float)cfg.beta2;
  c.one_m_b1 = (float)(1.0 - cfg.beta1);
  c.one_m_b2 = (float)(1.0 - cfg.beta2);
  c.inv_bc1 = (float)(1.0 / (1.0 - std::pow(cfg.beta1, (double)step)));
  c.inv_bc2 = (float)(1.0 / (1.0 - std::pow(cfg.beta2, (double)step)));
  c.eps = (float)cfg.eps;
  adamw_kernel<<<grid_for(n, sms), kThreads, 0, st>>>(w, static_cast<uint16_t*>(w_bf16), grad, m, v, n, c, grad_scale,
                                                      zero_grad);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(cudaStream_t st, const float* grad, int64_t n, double* partial_ws, double* sumsq,
                         int accumulate, float max_norm, float inv_steps, float* scale_out, float* norm_out) {
  sumsq_kernel<<<kSumsqBlocks, kThreads, 0, st>>>(grad, n, partial_ws);
  sumsq_finish_kernel<<<1, 32, 0, st>>>(partial_ws, kSumsqBlocks, sumsq, accumulate, max_norm, inv_steps, scale_out,
                                        norm_out);
  return cudaGetLastError();
}

cudaError_t launch_accumulate(cudaStream_t st, int sms, float* into, const float* from, int64_t n) {
  accumulate_kernel<<<grid_for(n, sms), kThreads, 0, st>>>(into, from, n);
  return cudaGetLastError();
}

}  // namespace mst_optim
