// Per-SM issue rates of the softmax / epilogue instruction mix on one B200
// (dev tool): MUFU.EX2, F2FP.BF16.F32.PACK_AB, FFMA, and their mixes, one
// CTA per SM, 4..16 warps, 8 independent chains per thread.  Prints warp
// instructions per cycle per SM for each op (clock64 around the loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates tools/pipe_rates.cu && ./pipe_rates
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void bench(float* out, long long* cyc, float seed) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed + threadIdx.x * 1e-3f + i;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // ex2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      } else if (OP == 1) {  // pack
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) & 7]));
        acc ^= r;
        v[i] += 1.0f;
      } else if (OP == 2) {  // ffma
        asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(v[i]));
      } else if (OP == 3) {  // ex2 + pack (1:0.5, the softmax mix)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        if (i & 1) {
          uint32_t r;
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[i - 1]));
          acc ^= r;
        }
      } else if (OP == 4) {  // ex2 + ffma (1:1)
        asm volatile("fma.rn.f32 %0, %0, 0f3F000000, 0fBF000000;" : "+f"(v[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps, float* out, long long* cyc, int sms) {
  bench<OP><<<sms, 32 * warps>>>(out, cyc, 0.5f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  const double inst = static_cast<double>(kIters) * 8 * warps;  // warp instructions of the op per SM
  printf("%-12s warps %2d: %.1f cycles, %.3f warp-inst/cycle/SM (%.1f lanes/clk/SM)\n", name, warps, c, inst / c,
         32 * inst / c);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  for (int w : {4, 8, 16}) {
    run<0>("ex2", w, out, cyc, sms);
    run<1>("cvt.bf16x2", w, out, cyc, sms);
    run<2>("ffma", w, out, cyc, sms);
    run<3>("ex2+pack", w, out, cyc, sms);
    run<4>("ffma+ex2", w, out, cyc, sms);
  }
  return 0;
}
