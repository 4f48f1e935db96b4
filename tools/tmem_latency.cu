// TMEM access latency on one B200 (dev tool): one CTA per SM, 4 warps (one
// per TMEM lane quadrant), a dependent chain of tcgen05.ld.32x32b.x32 ->
// tcgen05.wait::ld (the load address depends on the previous value), and of
// tcgen05.st.32x32b.x32 -> tcgen05.wait::st; clock64 per iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2407_15892_b200/csrc -o tmem_latency tools/tmem_latency.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace mst;

__global__ void __launch_bounds__(128, 1) tmem_lat(long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc_cg1(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot + (static_cast<uint32_t>(warp * 32) << 16);
  uint32_t r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = 0;
  ptx::tmem_st_32x32b_x32(tmem, r);
  ptx::tmem_st_wait();
  // ld latency: dependent chain
  uint32_t col = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    ptx::tmem_ld_32x32b_x32(tmem + (col & 32), r);
    ptx::tmem_ld_wait();
    col += r[0] + r[31] + 32;
  }
  long long t1 = clock64();
  // two loads then one wait (the attention passes' pattern)
  for (int i = 0; i < iters; ++i) {
    uint32_t s[32];
    ptx::tmem_ld_32x32b_x32(tmem + (col & 32), r);
    ptx::tmem_ld_32x32b_x32(tmem + 64 + (col & 32), s);
    ptx::tmem_ld_wait();
    col += r[0] + s[31] + 32;
  }
  long long t2 = clock64();
  // st -> wait::st
  for (int i = 0; i < iters; ++i) {
    r[0] = col + i;
    ptx::tmem_st_32x32b_x32(tmem + 128 + (i & 1) * 32, r);
    ptx::tmem_st_wait();
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = (t1 - t0) / iters;
    out[blockIdx.x * 4 + 1] = (t2 - t1) / iters;
    out[blockIdx.x * 4 + 2] = (t3 - t2) / iters;
    out[blockIdx.x * 4 + 3] = col;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(slot, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 4 * 148);
  tmem_lat<<<148, 128>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4 * 148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  printf("tcgen05.ld.32x32b.x32 + wait::ld (dependent): %lld cycles\n", h[0]);
  printf("2 x tcgen05.ld.32x32b.x32 + one wait::ld: %lld cycles\n", h[1]);
  printf("tcgen05.st.32x32b.x32 + wait::st: %lld cycles\n", h[2]);
  return 0;
}
