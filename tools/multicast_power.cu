// Energy of operand delivery: TMA unicast vs cluster multicast (dev tool, not
// part of libmst).  One CTA per SM in clusters of 2; every CTA streams 32 KB
// stages of an L2-resident buffer into a 6-stage shared-memory ring (no MMA),
// both CTAs of a cluster reading the same rows:
//   mode 0: each CTA loads both 16 KB boxes itself (2 L2 reads per box pair)
//   mode 1: CTA r loads box r once and multicasts it to both CTAs
// Each SM receives the same bytes in both modes; mode 1 halves the L2 reads.
// Prints ingress bytes per SM cycle; board power / SM clock are sampled by
// the caller (nvidia-smi) while it runs for ~`seconds`.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/mcast tools/multicast_power.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e_));               \
      return 1;                                                            \
    }                                                                      \
  } while (0)

constexpr int kStages = 6;
constexpr int kBox = 16384;  // 128 rows x 128 B
constexpr int kRows = 16384;  // tensor: 16384 rows x 64 bf16 (2 MB), L2 resident

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar),
               "r"(par)
               : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    stream(const __grid_constant__ CUtensorMap tm, int iters, int mode, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int cl = blockIdx.x >> 1;
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      const uint32_t par = (it / kStages) & 1;
      if (it >= kStages) wait(su32(&empty[s]), par ^ 1);
      const uint32_t fb = su32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2 * kBox) : "memory");
      const int row = ((cl * 13 + it) * 256) % kRows;
      const uint32_t dst = su32(smem + s * 2 * kBox);
      if (mode == 0) {
        for (int b = 0; b < 2; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  dst + b * kBox),
              "l"(&tm), "r"(fb), "r"(0), "r"(row + b * 128)
              : "memory");
      } else {
        // box `rank` of the pair, written into both CTAs at the same offset
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
            "{%3, %4}], [%2], %5;" ::"r"(dst + rank * kBox),
            "l"(&tm), "r"(fb), "r"(0), "r"(row + (int)rank * 128), "h"((uint16_t)0x3)
            : "memory");
      }
      // consume the stage issued kStages-1 iterations ago: wait for it, then
      // free it in both CTAs (the peer's multicast writes into this CTA's slot too)
      const int c = it - (kStages - 1);
      if (c >= 0) {
        const int cs = c % kStages;
        wait(su32(&full[cs]), (c / kStages) & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[cs])) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         mapa(su32(&empty[cs]), rank ^ 1))
                     : "memory");
      }
    }
    for (int c = iters - (kStages - 1); c < iters; ++c) wait(su32(&full[c % kStages]), (c / kStages) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cycles, clock64() - t0);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const double seconds = argc > 2 ? atof(argv[2]) : 10.0;
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* buf;
  CK(cudaMalloc(&buf, (size_t)kRows * 128));
  CK(cudaMemset(buf, 1, (size_t)kRows * 128));
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)kRows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("tensor map failed\n");
    return 1;
  }
  const int smem = kStages * 2 * kBox + 1024;
  CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  const int grid = sms / 2 * 2;
  const int iters = 20000;
  double tot_bytes = 0, tot_cyc = 0;
  auto t0 = std::chrono::steady_clock::now();
  int launches = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < seconds) {
    CK(cudaMemset(cyc, 0, 8));
    stream<<<grid, 128, smem>>>(tm, iters, mode, cyc);
    CK(cudaGetLastError());
    unsigned long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    tot_cyc += (double)c / grid;
    tot_bytes += (double)iters * 2 * kBox;
    ++launches;
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("mode %d (%s): %d launches, %.1f B/cycle/SM ingress, %.2f TB/s delivered to SMs, %.2f TB/s L2 reads\n", mode,
         mode ? "multicast" : "unicast", launches, tot_bytes / tot_cyc, tot_bytes * grid / secs / 1e12,
         tot_bytes * grid / secs / 1e12 / (mode ? 2 : 1));
  return 0;
}
