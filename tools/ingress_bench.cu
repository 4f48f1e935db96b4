// Per-SM operand-ingress microbenchmark (dev tool, not part of libmst).
// Question: is the ~55 B/cycle/SM L2->SMEM rate seen by the GEMM engine's
// TMA producer (MMA disabled) a TMA-unit limit or an SM-port limit?  Each
// CTA (one per SM) streams an L2-resident buffer:
//   mode 0: TMA 2-D boxes (128 rows x 128 B, SWIZZLE_128B) into a 6-stage
//           smem ring (mbarrier complete_tx), one issuing thread
//   mode 1: 16-byte LDG (ld.global.v4, no smem) by all 8 warps
//   mode 2: cp.async 16-byte (LDGSTS) into smem by all 8 warps
//   mode 3: mode 0 (warp 0) and mode 1 (warps 1..7) concurrently
// and reports bytes per SM cycle.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ingress tools/ingress_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

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

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256, 1) ingress(const __grid_constant__ CUtensorMap tm,
                                                  const __grid_constant__ CUtensorMap tm3, const uint4* __restrict__ buf,
                                                  int64_t buf_vec, int iters, int mode, unsigned long long* cycles,
                                                  unsigned long long* bytes, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  unsigned long long nb = 0;
  uint32_t acc = 0;
  const int rows_total = 8192;  // tensor map: [8192 rows x 64 cols bf16] = 1 MB per CTA region
  if (mode == 4 && warp == 0) {  // GEMM-like stage: A 2-D box + B 3-D box (MN-major slab), 32 KB
    if (lane == 0) {
      uint32_t phase = 0;
      int stage = 0;
      for (int it = 0; it < iters; ++it) {
        const int row = ((blockIdx.x * 7 + it) * 128) % rows_total;
        if (it >= kStages / 2) {
          const uint32_t par = phase ^ 1;
          asm volatile(
              "{\n.reg .pred p;\nW4: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W4;\n}" ::"r"(
                  su32(&full[stage])),
              "r"(par));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(2 * kBox));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                "r"(su32(smem + stage * 2 * kBox)),
            "l"((uint64_t)&tm), "r"(su32(&full[stage])), "r"(0), "r"(row)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
                "r"(su32(smem + stage * 2 * kBox + kBox)),
            "l"((uint64_t)&tm3), "r"(su32(&full[stage])), "r"(0), "r"((it * 64) % 4096), "r"((blockIdx.x * 2) % 64)
            : "memory");
        nb += 2 * kBox;
        if (++stage == kStages / 2) {
          stage = 0;
          phase ^= 1;
        }
      }
      for (int s = 0; s < kStages / 2; ++s) {
        const uint32_t par = (s < stage) ? phase : (phase ^ 1);
        asm volatile(
            "{\n.reg .pred p;\nW5: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W5;\n}" ::"r"(
                su32(&full[s])),
            "r"(par));
      }
    }
  }
  if ((mode == 0 || mode == 3) && warp == 0) {
    if (lane == 0) {
      uint32_t phase = 0;
      int stage = 0;
      for (int it = 0; it < iters; ++it) {
        const int row = ((blockIdx.x * 7 + it) * 128) % rows_total;
        if (it >= kStages) {  // wait for the load issued kStages ago before reusing its stage
          const uint32_t par = phase ^ 1;
          asm volatile(
              "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                  su32(&full[stage])),
              "r"(par));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(kBox));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                "r"(su32(smem + stage * kBox)),
            "l"((uint64_t)&tm), "r"(su32(&full[stage])), "r"(0), "r"(row)
            : "memory");
        nb += kBox;
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      for (int s = 0; s < kStages; ++s) {  // drain
        const uint32_t par = (s < stage) ? phase : (phase ^ 1);
        asm volatile(
            "{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(
                su32(&full[s])),
            "r"(par));
      }
    }
  }
  if (mode == 1 || (mode == 3 && warp > 0)) {
    const int nthr = mode == 1 ? 256 : 224;
    const int tid = mode == 1 ? threadIdx.x : threadIdx.x - 32;
    const int64_t region = (int64_t)blockIdx.x * 65536;  // 1 MB of uint4 per CTA
    const int per_iter = kBox / 16;                       // same bytes per iteration as one TMA box
    for (int it = 0; it < iters; ++it) {
      const int64_t base = region + ((int64_t)it * per_iter) % 65536;
      for (int v = tid; v < per_iter; v += nthr) {
        const uint4 x = __ldcg(buf + ((base + v) % buf_vec));
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
      }
      if (tid == 0) nb += kBox;
    }
  }
  if (mode == 2) {
    const int64_t region = (int64_t)blockIdx.x * 65536;
    const int per_iter = kBox / 16;
    for (int it = 0; it < iters; ++it) {
      const int64_t base = region + ((int64_t)it * per_iter) % 65536;
      uint8_t* dst = smem + (it % kStages) * kBox;
      for (int v = threadIdx.x; v < per_iter; v += 256)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + v * 16)),
                     "l"(buf + ((base + v) % buf_vec)));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 4;");
      if (threadIdx.x == 0) nb += kBox;
    }
    asm volatile("cp.async.wait_group 0;");
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (acc == 0x12345678u) sink[0] = acc;
  atomicAdd(bytes, nb);
  if (threadIdx.x == 0) atomicAdd(cycles, t1 - t0);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t bytes = 64ll << 20;  // 64 MB: L2-resident
  void* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, 8192}, strides[1] = {128};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  // 3-D MN-major map: {64 elems, K rows, MN/64 blocks} over an [4096 x 4096] bf16 matrix
  CUtensorMap tm3;
  {
    cuuint64_t d3[3] = {64, 4096, 64}, s3[2] = {4096 * 2, 128};
    cuuint32_t b3[3] = {64, 64, 2}, e3[3] = {1, 1, 1};
    if (enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode3 failed\n");
      return 1;
    }
  }
  unsigned long long *cyc, *nb;
  uint32_t* sink;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&nb, 8));
  CK(cudaMalloc(&sink, 4));
  const int smem = kStages * kBox + 1024;
  CK(cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[5] = {"TMA 2D 16KB boxes (1 thread)", "LDG.128 (8 warps)", "cp.async 16B (8 warps)",
                          "TMA (warp 0) + LDG.128 (warps 1-7)", "GEMM-like stage: 2D A + 3D B box, 3 stages"};
  for (int grid : {sms, 16}) {
    for (int mode : {0, 4}) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(cyc, 0, 8));
        CK(cudaMemset(nb, 0, 8));
        const int iters = 4000;
        ingress<<<grid, 256, smem>>>(tm, tm3, (const uint4*)buf, bytes / 16, iters, mode, cyc, nb, sink);
        CK(cudaDeviceSynchronize());
        unsigned long long c = 0, b = 0;
        CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&b, nb, 8, cudaMemcpyDeviceToHost));
        if (rep == 1)
          printf("grid %3d  %-38s %7.1f B/cycle/SM\n", grid, names[mode], (double)b / ((double)c / grid) / grid);
      }
    }
  }
  return 0;
}
