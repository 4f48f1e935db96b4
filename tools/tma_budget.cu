// Per-SM data-movement budget microbenchmark (dev tool, not part of libmst).
//
// Question (engine design): the GEMM launches run at ~57-60 B/cycle/SM of
// TMA traffic counting loads AND the epilogue's TMA stores / reduce-adds
// (K6 with its fp32 read-modify-write epilogue: 32 KB in + 8 KB out per K
// block, ~650-700 cycles).  Is that budget shared between TMA loads and TMA
// stores (one TMA unit), and would the same stores issued from registers by
// the LSU path (red.global.add.v4.f32, coalesced) add to it instead?
//
// One CTA per SM (grid = #SMs, 256 threads).  Warp 0 lane 0 streams 2 x 16 KB
// TMA boxes per stage (6-stage ring) from an L2-resident bf16 matrix; warp 1
// consumes the stages (wait full, arrive empty).  Warps 4..7 (the
// "epilogue") concurrently write fp32 data to an L2-resident fp32 matrix:
//   mode 0: nothing (load rate alone)
//   mode 1: TMA reduce-add of 16 KB boxes (128 rows x 32 fp32) from shared memory
//   mode 2: TMA store of the same boxes
//   mode 3: red.global.add.v4.f32 from registers, each warp instruction 4 rows x 128 B
//   mode 4: st.global.v4 (plain stores), same pattern
//   mode 5: mode 1 without loads (store rate alone)
//   mode 6: mode 3 without loads
// Both streams run for the whole window (the store warps stop when the
// producer is done); reported per SM cycle: load bytes, store bytes, sum.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmab tools/tma_budget.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e_));                        \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

constexpr int kStages = 6;
constexpr int kBox = 16384;          // 128 rows x 128 B
constexpr int kStage = 2 * kBox;     // A + B box
constexpr int kOutBox = 16384;       // 128 rows x 32 fp32
constexpr int kOutBufs = 2;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar),
      "r"(par)
      : "memory");
}

__global__ void __launch_bounds__(256, 1)
    budget(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, float* out,
           int64_t out_rows, int iters, int mode, unsigned long long* res) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = smem;
  uint8_t* obuf = smem + kStages * kStage;
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  for (int i = threadIdx.x; i < kOutBufs * kOutBox / 4; i += 256) reinterpret_cast<float*>(obuf)[i] = 1e-3f;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  const bool loads = mode <= 4;
  const unsigned long long t0 = clock64();
  unsigned long long lbytes = 0, sbytes = 0;
  const int in_rows = 4096;
  if (warp == 0 && lane == 0) {
    if (loads) {
      for (int it = 0; it < iters; ++it) {
        const int s = it % kStages;
        if (it >= kStages) mbar_wait(su32(&empty[s]), ((it / kStages) - 1) & 1);
        const uint32_t bar = su32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kStage) : "memory");
        const int k = (it * 64) % 4096;
        const int r0 = ((blockIdx.x * 128) + (it / 64) * 256) % in_rows;
        const int r1 = ((blockIdx.x * 128) + 2048 + (it / 64) * 256) % in_rows;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
            "[%2];" ::"r"(su32(ring + s * kStage)),
            "l"(&tin), "r"(bar), "r"(k), "r"(r0)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
            "[%2];" ::"r"(su32(ring + s * kStage + kBox)),
            "l"(&tin), "r"(bar), "r"(k), "r"(r1)
            : "memory");
        lbytes += kStage;
      }
      // drain
      for (int it = iters > kStages ? iters - kStages : 0; it < iters; ++it)
        mbar_wait(su32(&empty[it % kStages]), (it / kStages) & 1);
    } else {
      // store-only modes: run a fixed window of clock cycles
      const unsigned long long tw = clock64();
      while (clock64() - tw < (unsigned long long)iters * 600ull) {
      }
    }
    done = 1;
  } else if (warp == 1 && lane == 0 && loads) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      mbar_wait(su32(&full[s]), (it / kStages) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  } else if (warp >= 4 && mode != 0) {
    const int q = warp - 4;
    int it = 0;
    const int64_t cols = 4096;
    const bool tma = mode == 1 || mode == 2 || mode == 5;
    while (!done) {
      const int64_t rb = ((int64_t)blockIdx.x * 128 + (it / 16) * 256 * 148) % out_rows;
      const int cb = (it * 32) % (int)cols;
      if (tma) {
        if (q == 0 && lane == 0) {
          const int b = it % kOutBufs;
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (mode == 2)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tout),
                         "r"(su32(obuf + b * kOutBox)), "r"(cb), "r"((int)rb)
                         : "memory");
          else
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tout),
                "r"(su32(obuf + b * kOutBox)), "r"(cb), "r"((int)rb)
                : "memory");
          asm volatile("cp.async.bulk.commit_group;");
          sbytes += kOutBox;
        }
      } else {
        // 128 rows x 32 fp32 per iteration over the 4 warps: warp q rows [32q, 32q+32), 4 rows per instruction
        const float4 v = make_float4(1e-3f, 1e-3f, 1e-3f, 1e-3f);
        for (int r = 0; r < 32; r += 4) {
          const int64_t row = rb + q * 32 + r + (lane >> 3);
          float* dst = out + row * cols + cb + (lane & 7) * 4;
          if (mode == 3 || mode == 6)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                         "f"(v.w)
                         : "memory");
          else
            asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                         "f"(v.w)
                         : "memory");
        }
        if (lane == 0) sbytes += kOutBox / 4;
      }
      ++it;
    }
    if (tma && q == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (lbytes) atomicAdd(res + 0, lbytes);
  if (sbytes) atomicAdd(res + 1, sbytes);
  if (threadIdx.x == 0) atomicAdd(res + 2, t1 - t0);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t in_bytes = 4096ll * 4096 * 2;  // 32 MB bf16
  const int64_t out_rows = 2048;
  const int64_t out_bytes = out_rows * 4096 * 4;  // 32 MB fp32
  void *bin, *bout;
  CK(cudaMalloc(&bin, in_bytes));
  CK(cudaMalloc(&bout, out_bytes));
  CK(cudaMemset(bin, 0, in_bytes));
  CK(cudaMemset(bout, 0, out_bytes));
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tin, tout;
  {
    cuuint64_t d[2] = {4096, 4096}, s[1] = {4096 * 2};
    cuuint32_t b[2] = {64, 128}, e[2] = {1, 1};
    if (enc(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bin, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      return printf("encode in failed\n"), 1;
  }
  {
    cuuint64_t d[2] = {4096, (cuuint64_t)out_rows}, s[1] = {4096 * 4};
    cuuint32_t b[2] = {32, 128}, e[2] = {1, 1};
    if (enc(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, bout, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      return printf("encode out failed\n"), 1;
  }
  unsigned long long* res;
  CK(cudaMalloc(&res, 3 * sizeof(unsigned long long)));
  const int smem = kStages * kStage + kOutBufs * kOutBox + 1024;
  CK(cudaFuncSetAttribute(budget, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[] = {"TMA loads only",
                         "TMA loads + TMA reduce-add",
                         "TMA loads + TMA store",
                         "TMA loads + red.global.add.v4 (LSU)",
                         "TMA loads + st.global.v4 (LSU)",
                         "TMA reduce-add only",
                         "red.global.add.v4 only"};
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  for (int grid : {sms, sms / 4}) {
    for (int mode = 0; mode <= 6; ++mode) {
      budget<<<grid, 256, smem>>>(tin, tout, (float*)bout, out_rows, 200, mode, res);  // warm-up
      CK(cudaDeviceSynchronize());
      CK(cudaMemset(res, 0, 3 * sizeof(unsigned long long)));
      budget<<<grid, 256, smem>>>(tin, tout, (float*)bout, out_rows, iters, mode, res);
      CK(cudaDeviceSynchronize());
      unsigned long long h[3];
      CK(cudaMemcpy(h, res, sizeof(h), cudaMemcpyDeviceToHost));
      const double cyc = (double)h[2] / grid;
      const double l = (double)h[0] / grid / cyc, s = (double)h[1] / grid / cyc;
      printf("grid %3d  %-40s load %6.1f  store %6.1f  sum %6.1f B/cycle/SM\n", grid, names[mode], l, s, l + s);
    }
  }
  return 0;
}
