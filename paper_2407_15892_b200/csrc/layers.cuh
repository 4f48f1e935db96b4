// Host launchers of the decoder-layer kernels (csrc/layers.cu); the C ABI
// entry points that validate arguments live in mst_api.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mst_layers {
int rmsnorm_bwd_parts(int64_t n, int sms);
cudaError_t rmsnorm_fwd(cudaStream_t st, int sms, const void* x, const void* r, const float* g, void* y, void* s_out,
                        float* rstd, int64_t n, int d, float eps);
cudaError_t rmsnorm_bwd(cudaStream_t st, int sms, const void* s, const float* g, const float* rstd, const void* dy,
                        const void* dres, void* dx, float* part, float* dgain, int accumulate, int64_t n, int d);
cudaError_t embed_fwd(cudaStream_t st, int sms, const void* E, const int32_t* tok, void* out, int64_t n, int d,
                      int64_t vocab, int* bad);
cudaError_t embed_bwd(cudaStream_t st, int sms, const int32_t* order, const int32_t* seg, const int32_t* uniq, int nseg,
                      const void* dX, float* dE, int d, int accumulate);
}  // namespace mst_layers
