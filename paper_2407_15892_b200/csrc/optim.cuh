// Host launchers of the optimizer kernels (csrc/optim.cu); the C ABI entry
// points that validate arguments live in mst_api.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mst/mst.h"

namespace mst_optim {
constexpr int kSumsqBlocks = 1184;  // 8 x 148 SMs: fixed grid -> fixed reduction order
bool aligned16(const void* p);
cudaError_t launch_adamw(cudaStream_t st, int sms, int64_t n, float* w, void* w_bf16, float* grad, float* m, float* v,
                         const mst_adamw_config& cfg, int64_t step, const float* grad_scale, int zero_grad);
cudaError_t launch_sumsq(cudaStream_t st, const float* grad, int64_t n, double* partial_ws, double* sumsq,
                         int accumulate, float max_norm, float inv_steps, float* scale_out, float* norm_out);
cudaError_t launch_accumulate(cudaStream_t st, int sms, float* into, const float* from, int64_t n);
}  // namespace mst_optim
