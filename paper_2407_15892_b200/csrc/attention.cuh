// Causal GQA attention on tcgen05 (csrc/attention.cu); host entry points used
// by the C ABI (mst_attention_forward / mst_attention_backward in mst.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mst_attn {

// Tuning knobs, owned by the calling context (mst_ctx_set_tuning keys in
// brackets); the defaults are the measured-best settings.
struct AttnTuning {
  int fwd_version = 2;  // 2: two q tiles per CTA, 1: one ("attn_fwd")
  int bwd_version = 2;  // 2: TMEM A operands + rings, 1: the first kernels ("attn_bwd")
  // 1: rely on tcgen05.mma executing in issue order (an MMA that overwrites
  // TMEM columns an earlier MMA of the same thread reads as its A operand is
  // issued without waiting for that MMA's completion); 0: wait for the commit.
  int mma_inorder = 0;  // ("attn_inorder")
  // Backward issue orders (bit mask): bit 0 = the dK/dV kernel issues the next
  // tile's scores under the dS pass; bit 1 = the dQ kernel writes dS over S so
  // dP(j+1) does not wait for dQ(j).  0 = the earlier round-2 orders.
  int bwd_order = 3;    // ("attn_bwd_order")
  int poly_exp = 0;     // forward softmax exp2 pairs (of 4) on the FMA pipe, 0..3 ("attn_poly")
};

struct AttnShape {
  int B, S, heads, kvh, hd;
};

// Kernel attributes on the current device (called once per context).
cudaError_t init_device();

// Return 0 on success; otherwise *err names the failure (1: tensor map, 2: CUDA).
int forward(void* encode_fn, cudaStream_t st, const AttnTuning& tune, const AttnShape& s, const void* q, int64_t ldq, const void* k,
            int64_t ldk, const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, const char** err);
int backward(void* encode_fn, cudaStream_t st, const AttnTuning& tune, const AttnShape& s, const void* q, int64_t ldq, const void* k,
             int64_t ldk, const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
             const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv, float* delta,
             const char** err);

}  // namespace mst_attn
