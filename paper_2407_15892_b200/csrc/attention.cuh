// Causal GQA attention on tcgen05 (csrc/attention.cu); host entry points used
// by the C ABI (mst_attention_forward / mst_attention_backward in mst.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mst_attn {

extern int g_fwd_version;  // 2: two q tiles per CTA (default), 1: one (tuning "attn_fwd")
extern int g_mma_inorder;  // 1: no completion wait between dependent MMAs of one thread (tuning "attn_inorder")
extern int g_bwd_order;    // backward issue orders, bit 0 dK/dV, bit 1 dQ (tuning "attn_bwd_order")
extern int g_poly_exp;     // forward softmax exp2 pairs (of 4) on the FMA pipe, 0..3 (tuning "attn_poly")
extern int g_bwd_version;  // 2: TMEM A operands + 2-stage ring (default), 1: the first kernels (tuning "attn_bwd")

struct AttnShape {
  int B, S, heads, kvh, hd;
};

// Return 0 on success; otherwise *err names the failure (1: tensor map, 2: CUDA).
int forward(void* encode_fn, cudaStream_t st, const AttnShape& s, const void* q, int64_t ldq, const void* k,
            int64_t ldk, const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, const char** err);
int backward(void* encode_fn, cudaStream_t st, const AttnShape& s, const void* q, int64_t ldq, const void* k,
             int64_t ldk, const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
             const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv, float* delta,
             const char** err);

}  // namespace mst_attn
