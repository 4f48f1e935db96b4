"""Attention kernels only, for compute-sanitizer (dev tool): several kv / q tiles, hd 128 / 64, both backward orders."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import attention as A, miniseq as ms
ctx = ms.Context.get(0)
for hd in (128, 64):
    Sa, Ha, KVa = 700, 4, 2
    q = torch.randn(Sa, Ha * hd, device="cuda").bfloat16(); k = torch.randn(Sa, KVa * hd, device="cuda").bfloat16()
    v = torch.randn(Sa, KVa * hd, device="cuda").bfloat16(); do = torch.randn(Sa, Ha * hd, device="cuda").bfloat16()
    o, lse = A.attention_forward(q, k, v, 1, Sa, Ha, KVa)
    for order in (3, 0):
        ctx.set_tuning("attn_bwd_order", order)
        A.attention_backward(q, k, v, o, do, lse, 1, Sa, Ha, KVa)
torch.cuda.synchronize(); print("attn san done")
