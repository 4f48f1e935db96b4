"""A/B of the attention backward issue orders (tuning attn_bwd_order, bit 0
dK/dV kernel, bit 1 dQ kernel) and of attn_inorder, interleaved rounds; every
variant's dq / dk / dv must be bitwise equal to order 0's (same GEMMs, same
accumulation order, only the issue order moves).

  python tools/attn_bwd_ab.py [S] [heads] [kv_heads] [hd] [rounds]
"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_15892_b200 import attention as A, miniseq as ms  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
KV = int(sys.argv[3]) if len(sys.argv) > 3 else 8
hd = int(sys.argv[4]) if len(sys.argv) > 4 else 128
R = int(sys.argv[5]) if len(sys.argv) > 5 else 6
torch.manual_seed(0)
q = torch.randn(S, H * hd, device="cuda").bfloat16()
k = torch.randn(S, KV * hd, device="cuda").bfloat16()
v = torch.randn(S, KV * hd, device="cuda").bfloat16()
do = torch.randn(S, H * hd, device="cuda").bfloat16()
ctx = ms.Context.get(0)
fl = 5.0 * S * S * hd * H
o, lse = A.attention_forward(q, k, v, 1, S, H, KV)
variants = [(0, 0), (1, 0), (2, 0), (3, 0), (3, 1)]  # (bwd_order, inorder)
ref = None
res = {vv: [] for vv in variants}
same = {}
for r in range(R):
    order = variants if r % 2 == 0 else variants[::-1]
    for vv in order:
        ctx.set_tuning("attn_bwd_order", vv[0])
        ctx.set_tuning("attn_inorder", vv[1])
        g = A.attention_backward(q, k, v, o, do, lse, 1, S, H, KV)
        torch.cuda.synchronize()
        if vv == (0, 0) and ref is None:
            ref = [t.clone() for t in g]
        if ref is not None:
            same[vv] = same.get(vv, True) and all(torch.equal(a, b) for a, b in zip(g, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            A.attention_backward(q, k, v, o, do, lse, 1, S, H, KV)
        e1.record()
        torch.cuda.synchronize()
        res[vv].append(e0.elapsed_time(e1) / 5)
ctx.set_tuning("attn_bwd_order", 3)
ctx.set_tuning("attn_inorder", 0)
for vv in variants:
    ms_ = statistics.median(res[vv])
    print(json.dumps({"shape": dict(S=S, heads=H, kv_heads=KV, hd=hd), "attn_bwd_order": vv[0], "attn_inorder": vv[1],
                      "bwd_ms": ms_, "bwd_tflops": fl / ms_ / 1e9, "bitwise_equal_to_order0": same.get(vv)}))
