"""A/B of the attention kernels' MMA ordering knob (tuning "attn_inorder"):
outputs with the completion waits between dependent MMAs of one thread
removed must be bitwise those with the waits, over many shapes and reruns;
then both variants are timed.  (dev tool)"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_15892_b200 import attention as A  # noqa: E402
from paper_2407_15892_b200 import miniseq as ms  # noqa: E402

ctx = ms.Context.get(0)
shapes = [(1, 4096, 32, 8, 128), (2, 1000, 8, 2, 64), (1, 8192, 16, 16, 64), (3, 513, 8, 4, 96), (1, 257, 4, 1, 16)]
bad = 0
for (B, S, H, KV, hd) in shapes:
    torch.manual_seed(S)
    q = torch.randn(B * S, H * hd, device="cuda").bfloat16()
    k = torch.randn(B * S, KV * hd, device="cuda").bfloat16()
    v = torch.randn(B * S, KV * hd, device="cuda").bfloat16()
    do = torch.randn(B * S, H * hd, device="cuda").bfloat16()
    res = {}
    for mode in (0, 1):
        ctx.set_tuning("attn_inorder", mode)
        outs = []
        for rep in range(5):
            o, lse = A.attention_forward(q, k, v, B, S, H, KV)
            g = A.attention_backward(q, k, v, o, do, lse, B, S, H, KV)
            outs.append([o.clone(), lse.clone()] + [t.clone() for t in g])
        torch.cuda.synchronize()
        res[mode] = outs
    for rep in range(5):
        for x, y in zip(res[0][0], res[1][rep]):
            if not torch.equal(x, y):
                bad += 1
    print(json.dumps({"shape": [B, S, H, KV, hd], "mismatches_so_far": bad}), flush=True)
for mode in (0, 1):
    ctx.set_tuning("attn_inorder", mode)
    B, S, H, KV, hd = 1, 8192, 32, 8, 128
    q = torch.randn(B * S, H * hd, device="cuda").bfloat16()
    k = torch.randn(B * S, KV * hd, device="cuda").bfloat16()
    v = torch.randn(B * S, KV * hd, device="cuda").bfloat16()
    do = torch.randn(B * S, H * hd, device="cuda").bfloat16()
    o, lse = A.attention_forward(q, k, v, B, S, H, KV)
    for _ in range(3):
        A.attention_forward(q, k, v, B, S, H, KV, out=o)
        A.attention_backward(q, k, v, o, do, lse, B, S, H, KV)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(10):
        A.attention_forward(q, k, v, B, S, H, KV, out=o)
    ev[1].record()
    for _ in range(10):
        A.attention_backward(q, k, v, o, do, lse, B, S, H, KV)
    ev[2].record()
    torch.cuda.synchronize()
    tf, tb = ev[0].elapsed_time(ev[1]) / 10, ev[1].elapsed_time(ev[2]) / 10
    fl = 2.0 * S * S * hd * H
    print(json.dumps({"inorder": mode, "fwd_ms": tf, "fwd_tflops": fl / tf / 1e9, "bwd_ms": tb,
                      "bwd_tflops": 2.5 * fl / tb / 1e9}), flush=True)
print("total mismatches", bad)
