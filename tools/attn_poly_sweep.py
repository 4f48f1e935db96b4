"""Forward attention throughput vs the share of softmax exponentials computed
on the FMA pipe (tuning attn_poly = pairs of every 4), interleaved rounds in
one process, plus the output / lse deviation from attn_poly=0 (dev tool).
usage: python tools/attn_poly_sweep.py [S] [heads] [kv_heads] [hd]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_15892_b200 import attention as A  # noqa: E402
from paper_2407_15892_b200 import miniseq as ms  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
KV = int(sys.argv[3]) if len(sys.argv) > 3 else 8
hd = int(sys.argv[4]) if len(sys.argv) > 4 else 128
torch.manual_seed(0)
q = torch.randn(S, H * hd, device="cuda").bfloat16()
k = torch.randn(S, KV * hd, device="cuda").bfloat16()
v = torch.randn(S, KV * hd, device="cuda").bfloat16()
ctx = ms.Context.get(0)
fl = 2.0 * S * S * hd * H
ref = None
res = {p: [] for p in range(4)}
for p in range(4):
    ctx.set_tuning("attn_poly", p)
    o, lse = A.attention_forward(q, k, v, 1, S, H, KV)
    torch.cuda.synchronize()
    if ref is None:
        ref = (o.float(), lse.clone())
    else:
        do = (o.float() - ref[0]).norm() / ref[0].norm()
        dl = (lse - ref[1]).abs().max()
        print(f"attn_poly={p}: |o - o0|/|o0| = {do:.2e}, max |lse - lse0| = {dl:.2e}")
for r in range(6):
    for p in (range(4) if r % 2 == 0 else reversed(range(4))):
        ctx.set_tuning("attn_poly", p)
        for _ in range(2):
            A.attention_forward(q, k, v, 1, S, H, KV, out=o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            A.attention_forward(q, k, v, 1, S, H, KV, out=o)
        e1.record()
        torch.cuda.synchronize()
        res[p].append(e0.elapsed_time(e1) / 5)
ctx.set_tuning("attn_poly", 1)
for p in range(4):
    t = statistics.median(res[p])
    print(f"attn_poly={p}: {t:.3f} ms  {fl / t / 1e9:.1f} TFLOP/s (S={S} heads={H}/{KV} hd={hd})")
