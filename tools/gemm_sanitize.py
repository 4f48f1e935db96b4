"""Grouped-GEMM engine at a shape with many tiles per CTA pair (ring and TMEM
double-buffer wrap-around, dynamic tile claims over several waves), every
block-step schedule variant, for compute-sanitizer (dev tool)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms  # noqa: E402

torch.manual_seed(0)
N, H, I, V = 2048, 512, 1536, 8192
X = torch.randn(N, H, device="cuda").bfloat16()
W = [(0.03 * torch.randn(*s, device="cuda")).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
L = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
ctx = ms.Context.get(0)
for pair in (1, 0):
    ctx.set_tuning("pair_dw", pair)
    for mm, mh in ((4, 4), (2, 8), (1, 1), (3, 3)):
        ms.block_step(X, L, mlp, head, mm, mh)
ctx.set_tuning("pair_dw", 1)
torch.cuda.synchronize()
print("gemm sanitize done")
