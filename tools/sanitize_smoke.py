"""Small end-to-end run of every device entry point, for compute-sanitizer
(dev tool): python -m ... under `compute-sanitizer --tool memcheck`."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms, model as mdl, optim

torch.manual_seed(0)
N, H, I, V = 300, 64, 136, 520
X = torch.randn(N, H, device="cuda").bfloat16()
W = [(0.05 * torch.randn(*s, device="cuda")).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
L = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
L[::7] = -100
mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
ctx = ms.Context.get(0)
for chunked in (1, 0):
    ctx.set_tuning("chunked_block", chunked)
    st, gr = ms.block_step(X, L, mlp, head, 3, 3, check=True)
ctx.set_tuning("chunked_block", 1)
# round-2 schedule variants: paired dW GEMMs (even / odd chunk counts), row-scaled head on / off
for pair in (1, 0):
    for rs in (1, 0):
        ctx.set_tuning("pair_dw", pair)
        ctx.set_tuning("dl_rowscale", rs)
        for mm, mh in ((4, 4), (5, 5), (2, 6)):
            ms.block_step(X, L, mlp, head, mm, mh, check=True)
        ms.miniseq_lmhead_fused(X, L, head, ms.make_chunk_plan(N, 3))
ctx.set_tuning("pair_dw", 1)
ctx.set_tuning("dl_rowscale", 1)
# host-resident X / labels / dX (mst_block_step_host)
dXh = torch.empty(N, H, dtype=torch.bfloat16).pin_memory()
ms.block_step_host(X.cpu().pin_memory(), L.cpu().pin_memory(), mlp, head, 4, dXh)
plan = ms.make_chunk_plan(N, 4)
O, sv = ms.miniseq_mlp_forward(X, mlp, plan)
loss, hs = ms.miniseq_lmhead_forward(O, L, head, plan)
dO, _ = ms.miniseq_lmhead_backward(hs, head, plan)
ms.miniseq_mlp_backward(dO, sv, mlp, plan)
cfg = mdl.ModelConfig(d=64, I=224, V=512, heads=4, G=2, layers=1, S=128, B=1, M_mlp=2, M_head=4)
m = mdl.Model(cfg)
opt = optim.AdamW(m.w.named(), optim.OptimConfig())
tok = torch.randint(0, 512, (1, 128), device="cuda", dtype=torch.int32)
m.train_step(tok, tok, opt)
# attention kernels over several kv / q tiles (dK/dV ring, 3-stage K ring of the dQ kernel),
# every backward issue order, head dims 128 and 64, GQA 2
from paper_2407_15892_b200 import attention as A  # noqa: E402
for hd in (128, 64):
    Sa, Ha, KVa = 700, 4, 2
    q = torch.randn(Sa, Ha * hd, device="cuda").bfloat16()
    k = torch.randn(Sa, KVa * hd, device="cuda").bfloat16()
    v = torch.randn(Sa, KVa * hd, device="cuda").bfloat16()
    do = torch.randn(Sa, Ha * hd, device="cuda").bfloat16()
    o, lse = A.attention_forward(q, k, v, 1, Sa, Ha, KVa)
    for order in (3, 0):
        ctx.set_tuning("attn_bwd_order", order)
        A.attention_backward(q, k, v, o, do, lse, 1, Sa, Ha, KVa)
ctx.set_tuning("attn_bwd_order", 3)
torch.cuda.synchronize()
print("sanitize smoke done", float(st[2]))
