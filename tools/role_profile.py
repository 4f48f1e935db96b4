"""Per-launch role wait breakdown with the MST_PROFILE build (dev tool).
MST_LIB=.../libmst_prof.so python tools/role_profile.py"""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
S, M = 8192, 8
H, I, V = 4096, 14336, 128256
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
plan = ms.make_chunk_plan(S, M)
st, gr = ms.block_step(X, L, mlp, head, M, M)
ctx = ms.Context.get(0)
buf = torch.zeros(64 * 8, dtype=torch.int64, device=dev)
O, sv = ms.miniseq_mlp_forward(X, mlp, plan)
loss, hs = ms.miniseq_lmhead_forward(O, L, head, plan)
dO, _ = ms.miniseq_lmhead_backward(hs, head, plan, dW_out=gr.W_out)
torch.cuda.synchronize()
ops = {
    'mlp_fwd': lambda: ms.miniseq_mlp_forward(X, mlp, plan),
    'head_fwd': lambda: ms.miniseq_lmhead_forward(O, L, head, plan),
    'head_bwd': lambda: ms.miniseq_lmhead_backward(hs, head, plan, dW_out=gr.W_out),
    'mlp_bwd': lambda: ms.miniseq_mlp_backward(dO, sv, mlp, plan, grads=ms.MlpGrads(gr.W_gate, gr.W_up, gr.W_down)),
}
for name, fn in ops.items():
    buf.zero_()
    ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, buf.data_ptr()))
    ctx.set_timing(True)
    fn()
    torch.cuda.synchronize()
    recs = ctx.take_timing_records()
    ctx.set_timing(False)
    ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, None))
    c = buf.view(64, 8).cpu().tolist()
    print(f"== {name}")
    for k, (t, f) in enumerate(recs[:6]):
        v = c[k]
        pw, pt, mf, mt, mtot, ew, eb, etot = v
        pr = lambda a, b: f"{100 * a / max(b, 1):5.1f}%"
        print(f"  launch {k}: {t:6.3f} ms {f / t / 1e9:7.1f} TF/s | prod wait-empty {pr(pw, pt)} | "
              f"mma wait-full {pr(mf, mtot)} wait-tmem {pr(mt, mtot)} | epi wait {pr(ew, etot)} busy {pr(eb, etot)}")
