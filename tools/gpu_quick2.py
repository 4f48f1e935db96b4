"""Quick GPU check of the miniseq ops against the torch fp32 reference (dev tool)."""
import sys, time, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2407_15892_b200 import miniseq as ms
import torch_ref as R

dev = 'cuda'
def mk(N, H, I, V, seed=0, ign=0.05):
    g = torch.Generator(device=dev).manual_seed(seed)
    X = torch.randn(N, H, device=dev, generator=g).bfloat16()
    Wg = (0.02 * torch.randn(H, I, device=dev, generator=g)).bfloat16()
    Wu = (0.02 * torch.randn(H, I, device=dev, generator=g)).bfloat16()
    Wd = (0.02 * torch.randn(I, H, device=dev, generator=g)).bfloat16()
    Wo = (0.02 * torch.randn(H, V, device=dev, generator=g)).bfloat16()
    L = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    L[torch.rand(N, device=dev, generator=g) < ign] = -100
    return X, L, Wg, Wu, Wd, Wo

for (N, H, I, V, Mm, Mh) in [(1024, 256, 688, 4096, 4, 4), (512, 256, 512, 1024, 1, 1), (1000, 136, 200, 520, 3, 7), (8192//4, 4096, 14336, 128256, 2, 2)]:
    X, L, Wg, Wu, Wd, Wo = mk(N, H, I, V)
    plan = ms.make_chunk_plan(N, Mm)
    w = ms.MlpWeights(Wg, Wu, Wd)
    O, saved = ms.miniseq_mlp_forward(X, w, plan)
    ref = R.block(X, L, Wg, Wu, Wd, Wo, exact=False)
    print(f"N={N} H={H} I={I} V={V} M={Mm}/{Mh}: O rel {R.relerr(O, ref['O']):.2e}", flush=True)
    hplan = ms.make_chunk_plan(N, Mh)
    loss, hs = ms.miniseq_lmhead_forward(O, L, ms.LmHeadWeights(Wo), hplan)
    rl, rlse, _, _ = R.head_fwd(O, L, Wo)
    print(f"  loss {loss.item():.6f} ref {rl.item():.6f}  lse rel {R.relerr(hs.lse, rlse):.2e}", flush=True)
    dO, dWo = ms.miniseq_lmhead_backward(hs, ms.LmHeadWeights(Wo), hplan)
    valid = (L >= 0)
    scale = torch.where(valid, 1.0 / valid.sum(), 0.0).float()
    rdO, rdWo, _ = R.head_bwd(O, L, Wo, scale)
    print(f"  dO rel {R.relerr(dO, rdO):.2e} dWout rel {R.relerr(dWo, rdWo):.2e}", flush=True)
    dX, gr = ms.miniseq_mlp_backward(dO, saved, w, plan)
    rdX, rdWg, rdWu, rdWd = R.mlp_bwd(dO, X, Wg, Wu, Wd)
    print(f"  dX rel {R.relerr(dX, rdX):.2e} dWg {R.relerr(gr.W_gate, rdWg):.2e} dWu {R.relerr(gr.W_up, rdWu):.2e} dWd {R.relerr(gr.W_down, rdWd):.2e}", flush=True)
    # block step
    st, bg = ms.block_step(X, L, w, ms.LmHeadWeights(Wo), Mm, Mh)
    print(f"  block loss {st[2].item():.6f} dX rel {R.relerr(bg.dX, ref['dX']):.2e} dWout {R.relerr(bg.W_out, ref['dWout']):.2e} dWg {R.relerr(bg.W_gate, ref['dWg']):.2e} dWd {R.relerr(bg.W_down, ref['dWd']):.2e}", flush=True)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    for _ in range(2): ms.block_step(X, L, w, ms.LmHeadWeights(Wo), Mm, Mh, grads=bg, stats=st)
    t0.record()
    for _ in range(3): ms.block_step(X, L, w, ms.LmHeadWeights(Wo), Mm, Mh, grads=bg, stats=st)
    t1.record(); torch.cuda.synchronize()
    ms_ = t0.elapsed_time(t1) / 3
    fl = N * (22 * H * I + 8 * H * V)
    print(f"  block step {ms_:.3f} ms  {N/ms_*1e3:.0f} tok/s  {fl/ms_/1e9:.1f} TFLOP/s", flush=True)
