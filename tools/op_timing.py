"""Per-op / per-launch timing of the config-2 block (dev tool; prints a table)."""
import sys, json, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
M = int(sys.argv[2]) if len(sys.argv) > 2 else 8
H, I, V = 4096, 14336, 128256
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
ctx = ms.Context.get(0)
plan = ms.make_chunk_plan(S, M)
grads = ms.MlpGrads(torch.empty(H, I, device=dev), torch.empty(H, I, device=dev), torch.empty(I, H, device=dev))
dWo = torch.empty(H, V, device=dev)
def run():
    O, sv = ms.miniseq_mlp_forward(X, mlp, plan)
    ctx_rec.append(('mlp_fwd', ctx.take_timing_records()))
    loss, hs = ms.miniseq_lmhead_forward(O, L, head, plan)
    ctx_rec.append(('head_fwd', ctx.take_timing_records()))
    dO, _ = ms.miniseq_lmhead_backward(hs, head, plan, dW_out=dWo)
    ctx_rec.append(('head_bwd', ctx.take_timing_records()))
    dX, _ = ms.miniseq_mlp_backward(dO, sv, mlp, plan, grads=grads)
    ctx_rec.append(('mlp_bwd', ctx.take_timing_records()))
ctx.set_timing(True)
sys.path.insert(0, '.')
from bench import ClockSampler
for it in range(3):
    ctx_rec = []
    if it == 2:
        with ClockSampler(0, 0.005) as clk:
            run()
            torch.cuda.synchronize()
        print("clocks", clk.summary())
    else:
        run()
torch.cuda.synchronize()
tot_ms = tot_fl = 0
out = {}
for name, recs in ctx_rec:
    ms_ = sum(r[0] for r in recs); fl = sum(r[1] for r in recs)
    tot_ms += ms_; tot_fl += fl
    print(f"{name:9s} launches={len(recs):3d} {ms_:8.3f} ms  {fl/ms_/1e9:7.1f} TFLOP/s")
    for k, (t, f) in enumerate(recs[:4]):
        print(f"     launch {k}: {t:7.3f} ms {f/1e12:7.3f} TFLOP -> {f/t/1e9:7.1f} TFLOP/s")
    out[name] = dict(launches=len(recs), ms=ms_, tflops=fl / ms_ / 1e9, per_launch=[(t, f) for t, f in recs])
print(f"total gemm {tot_ms:.3f} ms {tot_fl/tot_ms/1e9:.1f} TFLOP/s; tokens/s (gemm only) {S/tot_ms*1e3:.0f}")
json.dump(out, open('gpurun_out/op_timing.json', 'w'))
