"""Per-op / per-launch timing of the config-2 block at sustained clocks (dev tool).
Warms up ~2 s of block steps, then times each op with per-launch CUDA events
while sampling the SM clock; reports TFLOP/s and efficiency = achieved /
(148 SMs x 8192 FLOP/cycle x sampled clock)."""
import sys, json, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
from bench import ClockSampler

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
st, gr = ms.block_step(X, L, mlp, head, M, M)
t0 = time.time()
while time.time() - t0 < 2.0:
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
ctx.set_timing(True)
ctx.take_timing_records()
out = {}
with ClockSampler(0, 0.005) as clk:
    recs_all = []
    for it in range(2):
        recs = []
        O, sv = ms.miniseq_mlp_forward(X, mlp, plan); recs.append(('mlp_fwd', ctx.take_timing_records()))
        loss, _, _, dO, _ = ms.miniseq_lmhead_fused(O, L, head, plan, dW_out=dWo); recs.append(('head_fused', ctx.take_timing_records()))
        dX, _ = ms.miniseq_mlp_backward(dO, sv, mlp, plan, grads=grads); recs.append(('mlp_bwd', ctx.take_timing_records()))
        recs_all.append(recs)
cs = clk.summary()
mhz = cs['sm_mhz'] or 1965
peak = 148 * 8192 * mhz * 1e6
print("clocks", cs)
tot_ms = tot_fl = 0
for name, recs in recs_all[-1]:
    ms_ = sum(r[0] for r in recs); fl = sum(r[1] for r in recs)
    tot_ms += ms_; tot_fl += fl
    eff = fl / (ms_ / 1e3) / peak
    print(f"{name:9s} launches={len(recs):3d} {ms_:8.3f} ms  {fl/ms_/1e9:7.1f} TFLOP/s  eff/clock {100*eff:5.1f}%")
    kinds = {}
    for t, f in recs:
        kinds.setdefault(round(f / 1e9), []).append(t)
    for gf, ts in sorted(kinds.items()):
        avg = sum(ts) / len(ts)
        print(f"     {len(ts):2d} x {gf/1e3:6.3f} TFLOP  avg {avg:7.3f} ms  {gf/avg/1e6:7.1f} TFLOP/s  eff/clock {100*gf*1e9/(avg/1e3)/peak:5.1f}%")
    out[name] = dict(launches=len(recs), ms=ms_, tflops=fl / ms_ / 1e9, eff=eff, per_launch=recs)
print(f"total gemm {tot_ms:.3f} ms {tot_fl/tot_ms/1e9:.1f} TFLOP/s eff/clock {100*tot_fl/(tot_ms/1e3)/peak:.1f}%; tokens/s (gemm only) {S/tot_ms*1e3:.0f}")
out['clocks'] = cs
json.dump(out, open('gpurun_out/op_timing.json', 'w'))
