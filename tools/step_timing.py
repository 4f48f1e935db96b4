"""Per-launch timing of the config-2 block_step (chunk-wise schedule) at
sustained clocks (dev tool).  Warms up ~2 s, then records every grouped GEMM
launch of one step with CUDA events while sampling the SM clock; prints
TFLOP/s and efficiency = achieved / (148 SMs x 8192 FLOP/cycle x clock).
With an MST_PROFILE build (MST_LIB=...) also prints per-role wait shares.
usage: python tools/step_timing.py [S] [M] [--prof]"""
import sys, json, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
from bench import ClockSampler

args = [a for a in sys.argv[1:] if not a.startswith('--')]
S = int(args[0]) if args else 8192
M = int(args[1]) if len(args) > 1 else 8
prof = '--prof' in sys.argv
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
import os
for kv in filter(None, os.environ.get('MST_TUNE', '').split(',')):
    k, v = kv.split('=')
    ctx.set_tuning(k, int(v))
st, gr = ms.block_step(X, L, mlp, head, M, M)
t0 = time.time()
while time.time() - t0 < 2.0:
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
buf = torch.zeros(128 * 8, dtype=torch.int64, device=dev)
if prof:
    ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, buf.data_ptr()))
ctx.set_timing(True)
ctx.take_timing_records()
with ClockSampler(0, 0.005) as clk:
    for it in range(3):
        if prof:
            buf.zero_()
            ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, buf.data_ptr()))
        ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
        torch.cuda.synchronize()
        recs = ctx.take_timing_records()
cs = clk.summary()
mhz = cs['sm_mhz'] or 1965
peak = 148 * 8192 * mhz * 1e6
print("clocks", cs)
tot_ms = sum(r[0] for r in recs)
tot_fl = sum(r[1] for r in recs)
kinds = {}
for k, (t, f) in enumerate(recs):
    kinds.setdefault(round(f / 1e9), []).append((k, t))
for gf, ts in sorted(kinds.items()):
    avg = sum(t for _, t in ts) / len(ts)
    print(f"{len(ts):3d} x {gf/1e3:6.3f} TFLOP avg {avg:7.3f} ms  {gf/avg:7.1f} TFLOP/s  "
          f"eff/clock {100*gf*1e9/(avg/1e3)/peak:5.1f}%  share {100*avg*len(ts)/tot_ms:5.1f}%  launches {[k for k,_ in ts][:4]}...")
print(f"total gemm {tot_ms:.3f} ms {tot_fl/tot_ms/1e9:.1f} TFLOP/s eff/clock {100*tot_fl/(tot_ms/1e3)/peak:.1f}%; "
      f"tokens/s (gemm only) {S/tot_ms*1e3:.0f}")
out = dict(clocks=cs, per_launch=recs)
if prof:
    c = buf.view(128, 8).cpu().tolist()
    for k, (t, f) in enumerate(recs[:16]):
        pw, pt, mf, mt, mtot, ew, eb, etot = c[k]
        pr = lambda a, b: f"{100 * a / max(b, 1):5.1f}%"
        npairs = ctx.num_pairs
        kb = f / (2 * 256 * 256 * 64) / npairs
        cyc = mtot / npairs
        print(f"  launch {k}: {t:6.3f} ms {f / t / 1e9:7.1f} TF/s | prod wait-empty {pr(pw, pt)} | "
              f"mma wait-full {pr(mf, mtot)} wait-tmem {pr(mt, mtot)} | epi wait {pr(ew, etot)} busy {pr(eb, etot)} | "
              f"{cyc / kb:5.0f} cyc/kblock (floor 512) clock {cyc / (t * 1e3):5.0f} MHz")
    out['roles'] = c[:len(recs)]
json.dump(out, open('gpurun_out/step_timing%s.json' % ('_prof' if prof else ''), 'w'))
