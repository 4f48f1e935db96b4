"""GPU timeline of one config-2 block step from CUPTI (torch.profiler):
per-kernel device intervals, idle gaps between consecutive kernels, and the
busy share per kernel family (dev tool).  usage: python tools/gap_profile.py"""
import json, sys, time, torch
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
st, gr = ms.block_step(X, L, mlp, head, M, M)
t0 = time.time()
while time.time() - t0 < 2.0:
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == 'CUDA' and e.time_range.end > e.time_range.start]
evs.sort(key=lambda e: e.time_range.start)
# keep the second step only: split on the first chunk_valid kernel of step 2
starts = [i for i, e in enumerate(evs) if 'chunk_valid' in e.name]
seg = evs[starts[1]:] if len(starts) > 1 else evs
t_begin, t_end = seg[0].time_range.start, max(e.time_range.end for e in seg)
busy = {}
gaps = []
prev_end = t_begin
for e in seg:
    k = e.name.replace('(anonymous namespace)::', '').split('(')[0].split('::')[-1][:40]
    d = e.time_range.end - e.time_range.start
    busy.setdefault(k, [0, 0.0])
    busy[k][0] += 1
    busy[k][1] += d
    gaps.append((e.time_range.start - prev_end, k))
    prev_end = max(prev_end, e.time_range.end)
wall = t_end - t_begin
tot_busy = sum(v[1] for v in busy.values())
print(f"step wall {wall/1e3:.3f} ms, kernels busy {tot_busy/1e3:.3f} ms, gaps {sum(max(0, g) for g, _ in gaps)/1e3:.3f} ms "
      f"over {len(seg)} kernels")
for k, (n, d) in sorted(busy.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:42s} x{n:3d} {d/1e3:8.3f} ms  {100*d/wall:5.1f}%")
big = sorted(gaps, reverse=True)[:10]
print("largest gaps (us) before:", [(round(g, 1), k) for g, k in big])
json.dump({"wall_us": wall, "busy": busy, "gaps": gaps}, open('gpurun_out/gap_profile.json', 'w'))
