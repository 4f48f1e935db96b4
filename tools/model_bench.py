"""Whole-decoder measurement at Llama3-8B layer shapes (dev tool): tokens/s
of forward+backward and peak device memory for standard (M=1) vs
mini-sequence blocks, with and without the per-layer recompute policy —
the paper's model-level claim (memory down, throughput kept).  Each
configuration runs in a fresh process so the peaks are clean.
usage: python tools/model_bench.py [layers] [S ...]"""
import json, subprocess, sys

CHILD = r'''
import json, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import model as mdl
layers, S, mm, mh, rc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5] == "1"
cfg = mdl.ModelConfig(d=4096, I=14336, V=128256, heads=32, G=4, layers=layers, S=S, B=1, M_mlp=mm, M_head=mh,
                      recompute=rc)
m = mdl.Model(cfg)
g = torch.Generator().manual_seed(0)
tok = torch.randint(0, cfg.V, (1, S), generator=g).int().cuda()
lab = torch.randint(0, cfg.V, (1, S), generator=g).int().cuda()
torch.cuda.synchronize()
base = torch.cuda.memory_allocated()
nparam = sum(t.numel() for t in m.w.named().values())
try:
    for _ in range(2):
        loss, saved = m.forward(tok, lab, check=False)
        grads = m.backward(saved)
        del saved, grads
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        loss, saved = m.forward(tok, lab, check=False)
        grads = m.backward(saved)
        del saved, grads
    e1.record()
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / n
    peak = torch.cuda.max_memory_allocated() - base
    print(json.dumps(dict(layers=layers, S=S, M_mlp=mm, M_head=mh, recompute=rc, ms_per_step=ms_step,
                          tokens_per_s=S / ms_step * 1e3, peak_over_weights_gb=peak / 1e9,
                          fp32_grads_gb=4 * nparam / 1e9, activations_and_workspace_gb=(peak - 4 * nparam) / 1e9,
                          weights_gb=base / 1e9, loss=float(loss))))
except torch.OutOfMemoryError as e:
    print(json.dumps(dict(layers=layers, S=S, M_mlp=mm, M_head=mh, recompute=rc, oom=str(e)[:160])))
'''

layers = sys.argv[1] if len(sys.argv) > 1 else "2"
seqs = sys.argv[2:] or ["8192", "32768"]
for S in seqs:
    for (mm, mh, rc) in ((1, 1, 0), (4, 16, 0), (1, 1, 1), (4, 16, 1)):
        out = subprocess.run([sys.executable, "-c", CHILD, layers, S, str(mm), str(mh), str(rc)], capture_output=True,
                             text=True)
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        print(lines[-1] if lines else json.dumps(dict(S=S, M_mlp=mm, M_head=mh, recompute=rc,
                                                       error=out.stderr[-300:])), flush=True)
