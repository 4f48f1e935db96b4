"""Longest sequence one B200 trains on (one forward + backward of the
decoder, fp32 gradients, per-layer recompute), standard blocks (M=1) vs
mini-sequence blocks — the paper's model-level claim (Table 3
kind of result) on Llama3-8B layer shapes with `layers` decoder layers.
Each probe runs in a fresh process; bisection on S in multiples of 8192.
usage: python tools/model_maxseq.py [layers]  (dev tool, JSON lines)"""
import json, subprocess, sys, time

CHILD = r'''
import json, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import model as mdl
layers, S, mm, mh = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = mdl.ModelConfig(d=4096, I=14336, V=128256, heads=32, G=4, layers=layers, S=S, B=1, M_mlp=mm, M_head=mh,
                      recompute=True)
try:
    m = mdl.Model(cfg)
    g = torch.Generator().manual_seed(0)
    tok = torch.randint(0, cfg.V, (1, S), generator=g).int().cuda()
    lab = torch.randint(0, cfg.V, (1, S), generator=g).int().cuda()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    loss, saved = m.forward(tok, lab, check=False)
    grads = m.backward(saved)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps(dict(fits=True, S=S, M_mlp=mm, M_head=mh, ms=e0.elapsed_time(e1),
                          peak_gb=torch.cuda.max_memory_allocated() / 1e9, loss=float(loss))))
except (torch.OutOfMemoryError, RuntimeError) as e:
    print(json.dumps(dict(fits=False, S=S, M_mlp=mm, M_head=mh, error=str(e)[:120])))
'''


def probe(layers, S, mst):
    mm, mh = ((S + 8191) // 8192, (S + 4095) // 4096) if mst else (1, 1)
    out = subprocess.run([sys.executable, "-c", CHILD, str(layers), str(S), str(mm), str(mh)], capture_output=True,
                         text=True, timeout=900)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else dict(fits=False, S=S, error=out.stderr[-200:])


layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for mst in (False, True):
    lo, hi, best = 8192, 1024 * 1024, None
    t0 = time.time()
    while hi - lo > 8192 and time.time() - t0 < 1500:
        mid = (lo + hi) // 2 // 8192 * 8192
        r = probe(layers, mid, mst)
        r["mode"] = "mini-sequence" if mst else "standard"
        print(json.dumps(r), flush=True)
        if r["fits"]:
            lo, best = mid, r
        else:
            hi = mid
    print(json.dumps(dict(summary=True, layers=layers, mode="mini-sequence" if mst else "standard",
                          max_seq_len=lo, best=best)), flush=True)
