"""A/B/C.. of libmst builds and/or tuning knobs on the chunk-wise block step,
interleaved in one process so every variant sees the same clocks and power
state (dev tool).  Also compares each variant's outputs with variant 0's:
loss, dX (bitwise count) and the weight gradients (max |diff| / max |ref|).

usage: python tools/ab_multi.py [--S 8192] [--M 8] [--MH M] [--rounds 8] [--steps 5]
                                 spec [spec ...]
spec = path/to/libmst.so[:key=value[:key=value ...]]   (knobs: mst_ctx_set_tuning)
"""
import argparse
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--S', type=int, default=8192)
ap.add_argument('--M', type=int, default=8)
ap.add_argument('--MH', type=int, default=0)
ap.add_argument('--H', type=int, default=4096)
ap.add_argument('--I', type=int, default=14336)
ap.add_argument('--V', type=int, default=128256)
ap.add_argument('--rounds', type=int, default=8)
ap.add_argument('--steps', type=int, default=5)
ap.add_argument('specs', nargs='+')
a = ap.parse_args()
S, M, MH, H, I, V = a.S, a.M, a.MH or a.M, a.H, a.I, a.V
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
stats = torch.empty(ms.stats_len(max(M, MH)), device=dev)
handles = []
for spec in a.specs:
    p, *opts = spec.split(':')
    lib = ctypes.CDLL(p)
    for name, (args, res) in ms._SIGS.items():
        if not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    h = ctypes.c_void_p()
    assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0, lib.mst_last_error()
    for o in opts:
        k, v = o.split('=')
        assert lib.mst_ctx_set_tuning(h, k.encode(), int(v)) == 0, lib.mst_last_error()
    nb = ctypes.c_size_t()
    assert lib.mst_ctx_block_workspace(h, S, H, I, V, M, MH, ctypes.byref(nb)) == 0, lib.mst_last_error()
    handles.append((lib, h, nb.value))
ws = torch.empty(max(x[2] for x in handles), dtype=torch.uint8, device=dev)
grads = [ms.alloc_block_grads(S, H, I, V, dev) for _ in handles]
st = torch.cuda.current_stream().cuda_stream


def step(k):
    lib, h, _ = handles[k]
    g = grads[k]
    r = lib.mst_block_step(h, st, X.data_ptr(), L.data_ptr(), Wg.data_ptr(), Wu.data_ptr(), Wd.data_ptr(),
                           Wo.data_ptr(), S, H, I, V, M, MH, 0, 1.0, stats.data_ptr(), g.dX.data_ptr(),
                           g.W_gate.data_ptr(), g.W_up.data_ptr(), g.W_down.data_ptr(), g.W_out.data_ptr(), 0,
                           ws.data_ptr(), ws.numel())
    assert r == 0, lib.mst_last_error()


losses = []
for k in range(len(handles)):
    for _ in range(3):
        step(k)
    torch.cuda.synchronize()
    losses.append(float(stats[2]))
ref = grads[0]
for k in range(1, len(handles)):
    g = grads[k]
    same_dx = int((g.dX.view(torch.int16) == ref.dX.view(torch.int16)).sum())
    rel = {n: float((getattr(g, n) - getattr(ref, n)).abs().max() / getattr(ref, n).abs().max())
           for n in ('W_gate', 'W_up', 'W_down', 'W_out')}
    print(f"variant {k}: loss {losses[k]:.6f} vs {losses[0]:.6f}; dX bitwise {same_dx}/{g.dX.numel()}; "
          + " ".join(f"{n} {v:.2e}" for n, v in rel.items()))
res = {k: [] for k in range(len(handles))}
for r in range(a.rounds):
    order = list(range(len(handles)))
    if r % 2:
        order.reverse()
    for k in order:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            step(k)
        e1.record()
        torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / a.steps)
base = sorted(res[0])[a.rounds // 2]
for k in range(len(handles)):
    v = sorted(res[k])
    med = v[a.rounds // 2]
    print(f"{a.specs[k].split('/')[-1]:48s} median {med:7.3f} ms  min {v[0]:7.3f}  -> {S / med * 1e3:8.0f} tok/s"
          f"  x{base / med:.4f}  ws {handles[k][2] / 1e9:.3f} GB")
