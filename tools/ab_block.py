"""A/B two libmst builds on the config-2 block step, alternating in one process
so both see the same clocks/power state (dev tool).
usage: python tools/ab_block.py libA.so libB.so [rounds]"""
import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
S, M = 8192, 8
H, I, V = 4096, 14336, 128256
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
g = ms.alloc_block_grads(S, H, I, V, dev)
stats = torch.empty(ms.stats_len(M), device=dev)
handles = []
for spec in libs:
    p, *opts = spec.split(':')
    lib = ctypes.CDLL(p)
    for name, (args, res) in ms._SIGS.items():
        if not hasattr(lib, name): continue  # older build (A/B against a previous revision)
        f = getattr(lib, name); f.argtypes = args; f.restype = res
    h = ctypes.c_void_p()
    assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0, lib.mst_last_error()
    for o in opts:
        k, v = o.split('=')
        assert lib.mst_ctx_set_tuning(h, k.encode(), int(v)) == 0, lib.mst_last_error()
    handles.append((lib, h))
def ws_bytes(lib):
    import ctypes as C
    nb = C.c_size_t()
    assert lib.mst_block_workspace(S, H, I, V, M, M, C.byref(nb)) == 0
    return nb.value


ws = torch.empty(max(ws_bytes(lib) for lib, _ in handles), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
def step(k):
    lib, h = handles[k]
    r = lib.mst_block_step(h, st, X.data_ptr(), L.data_ptr(), Wg.data_ptr(), Wu.data_ptr(), Wd.data_ptr(), Wo.data_ptr(),
                           S, H, I, V, M, M, 0, 1.0, stats.data_ptr(), g.dX.data_ptr(), g.W_gate.data_ptr(),
                           g.W_up.data_ptr(), g.W_down.data_ptr(), g.W_out.data_ptr(), 0, ws.data_ptr(), ws.numel())
    assert r == 0, lib.mst_last_error()
res = {0: [], 1: []}
losses = {}
for k in (0, 1):
    for _ in range(3): step(k)
    torch.cuda.synchronize(); losses[k] = float(stats[2])
for r in range(rounds):
    for k in ((0, 1) if r % 2 == 0 else (1, 0)):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): step(k)
        e1.record(); torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 5)
for k in (0, 1):
    v = sorted(res[k])
    print(f"{libs[k].split('/')[-1]:32s} median {v[len(v)//2]:7.3f} ms  min {v[0]:7.3f}  loss {losses[k]:.6f}  -> {S/v[len(v)//2]*1e3:.0f} tok/s")
print(f"speedup B/A (median): {sorted(res[0])[rounds//2] / sorted(res[1])[rounds//2]:.4f}")
