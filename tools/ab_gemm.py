"""A/B two libmst builds on debug_gemm shapes, alternating in one process (dev tool).
usage: python tools/ab_gemm.py libA.so[:key=v,...] libB.so[:key=v,...]"""
import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
dev = 'cuda'
handles = []
for spec in sys.argv[1:3]:
    p, *opts = spec.split(':')
    lib = ctypes.CDLL(p)
    for name, (args, res) in ms._SIGS.items():
        if not hasattr(lib, name): continue  # older build (A/B against a previous revision)
        f = getattr(lib, name); f.argtypes = args; f.restype = res
    h = ctypes.c_void_p(); assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0
    for o in opts:
        for kv in o.split(','):
            k, v = kv.split('=')
            assert lib.mst_ctx_set_tuning(h, k.encode(), int(v)) == 0, lib.mst_last_error()
    handles.append((spec, lib, h))
st = torch.cuda.current_stream().cuda_stream


def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


torch.manual_seed(0)
for name, M, N, K, amn, bmn in [("square 8192", 8192, 8192, 8192, 0, 1), ("K3-like", 1024, 128256, 4096, 0, 1),
                                 ("K5-like", 1024, 4096, 128256, 0, 0), ("K6T-like", 4096, 128256, 1024, 0, 1)]:
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if bmn else torch.randn(N, K, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    fl = 2 * M * N * K
    res = [[] for _ in handles]
    for r in range(4):
        for i, (spec, lib, h) in enumerate(handles):
            f = lambda: lib.mst_debug_gemm(h, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, amn, bmn, 0, 0)
            res[i].append(t_ms(f))
    print(f"{name:12s} " + " | ".join(f"{handles[i][0].split('/')[-1]} {min(r):.3f} ms {fl/min(r)/1e9:6.0f} TF/s"
                                       for i, r in enumerate(res)), flush=True)
