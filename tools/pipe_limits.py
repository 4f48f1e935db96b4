"""Mainloop limits: full kernel vs no-MMA (TMA only) vs no-TMA (MMA only) builds (dev tool)."""
import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
dev = 'cuda'
libs = {}
for tag in ('', '_nomma', '_notma'):
    lib = ctypes.CDLL(f'paper_2407_15892_b200/lib/libmst{tag}.so')
    for name, (args, res) in ms._SIGS.items():
        f = getattr(lib, name); f.argtypes = args; f.restype = res
    h = ctypes.c_void_p(); assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0
    libs[tag or 'full'] = (lib, h)
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
for name, M, N, K, amn, bmn in [("K3-like", 1024, 128256, 4096, 0, 1), ("square 8192", 8192, 8192, 8192, 0, 1),
                                 ("K5-like", 1024, 4096, 128256, 0, 0), ("K6T-like", 4096, 128256, 1024, 0, 1)]:
    A = torch.randn(M, K, device=dev).bfloat16() if not amn else torch.randn(K, M, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if bmn else torch.randn(N, K, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    fl = 2 * M * N * K
    out = []
    for tag, (lib, h) in libs.items():
        f = lambda: lib.mst_debug_gemm(h, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, amn, bmn, 0, 0)
        t = min(t_ms(f) for _ in range(2))
        out.append(f"{tag} {t:.3f} ms ({fl/t/1e9:.0f} TF/s-equiv)")
    print(f"{name:12s} " + " | ".join(out), flush=True)
