"""K6-shaped GEMM with MN-major vs K-major operands; long-K with MN-major (dev tool)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
dev = 'cuda'
n, H, V = 1024, 4096, 128256
torch.manual_seed(0)
dl = (torch.randn(n, V, device=dev) * 1e-4).bfloat16()
O = torch.randn(n, H, device=dev).bfloat16()
OT = O.t().contiguous(); dlT = dl.t().contiguous()
out = torch.zeros(H, V, device=dev, dtype=torch.bfloat16)
X = torch.randn(n, 16384, device=dev).bfloat16(); W = torch.randn(16384, 4096, device=dev).bfloat16()
XT = X.t().contiguous()
o2 = torch.zeros(n, 4096, device=dev, dtype=torch.bfloat16)
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
fl6 = 2 * n * H * V; fl2 = 2 * n * 16384 * 4096
t_ms(lambda: ms.debug_gemm(OT, dlT, H, V, n, 0, 0, out), 30)
for r in range(2):
    a = t_ms(lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, out))
    b = t_ms(lambda: ms.debug_gemm(OT, dlT, H, V, n, 0, 0, out))
    c = t_ms(lambda: ms.debug_gemm(OT, dl, H, V, n, 0, 1, out))
    d = t_ms(lambda: ms.debug_gemm(O, dlT, H, V, n, 1, 0, out))
    e = t_ms(lambda: ms.debug_gemm(X, W, n, 4096, 16384, 0, 1, o2))
    f = t_ms(lambda: ms.debug_gemm(XT, W, n, 4096, 16384, 1, 1, o2))
    print(f"K6 A MN,B MN {fl6/a/1e9:5.0f} | A K,B K {fl6/b/1e9:5.0f} | A K,B MN {fl6/c/1e9:5.0f} | A MN,B K {fl6/d/1e9:5.0f} TF/s || long-K(16384) A K,B MN {fl2/e/1e9:5.0f} | A MN,B MN {fl2/f/1e9:5.0f}")
