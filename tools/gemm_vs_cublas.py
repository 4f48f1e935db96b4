"""Engine vs cuBLAS (torch.matmul) on identical shapes, same process, interleaved (dev tool)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
torch.manual_seed(0)
dev = 'cuda'
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
shapes = [("square 8192^3", 8192, 8192, 8192, 0, 1),
          ("K1-like n=1024 N=28672 K=4096", 1024, 28672, 4096, 0, 1),
          ("K2-like n=1024 N=4096 K=14336", 1024, 4096, 14336, 0, 1),
          ("K3-like n=1024 N=128256 K=4096", 1024, 128256, 4096, 0, 1),
          ("K5-like n=1024 N=4096 K=128256", 1024, 4096, 128256, 0, 0),
          ("big 4096x28672x4096", 4096, 28672, 4096, 0, 1)]
for name, M, N, K, a_mn, b_mn in shapes:
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if b_mn else torch.randn(N, K, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ours = lambda: ms.debug_gemm(A, B, M, N, K, a_mn, b_mn, C)
    ref = (lambda: torch.matmul(A, B, out=C)) if b_mn else (lambda: torch.matmul(A, B.t(), out=C))
    r = []
    for _ in range(3):
        r.append((t_ms(ours), t_ms(ref)))
    o = min(x[0] for x in r); c = min(x[1] for x in r)
    fl = 2 * M * N * K
    print(f"{name:34s} ours {o:7.3f} ms {fl/o/1e9:7.1f} TF/s | cuBLAS {c:7.3f} ms {fl/c/1e9:7.1f} TF/s | ratio {c/o:5.3f}", flush=True)
