"""Forward GEMM shapes with the weight operand MN-major (SPEC layout) vs K-major (pre-transposed)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
dev = 'cuda'
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
torch.manual_seed(0)
for name, M, N, K in [("K1-like", 1024, 28672, 4096), ("K2-like", 1024, 4096, 14336), ("K3-like", 1024, 128256, 4096)]:
    A = torch.randn(M, K, device=dev).bfloat16()
    W = torch.randn(K, N, device=dev).bfloat16(); WT = W.t().contiguous()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    fl = 2 * M * N * K
    for r in range(2):
        mn = t_ms(lambda: ms.debug_gemm(A, W, M, N, K, 0, 1, C))
        km = t_ms(lambda: ms.debug_gemm(A, WT, M, N, K, 0, 0, C))
    print(f"{name}: B MN-major {fl/mn/1e9:6.0f} TF/s | B K-major {fl/km/1e9:6.0f} TF/s | gain {mn/km:.3f}")
