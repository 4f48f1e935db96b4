"""K5 / K6 in isolation vs grouped (dev tool)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
dev = 'cuda'
n, H, V = 1024, 4096, 128256
torch.manual_seed(0)
dl = (torch.randn(n, V, device=dev) * 1e-4).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
O = torch.randn(n, H, device=dev).bfloat16()
dX = torch.empty(n, H, device=dev, dtype=torch.bfloat16)
dW = torch.zeros(H, V, device=dev, dtype=torch.float32)
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
# warm clocks
t_ms(lambda: ms.debug_gemm(dl, Wo, n, H, V, 0, 0, dX), 30)
for r in range(2):
    k5 = t_ms(lambda: ms.debug_gemm(dl, Wo, n, H, V, 0, 0, dX))            # dX = dl W^T  (A K-major, B K-major)
    k6s = t_ms(lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, dW, beta=0))     # dW = O^T dl  store
    k6r = t_ms(lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, dW, beta=1))     # dW += O^T dl reduce-add
    fl = 2 * n * H * V
    print(f"K5 {k5:.3f} ms ({fl/k5/1e9:.0f} TF/s) | K6 store {k6s:.3f} ms ({fl/k6s/1e9:.0f}) | K6 reduce-add {k6r:.3f} ms ({fl/k6r/1e9:.0f}) | sum K5+K6r {k5+k6r:.3f}")
