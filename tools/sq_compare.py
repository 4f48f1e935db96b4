"""8192^3 bf16 GEMM: cuBLAS (torch.matmul) and the engine (mst_debug_gemm), a
few launches each (dev tool: ncu target for comparing the two kernels)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
n = 8192
A = torch.randn(n, n, device='cuda').bfloat16()
B = torch.randn(n, n, device='cuda').bfloat16()
C = torch.empty(n, n, device='cuda').bfloat16()
ctx = ms.Context.get(0)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    torch.matmul(A, B, out=C)
for _ in range(3):
    ms._check(ctx.lib.mst_debug_gemm(ctx.handle, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), n, n, n, 0, 1, 0, 0))
torch.cuda.synchronize()
