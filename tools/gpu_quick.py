"""Quick GPU sanity check of the tcgen05 engine against torch fp32 (dev tool)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms

torch.manual_seed(0)
dev = 'cuda'
def rel(a, b):
    a = a.float(); b = b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()

ok = True
for (M, N, K) in [(256, 256, 64), (256, 256, 1024), (512, 768, 4096), (296, 200, 136), (1024, 4096, 14336)]:
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            A = torch.randn(M, K, device=dev).bfloat16()
            B = torch.randn(K, N, device=dev).bfloat16()
            a_in = A.t().contiguous() if a_mn else A
            b_in = B if b_mn else B.t().contiguous()
            ref = A.float() @ B.float()
            for f32 in (0, 1):
                out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
                ms.debug_gemm(a_in, b_in, M, N, K, a_mn, b_mn, out)
                torch.cuda.synchronize()
                e = rel(out, ref)
                flag = e < (1e-5 if f32 else 8e-3)
                ok &= flag
                print(f"gemm M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} f32={f32} rel={e:.2e} {'OK' if flag else 'FAIL'}", flush=True)
print("GEMM", "PASS" if ok else "FAIL")
