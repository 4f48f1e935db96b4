"""Role wait breakdown (MST_PROFILE build) for single K5/K6-shaped GEMMs (dev tool)."""
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
dWb = torch.zeros(H, V, device=dev, dtype=torch.bfloat16)
ctx = ms.Context.get(0)
buf = torch.zeros(64 * 8, dtype=torch.int64, device=dev)
cases = {'K5 dX=dl W^T': lambda: ms.debug_gemm(dl, Wo, n, H, V, 0, 0, dX),
         'K6 store f32': lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, dW, beta=0),
         'K6 reduce f32': lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, dW, beta=1),
         'K6-shape bf16 out': lambda: ms.debug_gemm(O, dl, H, V, n, 1, 1, dWb)}
for name, fn in cases.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    buf.zero_()
    ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, buf.data_ptr()))
    ctx.set_timing(True)
    fn()
    torch.cuda.synchronize()
    (t, f), = ctx.take_timing_records()
    ctx.set_timing(False)
    ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, None))
    pw, pt, mf, mt, mtot, ew, eb, etot = buf.view(64, 8)[0].tolist()
    pr = lambda a, b: f"{100 * a / max(b, 1):5.1f}%"
    print(f"{name:20s} {t:6.3f} ms {f/t/1e9:6.0f} TF/s | prod wait-empty {pr(pw, pt)} | mma wait-full {pr(mf, mtot)} "
          f"wait-tmem {pr(mt, mtot)} | epi wait {pr(ew, etot)} busy {pr(eb, etot)}")
