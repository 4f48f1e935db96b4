"""Role wait shares of the engine on one GEMM shape (MST_PROFILE build; dev tool).
usage: MST_LIB=.../libmst_prof.so [MST_TUNE=k=v] python tools/shape_prof.py M N K a_mn b_mn [out_f32 beta]"""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
M, N, K, amn, bmn = map(int, sys.argv[1:6])
f32, beta = (map(int, sys.argv[6:8]) if len(sys.argv) > 7 else (0, 0))
ctx = ms.Context.get(0)
for kv in filter(None, os.environ.get('MST_TUNE', '').split(',')):
    k, v = kv.split('=')
    ctx.set_tuning(k, int(v))
st = torch.cuda.current_stream().cuda_stream
A = torch.randn(K, M, device='cuda').bfloat16() if amn else torch.randn(M, K, device='cuda').bfloat16()
B = torch.randn(K, N, device='cuda').bfloat16() if bmn else torch.randn(N, K, device='cuda').bfloat16()
C = torch.zeros(M, N, device='cuda', dtype=torch.float32 if f32 else torch.bfloat16)
f = lambda: ms._check(ctx.lib.mst_debug_gemm(ctx.handle, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                             amn, bmn, f32, beta))
for _ in range(20): f()
torch.cuda.synchronize()
buf = torch.zeros(64 * 8, dtype=torch.int64, device='cuda')
ms._check(ctx.lib.mst_ctx_set_profile_buffer(ctx.handle, buf.data_ptr()))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
c = [int(x) for x in buf.view(64, 8).sum(0).cpu().tolist()]
pw, pt, mf, mt, mtot, ew, eb, etot = c
npairs = ctx.num_pairs
kb = 2 * M * N * K / (2 * 256 * 256 * 64) / npairs
tiles = (M // 256) * (N // 256) / npairs
cyc = mtot / npairs
pr = lambda a, b: f"{100 * a / max(b, 1):5.1f}%"
feed = f"mma wait-feed {pr(pt, mtot)} | " if os.environ.get('MST_PROF2') else f"prod wait-empty {pr(pw, pt)} | "
print(f"{M}x{N}x{K} a_mn={amn} b_mn={bmn}: {t:.3f} ms | {feed} mma wait-full {pr(mf, mtot)} "
      f"wait-tmem {pr(mt, mtot)} | epi wait {pr(ew, etot)} busy {pr(eb, etot)} | {cyc / kb:5.0f} cyc/kblock "
      f"{cyc / tiles:7.0f} cyc/tile (mma floor {512 * kb / tiles:5.0f}) clock {cyc / (t * 1e3):5.0f} MHz")
