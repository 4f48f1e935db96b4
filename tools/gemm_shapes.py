"""Sustained TFLOP/s and per-clock efficiency of the engine on single GEMM
shapes (mst_debug_gemm), each run back to back for ~1.5 s (dev tool).
usage: MST_TUNE=k=v,... python tools/gemm_shapes.py"""
import os, sys, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
from bench import ClockSampler
ctx = ms.Context.get(0)
for kv in filter(None, os.environ.get('MST_TUNE', '').split(',')):
    k, v = kv.split('=')
    ctx.set_tuning(k, int(v))
st = torch.cuda.current_stream().cuda_stream
SHAPES = [  # name, M, N, K, a_mn, b_mn, out_f32, beta
    ("square 8192 bf16", 8192, 8192, 8192, 0, 1, 0, 0),
    ("K3 1024x128256x4096", 1024, 128256, 4096, 0, 1, 0, 0),
    ("K5 1024x4096x128256", 1024, 4096, 128256, 0, 0, 0, 0),
    ("K6 K=1024 bf16", 4096, 128256, 1024, 0, 1, 0, 0),
    ("K6 K=1024 f32 store", 4096, 128256, 1024, 0, 1, 1, 0),
    ("K6 K=1024 f32 reduce", 4096, 128256, 1024, 0, 1, 1, 1),
    ("K6 K=2048 f32 reduce", 4096, 128256, 2048, 0, 1, 1, 1),
    ("K6 K=4096 f32 reduce", 4096, 128256, 4096, 0, 1, 1, 1),
    ("K8 14336x4096x1024 f32 reduce", 14336, 4096, 1024, 0, 1, 1, 1),
    ("T K=512 bf16", 4096, 128256, 512, 0, 1, 0, 0),
    ("T K=2048 bf16", 4096, 128256, 2048, 0, 1, 0, 0),
    ("T K=4096 bf16", 4096, 65536, 4096, 0, 1, 0, 0),
    ("T K=1024 bf16 B K-major", 4096, 128256, 1024, 0, 0, 0, 0),
    ("T K=1024 bf16 A MN-major", 4096, 128256, 1024, 1, 1, 0, 0),
]
only = sys.argv[1:]
for name, M, N, K, amn, bmn, f32, beta in SHAPES:
    if only and not any(o in name for o in only):
        continue
    A = torch.randn(K, M, device='cuda').bfloat16() if amn else torch.randn(M, K, device='cuda').bfloat16()
    B = torch.randn(K, N, device='cuda').bfloat16() if bmn else torch.randn(N, K, device='cuda').bfloat16()
    C = torch.zeros(M, N, device='cuda', dtype=torch.float32 if f32 else torch.bfloat16)
    f = lambda: ms._check(ctx.lib.mst_debug_gemm(ctx.handle, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                                 amn, bmn, f32, beta))
    for _ in range(3): f()
    torch.cuda.synchronize()
    t0 = time.time()
    while time.time() - t0 < 0.7: f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    n = 0
    with ClockSampler(0, 0.01) as clk:
        e0.record()
        t0 = time.time()
        while time.time() - t0 < 1.0:
            for _ in range(4): f()
            n += 4
            torch.cuda.synchronize()
        e1.record(); torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1) / n
    cs = clk.summary()
    tf = 2 * M * N * K / ms_ / 1e9
    print(f"{name:32s} {ms_:8.3f} ms {tf:7.1f} TF/s  clock {cs['sm_mhz']} MHz  eff/clock "
          f"{100 * tf / (148 * 8192 * cs['sm_mhz'] * 1e-6):5.1f}%  power {cs['power_w_median']:.0f} W", flush=True)
    del A, B, C
