"""Cycle-level MMA pacing of the engine (dev tool): runs debug_gemm shapes with
MST_PROFILE builds (full and MST_DIAG_NO_TMA), reads the MMA-issuer cycle
counters and reports cycles per 64-deep K block per CTA pair (the tcgen05
floor for 256x256x64 over a pair is 4 x 128 = 512 cycles) and the effective
SM clock = cycles / event time.
usage: python tools/mma_rate.py lib1.so[,lib2.so...]"""
import ctypes, sys, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
from bench import ClockSampler
dev = 'cuda'
import os
PAIRS = [int(x) for x in os.environ.get('PAIRS', '0').split(',')]
NBLK = [int(x) for x in os.environ.get('NBLK', '1').split(',')]
SHAPES = os.environ.get('SHAPES', 'square 8192,K3-like,K6T-like').split(',')
libs = {}
for p in sys.argv[1].split(','):
    lib = ctypes.CDLL(p)
    for name, (args, res) in ms._SIGS.items():
        f = getattr(lib, name); f.argtypes = args; f.restype = res
    h = ctypes.c_void_p(); assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0
    libs[p.split('/')[-1]] = (lib, h)
st = torch.cuda.current_stream().cuda_stream
buf = torch.zeros(64 * 8, dtype=torch.int64, device=dev)
torch.manual_seed(0)
for name, M, N, K, amn, bmn in [("square 8192", 8192, 8192, 8192, 0, 1), ("K3-like", 1024, 128256, 4096, 0, 1),
                                 ("K6T-like", 4096, 128256, 1024, 0, 1), ("l2res", 1024, 8192, 4096, 0, 1),
                                 ("l2res-kmaj", 1024, 8192, 4096, 0, 0)]:
    if name not in SHAPES:
        continue
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if bmn else torch.randn(N, K, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    fl = 2 * M * N * K
    tiles = (M // 256) * ((N + 255) // 256)
    for (tag, (lib, h)), pairs, nbk in [(kv, pr, nb) for kv in libs.items() for pr in PAIRS for nb in NBLK]:
        if pairs:
            assert lib.mst_ctx_set_tuning(h, b"pairs", pairs) == 0
        assert lib.mst_ctx_set_tuning(h, b"debug_nblk", nbk) == 0
        npairs = lib.mst_ctx_num_pairs(h)
        tag = f"{tag} pairs={npairs} nblk={nbk}"
        f = lambda: lib.mst_debug_gemm(h, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, amn, bmn, 0, 0)
        t0 = time.time()
        while time.time() - t0 < 1.0:
            f()
        torch.cuda.synchronize()
        buf.zero_()
        lib.mst_ctx_set_profile_buffer(h, ctypes.c_void_p(buf.data_ptr()))
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(0, 0.002) as clk:
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
        lib.mst_ctx_set_profile_buffer(h, None)
        t = e0.elapsed_time(e1)
        c = buf.view(64, 8)[0].tolist()
        mma_tot = c[4] / npairs
        kb_per_pair = tiles * (K // 64) / npairs  # in 256-column K blocks (a wide K block counts twice)
        print(f"{name:11s} {tag:32s} {t:.3f} ms {fl/t/1e9:6.0f} TF/s | MMA cycles/pair {mma_tot:9.0f} "
              f"-> {mma_tot/kb_per_pair:6.1f} cyc/kblock (floor 512), wait-full {100*c[2]/max(c[4],1):4.1f}% "
              f"| clock {mma_tot/(t*1e3):6.0f} MHz (nvml {clk.summary()['sm_mhz']})", flush=True)
