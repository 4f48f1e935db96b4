import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
tag, shape = sys.argv[1], int(sys.argv[2])
dev = 'cuda'
lib = ctypes.CDLL(f'paper_2407_15892_b200/lib/libmst{tag}.so')
for name, (args, res) in ms._SIGS.items():
    f = getattr(lib, name); f.argtypes = args; f.restype = res
h = ctypes.c_void_p(); assert lib.mst_ctx_create(0, ctypes.byref(h)) == 0
st = torch.cuda.current_stream().cuda_stream
M, N, K, amn, bmn = [(1024, 128256, 4096, 0, 1), (8192, 8192, 8192, 0, 1), (1024, 4096, 128256, 0, 0), (4096, 128256, 1024, 0, 1)][shape]
A = torch.randn(M, K, device=dev).bfloat16(); B = (torch.randn(K, N, device=dev) if bmn else torch.randn(N, K, device=dev)).bfloat16()
C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
r = lib.mst_debug_gemm(h, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, amn, bmn, 0, 0)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): lib.mst_debug_gemm(h, st, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, amn, bmn, 0, 0)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f"lib{tag or '-full'} shape{shape} rc={r} {t:.3f} ms {2*M*N*K/t/1e9:.0f} TF/s-equiv", flush=True)
