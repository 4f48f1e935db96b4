"""cuBLAS (torch.matmul) running the same GEMM sequence as one chunk-wise
config-2 block step (8 chunks of 1024 tokens, K1..K10 shapes, no fused
epilogues) in steady state under the power cap (dev tool).  The comparison
point for the engine's GEMM time per step (tools/step_timing.py).
usage: python tools/cublas_step.py"""
import sys, time, torch
sys.path.insert(0, '.')
from bench import ClockSampler
dev = 'cuda'
n, H, I, V, M = 1024, 4096, 14336, 128256, 8
torch.manual_seed(0)
bf = torch.bfloat16
X = torch.randn(n, H, device=dev, dtype=bf)
Wgu = torch.randn(H, 2 * I, device=dev, dtype=bf) * 0.02
Wd = torch.randn(I, H, device=dev, dtype=bf) * 0.02
Wo = torch.randn(H, V, device=dev, dtype=bf) * 0.02
h = torch.randn(n, I, device=dev, dtype=bf)
dl = torch.randn(n, V, device=dev, dtype=bf)
dGU = torch.randn(n, 2 * I, device=dev, dtype=bf)
dWo = torch.zeros(H, V, device=dev, dtype=torch.float32)
dWd = torch.zeros(I, H, device=dev, dtype=torch.float32)
dWgu = torch.zeros(H, 2 * I, device=dev, dtype=torch.float32)
has_out_dtype = True
try:
    torch.mm(X.t(), h[:, :8], out_dtype=torch.float32)
except TypeError:
    has_out_dtype = False
flops = 0


def acc(dst, a, b):
    # fp32 accumulate like the engine's dW reduce-add (bf16 x bf16 -> fp32 when available)
    if has_out_dtype:
        dst.add_(torch.mm(a, b, out_dtype=torch.float32))
    else:
        dst.add_(torch.mm(a, b).float())


def step():
    for j in range(M):
        torch.mm(X, Wgu)                 # K1
        torch.mm(h, Wd)                  # K2
        torch.mm(X, Wo)                  # K3'
        torch.mm(dl, Wo.t())             # K5
        acc(dWo, X.t(), dl)              # K6
        torch.mm(X, Wd.t())              # K7a
        acc(dWd, h.t(), X)               # K8
        torch.mm(dGU, Wgu.t())           # K9
        acc(dWgu, X.t(), dGU)            # K10


fl = M * (2 * n * H * 2 * I + 2 * n * I * H + 3 * 2 * n * H * V + 2 * n * H * I + 2 * n * I * H + 2 * 2 * n * I * H * 2)
t0 = time.time()
while time.time() - t0 < 3.0:
    step()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
with ClockSampler(0, 0.005) as clk:
    e0.record()
    for _ in range(5):
        step()
    e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
print(f"cuBLAS chunk-wise step GEMMs: {t:.3f} ms, {fl / t / 1e9:.0f} TFLOP/s executed ({fl/1e12:.2f} TFLOP/step), "
      f"out_dtype fp32: {has_out_dtype}, clocks {clk.summary()}")
