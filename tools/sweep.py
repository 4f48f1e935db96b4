"""M-sweep and max-sequence measurements (BASELINE.json configs 3 and 4).

  python tools/sweep.py sweep-m   # config 3: Llama2-7B widths, S=16384, M in {1,2,4,8}
  python tools/sweep.py sweep-m2  # config 2: Llama3-8B widths, S=8192, M in {1,2,4,8,16}
  python tools/sweep.py sweep-pairs  # config 2: (M_mlp, M_head) pairs incl. the paper's (4, 16)
  python tools/sweep.py seq       # Llama3-8B widths, S = 8K..128K at chunk 1024 / 4096
  python tools/sweep.py max-seq   # config 4: Llama3-8B widths, bisection on S under the device budget
  python tools/sweep.py long      # config 4: S=65536, M=16, timed steps

Mirrors the reference's `cmd_sweep_m` (one row per M with
peak bytes, flops, step time) and `cmd_max_seq` (bisection
on S with dry runs).  Every row runs real steps on the GPU through the C ABI.
Writes JSON lines to stdout.
"""
from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_15892_b200 import miniseq as ms  # noqa: E402


def flops_per_token(H, I, V):
    """FLOPs the block step executes per token (18HI + 6HV: no recompute GEMM
    is left in the chunk-wise schedule with the single-pass head), so the
    reported rate can be compared with the hardware peak."""
    return 18.0 * H * I + 6.0 * H * V


def make(S, H, I, V, dev, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    X = torch.randn(S, H, device=dev, generator=g, dtype=torch.bfloat16)  # no fp32 temporary (max-seq)
    W = [(0.02 * torch.randn(*s, device=dev, generator=g)).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (S,), device=dev, generator=g, dtype=torch.int32)
    return X, L, W


def timed_steps(X, L, W, M_mlp, M_head, steps=3, warmup=2):
    S, H = X.shape
    I, V = W[0].shape[1], W[3].shape[1]
    mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
    grads = ms.alloc_block_grads(S, H, I, V, X.device)
    stats = torch.empty(ms.stats_len(min(S, M_head)), device=X.device)
    ws = torch.empty(ms.block_workspace_bytes(S, H, I, V, M_mlp, M_head, ms.Context.get(X.device.index)),
                     dtype=torch.uint8, device=X.device)
    for _ in range(warmup):
        ms.block_step(X, L, mlp, head, M_mlp, M_head, grads=grads, stats=stats, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ms.block_step(X, L, mlp, head, M_mlp, M_head, grads=grads, stats=stats, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / steps
    loss = float(stats[2])
    del grads, ws
    return ms_step, loss


def intermediate_bytes(S, I, V, M_mlp, M_head):
    nm = math.ceil(S / min(S, M_mlp))
    nh = math.ceil(S / min(S, M_head))
    return max(nm * I * (3 * 2 + 4), nh * V * 2 + nh * math.ceil(V / 256) * 8)


def sweep_m():
    dev = torch.device("cuda")
    H, I, V, S = 4096, 11008, 32000, 16384
    X, L, W = make(S, H, I, V, dev)
    for M in (1, 2, 4, 8):
        torch.cuda.reset_peak_memory_stats()
        ms_step, loss = timed_steps(X, L, W, M, M)
        peak = torch.cuda.max_memory_allocated()
        print(json.dumps({"config": "3 (Llama2-7B widths H=4096 I=11008 V=32000, S=16384)", "M": M,
                          "ms_per_step": ms_step, "tokens_per_s": S / ms_step * 1e3,
                          "executed_tflops": S * flops_per_token(H, I, V) / ms_step / 1e9,
                          "peak_intermediate_gb": intermediate_bytes(S, I, V, M, M) / 1e9,
                          "workspace_gb": ms.block_workspace_bytes(S, H, I, V, M, M, ms.Context.get(0)) / 1e9,
                          "device_peak_allocated_gb": peak / 1e9, "loss": loss}), flush=True)


def sweep_m2():
    """Config 2 (the bench workload) across M: the throughput cost of smaller chunks."""
    dev = torch.device("cuda")
    H, I, V, S = 4096, 14336, 128256, 8192
    X, L, W = make(S, H, I, V, dev)
    for M in (1, 2, 4, 8, 16):
        torch.cuda.reset_peak_memory_stats()
        ms_step, loss = timed_steps(X, L, W, M, M)
        print(json.dumps({"config": "2 (Llama3-8B widths, S=8192)", "M": M, "ms_per_step": ms_step,
                          "tokens_per_s": S / ms_step * 1e3,
                          "executed_tflops": S * flops_per_token(H, I, V) / ms_step / 1e9,
                          "peak_intermediate_gb": intermediate_bytes(S, I, V, M, M) / 1e9,
                          "workspace_gb": ms.block_workspace_bytes(S, H, I, V, M, M, ms.Context.get(0)) / 1e9,
                          "device_peak_allocated_gb": torch.cuda.max_memory_allocated() / 1e9, "loss": loss}),
              flush=True)


def sweep_pairs():
    """Config 2 widths, S=8192, independent (M_mlp, M_head) -- the paper's
    chosen setting is M=4 for the MLP and M=16 for the LM-Head;
    with nested plans block_step runs the chunk-wise schedule for all of them."""
    dev = torch.device("cuda")
    H, I, V, S = 4096, 14336, 128256, 8192
    X, L, W = make(S, H, I, V, dev)
    from paper_2407_15892_b200 import estimator

    for mm, mh in ((1, 1), (4, 4), (4, 16), (8, 8), (8, 16), (2, 16), (16, 16)):
        torch.cuda.reset_peak_memory_stats()
        ms_step, loss = timed_steps(X, L, W, mm, mh)
        print(json.dumps({"config": "2 (Llama3-8B widths, S=8192)", "M_mlp": mm, "M_head": mh,
                          "ms_per_step": ms_step, "tokens_per_s": S / ms_step * 1e3,
                          "executed_tflops": S * flops_per_token(H, I, V) / ms_step / 1e9,
                          "tracked_peak_intermediate_gb": estimator.predict_block_peak(S, H, I, V, mm, mh)["inter."] / 1e9,
                          "workspace_gb": ms.block_workspace_bytes(S, H, I, V, mm, mh, ms.Context.get(0)) / 1e9,
                          "device_peak_allocated_gb": torch.cuda.max_memory_allocated() / 1e9, "loss": loss}),
              flush=True)


def seq_sweep():
    """Config-2 widths across sequence lengths at fixed chunk lengths (n = 1024
    and 4096 tokens): throughput and workspace versus S."""
    dev = torch.device("cuda")
    H, I, V = 4096, 14336, 128256
    for S in (8192, 16384, 32768, 65536, 131072):
        X, L, W = make(S, H, I, V, dev)
        for n in (1024, 4096):
            M = S // n
            ms_step, loss = timed_steps(X, L, W, M, M, steps=2, warmup=1)
            print(json.dumps({"config": "Llama3-8B widths, sequence sweep", "S": S, "chunk": n, "M": M,
                              "ms_per_step": ms_step, "tokens_per_s": S / ms_step * 1e3,
                              "workspace_gb": ms.block_workspace_bytes(S, H, I, V, M, M, ms.Context.get(0)) / 1e9,
                              "loss": loss}), flush=True)
        del X, L, W
        torch.cuda.empty_cache()


def long_context():
    dev = torch.device("cuda")
    H, I, V, S, M = 4096, 14336, 128256, 65536, 16
    X, L, W = make(S, H, I, V, dev)
    torch.cuda.reset_peak_memory_stats()
    ms_step, loss = timed_steps(X, L, W, M, M, steps=2, warmup=1)
    print(json.dumps({"config": "4 (Llama3-8B widths, S=65536, M=16)", "ms_per_step": ms_step,
                      "tokens_per_s": S / ms_step * 1e3, "executed_tflops": S * flops_per_token(H, I, V) / ms_step / 1e9,
                      "peak_intermediate_gb": intermediate_bytes(S, I, V, M, M) / 1e9,
                      "peak_intermediate_gb_at_M1": intermediate_bytes(S, I, V, 1, 1) / 1e9,
                      "device_peak_allocated_gb": torch.cuda.max_memory_allocated() / 1e9, "loss": loss}),
          flush=True)


def max_seq(chunk=8192):
    """Largest S (multiple of 1024) whose block step fits the device, at a
    fixed chunk length (M = S / chunk): bisection with real dry-run steps."""
    dev = torch.device("cuda")
    H, I, V = 4096, 14336, 128256
    free, total = torch.cuda.mem_get_info()

    def fits(S):
        M = max(1, S // chunk)
        try:
            torch.cuda.empty_cache()
            X, L, W = make(S, H, I, V, dev)
            ms_step, loss = timed_steps(X, L, W, M, M, steps=1, warmup=0)
            peak = torch.cuda.max_memory_allocated()
            del X, L, W
            return True, ms_step, peak, loss
        except (torch.OutOfMemoryError, ms.Error) as e:  # pragma: no cover
            return False, str(e)[:80], 0, None

    lo, hi = 65536, 16 * 1024 * 1024
    best = None
    t0 = time.time()
    while hi - lo > 65536 and time.time() - t0 < 900:
        mid = (lo + hi) // 2 // 65536 * 65536
        torch.cuda.reset_peak_memory_stats()
        ok, a, peak, loss = fits(mid)
        print(json.dumps({"probe_S": mid, "fits": ok, "ms": a if ok else None, "peak_gb": peak / 1e9}), flush=True)
        if ok:
            lo, best = mid, (mid, a, peak, loss)
        else:
            hi = mid
    S, ms_step, peak, loss = best
    print(json.dumps({"config": "4 (Llama3-8B widths) max sequence length, chunk 8192 tokens",
                      "max_seq_len": S, "device_total_gb": total / 1e9, "device_peak_allocated_gb": peak / 1e9,
                      "ms_per_step": ms_step, "tokens_per_s": S / ms_step * 1e3, "loss": loss}), flush=True)


if __name__ == "__main__":
    {"sweep-m": sweep_m, "sweep-m2": sweep_m2, "sweep-pairs": sweep_pairs, "seq": seq_sweep, "max-seq": max_seq,
     "long": long_context}[sys.argv[1]]()
