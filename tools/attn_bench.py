"""Throughput of libmst's tcgen05 causal GQA attention (csrc/attention.cu)
next to flash_attn / torch SDPA (library kernels, for scale only).

  python tools/attn_bench.py [S] [heads] [kv_heads] [hd] [B]

Algorithmic FLOPs per (batch, head): forward 2 * S^2 * hd (causal half of
QK^T and PV), backward 5 * S^2 * hd (S, dP, dV, dK, dQ; libmst's
deterministic split recomputes S and dP in its dQ kernel, 7 GEMMs executed).
CUDA events on the launching stream, warm-up first, median of reps.
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_15892_b200 import attention as A  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    KV = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    hd = int(sys.argv[4]) if len(sys.argv) > 4 else 128
    B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    N = B * S
    torch.manual_seed(0)
    q = torch.randn(N, H * hd, device="cuda").bfloat16()
    k = torch.randn(N, KV * hd, device="cuda").bfloat16()
    v = torch.randn(N, KV * hd, device="cuda").bfloat16()
    do = torch.randn(N, H * hd, device="cuda").bfloat16()
    fwd_fl = 2.0 * S * S * hd * H * B
    bwd_fl = 5.0 * S * S * hd * H * B
    o, lse = A.attention_forward(q, k, v, B, S, H, KV)
    t_f = timeit(lambda: A.attention_forward(q, k, v, B, S, H, KV, out=o))
    t_b = timeit(lambda: A.attention_backward(q, k, v, o, do, lse, B, S, H, KV))
    out = {"shape": dict(B=B, S=S, heads=H, kv_heads=KV, hd=hd),
           "mst_fwd_ms": t_f, "mst_fwd_tflops": fwd_fl / t_f / 1e9,
           "mst_bwd_ms": t_b, "mst_bwd_tflops": bwd_fl / t_b / 1e9}
    try:
        from flash_attn import flash_attn_func

        q4 = q.reshape(B, S, H, hd)
        k4 = k.reshape(B, S, KV, hd)
        v4 = v.reshape(B, S, KV, hd)
        tf = timeit(lambda: flash_attn_func(q4, k4, v4, causal=True))
        q4r, k4r, v4r = (t.clone().requires_grad_(True) for t in (q4, k4, v4))
        o4 = flash_attn_func(q4r, k4r, v4r, causal=True)
        tb = timeit(lambda: torch.autograd.grad(o4, (q4r, k4r, v4r), do.reshape(B, S, H, hd), retain_graph=True))
        out.update(flash_attn_fwd_ms=tf, flash_attn_fwd_tflops=fwd_fl / tf / 1e9, flash_attn_bwd_ms=tb,
                   flash_attn_bwd_tflops=bwd_fl / tb / 1e9)
    except Exception as exc:  # pragma: no cover
        out["flash_attn"] = repr(exc)[:120]
    try:
        import torch.nn.functional as F

        qs = q.reshape(B, S, H, hd).transpose(1, 2)
        ks = k.reshape(B, S, KV, hd).transpose(1, 2)
        vs = v.reshape(B, S, KV, hd).transpose(1, 2)
        ts = timeit(lambda: F.scaled_dot_product_attention(qs, ks, vs, is_causal=True, enable_gqa=KV != H))
        out.update(sdpa_fwd_ms=ts, sdpa_fwd_tflops=fwd_fl / ts / 1e9)
    except Exception as exc:  # pragma: no cover
        out["sdpa"] = repr(exc)[:120]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
