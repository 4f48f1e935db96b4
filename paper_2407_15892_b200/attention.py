"""Causal grouped-query attention on libmst's tcgen05 kernels
(csrc/attention.cu; attn_forward / attn_backward of SPEC.md:233-241).

Tensors are token-major 2-D views: q [B*S, heads*hd], k / v [B*S, kv_heads*hd]
with unit stride along the features and any row stride (so column slices of
the decoder's fused qkv buffer are read in place); o, dq, dk, dv likewise.
The forward returns o and the fp32 log-sum-exp [B, heads, S] that the
backward needs; nothing of size S x S is ever stored.  No fallback: the
library must be built (miniseq.load_library raises otherwise).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import torch

from . import miniseq as ms


def _rows(t: torch.Tensor, name: str, width: int, n: int) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.bfloat16:
        raise ms.DtypeError(f"{name} must be a bf16 CUDA tensor")
    if t.dim() != 2 or t.shape[0] != n or t.shape[1] != width:
        raise ms.ShapeError(f"{name} must be [{n}, {width}], got {tuple(t.shape)}")
    if t.stride(1) != 1:
        raise ms.ConfigError(f"{name} needs unit stride along the features")
    return t.stride(0)


def attention_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, B: int, S: int, heads: int, kv_heads: int,
                      out: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """o = softmax(q k^T / sqrt(hd) + causal mask) v per head; returns (o, lse)."""
    hd = q.shape[1] // heads
    N = B * S
    ldq, ldk, ldv = _rows(q, "q", heads * hd, N), _rows(k, "k", kv_heads * hd, N), _rows(v, "v", kv_heads * hd, N)
    if out is None:
        out = torch.empty(N, heads * hd, device=q.device, dtype=torch.bfloat16)
    ldo = _rows(out, "o", heads * hd, N)
    lse = torch.empty(B, heads, S, device=q.device, dtype=torch.float32)
    ctx = ms.Context.get(q.device.index)
    ms._check(ctx.lib.mst_attention_forward(ctx.handle, ms._stream(q), q.data_ptr(), ldq, k.data_ptr(), ldk,
                                            v.data_ptr(), ldv, out.data_ptr(), ldo, lse.data_ptr(), B, S, heads,
                                            kv_heads, hd, 1))
    return out, lse


def attention_backward(q, k, v, o, do, lse, B: int, S: int, heads: int, kv_heads: int,
                       dq: Optional[torch.Tensor] = None, dk: Optional[torch.Tensor] = None,
                       dv: Optional[torch.Tensor] = None):
    """(dq, dk, dv) of the causal attention; dq / dk / dv may be column slices
    of one buffer (the decoder's d qkv)."""
    hd = q.shape[1] // heads
    N = B * S
    lds = [_rows(q, "q", heads * hd, N), _rows(k, "k", kv_heads * hd, N), _rows(v, "v", kv_heads * hd, N),
           _rows(o, "o", heads * hd, N), _rows(do, "dO", heads * hd, N)]
    dev = q.device
    dq = torch.empty(N, heads * hd, device=dev, dtype=torch.bfloat16) if dq is None else dq
    dk = torch.empty(N, kv_heads * hd, device=dev, dtype=torch.bfloat16) if dk is None else dk
    dv = torch.empty(N, kv_heads * hd, device=dev, dtype=torch.bfloat16) if dv is None else dv
    lds += [_rows(dq, "dq", heads * hd, N), _rows(dk, "dk", kv_heads * hd, N), _rows(dv, "dv", kv_heads * hd, N)]
    if lse.dtype != torch.float32 or lse.numel() != B * heads * S or not lse.is_contiguous():
        raise ms.ShapeError("lse must be a contiguous fp32 [B, heads, S] tensor")
    ctx = ms.Context.get(dev.index)
    nb = ctypes.c_size_t()
    ms._check(ctx.lib.mst_attention_workspace(B, S, heads, ctypes.byref(nb)))
    ws = torch.empty(nb.value, device=dev, dtype=torch.uint8)
    ms._check(ctx.lib.mst_attention_backward(ctx.handle, ms._stream(q), q.data_ptr(), lds[0], k.data_ptr(), lds[1],
                                             v.data_ptr(), lds[2], o.data_ptr(), lds[3], do.data_ptr(), lds[4],
                                             lse.data_ptr(), dq.data_ptr(), lds[5], dk.data_ptr(), lds[6],
                                             dv.data_ptr(), lds[7], B, S, heads, kv_heads, hd, 1, ws.data_ptr(),
                                             ws.numel()))
    return dq, dk, dv


class CausalAttention(torch.autograd.Function):
    """Autograd wrapper (used where the surrounding ops are autograd-tracked:
    the Ulysses all-to-alls in ulysses.py).  Saves q, k, v, o and lse; the
    backward never re-runs the forward."""

    @staticmethod
    def forward(ctx, q, k, v, B: int, S: int, heads: int, kv_heads: int):
        q, k, v = (t if t.stride(1) == 1 else t.contiguous() for t in (q, k, v))
        o, lse = attention_forward(q, k, v, B, S, heads, kv_heads)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.dims = (B, S, heads, kv_heads)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attention_backward(q, k, v, o, do.contiguous(), lse, *ctx.dims)
        return dq, dk, dv, None, None, None, None
