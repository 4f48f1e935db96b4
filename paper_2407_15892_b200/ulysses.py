"""Ulysses sequence parallelism around attention (the
reference's distributed MsT, SPEC.md:606-657, PAPER.md:221-225 and Table 8).

Every rank holds a contiguous shard of S/P tokens.  MLP, LM-Head, norms and
embedding are token-local (the MsT blocks run unchanged on the shard); only
attention needs the whole sequence, so around it the activations are
re-sharded by an all-to-all from "sequence shard, all heads" to "whole
sequence, heads / P" and back (DeepSpeed-Ulysses).  Collectives go through
torch.distributed's autograd-aware all_to_all_single (NCCL over NVLink on
B200 boxes; gloo in the CPU tests), so the attention backward re-shards the
gradients with the transposed all-to-alls automatically.

Requirements: heads % P == 0 and kv_heads % P == 0 (each rank owns whole
query groups), equal shard lengths.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist
from torch.distributed.nn.functional import all_to_all_single as _a2a


def _world(group) -> int:
    return dist.get_world_size(group) if dist.is_initialized() else 1


def _a2a_any(x: torch.Tensor, group) -> torch.Tensor:
    """Autograd-aware all-to-all along dim 0 (equal splits).  gloo has no CUDA
    all-to-all: stage through host memory there (tests only)."""
    if dist.get_backend(group) == "gloo" and x.is_cuda:
        return _a2a(torch.empty_like(x.cpu()), x.cpu(), group=group).to(x.device)
    return _a2a(torch.empty_like(x), x, group=group)


def seq_to_head(x: torch.Tensor, heads: int, group=None) -> torch.Tensor:
    """[S/P, heads, hd] (sequence shard, all heads) -> [S, heads/P, hd] (all
    tokens in rank order, this rank's head slice)."""
    P = _world(group)
    if P == 1:
        return x
    s, h, hd = x.shape
    if h % P:
        raise ValueError(f"{h} heads not divisible by {P} ranks")
    # chunk p of the send buffer = my tokens for rank p's heads
    send = x.reshape(s, P, h // P, hd).permute(1, 0, 2, 3).contiguous()      # [P, s, h/P, hd]
    recv = _a2a_any(send.reshape(P * s, h // P, hd), group)                  # [P*s, h/P, hd]: rank-ordered tokens
    return recv


def head_to_seq(y: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse of seq_to_head: [S, heads/P, hd] -> [S/P, heads, hd]."""
    P = _world(group)
    if P == 1:
        return y
    S, hp, hd = y.shape
    s = S // P
    recv = _a2a_any(y.contiguous(), group).reshape(P, s, hp, hd)            # [P (head block), s, h/P, hd]
    return recv.permute(1, 0, 2, 3).reshape(s, P * hp, hd)


def _mst_attention(qh: torch.Tensor, kh: torch.Tensor, vh: torch.Tensor, heads: int, kv_heads: int) -> torch.Tensor:
    """libmst's tcgen05 causal GQA attention (attention.CausalAttention) on the
    head-sharded layout: q [S, h, hd], k / v [S, kvh, hd] -> [S, h, hd]."""
    from .attention import CausalAttention

    S, _, hd = qh.shape
    o = CausalAttention.apply(qh.reshape(S, heads * hd), kh.reshape(S, kv_heads * hd), vh.reshape(S, kv_heads * hd),
                              1, S, heads, kv_heads)
    return o.reshape(S, heads, hd)


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int, kv_heads: int,
              group=None, attn_fn=None) -> torch.Tensor:
    """Causal grouped-query attention of one sequence sharded over `group`.
    q [S/P, heads*hd], k, v [S/P, kv_heads*hd] (this rank's tokens) ->
    [S/P, heads*hd].  Differentiable (autograd through the all-to-alls and
    libmst's attention kernels, whose backward does not re-run the forward).
    attn_fn(qh, kh, vh, heads_local, kv_heads_local) on [S, h, hd] views
    replaces the kernel -- for host-tensor tests of the re-sharding only; CUDA
    tensors always go through libmst."""
    P = _world(group)
    s = q.shape[0]
    hd = q.shape[1] // heads
    if heads % P or kv_heads % P:
        raise ValueError(f"Ulysses needs heads ({heads}) and kv heads ({kv_heads}) divisible by {P}")
    if attn_fn is None or q.is_cuda:
        if not q.is_cuda:
            raise ValueError("ulysses.attention runs libmst's CUDA kernels: pass CUDA tensors")
        attn_fn = _mst_attention
    qh = seq_to_head(q.reshape(s, heads, hd), heads, group)        # [S, h/P, hd]
    kh = seq_to_head(k.reshape(s, kv_heads, hd), kv_heads, group)  # [S, kvh/P, hd]
    vh = seq_to_head(v.reshape(s, kv_heads, hd), kv_heads, group)
    o = attn_fn(qh, kh, vh, heads // P, kv_heads // P)             # [S, h/P, hd]
    return head_to_seq(o, group).reshape(s, heads * hd)


def all_reduce_grads(grads: dict, group=None) -> None:
    """SUM all-reduce of replicated-weight gradients across the sequence shards."""
    if _world(group) == 1:
        return
    for g in grads.values():
        if dist.get_backend(group) == "gloo" and g.is_cuda:
            c = g.cpu()
            dist.all_reduce(c, group=group)
            g.copy_(c)
        else:
            dist.all_reduce(g, group=group)
