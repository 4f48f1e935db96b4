"""Ulysses attention re-sharding (paper_2407_15892_b200/ulysses.py) on CPU
with the gloo backend, world size 2 and 4: the sequence-sharded attention
(all-to-all to head shards, causal GQA on the whole sequence, all-to-all
back) equals single-process attention, forward and backward."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _full(q, k, v, heads, kvh):
    S = q.shape[0]
    hd = q.shape[1] // heads
    o = torch.nn.functional.scaled_dot_product_attention(
        q.reshape(S, heads, hd).transpose(0, 1)[None], k.reshape(S, kvh, hd).transpose(0, 1)[None],
        v.reshape(S, kvh, hd).transpose(0, 1)[None], is_causal=True, enable_gqa=kvh != heads)
    return o[0].transpose(0, 1).reshape(S, heads * hd)


def _sdpa_heads(qh, kh, vh, h, kvh):
    """Host stand-in for libmst's kernel on the head-sharded [S, h, hd] views
    (this test checks the re-sharding collectives, not the kernel)."""
    o = torch.nn.functional.scaled_dot_product_attention(qh.transpose(0, 1)[None], kh.transpose(0, 1)[None],
                                                         vh.transpose(0, 1)[None], is_causal=True,
                                                         enable_gqa=kvh != h)
    return o[0].transpose(0, 1)


def _worker(rank, world, port, ret, S, heads, kvh, hd):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_15892_b200 import ulysses

        g = torch.Generator().manual_seed(0)
        q = torch.randn(S, heads * hd, generator=g, dtype=torch.float64)
        k = torch.randn(S, kvh * hd, generator=g, dtype=torch.float64)
        v = torch.randn(S, kvh * hd, generator=g, dtype=torch.float64)
        do = torch.randn(S, heads * hd, generator=g, dtype=torch.float64)
        s = S // world
        sl = slice(rank * s, (rank + 1) * s)
        ql, kl, vl = (t[sl].clone().requires_grad_(True) for t in (q, k, v))
        o = ulysses.attention(ql, kl, vl, heads, kvh, attn_fn=_sdpa_heads)
        o.backward(do[sl])
        qf, kf, vf = (t.clone().requires_grad_(True) for t in (q, k, v))
        of = _full(qf, kf, vf, heads, kvh)
        of.backward(do)
        # k/v gradients of this rank's tokens collect contributions from every
        # rank's queries: they come back through the transposed all-to-all
        ret[rank] = dict(o=float((o - of[sl]).abs().max()), dq=float((ql.grad - qf.grad[sl]).abs().max()),
                         dk=float((kl.grad - kf.grad[sl]).abs().max()), dv=float((vl.grad - vf.grad[sl]).abs().max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,heads,kvh", [(2, 4, 2), (2, 8, 8), (4, 8, 4)])
def test_ulysses_attention_matches_full_sequence(world, heads, kvh):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ret, 64, heads, kvh, 8), nprocs=world, join=True)
    assert len(ret) == world
    for r, e in ret.items():
        for k, v in e.items():
            assert v < 1e-12, (r, k, v)
