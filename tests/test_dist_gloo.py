"""Sequence-parallel host logic (paper_2407_15892_b200/parallel.py) on CPU
with the gloo backend, world size 2 and 4 (acceptance 10).

The collectives, sharding and global token-weighted scaling are the product
code; the per-rank compute is the f64 oracle (`OracleOps`, test-only), so the
P>1 result can be compared with the single-process oracle: loss and
gradients within 1e-10."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, H, I, V, M_MLP, M_HEAD = 48, 8, 16, 24, 3, 4


class OracleOps:
    """CPU stand-in for GpuOps with the same interface (tests only)."""

    def __init__(self, orc):
        self.orc = orc

    def mlp_forward(self, X, w, M):
        O = self.orc.miniseq_mlp_forward(X.numpy(), *[t.numpy() for t in w], M)
        return torch.from_numpy(O), (X, M)

    def lmhead_forward(self, O, L, Wout, M):
        loss, lse, cs, cv = self.orc.miniseq_lmhead_forward(O.numpy(), L.numpy(), Wout.numpy(), M)
        stats = torch.tensor([cs.sum(), cv.sum(), loss, 0.0, *cs, *cv], dtype=torch.float64)
        return stats, (O, L, M, float(cv.sum()))

    def lmhead_backward(self, saved, Wout, gstats, dW_out):
        O, L, M, n_local = saved
        # token-weighted with the GLOBAL count: scale = 1 / n_global
        gl = n_local / float(gstats[1])
        dX, dW = self.orc.miniseq_lmhead_backward(O.numpy(), L.numpy(), Wout.numpy(), M, 0, gl)
        dW_out.copy_(torch.from_numpy(dW))
        return torch.from_numpy(dX)

    def count_valid(self, L, V):
        return torch.tensor([float(((L >= 0) & (L < V)).sum())], dtype=torch.float64)

    def lmhead_fused(self, O, L, Wout, M, global_valid, dW_out):
        stats, saved = self.lmhead_forward(O, L, Wout, M)
        dO = self.lmhead_backward(saved, Wout, torch.stack([stats[0], global_valid[0]]), dW_out)
        return stats, dO

    def mlp_backward(self, dO, saved, w, grads):
        X, M = saved
        dX, dWg, dWu, dWd = self.orc.miniseq_mlp_backward(dO.numpy(), X.numpy(), *[t.numpy() for t in w], M)
        for g, v in zip(grads, (dWg, dWu, dWd)):
            g.copy_(torch.from_numpy(v))
        return torch.from_numpy(dX)

    def block_step(self, X, L, w, Wout, M_mlp, M_head, grads, global_valid, grad_slab, slabs=1):
        """Stand-in for GpuOps.block_step (mst_block_step_sp): same order of the
        gradient-slab reports (dW_out's row slabs after the head, then dW_down
        whole and the dW_gate / dW_up slabs), slabs of ceil(rows / slabs)."""
        O, ms = self.mlp_forward(X, w, M_mlp)
        stats, dO = self.lmhead_fused(O, L, Wout, M_head, global_valid, grads[3])
        H = X.shape[1]
        per = -(-H // slabs)
        for r0 in range(0, H, per):
            grad_slab(3, r0, min(H, r0 + per))
        dX = self.mlp_backward(dO, ms, w, grads[:3])
        grad_slab(2, 0, grads[2].shape[0])
        for r0 in range(0, H, per):
            grad_slab(0, r0, min(H, r0 + per))
            grad_slab(1, r0, min(H, r0 + per))
        return stats, dX


def _inputs(orc):
    c = orc.make_inputs(31, N, H, I, V, p_ignore=0.15, w_std=0.3)
    c["L"][:5] = -100  # make rank shards hold different valid counts
    return c


def _worker(rank, world, port, ret, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2407_15892_b200.parallel import shard_rows, sp_block_step, sp_block_step_fused

        c = _inputs(orc)
        s, e = shard_rows(N, world, rank)
        f = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
        X, L = f(c["X"][s:e]), torch.from_numpy(c["L"][s:e].copy())
        w = (f(c["Wg"]), f(c["Wu"]), f(c["Wd"]))
        grads = tuple(torch.zeros_like(t) for t in (*w, f(c["Wout"])))
        if mode == "block":  # the bench's fast path: whole fused block + hook-driven gradient all-reduces
            r = sp_block_step_fused(OracleOps(orc), X, L, w, f(c["Wout"]), M_MLP, M_HEAD, grads, slabs=3)
        else:
            r = sp_block_step(OracleOps(orc), X, L, w, f(c["Wout"]), M_MLP, M_HEAD, grads, fused=mode == "fused")
        ref = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], M_MLP, M_HEAD, round_bf16=False)
        errs = dict(loss=abs(float(r.loss) - ref["loss"]),
                    dX=float(np.abs(r.dX.numpy() - ref["dX"][s:e]).max()),
                    dWg=float(np.abs(r.dW_gate.numpy() - ref["dWg"]).max()),
                    dWu=float(np.abs(r.dW_up.numpy() - ref["dWu"]).max()),
                    dWd=float(np.abs(r.dW_down.numpy() - ref["dWd"]).max()),
                    dWout=float(np.abs(r.dW_out.numpy() - ref["dWout"]).max()))
        ret[rank] = errs
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,mode", [(1, "fused"), (2, "fused"), (4, "fused"), (2, "separate"), (1, "block"),
                                        (2, "block"), (4, "block")])
def test_sequence_parallel_matches_single_process(world, mode, orc):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ret, mode), nprocs=world, join=True)
    assert len(ret) == world
    for rank, errs in ret.items():
        assert errs["loss"] <= 1e-12, (rank, errs)
        for k, v in errs.items():
            assert v <= 1e-10, (rank, k, v)  # SPEC.md:633 / acceptance 10


def test_shard_rows_partition():
    from paper_2407_15892_b200.parallel import shard_rows

    for total in (8, 9, 1000, 8192):
        for world in (1, 2, 3, 8):
            parts = [shard_rows(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(3, 4, 0)
