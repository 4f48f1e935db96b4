"""Sequence-parallel MsT step across ranks (SPEC.md:606-657 made real).

Tokens are independent through the MLP and LM-Head blocks, so each rank owns
a contiguous sequence shard (WorkerState) and runs the full
mini-sequence pipeline on it.  The only cross-rank traffic is:

  1. the valid-token count: all-reduce SUM of one float before the LM-Head,
     so every rank scales its dlogits by the GLOBAL count (token-weighted
     loss) — the per-rank gradients then already sum to the
     P=1 gradient; then the (loss sum, valid) pair for the reported loss;
  2. the weight gradients: all-reduce SUM.  On the fused chunk-wise block
     (sp_block_step_fused) each row slab is reduced asynchronously as soon
     as the library reports it final (mst_ctx_set_grad_slab_hook), so the
     reduction overlaps the last chunks' launches; sp_block_step (the SPEC
     op sequence) reduces dW_out while the MLP backward runs and
     dW_{gate,up,down} at the end.

The collective backend is whatever torch.distributed was initialised with:
NCCL over NVLink on B200 boxes, gloo in the CPU tests.  The compute is an
`ops` object; `GpuOps` (libmst, sm_100a) is the only product implementation.
"""
from __future__ import annotations

from dataclasses import dataclass
import torch
import torch.distributed as dist


def shard_rows(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced sequence shard of `rank` (first total % world ranks get one more row)."""
    if total < world:
        raise ValueError(f"cannot shard {total} rows over {world} ranks")
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


@dataclass
class StepResult:
    loss: torch.Tensor       # 0-d global loss (device of the ops)
    stats: torch.Tensor      # all-reduced stats (loss_sum, valid, ...)
    dX: torch.Tensor
    dW_gate: torch.Tensor
    dW_up: torch.Tensor
    dW_down: torch.Tensor
    dW_out: torch.Tensor


class GpuOps:
    """libmst-backed compute for one rank (CUDA tensors)."""

    def __init__(self):
        from . import miniseq as ms

        self.ms = ms

    def mlp_forward(self, X, w, M):
        return self.ms.miniseq_mlp_forward(X, self.ms.MlpWeights(*w), self.ms.make_chunk_plan(X.shape[0], M))

    def lmhead_forward(self, O, L, Wout, M):
        plan = self.ms.make_chunk_plan(O.shape[0], M)
        _, saved = self.ms.miniseq_lmhead_forward(O, L, self.ms.LmHeadWeights(Wout), plan)
        return saved.stats, saved

    def count_valid(self, L, V):
        return self.ms.count_valid(L, V)

    def lmhead_fused(self, O, L, Wout, M, global_valid, dW_out):
        plan = self.ms.make_chunk_plan(O.shape[0], M)
        _, stats, _, dO, _ = self.ms.miniseq_lmhead_fused(O, L, self.ms.LmHeadWeights(Wout), plan,
                                                          global_valid=global_valid, dW_out=dW_out)
        return stats, dO

    def lmhead_backward(self, saved, Wout, global_stats, dW_out):
        return self.ms.miniseq_lmhead_backward(saved, self.ms.LmHeadWeights(Wout), saved.plan,
                                               global_stats=global_stats, dW_out=dW_out)[0]

    def mlp_backward(self, dO, saved, w, grads):
        g = self.ms.MlpGrads(*grads)
        return self.ms.miniseq_mlp_backward(dO, saved, self.ms.MlpWeights(*w), saved.plan, grads=g)[0]

    def block_step(self, X, L, w, Wout, M_mlp, M_head, grads, global_valid, grad_slab, slabs=1, workspace=None,
                   stats=None):
        """The whole fused block (mst_block_step_sp, chunk-wise schedule) with the
        global valid count; grad_slab(which, r0, r1) fires as rows of each dW
        become final (`slabs` row slabs for dW_out / dW_gate / dW_up)."""
        ms = self.ms
        N, H = X.shape
        bg = ms.BlockGrads(dX=torch.empty(N, H, device=X.device, dtype=torch.bfloat16), W_gate=grads[0],
                           W_up=grads[1], W_down=grads[2], W_out=grads[3]) if not isinstance(grads, ms.BlockGrads) \
            else grads
        stats, bg = ms.block_step(X, L, ms.MlpWeights(*w), ms.LmHeadWeights(Wout), M_mlp, M_head, grads=bg,
                                  stats=stats, workspace=workspace, global_valid=global_valid, grad_slab=grad_slab,
                                  slabs=slabs)
        return stats, bg.dX


def sp_block_step_fused(ops, X: torch.Tensor, L: torch.Tensor, w: tuple, Wout: torch.Tensor, M_mlp: int,
                        M_head: int, grads: tuple, group=None, overlap: bool = True, slabs: int = 4,
                        **kw) -> StepResult:
    """Sequence-parallel step on the fused chunk-wise block (the fast path):
    one all-reduce of the valid count before the step, the block itself with
    the global count (mst_block_step_sp), then each weight gradient's SUM
    all-reduce issued per row slab from the library's gradient-slab hook the
    moment the slab is final: dW_out's slabs during the last head chunk's
    launches (overlapping them and the last chunk's MLP backward), dW_down
    and the dW_gate / dW_up slabs during the last MLP chunk's launches; only
    the last slab's reduction is exposed.  Then the loss pair.  Same results
    as sp_block_step (tests/test_dist_gloo.py)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    valid = ops.count_valid(L, Wout.shape[1])
    if world > 1:
        # fp64 integer counts: the SUM is exact up to 2^53 tokens
        dist.all_reduce(valid, op=dist.ReduceOp.SUM, group=group)
    works = []
    reported = {}
    gl = (grads.W_gate, grads.W_up, grads.W_down, grads.W_out) if hasattr(grads, "W_out") else tuple(grads)

    def slab(which: int, r0: int, r1: int) -> None:
        reported[which] = reported.get(which, 0) + (r1 - r0)
        if world > 1:
            works.append(dist.all_reduce(gl[which][r0:r1], op=dist.ReduceOp.SUM, group=group, async_op=overlap))

    stats, dX = ops.block_step(X, L, w, Wout, M_mlp, M_head, grads, valid, slab, slabs, **kw)
    for k, t in enumerate(gl):  # every gradient row reduced exactly once
        if reported.get(k) != t.shape[0]:
            raise RuntimeError(f"gradient {k}: {reported.get(k)} of {t.shape[0]} rows reported final")
    gstats = stats.clone()
    if world > 1:
        head = gstats[:2].contiguous()
        dist.all_reduce(head, op=dist.ReduceOp.SUM, group=group)
        gstats[:2] = head
    for wk in works:
        if wk is not None:
            wk.wait()
    loss = gstats[0] / gstats[1]
    return StepResult(loss=loss, stats=gstats, dX=dX, dW_gate=gl[0], dW_up=gl[1], dW_down=gl[2], dW_out=gl[3])


def sp_block_step(ops, X: torch.Tensor, L: torch.Tensor, w: tuple, Wout: torch.Tensor, M_mlp: int, M_head: int,
                  grads: tuple, group=None, overlap: bool = True, fused: bool = True) -> StepResult:
    """One sequence-parallel MLP -> LM-Head forward+backward on this rank's shard.

    w = (W_gate, W_up, W_down); grads = (dW_gate, dW_up, dW_down, dW_out) buffers
    (overwritten).  Returns global loss and SUM-reduced gradients."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dWg, dWu, dWd, dWo = grads
    O, msaved = ops.mlp_forward(X, w, M_mlp)
    if fused and hasattr(ops, "lmhead_fused"):
        # single-pass head: the global valid count must be known up front
        valid = ops.count_valid(L, Wout.shape[1])
        if world > 1:
            dist.all_reduce(valid, op=dist.ReduceOp.SUM, group=group)
        stats, dO = ops.lmhead_fused(O, L, Wout, M_head, valid, dWo)
        gstats = stats.clone()
        if world > 1:
            head = gstats[:2].contiguous()
            dist.all_reduce(head, op=dist.ReduceOp.SUM, group=group)
            gstats[:2] = head
    else:
        stats, hsaved = ops.lmhead_forward(O, L, Wout, M_head)
        gstats = stats.clone()
        if world > 1:
            head = gstats[:2].contiguous()
            dist.all_reduce(head, op=dist.ReduceOp.SUM, group=group)
            gstats[:2] = head
        dO = ops.lmhead_backward(hsaved, Wout, gstats, dWo)
    work = None
    if world > 1:
        # The process group runs the collective on its own stream, ordered
        # after the head backward; the MLP backward below overlaps it.
        work = dist.all_reduce(dWo, op=dist.ReduceOp.SUM, group=group, async_op=overlap)
    dX = ops.mlp_backward(dO, msaved, w, (dWg, dWu, dWd))
    if world > 1:
        for t in (dWg, dWu, dWd):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        if work is not None:
            work.wait()
    loss = gstats[0] / gstats[1]
    return StepResult(loss=loss, stats=gstats, dX=dX, dW_gate=dWg, dW_up=dWu, dW_down=dWd, dW_out=dWo)
