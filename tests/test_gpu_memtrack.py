"""memtrack on the GPU path: libmst's op counters and
memory events (include/mst/mst.h "memtrack") checked against the f64
oracle's counters (memtrack.hpp:19-35 conventions) and the paper's theorems
on the device implementation:
  * Thm 3.1: FLOPs are independent of M;
  * Thm 3.2: weight reads grow by exactly the per-chunk
    weight traffic per extra mini-sequence;
  * the tracked peak of the [S/M, V] / [S/M, I] intermediates falls as 1/M
    (the memory claim), every chunk buffer is freed, and the
    timeline exports in the reference's CSV format (memtrack.hpp:277-284).
"""
import io

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2407_15892_b200 import memtrack as mt
from paper_2407_15892_b200 import miniseq as ms

pytestmark = pytest.mark.gpu

N, H, I, V = 512, 128, 256, 1024


def _inputs(seed=5):
    c = oracle.make_inputs(seed, N, H, I, V)
    g = {k: torch.from_numpy(c[k]).cuda().bfloat16() for k in ("X", "Wg", "Wu", "Wd", "Wout")}
    return c, g, torch.from_numpy(c["L"]).cuda()


def _ctx():
    ctx = ms.Context.get(0)
    ctx.reset_counters()
    return ctx


@pytest.mark.parametrize("M", [1, 4])
def test_mlp_counters_match_oracle(M):
    c, g, _ = _inputs()
    w = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"])
    plan = ms.make_chunk_plan(N, M)
    ctx = _ctx()
    O, saved = ms.miniseq_mlp_forward(g["X"], w, plan)
    fwd = ctx.counters()
    oracle.counters_reset()
    oracle.miniseq_mlp_forward(c["X"], c["Wg"], c["Wu"], c["Wd"], M)
    ref = oracle.counters()
    assert (fwd.flops, fwd.matmul_flops, fwd.weight_read_elements) == \
        (ref["flops"], ref["matmul_flops"], ref["weight_read_elements"])
    # the oracle's slice_rows / concat_rows copy 2*n*H elements each per chunk;
    # libmst's chunk slices are zero-copy tensor-map offsets
    assert fwd.hbm_elements == ref["hbm_elements"] - 4 * N * H
    ctx.reset_counters()
    dO = torch.randn(N, H, device="cuda").bfloat16()
    ms.miniseq_mlp_backward(dO, saved, w, plan)
    bwd = ctx.counters()
    oracle.counters_reset()
    oracle.miniseq_mlp_backward(dO.double().cpu().numpy(), c["X"], c["Wg"], c["Wu"], c["Wd"], M)
    ref = oracle.counters()
    assert bwd.as_tuple() == (ref["flops"], ref["matmul_flops"], ref["hbm_elements"], ref["weight_read_elements"])


def _block_counts(M, tracker=None, pair_dw=1):
    _, g, L = _inputs()
    ctx = _ctx()
    ctx.attach_tracker(tracker)
    ctx.set_tuning("pair_dw", pair_dw)
    try:
        if tracker is not None:
            tracker.region_begin("block")
        _, gr = ms.block_step(g["X"], L, ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"]), M, M)
        torch.cuda.synchronize()
        if tracker is not None:  # deferred optimizer: the caller releases the gradients
            for k, t in (("W_gate", gr.W_gate), ("W_up", gr.W_up), ("W_down", gr.W_down), ("W_out", gr.W_out)):
                tracker.on_free(t.numel() * 4, f"grad.{k}")
        region = tracker.region_end("block") if tracker is not None else None
    finally:
        ctx.attach_tracker(None)
        ctx.set_tuning("pair_dw", 1)
    return ctx.counters(), region


def test_block_flops_independent_of_M_thm31():
    base = _block_counts(1)[0]
    for M in (2, 4, 8):
        c = _block_counts(M)[0]
        assert c.flops == base.flops and c.matmul_flops == base.matmul_flops
    # executed matmul FLOPs of the chunk-wise block: 18HI + 6HV per token
    assert base.matmul_flops == N * (18 * H * I + 6 * H * V)


def test_block_weight_reads_linear_in_M_thm32():
    reads = {M: _block_counts(M)[0].weight_read_elements for M in (1, 2, 4, 8)}
    per_chunk = 6 * H * I + 2 * H * V  # K1 + K2 + K7a + K9 (MLP), K3' + K5 (head)
    for M, r in reads.items():
        assert r == M * per_chunk


def test_tracked_peak_intermediate_scales_as_one_over_M():
    """With per-chunk dW accumulation (pair_dw off) every chunk buffer is 1/M
    of its M=1 size; the default pairs the dW GEMMs of two chunks and keeps
    one extra dG / dU / h^T set (checked exactly against the estimator in
    test_estimator_block_peak_matches_tracked_device_allocations)."""
    peaks = {}
    for M in (1, 8):
        t = mt.MemTracker()
        _, reg = _block_counts(M, t, pair_dw=0)
        assert t.live_bytes() == 0 and reg.report.final_live() == 0  # every chunk buffer freed
        n = N // M
        head = reg.report.peak_for_prefix("inter.head.")
        assert head == n * V * 2 + n * ((V + 255) // 256) * 8 + n * 8  # dlogits (bf16) + CE partials
        peaks[M] = (head, reg.report.peak_for_prefix("inter.mlp."), reg.report.peak_for_prefix("inter."))
        # the chunk-wise schedule keeps one O chunk and two dO chunks (dO_j feeds chunk j+1's dW_down GEMM)
        assert reg.report.peak_for_prefix("act.O") == n * H * 2
        assert reg.report.peak_for_prefix("act.dO") == 2 * n * H * 2
    assert peaks[1][0] == 8 * peaks[8][0]
    assert peaks[1][1] == 8 * peaks[8][1]
    assert peaks[1][2] == 8 * peaks[8][2]


def test_separate_ops_events_balanced_and_timeline():
    c, g, L = _inputs()
    plan = ms.make_chunk_plan(N, 4)
    t = mt.MemTracker()
    ctx = _ctx()
    ctx.attach_tracker(t)
    try:
        t.region_begin("ops")
        O, sv = ms.miniseq_mlp_forward(g["X"], ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), plan)
        loss, hs = ms.miniseq_lmhead_forward(O, L, ms.LmHeadWeights(g["Wout"]), plan)
        dO, _ = ms.miniseq_lmhead_backward(hs, ms.LmHeadWeights(g["Wout"]), plan)
        ms.miniseq_mlp_backward(dO, sv, ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), plan)
        torch.cuda.synchronize()
        reg = t.region_end("ops")
    finally:
        ctx.attach_tracker(None)
    assert reg.report.final_live() == 0
    # the tracker's own counters equal the context's (same stream of counts)
    assert reg.counters.as_tuple() == ctx.counters().as_tuple()
    lines = mt.export_timeline(reg.report, io.StringIO()).splitlines()
    assert lines[0] == "seq_no,kind,bytes,label,live_after"
    labels = {ln.split(",")[3] for ln in lines[1:]}
    assert {"inter.mlp.h", "inter.mlp.dh", "inter.mlp.dG", "inter.head.dlogits", "inter.head.partials"} <= labels
    # the one live [S/M, V] buffer: dlogits of one 128-row chunk
    assert reg.report.peak_for_prefix("inter.head.dlogits") == (N // 4) * V * 2


@pytest.mark.parametrize("M", [1, 2, 8])
def test_estimator_block_peak_matches_tracked_device_allocations(M):
    """estimator.predict_block_peak == the tracked peaks of a real block step
    on the device, per label class (SPEC.md:579 'tracker agreement', exact
    here rather than within 10%)."""
    from paper_2407_15892_b200 import estimator

    for pair in (1, 0):
        t = mt.MemTracker()
        _, reg = _block_counts(M, t, pair_dw=pair)
        pred = estimator.predict_block_peak(N, H, I, V, M, pair_dw=bool(pair))
        for prefix, b in pred.items():
            assert reg.report.peak_for_prefix(prefix) == b, (pair, prefix, reg.report.peak_for_prefix(prefix), b)
