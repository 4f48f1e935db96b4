"""Estimator formulas (paper_2407_15892_b200/estimator.py) against the
SPEC's estimator examples and the oracle's counters."""
from fractions import Fraction

import numpy as np

from paper_2407_15892_b200 import estimator as E


def test_intermediate_ratios_kats():
    r = E.intermediate_ratios(4096, 14336, 128256, 4)
    assert float(r["head"]) == 128256 / 4096 and round(float(r["head"]), 2) == 31.31
    assert r["mlp"] == 7  # SPEC.md:556 (paper prints 16: logged discrepancy)
    assert E.intermediate_ratios(64, 224, 2048, 4)["attn"] == 1 + Fraction(2, 4)


def test_predict_flops_kats_and_m_invariance():
    assert E.predict_flops(4, 16, 32, 8)["mlp"] == 3072
    assert E.predict_flops(64, 224, 2048, 512, 1) == E.predict_flops(64, 224, 2048, 512, 8)
    h = [E.predict_flops(64, 224, 2048, s)["head"] for s in (128, 256, 512)]
    assert h[1] - h[0] == (h[2] - h[1]) / 2  # linear in S


def test_predict_hbm_kats():
    d, I, V, S = 64, 224, 2048, 1024
    std = E.predict_hbm(d, I, V, S, 1)
    assert std == {"mlp": S * d + S * I + 3 * d * I, "head": S * d + S * V + d * V}
    for M in (2, 4, 8):
        p = E.predict_hbm(d, I, V, S, M)
        assert p["mlp"] - E.predict_hbm(d, I, V, S, M - 1)["mlp"] == 3 * d * I
        assert p["head"] - E.predict_hbm(d, I, V, S, M - 1)["head"] == d * V


def test_predict_flops_matches_oracle_counters(orc):
    """Counter agreement: the matmul part of predict_flops equals
    the oracle's memtrack counters of a forward at desk scale."""
    N, H, I, V, M = 32, 8, 16, 24, 4
    c = orc.make_inputs(1, N, H, I, V)
    orc.counters_reset()
    orc.miniseq_mlp_forward(c["X"], c["Wg"], c["Wu"], c["Wd"], M)
    assert orc.counters()["matmul_flops"] == E.predict_flops(H, I, V, N, M)["mlp"]
    orc.counters_reset()
    orc.miniseq_lmhead_forward(c["X"], c["L"], c["Wout"], M)
    ctr = orc.counters()
    assert ctr["flops"] == E.predict_flops(H, I, V, N, M)["head"]
    w = ctr["weight_read_elements"]
    assert w == M * H * V  # per-chunk W_out re-read (Theorem 3.2)


def test_block_peak_scales_as_one_over_m():
    p1, p8 = E.predict_block_peak(8192, 4096, 14336, 128256, 1), E.predict_block_peak(8192, 4096, 14336, 128256, 8)
    assert p1["inter.head."] == 8 * p8["inter.head."] and p1["inter."] == 8 * p8["inter."]
    assert np.isclose(p8["inter.head."] / 1e6, 266.8, atol=0.1)  # dlogits [S/M, V] bf16 + CE partials at config 2
