"""Randomised shapes through the C ABI against the f64 oracle (bf16-emulating
and exact checkers): extents multiples of 8 from
8 up to a few hundred (partial 256-row / 256-column tiles, K shorter than one
64-deep block, more chunks than rows), M_mlp and M_head drawn independently,
so both block schedules (chunk-wise when M_mlp == M_head, op-by-op
otherwise) and every grouped launch composition are exercised."""
import random

import numpy as np
import pytest
import torch

from paper_2407_15892_b200 import miniseq as ms
from test_gpu_parity import LOOSE, rel, to_gpu

pytestmark = pytest.mark.gpu

# block_step runs the single-pass LM-Head: its dlogits carry one extra bf16
# rounding (the stored softmax numerator); the bf16-emulating
# checker replays it (oracle.block(single_pass=True)), so the tight bounds of
# test_gpu_parity.py apply.
from test_gpu_parity import TIGHT_BF16 as FUSED_BF16, TIGHT_F32 as FUSED_F32  # noqa: E402


def _cases(n=48, seed=20261017):
    rnd = random.Random(seed)
    out = []
    for k in range(n):
        N = rnd.randint(1, 600)
        H = 8 * rnd.randint(1, 48)
        I = 8 * rnd.randint(1, 100)
        V = 8 * rnd.randint(1, 400)
        Mm = rnd.randint(1, 12)
        Mh = Mm if k % 2 == 0 else rnd.randint(1, 12)  # half the cases take the chunk-wise schedule
        out.append((N, H, I, V, Mm, Mh))
    return out


@pytest.mark.parametrize("shape", _cases(), ids=lambda c: "N{}_H{}_I{}_V{}_M{}-{}".format(*c))
def test_random_shapes_match_oracle(orc, shape):
    N, H, I, V, Mm, Mh = shape
    c = orc.make_inputs(hash(shape) % 100000, N, H, I, V, p_ignore=0.05)
    if (c["L"] >= 0).sum() == 0:
        c["L"][0] = 0
    t = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=True, single_pass=True)
    e = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=False)
    g = to_gpu(c)
    stats, gr = ms.block_step(g["X"], g["L"], ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"]),
                              Mm, Mh)
    torch.cuda.synchronize()
    loss = float(stats[2])
    assert abs(loss - t["loss"]) <= 1e-4 * abs(t["loss"])
    assert abs(loss - e["loss"]) <= 2e-3 * abs(e["loss"])
    assert rel(gr.dX, t["dX"]) <= FUSED_BF16
    assert rel(gr.dX, e["dX"]) <= LOOSE
    for k, name in (("dWg", "W_gate"), ("dWu", "W_up"), ("dWd", "W_down"), ("dWout", "W_out")):
        assert rel(getattr(gr, name), t[k]) <= FUSED_F32, k
        assert rel(getattr(gr, name), e[k]) <= LOOSE, k


@pytest.mark.parametrize("shape", _cases(16, seed=7), ids=lambda c: "N{}_H{}_I{}_V{}_M{}-{}".format(*c))
def test_random_shapes_separate_ops_match_oracle(orc, shape):
    """The SPEC ops one by one (two-pass LM-Head: logits recomputed in the
    backward, one bf16 rounding of dlogits) against the bf16-emulating
    checker at the tight bounds of test_gpu_parity.py."""
    from test_gpu_parity import TIGHT_BF16, TIGHT_F32

    N, H, I, V, Mm, Mh = shape
    c = orc.make_inputs(hash(shape) % 100000 + 1, N, H, I, V, p_ignore=0.05)
    if (c["L"] >= 0).sum() == 0:
        c["L"][0] = 0
    t = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=True)
    g = to_gpu(c)
    w = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"])
    plan, hplan = ms.make_chunk_plan(N, Mm), ms.make_chunk_plan(N, Mh)
    O, saved = ms.miniseq_mlp_forward(g["X"], w, plan)
    loss, hs = ms.miniseq_lmhead_forward(O, g["L"], ms.LmHeadWeights(g["Wout"]), hplan)
    dO, dWo = ms.miniseq_lmhead_backward(hs, ms.LmHeadWeights(g["Wout"]), hplan)
    dX, gr = ms.miniseq_mlp_backward(dO, saved, w, plan)
    torch.cuda.synchronize()
    assert abs(float(loss) - t["loss"]) <= 1e-4 * abs(t["loss"])
    assert rel(O, t["O"]) <= TIGHT_BF16
    assert rel(dO, t["dO"]) <= TIGHT_BF16
    assert rel(dX, t["dX"]) <= TIGHT_BF16
    assert rel(dWo, t["dWout"]) <= TIGHT_F32
    for k, name in (("dWg", "W_gate"), ("dWu", "W_up"), ("dWd", "W_down")):
        assert rel(getattr(gr, name), t[k]) <= TIGHT_F32, k


def _gemm_cases(n=32, seed=11):
    rnd = random.Random(seed)
    return [(8 * rnd.randint(1, 160), 8 * rnd.randint(1, 160), 8 * rnd.randint(1, 160), rnd.randint(0, 1),
             rnd.randint(0, 1), rnd.randint(0, 1), rnd.randint(0, 1)) for _ in range(n)]


@pytest.mark.parametrize("case", _gemm_cases(), ids=lambda c: "M{}_N{}_K{}_amn{}_bmn{}_f32{}_beta{}".format(*c))
def test_random_engine_gemms_match_fp64(case):
    """mst_gemm (the decoder's projection GEMMs on the same engine) over random
    extents and every operand orientation, store and accumulate."""
    from paper_2407_15892_b200 import model as mdl

    M, N, K, amn, bmn, f32, beta = case
    beta = beta if f32 else 0  # accumulation is defined for the fp32 output only (mst.h)
    torch.manual_seed(hash(case) % 1000)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    base = torch.randn(M, N, device="cuda")
    out = (base if f32 else base.bfloat16()).clone()
    mdl.gemm(A.t().contiguous() if amn else A, B if bmn else B.t().contiguous(), M, N, K, bool(amn), bool(bmn), out,
             beta=beta)
    ref = A.double() @ B.double() + (base.double() if beta else 0)
    assert rel(out.float(), ref.cpu().numpy()) <= (1e-5 if f32 else 4e-3), case


def test_engine_gemm_rejects_bf16_accumulation():
    A = torch.randn(64, 64, device="cuda").bfloat16()
    out = torch.zeros(64, 64, device="cuda").bfloat16()
    with pytest.raises(ms.ConfigError):
        ms.debug_gemm(A, A, 64, 64, 64, 0, 1, out, beta=1)

