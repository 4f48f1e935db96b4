"""GPU parity: libmst (sm_100a, through the C ABI) against the f64 oracle.

Inputs are the oracle's Rng-generated bf16 values (oracle.make_inputs), so the
GPU and the checker see bit-identical operands.  Two checkers:
  * oracle with round_bf16=True rounds to bf16 exactly where libmst stores
    bf16 (h, O, dlogits, dO, dG, dU, dX): only fp32-vs-f64 accumulation and
    rare bf16 rounding-boundary flips differ -> tight tolerances;
  * the exact f64 oracle (no intermediate rounding) -> the end-to-end
    error of bf16 compute with fp32 accumulation (north-star tolerance).
Tolerances (normwise relative ||gpu - ref||_F / ||ref||_F unless noted):
  TIGHT  = 4e-3 for bf16-stored tensors, 2e-3 for fp32 dW, loss rel 1e-4
  LOOSE  = 2e-2 for every tensor vs the exact f64 oracle, loss rel 2e-3
"""
import numpy as np
import pytest
import torch

from paper_2407_15892_b200 import miniseq as ms

pytestmark = pytest.mark.gpu

TIGHT_BF16 = 4e-3
TIGHT_F32 = 2e-3
LOOSE = 2e-2


def rel(a, b):
    a = np.asarray(a.float().cpu().numpy() if torch.is_tensor(a) else a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_gpu(c):
    d = {}
    for k in ("X", "Wg", "Wu", "Wd", "Wout"):
        d[k] = torch.from_numpy(c[k]).to("cuda").bfloat16()
    d["L"] = torch.from_numpy(c["L"]).to("cuda")
    return d


CASES = [
    # (N, H, I, V, M_mlp, M_head)       config 1 of BASELINE.json first
    (1024, 256, 688, 4096, 4, 4),
    (1024, 256, 688, 4096, 1, 16),
    (257, 64, 136, 520, 3, 7),    # ragged: partial 256-row tiles, I/V not multiples of 128/256
    (5, 16, 32, 40, 16, 16),      # M > N: singleton chunks
    (300, 8, 8, 8, 2, 2),         # tiny extents (TMA boxes larger than the tensor)
]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: "N{}_H{}_I{}_V{}_M{}-{}".format(*c))
def case(request, orc):
    N, H, I, V, Mm, Mh = request.param
    c = orc.make_inputs(request.param_index + 11, N, H, I, V, p_ignore=0.05)
    if (c["L"] >= 0).sum() == 0:
        c["L"][0] = 0
    tight = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=True)
    tight_sp = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=True,
                         single_pass=True)
    exact = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], Mm, Mh, round_bf16=False)
    return dict(shape=request.param, c=c, g=to_gpu(c), tight=tight, tight_sp=tight_sp, exact=exact)


def test_block_step_matches_oracle(case):
    """block_step runs the single-pass head: its checker replays the bf16
    softmax numerators (oracle.block(single_pass=True))."""
    N, H, I, V, Mm, Mh = case["shape"]
    g, t, e = case["g"], case["tight_sp"], case["exact"]
    stats, gr = ms.block_step(g["X"], g["L"], ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"]),
                              Mm, Mh)
    torch.cuda.synchronize()
    loss = float(stats[2])
    assert abs(loss - t["loss"]) <= 1e-4 * abs(t["loss"])
    assert abs(loss - e["loss"]) <= 2e-3 * abs(e["loss"])
    assert rel(gr.dX, t["dX"]) <= TIGHT_BF16
    for k, name in (("dWg", "W_gate"), ("dWu", "W_up"), ("dWd", "W_down"), ("dWout", "W_out")):
        assert rel(getattr(gr, name), t[k]) <= TIGHT_F32, k
        assert rel(getattr(gr, name), e[k]) <= LOOSE, k
    assert rel(gr.dX, e["dX"]) <= LOOSE


def test_ops_match_oracle(case):
    N, H, I, V, Mm, Mh = case["shape"]
    g, t = case["g"], case["tight"]
    w = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"])
    plan = ms.make_chunk_plan(N, Mm)
    O, saved = ms.miniseq_mlp_forward(g["X"], w, plan)
    assert rel(O, t["O"]) <= TIGHT_BF16
    hplan = ms.make_chunk_plan(N, Mh)
    loss, hs = ms.miniseq_lmhead_forward(O, g["L"], ms.LmHeadWeights(g["Wout"]), hplan)
    ms.check_lmhead_stats(hs)
    assert abs(float(loss) - t["loss"]) <= 1e-4 * abs(t["loss"])
    assert np.abs(hs.lse.cpu().numpy() - t["lse"]).max() <= 2e-3 * max(1.0, np.abs(t["lse"]).max())
    dO, dWo = ms.miniseq_lmhead_backward(hs, ms.LmHeadWeights(g["Wout"]), hplan)
    assert rel(dO, t["dO"]) <= TIGHT_BF16
    assert rel(dWo, t["dWout"]) <= TIGHT_F32
    dX, gr = ms.miniseq_mlp_backward(dO, saved, w, plan)
    assert rel(dX, t["dX"]) <= TIGHT_BF16
    assert rel(gr.W_gate, t["dWg"]) <= TIGHT_F32
    assert rel(gr.W_up, t["dWu"]) <= TIGHT_F32
    assert rel(gr.W_down, t["dWd"]) <= TIGHT_F32


def test_m_consistency_bitwise(orc):
    """O, lse, dO and dX are bitwise equal across M (row results do not depend
    on chunk placement); dW agrees within fp32 reassociation."""
    N, H, I, V = 1536, 128, 384, 1024
    g = to_gpu(orc.make_inputs(77, N, H, I, V))
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    ref = None
    for M in (1, 2, 3, 6, 8):
        stats, gr = ms.block_step(g["X"], g["L"], mlp, head, M, M)
        plan = ms.make_chunk_plan(N, M)
        O, _ = ms.miniseq_mlp_forward(g["X"], mlp, plan)
        _, hs = ms.miniseq_lmhead_forward(O, g["L"], head, plan)
        cur = dict(O=O.clone(), lse=hs.lse.clone(), dX=gr.dX.clone(), loss=float(stats[2]),
                   dWg=gr.W_gate.clone(), dWout=gr.W_out.clone())
        if ref is None:
            ref = cur
            continue
        assert torch.equal(cur["O"], ref["O"]), M
        assert torch.equal(cur["lse"], ref["lse"]), M
        assert torch.equal(cur["dX"], ref["dX"]), M
        assert abs(cur["loss"] - ref["loss"]) <= 1e-6 * abs(ref["loss"])
        assert rel(cur["dWg"], ref["dWg"].double().cpu().numpy()) <= 1e-5
        assert rel(cur["dWout"], ref["dWout"].double().cpu().numpy()) <= 1e-5


def test_rerun_bitwise_deterministic(orc):
    g = to_gpu(orc.make_inputs(5, 777, 64, 128, 264))
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    a = ms.block_step(g["X"], g["L"], mlp, head, 3, 5)
    a = [t.clone() for t in (a[0], a[1].dX, a[1].W_gate, a[1].W_out)]
    b = ms.block_step(g["X"], g["L"], mlp, head, 3, 5)
    b = [b[0], b[1].dX, b[1].W_gate, b[1].W_out]
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_paper_mean_mode(orc):
    N, H, V, M = 512, 64, 256, 4
    c = orc.make_inputs(9, N, H, 64, V, p_ignore=0.0)
    c["L"][128:256] = -100  # one chunk fully ignored -> modes differ
    g = to_gpu(c)
    head = ms.LmHeadWeights(g["Wout"])
    plan = ms.make_chunk_plan(N, M)
    for mode in (ms.TOKEN_WEIGHTED, ms.PAPER_MEAN):
        loss, hs = ms.miniseq_lmhead_forward(g["X"], g["L"], head, plan, mode)
        ref_loss, _, _, _ = orc.miniseq_lmhead_forward(c["X"], c["L"], c["Wout"], M, mode)
        assert abs(float(loss) - ref_loss) <= 1e-4 * abs(ref_loss)
        dX, dW = ms.miniseq_lmhead_backward(hs, head, plan, grad_loss=0.5)
        rdX, rdW = orc.miniseq_lmhead_backward(c["X"], c["L"], c["Wout"], M, mode, 0.5, True)
        assert rel(dX, rdX) <= TIGHT_BF16 and rel(dW, rdW) <= TIGHT_F32


def test_grad_accumulation(orc):
    """accumulate=1 adds onto existing dW (gradient accumulation)."""
    g = to_gpu(orc.make_inputs(3, 512, 64, 128, 256))
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    _, g1 = ms.block_step(g["X"], g["L"], mlp, head, 2, 2)
    once = g1.W_out.clone(), g1.W_gate.clone()
    ms.block_step(g["X"], g["L"], mlp, head, 2, 2, grads=g1, accumulate=True)
    assert torch.allclose(g1.W_out, 2 * once[0], rtol=1e-5, atol=1e-7)
    assert torch.allclose(g1.W_gate, 2 * once[1], rtol=1e-5, atol=1e-7)


def test_error_behaviour():
    dev = "cuda"
    X = torch.zeros(16, 64, dtype=torch.bfloat16, device=dev)
    W = torch.zeros(64, 64, dtype=torch.bfloat16, device=dev)
    plan = ms.make_chunk_plan(16, 2)
    with pytest.raises(ms.DtypeError):
        ms.miniseq_mlp_forward(X.float(), ms.MlpWeights(W, W, W), plan)
    with pytest.raises(ms.ShapeError):
        ms.miniseq_mlp_forward(X, ms.MlpWeights(W[:, :32].contiguous(), W, W), plan)
    with pytest.raises(ms.ConfigError):
        ms.miniseq_mlp_forward(X, ms.MlpWeights(W.t(), W, W), plan)  # non-contiguous
    with pytest.raises(ms.ConfigError):
        ms.miniseq_mlp_forward(X, ms.MlpWeights(W, W, W), ms.make_chunk_plan(15, 2))
    O, saved = ms.miniseq_mlp_forward(X, ms.MlpWeights(W, W, W), plan)
    W2 = W.clone()
    with pytest.raises(ms.StateError):  # saved state from other weights
        ms.miniseq_mlp_backward(O, saved, ms.MlpWeights(W2, W, W), plan)
    saved.rec.n = 8  # tampered record
    with pytest.raises(ms.StateError):
        ms.miniseq_mlp_backward(O, saved, ms.MlpWeights(W, W, W), plan)
    L = torch.full((16,), -100, dtype=torch.int32, device=dev)
    _, hs = ms.miniseq_lmhead_forward(X, L, ms.LmHeadWeights(W), plan)
    with pytest.raises(ms.DataError):  # all labels ignored
        ms.check_lmhead_stats(hs)
    L[0] = 64  # out of range label
    _, hs = ms.miniseq_lmhead_forward(X, L, ms.LmHeadWeights(W), plan)
    with pytest.raises(ms.DataError):
        ms.check_lmhead_stats(hs)


@pytest.mark.parametrize("nblk", [1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_engine_gemm_all_operand_majorness(a_mn, b_mn, nblk):
    """Every operand orientation, ragged extents, normal (256x256 per CTA
    pair) and wide (256x512: two N blocks sharing the A slot) tiles; N=768
    makes the last wide tile a single N block."""
    torch.manual_seed(0)
    ctx = ms.Context.get(0)
    ctx.set_tuning("debug_nblk", nblk)
    try:
        for (M, N, K) in [(256, 256, 64), (296, 200, 136), (512, 768, 4096), (256, 1024, 192)]:
            A = torch.randn(M, K, device="cuda").bfloat16()
            B = torch.randn(K, N, device="cuda").bfloat16()
            ref = A.double() @ B.double()
            for f32 in (True, False):
                out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
                ms.debug_gemm(A.t().contiguous() if a_mn else A, B if b_mn else B.t().contiguous(), M, N, K, a_mn,
                              b_mn, out)
                assert rel(out.float(), ref.cpu().numpy()) <= (1e-5 if f32 else 4e-3), (M, N, K, f32)
    finally:
        ctx.set_tuning("debug_nblk", 1)


def test_llama3_8b_shapes_against_torch_fp32():
    """Full Llama3-8B widths (H=4096, I=14336, V=128256) at S=1024, M=4: the
    oracle is too slow here, so the fp32 torch reference of the same block
    (bf16 rounding at the same points, tests/torch_ref.py) is the checker."""
    import torch_ref as R

    torch.manual_seed(1)
    N, H, I, V = 1024, 4096, 14336, 128256
    dev = "cuda"
    X = torch.randn(N, H, device=dev).bfloat16()
    Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
    Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
    Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
    L = torch.randint(0, V, (N,), device=dev, dtype=torch.int32)
    L[::17] = -100
    stats, gr = ms.block_step(X, L, ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo), 4, 4)
    ref = R.block(X, L, Wg, Wu, Wd, Wo)
    assert abs(float(stats[2]) - float(ref["loss"])) <= 1e-3 * float(ref["loss"])
    assert R.relerr(gr.dX, ref["dX"]) <= 1e-2
    assert R.relerr(gr.W_out, ref["dWout"]) <= 1e-2
    assert R.relerr(gr.W_gate, ref["dWg"]) <= 1e-2
    assert R.relerr(gr.W_down, ref["dWd"]) <= 1e-2


@pytest.mark.parametrize("shape", [(1024, 256, 4096, 4), (257, 64, 520, 3), (600, 128, 1000, 16)])
def test_lmhead_fused_matches_oracle(orc, shape):
    """Single-pass head (mst_lmhead_fused) against the oracle with its bf16
    softmax numerators replayed, at the tight bounds; loss to 1e-4 relative
    (SPEC.md:313-330)."""
    N, H, V, M = shape
    c = orc.make_inputs(41, N, H, 64, V, p_ignore=0.1)
    g = to_gpu(c)
    head = ms.LmHeadWeights(g["Wout"])
    plan = ms.make_chunk_plan(N, M)
    ctx = ms.Context.get(0)
    try:
        for knob, replay in ((1, 3), (0, 2)):  # row-scaled (default) / per-tile numerators + normalize
            ctx.set_tuning("dl_rowscale", knob)
            for mode in (ms.TOKEN_WEIGHTED, ms.PAPER_MEAN):
                loss, stats, lse, dX, dW = ms.miniseq_lmhead_fused(g["X"], g["L"], head, plan, mode, grad_loss=0.7)
                ref_loss, ref_lse, _, _ = orc.miniseq_lmhead_forward(c["X"], c["L"], c["Wout"], M, mode)
                rdX, rdW = orc.miniseq_lmhead_backward(c["X"], c["L"], c["Wout"], M, mode, 0.7, replay)
                assert abs(float(loss) - ref_loss) <= 1e-4 * abs(ref_loss)
                assert np.abs(lse.cpu().numpy() - ref_lse).max() <= 2e-3 * max(1.0, np.abs(ref_lse).max())
                assert rel(dX, rdX) <= TIGHT_BF16, (knob, rel(dX, rdX))
                assert rel(dW, rdW) <= TIGHT_F32, (knob, rel(dW, rdW))
    finally:
        ctx.set_tuning("dl_rowscale", 1)


def test_block_step_fused_vs_two_pass_head():
    """block_step with the single-pass head agrees with the two-pass head."""
    import ctypes

    torch.manual_seed(3)
    N, H, I, V, M = 1024, 256, 512, 2048, 4
    X = torch.randn(N, H, device="cuda").bfloat16()
    W = [(0.05 * torch.randn(*s, device="cuda")).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
    mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
    ctx = ms.Context.get(0)
    out = {}
    for fused in (1, 0):
        ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"fused_head", fused))
        st, gr = ms.block_step(X, L, mlp, head, M, M)
        out[fused] = (float(st[2]), gr.dX.clone(), gr.W_out.clone(), gr.W_gate.clone())
    ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"fused_head", 1))
    assert abs(out[1][0] - out[0][0]) <= 1e-5 * abs(out[0][0])
    for a, b in zip(out[1][1:], out[0][1:]):
        assert rel(a, b.double().cpu().numpy()) <= 6e-3


@pytest.mark.parametrize("shape", [(1024, 256, 688, 4096, 4), (777, 64, 136, 520, 3)])
def test_block_step_chunked_matches_op_by_op(shape):
    """Chunk-wise block schedule (saved G,U, no recompute) == op-by-op
    schedule: same kernels and accumulation orders, so agreement is at
    fp32-rounding level (FMA contraction may differ in the SwiGLU backward)."""
    N, H, I, V, M = shape
    torch.manual_seed(7)
    X = torch.randn(N, H, device="cuda").bfloat16()
    W = [(0.05 * torch.randn(*s, device="cuda")).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
    L[::9] = -100
    mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
    ctx = ms.Context.get(0)
    out = {}
    for key, (chunked, fused) in {1: (1, 0), 0: (0, 0), "f": (1, 1)}.items():
        ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"chunked_block", chunked))
        ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"fuse_swiglu_bwd", fused))
        st, gr = ms.block_step(X, L, mlp, head, M, M)
        torch.cuda.synchronize()
        out[key] = (float(st[2]), gr.dX.clone(), gr.W_gate.clone(), gr.W_up.clone(), gr.W_down.clone(),
                    gr.W_out.clone())
    ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"chunked_block", 1))
    ms._check(ctx.lib.mst_ctx_set_tuning(ctx.handle, b"fuse_swiglu_bwd", 0))
    assert out[1][0] == out[0][0]
    for a, b in zip(out[1][1:], out[0][1:]):
        assert rel(a, b.double().cpu().numpy()) <= 1e-5
    # SwiGLU backward fused into the dh GEMM epilogue (tuning fuse_swiglu_bwd=1): same values
    assert out["f"][0] == out[1][0]
    for a, b in zip(out["f"][1:], out[1][1:]):
        assert rel(a, b.double().cpu().numpy()) <= 1e-6


def test_nonfinite_scan_counts_nan_and_inf():
    """mst_count_nonfinite: bf16 and fp32, ragged lengths (tail bytes), NaN and
    +-Inf anywhere."""
    for dtype in (torch.bfloat16, torch.float32):
        for n in (1, 7, 8, 1000, 4099, 1 << 20):
            t = torch.randn(n, device="cuda").to(dtype)
            assert int(ms.count_nonfinite(t).item()) == 0
            idx = sorted({0, n // 3, n - 1})
            vals = [float("nan"), float("inf"), float("-inf")]
            for k, i in enumerate(idx):
                t[i] = vals[k % 3]
            assert int(ms.count_nonfinite(t).item()) == len(idx), (dtype, n)
            if n > 8:  # unaligned views: leading bytes before the first 16-byte boundary
                assert int(ms.count_nonfinite(t[1:]).item()) == len(idx) - 1, (dtype, n)


def test_nonfinite_inputs_and_loss_raise_nonfinite_error(orc):
    N, H, I, V = 256, 128, 128, 512
    c = orc.make_inputs(9, N, H, I, V)
    g = {k: torch.from_numpy(c[k]).cuda().bfloat16() for k in ("X", "Wg", "Wu", "Wd", "Wout")}
    L = torch.from_numpy(c["L"]).cuda()
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    ms.block_step(g["X"], L, mlp, head, 2, 2, check=True)  # clean inputs pass
    X = g["X"].clone()
    X[17, 5] = float("nan")
    with pytest.raises(ms.NonFiniteError, match="X"):
        ms.block_step(X, L, mlp, head, 2, 2, check=True)
    Wo = g["Wout"].clone()
    Wo[3, 7] = float("inf")
    _, hs = ms.miniseq_lmhead_forward(g["X"], L, ms.LmHeadWeights(Wo), ms.make_chunk_plan(N, 2))
    with pytest.raises(ms.NonFiniteError):
        ms.check_lmhead_stats(hs)
    Lbad = L.clone()
    Lbad[0] = V + 3
    with pytest.raises(ms.DataError):
        ms.block_step(g["X"], Lbad, mlp, head, 2, 2, check=True)


def test_block_step_sp_global_valid_scaling(orc):
    """mst_block_step_sp: global_valid == the local count reproduces
    block_step bitwise; twice the count halves every gradient exactly
    (the scale is a power of two, so bf16 dlogits and fp32 sums are exact)."""
    N, H, I, V = 512, 128, 256, 1024
    c = orc.make_inputs(21, N, H, I, V)
    g = to_gpu(c)
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    _, ref = ms.block_step(g["X"], g["L"], mlp, head, 4, 4)
    ref = {k: getattr(ref, k).clone() for k in ("dX", "W_gate", "W_up", "W_down", "W_out")}
    nv = ms.count_valid(g["L"], V)
    # exact fp64 integer count (SPEC.md:648 int64 all-reduce), fp32 rejected
    assert nv.dtype == torch.float64 and nv.item() == int(((g["L"] >= 0) & (g["L"] < V)).sum())
    with pytest.raises(ms.DtypeError):
        ms.block_step(g["X"], g["L"], mlp, head, 4, 4, global_valid=nv.float())
    calls = []
    _, same = ms.block_step(g["X"], g["L"], mlp, head, 4, 4, global_valid=nv.clone(), grad_ready=calls.append)
    assert calls == [3, 0, 1, 2]  # W_out after the head, the MLP weights at the end
    for k, t in ref.items():
        assert torch.equal(getattr(same, k), t), k
    _, half = ms.block_step(g["X"], g["L"], mlp, head, 4, 4, global_valid=2 * nv)
    for k, t in ref.items():
        assert torch.equal(getattr(half, k).float(), t.float() * 0.5), k


def test_count_valid_exact_beyond_fp32():
    """The valid-label count stays an exact integer past 2^24 tokens (fp32
    would round 2^24 + 3 to 2^24 + 4): mst_count_valid counts in int64 and
    returns fp64."""
    n = (1 << 24) + 3
    L = torch.zeros(n, dtype=torch.int32, device="cuda")
    L[::1000] = -100
    want = n - len(range(0, n, 1000))
    assert ms.count_valid(L, 10).item() == want


def test_config2_full_size_properties():
    """BASELINE config 2 at full size (Llama3-8B widths, S=8192): the bench's
    M=8 chunk-wise block step against (a) the fp32 torch reference of the
    same block and (b) itself at M=1 and M=2: dX and the loss are independent
    of M (chunk boundaries are multiples of the 256-row tile), dW within fp32
    reassociation; reruns are bitwise."""
    import torch_ref as R

    torch.manual_seed(5)
    N, H, I, V = 8192, 4096, 14336, 128256
    dev = "cuda"
    X = torch.randn(N, H, device=dev).bfloat16()
    Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
    Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
    Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
    L = torch.randint(0, V, (N,), device=dev, dtype=torch.int32)
    L[torch.rand(N, device=dev) < 0.05] = -100
    mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
    res = {}
    for M in (8, 2, 1):
        st, gr = ms.block_step(X, L, mlp, head, M, M)
        res[M] = (float(st[2]), {k: getattr(gr, k).clone() for k in ("dX", "W_gate", "W_up", "W_down", "W_out")})
    st, gr = ms.block_step(X, L, mlp, head, 8, 8)
    for k, t in res[8][1].items():
        assert torch.equal(getattr(gr, k), t), k  # bitwise rerun
    for M in (2, 1):
        assert abs(res[M][0] - res[8][0]) <= 1e-5 * res[8][0]
        assert torch.equal(res[M][1]["dX"], res[8][1]["dX"])
        for k in ("W_gate", "W_up", "W_down", "W_out"):
            assert R.relerr(res[M][1][k], res[8][1][k].float()) <= 1e-5, (M, k)
    ref = R.block(X, L, Wg, Wu, Wd, Wo)
    assert abs(res[8][0] - float(ref["loss"])) <= 1e-3 * float(ref["loss"])
    for k, rk in (("dX", "dX"), ("W_out", "dWout"), ("W_gate", "dWg"), ("W_up", "dWu"), ("W_down", "dWd")):
        assert R.relerr(res[8][1][k], ref[rk]) <= 1e-2, k


def test_tile_scheduler_back_to_back_launches():
    """The dynamic tile scheduler (one claiming thread per CTA pair, an
    8-entry code ring, a claim counter the last pair re-zeroes on exit):
    back-to-back launches with fewer tiles than pairs, exactly one tile per
    pair, and many waves, in both scheduling modes, with no host sync in
    between.  Results must equal the static per-pair lists bitwise (the tile
    order does not change any tile's arithmetic)."""
    torch.manual_seed(5)
    ctx = ms.Context.get(0)
    pairs = ctx.lib.mst_ctx_num_pairs(ctx.handle)
    shapes = [(256, 256, 128), (256, 256 * pairs, 64), (512, 256 * (pairs - 1), 1024), (2048, 4096, 512),
              (296, 520, 72)]
    data = []
    for (M, N, K) in shapes:
        data.append((torch.randn(M, K, device="cuda").bfloat16(), torch.randn(K, N, device="cuda").bfloat16(),
                     M, N, K))
    outs = {}
    try:
        for mode in (0, 1):
            ctx.set_tuning("dynamic", mode)
            res = []
            for rep in range(3):
                for A, B, M, N, K in data:
                    out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
                    ms.debug_gemm(A, B, M, N, K, 0, 1, out)
                    res.append(out)
            torch.cuda.synchronize()
            outs[mode] = res
    finally:
        ctx.set_tuning("dynamic", 1)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    for (A, B, M, N, K), out in zip(data, outs[1]):
        assert rel(out, (A.double() @ B.double()).cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("shape", [(1024, 256, 688, 4096, 4), (777, 512, 136, 520, 3), (300, 64, 136, 520, 1),
                                   (2048, 1024, 2816, 32000, 8)])
def test_block_step_host_streams_bitwise_equal(shape):
    """mst_block_step_host (X / labels / dX in pinned host memory, chunks
    streamed on a copy stream) == mst_block_step on device tensors, bitwise,
    including back-to-back calls that reuse the chunk buffers and events."""
    N, H, I, V, M = shape
    torch.manual_seed(3)
    X = torch.randn(N, H, device="cuda").bfloat16()
    W = [(0.05 * torch.randn(*s, device="cuda")).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
    L[::11] = -100
    mlp, head = ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])
    st, gr = ms.block_step(X, L, mlp, head, M, M)
    Xh, Lh = X.cpu().pin_memory(), L.cpu().pin_memory()
    for rep in range(2):
        dXh = torch.full((N, H), float("nan"), dtype=torch.bfloat16).pin_memory()
        sth, grh = ms.block_step_host(Xh, Lh, mlp, head, M, dXh)
        torch.cuda.synchronize()
        assert torch.equal(sth[:3], st[:3])
        assert torch.equal(dXh, gr.dX.cpu())
        for a, b in ((grh.W_gate, gr.W_gate), (grh.W_up, gr.W_up), (grh.W_down, gr.W_down), (grh.W_out, gr.W_out)):
            assert torch.equal(a, b)
