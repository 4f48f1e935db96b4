"""The CPU oracle against every SPEC known-answer example and property of the
hot path."""
import math

import numpy as np
import pytest

RNG = np.random.default_rng(0)


def rand_case(orc, seed, N, H, I, V, p_ignore=0.1):
    return orc.make_inputs(seed, N, H, I, V, p_ignore=p_ignore, x_std=1.0, w_std=0.3)


# ----------------------------------------------------------------- tensor-core KATs
def test_matmul_kats(orc):
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(orc.matmul(a, np.array([[5.0], [6.0]])), np.array([[17.0], [39.0]]))
    assert np.array_equal(orc.matmul(a, np.eye(2)), a)
    x = RNG.standard_normal((2, 3))
    assert np.array_equal(orc.matmul(x, np.eye(3)), x)


def test_matmul_associativity(orc):
    a, b, c = (RNG.uniform(-1, 1, (s, s)) for s in (16, 16, 16))
    assert np.abs(orc.matmul(orc.matmul(a, b), c) - orc.matmul(a, orc.matmul(b, c))).max() <= 1e-10


def test_silu_kats(orc):
    assert orc.silu(0.0) == 0.0
    assert abs(orc.silu(1.0) - 0.7310585786300049) < 1e-12
    assert abs(orc.silu(-20.0) - (-4.12230724e-8)) < 1e-14


def test_silu_backward_kats(orc):
    assert orc.silu_backward(0.0, 1.0) == 0.5
    fd = (orc.silu(1.0 + 1e-6) - orc.silu(1.0 - 1e-6)) / 2e-6
    assert abs(orc.silu_backward(1.0, 1.0) - 0.9276705) < 1e-7
    assert abs(orc.silu_backward(1.0, 1.0) - fd) < 1e-8
    assert orc.silu_backward(3.7, 0.0) == 0.0


# ----------------------------------------------------------------- chunk plan
def test_chunk_plan_examples(orc):
    assert orc.make_chunk_plan(8, 2) == [(0, 4), (4, 8)]
    assert orc.make_chunk_plan(8, 1) == [(0, 8)]
    assert orc.make_chunk_plan(7, 2) == [(0, 4), (4, 7)]


@pytest.mark.parametrize("M", [1, 2, 3, 4, 7, 8, 16])
def test_chunk_plan_invariants(orc, M):
    for N in range(1, 65):
        p = orc.make_chunk_plan(N, M)
        assert len(p) == min(M, N)
        assert p[0][0] == 0 and p[-1][1] == N
        assert all(a[1] == b[0] for a, b in zip(p, p[1:]))
        sizes = [e - s for s, e in p]
        assert max(sizes) == math.ceil(N / min(M, N)) and max(sizes) - min(sizes) <= 1


def test_chunk_plan_errors(orc):
    with pytest.raises(orc.OracleError) as e:
        orc.make_chunk_plan(0, 4)
    assert e.value.code == 5


# ----------------------------------------------------------------- blocks-std KATs
def test_lmhead_uniform_logits_is_ln_v(orc):
    X = RNG.standard_normal((5, 4))
    L = np.array([0, 3, 7, 1, 2], dtype=np.int32)
    loss, _ = orc.lmhead_forward(X, L, np.zeros((4, 8)))
    assert abs(loss - 2.0794415416798357) < 1e-12


def test_lmhead_all_ignored_is_error(orc):
    with pytest.raises(orc.OracleError) as e:
        orc.lmhead_forward(np.ones((3, 4)), np.full(3, -100, np.int32), np.ones((4, 8)))
    assert e.value.code == 5


def test_mlp_zero_input(orc):
    c = rand_case(orc, 1, 4, 8, 16, 8)
    O = orc.mlp_forward(np.zeros((4, 8)), c["Wg"], c["Wu"], c["Wd"])
    assert not O.any()


def test_mlp_zero_grad(orc):
    c = rand_case(orc, 2, 6, 8, 16, 8)
    for M in (1, 3):
        g = orc.miniseq_mlp_backward(np.zeros((6, 8)), c["X"], c["Wg"], c["Wu"], c["Wd"], M)
        assert all(not t.any() for t in g)


def test_dlogits_rows_sum_to_zero(orc):
    c = rand_case(orc, 3, 9, 8, 16, 12)
    # sum_v dW_out[h, v] = sum_r X[r,h] sum_v dl[r,v] = 0
    _, dW = orc.lmhead_backward(c["X"], c["L"], c["Wout"])
    assert np.abs(dW.sum(axis=1)).max() < 1e-12


def test_loss_permutation_equivariant(orc):
    c = rand_case(orc, 4, 16, 8, 16, 32)
    perm = RNG.permutation(16)
    l1, _ = orc.lmhead_forward(c["X"], c["L"], c["Wout"])
    l2, _ = orc.lmhead_forward(c["X"][perm], c["L"][perm], c["Wout"])
    assert abs(l1 - l2) <= 1e-12


def test_ignored_rows_have_zero_dx(orc):
    c = rand_case(orc, 5, 8, 8, 16, 16, p_ignore=0.0)
    L = np.full(8, -100, np.int32)
    L[3] = 5
    dX, _ = orc.lmhead_backward(c["X"], L, c["Wout"])
    assert np.abs(np.delete(dX, 3, axis=0)).max() == 0.0 and np.abs(dX[3]).max() > 0


# ----------------------------------------------------------------- finite differences
def _fd_check(f, x, grad, n_probe=20, h=1e-5, seed=0):
    r = np.random.default_rng(seed)
    idx = [tuple(r.integers(0, s) for s in x.shape) for _ in range(n_probe)]
    for i in idx:
        xp = x.copy()
        xp[i] += h
        xm = x.copy()
        xm[i] -= h
        fd = (f(xp) - f(xm)) / (2 * h)
        g = grad[i]
        assert abs(fd - g) <= 1e-6 * max(1.0, abs(fd), abs(g)) + 1e-9, (i, fd, g)


@pytest.mark.parametrize("seed", range(5))
def test_mlp_grad_finite_difference(orc, seed):
    c = rand_case(orc, 100 + seed, 6, 8, 16, 8)
    R = np.random.default_rng(seed).standard_normal((6, 8))  # scalar loss = <R, O>
    dX, dWg, dWu, dWd = orc.mlp_backward(R, c["X"], c["Wg"], c["Wu"], c["Wd"])
    f = lambda **kw: float((R * orc.mlp_forward(kw.get("X", c["X"]), kw.get("Wg", c["Wg"]), kw.get("Wu", c["Wu"]),
                                                kw.get("Wd", c["Wd"]))).sum())  # noqa: E731
    _fd_check(lambda v: f(X=v), c["X"].astype(np.float64), dX, seed=seed)
    _fd_check(lambda v: f(Wg=v), c["Wg"].astype(np.float64), dWg, seed=seed)
    _fd_check(lambda v: f(Wu=v), c["Wu"].astype(np.float64), dWu, seed=seed)
    _fd_check(lambda v: f(Wd=v), c["Wd"].astype(np.float64), dWd, seed=seed)


@pytest.mark.parametrize("seed", range(5))
def test_lmhead_grad_finite_difference(orc, seed):
    c = rand_case(orc, 200 + seed, 7, 8, 16, 12)
    dX, dW = orc.lmhead_backward(c["X"], c["L"], c["Wout"])
    _fd_check(lambda v: orc.lmhead_forward(v, c["L"], c["Wout"])[0], c["X"].astype(np.float64), dX, seed=seed)
    _fd_check(lambda v: orc.lmhead_forward(c["X"], c["L"], v)[0], c["Wout"].astype(np.float64), dW, seed=seed)


# ----------------------------------------------------------------- miniseq equivalence
def test_miniseq_m1_bitwise_equals_standard(orc):
    c = rand_case(orc, 7, 13, 8, 24, 16)
    X, Wg, Wu, Wd, Wo, L = c["X"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], c["L"]
    assert np.array_equal(orc.miniseq_mlp_forward(X, Wg, Wu, Wd, 1), orc.mlp_forward(X, Wg, Wu, Wd))
    dO = np.random.default_rng(1).standard_normal(X.shape)
    for a, b in zip(orc.miniseq_mlp_backward(dO, X, Wg, Wu, Wd, 1), orc.mlp_backward(dO, X, Wg, Wu, Wd)):
        assert np.array_equal(a, b)
    assert orc.miniseq_lmhead_forward(X, L, Wo, 1)[0] == orc.lmhead_forward(X, L, Wo)[0]
    for a, b in zip(orc.miniseq_lmhead_backward(X, L, Wo, 1), orc.lmhead_backward(X, L, Wo)):
        assert np.array_equal(a, b)


def test_miniseq_mlp_examples(orc):
    c = rand_case(orc, 8, 16, 8, 32, 8)
    X, Wg, Wu, Wd = c["X"], c["Wg"], c["Wu"], c["Wd"]
    O = orc.miniseq_mlp_forward(X, Wg, Wu, Wd, 4)
    assert np.abs(O - orc.mlp_forward(X, Wg, Wu, Wd)).max() <= 1e-12
    dO = np.random.default_rng(2).standard_normal(X.shape)
    for a, b in zip(orc.miniseq_mlp_backward(dO, X, Wg, Wu, Wd, 4), orc.mlp_backward(dO, X, Wg, Wu, Wd)):
        assert np.abs(a - b).max() <= 1e-10


def test_miniseq_lmhead_example(orc):
    c = rand_case(orc, 9, 64, 8, 8, 32)
    X, L, Wo = c["X"], c["L"], c["Wout"]
    for a, b in zip(orc.miniseq_lmhead_backward(X, L, Wo, 16), orc.lmhead_backward(X, L, Wo)):
        assert np.abs(a - b).max() <= 1e-10


def test_randomized_equivalence_100_cases(orc):
    """Acceptance 1: >=100 randomized (shape, seed, M) cases,
    non-divisible N included; fwd <= 1e-12, grads <= 1e-10 (f64, token-weighted)."""
    r = np.random.default_rng(1234)
    n_cases = 0
    for case in range(104):
        N = int(r.integers(4, 65))
        M = int(r.choice([1, 2, 3, 4, 7, 8, 16]))
        H, I, V = int(r.choice([4, 8])), int(r.choice([8, 16])), int(r.choice([8, 16, 32]))
        c = rand_case(orc, 5000 + case, N, H, I, V, p_ignore=0.2)
        if (c["L"] >= 0).sum() == 0:
            c["L"][0] = 1
        X, L, Wg, Wu, Wd, Wo = c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"]
        assert np.abs(orc.miniseq_mlp_forward(X, Wg, Wu, Wd, M) - orc.mlp_forward(X, Wg, Wu, Wd)).max() <= 1e-12
        dO = r.standard_normal(X.shape)
        for a, b in zip(orc.miniseq_mlp_backward(dO, X, Wg, Wu, Wd, M), orc.mlp_backward(dO, X, Wg, Wu, Wd)):
            assert np.abs(a - b).max() <= 1e-10
        l_ms = orc.miniseq_lmhead_forward(X, L, Wo, M)[0]
        assert abs(l_ms - orc.lmhead_forward(X, L, Wo)[0]) <= 1e-12
        for a, b in zip(orc.miniseq_lmhead_backward(X, L, Wo, M), orc.lmhead_backward(X, L, Wo)):
            assert np.abs(a - b).max() <= 1e-10
        n_cases += 1
    assert n_cases >= 100


def test_loss_modes(orc):
    c = rand_case(orc, 10, 16, 8, 8, 16, p_ignore=0.0)
    X, L, Wo = c["X"], c["L"].copy(), c["Wout"]
    tw = orc.miniseq_lmhead_forward(X, L, Wo, 4, 0)[0]
    pm = orc.miniseq_lmhead_forward(X, L, Wo, 4, 1)[0]
    assert abs(tw - pm) <= 1e-12  # equal valid counts
    L[4:8] = -100  # one chunk fully ignored
    std = orc.lmhead_forward(X, L, Wo)[0]
    tw = orc.miniseq_lmhead_forward(X, L, Wo, 4, 0)[0]
    pm = orc.miniseq_lmhead_forward(X, L, Wo, 4, 1)[0]
    assert abs(tw - std) <= 1e-12 and abs(pm - std) > 1e-6


# ----------------------------------------------------------------- counters (Thm 3.1 / 3.2)
def test_flop_invariance_and_weight_read_scaling(orc):
    """Acceptance 3/4: FLOPs equal across M | S; weight reads
    a + b*M with b = 3dI (MLP fwd) and dV (head fwd)."""
    S, H, I, V = 16, 4, 8, 12
    c = rand_case(orc, 11, S, H, I, V)
    fl, wr, hfl, hwr = [], [], [], []
    for M in (1, 2, 4, 8):
        orc.counters_reset()
        orc.miniseq_mlp_forward(c["X"], c["Wg"], c["Wu"], c["Wd"], M)
        k = orc.counters()
        fl.append(k["flops"])
        wr.append(k["weight_read_elements"])
        orc.counters_reset()
        orc.miniseq_lmhead_forward(c["X"], c["L"], c["Wout"], M)
        k = orc.counters()
        hfl.append(k["flops"])
        hwr.append(k["weight_read_elements"])
    assert len(set(fl)) == 1 and len(set(hfl)) == 1
    Ms = np.array([1, 2, 4, 8])
    b, a = np.polyfit(Ms, np.array(wr, float), 1)
    assert abs(b - 3 * H * I) < 1e-9 and abs(a) < 1e-9
    b, a = np.polyfit(Ms, np.array(hwr, float), 1)
    assert abs(b - H * V) < 1e-9 and abs(a) < 1e-9


# ----------------------------------------------------------------- memory
def test_peak_intermediate_scales_with_m(orc):
    S, H, I, V = 64, 8, 32, 64
    c = rand_case(orc, 12, S, H, I, V)
    peaks, hpeaks = [], []
    for M in (1, 2, 4, 8, 16):
        orc.mem_reset()
        orc.miniseq_mlp_forward(c["X"], c["Wg"], c["Wu"], c["Wd"], M)
        peaks.append(orc.mem_peak(orc.MEM_INTER_MLP))
        orc.mem_reset()
        orc.miniseq_lmhead_forward(c["X"], c["L"], c["Wout"], M)
        hpeaks.append(orc.mem_peak(orc.MEM_INTER_HEAD))
    assert all(a >= b for a, b in zip(peaks, peaks[1:]))  # non-increasing
    assert all(a >= b for a, b in zip(hpeaks, hpeaks[1:]))
    assert peaks[2] <= peaks[0] * math.ceil(S / 4) / S
    assert hpeaks[4] <= hpeaks[0] / 16


def test_determinism(orc):
    c = rand_case(orc, 13, 20, 8, 16, 16)
    a = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], 3, 5)
    b = orc.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], 3, 5)
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k]))


@pytest.mark.parametrize("scale_to", [None, 55.0, 100.0])
def test_rowscale_replay_close_to_exact(scale_to):
    """Replay mode 3 (the GPU's row-scaled LM-Head: numerators relative to one
    reference per row, per-row factor on dX and on the transposed head input)
    stays within bf16-level error of the exact f64 backward, also for logits
    far outside its +-64 log2-unit reference window."""
    from oracle import oracle as orc

    c = orc.make_inputs(41, 600, 128, 64, 1000, p_ignore=0.1)
    W = c["Wout"].astype(np.float64)
    if scale_to:
        W = (W * (scale_to / np.abs(c["X"].astype(np.float64) @ W).max())).astype(np.float32)
    e = orc.miniseq_lmhead_backward(c["X"], c["L"], W, 4, 0, 0.7, 0)
    t = orc.miniseq_lmhead_backward(c["X"], c["L"], W, 4, 0, 0.7, 3)
    for a, b in zip(t, e):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 5e-3
