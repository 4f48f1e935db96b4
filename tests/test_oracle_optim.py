"""The optimizer oracle (oracle/optim_ref.py) against every example the SPEC
gives for the `optim` module.  CPU only."""
import numpy as np
import pytest

from oracle import optim_ref as O


def test_clip_kats():
    # ||g|| = 0.5, max 1.0 -> unchanged
    g = [np.array([0.3, 0.4])]
    out, n = O.clip_global_norm(g, 1.0)
    assert n == pytest.approx(0.5) and np.array_equal(out[0], g[0])
    # single grad [3,4], max 1.0 -> [0.6, 0.8]
    out, n = O.clip_global_norm([np.array([3.0, 4.0])], 1.0)
    assert n == 5.0 and np.allclose(out[0], [0.6, 0.8], rtol=0, atol=1e-15)
    # post-clip global norm <= max-norm + 1e-12
    rng = np.random.default_rng(0)
    gs = [rng.normal(size=(7, 5)) * 10, rng.normal(size=13)]
    out, _ = O.clip_global_norm(gs, 1.0)
    assert O.global_norm(out) <= 1.0 + 1e-12
    with pytest.raises(FloatingPointError):
        O.clip_global_norm([np.array([1.0, np.nan])], 1.0)


def test_adamw_kats():
    # zero grads, zero wd -> weights unchanged
    w = np.array([1.0, -2.0, 3.0])
    w2, _, _ = O.adamw_step(w, np.zeros(3), np.zeros(3), np.zeros(3), 1, weight_decay=0.0)
    assert np.array_equal(w2, w)
    # scalar w=1, g=1, step 1 -> 1 - lr*wd*1 - lr/(1+1e-8)
    w2, m, v = O.adamw_step(np.array([1.0]), np.array([1.0]), np.zeros(1), np.zeros(1), 1)
    assert w2[0] == pytest.approx(1 - 1e-4 * 0.001 * 1 - 1e-4 / (1 + 1e-8), abs=1e-15)
    # two steps with identical grads -> ||dw|| per step within 5%
    rng = np.random.default_rng(1)
    w0 = rng.normal(size=100)
    g = rng.normal(size=100)
    w1, m, v = O.adamw_step(w0, g, np.zeros(100), np.zeros(100), 1)
    w2, m, v = O.adamw_step(w1, g, m, v, 2)
    d1, d2 = np.linalg.norm(w1 - w0), np.linalg.norm(w2 - w1)
    assert abs(d2 - d1) / d1 < 0.05


def test_accumulation_kats():
    rng = np.random.default_rng(2)
    g = [rng.normal(size=(4, 3))]
    # steps=1 -> identity
    assert np.array_equal(O.accumulate([g], 1)[0], g[0])
    # g and -g -> zero
    assert np.array_equal(O.accumulate([g, [-g[0]]], 2)[0], np.zeros((4, 3)))
    # k identical micro-batches == one k-times batch, within 1e-12
    k = 5
    assert np.allclose(O.accumulate([g] * k, k)[0], g[0], rtol=0, atol=1e-12)
    with pytest.raises(RuntimeError):
        O.accumulate([], 2)


def test_in_backward_equals_deferred_without_clip():
    """with clipping off, stepping each parameter during
    backward == stepping all after backward (the update is per-element)."""
    rng = np.random.default_rng(3)
    ws = [rng.normal(size=8), rng.normal(size=(3, 4))]
    gs = [rng.normal(size=8), rng.normal(size=(3, 4))]
    deferred = [O.adamw_step(w, g, np.zeros_like(w), np.zeros_like(w), 1)[0] for w, g in zip(ws, gs)]
    inb = []
    for w, g in reversed(list(zip(ws, gs))):  # backward order
        inb.insert(0, O.adamw_step(w, g, np.zeros_like(w), np.zeros_like(w), 1)[0])
    for a, b in zip(deferred, inb):
        assert np.array_equal(a, b)
