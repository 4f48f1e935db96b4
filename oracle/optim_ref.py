"""CPU restatement of the reference's `optim` module in
numpy float64 — TEST INFRASTRUCTURE ONLY (the checker for libmst's AdamW /
clip / accumulation kernels, csrc/optim.cu).

Parity pinned to the SPEC's own examples (tests/test_oracle_optim.py):
SPEC.md:489-491 (clip KATs), SPEC.md:497-499 (AdamW KATs),
SPEC.md:504-506 (accumulation KATs), SPEC.md:512-514 (in-backward
equivalence).  The reference ships no optimizer code, so there is nothing
else to pin against.
"""
from __future__ import annotations

import numpy as np

DEFAULTS = dict(lr=1e-4, weight_decay=0.001, clip_norm=1.0, beta1=0.9, beta2=0.999, eps=1e-8)


def global_norm(grads) -> float:
    """||g||_2 over every element of every gradient."""
    return float(np.sqrt(sum(float(np.sum(np.asarray(g, dtype=np.float64) ** 2)) for g in grads)))


def clip_global_norm(grads, max_norm: float):
    """if ||g|| > max-norm scale all grads by max-norm/||g||;
    non-finite gradient -> error."""
    norm = global_norm(grads)
    if not np.isfinite(norm):
        raise FloatingPointError("non-finite gradient (SPEC.md:488)")
    s = max_norm / norm if norm > max_norm else 1.0
    return [np.asarray(g, dtype=np.float64) * s for g in grads], norm


def adamw_step(w, g, m, v, step: int, lr=DEFAULTS["lr"], weight_decay=DEFAULTS["weight_decay"],
               beta1=DEFAULTS["beta1"], beta2=DEFAULTS["beta2"], eps=DEFAULTS["eps"]):
    """decoupled weight decay (w <- w - lr*wd*w), then the Adam
    moment update with bias correction.  Returns (w', m', v')."""
    w, g, m, v = (np.asarray(a, dtype=np.float64) for a in (w, g, m, v))
    w = w - lr * weight_decay * w
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mh = m / (1.0 - beta1 ** step)
    vh = v / (1.0 - beta2 ** step)
    w = w - lr * mh / (np.sqrt(vh) + eps)
    return w, m, v


def accumulate(micro_grads, steps: int):
    """sum, then divide by accumulation-steps at flush;
    flush before any accumulation -> error."""
    if not micro_grads:
        raise RuntimeError("flush before any accumulation (SPEC.md:503)")
    acc = [np.zeros_like(np.asarray(g, dtype=np.float64)) for g in micro_grads[0]]
    for gs in micro_grads:
        for a, g in zip(acc, gs):
            a += np.asarray(g, dtype=np.float64)
    return [a / steps for a in acc]
