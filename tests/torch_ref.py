"""Plain-PyTorch fp32 reference of the MLP -> LM-Head block (test helper).

Two flavours:
  * exact=True  : everything in fp32 from the bf16 inputs (the math of
                  SPEC.md:197-232 / Alg. 1-4 without any intermediate rounding).
  * exact=False : rounds to bf16 exactly where libmst stores bf16 tensors
                  (h, O, dlogits, dO, dG, dU, dX) so only fp32 accumulation
                  order differs — the tight parity target.
Used only by tests (never by the product path).
"""
from __future__ import annotations

import torch


def _r(t: torch.Tensor, exact: bool) -> torch.Tensor:
    return t if exact else t.bfloat16().float()


def mlp_fwd(X, Wg, Wu, Wd, exact=False):
    X, Wg, Wu, Wd = (t.float() for t in (X, Wg, Wu, Wd))
    G = X @ Wg
    U = X @ Wu
    s = torch.sigmoid(G)
    h = _r((G * s) * U, exact)
    O = _r(h @ Wd, exact)
    return O, (G, U, h)


def mlp_bwd(dO, X, Wg, Wu, Wd, exact=False):
    X, Wg, Wu, Wd, dO = (t.float() for t in (X, Wg, Wu, Wd, dO))
    G = X @ Wg
    U = X @ Wu
    s = torch.sigmoid(G)
    act = G * s
    h = _r(act * U, exact)
    dh = dO @ Wd.t()
    dG = _r(dh * U * (s * (1 + G * (1 - s))), exact)
    dU = _r(dh * act, exact)
    dWd = h.t() @ dO
    dX = _r(dG @ Wg.t() + dU @ Wu.t(), exact)
    dWg = X.t() @ dG
    dWu = X.t() @ dU
    return dX, dWg, dWu, dWd


def head_fwd(X, L, Wout, chunks=None, mode=0):
    X, Wout = X.float(), Wout.float()
    Z = X @ Wout
    lse = torch.logsumexp(Z, dim=1)
    Ll = L.long()
    valid = (Ll >= 0) & (Ll < Z.shape[1])
    zt = torch.where(valid, Z.gather(1, Ll.clamp(0, Z.shape[1] - 1)[:, None])[:, 0], torch.zeros_like(lse))
    row = torch.where(valid, lse - zt, torch.zeros_like(lse))
    if mode == 0 or chunks is None:
        loss = row.sum() / valid.sum()
    else:
        means = [row[s:e].sum() / valid[s:e].sum() for s, e in chunks if valid[s:e].sum() > 0]
        loss = sum(means) / len(chunks)
    return loss, lse, row, valid


def head_bwd(X, L, Wout, scale_rows, exact=False):
    """dlogits = (softmax - onehot) * scale_row; returns dX, dWout, dl."""
    X, Wout = X.float(), Wout.float()
    Z = X @ Wout
    P = torch.softmax(Z, dim=1)
    Ll = L.long()
    valid = (Ll >= 0) & (Ll < Z.shape[1])
    onehot = torch.zeros_like(P)
    onehot[valid, Ll[valid]] = 1.0
    dl = _r((P - onehot) * scale_rows[:, None], exact)
    dX = _r(dl @ Wout.t(), exact)
    dWout = X.t() @ dl
    return dX, dWout, dl


def block(X, L, Wg, Wu, Wd, Wout, grad_loss=1.0, exact=False):
    O, _ = mlp_fwd(X, Wg, Wu, Wd, exact)
    loss, lse, _, valid = head_fwd(O, L, Wout)
    scale = torch.where(valid, torch.full_like(lse, grad_loss) / valid.sum(), torch.zeros_like(lse))
    dO, dWout, _ = head_bwd(O, L, Wout, scale, exact)
    dX, dWg, dWu, dWd = mlp_bwd(dO, X, Wg, Wu, Wd, exact)
    return dict(loss=loss, lse=lse, O=O, dO=dO, dX=dX, dWg=dWg, dWu=dWu, dWd=dWd, dWout=dWout)


def relerr(a: torch.Tensor, b: torch.Tensor) -> float:
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))
