"""Analytic predictions for the MsT path — the reference's `estimator`
module restricted to what this repository builds.

  intermediate_ratios(cfg)            Table 1 ratios
  predict_flops(d, I, V, S, M)        Thm 3.1 counts, M-independent
  predict_hbm(d, I, V, S, M)          Thm 3.2 element accesses
  predict_block_peak(N, H, I, V, M)   peak bytes of the GPU block step's chunk
                                      buffers per memtrack label class, exactly
                                      as libmst reports them (mst.h "memtrack"):
                                      the cross-check of predict_peak against
                                      tracked device allocations

Not reproduced: predict_peak's whole-model Appendix D rows (weights /
gradients / optimizer / activation for Llama3-8B, Tables 4-7) — those need
the full model's activation inventory under the paper's PyTorch allocator.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict


def intermediate_ratios(d: int, I: int, V: int, G: int) -> Dict[str, Fraction]:
    """Table 1 'Ratio Intermediate/Input': attention 1 + 2/G (the dimensionally
    consistent reading), MLP 2I/d, LM-Head V/d."""
    return {"attn": 1 + Fraction(2, G), "mlp": Fraction(2 * I, d), "head": Fraction(V, d)}


def predict_flops(d: int, I: int, V: int, S: int, M: int = 1, c: int = 5) -> Dict[str, int]:
    """mlp 6 S d I, head 2 S d V + c S V (c = 5, the memtrack
    cross-entropy convention); no M in the formula (Theorem 3.1)."""
    return {"mlp": 6 * S * d * I, "head": 2 * S * d * V + c * S * V}


def predict_hbm(d: int, I: int, V: int, S: int, M: int = 1) -> Dict[str, int]:
    """SPEC.md:566-573 (Theorem 3.2): mlp S d + S I + 3 d I M, head S d + S V + d V M
    element accesses; each extra mini-sequence re-reads the weights once."""
    return {"mlp": S * d + S * I + 3 * d * I * M, "head": S * d + S * V + d * V * M}


def _chunk(N: int, M: int) -> int:
    c = min(N, M)
    return -(-N // c)  # the longest chunk of the balanced plan (App. A-1)


def predict_block_peak(N: int, H: int, I: int, V: int, M: int, M_head: int | None = None) -> Dict[str, int]:
    """Peak live bytes per label class of one chunk-wise block step
    (mst_block_step; M_mlp = M, M_head = M unless given, head chunks nested in
    the MLP chunks), as the library's memtrack events report them: the MLP
    chunk buffers h (bf16), G and U (fp32, kept for the backward), dh (fp32),
    dG, dU, h^T (bf16) -> 20 n I bytes at their common peak; one LM-Head
    chunk's softmax numerators / dlogits (bf16) plus the per-256-column CE
    partials and two fp32 row scalars; the activations: one O chunk and two
    dO chunks of the MLP chunk length (bf16; dO_j is read by chunk j+1's
    dW_down GEMM) and the sequence-wide lse (fp32)."""
    n = _chunk(N, M)
    nh = _chunk(N, M if M_head is None else M_head)
    head = nh * V * 2 + nh * (-(-V // 256)) * 8 + nh * 8
    mlp = 20 * n * I
    # the head's chunk buffers coexist with the forward MLP buffers of the same chunk (h, G, U = 10 n I)
    inter = max(mlp, 10 * n * I + head)
    return {"inter.mlp.": mlp, "inter.head.": head, "inter.": inter, "act.O": n * H * 2, "act.dO": 2 * n * H * 2,
            "act.lse": N * 4}
