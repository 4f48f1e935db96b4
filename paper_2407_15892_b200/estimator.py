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

  predict_peak(cfg, S, B, M_mlp, M_head, recompute, in_backward, convention)
                                      SPEC.md:590-596 -> MemBreakdown:
                                      "paper"  the Appendix D convention (PAPER.md:665-777:
                                               bf16 weights / gradients / Adam moments, the
                                               HF-Llama saved-tensor inventory);
                                      "repo"   this repository's model.py + optim.AdamW
                                               (bf16 weights, fp32 gradients, fp32 master +
                                               moments, model.py's saved set, libmst's
                                               chunk workspace) -- cross-checked against
                                               tracked device allocations (tests/test_gpu_estimator.py)
"""
from __future__ import annotations

from dataclasses import dataclass, field
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


def _bounds(N: int, M: int):
    """Balanced chunk plan (make_chunk_plan): min(N, M)
    chunks, the first N mod M one row longer."""
    c = min(N, M)
    q, r = divmod(N, c)
    b = [0]
    for j in range(c):
        b.append(b[-1] + q + (1 if j < r else 0))
    return b


def predict_block_peak(N: int, H: int, I: int, V: int, M: int, M_head: int | None = None,
                       pair_dw: bool = True) -> Dict[str, int]:
    """Peak live bytes per label class of one chunk-wise block step
    (mst_block_step; M_mlp = M, M_head = M unless given, head chunks nested in
    the MLP chunks), as the library's memtrack events report them.  The
    events are replayed in the library's order (block_step_chunked in
    csrc/mst_api.cu), so ragged plans are exact too:

      K1(j)        + inter.mlp.{h (bf16), G, U (fp32)} of chunk j
      K2(j) launch - the dW operand sets whose K8 / K10 ran in it
      head chunk k + act.oT, inter.head.{partials, dlogits}, then - all three
      K7a(j)       + inter.mlp.dh (fp32); SwiGLU backward + inter.mlp.{dG, dU,
                   hT} and act.xT (the dW operand set of chunk j); - dh
      end of j     - h, G, U of chunk j; K1(j+1) + those of chunk j+1
      last launch  - the remaining dW operand sets

    With `pair_dw` (the library default, tuning "pair_dw") K8 / K10 run once
    per chunk pair, so the set of an even chunk stays live through the next
    chunk's head and MLP backward.  Fixed for the step: act.O (one MLP
    chunk), act.dO (two), act.lse (sequence-wide, fp32)."""
    MH = M if M_head is None else M_head
    b, bh = _bounds(N, M), _bounds(N, MH)
    nch = len(b) - 1
    nparts = -(-V // 256)
    n = _chunk(N, M)
    live: Dict[str, int] = {}
    peaks: Dict[str, int] = {}
    prefixes = ("inter.mlp.", "inter.head.", "inter.", "act.O", "act.dO", "act.lse", "act.xT", "act.oT")

    def ev(label: str, nbytes: int):
        live[label] = live.get(label, 0) + nbytes
        for p in prefixes:
            if label.startswith(p):
                peaks[p] = max(peaks.get(p, 0), sum(v for k, v in live.items() if k.startswith(p)))

    def rows(j):
        return b[j + 1] - b[j]

    def mlp_fwd(j, on):
        s = 1 if on else -1
        for lab, eb in (("inter.mlp.h", 2), ("inter.mlp.G", 4), ("inter.mlp.U", 4)):
            ev(lab, s * rows(j) * I * eb)

    def grads(j, on):
        s = 1 if on else -1
        for lab in ("inter.mlp.dG", "inter.mlp.dU", "inter.mlp.hT"):
            ev(lab, s * rows(j) * I * 2)
        ev("act.xT", s * rows(j) * H * 2)

    pair = pair_dw and nch > 1
    ev("act.O", n * H * 2)
    ev("act.dO", 2 * n * H * 2)
    ev("act.lse", N * 4)
    mlp_fwd(0, True)
    for j in range(nch):
        if j > 0:  # K2(j) launch: K8 / K10 of chunk j-1, or of the pair (j-2, j-1)
            if not pair:
                grads(j - 1, False)
            elif (j - 1) & 1:
                grads(j - 2, False)
                grads(j - 1, False)
        for k in range(len(bh) - 1):
            if not (b[j] <= bh[k] < b[j + 1]):
                continue
            hr = bh[k + 1] - bh[k]
            ev("act.oT", hr * H * 2)
            ev("inter.head.partials", hr * nparts * 8 + hr * 8)
            ev("inter.head.dlogits", hr * V * 2)
            ev("inter.head.dlogits", -hr * V * 2)
            ev("inter.head.partials", -(hr * nparts * 8 + hr * 8))
            ev("act.oT", -hr * H * 2)
        ev("inter.mlp.dh", rows(j) * I * 4)
        grads(j, True)
        ev("inter.mlp.dh", -rows(j) * I * 4)
        mlp_fwd(j, False)
        if j + 1 < nch:
            mlp_fwd(j + 1, True)
    return {"inter.mlp.": peaks["inter.mlp."], "inter.head.": peaks["inter.head."], "inter.": peaks["inter."],
            "act.O": peaks["act.O"], "act.dO": peaks["act.dO"], "act.lse": peaks["act.lse"],
            "act.xT": peaks["act.xT"]}


# ------------------------------------------------------------------ predict_peak
@dataclass
class MemBreakdown:
    """bytes per component at the predicted peak; formulas
    recorded as strings for the report.  total == sum of the components."""
    weights: int
    gradients: int
    optimizer: int
    activation: int
    peak_intermediate: int
    phase: str = ""
    formulas: Dict[str, str] = field(default_factory=dict)

    def __post_init__(self):
        for k in ("weights", "gradients", "optimizer", "activation", "peak_intermediate"):
            if getattr(self, k) < 0:
                raise ValueError(f"{k} < 0")

    @property
    def total(self) -> int:
        return self.weights + self.gradients + self.optimizer + self.activation + self.peak_intermediate

    def rows(self, unit: float = 2 ** 30) -> Dict[str, float]:
        """The `estimate` report rows: weights, gradients,
        optimizer, activation, peak-intermediate, total (GiB by default, the
        unit of Appendix D's "GB")."""
        return {k: getattr(self, k) / unit for k in ("weights", "gradients", "optimizer", "activation",
                                                     "peak_intermediate", "total")}


def param_counts(d: int, I: int, V: int, heads: int, G: int, layers: int) -> Dict[str, int]:
    """Parameters of the Llama-style decoder: untied
    embedding and W_out, per layer W_qkv [d, d + 2d/G], W_o, three MLP
    matrices, two RMSNorm gains; the final gain."""
    kv = d // G
    mats = V * d + layers * (d * (d + 2 * kv) + d * d + 3 * d * I) + d * V
    gains = layers * 2 * d + d
    return {"matrices": mats, "gains": gains, "total": mats + gains}


def _paper_activation(d, I, V, G, L, N, M_mlp, M_head, recompute) -> Dict[str, int]:
    """Appendix D's activation (bf16, HF Llama with FlashAttention2): per layer
    the saved tensors 11 N d (two fp32 RMSNorm inputs counted double, their
    outputs, q/k/v incl. the pre-rotary copies, attention output) + 4 N I
    (the MLP input products G, silu(G), U, h) elements; the head keeps bf16
    logits, their fp32 copy and the fp32 log-softmax: N V (2 + 4 + 4) bytes.
    Recompute keeps one N d layer input per layer and rebuilds one layer at a
    time; MsT divides the MLP and head intermediates by M_mlp / M_head."""
    layer_d, layer_i = 11 * N * d * 2, 4 * N * I * 2
    head = N * V * 10
    if not recompute:
        return {"saved": L * (layer_d + layer_i), "inter": head}
    return {"saved": L * N * d * 2, "inter": layer_d + layer_i // M_mlp + head // M_head}


def _repo_activation(d, I, V, G, L, N, M_mlp, M_head, recompute, heads=1) -> Dict[str, int]:
    """model.py's saved set (bf16 unless noted): per layer the residual sum xs,
    and unless per-layer recompute: a = rmsnorm(xs), qkv [N, d + 2d/G], the
    attention output o and its fp32 log-sum-exp per head, x2, b = rmsnorm(x2)
    and two fp32 rstd rows; then the
    final norm's input / rstd, the head-input gradient dF, the LM-Head lse and
    the int32 tokens / labels.  Intermediates: libmst's persistent context
    workspace (the largest of the MLP and LM-Head chunk workspaces) plus one
    layer's transient backward buffers (dqkv, da, do, db, dx, the attention
    gradients) -- and with recompute the rebuilt layer's saved set."""
    from . import miniseq as ms

    kv = d // G
    per_layer_full = N * (6 * d + 2 * kv) * 2 + 8 * N + 4 * N * heads
    saved = L * (N * d * 2 if recompute else per_layer_full) + N * d * 2 * 3 + 4 * N * 2 + 8 * N
    lib = ms.load_library()
    import ctypes

    a, b = ctypes.c_size_t(), ctypes.c_size_t()
    ms._check(lib.mst_mlp_workspace(N, d, I, M_mlp, ctypes.byref(a)))
    ms._check(lib.mst_lmhead_workspace(N, d, V, M_head, ctypes.byref(b)))
    ws = max(a.value, b.value)
    transient = N * (d + 2 * kv) * 2 * 2 + N * d * 2 * 4
    return {"saved": saved, "inter": ws + transient + (per_layer_full if recompute else 0)}


def predict_peak(d: int, I: int, V: int, heads: int, G: int, layers: int, S: int, B: int = 1, M_mlp: int = 1,
                 M_head: int = 1, recompute: bool = False, in_backward: bool = False,
                 convention: str = "paper") -> MemBreakdown:
    """predict_peak: the larger of two phases --
    (A) the end of the forward / the backward: weights + optimizer state +
        activations + the peak intermediate (+ the fp32 gradients already
        produced, "repo" convention: model.py keeps every gradient until the
        optimizer step);
    (B) the optimizer step (absent with optimizer-in-backward): weights +
        gradients + optimizer state + the optimizer's intermediate.
    "paper": Appendix D: bf16 weights (2 B/param),
    gradients (2 B), Adam moments (2 x 2 B) plus a weight-sized optimizer
    intermediate; Llama3-8B / S=4096 gives 75 (vanilla), 74 (in-backward),
    52 (recompute) GiB.  "repo": bf16 weights + fp32 gains, fp32 gradients,
    AdamW fp32 master + moments (12 B/param, no intermediate: the update is
    one fused kernel)."""
    if convention not in ("paper", "repo"):
        raise ValueError("convention is 'paper' or 'repo'")
    N = S * B
    P = param_counts(d, I, V, heads, G, layers)
    if convention == "paper":
        act = _paper_activation(d, I, V, G, layers, N, M_mlp, M_head, recompute)
    else:
        act = _repo_activation(d, I, V, G, layers, N, M_mlp, M_head, recompute, heads)
    if convention == "paper":
        w = 2 * P["total"]
        g = 2 * P["total"]
        opt_state, opt_inter = 4 * P["total"], 2 * P["total"]
        grads_in_a = 0
        f = {"weights": "2 B x params", "gradients": "2 B x params (0 with optimizer-in-backward)",
             "optimizer": "Adam moments 2 x 2 B x params (+ 2 B x params intermediate at the step)",
             "activation": "per layer 11 N d + 4 N I bf16 elements; recompute: N d per layer",
             "peak_intermediate": "head N V (2+4+4) B / M_head; recompute: one layer's set, MLP part / M_mlp"}
    else:
        w = 2 * P["matrices"] + 4 * P["gains"]
        g = 4 * P["total"]
        opt_state, opt_inter = 12 * P["matrices"] + 8 * P["gains"], 0
        grads_in_a = 0 if in_backward else g
        f = {"weights": "2 B x matrix params + 4 B x gains", "gradients": "4 B x params (fp32)",
             "optimizer": "AdamW fp32 master + m + v (12 B / matrix param, 8 B / gain)",
             "activation": "model.py saved set: per layer N(6d + 2d/G) bf16 + 8N; recompute: N d per layer",
             "peak_intermediate": "libmst chunk workspace max(MLP, head) + one layer's backward buffers"}
    phase_a = w + opt_state + act["saved"] + act["inter"] + grads_in_a
    phase_b = -1 if in_backward else w + g + opt_state + opt_inter
    if phase_b > phase_a:
        return MemBreakdown(w, g, opt_state + opt_inter, 0, 0, "optimizer step", f)
    return MemBreakdown(w, grads_in_a, opt_state, act["saved"], act["inter"], "forward/backward", f)
