"""Llama-style decoder around the MsT blocks — the reference's `model` module
 on the B200 path (the real caller of
the hot path).

  embedding -> L x [RMSNorm, causal GQA attention, residual, RMSNorm, MLP,
  residual] -> final RMSNorm -> LM-Head + cross-entropy

with swappable standard (M = 1) / mini-sequence (M > 1) MLP and LM-Head
blocks (`ModelConfig.M_mlp`, `M_head`) and the per-layer
recompute policy (`recompute`).

Where the arithmetic runs:
  * MLP blocks, LM-Head + CE: libmst's MsT kernels (miniseq.py);
  * QKV / output projections and their gradients: libmst's tcgen05 GEMM
    engine (mst_gemm); Q, K, V come out of one fused [d, d + 2 d/G] weight;
  * RMSNorm (+ fused residual add) forward/backward, embedding gather /
    deterministic grouped scatter: libmst's HBM-bound kernels (csrc/layers.cu);
  * causal grouped-query attention: libmst's tcgen05 attention kernels
    (csrc/attention.cu, attention.py: forward with online softmax saving one
    fp32 log-sum-exp per row and head, deterministic dK/dV and dQ backward
    kernels), reading q / k / v as column slices of the fused qkv buffer and
    writing dq / dk / dv into one d qkv buffer; the backward never re-runs
    the forward (the paper uses FlashAttention2).
bf16 activations, fp32 accumulation, fp32 weight gradients (and RMSNorm
gains), token-weighted mean loss over non-ignored labels (-100).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch

from . import miniseq as ms
from .attention import attention_backward, attention_forward
from .memtrack import MemTracker  # noqa: F401  (re-exported for callers)


@dataclass
class ModelConfig:
    d: int = 64
    I: int = 224
    V: int = 2048
    heads: int = 4
    G: int = 2            # query groups: K and V have d / G columns (Table 1 "2 x (B,S,d/G)")
    layers: int = 2
    S: int = 256
    B: int = 1
    M_mlp: int = 1
    M_head: int = 1
    recompute: bool = False
    seed: int = 0
    eps: float = 1e-5

    @property
    def kv(self) -> int:
        return self.d // self.G

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    def validate(self) -> None:
        for k in ("d", "I", "V", "heads", "G", "S", "B", "M_mlp", "M_head"):
            if getattr(self, k) < 1:
                raise ms.ConfigError(f"{k} must be >= 1 (SPEC.md:416)")
        if self.layers < 0:
            raise ms.ConfigError("layers must be >= 0")
        if self.d % self.heads or self.heads % self.G:
            raise ms.ConfigError("d % heads == 0 and heads % G == 0 required (SPEC.md:416)")
        if self.d % 8 or self.I % 8 or self.V % 8 or self.kv % 8:
            raise ms.ShapeError("d, I, V and d/G must be multiples of 8 (16-byte TMA rows)")


@dataclass
class LayerWeights:
    W_qkv: torch.Tensor   # [d, d + 2 d/G] bf16: W_q | W_k | W_v (X W orientation)
    W_o: torch.Tensor     # [d, d] bf16
    g_attn: torch.Tensor  # [d] fp32 RMSNorm gain
    g_mlp: torch.Tensor   # [d] fp32
    W_gate: torch.Tensor  # [d, I] bf16
    W_up: torch.Tensor    # [d, I]
    W_down: torch.Tensor  # [I, d]

    def named(self, prefix: str) -> Dict[str, torch.Tensor]:
        return {f"{prefix}.{k}": getattr(self, k) for k in ("W_qkv", "W_o", "g_attn", "g_mlp", "W_gate", "W_up",
                                                             "W_down")}


@dataclass
class ModelWeights:
    embedding: torch.Tensor  # [V, d] bf16 (untied from W_out)
    layers: List[LayerWeights]
    g_final: torch.Tensor    # [d] fp32
    W_out: torch.Tensor      # [d, V] bf16

    def named(self) -> Dict[str, torch.Tensor]:
        out = {"embedding": self.embedding}
        for i, l in enumerate(self.layers):
            out.update(l.named(f"layers.{i}"))
        out.update({"g_final": self.g_final, "W_out": self.W_out})
        return out


def _fnv1a64(s: str) -> int:
    h = 0xcbf29ce484222325
    for b in s.encode():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def init_weights(cfg: ModelConfig, device="cuda") -> ModelWeights:
    """deterministic seeded init, N(0, 0.02^2) matrices, unit
    gains; every parameter draws from its own sub-seed (seed ^ fnv1a(name)),
    so adding layers does not perturb earlier ones."""
    cfg.validate()

    def normal(name, *shape):
        g = torch.Generator(device="cpu").manual_seed((cfg.seed ^ _fnv1a64(name)) & 0x7FFFFFFFFFFFFFFF)
        return (0.02 * torch.randn(*shape, generator=g)).to(device=device, dtype=torch.bfloat16)

    ones = lambda: torch.ones(cfg.d, device=device, dtype=torch.float32)  # noqa: E731
    layers = []
    for i in range(cfg.layers):
        p = f"layers.{i}"
        layers.append(LayerWeights(W_qkv=normal(f"{p}.W_qkv", cfg.d, cfg.d + 2 * cfg.kv),
                                   W_o=normal(f"{p}.W_o", cfg.d, cfg.d), g_attn=ones(), g_mlp=ones(),
                                   W_gate=normal(f"{p}.W_gate", cfg.d, cfg.I), W_up=normal(f"{p}.W_up", cfg.d, cfg.I),
                                   W_down=normal(f"{p}.W_down", cfg.I, cfg.d)))
    return ModelWeights(embedding=normal("embedding", cfg.V, cfg.d), layers=layers, g_final=ones(),
                        W_out=normal("W_out", cfg.d, cfg.V))


# ------------------------------------------------------------------ libmst ops
def _ctx(t):
    return ms.Context.get(t.device.index)


def gemm(A: torch.Tensor, B: torch.Tensor, M: int, N: int, K: int, a_mn: bool, b_mn: bool,
         out: torch.Tensor, beta: int = 0) -> torch.Tensor:
    """out[M,N] (+)= A B on the tcgen05 engine (mst_gemm; operand layouts as mst_debug_gemm)."""
    ctx = _ctx(A)
    ms._check(ctx.lib.mst_gemm(ctx.handle, ms._stream(A), A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K,
                               int(a_mn), int(b_mn), int(out.dtype == torch.float32), int(beta)))
    return out


def rmsnorm_forward(x: torch.Tensor, gain: torch.Tensor, eps: float, residual: Optional[torch.Tensor] = None):
    """(y, s, rstd): s = x (+ residual) in bf16, y = rmsnorm(s) * gain."""
    ctx = _ctx(x)
    n, d = x.shape
    y = torch.empty_like(x)
    s = torch.empty_like(x) if residual is not None else x
    rstd = torch.empty(n, device=x.device, dtype=torch.float32)
    ms._check(ctx.lib.mst_rmsnorm_forward(ctx.handle, ms._stream(x), x.data_ptr(), ms._ptr(residual), gain.data_ptr(),
                                          y.data_ptr(), s.data_ptr() if residual is not None else None,
                                          rstd.data_ptr(), n, d, float(eps)))
    return y, s, rstd


def rmsnorm_backward(s: torch.Tensor, gain: torch.Tensor, rstd: torch.Tensor, dy: torch.Tensor,
                     dres: Optional[torch.Tensor], dgain: torch.Tensor, accumulate: bool) -> torch.Tensor:
    ctx = _ctx(s)
    n, d = s.shape
    nb = ctypes.c_size_t()
    ms._check(ctx.lib.mst_rmsnorm_workspace(ctx.handle, n, d, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    dx = torch.empty_like(s)
    ms._check(ctx.lib.mst_rmsnorm_backward(ctx.handle, ms._stream(s), s.data_ptr(), gain.data_ptr(), rstd.data_ptr(),
                                           dy.data_ptr(), ms._ptr(dres), dx.data_ptr(), dgain.data_ptr(),
                                           int(accumulate), n, d, ws.data_ptr(), ws.numel()))
    return dx


def embedding_forward(table: torch.Tensor, tokens: torch.Tensor) -> torch.Tensor:
    ctx = _ctx(table)
    V, d = table.shape
    n = tokens.numel()
    out = torch.empty(n, d, device=table.device, dtype=table.dtype)
    bad = torch.empty(1, device=table.device, dtype=torch.int32)
    ms._check(ctx.lib.mst_embedding_forward(ctx.handle, ms._stream(table), table.data_ptr(), tokens.data_ptr(),
                                            out.data_ptr(), n, d, V, bad.data_ptr()))
    return out, bad


def embedding_backward(tokens: torch.Tensor, dx: torch.Tensor, dtable: torch.Tensor, accumulate: bool) -> None:
    """Deterministic: positions grouped by token (stable sort) and summed in
    position order per token."""
    ctx = _ctx(dx)
    V, d = dtable.shape
    t = tokens.reshape(-1).long()
    order = torch.sort(t, stable=True).indices.to(torch.int32)
    uniq, counts = torch.unique_consecutive(t[order.long()], return_counts=True)
    seg = torch.zeros(uniq.numel() + 1, device=dx.device, dtype=torch.int32)
    seg[1:] = torch.cumsum(counts, 0).to(torch.int32)
    u32 = uniq.to(torch.int32)
    ms._check(ctx.lib.mst_embedding_backward(ctx.handle, ms._stream(dx), order.data_ptr(), seg.data_ptr(),
                                             u32.data_ptr(), uniq.numel(), dx.data_ptr(), dtable.data_ptr(), d, V,
                                             int(accumulate)))


# ------------------------------------------------------------------ the model
@dataclass
class _LayerSaved:
    x: torch.Tensor                      # layer input (residual stream)
    a: Optional[torch.Tensor] = None     # rmsnorm_attn(x)
    rstd1: Optional[torch.Tensor] = None
    qkv: Optional[torch.Tensor] = None
    o: Optional[torch.Tensor] = None     # attention output [N, d] (before W_o)
    lse: Optional[torch.Tensor] = None   # attention log-sum-exp [B, heads, S] (fp32)
    attn_graph: Optional[tuple] = None   # Ulysses: (o with its autograd graph, (q, k, v) leaves)
    x2: Optional[torch.Tensor] = None    # x + attn
    b: Optional[torch.Tensor] = None     # rmsnorm_mlp(x2)
    rstd2: Optional[torch.Tensor] = None
    mlp_saved: Optional[ms.MlpSaved] = None
    m: Optional[torch.Tensor] = None     # MLP output


@dataclass
class Saved:
    tokens: torch.Tensor
    layers: List[_LayerSaved]
    x_last: torch.Tensor
    rstd_f: torch.Tensor
    dF: torch.Tensor                     # LM-Head input gradient (single-pass head)
    dW_out: torch.Tensor
    stats: torch.Tensor
    loss: torch.Tensor


class Model:
    """forward / backward of SPEC.md:430-451 over libmst kernels.

    group: a torch.distributed process group over which ONE sequence is
    sharded (Ulysses sequence parallelism, ulysses.py): cfg.S is then this
    rank's shard length (B must be 1), attention re-shards to heads with
    all-to-alls, the LM-Head uses the global valid-label count, the loss is
    the global token-weighted mean and backward() returns SUM-all-reduced
    weight gradients."""

    def __init__(self, cfg: ModelConfig, weights: Optional[ModelWeights] = None, device="cuda", group=None):
        cfg.validate()
        self.cfg = cfg
        self.w = weights if weights is not None else init_weights(cfg, device)
        self.group = group
        self.world = 1
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
            if self.world > 1 and cfg.B != 1:
                raise ms.ConfigError("sequence parallelism shards one sequence: B must be 1")

    # ---------------------------------------------------------------- attention
    def _attention(self, qkv: torch.Tensor):
        """Causal GQA over qkv [N, d + 2d/G] -> (o [N, d], lse, graph).
        One rank: libmst's kernel on the qkv column slices (lse saved for the
        backward).  Sequence-parallel: Ulysses all-to-alls around the same
        kernel under autograd; the graph is kept for the backward (no re-run)."""
        cfg = self.cfg
        h, kvh = cfg.heads, cfg.heads // cfg.G
        q, k, v = qkv[:, :cfg.d], qkv[:, cfg.d:cfg.d + cfg.kv], qkv[:, cfg.d + cfg.kv:]
        if self.world > 1:
            from . import ulysses

            q, k, v = (t.contiguous().requires_grad_(True) for t in (q, k, v))
            with torch.enable_grad():
                o = ulysses.attention(q, k, v, h, kvh, self.group)
            return o.detach().contiguous(), None, (o, (q, k, v))
        o, lse = attention_forward(q, k, v, cfg.B, cfg.S, h, kvh)
        return o, lse, None

    def _attention_backward(self, qkv: torch.Tensor, o: torch.Tensor, lse, graph, do: torch.Tensor) -> torch.Tensor:
        """d qkv [N, d + 2d/G] of the attention (dq | dk | dv written in place)."""
        cfg = self.cfg
        if graph is not None:  # Ulysses: backward through the saved graph (transposed all-to-alls)
            o_g, (q, k, v) = graph
            o_g.backward(do)
            return torch.cat([q.grad, k.grad, v.grad], dim=1)
        d, kv = cfg.d, cfg.kv
        dqkv = torch.empty_like(qkv)
        attention_backward(qkv[:, :d], qkv[:, d:d + kv], qkv[:, d + kv:], o, do, lse, cfg.B, cfg.S, cfg.heads,
                           cfg.heads // cfg.G, dq=dqkv[:, :d], dk=dqkv[:, d:d + kv], dv=dqkv[:, d + kv:])
        return dqkv

    # ---------------------------------------------------------------- forward
    def _layer_forward(self, lw: LayerWeights, x: torch.Tensor, resid: Optional[torch.Tensor]):
        """x: previous MLP output (or the embedding when resid is None), resid: the
        residual stream it is added to.  Returns (saved, m, x2) with the layer's
        own output = x2 + m (added by the next rmsnorm)."""
        cfg = self.cfg
        N = cfg.B * cfg.S
        a, xs, rstd1 = rmsnorm_forward(x, lw.g_attn, cfg.eps, residual=resid)
        qkv = torch.empty(N, cfg.d + 2 * cfg.kv, device=x.device, dtype=torch.bfloat16)
        gemm(a, lw.W_qkv, N, cfg.d + 2 * cfg.kv, cfg.d, False, True, qkv)
        o, lse, graph = self._attention(qkv)
        ao = torch.empty_like(o)
        gemm(o, lw.W_o, N, cfg.d, cfg.d, False, True, ao)
        b, x2, rstd2 = rmsnorm_forward(ao, lw.g_mlp, cfg.eps, residual=xs)
        m, msaved = ms.miniseq_mlp_forward(b, ms.MlpWeights(lw.W_gate, lw.W_up, lw.W_down),
                                           ms.make_chunk_plan(N, cfg.M_mlp))
        sv = _LayerSaved(x=xs)
        if not cfg.recompute:
            sv.a, sv.rstd1, sv.qkv, sv.o, sv.x2, sv.b, sv.rstd2, sv.mlp_saved = a, rstd1, qkv, o, x2, b, rstd2, msaved
            sv.lse, sv.attn_graph = lse, graph
        return sv, m, x2

    def forward(self, tokens: torch.Tensor, labels: torch.Tensor, check: bool = True):
        """(loss, saved) — SPEC.md:430-437.  The LM-Head runs single-pass
        (forward + backward of the head in one chunk loop), so saved holds the
        head-input gradient and dW_out for backward()."""
        cfg = self.cfg
        if tokens.shape != (cfg.B, cfg.S) or labels.shape != (cfg.B, cfg.S):
            raise ms.ShapeError(f"tokens/labels must be [{cfg.B}, {cfg.S}]")
        N = cfg.B * cfg.S
        tok = tokens.reshape(-1).to(torch.int32).contiguous()
        lab = labels.reshape(-1).to(torch.int32).contiguous()
        x, bad = embedding_forward(self.w.embedding, tok)
        if check and int(bad.item()):
            raise ms.DataError(f"{int(bad.item())} tokens outside [0, V) (SPEC.md:437)")
        saved_layers = []
        resid = None
        for lw in self.w.layers:
            sv, m, x2 = self._layer_forward(lw, x, resid)
            saved_layers.append(sv)
            x, resid = m, x2
        f, x_last, rstd_f = rmsnorm_forward(x, self.w.g_final, cfg.eps, residual=resid)
        dW_out = torch.empty(cfg.d, cfg.V, device=f.device, dtype=torch.float32)
        gv = None
        if self.world > 1:  # token-weighted loss over the whole sequence
            gv = ms.count_valid(lab, cfg.V)
            self._all_reduce(gv)
        loss, stats, _, dF, _ = ms.miniseq_lmhead_fused(f, lab, ms.LmHeadWeights(self.w.W_out),
                                                        ms.make_chunk_plan(N, cfg.M_head), dW_out=dW_out,
                                                        global_valid=gv)
        if self.world > 1:
            pair = stats[:2].clone()
            self._all_reduce(pair)
            stats = stats.clone()
            stats[:2] = pair
            loss = pair[0] / pair[1]
        if check:
            s = stats[:4].tolist()
            if s[1] == 0:
                raise ms.DataError("all labels ignored (SPEC.md:219)")
            if s[3] > 0:
                raise ms.DataError(f"{int(s[3])} labels outside [0, V) and != -100")
        return loss, Saved(tok, saved_layers, x_last, rstd_f, dF, dW_out, stats, loss)

    # ---------------------------------------------------------------- backward
    def backward(self, saved: Saved) -> Dict[str, torch.Tensor]:
        """GradSet of every parameter: fp32 tensors keyed as
        ModelWeights.named()."""
        cfg = self.cfg
        N = cfg.B * cfg.S
        grads: Dict[str, torch.Tensor] = {"W_out": saved.dW_out}
        g_final = torch.empty(cfg.d, device=saved.dF.device, dtype=torch.float32)
        # d(layer-L output): rmsnorm_final backward; the residual stream carries it on
        dx = rmsnorm_backward(saved.x_last, self.w.g_final, saved.rstd_f, saved.dF, None, g_final, False)
        grads["g_final"] = g_final
        for li in range(cfg.layers - 1, -1, -1):
            lw, sv = self.w.layers[li], saved.layers[li]
            dx = self._layer_backward(li, lw, sv, dx, grads)
        dE = torch.empty(cfg.V, cfg.d, device=dx.device, dtype=torch.float32)
        embedding_backward(saved.tokens, dx, dE, accumulate=False)
        grads["embedding"] = dE
        if self.world > 1:
            from . import ulysses

            ulysses.all_reduce_grads(grads, self.group)
        return grads

    def _all_reduce(self, t: torch.Tensor) -> None:
        import torch.distributed as dist

        if dist.get_backend(self.group) == "gloo" and t.is_cuda:
            c = t.cpu()
            dist.all_reduce(c, group=self.group)
            t.copy_(c)
        else:
            dist.all_reduce(t, group=self.group)

    def _layer_backward(self, li: int, lw: LayerWeights, sv: _LayerSaved, dx3: torch.Tensor, grads) -> torch.Tensor:
        cfg = self.cfg
        N = cfg.B * cfg.S
        p = f"layers.{li}"
        if cfg.recompute:  # per-layer checkpoint: rebuild the layer's activations from its input
            a, _, rstd1 = rmsnorm_forward(sv.x, lw.g_attn, cfg.eps)
            qkv = torch.empty(N, cfg.d + 2 * cfg.kv, device=a.device, dtype=torch.bfloat16)
            gemm(a, lw.W_qkv, N, cfg.d + 2 * cfg.kv, cfg.d, False, True, qkv)
            o, lse, graph = self._attention(qkv)  # part of the per-layer recompute policy
            ao = torch.empty_like(o)
            gemm(o, lw.W_o, N, cfg.d, cfg.d, False, True, ao)
            b, x2, rstd2 = rmsnorm_forward(ao, lw.g_mlp, cfg.eps, residual=sv.x)
            _, msaved = ms.miniseq_mlp_forward(b, ms.MlpWeights(lw.W_gate, lw.W_up, lw.W_down),
                                               ms.make_chunk_plan(N, cfg.M_mlp))
        else:
            a, rstd1, qkv, o, x2, b, rstd2, msaved = sv.a, sv.rstd1, sv.qkv, sv.o, sv.x2, sv.b, sv.rstd2, sv.mlp_saved
            lse, graph = sv.lse, sv.attn_graph
        mg = ms.MlpGrads(torch.empty(cfg.d, cfg.I, device=a.device), torch.empty(cfg.d, cfg.I, device=a.device),
                         torch.empty(cfg.I, cfg.d, device=a.device))
        db, _ = ms.miniseq_mlp_backward(dx3, msaved, ms.MlpWeights(lw.W_gate, lw.W_up, lw.W_down),
                                        ms.make_chunk_plan(N, cfg.M_mlp), grads=mg)
        grads[f"{p}.W_gate"], grads[f"{p}.W_up"], grads[f"{p}.W_down"] = mg.W_gate, mg.W_up, mg.W_down
        g2 = torch.empty(cfg.d, device=a.device, dtype=torch.float32)
        dx2 = rmsnorm_backward(x2, lw.g_mlp, rstd2, db, dx3, g2, False)   # residual: dx2 = dx3 + d(norm)
        grads[f"{p}.g_mlp"] = g2
        # output projection: ao = o W_o
        dWo = torch.empty(cfg.d, cfg.d, device=a.device, dtype=torch.float32)
        gemm(o, dx2, cfg.d, cfg.d, N, True, True, dWo)                    # o^T dx2
        grads[f"{p}.W_o"] = dWo
        do = torch.empty_like(o)
        gemm(dx2, lw.W_o, N, cfg.d, cfg.d, False, False, do)              # dx2 W_o^T
        # attention backward (libmst kernels from the saved lse; Ulysses all-to-alls when sharded)
        dqkv = self._attention_backward(qkv, o, lse, graph, do)
        dWqkv = torch.empty(cfg.d, cfg.d + 2 * cfg.kv, device=a.device, dtype=torch.float32)
        gemm(a, dqkv, cfg.d, cfg.d + 2 * cfg.kv, N, True, True, dWqkv)    # a^T dqkv
        grads[f"{p}.W_qkv"] = dWqkv
        da = torch.empty_like(a)
        gemm(dqkv, lw.W_qkv, N, cfg.d, cfg.d + 2 * cfg.kv, False, False, da)  # dqkv W_qkv^T
        g1 = torch.empty(cfg.d, device=a.device, dtype=torch.float32)
        dx = rmsnorm_backward(sv.x, lw.g_attn, rstd1, da, dx2, g1, False)
        grads[f"{p}.g_attn"] = g1
        return dx

    def train_step(self, tokens, labels, opt=None):
        loss, saved = self.forward(tokens, labels)
        grads = self.backward(saved)
        if opt is not None:
            opt.step(grads)
        return loss, grads
