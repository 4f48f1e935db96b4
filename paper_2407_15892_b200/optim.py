"""The reference's `optim` module on the B200 path.

AdamW with global-norm gradient clipping, micro-batch gradient accumulation
and an optimizer-in-backward mode, over the MsT block's parameters.  The
arithmetic runs in libmst's HBM-bound kernels (csrc/optim.cu, C ABI
`mst_adamw_step`, `mst_grad_sumsq`, `mst_grad_accumulate`); this module is
the host-side mirror of the SPEC operations:

  clip_global_norm(grads, max_norm)
  adamw_step(params, grads, state, cfg)
  accumulate(into, from_, ...) / GradAccumulator
  step_in_backward(name, state, cfg)

Parameters keep an fp32 master copy and fp32 moments (Appendix D: "optimizer
would take 2x of weights when using Adam"); the bf16 tensor the GEMMs read
is rewritten by the same kernel.  Gradients are the fp32 dW accumulators of
`miniseq.block_step`.  The clip factor and the 1/steps of accumulation are a
device scalar folded into the AdamW kernel, so a step needs no host sync
unless the caller asks for the norm.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Dict, Iterable, Optional, Tuple

import torch

from . import miniseq as ms


@dataclass
class OptimConfig:
    lr: float = 1e-4
    weight_decay: float = 0.001
    clip_norm: float = 1.0
    betas: Tuple[float, float] = (0.9, 0.999)
    eps: float = 1e-8
    accumulation_steps: int = 1
    in_backward: bool = False

    def validate(self) -> None:
        if not self.lr > 0:
            raise ms.ConfigError("lr must be > 0 (SPEC.md:478)")
        if not self.clip_norm > 0:
            raise ms.ConfigError("clip-norm must be > 0 (SPEC.md:478)")
        if not all(0 < b < 1 for b in self.betas):
            raise ms.ConfigError("betas must lie in (0, 1) (SPEC.md:478)")
        if self.accumulation_steps < 1:
            raise ms.ConfigError("accumulation-steps must be >= 1")

    def _c(self) -> "ms._AdamCfg":
        return ms._AdamCfg(self.lr, self.weight_decay, self.betas[0], self.betas[1], self.eps)


_GRAD_READY = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


def _lib():
    return ms.load_library()


def _ctx(t: torch.Tensor) -> ms.Context:
    return ms.Context.get(t.device.index)


@dataclass
class ParamState:  # one parameter's slice of OptimState
    weight: torch.Tensor          # bf16 model copy (read by the GEMMs, rewritten by each step)
    master: torch.Tensor          # fp32
    m: torch.Tensor               # fp32 first moment
    v: torch.Tensor               # fp32 second moment
    stepped: bool = False         # stepped in the current backward (in-backward mode)


@dataclass
class OptimState:
    params: Dict[str, ParamState] = field(default_factory=dict)
    step: int = 0

    @staticmethod
    def create(weights: Dict[str, torch.Tensor]) -> "OptimState":
        st = OptimState()
        for k, w in weights.items():
            if w.dtype not in (torch.bfloat16, torch.float32) or not w.is_cuda or not w.is_contiguous():
                raise ms.DtypeError(f"{k}: parameters are contiguous bf16 or fp32 CUDA tensors")
            if w.dtype == torch.float32:  # fp32 parameter (e.g. RMSNorm gains): it is its own master copy
                st.params[k] = ParamState(torch.empty(w.shape, device=w.device, dtype=torch.bfloat16), w,
                                          torch.zeros(w.shape, device=w.device), torch.zeros(w.shape, device=w.device))
            else:
                st.params[k] = ParamState(w, w.float().contiguous(), torch.zeros(w.shape, device=w.device),
                                          torch.zeros(w.shape, device=w.device))
        return st


class _NormWork:
    """Device scratch of one global-norm reduction (partials, fp64 sum, scale, norm)."""

    def __init__(self, device):
        nparts = _lib().mst_grad_sumsq_workspace()
        self.partial = torch.empty(nparts, dtype=torch.float64, device=device)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)
        self.scale = torch.ones(1, dtype=torch.float32, device=device)
        self.norm = torch.zeros(1, dtype=torch.float32, device=device)


def global_norm_scale(grads: Iterable[torch.Tensor], max_norm: Optional[float], inv_steps: float = 1.0,
                      work: Optional[_NormWork] = None) -> _NormWork:
    """Device-side ||g||_2 over all gradients and the clip factor of SPEC.md:486-491
    (times inv_steps); no host sync.  max_norm=None: factor = inv_steps."""
    grads = [g for g in grads]
    if not grads:
        raise ms.ConfigError("no gradients")
    lib, ctx = _lib(), _ctx(grads[0])
    w = work or _NormWork(grads[0].device)
    for i, g in enumerate(grads):
        if g.dtype != torch.float32 or not g.is_contiguous():
            raise ms.DtypeError("gradients are contiguous fp32 tensors")
        last = i == len(grads) - 1
        ms._check(lib.mst_grad_sumsq(ctx.handle, ms._stream(g), g.data_ptr(), g.numel(), w.partial.data_ptr(),
                                     w.sumsq.data_ptr(), int(i > 0),
                                     float(max_norm if max_norm is not None else 3.0e38), float(inv_steps),
                                     w.scale.data_ptr() if last else None, w.norm.data_ptr() if last else None))
    return w


def clip_global_norm(grads: Iterable[torch.Tensor], max_norm: float) -> float:
    """clip_global_norm: scales every gradient in place by
    max_norm / ||g|| when ||g|| > max_norm; returns the pre-clip norm.
    Non-finite gradients raise NonFiniteError."""
    grads = list(grads)
    if not max_norm > 0:
        raise ms.ConfigError("max-norm must be > 0")
    w = global_norm_scale(grads, max_norm)
    norm = float(w.norm.item())
    if not math.isfinite(norm):
        raise ms.NonFiniteError(f"non-finite gradient norm {norm} (SPEC.md:488)")
    if norm > max_norm:
        s = max_norm / norm
        for g in grads:
            g.mul_(s)
    return norm


def _adamw_one(p: ParamState, grad: torch.Tensor, cfg: OptimConfig, step: int,
               grad_scale: Optional[torch.Tensor], zero_grad: bool) -> None:
    lib, ctx = _lib(), _ctx(grad)
    if grad.shape != p.master.shape or grad.dtype != torch.float32:
        raise ms.ShapeError(f"gradient {tuple(grad.shape)} {grad.dtype} does not match parameter "
                            f"{tuple(p.master.shape)} fp32 (SPEC.md:495)")
    c = cfg._c()
    ms._check(lib.mst_adamw_step(ctx.handle, ms._stream(grad), p.master.numel(), p.master.data_ptr(),
                                 p.weight.data_ptr(), grad.data_ptr(), p.m.data_ptr(), p.v.data_ptr(), ctypes.byref(c),
                                 int(step), grad_scale.data_ptr() if grad_scale is not None else None,
                                 int(zero_grad)))


def adamw_step(grads: Dict[str, torch.Tensor], state: OptimState, cfg: OptimConfig,
               grad_scale: Optional[torch.Tensor] = None) -> None:
    """adamw_step for every parameter of `state`:
    decoupled weight decay, Adam moments with bias correction."""
    cfg.validate()
    if set(grads) != set(state.params):
        raise ms.ShapeError(f"gradient set {sorted(grads)} != parameters {sorted(state.params)}")
    state.step += 1
    for k, p in state.params.items():
        _adamw_one(p, grads[k], cfg, state.step, grad_scale, zero_grad=False)


def accumulate(into: Dict[str, torch.Tensor], from_: Dict[str, torch.Tensor]) -> None:
    """into += from_ (the sum half of SPEC.md:500-506; flush divides)."""
    lib = _lib()
    for k, g in from_.items():
        d = into[k]
        if d.shape != g.shape:
            raise ms.ShapeError(f"{k}: accumulation shape mismatch")
        ms._check(lib.mst_grad_accumulate(_ctx(d).handle, ms._stream(d), d.data_ptr(), g.data_ptr(), g.numel()))


class GradAccumulator:
    """accumulate(grads-into, grads-from, steps): sums
    micro-batch gradients.  One contract: flush() returns the SUM and the
    division by `steps` happens in AdamW.step (OptimConfig.accumulation_steps
    = steps folds 1/steps into the AdamW kernel's gradient scale and clips the
    norm of the averaged set, so no extra pass over the gradients);
    flush(scale=True) returns the averaged set for any other consumer.
    Flushing before any add is an error."""

    def __init__(self, steps: int):
        if steps < 1:
            raise ms.ConfigError("accumulation steps must be >= 1")
        self.steps = steps
        self.sum: Optional[Dict[str, torch.Tensor]] = None
        self.count = 0

    def add(self, grads: Dict[str, torch.Tensor]) -> None:
        if self.sum is None:
            self.sum = {k: g.clone() for k, g in grads.items()}
        else:
            accumulate(self.sum, grads)
        self.count += 1

    def flush(self, scale: bool = False) -> Dict[str, torch.Tensor]:
        if self.sum is None:
            raise ms.StateError("flush before any accumulation (SPEC.md:503)")
        out = self.sum
        if scale and self.steps != 1:
            for g in out.values():
                g.mul_(1.0 / self.steps)
        self.sum, self.count = None, 0
        return out


class AdamW:
    """AdamW over the MsT block with the SPEC's clip / accumulation /
    in-backward options.  `step(grads)` = clip_global_norm + adamw_step with
    the clip factor and 1/accumulation_steps folded into the kernel."""

    def __init__(self, weights: Dict[str, torch.Tensor], cfg: OptimConfig = OptimConfig()):
        cfg.validate()
        self.cfg = cfg
        self.state = OptimState.create(weights)
        dev = next(iter(weights.values())).device
        self._work = _NormWork(dev)

    def step(self, grads: Dict[str, torch.Tensor], check_finite: bool = False) -> Optional[float]:
        cfg = self.cfg
        inv = 1.0 / cfg.accumulation_steps
        w = global_norm_scale([grads[k] for k in self.state.params], None if cfg.in_backward else cfg.clip_norm,
                              inv, self._work)
        norm = None
        if check_finite:
            norm = float(w.norm.item())
            if not math.isfinite(norm):
                raise ms.NonFiniteError(f"non-finite gradient norm {norm} (SPEC.md:488)")
        adamw_step(grads, self.state, cfg, grad_scale=w.scale)
        return norm

    # ---------------------------------------------------------- in-backward
    def begin_backward(self) -> None:
        self.state.step += 1
        for p in self.state.params.values():
            p.stepped = False

    def step_in_backward(self, name: str, grad: torch.Tensor) -> None:
        """step_in_backward: one parameter, clipping off,
        gradient cleared right after use; stepping a parameter twice in one
        backward is a StateError."""
        p = self.state.params[name]
        if p.stepped:
            raise ms.StateError(f"parameter {name} already stepped in this backward (SPEC.md:511)")
        p.stepped = True
        scale = None
        if self.cfg.accumulation_steps != 1:
            scale = torch.full((1,), 1.0 / self.cfg.accumulation_steps, device=grad.device)
        _adamw_one(p, grad, self.cfg, self.state.step, scale, zero_grad=True)


_NAMES = ("W_gate", "W_up", "W_down", "W_out")


def train_step(X: torch.Tensor, L: torch.Tensor, opt: AdamW, M_mlp: int, M_head: int,
               grads: Optional[ms.BlockGrads] = None, tracker=None):
    """One training step of the MsT block: block_step (forward + backward)
    then the optimizer.  cfg.in_backward: each parameter is stepped as soon
    as its gradient is final in stream order (W_out after the LM-Head
    backward, the MLP weights after the MLP backward) through the library's
    gradient-ready hook, and its gradient is released (zeroed; with a
    memtrack tracker attached a "grad.*" free is recorded).  Otherwise
    clip + AdamW after the backward.  Returns (stats, grads)."""
    P = opt.state.params
    mlp = ms.MlpWeights(P["W_gate"].weight, P["W_up"].weight, P["W_down"].weight)
    head = ms.LmHeadWeights(P["W_out"].weight)
    N, H = X.shape
    I, V = mlp.W_gate.shape[1], head.W_out.shape[1]
    if grads is None:
        grads = ms.alloc_block_grads(N, H, I, V, X.device)
    gmap = {"W_gate": grads.W_gate, "W_up": grads.W_up, "W_down": grads.W_down, "W_out": grads.W_out}
    ctx = ms.Context.get(X.device.index)
    if tracker is not None:
        ctx.attach_tracker(tracker)  # the library records chunk buffers and grad.* lifetimes
    try:
        if not opt.cfg.in_backward:
            stats, grads = ms.block_step(X, L, mlp, head, M_mlp, M_head, grads=grads)
            opt.step(gmap)
            if tracker is not None:  # deferred: gradients released after the optimizer step
                for k, g in gmap.items():
                    tracker.on_free(g.numel() * 4, f"grad.{k}")
            return stats, grads
        return _train_step_in_backward(X, L, opt, M_mlp, M_head, grads, gmap, mlp, head, ctx)
    finally:
        if tracker is not None:
            ctx.attach_tracker(None)


def _train_step_in_backward(X, L, opt, M_mlp, M_head, grads, gmap, mlp, head, ctx):
    P = opt.state.params
    lib = _lib()
    opt.begin_backward()

    errors = []

    def ready(_user, which, _stream):  # the library records the grad.* release
        # ctypes prints and drops exceptions raised in a callback: keep the
        # first one and re-raise it once block_step has returned.
        try:
            name = _NAMES[which]
            opt.step_in_backward(name, gmap[name])
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    hook = _GRAD_READY(ready)
    ms._check(lib.mst_ctx_set_grad_ready_hook(ctx.handle, ctypes.cast(hook, ctypes.c_void_p), None))
    try:
        stats, grads = ms.block_step(X, L, mlp, head, M_mlp, M_head, grads=grads)
    finally:
        ms._check(lib.mst_ctx_set_grad_ready_hook(ctx.handle, None, None))
    if errors:
        raise errors[0]
    missing = [k for k, p in P.items() if not p.stepped]
    if missing:
        raise ms.StateError(f"parameters not stepped in backward: {missing}")
    return stats, grads
