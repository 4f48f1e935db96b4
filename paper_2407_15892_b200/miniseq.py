"""Python mirror of the reference `miniseq` operator API over the libmst C ABI.

The reference specifies the operations

    make_chunk_plan(N, M)
    miniseq_mlp_forward(X, w, plan) -> (O, saved)
    miniseq_mlp_backward(dO, saved, w, plan) -> (dX, dw)
    miniseq_lmhead_forward(X, L, w, plan, mode)
    miniseq_lmhead_backward(saved, w, plan, mode)
    mask_labels_for_chunk(L, range)

with the error taxonomy of proj/include/minitrain/error.hpp.  This module
keeps those names, argument meanings and errors; tensors are torch CUDA
tensors (bf16 activations/weights, fp32 gradients, int32 labels).  Every
call goes through `lib/libmst.so` (sm_100a); there is no CPU fallback — if
the library is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import torch

import os

# MST_LIB overrides the library path (tuning variants built by tools/); the
# default is the in-tree product build.
_LIB_PATH = Path(os.environ.get("MST_LIB", Path(__file__).resolve().parent / "lib" / "libmst.so"))

# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """minitrain::Error (error.hpp:10)."""


class ShapeError(Error):
    pass


class BoundsError(Error):
    pass


class DtypeError(Error):
    pass


class ConfigError(Error):
    pass


class DataError(Error):
    pass


class StateError(Error):
    pass


class NonFiniteError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: ShapeError, 2: BoundsError, 3: DtypeError, 4: ConfigError, 5: DataError, 6: StateError,
           7: NonFiniteError, 8: CudaError, 9: Error}

TOKEN_WEIGHTED = 0
PAPER_MEAN = 1


class _MlpSaved(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("w_gate", ctypes.c_void_p), ("w_up", ctypes.c_void_p),
                ("w_down", ctypes.c_void_p), ("n", ctypes.c_int64), ("h", ctypes.c_int64),
                ("i", ctypes.c_int64), ("m", ctypes.c_int64), ("fingerprint", ctypes.c_uint64)]


class _HeadSaved(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("labels", ctypes.c_void_p), ("w_out", ctypes.c_void_p),
                ("lse", ctypes.c_void_p), ("stats", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("h", ctypes.c_int64), ("v", ctypes.c_int64), ("m", ctypes.c_int64),
                ("loss_mode", ctypes.c_int32), ("_pad", ctypes.c_int32), ("fingerprint", ctypes.c_uint64)]


_VP, _I64, _I32, _F32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
_SIGS = {
    "mst_abi_version": ([], ctypes.c_int),
    "mst_last_error": ([], ctypes.c_char_p),
    "mst_ctx_create": ([_I32, ctypes.POINTER(_VP)], ctypes.c_int),
    "mst_ctx_destroy": ([_VP], None),
    "mst_ctx_num_pairs": ([_VP], ctypes.c_int),
    "mst_ctx_launch_count": ([_VP], ctypes.c_int64),
    "mst_ctx_set_timing": ([_VP, _I32], ctypes.c_int),
    "mst_ctx_take_timing": ([_VP, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(_I64)], ctypes.c_int),
    "mst_ctx_set_profile_buffer": ([_VP, _VP], ctypes.c_int),
    "mst_ctx_set_tuning": ([_VP, ctypes.c_char_p, _I32], ctypes.c_int),
    "mst_ctx_take_timing_records": ([_VP, _I64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(_I64)], ctypes.c_int),
    "mst_make_chunk_plan": ([_I64, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)], ctypes.c_int),
    "mst_mlp_workspace": ([_I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "mst_lmhead_workspace": ([_I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "mst_block_workspace": ([_I64, _I64, _I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "mst_ctx_block_workspace": ([_VP, _I64, _I64, _I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
                                ctypes.c_int),
    "mst_ctx_block_host_workspace": ([_VP, _I64, _I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
                                     ctypes.c_int),
    "mst_block_step_host": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _I64, _I32,
                             ctypes.c_float, _VP, _VP, _VP, _VP, _VP, _VP, _I32, _VP, ctypes.c_size_t], ctypes.c_int),
    "mst_mlp_forward": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _VP, ctypes.c_size_t,
                         ctypes.POINTER(_MlpSaved)], ctypes.c_int),
    "mst_mlp_backward": ([_VP, _VP, _VP, ctypes.POINTER(_MlpSaved), _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32,
                          _VP, ctypes.c_size_t], ctypes.c_int),
    "mst_lmhead_forward": ([_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _I32, _VP, _VP, _VP, ctypes.c_size_t,
                            ctypes.POINTER(_HeadSaved)], ctypes.c_int),
    "mst_lmhead_backward": ([_VP, _VP, ctypes.POINTER(_HeadSaved), _VP, _VP, _F32, _VP, _VP, _I32, _VP,
                             ctypes.c_size_t], ctypes.c_int),
    "mst_lmhead_fused": ([_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _I32, _F32, _VP, _VP, _VP, _VP, _VP, _I32,
                          _VP, ctypes.c_size_t], ctypes.c_int),
    "mst_count_valid": ([_VP, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "mst_block_step": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _F32,
                        _VP, _VP, _VP, _VP, _VP, _VP, _I32, _VP, ctypes.c_size_t], ctypes.c_int),
    "mst_block_step_sp": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _F32,
                           _VP, _VP, _VP, _VP, _VP, _VP, _I32, _VP, ctypes.c_size_t, _VP], ctypes.c_int),
    "mst_debug_gemm": ([_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _I32], ctypes.c_int),
    "mst_ctx_get_counters": ([_VP, _VP], ctypes.c_int),
    "mst_count_nonfinite": ([_VP, _VP, _VP, _I64, _I32, _VP], ctypes.c_int),
    "mst_ctx_reset_counters": ([_VP], ctypes.c_int),
    "mst_ctx_set_mem_hook": ([_VP, _VP, _VP], ctypes.c_int),
    "mst_ctx_set_count_hook": ([_VP, _VP, _VP], ctypes.c_int),
}

# memtrack hooks (mst.h): kind 0 alloc / 1 free; count kind 0 matmul / 1 op.
_MEM_HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p)
_COUNT_HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                               ctypes.c_uint64)


class _AdamCfg(ctypes.Structure):  # mst_adamw_config
    _fields_ = [("lr", ctypes.c_double), ("weight_decay", ctypes.c_double), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("eps", ctypes.c_double)]


_SIGS.update({  # optimizer, used by optim.py
    "mst_adamw_step": ([_VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, ctypes.POINTER(_AdamCfg), _I64, _VP, _I32],
                       ctypes.c_int),
    "mst_grad_sumsq_workspace": ([], ctypes.c_int),
    "mst_grad_sumsq": ([_VP, _VP, _VP, _I64, _VP, _VP, _I32, ctypes.c_float, ctypes.c_float, _VP, _VP], ctypes.c_int),
    "mst_grad_accumulate": ([_VP, _VP, _VP, _VP, _I64], ctypes.c_int),
    "mst_ctx_set_grad_ready_hook": ([_VP, _VP, _VP], ctypes.c_int),
})


_SIGS.update({  # decoder-layer plumbing (model module), used by model.py
    "mst_gemm": ([_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _I32], ctypes.c_int),
    "mst_rmsnorm_forward": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, ctypes.c_float], ctypes.c_int),
    "mst_rmsnorm_workspace": ([_VP, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "mst_rmsnorm_backward": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32, _I64, _I64, _VP, ctypes.c_size_t],
                             ctypes.c_int),
    "mst_embedding_forward": ([_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP], ctypes.c_int),
    "mst_embedding_backward": ([_VP, _VP, _VP, _VP, _VP, _I64, _VP, _VP, _I64, _I64, _I32], ctypes.c_int),
})

_GRAD_READY_HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)
# mst_grad_slab_hook(user, which, row0, row1, stream)
_GRAD_SLAB_HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p)
_SIGS["mst_ctx_set_grad_slab_hook"] = ([_VP, _VP, _VP, _I32], ctypes.c_int)
_SIGS["mst_ctx_check"] = ([_VP, _VP], ctypes.c_int)
_SIGS.update({  # causal GQA attention, used by attention.py
    "mst_attention_forward": ([_VP, _VP, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64,
                               _I64, _I32], ctypes.c_int),
    "mst_attention_workspace": ([_I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "mst_attention_backward": ([_VP, _VP, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _VP, _I64, _VP,
                                _I64, _VP, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _VP, ctypes.c_size_t],
                               ctypes.c_int),
})


class _Counters(ctypes.Structure):
    _fields_ = [("flops", ctypes.c_uint64), ("matmul_flops", ctypes.c_uint64), ("hbm_elements", ctypes.c_uint64),
                ("weight_read_elements", ctypes.c_uint64)]

_lib = None
_lib_lock = threading.Lock()


def load_library() -> ctypes.CDLL:
    """Load libmst.so (raises if it was not built — no fallback path exists)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ImportError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def _check(status: int) -> None:
    if status != 0:
        msg = load_library().mst_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


# ----------------------------------------------------------------- context
class Context:
    """One libmst context per device (one context per thread/device)."""

    _per_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        self.lib = load_library()
        self.device = device
        h = ctypes.c_void_p()
        _check(self.lib.mst_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self._ws: Optional[torch.Tensor] = None

    @classmethod
    def get(cls, device: Optional[int] = None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        ctx = cls._per_device.get(device)
        if ctx is None:
            ctx = cls._per_device[device] = Context(device)
        return ctx

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = None
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def counters(self):
        """Op counters of this context (memtrack.hpp:19-35 conventions)."""
        from .memtrack import OpCounters

        c = _Counters()
        _check(self.lib.mst_ctx_get_counters(self.handle, ctypes.byref(c)))
        return OpCounters(c.flops, c.matmul_flops, c.hbm_elements, c.weight_read_elements)

    def reset_counters(self) -> None:
        _check(self.lib.mst_ctx_reset_counters(self.handle))

    def attach_tracker(self, tracker) -> None:
        """Route the library's memory events and op counts into a
        memtrack.MemTracker (or anything with on_alloc/on_free/count_matmul/
        count_op); None detaches."""
        if tracker is None:
            _check(self.lib.mst_ctx_set_mem_hook(self.handle, None, None))
            _check(self.lib.mst_ctx_set_count_hook(self.handle, None, None))
            self._hooks = None
            return

        def mem(_user, kind, nbytes, label):
            (tracker.on_alloc if kind == 0 else tracker.on_free)(int(nbytes), label.decode())

        def cnt(_user, kind, a, b, c, w):
            if kind == 0:
                tracker.count_matmul(int(a), int(b), int(c), int(w))
            else:
                tracker.count_op(int(a), int(b))

        self._hooks = (_MEM_HOOK(mem), _COUNT_HOOK(cnt))  # keep the trampolines alive
        _check(self.lib.mst_ctx_set_mem_hook(self.handle, ctypes.cast(self._hooks[0], ctypes.c_void_p), None))
        _check(self.lib.mst_ctx_set_count_hook(self.handle, ctypes.cast(self._hooks[1], ctypes.c_void_p), None))

    def check(self, stream: Optional[int] = None) -> None:
        """Synchronise `stream` (default: the current stream) and raise the
        context's deferred device-side error, if any (mst_ctx_check: all
        labels ignored / invalid labels -> DataError, non-finite loss ->
        NonFiniteError); clears it."""
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        _check(self.lib.mst_ctx_check(self.handle, stream))

    def set_tuning(self, key: str, value: int) -> None:
        """Engine tuning / diagnostic knobs (mst_ctx_set_tuning in mst.h)."""
        _check(self.lib.mst_ctx_set_tuning(self.handle, key.encode(), int(value)))

    @property
    def num_pairs(self) -> int:
        return self.lib.mst_ctx_num_pairs(self.handle)

    @property
    def launch_count(self) -> int:
        return self.lib.mst_ctx_launch_count(self.handle)

    def set_timing(self, enable: bool) -> None:
        _check(self.lib.mst_ctx_set_timing(self.handle, int(enable)))

    def take_timing(self) -> tuple[float, float, int]:
        """(gemm device ms, algorithmic gemm FLOPs, launches) since the last call."""
        ms_, fl, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(self.lib.mst_ctx_take_timing(self.handle, ctypes.byref(ms_), ctypes.byref(fl), ctypes.byref(n)))
        return ms_.value, fl.value, n.value

    def take_timing_records(self, cap: int = 4096) -> list[tuple[float, float]]:
        """Per-launch (device ms, algorithmic FLOPs) since the last take."""
        ms_, fl, n = (ctypes.c_double * cap)(), (ctypes.c_double * cap)(), ctypes.c_int64()
        _check(self.lib.mst_ctx_take_timing_records(self.handle, cap, ms_, fl, ctypes.byref(n)))
        return [(ms_[k], fl[k]) for k in range(n.value)]


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _req(t: torch.Tensor, name: str, dtype: torch.dtype, shape: tuple) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ConfigError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise DtypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ConfigError(f"{name} must be contiguous")


# ----------------------------------------------------------------- types
@dataclass(frozen=True)
class ChunkPlan:
    """contiguous ranges covering [0, N)."""
    M: int
    N: int
    ranges: tuple

    def __len__(self) -> int:
        return len(self.ranges)


@dataclass
class MlpWeights:
    """W_gate, W_up [d x I]; W_down [I x d]."""
    W_gate: torch.Tensor
    W_up: torch.Tensor
    W_down: torch.Tensor


@dataclass
class MlpGrads:
    W_gate: torch.Tensor
    W_up: torch.Tensor
    W_down: torch.Tensor


@dataclass
class LmHeadWeights:
    """W_out [d x V]."""
    W_out: torch.Tensor


@dataclass
class MlpSaved:
    X: torch.Tensor
    plan: ChunkPlan
    rec: _MlpSaved


@dataclass
class LmHeadSaved:
    X: torch.Tensor
    labels: torch.Tensor
    lse: torch.Tensor
    stats: torch.Tensor
    plan: ChunkPlan
    mode: int
    rec: _HeadSaved

    @property
    def valid_count(self) -> torch.Tensor:
        return self.stats[1]


def make_chunk_plan(N: int, M: int) -> ChunkPlan:
    """SPEC.md:286-294 (balanced rule)."""
    lib = load_library()
    if N < 1:
        raise DataError("make_chunk_plan: N must be >= 1")
    if M < 1:
        raise ConfigError("make_chunk_plan: M must be >= 1")
    cap = min(N, M) + 1
    buf = (ctypes.c_int64 * cap)()
    cnt = ctypes.c_int64()
    _check(lib.mst_make_chunk_plan(N, M, buf, ctypes.byref(cnt)))
    b = list(buf)[: cnt.value + 1]
    return ChunkPlan(M=M, N=N, ranges=tuple((b[i], b[i + 1]) for i in range(cnt.value)))


def mask_labels_for_chunk(L: torch.Tensor, rng: tuple) -> torch.Tensor:
    """label slice of a chunk, ignore value -100 preserved."""
    s, e = rng
    if not (0 <= s <= e <= L.shape[0]):
        raise BoundsError(f"range {rng} outside [0, {L.shape[0]})")
    return L[s:e]


def _plan_check(plan: ChunkPlan, N: int) -> None:
    if plan.N != N:
        raise ConfigError(f"plan covers N={plan.N} rows but X has {N} (SPEC.md:297)")


# ----------------------------------------------------------------- MLP
def miniseq_mlp_forward(X: torch.Tensor, w: MlpWeights, plan: ChunkPlan, out: Optional[torch.Tensor] = None):
    """SPEC.md:295-303 / Alg. 1: O = silu(X W_g) * (X W_u) W_d, chunk by chunk."""
    ctx = Context.get(X.device.index)
    N, H = X.shape
    I = w.W_gate.shape[1]
    _plan_check(plan, N)
    _req(X, "X", torch.bfloat16, (N, H))
    _req(w.W_gate, "W_gate", torch.bfloat16, (H, I))
    _req(w.W_up, "W_up", torch.bfloat16, (H, I))
    _req(w.W_down, "W_down", torch.bfloat16, (I, H))
    if out is None:
        out = torch.empty_like(X)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_mlp_workspace(N, H, I, plan.M, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    rec = _MlpSaved()
    _check(ctx.lib.mst_mlp_forward(ctx.handle, _stream(X), X.data_ptr(), w.W_gate.data_ptr(), w.W_up.data_ptr(),
                                   w.W_down.data_ptr(), out.data_ptr(), N, H, I, plan.M, ws.data_ptr(), ws.numel(),
                                   ctypes.byref(rec)))
    return out, MlpSaved(X=X, plan=plan, rec=rec)


def miniseq_mlp_backward(dO: torch.Tensor, saved: MlpSaved, w: MlpWeights, plan: ChunkPlan,
                         grads: Optional[MlpGrads] = None, accumulate: bool = False):
    """SPEC.md:304-312 / Alg. 3: per-chunk recompute; dW accumulated in fp32, ascending chunks."""
    if saved.plan != plan:
        raise StateError("saved state was produced under a different chunk plan")
    X = saved.X
    ctx = Context.get(X.device.index)
    N, H = X.shape
    I = w.W_gate.shape[1]
    _req(dO, "dO", torch.bfloat16, (N, H))
    if grads is None:
        dev = X.device
        grads = MlpGrads(torch.empty(H, I, dtype=torch.float32, device=dev),
                         torch.empty(H, I, dtype=torch.float32, device=dev),
                         torch.empty(I, H, dtype=torch.float32, device=dev))
        accumulate = False
    _req(grads.W_gate, "dW_gate", torch.float32, (H, I))
    _req(grads.W_up, "dW_up", torch.float32, (H, I))
    _req(grads.W_down, "dW_down", torch.float32, (I, H))
    dX = torch.empty_like(X)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_mlp_workspace(N, H, I, plan.M, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    _check(ctx.lib.mst_mlp_backward(ctx.handle, _stream(X), dO.data_ptr(), ctypes.byref(saved.rec),
                                    w.W_gate.data_ptr(), w.W_up.data_ptr(), w.W_down.data_ptr(), dX.data_ptr(),
                                    grads.W_gate.data_ptr(), grads.W_up.data_ptr(), grads.W_down.data_ptr(),
                                    int(accumulate), ws.data_ptr(), ws.numel()))
    return dX, grads


# ----------------------------------------------------------------- LM-Head
def stats_len(num_chunks: int) -> int:
    return 4 + 2 * num_chunks


def miniseq_lmhead_forward(X: torch.Tensor, L: torch.Tensor, w: LmHeadWeights, plan: ChunkPlan,
                           mode: int = TOKEN_WEIGHTED):
    """SPEC.md:313-321 / Alg. 2.  Returns (loss, saved); loss is a 0-d device tensor.

    The per-chunk logits never reach HBM: the GEMM epilogue keeps an online
    softmax, so the saved state is X, L and one fp32 lse per row."""
    ctx = Context.get(X.device.index)
    N, H = X.shape
    V = w.W_out.shape[1]
    _plan_check(plan, N)
    _req(X, "X", torch.bfloat16, (N, H))
    _req(L, "L", torch.int32, (N,))
    _req(w.W_out, "W_out", torch.bfloat16, (H, V))
    stats = torch.empty(stats_len(len(plan)), dtype=torch.float32, device=X.device)
    lse = torch.empty(N, dtype=torch.float32, device=X.device)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_lmhead_workspace(N, H, V, plan.M, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    rec = _HeadSaved()
    _check(ctx.lib.mst_lmhead_forward(ctx.handle, _stream(X), X.data_ptr(), L.data_ptr(), w.W_out.data_ptr(), N, H,
                                      V, plan.M, int(mode), stats.data_ptr(), lse.data_ptr(), ws.data_ptr(),
                                      ws.numel(), ctypes.byref(rec)))
    return stats[2], LmHeadSaved(X=X, labels=L, lse=lse, stats=stats, plan=plan, mode=int(mode), rec=rec)


def check_lmhead_stats(saved: LmHeadSaved) -> None:
    """Host-side checks the asynchronous C ABI defers (forces a sync):
    invalid label ids (DataError) and all-ignored input."""
    s = saved.stats[:4].tolist()
    Context.get(saved.stats.device.index).check()  # consumes the deferred flag this forward raised
    if s[3] > 0:
        raise DataError(f"{int(s[3])} labels outside [0, V) and != -100")
    if s[1] == 0:
        raise DataError("all labels ignored: loss undefined (SPEC.md:219)")
    if not math.isfinite(s[2]):
        raise NonFiniteError(f"non-finite loss {s[2]} (SPEC.md:26)")


def miniseq_lmhead_backward(saved: LmHeadSaved, w: LmHeadWeights, plan: ChunkPlan, mode: Optional[int] = None,
                            grad_loss: float = 1.0, global_stats: Optional[torch.Tensor] = None,
                            dW_out: Optional[torch.Tensor] = None, accumulate: bool = False):
    """SPEC.md:322-330 / Alg. 4: recompute logits per chunk, CE backward with the
    mode's scaling x grad_loss, dX concatenated, dW_out accumulated in fp32."""
    if saved.plan != plan:
        raise StateError("saved state was produced under a different chunk plan")
    if mode is not None and mode != saved.mode:
        raise StateError("loss mode differs from the forward's")
    X = saved.X
    ctx = Context.get(X.device.index)
    N, H = X.shape
    V = w.W_out.shape[1]
    if dW_out is None:
        dW_out = torch.empty(H, V, dtype=torch.float32, device=X.device)
        accumulate = False
    _req(dW_out, "dW_out", torch.float32, (H, V))
    dX = torch.empty_like(X)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_lmhead_workspace(N, H, V, plan.M, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    gs = saved.stats if global_stats is None else global_stats
    _check(ctx.lib.mst_lmhead_backward(ctx.handle, _stream(X), ctypes.byref(saved.rec), w.W_out.data_ptr(),
                                       gs.data_ptr(), float(grad_loss), dX.data_ptr(), dW_out.data_ptr(),
                                       int(accumulate), ws.data_ptr(), ws.numel()))
    return dX, dW_out


def count_nonfinite(t: torch.Tensor) -> torch.Tensor:
    """Device count of NaN/Inf elements of a bf16 / fp32 tensor (int32, no sync)."""
    ctx = Context.get(t.device.index)
    if t.dtype not in (torch.bfloat16, torch.float32):
        raise DtypeError(f"non-finite scan supports bf16 / fp32, got {t.dtype}")
    if not t.is_contiguous():
        raise ShapeError("non-finite scan needs a contiguous tensor")
    out = torch.empty(1, dtype=torch.int32, device=t.device)
    _check(ctx.lib.mst_count_nonfinite(ctx.handle, _stream(t), t.data_ptr(), t.numel(),
                                       1 if t.dtype == torch.float32 else 0, out.data_ptr()))
    return out


def check_finite(**tensors: torch.Tensor) -> None:
    """Raise NonFiniteError naming every tensor with NaN/Inf elements
    (SPEC.md:26); one host sync for all of them."""
    counts = {k: count_nonfinite(t) for k, t in tensors.items() if t is not None and t.numel()}
    bad = {k: int(v.item()) for k, v in counts.items()}
    bad = {k: v for k, v in bad.items() if v}
    if bad:
        raise NonFiniteError("non-finite elements (SPEC.md:26): " + ", ".join(f"{k}: {v}" for k, v in bad.items()))


def count_valid(L: torch.Tensor, V: int) -> torch.Tensor:
    """Device count of labels in [0, V) (1-element fp64 tensor holding an
    exact integer, no sync): the term a sequence shard SUM-all-reduces."""
    ctx = Context.get(L.device.index)
    out = torch.empty(1, dtype=torch.float64, device=L.device)
    _check(ctx.lib.mst_count_valid(ctx.handle, _stream(L), L.data_ptr(), L.shape[0], V, out.data_ptr()))
    return out


def miniseq_lmhead_fused(X: torch.Tensor, L: torch.Tensor, w: LmHeadWeights, plan: ChunkPlan,
                         mode: int = TOKEN_WEIGHTED, grad_loss: float = 1.0,
                         global_valid: Optional[torch.Tensor] = None, dW_out: Optional[torch.Tensor] = None,
                         accumulate: bool = False):
    """LM-Head forward + backward in one pass over the chunks (SPEC.md:313-330
    back to back): returns (loss, stats, lse, dX, dW_out).  `global_valid`
    (1-elem device fp64 count) overrides the local valid count (sequence sharding)."""
    ctx = Context.get(X.device.index)
    N, H = X.shape
    V = w.W_out.shape[1]
    _plan_check(plan, N)
    _req(X, "X", torch.bfloat16, (N, H))
    _req(L, "L", torch.int32, (N,))
    _req(w.W_out, "W_out", torch.bfloat16, (H, V))
    if dW_out is None:
        dW_out = torch.empty(H, V, dtype=torch.float32, device=X.device)
        accumulate = False
    _req(dW_out, "dW_out", torch.float32, (H, V))
    if global_valid is not None:
        _req(global_valid, "global_valid", torch.float64, (1,))
    stats = torch.empty(stats_len(len(plan)), dtype=torch.float32, device=X.device)
    lse = torch.empty(N, dtype=torch.float32, device=X.device)
    dX = torch.empty_like(X)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_lmhead_workspace(N, H, V, plan.M, ctypes.byref(nb)))
    ws = ctx.workspace(nb.value)
    _check(ctx.lib.mst_lmhead_fused(ctx.handle, _stream(X), X.data_ptr(), L.data_ptr(), w.W_out.data_ptr(), N, H, V,
                                    plan.M, int(mode), float(grad_loss), _ptr(global_valid), stats.data_ptr(),
                                    lse.data_ptr(), dX.data_ptr(), dW_out.data_ptr(), int(accumulate), ws.data_ptr(),
                                    ws.numel()))
    return stats[2], stats, lse, dX, dW_out


# ----------------------------------------------------------------- block
@dataclass
class BlockGrads:
    dX: torch.Tensor
    W_gate: torch.Tensor
    W_up: torch.Tensor
    W_down: torch.Tensor
    W_out: torch.Tensor


def block_workspace_bytes(N: int, H: int, I: int, V: int, M_mlp: int, M_head: int,
                          ctx: Optional["Context"] = None) -> int:
    """Workspace of block_step: for `ctx`'s schedule knobs (mst_ctx_block_workspace),
    else the maximum over all schedules (mst_block_workspace)."""
    nb = ctypes.c_size_t()
    if ctx is not None:
        _check(ctx.lib.mst_ctx_block_workspace(ctx.handle, N, H, I, V, M_mlp, M_head, ctypes.byref(nb)))
    else:
        _check(load_library().mst_block_workspace(N, H, I, V, M_mlp, M_head, ctypes.byref(nb)))
    return nb.value


def alloc_block_grads(N: int, H: int, I: int, V: int, device) -> BlockGrads:
    return BlockGrads(torch.empty(N, H, dtype=torch.bfloat16, device=device),
                      torch.empty(H, I, dtype=torch.float32, device=device),
                      torch.empty(H, I, dtype=torch.float32, device=device),
                      torch.empty(I, H, dtype=torch.float32, device=device),
                      torch.empty(H, V, dtype=torch.float32, device=device))


def block_step(X: torch.Tensor, L: torch.Tensor, mlp: MlpWeights, head: LmHeadWeights, M_mlp: int, M_head: int,
               mode: int = TOKEN_WEIGHTED, grad_loss: float = 1.0, grads: Optional[BlockGrads] = None,
               stats: Optional[torch.Tensor] = None, accumulate: bool = False,
               workspace: Optional[torch.Tensor] = None, check: bool = False,
               global_valid: Optional[torch.Tensor] = None, grad_ready=None, grad_slab=None, slabs: int = 1):
    """One MLP -> LM-Head block, forward + backward (the unit the paper times,
    PAPER.md:475).  Returns (stats, grads); stats[2] is the loss.
    check=True surfaces the SPEC's errors synchronously: NonFiniteError for
    NaN/Inf inputs or outputs, DataError for invalid labels or an
    all-ignored batch.
    global_valid: device fp64 [1] valid-label count all-reduced over a
    sequence-parallel group (mst_block_step_sp).  grad_ready(which): called
    while the step is enqueued, right after the launch that makes gradient
    `which` (0 W_gate, 1 W_up, 2 W_down, 3 W_out) final in stream order
    (mst_ctx_set_grad_ready_hook).  grad_slab(which, row0, row1): called
    as rows [row0, row1) of gradient `which` become final; `slabs` > 1 cuts
    the finalising launches into that many row slabs (mst_ctx_set_grad_slab_hook:
    the sequence-parallel all-reduce overlap).  Exceptions raised inside either
    callback are re-raised after the step is enqueued."""
    if check:
        check_finite(X=X, W_gate=mlp.W_gate, W_up=mlp.W_up, W_down=mlp.W_down, W_out=head.W_out)
    ctx = Context.get(X.device.index)
    N, H = X.shape
    I = mlp.W_gate.shape[1]
    V = head.W_out.shape[1]
    _req(X, "X", torch.bfloat16, (N, H))
    _req(L, "L", torch.int32, (N,))
    _req(mlp.W_gate, "W_gate", torch.bfloat16, (H, I))
    _req(mlp.W_up, "W_up", torch.bfloat16, (H, I))
    _req(mlp.W_down, "W_down", torch.bfloat16, (I, H))
    _req(head.W_out, "W_out", torch.bfloat16, (H, V))
    if grads is None:
        grads = alloc_block_grads(N, H, I, V, X.device)
    nch = min(N, M_head)
    if stats is None:
        stats = torch.empty(stats_len(nch), dtype=torch.float32, device=X.device)
    need = block_workspace_bytes(N, H, I, V, M_mlp, M_head, ctx)
    ws = workspace if workspace is not None else ctx.workspace(need)
    if global_valid is not None:
        _req(global_valid, "global_valid", torch.float64, (1,))
    hook = slab_hook = None
    errors = []

    def guarded(fn, *a):  # ctypes prints and drops callback exceptions: keep them
        try:
            fn(*a)
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    if grad_ready is not None:
        hook = _GRAD_READY_HOOK(lambda _u, which, _s: guarded(grad_ready, int(which)))
        _check(ctx.lib.mst_ctx_set_grad_ready_hook(ctx.handle, ctypes.cast(hook, ctypes.c_void_p), None))
    if grad_slab is not None:
        slab_hook = _GRAD_SLAB_HOOK(lambda _u, which, r0, r1, _s: guarded(grad_slab, int(which), int(r0), int(r1)))
        _check(ctx.lib.mst_ctx_set_grad_slab_hook(ctx.handle, ctypes.cast(slab_hook, ctypes.c_void_p), None,
                                                  int(slabs)))
    try:
        _check(ctx.lib.mst_block_step_sp(ctx.handle, _stream(X), X.data_ptr(), L.data_ptr(), mlp.W_gate.data_ptr(),
                                         mlp.W_up.data_ptr(), mlp.W_down.data_ptr(), head.W_out.data_ptr(), N, H, I,
                                         V, M_mlp, M_head, int(mode), float(grad_loss), stats.data_ptr(),
                                         grads.dX.data_ptr(), grads.W_gate.data_ptr(), grads.W_up.data_ptr(),
                                         grads.W_down.data_ptr(), grads.W_out.data_ptr(), int(accumulate),
                                         ws.data_ptr(), ws.numel(), _ptr(global_valid)))
    finally:
        if hook is not None:
            _check(ctx.lib.mst_ctx_set_grad_ready_hook(ctx.handle, None, None))
        if slab_hook is not None:
            _check(ctx.lib.mst_ctx_set_grad_slab_hook(ctx.handle, None, None, 1))
    if errors:
        raise errors[0]
    if check:
        s = stats[:4].tolist()
        ctx.check()  # the deferred device-side error of this step, if any
        if s[3] > 0:
            raise DataError(f"{int(s[3])} labels outside [0, V) and != -100")
        if s[1] == 0:
            raise DataError("all labels ignored: loss undefined (SPEC.md:219)")
        check_finite(loss=stats[2:3], dX=grads.dX, dW_gate=grads.W_gate, dW_up=grads.W_up, dW_down=grads.W_down,
                     dW_out=grads.W_out)
    return stats, grads


def block_step_host(X: torch.Tensor, L: torch.Tensor, mlp: MlpWeights, head: LmHeadWeights, M: int,
                    dX: torch.Tensor, grads: Optional[BlockGrads] = None, stats: Optional[torch.Tensor] = None,
                    mode: int = TOKEN_WEIGHTED, grad_loss: float = 1.0, accumulate: bool = False,
                    workspace: Optional[torch.Tensor] = None):
    """block_step with host-resident X, labels and dX (mst_block_step_host):
    X / L are pinned CPU tensors, dX a pinned CPU bf16 output; the chunks are
    streamed in and out on a copy stream while the GEMMs run.  Weights and
    the fp32 weight gradients (grads.W_*) live on the device.  Returns
    (stats, grads); dX is filled once the current stream is synchronised."""
    dev = mlp.W_gate.device
    ctx = Context.get(dev.index)
    N, H = X.shape
    I = mlp.W_gate.shape[1]
    V = head.W_out.shape[1]
    for t, name, dt, shape in ((X, "X", torch.bfloat16, (N, H)), (L, "L", torch.int32, (N,)),
                               (dX, "dX", torch.bfloat16, (N, H))):
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise ConfigError(f"{name} must be a host (CPU) tensor, pinned for overlapped copies")
        if t.dtype != dt:
            raise DtypeError(f"{name} must be {dt}, got {t.dtype}")
        if tuple(t.shape) != shape:
            raise ShapeError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ConfigError(f"{name} must be contiguous")
    if grads is None:
        grads = BlockGrads(dX, *(torch.empty(*s, dtype=torch.float32, device=dev) for s in ((H, I), (H, I), (I, H),
                                                                                          (H, V))))
    nch = min(N, M)
    if stats is None:
        stats = torch.empty(stats_len(nch), dtype=torch.float32, device=dev)
    nb = ctypes.c_size_t()
    _check(ctx.lib.mst_ctx_block_host_workspace(ctx.handle, N, H, I, V, M, ctypes.byref(nb)))
    ws = workspace if workspace is not None else ctx.workspace(nb.value)
    _check(ctx.lib.mst_block_step_host(ctx.handle, _stream(mlp.W_gate), X.data_ptr(), L.data_ptr(),
                                       mlp.W_gate.data_ptr(), mlp.W_up.data_ptr(), mlp.W_down.data_ptr(),
                                       head.W_out.data_ptr(), N, H, I, V, M, mode, grad_loss, stats.data_ptr(),
                                       dX.data_ptr(), grads.W_gate.data_ptr(), grads.W_up.data_ptr(),
                                       grads.W_down.data_ptr(), grads.W_out.data_ptr(), int(accumulate),
                                       ws.data_ptr(), ws.numel()))
    return stats, grads


def debug_gemm(A: torch.Tensor, B: torch.Tensor, M: int, N: int, K: int, a_mn: bool, b_mn: bool,
               out: torch.Tensor, beta: int = 0) -> torch.Tensor:
    """C = A B through the tcgen05 engine (diagnostics; see mst.h)."""
    ctx = Context.get(A.device.index)
    _check(ctx.lib.mst_debug_gemm(ctx.handle, _stream(A), A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K,
                                  int(a_mn), int(b_mn), int(out.dtype == torch.float32), int(beta)))
    return out
