"""ctypes/numpy front end of the C oracle (oracle/mst_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker for parity tests and the timed CPU
baseline.  Every function restates a reference operation; the C source
carries the SPEC.md / rng.hpp / memtrack.hpp line citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libmst_oracle.so"
REF_DRIVER = HERE / "_ref" / "ref_driver"
REFERENCE_INCLUDE = Path("/root/reference/proj/include")

_lock = threading.Lock()
_lib = None


def build(ref: bool = False) -> None:
    """Compile the oracle (and, if the reference is mounted, the reference driver)."""
    targets = ["all"] + (["ref"] if ref and REFERENCE_INCLUDE.exists() else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class Rng(ctypes.Structure):
    _fields_ = [("root_seed", ctypes.c_uint64), ("s", ctypes.c_uint64 * 4)]


class Counters(ctypes.Structure):
    _fields_ = [("flops", ctypes.c_uint64), ("matmul_flops", ctypes.c_uint64), ("hbm_elements", ctypes.c_uint64),
                ("weight_read_elements", ctypes.c_uint64)]


class BlockF32(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("N", "H", "I", "V", "M_mlp", "M_head")] + \
               [(n, ctypes.c_void_p) for n in ("X", "Wg", "Wu", "Wd", "Wout", "WgT", "WuT", "WdT", "WoutT", "L",
                                               "dX", "dWg", "dWu", "dWd", "dWout")] + [("loss", ctypes.c_double)]


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            src = HERE / "mst_oracle.c"
            if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
                build()
            L = ctypes.CDLL(str(LIB))
            d, i64, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
            L.orc_rng_next_u64.restype = ctypes.c_uint64
            L.orc_rng_uniform.restype = d
            L.orc_rng_gaussian.restype = d
            L.orc_rng_uniform_below.restype = ctypes.c_uint64
            L.orc_rng_uniform_below.argtypes = [ctypes.POINTER(Rng), ctypes.c_uint64]
            L.orc_rng_init.argtypes = [ctypes.POINTER(Rng), ctypes.c_uint64]
            L.orc_fnv1a64.restype = ctypes.c_uint64
            L.orc_fnv1a64.argtypes = [ctypes.c_char_p]
            L.orc_splitmix64.restype = ctypes.c_uint64
            L.orc_silu_f64.restype = d
            L.orc_silu_f64.argtypes = [d]
            L.orc_silu_backward_f64.restype = d
            L.orc_silu_backward_f64.argtypes = [d, d]
            L.orc_round_bf16.restype = ctypes.c_float
            L.orc_round_bf16.argtypes = [ctypes.c_float]
            L.orc_fill_gaussian_bf16.argtypes = [ctypes.POINTER(Rng), vp, i64, d]
            L.orc_fill_labels.argtypes = [ctypes.POINTER(Rng), vp, i64, i64, d]
            L.orc_mem_peak.restype = ctypes.c_uint64
            L.orc_mem_peak_class.restype = ctypes.c_uint64
            L.orc_mem_live.restype = ctypes.c_uint64
            L.orc_matmul_f64.argtypes = [vp, vp, vp, i64, i64, i64]
            L.orc_make_chunk_plan.argtypes = [i64, i64, vp, vp]
            L.orc_mlp_forward_f64.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp, ctypes.c_int]
            L.orc_mlp_backward_f64.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, vp, vp, vp, vp, ctypes.c_int]
            L.orc_lmhead_forward_f64.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp]
            L.orc_lmhead_backward_f64.argtypes = [vp, vp, vp, i64, i64, i64, d, vp, vp, ctypes.c_int]
            L.orc_miniseq_mlp_forward_f64.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, vp, ctypes.c_int]
            L.orc_miniseq_mlp_backward_f64.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp, vp, vp,
                                                       ctypes.c_int]
            L.orc_miniseq_lmhead_forward_f64.argtypes = [vp, vp, vp, i64, i64, i64, i64, ctypes.c_int, vp, vp, vp,
                                                         vp]
            L.orc_miniseq_lmhead_backward_f64.argtypes = [vp, vp, vp, i64, i64, i64, i64, ctypes.c_int, d, vp, vp,
                                                          ctypes.c_int]
            L.orc_block_step_f32.argtypes = [ctypes.POINTER(BlockF32), ctypes.c_int]
            L.orc_transpose_f32.argtypes = [vp, vp, i64, i64, ctypes.c_int]
            _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _chk(code: int, what: str) -> None:
    if code != 0:
        raise OracleError(code, what)


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------ rng
class OracleRng:
    """rng.hpp:28-72 restated (Rng, fork, next_u64, uniform, uniform_below, gaussian)."""

    def __init__(self, seed: int):
        self._r = Rng()
        lib().orc_rng_init(ctypes.byref(self._r), ctypes.c_uint64(seed))

    def fork(self, name: str) -> "OracleRng":
        out = OracleRng(0)
        lib().orc_rng_fork(ctypes.byref(self._r), name.encode(), ctypes.byref(out._r))
        return out

    def next_u64(self) -> int:
        return lib().orc_rng_next_u64(ctypes.byref(self._r))

    def uniform(self) -> float:
        return lib().orc_rng_uniform(ctypes.byref(self._r))

    def uniform_below(self, n: int) -> int:
        return lib().orc_rng_uniform_below(ctypes.byref(self._r), n)

    def gaussian(self) -> float:
        return lib().orc_rng_gaussian(ctypes.byref(self._r))

    def gaussian_bf16(self, shape, std: float) -> np.ndarray:
        out = np.empty(int(np.prod(shape)), dtype=np.float32)
        lib().orc_fill_gaussian_bf16(ctypes.byref(self._r), _p(out), out.size, std)
        return out.reshape(shape)

    def labels(self, n: int, vocab: int, p_ignore: float = 0.05) -> np.ndarray:
        out = np.empty(n, dtype=np.int32)
        lib().orc_fill_labels(ctypes.byref(self._r), _p(out), n, vocab, p_ignore)
        return out


def fnv1a64(s: str) -> int:
    return lib().orc_fnv1a64(s.encode())


def splitmix64_seq(seed: int, n: int) -> list:
    st = ctypes.c_uint64(seed)
    return [lib().orc_splitmix64(ctypes.byref(st)) for _ in range(n)]


def round_bf16(x: float) -> float:
    return lib().orc_round_bf16(x)


def make_inputs(seed: int, N: int, H: int, I: int, V: int, p_ignore: float = 0.05, x_std: float = 1.0,
                w_std: float = 0.02):
    """Golden synthetic inputs: bf16-valued X ~ N(0,1), W ~ N(0, 0.02^2)
    (SPEC.md:428), labels uniform in [0,V) with p_ignore set to -100; each tensor
    drawn from its own named fork of Rng(seed) so shapes never perturb each other."""
    r = OracleRng(seed)
    return dict(X=r.fork("X").gaussian_bf16((N, H), x_std),
                Wg=r.fork("weights.mlp.gate").gaussian_bf16((H, I), w_std),
                Wu=r.fork("weights.mlp.up").gaussian_bf16((H, I), w_std),
                Wd=r.fork("weights.mlp.down").gaussian_bf16((I, H), w_std),
                Wout=r.fork("weights.head.out").gaussian_bf16((H, V), w_std),
                L=r.fork("labels").labels(N, V, p_ignore))


# ------------------------------------------------------------------ counters / memory
def counters_reset() -> None:
    lib().orc_counters_reset()


def counters() -> dict:
    c = Counters()
    lib().orc_counters_get(ctypes.byref(c))
    return dict(flops=c.flops, matmul_flops=c.matmul_flops, hbm_elements=c.hbm_elements,
                weight_read_elements=c.weight_read_elements)


MEM_ACT, MEM_INTER_MLP, MEM_INTER_HEAD, MEM_GRAD = 0, 1, 2, 3


def mem_reset() -> None:
    lib().orc_mem_reset()


def mem_peak(cls: int | None = None) -> int:
    return lib().orc_mem_peak() if cls is None else lib().orc_mem_peak_class(cls)


# ------------------------------------------------------------------ ops (f64)
def make_chunk_plan(N: int, M: int):
    b = np.zeros(max(1, min(N, M)) + 1, dtype=np.int64)
    c = np.zeros(1, dtype=np.int64)
    _chk(lib().orc_make_chunk_plan(N, M, _p(b), _p(c)), "make_chunk_plan")
    return [(int(b[i]), int(b[i + 1])) for i in range(int(c[0]))]


def matmul(a, b):
    a, b = _f64(a), _f64(b)
    c = np.empty((a.shape[0], b.shape[1]))
    lib().orc_matmul_f64(_p(a), _p(b), _p(c), a.shape[0], a.shape[1], b.shape[1])
    return c


def silu(x: float) -> float:
    return lib().orc_silu_f64(x)


def silu_backward(x: float, up: float) -> float:
    return lib().orc_silu_backward_f64(x, up)


def mlp_forward(X, Wg, Wu, Wd, round_bf16=False):
    X, Wg, Wu, Wd = map(_f64, (X, Wg, Wu, Wd))
    O = np.empty_like(X)
    _chk(lib().orc_mlp_forward_f64(_p(X), _p(Wg), _p(Wu), _p(Wd), X.shape[0], X.shape[1], Wg.shape[1], _p(O),
                                   int(round_bf16)), "mlp_forward")
    return O


def mlp_backward(dO, X, Wg, Wu, Wd, round_bf16=False):
    dO, X, Wg, Wu, Wd = map(_f64, (dO, X, Wg, Wu, Wd))
    dX, dWg, dWu, dWd = np.empty_like(X), np.empty_like(Wg), np.empty_like(Wu), np.empty_like(Wd)
    _chk(lib().orc_mlp_backward_f64(_p(dO), _p(X), _p(Wg), _p(Wu), _p(Wd), X.shape[0], X.shape[1], Wg.shape[1],
                                    _p(dX), _p(dWg), _p(dWu), _p(dWd), int(round_bf16)), "mlp_backward")
    return dX, dWg, dWu, dWd


def miniseq_mlp_forward(X, Wg, Wu, Wd, M, round_bf16=False):
    X, Wg, Wu, Wd = map(_f64, (X, Wg, Wu, Wd))
    O = np.empty_like(X)
    _chk(lib().orc_miniseq_mlp_forward_f64(_p(X), _p(Wg), _p(Wu), _p(Wd), X.shape[0], X.shape[1], Wg.shape[1], M,
                                           _p(O), int(round_bf16)), "miniseq_mlp_forward")
    return O


def miniseq_mlp_backward(dO, X, Wg, Wu, Wd, M, round_bf16=False):
    dO, X, Wg, Wu, Wd = map(_f64, (dO, X, Wg, Wu, Wd))
    dX, dWg, dWu, dWd = np.empty_like(X), np.empty_like(Wg), np.empty_like(Wu), np.empty_like(Wd)
    _chk(lib().orc_miniseq_mlp_backward_f64(_p(dO), _p(X), _p(Wg), _p(Wu), _p(Wd), X.shape[0], X.shape[1],
                                            Wg.shape[1], M, _p(dX), _p(dWg), _p(dWu), _p(dWd), int(round_bf16)),
         "miniseq_mlp_backward")
    return dX, dWg, dWu, dWd


def lmhead_forward(X, L, Wout):
    X, L, Wout = _f64(X), _i32(L), _f64(Wout)
    loss = np.zeros(1)
    lse = np.empty(X.shape[0])
    _chk(lib().orc_lmhead_forward_f64(_p(X), _p(L), _p(Wout), X.shape[0], X.shape[1], Wout.shape[1], _p(loss),
                                      _p(lse)), "lmhead_forward")
    return float(loss[0]), lse


def lmhead_backward(X, L, Wout, grad_loss=1.0, round_bf16=False):
    X, L, Wout = _f64(X), _i32(L), _f64(Wout)
    dX, dW = np.empty_like(X), np.empty_like(Wout)
    _chk(lib().orc_lmhead_backward_f64(_p(X), _p(L), _p(Wout), X.shape[0], X.shape[1], Wout.shape[1], grad_loss,
                                       _p(dX), _p(dW), int(round_bf16)), "lmhead_backward")
    return dX, dW


def miniseq_lmhead_forward(X, L, Wout, M, mode=0):
    X, L, Wout = _f64(X), _i32(L), _f64(Wout)
    loss = np.zeros(1)
    lse = np.empty(X.shape[0])
    c = min(X.shape[0], M)
    cs, cv = np.zeros(c), np.zeros(c)
    _chk(lib().orc_miniseq_lmhead_forward_f64(_p(X), _p(L), _p(Wout), X.shape[0], X.shape[1], Wout.shape[1], M,
                                              mode, _p(loss), _p(lse), _p(cs), _p(cv)), "miniseq_lmhead_forward")
    return float(loss[0]), lse, cs, cv


def miniseq_lmhead_backward(X, L, Wout, M, mode=0, grad_loss=1.0, round_bf16=False):
    X, L, Wout = _f64(X), _i32(L), _f64(Wout)
    dX, dW = np.empty_like(X), np.empty_like(Wout)
    _chk(lib().orc_miniseq_lmhead_backward_f64(_p(X), _p(L), _p(Wout), X.shape[0], X.shape[1], Wout.shape[1], M,
                                               mode, grad_loss, _p(dX), _p(dW), int(round_bf16)),
         "miniseq_lmhead_backward")
    return dX, dW


def block(X, L, Wg, Wu, Wd, Wout, M_mlp, M_head, round_bf16=True, grad_loss=1.0, single_pass=False):
    """MLP -> LM-Head block fwd+bwd in f64 (the GPU block_step's checker).
    With round_bf16 the intermediates libmst stores in bf16 are rounded here
    too; single_pass additionally replays the single-pass head's bf16
    rounding: True / "rowscale" the row-scaled head
    (block_step's default: numerators relative to one reference per row,
    per-row factor applied to dX and to the transposed head input),
    "normalize" the per-tile numerators + normalize pass (dl_rowscale=0)."""
    O = miniseq_mlp_forward(X, Wg, Wu, Wd, M_mlp, round_bf16)
    loss, lse, _, _ = miniseq_lmhead_forward(O, L, Wout, M_head)
    sp = {False: 1, True: 3, "rowscale": 3, "normalize": 2}[single_pass]
    rnd = sp if round_bf16 else 0
    dO, dWout = miniseq_lmhead_backward(O, L, Wout, M_head, 0, grad_loss, rnd)
    dX, dWg, dWu, dWd = miniseq_mlp_backward(dO, X, Wg, Wu, Wd, M_mlp, round_bf16)
    return dict(O=O, loss=loss, lse=lse, dO=dO, dWout=dWout, dX=dX, dWg=dWg, dWu=dWu, dWd=dWd)


# ------------------------------------------------------------------ f32 CPU baseline
def transpose_f32(a: np.ndarray, nthreads: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    at = np.empty((a.shape[1], a.shape[0]), dtype=np.float32)
    lib().orc_transpose_f32(_p(a), _p(at), a.shape[0], a.shape[1], nthreads)
    return at


class CpuBlock:
    """The reference path on host cores: f32 block fwd+bwd (SPEC.md:96 performance dtype)."""

    def __init__(self, X, L, Wg, Wu, Wd, Wout, M_mlp, M_head, nthreads: int):
        f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
        self.X, self.Wg, self.Wu, self.Wd, self.Wout = map(f, (X, Wg, Wu, Wd, Wout))
        self.L = _i32(L)
        self.nthreads = nthreads
        self.WgT = transpose_f32(self.Wg, nthreads)
        self.WuT = transpose_f32(self.Wu, nthreads)
        self.WdT = transpose_f32(self.Wd, nthreads)
        self.WoutT = transpose_f32(self.Wout, nthreads)
        N, H = self.X.shape
        I, V = self.Wg.shape[1], self.Wout.shape[1]
        self.dX = np.empty((N, H), np.float32)
        self.dWg = np.empty((H, I), np.float32)
        self.dWu = np.empty((H, I), np.float32)
        self.dWd = np.empty((I, H), np.float32)
        self.dWout = np.empty((H, V), np.float32)
        b = BlockF32()
        b.N, b.H, b.I, b.V, b.M_mlp, b.M_head = N, H, I, V, M_mlp, M_head
        for n in ("X", "Wg", "Wu", "Wd", "Wout", "WgT", "WuT", "WdT", "WoutT", "L", "dX", "dWg", "dWu", "dWd",
                  "dWout"):
            setattr(b, n, _p(getattr(self, n)))
        self.b = b

    def step(self) -> float:
        _chk(lib().orc_block_step_f32(ctypes.byref(self.b), self.nthreads), "block_step_f32")
        return self.b.loss


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
