"""C-ABI boundary checks that need no GPU: libmst.so loads, exports every
symbol include/mst/mst.h declares, and its host-only entry points (chunk
plan, workspace sizing, argument validation) behave like the reference
(error.hpp:14-20)."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest
import torch

from paper_2407_15892_b200 import LIB_PATH, build_lib
from paper_2407_15892_b200 import miniseq as ms

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    txt = (ROOT / "include" / "mst" / "mst.h").read_text()
    return sorted(set(re.findall(r"MST_API\s+[\w\s\*]+?\b(mst_\w+)\s*\(", txt)))


def test_library_builds_and_exports_every_header_symbol():
    build_lib()
    assert LIB_PATH.exists()
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (mst_\w+)", out))
    declared = header_symbols()
    assert len(declared) >= 16
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # the Python mirror binds exactly the declared ABI
    assert sorted(ms.exported_symbols()) == declared


def test_library_contains_sm100a_tcgen05_code():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_abi_version():
    assert ms.load_library().mst_abi_version() == 1


@pytest.mark.parametrize("N,M", [(8, 2), (8, 1), (7, 2), (9, 4), (64, 16), (5, 7), (8192, 8), (1000, 3)])
def test_chunk_plan_matches_oracle(orc, N, M):
    p = ms.make_chunk_plan(N, M)
    assert list(p.ranges) == orc.make_chunk_plan(N, M)


def test_chunk_plan_errors():
    with pytest.raises(ms.DataError):
        ms.make_chunk_plan(0, 4)
    with pytest.raises(ms.ConfigError):
        ms.make_chunk_plan(8, 0)


def test_mask_labels_for_chunk():
    L = torch.tensor([-100, -100, 3, 4, -100], dtype=torch.int32)
    plan = ms.make_chunk_plan(5, 2)
    parts = [ms.mask_labels_for_chunk(L, r) for r in plan.ranges]
    assert int((parts[0] >= 0).sum()) == 1 and torch.equal(torch.cat(parts), L)
    assert int((ms.mask_labels_for_chunk(L, (0, 2)) >= 0).sum()) == 0
    with pytest.raises(ms.BoundsError):
        ms.mask_labels_for_chunk(L, (3, 9))


def test_workspace_sizes_scale_with_chunk_length():
    lib = ms.load_library()
    nb = ctypes.c_size_t()

    def ws(fn, *a):
        assert fn(*a, ctypes.byref(nb)) == 0
        return nb.value

    # head scratch is one [S/M, V] dlogits chunk + partials: ~M x smaller
    full = ws(lib.mst_lmhead_workspace, 8192, 4096, 128256, 1)
    m8 = ws(lib.mst_lmhead_workspace, 8192, 4096, 128256, 8)
    assert 7.5 < full / m8 < 8.5
    assert ws(lib.mst_mlp_workspace, 8192, 4096, 14336, 1) > 7.5 * ws(lib.mst_mlp_workspace, 8192, 4096, 14336, 8)


def test_argument_validation_maps_to_reference_errors():
    lib = ms.load_library()
    nb = ctypes.c_size_t()
    assert lib.mst_mlp_workspace(0, 64, 64, 1, ctypes.byref(nb)) == 5  # DataError: N=0
    assert lib.mst_mlp_workspace(8, 60, 64, 1, ctypes.byref(nb)) == 1  # ShapeError: H % 8
    assert b"multiples of 8" in lib.mst_last_error()
    assert lib.mst_mlp_workspace(8, 64, 64, 0, ctypes.byref(nb)) == 4  # ConfigError: M=0


def test_backward_rejects_stale_saved_state_without_gpu():
    lib = ms.load_library()
    rec = ms._MlpSaved()
    rec.n, rec.h, rec.i, rec.m = 8, 8, 8, 1
    rec.fingerprint = 12345  # not produced by a forward
    st = lib.mst_mlp_backward(None, None, None, ctypes.byref(rec), None, None, None, None, None, None, None, 0,
                              None, 0)
    assert st == 6  # NULL ctx is reported as StateError too
    assert st in ms._STATUS and ms._STATUS[st] is ms.StateError


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    with pytest.raises(ms.Error):
        ms.Context(0)
