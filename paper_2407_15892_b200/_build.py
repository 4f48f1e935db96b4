"""Build recipes for the in-tree native artefacts.

`build_lib()` compiles the sm_100a product library `lib/libmst.so` (CUDA
kernels + C ABI, include/mst/mst.h) with nvcc.  The result is written inside
the package so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB_PATH = LIB_DIR / "libmst.so"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return cand


def lib_sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def lib_inputs() -> list[Path]:
    return lib_sources() + sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").rglob("*.h"))


def needs_rebuild(out: Path, inputs: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def build_lib(force: bool = False, verbose: bool = False, out: Path | None = None,
              defines: tuple[str, ...] = ()) -> Path:
    """Compile libmst.so (or a tuning variant at `out` with extra -D defines)."""
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    target = out or LIB_PATH
    if not force and not defines and not needs_rebuild(target, lib_inputs()):
        return target
    tmp = target.with_suffix(".so.tmp")
    cmd = [
        nvcc(), *ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
        "-I", str(ROOT / "include"), "-I", str(CSRC),
        "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines],
        "-o", str(tmp), *map(str, lib_sources()),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    import sys

    print(build_lib(force="-f" in sys.argv, verbose="-v" in sys.argv))
