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


CPP_BIN = ROOT / "tests" / "cpp" / "_bin"


def build_cpp_device(ref_include: Path | None = None, out: Path | None = None) -> Path:
    """Compile tests/cpp/device_run.cpp (the C++ binding run on the GPU,
    tests/test_cpp_device.py) against libmst.so; with the reference's headers
    on the include path it forwards the library's memory events into the
    reference's own minitrain::MemTracker.  Host compile only (g++ + the
    CUDA runtime), so it builds here and travels to the GPU box prebuilt."""
    lib = build_lib()
    target = out or (CPP_BIN / "device_run")
    target.parent.mkdir(parents=True, exist_ok=True)
    cuda = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else (shutil.which("g++") or "g++")
    cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"), "-I", str(cuda / "include")]
    if ref_include is not None:
        cmd += ["-I", str(ref_include)]
    else:
        cmd += ["-DMST_STANDALONE_ERRORS"]
    cmd += [str(ROOT / "tests" / "cpp" / "device_run.cpp"), str(lib), f"-Wl,-rpath,{lib.parent}",
            "-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}", "-o", str(target)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return target


if __name__ == "__main__":
    import sys

    print(build_lib(force="-f" in sys.argv, verbose="-v" in sys.argv))
