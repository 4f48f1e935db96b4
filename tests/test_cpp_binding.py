"""The C++ drop-in header (include/mst/miniseq.hpp) compiles against libmst.so,
standalone and against the reference's own minitrain/error.hpp, and maps
status codes to the reference exception types (host-only, no GPU)."""
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2407_15892_b200 import LIB_PATH, build_lib

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")


def _cxx():
    return "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")


@pytest.mark.parametrize("with_reference", [False, True])
def test_cpp_binding(tmp_path, with_reference):
    if with_reference and not REF_INC.exists():
        pytest.skip("reference headers not mounted (GPU box)")
    build_lib()
    exe = tmp_path / "abi_smoke"
    cmd = [_cxx(), "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", str(ROOT / "include")]
    if with_reference:
        cmd += ["-I", str(REF_INC)]
    else:
        cmd += ["-DMST_STANDALONE_ERRORS"]
    cmd += [str(ROOT / "tests" / "cpp" / "abi_smoke.cpp"), str(LIB_PATH), f"-Wl,-rpath,{LIB_PATH.parent}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi_smoke OK" in out.stdout
    assert ("reference minitrain" in out.stdout) == with_reference
