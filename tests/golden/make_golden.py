"""Regenerate tests/golden/reference_rng_memtrack.json from the REFERENCE.

Compiles the reference's own header-only rng.hpp / memtrack.hpp from
/root/reference/proj/include via oracle/Makefile (target `ref`, output in
oracle/_ref/) and records its output.  Run here (the reference is not on
the GPU box); the JSON is committed.
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402


def main() -> None:
    oracle.build(ref=True)
    out = subprocess.run([str(oracle.REF_DRIVER)], capture_output=True, text=True, check=True).stdout
    data = json.loads(out)
    data["_source"] = "oracle/_ref/ref_driver compiled from /root/reference/proj/include (rng.hpp, memtrack.hpp)"
    dst = Path(__file__).with_name("reference_rng_memtrack.json")
    dst.write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()
