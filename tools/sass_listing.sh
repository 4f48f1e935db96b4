#!/bin/bash
# Commit-able SASS evidence for libmst.so (north star: "a committed SASS listing").
# Writes profiles/sass/<kernel>.sass per kernel function and a mnemonic census
# (tcgen05 -> UTC*MMA / LDTM, TMA -> UTMALDG / UTMASTG / UTMAREDG) in
# profiles/sass/SUMMARY.md.  usage: tools/sass_listing.sh [lib]
set -e
lib=${1:-paper_2407_15892_b200/lib/libmst.so}
out=profiles/sass
mkdir -p $out
cuobjdump -sass $lib > /tmp/mst_all.sass
python3 - "$out" <<'PY'
import re, sys, collections
out = sys.argv[1]
txt = open('/tmp/mst_all.sass').read()
funcs = re.split(r'\n\s*Function : ', txt)[1:]
lines = ["# SASS census of libmst.so (sm_100a, cuobjdump -sass)", "",
         "| kernel | SASS lines | UTC*MMA | LDTM | UTMALDG | UTMASTG | UTMAREDG | HMMA (legacy) |", "|---|---|---|---|---|---|---|---|"]
for f in funcs:
    name = f.split('\n', 1)[0].strip()
    body = f
    short = re.sub(r'[^A-Za-z0-9_]+', '_', name)[:80]
    cnt = lambda pat: len(re.findall(pat, body))
    n = body.count('\n')
    lines.append(f"| `{name[:70]}` | {n} | {cnt(r'UTC[A-Z]*MMA')} | {cnt(r'LDTM')} | {cnt(r'UTMALDG')} | {cnt(r'UTMASTG')} | {cnt(r'UTMAREDG')} | {cnt(r' HMMA')} |")
    if 'grouped_gemm' in name:
        import gzip; gzip.open(f"{out}/mst_grouped_gemm_kernel.sass.gz", "wt").write("Function : " + f)
ops = collections.Counter(re.findall(r'\b(UTC[A-Z]*MMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG[.A-Z0-9]*|UTMAREDG[.A-Z0-9]*|LDTM[.A-Z0-9x]*|UTCBAR[.A-Z0-9]*)', txt))
lines += ["", "Distinct tcgen05 / TMA mnemonics in the library:", ""] + [f"* `{k}` x{v}" for k, v in sorted(ops.items())]
open(f"{out}/SUMMARY.md", 'w').write("\n".join(lines) + "\n")
print("\n".join(lines))
PY
