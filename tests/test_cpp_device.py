"""The reference-facing C++ binding (include/mst/miniseq.hpp) executed on the
GPU: tests/cpp/device_run.cpp runs the SPEC ops one by
one and mst::block_step through the header, with the reference's own
minitrain::MemTracker attached when the binary was built against its headers
(__graft_entry__.build() does that in the container where /root/reference is
mounted; the prebuilt binary travels to the GPU box).  Every output must be
bitwise equal to the Python ctypes path over the same C ABI, and the tracked
peak of the "inter." chunk buffers must equal estimator.predict_block_peak."""
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2407_15892_b200 import estimator
from paper_2407_15892_b200 import miniseq as ms
from paper_2407_15892_b200._build import CPP_BIN, build_cpp_device

pytestmark = pytest.mark.gpu


def _binary(tmp_path: Path) -> Path:
    exe = CPP_BIN / "device_run"
    if exe.exists():
        return exe
    return build_cpp_device(None, tmp_path / "device_run")  # standalone (no reference headers on this host)


@pytest.mark.parametrize("shape", [(1024, 256, 688, 4096, 4, 4), (1000, 128, 256, 1000, 2, 10),
                                   (777, 64, 136, 520, 3, 5)])
def test_cpp_binding_on_device_bitwise_equal_to_python(orc, tmp_path, shape):
    N, H, I, V, Mm, Mh = shape
    c = orc.make_inputs(606, N, H, I, V, p_ignore=0.05)
    bf = {k: torch.from_numpy(c[k]).bfloat16() for k in ("X", "Wg", "Wu", "Wd", "Wout")}
    for k, t in bf.items():
        t.view(torch.int16).numpy().tofile(tmp_path / f"{k}.bf16")
    c["L"].astype(np.int32).tofile(tmp_path / "L.i32")
    out = subprocess.run([str(_binary(tmp_path)), str(tmp_path), *map(str, shape)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "device_run OK" in out.stdout, out.stdout + out.stderr

    def load(name, dtype, shape_):
        raw = np.fromfile(tmp_path / name, dtype=np.int16 if dtype == "bf16" else np.float32)
        t = torch.from_numpy(raw.reshape(shape_))
        return t.view(torch.bfloat16) if dtype == "bf16" else t

    g = {k: t.cuda() for k, t in bf.items()}
    L = torch.from_numpy(c["L"]).cuda()
    mlp, head = ms.MlpWeights(g["Wg"], g["Wu"], g["Wd"]), ms.LmHeadWeights(g["Wout"])
    # the SPEC ops through ctypes
    pm, ph = ms.make_chunk_plan(N, Mm), ms.make_chunk_plan(N, Mh)
    O, saved = ms.miniseq_mlp_forward(g["X"], mlp, pm)
    _, hs = ms.miniseq_lmhead_forward(O, L, head, ph)
    dO, dWo = ms.miniseq_lmhead_backward(hs, head, ph)
    dX, gr = ms.miniseq_mlp_backward(dO, saved, mlp, pm)
    torch.cuda.synchronize()
    nst = ms.stats_len(len(ph))
    for name, ref, dt, shp in (("ops_O", O, "bf16", (N, H)), ("ops_dO", dO, "bf16", (N, H)),
                               ("ops_dX", dX, "bf16", (N, H)), ("ops_lse", hs.lse, "f32", (N,)),
                               ("ops_stats", hs.stats, "f32", (nst,)), ("ops_dWg", gr.W_gate, "f32", (H, I)),
                               ("ops_dWu", gr.W_up, "f32", (H, I)), ("ops_dWd", gr.W_down, "f32", (I, H)),
                               ("ops_dWout", dWo, "f32", (H, V))):
        got = load(name + (".bf16" if dt == "bf16" else ".f32"), dt, shp)
        assert torch.equal(got, ref.cpu()), name
    # the fused block step
    ctx = ms.Context.get(0)
    ctx.reset_counters()
    st, bg = ms.block_step(g["X"], L, mlp, head, Mm, Mh)
    torch.cuda.synchronize()
    flops = ctx.counters().flops
    for name, ref, dt, shp in (("blk_dX", bg.dX, "bf16", (N, H)), ("blk_stats", st, "f32", (nst,)),
                               ("blk_dWg", bg.W_gate, "f32", (H, I)), ("blk_dWu", bg.W_up, "f32", (H, I)),
                               ("blk_dWd", bg.W_down, "f32", (I, H)), ("blk_dWout", bg.W_out, "f32", (H, V))):
        got = load(name + (".bf16" if dt == "bf16" else ".f32"), dt, shp)
        assert torch.equal(got, ref.cpu()), name
    if H % 128 == 0:  # attention through the header (device_run.cpp): q = X, k / v = column slices of X
        from paper_2407_15892_b200 import attention as A

        heads, kvh = H // 64, H // 128
        kvw = kvh * 64
        Xg = g["X"]
        ao, alse = A.attention_forward(Xg, Xg[:, :kvw], Xg[:, kvw:2 * kvw], 1, N, heads, kvh)
        dq, dk, dv = A.attention_backward(Xg, Xg[:, :kvw], Xg[:, kvw:2 * kvw], ao, O, alse, 1, N, heads, kvh)
        torch.cuda.synchronize()
        for name, ref, dt, shp in (("attn_o", ao, "bf16", (N, H)), ("attn_lse", alse.reshape(-1), "f32", (heads * N,)),
                                   ("attn_dq", dq, "bf16", (N, H)), ("attn_dk", dk, "bf16", (N, kvw)),
                                   ("attn_dv", dv, "bf16", (N, kvw))):
            got = load(name + (".bf16" if dt == "bf16" else ".f32"), dt, shp)
            assert torch.equal(got, ref.cpu()), name
    lines = dict(line.rsplit(" ", 1) for line in out.stdout.splitlines() if line.startswith("tracked"))
    if lines:  # built against the reference's minitrain/memtrack.hpp
        nested = {r[0] for r in pm.ranges} <= {r[0] for r in ph.ranges}
        if nested:
            assert int(lines["tracked inter. peak"]) == estimator.predict_block_peak(N, H, I, V, Mm, Mh)["inter."]
        assert int(lines["tracked block flops"]) == flops
