"""The host-side MemTracker mirror (paper_2407_15892_b200/memtrack.py) against
the reference's own memtrack.hpp, compiled here by oracle/Makefile target
`ref`: tests/golden/reference_rng_memtrack.json "memtrack" / "memtrack_script"
were produced by that binary (tests/golden/make_golden.py) running the same
script as `_script()` below."""
import io
import json
from pathlib import Path

import pytest

from paper_2407_15892_b200 import memtrack as mt

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_rng_memtrack.json").read_text())


def _script():
    """Mirror of the scripted session in oracle/ref_driver.cpp."""
    t = mt.MemTracker()
    t.on_alloc(64, "weights.w")
    t.region_begin("step")
    t.on_alloc(1000, "act.O")
    t.on_alloc(4000, "inter.mlp.h")
    t.on_alloc(8000, "inter.mlp.G")
    t.count_matmul(4, 8, 16, 128)
    t.count_op(64, 128)
    t.on_free(4000, "inter.mlp.h")
    t.on_alloc(2000, "inter.head.dlogits")
    t.region_begin("inner")
    t.on_alloc(500, "inter.head.partials")
    t.count_matmul(2, 3, 5)
    t.on_free(500, "inter.head.partials")
    inner = t.region_end("inner")
    t.on_free(8000, "inter.mlp.G")
    t.on_free(2000, "inter.head.dlogits")
    t.on_alloc(3000, "inter.mlp.h")
    t.on_free(3000, "inter.mlp.h")
    t.on_free(1000, "act.O")
    step = t.region_end("step")
    return t, step, inner


@pytest.mark.parametrize("name", ["step", "inner"])
def test_region_stats_match_reference(name):
    _, step, inner = _script()
    r = {"step": step, "inner": inner}[name]
    g = GOLD["memtrack_script"][name]
    assert r.report.peak_bytes() == g["peak"]
    assert r.report.final_live() == g["final_live"]
    assert r.report.entry_live == g["entry_live"]
    assert r.report.peak_for_prefix("inter.") == g["peak_inter"]
    assert r.report.peak_for_prefix("inter.mlp.") == g["peak_inter_mlp"]
    assert r.report.peak_excluding_prefix("inter.head.") == g["peak_excl_head"]
    assert r.report.peak_by_label() == g["peak_by_label"]
    assert list(r.counters.as_tuple()) == g["counters"]
    assert mt.export_timeline(r.report, io.StringIO()).splitlines() == g["timeline"]


def test_tracker_errors_match_reference():
    t, _, _ = _script()
    assert GOLD["memtrack_script"]["errors"] == {"free_exceeds_live": True, "region_mismatch": True}
    with pytest.raises(mt.StateError):
        t.on_free(1, "act.none")
    t.region_begin("a")
    with pytest.raises(mt.StateError):
        t.region_end("b")


def test_counting_kats_match_reference():
    g = GOLD["memtrack"]
    t = mt.MemTracker()
    t.region_begin("r")
    t.on_alloc(10 * 10 * 8, "act.x")
    t.on_free(10 * 10 * 8, "act.x")
    assert t.region_end("r").report.peak_bytes() == g["peak_10x10_f64"]
    t.region_begin("m")
    t.count_matmul(8, 4, 16)
    m = t.region_end("m").counters
    assert (m.flops, m.hbm_elements) == (g["flops_8_4_16"], g["hbm_8_4_16"])
    t.region_begin("mlp")
    t.count_matmul(8, 4, 16, 4 * 16)
    t.count_matmul(8, 4, 16, 4 * 16)
    t.count_matmul(8, 16, 4, 16 * 4)
    c = t.region_end("mlp").counters
    assert (c.flops, c.weight_read_elements) == (g["mlp_S8_d4_I16_flops"], g["mlp_S8_d4_I16_weight_reads"])


def test_timeline_file_export(tmp_path):
    _, step, _ = _script()
    p = tmp_path / "timeline.csv"
    mt.export_timeline(step.report, str(p))
    assert p.read_text().splitlines() == GOLD["memtrack_script"]["step"]["timeline"]
