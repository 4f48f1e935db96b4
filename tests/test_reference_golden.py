"""Pin the oracle against outputs of the REFERENCE itself.

tests/golden/reference_rng_memtrack.json was produced by compiling the
reference's own proj/include/minitrain/rng.hpp and memtrack.hpp (see
tests/golden/make_golden.py, oracle/Makefile target `ref`)."""
import json
from pathlib import Path

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_rng_memtrack.json").read_text())


def test_splitmix64_matches_reference(orc):
    assert [str(v) for v in orc.splitmix64_seq(42, 4)] == GOLD["splitmix64_seed42"]


def test_fnv1a64_matches_reference(orc):
    for k, v in GOLD["fnv1a64"].items():
        assert str(orc.fnv1a64(k)) == v


def test_xoshiro_streams_match_reference(orc):
    r = orc.OracleRng(0)
    assert [str(r.next_u64()) for _ in range(8)] == GOLD["xoshiro_seed0"]
    r = orc.OracleRng(1234)
    assert [str(r.next_u64()) for _ in range(8)] == GOLD["xoshiro_seed1234"]
    f = orc.OracleRng(1234).fork("X")
    assert [str(f.next_u64()) for _ in range(8)] == GOLD["xoshiro_seed1234_fork_X"]


def test_uniform_gaussian_below_match_reference_bitwise(orc):
    r = orc.OracleRng(7)
    assert [r.uniform() for _ in range(8)] == GOLD["uniform_seed7"]
    r = orc.OracleRng(7)
    assert [r.gaussian() for _ in range(8)] == GOLD["gaussian_seed7"]
    r = orc.OracleRng(99)
    assert [r.uniform_below(1000) for _ in range(8)] == GOLD["below_seed99_v1000"]


def test_counting_conventions_match_reference_memtrack(orc):
    m = GOLD["memtrack"]
    assert m["peak_10x10_f64"] == 800
    orc.counters_reset()
    orc.lib().orc_counters_reset()
    # count_matmul(8,4,16): reproduce through a real oracle matmul-bearing op is
    # not possible in isolation, so check the MLP example end to end instead.
    import numpy as np

    X = np.ones((8, 4))
    Wg = np.ones((4, 16))
    Wu = np.ones((4, 16))
    Wd = np.ones((16, 4))
    orc.counters_reset()
    orc.mlp_forward(X, Wg, Wu, Wd)
    c = orc.counters()
    assert c["matmul_flops"] == m["mlp_S8_d4_I16_flops"] == 3072
    assert c["weight_read_elements"] == m["mlp_S8_d4_I16_weight_reads"]
    assert m["flops_8_4_16"] == 2 * 8 * 4 * 16
