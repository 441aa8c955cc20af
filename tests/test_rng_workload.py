"""splitmix64 and arrival streams vs the reference's golden vectors
(tests/test_rng.py:15-37 of the reference; fixtures from make_golden.py)."""

import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2603_14371_b200 import SplitMix64, WorkloadSpec, generate_arrivals
from paper_2603_14371_b200.rng import counter_u64, counter_uniform

ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle_splitmix.so")


def test_published_check_values(golden):
    g = golden("rng.json")
    r = SplitMix64(0)
    assert [r.next_u64() for _ in range(5)] == [int(x) for x in g["seed0_u64"]]
    assert int(g["seed0_u64"][0]) == 0xE220A8397B1DCDAF
    r = SplitMix64(0xDEADBEEF)
    assert [r.next_u64() for _ in range(3)] == [int(x) for x in g["deadbeef_u64"]]


def test_streams_match_reference(golden):
    g = golden("rng.json")
    r = SplitMix64(7)
    assert [r.next_u64() for _ in range(64)] == [int(x) for x in g["seed7_u64"]]
    r = SplitMix64(7)
    assert [r.uniform() for _ in range(64)] == g["seed7_uniform"]
    r = SplitMix64(9)
    assert [r.below(10) for _ in range(50)] == g["seed9_below10"]
    r = SplitMix64(11)
    assert [r.poisson(2.5) for _ in range(50)] == g["seed11_poisson2.5"]


def test_counter_form_is_the_stream(golden):
    g = golden("rng.json")
    assert counter_u64(7, 0, 64).tolist() == [int(x) for x in g["seed7_u64"]]
    assert counter_uniform(7, 0, 64).tolist() == g["seed7_uniform"]
    r = SplitMix64(7)
    r.skip(40)
    assert r.next_u64() == int(g["seed7_u64"][40])


def test_oracle_counter_form_is_the_stream(golden):
    """The oracle's own restatement (oracle/rng_ref.py) is pinned to the same
    reference vectors, independently of the product's rng module."""
    from oracle import rng_ref
    g = golden("rng.json")
    assert rng_ref.counter_u64(7, 0, 64).tolist() == [int(x) for x in g["seed7_u64"]]
    assert rng_ref.counter_uniform(7, 0, 64).tolist() == g["seed7_uniform"]
    assert rng_ref.counter_u64(0, 0, 5).tolist() == [int(x) for x in g["seed0_u64"]]
    assert rng_ref.counter_u64(0xDEADBEEF, 0, 3).tolist() == [int(x) for x in g["deadbeef_u64"]]


def test_below_and_poisson_guards():
    with pytest.raises(ValueError, match="positive bound"):
        SplitMix64(1).below(0)
    with pytest.raises(ValueError, match="nonnegative"):
        SplitMix64(1).poisson(-1.0)
    assert SplitMix64(1).poisson(0.0) == 0


@pytest.fixture(scope="module")
def oracle_c():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)
    lib = C.CDLL(ORACLE_SO)
    return lib


def test_c_oracle_matches_golden(golden, oracle_c):
    g = golden("rng.json")
    out = np.zeros(64, np.uint64)
    oracle_c.oracle_splitmix_u64(C.c_uint64(7), C.c_int64(64), out.ctypes.data_as(C.c_void_p))
    assert out.tolist() == [int(x) for x in g["seed7_u64"]]
    w = np.zeros(64, np.float64)
    oracle_c.oracle_toy_weights(C.c_uint64(7), C.c_int64(0), C.c_int64(64),
                                w.ctypes.data_as(C.c_void_p))
    assert w.tolist() == [-0.1 + 0.2 * u for u in g["seed7_uniform"]]


def test_arrivals_match_reference(golden):
    for case in golden("workload.json"):
        got = generate_arrivals(WorkloadSpec(**case["spec"]), case["vocab"])
        assert [[a.frame, a.n_tokens, list(a.observation.obs_tokens)] for a in got] == \
            case["arrivals"]


@pytest.mark.parametrize("kw, msg", [
    (dict(pattern="Bogus"), "unknown pattern"),
    (dict(num_frames=-1), "nonnegative"),
    (dict(default_N=0), "budgets"),
    (dict(p_long=1.5), "p_long"),
    (dict(obs_len=0), "obs_len"),
])
def test_workload_validation(kw, msg):
    with pytest.raises(ValueError, match=msg):
        WorkloadSpec(**kw)


def test_rates_and_budgets():
    assert WorkloadSpec(pattern="Uniform", r=3).arrivals_per_frame == 3.0
    assert WorkloadSpec(pattern="Poisson", lam=0.7).arrivals_per_frame == 0.7
    assert WorkloadSpec(pattern="MixedLength", short_N=3, long_N=9).max_budget == 9
    assert WorkloadSpec(pattern="MixedLength", short_N=3, long_N=9, p_long=0.0).max_budget == 3
    assert generate_arrivals(WorkloadSpec(pattern="Uniform", r=0, num_frames=5)) == []
