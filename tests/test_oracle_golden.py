"""Pin the CPU oracle to the reference: every golden vector, bit for bit.

tests/golden/reference_vectors.npz was written by the reference's own public
API (tests/golden/make_golden.py).  Both oracle restatements -- the C port
(liboracle.so) and the numpy port of the executor -- must reproduce it
exactly, signed zeros included; only then is the oracle trusted as the GPU
checker.
"""

import os

import numpy as np
import pytest

from oracle import oracle

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


CASES = [(m, algo, inv) for m in list(range(0, 13)) + [13, 14] for algo in ("dit", "dif")
         for inv in (False, True)]


@pytest.mark.parametrize("m,algo,inv", CASES)
def test_c_oracle_bitwise(m, algo, inv):
    tag = f"m{m}_{algo}_{'inv' if inv else 'fwd'}"
    yr, yi = oracle.fft_split_c(GOLD[f"m{m}_x_re"], GOLD[f"m{m}_x_im"], algo, inv)
    assert same_bits(yr, GOLD[tag + "_re"]) and same_bits(yi, GOLD[tag + "_im"])


@pytest.mark.parametrize("m,algo,inv", [c for c in CASES if c[0] <= 14])
def test_numpy_port_bitwise(m, algo, inv):
    tag = f"m{m}_{algo}_{'inv' if inv else 'fwd'}"
    yr, yi = oracle.fft_split_numpy(GOLD[f"m{m}_x_re"], GOLD[f"m{m}_x_im"], algo, inv)
    assert same_bits(yr, GOLD[tag + "_re"]) and same_bits(yi, GOLD[tag + "_im"])


@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_config1_full_batch(algo):
    # BASELINE configs[0]: N=8 fp64 B=1024, the reference's own CPU case
    yr, yi = oracle.fft_split_c(GOLD["cfg1_x_re"], GOLD["cfg1_x_im"], algo)
    assert same_bits(yr, GOLD[f"cfg1_{algo}_re"]) and same_bits(yi, GOLD[f"cfg1_{algo}_im"])


@pytest.mark.parametrize("name", ["cfg2_n64_f32", "cfg3_n1024_f32", "cfg3_n1024_f64", "cfg4_n4096_f32"])
def test_config_prefixes(name):
    xr = GOLD[f"{name}_x_re"]
    xi = GOLD[f"{name}_x_im"]
    yr, yi = oracle.fft_split_c(xr, xi, "dit")
    assert same_bits(yr, GOLD[f"{name}_dit_re"]) and same_bits(yi, GOLD[f"{name}_dit_im"])


@pytest.mark.parametrize("m", [1, 2, 3, 6, 12, 16])
def test_oracle_tables(m):
    w = oracle.stage_factors(m)[m - 1]
    assert same_bits(w.real, GOLD[f"stage_factor_m{m}_re"])
    assert same_bits(w.imag, GOLD[f"stage_factor_m{m}_im"])
    c, s = oracle.cos_sin(m)
    assert same_bits(c, GOLD[f"cos_m{m}"]) and same_bits(s, GOLD[f"sin_m{m}"])


@pytest.mark.parametrize("m", [0, 3, 5, 10])
def test_oracle_bitrev(m):
    assert np.array_equal(oracle.bitrev(m), GOLD[f"bitrev_m{m}"])


def test_golden_known_answer_4_point():
    # the reference's printed example (test_transform.py:57-62): sanity of the file itself
    yr, yi = oracle.fft_split_c(np.array([1.0, 2.0, 3.0, 4.0]), np.zeros(4))
    assert yr.tolist() == [10.0, -2.0, -2.0, -2.0] and yi.tolist() == [0.0, 2.0, 0.0, -2.0]


# ---- m > 14: the reference's stage-pair slab path (transform.py:160-200,
# 227-237), pinned by SHA-256 of the reference's output bytes
# (tests/golden/reference_large_pins.json, written by make_golden.py --large)
import hashlib  # noqa: E402
import json  # noqa: E402

LARGE = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_large_pins.json")))["pins"]


def large_input(m):
    rng = np.random.default_rng(5000 + m)
    return rng.standard_normal(1 << m), rng.standard_normal(1 << m)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


@pytest.mark.parametrize("tag", sorted(LARGE))
def test_c_oracle_large_m_pins(tag):
    m = int(tag.split("_")[0][1:])
    algo, inv = tag.split("_")[1], tag.endswith("inv")
    re, im = large_input(m)
    yr, yi = oracle.fft_split_c(re, im, algo, inv)
    pin = LARGE[tag]
    idx = np.array(pin["sample_index"])
    assert same_bits(yr[idx], np.array(pin["sample_re"])) and same_bits(yi[idx], np.array(pin["sample_im"]))
    assert digest(yr) == pin["sha256_re"] and digest(yi) == pin["sha256_im"]
