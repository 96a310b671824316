"""The reference's transform tests (pkg/tests/test_transform.py), run on the
GPU path through the drop-in API with the reference's own tolerances.

Each test cites the reference test it mirrors.  Inputs follow the reference's
conventions (seeded default_rng, standard normal re then im).  The checkers
are the oracle (tests/test_oracle_golden.py pins it to the reference) and
numpy's FFT where the reference itself uses it.
"""

import threading

import numpy as np
import pytest
import torch

import paper_2504_07264_b200 as sf
from oracle import oracle

pytestmark = pytest.mark.gpu
VARIANTS = ["dit", "dif"]


def _transform(re, im, m, algo, inverse=False):
    plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0")
    buf = sf.interleave(sf.SplitSignal(torch.as_tensor(re, dtype=torch.float64).cuda(),
                                       torch.as_tensor(im, dtype=torch.float64).cuda()))
    (sf.ifft if inverse else sf.fft)(plan, buf)
    out = sf.deinterleave(buf)
    return out.re.cpu().numpy(), out.im.cpu().numpy()


def _rand(rng, n):
    return rng.standard_normal(n), rng.standard_normal(n)


@pytest.mark.parametrize("m", range(0, 9))
@pytest.mark.parametrize("algo", VARIANTS)
def test_matches_naive_oracle(cuda, m, algo):
    # test_transform.py:82-93 (naive O(N^2) DFT, 1e-10 * (1 + max|y|))
    rng = np.random.default_rng(100 + m)
    n = 1 << m
    for _ in range(3):
        re, im = _rand(rng, n)
        gr, gi = _transform(re, im, m, algo)
        k = np.arange(n)
        ang = 2.0 * np.pi * (np.outer(k, k) % n) / n
        c, s = np.cos(ang), np.sin(ang)
        wr, wi = c @ re + s @ im, c @ im - s @ re
        scale = 1.0 + max(np.max(np.abs(wr)), np.max(np.abs(wi)))
        assert np.max(np.abs(gr - wr)) <= 1e-10 * scale and np.max(np.abs(gi - wi)) <= 1e-10 * scale


@pytest.mark.parametrize("m", [0, 1, 2, 3, 5, 7, 10, 13])
def test_matches_numpy_fft(cuda, m):
    # test_transform.py:96-104
    rng = np.random.default_rng(m)
    re, im = _rand(rng, 1 << m)
    ref = np.fft.fft(re + 1j * im)
    for algo in VARIANTS:
        gr, gi = _transform(re, im, m, algo)
        assert np.max(np.abs((gr + 1j * gi) - ref)) <= 1e-11 * (1.0 + np.max(np.abs(ref)))


@pytest.mark.parametrize("m", range(0, 12))
def test_dit_and_dif_agree(cuda, m):
    # test_transform.py:107-115
    rng = np.random.default_rng(7 * m + 1)
    re, im = _rand(rng, 1 << m)
    ar, ai = _transform(re, im, m, "dit")
    br, bi = _transform(re, im, m, "dif")
    scale = 1.0 + np.max(np.abs(ar + 1j * ai))
    assert np.max(np.abs(ar - br)) <= 1e-12 * scale and np.max(np.abs(ai - bi)) <= 1e-12 * scale


def test_linearity(cuda):
    # test_transform.py:170-183
    rng = np.random.default_rng(77)
    m, n = 6, 64
    for _ in range(10):
        xr, xi = _rand(rng, n)
        yr, yi = _rand(rng, n)
        a, b = rng.standard_normal(2)
        fx = _transform(xr, xi, m, "dit")
        fy = _transform(yr, yi, m, "dit")
        fc = _transform(a * xr + b * yr, a * xi + b * yi, m, "dit")
        scale = 1.0 + np.max(np.abs(fc[0] + 1j * fc[1]))
        assert np.max(np.abs(fc[0] - (a * fx[0] + b * fy[0]))) <= 1e-10 * scale
        assert np.max(np.abs(fc[1] - (a * fx[1] + b * fy[1]))) <= 1e-10 * scale


@pytest.mark.parametrize("m", [0, 1, 4, 8, 11])
def test_parseval(cuda, m):
    # test_transform.py:186-194
    rng = np.random.default_rng(m + 3)
    n = 1 << m
    re, im = _rand(rng, n)
    gr, gi = _transform(re, im, m, "dit")
    te = np.sum(re ** 2 + im ** 2)
    fe = np.sum(gr ** 2 + gi ** 2) / n
    assert abs(te - fe) <= 1e-9 * (1.0 + te)


@pytest.mark.parametrize("m", [1, 3, 6, 10])
def test_conjugate_symmetry_for_real_input(cuda, m):
    # test_transform.py:197-205
    rng = np.random.default_rng(m + 13)
    n = 1 << m
    gr, gi = _transform(rng.standard_normal(n), np.zeros(n), m, "dit")
    scale = 1.0 + np.max(np.abs(gr + 1j * gi))
    mirror = (-np.arange(n)) % n
    assert np.max(np.abs(gr - gr[mirror])) <= 1e-10 * scale
    assert np.max(np.abs(gi + gi[mirror])) <= 1e-10 * scale


@pytest.mark.parametrize("m", [0, 1, 5, 9, 12])
@pytest.mark.parametrize("algo", VARIANTS)
def test_ifft_inverts_fft(cuda, m, algo):
    # test_transform.py:208-220 (in place on one InterleavedBuffer)
    rng = np.random.default_rng(m + 29)
    re, im = _rand(rng, 1 << m)
    plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0")
    buf = sf.interleave(sf.SplitSignal(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda()))
    sf.fft(plan, buf)
    sf.ifft(plan, buf)
    back = sf.deinterleave(buf)
    scale = 1.0 + np.max(np.abs(re + 1j * im))
    assert np.max(np.abs(back.re.cpu().numpy() - re)) <= 1e-10 * scale
    assert np.max(np.abs(back.im.cpu().numpy() - im)) <= 1e-10 * scale


def test_buffer_plan_size_mismatch(cuda):
    # test_transform.py:249-256
    plan = sf.make_plan(3, device="cuda:0")
    buf = sf.interleave(sf.SplitSignal(torch.zeros(4, dtype=torch.float64).cuda(),
                                       torch.zeros(4, dtype=torch.float64).cuda()))
    for op in (sf.fft, sf.fft_dit, sf.fft_dif, sf.ifft):
        with pytest.raises(ValueError, match="buffer is for m=2"):
            op(plan, buf)


def test_plans_are_thread_safe(cuda):
    # test_transform.py:267-290: one plan, 4 host threads x 20 transforms,
    # each on its own buffers and its own stream
    m = 10
    rng = np.random.default_rng(4)
    re, im = _rand(rng, 1 << m)
    plan = sf.make_plan(m, dtype=torch.float64, device="cuda:0")
    xr, xi = torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda()
    er, ei = sf.fft_split(xr, xi, plan=plan)
    torch.cuda.synchronize()
    failures = []

    def worker():
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(20):
                yr, yi = sf.fft_split(xr.clone(), xi.clone(), plan=plan)
                s.synchronize()
                if not (torch.equal(yr, er) and torch.equal(yi, ei)):
                    failures.append(1)

    threads = [threading.Thread(target=worker) for _ in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not failures


def test_empty_batch_and_single_row(cuda):
    x = torch.zeros(0, 64, device="cuda:0")
    yr, yi = sf.fft_split(x, x)
    assert yr.shape == (0, 64)
    one = torch.randn(1, 64, device="cuda:0", dtype=torch.float64)
    a = sf.fft_split(one, one)
    b = sf.fft_split(one[0], one[0])
    assert torch.equal(a[0][0], b[0]) and torch.equal(a[1][0], b[1])


def test_oracle_agreement_many_random_inputs(cuda):
    # test_acceptance.py:67-89 (m = 1..12, 100 random inputs per size, both
    # variants, 1e-10 bound) -- one batched GPU call per size and variant
    rng = np.random.default_rng(1234)
    for m in range(1, 13):
        re = rng.standard_normal((100, 1 << m))
        im = rng.standard_normal((100, 1 << m))
        for algo in VARIANTS:
            plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0")
            gr, gi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), plan=plan)
            wr, wi = oracle.fft_split_c(re, im, algo)
            bound = 1e-10 * (1.0 + np.maximum(np.abs(wr).max(axis=1), np.abs(wi).max(axis=1)))
            dev = np.maximum(np.abs(gr.cpu().numpy() - wr).max(axis=1), np.abs(gi.cpu().numpy() - wi).max(axis=1))
            assert np.all(dev <= bound)
