"""Edge cases of the batched planar drop-in on the GPU (the reference's own
edge tests are 1-D: tests/test_gpu_reference_suite.py runs those): empty and
one-row batches, N = 1 and N = 2, ragged last tiles, non-contiguous and
misaligned planes on every size class (fused, TMA, multi-launch, L2-fused
pairs), shape / dtype / device mismatches, and the capacity limit.
All results are checked against the C oracle (fp64: bit for bit)."""

import numpy as np
import pytest
import torch

import paper_2504_07264_b200 as sf
from oracle import oracle

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def check64(yr, yi, re, im, algo="dit", inverse=False):
    wr, wi = oracle.fft_split_c(re, im, algo, inverse)
    assert np.array_equal(bits(yr.cpu().numpy()), bits(wr))
    assert np.array_equal(bits(yi.cpu().numpy()), bits(wi))


@pytest.mark.parametrize("m", [0, 1, 6, 10, 12, 14, 20])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_empty_batch(cuda, m, dtype):
    xr = torch.empty((0, 1 << m), dtype=dtype, device="cuda:0")
    xi = torch.empty((0, 1 << m), dtype=dtype, device="cuda:0")
    yr, yi = sf.fft_split(xr, xi)
    assert yr.shape == (0, 1 << m) and yi.shape == (0, 1 << m) and yr.dtype == dtype
    zr, zi = sf.ifft_split(yr, yi)
    assert zr.shape == (0, 1 << m)


@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_one_and_two_point_transforms(cuda, algo):
    rng = np.random.default_rng(8100)
    for m in (0, 1):
        re, im = rng.standard_normal((37, 1 << m)), rng.standard_normal((37, 1 << m))
        for inverse in (False, True):
            yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), algorithm=algo,
                                  inverse=inverse)
            check64(yr, yi, re, im, algo, inverse)
    # a single 1-D signal of one sample is its own transform
    yr, yi = sf.fft_split(torch.tensor([2.5], dtype=torch.float64, device="cuda:0"),
                          torch.tensor([-0.0], dtype=torch.float64, device="cuda:0"))
    assert yr.item() == 2.5 and np.signbit(yi.item()) == np.signbit(
        oracle.fft_split_c(np.array([[2.5]]), np.array([[-0.0]]), "dit", False)[1][0, 0])


@pytest.mark.parametrize("m,b", [(6, 1), (6, 257), (7, 33), (10, 1), (10, 10), (10, 1333), (12, 1), (12, 9),
                                 (14, 1), (14, 3), (20, 1)])
def test_one_row_and_ragged_batches_fp64(cuda, m, b):
    # batches that are not multiples of any tile / warp / CTA count, down to one row
    rng = np.random.default_rng(8200 + 31 * m + b)
    re, im = rng.standard_normal((b, 1 << m)), rng.standard_normal((b, 1 << m))
    for algo in ("dit", "dif"):
        yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), algorithm=algo)
        check64(yr, yi, re, im, algo)


@pytest.mark.parametrize("m", [6, 10, 12, 14, 20])
def test_misaligned_and_padded_rows_fp64(cuda, m):
    # planes that start 8 bytes into an allocation with an odd row stride: no
    # 16-byte alignment anywhere (the TMA / bulk-copy / cp.async paths must
    # fall back or cope), for the fused, multi-launch and L2-fused schedules
    rng = np.random.default_rng(8300 + m)
    b, n = 5, 1 << m
    stride = n + 3
    re, im = rng.standard_normal((b, n)), rng.standard_normal((b, n))
    bufr = torch.zeros(1 + b * stride, dtype=torch.float64, device="cuda:0")
    bufi = torch.zeros(1 + b * stride, dtype=torch.float64, device="cuda:0")
    xr = bufr[1:].view(b, stride)[:, :n]
    xi = bufi[1:].view(b, stride)[:, :n]
    xr.copy_(torch.from_numpy(re))
    xi.copy_(torch.from_numpy(im))
    assert xr.data_ptr() % 16 == 8
    kernels = ["auto"] + (["pass", "pass2"] if m == 20 else [])
    for kern in kernels:
        plan = sf.make_plan(m, dtype=torch.float64, device="cuda:0", kernel=kern)
        yr, yi = sf.fft_split(xr, xi, plan=plan)
        check64(yr, yi, re, im)
        # the same into a misaligned, padded output
        outr = torch.zeros(1 + b * stride, dtype=torch.float64, device="cuda:0")
        outi = torch.zeros(1 + b * stride, dtype=torch.float64, device="cuda:0")
        orr, oi = outr[1:].view(b, stride)[:, :n], outi[1:].view(b, stride)[:, :n]
        sf.fft_split(xr, xi, out=(orr, oi), plan=plan)
        check64(orr, oi, re, im)
        assert float(outr[0]) == 0.0 and float(outr[1:].view(b, stride)[:, n:].abs().max()) == 0.0   # padding untouched


def test_non_contiguous_planes_are_handled(cuda):
    # a transposed view (inner stride != 1) and planes with different strides
    rng = np.random.default_rng(8400)
    re, im = rng.standard_normal((64, 48)), rng.standard_normal((48, 64))
    xr = torch.from_numpy(re).cuda().t()            # [48, 64], inner stride 48
    xi = torch.from_numpy(im).cuda()                # [48, 64], contiguous
    yr, yi = sf.fft_split(xr, xi)
    check64(yr, yi, np.ascontiguousarray(re.T), im)


def test_mismatches_raise_before_any_launch(cuda):
    from paper_2504_07264_b200 import _ffi
    x = torch.zeros((4, 64), dtype=torch.float64, device="cuda:0")
    n0 = _ffi.launch_count()
    with pytest.raises(ValueError):
        sf.fft_split(x, torch.zeros((4, 32), dtype=torch.float64, device="cuda:0"))          # shapes differ
    with pytest.raises(ValueError):
        sf.fft_split(torch.zeros((4, 48), dtype=torch.float64, device="cuda:0"),
                     torch.zeros((4, 48), dtype=torch.float64, device="cuda:0"))              # not a power of two
    with pytest.raises(ValueError):
        sf.fft_split(x, x, plan=sf.make_plan(5, dtype=torch.float64, device="cuda:0"))        # plan for another N
    with pytest.raises(ValueError):
        sf.fft_split(x, x, plan=sf.make_plan(6, dtype=torch.float32, device="cuda:0"))        # plan for another dtype
    with pytest.raises(ValueError):
        sf.fft_split(x, x, out=(torch.zeros((4, 64), dtype=torch.float32, device="cuda:0"),) * 2)
    with pytest.raises(ValueError):
        sf.fft_split(x, x, out=(torch.zeros((3, 64), dtype=torch.float64, device="cuda:0"),) * 2)
    assert _ffi.launch_count() == n0


def test_capacity_limit_matches_the_reference(cuda):
    # make_plan's max_m guard (transform.py:32, 69-73): CapacityError, a ValueError subclass
    assert sf.MAX_PLAN_M == 30
    with pytest.raises(sf.CapacityError):
        sf.make_plan(31)
    with pytest.raises(sf.CapacityError):
        sf.make_plan(10, max_m=9)
    with pytest.raises(sf.CapacityError):
        sf.make_plan(31, max_m=40)       # beyond what the library addresses at all
    assert issubclass(sf.CapacityError, ValueError)
    assert sf.make_plan(20, max_m=20, dtype=torch.float32, device="cuda:0").sample_count == 1 << 20


def test_special_values_propagate_like_the_reference(cuda):
    # infinities, NaNs, signed zeros and denormals go through the same fp64
    # operations as the reference's: bit-identical results, NaN payloads aside
    rng = np.random.default_rng(8500)
    re, im = rng.standard_normal((6, 1024)), rng.standard_normal((6, 1024))
    re[0, 3], im[1, 7] = np.inf, -np.inf
    re[2, :] = 0.0
    im[2, :] = -0.0
    re[3, 5] = 5e-324
    im[3, 9] = -2.2250738585072014e-308
    re[4, 100] = np.nan
    yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda())
    wr, wi = oracle.fft_split_c(re, im, "dit", False)
    gr, gi = yr.cpu().numpy(), yi.cpu().numpy()
    for g, w in ((gr, wr), (gi, wi)):
        assert np.array_equal(np.isnan(g), np.isnan(w))
        ok = ~np.isnan(w)
        assert np.array_equal(bits(g[ok]), bits(w[ok]))
