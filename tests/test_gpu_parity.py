"""GPU parity: the CUDA path through the C ABI vs the pinned CPU oracle.

fp64: bit-for-bit equality with the oracle, which is itself bit-identical to
the reference (tests/test_oracle_golden.py), so fp64 GPU == reference.
fp32: relative L2 <= 1e-5 * log2 N against the fp64 oracle on the same
fp32-rounded inputs (BASELINE.json north_star tolerance).
"""

import numpy as np
import pytest
import torch

import paper_2504_07264_b200 as sf
from oracle import oracle

pytestmark = pytest.mark.gpu

F32_TOL = lambda m: 1e-5 * max(m, 1)   # noqa: E731  north_star: <= 1e-5*log2N


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def rel_l2(got_re, got_im, want_re, want_im):
    num = np.sqrt(np.sum((got_re - want_re) ** 2 + (got_im - want_im) ** 2))
    den = np.sqrt(np.sum(want_re ** 2 + want_im ** 2))
    return num / max(den, 1e-300)


def rand(rng, b, n, dtype):
    re = rng.standard_normal((b, n)).astype(dtype)
    im = rng.standard_normal((b, n)).astype(dtype)
    return re, im


def gpu_split(re, im, algo="dit", inverse=False, radix_log=0, kernel="auto", prefetch=None):
    dt = torch.float32 if re.dtype == np.float32 else torch.float64
    m = re.shape[-1].bit_length() - 1
    plan = sf.make_plan(m, algo, dtype=dt, device="cuda:0", radix_log=radix_log, kernel=kernel,
                        prefetch_factors=prefetch)
    xr = torch.from_numpy(re).cuda()
    xi = torch.from_numpy(im).cuda()
    yr, yi = sf.fft_split(xr, xi, inverse=inverse, plan=plan)
    torch.cuda.synchronize()
    return yr.cpu().numpy(), yi.cpu().numpy()


FUSED_M = list(range(0, 13))
LARGE_M = [13, 14, 16, 17, 20, 22]


@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("algo", ["dit", "dif"])
@pytest.mark.parametrize("m", FUSED_M + LARGE_M)
def test_f64_bitwise_vs_oracle(cuda, m, algo, inverse):
    rng = np.random.default_rng(1000 + m)
    b = 37 if m <= 12 else 3          # batch not a multiple of the CTA tile
    re, im = rand(rng, b, 1 << m, np.float64)
    gr, gi = gpu_split(re, im, algo, inverse)
    wr, wi = oracle.fft_split_c(re, im, algo, inverse)
    assert np.array_equal(bits(gr), bits(wr)), f"re differs, max abs {np.abs(gr - wr).max()}"
    assert np.array_equal(bits(gi), bits(wi)), f"im differs, max abs {np.abs(gi - wi).max()}"


@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("algo", ["dit", "dif"])
@pytest.mark.parametrize("m", FUSED_M + LARGE_M)
def test_f32_rel_l2_vs_oracle(cuda, m, algo, inverse):
    rng = np.random.default_rng(2000 + m)
    b = 37 if m <= 12 else 3
    re, im = rand(rng, b, 1 << m, np.float32)
    gr, gi = gpu_split(re, im, algo, inverse)
    wr, wi = oracle.fft_split_c(re, im, algo, inverse)
    err = rel_l2(gr.astype(np.float64), gi.astype(np.float64), wr, wi)
    assert err <= F32_TOL(m), f"relL2 {err:.3e} > {F32_TOL(m):.1e}"


@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("algo", ["dit", "dif"])
@pytest.mark.parametrize("m,lr", [(m, lr) for m in (4, 5, 6, 7, 9, 10, 11, 12) for lr in (2, 3, 4, 5)
                                  if (1 << (m - min(lr, m))) <= 1024])
def test_every_radix_schedule(cuda, m, lr, algo, dtype, prefetch):
    if dtype == np.float64 and prefetch:
        pytest.skip("fp64 reads every factor from the table")
    rng = np.random.default_rng(3000 + 16 * m + lr)
    re, im = rand(rng, 19, 1 << m, dtype)
    gr, gi = gpu_split(re, im, algo, False, radix_log=lr, kernel="ldg", prefetch=prefetch)
    wr, wi = oracle.fft_split_c(re, im, algo, False)
    if dtype == np.float64:
        assert np.array_equal(bits(gr), bits(wr)) and np.array_equal(bits(gi), bits(wi))
    else:
        assert rel_l2(gr.astype(np.float64), gi.astype(np.float64), wr, wi) <= F32_TOL(m)


@pytest.mark.parametrize("m", [3, 6, 10, 12, 14])
@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_interleaved_in_place_matches_split(cuda, m, algo):
    rng = np.random.default_rng(4000 + m)
    b = 5
    re, im = rand(rng, b, 1 << m, np.float64)
    data = np.empty((b, 2 << m))
    data[:, 0::2] = re
    data[:, 1::2] = im
    plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0")
    buf = sf.InterleavedBuffer(torch.from_numpy(data).cuda(), m)
    sf.fft(plan, buf)
    out = buf.data.cpu().numpy()
    wr, wi = oracle.fft_split_c(re, im, algo, False)
    assert np.array_equal(bits(out[:, 0::2]), bits(wr))
    assert np.array_equal(bits(out[:, 1::2]), bits(wi))
    sf.ifft(plan, buf)
    back = buf.data.cpu().numpy()
    assert np.max(np.abs(back - data)) <= 1e-12 * (1 + np.abs(data).max())


@pytest.mark.parametrize("m", [6, 10, 13])
def test_in_place_and_strided_rows(cuda, m):
    rng = np.random.default_rng(5000 + m)
    n = 1 << m
    wide_re = torch.from_numpy(rng.standard_normal((9, n + 64))).cuda()
    wide_im = torch.from_numpy(rng.standard_normal((9, n + 64))).cuda()
    xr, xi = wide_re[:, 32:32 + n], wide_im[:, 32:32 + n]   # row stride n + 64
    want = oracle.fft_split_c(xr.cpu().numpy(), xi.cpu().numpy())
    yr, yi = sf.fft_split(xr, xi, out=(xr, xi))             # in place, strided
    torch.cuda.synchronize()
    assert yr.data_ptr() == xr.data_ptr()
    assert np.array_equal(bits(xr.cpu().numpy()), bits(want[0]))
    assert np.array_equal(bits(xi.cpu().numpy()), bits(want[1]))
    # the pad columns were not touched
    assert torch.equal(wide_re[:, :32], torch.from_numpy(np.asarray(wide_re[:, :32].cpu())).cuda())


def test_host_arrays_round_trip_through_gpu(cuda):
    # numpy in -> numpy out, computed on the GPU (reference-style call)
    rng = np.random.default_rng(6)
    re, im = rng.standard_normal(64), rng.standard_normal(64)
    yr, yi = sf.fft_split(re, im)
    assert isinstance(yr, np.ndarray)
    wr, wi = oracle.fft_split_c(re, im)
    assert np.array_equal(bits(yr), bits(wr)) and np.array_equal(bits(yi), bits(wi))


# ---- the reference's inline known answers, on the GPU ---------------------

def _known(re, im, m, algo="dit", dtype=torch.float64, inverse=False):
    plan = sf.make_plan(m, algo, dtype=dtype, device="cuda:0")
    xr = torch.tensor(re, dtype=dtype, device="cuda:0")
    xi = torch.tensor(im, dtype=dtype, device="cuda:0")
    yr, yi = sf.fft_split(xr, xi, plan=plan, inverse=inverse)
    return yr.cpu().tolist(), yi.cpu().tolist()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_known_answers(cuda, algo, dtype):
    # impulse -> ones (test_transform.py:41-47)
    assert _known([1.0] + [0.0] * 7, [0.0] * 8, 3, algo, dtype) == ([1.0] * 8, [0.0] * 8)
    # constant 2.5 -> 40 delta (test_transform.py:50-54)
    assert _known([2.5] * 16, [0.0] * 16, 4, algo, dtype) == ([40.0] + [0.0] * 15, [0.0] * 16)
    # 4-point ramp (test_transform.py:57-62, README.md:41-47)
    assert _known([1.0, 2.0, 3.0, 4.0], [0.0] * 4, 2, algo, dtype) == (
        [10.0, -2.0, -2.0, -2.0], [0.0, 2.0, 0.0, -2.0])
    # N = 1 identity (test_transform.py:76-79)
    assert _known([3.5], [-1.25], 0, algo, dtype) == ([3.5], [-1.25])
    # ifft(ones) = delta (test_transform.py:223-229)
    assert _known([1.0] * 8, [0.0] * 8, 3, algo, dtype, inverse=True) == ([1.0] + [0.0] * 7, [0.0] * 8)


def test_single_tone(cuda):
    # test_transform.py:65-73
    n = 16
    t = 2.0 * np.pi * np.arange(n) / n
    yr, yi = _known(np.cos(t).tolist(), np.sin(t).tolist(), 4)
    want = np.zeros(n)
    want[1] = n
    assert np.max(np.abs(np.array(yr) - want)) <= 1e-13 * n
    assert np.max(np.abs(np.array(yi))) <= 1e-13 * n


def test_launches_are_counted(cuda):
    from paper_2504_07264_b200 import _ffi
    before = _ffi.launch_count()
    x = torch.zeros(4, 64, device="cuda:0")
    sf.fft_split(x, x)
    torch.cuda.synchronize()
    assert _ffi.launch_count() == before + 1


# ---- the TMA-fed persistent kernel vs the LDG kernel vs the oracle -----------

TMA_CASES = [("f32", m, lr) for m, lrs in {5: [3], 6: [3, 2], 7: [3, 4], 8: [3, 4], 9: [3, 4],
                                            10: [4, 3, 5], 11: [4, 3], 12: [4, 3, 6]}.items() for lr in lrs] + \
            [("f64", m, lr) for m, lrs in {4: [2], 5: [3], 6: [3], 7: [3, 4], 8: [3, 4], 9: [3],
                                            10: [3, 4, 5], 11: [4]}.items() for lr in lrs]


@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("algo", ["dit", "dif"])
@pytest.mark.parametrize("dt,m,lr", TMA_CASES)
def test_tma_kernel_many_tiles(cuda, dt, m, lr, algo, prefetch):
    if dt == "f64" and prefetch:
        pytest.skip("fp64 reads every factor from the table")
    # enough rows for several tiles per persistent CTA (stage and output-buffer
    # reuse) plus a ragged tail tile
    dtype = np.float32 if dt == "f32" else np.float64
    tdt = torch.float32 if dt == "f32" else torch.float64
    b = (1 << 22 >> m) + 3
    rng = np.random.default_rng(7000 + m + 31 * lr)
    re, im = rand(rng, b, 1 << m, dtype)
    plan = sf.make_plan(m, algo, dtype=tdt, device="cuda:0", radix_log=lr, kernel="tma",
                        prefetch_factors=prefetch)
    assert plan.kernel == "tma"
    xr, xi = torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda()
    for inverse in (False, True):
        yr, yi = sf.fft_split(xr, xi, plan=plan, inverse=inverse)
        gr, gi = yr.cpu().numpy(), yi.cpu().numpy()
        wr, wi = oracle.fft_split_c(re, im, algo, inverse)
        if dt == "f64":
            assert np.array_equal(bits(gr), bits(wr)) and np.array_equal(bits(gi), bits(wi))
        else:
            assert rel_l2(gr.astype(np.float64), gi.astype(np.float64), wr, wi) <= F32_TOL(m)
            # and bit-identical to the LDG kernel (same arithmetic, other data
            # path); radix 64 (the signal-group kernel) has no LDG twin
            if lr > 5:
                continue
            ldg = sf.make_plan(m, algo, dtype=tdt, device="cuda:0", radix_log=lr, kernel="ldg",
                               prefetch_factors=prefetch)
            lr_, li_ = sf.fft_split(xr, xi, plan=ldg, inverse=inverse)
            assert torch.equal(lr_, yr) and torch.equal(li_, yi)


@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_warp_kernel_long_persistent_loop(cuda, algo):
    # fp64 N = 1024 radix 32 (sfft_tma_warp.cuh): ~40 signals per warp, so
    # both slots of every warp are refilled many times (in-place exchange in
    # the slot, bulk-copy refill after the exchange read), ragged tail, row
    # strides > N on both sides
    m, b = 10, 148 * 7 * 40 + 5
    rng = np.random.default_rng(9100)
    re, im = rand(rng, b, 1 << m, np.float64)
    pad_in, pad_out = 1024 + 32, 1024 + 64
    xr = torch.zeros(b, pad_in, dtype=torch.float64, device="cuda:0")
    xi = torch.zeros_like(xr)
    xr[:, :1024] = torch.from_numpy(re).cuda()
    xi[:, :1024] = torch.from_numpy(im).cuda()
    plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0", radix_log=5, kernel="tma")
    for inverse in (False, True):
        yr = torch.full((b, pad_out), 7.0, dtype=torch.float64, device="cuda:0")
        yi = torch.full_like(yr, 7.0)
        sf.fft_split(xr[:, :1024], xi[:, :1024], plan=plan, inverse=inverse, out=(yr[:, :1024], yi[:, :1024]))
        wr, wi = oracle.fft_split_c(re, im, algo, inverse)
        assert np.array_equal(bits(yr[:, :1024].cpu().numpy()), bits(wr))
        assert np.array_equal(bits(yi[:, :1024].cpu().numpy()), bits(wi))
        assert bool((yr[:, 1024:] == 7.0).all()) and bool((yi[:, 1024:] == 7.0).all())


@pytest.mark.parametrize("b", [1, 5, 9, 10, 11, 148 * 9 + 1, 148 * 10 * 3 + 7])
def test_warp_kernel_small_and_ragged_batches(cuda, b):
    # the slot ring with fewer signals than slots / warps, partial last
    # rounds and idle warps (they still meet the CTA's final barrier)
    rng = np.random.default_rng(9300 + b)
    re, im = rand(rng, b, 1024, np.float64)
    xr, xi = torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda()
    for algo in ("dit", "dif"):
        plan = sf.make_plan(10, algo, dtype=torch.float64, device="cuda:0", radix_log=5, kernel="tma")
        assert plan.exec_kernel(b)[2] == "sfft_tmaw_kernel"
        for inverse in (False, True):
            yr, yi = sf.fft_split(xr, xi, plan=plan, inverse=inverse)
            wr, wi = oracle.fft_split_c(re, im, algo, inverse)
            assert np.array_equal(bits(yr.cpu().numpy()), bits(wr))
            assert np.array_equal(bits(yi.cpu().numpy()), bits(wi))


def test_auto_batch_switch_fp64_n1024(cuda):
    # kernel=auto switches fp64 N = 1024 between the radix-8 TMA kernel (small
    # batches) and the warp-per-signal radix-32 kernel (>= 2^16 rows); both
    # are the reference's arithmetic, so results are bitwise equal either way
    plan = sf.make_plan(10, "dit", dtype=torch.float64, device="cuda:0")
    assert plan.exec_kernel(1 << 16) == ("tma", 5, "sfft_tmaw_kernel")
    assert plan.exec_kernel((1 << 16) - 1) == ("tma", 3, "sfft_tma_kernel")
    assert plan.exec_kernel(1 << 16, interleaved=True)[0] == "ldg"
    # fp32 N = 4096: the two-warp radix-64 signal-group kernel from 2^13 rows,
    # the LDG radix-16 kernel below
    p32 = sf.make_plan(12, "dit", dtype=torch.float32, device="cuda:0")
    assert p32.exec_kernel(1 << 13) == ("tma", 6, "sfft_tmaw_kernel")
    assert p32.exec_kernel((1 << 13) - 1)[0] == "ldg"
    rng = np.random.default_rng(9200)
    b = 1 << 16
    re, im = rand(rng, b, 1024, np.float64)
    xr, xi = torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda()
    big_r, big_i = sf.fft_split(xr, xi, plan=plan)
    small_r, small_i = sf.fft_split(xr[:4096], xi[:4096], plan=plan)
    assert torch.equal(big_r[:4096], small_r) and torch.equal(big_i[:4096], small_i)
    wr, wi = oracle.fft_split_c(re[:4096], im[:4096])
    assert np.array_equal(bits(small_r.cpu().numpy()), bits(wr))
    assert np.array_equal(bits(small_i.cpu().numpy()), bits(wi))


def test_tma_falls_back_for_unaligned_rows(cuda):
    m = 6
    rng = np.random.default_rng(8)
    base_r = torch.from_numpy(rng.standard_normal(64 * 100 + 1).astype(np.float32)).cuda()
    base_i = torch.from_numpy(rng.standard_normal(64 * 100 + 1).astype(np.float32)).cuda()
    xr, xi = base_r[1:].view(100, 64), base_i[1:].view(100, 64)     # 4-byte aligned only
    plan = sf.make_plan(m, dtype=torch.float32, device="cuda:0")
    assert plan.kernel == "tma"
    yr, yi = sf.fft_split(xr, xi, plan=plan)                         # auto -> LDG path
    wr, wi = oracle.fft_split_c(xr.cpu().numpy(), xi.cpu().numpy())
    assert rel_l2(yr.cpu().numpy().astype(np.float64), yi.cpu().numpy().astype(np.float64), wr, wi) <= 6e-5
    forced = sf.make_plan(m, dtype=torch.float32, device="cuda:0", kernel="tma")
    with pytest.raises(ValueError, match="TMA kernel needs"):
        sf.fft_split(xr, xi, plan=forced)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_pipeline_many_chunks(cuda, monkeypatch, pinned):
    # host planes go through the chunked H2D/compute/D2H pipeline; force many
    # chunks (and a ragged last one) and compare with the device-resident path
    from paper_2504_07264_b200 import transform
    monkeypatch.setattr(transform, "_PIPE_CHUNK_BYTES", 64 * 4 * 1000)
    rng = np.random.default_rng(11)
    b, n = 10007, 64
    re = torch.from_numpy(rng.standard_normal((b, n)).astype(np.float32))
    im = torch.from_numpy(rng.standard_normal((b, n)).astype(np.float32))
    if pinned:
        re, im = re.pin_memory(), im.pin_memory()
    out_r = torch.empty_like(re)
    out_i = torch.empty_like(im)
    for inverse in (False, True):
        sf.fft_split(re, im, out=(out_r, out_i), inverse=inverse)
        dr, di = sf.fft_split(re.cuda(), im.cuda(), inverse=inverse)
        assert torch.equal(out_r, dr.cpu()) and torch.equal(out_i, di.cpu())


PASS_VARIANTS = {"plain": {}, "split_8_5": {"SFFT_PASS_SPLIT": "8,5"}}


@pytest.mark.parametrize("variant", sorted(PASS_VARIANTS))
@pytest.mark.parametrize("algo", ["dit", "dif"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m", [13, 16, 20])
def test_pass_kernel_variants(cuda, m, dtype, algo, variant):
    # the pass schedule in a subprocess: default group split, and (m = 13
    # only) an unbalanced split through the developer knob
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, sys
sys.path.insert(0, {repr(__import__('os').path.dirname(__import__('os').path.dirname(__file__)))})
import paper_2504_07264_b200 as sf
from oracle import oracle
rng = np.random.default_rng({m})
re = rng.standard_normal((3, 1 << {m})).astype(np.{np.dtype(dtype).name})
im = rng.standard_normal((3, 1 << {m})).astype(np.{np.dtype(dtype).name})
for inv in (False, True):
    yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), algorithm="{algo}", inverse=inv)
    wr, wi = oracle.fft_split_c(re, im, "{algo}", inv)
    gr, gi = yr.cpu().numpy().astype(np.float64), yi.cpu().numpy().astype(np.float64)
    if re.dtype == np.float64:
        assert np.array_equal(gr.view(np.int64), wr.view(np.int64)) and np.array_equal(gi.view(np.int64), wi.view(np.int64))
    else:
        err = np.sqrt(np.sum((gr - wr) ** 2 + (gi - wi) ** 2) / np.sum(wr ** 2 + wi ** 2))
        assert err <= 1e-5 * {m}, err
print("ok")
"""
    env = dict(__import__('os').environ, **PASS_VARIANTS[variant])
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("m", [6, 10, 14])
def test_cuda_graph_capture_and_replay(cuda, m):
    # exec is a pure stream-ordered launch sequence (no sync, no allocation
    # in the C ABI), so it can be captured in a CUDA graph and replayed
    rng = np.random.default_rng(12)
    xr = torch.from_numpy(rng.standard_normal((64, 1 << m)).astype(np.float32)).cuda()
    xi = torch.from_numpy(rng.standard_normal((64, 1 << m)).astype(np.float32)).cuda()
    plan = sf.make_plan(m, dtype=torch.float32, device="cuda:0")
    yr, yi = torch.empty_like(xr), torch.empty_like(xi)
    sf.fft_split(xr, xi, out=(yr, yi), plan=plan)          # warm up outside the capture
    want = (yr.clone(), yi.clone())
    yr.zero_()
    yi.zero_()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(yr, want[0]) and torch.equal(yi, want[1])


# ---- the GPU pinned straight to the reference at m > 14 (no oracle in the
# loop): SHA-256 of the fp64 output bytes equals the reference's
# (tests/golden/reference_large_pins.json; the reference's stage-pair slab
# path, transform.py:160-200, 227-237)
def _large_pins():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "reference_large_pins.json")) as f:
        return json.load(f)["pins"]


@pytest.mark.parametrize("tag", sorted(_large_pins()))
def test_gpu_fp64_large_m_matches_reference_digest(cuda, tag):
    import hashlib
    pin = _large_pins()[tag]
    m = int(tag.split("_")[0][1:])
    algo, inv = tag.split("_")[1], tag.endswith("inv")
    rng = np.random.default_rng(5000 + m)
    re, im = rng.standard_normal(1 << m), rng.standard_normal(1 << m)
    plan = sf.make_plan(m, algo, dtype=torch.float64, device="cuda:0")
    yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), plan=plan, inverse=inv)
    gr, gi = yr.cpu().numpy(), yi.cpu().numpy()
    d = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()   # noqa: E731
    assert d(gr) == pin["sha256_re"] and d(gi) == pin["sha256_im"]


# ---- the literal per-stage operators (transform.py:88-120) on the GPU ----
@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("m", [1, 3, 8, 13, 14])
def test_stage_operators_batched_torch(cuda, dt, m):
    # batched torch buffers (the extension) equal the reference-mode numpy
    # buffers row by row; composed with the bit reversal they give fft_dit /
    # fft_dif (fp64: bit for bit)
    tdt = torch.float64 if dt == "f64" else torch.float32
    rng = np.random.default_rng(70 + m)
    b = 3
    data = rng.standard_normal((b, 2 << m))
    plan = sf.make_plan(m, "dit", dtype=tdt, device="cuda:0")
    for i in range(1, m + 1):
        t = sf.InterleavedBuffer(torch.from_numpy(data).to("cuda:0", tdt), m)
        sf.butterfly_stage(t, i)
        sf.twiddle_stage(t, plan, i)
        for r in range(b):
            nb = sf.InterleavedBuffer(data[r].astype(np.float32 if dt == "f32" else np.float64), m)
            sf.butterfly_stage(nb, i)
            sf.twiddle_stage(nb, plan, i)
            got = t.data[r].cpu().numpy().astype(np.float64)
            if dt == "f64":
                assert np.array_equal(got, nb.data)
            else:
                assert np.max(np.abs(got - nb.data)) <= 1e-5 * (1 + np.abs(nb.data).max())
    if dt == "f64":
        sig = sf.SplitSignal(data[0, 0::2].copy(), data[0, 1::2].copy())
        fast = sf.interleave(sig)
        sf.fft_dit(plan, fast)
        slow = sf.permute_pairwise_bitrev(sf.interleave(sig))
        for i in range(1, m + 1):
            sf.twiddle_stage(slow, plan, i)
            sf.butterfly_stage(slow, i)
        assert np.array_equal(fast.data, slow.data)


def test_numpy_containers_follow_the_reference(cuda):
    # fp32 numpy input is upcast to float64 and computed in fp64, like
    # layout.py:29-30 -- through the default plan and through fft_split
    rng = np.random.default_rng(3)
    re = rng.standard_normal(256).astype(np.float32)
    im = rng.standard_normal(256).astype(np.float32)
    buf = sf.interleave(sf.SplitSignal(re, im))
    assert buf.data.dtype == np.float64
    sf.fft(sf.make_plan(8), buf)
    out = sf.deinterleave(buf)
    wr, wi = oracle.fft_split_c(re.astype(np.float64), im.astype(np.float64))
    assert np.array_equal(out.re, wr) and np.array_equal(out.im, wi)
    yr, yi = sf.fft_split(re, im)
    assert yr.dtype == np.float64 and np.array_equal(yr, wr) and np.array_equal(yi, wi)
