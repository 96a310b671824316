"""The seeded synthetic inputs (workloads.py) follow the stated convention."""

import numpy as np

import workloads


def test_chunked_draws_equal_one_shot_draws():
    cfg = workloads.Config("t", 6, 300, "f64", 1, "normal")
    workloads_chunk = workloads._CHUNK_ELEMS
    try:
        workloads._CHUNK_ELEMS = 64 * 7          # force many chunks
        re, im = workloads.generate(cfg)
    finally:
        workloads._CHUNK_ELEMS = workloads_chunk
    rng = np.random.default_rng(1)
    assert np.array_equal(re, rng.standard_normal((300, 64)))
    assert np.array_equal(im, rng.standard_normal((300, 64)))


def test_prefix_rows_are_the_full_stream_prefix():
    cfg = workloads.Config("t", 4, 100, "f64", 2, "uniform")
    full = workloads.generate(cfg)
    part = workloads.generate(cfg, rows=7)
    assert np.array_equal(full[0][:7], part[0]) and np.array_equal(full[1][:7], part[1])


def test_config_shapes_and_dtypes():
    c = workloads.CONFIGS
    assert (c["cfg1_n8_f64"].n, c["cfg1_n8_f64"].batch, c["cfg1_n8_f64"].dtype) == (8, 1024, "f64")
    assert (c["cfg2_n64_f32"].n, c["cfg2_n64_f32"].batch) == (64, 1 << 20)
    assert (c["cfg3_n1024_f32"].n, c["cfg3_n1024_f32"].batch) == (1024, 1 << 18)
    assert (c["cfg4_n4096_f32"].n, c["cfg4_n4096_f32"].batch) == (4096, 1 << 16)
    assert c["cfg5_n2p28_f32"].n == 1 << 28
    re, im = workloads.generate(c["cfg1_n8_f64"])
    assert re.shape == (1024, 8) and re.dtype == np.float64
    assert re.min() >= -1.0 and re.max() < 1.0
    assert c["cfg2_n64_f32"].algorithmic_bytes == 1 << 30


def test_tone_config_has_its_tones():
    from oracle import oracle
    cfg = workloads.CONFIGS["cfg4_n4096_f32"]
    re, im = workloads.generate(cfg, rows=3)
    k, amp, _ = workloads.tone_params(cfg, np.random.default_rng(cfg.seed))
    yr, yi = oracle.fft_split_c(re, im)
    mag = np.hypot(yr, yi)
    for b in range(3):
        for kk in np.unique(k[b]):
            want = cfg.n * amp[b][k[b] == kk]
            # |y[k_j]| ~ N * A_j (tones sharing a bin add with their phases)
            if len(want) == 1:
                assert abs(mag[b, kk] - want[0]) <= 0.01 * want[0] + 5.0
