"""Host-side logic of the drop-in API (no GPU needed).

Mirrors the reference's validation tests (test_transform.py:232-264,
test_layout.py:22-169, test_twiddle.py) against the B200 package, checks the
host-built twiddle tables bit-for-bit against the reference's, and checks
that there is no CPU fallback.
"""

import os

import numpy as np
import pytest
import torch

import paper_2504_07264_b200 as sf
from paper_2504_07264_b200 import twiddle

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a, np.float64).view(np.int64),
                          np.ascontiguousarray(b, np.float64).view(np.int64))


@pytest.mark.parametrize("m", [1, 2, 3, 6, 12, 16])
def test_library_twiddles_match_reference_bitwise(m):
    wr, wi = twiddle.stage_factor_table(m)
    assert same_bits(wr, GOLD[f"stage_factor_m{m}_re"])
    assert same_bits(wi, GOLD[f"stage_factor_m{m}_im"])
    st = sf.build_twiddle_table(m).stage(m)
    assert same_bits(st.cos, GOLD[f"cos_m{m}"]) and same_bits(st.sin, GOLD[f"sin_m{m}"])


def test_stage_tables_are_strided_views_of_the_top_table():
    t = sf.build_twiddle_table(12)
    for i in range(1, 13):
        c, s = twiddle._snapped_cos_sin(i)
        assert same_bits(t.stage(i).cos, c) and same_bits(t.stage(i).sin, s)


def test_rotation_fixtures():
    # test_twiddle.py:20-54 and the omega^(3,3) erratum
    assert sf.rotation_block(1, 0).kind is sf.RotationKind.IDENTITY
    rb = sf.rotation_block(2, 1)
    assert rb.kind is sf.RotationKind.QUARTER_TURN and (rb.c, rb.s) == (0.0, 1.0)
    sq2 = np.sqrt(2.0) / 2.0
    rb = sf.rotation_block(3, 3)
    assert abs(rb.c + sq2) <= 1e-15 and abs(rb.s - sq2) <= 1e-15
    with pytest.raises(ValueError, match="out of range"):
        sf.rotation_block(3, 4)


@pytest.mark.parametrize("m", range(0, 21))
def test_count_flops_matches_reference_census(m):
    row = GOLD["census"][m]
    r = sf.count_flops(m)
    assert [r.real_mults, r.real_adds, r.generic_rotations, r.quarter_turns,
            r.identity_rotations] == row[1:].tolist()


def test_count_flops_eight_point_fixture():
    r = sf.count_flops(3)   # test_transform.py:308-314
    assert (r.generic_rotations, r.real_mults, r.quarter_turns, r.identity_rotations, r.real_adds) == \
        (2, 8, 2, 3, 48)


def test_plan_validation_messages():
    # test_transform.py:232-240 -- raised before any device work
    with pytest.raises(ValueError, match="must be >= 0"):
        sf.make_plan(-1)
    with pytest.raises(sf.CapacityError, match="exceeds the plan limit"):
        sf.make_plan(31)
    with pytest.raises(sf.CapacityError):
        sf.make_plan(9, max_m=8)
    with pytest.raises(ValueError):
        sf.make_plan(3, "fast")


def test_split_signal_validation():
    with pytest.raises(ValueError, match="channel lengths differ"):
        sf.SplitSignal(np.zeros(4), np.zeros(8))
    with pytest.raises(ValueError, match="one-dimensional"):
        sf.SplitSignal(np.zeros((2, 2, 2)), np.zeros((2, 2, 2)))
    s = sf.SplitSignal([1, 2], [3, 4])
    assert s.re.dtype == np.float64         # non-torch input: the reference's container (layout.py:29-30)
    assert sf.SplitSignal(np.ones(4, dtype=np.float32), np.ones(4)).re.dtype == np.float64
    with pytest.raises(ValueError, match="one-dimensional"):
        sf.SplitSignal(np.zeros((2, 4)), np.zeros((2, 4)))       # numpy: 1-D only, as the reference
    t = sf.SplitSignal(torch.zeros(2, 4, dtype=torch.float32), torch.zeros(2, 4, dtype=torch.float32))
    assert t.re.dtype == torch.float32 and t.batch == 2          # torch: the batched extension
    with pytest.raises(ValueError, match="not a power of two"):
        sf.interleave(sf.SplitSignal(np.zeros(6), np.zeros(6)))
    with pytest.raises(ValueError, match="does not match m"):
        sf.InterleavedBuffer(torch.zeros(10, dtype=torch.float64), 2)


def test_interleave_round_trip_is_bitwise():
    rng = np.random.default_rng(3)
    re = rng.standard_normal(16)
    im = rng.standard_normal(16)
    re[3] = -0.0
    im[5] = 5e-324
    buf = sf.interleave(sf.SplitSignal(re, im))
    assert buf.data[0::2].tolist() == re.tolist()
    back = sf.deinterleave(buf)
    assert same_bits(back.re, re) and same_bits(back.im, im)
    assert np.signbit(back.re[3])
    # torch containers: the same bits
    tb = sf.interleave(sf.SplitSignal(torch.from_numpy(re), torch.from_numpy(im)))
    tback = sf.deinterleave(tb)
    assert same_bits(tback.re.numpy(), re) and same_bits(tback.im.numpy(), im)


def test_bit_reverse_helpers():
    assert sf.bit_reverse_indices(3).tolist() == [0, 4, 2, 6, 1, 5, 3, 7]
    assert sf.bit_reverse_index(1, 3) == 4
    for m in (0, 3, 5, 10):
        assert np.array_equal(sf.bit_reverse_indices(m), GOLD[f"bitrev_m{m}"])
    buf = sf.InterleavedBuffer(torch.arange(16, dtype=torch.float64), 3)
    p = sf.permute_pairwise_bitrev(buf)
    assert p.data.view(8, 2)[:, 0].tolist() == [0.0, 8.0, 4.0, 12.0, 2.0, 10.0, 6.0, 14.0]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the behaviour without a GPU")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sf.fft_split(np.zeros(8), np.zeros(8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sf.make_plan(3)


def test_split_validation_happens_before_device_work():
    with pytest.raises(ValueError, match="not a power of two"):
        sf.fft_split(np.zeros(12), np.zeros(12))
    with pytest.raises(ValueError, match="channel lengths differ"):
        sf.fft_split(np.zeros(8), np.zeros(4))
