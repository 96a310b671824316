"""The reference's own tests against the drop-in (tests/refsuite.py).

CPU: test_layout.py + test_twiddle.py (containers, bit reversal, twiddle
tables -- no transform).  GPU: test_transform.py as well (every fft / ifft /
stage operator runs on the B200 through the shim).  Zero failures is the
bar; the staged copy is git-ignored and made from /root/reference by
``build()`` or by the CPU test itself.
"""

import pytest

import refsuite


def _require_staged():
    if not refsuite.stage():
        pytest.skip("reference suite not staged (needs /root/reference once, e.g. __graft_entry__.build())")


def test_reference_layout_and_twiddle_suites():
    _require_staged()
    rc, summary, out = refsuite.run(["test_layout.py", "test_twiddle.py"])
    assert rc == 0 and "failed" not in summary and "error" not in summary, out[-4000:]
    print(summary)


@pytest.mark.gpu
def test_reference_transform_suite_on_gpu(cuda):
    if not refsuite.staged():
        pytest.skip("reference suite not staged")
    rc, summary, out = refsuite.run(["test_layout.py", "test_twiddle.py", "test_transform.py"])
    assert rc == 0 and "failed" not in summary and "error" not in summary, out[-4000:]
    print(summary)
