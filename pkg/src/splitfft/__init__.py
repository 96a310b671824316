"""``splitfft`` import shim for the B200 package (north_star: the reference's
public transform functions stay in pkg/src).

``import splitfft`` here resolves to ``paper_2504_07264_b200`` -- the same
names (splitfft/__init__.py:14-55), with every transform executed by the
sm_100a kernels through the C ABI -- and its submodules
``splitfft.layout``, ``splitfft.transform``, ``splitfft.twiddle``,
``splitfft.errors``, ``splitfft.signalio`` and ``splitfft.cli`` are the
package's own modules, so ``from splitfft.transform import fft`` keeps
working after ``PYTHONPATH=pkg/src``.

Not provided (outside the GPU hot path): the dense O(4^m)
proof tools (``densealg``, ``verify_factorization``), the O(N^2) test oracle
(``oracle.naive_dft``), the CPU wall-clock harness (``bench``) and the
/verify and /bench service routes.
"""

import importlib
import os
import sys

try:
    import paper_2504_07264_b200 as _pkg
except ImportError:   # repo checkout: the package sits three levels up
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
    import paper_2504_07264_b200 as _pkg

from paper_2504_07264_b200 import *  # noqa: F401,F403,E402
from paper_2504_07264_b200 import __all__, __version__  # noqa: F401,E402

for _name in ("layout", "transform", "twiddle", "errors", "signalio", "cli"):
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"paper_2504_07264_b200.{_name}")
    globals()[_name] = sys.modules[f"{__name__}.{_name}"]

_OUT_OF_SCOPE = {"naive_dft": "splitfft.oracle (the reference's O(N^2) test oracle)",
                 "verify_factorization": "splitfft.densealg (the dense O(4^m) proof tool)"}


def __getattr__(name):
    if name in _OUT_OF_SCOPE:
        raise AttributeError(f"splitfft.{name} is not part of the B200 drop-in: {_OUT_OF_SCOPE[name]} is "
                             "outside the GPU hot path (SURVEY.md sec. 2)")
    raise AttributeError(f"module 'splitfft' has no attribute {name!r}")
