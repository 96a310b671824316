"""B200-native split-format DFT (arXiv 2504.07264), drop-in for ``splitfft``.

The complex N-point DFT on separate real and imaginary planes, computed
through the paper's factorization -- I (x) H2 butterflies, diagonal cos/sin
rotations mixing the two planes, and the pairwise bit-reversal -- batched
over many signals in hand-written sm_100a CUDA kernels reached through the C
ABI in include/splitfft_b200.h.  The public names mirror the reference
package (splitfft/__init__.py:14-55); ``fft_split`` / ``ifft_split`` are the
batched planar ``(x_re, x_im) -> (y_re, y_im)`` entry points.
"""

__version__ = "0.1.0"

from .errors import CapacityError
from .layout import (
    InterleavedBuffer,
    SplitSignal,
    bit_reverse_index,
    bit_reverse_indices,
    deinterleave,
    interleave,
    is_power_of_two,
    permute_pairwise_bitrev,
)
from .transform import (
    MAX_PLAN_M,
    Algorithm,
    FftPlan,
    FlopReport,
    butterfly_stage,
    count_flops,
    fft,
    fft_dif,
    fft_dit,
    fft_split,
    ifft,
    ifft_split,
    make_plan,
    twiddle_stage,
)
from .twiddle import RotationBlock, RotationKind, build_twiddle_table, rotation_block

__all__ = [
    "Algorithm",
    "CapacityError",
    "FftPlan",
    "FlopReport",
    "InterleavedBuffer",
    "MAX_PLAN_M",
    "RotationBlock",
    "RotationKind",
    "SplitSignal",
    "bit_reverse_index",
    "bit_reverse_indices",
    "build_twiddle_table",
    "butterfly_stage",
    "count_flops",
    "deinterleave",
    "fft",
    "fft_dif",
    "fft_dit",
    "fft_split",
    "ifft",
    "ifft_split",
    "interleave",
    "is_power_of_two",
    "make_plan",
    "permute_pairwise_bitrev",
    "rotation_block",
    "twiddle_stage",
    "__version__",
]
