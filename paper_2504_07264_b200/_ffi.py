"""ctypes binding of the C ABI in include/splitfft_b200.h.

The shared library ``libsplitfft_b200.so`` sits next to this file (built by
``__graft_entry__.build()`` / ``make -C paper_2504_07264_b200/csrc``).  There
is no fallback: if the library is missing, importing the package fails with
the build command in the message.
"""

import ctypes
import os

from .errors import CapacityError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsplitfft_b200.so")
# developer knob (A/B of two builds on one box, tools/p2_sweep.py): another build of the same library
LIB_PATH = os.environ.get("SFFT_B200_LIB", LIB_PATH)

SFFT_OK, SFFT_EINVAL, SFFT_ECAPACITY, SFFT_ECUDA = 0, 1, 2, 3
SFFT_F32, SFFT_F64 = 0, 1
SFFT_DIT, SFFT_DIF = 0, 1
SFFT_FORWARD, SFFT_INVERSE = -1, 1
SFFT_MAX_LOG2N = 30
SFFT_KERNEL_AUTO, SFFT_KERNEL_LDG, SFFT_KERNEL_TMA, SFFT_KERNEL_PASS, SFFT_KERNEL_PASS2 = 0, 1, 2, 3, 4
ABI_VERSION = 1

# every symbol include/splitfft_b200.h declares: name -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
SIGNATURES = {
    "sfft_abi_version": (_I, []),
    "sfft_last_error": (ctypes.c_char_p, []),
    "sfft_plan_create": (_I, [_I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "sfft_plan_create_ex": (_I, [_I, _I, _I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "sfft_plan_destroy": (_I, [_P]),
    "sfft_plan_info": (_I, [_P] + [ctypes.POINTER(_I)] * 7),
    "sfft_workspace_bytes": (_I, [_P, _I64, ctypes.POINTER(ctypes.c_size_t)]),
    "sfft_exec_schedule": (_I, [_P, _I64, _I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "sfft_exec_kernel": (_I, [_P, _I64, _I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                             ctypes.POINTER(ctypes.c_int)]),
    "sfft_exec_split": (_I, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I, _P, _P]),
    "sfft_exec_interleaved": (_I, [_P, _P, _P, _I64, _I64, _I64, _I, _P, _P]),
    "sfft_exec_butterfly_stage": (_I, [_I, _I, _I, _P, _I64, _I64, _I, _P]),
    "sfft_exec_twiddle_stage": (_I, [_P, _I, _P, _I64, _I64, _P]),
    "sfft_twiddle_table": (_I, [_I, _P, _P]),
    "sfft_count_flops": (_I, [_I, ctypes.POINTER(_I64)]),
    "sfft_launch_count": (_I64, []),
    "sfft_dist_plan_create": (_I, [_I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "sfft_dist_plan_destroy": (_I, [_P]),
    "sfft_dist_layout": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I), ctypes.POINTER(_I64)]),
    "sfft_dist_workspace_bytes": (_I, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "sfft_dist_schedule": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "sfft_dist_exec_phase": (_I, [_P, _I, _P, _P, _P, _P, _I, _P, _P]),
    "sfft_dist_exec_phase0_p2p": (_I, [_P, _P, _P, ctypes.POINTER(_P), ctypes.POINTER(_P), _I, _I, _P, _P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2504_07264_b200/csrc` (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sfft_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.sfft_abi_version()} != {ABI_VERSION}")
    return lib


lib = _load()


def check(status: int) -> None:
    """Map a C status to the reference's exception types."""
    if status == SFFT_OK:
        return
    msg = lib.sfft_last_error().decode("utf-8", "replace")
    if status == SFFT_EINVAL:
        raise ValueError(msg)
    if status == SFFT_ECAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib.sfft_launch_count())


# Optional NVTX ranges around the exec calls and the sharded phases
# (SFFT_NVTX=1; off by default: a range push/pop costs a few microseconds per
# exec, comparable to a small launch).  Timelines: nsys / ncu --nvtx.
NVTX = os.environ.get("SFFT_NVTX", "0") == "1"


class nvtx_range:
    """``with nvtx_range("name"):`` -- a no-op unless SFFT_NVTX=1."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if NVTX:
            import torch
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        if NVTX:
            import torch
            torch.cuda.nvtx.range_pop()
        return False
