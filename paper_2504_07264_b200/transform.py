"""Plans and transforms on the GPU (mirrors splitfft/transform.py).

Public surface kept from the reference: ``MAX_PLAN_M``, ``Algorithm``,
``FftPlan``, ``make_plan``, ``fft``, ``fft_dit``, ``fft_dif``, ``ifft``,
``FlopReport``, ``count_flops`` (transform.py:32-335), plus the batched
split->split drop-in ``fft_split`` / ``ifft_split`` -- the planar
``(x_re, x_im) -> (y_re, y_im)`` form of the reference's service path
(service/app.py:43-52).

Every transform runs on the GPU through the C ABI (``_ffi``); there is no
CPU fallback.  Host inputs (numpy arrays, CPU tensors) are copied to the
current CUDA device, transformed there and copied back, so reference users
can switch without touching their arrays; with no CUDA device the call
raises.
"""

import enum
import ctypes
import threading
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _ffi
from .errors import CapacityError
from .layout import InterleavedBuffer, SplitSignal, bit_reverse_indices, is_power_of_two
from .twiddle import TwiddleTable, build_twiddle_table, stage_factor_table

MAX_PLAN_M = _ffi.SFFT_MAX_LOG2N   # transform.py:32

_DTYPE_CODE = {torch.float32: _ffi.SFFT_F32, torch.float64: _ffi.SFFT_F64}


class Algorithm(enum.Enum):
    DIT = "dit"
    DIF = "dif"


def _resolve_device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("splitfft-b200 needs a CUDA device (there is no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError(f"plans live on a CUDA device, got {device} (there is no CPU fallback)")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


class FftPlan:
    """Device-resident tables for transforms of one size (transform.py:46-62).

    Immutable and safe to share across threads; every call works on its own
    buffers (and its own workspace for log2 N > 12).
    """

    __slots__ = ("m", "algorithm", "dtype", "device", "_handle", "_lock", "_tables", "__weakref__")

    def __init__(self, m, algorithm, dtype, device, handle):
        object.__setattr__(self, "m", m)
        object.__setattr__(self, "algorithm", algorithm)
        object.__setattr__(self, "dtype", dtype)
        object.__setattr__(self, "device", device)
        object.__setattr__(self, "_handle", handle)
        object.__setattr__(self, "_lock", threading.Lock())
        object.__setattr__(self, "_tables", None)

    def __setattr__(self, name, value):
        raise AttributeError("FftPlan is immutable")

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                _ffi.lib.sfft_plan_destroy(h)
            except Exception:
                pass

    def __repr__(self):
        return (f"FftPlan(m={self.m}, algorithm={self.algorithm}, dtype={self.dtype}, "
                f"device={self.device}, kernel={self.kernel}, radix=2^{self.radix_log}, "
                f"launches={self.launches_per_exec})")

    @property
    def sample_count(self) -> int:
        return 1 << self.m

    def _info(self):
        vals = [ctypes.c_int() for _ in range(7)]
        _ffi.check(_ffi.lib.sfft_plan_info(self._handle, *[ctypes.byref(v) for v in vals]))
        return [v.value for v in vals]

    @property
    def launches_per_exec(self) -> int:
        return self._info()[4]

    def schedule(self, batch: int = 1, interleaved: bool = False):
        """(kernel launches, HBM sweeps) one exec of `batch` rows uses."""
        nl, ns = ctypes.c_int(), ctypes.c_int()
        _ffi.check(_ffi.lib.sfft_exec_schedule(self._handle, int(batch), int(bool(interleaved)),
                                               ctypes.byref(nl), ctypes.byref(ns)))
        return nl.value, ns.value

    def exec_kernel(self, batch: int = 1, interleaved: bool = False):
        """(family, log2 radix, kernel name) of the kernel one exec of `batch`
        aligned planar rows launches (kernel='auto' switches by batch size)."""
        fam, lr, warp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _ffi.check(_ffi.lib.sfft_exec_kernel(self._handle, int(batch), int(bool(interleaved)),
                                             ctypes.byref(fam), ctypes.byref(lr), ctypes.byref(warp)))
        family = {_ffi.SFFT_KERNEL_TMA: "tma", _ffi.SFFT_KERNEL_LDG: "ldg", _ffi.SFFT_KERNEL_PASS: "pass",
                  _ffi.SFFT_KERNEL_PASS2: "pass2"}[fam.value]
        name = ("sfft_tmaw_kernel" if warp.value else
                {"tma": "sfft_tma_kernel", "ldg": "sfft_fused_kernel", "pass": "sfft_pass_kernel",
                 "pass2": "sfft_pass2_kernel"}[family])
        return family, lr.value, name

    @property
    def radix_log(self) -> int:
        return self._info()[5]

    @property
    def kernel(self) -> str:
        """Kernel family used for aligned planar rows: 'tma', 'ldg', 'pass' or
        'pass2' (the L2-fused group pairs)."""
        return {_ffi.SFFT_KERNEL_TMA: "tma", _ffi.SFFT_KERNEL_LDG: "ldg",
                _ffi.SFFT_KERNEL_PASS: "pass", _ffi.SFFT_KERNEL_PASS2: "pass2"}[self._info()[6]]

    def workspace_bytes(self, batch: int) -> int:
        out = ctypes.c_size_t()
        _ffi.check(_ffi.lib.sfft_workspace_bytes(self._handle, int(batch), ctypes.byref(out)))
        return int(out.value)

    # host-side views the reference exposes on its plan (read-only)
    @property
    def twiddles(self) -> TwiddleTable:
        return build_twiddle_table(self.m)

    @property
    def bitrev(self) -> np.ndarray:
        idx = bit_reverse_indices(self.m)
        idx.flags.writeable = False
        return idx

    @property
    def stage_factors(self) -> tuple:
        """Host copies of w_i = cos - j sin per stage (transform.py:80-84)."""
        if self.m == 0:
            return ()
        wr, wi = stage_factor_table(self.m)
        out = []
        for i in range(1, self.m + 1):
            step = 1 << (self.m - i)
            w = np.empty(1 << (i - 1), dtype=np.complex128)
            w.real = wr[::step]
            w.imag = wi[::step]
            w.flags.writeable = False
            out.append(w)
        return tuple(out)


def make_plan(m: int, algorithm=Algorithm.DIT, *, max_m: int = MAX_PLAN_M,
              dtype=torch.float64, device=None, radix_log: int = 0, kernel: str = "auto",
              prefetch_factors=None) -> FftPlan:
    """Build an FftPlan for 2**m samples on a CUDA device (transform.py:65-85).

    Same validation order and messages as the reference: m < 0 -> ValueError,
    m > max_m -> CapacityError, unknown algorithm -> ValueError.  ``dtype`` is
    the plane dtype (float64 like the reference, or float32); ``radix_log``
    overrides the register radix of the fused kernel (0 = tuned default);
    ``kernel`` picks the fused kernel family: "auto" (TMA-fed when the rows
    allow it), "ldg" (per-thread loads) or "tma" (required); for m > 12
    "pass" forces one launch per stage group and "pass2" (20 <= m <= 28,
    planar rows) the L2-fused group pairs (auto takes them for fp64 m = 28);
    ``prefetch_factors`` (fp32) forces fetching each pass's base factors
    before the data on/off (None = tuned default).
    """
    if m < 0:
        raise ValueError(f"stage count m must be >= 0, got {m}")
    if m > max_m:
        raise CapacityError(f"m={m} exceeds the plan limit max_m={max_m}")
    algorithm = Algorithm(algorithm) if not isinstance(algorithm, Algorithm) else algorithm
    if dtype not in _DTYPE_CODE:
        raise ValueError(f"dtype must be torch.float32 or torch.float64, got {dtype}")
    device = _resolve_device(device)
    kernels = {"auto": _ffi.SFFT_KERNEL_AUTO, "ldg": _ffi.SFFT_KERNEL_LDG, "tma": _ffi.SFFT_KERNEL_TMA,
               "pass": _ffi.SFFT_KERNEL_PASS, "pass2": _ffi.SFFT_KERNEL_PASS2}
    if kernel not in kernels:
        raise ValueError(f"kernel must be one of {sorted(kernels)}, got {kernel!r}")
    kcode = kernels[kernel] | {None: 0, False: 0x10, True: 0x20}[prefetch_factors]
    handle = ctypes.c_void_p()
    algo = _ffi.SFFT_DIF if algorithm is Algorithm.DIF else _ffi.SFFT_DIT
    _ffi.check(_ffi.lib.sfft_plan_create_ex(int(m), _DTYPE_CODE[dtype], algo, device.index,
                                            int(min(max_m, MAX_PLAN_M)),
                                            int(radix_log), kcode, ctypes.byref(handle)))
    return FftPlan(m, algorithm, dtype, device, handle.value)


@lru_cache(maxsize=32)
def _cached_plan(m, algorithm, dtype, device_index):
    # plan cache of the service path (service/app.py:28-30)
    return make_plan(m, algorithm, dtype=dtype, device=torch.device("cuda", device_index))


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _rows(t: torch.Tensor):
    """(batch, row stride) of a [N] or [B, N] tensor with unit inner stride."""
    if t.ndim == 1:
        return 1, t.shape[0]
    return t.shape[0], t.stride(0)


def _workspace(plan: FftPlan, batch: int):
    nbytes = plan.workspace_bytes(batch)
    if nbytes == 0:
        return None, 0
    ws = torch.empty(nbytes, dtype=torch.uint8, device=plan.device)
    return ws, ws.data_ptr()


def _exec_split_device(plan, xr, xi, yr, yi, inverse):
    batch, istr = _rows(xr)
    _, ostr = _rows(yr)
    ws, wsp = _workspace(plan, batch)
    direction = _ffi.SFFT_INVERSE if inverse else _ffi.SFFT_FORWARD
    with _ffi.nvtx_range("sfft_exec_split"):
        _ffi.check(_ffi.lib.sfft_exec_split(plan._handle, xr.data_ptr(), xi.data_ptr(), yr.data_ptr(),
                                            yi.data_ptr(), batch, istr, ostr, direction, wsp,
                                            _stream_ptr(plan.device)))
    if ws is not None:
        ws.record_stream(torch.cuda.current_stream(plan.device))


def _unit_rows(t: torch.Tensor) -> torch.Tensor:
    if t.stride(-1) != 1 or (t.ndim == 2 and t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        t = t.contiguous()
    return t


def fft_split(x_re, x_im, *, algorithm="dit", inverse: bool = False, out=None, plan=None):
    """Batched split-format DFT: ``(x_re, x_im) -> (y_re, y_im)``.

    ``x_re``/``x_im``: planes of shape ``[N]`` or ``[B, N]`` (N = 2**m),
    float32 or float64 torch tensors on a CUDA device -- the hot path -- or
    host arrays/tensors (copied to the current CUDA device and back).
    Forward kernel exp(-j 2 pi n k / N), unnormalised; ``inverse=True`` gives
    the reference's ifft (channel swap + 1/N, transform.py:286-298).
    ``out=(y_re, y_im)`` may alias the inputs (in place).  Returns the output
    planes in the input's container type.
    """
    was_numpy = not isinstance(x_re, torch.Tensor) and not isinstance(x_im, torch.Tensor)
    if was_numpy:
        # host arrays follow the reference's containers: float64 (fp32 is
        # upcast exactly, layout.py:29-30), results returned as float64
        x_re = torch.from_numpy(np.ascontiguousarray(x_re, dtype=np.float64))
        x_im = torch.from_numpy(np.ascontiguousarray(x_im, dtype=np.float64))
    sig = SplitSignal(x_re, x_im)
    n = len(sig)
    if not is_power_of_two(n):
        raise ValueError(f"sample count {n} is not a power of two")
    m = n.bit_length() - 1
    host = sig.re.device.type != "cuda"
    device = _resolve_device(None if host else sig.re.device)
    algorithm = Algorithm(algorithm) if not isinstance(algorithm, Algorithm) else algorithm
    if plan is None:
        plan = _cached_plan(m, algorithm, sig.re.dtype, device.index)
    else:
        if plan.m != m:
            raise ValueError(f"buffer is for m={m} but plan is for m={plan.m}")
        if plan.dtype != sig.re.dtype:
            raise ValueError(f"signal dtype {sig.re.dtype} does not match plan dtype {plan.dtype}")
        device = plan.device

    if not host:
        if sig.re.device != device:
            raise ValueError(f"signal is on {sig.re.device} but plan is on {device}")
        xr, xi = _unit_rows(sig.re), _unit_rows(sig.im)
        if out is None:
            yr, yi = torch.empty_like(xr), torch.empty_like(xi)
        else:
            yr, yi = out
            if yr.shape != xr.shape or yi.shape != xr.shape or yr.dtype != xr.dtype or yi.dtype != xr.dtype:
                raise ValueError("out planes must match the input shape and dtype")
            if yr.device != device or yi.device != device:
                raise ValueError("out planes must be on the plan's device")
            if yr.stride(-1) != 1 or yi.stride(-1) != 1 or yr.stride() != yi.stride():
                raise ValueError("out planes must have unit inner stride and equal strides")
        if xr.stride() != xi.stride():
            xr, xi = xr.contiguous(), xi.contiguous()
        _exec_split_device(plan, xr, xi, yr, yi, inverse)
        return yr, yi

    # host buffers: chunked H2D -> transform -> D2H pipeline (the e2e path)
    hr_in, hi_in = sig.re, sig.im
    if out is not None:
        hr, hi = out
        hr = torch.from_numpy(hr) if not isinstance(hr, torch.Tensor) else hr
        hi = torch.from_numpy(hi) if not isinstance(hi, torch.Tensor) else hi
        if hr.dtype != hr_in.dtype and was_numpy:
            raise ValueError("out arrays for numpy input must be float64 (the reference's dtype)")
        if hr.shape != hr_in.shape or hi.shape != hr_in.shape or hr.dtype != hr_in.dtype:
            raise ValueError("out planes must match the input shape and dtype")
    else:
        pin = hr_in.is_pinned()
        hr = torch.empty(hr_in.shape, dtype=hr_in.dtype, pin_memory=pin)
        hi = torch.empty(hr_in.shape, dtype=hr_in.dtype, pin_memory=pin)
    _host_pipeline(plan, device, hr_in, hi_in, hr, hi, inverse)
    if out is not None:
        return out
    if was_numpy:
        return hr.numpy(), hi.numpy()
    return hr, hi


_PIPE_CHUNK_BYTES = 8 << 20    # per plane per chunk (tools/e2e_probe.py sweep)
_PIPE_SLOTS = 4


def _host_pipeline(plan, device, hr_in, hi_in, hr_out, hi_out, inverse):
    """Host planes -> device -> transform -> host planes, in row chunks on
    three streams (H2D, compute, D2H) so that both PCIe directions and the
    kernel overlap; with pinned host memory every copy is asynchronous."""
    one = hr_in.ndim == 1
    xr2 = hr_in.reshape(1, -1) if one else hr_in
    xi2 = hi_in.reshape(1, -1) if one else hi_in
    yr2 = hr_out.reshape(1, -1) if one else hr_out
    yi2 = hi_out.reshape(1, -1) if one else hi_out
    b, n = xr2.shape
    esz = xr2.element_size()
    rows = max(1, min(b, _PIPE_CHUNK_BYTES // (n * esz)))
    nchunks = (b + rows - 1) // rows
    slots = min(_PIPE_SLOTS, nchunks)
    with torch.cuda.device(device):
        caller = torch.cuda.current_stream(device)
        s_in, s_cmp, s_out = (torch.cuda.Stream(device) for _ in range(3))
        for s_ in (s_in, s_cmp, s_out):
            s_.wait_stream(caller)
        bufs = [tuple(torch.empty((rows, n), dtype=xr2.dtype, device=device) for _ in range(4))
                for _ in range(slots)]
        freed = [None] * slots
        for k in range(nchunks):
            r0, r1 = k * rows, min(b, (k + 1) * rows)
            sl = k % slots
            dxr, dxi, dyr, dyi = (t[: r1 - r0] for t in bufs[sl])
            with torch.cuda.stream(s_in):
                if freed[sl] is not None:
                    s_in.wait_event(freed[sl])
                dxr.copy_(xr2[r0:r1], non_blocking=True)
                dxi.copy_(xi2[r0:r1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in)
                _exec_split_device(plan, dxr, dxi, dyr, dyi, inverse)
                ev_cmp = torch.cuda.Event()
                ev_cmp.record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp)
                yr2[r0:r1].copy_(dyr, non_blocking=True)
                yi2[r0:r1].copy_(dyi, non_blocking=True)
                ev_out = torch.cuda.Event()
                ev_out.record(s_out)
                freed[sl] = ev_out
        s_out.synchronize()
        for s_ in (s_in, s_cmp, s_out):
            caller.wait_stream(s_)


def ifft_split(x_re, x_im, *, algorithm="dit", out=None, plan=None):
    """Inverse of :func:`fft_split` (transform.py:286-298)."""
    return fft_split(x_re, x_im, algorithm=algorithm, inverse=True, out=out, plan=plan)


def _check_pair(plan: FftPlan, buf: InterleavedBuffer) -> None:
    if buf.m != plan.m:
        raise ValueError(f"buffer is for m={buf.m} but plan is for m={plan.m}")


def _run_interleaved(plan: FftPlan, buf: InterleavedBuffer, inverse: bool, algorithm: Algorithm):
    _check_pair(plan, buf)
    if algorithm is not plan.algorithm:
        # fft_dit/fft_dif on a plan built for the other variant: same tables,
        # other kernel family (the reference's plans serve both, :208-270)
        plan = _cached_plan(plan.m, algorithm, plan.dtype, plan.device.index)
    direction = _ffi.SFFT_INVERSE if inverse else _ffi.SFFT_FORWARD
    if not buf.is_torch:
        # the reference's float64 numpy buffer: transformed on the GPU in the
        # plan's dtype and written back in place (transform.py:208-298
        # mutate buf.data)
        work = torch.from_numpy(buf.data).to(plan.device, plan.dtype)
        n = plan.sample_count
        ws, wsp = _workspace(plan, 1)
        _ffi.check(_ffi.lib.sfft_exec_interleaved(plan._handle, work.data_ptr(), work.data_ptr(), 1, n, n,
                                                  direction, wsp, _stream_ptr(plan.device)))
        buf.data[...] = work.cpu().numpy()
        return buf
    data = buf.data
    if data.dtype != plan.dtype:
        raise ValueError(f"buffer dtype {data.dtype} does not match plan dtype {plan.dtype}")
    host = data.device.type != "cuda"
    work = data.to(plan.device, non_blocking=True) if host else data
    if work.device != plan.device:
        raise ValueError(f"buffer is on {work.device} but plan is on {plan.device}")
    if not work.is_contiguous():
        work = work.contiguous()
    batch = 1 if work.ndim == 1 else work.shape[0]
    n = plan.sample_count
    ws, wsp = _workspace(plan, batch)
    _ffi.check(_ffi.lib.sfft_exec_interleaved(plan._handle, work.data_ptr(), work.data_ptr(), batch, n, n,
                                              direction, wsp, _stream_ptr(plan.device)))
    if ws is not None:
        ws.record_stream(torch.cuda.current_stream(plan.device))
    if work.data_ptr() != data.data_ptr():
        data.copy_(work)
    return buf


def _stage_operand(buf: InterleavedBuffer, device, dtype):
    """(device tensor the stage kernel runs on, write-back) for a buffer."""
    if not buf.is_torch:
        work = torch.from_numpy(buf.data).to(device, dtype)

        def back():
            buf.data[...] = work.cpu().numpy()
        return work, back
    data = buf.data
    if data.device.type == "cuda" and data.is_contiguous() and data.dtype == dtype:
        return data, lambda: None
    work = data.to(device, dtype).contiguous()
    return work, lambda: data.copy_(work)


def butterfly_stage(buf: InterleavedBuffer, i: int) -> None:
    """Apply the stage-``i`` butterflies W^(i) in place (transform.py:88-101):
    within each block of ``2**i`` pairs, pair q and pair q + 2**(i-1) become
    their sum and difference.  Runs on the GPU (sfft_stage.cuh)."""
    if not 1 <= i <= buf.m:
        raise ValueError(f"stage index {i} out of range for m={buf.m}")
    if buf.is_torch and buf.data.device.type == "cuda":
        device, dtype = buf.data.device, buf.data.dtype
    else:
        device = _resolve_device(None)
        dtype = buf.data.dtype if buf.is_torch else torch.float64
    work, back = _stage_operand(buf, device, dtype)
    batch = 1 if work.ndim == 1 else work.shape[0]
    _ffi.check(_ffi.lib.sfft_exec_butterfly_stage(_DTYPE_CODE[dtype], buf.m, int(i), work.data_ptr(), batch,
                                                  buf.sample_count, device.index, _stream_ptr(device)))
    back()


def twiddle_stage(buf: InterleavedBuffer, plan: FftPlan, i: int) -> None:
    """Apply the stage-``i`` rotations D^(i) in place (transform.py:104-120):
    pair q >= 1 of each block's second half is multiplied by the stage-i
    factor (the identity column is skipped, as the reference does).  Runs on
    the GPU with the plan's tables and dtype (sfft_stage.cuh)."""
    if buf.m != plan.m:
        raise ValueError(f"buffer is for m={buf.m} but plan is for m={plan.m}")
    if not 1 <= i <= plan.m:
        raise ValueError(f"stage index {i} out of range for m={plan.m}")
    if i == 1:
        return  # the single stage-1 rotation is the identity
    work, back = _stage_operand(buf, plan.device, plan.dtype)
    batch = 1 if work.ndim == 1 else work.shape[0]
    _ffi.check(_ffi.lib.sfft_exec_twiddle_stage(plan._handle, int(i), work.data_ptr(), batch, plan.sample_count,
                                                _stream_ptr(plan.device)))
    back()


def fft_dit(plan: FftPlan, buf: InterleavedBuffer) -> InterleavedBuffer:
    """Forward transform, decimation in time; mutates ``buf`` (transform.py:208)."""
    return _run_interleaved(plan, buf, False, Algorithm.DIT)


def fft_dif(plan: FftPlan, buf: InterleavedBuffer) -> InterleavedBuffer:
    """Forward transform, decimation in frequency; mutates ``buf`` (transform.py:241)."""
    return _run_interleaved(plan, buf, False, Algorithm.DIF)


def fft(plan: FftPlan, buf: InterleavedBuffer) -> InterleavedBuffer:
    """Forward transform using the plan's variant (transform.py:273-277)."""
    return _run_interleaved(plan, buf, False, plan.algorithm)


def ifft(plan: FftPlan, buf: InterleavedBuffer) -> InterleavedBuffer:
    """Inverse transform by the channel-swap identity (transform.py:286-298)."""
    return _run_interleaved(plan, buf, True, plan.algorithm)


@dataclass(frozen=True)
class FlopReport:
    """Real-arithmetic census for one transform size (transform.py:301-309)."""

    real_mults: int
    real_adds: int
    generic_rotations: int
    quarter_turns: int
    identity_rotations: int


def count_flops(plan) -> FlopReport:
    """Census of rotation kinds and real ops (transform.py:312-335)."""
    m = plan.m if isinstance(plan, FftPlan) else int(plan)
    out = (ctypes.c_int64 * 5)()
    _ffi.check(_ffi.lib.sfft_count_flops(m, out))
    return FlopReport(*[int(v) for v in out])
