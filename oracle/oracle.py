"""TEST INFRASTRUCTURE, NOT PRODUCT CODE: the CPU parity oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline -- never on the product path (paper_2504_07264_b200 never imports
it).

Two restatements of the reference's CPU algorithm
(/root/reference/pkg/src/splitfft/transform.py):

* ``fft_split_c`` -- ctypes wrapper of splitfft_oracle.c (liboracle.so):
  batched fp64 DIT/DIF/inverse, bit-identical to the reference (pinned by
  tests/test_oracle_golden.py against tests/golden/*.npz written by the
  reference itself), multi-threaded over independent rows.
* ``fft_split_numpy`` -- a numpy restatement of the reference executor
  (transform.py:123-270: gather, stage 1, 2^14-pair segments, two-stage
  column slabs) for one signal at a time, on complex128 views of an
  interleaved buffer.  It is the "reference port" that bench.py's
  ``--impl reference`` arm times: the same numpy ufunc sequence per signal
  as the reference, hence the same cost profile.

Parity status: PINNED (bitwise vs reference-generated golden vectors).
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        L.oracle_fft_split.argtypes = [I, I, I, P, P, P, P, I64, I64, I64, I]
        L.oracle_fft_split.restype = I
        L.oracle_twiddle_table.argtypes = [I, P, P]
        L.oracle_twiddle_table.restype = I
        L.oracle_cos_sin.argtypes = [I, P, P]
        L.oracle_cos_sin.restype = I
        L.oracle_bitrev.argtypes = [I, P]
        L.oracle_bitrev.restype = None
        _lib = L
    return _lib


def fft_split_c(x_re, x_im, algorithm="dit", inverse=False, threads=None):
    """fp64 split->split transform of [N] or [B, N] planes (any float dtype is
    upcast exactly to float64, as layout.py:29-30 does)."""
    xr = np.ascontiguousarray(np.asarray(x_re, dtype=np.float64))
    xi = np.ascontiguousarray(np.asarray(x_im, dtype=np.float64))
    one = xr.ndim == 1
    if one:
        xr, xi = xr[None, :], xi[None, :]
    b, n = xr.shape
    m = n.bit_length() - 1
    if n != 1 << m:
        raise ValueError(f"sample count {n} is not a power of two")
    yr = np.empty_like(xr)
    yi = np.empty_like(xi)
    if threads is None:
        # rows split across threads; fewer rows than cores and m >= 16: the
        # threads split each stage of a row instead (bit-identical)
        threads = os.cpu_count() or 1 if (b < (os.cpu_count() or 1) and m >= 16) else \
            min(os.cpu_count() or 1, max(1, b))
    rc = lib().oracle_fft_split(m, 1 if algorithm == "dif" else 0, 1 if inverse else 0,
                                xr.ctypes.data, xi.ctypes.data, yr.ctypes.data, yi.ctypes.data,
                                b, n, n, int(threads))
    if rc == 2:
        raise MemoryError("oracle: out of host memory")
    if rc:
        raise ValueError("oracle rejected the arguments")
    if one:
        return yr[0], yi[0]
    return yr, yi


def stage_factors(m):
    """FftPlan.stage_factors (transform.py:80-84) restated via the C oracle."""
    if m == 0:
        return ()
    h = 1 << (m - 1)
    wr = np.empty(h)
    wi = np.empty(h)
    lib().oracle_twiddle_table(m, wr.ctypes.data, wi.ctypes.data)
    top = wr + 1j * wi
    return tuple(np.ascontiguousarray(top[:: 1 << (m - i)]) for i in range(1, m + 1))


def cos_sin(i):
    h = 1 << (i - 1)
    c = np.empty(h)
    s = np.empty(h)
    lib().oracle_cos_sin(i, c.ctypes.data, s.ctypes.data)
    return c, s


def bitrev(m):
    idx = np.empty(1 << m, dtype=np.int64)
    lib().oracle_bitrev(m, idx.ctypes.data)
    return idx


# ---------------------------------------------------------------------------
# numpy restatement of the reference executor (the timed "reference port")
# ---------------------------------------------------------------------------
_SEG_LOG = 14          # transform.py:35
_SLAB = 1 << 13        # transform.py:38


class NumpyPlan:
    """make_plan restated (transform.py:65-85): stage factors + bitrev."""

    def __init__(self, m, algorithm="dit"):
        self.m = m
        self.algorithm = algorithm
        self.factors = stage_factors(m)
        self.bitrev = bitrev(m).astype(np.intp)


def _butterfly_all(src, dst):                      # transform.py:123-128
    s = src.reshape(-1, 2)
    d = dst.reshape(-1, 2)
    np.add(s[:, 0], s[:, 1], out=d[:, 0])
    np.subtract(s[:, 0], s[:, 1], out=d[:, 1])


def _dit_stage(z, w, temp):                        # transform.py:131-139
    v = z.reshape(-1, 2, w.size)
    a = v[:, 0, :]
    b = v[:, 1, :]
    t = temp[: a.size].reshape(a.shape)
    np.multiply(b, w, out=t)
    np.subtract(a, t, out=b)
    np.add(a, t, out=a)


def _dif_stage(z, w, temp):                        # transform.py:142-150
    v = z.reshape(-1, 2, w.size)
    a = v[:, 0, :]
    b = v[:, 1, :]
    t = temp[: a.size].reshape(a.shape)
    np.subtract(a, b, out=t)
    np.add(a, b, out=a)
    np.multiply(t, w, out=b)


def _slab_columns(v, r):                           # transform.py:153-157
    c = max(1, min(r, _SLAB // v.shape[0]))
    for c0 in range(0, r, c):
        yield c0, min(r, c0 + c)


def _dit_stage_pair(z, w1, w2, temp):              # transform.py:160-179
    r = w1.size
    v = z.reshape(-1, 2, 2, r)
    w2v = w2.reshape(2, r)
    for c0, c1 in _slab_columns(v, r):
        a0, b0 = v[:, 0, 0, c0:c1], v[:, 0, 1, c0:c1]
        a1, b1 = v[:, 1, 0, c0:c1], v[:, 1, 1, c0:c1]
        t = temp[: a0.size].reshape(a0.shape)
        for a, b in ((a0, b0), (a1, b1)):
            np.multiply(b, w1[c0:c1], out=t)
            np.subtract(a, t, out=b)
            np.add(a, t, out=a)
        for h, (a, b) in enumerate(((a0, a1), (b0, b1))):
            np.multiply(b, w2v[h, c0:c1], out=t)
            np.subtract(a, t, out=b)
            np.add(a, t, out=a)


def _dif_stage_pair(z, w1, w2, temp):              # transform.py:182-200
    r = w1.size
    v = z.reshape(-1, 2, 2, r)
    w2v = w2.reshape(2, r)
    for c0, c1 in _slab_columns(v, r):
        a0, b0 = v[:, 0, 0, c0:c1], v[:, 0, 1, c0:c1]
        a1, b1 = v[:, 1, 0, c0:c1], v[:, 1, 1, c0:c1]
        t = temp[: a0.size].reshape(a0.shape)
        for h, (a, b) in enumerate(((a0, a1), (b0, b1))):
            np.subtract(a, b, out=t)
            np.add(a, b, out=a)
            np.multiply(t, w2v[h, c0:c1], out=b)
        for a, b in ((a0, b0), (a1, b1)):
            np.subtract(a, b, out=t)
            np.add(a, b, out=a)
            np.multiply(t, w1[c0:c1], out=b)


def _fft_dit(plan, z):                             # transform.py:208-238
    m = plan.m
    if m == 0:
        return
    n = z.size
    scratch = np.empty(n, dtype=np.complex128)
    np.take(z, plan.bitrev, out=scratch)
    _butterfly_all(scratch, z)
    k = min(m, _SEG_LOG)
    if k >= 2:
        temp = np.empty(1 << (k - 1), dtype=np.complex128)
        seg = 1 << k
        for s0 in range(0, n, seg):
            zs = z[s0: s0 + seg]
            for i in range(2, k + 1):
                _dit_stage(zs, plan.factors[i - 1], temp)
    slab = None
    i = k + 1
    while i <= m:
        if i < m:
            if slab is None:
                slab = np.empty(max(_SLAB, n >> (k + 2)), dtype=np.complex128)
            _dit_stage_pair(z, plan.factors[i - 1], plan.factors[i], slab)
            i += 2
        else:
            _dit_stage(z, plan.factors[i - 1], scratch[: n >> 1])
            i += 1


def _fft_dif(plan, z):                             # transform.py:241-270
    m = plan.m
    if m == 0:
        return
    n = z.size
    scratch = np.empty(n, dtype=np.complex128)
    k = min(m, _SEG_LOG)
    slab = None
    i = m
    while i > k:
        if i - 1 > k:
            if slab is None:
                slab = np.empty(max(_SLAB, n >> (k + 2)), dtype=np.complex128)
            _dif_stage_pair(z, plan.factors[i - 2], plan.factors[i - 1], slab)
            i -= 2
        else:
            _dif_stage(z, plan.factors[i - 1], scratch[: n >> 1])
            i -= 1
    temp = np.empty(1 << (k - 1), dtype=np.complex128) if k >= 2 else None
    seg = 1 << k
    for s0 in range(0, n, seg):
        zs = z[s0: s0 + seg]
        for i in range(k, 1, -1):
            _dif_stage(zs, plan.factors[i - 1], temp)
        _butterfly_all(zs, scratch[s0: s0 + seg])
    np.take(scratch, plan.bitrev, out=z)


def split_to_split_numpy(plan, re, im, inverse=False):
    """One signal through the reference's split->split composite
    (service/app.py:43-52: SplitSignal -> interleave -> fft|ifft -> deinterleave)."""
    re = np.ascontiguousarray(re, dtype=np.float64)       # layout.py:29-30
    im = np.ascontiguousarray(im, dtype=np.float64)
    n = re.size
    data = np.empty(2 * n, dtype=np.float64)              # layout.py:98-100
    data[0::2] = re
    data[1::2] = im
    run = _fft_dif if plan.algorithm == "dif" else _fft_dit
    if inverse:                                           # transform.py:286-298
        r = data[0::2].copy()
        data[0::2] = data[1::2]
        data[1::2] = r
        run(plan, data.view(np.complex128))
        r = data[0::2].copy()
        data[0::2] = data[1::2]
        data[1::2] = r
        data *= 1.0 / n
    else:
        run(plan, data.view(np.complex128))
    return data[0::2].copy(), data[1::2].copy()           # layout.py:104-106


def fft_split_numpy(x_re, x_im, algorithm="dit", inverse=False, plan=None):
    xr = np.asarray(x_re)
    xi = np.asarray(x_im)
    one = xr.ndim == 1
    if one:
        xr, xi = xr[None, :], xi[None, :]
    n = xr.shape[1]
    m = n.bit_length() - 1
    plan = plan or NumpyPlan(m, algorithm)
    yr = np.empty(xr.shape, dtype=np.float64)
    yi = np.empty(xr.shape, dtype=np.float64)
    for b in range(xr.shape[0]):
        yr[b], yi[b] = split_to_split_numpy(plan, xr[b], xi[b], inverse)
    if one:
        return yr[0], yi[0]
    return yr, yi
