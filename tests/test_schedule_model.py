"""CPU model of the kernels' Stockham register-pass index map.

sfft_common.cuh/sfft_fused.cuh execute the reference's radix-2 stages
grouped 2^K at a time, with the data exchanged between groups in Stockham
order.  This numpy restatement uses exactly the kernels' index formulas
(virtual thread j, c = j mod ns, q = c + f*ns, register rev_K(f), writes
out[(j>>s)*ns*R + c + ns*f]; DIF the transpose) and numpy's own complex
multiply (the rounding the reference uses), and must equal the reference
oracle bit for bit for every size and radix.  It documents -- and guards --
the claim that regrouping the stages changes no arithmetic.
"""

import numpy as np
import pytest

from oracle import oracle


def rev(f, b):
    r = 0
    for _ in range(b):
        r = (r << 1) | (f & 1)
        f >>= 1
    return r


def schedule(m, logr):
    out, s = [], 0
    while s < m:
        k = min(logr, m - s)
        out.append((s, k))
        s += k
    return out


def top_table(m):
    return oracle.stage_factors(m)[m - 1] if m else None


def model_dit(x, m, logr):
    n = x.shape[1]
    top = top_table(m)
    buf = x.copy()
    for s, k in schedule(m, logr):
        r_, ns = 1 << k, 1 << s
        j = np.arange(n // r_)
        g, c = j >> s, j & (ns - 1)
        v = buf[:, j[:, None] + np.arange(r_)[None, :] * (n // r_)].copy()
        for t in range(1, k + 1):
            half, i = r_ >> t, s + t
            for f in range(1 << (t - 1)):
                rf = rev(f, t - 1) * 2 * half
                w = top[(c + (f << s)) << (m - i)]
                for r in range(half):
                    p1, p2 = r + rf, r + rf + half
                    a = v[:, :, p1].copy()
                    tt = v[:, :, p2].copy() if i == 1 else np.multiply(v[:, :, p2], w)
                    v[:, :, p2] = a - tt
                    v[:, :, p1] = a + tt
        out = np.empty_like(buf)
        for f in range(r_):
            out[:, g * ns * r_ + c + ns * f] = v[:, :, rev(f, k)]
        buf = out
    return buf


def model_dif(x, m, logr):
    n = x.shape[1]
    top = top_table(m)
    buf = x.copy()
    for s, k in reversed(schedule(m, logr)):
        r_, ns = 1 << k, 1 << s
        j = np.arange(n // r_)
        g, c = j >> s, j & (ns - 1)
        v = np.empty((x.shape[0], n // r_, r_), dtype=complex)
        for f in range(r_):
            v[:, :, rev(f, k)] = buf[:, g * ns * r_ + c + ns * f]
        for t in range(k, 0, -1):
            half, i = r_ >> t, s + t
            for f in range(1 << (t - 1)):
                rf = rev(f, t - 1) * 2 * half
                w = top[(c + (f << s)) << (m - i)]
                for r in range(half):
                    p1, p2 = r + rf, r + rf + half
                    a, b = v[:, :, p1].copy(), v[:, :, p2].copy()
                    tt = a - b
                    v[:, :, p1] = a + b
                    v[:, :, p2] = tt if i == 1 else np.multiply(tt, w)
        out = np.empty_like(buf)
        out[:, j[:, None] + np.arange(r_)[None, :] * (n // r_)] = v
        buf = out
    return buf


def bits(z):
    z = np.ascontiguousarray(z)
    return np.concatenate([z.real.ravel().view(np.int64), z.imag.ravel().view(np.int64)])


@pytest.mark.parametrize("m", range(0, 11))
@pytest.mark.parametrize("logr", [1, 2, 3, 4, 5])
def test_register_pass_map_is_bitwise_the_reference(m, logr):
    rng = np.random.default_rng(50 + m)
    n = 1 << m
    x = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
    for algo, model in (("dit", model_dit), ("dif", model_dif)):
        wr, wi = oracle.fft_split_c(x.real.copy(), x.imag.copy(), algo)
        assert np.array_equal(bits(model(x, m, logr)), bits(wr + 1j * wi)), (algo, m, logr)


@pytest.mark.parametrize("m,logr", [(m, lr) for m in range(2, 13) for lr in (2, 3, 4, 5) if lr < m])
def test_partial_last_exchange_keeps_own_values(m, logr):
    """sfft_fused.cuh LastX: before a last register pass of KPL < LR stages,
    the Stockham exchange permutes values only inside groups of RPL = 2^KPL
    threads (t = g * P/RPL + c), and the value thread t reads at (u, r = g)
    is the one it wrote itself at position f = g + RPL*u -- so the kernels
    keep those in registers (DIT: the gather of the last pass; DIF: the
    transpose, first pass -> second).  Checked on the kernels' index formulas
    for every physical thread."""
    n, r_ = 1 << m, 1 << logr
    p_ = n // r_
    sched = schedule(m, logr)
    if len(sched) < 2 or sched[-1][1] == logr:
        return
    sp_prev, _ = sched[-2]
    sp_last, kpl = sched[-1]
    rpl, ns_prev, ns_last = 1 << kpl, 1 << sp_prev, 1 << sp_last
    gstride = p_ // rpl
    writer = {}
    for i in range(p_):                       # pass NPASS-2 scatter (U = 1, full radix)
        base = (i >> sp_prev) * ns_prev * r_ + (i & (ns_prev - 1))
        for f in range(r_):
            writer[base + ns_prev * f] = (i, f)
    assert len(writer) == n
    for t in range(p_):                       # last pass gather
        g = t // gstride
        for u in range(r_ // rpl):
            j = t + p_ * u
            for r in range(rpl):
                wi, wf = writer[j + r * (n // rpl)]
                assert wi % gstride == t % gstride   # same group of RPL threads
                if r == g:
                    assert (wi, wf) == (t, g + rpl * u)
                else:
                    assert wi != t
