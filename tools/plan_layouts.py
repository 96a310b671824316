"""Shared-memory exchange layouts for the fused kernels (build-time planner).

Between register pass x and x+1 every fused kernel writes its registers to a
shared-memory exchange buffer with the Stockham pattern
    e = (j >> s) * ns * R' + (j & (ns-1)) + ns * f
and the next pass reads  e = j' + r * N / R''.  Which physical word each
logical element e goes to is free, as long as writer and reader agree.  This
script searches, per (element size, log2 N, log2 radix, threads per CTA) and
per exchange, a layout
    none:   phys = e
    pad A:  phys = e + (e >> A)
    xor A:  phys = e ^ ((e >> A) & (banks - 1))
    shifted pad A, B:  phys = e + ((e >> A) << B)
plus a per-signal stride, that makes every warp-wide access of both patterns
bank-conflict free under the shared-memory model of B300_MICROARCH.md
(32 four-byte banks; 64-bit accesses split into two half-warp wavefronts),
and writes csrc/sfft_layouts.h.  Run it when the kernel shapes change:

    python tools/plan_layouts.py
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2504_07264_b200", "csrc")
sys.path.insert(0, CSRC)

import gen_inst  # noqa: E402  (kernel shape tables)


def wavefronts(addrs, esz):
    tot = 0
    groups = [addrs] if esz == 4 else [addrs[:16], addrs[16:]]
    for g in groups:
        banks = {}
        for a in g:
            for w in range(esz // 4):
                word = a // 4 + w
                banks.setdefault(word % 32, set()).add(word)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


def schedule(m, lr):
    out, s = [], 0
    while s < m:
        k = min(lr, m - s)
        out.append((s, k))
        s += k
    return out


def phys_fn(kind, a, esz):
    mask = 31 if esz == 4 else 15
    if kind == 0:
        return lambda e: e
    if kind == 1:
        return lambda e: e + (e >> a)
    if kind == 3:   # shifted pad: arg = A | B << 8, phys = e + ((e >> A) << B)
        sa, sb = a & 255, a >> 8
        return lambda e: e + ((e >> sa) << sb)
    return lambda e: e ^ ((e >> a) & mask)


def exchange_cost(n, lr, esz, nt, x, fn, sstr):
    m = n.bit_length() - 1
    r_ = 1 << lr
    p_ = n // r_
    sched = schedule(m, lr)
    tot = cnt = 0
    for p, kind in ((x, "wr"), (x + 1, "rd")):
        s, k = sched[p]
        rp = 1 << k
        u_n = r_ // rp
        ns = 1 << s
        for w in range(min(nt, 256) // 32):
            for u in range(u_n):
                for idx in range(rp):
                    addrs = []
                    for tid in range(w * 32, w * 32 + 32):
                        sig, t = divmod(tid, p_)
                        j = t + p_ * u
                        e = j + idx * (n // rp) if kind == "rd" else (j >> s) * ns * rp + (j & (ns - 1)) + ns * idx
                        addrs.append((sig * sstr + fn(e)) * esz)
                    tot += wavefronts(addrs, esz)
                    cnt += 1
    return tot / cnt / (2 if esz == 8 else 1)


def linear_sides(n, lr, x, fn):
    """Bit 0: every write of exchange x is phys(e(t,0,0)) + phys(e(0,u,f)); bit 1:
    the same for every read -- the kernels then address the exchange as a
    per-thread base plus compile-time offsets (ex_wr / ex_rd)."""
    m = n.bit_length() - 1
    r_ = 1 << lr
    p_ = n // r_
    sched = schedule(m, lr)
    bits = 0
    for bit, (p, kind) in enumerate(((x, "wr"), (x + 1, "rd"))):
        s, k = sched[p]
        rp = 1 << k
        ns = 1 << s

        def e_of(j, idx):
            return j + idx * (n // rp) if kind == "rd" else (j >> s) * ns * rp + (j & (ns - 1)) + ns * idx
        ok = all(fn(e_of(t + p_ * u, idx)) == fn(e_of(t, 0)) + fn(e_of(p_ * u, idx))
                 for u in range(r_ // rp) for idx in range(rp) for t in range(p_))
        bits |= ok << bit
    return bits


def nonlinear_sites(n, lr, x, fn):
    """Accesses of exchange x (the Stockham write of pass x and the read of
    pass x+1) whose physical slot is NOT the thread's first slot plus a
    thread-independent constant: each of those costs the kernel address
    arithmetic per access instead of an immediate offset."""
    m = n.bit_length() - 1
    r_ = 1 << lr
    p_ = n // r_
    sched = schedule(m, lr)
    cnt = 0
    for p, kind in ((x, "wr"), (x + 1, "rd")):
        s, k = sched[p]
        rp = 1 << k
        ns = 1 << s

        def e_of(j, idx):
            return j + idx * (n // rp) if kind == "rd" else (j >> s) * ns * rp + (j & (ns - 1)) + ns * idx
        for u in range(r_ // rp):
            for idx in range(rp):
                deltas = {fn(e_of(t + p_ * u, idx)) - fn(e_of(t, 0)) for t in range(p_)}
                cnt += len(deltas) > 1
    return cnt


def plan(n, lr, esz, nt):
    m = n.bit_length() - 1
    sched = schedule(m, lr)
    p_ = n // (1 << lr)
    s_ = nt // p_
    lb = 5 if esz == 4 else 4
    order = ([(1, lr), (1, lb), (2, lr), (0, 0)] + [(1, a) for a in range(2, 11)]
             + [(3, a | (b << 8)) for a in range(2, 12) for b in range(1, 6)] + [(2, a) for a in range(2, 11)])
    result = []
    for x in range(len(sched) - 1):
        # every conflict-free layout, then the one with the fewest accesses
        # that need per-access address arithmetic (ties: planner order)
        best, free = None, []
        for kind, a in order:
            fn = phys_fn(kind, a, esz)
            span = fn(n - 1) + 1
            base = (span + 7) // 8 * 8 if s_ > 1 else span
            for extra in (range(0, 33) if s_ > 1 else (0,)):
                sstr = base + extra if s_ > 1 else span
                c = exchange_cost(n, lr, esz, nt, x, fn, sstr)
                if best is None or c < best[0] - 1e-9:
                    best = (c, kind, a, sstr)
                if c <= 1.0 + 1e-9:
                    free.append((nonlinear_sites(n, lr, x, fn), len(free), (c, kind, a, sstr)))
                    break
        result.append(min(free)[2] if free else best)
    return result


def chain(vals, n=None):
    """C conditional chain of vals[0..n) (n = the number of exchanges; the
    last value also answers every x >= n-1)."""
    if n is None:
        n = len(vals)
        while n > 1 and vals[n - 1] == 0:
            n -= 1
    expr = str(vals[n - 1])
    for x in range(n - 2, -1, -1):
        expr = f"x == {x} ? {vals[x]} : ({expr})"
    return expr


def shapes():
    out = set()
    for dt, esz in (("f32", 4), ("f64", 8)):
        for logn in range(1, 13):
            lrs = sorted({min(lr, logn) for lr in gen_inst.RADIX_CHOICES[dt]})
            for lr in lrs:
                p_ = 1 << (logn - lr)
                if p_ > 1024:
                    continue
                out.add((esz, logn, lr, gen_inst.fused_nt(logn, lr)))   # LDG kernel
        for logn, cfgs in gen_inst.TMA_CONFIGS[dt].items():
            for c in cfgs:
                lr, nt = c[0], c[1]
                p_ = 1 << (logn - lr)
                out.add((esz, logn, lr, max(p_, nt)))          # TMA kernel
    return sorted(out)


def main():
    lines = [
        "// GENERATED by tools/plan_layouts.py -- shared-memory exchange layouts",
        "// (per exchange x: kind 0 none / 1 pad A / 2 xor A / 3 shifted pad A | B << 8,\n// and the per-signal",
        "// stride), each checked bank-conflict free for both the Stockham write",
        "// and the next pass's read pattern.  Unlisted shapes use ExLayoutDefault.",
        "#pragma once",
        "namespace sfft {",
        "template <int ESZ, int LOGN, int LR, int NT> struct ExLayout {",
        "    static constexpr bool planned = false;",
        "    __host__ __device__ static constexpr int kind(int) { return 1; }",
        "    __host__ __device__ static constexpr int arg(int) { return LR; }",
        "    __host__ __device__ static constexpr int lin(int) { return 0; }",
        "    static constexpr int sstr = (1 << LOGN) + ((1 << LOGN) >> LR);",
        "};",
    ]
    worst = 1.0
    for esz, logn, lr, nt in shapes():
        n = 1 << logn
        res = plan(n, lr, esz, nt)
        if not res:
            continue
        worst = max(worst, max(r[0] for r in res))
        kinds = [r[1] for r in res] + [0] * (12 - len(res))
        args = [r[2] for r in res] + [0] * (12 - len(res))
        lins = [linear_sides(n, lr, x, phys_fn(r[1], r[2], esz)) for x, r in enumerate(res)] + [0] * (12 - len(res))
        sstr = max(r[3] for r in res)
        costs = " ".join(f"{r[0]:.2f}" for r in res)
        lines += [
            f"template <> struct ExLayout<{esz}, {logn}, {lr}, {nt}> {{   // wavefronts/ideal: {costs}",
            "    static constexpr bool planned = true;",
            f"    __host__ __device__ static constexpr int kind(int x) {{ return {chain(kinds, len(res))}; }}",
            f"    __host__ __device__ static constexpr int arg(int x) {{ return {chain(args, len(res))}; }}",
            f"    __host__ __device__ static constexpr int lin(int x) {{ return {chain(lins, len(res))}; }}",
            f"    static constexpr int sstr = {sstr};",
            "};",
        ]
        print(f"esz{esz} N{n} LR{lr} NT{nt}: {costs} sstr={sstr}", flush=True)
    lines.append("}  // namespace sfft")
    with open(os.path.join(CSRC, "sfft_layouts.h"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"worst exchange cost {worst:.2f}")


if __name__ == "__main__":
    main()
