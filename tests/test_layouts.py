"""The generated shared-memory exchange layouts (csrc/sfft_layouts.h) are what
the planner (tools/plan_layouts.py) proves: every planned exchange is
bank-conflict free for both the Stockham write and the next pass's read, and
its additivity bits (ExLayout::lin, which let the kernels address an exchange
as a per-thread base plus compile-time offsets, ex_wr/ex_rd) hold for every
thread.  A wrong `lin` bit would silently corrupt results, so the header is
re-checked here from its own text."""

import os
import re
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import plan_layouts as pl  # noqa: E402

HEADER = os.path.join(ROOT, "paper_2504_07264_b200", "csrc", "sfft_layouts.h")


def chain_values(expr, count):
    """Evaluate a generated `x == 0 ? a : (x == 1 ? b : (c))` chain for x < count."""
    vals = []
    for x in range(count):
        e = expr
        # innermost-first evaluation of the C conditional chain
        while "?" in e:
            m = re.match(r"x == (\d+) \? (\d+) : \((.*)\)$", e.strip())
            if not m:
                break
            e = m.group(2) if int(m.group(1)) == x else m.group(3)
        vals.append(int(e.strip().strip("()")))
    return vals


def planned_layouts():
    text = open(HEADER).read()
    pat = re.compile(
        r"template <> struct ExLayout<(\d+), (\d+), (\d+), (\d+)> \{[^\n]*\n"
        r"\s+static constexpr bool planned = true;\n"
        r"\s+__host__ __device__ static constexpr int kind\(int x\) \{ return (.*?); \}\n"
        r"\s+__host__ __device__ static constexpr int arg\(int x\) \{ return (.*?); \}\n"
        r"\s+__host__ __device__ static constexpr int lin\(int x\) \{ return (.*?); \}\n"
        r"\s+static constexpr int sstr = (\d+);")
    out = []
    for m in pat.finditer(text):
        esz, logn, lr, nt = (int(m.group(i)) for i in range(1, 5))
        out.append((esz, logn, lr, nt, m.group(5), m.group(6), m.group(7), int(m.group(8))))
    return out


LAYOUTS = planned_layouts()


def test_header_has_every_planned_shape():
    assert len(LAYOUTS) == len([s for s in pl.shapes() if len(pl.schedule(s[1], s[2])) >= 2])


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: f"esz{l[0]}-m{l[1]}-lr{l[2]}-nt{l[3]}")
def test_layout_conflict_free_and_lin_bits_exact(lay):
    esz, logn, lr, nt, kinds, args, lins, sstr = lay
    n = 1 << logn
    nx = len(pl.schedule(logn, lr)) - 1
    kv, av, lv = chain_values(kinds, nx), chain_values(args, nx), chain_values(lins, nx)
    for x in range(nx):
        fn = pl.phys_fn(kv[x], av[x], esz)
        assert fn(n - 1) < sstr, "slots must fit the per-signal stride"
        assert pl.exchange_cost(n, lr, esz, nt, x, fn, sstr) <= 1.0 + 1e-9
        # the bits the kernels rely on must be exactly the planner's proof
        assert lv[x] == pl.linear_sides(n, lr, x, fn)
