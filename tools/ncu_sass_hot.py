"""Per-instruction view of an ncu capture (--page source, SASS): the
instructions with excess shared wavefronts (bank conflicts) and the top
stall-sampled instructions.
    python tools/ncu_sass_hot.py REP [top]"""
import csv
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rd = list(csv.reader(lines[1:]))
    hdr = rd[0]
    return hdr, rd[1:]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    hdr, rs = rows(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    num = lambda r, k: float(r[ix[k]] or 0) if r[ix[k]] not in ("-", "") else 0.0   # noqa: E731
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in rs)
    ex = [(num(r, "L1 Wavefronts Shared Excessive"), r) for r in rs]
    ex = [e for e in ex if e[0] > 0]
    print(f"instructions with excess shared wavefronts: {len(ex)}, total excess "
          f"{sum(e[0] for e in ex):.0f}")
    for v, r in sorted(ex, key=lambda e: -e[0])[:top]:
        print(f"  {v:12.0f}  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()}")
    print(f"top stall samples (of {tot:.0f}):")
    st = sorted(rs, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in st:
        print(f"  {num(r, 'Warp Stall Sampling (All Samples)'):8.0f}  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()}")


if __name__ == "__main__":
    main()
