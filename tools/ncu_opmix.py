"""Executed-instruction mix of one kernel in an ncu capture, by SASS opcode
(--page source): python tools/ncu_opmix.py REP [kernel-index] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if kid is not None:
    cmd += ["--launch-skip", kid, "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rd = list(csv.reader(lines[start:]))
hdr = rd[0]
ix = {h: i for i, h in enumerate(hdr)}
ex_key = "Instructions Executed" if "Instructions Executed" in ix else [h for h in hdr if "Executed" in h][0]
st_key = "Warp Stall Sampling (All Samples)"
cnt, stall = collections.Counter(), collections.Counter()
for r in rd[1:]:
    if len(r) < len(hdr) or r[0] == "Address":
        continue
    src = r[ix["Source"]].strip()
    if not src:
        continue
    op = src.split()[0]
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        cnt[op] += float(r[ix[ex_key]] or 0)
        stall[op] += float(r[ix[st_key]] or 0)
    except ValueError:
        pass
tot, tst = sum(cnt.values()), sum(stall.values())
print(f"total warp instructions {tot:.4g}, stall samples {tst:.4g}")
for op, v in cnt.most_common(top):
    print(f"{op:10s} {v:12.4g} {100 * v / tot:6.2f}%   stall {100 * stall[op] / max(tst, 1):6.2f}%")
