"""Executed instructions and stall samples per CUDA source line of one kernel
in an ncu capture (needs -lineinfo and --import-source on):
python tools/ncu_lines.py REP [kernel-index] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda", "--launch-skip", kid,
       "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        print(r[1])
    elif r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
    elif hdr and r[0] not in ("", "-"):
        try:
            ex = float(r[hdr["Instructions Executed"]])
            st = float(r[hdr["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        rows.append((ex, st, fname, r[0], r[1].strip()))
tot = sum(r[0] for r in rows)
tst = sum(r[1] for r in rows)
print(f"total warp instructions {tot:.4g}, stall samples {tst:.4g}")
for ex, st, f, ln, src in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100 * ex / tot:6.2f}% inst {100 * st / max(tst, 1):6.2f}% stall  {f}:{ln}  {src[:100]}")
