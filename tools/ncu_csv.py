"""Print (launch id, kernel, metric, value) from `ncu --csv` output on stdin,
skipping the program's own stdout lines (developer tool)."""
import csv
import sys

lines = sys.stdin.read().splitlines()
start = next((i for i, l in enumerate(lines) if l.startswith('"ID"')), None)
if start is None:
    sys.exit("no ncu csv header found")
rows = list(csv.reader(lines[start:]))
h = rows[0]
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for r in rows[1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    print(tag, d["ID"], d["Kernel Name"][:60], d["Metric Name"], d["Metric Value"])
