"""List register counts / spills of the kernels in ptxas -v logs:
python tools/ptxas_spills.py build/csrc/sfft_inst_pass2_f32.ptxas.log [--all]"""
import re
import subprocess
import sys

show_all = "--all" in sys.argv
for f in [a for a in sys.argv[1:] if not a.startswith("--")]:
    t = open(f).read()
    pat = (r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, "
           r"(\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers")
    for m in re.finditer(pat, t):
        if not show_all and m.group(3) == "0":
            continue
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        print(f"{name[:110]}  stack {m.group(2)} spill st/ld {m.group(3)}/{m.group(4)} regs {m.group(5)}")
