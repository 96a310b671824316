"""Refresh profiles/ncu_traffic.json (bench.py's roofline.traffic) from ncu
--set full captures: dram__bytes_read.sum + dram__bytes_write.sum per launch
(mean over the captured launches).

    python tools/ncu_traffic_update.py cfg2_n64_f32=gpurun_out/prof_r01p_cfg2_n64_f32.ncu-rep ...

The kernel-source hash is read from gpurun_out/prof_<TAG>.srchash (written
by tools/prof_cfgs.sh on the box at capture time); bench.py only reports a
capture whose hash matches the sources it runs.  An entry named
"cfg:dif" records a DIF capture.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rd = float(d["dram__bytes_read.sum"]) * SCALE[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(d["dram__bytes_write.sum"]) * SCALE[units[hdr.index("dram__bytes_write.sum")]]
        yield d["Kernel Name"], rd, wr


def main():
    with open(PATH) as f:
        table = json.load(f)
    for arg in sys.argv[1:]:
        cfg, rep = arg.split("=", 1)
        algo = "dit"
        if ":" in cfg:
            cfg, algo = cfg.split(":", 1)
        tag = os.path.basename(rep).split("_")[1]     # prof_<TAG>_<cfg>.ncu-rep
        hpath = os.path.join(os.path.dirname(rep), f"prof_{tag}.srchash")
        src = open(hpath).read().strip() if os.path.exists(hpath) else None
        ls = list(launches(rep))
        rd = sum(x[1] for x in ls) / len(ls)
        wr = sum(x[2] for x in ls) / len(ls)
        table[cfg] = {"kernel": ls[0][0][:120], "dram_bytes_read": rd, "dram_bytes_write": wr,
                      "dram_bytes_per_launch": rd + wr, "launches_captured": len(ls),
                      "source": os.path.relpath(rep, ROOT), "src_hash": src, "algorithm": algo}
        print(cfg, len(ls), f"{(rd + wr) / 1e9:.4f} GB per launch", ls[0][0][:80])
    with open(PATH, "w") as f:
        json.dump(table, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
