"""profiles/<tag>_ncu_cfg5.md from tools/ncu_cfg5.sh's launch lists: per
launch time and DRAM bytes of one 2^27-pair sort at buffer 1.0 and 0.5, the
sum of DRAM bytes against the algorithmic lower bound P * 2 * n * 12 B.
usage: python tools/summarize_cfg5.py [gpurun_out] [tag]"""
import csv
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r2"
N, S = 1 << 27, 12
PEAK = 6533.5      # MEASURED_PEAKS.json hbm_gbs (copy read + write)
OURS = ("tile_sort2", "merge_tstore", "merge_inplace", "partition", "inplace_deps", "gather_samples", "reverse")


def launches(path):
    per = OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = next((k for k in OURS if k in d["Kernel Name"]), None)
        if name is None:
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        if d["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
        elif unit in ("ns", "nsecond"):
            v *= 1e-3
        elif unit in ("ms", "msecond"):
            v *= 1e3
        per.setdefault((int(d["ID"]), name), {})[d["Metric Name"]] = v
    return per


out = [f"# ncu launch lists ({TAG}) — BASELINE config 5: n = 2^27 f64 U(0,1) + u32 index, one sort per mode",
       "", "`tools/ncu_cfg5.sh` (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
       "--clock-control none`; cold-cache serialised replay: compare shares and bytes, not absolutes).", ""]
for f in ("1.0", "0.5"):
    p = os.path.join(D, f"launches_cfg5_{f}.csv")
    if not os.path.exists(p):
        continue
    per = launches(p)
    out += [f"## buffer fraction {f}", "", "| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |",
            "|---|---|---|---|---|"]
    tt = rb = wb = 0.0
    for i, ((_, k), m) in enumerate(per.items()):
        t = m.get("gpu__time_duration.sum", 0.0)
        r = m.get("dram__bytes_read.sum", 0.0)
        w = m.get("dram__bytes_write.sum", 0.0)
        tt += t
        rb += r
        wb += w
        out.append(f"| {i} | {k} | {t:.1f} | {r:.1f} | {w:.1f} |")
    lb = 15 * 2 * N * S / 1e6
    out += ["", f"Sum: {tt / 1e3:.2f} ms of kernel time, DRAM {rb + wb:.0f} MB (read {rb:.0f} + write {wb:.0f}) "
            f"against the lower bound P*2*n*s = 15 * 2 * 2^27 * 12 B = {lb:.0f} MB; "
            f"{(rb + wb) / (tt / 1e3):.0f} GB/s over the kernel time ({(rb + wb) / (tt / 1e3) / PEAK:.2f} "
            f"of the measured copy peak).", ""]
open(os.path.join(ROOT, "profiles", f"{TAG}_ncu_cfg5.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
