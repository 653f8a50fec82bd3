"""Summarise the ncu outputs of tools/gpu_round.sh into profiles/.

    python tools/summarize_ncu.py [gpurun_out] [tag]

Reads <dir>/launches.csv (per-launch gpu__time_duration + DRAM bytes, one
--profile-only bench run = warm-up sort + measured sort of BASELINE config 2)
and <dir>/prof_full.ncu-rep (--set full of the top kernels), writes
profiles/<tag>_ncu_summary.md and profiles/ncu_merge_traffic.json (the DRAM
traffic per merge-pass launch that bench.py reports as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r2"
PROF = os.path.join(ROOT, "profiles")
os.makedirs(PROF, exist_ok=True)


def short(name):
    for k in ("tile_sort2_kernel", "merge_tstore_kernel", "partition_kernel", "inplace_deps_kernel",
              "merge_kernel", "vectorized_elementwise_kernel"):
        if k in name:
            return k
    return name[:40]


def launches():
    rows = list(csv.reader(open(os.path.join(D, "launches.csv"))))
    hdr = None
    per = OrderedDict()
    seq = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), short(d["Kernel Name"]))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0) \
            if d["Metric Name"].startswith("dram__bytes") else 1.0
        per.setdefault(key, {})[d["Metric Name"]] = v * scale          # DRAM bytes -> MB
    for (i, k), m in per.items():
        seq.append((i, k, m))
    return seq


def raw_full():
    out = subprocess.check_output(["ncu", "-i", os.path.join(D, "prof_full.ncu-rep"), "--page", "raw", "--csv"],
                                  stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append(d)
    return res


def main():
    seq = launches()
    # the second sort of the run is the measured one: take launches after the second fill kernel
    fills = [i for i, (_, k, _) in enumerate(seq) if k == "vectorized_elementwise_kernel"]
    start = fills[-1] + 1 if fills else len(seq) // 2
    step = [x for x in seq[start:] if x[1] != "vectorized_elementwise_kernel"]
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, _, m in step)
    lines = [f"# ncu summary ({TAG}) — BASELINE config 2 (n = 2^24 f64 U(0,1), key-only, buffer 1.0)", "",
             "Launch list of one sort (`bench.py --profile-only`, ncu `--clock-control none`, cold-cache "
             "serialised replay: compare shares, not absolutes).", "",
             "| # | kernel | time (us) | share | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|---|"]
    merge_bytes = []
    merge_t = []
    for j, (i, k, m) in enumerate(step):
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        rd = m.get("dram__bytes_read.sum", 0)
        wr = m.get("dram__bytes_write.sum", 0)
        # ncu reports bytes in the unit the csv states (MB for these metrics by default)
        lines.append(f"| {j} | {k} | {t:.1f} | {100 * m.get('gpu__time_duration.sum', 0) / tot:.1f}% | "
                     f"{rd:.1f} | {wr:.1f} |")
        if k == "merge_tstore_kernel":
            merge_bytes.append((rd + wr) * 1e6)
            merge_t.append(t)
    lines.append("")
    lines.append(f"Sum of kernel times: {tot / 1e3:.1f} us.  Merge passes: {len(merge_t)}, share "
                 f"{100 * sum(merge_t) * 1e3 / tot:.1f}%.")
    n = 1 << 24
    if merge_bytes:
        avg = sum(merge_bytes) / len(merge_bytes)
        lines.append(f"Average DRAM traffic per merge-pass launch: {avg / 1e6:.1f} MB "
                     f"(algorithmic 2*n*8 = {2 * n * 8 / 1e6:.1f} MB).")
        json.dump({"n": n, "payload": False, "dram_bytes_per_launch": avg,
                   "algorithmic_bytes_per_launch": 2 * n * 8,
                   "source": f"profiles/{TAG}_ncu_summary.md (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                             f"mean over the {len(merge_bytes)} merge_tstore_kernel launches of one sort)"},
                  open(os.path.join(PROF, "ncu_merge_traffic.json"), "w"), indent=1)
    try:
        full = raw_full()
        lines += ["", "## `--set full` captures", "",
                  "| kernel | time (us) | DRAM R+W (MB) | DRAM % peak | L1/TEX % | issue active % | regs | warps/SM | "
                  "smem bank conflicts / wavefronts | UBLKCP/UTMA in SASS |", "|---|---|---|---|---|---|---|---|---|---|"]
        for d in full:
            def g(k, default="-"):
                return d.get(k, default)
            rd = float(g("dram__bytes_read.sum", 0) or 0)
            wr = float(g("dram__bytes_write.sum", 0) or 0)
            lines.append(
                f"| {short(g('Kernel Name'))} | {float(g('gpu__time_duration.sum', 0)):.1f} | {rd + wr:.1f} | "
                f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                f"{g('l1tex__throughput.avg.pct_of_peak_sustained_active')} | "
                f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | {g('launch__registers_per_thread')} | "
                f"{g('sm__warps_active.avg.per_cycle_active')} | "
                f"{g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')} / "
                f"{g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')} | profiles/r2_sass_tma.txt |")
    except Exception as e:  # noqa: BLE001
        lines.append(f"(full capture unavailable: {e})")
    open(os.path.join(PROF, f"{TAG}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
