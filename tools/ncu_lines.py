"""Per-source-line hot spots from an `ncu --page source --csv --print-source cuda,sass` dump.
usage: python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
tot = 0
lines = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[0] == "":
        continue
    s = num(r[ix["Warp Stall Sampling (All Samples)"]])
    lines.append((s, r[0], r[1].strip()[:100], num(r[ix["L1 Wavefronts Shared"]]),
                  num(r[ix["L1 Wavefronts Shared Ideal"]]), num(r[ix["Instructions Executed"]])))
    tot += s
lines.sort(reverse=True)
print("total samples", tot)
for s, ln, src, wf, ideal, inst in lines[:top]:
    print(f"{s:8.0f} {100 * s / max(tot, 1):5.1f}% L{ln:>5} wf={wf:.0f} ideal={ideal:.0f} inst={inst:.0f} | {src}")
