"""Counts the Blackwell data-movement instructions in the SASS of each kernel
of libgns.so (TMA tensor loads/stores UTMALDG/UTMASTG, bulk copies UBLKCP,
mbarrier ops SYNCS, programmatic-launch control) -> profiles/r2_sass_tma.txt.
usage: python tools/sass_evidence.py"""
import os
import re
import subprocess
from collections import Counter, OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2402_01816_b200", "libgns.so")
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ("UTMALDG", "UTMASTG", "UBLKCP", "UTMACMDFLUSH", "SYNCS", "LDS", "STS", "LDG", "STG", "ACQBULK")
per = OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(2)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                per[cur][o] += 1
out = ["# SASS evidence (r2): data-movement instructions per kernel of libgns.so (sm_100a)", "",
       "UTMALDG / UTMASTG = TMA tensor load / store, UBLKCP = TMA 1-D bulk copy, SYNCS = mbarrier ops,",
       "ACQBULK = griddepcontrol.wait (programmatic dependent launch).  `python tools/sass_evidence.py`.", "",
       "| kernel (mangled, ORD 0 instances) | " + " | ".join(OPS) + " |", "|---|" + "---|" * len(OPS)]
for f, c in per.items():
    if not re.search(r"ILi0E|ILb0ELi0E|ILb1ELi0E|Kernel[^I]*$|nan_count|iota|gather|f32_|reverse|split_cuts|inplace_deps", f):
        continue
    out.append(f"| `{f[:90]}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
open(os.path.join(ROOT, "profiles", "r2_sass_tma.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
