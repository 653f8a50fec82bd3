"""Per-launch times (gns_timing_begin/end) of one sort.
usage: python tools/time_launches.py [--n 27] [--pairs] [--frac 0.5]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=27)
ap.add_argument("--pairs", action="store_true")
ap.add_argument("--frac", type=float, default=0.5)
ap.add_argument("--omit", action="store_true")
ap.add_argument("--input", default="uniform")
ap.add_argument("--u64", action="store_true", help="gns_sort_keys_u64 (64-bit payload)")
a = ap.parse_args()
n = 1 << a.n
src = torch.from_numpy(synth.uniform(n, 9) if a.input == "uniform" else synth.config(4, a.input, n).keys).cuda()
srcv = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
k = torch.empty_like(src)
v = torch.empty_like(srcv) if a.pairs else None
ws = gns.alloc_workspace(n, a.frac, a.pairs)
if a.u64:
    v64 = torch.arange(n, device="cuda", dtype=torch.int64)
    ws64 = torch.empty(gns.workspace_bytes_u64(n), dtype=torch.uint8, device="cuda")
per = []
for i in range(3):
    k.copy_(src)
    if a.pairs:
        v.copy_(srcv)
    assert gns.gns_timing_begin(512) == 0
    if a.u64:
        gns.sort_u64_(k, v64, workspace=ws64)
    elif a.omit:
        gns.sort_omit_(k, v, workspace=ws)
    else:
        gns.sort_(k, v, a.frac, workspace=ws)
    per.append(gns.gns_timing_end())
kinds = [gns.LAUNCH_KINDS.get(kd, "?") for kd, _ in per[-1]]
med = [float(np.median([r[j][1] for r in per[1:]])) for j in range(len(kinds))]
tot = sum(med)
agg = {}
for kd, t in zip(kinds, med):
    agg[kd] = agg.get(kd, 0.0) + t
print(f"n=2^{a.n} pairs={a.pairs} frac={a.frac} total {tot:.3f} ms over {len(med)} launches")
for kd, t in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {kd:14s} {t:.3f} ms ({100 * t / tot:.1f}%)  launches {kinds.count(kd)}")
big = [(kd, t) for kd, t in zip(kinds, med) if kd in ("inplace_merge", "partition", "inplace_deps")]
print("  in-place steps:", " ".join(f"{kd}:{t*1e3:.0f}us" for kd, t in big))
print("  per launch:", " ".join(f"{kd}:{t*1e3:.1f}" for kd, t in zip(kinds, med)))
