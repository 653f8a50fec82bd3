"""Times gns_sort_* on one config (CUDA events, L2 flushed, input restored
untimed); prints one line.  For A/B experiments: python tools/time_sort.py
[--n 24] [--pairs] [--frac 1.0] [--reps 20] [--omit] [--input uniform|asc|desc|swap1pct|runs16]."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--pairs", action="store_true")
ap.add_argument("--frac", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--tag", default="")
ap.add_argument("--omit", action="store_true", help="gns_sort_omit (Omitsort schedule)")
ap.add_argument("--input", default="uniform")
ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between reps (code + data)")
a = ap.parse_args()
n = 1 << a.n
src = torch.from_numpy(synth.uniform(n, 2000) if a.input == "uniform" else synth.config(4, a.input, n).keys).cuda()
srcv = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
k = torch.empty_like(src)
v = torch.empty_like(srcv) if a.pairs else None
ws = gns.alloc_workspace(n, a.frac, a.pairs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(a.reps + 3):
    k.copy_(src)
    if a.pairs:
        v.copy_(srcv)
    if not a.no_flush:
        flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if a.omit:
        gns.sort_omit_(k, v, workspace=ws)
    else:
        gns.sort_(k, v, a.frac, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ok = bool((k[1:] >= k[:-1]).all())
print(f"{a.tag} {a.input} omit={a.omit} n=2^{a.n} pairs={a.pairs} frac={a.frac} median_ms={np.median(ts):.4f} min_ms={min(ts):.4f} "
      f"Gkeys/s={n / np.median(ts) / 1e6:.2f} sorted={ok}", flush=True)
