"""Per-kind launch times of one gns_sort_f32 sort (gns_timing).
usage: python tools/f32_launches.py [--n 24] [--pairs]"""
import argparse
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
n = 1 << a.n
k = torch.rand(n, device="cuda", dtype=torch.float32)
v = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32) if a.pairs else None
ws = torch.empty(gns.workspace_bytes_f32(n, True), dtype=torch.uint8, device="cuda")
gns.sort_f32_(k.clone(), None if v is None else v.clone(), workspace=ws)
torch.cuda.synchronize()
kk, vv = k.clone(), (None if v is None else v.clone())
gns.gns_timing_begin(256)
gns.sort_f32_(kk, vv, workspace=ws)
torch.cuda.synchronize()
agg = defaultdict(float)
cnt = defaultdict(int)
for kd, ms in gns.gns_timing_end():
    agg[gns.LAUNCH_KINDS.get(kd, kd)] += ms
    cnt[gns.LAUNCH_KINDS.get(kd, kd)] += 1
print(f"n=2^{a.n} pairs={a.pairs}", {k: (round(v, 3), cnt[k]) for k, v in agg.items()})
