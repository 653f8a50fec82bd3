"""Times gns_sort_f32 (binary32 keys, key-only and with u32 payload) at 2^n
(CUDA events, L2 flushed).  usage: python tools/time_f32.py [--n 24]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
a = ap.parse_args()
n = 1 << a.n
g = torch.Generator(device="cuda")
g.manual_seed(1)
src = torch.rand(n, device="cuda", generator=g, dtype=torch.float32)
pay = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = torch.empty(gns.workspace_bytes_f32(n, True), dtype=torch.uint8, device="cuda")
for hv in (False, True):
    ts = []
    for i in range(13):
        k = src.clone()
        v = pay.clone() if hv else None
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gns.sort_f32_(k, v, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ok = bool((k[1:] >= k[:-1]).all())
    print(f"n=2^{a.n} f32 payload={hv} median_ms={np.median(ts):.4f} Gkeys/s={n / np.median(ts) / 1e6:.2f} "
          f"sorted={ok}", flush=True)
