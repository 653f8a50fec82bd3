"""Times gns_sort_keys_u64 (f64 keys + 64-bit payload) against the u32-payload
sort on BASELINE config 2 keys (CUDA events, L2 flushed).
usage: python tools/time_u64.py [--n 24]"""
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
a = ap.parse_args()
n = 1 << a.n
src = torch.from_numpy(synth.uniform(n, 2000)).cuda()
p64 = torch.arange(n, dtype=torch.int64, device="cuda")
p32 = torch.arange(n, dtype=torch.int64, device="cuda").to(torch.uint32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws64 = torch.empty(gns.workspace_bytes_u64(n), dtype=torch.uint8, device="cuda")
ws32 = gns.alloc_workspace(n, 1.0, True)
for name in ("u32", "u64"):
    ts = []
    for i in range(13):
        k = src.clone()
        v = (p64 if name == "u64" else p32).clone()
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "u64":
            gns.sort_u64_(k, v, workspace=ws64)
        else:
            gns.sort_(k, v, 1.0, workspace=ws32)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(f"n=2^{a.n} payload={name} median_ms={np.median(ts):.4f}", flush=True)
