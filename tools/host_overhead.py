"""Host-side cost of one sort call (no sync), and the GPU time of the same
sort replayed from a CUDA graph: small sorts are launch/host-bound.
usage: python tools/host_overhead.py [--n 16] [--pairs]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
n = 1 << a.n
src = torch.from_numpy(synth.uniform(n, 2000)).cuda()
srcv = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
k = src.clone()
v = srcv.clone() if a.pairs else None
ws = gns.alloc_workspace(n, 1.0, a.pairs)
st = torch.cuda.current_stream()
for _ in range(10):
    gns.sort_(k, v, 1.0, workspace=ws)
torch.cuda.synchronize()
# host time per call (python wrapper + C-ABI + launches), GPU queue kept busy
reps = 200
t0 = time.perf_counter()
for _ in range(reps):
    gns.sort_(k, v, 1.0, workspace=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"n=2^{a.n} pairs={a.pairs}: host {1e6 * (t1 - t0) / reps:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / reps:.1f} us/call")
# GPU time per sort: a CUDA graph of 20 sorts (input restored inside the graph)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(st)
with torch.cuda.stream(s):
    for _ in range(3):
        k.copy_(src)
        if a.pairs:
            v.copy_(srcv)
        gns.sort_(k, v, 1.0, workspace=ws, stream=s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            k.copy_(src)
            if a.pairs:
                v.copy_(srcv)
            gns.sort_(k, v, 1.0, workspace=ws, stream=s)
st.wait_stream(s)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 20)
ok = bool((k[1:] >= k[:-1]).all())
print(f"  graph replay: {1e3 * float(np.median(ts)):.1f} us per (restore + sort), sorted={ok}")
