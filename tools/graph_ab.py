"""Stream launches vs one CUDA-graph replay of the same sort (2^24 f64)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
src = torch.from_numpy(synth.uniform(n, 5)).cuda()
k = src.clone()
ws = gns.alloc_workspace(n, 1.0, False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    for _ in range(3):
        k.copy_(src)
        gns.sort_(k, None, 1.0, workspace=ws, stream=s)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    gns.sort_(k, None, 1.0, workspace=ws, stream=s)
torch.cuda.synchronize()


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        k.copy_(src)
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[3:]))


t_stream = timeit(lambda: gns.sort_(k, None, 1.0, workspace=ws))
t_graph = timeit(lambda: g.replay())
ok = bool((k[1:] >= k[:-1]).all())
print(f"n=2^{n.bit_length()-1} stream {t_stream:.4f} ms  graph {t_graph:.4f} ms  sorted={ok}")
