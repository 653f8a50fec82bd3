"""Two binary32 sorts of 2^24 keys (for ncu captures of the f32 kernels).
usage: python tools/f32_once.py [--pairs]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402

pairs = "--pairs" in sys.argv
n = 1 << 24
g = torch.Generator(device="cuda")
g.manual_seed(3)
src = torch.rand(n, device="cuda", generator=g, dtype=torch.float32)
ws = torch.empty(max(1, gns.workspace_bytes_f32(n, pairs)), dtype=torch.uint8, device="cuda")
for _ in range(2):
    k = src.clone()
    v = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32) if pairs else None
    gns.sort_f32_(k, v, workspace=ws)
torch.cuda.synchronize()
print("sorted", bool((k[1:] >= k[:-1]).all()))
