"""Exactly one sort of a BASELINE-shaped input (for ncu launch lists).
usage: python tools/one_sort.py [--n 27] [--pairs] [--frac 1.0]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=27)
ap.add_argument("--pairs", action="store_true")
ap.add_argument("--frac", type=float, default=1.0)
a = ap.parse_args()
n = 1 << a.n
k = torch.from_numpy(synth.uniform(n, 2000)).cuda()
v = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
ws = gns.alloc_workspace(n, a.frac, a.pairs)
gns.sort_(k, v, a.frac, workspace=ws)
torch.cuda.synchronize()
print("sorted", bool((k[1:] >= k[:-1]).all()))
