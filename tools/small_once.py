"""A few on-chip small sorts (2^16 keys + u32 payload, one 16-CTA cluster) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

n = 1 << 16
k = torch.from_numpy(synth.uniform(n, 5)).cuda()
v = torch.from_numpy(synth.iota_u32(n)).cuda()
for _ in range(3):
    gns.sort_(k, v)
torch.cuda.synchronize()
print("sorted", bool((k[1:] >= k[:-1]).all()))
