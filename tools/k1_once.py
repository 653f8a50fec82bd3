"""One K1 tile sort of 2^24 uniform keys (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

n = 1 << int(os.environ.get("K1_N", "24"))
pairs = os.environ.get("K1_PAIRS", "0") == "1"
src = torch.from_numpy(synth.uniform(n, 5)).cuda()
sv = torch.from_numpy(synth.iota_u32(n)).cuda() if pairs else None
dk = torch.empty_like(src)
dv = torch.empty_like(sv) if pairs else None
for _ in range(3):
    gns.tile_sort(src, sv, dk, dv)
torch.cuda.synchronize()
print("ok")
