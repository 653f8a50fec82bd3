"""Per-kernel times of one sort for a few input shapes (A/B tool).
usage: python tools/time_cfg.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

n = 1 << 24
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, keys, pairs in (("uniform key-only", synth.uniform(n, 1), False), ("uniform pairs", synth.uniform(n, 1), True),
                          ("ties24 key-only", synth.ties(n, 2, 24), False), ("ties24 pairs", synth.ties(n, 2, 24), True),
                          ("ties1000 pairs", synth.ties(n, 3, 1000), True)):
    src = torch.from_numpy(keys).cuda()
    srcv = torch.from_numpy(synth.iota_u32(n)).cuda() if pairs else None
    k = torch.empty_like(src)
    v = torch.empty_like(srcv) if pairs else None
    ws = gns.alloc_workspace(n, 1.0, pairs)
    per = []
    for i in range(4):
        k.copy_(src)
        if pairs:
            v.copy_(srcv)
        flush.fill_(1)
        assert gns.gns_timing_begin(64) == 0
        gns.sort_(k, v, 1.0, workspace=ws)
        per.append(gns.gns_timing_end())
    med = [float(np.median([r[j][1] for r in per[1:]])) for j in range(len(per[0]))]
    print(f"{name:18s} total {sum(med):.3f} ms  tile {med[0]*1e3:.0f} us  merges {' '.join(f'{x*1e3:.0f}' for x in med[1:])}",
          flush=True)
