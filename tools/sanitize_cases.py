"""Small sorts over every code path, for compute-sanitizer (memcheck / racecheck
/ synccheck / initcheck, one tool per run).  Exits 1 on a wrong result."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

T = gns.gns_tile_elems()
bad = 0
for n in (1, 100, T - 3, T + 1, 3 * T + 77, 9 * T + 5):
    for frac in (1.0, 0.5, 0.25):
        for hv in (False, True):
            for target in ("AscLeft", "DescRight"):
                k = synth.ties(n, n + 7, 50)
                v = synth.iota_u32(n)
                tk = torch.from_numpy(k).cuda()
                tv = torch.from_numpy(v).cuda() if hv else None
                gns.sort_(tk, tv, frac, target=target)
                torch.cuda.synchronize()
                order = np.argsort(k, kind="stable")
                exp = k[order]
                if target == "DescRight":
                    exp = exp[::-1]
                if not np.array_equal(tk.cpu().numpy(), exp):
                    print("MISMATCH", n, frac, hv, target)
                    bad += 1
print("cases done, mismatches:", bad)
sys.exit(1 if bad else 0)
