"""Quick bit-exact check of the product sort against torch's stable sort on
the GPU (keys-only and with a u32 index payload) over sizes that exercise
the schedules (split-stream halves with odd and even level counts, ragged
right halves) and presorted inputs.  For schedule A/B work before the full
oracle suite: python tools/check_sched.py."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

sizes = [(1 << 20) + 777, (1 << 21) + 5, 3 * (1 << 21) + 13, 1 << 22, (1 << 23) - 1, 1 << 23,
         (1 << 23) + 4096 * 3 + 1, 1 << 24, (1 << 24) - 123]
bad = 0
for n in sizes:
    for inp in ("uniform", "ties", "asc", "desc", "swap1pct"):
        if inp == "uniform":
            src = synth.uniform(n, 77 + n % 1000)
        elif inp == "ties":
            src = synth.ties(n, 5, 24)
        else:
            src = synth.config(4, inp, n).keys
        ks = torch.from_numpy(src).cuda()
        ek, ei = torch.sort(ks, stable=True)
        for hv in (False, True):
            for frac in (1.0, 0.5):
                k = ks.clone()
                v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if hv else None
                gns.sort_(k, v, frac)
                torch.cuda.synchronize()
                ok = torch.equal(k.view(torch.int64), ek.view(torch.int64))
                if hv:
                    ok = ok and torch.equal(v.view(torch.int32).to(torch.int64), ei)
                if not ok:
                    bad += 1
                    print(f"MISMATCH n={n} input={inp} payload={hv} frac={frac}", flush=True)
print(f"check_sched: {len(sizes) * 5 * 4} cases, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
