"""Bit-exact check of small sorts (the one-cluster path, n <= 65536) against
torch's stable sort on the GPU, keys-only and with a u32 index payload, for
the library named by GNS_LIB: python tools/check_small.py."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

bad = 0
cases = 0
for n in (2, 7, 100, 4095, 4096, 4097, 8191, 12345, 20000, 32768, 40000, 65535, 65536):
    for inp in ("uniform", "ties", "desc"):
        src = {"uniform": lambda: synth.uniform(n, 11 + n), "ties": lambda: synth.ties(n, 3, 5),
               "desc": lambda: synth.uniform(n, 5 + n)}[inp]()
        ks = torch.from_numpy(src).cuda()
        if inp == "desc":
            ks = torch.sort(ks, descending=True).values.contiguous()
        ek, ei = torch.sort(ks, stable=True)
        for hv in (False, True):
            k = ks.clone()
            v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if hv else None
            gns.sort_(k, v)
            torch.cuda.synchronize()
            ok = torch.equal(k.view(torch.int64), ek.view(torch.int64))
            if hv:
                ok = ok and torch.equal(v.view(torch.int32).to(torch.int64), ei)
            cases += 1
            if not ok:
                bad += 1
                print(f"MISMATCH n={n} input={inp} payload={hv}", flush=True)
print(f"check_small: {cases} cases, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
