"""Event-timed K1 tile sort (gns_tile_sort) and whole sorts, for A/B runs.
usage: python tools/time_k1.py [--n 24] [--reps 20]   (GNS_K1=2 selects the 256x32 key-only K1)"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
n = 1 << a.n
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:])), float(np.min(ts[2:]))


for name, keys in (("uniform", synth.uniform(n, 5)), ("ties24", synth.ties(n, 6, 24))):
    for pairs in (False, True):
        src = torch.from_numpy(keys).cuda()
        sv = torch.from_numpy(synth.iota_u32(n)).cuda() if pairs else None
        dk = torch.empty_like(src)
        dv = torch.empty_like(sv) if pairs else None
        med, mn = timed(lambda: gns.tile_sort(src, sv, dk, dv), a.reps)
        # spot-check the tile sort against the oracle on a few tiles
        T1 = gns.gns_tile_elems()
        hk = dk.cpu().numpy()
        hv = dv.cpu().numpy() if pairs else None
        for t in (0, 7, n // T1 - 1):
            sl = slice(t * T1, (t + 1) * T1)
            ek, ev = oracle.sort(keys[sl], synth.iota_u32(n)[sl] if pairs else None)
            assert np.array_equal(hk[sl].view(np.uint64), ek.view(np.uint64)), f"tile {t} keys"
            if pairs:
                assert np.array_equal(hv[sl], ev), f"tile {t} vals"
        ws = gns.alloc_workspace(n, 1.0, pairs)
        k2 = torch.empty_like(src)
        v2 = torch.empty_like(sv) if pairs else None

        def whole():
            k2.copy_(src)
            if pairs:
                v2.copy_(sv)
            gns.sort_(k2, v2, 1.0, workspace=ws)
        # (the copy is inside the timed region: subtract it)
        cmed, _ = timed(lambda: (k2.copy_(src), v2.copy_(sv) if pairs else None), a.reps)
        wmed, _ = timed(whole, a.reps)
        ek, ev = oracle.sort(keys[: 1 << 20], synth.iota_u32(1 << 20) if pairs else None)
        ok = bool(np.all(np.diff(k2.cpu().numpy()) >= 0))
        print(f"K1={os.environ.get('GNS_K1', '3')} n=2^{a.n} {name:8s} pairs={int(pairs)} tile_sort {med*1e3:7.1f} us "
              f"(min {mn*1e3:7.1f})  whole sort {(wmed - cmed)*1e3:7.1f} us  sorted={ok}", flush=True)
