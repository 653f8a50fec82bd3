"""Timeline of the pipelined multi-pass merge (profiling build libgns_prof.so).
usage: GNS_LIB=libgns_prof.so python tools/prof_multi.py [--n 24] [--pairs]"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
lib = gns._lib
lib.gns_prof_read.argtypes = [ctypes.c_void_p]
lib.gns_prof_timeline.argtypes = [ctypes.c_void_p]
n = 1 << a.n
src = torch.from_numpy(synth.uniform(n, 2000)).cuda()
sv = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
ws = gns.alloc_workspace(n, 1.0, a.pairs)
for rep in range(3):
    k = src.clone()
    v = sv.clone() if a.pairs else None
    torch.cuda.synchronize()
    lib.gns_prof_reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gns.sort_(k, v, 1.0, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
tl = (ctypes.c_ulonglong * 64)()
lib.gns_prof_timeline(tl)
pr = (ctypes.c_ulonglong * 16)()
lib.gns_prof_read(pr)
print(f"n=2^{a.n} pairs={a.pairs} sort {e0.elapsed_time(e1) * 1e3:.1f} us, sorted={bool((k[1:] >= k[:-1]).all())}")
t0 = min(tl[2 * i] for i in range(32) if tl[2 * i] != 2**64 - 1)
for i in range(32):
    if tl[2 * i] != 2**64 - 1:
        print(f"  slot {i:2d}: {(tl[2 * i] - t0) / 1e3:8.1f} .. {(tl[2 * i + 1] - t0) / 1e3:8.1f} us")
cnt = max(pr[2], 1)
print(f"  searches: {pr[2]} tiles, dep wait {pr[0] / cnt / 1965:.2f} us/tile, search {pr[1] / cnt / 1965:.2f} us/tile, "
      f"producer idle {pr[3] / 1965 / 296:.1f} us/CTA")
print(f"  producer per CTA: issue {pr[5] / 1965 / 296:.1f} us, "
      f"wait_pend {pr[6] / 1965 / 296:.1f} us, wait_read {pr[7] / 1965 / 296:.1f} us")
