"""Phase breakdown of the merge passes (profiling build libgns_prof.so).
usage: GNS_LIB=libgns_prof.so python tools/prof_merge.py [--n 24]
Prints, per pass, the average per-CTA time (us at 1965 MHz) thread 0 spent in
each phase of merge_tstore_kernel."""
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
ap.add_argument("--ties", type=int, default=0, help="heavy ties: keys uniform integers in [0, T)")
a = ap.parse_args()
lib = gns._lib
lib.gns_prof_read.argtypes = [ctypes.c_void_p]
n = 1 << a.n
T = gns.gns_tile_elems()
src = torch.from_numpy(synth.ties(n, 2000, a.ties) if a.ties else synth.uniform(n, 2000)).cuda()
names = ["startup", "wait_load", "compute", "bar1", "staging+bar2", "store_read", "issue", "total", "split_spin"]
cur = torch.empty_like(src)
oth = torch.empty_like(src)
mws = torch.empty(gns.gns_merge_workspace_bytes(n), dtype=torch.uint8, device="cuda")
vp, sz = ctypes.c_void_p, ctypes.c_size_t
assert lib.gns_tile_sort(vp(src.data_ptr()), None, vp(cur.data_ptr()), None, sz(n), None) == 0
print(f"n=2^{a.n}")
L = T
while L < n:
    for rep in range(2):
        lib.gns_prof_reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.gns_merge_pass(vp(cur.data_ptr()), None, vp(oth.data_ptr()), None, sz(n), sz(L),
                                vp(mws.data_ptr()), sz(mws.numel()), None)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0
    buf = (ctypes.c_ulonglong * 16)()
    lib.gns_prof_read(buf)
    ctas = max(buf[10], 1)
    us = e0.elapsed_time(e1) * 1e3
    row = " ".join(f"{names[q]}={buf[q] / ctas / 1965:.1f}" for q in range(9))
    row += " | merge t0: " + " ".join(f"{nm}={buf[q] / ctas / 1965:.1f}" for q, nm in
                                      ((11, "flag"), (12, "split0"), (13, "full0"), (14, "end")))
    print(f"L=2^{L.bit_length() - 1} {us:.1f}us tiles/cta={buf[9] / ctas:.1f} | {row}", flush=True)
    cur, oth = oth, cur
    L *= 2
ok = bool((cur[1:] >= cur[:-1]).all())
print("sorted:", ok)
# the product path (sample-guided searches): counters summed over one whole sort
k = src.clone()
ws = gns.alloc_workspace(n, 1.0, False)
gns.sort_(k, None, 1.0, workspace=ws)
for rep in range(2):
    k.copy_(src)
    torch.cuda.synchronize()
    lib.gns_prof_reset()
    gns.sort_(k, None, 1.0, workspace=ws)
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib.gns_prof_read(buf)
ctas = max(buf[10], 1)
row = " ".join(f"{names[q]}={buf[q] / ctas / 1965:.1f}" for q in range(9))
row += " | merge t0: " + " ".join(f"{nm}={buf[q] / ctas / 1965:.1f}" for q, nm in
                                  ((11, "flag"), (12, "split0"), (13, "full0"), (14, "end")))
print(f"whole sort, avg per pass: {row}")
tl = (ctypes.c_ulonglong * 64)()
lib.gns_prof_timeline(tl)
t0 = tl[0]
prev_end = None
for i in range(32):
    a, b = tl[2 * i], tl[2 * i + 1]
    if b == 0:
        continue
    gap = f" gap {(a - prev_end) / 1e3:6.2f}" if prev_end else ""
    print(f"  slot {i:2d}: start {(a - t0) / 1e3:8.2f} us  end {(b - t0) / 1e3:8.2f} us  dur {(b - a) / 1e3:7.2f}{gap}")
    prev_end = b
