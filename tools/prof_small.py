"""Phase clocks of the one-cluster small sort (CTA 0, profiling build):
GNS_LIB=libgns_prof.so python tools/prof_small.py [--pairs]"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
lib = gns._lib
lib.gns_prof_read.argtypes = [ctypes.c_void_p]
n = 1 << 16
src = torch.from_numpy(synth.uniform(n, 5)).cuda()
srcv = torch.from_numpy(synth.iota_u32(n)).cuda() if a.pairs else None
k, v = src.clone(), (srcv.clone() if a.pairs else None)
for _ in range(3):
    k.copy_(src)
    if a.pairs:
        v.copy_(srcv)
    gns.sort_(k, v)
torch.cuda.synchronize()
reps = 20
lib.gns_prof_reset()
for _ in range(reps):
    k.copy_(src)
    if a.pairs:
        v.copy_(srcv)
    gns.sort_(k, v)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib.gns_prof_read(buf)
names = ["pdl_wait", "loaded", "transposed", "local_rounds", "cl_sync1", "cl_search1", "cl_copy1", "cluster_levels", "end"]
print(f"pairs={a.pairs}: " + " ".join(f"{nm}={buf[q] / reps / 1965:.2f}us" for q, nm in enumerate(names)))
