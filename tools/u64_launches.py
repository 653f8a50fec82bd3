"""Per-kind launch times of one gns_sort_keys_u64 sort of 2^27 keys (gns_timing)."""
import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2402_01816_b200 as gns, synth
n = 1 << 27
k = torch.from_numpy(synth.uniform(n, 2000)).cuda()
p = torch.arange(n, dtype=torch.int64, device="cuda")
ws = torch.empty(gns.workspace_bytes_u64(n), dtype=torch.uint8, device="cuda")
gns.sort_u64_(k.clone(), p.clone(), workspace=ws)
torch.cuda.synchronize()
kk, pp = k.clone(), p.clone()
gns.gns_timing_begin(256)
gns.sort_u64_(kk, pp, workspace=ws)
torch.cuda.synchronize()
res = gns.gns_timing_end()
from collections import defaultdict
agg = defaultdict(float)
for kd, ms in res:
    agg[gns.LAUNCH_KINDS.get(kd, kd)] += ms
print({k: round(v, 3) for k, v in agg.items()})
