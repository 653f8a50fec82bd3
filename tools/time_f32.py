"""Per-kernel times (gns_timing) of binary32 sorts of 2^24 keys, key-only and with u32 payload."""
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2402_01816_b200 as gns
n = 1 << 24
g = torch.Generator(device="cuda"); g.manual_seed(3)
src = torch.rand(n, device="cuda", generator=g, dtype=torch.float32)
for pairs in (False, True):
    ws = torch.empty(max(1, gns.workspace_bytes_f32(n, pairs)), dtype=torch.uint8, device="cuda")
    per = []
    for i in range(4):
        k = src.clone(); v = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32) if pairs else None
        gns.gns_timing_begin(64)
        gns.sort_f32_(k, v, workspace=ws)
        per.append(gns.gns_timing_end())
    kinds = [gns.LAUNCH_KINDS.get(kd, "?") for kd, _ in per[-1]]
    med = [float(np.median([r[j][1] for r in per[1:]])) for j in range(len(kinds))]
    agg = {}
    for kd, t in zip(kinds, med): agg[kd] = agg.get(kd, 0) + t
    print("pairs", pairs, {a: round(b * 1e3, 1) for a, b in agg.items()}, "total", round(sum(med) * 1e3, 1), "us; per merge", [round(t*1e3,1) for kd,t in zip(kinds,med) if kd=="f32_merge"][:3])
