import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2402_01816_b200 as gns, synth, oracle
ok_all = True
for n in [2*8192*2 + 5, 4*8192, 4*8192 + 1, 16*8192 + 333, 1 << 20, (1 << 22) + 12345, 1 << 24]:
    for kind in ("uniform", "ties", "asc", "desc"):
        if kind == "uniform": k = synth.uniform(n, n)
        elif kind == "ties": k = synth.ties(n, n, 24)
        elif kind == "asc": k = np.arange(n, dtype=np.float64)
        else: k = np.arange(n, 0, -1, dtype=np.float64)
        t = torch.from_numpy(k).cuda()
        gns.sort_(t, None, 1.0, workspace=gns.alloc_workspace(n, 1.0, False))
        torch.cuda.synchronize()
        g = t.cpu().numpy()
        e = np.sort(k, kind="stable")
        ok = np.array_equal(g.view(np.uint64), e.view(np.uint64))
        ok_all &= ok
        if not ok:
            bad = np.flatnonzero(g.view(np.uint64) != e.view(np.uint64))
            print("FAIL", n, kind, bad.size, bad[:5], flush=True)
print("all ok" if ok_all else "FAILURES")
