"""The A/B code paths selected by environment knobs (read once per process,
so each runs in a subprocess): GNS_MULTI=1 (all merge levels in one
persistent launch), GNS_CHAIN=1 (chained passes on region counters),
GNS_K1=2 (the 256 x 32 key-only tile sort), GNS_K1_CL=8 / 16 (the key-only
tile sort merging a thread-block cluster's tiles on chip), GNS_MERGE_MODE=1
(ticket passes for every size), GNS_SMALL=0 (tile sort + merge passes for
n <= 65536), GNS_FOUR=1 (key-only 4-way merge passes, gns_merge4.cuh),
GNS_COOP=0 (the merge pass's TMA boxes issued by one producer lane).  Each sorts a few seeded inputs through the C-ABI and
compares bit-exactly with the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT_DIR)
import oracle, synth, paper_2402_01816_b200 as gns
bad = 0
for n, seed, pay in ((3 * 8192 + 77, 1, True), (1 << 20, 2, False), ((1 << 21) + 5, 3, True), (40000, 4, False),
                     (65536, 5, True), (9000, 6, False)):
    k = synth.ties(n, seed, 1000) if seed % 2 else synth.uniform(n, seed)
    v = synth.iota_u32(n) if pay else None
    ek, ev = oracle.sort(k, v)
    for frac in (1.0, 0.5):
        tk = torch.from_numpy(k.copy()).cuda()
        tv = None if v is None else torch.from_numpy(v.copy()).cuda()
        gns.sort_(tk, tv, frac)
        torch.cuda.synchronize()
        ok = np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64))
        ok = ok and (v is None or np.array_equal(tv.cpu().numpy(), ev))
        if not ok:
            bad += 1
            print("FAIL", n, frac, pay)
# ordered / strictly reversed inputs (the adaptive shortcuts inside the variant)
for k in (np.arange(3 * 8192 + 5, dtype=np.float64), np.arange(5 * 8192, 0, -1).astype(np.float64),
          np.arange(20 * 8192, 0, -1).astype(np.float64), np.arange(37 * 8192 + 11, dtype=np.float64)):
    tk = torch.from_numpy(k.copy()).cuda()
    gns.sort_(tk, None, 1.0)
    torch.cuda.synchronize()
    if not np.array_equal(tk.cpu().numpy(), np.sort(k)):
        bad += 1
        print("FAIL presorted", k.size)
print("bad", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("env", [{"GNS_MULTI": "1"}, {"GNS_CHAIN": "1"}, {"GNS_K1": "2"}, {"GNS_MERGE_MODE": "1"}, {"GNS_SMALL": "0"},
                                 {"GNS_MERGE_MODE": "0"}, {"GNS_K1_CL": "8"}, {"GNS_K1_CL": "16"}, {"GNS_FOUR": "1"},
                                 {"GNS_FOUR": "1", "GNS_MERGE_MODE": "1"}, {"GNS_COOP": "0"}])
def test_env_variant_bitexact(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT_DIR", repr(ROOT))], capture_output=True, text=True, env=e, timeout=600)
    assert r.returncode == 0, (env, r.stdout[-2000:], r.stderr[-2000:])


# The 4-way passes (GNS_FOUR=1) on what only they see: an even level count
# (every pass 4-way, the tile sort writes the fine samples), partial last
# groups (1, 2 or 3 runs), heavy ties and signed zeros across the runs (the
# pivot tie rule), both directions and the integer key types, both buffer modes.
SCRIPT4 = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT_DIR)
import oracle, synth, paper_2402_01816_b200 as gns
T1 = 8192
bad = 0
sizes = [4 * T1, 4 * T1 + 1, 6 * T1 + 333, 7 * T1 - 3, 16 * T1, 17 * T1 + 9, (1 << 19) + 1, 1 << 20, 3 * (1 << 18) + 77]
for n in sizes:
    for kind in ("uniform", "ties3", "zeros", "runs"):
        if kind == "uniform":
            k = synth.uniform(n, n)
        elif kind == "ties3":
            k = synth.ties(n, n + 1, 3)
        elif kind == "zeros":
            k = synth.ties(n, n + 2, 3) - 1.0
            k[::5] = -0.0
            k[1::7] = 0.0
        else:
            k = synth.config(4, "runs16", n).keys
        for frac in (1.0, 0.5):
            tk = torch.from_numpy(k.copy()).cuda()
            gns.sort_(tk, None, frac)
            torch.cuda.synchronize()
            ek, _ = oracle.sort(k, None)
            if not np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64)):
                bad += 1
                print("FAIL", n, kind, frac)
# the four targets and the integer key types (gns_sort_keys), with payload-free keys
n = 9 * T1 + 5
rng = np.random.default_rng(7)
for target in ("AscLeft", "AscRight", "DescLeft", "DescRight"):
    k = synth.ties(n, 11, 50)
    tk = torch.from_numpy(k.copy()).cuda()
    gns.sort_(tk, None, 1.0, target=target)
    torch.cuda.synchronize()
    ek, _ = oracle.sort_target(k, None, target)
    if not np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64)):
        bad += 1
        print("FAIL target", target)
for kt, dt in (("i64", np.int64), ("u64", np.uint64)):
    k = rng.integers(0, 1000, n).astype(dt)
    k[::3] = np.iinfo(dt).max
    tk = torch.from_numpy(k.copy()).cuda()
    gns.sort_(tk, None, 1.0, target="DescLeft")
    torch.cuda.synchronize()
    ek, _ = oracle.sort_keys(k, None, kt, "DescLeft")
    if not np.array_equal(tk.cpu().numpy(), ek):
        bad += 1
        print("FAIL key type", kt)
print("bad", bad)
sys.exit(1 if bad else 0)
"""


def test_four_way_passes_bitexact():
    e = dict(os.environ, GNS_FOUR="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT4.replace("ROOT_DIR", repr(ROOT))], capture_output=True, text=True, env=e,
                       timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])


# The register network merges (compile-time knobs GNS_F2_NET / GNS_K1_NET, `make net`
# -> libgns_net.so): the binary32 key-only merge pass and K1's merge-path rounds (both
# key widths) merge a thread's outputs by a bitonic network unless -0.0 / NaN keys are
# present.  The f64 knob script and the binary32 parity tests run against that build.
NET_LIB = os.path.join(ROOT, "paper_2402_01816_b200", "libgns_net.so")


@pytest.mark.skipif(not os.path.exists(NET_LIB), reason="libgns_net.so not built (make net)")
def test_network_merge_build_bitexact():
    e = dict(os.environ, GNS_LIB="libgns_net.so")
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT_DIR", repr(ROOT))], capture_output=True, text=True, env=e, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x", "-m", "gpu",
                        "-k", "f32 or tile_sort_step"], capture_output=True, text=True, env=e, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
