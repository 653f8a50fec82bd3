"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/gns.h declares, plans passes/bytes correctly, and rejects bad
arguments before touching CUDA."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gns.h")


@pytest.fixture(scope="session")
def gns():
    lib = os.path.join(ROOT, "paper_2402_01816_b200", "libgns.so")
    srcs = [os.path.join(ROOT, "paper_2402_01816_b200", "csrc", f) for f in ("gns.cu", "gns_kernels.cuh")] + [HEADER]
    if not os.path.exists(lib) or any(os.path.getmtime(s) > os.path.getmtime(lib) for s in srcs):
        subprocess.check_call(["make", "-C", ROOT, "paper_2402_01816_b200/libgns.so"])
    import paper_2402_01816_b200 as g
    return g


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gns_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(gns):
    names = declared_functions()
    assert len(names) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only", gns.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (gns_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(gns.EXPORTED)


def test_sm100a_only(gns):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gns.LIB_PATH]).decode()
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_geometry_and_plan(gns):
    T = gns.gns_tile_elems()
    M = gns.gns_merge_tile_elems()
    assert M == 4096 and T % M == 0 and T >= M

    def passes(n):
        runs = -(-n // T)
        return 0 if n <= T else (runs - 1).bit_length()

    p = gns.plan(1 << 24, 1.0, False)
    assert p["merge_passes"] == passes(1 << 24) and p["hbm_passes"] == 1 + passes(1 << 24)
    assert p["bytes_lower_bound"] == p["hbm_passes"] * 2 * (1 << 24) * 8
    assert p["buffer_elems"] == 1 << 24
    p = gns.plan(1 << 27, 0.5, True)
    assert p["hbm_passes"] == 1 + passes(1 << 27) and p["left_len"] == 1 << 26 and p["buffer_elems"] == 1 << 26
    assert p["bytes_lower_bound"] == p["hbm_passes"] * 2 * (1 << 27) * 12
    p = gns.plan(T, 0.5, True)
    assert p["workspace_bytes"] == 0 and p["hbm_passes"] == 1
    # up to 16 x 4096 keys: one thread-block cluster sorts on chip (no buffer,
    # one read + one write, no merge pass)
    small = 16 * 4096
    for n in (T + 1, small):
        p = gns.plan(n, 1.0, True)
        assert p["merge_passes"] == 0 and p["hbm_passes"] == 1 and p["workspace_bytes"] == 0
    p = gns.plan(small + 1, 1.0, False)
    assert p["merge_passes"] == passes(small + 1) and p["workspace_bytes"] > 0
    assert gns.plan(0, 1.0, False)["hbm_passes"] == 0


def test_workspace_ram_pct(gns):
    from oracle import footprint
    n = 1 << 27
    for frac, want in ((1.0, 2.0), (0.5, 1.5)):
        ws = gns.workspace_bytes(n, frac, True)
        r = footprint.ram_pct(n * 12, ws)
        assert want <= r < want + 5e-3, (frac, r)   # + index arrays and split-search samples (DESIGN R7)
    assert gns.workspace_bytes(n, 0.7, True) == 0


def test_limited_buffer_fractions(gns):
    """NEXT f1: buffer fractions p in [1/64, 0.5]: %RAM ~ 1 + p, more passes
    as p shrinks (the Frogsort2 trade-off)."""
    from oracle import footprint
    n = 1 << 27
    prev = None
    for p in (0.5, 0.25, 0.125, 1 / 16, 1 / 64):
        info = gns.plan(n, p, True)
        r = footprint.ram_pct(n * 12, info["workspace_bytes"])
        assert 1 + p <= r < 1 + p + 5e-3, (p, r)
        if prev is not None:
            assert info["element_passes"] >= prev
        prev = info["element_passes"]
        assert info["bytes_lower_bound"] == round(info["element_passes"] * n) * 2 * 12
    assert gns.plan(n, 0.5, True)["element_passes"] == gns.plan(n, 1.0, True)["element_passes"]
    for bad in (0.0, 0.75, 1 / 128, 1.5, -1.0):
        assert gns.workspace_bytes(n, bad, True) == 0
        assert gns.gns_sort_f64(256, 10000, bad, None) == 2


def test_argument_errors_before_any_cuda_call(gns):
    # all of these must return before touching CUDA (there is no GPU here)
    assert gns.gns_sort_f64(None, 10, 1.0, None) == 1
    assert gns.gns_sort_f64(256, 10, 0.75, None) == 2
    assert gns.gns_sort_f64(260, 10, 1.0, None) == 6            # below natural (8-byte) alignment
    assert gns.gns_sort_pairs_f64_u32(256, 258, 10, 1.0, None) == 6   # vals below 4-byte alignment
    assert gns.gns_tile_sort(264, None, 512, None, 10, None) == 6     # per-step entry points: 32-byte
    assert gns.gns_sort_pairs_f64_u32(256, None, 10, 1.0, None) == 1
    assert gns.gns_sort_f64(256, (1 << 31), 1.0, None) == 1
    assert gns.gns_sort_f64_ws(256, 1 << 20, 1.0, None, 0, None) == 5
    assert gns.gns_sort_f64_ws(256, 1 << 20, 1.0, 256, 10, None) == 5
    assert gns.gns_merge_pass(256, None, 512, None, 1000, 100, 256, 1 << 20, None) == 1   # run_len % 2048
    assert gns.gns_merge_inplace_top(256, None, 512, None, 10, 100, 256, 1 << 20, None) == 1
    # n in {0, 1}: OK, no launch
    assert gns.gns_sort_f64(None, 0, 1.0, None) == 0
    assert gns.gns_sort_f64(256, 1, 0.5, None) == 0
    assert gns.gns_status_string(6) == "GNS_ERR_MISALIGNED"
    assert gns.gns_sort_f64(260, 10, 1.0, None) == 6
    assert "aligned" in gns.gns_last_error_string()


def test_sort_keys_argument_errors(gns):
    """gns_sort_keys (NEXT f3 key types): unknown key type / target rejected
    before any CUDA call; the f64/i64/u64 paths share the alignment rules."""
    assert gns.gns_sort_keys(256, 3, None, 10, 1.0, 0, None, 0, None) == 1
    assert gns.gns_sort_keys(256, -1, None, 10, 1.0, 0, None, 0, None) == 1
    assert gns.gns_sort_keys(256, 1, None, 10, 1.0, 4, None, 0, None) == 1
    assert gns.gns_sort_keys(260, 2, None, 10, 1.0, 0, None, 0, None) == 6
    assert gns.gns_sort_keys(256, 1, None, 10, 0.75, 0, None, 0, None) == 2
    assert gns.gns_sort_keys(None, 2, None, 0, 1.0, 0, None, 0, None) == 0
