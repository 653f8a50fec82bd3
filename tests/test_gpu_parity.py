"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
bit-exact on keys and payload (the stable result is unique).

Covers every §8(a) row: the full sort in both buffer modes (a1, a5, a7), the
tile sort (a2), one merge pass incl. its co-rank partition (a3+a4), the
in-place top merge with its hazard protocol (a6), at edge sizes (empty, 1,
tile +-1, several tiles with ragged tails, pass boundaries), all five
BASELINE configs at full size, ties, signed zeros and +-inf.
"""
import numpy as np
import pytest

import oracle
import synth
from checks import assert_bitexact, check_invariants

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gns():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2402_01816_b200 as g
    return g


def to_dev(k, v):
    tk = torch.from_numpy(np.ascontiguousarray(k)).cuda()
    tv = None if v is None else torch.from_numpy(np.ascontiguousarray(v, dtype=np.uint32)).cuda()
    return tk, tv


def gpu_sort(gns, k, v, frac, use_ws=False):
    tk, tv = to_dev(k, v)
    ws = gns.alloc_workspace(k.size, frac, v is not None) if use_ws else None
    gns.sort_(tk, tv, frac, workspace=ws)
    torch.cuda.synchronize()
    return tk.cpu().numpy(), (None if tv is None else tv.cpu().numpy())


def check_against_oracle(gns, k, v, frac, use_ws=False, what=""):
    gk, gv = gpu_sort(gns, k, v, frac, use_ws)
    ek, ev = oracle.sort(k, v)
    assert_bitexact(gk, ek, gv, ev, what=what)


T = 4096          # merge tile; the tile-sort tile (gns_tile_elems) is a multiple of it
T1 = 8192         # tile-sort tile of this build (checked in test_tile_geometry)
EDGE_SIZES = [0, 1, 2, 3, 31, 32, 33, 255, 1000, T - 1, T, T + 1, 2 * T - 1, 2 * T, 2 * T + 1,
              3 * T, 3 * T + 17, 4 * T + 1, 8 * T - 5, 8 * T + 3, 9 * T, 65521, (1 << 16) + 1,
              (1 << 17) - 1, 100003, T1 - 1, T1 + 1, 2 * T1 + 7, 4 * T1 + 1]


def test_tile_geometry(gns):
    assert gns.gns_tile_elems() == T1 and gns.gns_merge_tile_elems() == T


@pytest.mark.parametrize("frac", [1.0, 0.5])
@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("n", EDGE_SIZES)
def test_edge_sizes_ties(gns, n, payload, frac):
    k = synth.ties(n, 77 + n, 7)
    k[::5] *= -1.0                      # -0.0 / +0.0 mix, negative keys
    v = synth.iota_u32(n) if payload else None
    check_against_oracle(gns, k, v, frac, what=f"n={n}")


@pytest.mark.parametrize("frac", [1.0, 0.5])
@pytest.mark.parametrize("n", [T + 1, 5 * T + 77, 1 << 18, (1 << 20) + 12345])
def test_uniform_pairs_ws(gns, n, frac):
    k = synth.uniform(n, 9000 + n)
    v = synth.iota_u32(n)[::-1].copy()   # payload need not be the index
    check_against_oracle(gns, k, v, frac, use_ws=True, what=f"n={n}")


@pytest.mark.parametrize("frac", [0.25, 0.3, 0.125, 1 / 16, 1 / 64])
@pytest.mark.parametrize("n", [T1 + 1, 5 * T1 + 333, 20 * T1 + 7])
def test_limited_buffer_fractions(gns, n, frac):
    """NEXT f1: buffer fraction p < 0.5 (recursive imbalanced split + in-place
    merges); same unique stable result."""
    k = synth.ties(n, 600 + n, 11)
    v = synth.iota_u32(n)
    check_against_oracle(gns, k, v, frac, use_ws=True, what=f"n={n} p={frac}")
    check_against_oracle(gns, synth.uniform(n, 700 + n), None, frac, what=f"n={n} p={frac} key-only")


@pytest.mark.parametrize("target", ["AscRight", "DescLeft", "DescRight"])
@pytest.mark.parametrize("frac", [1.0, 0.5, 0.25])
@pytest.mark.parametrize("n", [1, 1000, T1, 3 * T1 + 5, 100003])
def test_targets(gns, n, frac, target):
    """NEXT f3: the other three API targets, vs the oracle."""
    k = synth.ties(n, 900 + n, 13)
    k[::4] *= -1.0
    k[::11] = np.inf
    k[::13] = -np.inf
    v = synth.iota_u32(n)
    tk, tv = to_dev(k, v)
    gns.sort_(tk, tv, frac, target=target)
    torch.cuda.synchronize()
    ek, ev = oracle.sort_target(k, v, target)
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"{target} n={n} p={frac}")
    tk, _ = to_dev(k, None)
    gns.sort_(tk, None, frac, target=target)
    torch.cuda.synchronize()
    assert_bitexact(tk.cpu().numpy(), ek, what=f"{target} key-only n={n}")


@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [3 * T1, 5 * T1 + 17, 16 * T1, 33 * T1 - 1])
def test_presorted_fast_path(gns, n, target):
    """NEXT f2: already-ordered input takes the omission path (no merge pass
    moves data); one descent anywhere must take the full path.  Covers odd and
    even merge-pass counts (the copy-back case) and ties."""
    desc = target in ("DescLeft", "AscRight")        # AscRight = reverse(DescLeft)
    base = np.sort(synth.ties(n, 55 + n, 1000))       # ordered, with ties
    if desc:
        base = base[::-1].copy()
    v = synth.iota_u32(n)
    cases = {"ordered": base}
    for where in (T1 - 1, T1 + 100, n - 2):          # a descent at a tile boundary / inside / at the end
        k = base.copy()
        k[where], k[where + 1] = k[where + 1], k[where]
        if k[where] != k[where + 1]:
            cases[f"swap@{where}"] = k
    for name, k in cases.items():
        tk, tv = to_dev(k, v)
        gns.sort_(tk, tv, 1.0, target=target)
        torch.cuda.synchronize()
        ek, ev = oracle.sort_target(k, v, target)
        assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"{target} {name} n={n}")


def test_specials_inf_zero(gns):
    n = 3 * T + 5
    rng = np.random.default_rng(5)
    pool = np.array([-np.inf, np.inf, -0.0, 0.0, 1.0, -1.0, 5e-324, -5e-324, np.finfo(np.float64).max])
    k = pool[rng.integers(0, pool.size, n)]
    v = synth.iota_u32(n)
    for frac in (1.0, 0.5):
        check_against_oracle(gns, k, v, frac, what="specials")


def test_exhaustive_tiny(gns):
    import itertools
    for alphabet in ((0.0, 1.0, 2.0), (-0.0, 0.0, 1.0)):
        for n in range(0, 7):
            for seq in itertools.product(alphabet, repeat=n):
                k = np.array(seq, dtype=np.float64)
                v = synth.iota_u32(n)
                check_against_oracle(gns, k, v, 1.0, what=str(seq))


# ------------------------------------------------------------- per-step parity

def test_tile_sort_step(gns):
    T = gns.gns_tile_elems()
    n = 7 * T + 123
    k = synth.ties(n, 4242, 50)
    v = synth.iota_u32(n)
    tk, tv = to_dev(k, v)
    ok, ov = torch.empty_like(tk), torch.empty_like(tv)
    gns.tile_sort(tk, tv, ok, ov)
    torch.cuda.synchronize()
    gk, gv = ok.cpu().numpy(), ov.cpu().numpy()
    for lo in range(0, n, T):
        ek, ev = oracle.sort(k[lo:lo + T], v[lo:lo + T])
        assert_bitexact(gk[lo:lo + T], ek, gv[lo:lo + T], ev, what=f"tile {lo // T}")


@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("L_tiles,n", [(1, 2 * T), (1, 5 * T + 3), (2, 11 * T + 999), (4, 9 * T), (8, 3 * T + 1)])
def test_merge_pass_step(gns, L_tiles, n, payload):
    L = L_tiles * T
    k = synth.ties(n, 31 + n, 9)
    v = synth.iota_u32(n) if payload else None
    # presort runs of L with the oracle, then one merge level on both sides
    k2 = k.copy()
    v2 = None if v is None else v.copy()
    for lo in range(0, n, L):
        sk, sv = oracle.sort(k2[lo:lo + L], None if v2 is None else v2[lo:lo + L])
        k2[lo:lo + L] = sk
        if v2 is not None:
            v2[lo:lo + L] = sv
    ek, ev = oracle.merge_runs(k2, v2, L)
    tk, tv = to_dev(k2, v2)
    ok = torch.empty_like(tk)
    ov = None if tv is None else torch.empty_like(tv)
    ws = torch.empty(gns.gns_merge_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    gns.merge_pass(tk, tv, ok, ov, L, ws)
    torch.cuda.synchronize()
    assert_bitexact(ok.cpu().numpy(), ek, None if ov is None else ov.cpu().numpy(), ev)


def _inplace_case(layout, n, nl, rng):
    nr = n - nl
    if layout == "left_small":          # all left < all right: no cross-tile hazard
        a = np.sort(rng.random(nl)); b = np.sort(rng.random(nr)) + 2.0
    elif layout == "left_big":          # all left > all right: hazard n/(2T) tiles back
        a = np.sort(rng.random(nl)) + 2.0; b = np.sort(rng.random(nr))
    elif layout == "interleave":        # hazard with the previous tile
        a = np.arange(nl, dtype=np.float64) * 2.0; b = np.arange(nr, dtype=np.float64) * 2.0 + 1.0
    elif layout == "ties":
        a = np.sort(rng.integers(0, 3, nl)).astype(np.float64)
        b = np.sort(rng.integers(0, 3, nr)).astype(np.float64)
    else:
        a = np.sort(rng.random(nl)); b = np.sort(rng.random(nr))
    return a, b


@pytest.mark.parametrize("layout", ["left_small", "left_big", "interleave", "ties", "random"])
def test_inplace_top_merge_hazards(gns, layout):
    """Row a6 stress: the dead region of the data array and
    the unused buffer tail are poisoned with NaN, so a read-after-overwrite
    shows up as a wrong output.  Repeated to give races a chance."""
    rng = np.random.default_rng(123)
    # 100 repetitions per layout, the three geometries in turn
    for rep, (n, nl) in enumerate(([(64 * T, 32 * T), (64 * T + 40, 32 * T + 32), (20 * T + 7, 10 * T + 32)] * 34)[:100]):
        a, b = _inplace_case(layout, n, nl, rng)
        va = np.arange(nl, dtype=np.uint32)
        vb = np.arange(nl, n, dtype=np.uint32)
        ek, ev = oracle.merge_runs(np.concatenate([a, b]), np.concatenate([va, vb]), nl)
        data = np.full(n, np.nan)
        data[nl:] = b
        vals = np.full(n, 0xDEADBEEF, dtype=np.uint32)
        vals[nl:] = vb
        tk, tv = to_dev(data, vals)
        lk, lv = to_dev(a, va)
        ws = torch.empty(gns.gns_merge_workspace_bytes(n), dtype=torch.uint8, device="cuda")
        gns.merge_inplace_top(tk, tv, lk, lv, nl, ws)
        torch.cuda.synchronize()
        assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"{layout} rep {rep}")


# ------------------------------------------------------- BASELINE configs, full size

def _config_cases():
    cases = [(1, ""), (2, ""), (3, "")] + [(4, s) for s in synth.CONFIG4_SUBS] + [(5, "")]
    return cases


@pytest.mark.slow
@pytest.mark.parametrize("c,sub", _config_cases())
def test_baseline_configs_full_size(gns, c, sub):
    case = synth.config(c, sub)
    k, v = case.keys, case.vals
    n = k.size
    ek, ev = oracle.sort(k, v)
    if c in (1, 4):
        # also the closed form (permutations of 0..n-1): keys -> i, payload ->
        # inverse permutation -- an expectation independent of the oracle
        ck = np.arange(n, dtype=np.float64)
        assert_bitexact(ek, ck, what=f"{case.name} oracle vs closed form")
        if v is not None:
            cv = np.empty(n, dtype=np.uint32)
            cv[k.astype(np.int64)] = v
            assert np.array_equal(ev, cv), f"{case.name} oracle payload vs closed form"
    for frac in case.fractions + ([0.5] if c in (2, 3) else []):
        gk, gv = gpu_sort(gns, k, v, frac, use_ws=True)
        assert_bitexact(gk, ek, gv, ev, what=f"{case.name} frac={frac}")
        if c == 3:
            check_invariants(k, gk, v, gv, payload_is_index=True)


def test_error_paths_leave_data_untouched(gns):
    n = 16 * 4096 + 5                         # > the on-chip small sort, so a workspace is required
    k = synth.uniform(n, 1)
    tk, _ = to_dev(k, None)
    before = tk.clone()
    assert gns.gns_sort_f64(int(tk.data_ptr()), n, 0.7, 0) == 2
    assert gns.gns_sort_f64(int(tk.data_ptr()) + 4, n - 1, 1.0, 0) == 6      # below natural alignment
    assert gns.gns_sort_f64_ws(int(tk.data_ptr()), n, 1.0, 0, 0, 0) == 5
    assert gns.gns_sort_f64_ws(int(tk.data_ptr()), n, 1.0, 256, 64, 0) == 5
    torch.cuda.synchronize()
    assert torch.equal(before, tk)


def test_nan_memory_safe(gns):
    """NaN is a precondition violation (header: contents unspecified), but the
    call must not fault, must terminate, and the context must stay usable."""
    n = 6 * T + 11
    k = synth.uniform(n, 3)
    k[::7] = np.nan
    v = synth.iota_u32(n)
    for frac in (1.0, 0.5):
        gpu_sort(gns, k, v, frac)
    check_against_oracle(gns, synth.uniform(n, 4), v, 0.5, what="after NaN")


def test_nan_rejected_with_gns_debug(gns, monkeypatch):
    """GNS_DEBUG=1: a NaN key makes every f64 sort return
    GNS_ERR_INVALID_ARGUMENT before anything moves (pre-scan, header R1);
    NaN-free input still sorts bit-exact."""
    monkeypatch.setenv("GNS_DEBUG", "1")
    n = 5 * T + 3
    k = synth.uniform(n, 8)
    k[n // 2] = np.nan
    v = synth.iota_u32(n)
    for frac in (1.0, 0.5):
        tk, tv = to_dev(k, v)
        with pytest.raises(gns.GnsError) as ei:
            gns.sort_(tk, tv, frac)
        assert ei.value.status == 1
        torch.cuda.synchronize()
        assert np.array_equal(tk.cpu().numpy().view(np.uint64), k.view(np.uint64))
        assert np.array_equal(tv.cpu().numpy(), v)
    tk, _ = to_dev(k, None)
    with pytest.raises(gns.GnsError):
        gns.sort_omit_(tk, None)
    check_against_oracle(gns, synth.uniform(n, 9), v, 1.0, what="GNS_DEBUG=1, no NaN")


def _int_keys(key_type, n, seed):
    """Seeded 8-byte integer keys with ties and the type's extreme values."""
    rng = np.random.default_rng(seed)
    if key_type == "i64":
        lo, hi = np.iinfo(np.int64).min, np.iinfo(np.int64).max
        k = rng.integers(lo, hi, n, dtype=np.int64, endpoint=True)
        k[::9] = rng.integers(-20, 20, k[::9].size)          # heavy ties around zero
        ext = np.array([lo, hi, -1, 0, 1], dtype=np.int64)
    else:
        hi = np.iinfo(np.uint64).max
        k = rng.integers(0, hi, n, dtype=np.uint64, endpoint=True)
        k[::9] = rng.integers(0, 40, k[::9].size).astype(np.uint64)
        ext = np.array([0, 1, 1 << 63, (1 << 63) - 1, hi], dtype=np.uint64)
    k[::17] = ext[np.arange(k[::17].size) % ext.size]
    return k


@pytest.mark.parametrize("key_type", ["i64", "u64"])
@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("frac", [1.0, 0.5, 0.25])
@pytest.mark.parametrize("n", [1, 777, T1, 3 * T1 + 5, 100003, (1 << 18) + 3])
def test_int_key_types(gns, n, frac, target, key_type):
    """NEXT f3: int64 / uint64 keys (gns_sort_keys) vs the oracle, bit-exact,
    with payload and key-only, every target and buffer mode."""
    k = _int_keys(key_type, n, 4000 + n)
    v = synth.iota_u32(n)
    ek, ev = oracle.sort_keys(k, v, key_type, target)
    tk, tv = to_dev(k, v)
    gns.sort_(tk, tv, frac, target=target)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy(), ek), f"{key_type} {target} n={n} p={frac} keys"
    assert np.array_equal(tv.cpu().numpy(), ev), f"{key_type} {target} n={n} p={frac} payload"
    tk, _ = to_dev(k, None)
    gns.sort_(tk, None, frac, target=target)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy(), ek), f"{key_type} {target} n={n} p={frac} key-only"


def test_key_type_f64_through_sort_keys(gns):
    """gns_sort_keys with GNS_KEY_F64 is the f64 path (same result as sort_)."""
    n = 3 * T1 + 11
    k = synth.ties(n, 77, 50)
    k[::5] *= -1.0
    v = synth.iota_u32(n)
    tk, tv = to_dev(k, v)
    rc = gns.gns_sort_keys(tk.data_ptr(), 0, tv.data_ptr(), n, 1.0, 0, None, 0, 0)
    assert rc == 0
    torch.cuda.synchronize()
    ek, ev = oracle.sort(k, v)
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev)


@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [T1 + 1, 3 * T1, 5 * T1 + 17, 16 * T1, 33 * T1 - 1, 100003])
def test_reversed_fast_path(gns, n, target):
    """NEXT f2 (Octosort's reversal): a strictly reversed
    input is sorted by one tile-order reversal (odd merge-pass counts) or a
    reversal + copy (even counts); a single tie or a single ordered pair must
    take the full path.  Ragged last tiles included."""
    desc = target in ("DescLeft", "AscRight")
    base = synth.uniform(n, 66 + n)
    base = np.unique(base)                             # distinct keys
    while base.size < n:
        base = np.unique(np.concatenate([base, synth.uniform(n, 67 + base.size)]))
    base = np.sort(base[:n])[::-1].copy()              # strictly descending
    if desc:
        base = base[::-1].copy()                       # strictly ascending = reversed for Desc
    v = synth.iota_u32(n)
    cases = {"reversed": base}
    k = base.copy()
    k[n // 2] = k[n // 2 + 1]                          # one tie
    cases["tie"] = k
    k = base.copy()
    k[T1 - 1], k[T1] = k[T1], k[T1 - 1]                # one ordered pair across a tile boundary
    cases["swap"] = k
    for name, k in cases.items():
        tk, tv = to_dev(k, v)
        gns.sort_(tk, tv, 1.0, target=target)
        torch.cuda.synchronize()
        ek, ev = oracle.sort_target(k, v, target)
        assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"{target} {name} n={n}")
        tk, _ = to_dev(k, None)
        gns.sort_(tk, None, 1.0, target=target)
        torch.cuda.synchronize()
        assert_bitexact(tk.cpu().numpy(), ek, what=f"{target} {name} key-only n={n}")


@pytest.mark.parametrize("frac", [1.0, 0.5])
@pytest.mark.parametrize("name", synth.PATTERNS)
@pytest.mark.parametrize("n", [5 * T1 + 123, 40 * T1])
def test_paper_patterns(gns, n, name, frac):
    """The paper's eight input patterns incl. locally and
    globally presorted / reversed ones, which exercise the per-tile omission
    and reversal (NEXT f2) next to the full path, vs the oracle."""
    k = synth.pattern(name, n, 500 + n)
    v = synth.iota_u32(n)
    tk, tv = to_dev(k, v)
    gns.sort_(tk, tv, frac)
    torch.cuda.synchronize()
    ek, ev = oracle.sort(k, v)
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"{name} n={n} p={frac}")


@pytest.mark.parametrize("target", ["AscLeft", "DescLeft"])
def test_tile_local_order_mix(gns, target):
    """Tiles that are in order, strictly reversed, reversed with a tie, and
    random, side by side (per-tile mode decisions), plus the tile sort step."""
    rng = np.random.default_rng(5)
    parts = []
    for i in range(12):
        t = np.unique(rng.random(T1 + 64))[:T1]
        kind = i % 4
        if kind == 0:
            t = np.sort(t)
        elif kind == 1:
            t = np.sort(t)[::-1].copy()
        elif kind == 2:
            t = np.sort(t)[::-1].copy()
            t[100] = t[101]
        parts.append(t)
    k = np.concatenate(parts + [rng.random(777)])
    v = synth.iota_u32(k.size)
    tk, tv = to_dev(k, v)
    gns.sort_(tk, tv, 1.0, target=target)
    torch.cuda.synchronize()
    ek, ev = oracle.sort_target(k, v, target)
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=target)
    if target == "AscLeft":
        sk_, sv_ = to_dev(k, v)
        dk, dv = torch.empty_like(sk_), torch.empty_like(sv_)
        gns.tile_sort(sk_, sv_, dk, dv)
        torch.cuda.synchronize()
        for t0 in range(0, k.size, T1):
            ek, ev = oracle.sort(k[t0:t0 + T1], v[t0:t0 + T1])
            assert_bitexact(dk.cpu().numpy()[t0:t0 + T1], ek, dv.cpu().numpy()[t0:t0 + T1], ev, what=f"tile {t0}")


# ---------------------------------------------- NEXT f4: distributed sort steps
@pytest.mark.parametrize("key_type", ["f64", "i64", "u64"])
@pytest.mark.parametrize("la,lb", [(1, 1), (0, 5), (7, 0), (4095, 4097), (10000, 333), (333, 10000),
                                   (3 * T1 + 5, 2 * T1 + 11), (1 << 18, (1 << 17) + 3)])
def test_merge_two(gns, la, lb, key_type):
    """gns_merge_two: two sorted runs of any lengths, at unaligned offsets,
    stable (a wins ties) == the oracle's stable sort of a ++ b."""
    rng = np.random.default_rng(la * 7 + lb)
    if key_type == "f64":
        k = rng.integers(-20, 20, la + lb).astype(np.float64)
        k[k == 0] = -0.0
    else:
        k = _int_keys(key_type, la + lb, la + 3 * lb)
        k[::4] = k[1]
    a = oracle.sort_keys(k[:la], None, key_type)[0]
    b = oracle.sort_keys(k[la:], None, key_type)[0]
    cat = np.concatenate([a, b])
    v = synth.iota_u32(la + lb)
    ek, ev = oracle.sort_keys(cat, v, key_type)
    # place a and b at odd element offsets of one buffer (8-byte, not 32-byte aligned)
    pad = np.zeros(3, dtype=cat.dtype)
    vpad = np.zeros(3, dtype=np.uint32)
    buf = torch.from_numpy(np.concatenate([pad[:1], a, pad, b])).cuda()
    vb = torch.from_numpy(np.concatenate([vpad[:1], v[:la], vpad, v[la:]])).cuda()
    ak, av = buf[1:1 + la], vb[1:1 + la]
    bk, bv = buf[4 + la:4 + la + lb], vb[4 + la:4 + la + lb]
    gk, gv = gns.merge_two(ak, av, bk, bv)
    torch.cuda.synchronize()
    assert np.array_equal(gk.cpu().numpy().view(np.uint64), ek.view(np.uint64)), (la, lb, key_type)
    assert np.array_equal(gv.cpu().numpy(), ev), (la, lb, key_type)
    gk, _ = gns.merge_two(ak, None, bk, None)
    torch.cuda.synchronize()
    assert np.array_equal(gk.cpu().numpy().view(np.uint64), ek.view(np.uint64)), (la, lb, key_type, "key-only")


@pytest.mark.parametrize("key_type", ["f64", "i64", "u64"])
def test_split_cuts(gns, key_type):
    """gns_split_cuts == the definition via numpy.searchsorted (upper bound for
    lower ranks, lower bound for higher ranks, the position for the owner)."""
    n = 50000
    if key_type == "f64":
        k = np.sort(np.random.default_rng(1).integers(-100, 100, n).astype(np.float64))
        spl = np.array([-100.0, -3.0, 0.0, 7.5, 99.0, 1000.0])
    else:
        k = oracle.sort_keys(_int_keys(key_type, n, 2), None, key_type)[0]
        spl = k[[0, 10, 20000, 20001, n - 1]]
    for me in (0, 2, 4):
        ranks = np.array([1, 2, 3, 2, 5, 0][:spl.size], dtype=np.int32)
        pos = np.array([5, 17, 0, n, 123, 9][:spl.size], dtype=np.int64)
        got = gns.split_cuts(torch.from_numpy(k).cuda(), torch.from_numpy(spl).cuda(), torch.from_numpy(ranks).cuda(),
                             torch.from_numpy(pos).cuda(), me)
        torch.cuda.synchronize()
        want = [int(p) if r == me else int(np.searchsorted(k, x, side="right" if me < r else "left"))
                for x, r, p in zip(spl, ranks, pos)]
        assert got.cpu().tolist() == want, (key_type, me)


@pytest.mark.parametrize("balanced", [True, False])
@pytest.mark.parametrize("k", [2, 3, 4, 8])
@pytest.mark.parametrize("pattern", ["uniform", "ties", "skewed"])
def test_distributed_sort_simulated(gns, k, pattern, balanced):
    """The f4 path's kernels end to end on one GPU: dist.simulate runs the k
    ranks' steps in one process (exchange = slices, no collectives), vs the
    oracle's stable sort of the rank-major concatenation; with exact co-ranks
    (balanced) every piece has exactly its share of the N keys."""
    from paper_2402_01816_b200 import dist as gdist
    rng = np.random.default_rng(k * 100 + len(pattern))
    shards = []
    for r in range(k):
        n = int(rng.integers(0, 3 * T1)) if pattern == "skewed" else 2 * T1 + 37 * r
        if pattern == "ties":
            s = rng.integers(0, 5, n).astype(np.float64)
        elif pattern == "skewed":
            s = rng.random(n) + r          # rank r holds [r, r+1): no interleaving
        else:
            s = synth.uniform(n, 70 + r)
        shards.append(s)
    base = np.cumsum([0] + [s.size for s in shards])
    ins = [(torch.from_numpy(s).cuda(), torch.from_numpy((np.arange(s.size) + base[r]).astype(np.uint32)).cuda())
           for r, s in enumerate(shards)]
    outs = gdist.simulate(ins, samples=32, balanced=balanced)
    torch.cuda.synchronize()
    allk = np.concatenate(shards)
    ek, ev = oracle.sort(allk, np.arange(allk.size, dtype=np.uint32))
    gk = np.concatenate([o[0].cpu().numpy() for o in outs])
    gv = np.concatenate([o[1].cpu().numpy() for o in outs])
    assert_bitexact(gk, ek, gv, ev, what=f"k={k} {pattern}")
    if balanced:
        N = allk.size
        assert [o[0].numel() for o in outs] == [((g + 1) * N) // k - (g * N) // k for g in range(k)]


def test_distributed_sort_single_rank_nccl(gns):
    """sort_distributed through a real NCCL process group (world size 1 on
    this one-GPU box): the collective path's set-up and the local sort."""
    import torch.distributed as dist
    from paper_2402_01816_b200 import dist as gdist
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        k = synth.ties(3 * T1 + 5, 8, 30)
        v = synth.iota_u32(k.size)
        gk, gv = gdist.sort_distributed(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        torch.cuda.synchronize()
        ek, ev = oracle.sort(k, v)
        assert_bitexact(gk.cpu().numpy(), ek, gv.cpu().numpy(), ev)
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
@pytest.mark.parametrize("n,frac", [((1 << 31) - 1, 1.0), ((1 << 30) + 12345, 0.5)])
def test_max_size_properties(gns, n, frac):
    """GNS_MAX_N-scale sorts (int32 tile/row/co-rank arithmetic at its limit),
    checked by properties that together fix the stable sort uniquely
    (SURVEY.md §8(c) I1-I3 plus the payload gather): output non-decreasing,
    payload a permutation of 0..n-1 (the original indices), every output key
    bit-identical to the input key its payload names, and equal keys in
    ascending payload order.  Seeded device-side inputs with ties."""
    torch.cuda.empty_cache()                  # (blocks cached by earlier tests count as used)
    free, _ = torch.cuda.mem_get_info()
    need = n * (8 + 4) * 3 + n * 8
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of device memory")
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    keys = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g).to(torch.float64)   # heavy ties
    keys[::3] = torch.rand(keys[::3].shape, device="cuda", generator=g, dtype=torch.float64)
    src = keys.clone()
    vals = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32)
    ws = gns.alloc_workspace(n, frac, True)
    gns.sort_(keys, vals, frac, workspace=ws)
    torch.cuda.synchronize()
    del ws
    assert bool((keys[1:] >= keys[:-1]).all())
    idx = vals.to(torch.int64)
    assert bool((src.view(torch.int64)[idx] == keys.view(torch.int64)).all())      # gather: bit-exact keys
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    seen[idx] = 1
    assert int(seen.sum()) == n                                                       # a permutation
    tie = keys[1:] == keys[:-1]
    assert bool((idx[1:][tie] > idx[:-1][tie]).all())                                 # stable ties


@pytest.mark.slow
@pytest.mark.parametrize("pattern", ["uniform", "ties", "ascending", "reversed", "runs"])
def test_ticket_merge_passes_large_pairs(gns, pattern):
    """Passes of >= 8192 tiles with payload run as partition + ticket-scheduled
    merge (gns.cu ticket_pass): 2^25 + ragged pairs, several patterns
    (including the f2 ordered / reversed fast paths through that kernel), both
    buffer modes and a descending target, vs the oracle."""
    n = (1 << 25) + 777
    if pattern == "uniform":
        k = synth.uniform(n, 31)
    elif pattern == "ties":
        k = synth.ties(n, 32, 24)
    elif pattern == "ascending":
        k = np.arange(n, dtype=np.float64)
    elif pattern == "reversed":
        k = np.arange(n, 0, -1, dtype=np.float64)
    else:
        k = synth.runs(n, 33)
    v = synth.iota_u32(n)
    ek, ev = oracle.sort(k, v)
    for frac in (1.0, 0.5):
        gk, gv = gpu_sort(gns, k, v, frac, use_ws=True)
        assert_bitexact(gk, ek, gv, ev, what=f"{pattern} frac={frac}")
    if pattern in ("uniform", "ties"):
        tk, tv = to_dev(k, v)
        gns.sort_(tk, tv, 1.0, target="DescLeft")
        torch.cuda.synchronize()
        dk, dv = oracle.sort_target(k, v, "DescLeft")
        assert_bitexact(tk.cpu().numpy(), dk, tv.cpu().numpy(), dv, what=f"{pattern} DescLeft")


@pytest.mark.slow
@pytest.mark.parametrize("key_type,target", [("u64", "AscLeft"), ("i64", "DescRight")])
def test_ticket_merge_passes_int_keys(gns, key_type, target):
    """The partition + ticket-merge passes (>= 8192 tiles with payload) with
    64-bit integer keys and a Right target, vs the oracle."""
    n = (1 << 25) + 33
    k = _int_keys(key_type, n, 77)
    v = synth.iota_u32(n)
    ek, ev = oracle.sort_keys(k, v, key_type, target)
    tk, tv = to_dev(k, v)
    gns.sort_(tk, tv, 1.0, target=target)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy(), ek) and np.array_equal(tv.cpu().numpy(), ev)


@pytest.mark.slow
def test_ticket_merge_passes_large_keys(gns):
    """Key-only passes of >= 32768 tiles (2^27 + ragged keys) also run as
    partition + ticket-scheduled merge; vs the oracle, both buffer modes."""
    n = (1 << 27) + 5
    k = synth.ties(n, 41, 1 << 20)
    k[::5] = synth.uniform(k[::5].size, 42)
    ek, _ = oracle.sort(k, None)
    for frac in (1.0, 0.5):
        gk, _ = gpu_sort(gns, k, None, frac, use_ws=True)
        assert_bitexact(gk, ek, what=f"frac={frac}")


def test_concurrent_streams_and_threads(gns):
    """Reentrancy (header): sorts enqueued on different streams from two host
    threads at once, each with its own workspace (and one stream-ordered
    allocation), all bit-exact."""
    import threading
    cases = []
    for i, (n, frac, hv) in enumerate([(5 * T1 + 17, 1.0, True), (7 * T1 + 3, 0.5, False),
                                       (3 * T1 + 1, 0.25, True), (9 * T1, 1.0, False)]):
        k = synth.ties(n, 300 + i, 50) if i % 2 else synth.uniform(n, 300 + i)
        v = synth.iota_u32(n) if hv else None
        cases.append((k, v, frac))
    results = [None] * len(cases)
    errors = []

    def run(idx):
        try:
            k, v, frac = cases[idx]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                tk, tv = to_dev(k, v)
                ws = gns.alloc_workspace(k.size, frac, v is not None) if idx % 2 == 0 else None
                for _ in range(3):                     # re-sorting sorted data is a no-op, result unchanged
                    gns.sort_(tk, tv, frac, workspace=ws, stream=s)
            s.synchronize()
            results[idx] = (tk.cpu().numpy(), None if tv is None else tv.cpu().numpy())
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (k, v, frac), (gk, gv) in zip(cases, results):
        ek, ev = oracle.sort(k, v)
        assert_bitexact(gk, ek, gv, ev, what=f"n={k.size} frac={frac}")


@pytest.mark.parametrize("key_type", ["f64", "i64", "u64"])
@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [0, 1, 2, 777, T1, T1 + 1, 3 * T1 + 5, 100003, (1 << 20) + 3])
def test_u64_payload(gns, n, target, key_type):
    """NEXT f3: 64-bit payloads (gns_sort_keys_u64) vs the oracle: keys
    bit-exact, payload[i] = the input payload of the key's stable position
    (the oracle's index permutation), every target and key type; with and
    without a caller workspace."""
    rng = np.random.default_rng(n + len(target) + len(key_type))
    if key_type == "f64":
        k = synth.ties(n, 600 + n, 40)
        k[::5] *= -1.0
    else:
        k = _int_keys(key_type, n, 600 + n)
    pay = rng.integers(0, 1 << 64, n, dtype=np.uint64, endpoint=False)
    ek, ev = oracle.sort_keys(k, synth.iota_u32(n), key_type, target)
    for use_ws in (False, True):
        tk = torch.from_numpy(k.copy()).cuda()
        tp = torch.from_numpy(pay.copy()).cuda()
        ws = (torch.empty(max(1, gns.workspace_bytes_u64(n)), dtype=torch.uint8, device="cuda") if use_ws else None)
        gns.sort_u64_(tk, tp, workspace=ws, target=target)
        torch.cuda.synchronize()
        assert np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64)), f"keys n={n} {target}"
        assert np.array_equal(tp.cpu().numpy(), pay[ev.astype(np.int64)]), f"payload n={n} {target} ws={use_ws}"


def test_u64_payload_full_size_and_errors(gns):
    """BASELINE config 2 keys with a 64-bit payload at full size; argument
    errors leave the data untouched."""
    k = synth.config(2).keys
    n = k.size
    pay = np.arange(n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    ek, ev = oracle.sort(k, synth.iota_u32(n))
    tk, tp = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(pay).cuda()
    gns.sort_u64_(tk, tp)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64))
    assert np.array_equal(tp.cpu().numpy(), pay[ev.astype(np.int64)])
    small = torch.empty(64, dtype=torch.uint8, device="cuda")
    tk2, tp2 = torch.from_numpy(k[:3 * T1].copy()).cuda(), torch.from_numpy(pay[:3 * T1].copy()).cuda()
    with pytest.raises(gns.GnsError) as ei:
        gns.sort_u64_(tk2, tp2, workspace=small)
    assert ei.value.status == 5
    torch.cuda.synchronize()
    assert np.array_equal(tk2.cpu().numpy(), k[:3 * T1]) and np.array_equal(tp2.cpu().numpy(), pay[:3 * T1])


def _f32_keys(n, seed):
    """Seeded binary32 keys with ties, signed zeros, infinities, subnormals."""
    rng = np.random.default_rng(seed)
    k = (rng.standard_normal(n) * 1e3).astype(np.float32)
    k[::7] = rng.integers(-20, 20, k[::7].size).astype(np.float32)          # ties
    ext = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 3.4e38, -3.4e38], dtype=np.float32)
    k[::13] = ext[np.arange(k[::13].size) % ext.size]
    return k


@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [0, 1, 2, 777, T1, T1 + 1, 3 * T1 + 5, 100003, (1 << 20) + 3])
def test_f32_keys(gns, n, target, payload):
    """NEXT f3: binary32 keys (gns_sort_f32) vs the oracle: the oracle sorts
    the exactly widened keys (same IEEE order, -0.0 == +0.0) with the index as
    payload; the expected output is the input permuted by that stable order,
    bit-exact (signed zeros keep their bits)."""
    k = _f32_keys(n, 900 + n + len(target))
    v = synth.iota_u32(n)[::-1].copy() if payload else None
    _, ev = oracle.sort_target(k.astype(np.float64), synth.iota_u32(n), target)
    perm = ev.astype(np.int64)
    for use_ws in (False, True):
        tk = torch.from_numpy(k.copy()).cuda()
        tv = None if v is None else torch.from_numpy(v.copy()).cuda()
        ws = (torch.empty(max(1, gns.workspace_bytes_f32(n, v is not None)), dtype=torch.uint8, device="cuda") if use_ws else None)
        gns.sort_f32_(tk, tv, workspace=ws, target=target)
        torch.cuda.synchronize()
        assert np.array_equal(tk.cpu().numpy().view(np.uint32), k[perm].view(np.uint32)), f"keys n={n} {target}"
        if v is not None:
            assert np.array_equal(tv.cpu().numpy(), v[perm]), f"vals n={n} {target}"


def _f32_keys_shape(n, seed, shape):
    """binary32 keys without zeros (uniform / heavy ties) or with a few zeros
    of both signs: the key-only merge pass merges a thread's outputs by a
    register network unless its warp holds a zero (csrc/gns_f32.cuh)."""
    rng = np.random.default_rng(seed)
    if shape == "uniform":
        k = (rng.random(n, dtype=np.float32) + np.float32(0.5)) * np.where(rng.random(n) < 0.5, -1, 1).astype(np.float32)
    elif shape == "ties":
        k = rng.integers(1, 24, n).astype(np.float32) * np.where(rng.random(n) < 0.3, -1, 1).astype(np.float32)
    elif shape == "sparse_zeros":
        k = (rng.standard_normal(n) * 4).astype(np.float32)
        k[k == 0] = 1.0
        z = rng.integers(0, max(n, 1), max(1, n // 3000))
        k[z] = np.where(rng.random(z.size) < 0.5, np.float32(-0.0), np.float32(0.0))
    elif shape == "runs":
        k = np.sort((rng.random(n, dtype=np.float32) + np.float32(1.0)))      # presorted halves interleaving by blocks
        h = n // 2
        k = np.concatenate([k[h:], k[:h]])
    else:
        raise ValueError(shape)
    return k


@pytest.mark.parametrize("shape", ["uniform", "ties", "sparse_zeros", "runs"])
@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [4096, T1 + 1, 2 * T1, 3 * T1 + 5, 100003, (1 << 20) + 3, (1 << 22) + 4099])
def test_f32_keys_network_merge(gns, n, target, shape):
    """NEXT f3: binary32 key-only merge passes on inputs whose warps hold no
    zero (the register bitonic merge of a thread's 16 outputs) and on inputs
    with a few signed zeros (warps falling back to the serial stable merge),
    vs the oracle's stable order of the exactly widened keys, bit-exact."""
    k = _f32_keys_shape(n, 77 + n + len(target), shape)
    _, ev = oracle.sort_target(k.astype(np.float64), synth.iota_u32(n), target)
    perm = ev.astype(np.int64)
    tk = torch.from_numpy(k.copy()).cuda()
    gns.sort_f32_(tk, None, target=target)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy().view(np.uint32), k[perm].view(np.uint32)), f"keys n={n} {target} {shape}"


def test_f32_keys_full_size(gns):
    """2^24 binary32 keys with payload at full size, vs the oracle."""
    n = 1 << 24
    k = _f32_keys(n, 4242)
    v = synth.iota_u32(n)
    _, ev = oracle.sort(k.astype(np.float64), v)
    tk, tv = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(v.copy()).cuda()
    gns.sort_f32_(tk, tv)
    torch.cuda.synchronize()
    perm = ev.astype(np.int64)
    assert np.array_equal(tk.cpu().numpy().view(np.uint32), k[perm].view(np.uint32))
    assert np.array_equal(tv.cpu().numpy(), v[perm])


@pytest.mark.slow
def test_f32_max_size_properties(gns):
    """binary32 keys at GNS_MAX_N with payload = index (int32 offsets of the
    4-byte kernels at their limit), by the properties that fix the stable
    sort: non-decreasing, payload a permutation, every key bit-identical to
    the input key its payload names, ties in ascending payload order."""
    n = (1 << 31) - 1
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    need = n * (4 + 4) * 3 + n * 8
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of device memory")
    g = torch.Generator(device="cuda")
    g.manual_seed(31)
    keys = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g).to(torch.float32)   # heavy ties
    keys[::3] = torch.rand(keys[::3].shape, device="cuda", generator=g, dtype=torch.float32)
    src = keys.clone()
    vals = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32)
    gns.sort_f32_(keys, vals)
    torch.cuda.synchronize()
    assert bool((keys[1:] >= keys[:-1]).all())
    idx = vals.to(torch.int64)
    assert bool((src.view(torch.int32)[idx] == keys.view(torch.int32)).all())
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    seen[idx] = 1
    assert int(seen.sum()) == n
    tie = keys[1:] == keys[:-1]
    assert bool((idx[1:][tie] > idx[:-1][tie]).all())


@pytest.mark.slow
def test_u64_payload_max_size_properties(gns):
    """64-bit payloads at GNS_MAX_N: keys non-decreasing, each payload (the
    input index as uint64) names the input key its key equals bit-exactly,
    ties in ascending payload order."""
    n = (1 << 31) - 1
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    need = n * (8 + 8) * 3 + n * 8
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of device memory")
    g = torch.Generator(device="cuda")
    g.manual_seed(64)
    keys = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g).to(torch.float64)
    src = keys.clone()
    vals = torch.arange(n, device="cuda", dtype=torch.int64)
    gns.sort_u64_(keys, vals)
    torch.cuda.synchronize()
    assert bool((keys[1:] >= keys[:-1]).all())
    assert bool((src.view(torch.int64)[vals] == keys.view(torch.int64)).all())
    tie = keys[1:] == keys[:-1]
    assert bool((vals[1:][tie] > vals[:-1][tie]).all())
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    seen[vals] = 1
    assert int(seen.sum()) == n


@pytest.mark.parametrize("payload", [False, True])
def test_f32_nan_memory_safe(gns, payload):
    """binary32 keys with NaN (a precondition violation, R1): the
    merge pass must clamp non-monotone split points so its bulk
    copies stay inside their shared slots.  Crafted inputs: a tile of zeros
    with NaNs (at every position a search can probe, and sparse), followed by
    a tile of -1.0; plus random NaNs over several passes.  The call must
    terminate without a fault and the context must still sort correctly."""
    t = T1
    cases = []
    a = np.zeros(2 * t, np.float32)
    a[:t:7] = np.nan
    a[t:] = -1.0
    cases.append(a)
    b = np.zeros(2 * t, np.float32)
    b[:t][np.arange(0, t, 1)[::2]] = np.nan
    b[t:] = -1.0
    cases.append(b)
    c = np.zeros(4 * t + 5, np.float32)
    c[::3] = np.nan
    c[2 * t:] = -2.0
    cases.append(c)
    r = synth.uniform(9 * t + 3, 77).astype(np.float32)
    r[::5] = np.nan
    cases.append(r)
    for k in cases:
        n = k.size
        tk = torch.from_numpy(k.copy()).cuda()
        tv = torch.from_numpy(synth.iota_u32(n)).cuda() if payload else None
        gns.sort_f32_(tk, tv)
        torch.cuda.synchronize()
    n = 3 * t + 11
    k = _f32_keys(n, 31337)
    v = synth.iota_u32(n)
    _, ev = oracle.sort(k.astype(np.float64), v)
    tk, tv = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(v.copy()).cuda()
    gns.sort_f32_(tk, tv)
    torch.cuda.synchronize()
    perm = ev.astype(np.int64)
    assert np.array_equal(tk.cpu().numpy().view(np.uint32), k[perm].view(np.uint32)), "after NaN"


# ---------------------------------------------------------------- row b: natural alignment
# keys need only 8-byte, vals 4-byte alignment; the sort of a
# sliced view (not 32-byte aligned) takes the peel path (gns_peel.cuh) and is
# bit-exact like any other (sorting applies to any contiguous
# sequence).
VIEW_SIZES = [1, 2, 5, 7, 9, 100, T1 - 3, T1 + 9, 3 * T1 + 77, 2 * 4096 * 3 + 5, (1 << 20) + 13]


@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("frac", [1.0, 0.5, 0.25])
@pytest.mark.parametrize("view", [(1, 0), (3, 0), (5, 7), (2, 1), (7, 0)])
@pytest.mark.parametrize("n", VIEW_SIZES)
def test_sliced_views(gns, n, view, frac, payload):
    lo, hi = view
    full = n + lo + hi
    k = synth.ties(full, 4100 + n + lo, 50)
    k[::11] *= -1.0
    v = synth.iota_u32(full)[::-1].copy() if payload else None
    ek, ev = oracle.sort(k[lo:full - hi], None if v is None else v[lo:full - hi])
    for use_ws in (False, True):
        tk, tv = to_dev(k, v)
        sk = tk[lo:full - hi]
        sv = None if tv is None else tv[lo:full - hi]
        ws = gns.alloc_workspace(n, frac, payload) if use_ws else None
        gns.sort_(sk, sv, frac, workspace=ws)
        torch.cuda.synchronize()
        gk = tk.cpu().numpy()
        assert_bitexact(gk[lo:full - hi], ek, None if tv is None else tv.cpu().numpy()[lo:full - hi], ev,
                        what=f"view {view} n={n} frac={frac}")
        # nothing outside the view moved
        assert np.array_equal(gk[:lo].view(np.uint64), k[:lo].view(np.uint64))
        assert np.array_equal(gk[full - hi:].view(np.uint64), k[full - hi:].view(np.uint64))


@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("key_type", ["f64", "i64", "u64"])
@pytest.mark.parametrize("frac", [1.0, 0.5])
def test_sliced_views_targets_key_types(gns, target, key_type, frac):
    """Views of every key type and target (the peel merge runs in the
    target's direction; Right targets reverse the whole view at the end)."""
    n = 5 * T1 + 3
    if key_type == "f64":
        k = synth.ties(n + 3, 4200, 30)
        k[::7] *= -1.0
    else:
        k = _int_keys(key_type, n + 3, 4201)
    v = synth.iota_u32(n + 3)
    kk, vv = k[3:], v[3:]
    if key_type == "f64":
        ek, ev = oracle.sort_target(kk, vv, target)
    else:
        ek, ev = oracle.sort_keys(kk, vv, key_type, target)
    tk, tv = to_dev(k, v)
    gns.sort_(tk[3:], tv[3:], frac, target=target)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy()[3:].view(np.uint64), ek.view(np.uint64)), f"{key_type} {target}"
    assert np.array_equal(tv.cpu().numpy()[3:], ev), f"{key_type} {target}"


def test_sliced_view_ticket_passes(gns):
    """A view at a size whose merge passes use the ticket-scheduled kernel
    (>= 2^25 pairs), both buffer modes."""
    n = (1 << 25) + 3
    k = synth.uniform(n + 1, 4300)
    v = synth.iota_u32(n + 1)
    ek, ev = oracle.sort(k[1:], v[1:])
    for frac in (1.0, 0.5):
        tk, tv = to_dev(k, v)
        gns.sort_(tk[1:], tv[1:], frac)
        torch.cuda.synchronize()
        assert_bitexact(tk.cpu().numpy()[1:], ek, tv.cpu().numpy()[1:], ev, what=f"frac={frac}")


def test_sliced_views_incompatible_offsets(gns):
    """keys and vals with no common 32-byte boundary (keys[1:] with vals[2:]):
    vals go through an aligned temporary; still bit-exact."""
    n = 3 * T1 + 5
    k = synth.ties(n + 2, 4400, 20)
    v = synth.iota_u32(n + 2)
    ek, ev = oracle.sort(k[1:n + 1], v[2:n + 2])
    tk, tv = to_dev(k, v)
    gns.sort_(tk[1:n + 1], tv[2:n + 2], 1.0)
    torch.cuda.synchronize()
    assert_bitexact(tk.cpu().numpy()[1:n + 1], ek, tv.cpu().numpy()[2:n + 2], ev, what="incompatible")


# ------------------------------------------------- all-equal keys through the merges
@pytest.mark.parametrize("frac", [1.0, 0.5, 0.125])
@pytest.mark.parametrize("n", [3 * T1 + 5, 20 * T1 + 1, (1 << 20) + 7])
@pytest.mark.parametrize("sched", ["default", "omit"])
def test_all_equal_keys_defeat_shortcut(gns, n, frac, sched):
    """All keys equal except a smaller LAST key: the whole-input "in order"
    shortcut does not fire (one descent), so every tie goes through the tile
    sort, every merge pass and (limited buffer) the in-place top merge; the
    payload (= index) must come out as n-1 followed by 0..n-2 (stability).
    Same with the Omitsort schedule (full buffer)."""
    if sched == "omit" and frac != 1.0:
        pytest.skip("the Omitsort schedule runs with the full buffer")
    k = np.full(n, 7.0)
    k[-1] = 3.0
    v = synth.iota_u32(n)
    ek, ev = oracle.sort(k, v)
    assert ev[0] == n - 1 and np.array_equal(ev[1:], np.arange(n - 1, dtype=np.uint32))
    tk, tv = to_dev(k, v)
    if sched == "omit":
        gns.sort_omit_(tk, tv)
    else:
        gns.sort_(tk, tv, frac)
    torch.cuda.synchronize()
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"all-equal n={n} frac={frac} {sched}")
    # signed zeros: all +-0.0 (equal under IEEE <) but one -1.0 at the end:
    # the zeros' bit patterns must keep their input order
    z = np.where(np.arange(n) % 3 == 0, -0.0, 0.0)
    z[-1] = -1.0
    ek, ev = oracle.sort(z, v)
    tk, tv = to_dev(z, v)
    if sched == "omit":
        gns.sort_omit_(tk, tv)
    else:
        gns.sort_(tk, tv, frac)
    torch.cuda.synchronize()
    assert_bitexact(tk.cpu().numpy(), ek, tv.cpu().numpy(), ev, what=f"zeros n={n} frac={frac} {sched}")
    # key-only (the 64-key network path with its zero-sign fix-up)
    tk, _ = to_dev(z, None)
    if sched == "omit":
        gns.sort_omit_(tk, None)
    else:
        gns.sort_(tk, None, frac)
    torch.cuda.synchronize()
    assert_bitexact(tk.cpu().numpy(), ek, what=f"zeros key-only n={n} frac={frac} {sched}")


@pytest.mark.parametrize("off", [1, 2, 3, 5, 7])
@pytest.mark.parametrize("la,lb", [(1, 1), (3, 9), (T + 5, 2 * T + 1), (5 * T1 + 3, 17)])
def test_merge_two_into_unaligned_views(gns, la, lb, off):
    """gns_merge_two writing into a view at any element offset (natural
    alignment; the first outputs by the head kernel), keys and vals."""
    a = np.sort(synth.ties(la, 31 + la, 20), kind="stable")
    b = np.sort(synth.ties(lb, 32 + lb, 20), kind="stable")
    va = np.arange(la, dtype=np.uint32)
    vb = np.arange(la, la + lb, dtype=np.uint32)
    # the stable merge of two sorted runs = the stable sort of their concatenation
    ek, ev = oracle.sort(np.concatenate([a, b]), np.concatenate([va, vb]))
    dk = torch.full((la + lb + 16,), np.nan, dtype=torch.float64, device="cuda")
    dv = torch.full((la + lb + 16,), 7, dtype=torch.int64, device="cuda").to(torch.uint32)
    ta, tva = to_dev(a, va)
    tb, tvb = to_dev(b, vb)
    gns.merge_two(ta, tva, tb, tvb, out=(dk[off:off + la + lb], dv[off:off + la + lb]))
    torch.cuda.synchronize()
    assert_bitexact(dk.cpu().numpy()[off:off + la + lb], ek, dv.cpu().numpy()[off:off + la + lb], ev,
                    what=f"off={off} la={la} lb={lb}")
    assert np.isnan(dk.cpu().numpy()[:off]).all() and np.isnan(dk.cpu().numpy()[off + la + lb:]).all()
