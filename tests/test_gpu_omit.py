"""GPU parity of the Omitsort schedule (NEXT f2, gns_sort_omit; PAPER.md:228
§Full adaptivity): runs carry their location (data / buffer), a pair in
different regions first moves its buffer-resident run to the data region,
non-overlapping pairs are not merged, the others merge into the other region,
a run ending in the buffer is copied back.  The result must be the unique
stable sort, bit-exact against the oracle, whatever mix of omitted, copied and
merged pairs the input produces.
"""
import numpy as np
import pytest

import oracle
import synth
from checks import assert_bitexact

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

T = 4096          # merge tile
T1 = 8192         # tile-sort tile = level-0 run


@pytest.fixture(scope="module")
def gns():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2402_01816_b200 as g
    return g


def to_dev(k, v):
    tk = torch.from_numpy(np.ascontiguousarray(k)).cuda()
    tv = None if v is None else torch.from_numpy(np.ascontiguousarray(v, dtype=np.uint32)).cuda()
    return tk, tv


def omit_sort(gns, k, v, target="AscLeft", use_ws=False):
    tk, tv = to_dev(k, v)
    ws = gns.alloc_workspace(k.size, 1.0, v is not None) if use_ws else None
    if ws is not None:
        ws.fill_(0xFF)                  # stale buffer contents must never leak into the result
    gns.sort_omit_(tk, tv, workspace=ws, target=target)
    torch.cuda.synchronize()
    return tk.cpu().numpy(), (None if tv is None else tv.cpu().numpy())


def run_blocks(n, seed, block, shuffle_frac):
    """Ascending blocks of `block` keys; a fraction of the blocks swapped with
    random partners, so neighbouring runs are sometimes disjoint (omitted),
    sometimes overlapping (merged), and locations diverge between levels."""
    rng = np.random.default_rng(seed)
    k = np.arange(n, dtype=np.float64)
    nb = (n + block - 1) // block
    idx = np.arange(nb)
    m = int(nb * shuffle_frac)
    if m > 1:
        sel = rng.choice(nb, m, replace=False)
        idx[sel] = idx[rng.permutation(sel)]
    parts = [k[i * block:(i + 1) * block] for i in idx]
    return np.concatenate(parts)


SIZES = [1, 2, 33, T1 - 1, T1, T1 + 1, 2 * T1, 2 * T1 + 7, 3 * T1 + 5, 4 * T1 + 1, 7 * T1 - 3, 8 * T1,
         9 * T1 + 100, 100003, (1 << 18) + 3, (1 << 20) + 12345]


@pytest.mark.parametrize("payload", [False, True])
@pytest.mark.parametrize("n", SIZES)
def test_omit_uniform_and_ties(gns, n, payload):
    """Random input: every pair overlaps, locations flip every level (odd and
    even level counts: final copy or not); ties with signed zeros."""
    v = synth.iota_u32(n) if payload else None
    for k in (synth.uniform(n, 31 + n), synth.ties(n, 32 + n, 7) * np.where(np.arange(n) % 5 == 0, -1.0, 1.0)):
        gk, gv = omit_sort(gns, k, v, use_ws=payload)
        ek, ev = oracle.sort(k, v)
        assert_bitexact(gk, ek, gv, ev, what=f"n={n}")


@pytest.mark.parametrize("name", synth.PATTERNS)
@pytest.mark.parametrize("n", [5 * T1 + 123, 40 * T1, (1 << 20) + 3])
def test_omit_paper_patterns(gns, n, name):
    """The paper's eight patterns: presorted ones omit
    whole subtrees, local ones mix omitted and merged pairs."""
    k = synth.pattern(name, n, 700 + n)
    v = synth.iota_u32(n)
    gk, gv = omit_sort(gns, k, v)
    ek, ev = oracle.sort(k, v)
    assert_bitexact(gk, ek, gv, ev, what=f"{name} n={n}")
    gk, _ = omit_sort(gns, k, None)
    assert_bitexact(gk, ek, what=f"{name} n={n} key-only")


@pytest.mark.parametrize("block", [T1 // 2, T1, 3 * T1, 8 * T1 + 5])
@pytest.mark.parametrize("shuffle", [0.0, 0.1, 0.5, 1.0])
@pytest.mark.parametrize("n", [37 * T1 + 11, 64 * T1])
def test_omit_block_mixes(gns, n, block, shuffle):
    """Mixed run locations: blocks of ascending keys, partially shuffled, so
    pairs of every kind (omitted in data, omitted in buffer, copied then
    omitted, copied then merged, merged either way) occur side by side."""
    k = run_blocks(n, 11 + block, block, shuffle)
    v = synth.iota_u32(n)[::-1].copy()
    gk, gv = omit_sort(gns, k, v, use_ws=True)
    ek, ev = oracle.sort(k, v)
    assert_bitexact(gk, ek, gv, ev, what=f"block={block} shuffle={shuffle} n={n}")


@pytest.mark.parametrize("target", ["AscLeft", "AscRight", "DescLeft", "DescRight"])
@pytest.mark.parametrize("n", [3 * T1 + 5, 100003])
def test_omit_targets_with_ties(gns, n, target):
    """The four targets through the Omitsort schedule; runs with
    ties across run boundaries (A's last key == B's first key is an omission
    for the Left targets)."""
    k = np.repeat(np.arange((n + 99) // 100, dtype=np.float64), 100)[:n].copy()
    k[n // 3: n // 3 + T1] = synth.ties(T1, 5, 9)
    v = synth.iota_u32(n)
    gk, gv = omit_sort(gns, k, v, target=target)
    ek, ev = oracle.sort_target(k, v, target)
    assert_bitexact(gk, ek, gv, ev, what=f"{target} n={n}")


@pytest.mark.parametrize("key_type", ["i64", "u64"])
def test_omit_int_keys(gns, key_type):
    """NEXT f3 key types through the Omitsort schedule."""
    n = 20 * T1 + 3
    rng = np.random.default_rng(9)
    if key_type == "i64":
        k = np.sort(rng.integers(-(1 << 62), 1 << 62, n)).astype(np.int64)
        k[5 * T1: 9 * T1] = rng.integers(-(1 << 62), 1 << 62, 4 * T1)
    else:
        k = np.sort(rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2)).astype(np.uint64)
        k[5 * T1: 9 * T1] = rng.integers(0, 1 << 63, 4 * T1, dtype=np.uint64)
    v = synth.iota_u32(n)
    ek, ev = oracle.sort_keys(k, v, key_type, "AscLeft")
    tk, tv = to_dev(k, v)
    gns.sort_omit_(tk, tv)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy(), ek) and np.array_equal(tv.cpu().numpy(), ev), key_type


@pytest.mark.parametrize("sub", ["asc", "desc", "swap1pct", "runs16"])
def test_omit_config4_full_size(gns, sub):
    """BASELINE config 4 (n = 2^24 presorted patterns) through gns_sort_omit,
    with payload = index (stability), vs the oracle."""
    case = synth.config(4, sub)
    v = synth.iota_u32(case.keys.size)
    gk, gv = omit_sort(gns, case.keys, v, use_ws=True)
    ek, ev = oracle.sort(case.keys, v)
    assert_bitexact(gk, ek, gv, ev, what=sub)


def test_omit_uniform_full_size(gns):
    """BASELINE config 2 (2^24 U(0,1), key-only) through gns_sort_omit: 11
    merge levels (odd: the run ends in the buffer and is copied back)."""
    case = synth.config(2)
    gk, _ = omit_sort(gns, case.keys, None, use_ws=True)
    ek, _ = oracle.sort(case.keys, None)
    assert_bitexact(gk, ek, what="cfg2")


def test_omit_errors(gns):
    """Argument errors as gns_sort_keys; the input stays untouched."""
    k = synth.uniform(9 * T1, 1)              # (above the on-chip small sort: a workspace is needed)
    tk, _ = to_dev(k, None)
    with pytest.raises(Exception):
        gns.sort_omit_(tk, None, target="Sideways")
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(RuntimeError):
        gns.sort_omit_(tk, None, workspace=small)
    torch.cuda.synchronize()
    assert np.array_equal(tk.cpu().numpy(), k)


def dir_blocks(n, seed, block, kinds):
    """Blocks of distinct keys, each ascending, strictly descending, or
    descending with one tie ('a', 'd', 't' cycling through `kinds`), in a
    seeded block order: descending runs are kept lazily (Octosort), merged
    with each other when disjoint, reversed when they meet an ascending run
    or overlap."""
    rng = np.random.default_rng(seed)
    base = np.arange(n, dtype=np.float64) * 2.0
    nb = (n + block - 1) // block
    order = rng.permutation(nb) if seed % 2 else np.arange(nb)[::-1]
    parts = []
    for j, b in enumerate(order):
        x = base[b * block:(b + 1) * block].copy()
        kind = kinds[j % len(kinds)]
        if kind != "a":
            x = x[::-1].copy()
        if kind == "t" and x.size > 3:
            x[1] = x[2]
        parts.append(x)
    return np.concatenate(parts)


@pytest.mark.parametrize("kinds", ["d", "dt", "ad", "dda", "t"])
@pytest.mark.parametrize("block", [T1, 2 * T1, 5 * T1 + 3])
@pytest.mark.parametrize("n", [33 * T1 + 17, 64 * T1])
def test_omit_descending_runs(gns, n, block, kinds):
    """Octosort inside the Omitsort schedule: strictly
    reversed tiles stay descending runs, disjoint descending pairs are omitted
    as descending, the rest is reversed (in place or while copied) before
    merging; a descending result is reversed once at the end."""
    k = dir_blocks(n, n + block + len(kinds), block, kinds)
    v = synth.iota_u32(n)
    gk, gv = omit_sort(gns, k, v, use_ws=True)
    ek, ev = oracle.sort(k, v)
    assert_bitexact(gk, ek, gv, ev, what=f"kinds={kinds} block={block} n={n}")
    gk, _ = omit_sort(gns, k, None)
    assert_bitexact(gk, ek, what=f"kinds={kinds} block={block} n={n} key-only")


@pytest.mark.parametrize("target", ["AscLeft", "DescLeft", "AscRight", "DescRight"])
@pytest.mark.parametrize("n", [T1 + 1, 4 * T1, 9 * T1 + 5, (1 << 20) + 3])
def test_omit_strictly_reversed(gns, n, target):
    """A strictly reversed input (for the target's direction): one final
    reversal (or reversed copy); with one tie it must take merges."""
    k = np.arange(n, dtype=np.float64)
    if target in ("AscLeft", "AscRight"):
        k = k[::-1].copy()
    v = synth.iota_u32(n)
    for name in ("strict", "tie"):
        x = k.copy()
        if name == "tie":
            x[n // 2] = x[n // 2 + 1]
        gk, gv = omit_sort(gns, x, v, target=target)
        ek, ev = oracle.sort_target(x, v, target)
        assert_bitexact(gk, ek, gv, ev, what=f"{target} {name} n={n}")


@pytest.mark.slow
@pytest.mark.parametrize("pattern", ["runs", "ties"])
def test_omit_max_size_properties(gns, pattern):
    """GNS_MAX_N-scale Omitsort schedule (32-bit positions in the plan at
    their limit), checked by properties that fix the stable sort uniquely:
    non-decreasing keys, payload a permutation of the original indices, every
    output key bit-identical to the input key its payload names, ties in
    ascending payload order.  Seeded device-side inputs: 64 shuffled
    ascending runs with a descending one (omitted, copied, reversed and
    merged pairs), or heavy ties."""
    n = (1 << 31) - 1
    torch.cuda.empty_cache()                  # (blocks cached by earlier tests count as used)
    free, _ = torch.cuda.mem_get_info()
    need = n * (8 + 4) * 3 + n * 8
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of device memory")
    g = torch.Generator(device="cuda")
    g.manual_seed(n + len(pattern))
    if pattern == "runs":
        base = torch.arange(n, device="cuda", dtype=torch.float64)
        blk = (n + 63) // 64
        perm = torch.randperm(64, device="cuda", generator=g)
        keys = torch.empty_like(base)
        for i in range(64):
            a, b = i * blk, min(n, (i + 1) * blk)
            c = int(perm[i]) * blk
            keys[a:b] = base[c:c + (b - a)] if c + (b - a) <= n else base[n - (b - a):]
        keys[:blk] = keys[:blk].flip(0)                       # one strictly descending run
    else:
        keys = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g).to(torch.float64)
    src = keys.clone()
    vals = torch.arange(n, device="cuda", dtype=torch.int64).to(torch.uint32)
    ws = gns.alloc_workspace(n, 1.0, True)
    gns.sort_omit_(keys, vals, workspace=ws)
    torch.cuda.synchronize()
    del ws
    assert bool((keys[1:] >= keys[:-1]).all())
    idx = vals.to(torch.int64)
    assert bool((src.view(torch.int64)[idx] == keys.view(torch.int64)).all())
    seen = torch.zeros(n, dtype=torch.uint8, device="cuda")
    seen[idx] = 1
    assert int(seen.sum()) == n
    tie = keys[1:] == keys[:-1]
    assert bool((idx[1:][tie] > idx[:-1][tie]).all())
