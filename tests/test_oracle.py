"""Pins for the CPU oracle (oracle/), none of which re-types its formula.

Each pin is chosen so a plausible oracle mistake fails it:
  * brute force (stable insertion sort written here, exhaustive tiny inputs)
    catches a wrong tie rule (taking B on `<=`), an off-by-one split, a lost
    payload;
  * the closed form for permutations catches a transposed key/payload move;
  * the textbook stable counting sort catches instability under heavy ties;
  * numpy.argsort(kind="stable") (a library routine) catches anything at scale;
  * the SPEC.md worked examples (tests/golden/spec_examples.json, cited).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth
from checks import assert_bitexact, check_invariants, key_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def insertion_sort_stable(keys, tags):
    """Brute force: shift while the previous key is strictly greater."""
    a = list(zip(keys, tags))
    for i in range(1, len(a)):
        x = a[i]
        j = i
        while j > 0 and a[j - 1][0] > x[0]:
            a[j] = a[j - 1]
            j -= 1
        a[j] = x
    return [k for k, _ in a], [t for _, t in a]


@pytest.mark.parametrize("alphabet", [(0.0, 1.0, 2.0), (-0.0, 0.0, 1.0)])
def test_exhaustive_tiny_vs_insertion_sort(alphabet):
    count = 0
    for n in range(0, 8):
        for seq in itertools.product(alphabet, repeat=n):
            keys = np.array(seq, dtype=np.float64)
            tags = np.arange(n, dtype=np.uint32)
            ek, et = insertion_sort_stable(list(keys), list(tags))
            gk, gt = oracle.sort(keys, tags)
            assert_bitexact(gk, np.array(ek, dtype=np.float64), gt, np.array(et, dtype=np.uint32),
                            what=f"seq={seq}")
            count += 1
    assert count == sum(3 ** n for n in range(8))


def test_signed_zero_keeps_bits_and_order():
    keys = np.array([0.0, -0.0, 0.0, -0.0, -1.0], dtype=np.float64)
    gk, gv = oracle.sort(keys, np.arange(5, dtype=np.uint32))
    assert list(gv) == [4, 0, 1, 2, 3]
    assert list(np.signbit(gk)) == [True, False, True, False, True]


def test_random_small_vs_numpy_stable():
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(0, 2000))
        d = int(rng.integers(1, 5))
        keys = rng.integers(0, d, n).astype(np.float64)
        keys[rng.random(n) < 0.1] *= -1.0   # mixes -0.0 into the zeros
        tags = np.arange(n, dtype=np.uint32)
        order = np.argsort(keys, kind="stable")
        gk, gt = oracle.sort(keys, tags)
        assert_bitexact(gk, keys[order], gt, tags[order], what=f"trial {trial}")


def test_uniform_vs_numpy_stable_and_invariants():
    n = 1 << 16
    keys = synth.uniform(n, 2000)
    keys[::97] = keys[5]      # force duplicates
    tags = np.arange(n, dtype=np.uint32)
    gk, gt = oracle.sort(keys, tags)
    order = np.argsort(keys, kind="stable")
    assert_bitexact(gk, keys[order], gt, tags[order])
    check_invariants(keys, gk, tags, gt, payload_is_index=True)


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 4097, 1 << 16])
def test_permutation_closed_form(n):
    """keys = a permutation of 0..n-1 (config 1 shape): sorted keys are i and
    the payload is the inverse permutation.  No sort needed to state it."""
    keys = synth.permutation(n, 1000 + n)
    tags = np.arange(n, dtype=np.uint32)
    gk, gt = oracle.sort(keys, tags)
    assert np.array_equal(gk, np.arange(n, dtype=np.float64))
    inv = np.empty(n, dtype=np.uint32)
    inv[keys.astype(np.int64)] = np.arange(n, dtype=np.uint32)
    assert np.array_equal(gt, inv)


def counting_sort_stable(keys_int, m):
    """Textbook stable counting sort (histogram, exclusive prefix sum,
    scatter in index order)."""
    n = len(keys_int)
    count = np.bincount(keys_int, minlength=m)
    start = np.concatenate([[0], np.cumsum(count)[:-1]])
    out_tag = np.empty(n, dtype=np.uint32)
    out_key = np.empty(n, dtype=np.int64)
    pos = start.copy()
    for i in range(n):             # index order = stability
        k = keys_int[i]
        out_tag[pos[k]] = i
        out_key[pos[k]] = k
        pos[k] += 1
    return out_key, out_tag


def test_heavy_ties_vs_counting_sort():
    n = 50000
    keys = synth.ties(n, 3000, 24)
    ek, et = counting_sort_stable(keys.astype(np.int64), 24)
    gk, gt = oracle.sort(keys, np.arange(n, dtype=np.uint32))
    assert np.array_equal(gk, ek.astype(np.float64))
    assert np.array_equal(gt, et)


def test_presorted_patterns_closed_form():
    n = 10007
    for k in (synth.ascending(n), synth.descending(n), synth.swapped(n, 4003), synth.runs(n, 4004)):
        gk, gt = oracle.sort(k, np.arange(n, dtype=np.uint32))
        assert np.array_equal(gk, np.arange(n, dtype=np.float64))
        inv = np.empty(n, dtype=np.uint32)
        inv[k.astype(np.int64)] = np.arange(n, dtype=np.uint32)
        assert np.array_equal(gt, inv)


def test_nan_rejected_and_input_untouched():
    keys = np.array([1.0, np.nan, 0.0])
    with pytest.raises(oracle.OracleNaNError):
        oracle.sort(keys)


def test_golden_spec_examples():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        g = json.load(f)
    for ex in g["stable_sort"]:
        gk, gt = oracle.sort(np.array(ex["keys"], dtype=np.float64), np.array(ex["tags"], dtype=np.uint32))
        assert list(gk) == ex["out_keys"], ex["cite"]
        assert list(gt) == ex["out_tags"], ex["cite"]
    for ex in g["merge"]:
        k = np.array(ex["left"] + ex["right"], dtype=np.float64)
        t = np.array(ex.get("left_tags", list(range(len(ex["left"])))) +
                     ex.get("right_tags", list(range(len(ex["left"]), len(k)))), dtype=np.uint32)
        mk, mt = oracle.merge_runs(k, t, len(ex["left"]))
        assert list(mk) == ex["out"], ex["cite"]
        if "out_tags" in ex:
            assert list(mt) == ex["out_tags"], ex["cite"]


def test_merge_runs_vs_brute_force():
    rng = np.random.default_rng(11)
    for trial in range(100):
        L = int(rng.integers(1, 40))
        n = int(rng.integers(0, 6 * L))
        keys = rng.integers(0, 4, n).astype(np.float64)
        tags = np.arange(n, dtype=np.uint32)
        # presort each run with the brute-force insertion sort
        for lo in range(0, n, L):
            sk, st = insertion_sort_stable(list(keys[lo:lo + L]), list(tags[lo:lo + L]))
            keys[lo:lo + L] = sk
            tags[lo:lo + L] = st
        mk, mt = oracle.merge_runs(keys, tags, L)
        for lo in range(0, n, 2 * L):
            ek, et = insertion_sort_stable(list(keys[lo:lo + 2 * L]), list(tags[lo:lo + 2 * L]))
            assert list(mk[lo:lo + 2 * L]) == ek
            assert list(mt[lo:lo + 2 * L]) == et


def test_oracle_sort_equals_repeated_merge_levels():
    """sort == tile-sort then log2 merge levels (the GPU path's structure),
    both taken from the oracle — a consistency pin of merge_runs vs sort."""
    n = 5000
    keys = synth.ties(n, 77, 5)
    tags = np.arange(n, dtype=np.uint32)
    T = 64
    k, t = keys.copy(), tags.copy()
    for lo in range(0, n, T):
        k[lo:lo + T], t[lo:lo + T] = oracle.sort(k[lo:lo + T], t[lo:lo + T])
    L = T
    while L < n:
        k, t = oracle.merge_runs(k, t, L)
        L *= 2
    ek, et = oracle.sort(keys, tags)
    assert_bitexact(k, ek, t, et)


# ------------------------------------------------------------ NEXT f3: targets

def brute_target(keys, tags, target):
    """Insertion sort on the composite order the target defines:
    AscLeft (k, i), AscRight (k, -i), DescLeft (-k, i), DescRight (-k, -i);
    IEEE comparisons on k (so -0.0 == +0.0)."""
    desc = target.startswith("Desc")
    right = target.endswith("Right")

    def before(a, b):     # a = (k, i) strictly precedes b
        ka, ia = a
        kb, ib = b
        if (kb < ka) if desc else (ka < kb):
            return True
        if ka == kb:
            return ia > ib if right else ia < ib
        return False
    a = list(zip(keys, tags))
    for i in range(1, len(a)):
        x = a[i]
        j = i
        while j > 0 and before(x, a[j - 1]):
            a[j] = a[j - 1]
            j -= 1
        a[j] = x
    return [k for k, _ in a], [t for _, t in a]


@pytest.mark.parametrize("target", ["AscLeft", "AscRight", "DescLeft", "DescRight"])
def test_targets_exhaustive_vs_brute_force(target):
    for alphabet in ((0.0, 1.0, 2.0), (-0.0, 0.0, 1.0)):
        for n in range(0, 7):
            for seq in itertools.product(alphabet, repeat=n):
                keys = np.array(seq, dtype=np.float64)
                tags = np.arange(n, dtype=np.uint32)
                ek, et = brute_target(list(keys), list(tags), target)
                gk, gt = oracle.sort_target(keys, tags, target)
                assert_bitexact(gk, np.array(ek, dtype=np.float64), gt, np.array(et, dtype=np.uint32),
                                what=f"{target} {seq}")


def test_targets_relations_and_golden():
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 5, 3000).astype(np.float64)
    tags = np.arange(3000, dtype=np.uint32)
    al = oracle.sort_target(keys, tags, "AscLeft")
    assert_bitexact(al[0], oracle.sort(keys, tags)[0], al[1], oracle.sort(keys, tags)[1])
    for a, b in (("AscRight", "DescLeft"), ("DescRight", "AscLeft")):
        ka, ta = oracle.sort_target(keys, tags, a)
        kb, tb = oracle.sort_target(keys, tags, b)
        assert_bitexact(ka, kb[::-1].copy(), ta, tb[::-1].copy(), what=f"{a} == reverse({b})")
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        g = json.load(f)
    for ex in g["targets"]:
        gk, gt = oracle.sort_target(np.array(ex["keys"], dtype=np.float64),
                                    np.array(ex["tags"], dtype=np.uint32), ex["target"])
        assert list(gk) == ex["out_keys"] and list(gt) == ex["out_tags"], ex["cite"]


# ------------------------------------------------- NEXT f3: 8-byte key types
I64_EXTREMES = (np.iinfo(np.int64).min, -1, 0, 1, np.iinfo(np.int64).max)
U64_EXTREMES = (0, 1, 1 << 63, (1 << 64) - 1)


@pytest.mark.parametrize("key_type,alphabet", [("i64", I64_EXTREMES[:3] + I64_EXTREMES[4:]),
                                               ("u64", U64_EXTREMES)])
@pytest.mark.parametrize("target", ["AscLeft", "DescRight"])
def test_int_keys_exhaustive_vs_brute_force(key_type, alphabet, target):
    """Brute force over every sequence of length <= 5 drawn from values at the
    ends of the type's range: treating u64 as i64 (or either as f64) puts
    2^63 / 2^64-1 / INT64_MIN in the wrong place and fails here."""
    dt = np.int64 if key_type == "i64" else np.uint64
    for n in range(0, 6):
        for seq in itertools.product(alphabet, repeat=n):
            keys = np.array([int(x) for x in seq], dtype=dt)
            tags = np.arange(n, dtype=np.uint32)
            ek, et = brute_target([int(x) for x in keys], list(tags), target)   # Python ints: exact order
            gk, gt = oracle.sort_keys(keys, tags, key_type, target)
            assert [int(x) for x in gk] == ek and list(gt) == et, (key_type, target, seq)


@pytest.mark.parametrize("key_type", ["f64", "i64", "u64"])
def test_key_types_vs_numpy_stable(key_type):
    rng = np.random.default_rng(11)
    n = 20000
    if key_type == "f64":
        keys = rng.integers(-50, 50, n).astype(np.float64)
    elif key_type == "i64":
        keys = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, n, dtype=np.int64, endpoint=True)
        keys[::7] = keys[3]                                     # ties
    else:
        keys = rng.integers(0, np.iinfo(np.uint64).max, n, dtype=np.uint64, endpoint=True)
        keys[::5] = keys[2]
    vals = np.arange(n, dtype=np.uint32)
    order = np.argsort(keys, kind="stable")
    gk, gv = oracle.sort_keys(keys, vals, key_type)
    assert np.array_equal(gk, keys[order]) and np.array_equal(gv, vals[order])
    # descending-left: stable sort by the reversed order, ties in input order
    rk, rv = oracle.sort_keys(keys, vals, key_type, "DescLeft")
    if key_type == "f64":
        order_d = np.argsort(-keys, kind="stable")
    else:
        order_d = np.lexsort((np.arange(n), [-int(x) for x in keys])) if key_type == "u64" else \
            np.argsort(-keys.astype(object), kind="stable")
    assert [int(x) for x in rk] == [int(x) for x in keys[order_d]] and np.array_equal(rv, vals[order_d])
