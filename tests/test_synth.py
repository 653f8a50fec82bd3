"""The shared input generators: PRNG pinned to published SplitMix64 outputs,
recipes checked against the readings in DESIGN.md §3."""
import json
import os

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vector():
    with open(os.path.join(GOLDEN, "splitmix64.json")) as f:
        g = json.load(f)
    got = synth.u64_stream(len(g["first"]), g["seed"])
    assert [int(x) for x in got] == [int(x) for x in g["first"]]


def test_determinism_and_ranges():
    a = synth.uniform(1000, 5)
    assert np.array_equal(a, synth.uniform(1000, 5))
    assert not np.array_equal(a, synth.uniform(1000, 6))
    assert a.min() >= 0.0 and a.max() < 1.0 and not np.isnan(a).any()
    t = synth.ties(100000, 3000, 24)
    assert set(np.unique(t)) == set(float(i) for i in range(24))


def test_permutation_is_permutation():
    p = synth.permutation(4096, 1000)
    assert np.array_equal(np.sort(p), np.arange(4096.0))
    assert not np.array_equal(p, np.arange(4096.0))


def test_swapped_exactly_one_percent():
    n = 4096
    k = synth.swapped(n, 4003, 10)
    assert int(np.sum(k != np.arange(n))) == 2 * (n // 200)
    assert np.array_equal(np.sort(k), np.arange(float(n)))


def test_runs16():
    n = 1 << 16
    k = synth.runs(n, 4004, 16)
    assert np.array_equal(np.sort(k), np.arange(float(n)))
    # 16 runs of consecutive integers -> at most 15 breaks in "k[i+1] == k[i] + 1"
    breaks = int(np.sum(np.diff(k) != 1))
    assert 1 <= breaks <= 15   # adjacent runs may happen to continue each other (A11)


def test_paper_patterns():
    n = 1000
    b = 32  # ceil(sqrt(1000))
    for name in synth.PATTERNS:
        k = synth.pattern(name, n, 9)
        if name == "tielog2":
            assert len(np.unique(k)) <= 10
            continue
        assert np.array_equal(np.sort(k), np.arange(float(n))), name
    al = synth.pattern("asclocal", n, 9)
    for s in range(0, n, b):
        assert np.all(np.diff(al[s:s + b]) > 0)
    dl = synth.pattern("desclocal", n, 9)
    for s in range(0, n, b):
        assert np.all(np.diff(dl[s:s + b]) < 0)
    ag = synth.pattern("ascglobal", n, 9)
    for s in range(0, n, b):
        assert sorted(ag[s:s + b]) == list(np.arange(s, min(n, s + b), dtype=float))
    assert list(synth.pattern("ascall", 5, 1)) == [0, 1, 2, 3, 4]
    assert list(synth.pattern("descall", 4, 1)) == [3, 2, 1, 0]
