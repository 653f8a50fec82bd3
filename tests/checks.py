"""Output checkers shared by the tests (no sort arithmetic of the method).

Invariants from BASELINE.json north_star / SURVEY.md §8(c):
  I1 output keys non-decreasing under IEEE `<`
  I2 multiset of (key bits, val) pairs equals the input's
  I3 among equal keys, the payload (original index) strictly ascends
"""
import numpy as np


def key_bits(k):
    return np.ascontiguousarray(k, dtype=np.float64).view(np.uint64)


def assert_bitexact(got_k, exp_k, got_v=None, exp_v=None, what=""):
    gk, ek = key_bits(got_k), key_bits(exp_k)
    if gk.shape != ek.shape:
        raise AssertionError(f"{what}: length {gk.shape} != {ek.shape}")
    bad = np.flatnonzero(gk != ek)
    if bad.size:
        i = bad[0]
        raise AssertionError(f"{what}: {bad.size} key mismatches, first at {i}: "
                             f"got {got_k[i]!r} want {exp_k[i]!r}")
    if exp_v is not None:
        bad = np.flatnonzero(np.asarray(got_v) != np.asarray(exp_v))
        if bad.size:
            i = bad[0]
            raise AssertionError(f"{what}: {bad.size} payload mismatches, first at {i}: "
                                 f"got {got_v[i]} want {exp_v[i]}")


def check_invariants(in_k, out_k, in_v=None, out_v=None, payload_is_index=False):
    in_k = np.asarray(in_k, dtype=np.float64)
    out_k = np.asarray(out_k, dtype=np.float64)
    assert in_k.shape == out_k.shape
    if out_k.size > 1:
        # I1: not (out[i+1] < out[i])
        assert not np.any(out_k[1:] < out_k[:-1]), "I1 violated: output not non-decreasing"
    # I2: multiset of (bits, val) equal
    ib, ob = key_bits(in_k), key_bits(out_k)
    if in_v is None:
        assert np.array_equal(np.sort(ib), np.sort(ob)), "I2 violated (keys)"
    else:
        ia = np.lexsort((np.asarray(in_v), ib))
        oa = np.lexsort((np.asarray(out_v), ob))
        assert np.array_equal(ib[ia], ob[oa]) and np.array_equal(np.asarray(in_v)[ia], np.asarray(out_v)[oa]), \
            "I2 violated (pairs)"
        if payload_is_index and out_k.size > 1:
            eq = out_k[1:] == out_k[:-1]
            ov = np.asarray(out_v).astype(np.int64)
            assert np.all(ov[1:][eq] > ov[:-1][eq]), "I3 violated: ties not in input order"
