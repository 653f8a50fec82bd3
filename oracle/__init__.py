"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2402_01816_b200``) never imports it and shares no code
with it.

Functions and the passages they follow:

* :func:`sort` — stable ascending sort of f64 keys (+ optional u32 payload),
  plain top-down mergesort with Knuth's merge, left run wins ties
  (§Definition of sorting; §Forgotten art).
  C implementation in ``oracle/oracle.c``.  Pinned (tests/test_oracle.py) by
  brute-force stable insertion sort (exhaustive tiny inputs), closed forms
  (permutations -> identity keys + inverse permutation), a textbook stable
  counting sort (heavy ties), ``numpy.argsort(kind="stable")`` and the SPEC.md
  worked examples in ``tests/golden/``.
* :func:`sort_target` — the four API targets AscLeft/AscRight/DescLeft/
  DescRight (NEXT f3): the same mergesort, merge rule per
  target.  Pinned by brute force on (key, +-index) orders, the SPEC.md:72
  DescLeft example, and AscLeft == :func:`sort`.
* :func:`sort_keys` — the same mergesort over 8-byte keys of type f64, i64
  or u64 (NEXT f3, key types), any target.  Pinned by brute force over tiny
  inputs with extreme values (INT64_MIN/MAX, 2^63, 2^64-1: sorting u64 as
  i64 or f64 fails the pin) and ``numpy.argsort(kind="stable")``.
* :func:`merge_runs` — one merge level over runs of length L.
  Pinned by the SPEC.md ``mergeKnuth`` examples and by brute force.
* :mod:`oracle.footprint` — %RAM and tFootprint.  Pinned by the
  paper's own Squidtab identity and SPEC.md examples.

Every function is pinned; nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleNaNError(ValueError):
    """Raised for NaN keys (reading R1)."""


def build() -> None:
    # -O2: the oracle is plain C, not tuned; optimisation flags do not change
    # its arithmetic (it has none besides comparisons and copies).
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        up = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_sort_f64_u32.argtypes = [dp, up, ctypes.c_size_t]
        L.oracle_sort_f64_u32.restype = ctypes.c_int
        L.oracle_sort_target.argtypes = [dp, up, ctypes.c_size_t, ctypes.c_int]
        L.oracle_sort_target.restype = ctypes.c_int
        L.oracle_sort_keys.argtypes = [ctypes.POINTER(ctypes.c_uint64), up, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_int]
        L.oracle_sort_keys.restype = ctypes.c_int
        L.oracle_merge_runs.argtypes = [dp, up, ctypes.c_size_t, ctypes.c_size_t, dp, up]
        L.oracle_merge_runs.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptrs(k: np.ndarray, v: Optional[np.ndarray]):
    dp = k.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    up = v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if v is not None else None
    return dp, up


def sort(keys: np.ndarray, vals: Optional[np.ndarray] = None
         ) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """Returns stably sorted copies of (keys, vals)."""
    k = np.array(keys, dtype=np.float64, copy=True, order="C")
    v = None if vals is None else np.array(vals, dtype=np.uint32, copy=True, order="C")
    if v is not None and v.shape != k.shape:
        raise ValueError("keys and vals differ in length")
    dp, up = _ptrs(k, v)
    rc = lib().oracle_sort_f64_u32(dp, up, k.size)
    if rc == 1:
        raise OracleNaNError("NaN key")
    if rc != 0:
        raise MemoryError("oracle")
    return k, v


TARGETS = {"AscLeft": 0, "AscRight": 1, "DescLeft": 2, "DescRight": 3}


def sort_target(keys: np.ndarray, vals: Optional[np.ndarray], target: str
                ) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """The four stable API targets, NEXT f3."""
    k = np.array(keys, dtype=np.float64, copy=True, order="C")
    v = None if vals is None else np.array(vals, dtype=np.uint32, copy=True, order="C")
    dp, up = _ptrs(k, v)
    rc = lib().oracle_sort_target(dp, up, k.size, TARGETS[target])
    if rc == 1:
        raise OracleNaNError("NaN key")
    if rc != 0:
        raise ValueError("oracle_sort_target failed")
    return k, v


KEY_TYPES = {"f64": 0, "i64": 1, "u64": 2}
_KEY_DTYPES = {"f64": np.float64, "i64": np.int64, "u64": np.uint64}


def sort_keys(keys: np.ndarray, vals: Optional[np.ndarray], key_type: str, target: str = "AscLeft"
              ) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """Stable sort of 8-byte keys of ``key_type`` (f64 / i64 / u64) for one of
    the four targets; returns sorted copies (keys in their own dtype)."""
    k = np.array(keys, dtype=_KEY_DTYPES[key_type], copy=True, order="C")
    v = None if vals is None else np.array(vals, dtype=np.uint32, copy=True, order="C")
    kp = k.view(np.uint64).ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    up = v.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if v is not None else None
    rc = lib().oracle_sort_keys(kp, up, k.size, KEY_TYPES[key_type], TARGETS[target])
    if rc == 1:
        raise OracleNaNError("NaN key")
    if rc != 0:
        raise ValueError("oracle_sort_keys failed")
    return k, v


def merge_runs(keys: np.ndarray, vals: Optional[np.ndarray], run_len: int
               ) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """One merge level: merges consecutive pairs of sorted runs of length
    ``run_len`` (left run wins ties)."""
    k = np.ascontiguousarray(keys, dtype=np.float64)
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32)
    ok = np.empty_like(k)
    ov = None if v is None else np.empty_like(v)
    dp, up = _ptrs(k, v)
    odp, oup = _ptrs(ok, ov)
    rc = lib().oracle_merge_runs(dp, up, k.size, run_len, odp, oup)
    if rc != 0:
        raise OracleNaNError("NaN key or run_len == 0")
    return ok, ov
