"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.

This module holds none of the method's arithmetic (no compare, merge or sort);
it draws inputs only.  The generators are C (``synth/gen.c``) so that the
2^27-element config is produced in about a second; this wrapper compiles the
shared object with gcc on first use if it is missing or stale.

Configs follow BASELINE.json ``configs`` (index 1..5 as in SURVEY.md §8(d));
seeds are ``1000 * config + sub``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def _build() -> None:
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            _build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        sz, u64 = ctypes.c_size_t, ctypes.c_uint64
        L.gen_u64.argtypes = [ctypes.POINTER(ctypes.c_uint64), sz, u64]
        L.gen_uniform.argtypes = [dp, sz, u64]
        L.gen_permutation.argtypes = [dp, sz, u64]
        L.gen_ties.argtypes = [dp, sz, u64, u64]
        L.gen_ascending.argtypes = [dp, sz]
        L.gen_descending.argtypes = [dp, sz]
        L.gen_swapped.argtypes = [dp, sz, u64, ctypes.c_uint]
        L.gen_swapped.restype = ctypes.c_int
        L.gen_runs.argtypes = [dp, sz, u64, ctypes.c_uint]
        L.gen_runs.restype = ctypes.c_int
        L.gen_pattern_local.argtypes = [dp, sz, u64, ctypes.c_int]
        L.gen_pattern_local.restype = ctypes.c_int
        L.gen_pattern_global.argtypes = [dp, sz, u64, ctypes.c_int]
        L.gen_pattern_global.restype = ctypes.c_int
        L.gen_iota_u32.argtypes = [ctypes.POINTER(ctypes.c_uint32), sz]
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def u64_stream(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().gen_u64(out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n, seed)
    return out


def uniform(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().gen_uniform(_dptr(out), n, seed)
    return out


def permutation(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().gen_permutation(_dptr(out), n, seed)
    return out


def ties(n: int, seed: int, m: int = 24) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().gen_ties(_dptr(out), n, seed, m)
    return out


def ascending(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().gen_ascending(_dptr(out), n)
    return out


def descending(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().gen_descending(_dptr(out), n)
    return out


def swapped(n: int, seed: int, permille: int = 10) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    if lib().gen_swapped(_dptr(out), n, seed, permille) != 0:
        raise MemoryError("gen_swapped")
    return out


def runs(n: int, seed: int, nruns: int = 16) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    if lib().gen_runs(_dptr(out), n, seed, nruns) != 0:
        raise MemoryError("gen_runs")
    return out


def pattern(name: str, n: int, seed: int) -> np.ndarray:
    """The paper's eight patterns on values 0..n-1."""
    out = np.empty(n, dtype=np.float64)
    L = lib()
    if name == "permut":
        L.gen_permutation(_dptr(out), n, seed)
    elif name == "tielog2":
        L.gen_ties(_dptr(out), n, seed, max(1, int(np.ceil(np.log2(max(n, 2))))))
    elif name == "ascall":
        L.gen_ascending(_dptr(out), n)
    elif name == "descall":
        L.gen_descending(_dptr(out), n)
    elif name in ("asclocal", "desclocal"):
        if L.gen_pattern_local(_dptr(out), n, seed, int(name == "desclocal")) != 0:
            raise MemoryError(name)
    elif name in ("ascglobal", "descglobal"):
        if L.gen_pattern_global(_dptr(out), n, seed, int(name == "descglobal")) != 0:
            raise MemoryError(name)
    else:
        raise ValueError(f"unknown pattern {name!r}")
    return out


PATTERNS = ("permut", "tielog2", "ascall", "asclocal", "ascglobal",
            "descall", "desclocal", "descglobal")


def iota_u32(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    lib().gen_iota_u32(out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), n)
    return out


@dataclass
class Case:
    """One concrete sort input: keys, optional u32 payload, buffer fractions."""
    name: str
    keys: np.ndarray
    vals: Optional[np.ndarray]
    fractions: List[float]
    shape: str          # which paper pattern it stands in for


def config(c: int, sub: str = "", n: Optional[int] = None) -> Case:
    """BASELINE.json configs[c-1] at its full size (or at ``n`` if given,
    same recipe).  Config 4 takes ``sub`` in {asc, desc, swap1pct, runs16}."""
    if c == 1:
        n = n or (1 << 16)
        return Case("cfg1_permut_2^%d" % n.bit_length(), permutation(n, 1000), iota_u32(n), [1.0],
                    "permut (PAPER.md:372)")
    if c == 2:
        n = n or (1 << 24)
        return Case("cfg2_uniform", uniform(n, 2000), None, [1.0], "random doubles (PAPER.md:313, 338)")
    if c == 3:
        n = n or (1 << 24)
        return Case("cfg3_ties24", ties(n, 3000, 24), iota_u32(n), [1.0], "tielog2 (PAPER.md:374)")
    if c == 4:
        n = n or (1 << 24)
        if sub == "asc":
            k = ascending(n)
        elif sub == "desc":
            k = descending(n)
        elif sub == "swap1pct":
            k = swapped(n, 4003, 10)
        elif sub == "runs16":
            k = runs(n, 4004, 16)
        else:
            raise ValueError("config 4 sub must be asc|desc|swap1pct|runs16")
        return Case("cfg4_" + sub, k, None, [1.0], "ascall/descall/near-sorted (PAPER.md:376, 388)")
    if c == 5:
        n = n or (1 << 27)
        return Case("cfg5_uniform_pairs", uniform(n, 5000), iota_u32(n), [1.0, 0.5],
                    "random doubles with payload")
    raise ValueError("config must be 1..5")


CONFIG4_SUBS = ("asc", "desc", "swap1pct", "runs16")
