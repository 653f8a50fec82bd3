"""Randomised parity fuzzing of every sort entry point against the oracle
(run under gpurun).  Each case draws: size (log-uniform, ragged), input shape
(uniform, heavy ties, presorted / reversed runs, blocks, specials), key type,
target, payload, buffer fraction, entry point (sort_, sort_omit_,
sort_u64_, sort_f32_) and, for sort_ / sort_omit_, a view offset (0..7 head
and tail elements: the natural-alignment path), then compares bit-exactly.
usage: python tools/fuzz.py [--seconds 600] [--max-log2 22] [--seed 1]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2402_01816_b200 as gns  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=600)
ap.add_argument("--max-log2", type=int, default=22)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
TARGETS = ["AscLeft", "AscRight", "DescLeft", "DescRight"]


def keys_f64(n):
    kind = rng.integers(0, 7)
    if kind == 0:
        k = rng.random(n)
    elif kind == 1:
        k = rng.integers(0, int(rng.integers(1, 50)), n).astype(np.float64)
    elif kind == 2:
        k = np.sort(rng.random(n))
        if rng.random() < 0.5:
            k = k[::-1].copy()
    elif kind == 3:                                   # shuffled ascending / descending blocks
        b = int(rng.integers(1, max(2, n // 3) + 1))
        parts = [np.sort(rng.random(min(b, n - i))) for i in range(0, n, b)]
        parts = [p[::-1].copy() if rng.random() < 0.3 else p for p in parts]
        rng.shuffle(parts)
        k = np.concatenate(parts) if parts else np.zeros(0)
    elif kind == 4:                                   # specials
        ext = np.array([0.0, -0.0, np.inf, -np.inf, 5e-324, -5e-324, 1.0, -1.0])
        k = ext[rng.integers(0, ext.size, n)]
    elif kind == 5:                                   # nearly sorted
        k = np.arange(n, dtype=np.float64)
        m = max(1, n // 100)
        i, j = rng.integers(0, max(1, n), m), rng.integers(0, max(1, n), m)
        k[i], k[j] = k[j], k[i].copy()
    else:
        k = synth.pattern(synth.PATTERNS[int(rng.integers(0, len(synth.PATTERNS)))], n, int(rng.integers(1 << 30)))
    return np.ascontiguousarray(k, dtype=np.float64)


def one():
    n = int(np.exp(rng.uniform(0, np.log(1 << a.max_log2))))
    n += int(rng.integers(0, 64))
    entry = rng.choice(["sort", "sort", "omit", "u64", "f32"])
    target = TARGETS[int(rng.integers(0, 4))]
    payload = bool(rng.random() < 0.5)
    if entry == "f32":
        k = keys_f64(n).astype(np.float32)
        v = synth.iota_u32(n)[::-1].copy() if payload else None
        _, ev = oracle.sort_target(k.astype(np.float64), synth.iota_u32(n), target)
        tk = torch.from_numpy(k.copy()).cuda()
        tv = None if v is None else torch.from_numpy(v.copy()).cuda()
        gns.sort_f32_(tk, tv, target=target)
        torch.cuda.synchronize()
        p = ev.astype(np.int64)
        ok = np.array_equal(tk.cpu().numpy().view(np.uint32), k[p].view(np.uint32))
        ok = ok and (v is None or np.array_equal(tv.cpu().numpy(), v[p]))
        return ok, (entry, n, target, payload)
    kt = rng.choice(["f64", "f64", "i64", "u64"])
    k = keys_f64(n)
    if kt == "i64":
        k = (k * 1e6).astype(np.int64) if np.isfinite(k).all() else rng.integers(-100, 100, n).astype(np.int64)
    elif kt == "u64":
        k = (np.abs(k) * 1e6).astype(np.uint64) if np.isfinite(k).all() else rng.integers(0, 100, n).astype(np.uint64)
    if entry == "u64":
        pay = rng.integers(0, 1 << 63, n, dtype=np.uint64)
        ek, ev = oracle.sort_keys(k, synth.iota_u32(n), kt, target)
        tk = torch.from_numpy(k.copy()).cuda()
        tp = torch.from_numpy(pay.copy()).cuda()
        gns.sort_u64_(tk, tp, target=target)
        torch.cuda.synchronize()
        ok = np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64))
        ok = ok and np.array_equal(tp.cpu().numpy(), pay[ev.astype(np.int64)])
        return ok, (entry, kt, n, target)
    v = synth.iota_u32(n)[::-1].copy() if payload else None
    ek, ev = oracle.sort_keys(k, v, kt, target)
    lo = int(rng.integers(0, 8)) if rng.random() < 0.4 else 0          # view t[lo:lo+n]
    hi = int(rng.integers(0, 8)) if lo else 0
    kk = np.concatenate([np.zeros(lo, k.dtype), k, np.zeros(hi, k.dtype)])
    tkf = torch.from_numpy(kk).cuda()
    tk = tkf[lo:lo + n]
    tvf = None if v is None else torch.from_numpy(np.concatenate([np.zeros(lo, np.uint32), v,
                                                                   np.zeros(hi, np.uint32)])).cuda()
    tv = None if tvf is None else tvf[lo:lo + n]
    frac = 1.0
    if entry == "omit":
        gns.sort_omit_(tk, tv, target=target)
    else:
        frac = float(rng.choice([1.0, 1.0, 0.5, 0.25, 0.125, 1 / 64]))
        gns.sort_(tk, tv, frac, target=target)
    torch.cuda.synchronize()
    ok = np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64))
    ok = ok and (v is None or np.array_equal(tv.cpu().numpy(), ev))
    return ok, (entry, kt, n, target, payload, frac, lo)


t_end = time.time() + a.seconds
cases = fails = 0
while time.time() < t_end:
    ok, desc = one()
    cases += 1
    if not ok:
        fails += 1
        print("FAIL", desc, flush=True)
print(f"fuzz: {cases} cases, {fails} failures (seed {a.seed})", flush=True)
