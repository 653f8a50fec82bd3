#!/usr/bin/env python3
"""bench.py — headline benchmark of the B200-native stable f64 mergesort.

Metric (BASELINE.json): sorted keys/s at n = 2^24 f64 (configs[1]: U(0,1),
key-only, buffer fraction 1.0) and its HBM-roofline fraction; tFootprint =
%RAM x time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--frac 1.0] [--no-footprint]

One process per GPU (torchrun for N > 1).  N > 1 (default): the sharded sort
(NEXT f4, dist.sort_distributed) of ONE array of N x 2^24 keys, rank r holding
the r-th 2^24-key shard (rank 0's = BASELINE config 2): local sort, exact
co-ranks, one NCCL all-to-all-v, merge of the received runs; "scaling":
"weak"; per-rank %RAM reported.  --replicas: N independent single-GPU sorts.  Timing: W untimed warm-up steps; each timed step restores
the unsorted input (untimed D2D copy) and flushes L2 (untimed 256 MiB write),
then CUDA events on the sort's stream bracket exactly one sort; the K step
times are summed; barrier + synchronize on both sides; max over ranks.

The oracle (oracle/) is executed only in the cpu_baseline leg and by
--impl reference, on the host cores, never on the GPU path.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (inputs only; holds none of the method)

METRIC = "sorted keys/sec at n=2^24 f64 (and HBM roofline %); tFootprint=%RAM x time"
UNIT = "keys/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, help="BASELINE config index (1..5)")
    ap.add_argument("--sub", default="asc", help="config 4 sub-pattern")
    ap.add_argument("--frac", type=float, default=1.0)
    ap.add_argument("--no-footprint", action="store_true",
                    help="skip the config-5 tFootprint comparison (1.0 vs 0.5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the sharded sort")
    ap.add_argument("--profile-only", action="store_true",
                    help="one warm-up + one sort, no timing loops (for ncu)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def workload(cfg: int, sub: str, frac: float, rank: int):
    case = synth.config(cfg, sub)
    if rank:   # weak-scaling replicas: each rank its own seeded input of the same recipe
        n = case.keys.size
        case.keys = {1: synth.permutation, 2: synth.uniform, 3: lambda n, s: synth.ties(n, s, 24),
                     5: synth.uniform}.get(cfg, lambda n, s: case.keys)(n, 1000 * cfg + 7919 * rank)
    return case


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm), rank 0 only."""
    if rank != 0:
        return
    import oracle
    case = synth.config(args.config, args.sub)
    n = case.keys.size
    keys = case.keys
    vals = case.vals
    for _ in range(min(args.warmup, 1)):
        oracle.sort(keys, vals)
    t = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sort(keys, vals)
        t += time.perf_counter() - t0
    v = n * args.steps / t
    sample = (f"each step: the oracle's stable mergesort of the full workload ({case.name}, n=2^{n.bit_length() - 1}) "
              f"on 1 host core (warm-up {min(args.warmup, 1)} step)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_json(case, args.frac),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_json(case, frac):
    n = case.keys.size
    return {"workload": f"{case.name}: n=2^{n.bit_length() - 1} f64 keys"
                        f"{' + u32 payload' if case.vals is not None else ' key-only'}, buffer fraction {frac}",
            "n": n, "payload": case.vals is not None, "buffer_fraction": frac, "shape": case.shape,
            "l2": "flushed (256 MiB write) before every timed step",
            "input_restore": "untimed device-to-device copy of the unsorted input before every timed step"}


# --------------------------------------------------------------------- ours
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2402_01816_b200 as gns

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (no CPU fallback)")
    # (GNS_BENCH_BACKEND=gloo: ranks may share GPUs -- a functional check of
    # the N > 1 paths on a one-GPU box; timings of shared GPUs mean nothing)
    backend = os.environ.get("GNS_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist

    if world > 1 and not args.replicas:
        run_sharded(args, rank, world, local, dev, pg)
        return

    case = workload(args.config, args.sub, args.frac, rank)
    n = case.keys.size
    hv = case.vals is not None
    s = 12 if hv else 8
    plan = gns.plan(n, args.frac, hv)
    stream = torch.cuda.current_stream(dev)
    st = int(stream.cuda_stream)

    src_k = torch.from_numpy(case.keys).to(dev)
    src_v = torch.from_numpy(case.vals).to(dev) if hv else None
    k = torch.empty_like(src_k)
    v = torch.empty_like(src_v) if hv else None
    ws = gns.alloc_workspace(n, args.frac, hv, dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(256 << 20, 2 * l2), dtype=torch.uint8, device=dev)

    def restore():
        k.copy_(src_k)
        if hv:
            v.copy_(src_v)
        flush.fill_(1)

    def sort_once():
        gns.sort_(k, v, args.frac, workspace=ws)

    for _ in range(max(args.warmup, 3 if not args.profile_only else 1)):
        restore()
        sort_once()
    torch.cuda.synchronize()
    if args.profile_only:
        restore()
        sort_once()
        torch.cuda.synchronize()
        print(json.dumps({"profile_only": True, "n": n}))
        return

    # ---------------------------------------------------------- timed region
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            restore()
            ev[i][0].record(stream)
            sort_once()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(step_ms)
    cdev = torch.device("cpu") if os.environ.get("GNS_BENCH_BACKEND") == "gloo" else dev
    t_max, value = aggregate(torch, pg, t_ms, n, args.steps, world, cdev)
    ms_per_step = t_max / args.steps

    # validity of the last output: GPU-side properties only (the oracle is not
    # used here): non-decreasing, same multiset of key bits (two wrapping
    # moment hashes), and for index payloads: ties in ascending index order.
    ok_sorted = bool((k[1:] >= k[:-1]).all().item()) if n > 1 else True
    kb, sb = k.view(torch.int64), src_k.view(torch.int64)
    ok_perm = bool((kb.sum() == sb.sum()).item() and ((kb * kb).sum() == (sb * sb).sum()).item())
    if hv and n > 1:
        tie = k[1:] == k[:-1]
        ok_perm = ok_perm and bool((v[1:].to(torch.int64)[tie] > v[:-1].to(torch.int64)[tie]).all().item())

    # ------------------------------------------- per-kernel timing (roofline)
    roof = kernel_roofline(gns, torch, dev, stream, src_k, src_v, k, v, n, hv, s, plan, restore, ws, args.frac)
    peak, peak_src = measured_peaks()
    achieved = roof["merge_pass_gbs"]
    traffic = ncu_traffic(case, args.frac)

    # ----------------------------------------------------------- end-to-end
    e2e = end_to_end(gns, torch, dev, stream, case, args, n, hv, ws)

    footprint = None
    presorted = None
    others = None
    keytypes = None
    half = None
    if rank == 0 and world == 1 and not args.no_footprint and args.config == 2:
        half = half_buffer(gns, torch, dev, stream, flush, src_k, k, n, s)
        footprint = footprint_cfg5(gns, torch, dev, stream, flush)
        presorted = config4(gns, torch, dev, stream, flush)
        others = other_configs(gns, torch, dev, stream, flush)
        keytypes = key_types(gns, torch, dev, stream, flush)

    cpu = None
    bitexact = None
    if rank == 0 and not args.no_cpu_baseline:
        # (rank 0's input is the BASELINE workload itself; other ranks' replicas
        # are checked by the GPU-side properties above)
        cpu, (ek, ev) = cpu_baseline(case)
        gk = k.cpu().numpy()
        bitexact = bool(np.array_equal(gk.view(np.uint64), ek.view(np.uint64)))
        if hv:
            bitexact = bitexact and bool(np.array_equal(v.cpu().numpy(), ev))
        if world > 1:
            cpu = None          # (cpu_baseline: rank 0 at N=1 only)

    # ------------------- the allocating C-ABI call (buffer allocated per call)
    alloc = allocating_api(gns, torch, dev, stream, src_k, src_v, k, v, n, hv, s, args.frac, restore,
                           max(3, min(args.steps, 10)))

    launches_per_step = launches(plan, args.frac, n)
    ram = 1.0 + plan["workspace_bytes"] / (n * s)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "step_ms_rank0": {"median": float(np.median(step_ms)), "min": float(min(step_ms))},
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, see DESIGN.md §3)",
        "config": dict(config_json(case, args.frac), parallelism=f"replicas{world}" if world > 1 else "single"),
        "roofline": {"bound": "hbm", "kernel": "merge pass (merge_tstore_kernel: K2 co-rank search warps + K3 TMA-pipelined merge, one launch per pass), avg over "
                     f"{plan['merge_passes']} passes", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "frac_vs_nominal_8tbs": achieved / 8000.0, "traffic": traffic,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": 2 * n * s,
                     "share_of_step": roof["merge_share"],
                     "whole_sort": {"bytes_lower_bound": plan["bytes_lower_bound"],
                                    "element_passes": plan["element_passes"],
                                    "achieved": plan["bytes_lower_bound"] / (ms_per_step / 1e3) / 1e9,
                                    "frac": plan["bytes_lower_bound"] / (ms_per_step / 1e3) / 1e9 / peak,
                                    "frac_vs_nominal_8tbs": plan["bytes_lower_bound"] / (ms_per_step / 1e3) / 8e12},
                     "per_kernel_ms": roof["per_kernel_ms"]},
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "ram_pct": ram, "tfootprint_ms": ram * ms_per_step,
        "bitexact": bitexact,
        "valid": {"sorted": ok_sorted, "same_multiset_and_stable_ties": ok_perm,
                  "bitexact_vs_oracle": bitexact},
        "allocating_api": alloc,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if half:
        line["buffer_0.5_same_config"] = half
    if footprint:
        line["footprint_cfg5"] = footprint
    if presorted:
        line["presorted_cfg4"] = presorted
    if others:
        line["other_configs"] = others
    if keytypes:
        line["key_types_f3"] = keytypes
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def run_sharded(args, rank, world, local, dev, pg):
    """N > 1: the distributed stable sort of one array (NEXT f4), weak
    scaling (2^24 keys per rank).  Device-timed per step with CUDA events on
    the sort's stream (collectives included), max over ranks."""
    import torch
    import paper_2402_01816_b200 as gns
    from paper_2402_01816_b200 import dist as gdist
    n = 1 << 24
    keys = synth.uniform(n, 1000 * 2 + (7919 * rank if rank else 0))       # rank 0: BASELINE config 2
    src = torch.from_numpy(keys).to(dev)
    k = torch.empty_like(src)
    ws = gns.alloc_workspace(n, args.frac, False, dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    info = {}
    out = None

    def step():
        nonlocal out
        k.copy_(src)
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = gdist.sort_distributed(k, None, samples=64, buffer_fraction=args.frac, workspace=ws, info=info)
        b.record(stream)
        return a, b

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    pg.barrier()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            evs.append(step())
        torch.cuda.synchronize()
    pg.barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    cdev = torch.device("cpu") if os.environ.get("GNS_BENCH_BACKEND") == "gloo" else dev   # (gloo: host tensors)
    t_max, value = aggregate(torch, pg, t_ms, n, args.steps, world, cdev)
    ok_k = out[0]
    # validity: every piece sorted, pieces in rank order (last key <= next first), balanced sizes
    ends = torch.tensor([ok_k[0].item() if ok_k.numel() else 0.0, ok_k[-1].item() if ok_k.numel() else 0.0,
                         float(ok_k.numel()), float(bool((ok_k[1:] >= ok_k[:-1]).all().item()))],
                        dtype=torch.float64, device=cdev)
    allends = [torch.empty_like(ends) for _ in range(world)]
    pg.all_gather(allends, ends)
    e = torch.stack(allends).cpu().numpy()
    ok = bool(all(e[:, 3] == 1.0) and all(e[i, 1] <= e[i + 1, 0] for i in range(world - 1))
              and all(e[:, 2] == n))
    ram = torch.tensor([info.get("ram_pct_peak", 0.0), info.get("ram_pct_sort", 0.0),
                        info.get("ram_pct_exchange", 0.0)], dtype=torch.float64, device=cdev)
    pg.all_reduce(ram, op=pg.ReduceOp.MAX)
    ms = t_max / args.steps
    if rank == 0:
        plan = gns.plan(n, args.frac, False)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64 U(0,1), see DESIGN.md §3)",
            "config": {"workload": f"sharded stable sort of one array of {world} x 2^24 f64 U(0,1) keys "
                                   f"(rank r holds shard r; rank 0's is BASELINE config 2), buffer fraction {args.frac}",
                       "n_per_rank": n, "parallelism": f"sharded{world} (local sort, exact co-ranks, one NCCL "
                                                       f"all-to-all-v, merge tree of the received runs)",
                       "l2": "flushed (256 MiB write) before every timed step"},
            "gpu_launches": args.steps * (plan["launches"] + world),
            "clocks": clk.summary(),
            "ram_pct": float(ram[0]), "ram_pct_local_sort": float(ram[1]), "ram_pct_exchange": float(ram[2]),
            "tfootprint_ms": float(ram[0]) * ms,
            "valid": {"pieces_sorted_in_rank_order_balanced": ok},
            "e2e": None,
        }
        print(json.dumps(line), flush=True)
    pg.barrier()
    pg.destroy_process_group()


def aggregate(torch, pg, t_ms, n, steps, world, device):
    """Whole-job throughput of `world` replicas: every rank sorted `steps`
    inputs of n keys in t_ms of device time; the job time is the max over
    ranks (all_reduce MAX), value = world * n * steps / max_t."""
    t_max = float(t_ms)
    if pg is not None and world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=device)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        t_max = float(tt.item())
    return t_max, world * n * steps / (t_max / 1e3)


def launches(plan, frac, n):
    """Kernel launches of one sort, from the library's own schedule (gns_plan)."""
    return plan["launches"]


def kernel_roofline(gns, torch, dev, stream, src_k, src_v, k, v, n, hv, s, plan, restore, ws, frac, reps=5):
    """Times every kernel of the product sort (gns_sort_*_ws, the same call the
    timed region makes) with CUDA events recorded by the library on the
    launching stream between launches (gns_timing_begin/end)."""
    per = []
    for _ in range(reps):
        restore()
        assert gns.gns_timing_begin(256) == 0
        gns.sort_(k, v, frac, workspace=ws, stream=stream)
        per.append(gns.gns_timing_end())
    kinds = [kd for kd, _ in per[0]]
    med = [float(np.median([r[i][1] for r in per])) for i in range(len(kinds))]
    tile = [t for kd, t in zip(kinds, med) if kd == 1]
    merge = [t for kd, t in zip(kinds, med) if kd == 2]
    total = sum(med)
    mavg = float(np.mean(merge)) if merge else 0.0
    return {"merge_pass_gbs": (2 * n * s) / (mavg / 1e3) / 1e9 if merge else 0.0,
            "merge_share": sum(merge) / total if total else 0.0,
            "per_kernel_ms": {"tile_sort": sum(tile), "merge_passes": merge,
                              "tile_sort_gbs": (2 * n * s) / (sum(tile) / 1e3) / 1e9 if tile else 0.0,
                              "launches": [[gns.LAUNCH_KINDS.get(kd, "other"), t] for kd, t in zip(kinds, med)]}}


def ncu_traffic(case, frac):
    """DRAM bytes per merge-pass launch from the committed ncu --set full
    summary for this workload (profiles/ncu_merge_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_merge_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("n") == case.keys.size and d.get("payload") == (case.vals is not None):
            return d["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def end_to_end(gns, torch, dev, stream, case, args, n, hv, ws, steps=None):
    """Same metric through the public C-ABI call, from pinned host memory:
    every step copies its input host->device, sorts it (gns_sort_*_ws) and
    copies the sorted result device->host, all inside the timed region.
    Steps rotate over three buffer sets on three streams, so step i+1's
    upload, step i's sort and step i-1's download overlap (PCIe is full
    duplex) -- a serving pipeline; the fully serial figure is reported beside
    it."""
    steps = steps or max(4, min(args.steps, 12))
    hk = torch.from_numpy(case.keys).pin_memory()
    hv_ = torch.from_numpy(case.vals).pin_memory() if hv else None
    nslot = 3
    slots = []
    for i in range(nslot):
        slots.append({
            "st": stream if i == 0 else torch.cuda.Stream(dev),
            "dk": torch.empty(n, dtype=torch.float64, device=dev),
            "dv": torch.empty(n, dtype=torch.uint32, device=dev) if hv else None,
            "ok": torch.empty(n, dtype=torch.float64).pin_memory(),
            "ov": torch.empty(n, dtype=torch.uint32).pin_memory() if hv else None,
            "ws": ws if i == 0 else gns.alloc_workspace(n, args.frac, hv, dev),
        })

    def step(sl):
        with torch.cuda.stream(sl["st"]):
            sl["dk"].copy_(hk, non_blocking=True)
            if hv:
                sl["dv"].copy_(hv_, non_blocking=True)
            gns.sort_(sl["dk"], sl["dv"], args.frac, workspace=sl["ws"], stream=sl["st"])
            sl["ok"].copy_(sl["dk"], non_blocking=True)
            if hv:
                sl["ov"].copy_(sl["dv"], non_blocking=True)

    def timed(pipelined):
        for sl in slots:
            step(sl)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for sl in slots[1:]:
            sl["st"].wait_event(a)
        for i in range(steps):
            sl = slots[i % nslot] if pipelined else slots[0]
            step(sl)
        for sl in slots[1:]:
            done = torch.cuda.Event()
            done.record(sl["st"])
            stream.wait_event(done)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3

    t_pipe = timed(True)
    t_serial = timed(False)
    ok = bool((slots[0]["ok"][1:] >= slots[0]["ok"][:-1]).all().item())
    by = n * (12 if hv else 8)
    return {"value": n * steps / t_pipe, "unit": UNIT, "h2d_bytes_per_step": by, "d2h_bytes_per_step": by,
            "steps": steps, "serial_value": n * steps / t_serial, "host_result_sorted": ok,
            "path": "pinned host -> H2D -> gns_sort_*_ws -> D2H -> pinned host, three buffer sets rotating on "
                    "three streams (upload of step i+1, sort of step i, download of step i-1 overlap)"}


def allocating_api(gns, torch, dev, stream, src_k, src_v, k, v, n, hv, s, frac, restore, reps):
    """The plain C-ABI call (gns_sort_f64 / gns_sort_pairs_f64_u32: the buffer
    is allocated and freed stream-ordered inside the call, SURVEY §8(a) a7,
    reading A8) timed like the headline (L2 flushed, input restored untimed),
    and the measured %RAM: the high-water mark of the device's default memory
    pool (the one the call allocates from) during the call."""
    ts = []
    hw = None
    for i in range(reps + 1):
        restore()
        torch.cuda.synchronize()
        gns.gns_pool_high_water(1)          # (torch's caching allocator is a separate pool)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gns.sort_(k, v, frac, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
        hw = gns.gns_pool_high_water(0)
    ms = float(np.median(ts))
    data = n * s
    return {"ms": ms, "keys_per_s": n / (ms / 1e3), "pool_high_water_bytes": hw,
            "ram_pct_measured": 1.0 + hw / data if hw is not None and hw != (1 << 64) - 1 else None,
            "ram_pct_nominal": 1.0 + gns.workspace_bytes(n, frac, hv) / data,
            "note": "cudaMallocAsync/cudaFreeAsync of the whole buffer inside every timed call"}


def half_buffer(gns, torch, dev, stream, flush, src_k, k, n, s, reps=10):
    """The headline workload at buffer fraction 0.5 (%RAM 1.5): runtime and
    tFootprint beside the 1.0 line."""
    ws = gns.alloc_workspace(n, 0.5, False, dev)
    ts = []
    for i in range(reps + 2):
        k.copy_(src_k)
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gns.sort_(k, None, 0.5, workspace=ws)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ram = 1.0 + ws.numel() / (n * s)
    return {"ms": ms, "keys_per_s": n / (ms / 1e3), "ram_pct": ram, "tfootprint_ms": ram * ms,
            "sorted": bool((k[1:] >= k[:-1]).all().item()),
            "element_passes": gns.plan(n, 0.5, False)["element_passes"]}


def footprint_cfg5(gns, torch, dev, stream, flush, reps=3):
    """configs[4]: n = 2^27 U(0,1) + u32 index at buffer fractions 1.0, 0.5
    (the BASELINE pair) and the NEXT-f1 sweep 0.25, 0.125, 1/16: runtime,
    %RAM (exact workspace bytes) and tFootprint = %RAM x runTime."""
    case = synth.config(5)
    n = case.keys.size
    src_k = torch.from_numpy(case.keys).to(dev)
    src_v = torch.from_numpy(case.vals).to(dev)
    k, v = torch.empty_like(src_k), torch.empty_like(src_v)
    out = {"workload": "cfg5: n=2^27 f64 U(0,1) + u32 index", "n": n}
    first = None
    agree = True
    for frac in (1.0, 0.5, 0.25, 0.125, 0.0625):
        ws = gns.alloc_workspace(n, frac, True, dev)
        times = []
        for i in range(reps + 1):
            k.copy_(src_k)
            v.copy_(src_v)
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gns.sort_(k, v, frac, workspace=ws)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= 1:
                times.append(a.elapsed_time(b))
        if first is None:
            first = k.clone(), v.clone()
        else:
            agree = agree and bool(torch.equal(first[0].view(torch.int64), k.view(torch.int64)) and
                                   torch.equal(first[1].view(torch.int32), v.view(torch.int32)))
        ram = 1.0 + ws.numel() / (n * 12)
        ms = float(np.median(times))
        out[str(frac)] = {"ms": ms, "keys_per_s": n / (ms / 1e3), "ram_pct": ram,
                          "tfootprint_ms": ram * ms, "workspace_bytes": int(ws.numel()),
                          "element_passes": gns.plan(n, frac, True)["element_passes"]}
        del ws
    out["all_fractions_agree_bitexact"] = agree
    out["tfootprint_0.5_lt_1.0"] = out["0.5"]["tfootprint_ms"] < out["1.0"]["tfootprint_ms"]
    out["argmin_tfootprint_fraction"] = min((f for f in out if f.replace(".", "").isdigit()),
                                            key=lambda f: out[f]["tfootprint_ms"])
    return out


def config4(gns, torch, dev, stream, flush, reps=5):
    """configs[3]: n = 2^24 presorted patterns, key-only, buffer 1.0, through
    the default schedule (``sort_``: a fully ordered or strictly reversed
    input skips the merge passes on the device) and through the Omitsort
    schedule (``sort_omit_``, NEXT f2: per-pair omission with run-location
    tracking)."""
    out = {}
    n = 1 << 24
    ws = gns.alloc_workspace(n, 1.0, False, dev)
    for sub in synth.CONFIG4_SUBS:
        src = torch.from_numpy(synth.config(4, sub).keys).to(dev)
        k = torch.empty_like(src)
        for sched in ("default", "omit"):
            ts = []
            for i in range(reps + 1):
                k.copy_(src)
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if sched == "omit":
                    gns.sort_omit_(k, None, workspace=ws)
                else:
                    gns.sort_(k, None, 1.0, workspace=ws)
                b.record(stream)
                torch.cuda.synchronize()
                if i:
                    ts.append(a.elapsed_time(b))
            ok = bool((k[1:] >= k[:-1]).all().item())
            ms = float(np.median(ts))
            r = {"ms": ms, "keys_per_s": n / (ms / 1e3), "sorted": ok}
            if sched == "omit":
                out[sub]["omit"] = r
            else:
                out[sub] = r
    return out


def key_types(gns, torch, dev, stream, flush, reps=5):
    """NEXT f3 at n = 2^24 (same timing rules): int64 keys (the 8-byte path),
    binary32 keys key-only and with a u32 payload (the 4-byte kernels), f64
    keys with a 64-bit payload (index sort + gather); median ms, keys/s,
    %RAM."""
    n = 1 << 24
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    cases = {
        "i64": (torch.randint(-(1 << 62), 1 << 62, (n,), device=dev, generator=g), None),
        "f32": (torch.rand(n, device=dev, generator=g, dtype=torch.float32), None),
        "f32_u32": (torch.rand(n, device=dev, generator=g, dtype=torch.float32),
                    torch.arange(n, device=dev, dtype=torch.int64).to(torch.uint32)),
        "f64_u64": (torch.rand(n, device=dev, generator=g, dtype=torch.float64),
                    torch.arange(n, device=dev, dtype=torch.int64)),
    }
    out = {}
    for name, (src, srcv) in cases.items():
        if name.startswith("f32"):
            ws = torch.empty(max(1, gns.workspace_bytes_f32(n, srcv is not None)), dtype=torch.uint8, device=dev)
            run = lambda k, v: gns.sort_f32_(k, v, workspace=ws, stream=stream)
            data = n * (4 + (4 if srcv is not None else 0))
        elif name == "f64_u64":
            ws = torch.empty(gns.workspace_bytes_u64(n), dtype=torch.uint8, device=dev)
            run = lambda k, v: gns.sort_u64_(k, v, workspace=ws, stream=stream)
            data = n * 16
        else:
            ws = gns.alloc_workspace(n, 1.0, False, dev)
            run = lambda k, v: gns.sort_(k, v, 1.0, workspace=ws, stream=stream)
            data = n * 8
        ts = []
        for i in range(reps + 1):
            k = src.clone()
            v = None if srcv is None else srcv.clone()
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run(k, v)
            b.record(stream)
            torch.cuda.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        out[name] = {"ms": ms, "keys_per_s": n / (ms / 1e3), "sorted": bool((k[1:] >= k[:-1]).all().item()),
                     "ram_pct": 1.0 + ws.numel() / data}
        del ws
    return out


def other_configs(gns, torch, dev, stream, flush, reps=5):
    """configs[0] (2^16 permutation + payload) and configs[2] (2^24 heavy
    ties + payload), buffer 1.0: median ms and keys/s (same timing rules)."""
    out = {}
    for c in (1, 3):
        case = synth.config(c)
        n = case.keys.size
        src = torch.from_numpy(case.keys).to(dev)
        srcv = torch.from_numpy(case.vals).to(dev)
        k, v = torch.empty_like(src), torch.empty_like(srcv)
        ws = gns.alloc_workspace(n, 1.0, True, dev)
        ts = []
        for i in range(reps + 3):
            k.copy_(src)
            v.copy_(srcv)
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gns.sort_(k, v, 1.0, workspace=ws)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        tie = k[1:] == k[:-1]
        ok = bool((k[1:] >= k[:-1]).all().item()) and bool(
            (v[1:].to(torch.int64)[tie] > v[:-1].to(torch.int64)[tie]).all().item())
        ms = float(np.median(ts))
        out[f"cfg{c}"] = {"workload": case.shape, "n": n, "payload": True, "ms": ms,
                          "keys_per_s": n / (ms / 1e3), "sorted_stable": ok}
    return out


def host_cpu():
    """The host CPU model and core count (report them beside the oracle)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model}, {os.cpu_count()} logical cores"


def cpu_baseline(case):
    """The oracle, as it stands, on the host: the full workload sorted 3x on 1
    core (~10 s).  Also returns its output, which the timed GPU output is
    compared with bit for bit."""
    import oracle
    keys = case.keys
    vals = case.vals
    reps = 3
    out = None
    t0 = time.perf_counter()
    for _ in range(reps):
        out = oracle.sort(keys, vals)
    t = time.perf_counter() - t0
    return ({"value": keys.size * reps / t, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_cpu(),
             "sample": f"{case.name}, full n={keys.size}, sorted {reps}x by the single-threaded oracle "
                       f"(host has {os.cpu_count()} cores)"}, out)


if __name__ == "__main__":
    main()
