"""NEXT f4: the distributed sort's orchestration
(paper_2402_01816_b200.dist) on CPU with the gloo backend, world_size 2 and 3.

The data steps (local sort, cuts, two-run merge) are the oracle's here
(test-only CPU ops); the splitter choice, counts, all-to-all-v exchange and
merge-tree order are the product code.  The concatenation of the ranks'
outputs must equal the oracle's stable sort of the concatenated shards,
bit-exact, payload included."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


KT = {torch.float64: "f64", torch.int64: "i64", torch.uint64: "u64"}


class CpuOracleOps:
    """Test-only CPU implementations of the three data steps (oracle /
    numpy), so the orchestration runs without a GPU."""

    def sort(self, keys, vals):
        import oracle
        kt = KT[keys.dtype]
        k, v = oracle.sort_keys(keys.numpy(), None if vals is None else vals.numpy(), kt)
        return torch.from_numpy(k), (None if v is None else torch.from_numpy(v))

    def cuts(self, sorted_keys, spl_key, spl_rank, spl_pos, me):
        a = sorted_keys.numpy()
        out = []
        for x, r, p in zip(spl_key.numpy(), spl_rank.numpy(), spl_pos.numpy()):
            if r == me:
                out.append(int(p))
            else:
                out.append(int(np.searchsorted(a, x, side="right" if me < r else "left")))
        return torch.tensor(out, dtype=torch.int64)

    def merge_two(self, a_k, a_v, b_k, b_v):
        k = torch.cat([a_k, b_k])
        v = None if a_v is None else torch.cat([a_v, b_v])
        return self.sort(k, v)


class CpuFootprintOps(CpuOracleOps):
    """The same CPU data steps plus the footprint-aware interface of the
    product ops: sort with a buffer fraction and workspace (sized by the
    library's own gns_workspace_bytes), and merge_into (the ping-pong tree
    writes into given views instead of allocating)."""

    def sort(self, keys, vals, buffer_fraction=1.0, workspace=None):
        k, v = CpuOracleOps.sort(self, keys, vals)
        keys.copy_(k)                         # in place, like the CUDA op
        if vals is not None:
            vals.copy_(v)
        return keys, vals

    def workspace_bytes(self, n, buffer_fraction, with_vals):
        import paper_2402_01816_b200 as gns
        return gns.workspace_bytes(n, buffer_fraction, with_vals)

    def merge_into(self, a_k, a_v, b_k, b_v, d_k, d_v):
        k, v = self.merge_two(a_k, a_v, b_k, b_v)
        d_k.copy_(k)
        if d_v is not None:
            d_v.copy_(v)


def make_shard(case, rank, world):
    rng = np.random.default_rng(1000 * case + rank)
    if case == 0:          # f64, heavy ties, signed zeros
        n = 3000 + 700 * rank
        k = rng.integers(-5, 6, n).astype(np.float64)
        k[k == 0] = np.where(rng.random((k == 0).sum()) < 0.5, -0.0, 0.0)
    elif case == 1:        # f64 distinct-ish, one empty shard
        n = 0 if rank == world - 1 else 5000
        k = rng.random(n)
    elif case == 2:        # int64 extremes
        n = 2000 + 13 * rank
        k = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, n, dtype=np.int64, endpoint=True)
        k[::3] = rng.integers(-3, 3, k[::3].size)
    elif case == 3:        # uint64, all keys equal on every rank (stability across ranks)
        n = 1500
        k = np.full(n, 7, dtype=np.uint64)
    else:                  # tiny shards (fewer elements than samples)
        n = 5 + rank
        k = rng.integers(0, 4, n).astype(np.float64)
    return k


CASES = (0, 1, 2, 3, 4)


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_01816_b200 import dist as gdist
    for case in CASES:
        k = make_shard(case, rank, world)
        base = sum(make_shard(case, r, world).size for r in range(rank))
        v = (np.arange(k.size) + base).astype(np.uint32)
        for bal in (True, False):
            ok, ov = gdist.sort_distributed(torch.from_numpy(k), torch.from_numpy(v), samples=16, ops=CpuOracleOps(),
                                            balanced=bal)
            q.put((case, bal, rank, ok.numpy(), ov.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_sort_gloo(world):
    """All five shard patterns in one world_size-`world` gloo group."""
    import oracle
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world * len(CASES) * 2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case in CASES:
        shards = [make_shard(case, r, world) for r in range(world)]
        allk = np.concatenate(shards)
        allv = np.arange(allk.size, dtype=np.uint32)
        kt = {np.dtype(np.float64): "f64", np.dtype(np.int64): "i64", np.dtype(np.uint64): "u64"}[allk.dtype]
        ek, ev = oracle.sort_keys(allk, allv, kt)
        N = allk.size
        for bal in (True, False):
            got = sorted([r for r in res if r[0] == case and r[1] == bal], key=lambda x: x[2])
            gk = np.concatenate([r[3] for r in got])
            gv = np.concatenate([r[4] for r in got])
            what = f"case {case} world {world} balanced={bal}"
            assert gk.view(np.uint64).tolist() == ek.view(np.uint64).tolist(), what
            assert gv.tolist() == ev.tolist(), what
            if bal:   # exact co-ranks: rank g holds global ranks [g N / k, (g+1) N / k)
                assert [r[3].size for r in got] == [((g + 1) * N) // world - (g * N) // world
                                                    for g in range(world)], what


@pytest.mark.parametrize("samples", [1, 16])
@pytest.mark.parametrize("balanced", [True, False])
@pytest.mark.parametrize("case", CASES)
def test_simulate_matches_collective_cpu(case, balanced, samples):
    """dist.simulate (one process, no collectives) == the oracle too; with
    exact co-ranks every piece has its balanced size."""
    import oracle
    from paper_2402_01816_b200 import dist as gdist
    world = 4
    shards = [make_shard(case, r, world) for r in range(world)]
    base = np.cumsum([0] + [s.size for s in shards])
    outs = gdist.simulate([(torch.from_numpy(s), torch.from_numpy((np.arange(s.size) + base[r]).astype(np.uint32)))
                           for r, s in enumerate(shards)], samples=samples, ops=CpuOracleOps(), balanced=balanced)
    allk = np.concatenate(shards)
    kt = {np.dtype(np.float64): "f64", np.dtype(np.int64): "i64", np.dtype(np.uint64): "u64"}[allk.dtype]
    ek, ev = oracle.sort_keys(allk, np.arange(allk.size, dtype=np.uint32), kt)
    assert np.concatenate([o[0].numpy() for o in outs]).view(np.uint64).tolist() == ek.view(np.uint64).tolist()
    assert np.concatenate([o[1].numpy() for o in outs]).tolist() == ev.tolist()
    if balanced:
        N = allk.size
        assert [o[0].numel() for o in outs] == [((g + 1) * N) // world - (g * N) // world for g in range(world)]


def _fp_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_01816_b200 import dist as gdist
    n = 40000                                   # equal shards: balanced pieces fit the shard's memory
    rng = np.random.default_rng(77 + rank)
    k = rng.integers(0, 50, n).astype(np.float64)
    v = (np.arange(n) + rank * n).astype(np.uint32)
    for frac in (1.0, 0.5):
        info = {}
        tk, tv = torch.from_numpy(k.copy()), torch.from_numpy(v.copy())
        ok, ov = gdist.sort_distributed(tk, tv, samples=8, ops=CpuFootprintOps(), buffer_fraction=frac, info=info)
        q.put((frac, rank, ok.numpy().copy(), ov.numpy().copy(), info))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_sort_footprint_gloo(world):
    """f4 footprint: the shard sorted in place with the caller's buffer
    fraction, one receive buffer, the ping-pong merge tree inside the
    shard's memory: per-rank peak %RAM <= 2.0 (1.0 + p for the local sort,
    2.0 for the exchange of balanced equal shards), output bit-exact."""
    import oracle
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world * 2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 40000
    allk = np.concatenate([np.random.default_rng(77 + r).integers(0, 50, n).astype(np.float64) for r in range(world)])
    ek, ev = oracle.sort(allk, np.arange(allk.size, dtype=np.uint32))
    for frac in (1.0, 0.5):
        got = sorted([r for r in res if r[0] == frac], key=lambda x: x[1])
        assert np.concatenate([g[2] for g in got]).view(np.uint64).tolist() == ek.view(np.uint64).tolist()
        assert np.concatenate([g[3] for g in got]).tolist() == ev.tolist()
        for g in got:
            info = g[4]
            assert info["partner_bytes"] == 0                       # the tree ping-pongs in the shard's memory
            assert info["ram_pct_sort"] <= 1.0 + frac + 0.02
            assert info["ram_pct_exchange"] <= 2.0 + 1e-9
            assert info["ram_pct_peak"] <= 2.0 + 0.02
