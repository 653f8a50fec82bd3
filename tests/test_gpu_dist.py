"""NEXT f4 on the GPU: the real ``sort_distributed`` (not ``simulate``) with
this package's CUDA kernels, k processes.

* several processes sharing cuda:0 with the gloo backend (collectives staged
  through the host; no kernel ever waits on another process, so sharing one
  GPU is safe -- B200_PROFILING.md);
* with >= 2 visible GPUs, one process per GPU over NCCL (skipped on the
  one-GPU boxes of this pool).

Checks: the ranks' outputs concatenated are the oracle's stable sort of the
rank-major concatenation (bit-exact, payload = global index); balanced pieces;
per-rank footprint (in-place local sort with the caller's buffer fraction,
one receive buffer, the merge tree inside the shard's memory: peak %RAM
<= 2.0, local sort 1 + p)."""
import os
import socket
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T1 = 8192


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(case, rank, world):
    n = [3 * T1 + 101 * rank, 5 * T1, 2 * T1 + 7][case]
    if case == 0:
        return synth.ties(n, 500 + rank, 40)
    if case == 1:
        return synth.uniform(n, 600 + rank)
    k = synth.uniform(n, 700 + rank) + rank          # rank r holds [r, r+1): no interleaving
    return k


def _worker(rank, world, port, backend, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_01816_b200 import dist as gdist
    try:
        for case in (0, 1, 2):
            k = _shard(case, rank, world)
            base = sum(_shard(case, r, world).size for r in range(rank))
            v = (np.arange(k.size) + base).astype(np.uint32)
            for frac in (1.0, 0.5):
                info = {}
                ok, ov = gdist.sort_distributed(torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev),
                                                samples=32, buffer_fraction=frac, info=info)
                torch.cuda.synchronize()
                q.put((case, frac, rank, ok.cpu().numpy(), ov.cpu().numpy(), info))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, backend):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world * 3 * 2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for case in (0, 1, 2):
        shards = [_shard(case, r, world) for r in range(world)]
        allk = np.concatenate(shards)
        N = allk.size
        ek, ev = oracle.sort(allk, np.arange(N, dtype=np.uint32))
        for frac in (1.0, 0.5):
            got = sorted([r for r in res if r[0] == case and r[1] == frac], key=lambda x: x[2])
            gk = np.concatenate([g[3] for g in got])
            gv = np.concatenate([g[4] for g in got])
            assert np.array_equal(gk.view(np.uint64), ek.view(np.uint64)), f"case {case} frac {frac}"
            assert np.array_equal(gv, ev), f"case {case} frac {frac}"
            assert [g[3].size for g in got] == [((r + 1) * N) // world - (r * N) // world for r in range(world)]
            for g in got:
                info = g[5]
                assert info["ram_pct_sort"] <= 1.0 + frac + 0.02, info
                if case == 1:                      # equal shards: the tree stays in the shard's memory
                    assert info["partner_bytes"] == 0 and info["ram_pct_peak"] <= 2.0 + 0.02, info


@pytest.mark.parametrize("world", [2, 3])
def test_sort_distributed_processes_sharing_one_gpu_gloo(world):
    assert torch.cuda.is_available()
    _run(world, "gloo")


def test_sort_distributed_nccl_multi_gpu():
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU visible: the NCCL multi-GPU run needs >= 2 (gloo-on-one-GPU covers the logic)")
    _run(min(torch.cuda.device_count(), 4), "nccl")
