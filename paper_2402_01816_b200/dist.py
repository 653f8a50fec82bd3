"""NEXT f4: stable sort of an array sharded over the ranks of
a ``torch.distributed`` group, one GPU per rank, with ONE data exchange.

The paper parallelises its merges "over an arbitrary number of processes"
(§Parallel sorting); across GPUs the natural form is
sort -> split -> exchange -> merge:

1. every rank stably sorts its shard with the single-GPU path
   (``gns_sort_keys``);
2. the ranks agree on k-1 splitters: each contributes ``samples`` regularly
   spaced elements of its sorted shard as (key, rank, position) triples, the
   triples are all-gathered in rank order and stably sorted by key -- which
   orders them by (key, rank, position) -- and every (V/k)-th one is taken;
3. each rank cuts its sorted shard at the splitters (``gns_split_cuts``:
   elements preceding splitter i in the global order (key, rank, position));
4. one all-to-all-v (NCCL over NVLink) sends piece j to rank j;
5. each rank merges the k received sorted runs in rank order with a pairwise
   tree of ``gns_merge_two`` launches (left run wins ties).

With ``balanced=True`` (default) steps 2-3 are exact instead (SURVEY.md
§8(e) step 2, "the k co-ranks across the k sorted shards"): rank g receives
exactly the elements of global stable rank [g N / k, (g+1) N / k).  For every
target rank R each rank keeps a window [lo, hi] of its cut; per round every
rank proposes ``samples`` elements evenly spaced in its window, all ranks
count (``gns_split_cuts``) how many of their elements precede each proposal,
one all-reduce sums the counts C(x), and each rank narrows its window:
C(x) < R puts x among the first R (lo >= its count, +1 on the owner),
C(x) >= R keeps it out (hi <= its count).  A rank's own proposals split its
window into ``samples`` + 1 parts, so about log_{samples+1}(n) rounds; the
cuts are exact when the windows' lower ends sum to R.

Global order: (key, rank, position in the rank's shard) = stable in the
rank-major input order, so the concatenation of the ranks' outputs is the
unique stable sort of the concatenated shards (bit-exact, payload included).
With sample splitters (``balanced=False``) output sizes vary per rank
(splitter quality) and a rank may receive nothing; with exact co-ranks
(default) they are the balanced shares.

Footprint (%RAM per rank; the paper's parallel claim is about
Footprint): the shard is sorted IN PLACE with the caller's
buffer fraction (1.0 or <= 0.5, optional caller workspace); the exchange
receives into ONE buffer of the received size; the k received runs are merged
by a pairwise tree that ping-pongs between that buffer and the shard's own
(then dead) memory -- no allocation per merge.  Peak bytes per rank: the
local sort (1 + p) and the exchange/merge phase (1 + received / shard size,
2.0 for balanced equal shards); ``info`` reports both.  The exact co-rank
rounds run on the device without host round trips (a fixed number of rounds
from the shard sizes, one convergence check).

Every step that touches the data runs in this package's CUDA kernels; the
``ops`` argument exists so the orchestration can be exercised on CPU with the
gloo backend in tests (tests/test_dist_sort.py passes oracle-based CPU ops);
the default ops are the CUDA ones and fail loudly without the extension.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import paper_2402_01816_b200 as gns


# Collectives: NCCL takes the CUDA tensors directly; the gloo backend (CPU
# tests, or several processes sharing one GPU in the GPU tests) stages CUDA
# tensors through host copies.
def _staged(group, t):
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _all_reduce(t, op=None, group=None):
    import torch.distributed as dist
    op = op if op is not None else dist.ReduceOp.SUM
    if _staged(group, t):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def _all_gather(outs, t, group=None):
    import torch.distributed as dist
    if _staged(group, t):
        ho = [o.cpu() for o in outs]
        dist.all_gather(ho, t.cpu(), group=group)
        for o, h in zip(outs, ho):
            o.copy_(h)
    else:
        dist.all_gather(outs, t, group=group)


def _all_to_all_single(out, inp, out_split=None, in_split=None, group=None):
    import torch.distributed as dist
    if _staged(group, inp):
        ho = out.cpu()
        dist.all_to_all_single(ho, inp.cpu(), out_split, in_split, group=group)
        out.copy_(ho)
    else:
        dist.all_to_all_single(out, inp, out_split, in_split, group=group)


class CudaOps:
    """The product steps: this package's kernels through the C-ABI."""

    def sort(self, keys, vals, buffer_fraction: float = 1.0, workspace=None):
        gns.sort_(keys, vals, buffer_fraction, workspace=workspace)
        return keys, vals

    def workspace_bytes(self, n, buffer_fraction, with_vals):
        return gns.workspace_bytes(n, buffer_fraction, with_vals)

    def cuts(self, sorted_keys, spl_keys, spl_rank, spl_pos, my_rank):
        return gns.split_cuts(sorted_keys, spl_keys, spl_rank, spl_pos, my_rank)

    def merge_two(self, a_k, a_v, b_k, b_v):
        return gns.merge_two(a_k, a_v, b_k, b_v)

    def merge_into(self, a_k, a_v, b_k, b_v, d_k, d_v):
        gns.merge_two(a_k, a_v, b_k, b_v, out=(d_k, d_v))


def _sample_positions(n: int, s: int) -> List[int]:
    """s regularly spaced positions of a shard of n elements (none if empty)."""
    if n == 0:
        return []
    return [(j * n) // s for j in range(s)]


def choose_splitters(torch, all_keys, all_rank, all_pos, k: int, ops):
    """Splitters from the all-gathered samples (rank-major, positions
    ascending within a rank): a stable key sort orders them by
    (key, rank, position); every (V/k)-th triple is a splitter."""
    V = all_keys.numel()
    if k <= 1 or V == 0:
        return all_keys[:0], all_rank[:0], all_pos[:0]
    idx = torch.arange(V, dtype=torch.int64, device=all_keys.device).to(torch.uint32)
    sk = all_keys.clone()
    sk, idx = ops.sort(sk, idx)
    pick = torch.tensor([(i * V) // k for i in range(1, k)], dtype=torch.int64, device=all_keys.device)
    order = idx.to(torch.int64)[pick]
    return sk[pick], all_rank[order], all_pos[order]


def merge_runs(runs, ops):
    """Pairwise tree merge of sorted runs given in rank order (left wins ties)."""
    runs = [r for r in runs if r[0].numel() > 0] or runs[:1]
    while len(runs) > 1:
        nxt = []
        for i in range(0, len(runs) - 1, 2):
            (ak, av), (bk, bv) = runs[i], runs[i + 1]
            nxt.append(ops.merge_two(ak, av, bk, bv))
        if len(runs) % 2:
            nxt.append(runs[-1])
        runs = nxt
    return runs[0]


def _proposals(torch, keys, lo, hi, s):
    """s positions evenly spaced in each window [lo_g, hi_g) of this rank's
    sorted keys (positions past an empty window are marked invalid)."""
    dev = keys.device
    j = torch.arange(1, s + 1, dtype=torch.int64, device=dev)
    span = (hi - lo).clamp(min=0)
    pos = lo[:, None] + (span[:, None] * j[None, :]) // (s + 1)
    valid = (span[:, None] > 0) & (pos < hi[:, None])
    pos = torch.where(valid, pos, torch.zeros_like(pos))
    key = keys[pos.clamp(max=max(keys.numel() - 1, 0))] if keys.numel() else torch.zeros(pos.shape, dtype=keys.dtype,
                                                                                            device=dev)
    return pos, key, valid


def _narrow(torch, lo, hi, R, cand_rank, cand_pos, valid, mine, C, me):
    """Window update of this rank from the global counts C of every proposal
    (targets x proposals): x with C(x) < R is among the first R elements (cut
    >= its count here, +1 if this rank owns it), else the cut <= its count."""
    inside = valid & (C < R[:, None])
    own = (cand_rank == me).to(torch.int64)
    big = torch.iinfo(torch.int64).max
    lo_new = torch.where(inside, mine + own * inside.to(torch.int64), torch.full_like(mine, -1)).amax(dim=1)
    hi_new = torch.where(valid & ~inside, mine, torch.full_like(mine, big)).amin(dim=1)
    return torch.maximum(lo, lo_new), torch.minimum(hi, hi_new)


def _count(torch, ops, keys, ck, cr, cp, cv, me):
    """This rank's count of elements preceding every proposal (0 for invalid
    ones -- they are counted like the others and masked, so no host round
    trip decides which to count); ck holds the proposals' keys as int64 bit
    patterns."""
    c = ops.cuts(keys, ck.reshape(-1).contiguous().view(keys.dtype), cr.reshape(-1).contiguous(),
                 cp.reshape(-1).contiguous(), me)
    return (c.to(torch.int64) * cv.reshape(-1).to(torch.int64)).reshape(ck.shape)


def _rounds_bound(n_max: int, s: int) -> int:
    """Rounds after which every window has collapsed: each round splits a
    window into s + 1 parts (plus one round of slack for the owner's +1)."""
    r, w = 0, max(1, n_max) + 1
    while w > 1:
        w = -(-w // (s + 1))
        r += 1
    return r + 2


def exact_cuts(keys, k, me, group, samples, ops):
    """Cuts of this rank's sorted shard at global stable ranks g N / k,
    g = 1..k-1 (collective over ``group``).  The rounds stay on the device:
    one all-reduce of the shard sizes (sum and max) fixes their number, one
    check at the end confirms convergence."""
    import torch
    import torch.distributed as dist
    dev = keys.device
    n = keys.numel()
    nt = torch.tensor([n, n], dtype=torch.int64, device=dev)
    _all_reduce(nt[:1], group=group)
    _all_reduce(nt[1:], op=dist.ReduceOp.MAX, group=group)
    N, n_max = (int(x) for x in nt.cpu())
    R = torch.tensor([(g * N) // k for g in range(1, k)], dtype=torch.int64, device=dev)
    lo = torch.zeros(k - 1, dtype=torch.int64, device=dev)
    hi = torch.full((k - 1,), n, dtype=torch.int64, device=dev)
    s = max(1, samples)
    bound = _rounds_bound(n_max, s)
    for it in range(64):
        pos, key, valid = _proposals(torch, keys, lo, hi, s)
        # every rank's proposals: (key bits, position, valid) gathered in rank order
        kb = key.contiguous().view(torch.int64)                    # 8-byte patterns of any key type
        gk = [torch.empty_like(kb) for _ in range(k)]
        gp = [torch.empty_like(pos) for _ in range(k)]
        gvl = [torch.empty_like(pos) for _ in range(k)]
        _all_gather(gk, kb, group=group)
        _all_gather(gp, pos.contiguous(), group=group)
        _all_gather(gvl, valid.to(torch.int64).contiguous(), group=group)
        ck = torch.stack(gk, dim=1).reshape(k - 1, k * s)          # target x (rank, j)
        cp = torch.stack(gp, dim=1).reshape(k - 1, k * s)
        cv = torch.stack(gvl, dim=1).reshape(k - 1, k * s).bool()
        cr = torch.arange(k, dtype=torch.int32, device=dev).repeat_interleave(s).repeat(k - 1, 1)
        mine = _count(torch, ops, keys, ck, cr, cp, cv, me)
        # global counts of every proposal, plus the windows' lower ends
        red = torch.cat([mine.reshape(-1), lo])
        _all_reduce(red, group=group)
        C = red[:mine.numel()].reshape(k - 1, k * s)
        if it + 1 >= bound and bool((red[mine.numel():] == R).all()):   # (host check only past the bound)
            break
        lo, hi = _narrow(torch, lo, hi, R, cr, cp, cv, mine, C, me)
    else:
        raise RuntimeError("exact_cuts did not converge")
    return lo


def sort_distributed(keys, vals=None, group=None, samples: int = 64, ops=None, balanced: bool = True,
                     buffer_fraction: float = 1.0, workspace=None, info: Optional[dict] = None
                     ) -> Tuple[object, Optional[object]]:
    """Stable sort of the rank-major concatenation of every rank's
    (keys, vals) shard.  Returns this rank's piece of the sorted array: with
    ``balanced`` exactly global ranks [g N / k, (g+1) N / k) on rank g, else
    the piece between sample splitters.  keys: float64 / int64 / uint64 (CUDA
    for the default ops); vals: uint32 or None.  Collective: every rank of
    ``group`` must call it.

    Footprint: ``keys``/``vals`` are sorted in place (their contents are
    consumed) with ``buffer_fraction`` (1.0 or <= 0.5) and the optional
    caller ``workspace``; the returned piece lives in one receive buffer or in
    the shard's own memory (when the tree's last merge lands there).  If
    ``info`` is a dict it receives the per-phase bytes and %RAM of this rank."""
    import torch
    import torch.distributed as dist
    ops = ops or CudaOps()
    k = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = keys.device
    n = keys.numel()
    s_el = keys.element_size() + (vals.element_size() if vals is not None else 0)
    ws_bytes = 0
    sized = hasattr(ops, "workspace_bytes")
    if workspace is None and sized and n > 1:
        ws_bytes = ops.workspace_bytes(n, buffer_fraction, vals is not None)
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    elif workspace is not None:
        ws_bytes = workspace.numel() * workspace.element_size()
    # 1. local stable sort of the shard, in place
    if sized:
        keys, vals = ops.sort(keys, vals, buffer_fraction, workspace)
    else:
        keys, vals = ops.sort(keys, vals)
    del workspace                                   # (the local sort's buffer is free from here on)
    if info is not None:
        info.update(shard_bytes=n * s_el, sort_buffer_bytes=ws_bytes,
                    ram_pct_sort=1.0 + (ws_bytes / (n * s_el) if n else 0.0))
    if k == 1:
        if info is not None:
            info.update(recv_bytes=0, partner_bytes=0, ram_pct_exchange=1.0, ram_pct_peak=info["ram_pct_sort"])
        return keys, vals
    if balanced:
        cuts = exact_cuts(keys, k, me, group, samples, ops)
        return _exchange_and_merge(torch, dist, keys, vals, cuts, n, k, group, ops, info, s_el)
    # 2. samples -> splitters (every rank contributes exactly `samples` slots;
    # an empty shard marks its slots invalid)
    pos = _sample_positions(n, samples)
    valid = torch.zeros(samples, dtype=torch.int64, device=dev)
    s_pos = torch.zeros(samples, dtype=torch.int64, device=dev)
    s_key = torch.zeros(samples, dtype=keys.dtype, device=dev)
    if pos:
        p = torch.tensor(pos, dtype=torch.int64, device=dev)
        valid[:] = 1
        s_pos[:] = p
        s_key[:] = keys[p]
    g_key = [torch.empty_like(s_key) for _ in range(k)]
    g_pos = [torch.empty_like(s_pos) for _ in range(k)]
    g_val = [torch.empty_like(valid) for _ in range(k)]
    _all_gather([g.view(torch.int64) for g in g_key], s_key.view(torch.int64), group=group)   # 8-byte patterns
    _all_gather(g_pos, s_pos, group=group)
    _all_gather(g_val, valid, group=group)
    a_key = torch.cat(g_key)
    a_pos = torch.cat(g_pos)
    a_rank = torch.arange(k, dtype=torch.int32, device=dev).repeat_interleave(samples)
    m = torch.cat(g_val).bool()
    spl_key, spl_rank, spl_pos = choose_splitters(torch, a_key[m], a_rank[m], a_pos[m], k, ops)
    # 3. cuts -> send counts
    if spl_key.numel():
        cuts = ops.cuts(keys, spl_key.contiguous(), spl_rank.contiguous(), spl_pos.contiguous(), me)
    else:
        cuts = torch.zeros(k - 1, dtype=torch.int64, device=dev)
    return _exchange_and_merge(torch, dist, keys, vals, cuts, n, k, group, ops, info, s_el)


def _exchange_and_merge(torch, dist, keys, vals, cuts, n, k, group, ops, info=None, s_el=8):
    """Steps 4-5: one all-to-all-v of the pieces between the cuts into ONE
    receive buffer, then the merge of the k received runs in rank order,
    ping-ponging between that buffer and the shard's own memory (dead after
    the exchange) when it is large enough (balanced equal shards), else a
    second buffer."""
    dev = keys.device
    edges = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), cuts.to(torch.int64),
                       torch.full((1,), n, dtype=torch.int64, device=dev)])
    send = (edges[1:] - edges[:-1]).contiguous()
    recv = torch.empty_like(send)
    _all_to_all_single(recv, send, group=group)
    sr = torch.cat([send, recv]).cpu()                     # (the split sizes are host arguments of NCCL)
    send_l = [int(x) for x in sr[:k]]
    recv_l = [int(x) for x in sr[k:]]
    m = sum(recv_l)
    # 4. one all-to-all-v of keys (and vals) into one receive buffer
    out_k = torch.empty(m, dtype=keys.dtype, device=dev)
    # (keys move as their 64-bit patterns: every key type is 8 bytes)
    _all_to_all_single(out_k.view(torch.int64), keys.view(torch.int64), recv_l, send_l, group=group)
    out_v = None
    if vals is not None:
        out_v = torch.empty(m, dtype=vals.dtype, device=dev)
        # (uint32 is not an NCCL type: move the payload as int32 bits)
        _all_to_all_single(out_v.view(torch.int32), vals.view(torch.int32), recv_l, send_l, group=group)
    # 5. merge the k received runs in rank order; partner = the shard's memory
    extra = 0
    runs, o = [], 0
    for c in recv_l:
        runs.append((o, c))
        o += c
    runs = [r for r in runs if r[1] > 0] or [(0, 0)]
    if hasattr(ops, "merge_into"):
        if n >= m:
            pk, pv = keys[:m], (None if vals is None else vals[:m])
        else:
            pk = torch.empty(m, dtype=keys.dtype, device=dev)
            pv = None if vals is None else torch.empty(m, dtype=vals.dtype, device=dev)
            extra = m * s_el
        where = merge_tree_pingpong(torch, [(out_k, out_v), (pk, pv)], runs, ops)
        rk, rv = ((out_k, out_v) if where == 0 else (pk, pv))
    else:   # (test ops without merge_into: tree of merge_two)
        rk, rv = merge_runs([(out_k[a:a + c], None if out_v is None else out_v[a:a + c]) for a, c in runs], ops)
    if info is not None:
        info.update(recv_bytes=m * s_el, partner_bytes=extra,
                    ram_pct_exchange=1.0 + ((m * s_el + extra) / (n * s_el) if n else 0.0))
        info["ram_pct_peak"] = max(info["ram_pct_sort"], info["ram_pct_exchange"])
    return rk.contiguous(), (None if rv is None else rv.contiguous())


def merge_tree_pingpong(torch, bufs, runs, ops):
    """Pairwise tree merge of consecutive sorted runs (rank order, left wins
    ties) that lie back to back in bufs[0] (runs = [(offset, length)]),
    ping-ponging between the two equally large buffers bufs[0], bufs[1]
    (each a (keys, vals-or-None) pair): level by level, runs 2i and 2i+1 are
    merged into the other buffer at the same offset; an unpaired last run is
    copied across.  Returns the index of the buffer holding the result."""
    cur = 0
    while len(runs) > 1:
        (xk, xv), (yk, yv) = bufs[cur], bufs[1 - cur]
        nxt = []
        for i in range(0, len(runs), 2):
            if i + 1 < len(runs):
                (oa, la), (ob, lb) = runs[i], runs[i + 1]
                ops.merge_into(xk[oa:oa + la], None if xv is None else xv[oa:oa + la],
                               xk[ob:ob + lb], None if xv is None else xv[ob:ob + lb],
                               yk[oa:oa + la + lb], None if yv is None else yv[oa:oa + la + lb])
                nxt.append((oa, la + lb))
            else:
                o, ln = runs[i]
                yk[o:o + ln].copy_(xk[o:o + ln])
                if yv is not None:
                    yv[o:o + ln].copy_(xv[o:o + ln])
                nxt.append((o, ln))
        runs = nxt
        cur = 1 - cur
    return cur


def simulate_exact_cuts(torch, keys_list, samples, ops):
    """exact_cuts for k shards in one process (the all-gather and all-reduce
    are concatenations and sums): every shard's k-1 cuts."""
    k = len(keys_list)
    dev = keys_list[0].device
    N = sum(x.numel() for x in keys_list)
    R = torch.tensor([(g * N) // k for g in range(1, k)], dtype=torch.int64, device=dev)
    lo = [torch.zeros(k - 1, dtype=torch.int64, device=dev) for _ in range(k)]
    hi = [torch.full((k - 1,), x.numel(), dtype=torch.int64, device=dev) for x in keys_list]
    s = max(1, samples)
    for _ in range(64):
        props = [_proposals(torch, keys_list[r], lo[r], hi[r], s) for r in range(k)]
        ck = torch.stack([p[1].contiguous().view(torch.int64) for p in props], dim=1).reshape(k - 1, k * s)
        cp = torch.stack([p[0] for p in props], dim=1).reshape(k - 1, k * s)
        cv = torch.stack([p[2] for p in props], dim=1).reshape(k - 1, k * s)
        cr = torch.arange(k, dtype=torch.int32, device=dev).repeat_interleave(s).repeat(k - 1, 1)
        mine = [_count(torch, ops, keys_list[r], ck, cr, cp, cv, r) for r in range(k)]
        C = sum(mine)
        if bool((sum(lo) == R).all()):
            break
        for r in range(k):
            lo[r], hi[r] = _narrow(torch, lo[r], hi[r], R, cr, cp, cv, mine[r], C, r)
    else:
        raise RuntimeError("exact_cuts did not converge")
    return lo


def simulate(shards, samples: int = 64, ops=None, balanced: bool = True):
    """The same steps for k shards in ONE process (no collectives: the
    all-gather and all-to-all are tensor concatenations / slices), for
    validating the kernels of the distributed path on a single GPU.  Returns
    the k output pieces."""
    import torch
    ops = ops or CudaOps()
    k = len(shards)
    srt = []
    for kk, vv in shards:
        kk = kk.clone()
        vv = None if vv is None else vv.clone()
        srt.append(ops.sort(kk, vv))
    if k == 1:
        return srt
    dev = srt[0][0].device
    if balanced:
        cuts = simulate_exact_cuts(torch, [kk for kk, _ in srt], samples, ops)
        pieces = []
        for r, (kk, vv) in enumerate(srt):
            e = [0] + [int(x) for x in cuts[r].cpu()] + [kk.numel()]
            pieces.append([(kk[e[j]:e[j + 1]], None if vv is None else vv[e[j]:e[j + 1]]) for j in range(k)])
        return [merge_runs([pieces[r][j] for r in range(k)], ops) for j in range(k)]
    a_key, a_pos, a_rank = [], [], []
    for r, (kk, _) in enumerate(srt):
        pos = _sample_positions(kk.numel(), samples)
        if pos:
            p = torch.tensor(pos, dtype=torch.int64, device=dev)
            a_key.append(kk[p])
            a_pos.append(p)
            a_rank.append(torch.full((len(pos),), r, dtype=torch.int32, device=dev))
    spl_key, spl_rank, spl_pos = choose_splitters(torch, torch.cat(a_key), torch.cat(a_rank), torch.cat(a_pos),
                                                  k, ops)
    pieces = []            # pieces[src][dst]
    for r, (kk, vv) in enumerate(srt):
        n = kk.numel()
        cuts = ops.cuts(kk, spl_key.contiguous(), spl_rank.contiguous(), spl_pos.contiguous(), r)
        e = [0] + [int(x) for x in cuts.cpu()] + [n]
        pieces.append([(kk[e[j]:e[j + 1]], None if vv is None else vv[e[j]:e[j + 1]]) for j in range(k)])
    out = []
    for j in range(k):
        runs = [pieces[r][j] for r in range(k)]
        out.append(merge_runs(runs, ops))
    return out
