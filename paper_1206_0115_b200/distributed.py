"""Host side of the multi-GPU path: one exchange per upward level.

Each rank owns a contiguous Morton range of cells per level (``FmmContext.partition``).
After the upward step of a partitioned level the library's plan
(``FmmContext.exchange_plan``, csrc/partition.cu) says what moves: kind 1 = every rank's
owned rows are all-gathered (the alignment level, when the replicated levels above it
run M2M), kind 2 = the halo -- each rank receives from each peer exactly the rows its
M2L reads. In-library NCCL does this inside ``evaluate`` (ncclBroadcast group /
ncclSend + ncclRecv per peer); the functions here run the same plan on host arrays:

* ``evaluate_partitioned`` -- N rank contexts driven from one process (single-device
  emulation, tests);
* ``evaluate_rank`` -- one process per rank with ``torch.distributed`` (gloo on CPU
  tensors: all_gather for kind 1, isend / irecv per peer for kind 2).
"""
from __future__ import annotations

import numpy as np


def exchange_segments(local: np.ndarray, begins: np.ndarray, rank: int, gather) -> np.ndarray:
    """All-gather the owned rows [begins[rank], begins[rank+1]) of ``local`` (cells x l^3).

    ``gather(segment) -> list of every rank's segment`` is the collective (e.g. a
    torch.distributed all_gather_object / padded all_gather); the result has every
    rank's rows in place and equals ``local`` on the caller's own rows."""
    seg = np.ascontiguousarray(local[begins[rank]:begins[rank + 1]])
    parts = gather(seg)
    out = np.array(local, copy=True)
    for r, part in enumerate(parts):
        assert part.shape[0] == begins[r + 1] - begins[r], (r, part.shape, begins)
        out[begins[r]:begins[r + 1]] = part
    return out


def exchange_halo(local: np.ndarray, plans, rank: int, sendrecv) -> np.ndarray:
    """Halo exchange of one level: ``plans[p] = (send_cells, recv_cells)`` with peer p;
    ``sendrecv(p, rows_to_send, n_recv) -> received rows`` is the point-to-point step.
    Received rows land in place; the caller's own rows are unchanged."""
    out = np.array(local, copy=True)
    for p, (snd, rcv) in enumerate(plans):
        if p == rank or (len(snd) == 0 and len(rcv) == 0):
            continue
        got = sendrecv(p, np.ascontiguousarray(local[snd]), len(rcv))
        if len(rcv):
            out[rcv] = got
    return out


def exchange_bytes(ctx, nranks: int) -> int:
    """Multipole bytes this rank receives per evaluation (kind 1 all-gather + kind 2 halo)."""
    total = 0
    ld = ((ctx.order ** 3 + 31) // 32) * 32  # padded row on the device (ldE)
    me = ctx.partition_info()["rank"]
    for v in range(2, ctx.height):
        kind = ctx.exchange_plan(v, 0)[0]
        if kind == 1:
            b = ctx.partition_ranges(v)
            total += (int(b[-1]) - int(b[me + 1] - b[me])) * ld * 8
        elif kind == 2:
            total += sum(len(ctx.exchange_plan(v, p)[2]) for p in range(nranks) if p != me) * ld * 8
    return total


def evaluate_partitioned(ctxs) -> list:
    """Stepped partitioned evaluation of N rank contexts driven from one host process
    (single-device emulation): ``ctxs[r]`` is partitioned as rank r of len(ctxs).
    Returns each rank's gathered fields (zero outside its owned particles)."""
    n = len(ctxs)
    height = ctxs[0].height
    for c in ctxs:
        c.reset()
    for v in range(height - 1, 1, -1):
        for c in ctxs:
            c.upward_level(v)
        kind = ctxs[0].exchange_plan(v, 0)[0]
        if kind == 0:
            continue
        full = [c.expansion(v, 0) for c in ctxs]
        if kind == 1:
            begins = ctxs[0].partition_ranges(v)
            segs = [full[r][begins[r]:begins[r + 1]] for r in range(n)]
            for r, c in enumerate(ctxs):
                c.set_expansion(v, 0, exchange_segments(full[r], begins, r, lambda _s: segs))
            continue
        for r, c in enumerate(ctxs):
            plans = [c.exchange_plan(v, p)[1:] for p in range(n)]

            def sendrecv(p, _rows, n_recv, r=r):
                snd_p = ctxs[p].exchange_plan(v, r)[1]  # what p sends to r
                assert np.array_equal(snd_p, plans[p][1]), (v, r, p)
                return full[p][snd_p]

            c.set_expansion(v, 0, exchange_halo(full[r], plans, r, sendrecv))
    out = []
    for c in ctxs:
        c.downward()
        out.append(c.gather())
    return out


def evaluate_rank(ctx, dist) -> list:
    """Stepped partitioned evaluation of this process's rank over ``torch.distributed``
    (CPU tensors: gloo). ``ctx`` is partitioned as dist.get_rank() of dist.get_world_size().
    Returns this rank's gathered fields (zero outside its owned particles)."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx.reset()
    for v in range(ctx.height - 1, 1, -1):
        ctx.upward_level(v)
        kind = ctx.exchange_plan(v, 0)[0]
        if kind == 0:
            continue
        local = ctx.expansion(v, 0)
        if kind == 1:
            begins = ctx.partition_ranges(v)
            width = local.shape[1]
            rows = int(max(begins[r + 1] - begins[r] for r in range(world)))

            def gather(seg):
                pad = torch.zeros(rows, width, dtype=torch.float64)
                pad[:seg.shape[0]] = torch.from_numpy(seg)
                parts = [torch.zeros_like(pad) for _ in range(world)]
                dist.all_gather(parts, pad)
                return [parts[r][:begins[r + 1] - begins[r]].numpy() for r in range(world)]

            ctx.set_expansion(v, 0, exchange_segments(local, begins, rank, gather))
            continue
        plans = [ctx.exchange_plan(v, p)[1:] for p in range(world)]
        reqs, bufs = [], {}
        for p in range(world):
            if p == rank:
                continue
            snd, rcv = plans[p]
            if len(snd):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(local[snd])), p))
            if len(rcv):
                bufs[p] = torch.zeros(len(rcv), local.shape[1], dtype=torch.float64)
                reqs.append(dist.irecv(bufs[p], p))
        for q in reqs:
            q.wait()
        out = np.array(local, copy=True)
        for p, b in bufs.items():
            out[plans[p][1]] = b.numpy()
        ctx.set_expansion(v, 0, out)
    ctx.downward()
    return ctx.gather()


# ---------------------------------------------------------------- distributed input
# Each rank holds one slice of the input (input order, slices in rank order); only the
# Morton keys are all-gathered, then each rank receives the particle records of its
# owned leaves and their 26-neighbour halo (csrc/dist.cu). The library does it over
# NCCL in one call (FmmContext.build_tree_distributed); these drive the same steps
# (fmmgpu_dist_*) with host collectives.

def _root(lohi_all, root):
    if root is not None:
        return np.ascontiguousarray(root, dtype=np.float64)
    from . import root_from_bounds
    g = np.concatenate([lohi_all[:, :3].min(axis=0), lohi_all[:, 3:6].max(axis=0)])
    return root_from_bounds(g)


def build_distributed_emulated(ctxs, slices, height: int, group_size: int = 250, root=None):
    """Distributed build of N rank contexts from one host process (single-device
    emulation): ``slices[r]`` is rank r's (n_r, 4) input slice. Raises like the library
    (every rank) when particles coincide. Returns the per-rank particle records received."""
    n = len(ctxs)
    lohi = np.stack([c.dist_local(s) for c, s in zip(ctxs, slices)])
    offsets = np.concatenate([[0], np.cumsum([len(s) for s in slices])]).astype(np.uint64)
    rt = _root(lohi, root)
    kf = [c.dist_keys(rt, height) for c in ctxs]
    keys = np.concatenate([k for k, _ in kf]) if offsets[-1] else np.zeros(0, np.uint64)
    flag = 0
    for _, f in kf:
        flag |= f
    for r, c in enumerate(ctxs):
        c.dist_build(keys, offsets, r, n, height, group_size, rt, flag)
    moved = [0] * n
    for r, c in enumerate(ctxs):
        for p in range(n):
            if p == r:
                continue
            rec = ctxs[p].dist_pack(r)  # what p sends to r
            assert len(rec) == len(c.dist_plan(p)[1]), (r, p)
            c.dist_unpack(p, rec)
            moved[r] += len(rec)
    cf = 0
    for c in ctxs:
        cf |= c.dist_check()
    for c in ctxs:
        c.dist_commit(cf)
    return moved


def build_distributed_rank(ctx, xyzw_local, height: int, group_size: int, dist, root=None) -> int:
    """Distributed build of this process's rank over ``torch.distributed`` (gloo, CPU
    tensors): all-gathers of the bounds and keys, isend / irecv of particle records per
    peer. Returns the number of particle records this rank received."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    lohi = ctx.dist_local(xyzw_local)
    nloc = len(np.asarray(xyzw_local).reshape(-1, 4))
    meta = torch.tensor(list(lohi) + [float(nloc)], dtype=torch.float64)
    parts = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(parts, meta)
    m = torch.stack(parts).numpy()
    counts = m[:, 6].astype(np.uint64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    rt = _root(m[:, :6], root)
    keys, flag = ctx.dist_keys(rt, height)
    width = int(counts.max()) if world else 0
    pad = torch.zeros(width, dtype=torch.int64)
    pad[:nloc] = torch.from_numpy(keys.view(np.int64))
    kparts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(kparts, pad)
    keys_all = np.concatenate([kparts[r][:int(counts[r])].numpy() for r in range(world)]).view(np.uint64)
    f = torch.tensor([flag], dtype=torch.int64)
    dist.all_reduce(f, op=dist.ReduceOp.MAX)
    ctx.dist_build(keys_all, offsets, rank, world, height, group_size, rt, int(f.item()))
    reqs, bufs = [], {}
    for p in range(world):
        if p == rank:
            continue
        snd, rcv = ctx.dist_plan(p)
        if len(snd):
            reqs.append(dist.isend(torch.from_numpy(ctx.dist_pack(p)), p))
        if len(rcv):
            bufs[p] = torch.zeros(len(rcv), 4, dtype=torch.float64)
            reqs.append(dist.irecv(bufs[p], p))
    for q in reqs:
        q.wait()
    for p, b in bufs.items():
        ctx.dist_unpack(p, b.numpy())
    cf = torch.tensor([ctx.dist_check()], dtype=torch.int64)
    dist.all_reduce(cf, op=dist.ReduceOp.MAX)
    ctx.dist_commit(int(cf.item()))
    return sum(len(b) for b in bufs.values())
