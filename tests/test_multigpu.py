"""Multi-GPU path: contiguous Morton ranges of leaves, one multipole
exchange per upward level (all-gather at the alignment level, per-peer halo below),
owner-computes downward pass.

* CPU: the balanced contiguous split (fmmgpu_plan_partition, host-only), and the
  exchange steps with real torch.distributed processes (gloo, world size 2): the
  all-gather of owned rows and the point-to-point halo step.
* GPU (one device): N partitioned contexts emulate N ranks through the stepped API and
  the library's exchange plan; the per-rank fields must partition the particles and
  their sum must equal the oracle (<= 1e-12) and the unpartitioned evaluation
  (<= 1e-13). Two real processes (both on the one device) run the library over gloo.
"""
import os
import socket

import numpy as np
import pytest

from oracles import Oracle, OracleOps, OracleTree, force_error, relative_l2_error

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1206_0115_b200", "libfmmgpu.so")
needs_lib = pytest.mark.skipif(not os.path.exists(LIB), reason="libfmmgpu.so not built")


@needs_lib
@pytest.mark.parametrize("nranks", [1, 2, 3, 8, 13])
def test_plan_partition_balanced_and_contiguous(nranks):
    import paper_1206_0115_b200 as P
    rng = np.random.default_rng(nranks)
    w = rng.integers(1, 1000, size=500).astype(np.uint64)
    b = P.plan_partition(w, nranks)
    assert b[0] == 0 and b[-1] == len(w) and np.all(np.diff(b.astype(np.int64)) >= 0)
    loads = [int(w[b[r]:b[r + 1]].sum()) for r in range(nranks)]
    assert sum(loads) == int(w.sum())
    # every rank within one item of the ideal share
    ideal = w.sum() / nranks
    assert max(abs(x - ideal) for x in loads) <= w.max()
    # degenerate inputs
    assert list(P.plan_partition(np.zeros(0, np.uint64), nranks)) == [0] * (nranks + 1)
    e = P.plan_partition(np.ones(3, np.uint64), nranks)
    assert e[-1] == 3 and np.all(np.diff(e.astype(np.int64)) >= 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import paper_1206_0115_b200 as P
        from paper_1206_0115_b200.distributed import exchange_segments
        # both ranks derive the same split from the same (replicated) weights
        w = (np.arange(1, 101) ** 2).astype(np.uint64)
        b = P.plan_partition(w, world)
        plans = [None] * world
        dist.all_gather_object(plans, b.tolist())
        assert all(p == b.tolist() for p in plans)
        # each rank computed only its owned rows of a level (others stale/zero)
        full_ref = np.arange(100 * 7, dtype=np.float64).reshape(100, 7)
        local = np.zeros_like(full_ref)
        local[b[rank]:b[rank + 1]] = full_ref[b[rank]:b[rank + 1]]

        def gather(seg):
            out = [None] * world
            dist.all_gather_object(out, seg)
            return out

        got = exchange_segments(local, b, rank, gather)
        q.put((rank, bool(np.array_equal(got, full_ref))))
    finally:
        dist.destroy_process_group()


def _gloo_halo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import torch
        from paper_1206_0115_b200.distributed import exchange_halo
        full_ref = np.arange(50 * 3, dtype=np.float64).reshape(50, 3) + 1
        own = [np.arange(0, 25), np.arange(25, 50)]
        local = np.zeros_like(full_ref)
        local[own[rank]] = full_ref[own[rank]]
        peer = 1 - rank
        # rank r needs these cells of its peer (the halo), ascending
        need = [np.array([25, 26, 30, 49]), np.array([0, 3, 24])]
        plans = [None, None]
        plans[peer] = (need[peer], need[rank])
        plans[rank] = (np.zeros(0, int), np.zeros(0, int))

        def sendrecv(p, rows, n_recv):
            buf = torch.zeros(n_recv, rows.shape[1], dtype=torch.float64)
            reqs = [dist.isend(torch.from_numpy(rows), p), dist.irecv(buf, p)]
            for r in reqs:
                r.wait()
            return buf.numpy()

        got = exchange_halo(local, plans, rank, sendrecv)
        expect = local.copy()
        expect[need[rank]] = full_ref[need[rank]]
        q.put((rank, bool(np.array_equal(got, expect))))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_with_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_halo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


@needs_lib
def test_exchange_with_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


CASES = [(20000, 5, 5, "uniform", 42), (12000, 5, 4, "sphere", 3), (30000, 6, 3, "uniform", 7)]


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_h{c[1]}_l{c[2]}_{c[3]}" for c in CASES])
def test_partitioned_evaluation_emulated(nranks, case):
    import paper_1206_0115_b200 as P
    from paper_1206_0115_b200.distributed import evaluate_partitioned
    n, h, l, dist, seed = case
    xyzw = Oracle.generate_particles(n, dist, seed)
    xyzw[:, 3] = 0.5 + np.random.default_rng(seed).random(n)
    full = P.FmmContext(None, order=l)
    full.build_tree(xyzw, h)
    full.evaluate()
    g_full = full.gather()
    ctxs = []
    for r in range(nranks):
        c = P.FmmContext(None, order=l)
        c.build_tree(xyzw, h)
        c.partition(r, nranks)
        ctxs.append(c)
    info = ctxs[0].partition_info()
    align = info["align_level"]
    kinds = [ctxs[0].exchange_plan(v, 0)[0] for v in range(h)]
    assert all(k == 0 for k in kinds[:max(2, align)]) and all(k in (1, 2) for k in kinds[max(2, align):])
    assert 2 in kinds  # the levels below the alignment level move only their halo
    outs = evaluate_partitioned(ctxs)
    # owned particles partition the set: each particle is nonzero on exactly one rank
    slots = [c.partition_info()["slots"] for c in ctxs]
    assert slots[0][0] == 0 and slots[-1][1] == n
    assert all(slots[r][1] == slots[r + 1][0] for r in range(nranks - 1))
    nz = sum((np.abs(o[0]) > 0).astype(int) for o in outs)
    assert np.all(nz == 1)
    g = [sum(o[k] for o in outs) for k in range(4)]
    assert relative_l2_error(g[0], g_full[0]) <= 1e-13
    assert force_error(*g[1:], *g_full[1:]) <= 1e-13
    ref = OracleTree(xyzw, h).evaluate(OracleOps.cached(l))
    assert relative_l2_error(g[0], ref[0]) <= 1e-12
    assert force_error(*g[1:], *ref[1:]) <= 1e-12
    # nranks = 1 restores the full evaluation on the same context
    ctxs[0].partition(0, 1)
    ctxs[0].evaluate()
    g1 = ctxs[0].gather()
    assert relative_l2_error(g1[0], g_full[0]) == 0.0
    for c in ctxs + [full]:
        c.close()


def _library_rank(rank, world, port, case, q):
    """One rank of a real 2-process run of the library (both processes on device 0):
    whole tree, partition(rank, world), stepped evaluation with the exchange over gloo."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import torch
        import paper_1206_0115_b200 as P
        from paper_1206_0115_b200.distributed import evaluate_rank, exchange_bytes
        n, h, l, dist_name, seed = case
        xyzw = Oracle.generate_particles(n, dist_name, seed)
        xyzw[:, 3] = 0.5 + np.random.default_rng(seed).random(n)
        c = P.FmmContext(None, order=l)
        c.build_tree(xyzw, h)
        c.partition(rank, world)
        g = evaluate_rank(c, dist)
        s0, s1 = c.partition_info()["slots"]
        # the fields of all ranks summed on every rank (each particle is owned once)
        tot = torch.from_numpy(np.stack(g))
        dist.all_reduce(tot)
        q.put((rank, tot.numpy(), exchange_bytes(c, world), (s0, s1)))
        c.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [(30000, 5, 5, "uniform", 11), (20000, 6, 4, "ellipsoid", 5)],
                         ids=["n30000_h5_l5_uniform", "n20000_h6_l4_ellipsoid"])
def test_two_processes_run_the_library_over_gloo(case):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_library_rank, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, tot, nbytes, slots = q.get(timeout=600)
        res[r] = (tot, nbytes, slots)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    n, h, l, dist_name, seed = case
    xyzw = Oracle.generate_particles(n, dist_name, seed)
    xyzw[:, 3] = 0.5 + np.random.default_rng(seed).random(n)
    ref = OracleTree(xyzw, h).evaluate(OracleOps.cached(l))
    for r in (0, 1):
        g = res[r][0]
        assert relative_l2_error(g[0], ref[0]) <= 1e-12
        assert force_error(*g[1:], *ref[1:]) <= 1e-12
    assert res[0][2][1] == res[1][2][0]  # the owned particle ranges meet
    assert res[0][1] > 0 and res[1][1] > 0  # something was exchanged


@pytest.mark.gpu
def test_halo_plan_smaller_than_allgather():
    """The halo exchange moves a fraction of the old whole-level all-gather (uniform
    cloud, 8 ranks), and every rank's receive list from p is p's send list to it."""
    import paper_1206_0115_b200 as P
    from paper_1206_0115_b200.distributed import exchange_bytes
    xyzw = Oracle.generate_particles(400000, "uniform", 3)
    h, l, nr = 6, 5, 8
    ctxs = []
    for r in range(nr):
        c = P.FmmContext(None, order=l)
        c.build_tree(xyzw, h)
        c.partition(r, nr)
        ctxs.append(c)
    ld = ((l ** 3 + 31) // 32) * 32
    a = ctxs[0].partition_info()["align_level"]
    allgather = sum((nr - 1) / nr * ctxs[0].level(v)[0].shape[0] * ld * 8 for v in range(max(2, a), h))
    for r, c in enumerate(ctxs):
        assert exchange_bytes(c, nr) < 0.3 * allgather
        for v in range(max(2, a), h):
            for p in range(nr):
                k, snd, rcv = c.exchange_plan(v, p)
                if k == 2 and p != r:
                    assert np.array_equal(rcv, ctxs[p].exchange_plan(v, r)[1])
    for c in ctxs:
        c.close()
