"""Distributed input of the multi-GPU path (halo particles; csrc/dist.cu).

Each rank holds only a slice of the input; only Morton keys are all-gathered and each
rank receives the particle records of its owned leaves and their 26-neighbour halo.

* the tree (every level's Cell array, block offsets, Morton order, ids, root cube) must
  be bit-exact with the single-device build of the whole set (geometry.cpp:73-161);
* each rank holds exactly the positions of its owned + halo leaves, and receives fewer
  records than the whole set;
* the partitioned evaluation over those particles equals the single-device evaluation
  (<= 1e-13) and the oracle (<= 1e-12);
* coincident particles held by different ranks raise domain_error on every rank;
* two real processes over gloo (both on the one device) build and evaluate.
"""
import os
import socket

import numpy as np
import pytest

from oracles import Oracle, OracleOps, OracleTree, force_error, relative_l2_error

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cloud(n, dist, seed):
    xyzw = Oracle.generate_particles(n, dist, seed)
    xyzw[:, 3] = 0.5 + np.random.default_rng(seed).random(n)
    return xyzw


def _slices(xyzw, nranks, seed):
    """Uneven contiguous slices in input order (one may be empty)."""
    n = len(xyzw)
    rng = np.random.default_rng(seed)
    cuts = np.sort(rng.integers(0, n, size=nranks - 1))
    if nranks > 2:
        cuts[1] = cuts[0]  # an empty slice
    b = np.concatenate([[0], cuts, [n]])
    return [xyzw[b[r]:b[r + 1]] for r in range(nranks)]


def _needed_slots(full, rank_ctx):
    """Morton slots of the owned leaves and their 26 neighbours (host restatement)."""
    cells, _ = full.level(full.height - 1)
    codes = cells["code"].astype(np.int64)
    first = cells["first_particle"].astype(np.int64)
    count = cells["particle_count"].astype(np.int64)
    b = rank_ctx.partition_ranges(full.height - 1)
    me = rank_ctx.partition_info()["rank"]
    own = set(range(int(b[me]), int(b[me + 1])))
    index = {int(c): i for i, c in enumerate(codes)}

    def demorton(c):
        ijk = [0, 0, 0]
        for bit in range(21):
            for a in range(3):
                ijk[a] |= ((c >> (3 * bit + 2 - a)) & 1) << bit
        return ijk

    def morton(i, j, k):
        c = 0
        for bit in range(21):
            c |= ((i >> bit) & 1) << (3 * bit + 2) | ((j >> bit) & 1) << (3 * bit + 1) | ((k >> bit) & 1) << (3 * bit)
        return c

    need = set()
    g = 1 << (full.height - 1)
    for c in own:
        i, j, k = demorton(int(codes[c]))
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    x, y, z = i + di, j + dj, k + dk
                    if 0 <= x < g and 0 <= y < g and 0 <= z < g:
                        q = index.get(morton(x, y, z))
                        if q is not None:
                            need.add(q)
    slots = np.zeros(full.n, dtype=bool)
    for q in need:
        slots[first[q]:first[q] + count[q]] = True
    return slots


CASES = [(20000, 5, 5, "uniform", 42), (15000, 6, 4, "ellipsoid", 5), (30000, 4, 3, "sphere", 9)]


@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_h{c[1]}_l{c[2]}_{c[3]}" for c in CASES])
def test_distributed_build_emulated(nranks, case):
    import paper_1206_0115_b200 as P
    from paper_1206_0115_b200.distributed import build_distributed_emulated, evaluate_partitioned
    n, h, l, dist, seed = case
    xyzw = _cloud(n, dist, seed)
    full = P.FmmContext(None, order=l)
    full.build_tree(xyzw, h)
    full.evaluate()
    g_full = full.gather()
    fx, fy, fz, fw, fid = full.particles()
    ctxs = [P.FmmContext(None, order=l) for _ in range(nranks)]
    moved = build_distributed_emulated(ctxs, _slices(xyzw, nranks, seed), h)
    for r, c in enumerate(ctxs):
        # tree bit-exact with the single-device build
        assert np.array_equal(c.root_cube(), full.root_cube())
        for v in range(h):
            a, ba = c.level(v)
            b, bb = full.level(v)
            assert np.array_equal(a, b) and np.array_equal(ba, bb), (r, v)
        x, y, z, w, ids = c.particles()
        assert np.array_equal(ids, fid)
        need = _needed_slots(full, c)
        for got, ref in ((x, fx), (y, fy), (z, fz), (w, fw)):
            assert np.array_equal(got[need], ref[need]), r
            assert np.all(got[~need] == 0)
        assert moved[r] < n  # halo, not the whole set
    outs = evaluate_partitioned(ctxs)
    g = [sum(o[k] for o in outs) for k in range(4)]
    assert relative_l2_error(g[0], g_full[0]) <= 1e-13
    assert force_error(*g[1:], *g_full[1:]) <= 1e-13
    ref = OracleTree(xyzw, h).evaluate(OracleOps.cached(l))
    assert relative_l2_error(g[0], ref[0]) <= 1e-12
    assert force_error(*g[1:], *ref[1:]) <= 1e-12
    # the distributed tree keeps its placement: another split is refused
    with pytest.raises(P.LogicError):
        ctxs[0].partition(0, 1)
    for c in ctxs + [full]:
        c.close()


def test_distributed_build_rejects_coincident_particles_across_ranks():
    import paper_1206_0115_b200 as P
    from paper_1206_0115_b200.distributed import build_distributed_emulated
    xyzw = _cloud(6000, "uniform", 1)
    xyzw[5500, :3] = xyzw[10, :3]  # same position, different slices
    ctxs = [P.FmmContext(None, order=3) for _ in range(2)]
    with pytest.raises(P.DomainError):
        build_distributed_emulated(ctxs, [xyzw[:3000], xyzw[3000:]], 4)
    # every rank refuses: the second context never committed and has no usable tree
    with pytest.raises(P.LogicError):
        ctxs[1].evaluate()
    for c in ctxs:
        c.close()


def test_distributed_build_explicit_root_outside_raises():
    import paper_1206_0115_b200 as P
    from paper_1206_0115_b200.distributed import build_distributed_emulated
    xyzw = _cloud(4000, "uniform", 2)
    ctxs = [P.FmmContext(None, order=3) for _ in range(2)]
    with pytest.raises(P.DomainError):
        build_distributed_emulated(ctxs, [xyzw[:2000], xyzw[2000:]], 4, root=[0.5, 0.5, 0.5, 0.5])
    for c in ctxs:
        c.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dist_rank(rank, world, port, case, q):
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
        from paper_1206_0115_b200.distributed import build_distributed_rank, evaluate_rank
        n, h, l, dist_name, seed = case
        xyzw = _cloud(n, dist_name, seed)
        b = [0, n // 3, n]  # uneven slices
        c = P.FmmContext(None, order=l)
        got = build_distributed_rank(c, xyzw[b[rank]:b[rank + 1]], h, 250, dist)
        g = evaluate_rank(c, dist)
        tot = torch.from_numpy(np.stack(g))
        dist.all_reduce(tot)
        q.put((rank, tot.numpy(), got))
        c.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(30000, 5, 5, "uniform", 11), (20000, 6, 4, "ellipsoid", 5)],
                         ids=["n30000_h5_l5_uniform", "n20000_h6_l4_ellipsoid"])
def test_two_processes_distributed_input_over_gloo(case):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_rank, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, tot, got = q.get(timeout=600)
        res[r] = (tot, got)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    n, h, l, dist_name, seed = case
    ref = OracleTree(_cloud(n, dist_name, seed), h).evaluate(OracleOps.cached(l))
    for r in (0, 1):
        g = res[r][0]
        assert relative_l2_error(g[0], ref[0]) <= 1e-12
        assert force_error(*g[1:], *ref[1:]) <= 1e-12
        assert 0 < res[r][1] < n  # halo records only


def test_nccl_distributed_build_single_rank():
    """The in-library NCCL path of the distributed build (fmmgpu_build_tree_distributed:
    bounds / keys / flags all-gathers as broadcast groups, per-peer record exchange,
    coincident check) on a one-rank communicator -- the only NCCL run one GPU allows --
    gives the single-device tree and fields bit for bit."""
    import paper_1206_0115_b200 as P
    xyzw = _cloud(30000, "uniform", 12)
    full = P.FmmContext(None, order=4)
    full.build_tree(xyzw, 5)
    full.evaluate()
    ref = full.gather()
    c = P.FmmContext(None, order=4)
    c.comm_init(P.comm_unique_id(), 1, 0)
    c.build_tree_distributed(xyzw, 5)
    for v in range(5):
        a, ba = c.level(v)
        b, bb = full.level(v)
        assert np.array_equal(a, b) and np.array_equal(ba, bb)
    c.evaluate()
    got = c.gather()
    for x, y in zip(got, ref):
        assert np.array_equal(x, y)
    # coincident particles are refused on every rank through the same path
    dup = xyzw.copy()
    dup[17, :3] = dup[4, :3]
    with pytest.raises(P.DomainError):
        c.build_tree_distributed(dup, 5)
    for x in (c, full):
        x.close()
