"""CPU, world size 2 over gloo: the host protocol of the distributed input
(paper_1206_0115_b200.distributed.build_distributed_rank: all-gathers of bounds and keys,
OR of the flags, per-peer isend / irecv of particle records) against a numpy stand-in for
the library's fmmgpu_dist_* steps (csrc/dist.cu semantics: leaf keys, stable sort of
(key, input index), contiguous leaf ranges per rank, owned + 26-neighbour halo leaves).
The GPU tests (tests/test_dist_input.py) run the same protocol against the library."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class MockDistContext:
    """The fmmgpu_dist_* steps in numpy (small inputs only)."""

    def __init__(self):
        self.loc = None

    def dist_local(self, xyzw_local):
        self.loc = np.asarray(xyzw_local, dtype=np.float64).reshape(-1, 4)
        if len(self.loc) == 0:
            return np.array([np.inf] * 3 + [-np.inf] * 3)
        return np.concatenate([self.loc[:, :3].min(axis=0), self.loc[:, :3].max(axis=0)])

    def dist_keys(self, root, height):
        g = 1 << (height - 1)
        lo = root[:3] - 0.5 * root[3]
        cw = root[3] / g
        ijk = np.clip(np.floor((self.loc[:, :3] - lo) / cw), 0, g - 1).astype(np.int64)
        key = np.zeros(len(ijk), dtype=np.uint64)
        for b in range(height - 1):
            for a in range(3):
                key |= ((ijk[:, a] >> b) & 1).astype(np.uint64) << np.uint64(3 * b + 2 - a)
        self._g = g
        return key, 0

    def dist_build(self, keys_all, offsets, rank, nranks, height, group, root, flag):
        self.rank, self.nranks, self.off = rank, nranks, np.asarray(offsets, dtype=np.int64)
        order = np.argsort(keys_all, kind="stable")  # stable sort of (key, input index)
        self.ids = order
        skeys = keys_all[order]
        leaves, first = np.unique(skeys, return_index=True)
        self.leaf_of_slot = np.searchsorted(leaves, skeys)
        nl = len(leaves)
        b = [r * nl // nranks for r in range(nranks + 1)]
        owner = np.searchsorted(np.asarray(b[1:]), np.arange(nl), side="right")
        # decode leaf coordinates
        ijk = np.zeros((nl, 3), dtype=np.int64)
        for bit in range(height - 1):
            for a in range(3):
                ijk[:, a] |= ((leaves >> np.uint64(3 * bit + 2 - a)) & np.uint64(1)).astype(np.int64) << bit
        index = {tuple(x): i for i, x in enumerate(ijk)}
        need = np.zeros((nl, nranks), dtype=bool)
        for i, x in enumerate(ijk):
            need[i, owner[i]] = True
            for d in np.ndindex(3, 3, 3):
                q = index.get((x[0] + d[0] - 1, x[1] + d[1] - 1, x[2] + d[2] - 1))
                if q is not None:
                    need[i, owner[q]] = True
        self.need = need
        n = len(keys_all)
        self.pw = np.zeros((n, 4))
        src_rank = np.searchsorted(self.off[1:], self.ids, side="right")
        self.src_rank = src_rank
        mine = (src_rank == rank) & need[self.leaf_of_slot, rank]
        self.pw[mine] = self.loc[self.ids[mine] - self.off[rank]]

    def dist_plan(self, peer):
        send = np.nonzero((self.src_rank == self.rank) & self.need[self.leaf_of_slot, peer])[0]
        recv = np.nonzero((self.src_rank == peer) & self.need[self.leaf_of_slot, self.rank])[0]
        return send.astype(np.uint32), recv.astype(np.uint32)

    def dist_pack(self, peer):
        send, _ = self.dist_plan(peer)
        return self.loc[self.ids[send] - self.off[self.rank]]

    def dist_unpack(self, peer, records):
        _, recv = self.dist_plan(peer)
        self.pw[recv] = records

    def dist_check(self):
        return 0

    def dist_commit(self, flag):
        self.committed = True


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from test_dist_protocol import MockDistContext
        from paper_1206_0115_b200.distributed import build_distributed_rank
        rng = np.random.default_rng(7)
        xyzw = np.concatenate([rng.random((3000, 3)), np.ones((3000, 1))], axis=1)
        b = [0, 1100, 3000]  # uneven slices
        ctx = MockDistContext()
        root = np.array([0.5, 0.5, 0.5, 1.0])
        got = build_distributed_rank(ctx, xyzw[b[rank]:b[rank + 1]], 4, 250, dist, root=root)
        needed = ctx.need[ctx.leaf_of_slot, rank]
        ok = np.array_equal(ctx.pw[needed], xyzw[ctx.ids[needed]]) and np.all(ctx.pw[~needed] == 0)
        q.put((rank, bool(ok), int(got), int(needed.sum()), bool(getattr(ctx, "committed", False))))
    finally:
        dist.destroy_process_group()


def test_distributed_input_protocol_with_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, ok, got, needed, committed = q.get(timeout=300)
        res[r] = (ok, got, needed, committed)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for r in (0, 1):
        ok, got, needed, committed = res[r]
        assert ok and committed
        assert 0 < got < needed  # records from the peer: part of the owned + halo set
