"""Host side of the multi-GPU path: one exchange per upward level.

Each rank owns a contiguous Morton range of cells per level (``FmmContext.partition``);
the exchange all-gathers every rank's owned segment of a level's multipoles (an
allgatherv). ``exchange_segments`` is that step on host arrays -- the same plan the
in-library NCCL path executes with one ncclBroadcast per rank -- and
``evaluate_partitioned`` drives the stepped API with a caller-supplied all-gather, so
the partitioned kernels can run with torch.distributed (gloo/nccl) plumbing or, for
tests, with N contexts emulating N ranks on one device.
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


def evaluate_partitioned(ctxs, levels_exchange) -> list:
    """Stepped partitioned evaluation of N rank contexts driven from one host process
    (single-device emulation): ``ctxs[r]`` is partitioned as rank r of len(ctxs).
    ``levels_exchange(v)`` tells whether level v is exchanged. Returns each rank's
    gathered fields (zero outside its owned particles)."""
    n = len(ctxs)
    height = ctxs[0].height
    for c in ctxs:
        c.reset()
    for v in range(height - 1, 1, -1):
        for c in ctxs:
            c.upward_level(v)
        if levels_exchange(v):
            begins = ctxs[0].partition_ranges(v)
            full = [c.expansion(v, 0) for c in ctxs]
            segs = [full[r][begins[r]:begins[r + 1]] for r in range(n)]
            for r, c in enumerate(ctxs):
                c.set_expansion(v, 0, exchange_segments(full[r], begins, r, lambda _s: segs))
    out = []
    for c in ctxs:
        c.downward()
        out.append(c.gather())
    return out
