"""Projected 1/2/4/8-GPU strong scaling of config B (and E) from one B200.

Every rank of the multi-GPU path (csrc/partition.cu, csrc/dist.cu) holds the
same tree (built from all-gathered keys) and evaluates only its owned Morton range of
leaves; the exchange after each upward level is the library's plan (all-gather at the
alignment level when needed, per-peer halo below). Without 8 GPUs, this times each rank's
partitioned evaluation on the one device (fmmgpu_set_measurement: the exchange is skipped
and the fields are refused) and adds the exchange volume the rank receives at an assumed
NVLink rate. Projection = max over ranks; it is an estimate, not a measurement of the
multi-GPU run. tree_build_ms_per_rank is the single-device build of the whole set.

    python tools/scaling_projection.py [config] > profiles/r01_scaling_projection.json
"""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_1206_0115_b200 as P  # noqa: E402
from paper_1206_0115_b200.distributed import exchange_bytes  # noqa: E402

CFG = {"B": (10_000_000, 7, 5), "E": (100_000_000, 8, 5)}
NVLINK_GBS = 600.0  # assumed achieved all-gather rate per GPU (NVLink 5: 900 GB/s per direction)

name = sys.argv[1] if len(sys.argv) > 1 else "B"
n, h, order = CFG[name]
c = P.FmmContext(None, order=order)
c.build_tree(P.generate_particles(n, "uniform", 42), h)
c.set_measurement(True)
for _ in range(2):
    c.evaluate()
t1, _, _ = c.time_evaluations(3)
t1 /= 3
tree_ms = c.timings()["TREE"]
rows = []
for N in (1, 2, 4, 8):
    per_rank = []
    xbytes = []
    for r in range(N):
        c.partition(r, N)
        for _ in range(2):
            c.evaluate()
        t, _, _ = c.time_evaluations(3)
        per_rank.append(t / 3)
        xbytes.append(exchange_bytes(c, N) if N > 1 else 0)
    gather_bytes = max(xbytes)
    c.partition(0, 1)
    exch_ms = gather_bytes / (NVLINK_GBS * 1e9) * 1e3
    proj = max(per_rank) + exch_ms
    rows.append({"gpus": N, "rank_ms": per_rank, "max_rank_ms": max(per_rank), "exchange_bytes_per_rank": xbytes,
                 "exchange_ms_at_%dGBs" % NVLINK_GBS: exch_ms, "projected_ms": proj,
                 "projected_mparticles_s": n / proj / 1e3, "efficiency": t1 / (N * proj)})
print(json.dumps({"config": name, "n": n, "height": h, "order": order, "single_gpu_eval_ms": t1,
                  "tree_build_ms_per_rank": tree_ms, "note": __doc__.split("\n\n")[1].replace("\n", " "),
                  "rows": rows}, indent=1))
