"""Projected 1/2/4/8-GPU strong scaling of config B (and E) from one B200.

Every rank of the multi-GPU path (csrc/partition.cu) builds the whole
tree and evaluates only its owned Morton range of leaves; the one exchange is an
all-gather of each upward level's multipoles. Without 8 GPUs, this times each rank's
partitioned evaluation on the one device (FMMGPU_PART_NO_EXCHANGE=1: the all-gather is
skipped, so the fields are not used) and adds the all-gather volume at an assumed
NVLink rate. Projection = max over ranks; it is an estimate, not a measurement of the
multi-GPU run.

    python tools/scaling_projection.py [config] > profiles/r01_scaling_projection.json
"""
import json
import os
import sys

os.environ["FMMGPU_PART_NO_EXCHANGE"] = "1"
sys.path.insert(0, ".")
import paper_1206_0115_b200 as P  # noqa: E402

CFG = {"B": (10_000_000, 7, 5), "E": (100_000_000, 8, 5)}
NVLINK_GBS = 600.0  # assumed achieved all-gather rate per GPU (NVLink 5: 900 GB/s per direction)

name = sys.argv[1] if len(sys.argv) > 1 else "B"
n, h, order = CFG[name]
c = P.FmmContext(None, order=order)
c.build_tree(P.generate_particles(n, "uniform", 42), h)
for _ in range(2):
    c.evaluate()
t1, _, _ = c.time_evaluations(3)
t1 /= 3
tree_ms = c.timings()["TREE"]
rows = []
for N in (1, 2, 4, 8):
    per_rank = []
    gather_bytes = 0
    for r in range(N):
        c.partition(r, N)
        for _ in range(2):
            c.evaluate()
        t, _, _ = c.time_evaluations(3)
        per_rank.append(t / 3)
        if r == 0 and N > 1:
            info = c.partition_info()
            a = max(2, info["align_level"])
            ld = ((order ** 3 + 31) // 32) * 32  # round_up(l^3, 32), the padded row (csrc ldE)
            for v in range(a, h):
                cells = c.level(v)[0].shape[0]
                gather_bytes += (N - 1) / N * cells * ld * 8
    c.partition(0, 1)
    exch_ms = gather_bytes / (NVLINK_GBS * 1e9) * 1e3
    proj = max(per_rank) + exch_ms
    rows.append({"gpus": N, "rank_ms": per_rank, "max_rank_ms": max(per_rank), "allgather_bytes_per_rank": gather_bytes,
                 "allgather_ms_at_%dGBs" % NVLINK_GBS: exch_ms, "projected_ms": proj,
                 "projected_mparticles_s": n / proj / 1e3, "efficiency": t1 / (N * proj)})
print(json.dumps({"config": name, "n": n, "height": h, "order": order, "single_gpu_eval_ms": t1,
                  "tree_build_ms_per_rank": tree_ms, "note": __doc__.split("\n\n")[1].replace("\n", " "),
                  "rows": rows}, indent=1))
