"""Bytes each rank receives in the distributed build (csrc/dist.cu) at config B, from
N rank contexts emulated on one device: the all-gathered Morton keys (8 B per particle
held by the other ranks) and the particle records of the rank's owned + halo leaves that
other ranks hold (32 B each), against replicating the input (32 B x N per rank).

    python tools/dist_input_volume.py [n] [height] > profiles/r02_dist_input_volume_B.json
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1206_0115_b200 as P  # noqa: E402
from paper_1206_0115_b200.distributed import build_distributed_emulated  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
h = int(sys.argv[2]) if len(sys.argv) > 2 else 7
xyzw = P.generate_particles(n, "uniform", 42)
rows = []
for N in (2, 4, 8):
    ctxs = [P.FmmContext(None, order=5) for _ in range(N)]
    b = [r * n // N for r in range(N + 1)]
    moved = build_distributed_emulated(ctxs, [xyzw[b[r]:b[r + 1]] for r in range(N)], h)
    owned = [int(np.diff(c.partition_info()["slots"])[0]) for c in ctxs]
    rows.append({"gpus": N, "records_received_per_rank": moved, "owned_particles_per_rank": owned,
                 "key_bytes_received_per_rank": [8 * (n - (b[r + 1] - b[r])) for r in range(N)],
                 "particle_bytes_received_per_rank": [32 * m for m in moved],
                 "replicated_input_bytes_per_rank": 32 * n,
                 "halo_fraction_of_owned": [m / o for m, o in zip(moved, owned)]})
    for c in ctxs:
        c.close()
print(json.dumps({"config": "B" if (n, h) == (10_000_000, 7) else f"n={n} h={h}", "n": n, "height": h,
                  "note": __doc__.split("\n\n")[0].replace("\n", " "), "rows": rows}, indent=1))
