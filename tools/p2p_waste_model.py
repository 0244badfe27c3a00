"""Lane-work model of the P2P unit decomposition at config B (development aid).

Counts, from the real leaf occupancies of the config-B cloud, the lane-interactions the
P2P kernel executes per evaluation under two partial-pass schemes and compares them with
the useful directional interactions:
  * one partial pass per child with S = floor(32 / m) source splits (the previous kernel);
  * the partial pass cut into 16/8/4/2/1-target chunks, chunk 2^b split 32/2^b ways
    (csrc/p2p.cu).
Both include the group-of-4 padding of the staged runs. CPU only, ~1 min.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1206_0115_b200 as P  # noqa: E402  (host-side generator only)

G = 64
x = P.generate_particles(10_000_000, "uniform", 42)
lo, hi = x[:, :3].min(0), x[:, :3].max(0)
c, w = (lo + hi) / 2, (hi - lo).max() * (1 + 1e-6)
ijk = np.clip(np.floor((x[:, :3] - (c - w / 2)) / (w / G)).astype(int), 0, G - 1)
cnt = np.zeros((G, G, G), int)
np.add.at(cnt, (ijk[:, 0], ijk[:, 1], ijk[:, 2]), 1)
pad = np.pad(cnt, 1)


def padrow(r):  # csrc/p2p.cu neigh_meta: qc = 0 and 3 padded to 4, (qc = 1, 2) jointly
    return [(r[0] + 3) // 4 * 4, r[1], (r[1] + r[2] + 3) // 4 * 4 - r[1], (r[3] + 3) // 4 * 4]


def cost(chunks, runs):
    return sum(32 * 4 * sum((g + 32 // mm - 1) // (32 // mm) for g in runs) for mm in chunks)


useful = old = new = 0
for a in range(0, G, 2):
    for b in range(0, G, 2):
        for cc in range(0, G, 2):
            blk = pad[a:a + 4, b:b + 4, cc:cc + 4]
            padded = np.array([[padrow(blk[qa, qb, :]) for qb in range(4)] for qa in range(4)])
            for ca in (0, 1):
                for cb in (0, 1):
                    for cz in (0, 1):
                        nt = blk[1 + ca, 1 + cb, 1 + cz]
                        useful += nt * blk[ca:ca + 3, cb:cb + 3, cz:cz + 3].sum()
                        runs = [padded[ca + q // 3, cb + q % 3, cz:cz + 3].sum() // 4 for q in range(9)]
                        full = (nt // 32) * 32 * 4 * sum(runs)
                        m = nt % 32
                        old += full + (cost([32 // (32 // m)], runs) if m else 0)
                        new += full + (cost([1 << k for k in range(4, -1, -1) if m >> k & 1], runs) if m else 0)
print(f"useful {useful:.4e}; one partial pass: waste {100 * (old / useful - 1):.1f}%; "
      f"binary chunks: waste {100 * (new / useful - 1):.1f}%")
