"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, built from
/root/reference/proj/src by oracle/build_ref.sh). Run in the dev container:

    python tests/golden/make_golden.py

The fixtures pin the CPU restatement (oracle/restate) wherever the reference
cannot be built (the GPU box has no /root/reference)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import Oracle, RefContext, RefLib  # noqa: E402

CONFIGS = [
    # name, n, height, order, dist, seed, random weights
    ("u2000_h3_l7", 2000, 3, 7, "uniform", 42, False),
    ("u10000_h4_l5", 10000, 4, 5, "uniform", 42, False),
    ("s5000_h5_l4", 5000, 5, 4, "sphere", 7, False),
    ("u3000_h4_l3_w", 3000, 4, 3, "uniform", 11, True),
]


def particles(n, dist, seed, rw):
    xyzw = Oracle.generate_particles(n, dist, seed)
    if rw:  # test_direct.cpp:15-21 style weights in [0.5, 1.5)
        rng = np.random.default_rng(seed)
        xyzw[:, 3] = 0.5 + rng.random(n)
    return xyzw


def main():
    assert RefLib.available(), "build oracle/_ref first (oracle/build_ref.sh)"
    for name, n, h, l, dist, seed, rw in CONFIGS:
        xyzw = particles(n, dist, seed, rw)
        ref = RefContext(xyzw, h, l)
        ref.execute(workers=1)
        pot, fx, fy, fz = ref.fields()
        out = {"n": n, "height": h, "order": l, "pot": pot, "fx": fx, "fy": fy, "fz": fz,
               "root": ref.root_cube(), "ranks": ref.ranks(), "xyzw": xyzw}
        out["ids"] = ref.particles()[4]
        for v in range(h):
            cells, bo = ref.level(v)
            cells["_pad"] = 0
            out[f"cells{v}"] = cells.view(np.uint8)
            out[f"blocks{v}"] = bo
        off, cells, ti, tot = ref.near()
        out["near_off"], out["near_cells"], out["task_interactions"], out["near_total"] = off, cells, ti, tot
        for v in range(2, h):
            t, s, vec, go = ref.far(v)
            out[f"far_t{v}"], out[f"far_s{v}"], out[f"far_v{v}"], out[f"far_g{v}"] = t, s, vec, go
        ref.save_m2l_cache(os.path.join(HERE, f"m2l_l{l}.bin"))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
