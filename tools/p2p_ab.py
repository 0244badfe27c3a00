"""Mutual vs one-sided near field on one configuration (development aid):
python tools/p2p_ab.py [B|C|D|E|A]. Prints the isolated P2P time of each kernel, the
evaluation time with each, and the relative difference of their fields."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1206_0115_b200 as P  # noqa: E402

CFG = {"A": (100_000, "uniform", 4, 5), "B": (10_000_000, "uniform", 7, 5), "C": (10_000_000, "uniform", 7, 7),
       "D": (20_000_000, "ellipsoid", 8, 5), "E": (100_000_000, "uniform", 8, 5)}


def rel(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / np.sum(b ** 2)))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "B"
    n, dist, h, order = CFG[name]
    c = P.FmmContext(None, order=order)
    c.build_tree(P.generate_particles(n, dist, 42), h)
    res = {}
    for mode in (False, True):
        c.set_p2p_mode(mode)
        c.evaluate()
        c.evaluate()
        p2p = c.time_operator("P2P", -1, 3)
        total, kinds, _ = c.time_evaluations(5)
        c.evaluate()
        res[mode] = c.gather()
        print(f"[{name}] {'mutual ' if mode else 'onesided'}: P2P isolated {p2p:.3f} ms, evaluation {total / 5:.3f} ms",
              flush=True)
    a, b = res[False], res[True]
    f = lambda g: np.stack(g[1:], 1).ravel()  # noqa: E731
    print(f"[{name}] mutual vs onesided: potential {rel(b[0], a[0]):.3e} force {rel(f(b), f(a)):.3e}", flush=True)


if __name__ == "__main__":
    main()
