"""Small runs of every kernel family for compute-sanitizer (development aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_1206_0115_b200 as P
from oracles import Oracle
from paper_1206_0115_b200.distributed import build_distributed_emulated, evaluate_partitioned

cache5 = "tests/golden/m2l_l5.bin"
for (n, h, l, dist) in [(20000, 4, 5, "uniform"), (30000, 5, 7, "uniform"), (15000, 6, 4, "ellipsoid"),
                        (4000, 12, 3, "uniform")]:
    xyzw = Oracle.generate_particles(n, dist, 3)
    c = P.FmmContext(None, order=l, m2l_cache=cache5 if l == 5 else None)
    c.build_tree(xyzw, h)
    for mode in (0, 1):
        c.set_p2p_mode(mode)
        c.evaluate()
    c.build_lists()
    c.gather()
    print("ok", n, h, l, dist, flush=True)
    c.close()
xyzw = Oracle.generate_particles(20000, "uniform", 5)
xyzw[:300, :3] = 0.3 + 0.001 * np.random.default_rng(1).random((300, 3))  # one big leaf
c = P.FmmContext(None, order=5, m2l_cache=cache5)
c.build_tree(xyzw, 4)
c.evaluate()
c.close()
ctxs = [P.FmmContext(None, order=5, m2l_cache=cache5) for _ in range(3)]
build_distributed_emulated(ctxs, [xyzw[:5000], xyzw[5000:5000], xyzw[5000:]], 4)
evaluate_partitioned(ctxs)
print("ok dist", flush=True)
