"""Which operator carries the force difference of the h=12 uniform case (development aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_1206_0115_b200 as P
from oracles import Oracle, OracleOps, OracleTree, RefContext, relative_l2_error, force_error

n, h, l, seed = int(sys.argv[1]) if len(sys.argv) > 1 else 12000, int(sys.argv[2]) if len(sys.argv) > 2 else 12, 4, 2
xyzw = Oracle.generate_particles(n, "uniform", seed)
ref = RefContext(xyzw, h, l)
ref.execute(workers=4)
rf = ref.fields()
cache = "/tmp/deep_ref.bin"
ref.save_m2l_cache(cache)
ot = OracleTree(xyzw, h)
ops = OracleOps(l, cache_path=cache)
of = ot.evaluate(ops)
print("oracle vs reference", relative_l2_error(of[0], rf[0]), force_error(*of[1:], *rf[1:]))
c = P.FmmContext(None, order=l)
c.load_m2l_cache(cache)
c.build_tree(xyzw, h)
for name, kinds, mask in (("near", {"P2P"}, 32), ("far", {"P2M", "M2M", "M2L", "L2L", "L2P"}, 31)):
    for mode in (0, 1):
        c.set_p2p_mode(mode)
        c.run_kinds(kinds)
        g = c.gather()
        o = ot.evaluate(ops, mask=mask)
        print(name, "p2p mode", mode, "vs oracle", relative_l2_error(g[0], o[0]), force_error(*g[1:], *o[1:]),
              "norms", np.linalg.norm(o[1]), flush=True)
c.set_p2p_mode(2)
c.evaluate()
g = c.gather()
print("full vs oracle", relative_l2_error(g[0], of[0]), force_error(*g[1:], *of[1:]))
print("full vs ref", relative_l2_error(g[0], rf[0]), force_error(*g[1:], *rf[1:]))
d = np.sqrt(sum((g[k] - rf[k]) ** 2 for k in (1, 2, 3)))
i = np.argsort(d)[::-1][:5]
print("largest abs force diffs", d[i], "at", i, "|f|", np.sqrt(sum(rf[k][i] ** 2 for k in (1, 2, 3))))
