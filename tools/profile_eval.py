"""Profiling driver: build config-B tree, run `evals` evaluations (for ncu)."""
import sys
sys.path.insert(0, ".")
import paper_1206_0115_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
h = int(sys.argv[2]) if len(sys.argv) > 2 else 7
l = int(sys.argv[3]) if len(sys.argv) > 3 else 5
evals = int(sys.argv[4]) if len(sys.argv) > 4 else 2
dist = sys.argv[5] if len(sys.argv) > 5 else "uniform"
xyzw = P.generate_particles(n, dist, 42)
c = P.FmmContext(None, order=l)
c.build_tree(xyzw, h)
for _ in range(evals):
    c.evaluate()
c.synchronize()
print("done", c.timings())
