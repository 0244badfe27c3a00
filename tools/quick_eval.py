"""Quick device timing of one configuration (development aid; bench.py is the contract)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1206_0115_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
h = int(sys.argv[2]) if len(sys.argv) > 2 else 7
l = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t0 = time.time(); xyzw = P.generate_particles(n, "uniform", 42); print("gen", time.time() - t0, flush=True)
t0 = time.time(); c = P.FmmContext(None, order=l); print("ctx", time.time() - t0, c.compression_report()["ranks"], flush=True)
for i in range(3):
    t0 = time.time(); c.build_tree(xyzw, h); print("tree", time.time() - t0, flush=True)
for i in range(4):
    c.evaluate(); c.synchronize()
    print({k: round(v, 3) for k, v in c.timings().items()}, "launches", c.launch_count(), flush=True)
g = c.gather()
print("pot", g[0][:3], "f", g[1][:3])
