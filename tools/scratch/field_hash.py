"""sha256 of one evaluation's gathered fields (development aid: a timing variant must give
bitwise the same fields). python tools/scratch/field_hash.py [N H ORDER DIST]"""
import hashlib
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1206_0115_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
h = int(sys.argv[2]) if len(sys.argv) > 2 else 7
order = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dist = sys.argv[4] if len(sys.argv) > 4 else "uniform"
c = P.FmmContext(None, order=order)
c.build_tree(P.generate_particles(n, dist, 42), h)
c.evaluate()
m = hashlib.sha256()
for f in c.gather():
    m.update(np.ascontiguousarray(f).tobytes())
print(f"fields n={n} h={h} l={order} {dist}: {m.hexdigest()[:16]}")
