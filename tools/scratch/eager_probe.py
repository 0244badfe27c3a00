"""Eager first evaluation after a tree build vs graph replay (development aid)."""
import sys

sys.path.insert(0, ".")
import torch

import paper_1206_0115_b200 as P

x = torch.from_numpy(P.generate_particles(10_000_000, "uniform", 42)).cuda()
c = P.FmmContext(None, order=5)
from ctypes import c_void_p
lib = P.lib()
for it in range(4):
    c._check(lib.fmmgpu_build_tree(c.h, c_void_p(x.data_ptr()), 10_000_000, 1, 7, 250, None))
    for k in range(3):
        c.evaluate()
        c.synchronize()
        print(f"build {it} eval {k}: {c.timings()['EVAL']:.3f} ms", flush=True)
