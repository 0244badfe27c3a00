"""ncu driver: two config-B tree builds from device memory (profile the second)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1206_0115_b200 as P
from ctypes import c_void_p
n, h = 10_000_000, 7
x = torch.from_numpy(P.generate_particles(n, "uniform", 42)).cuda()
c = P.FmmContext(None, order=5, m2l_cache="tests/golden/m2l_l5.bin")  # no device SVD under ncu
for _ in range(2):
    c._check(P.lib().fmmgpu_build_tree(c.h, c_void_p(x.data_ptr()), n, 1, h, 250, None))
torch.cuda.synchronize()
print("tree ms", c.timings()["TREE"])
