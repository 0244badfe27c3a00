"""Warm tree-build time at config B from device-resident particles (development aid):
CUDA events around fmmgpu_build_tree (timings()['TREE']) and the host wall time."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1206_0115_b200 as P

n, h = 10_000_000, 7
xyzw = P.generate_particles(n, "uniform", 42)
c = P.FmmContext(None, order=5)
c.build_tree(xyzw, h)
dev = torch.from_numpy(xyzw).cuda()
ev, wall = [], []
for _ in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c.build_tree(n, h, 250, on_device_ptr=dev.data_ptr())
    torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e3)
    ev.append(c.timings()["TREE"])
print(f"tree build: events best {min(ev):.3f} median {sorted(ev)[4]:.3f} ms; host wall best {min(wall):.3f} ms")
