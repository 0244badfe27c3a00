"""Timeline of pipelined runs at config B (development aid): FMMGPU_TRACE=1 makes
fmmgpu_run_wait print event times of every step's H2D, tree build, evaluation and D2H."""
import os
import sys
import time

os.environ["FMMGPU_TRACE"] = "1"
sys.path.insert(0, ".")
import torch

import paper_1206_0115_b200 as P

n, h = 10_000_000, 7
xyzw = P.generate_particles(n, "uniform", 42)
c = P.FmmContext(None, order=5)
pins = [torch.from_numpy(xyzw).pin_memory() for _ in range(2)]
outs = [[torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)] for _ in range(2)]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(6):
        c.run_async(pins[k % 2].data_ptr(), n, h, 250, [o.data_ptr() for o in outs[k % 2]])
    c.run_wait()
    print(f"rep {rep}: {(time.perf_counter() - t0) / 6 * 1e3:.2f} ms/step wall", flush=True)
