"""Steady-state breakdown of one e2e step at config B (development aid): tree build from
pinned host / device memory, evaluation, field download, serial and pipelined runs."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1206_0115_b200 as P

import os
n, h, dist = {"B": (10_000_000, 7, "uniform"), "D": (20_000_000, 8, "ellipsoid")}[os.environ.get("PROBE_CFG", "B")]
xyzw = P.generate_particles(n, dist, 42)
c = P.FmmContext(None, order=5)
pin = torch.from_numpy(xyzw).pin_memory()
dev = pin.cuda()
outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
lib = P.lib()
from ctypes import c_void_p


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    free, total = torch.cuda.mem_get_info()
    print(f"    [used {(total - free) / 1e9:.1f} GB]", end=" ")
    return ms


print("build_tree host  %.2f ms" % t(lambda: c._check(lib.fmmgpu_build_tree(c.h, c_void_p(pin.data_ptr()), n, 0, h, 250, None))))
print("build_tree dev   %.2f ms" % t(lambda: c._check(lib.fmmgpu_build_tree(c.h, c_void_p(dev.data_ptr()), n, 1, h, 250, None))))
print("  device-timed   %.2f ms" % c.timings()["TREE"])
print("evaluate         %.2f ms" % t(lambda: (c.evaluate(), c.synchronize())))
print("download         %.2f ms" % t(lambda: c._check(lib.fmmgpu_download_fields(c.h, *[c_void_p(o.data_ptr()) for o in outs], 0))))
print("run (serial)     %.2f ms" % t(lambda: c._check(lib.fmmgpu_run(c.h, c_void_p(pin.data_ptr()), n, h, 250, *[c_void_p(o.data_ptr()) for o in outs]))))


def pipe():
    for k in range(6):
        c.run_async(pin.data_ptr(), n, h, 250, [o.data_ptr() for o in outs])
    c.run_wait()


print("run_async x6     %.2f ms/step" % (t(pipe, 2) / 6))
