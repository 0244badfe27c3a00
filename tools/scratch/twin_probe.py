"""Prototype of a two-context pipeline (development aid): tree build k+1 on one context
while the other context evaluates step k. Device-resident inputs, wall clock per step."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1206_0115_b200 as P
from ctypes import c_void_p

n, h = 10_000_000, 7
dev = torch.from_numpy(P.generate_particles(n, "uniform", 42)).cuda()
lib = P.lib()
a = P.FmmContext(None, order=5)
b = P.FmmContext(None, order=5)
ctxs = [a, b]


def build(c):
    c._check(lib.fmmgpu_build_tree(c.h, c_void_p(dev.data_ptr()), n, 1, h, 250, None))


for c in ctxs:
    build(c)
    c.evaluate()
    c.synchronize()
# serial: build + evaluate on one context
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(8):
    build(a)
    a.evaluate()
a.synchronize()
print("serial     %.2f ms/step" % ((time.perf_counter() - t0) / 8 * 1e3), flush=True)
# alternating contexts
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(8):
    c = ctxs[k & 1]
    build(c)
    c.evaluate()
for c in ctxs:
    c.synchronize()
print("alternate  %.2f ms/step" % ((time.perf_counter() - t0) / 8 * 1e3), flush=True)
# alternating, evaluation k+1 ordered after evaluation k (no two evaluations at once)
torch.cuda.synchronize()
t0 = time.perf_counter()
ev = torch.cuda.Event()
for k in range(8):
    c = ctxs[k & 1]
    build(c)
    o = ctxs[(k + 1) & 1]
    o.synchronize() if k else None
    c.evaluate()
for c in ctxs:
    c.synchronize()
print("alt+order  %.2f ms/step" % ((time.perf_counter() - t0) / 8 * 1e3), flush=True)
