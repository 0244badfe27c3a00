"""Does a concurrent PCIe copy slow an evaluation down? (development aid) Times config-B
evaluations alone, with a 320 MB D2H, and with a 320 MB H2D running on a side stream."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1206_0115_b200 as P

c = P.FmmContext(None, order=5)
c.build_tree(P.generate_particles(10_000_000, "uniform", 42), 7)
for _ in range(3):
    c.evaluate()
c.synchronize()
dev = torch.empty(40_000_000, dtype=torch.float64, device="cuda")
host = torch.empty(40_000_000, dtype=torch.float64).pin_memory()
side = torch.cuda.Stream()


def run(mode, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if mode == "d2h":
            with torch.cuda.stream(side):
                host.copy_(dev, non_blocking=True)
        elif mode == "h2d":
            with torch.cuda.stream(side):
                dev.copy_(host, non_blocking=True)
        t0 = time.perf_counter()
        c.evaluate()
        c.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
    print(f"{mode:5s} eval wall {min(ts):.3f} ms (min of {reps}), device {c.timings()['EVAL']:.3f} ms", flush=True)


for mode in ("none", "d2h", "h2d", "none", "d2h"):
    run(mode)
