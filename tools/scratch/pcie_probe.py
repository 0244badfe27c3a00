"""PCIe copy-rate probe (development aid): pinned 320 MB H2D / D2H, repeated."""
import time
import torch
a = torch.empty(40_000_000, dtype=torch.float64).pin_memory()
b = torch.empty(40_000_000, dtype=torch.float64, device="cuda")
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter(); b.copy_(a, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); a.copy_(b, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"h2d {0.32/(t1-t0):6.1f} GB/s  d2h {0.32/(t2-t1):6.1f} GB/s", flush=True)
