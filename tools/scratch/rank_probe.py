"""Per-rank partitioned evaluation time at config B (measurement mode, exchange skipped) and
the per-launch trace of rank 0 of N (development aid)."""
import os
import sys
sys.path.insert(0, ".")
import paper_1206_0115_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = P.FmmContext(None, order=5)
c.build_tree(P.generate_particles(10_000_000, "uniform", 42), 7)
c.set_measurement(True)
ts = []
for r in range(N):
    c.partition(r, N)
    for _ in range(2):
        c.evaluate()
    t, kinds, _ = c.time_evaluations(5)
    ts.append(t / 5)
print("AUX", os.environ.get("FMMGPU_AUX"), "ranks", N, "max %.3f ms" % max(ts), ["%.3f" % x for x in ts], flush=True)
c.partition(0, N)
c.evaluate()
c.set_trace(True)
c.evaluate()
for k, lv, st, t0, t1 in c.trace_spans():
    print(f"  {k:10s} L{lv} s{st}: {t0:7.3f} -> {t1:7.3f} ({t1 - t0:6.3f})")
