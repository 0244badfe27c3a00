"""Per-launch spans of one config-B evaluation (development aid)."""
import sys
sys.path.insert(0, ".")
import paper_1206_0115_b200 as P
c = P.FmmContext(None, order=5)
c.build_tree(P.generate_particles(10_000_000, "uniform", 42), 7)
c.evaluate()
c.set_trace(True)
for _ in range(2):
    c.evaluate()
for k, lv, st, t0, t1 in c.trace_spans():
    print(f"{k:10s} L{lv} stream {st}: {t0:8.3f} -> {t1:8.3f} ({t1 - t0:7.3f} ms)")
