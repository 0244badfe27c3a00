"""Device time of whole config-B evaluations under an environment switch (development
aid): python tools/eval_ab.py ENVVAR VALUE [VALUE ...] -- one process per value.
N, H, DIST, ORDER select the configuration (default config B)."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import paper_1206_0115_b200 as P
    c = P.FmmContext(None, order=int(os.environ.get("ORDER", "5")))
    n, h, dist = int(os.environ.get("N", "10000000")), int(os.environ.get("H", "7")), os.environ.get("DIST", "uniform")
    c.build_tree(P.generate_particles(n, dist, 42), h)
    for _ in range(3):
        c.evaluate()
    total, kinds, _ = c.time_evaluations(10)
    p2p = c.time_operator("P2P", -1, 3)
    print(f"[{sys.argv[2]}] {total / 10:.3f} ms/eval  M2L in step {kinds['M2L'] / 10:.3f}  P2P isolated {p2p:.3f}",
          flush=True)
else:
    env, *vals = sys.argv[1:]
    for v in vals:
        subprocess.run([sys.executable, __file__, "--child", f"{env}={v}"], env=dict(os.environ, **{env: v}), check=True)
