"""Time the M2L variants (FMMGPU_M2L_VARIANT: 0 scatter in phase A, 1 dense phase A +
gather in phase B) in isolation at config B and check bitwise-identical local
expansions. One process per variant. Development aid."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, ".")
    import numpy as np
    import paper_1206_0115_b200 as P
    xyzw = P.generate_particles(10_000_000, "uniform", 42)
    c = P.FmmContext(None, order=int(os.environ.get("ORDER", "5")))
    c.build_tree(xyzw, 7)
    c.evaluate()
    c.synchronize()
    ms_all = c.time_operator("M2L", -1, 3)
    ms_leaf = c.time_operator("M2L", 6, 3)
    c.evaluate()
    g = c.gather()
    np.save(f"/tmp/m2l_v{sys.argv[1]}.npy", np.stack(g))
    print(f"variant {sys.argv[1]}: M2L all levels {ms_all:.3f} ms, leaf {ms_leaf:.3f} ms, eval {c.timings()['EVAL']:.3f} ms",
          flush=True)
else:
    for v in range(2):
        env = dict(os.environ, FMMGPU_M2L_VARIANT=str(v))
        subprocess.run([sys.executable, __file__, str(v)], env=env, check=True)
    import numpy as np
    a, b = np.load("/tmp/m2l_v0.npy"), np.load("/tmp/m2l_v1.npy")
    print("fields bitwise equal:", bool(np.array_equal(a, b)), "max rel diff", float(np.max(np.abs(a - b)) / np.max(np.abs(a))))
