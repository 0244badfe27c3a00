"""Time the M2L phase A tilings (FMMGPU_M2L_A) at config B and check the leaf locals
are bitwise identical. One process per variant. Development aid."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, ".")
    import numpy as np
    import paper_1206_0115_b200 as P
    order = int(os.environ.get("ORDER", "5"))
    xyzw = P.generate_particles(10_000_000, "uniform", 42)
    c = P.FmmContext(None, order=order)
    c.build_tree(xyzw, 7)
    c.time_operator("M2L", 6, 1)
    leaf = c.time_operator("M2L", 6, 5)
    import ctypes
    ms = ctypes.c_double()
    allv = c.time_operator("M2L", -1, 3)
    c.evaluate()
    c.synchronize()
    np.save(f"/tmp/m2l_v{sys.argv[1]}.npy", c.expansion(6, 1))
    print(f"variant {sys.argv[1]}: leaf {leaf:.3f} ms, all levels {allv:.3f} ms", flush=True)
else:
    # (FMMGPU_M2L_A, FMMGPU_M2L_LATE)
    SETS = {0: ("0", "0", "0"), 1: ("0", "0", "1"), 4: ("0", "0", "4")}
    VARIANTS = list(SETS)
    for v in VARIANTS:
        env = dict(os.environ, FMMGPU_M2L_A=SETS[v][0], FMMGPU_M2L_LATE=SETS[v][1], FMMGPU_M2L_DEBUG=SETS[v][2])
        subprocess.run([sys.executable, __file__, str(v)], env=env, check=True)
    import numpy as np
    base = np.load(f"/tmp/m2l_v{VARIANTS[0]}.npy")
    for v in VARIANTS[1:]:
        print(f"variant {v} bitwise equal to {VARIANTS[0]}:", bool(np.array_equal(np.load(f"/tmp/m2l_v{v}.npy"), base)))
