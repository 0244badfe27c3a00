"""Time the P2P kernel variants (FMMGPU_P2P_VARIANT) in isolation at config B and check
they produce bitwise-identical near fields. One process per variant (the variant is
read once per process). Development aid."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, ".")
    import numpy as np
    import paper_1206_0115_b200 as P
    xyzw = P.generate_particles(10_000_000, "uniform", 42)
    c = P.FmmContext(None, order=5)
    c.build_tree(xyzw, 7)
    c.time_operator("P2P", -1, 1)
    ms = c.time_operator("P2P", -1, 5)
    c.reset()
    c.run_kinds({"P2P"})
    f = c.sorted_fields()
    np.save(f"/tmp/p2p_v{sys.argv[1]}.npy", np.stack(f))
    print(f"variant {sys.argv[1]}: {ms:.3f} ms", flush=True)
else:
    VARIANTS = [0, 2, 3]  # 0 = k_p2p 12 warps (default), 2 = 16 warps, 3 = 8 warps
    for v in VARIANTS:
        env = dict(os.environ, FMMGPU_P2P_VARIANT=str(v))
        subprocess.run([sys.executable, __file__, str(v)], env=env, check=True)
    import numpy as np
    base = np.load(f"/tmp/p2p_v{VARIANTS[0]}.npy")
    for v in VARIANTS[1:]:
        print(f"variant {v} bitwise equal to {VARIANTS[0]}:", bool(np.array_equal(np.load(f"/tmp/p2p_v{v}.npy"), base)))
