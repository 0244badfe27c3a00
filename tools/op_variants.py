"""A/B timing of one operator under an environment switch at config B (development aid).

    python tools/op_variants.py ENVVAR KIND LEVEL VALUE [VALUE ...]

One process per value; prints the isolated device time (time_operator, 5 reps) and
whether the operator's output (leaf multipole for P2M, leaf local_own for M2L, the
sorted fields otherwise) is bitwise identical to the first value's."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    _, _, kind, level, tag = sys.argv
    sys.path.insert(0, ".")
    import numpy as np
    import paper_1206_0115_b200 as P
    level = int(level)
    xyzw = P.generate_particles(10_000_000, "uniform", 42)
    c = P.FmmContext(None, order=int(os.environ.get("ORDER", "5")))
    c.build_tree(xyzw, 7)
    c.time_operator(kind, level, 1)
    ms = c.time_operator(kind, level, 5)
    c.evaluate()
    c.synchronize()
    out = {"P2M": lambda: c.expansion(6, 0), "M2L": lambda: c.expansion(6, 1)}.get(kind, lambda: np.stack(c.sorted_fields()))()
    np.save(f"/tmp/opv_{tag}.npy", out)
    print(f"{kind} level {level} [{tag}]: {ms:.3f} ms", flush=True)
else:
    env, kind, level, *vals = sys.argv[1:]
    for v in vals:
        subprocess.run([sys.executable, __file__, "--child", kind, level, f"{env}={v}"],
                       env=dict(os.environ, **{env: v}), check=True)
    import numpy as np
    base = np.load(f"/tmp/opv_{env}={vals[0]}.npy")
    for v in vals[1:]:
        print(f"{env}={v} bitwise equal to {env}={vals[0]}:", bool(np.array_equal(np.load(f"/tmp/opv_{env}={v}.npy"), base)))
