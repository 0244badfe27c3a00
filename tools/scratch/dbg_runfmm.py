import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_1206_0115_b200 as P
from oracles import Oracle, OracleTree, OracleOps, relative_l2_error
for (n,h,acc) in [(10000,4,3),(10000,4,5),(20000,5,5)]:
    cfg = P.RunConfig(n=n, height=h, acc=acc, seed=42)
    f, ep, ef = P.run_fmm(cfg, check=1000)
    x = P.generate_particles(n, 'uniform', 42)
    o = OracleTree(x, h).evaluate(OracleOps.cached(acc))
    print(n, h, acc, 'eps', ep, ef, 'vs oracle', relative_l2_error(f[0], o[0]), flush=True)
