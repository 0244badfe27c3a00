"""First GPU test of the suite (collected before the others): one evaluation of every
kernel family of the hot path through the C ABI, with the M2L operators read from the
reference's own cache (tests/golden, M2LOperatorSet::save_cache) so no cuSOLVER
precompute runs first -- the launches recorded for this process begin with the tree
build, k_p2p_mutual / k_p2p_drain, k_p2p, k_m2l_phase_a / phase_b, the transfers and the
gather. Checked against the oracle with the same factors."""
import os

import numpy as np
import pytest

from oracles import Oracle, OracleOps, OracleTree, force_error, relative_l2_error

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_family_runs_first():
    import paper_1206_0115_b200 as P
    n, h, order = 40000, 5, 5
    xyzw = Oracle.generate_particles(n, "uniform", 42)
    xyzw[:, 3] = 0.5 + np.random.default_rng(1).random(n)
    cache = os.path.join(ROOT, "tests", "golden", "m2l_l5.bin")
    ref = OracleTree(xyzw, h).evaluate(OracleOps(order, cache_path=cache))
    with P.FmmContext(None, order=order, m2l_cache=cache) as c:
        c.build_tree(xyzw, h, 250)
        for mutual in (True, False):  # both near-field kernels
            c.set_p2p_mode(mutual)
            c.evaluate()
            g = c.gather()
            assert c.launch_count() > 0
            assert relative_l2_error(g[0], ref[0]) <= 1e-12
            assert force_error(*g[1:], *ref[1:]) <= 1e-12
