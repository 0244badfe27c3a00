"""CPU suite: pins the oracle (oracle/restate) before anything is compared with it.

1. Known-answer tests restated from the reference's own unit tests
   (test_geometry.cpp, test_chebyshev.cpp, test_m2l.cpp, test_direct.cpp).
2. The reference's recorded end-to-end numbers (proj/test_output.txt:7-11).
3. Golden fixtures generated from the reference itself (tests/golden, made by
   tests/golden/make_golden.py from oracle/_ref): bit-exact tree / lists, fields.
4. Live comparison with oracle/_ref when it is built here.
"""
import ctypes
import glob
import os

import numpy as np
import pytest

from oracles import (CELL_DTYPE, Oracle, OracleOps, OracleTree, RefContext, RefLib, force_error,
                     relative_l2_error)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
L = Oracle.lib()


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def direct(xyzw, targets):
    k = len(targets)
    out = [np.zeros(k) for _ in range(4)]
    t = np.ascontiguousarray(targets, dtype=np.uint32)
    L.orc_direct(_p(xyzw), ctypes.c_uint64(len(xyzw)), _p(t), ctypes.c_uint64(k), *[_p(a) for a in out])
    return out


# ---------------------------------------------------------------- KATs
def test_morton_kats():  # test_geometry.cpp:32-54
    assert L.orc_morton_encode(3, 1, 2, 2) == 46
    assert L.orc_morton_encode(0, 0, 0, 5) == 0
    assert L.orc_morton_encode(0, 0, 1, 3) == 1
    assert L.orc_morton_encode(1, 0, 0, 1) == 4


def test_bounding_cube():  # test_geometry.cpp:56-70
    ps = np.array([[0.0, 0.0, 0.0, 1.0], [1.0, 2.0, 0.5, 1.0]])
    out = np.zeros(4)
    assert L.orc_bounding_cube(_p(ps), ctypes.c_uint64(2), _p(out)) == 0
    assert abs(out[0] - 0.5) < 1e-12 and abs(out[1] - 1.0) < 1e-12 and abs(out[2] - 0.25) < 1e-12
    assert abs(out[3] - 2.0 * (1 + 1e-6)) < 1e-12 and out[3] > 2.0
    one = np.array([[0.3, 0.3, 0.3, 1.0]])
    L.orc_bounding_cube(_p(one), ctypes.c_uint64(1), _p(out))
    assert out[3] == 1.0
    assert L.orc_bounding_cube(_p(one), ctypes.c_uint64(0), _p(out)) == 1  # invalid_argument


def test_chebyshev_kats():  # test_chebyshev.cpp:56-69, 117-127
    r = np.zeros(3)
    L.orc_roots(3, _p(r))
    assert abs(r[0] - 0.86602540378443871) <= 1e-15 * 0.87 and abs(r[1]) < 1e-15
    m = np.zeros(4)
    L.orc_child_matrix(2, 0, _p(m))
    m1 = np.zeros(4)
    L.orc_child_matrix(2, 1, _p(m1))
    vals = sorted(np.round(np.concatenate([m, m1]), 14).tolist())
    for v in (0.39644660940672627, -0.10355339059327373, 0.60355339059327373, 1.1035533905932737):
        assert any(abs(v - x) < 1e-14 for x in vals), v
    # partition of unity at l=2..10 (test_chebyshev.cpp:71-85)
    for l in range(2, 11):
        roots = np.zeros(l)
        L.orc_roots(l, _p(roots))
        for x in (-1.0, -0.3, 0.0, 0.77, 1.0):
            s = sum(L.orc_s_eval(rt, x, l) for rt in roots)
            assert abs(s - 1.0) < 1e-12
        for a in range(l):  # Kronecker delta at the roots
            for b in range(l):
                assert abs(L.orc_s_eval(roots[a], roots[b], l) - (a == b)) < 1e-12


def test_m2l_kats():  # test_m2l.cpp:125-134, 33-34
    k = np.zeros((8, 8))
    L.orc_assemble_m2l(2, 0, 0, 2, ctypes.c_double(1.0), _p(k))
    assert abs(k[0, 0] - 0.5) < 1e-15
    assert abs(k[0, 7] - 0.61180988178458429) < 1e-14
    assert abs(k[7, 0] - 0.34651218019377489) < 1e-14
    assert abs(k[3, 5] - 0.678598344545847) < 1e-14
    ops = OracleOps.cached(5)
    ranks, mult = ops.ranks()
    assert list(mult) == [6, 24, 24, 12, 24, 8, 6, 24, 24, 24, 48, 24, 12, 24, 24, 8]
    assert list(ranks) == [23, 18, 16, 15, 14, 10, 13, 12, 10, 9, 9, 9, 9, 9, 9, 9]
    means = []
    for order in (3, 5, 7):
        r, m = OracleOps.cached(order).ranks()
        means.append(float(np.dot(r, m)) / 316.0)
    assert [round(x, 2) for x in means] == [4.66, 11.49, 23.11]  # test_output.txt:8


def test_symmetry_transport():  # acceptance criterion 3 (acceptance.cpp:100-130)
    perm = np.zeros(3, dtype=np.int32)
    sign = np.zeros(3, dtype=np.int32)
    worst = 0.0
    for order in (2, 3):
        n3 = order ** 3
        canon_list = [(i, j, k) for i in range(2, 4) for j in range(i + 1) for k in range(j + 1)]
        for i in range(-3, 4):
            for j in range(-3, 4):
                for kk in range(-3, 4):
                    if max(abs(i), abs(j), abs(kk)) < 2:
                        continue
                    c = L.orc_canonicalize(i, j, kk, _p(perm), _p(sign))
                    p = np.zeros(n3, dtype=np.uint32)
                    L.orc_grid_permutation(_p(perm), _p(sign), order, _p(p))
                    d = np.zeros((n3, n3))
                    L.orc_assemble_m2l(i, j, kk, order, ctypes.c_double(1.0), _p(d))
                    cm = np.zeros((n3, n3))
                    L.orc_assemble_m2l(*canon_list[c], order, ctypes.c_double(1.0), _p(cm))
                    worst = max(worst, np.abs(d - cm[np.ix_(p, p)]).max())
    assert worst <= 1e-12


def test_pair_kernel_kats():  # test_direct.cpp:25-45
    pts = np.array([[i, j, k, 1.0] for i in range(2) for j in range(2) for k in range(2)], dtype=np.float64)
    pot, fx, fy, fz = direct(pts, [0])
    assert abs(pot[0] - 5.6986706127492681) <= 1e-15 * 5.7
    two = np.array([[0, 0, 0, 1.0], [2, 0, 0, 1.0]])
    pot, fx, fy, fz = direct(two, [0])
    assert abs(fx[0] + 0.25) < 1e-15 and fy[0] == 0 and fz[0] == 0


def test_tree_errors():  # test_geometry.cpp:187-200
    ps = np.array([[0.1, 0.1, 0.1, 1.0], [0.1, 0.1, 0.1, 1.0], [0.9, 0.9, 0.9, 1.0]])
    from oracles import CheckerError
    with pytest.raises(CheckerError) as e:
        OracleTree(ps, 4, 10)
    assert e.value.code == 2
    ok = np.array([[0.1, 0.2, 0.3, 1.0], [0.9, 0.9, 0.9, 1.0]])
    for h, g in ((2, 10), (22, 10), (4, 0)):
        with pytest.raises(CheckerError) as e:
            OracleTree(ok, h, g)
        assert e.value.code == 1
    with pytest.raises(CheckerError) as e:
        OracleTree(ok, 4, 10, root=[0.5, 0.5, 0.5, 0.5])
    assert e.value.code == 2


def test_near_far_trichotomy():  # test_geometry.cpp:213-278: full 4^3 grid
    g = 4
    pts = np.array([[(i + 0.5) / g, (j + 0.5) / g, (k + 0.5) / g, 1.0]
                    for i in range(g) for j in range(g) for k in range(g)])
    t = OracleTree(pts, 3, 1000, root=[0.5, 0.5, 0.5, 1.0])
    off, cells, _, _ = t.near()
    counts = np.diff(off)
    assert counts.max() == 26 and counts.min() == 7
    tt, ss, vv, go = t.far(2)
    per_target = np.bincount(tt, minlength=64)
    assert per_target.max() <= 189
    for c in range(64):  # near + far + self partition the cells of the 6^3 parent window
        near = set(cells[off[c]:off[c + 1]].tolist())
        far = set(ss[tt == c].tolist())
        assert not (near & far) and c not in near and c not in far


# ---------------------------------------------------------------- recorded reference outputs
def test_reference_recorded_accuracy():
    """proj/test_output.txt:7 (criterion 1): eps_L2 = 1.242e-04 / 1.051e-06 / 1.150e-08 for
    orders 3/5/7 at N=1e4 uniform seed 42, h=4, 1000 sampled targets k*n/1000 (bench.cpp:369-377)."""
    n = 10000
    xyzw = Oracle.generate_particles(n, "uniform", 42)
    targets = np.array([k * n // 1000 for k in range(1000)], dtype=np.uint32)
    ref = direct(xyzw, targets)
    got = []
    for order in (3, 5, 7):
        t = OracleTree(xyzw, 4)
        f = t.evaluate(OracleOps.cached(order))
        got.append(relative_l2_error(f[0][targets], ref[0]))
    assert ["%.3e" % x for x in got] == ["1.242e-04", "1.051e-06", "1.150e-08"]


def test_reference_recorded_full_oracle():
    """proj/test_output.txt:11 (criterion 5): N=2000, h=3, order 7, every target:
    potential 1.825e-08, force 1.256e-06."""
    n = 2000
    xyzw = Oracle.generate_particles(n, "uniform", 42)
    t = OracleTree(xyzw, 3)
    f = t.evaluate(OracleOps.cached(7))
    ref = direct(xyzw, np.arange(n))
    assert "%.3e" % relative_l2_error(f[0], ref[0]) == "1.825e-08"
    assert "%.3e" % force_error(*f[1:], *ref[1:]) == "1.256e-06"


def test_mutual_equals_onesided():  # test_direct.cpp:179-214
    xyzw = Oracle.generate_particles(3000, "uniform", 5)
    xyzw[:, 3] = 0.5 + np.random.default_rng(5).random(3000)
    ops = OracleOps(3)
    a = OracleTree(xyzw, 4).evaluate(ops, mask=32, mutual=True)
    b = OracleTree(xyzw, 4).evaluate(ops, mask=32, mutual=False)
    assert relative_l2_error(a[0], b[0]) <= 1e-14
    assert force_error(*a[1:], *b[1:]) <= 1e-14


# ---------------------------------------------------------------- golden fixtures from the reference
GOLDEN_FILES = sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


@pytest.mark.parametrize("path", GOLDEN_FILES, ids=[os.path.basename(p)[:-4] for p in GOLDEN_FILES])
def test_oracle_against_golden(path):
    gd = np.load(path)
    n, h, l = int(gd["n"]), int(gd["height"]), int(gd["order"])
    xyzw = np.ascontiguousarray(gd["xyzw"])
    t = OracleTree(xyzw, h)
    assert np.array_equal(t.root_cube(), gd["root"])
    assert np.array_equal(t.particles()[4], gd["ids"])
    for v in range(h):
        cells, bo = t.level(v)
        cells["_pad"] = 0
        assert np.array_equal(cells.view(np.uint8), gd[f"cells{v}"]), v
        assert np.array_equal(bo, gd[f"blocks{v}"])
    off, cells, ti, tot = t.near()
    assert np.array_equal(off, gd["near_off"]) and np.array_equal(cells, gd["near_cells"])
    assert np.array_equal(ti, gd["task_interactions"]) and tot == int(gd["near_total"])
    for v in range(2, h):
        tt, ss, vv, go = t.far(v)
        assert np.array_equal(tt, gd[f"far_t{v}"]) and np.array_equal(ss, gd[f"far_s{v}"])
        assert np.array_equal(vv, gd[f"far_v{v}"]) and np.array_equal(go, gd[f"far_g{v}"])
    ops = OracleOps(l, cache_path=os.path.join(GOLDEN, f"m2l_l{l}.bin"))
    assert list(ops.ranks()[0]) == list(gd["ranks"])
    f = t.evaluate(ops)
    assert relative_l2_error(f[0], gd["pot"]) <= 1e-14
    assert force_error(*f[1:], gd["fx"], gd["fy"], gd["fz"]) <= 1e-13
    f2 = OracleTree(xyzw, h).evaluate(OracleOps.cached(l))  # own Jacobi SVD factors
    assert relative_l2_error(f2[0], gd["pot"]) <= 1e-13
    assert force_error(*f2[1:], gd["fx"], gd["fy"], gd["fz"]) <= 1e-13


@pytest.mark.skipif(not RefLib.available(), reason="oracle/_ref not built")
def test_oracle_against_live_reference(tmp_path):
    for (n, h, l, dist) in [(4000, 4, 4, "sphere"), (6000, 5, 3, "uniform")]:
        xyzw = Oracle.generate_particles(n, dist, 3)
        ref = RefContext(xyzw, h, l)
        t = OracleTree(xyzw, h)
        for v in range(h):
            a, ab = t.level(v)
            b, bb = ref.level(v)
            a["_pad"] = 0
            b["_pad"] = 0
            assert np.array_equal(a, b) and np.array_equal(ab, bb)
        ref.execute(workers=2)
        rf = ref.fields()
        cache = str(tmp_path / "c.bin")
        ref.save_m2l_cache(cache)
        f = t.evaluate(OracleOps(l, cache_path=cache))
        assert relative_l2_error(f[0], rf[0]) <= 1e-14
        assert force_error(*f[1:], *rf[1:]) <= 1e-13
