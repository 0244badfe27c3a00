"""Parity of the CUDA path with the reference itself at the BASELINE.json configurations
(test infrastructure: used by tests/test_gpu_configs.py and tools/parity_report.py).

The north-star bar (BASELINE.json): bit-exact tree, Morton keys and interaction lists,
and potentials / forces within relative L2 <= 1e-12 of the reference CPU implementation
at the same Chebyshev order. The reference is oracle/_ref (the unmodified reference
sources, FmmContext + execute with all host threads); the comparison is made twice:
with each side's own SVD factors (cuSOLVER on the device vs the reference's LAPACK
BDCSVD stand-in) and with the reference's factors loaded into the device context
through the reference cache format (m2l.cpp:212-288).

Checks, in the order the reference builds the structures:
* root cube (geometry.cpp:18-36), ParticleStore in Morton order with ids (:95-109);
* every level's Cell array and block_offsets (geometry.cpp:113-160);
* near CSR + total_directional (direct.cpp:22-61), far LevelM2L pairs / vec slots /
  group offsets per level (taskflow.cpp:67-105);
* the flop ledger per (kind, level) and the M2L pairs per (level, class)
  (count_interactions + build_ledger, taskflow.cpp:107-135, bench.cpp:151-181);
* fields in input order (bench.cpp:350-365), relative L2 (bench.cpp:91-100).
"""
from __future__ import annotations

import os
import tempfile
import time

import numpy as np

from oracles import Oracle, RefContext, force_error, relative_l2_error

# name: (n, dist, height, order, seed, random weights)
CONFIGS = {
    "A": (100_000, "uniform", 4, 5, 42, False),
    "H7": (300_000, "uniform", 7, 5, 7, True),   # leaf M2L large enough for unsplit phase A / B
    "B": (10_000_000, "uniform", 7, 5, 42, False),
    "C": (10_000_000, "uniform", 7, 7, 42, False),
    "D": (20_000_000, "ellipsoid", 8, 5, 42, False),
    "E": (100_000_000, "uniform", 8, 5, 42, False),
}


def particles(name):
    n, dist, h, l, seed, rw = CONFIGS[name]
    xyzw = Oracle.generate_particles(n, dist, seed)
    if rw:  # test_direct.cpp:15-21: w in [0.5, 1.5)
        xyzw[:, 3] = 0.5 + np.random.default_rng(seed).random(n)
    return xyzw


def _eq_cells(a, b):
    a = a.copy()
    b = b.copy()
    a["_pad"] = 0
    b["_pad"] = 0
    return np.array_equal(a, b)


def compare_tree(c, ref, h):
    out = {"root": bool(np.array_equal(c.root_cube(), ref.root_cube()))}
    ok = True
    for a, b in zip(c.particles(), ref.particles()):
        ok = ok and np.array_equal(a, b)
    out["particles_ids"] = bool(ok)
    bad = []
    for v in range(h):
        gc, gb = c.level(v)
        rc, rb = ref.level(v)
        if not (_eq_cells(gc, rc) and np.array_equal(gb, rb)):
            bad.append(v)
    out["levels_bad"] = bad
    out["cells_per_level"] = [int(c.level(v)[0].shape[0]) for v in range(h)]
    out["bit_exact"] = out["root"] and out["particles_ids"] and not bad
    return out


def compare_lists(c, ref, h):
    c.build_lists()
    goff, gcells, gtot = c.near()
    roff, rcells, _, rtot = ref.near()
    out = {"near": bool(np.array_equal(goff, roff) and np.array_equal(gcells, rcells) and gtot == rtot),
           "near_entries": int(len(rcells)), "near_directional": int(rtot)}
    # NearFieldPlan block arrays (partners_above, contributors_below, task_interactions)
    gb, rb = c.near_blocks(), ref.near_blocks()
    out["near_blocks"] = bool(all(np.array_equal(x, y) for x, y in zip(gb, rb)))
    out["near"] = out["near"] and out["near_blocks"]
    bad, pairs = [], 0
    for v in range(2, h):
        g = c.far(v)
        r = ref.far(v)
        pairs += len(r[0])
        if not all(np.array_equal(a, b) for a, b in zip(g, r)):
            bad.append(v)
        del g, r
        # LevelM2L::source_blocks (taskflow.cpp:96-102)
        if not all(np.array_equal(a, b) for a, b in zip(c.far_source_blocks(v), ref.far_source_blocks(v))):
            bad.append(v)
    out["far_levels_bad"] = bad
    out["m2l_pairs"] = pairs
    out["bit_exact"] = out["near"] and not bad
    return out


def compare_ledger(c, ref):
    g = c.ledger_rows()
    r = ref.ledger_rows()
    eq = {k: bool(np.array_equal(g[k], r[k])) for k in ("work", "flops", "m2l_pairs")}
    return {"equal": all(eq.values()), **eq, "total_flops": int(r["flops"].sum())}


def field_errors(g, r):
    return relative_l2_error(g[0], r[0]), force_error(*g[1:], *r[1:])


def run(name, P, workers=None, lists=True, shared=True, log=print):
    """Builds both sides for config `name` and compares everything; returns a dict."""
    n, dist, h, l, seed, rw = CONFIGS[name]
    workers = workers or os.cpu_count() or 1
    res = {"config": name, "n": n, "dist": dist, "height": h, "order": l, "seed": seed, "random_weights": rw}
    xyzw = particles(name)
    t0 = time.perf_counter()
    ref = RefContext(xyzw, h, l)
    res["ref_setup_seconds"] = ref.setup_seconds()
    res["ref_exec_seconds"] = ref.execute(workers=workers)
    res["ref_workers"] = workers
    rf = ref.fields()
    log(f"[{name}] reference: setup {res['ref_setup_seconds']:.1f} s, exec {res['ref_exec_seconds']:.1f} s "
        f"({workers} workers)")
    c = P.FmmContext(None, order=l)
    c.build_tree(xyzw, h, 250)
    res["tree"] = compare_tree(c, ref, h)
    if lists:
        res["lists"] = compare_lists(c, ref, h)
        res["ledger"] = compare_ledger(c, ref)
    c.evaluate()
    g = c.gather()
    ep, ef = field_errors(g, rf)
    res["own_factors"] = {"rel_l2_potential": ep, "rel_l2_force": ef}
    log(f"[{name}] own factors: potential {ep:.3e} force {ef:.3e}; tree {res['tree']['bit_exact']}"
        + (f", lists {res['lists']['bit_exact']}, ledger {res['ledger']['equal']}" if lists else ""))
    if shared:
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "m2l.bin")
            ref.save_m2l_cache(path)
            c.load_m2l_cache(path)
        c.evaluate()
        g = c.gather()
        ep, ef = field_errors(g, rf)
        res["reference_factors"] = {"rel_l2_potential": ep, "rel_l2_force": ef}
        log(f"[{name}] reference factors: potential {ep:.3e} force {ef:.3e}")
    c.close()
    res["wall_seconds"] = time.perf_counter() - t0
    return res
