"""Output formats of the reference (bench.cpp:504-584) written by the mirror: results.csv
round-trips every double (%.17g), summary.json carries the reference's keys."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1206_0115_b200 import RunConfig  # noqa: E402
from paper_1206_0115_b200.report import (flop_costs, read_results_csv, write_chrome_trace,  # noqa: E402
                                         write_results_csv, write_summary_json)


def test_results_csv_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    xyzw = rng.random((50, 4))
    fields = [rng.standard_normal(50) * 10.0 ** rng.integers(-5, 8, 50) for _ in range(4)]
    p = str(tmp_path / "results.csv")
    write_results_csv(p, xyzw, fields)
    head = open(p).readline().strip()
    assert head == "id,x,y,z,w,potential,fx,fy,fz"
    x2, f2 = read_results_csv(p)
    assert np.array_equal(x2, xyzw) and all(np.array_equal(a, b) for a, b in zip(f2, fields))


def test_summary_json_keys(tmp_path):
    cfg = RunConfig(n=100, height=4, acc=5)
    work = np.zeros((7, 4), dtype=np.uint64)
    flops = np.zeros((7, 4), dtype=np.uint64)
    work[0, 3], flops[0, 3] = 100, 10
    work[2, 2], flops[2, 2] = 7, 20
    work[2, 3], flops[2, 3] = 9, 30
    work[5, 3], flops[5, 3] = 12, 40
    comp = {"ranks": [23] * 16, "multiplicity": [6] * 16, "weighted_mean_rank": 11.49}
    p = str(tmp_path / "summary.json")
    write_summary_json(p, cfg=cfg, n=100, setup_seconds=0.1, exec_seconds=0.2, wall_seconds=0.3,
                       compression=comp, ledger_rows={"work": work, "flops": flops}, eps=(1e-6, 1e-5),
                       spans=[("P2P", 3, 1, 0.0, 2.0), ("M2L", 2, 0, 0.0, 1.0), ("M2L", 3, 0, 1.0, 2.0)])
    j = json.load(open(p))
    assert set(j) == {"config", "timings", "compression", "flop_costs", "ledger", "accuracy", "breakdown",
                      "occupancy"}
    assert j["ledger"]["total_flops"] == 100 and j["ledger"]["M2L"]["flops"] == 50
    assert [e["level"] for e in j["ledger"]["M2L"]["levels"]] == [2, 3]
    assert abs(j["ledger"]["M2L"]["levels"][1]["share_percent"] - 30) < 1e-12
    assert j["flop_costs"] == flop_costs(5) and j["flop_costs"]["l2p_per_particle"] == 16 * 125 + 150
    assert j["occupancy"]["busy_fraction"] == [1.0, 1.0] and j["occupancy"]["kind_share"]["P2P"] == 0.5


def _same_shape(a, b, path=""):
    """Recursive key / type / list-length equality of two JSON trees (occupancy's
    busy_fraction has one entry per worker thread in the reference, per CUDA stream on
    the device)."""
    assert type(a) is type(b) or {type(a), type(b)} <= {int, float}, (path, a, b)
    if isinstance(a, dict):
        assert set(a) == set(b), (path, set(a) ^ set(b))
        for k in a:
            _same_shape(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        if path.endswith("busy_fraction"):
            return
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _same_shape(x, y, f"{path}[{i}]")


def test_summary_json_matches_reference_writer(tmp_path):
    """Our writer fed the reference's own ledger rows reproduces the reference writer's
    summary.json (bench.cpp:516-584): same keys and nesting, identical ledger, shares and
    breakdown text. (The device ledger rows themselves are checked equal to the
    reference's in tests/test_gpu_configs.py.)"""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from oracles import Oracle, RefContext, RefLib, ref_run_fmm
    if not RefLib.available():
        import pytest
        pytest.skip("oracle/_ref not built")
    n, h, acc, seed = 6000, 4, 4, 42
    ref_dir = str(tmp_path / "ref")
    eps = ref_run_fmm(n, "uniform", seed, h, acc, ref_dir, workers=2, check=100)
    rj = json.load(open(os.path.join(ref_dir, "summary.json")))
    ref = RefContext(Oracle.generate_particles(n, "uniform", seed), h, acc)
    rows = ref.ledger_rows()
    ranks = ref.ranks()
    cfg = RunConfig(n=n, height=h, acc=acc, seed=seed)
    mult = [6, 24, 24, 12, 24, 8, 6, 24, 24, 24, 48, 24, 12, 24, 24, 8]
    comp = {"ranks": ranks, "multiplicity": mult,
            "weighted_mean_rank": sum(int(r) * m for r, m in zip(ranks, mult)) / 316.0}
    p = str(tmp_path / "summary.json")
    oj = write_summary_json(p, cfg=cfg, n=n, setup_seconds=rj["timings"]["setup_seconds"],
                            exec_seconds=rj["timings"]["exec_seconds"], wall_seconds=rj["timings"]["wall_seconds"],
                            compression=comp, ledger_rows=rows, eps=eps, check=100,
                            spans=[("P2P", h - 1, 1, 0.0, 1.0)])
    oj = json.load(open(p))
    _same_shape(oj, rj)
    assert oj["ledger"] == rj["ledger"]
    assert oj["breakdown"] == rj["breakdown"]
    assert oj["flop_costs"] == rj["flop_costs"]
    assert oj["compression"]["ranks"] == rj["compression"]["ranks"]
    assert oj["compression"]["multiplicity"] == rj["compression"]["multiplicity"]
    assert abs(oj["compression"]["weighted_mean_rank"] - rj["compression"]["weighted_mean_rank"]) < 1e-12
    for k in ("n", "dist", "height", "acc", "group_size", "seed", "check", "dry_run"):
        assert oj["config"][k] == rj["config"][k], k
    assert oj["accuracy"] == rj["accuracy"]


def test_chrome_trace_format(tmp_path):
    spans = [("P2P", 6, 1, 0.0, 12.5), ("P2M", 6, 0, 0.01, 0.8), ("M2L", 6, 0, 1.0, 13.0)]
    p = str(tmp_path / "trace.json")
    write_chrome_trace(p, spans, work={("M2L", 6): 123})
    ev = json.load(open(p))
    assert [e["name"] for e in ev] == ["P2P", "P2M", "M2L"]
    assert all(e["ph"] == "X" and e["pid"] == 0 for e in ev)
    assert ev[0]["tid"] == 1 and abs(ev[0]["dur"] - 12500.0) < 1e-9 and ev[2]["args"] == {"level": 6, "work": 123}
