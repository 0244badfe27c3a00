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
    ledger = {"flops": {"P2M": 10, "M2M": 1, "M2L": 50, "L2L": 1, "L2P": 20, "P2P": 18, "P2PREDUCE": 0},
              "near_directional": 12, "m2l_pairs": 34}
    comp = {"ranks": [23] * 16, "multiplicity": [6] * 16, "weighted_mean_rank": 11.49}
    p = str(tmp_path / "summary.json")
    write_summary_json(p, cfg=cfg, n=100, setup_seconds=0.1, exec_seconds=0.2, wall_seconds=0.3,
                       compression=comp, ledger=ledger, eps=(1e-6, 1e-5))
    j = json.load(open(p))
    assert set(j) >= {"config", "timings", "compression", "flop_costs", "ledger", "accuracy"}
    assert j["ledger"]["total_flops"] == 100 and abs(j["ledger"]["M2L"]["share_percent"] - 50) < 1e-12
    assert j["flop_costs"] == flop_costs(5) and j["flop_costs"]["l2p_per_particle"] == 16 * 125 + 150


def test_chrome_trace_format(tmp_path):
    spans = [("P2P", 6, 1, 0.0, 12.5), ("P2M", 6, 0, 0.01, 0.8), ("M2L", 6, 0, 1.0, 13.0)]
    p = str(tmp_path / "trace.json")
    write_chrome_trace(p, spans, work={("M2L", 6): 123})
    ev = json.load(open(p))
    assert [e["name"] for e in ev] == ["P2P", "P2M", "M2L"]
    assert all(e["ph"] == "X" and e["pid"] == 0 for e in ev)
    assert ev[0]["tid"] == 1 and abs(ev[0]["dur"] - 12500.0) < 1e-9 and ev[2]["args"] == {"level": 6, "work": 123}
