"""The reference's output formats (bench.cpp:504-584), so its tooling can diff results:

* ``write_results_csv``  results.csv, header ``id,x,y,z,w,potential,fx,fy,fz`` and %.17g
  (round-trip) values (bench.cpp:504-514);
* ``write_summary_json`` summary.json with the reference's keys: config, timings,
  accuracy, compression, flop_costs, ledger (per kind; the device ledger is not split per
  level), occupancy replaced by the device per-operator times (bench.cpp:516-584);
* ``write_chrome_trace`` trace.json in the reference's Chrome "ph":"X" format
  (runtime.cpp:277-292) from the device spans of FmmContext.trace_spans (one span per
  operator launch; tid = CUDA stream: 0 far field, 1 near field).
"""
from __future__ import annotations

import json

import numpy as np

KINDS = ("P2M", "M2M", "M2L", "L2L", "L2P", "P2P", "P2PREDUCE")


def write_results_csv(path: str, xyzw: np.ndarray, fields) -> None:
    pot, fx, fy, fz = fields
    data = np.column_stack([xyzw[:, 0], xyzw[:, 1], xyzw[:, 2], xyzw[:, 3], pot, fx, fy, fz])
    with open(path, "w") as f:
        f.write("id,x,y,z,w,potential,fx,fy,fz\n")
        for i, row in enumerate(data):
            f.write(str(i) + "," + ",".join("%.17g" % v for v in row) + "\n")


def read_results_csv(path: str):
    """Inverse of write_results_csv (and of the reference's results.csv)."""
    a = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    return a[:, 1:5], [a[:, 5], a[:, 6], a[:, 7], a[:, 8]]


def flop_costs(order: int) -> dict:
    """bench.cpp:102-122 (flop_cost)."""
    l = order
    return {"p2p_per_directional_interaction": 15, "p2m_per_particle": 4 * l ** 3 + 15 * l,
            "l2p_per_particle": 16 * l ** 3 + 30 * l, "transfer_per_child": 6 * l ** 4,
            "m2l_per_pair_rank1": 4 * l ** 3 + 1}


def write_summary_json(path: str, *, cfg, n: int, setup_seconds: float, exec_seconds: float,
                       wall_seconds: float, compression: dict, ledger: dict, eps=None,
                       device_ms: dict | None = None) -> dict:
    j = {"config": {"n": n, "dist": cfg.dist, "height": cfg.height, "acc": cfg.acc,
                    "group_size": cfg.group_size, "seed": cfg.seed},
         "timings": {"setup_seconds": setup_seconds, "exec_seconds": exec_seconds, "wall_seconds": wall_seconds},
         "compression": {"order": cfg.acc, "eps": 10.0 ** -cfg.acc,
                         "ranks": [int(r) for r in compression["ranks"]],
                         "multiplicity": [int(m) for m in compression["multiplicity"]],
                         "weighted_mean_rank": float(compression["weighted_mean_rank"])},
         "flop_costs": flop_costs(cfg.acc)}
    if eps is not None and eps[0] >= 0:
        j["accuracy"] = {"eps_l2_potential": float(eps[0]), "eps_l2_force": float(eps[1])}
    total = sum(int(v) for v in ledger["flops"].values())
    j["ledger"] = {k: {"flops": int(ledger["flops"][k]),
                       "share_percent": 100.0 * int(ledger["flops"][k]) / total if total else 0.0} for k in KINDS}
    j["ledger"]["total_flops"] = total
    j["ledger"]["near_directional"] = int(ledger["near_directional"])
    j["ledger"]["m2l_pairs"] = int(ledger["m2l_pairs"])
    if device_ms:
        j["device_ms"] = {k: float(v) for k, v in device_ms.items()}
    with open(path, "w") as f:
        json.dump(j, f, indent=2)
        f.write("\n")
    return j


def write_chrome_trace(path: str, spans, work=None) -> None:
    """runtime.cpp:277-292: a JSON array of {"name", "ph":"X", "ts", "dur" (microseconds),
    "pid":0, "tid", "args":{"level", "work"}}; spans = [(kind, level, stream, start_ms,
    end_ms)], work = optional {(kind, level): value}."""
    events = []
    for kind, level, stream, t0, t1 in spans:
        w = 0 if work is None else work.get((kind, level), 0)
        events.append({"name": kind, "ph": "X", "ts": t0 * 1e3, "dur": (t1 - t0) * 1e3, "pid": 0, "tid": stream,
                       "args": {"level": level, "work": w}})
    with open(path, "w") as f:
        json.dump(events, f, indent=0)
        f.write("\n")
