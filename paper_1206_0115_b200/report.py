"""The reference's output formats (bench.cpp:504-584), so its tooling can diff results:

* ``write_results_csv``  results.csv, header ``id,x,y,z,w,potential,fx,fy,fz`` and %.17g
  (round-trip) values (bench.cpp:504-514);
* ``write_summary_json`` summary.json with the reference's keys and nesting: config,
  timings, accuracy, compression, flop_costs, ledger (per kind and per level, from the
  device's ledger rows), breakdown, occupancy over the device spans (bench.cpp:516-584);
* ``write_chrome_trace`` trace.json in the reference's Chrome "ph":"X" format
  (runtime.cpp:277-292) from the device spans of FmmContext.trace_spans (one span per
  operator launch; tid = CUDA stream: 0 far field, 1 near field, 2 coarse M2L + L2L).
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


def ledger_totals(rows: dict) -> dict:
    """Per-kind totals of ledger rows ({"work", "flops"}: (7, height) arrays)."""
    return {k: int(np.asarray(rows["flops"])[i].sum()) for i, k in enumerate(KINDS)}


def format_breakdown(rows: dict) -> str:
    """format_breakdown (bench.cpp:183-218): the level x operator percentage grid."""
    work = np.asarray(rows["work"], dtype=np.uint64)
    flops = np.asarray(rows["flops"], dtype=np.uint64)
    total = int(flops.sum())

    def percent(f, w):
        if w == 0 and f == 0:
            return " %9s" % "-"
        return " %8.2f%%" % (100.0 * float(f) / float(total) if total else 0.0)

    out = "level" + "".join(" %9s" % k for k in KINDS) + "\n"
    for v in range(work.shape[1]):
        if not (work[:, v].any() or flops[:, v].any()):
            continue
        out += "%5d" % v + "".join(percent(int(flops[k, v]), int(work[k, v])) for k in range(7)) + "\n"
    out += "total" + "".join(percent(int(flops[k].sum()), int(work[k].sum())) for k in range(7)) + "\n"
    return out


def occupancy(spans, wall_ms: float | None = None, workers: int = 2) -> dict:
    """occupancy (runtime.cpp:260-276) over device spans: busy fraction per CUDA stream
    (the reference: per worker thread) and each kind's share of the busy time."""
    workers = max([workers] + [sp[2] + 1 for sp in spans])  # streams: 0 far, 1 near, 2 coarse far
    busy = [0.0] * workers
    share = {k: 0.0 for k in KINDS}
    if wall_ms is None:
        wall_ms = max((t1 for *_, t1 in spans), default=0.0) - min((t0 for *_, t0, _ in spans), default=0.0)
    total = 0.0
    for kind, _level, stream, t0, t1 in spans:
        busy[stream] += t1 - t0
        share[kind] += t1 - t0
        total += t1 - t0
    return {"busy_fraction": [b / wall_ms if wall_ms > 0 else 0.0 for b in busy],
            "kind_share": {k: (v / total if total > 0 else 0.0) for k, v in share.items()}}


def write_summary_json(path: str, *, cfg, n: int, setup_seconds: float, exec_seconds: float,
                       wall_seconds: float, compression: dict, ledger_rows: dict, eps=None,
                       spans=None, workers: int = 2, policy: str = "device-streams", check: int = 0,
                       device_ms: dict | None = None) -> dict:
    """summary.json with the reference writer's keys and nesting (bench.cpp:516-584):
    config, timings, accuracy, compression, flop_costs, ledger (per kind: work, flops and
    per-level rows with share_percent; total_flops), breakdown, occupancy. The device
    runs on two CUDA streams instead of worker threads: workers = 2, policy
    "device-streams", occupancy from the per-launch device spans (FmmContext.trace_spans)."""
    work = np.asarray(ledger_rows["work"], dtype=np.uint64)
    flops = np.asarray(ledger_rows["flops"], dtype=np.uint64)
    total = int(flops.sum())
    j = {"config": {"n": n, "dist": cfg.dist, "height": cfg.height, "acc": cfg.acc,
                    "group_size": cfg.group_size, "workers": workers, "policy": policy, "seed": cfg.seed,
                    "check": check, "dry_run": False},
         "timings": {"setup_seconds": setup_seconds, "exec_seconds": exec_seconds, "wall_seconds": wall_seconds}}
    if eps is not None and eps[0] >= 0:
        j["accuracy"] = {"eps_l2_potential": float(eps[0]), "eps_l2_force": float(eps[1])}
    j["compression"] = {"order": cfg.acc, "eps": 10.0 ** -cfg.acc,
                        "ranks": [int(r) for r in compression["ranks"]],
                        "multiplicity": [int(m) for m in compression["multiplicity"]],
                        "weighted_mean_rank": float(compression["weighted_mean_rank"])}
    j["flop_costs"] = flop_costs(cfg.acc)
    ledger = {}
    for k, name in enumerate(KINDS):
        levels = [{"level": v, "work": int(work[k, v]), "flops": int(flops[k, v]),
                   "share_percent": 100.0 * float(flops[k, v]) / float(total) if total else 0.0}
                  for v in range(work.shape[1]) if work[k, v] or flops[k, v]]
        ledger[name] = {"work": int(work[k].sum()), "flops": int(flops[k].sum()), "levels": levels}
    ledger["total_flops"] = total
    j["ledger"] = ledger
    j["breakdown"] = format_breakdown(ledger_rows)
    if spans is not None:
        j["occupancy"] = occupancy(spans, workers=workers)
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
