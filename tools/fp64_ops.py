"""Executed FP64 operations per operator of one evaluation, from an ncu CSV of the
thread-level DFMA / DADD / DMUL counters and the warp-level DMMA counter
(tools/gpu/gpu_r02y.sh) -> profiles/fp64_ops.json, which bench.py reads to report each
operator's EXECUTED-flop fraction beside the reference-ledger fraction (the factored P2M /
L2P kernels execute fewer flops than the ledger counts; M2L's DMMA executes padding).

    python tools/fp64_ops.py gpurun_out/r02y/fp64_ops.csv B
flops: 2 per DFMA, 1 per DADD / DMUL, 512 per DMMA m8n8k4 (8 x 8 x 4 FMAs).
"""
import csv
import json
import os
import sys

src = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "B"
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launch = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(int(r[ii]), {"name": r[ki]})
    try:
        d[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:  # n/a
        pass


def kind(name):
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    if "k_p2m" in n:
        return "P2M"
    if "k_l2p" in n:
        return "L2P"
    if "k_transfer" in n:
        return "M2M" if ", 1>" in n or ", true>" in n else "L2L"
    if "k_m2l_phase" in n:
        return "M2L"
    if "k_p2p" in n:
        return "P2P"
    if "k_gather" in n:
        return "GATHER"
    return None


out = {}
for d in launch.values():
    k = kind(d["name"])
    if k is None:
        continue
    o = out.setdefault(k, {"dfma": 0.0, "dadd": 0.0, "dmul": 0.0, "dmma": 0.0, "ms": 0.0, "launches": 0})
    o["dfma"] += d.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
    o["dadd"] += d.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
    o["dmul"] += d.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
    o["dmma"] += d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)
    o["ms"] += d.get("gpu__time_duration.sum", 0.0) / 1e6
    o["launches"] += 1
for o in out.values():
    o["exec_flops"] = 2 * o["dfma"] + o["dadd"] + o["dmul"] + 512 * o["dmma"]
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "fp64_ops.json")
allc = json.load(open(p)) if os.path.exists(p) else {}
allc[cfg] = out
allc["note"] = __doc__.split("\n\n")[0].replace("\n", " ")
json.dump(allc, open(p, "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))
