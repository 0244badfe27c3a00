"""Turn a gpurun_out/ capture into the committed evidence under profiles/.

    python tools/summarize_profiles.py <round-tag> [gpurun_out]

Writes
  profiles/<tag>_launches.txt   per-launch device time of ONE evaluation (ncu
                                gpu__time_duration, --clock-control none; cold-cache and
                                serialised, so compare shares, not absolutes)
  profiles/<tag>_ncu_<kernel>.txt   key counters + stall breakdown of each kernel in
                                prof*.ncu-rep (ncu --set full)
  profiles/traffic.json         dram bytes per launch of the captured kernels, keyed
                                "B:<KIND>" for bench.py's roofline.traffic
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

KIND_OF = {"k_p2p": "P2P", "k_m2l_phase_a": "M2L_A", "k_m2l_phase_b": "M2L_B", "k_p2m": "P2M", "k_l2p": "L2P",
           "k_transfer_warp<5, 1>": "M2M", "k_transfer_warp<5, 0>": "L2L", "k_gather": "GATHER"}


def short(name):
    n = name.replace("fmmgpu::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return n.split("(")[0].replace("void ", "").rsplit("::", 1)[-1]


# ---- launch list
lp = os.path.join(src, "launches.csv")
if os.path.exists(lp):
    rows = list(csv.reader(open(lp)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
    ends = [i for i, (k, _) in enumerate(data) if "k_gather" in k]
    one = data[ends[-2] + 1:ends[-1] + 1] if len(ends) >= 2 else data
    tot = sum(v for _, v in one)
    with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
        f.write(f"# one evaluation, config B (N=10M, h=7, l=5); ncu gpu__time_duration.sum, --clock-control none\n")
        f.write(f"# serialised sum {tot / 1e6:.3f} ms over {len(one)} launches\n")
        for k, v in one:
            f.write(f"{v / 1e3:10.1f} us  {100 * v / tot:5.1f}%  {short(k)}\n")
    print(open(os.path.join(out_dir, f"{tag}_launches.txt")).read())

# ---- full captures
traffic_path = os.path.join(out_dir, "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Theoretical Occupancy", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum"]
for rep in sorted(p for p in os.listdir(src) if p.endswith(".ncu-rep")):
    path = os.path.join(src, rep)
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    d = list(csv.reader(io.StringIO(det)))
    r = list(csv.reader(io.StringIO(raw)))
    if len(d) < 2 or len(r) < 3:
        continue
    dh, rh, units = d[0], r[0], r[1]
    by_id = {}
    for row in d[1:]:
        by_id.setdefault(row[dh.index("ID")], []).append(row)
    for row in r[2:]:
        kid = row[rh.index("ID")]
        name = short(row[rh.index("Kernel Name")])
        lines = [f"# ncu --set full --clock-control none ({rep}, launch id {kid})", f"kernel: {name}"]
        for dr in by_id.get(kid, []):
            if dr[dh.index("Metric Name")] in WANT:
                lines.append(f"  {dr[dh.index('Metric Name')]:36s} {dr[dh.index('Metric Value')]:>14s} "
                             f"{dr[dh.index('Metric Unit')]}")
        for k in RAW:
            if k in rh:
                lines.append(f"  {k:72s} {row[rh.index(k)]} {units[rh.index(k)]}")
        stalls = []
        for k in rh:
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(row[rh.index(k)].replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        lines.append("  stall breakdown (pc sampling):")
        for s, k in sorted(stalls, reverse=True)[:8]:
            lines.append(f"    {k:40s} {100 * s / tot:5.1f} %")
        fname = os.path.join(out_dir, f"{tag}_ncu_{name.replace('<', '_').replace('>', '').replace(', ', '_')}_{kid}.txt")
        open(fname, "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
        try:
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            byts = sum(float(row[rh.index(m)].replace(",", "")) * sc[units[rh.index(m)]]
                       for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            for key, kind in KIND_OF.items():
                if name.startswith(key):
                    traffic[f"B:{kind}:{rep}:{kid}"] = byts
                    if kind == "P2P":
                        traffic["B:P2P"] = byts
        except (ValueError, KeyError):
            pass
json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
