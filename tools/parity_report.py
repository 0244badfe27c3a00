"""Runs tests/config_parity.py for the named configs and writes one JSON per config
(default gpurun_out/parity_<name>.json): the evidence behind BASELINE.md §4's parity
columns.  python tools/parity_report.py A H7 B C D [E]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import config_parity  # noqa: E402
import paper_1206_0115_b200 as P  # noqa: E402


def main():
    names = sys.argv[1:] or ["A", "H7", "B", "C", "D"]
    out = os.environ.get("PARITY_OUT", os.path.join(ROOT, "gpurun_out"))
    os.makedirs(out, exist_ok=True)
    for name in names:
        res = config_parity.run(name, P, lists=name != "E")
        res["host_cpus"] = os.cpu_count()
        with open(os.path.join(out, f"parity_{name}.json"), "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
