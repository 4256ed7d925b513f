"""Copies the ncu evidence of a round into profiles/ (tracked):

    python tools/make_profiles.py --round 1 --config c2 \
        --launches gpurun_out/launches_c2.csv --full gpurun_out/prof_c2.ncu-rep

* <round>_<config>_launches.csv      every kernel launch of the bench command
                                     (gpu__time_duration, cold, serialised)
* <round>_<config>_launch_share.json per-kernel totals and the walk kernel's share
* <round>_<config>_walk_kernel.json  summary of the --set full capture
(profiles/ncu_traffic.json, the stamped per-config DRAM bytes bench.py reads,
comes from tools/capture_traffic.py.)
"""
import argparse
import csv
import json
import os
import shutil
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from ncu_summary import summarise  # noqa: E402


def launch_share(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:60]
        tot[name] += v * scale
        cnt[name] += 1
    total = sum(tot.values())
    out = sorted(({"kernel": k, "launches": cnt[k], "total_us": t, "share": t / total}
                  for k, t in tot.items()), key=lambda d: -d["total_us"])
    return {"total_us": total, "kernels": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    tag = f"r{args.round:02d}_{args.config}"
    if args.launches:
        shutil.copy(args.launches, os.path.join(prof, f"{tag}_launches.csv"))
        with open(os.path.join(prof, f"{tag}_launch_share.json"), "w") as f:
            json.dump(launch_share(args.launches), f, indent=1)
    if args.full:
        s = summarise(args.full)
        with open(os.path.join(prof, f"{tag}_walk_kernel.json"), "w") as f:
            json.dump(s, f, indent=1)
    print("ok", tag)


if __name__ == "__main__":
    main()
