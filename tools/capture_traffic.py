"""DRAM traffic of each bench config's walk kernel, stamped with the source hash.

On a GPU box (gpurun), from the repo root:

    python tools/capture_traffic.py run [c1 c2 ...]     # writes gpurun_out/ncu_traffic.json

then here:

    cp gpurun_out/ncu_traffic.json profiles/

For every config: one plain run of `tools/profile_walk.py --config cN --tune
--launches 1` (must exit 0), then the same command under ncu collecting
dram__bytes_read.sum + dram__bytes_write.sum + gpu__time_duration.sum of the
timed walk-kernel launch (NVTX range "timed", so the tuner's launches are not
captured).  The result records the moves of that launch and
paper_2107_11983_b200.build.source_hash(): bench.py reports a capture whose
stamp differs from the library it runs as stale (roofline.traffic_stamp).
"""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def parse_csv(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = {}
    for r in rows[1:]:
        out[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    return out


def run(configs):
    from paper_2107_11983_b200.build import source_hash
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    sha = source_hash()
    out = {"about": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one walk-kernel launch per "
                    "config at its tuned grid; src_sha = paper_2107_11983_b200.build.source_hash() of the "
                    "library captured (bench.py reports a capture of other sources as stale). Written by "
                    "tools/capture_traffic.py.", "configs": {}}
    for key in configs:
        cmd = [sys.executable, os.path.join(ROOT, "tools", "profile_walk.py"), "--config", key, "--tune",
               "--launches", "1"] + (["--counts"] if key == "c2" else [])
        plain = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        log = plain.stdout + plain.stderr
        if plain.returncode != 0:
            print(f"{key}: plain run failed, not profiled\n{log[-2000:]}", flush=True)
            continue
        m = re.search(r"launch 0: (\d+) moves", log)
        moves = int(m.group(1))
        csv_path = os.path.join(ROOT, "gpurun_out", f"traffic_{key}.csv")
        prof = subprocess.run(["ncu", "--clock-control", "none", "--nvtx", "--nvtx-include", "timed/",
                               "--metrics", METRICS, "-k", "regex:walk_kernel", "-c", "1", "--csv",
                               "--log-file", csv_path] + cmd, capture_output=True, text=True, cwd=ROOT)
        if prof.returncode != 0 or not os.path.exists(csv_path):
            print(f"{key}: ncu failed\n{(prof.stdout + prof.stderr)[-2000:]}", flush=True)
            continue
        v = parse_csv(csv_path)
        b = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        out["configs"][key] = {"bytes": b, "read": v["dram__bytes_read.sum"], "write": v["dram__bytes_write.sum"],
                               "moves": moves, "bytes_per_move": b / moves,
                               "ncu_seconds": v["gpu__time_duration.sum"], "src_sha": sha}
        print(key, json.dumps(out["configs"][key]), flush=True)
        with open(os.path.join(ROOT, "gpurun_out", "ncu_traffic.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    if len(sys.argv) >= 2 and sys.argv[1] == "run":
        run(sys.argv[2:] or ["c1", "c2", "c3", "c4", "c5", "g1", "g2", "g3"])
    else:
        print(__doc__)
