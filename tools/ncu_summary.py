"""Summarise an ncu report (raw page) into the numbers DESIGN.md / bench use."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "dram__sectors_read.sum", "dram__sectors_write.sum"]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:80]}
        for i, k in enumerate(h):
            if k in KEYS or ("smsp__average_warp_latency_issue_stalled" in k and k.endswith("pct")) \
                    or ("smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")):
                try:
                    d[k] = float(v[i].replace(",", ""))
                except ValueError:
                    d[k] = v[i]
                d[k + "@unit"] = u[i]
        res.append(d)
    return res


if __name__ == "__main__":
    for r in summarise(sys.argv[1]):
        stalls = {k: r[k] for k in r if "pcsamp" in k and not k.endswith("@unit") and r[k]}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        base = {k: (r[k], r.get(k + "@unit")) for k in r if k in KEYS}
        print(json.dumps({"kernel": r["kernel"], "metrics": base, "top_stall_samples": top}, indent=1))
