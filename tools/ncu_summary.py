"""Summarize an ncu report (raw page) into the numbers profiles/ records."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": dict(zip(hdr, vals)).get("Kernel Name", "")[:120]}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                d[h] = f"{v} {u}".strip()
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    if float(v) > 0.05:
                        d["stall:" + h.split("stalled_")[1].split("_per_issue")[0]] = round(float(v), 3)
                except ValueError:
                    pass
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))
