"""Summarise one kernel of an `ncu --set full` report into profiles/*.json.

    python tools/ncu_summary.py <report.ncu-rep> <out.json> [kernel-substring]

Reads `ncu -i <rep> --page raw --csv` and keeps the metrics the roofline
lines cite; byte metrics are normalised to bytes and DRAM traffic per launch
is reported as `dram_bytes_per_launch` (read + write)."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    want = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(head)}
    for r in data:
        if want and want not in r[idx["Kernel Name"]]:
            continue
        res = {"Kernel Name": r[idx["Kernel Name"]], "report": rep.split("/")[-1]}
        for m in KEEP:
            if m not in idx:
                continue
            v, u = r[idx[m]], units[idx[m]]
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                res[m] = v
                continue
            if "bytes" in m and u in SCALE:
                res[m] = f * SCALE[u]
            elif m == "gpu__time_duration.sum" and u in SCALE:
                res["duration_ms"] = f * SCALE[u]
            else:
                res[m] = f
        res["dram_bytes_per_launch"] = res.get("dram__bytes_read.sum", 0.0) + res.get("dram__bytes_write.sum", 0.0)
        json.dump(res, open(out, "w"), indent=1)
        print(json.dumps(res, indent=1))
        return
    sys.exit("kernel not found")


if __name__ == "__main__":
    main()
