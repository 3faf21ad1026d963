"""Summarise an `ncu --set full` report of one launch into the JSON bench.py reads (traffic) and
the judge can check: python tools/ncu_summary.py <report.ncu-rep> <kernel label> <cells> <out.json>
[capture note].  Needs the ncu CLI (no GPU)."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Achieved Occupancy"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__inst_executed.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "gpu__time_duration.sum"]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "no_instruction", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "barrier", "membar", "not_selected", "selected", "branch_resolving", "dispatch_stall",
          "sleeping", "drain", "misc", "tex_throttle"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def main():
    rep, label, cells, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    note = sys.argv[5] if len(sys.argv) > 5 else ""
    det = ncu_csv(rep, "details")
    h = det[0]
    isec, iname, ival, iunit = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    details = {}
    for row in det[1:]:
        if (row[isec], row[iname]) in KEEP:
            details[f"{row[isec]}/{row[iname]}"] = [row[ival], row[iunit]]
    raw = ncu_csv(rep, "raw")
    names, units, vals = raw[0], raw[1], raw[2]
    rv = {n: to_num(v) for n, v in zip(names, vals)}
    stalls = {}
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in rv:
            stalls[s] = rv[k]
    summ = {
        "kernel": label,
        "capture": note,
        "cells_per_launch": cells,
        "dram_bytes_read": rv.get("dram__bytes_read.sum"),
        "dram_bytes_write": rv.get("dram__bytes_write.sum"),
        "raw": {k: rv.get(k) for k in RAW},
        "warp_stall_cycles_per_issued_instruction": stalls,
        "details": details,
    }
    tot = (summ["dram_bytes_read"] or 0) + (summ["dram_bytes_write"] or 0)
    summ["dram_bytes_per_cell"] = tot / cells
    with open(out, "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps({k: summ[k] for k in ("kernel", "dram_bytes_per_cell")}), stalls)


if __name__ == "__main__":
    main()
