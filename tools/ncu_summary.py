"""Summarise an ncu report (raw page) into the metrics this project's rooflines use.

    python tools/ncu_summary.py gpurun_out/far_c4.ncu-rep [--flops-per-launch F] [--bytes-per-launch B]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.avg.per_cycle_active", "sm__inst_executed.avg.per_cycle_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_wait", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units, data = r[0], r[1], r[2:]
    return [{h: (v, u) for h, u, v in zip(hdr, units, d)} for d in data]


def main():
    rep = sys.argv[1]
    res = []
    for d in rows(rep):
        e = {}
        for k in d:
            if any(k.startswith(x) for x in KEYS) or "pipe_fp64" in k or "stall" in k and "pct" in k:
                e[k] = d[k][0] + (f" {d[k][1]}" if d[k][1] else "")
        res.append(e)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
