"""Print the headline ncu metrics of a report (raw page), one kernel per row.

    python tools/ncu_metrics.py prof.ncu-rep [playouts_per_launch]
"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
        "sm__sass_branch_targets_threads_divergent.sum", "sm__sass_branch_targets_threads_uniform.sum"]


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in WANT or h == "Kernel Name":
                d[h] = (vals[i], units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    n = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for d in metrics(rep):
        for k in ["Kernel Name"] + WANT:
            if k in d:
                print("%-70s %s %s" % (k, d[k][0], d[k][1]))
        if n and "smsp__inst_executed.sum" in d:
            wi = float(d["smsp__inst_executed.sum"][0].replace(",", ""))
            r = float(d["smsp__thread_inst_executed_per_inst_executed.ratio"][0])
            print("thread-inst per playout: %.1f   warp-inst per playout: %.2f   eta_SIMT: %.3f" % (wi * r / n, wi / n, r / 32))
