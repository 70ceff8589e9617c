"""Summarise an ncu --set full report into a small JSON for profiles/ (the
judged evidence: eta_SIMT, issue utilisation, pipe utilisation, stall mix,
thread-instructions per playout, DRAM traffic).

    python tools/summarize_profile.py REP.ncu-rep PLAYOUTS_PER_LAUNCH OUT.json [--unit]

--unit also writes profiles/roofline_unit.json (the per-playout instruction
count bench.py's roofline uses) when the report is the bench workload's
refill kernel.
"""

import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__thread_inst_executed.sum": "thread_inst",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__sass_average_branch_targets_threads_uniform.pct": "branch_targets_uniform_pct",
    "smsp__sass_branch_targets_threads_divergent.sum": "branch_targets_divergent",
    "smsp__inst_executed_op_branch.sum": "branch_inst",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "pipe_uniform_pct",
}


def to_float(v, unit):
    x = float(v.replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}
    return x * scale.get(unit, 1.0)


def summarize(rep, playouts):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"report": rep, "kernel": vals[hdr.index("Kernel Name")]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h in KEYS:
            res[KEYS[h]] = to_float(vals[i], units[i])
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    res["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v}
    res["eta_simt"] = res["threads_per_inst"] / 32.0
    res["playouts_per_launch"] = playouts
    res["thread_inst_per_playout"] = res["warp_inst"] * res["threads_per_inst"] / playouts
    res["warp_inst_per_playout"] = res["warp_inst"] / playouts
    res["dram_bytes_per_launch"] = res.get("dram_read", 0) + res.get("dram_write", 0)
    res["playouts_per_s_under_ncu"] = playouts / res["duration"]
    return res


def main():
    rep, n, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    res = summarize(rep, n)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
    if "--unit" in sys.argv:
        unit = {"workload": "fixtures/c2_d1.json", "kernel": res["kernel"],
                "thread_inst_per_playout": res["thread_inst_per_playout"],
                "dram_bytes_per_launch": res["dram_bytes_per_launch"],
                "eta_simt": res["eta_simt"], "issue_active_pct": res["issue_active_pct"],
                "pipe_alu_pct": res.get("pipe_alu_pct"), "pipe_xu_pct": res.get("pipe_xu_pct"),
                "pipe_fma_pct": res.get("pipe_fma_pct"),
                "source": os.path.relpath(os.path.abspath(out), os.path.dirname(os.path.dirname(os.path.abspath(__file__))))}
        with open("profiles/roofline_unit.json", "w") as f:
            json.dump(unit, f, indent=1)


if __name__ == "__main__":
    main()
