"""Key metrics of an `ncu --set full` report as JSON (for profiles/ncu_summary.json).

usage: python tools/ncu_summary.py report.ncu-rep paths_per_launch [name]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]
# executed FP32 operations (thread-level, predicated on): paired ops count two
# lanes, an FMA two flops
FLOPS = {"fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}
UNIT = {"dram__bytes_read.sum": None, "dram__bytes_write.sum": None}


def main():
    rep, paths = sys.argv[1], int(sys.argv[2])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        ent = {k: d.get(k) for k in KEYS}
        rd = float(ent["dram__bytes_read.sum"].replace(",", ""))
        wr = float(ent["dram__bytes_write.sum"].replace(",", ""))
        ent["paths_per_launch"] = paths
        ent["dram_bytes_per_path"] = (rd + wr) / paths
        ops = {o: d.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum") for o in FLOPS}
        if all(v not in (None, "") for v in ops.values()):
            ent["executed_fp32_ops"] = {o: float(v.replace(",", "")) for o, v in ops.items()}
            ent["executed_flop_per_path"] = sum(FLOPS[o] * v for o, v in ent["executed_fp32_ops"].items()) / paths
        ent["kernel"] = d["Kernel Name"]
        res[d["Kernel Name"]] = ent
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
