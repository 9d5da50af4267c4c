"""Key metrics of one kernel from an ncu report (raw page), for profiles/ summaries.
Usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["short_scoreboard", "wait", "long_scoreboard", "math_pipe_throttle", "mio_throttle", "barrier", "not_selected",
          "selected", "dispatch_stall", "no_instruction", "branch_resolving", "lg_throttle", "membar", "drain", "tex_throttle"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:80]}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u[k]}")
        st = {s: d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") for s in STALLS}
        print("  stalls per issue:", ", ".join(f"{s} {float(v):.2f}" for s, v in st.items() if v and float(v) > 0.05))


if __name__ == "__main__":
    main(sys.argv[1])
