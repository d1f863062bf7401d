"""Print the key metrics of an ncu report:  python tools/ncu_summary.py <rep> [more keys...]"""
import csv
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        for i, x in enumerate(h):
            if x in KEYS or x in extra:
                print(f"{x} = {v[i]} {u[i]}")
        for i, x in enumerate(h):
            if "warps_issue_stalled" in x and x.endswith("per_issue_active.ratio"):
                try:
                    if float(v[i]) > 0.25:
                        print(f"{x.replace('smsp__average_warps_issue_stalled_', 'stall:')} = {v[i]}")
                except ValueError:
                    pass
        print("--")


if __name__ == "__main__":
    main()
