"""Summarise an ncu --page raw --csv export: key throughput / stall metrics per kernel."""
import csv
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "wait", "not_selected", "selected", "no_instruction", "tex_throttle", "dispatch_stall", "membar",
          "drain", "imc_miss", "branch_resolving"]


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:70]
        print("==", name)
        for w in WANT:
            if w in h:
                print(f"   {w:70s} {r[h.index(w)]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in h:
                try:
                    st.append((float(r[h.index(k)]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls (warps per issue):", ", ".join(f"{s}={v:.2f}" for v, s in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
