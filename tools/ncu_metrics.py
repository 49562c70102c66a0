"""Key metrics + stall breakdown of the kernels in an ncu report.
    python tools/ncu_metrics.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for row in r[2:]:
        name = row[h.index("Kernel Name")][:60]
        print("==", name)
        for w in WANT:
            if w in h:
                print(f"  {w:70s} {row[h.index(w)]}")
        st = []
        for i, x in enumerate(h):
            if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(row[i]), x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:9]))


if __name__ == "__main__":
    main()
