"""Summarise an ncu report (raw page) per kernel: time, DRAM bytes, pipes, stalls.
    python tools/ncu_summary.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        name = r[ki]
        if pat and not pat.search(name):
            continue
        print("==", name[:100])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"   {w:70s} {r[i]} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith(STALL) and not h.endswith("not_issued") and r[i] not in ("", "0"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len(STALL):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        print("   stalls:", ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in stalls[:7]))


if __name__ == "__main__":
    main()
