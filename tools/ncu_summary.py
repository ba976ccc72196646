"""Per-kernel summary of an ncu --set full report (the metrics DESIGN.md §6
quotes): duration, DRAM / SM throughput, IPC, issue slots, occupancy,
registers, cache hit rates.

    python tools/ncu_summary.py report.ncu-rep > summary.txt
"""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ii, ui = hdr.index("ID"), hdr.index("Metric Unit")
    cur = None
    for r in rows[1:]:
        if r[mi] not in WANT:
            continue
        key = (r[ii], r[ki])
        if key != cur:
            print(f"\n[{r[ii]}] {r[ki][:110]}")
            cur = key
        print(f"    {r[mi]:32s} {r[vi]:>10s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
