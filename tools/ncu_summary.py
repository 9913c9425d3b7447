#!/usr/bin/env python
"""Summarise an ncu report: per kernel duration, DRAM/L2/SM throughput,
occupancy, issue activity and the top warp-stall reasons."""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]   # names, units, one row per launch


def main(rep):
    hdr, units, rows = raw(rep)
    unit = dict(zip(hdr, units))
    for v in rows:
        d = dict(zip(hdr, v))
        name = d.get("Kernel Name", "?")[:70]
        def g(k, default="n/a"):
            return d.get(k, default)
        print(f"== {name}")
        for k, lab in [("gpu__time_duration.sum", "duration"),
                       ("dram__bytes_read.sum", "dram read"),
                       ("dram__bytes_write.sum", "dram write"),
                       ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
                       ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
                       ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
                       ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
                       ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
                       ("launch__registers_per_thread", "regs"),
                       ("launch__grid_size", "grid"), ("launch__block_size", "block"),
                       ("smsp__inst_executed.sum", "warp instr")]:
            print(f"   {lab:16s} {g(k)} {unit.get(k, '')}")
        st = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls/issue:", ", ".join(f"{n}={x:.2f}" for x, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
