"""Summarise an ncu report's details page (key metrics) -- run locally on gpurun_out/*.ncu-rep."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Compute (SM) Throughput", "Executed Instructions", "Mem Busy", "Max Bandwidth", "Block Limit Registers",
        "Block Limit Shared Mem", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Dynamic Shared Memory Per Block"]


def main(path, raw_metrics=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    seen = set()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[mi] in WANT and (r[ki], r[mi]) not in seen:
            seen.add((r[ki], r[mi]))
            print(f"{r[ki][:40]:40s} {r[mi]:38s} {r[vi]:>14s} {r[ui]}")
    if raw_metrics:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[0]
        for m in raw_metrics:
            if m in h:
                i = h.index(m)
                for r in rows[2:]:
                    print(f"{m:50s} {r[i]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
