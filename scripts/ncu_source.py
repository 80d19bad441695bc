"""Per-source-line warp-stall samples from an ncu report (kernels built with -lineinfo).

    python scripts/ncu_source.py gpurun_out/x.ncu-rep [top] [kernel-regex]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40, kernel_regex=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    data, tot, fname, head = [], 0.0, "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            head = r
            si = head.index("Warp Stall Sampling (All Samples)")
            ii = head.index("Instructions Executed")
            continue
        if head is None or r[0] in ("Function Name", "Kernel Name"):
            continue
        if r[0]:                                # a source line (aggregate of its SASS)
            try:
                s = float(r[si] or 0)
            except ValueError:
                continue
            tot += s
            data.append((s, f"{fname}:{r[0]}", r[1].strip()[:100], r[ii]))
    data.sort(reverse=True)
    for s, loc, src, ie in data[:top]:
        print(f"{100 * s / max(tot, 1):5.1f}% {loc:22s} inst={ie:>11s}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)
