"""Per-source-line executed-instruction counts (and stall-sample share) from an
ncu report built with -lineinfo, in source order -- the dynamic instruction
budget of a kernel by line.

    python scripts/ncu_lines.py gpurun_out/x.ncu-rep [min_pct] [kernel-regex]
"""
import csv
import io
import subprocess
import sys


def main(path, min_pct=0.2, kernel_regex=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    data, fname, head = [], "?", None
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
        if head is None or not r[0].isdigit():
            continue
        try:
            n, st = float(r[ii] or 0), float(r[si] or 0)
        except ValueError:
            continue
        if n or st:
            data.append((fname, int(r[0]), n, st, r[1].strip()[:90]))
    tot = sum(d[2] for d in data) or 1
    tst = sum(d[3] for d in data) or 1
    for f, ln, n, st, src in sorted(data, key=lambda d: (d[0], d[1])):
        if 100 * n / tot >= min_pct or 100 * st / tst >= min_pct:
            print(f"{f[:20]:20s}:{ln:4d} inst {100 * n / tot:5.1f}%  stall {100 * st / tst:5.1f}%  {src}")
    print(f"total executed instructions {tot:.4g}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.2, sys.argv[3] if len(sys.argv) > 3 else None)
