"""Per-source-line warp-stall samples from an ncu report (kernels built with -lineinfo).

    python scripts/ncu_source.py gpurun_out/x.ncu-rep [top] [kernel-regex] [--lines A-B]

Prints the top source lines by stall samples with their instruction counts and
their three largest stall reasons; --lines A-B also sums the samples of
hash_bitslice.cu's lines A..B (a phase of the kernel) by reason.
"""
import csv
import io
import subprocess
import sys


def main(path, top=40, kernel_regex=None, span=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    data, tot, fname, head = [], 0.0, "?", None
    span_tot, span_reasons = 0.0, {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path" or r[0] == "File Name":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            head = r
            si = head.index("Warp Stall Sampling (All Samples)")
            ii = head.index("Instructions Executed")
            reasons = [(i, h[len("stall_"):]) for i, h in enumerate(head) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if head is None or r[0] in ("Function Name", "Kernel Name"):
            continue
        if r[0]:                                # a source line (aggregate of its SASS)
            try:
                s = float(r[si] or 0)
            except ValueError:
                continue
            tot += s
            rs = sorted(((float(r[i] or 0), n) for i, n in reasons), reverse=True)
            data.append((s, f"{fname}:{r[0]}", r[1].strip()[:90], r[ii], rs[:3]))
            if span and fname == "hash_bitslice.cu" and span[0] <= int(r[0]) <= span[1]:
                span_tot += s
                for v, n in rs:
                    span_reasons[n] = span_reasons.get(n, 0.0) + v
    data.sort(key=lambda x: -x[0])
    for s, loc, src, ie, rs in data[:top]:
        why = " ".join(f"{n}={100 * v / max(s, 1):.0f}%" for v, n in rs if v > 0)
        print(f"{100 * s / max(tot, 1):5.1f}% {loc:22s} inst={ie:>11s}  {src}\n{'':30s}[{why}]")
    if span:
        print(f"lines {span[0]}-{span[1]}: {100 * span_tot / max(tot, 1):.1f}% of samples: " +
              " ".join(f"{n}={100 * v / max(span_tot, 1):.0f}%" for n, v in
                       sorted(span_reasons.items(), key=lambda x: -x[1]) if v > 0))


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--lines")]
    span = None
    for a in sys.argv[1:]:
        if a.startswith("--lines="):
            lo, hi = a.split("=", 1)[1].split("-")
            span = (int(lo), int(hi))
    main(args[0], int(args[1]) if len(args) > 1 else 40, args[2] if len(args) > 2 else None, span)
