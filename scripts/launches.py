"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel count, total and mean time."""
import collections
import csv
import sys


def main(path, skip_first=0):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    head = rows[h]
    ki, ni, vi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) == len(head) and r[ni] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0][:70]
            v = float(r[vi].replace(",", ""))
            c, t = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, t + v)
    tot = sum(t for c, t in agg.values())
    for name, (c, t) in agg.items():
        print(f"{name:72s} n={c:4d} total={t / 1e6:9.3f} ms mean={t / c / 1e3:10.1f} us  {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
