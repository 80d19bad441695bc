#!/usr/bin/env python
"""Markdown results table from bench.py JSON lines.

    python scripts/results_table.py profiles/r2_end/bench_*.json
"""
import json
import sys


def row(path):
    d = json.loads(open(path).read().strip().split("\n")[-1])
    if d.get("impl") == "reference":
        return None
    r = d.get("roofline") or {}
    cfg = d["config"]["workload"].split(":")[0]
    tk = r.get("t_kernel_ms")
    floor = r.get("t_floor_ms")
    frac = r.get("frac")
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    kern = r.get("kernel", "?")
    return (f"| {cfg} | {d['n_gpus']} | {kern} | {d['value']:.3g} | {d['ms_per_step']:.3f} | "
            f"{tk:.3f} | " if tk is not None else f"| {cfg} | {d['n_gpus']} | {kern} | {d['value']:.3g} | "
            f"{d['ms_per_step']:.3f} | - | ") + \
        (f"{floor:.3f} | " if floor else "- | ") + \
        (f"{frac:.3f} ({r.get('bound')}, {r.get('unit')}) | " if frac is not None else "- | ") + \
        (f"{r.get('frac_vs_paper_loop', float('nan')):.2f} | ") + \
        (f"{e2e.get('value', float('nan')):.3g} | " if e2e else "- | ") + \
        (f"{cpu.get('value', float('nan')):.3g} ({cpu.get('cores')} cores) |" if cpu else "- |")


def main(paths):
    print("| Cfg | G | kernel | hashes/s | ms/step | t_kernel ms | t_floor ms | frac (bound, unit) | "
          "× paper-loop bound | e2e hashes/s | oracle hashes/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        r = row(p)
        if r:
            print(r)


if __name__ == "__main__":
    main(sys.argv[1:])
