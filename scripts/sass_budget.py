#!/usr/bin/env python
"""Static SASS instruction budget of a hot loop, by source region -- the
committed evidence behind the roofline constants bench.py uses.

Disassembles one kernel of a built object (cuobjdump -xelf + nvdisasm -g, so
every instruction carries the source line it came from, inlined helpers
included), takes the address range spanned by the instructions of the loop's
own source lines, and counts the instructions in that range by region:

    python scripts/sass_budget.py bitslice [--kernel-match ILi6ELi2ELb0ELi512] [--out profiles/r2_sass]

Regions are source-line ranges of paper_1602_08393_b200/csrc/*.cu located by
marker strings (so the script survives edits that move lines).  Writes
<out>.json (counts) and <out>.txt (the annotated SASS listing of the range).
"""
import argparse
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1602_08393_b200", "csrc")
BUILD = os.path.join(ROOT, "paper_1602_08393_b200", "build")


def line_of(path, marker, start=1):
    for i, l in enumerate(open(path).read().split("\n"), 1):
        if i >= start and marker in l:
            return i
    raise SystemExit(f"marker not found in {path}: {marker!r}")


def block_end(path, start):
    """Line of the brace closing the block opened on or after `start`."""
    depth, opened = 0, False
    for i, l in enumerate(open(path).read().split("\n"), 1):
        if i < start:
            continue
        for ch in l:
            if ch == "{":
                depth += 1
                opened = True
            elif ch == "}":
                depth -= 1
        if opened and depth == 0:
            return i
    raise SystemExit("unbalanced braces")


def disasm(obj, kernel_match):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=tmp, check=True, capture_output=True)
    cubins = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    text = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubins[0])], capture_output=True,
                          text=True, check=True).stdout
    out, cur, take, name = [], None, False, None
    for l in text.split("\n"):
        m = re.match(r"\s*\.section\s+\.text\.(\S+),", l)
        if m:
            take = all(k in m.group(1) for k in kernel_match)
            if take:
                name = m.group(1)
            continue
        if not take:
            continue
        m = re.search(r'//## File ".*/(\S+)", line (\d+)', l)
        if m:
            cur = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
        if m:
            out.append((int(m.group(1), 16), cur, m.group(2).strip()))
    if not out:
        raise SystemExit(f"no kernel matching {kernel_match}")
    return name, out


def bitslice_regions():
    f = os.path.join(CSRC, "hash_bitslice.cu")
    loop0 = line_of(f, "for (uint32_t tb = 0;; tb += 64) {")
    loop1 = block_end(f, loop0)
    t0 = line_of(f, "__device__ __forceinline__ void bv_test(")
    t1 = block_end(f, t0)
    chain0 = line_of(f, "__device__ __forceinline__ uint32_t bv_chain(")
    ld0 = line_of(f, "__device__ __forceinline__ void bv_load_group(")
    la0 = line_of(f, "__device__ __forceinline__ void bv_load_all(")
    tr0 = line_of(f, "struct BvTranspose {")
    prmt0 = line_of(f, "__device__ __forceinline__ uint32_t bv_prmt(")
    rotl0 = line_of(f, "__device__ __forceinline__ uint32_t bv_rotl(")
    comb0 = line_of(f, "// ---- a8: the first green draw of each pending row", loop0)
    late0 = line_of(f, "if (tb >= (uint32_t)T0) {", loop0)
    late1 = block_end(f, late0)
    cap0 = line_of(f, "if (tb >= p.cap) {", loop0)
    cap1 = block_end(f, cap0)
    fname = "hash_bitslice.cu"
    test_lines = set(range(t0, t1 + 1)) | set(range(chain0, block_end(f, chain0) + 1)) | \
        set(range(ld0, block_end(f, ld0) + 1)) | set(range(la0, block_end(f, la0) + 1)) | \
        set(range(prmt0, block_end(f, prmt0) + 1))
    comb_lines = set(range(comb0, loop1 + 1)) | set(range(tr0, block_end(f, tr0) + 1)) | \
        set(range(rotl0, block_end(f, rotl0) + 1))
    return {
        "loop": (fname, loop0, loop1),
        "regions": [
            ("late_draws (t >= T0, cold)", lambda c: c[0] == "common.cuh" or (c[0] == fname and late0 <= c[1] <= late1)),
            ("cap (cold)", lambda c: c[0] == fname and cap0 <= c[1] <= cap1),
            ("test (2 draws x G groups: decode, L masks, column-max skip, plane loads, carry chains)",
             lambda c: c[0] == fname and c[1] in test_lines),
            ("combine (REDUX, 32x32 transpose, first green, record)",
             lambda c: (c[0] == fname and c[1] in comb_lines) or c[0].startswith("sm_")),
            ("loop control + prefetch", lambda c: True),
        ],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["bitslice"])
    ap.add_argument("--kernel-match", nargs="+", default=["bitslice_kernel", "ILi6ELi2ELb0ELi512"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_sass_bitslice"))
    a = ap.parse_args()
    spec = bitslice_regions()
    name, ins = disasm(os.path.join(BUILD, "hash_bitslice.cu.o"), a.kernel_match)
    fname, l0, l1 = spec["loop"]
    addrs = [x[0] for x in ins if x[1] and x[1][0] == fname and l0 <= x[1][1] <= l1]
    lo, hi = min(addrs), max(addrs)
    rng = [x for x in ins if lo <= x[0] <= hi]
    counts = {r[0]: 0 for r in spec["regions"]}
    lines = []
    for addr, c, op in rng:
        c = c or ("?", 0)
        for rname, pred in spec["regions"]:
            if pred(c):
                counts[rname] += 1
                break
        lines.append(f"/*{addr:05x}*/ {op:60s} // {c[0]}:{c[1]}  [{rname.split(' ')[0]}]")
    mt = re.search(r"ILi(\d+)ELi(\d+)ELb(\d)ELi(\d+)E", name)
    res = {"kernel": name.split(",")[0], "planes": int(mt.group(1)), "groups": int(mt.group(2)),
           "clamp": int(mt.group(3)), "threads": int(mt.group(4)),
           "loop_source": f"{fname}:{l0}-{l1}", "address_range": [hex(lo), hex(hi)],
           "instructions_in_range": len(rng), "by_region": counts,
           "note": "static count of the round loop (64 draws per warp round: 2 per lane); cold regions run "
                   "only past T0 draws / at the cap"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".txt", "w").write("\n".join(lines) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
