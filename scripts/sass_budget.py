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
    labels, pending = {}, []
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
        m = re.match(r"^(\.L_x_\d+):", l.strip())
        if m:
            pending.append(m.group(1))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
        if m:
            a = int(m.group(1), 16)
            for lb in pending:
                labels[lb] = a
            pending = []
            out.append((a, cur, m.group(2).strip()))
    if not out:
        raise SystemExit(f"no kernel matching {kernel_match}")
    # branch targets as addresses
    out = [(a, c, re.sub(r"`\((\.L_x_\d+)\)", lambda mm: hex(labels.get(mm.group(1), -1)), op)) for a, c, op in out]
    return name, out


def bitslice_regions():
    f = os.path.join(CSRC, "hash_bitslice.cu")
    loop0 = line_of(f, "for (uint32_t tb = 0;; tb += BV_RD) {")
    loop1 = block_end(f, loop0)
    t0 = line_of(f, "__device__ __forceinline__ bool bv_test_c(")
    t1 = block_end(f, t0)
    chain0 = line_of(f, "__device__ __forceinline__ uint32_t bv_chain(")
    ld0 = line_of(f, "__device__ __forceinline__ void bv_load_group(")
    la0 = line_of(f, "__device__ __forceinline__ void bv_load_all(")
    tr0 = line_of(f, "struct BvTranspose {")
    prmt0 = line_of(f, "__device__ __forceinline__ uint32_t bv_prmt(")
    rotl0 = line_of(f, "__device__ __forceinline__ uint32_t bv_rotl(")
    comb0 = line_of(f, "// ---- a8: the first green draw of each pending row", loop0)
    late0 = line_of(f, "if (tb >= (uint32_t)BV_T0) {", loop0)
    late1 = block_end(f, late0)
    cap0 = line_of(f, "if (total == 0u) {", loop0)
    cap1 = block_end(f, cap0)
    slow0 = line_of(f, "if (CLAMP && slow) {", loop0)
    scr0 = line_of(f, "// ---- a5/a6 screen:", loop0)
    scr1 = line_of(f, "// ---- test the needed draws", scr0)
    pass0 = line_of(f, "for (uint32_t base = 0; base < total; base += 32) {", loop0)
    pass1 = block_end(f, pass0)
    slow1 = block_end(f, slow0)
    fname = "hash_bitslice.cu"
    test_lines = set(range(t0, t1 + 1)) | set(range(chain0, block_end(f, chain0) + 1)) | \
        set(range(ld0, block_end(f, ld0) + 1)) | set(range(la0, block_end(f, la0) + 1)) | \
        set(range(prmt0, block_end(f, prmt0) + 1))
    comb_lines = set(range(comb0, loop1 + 1)) | set(range(tr0, block_end(f, tr0) + 1)) | \
        set(range(rotl0, block_end(f, rotl0) + 1))
    return {
        "loop": (fname, loop0, loop1),
        "pass": (pass0, pass1),
        "regions": [
            ("late_draws (t >= T0, cold)", lambda c: c[0] == "common.cuh" or (c[0] == fname and late0 <= c[1] <= late1)),
            ("cap (cold)", lambda c: c[0] == fname and cap0 <= c[1] <= cap1),
            ("clamped top cells (cold)", lambda c: c[0] == fname and slow0 <= c[1] <= slow1),
            ("screen (decode 3 draws, column-max test, ballot compaction into the list)",
             lambda c: c[0] == fname and scr0 <= c[1] < scr1),
            ("test (a listed draw x G groups: decode, L masks, plane loads, carry chains)",
             lambda c: c[0] == fname and c[1] in test_lines),
            ("combine (a 32x32 transpose per group, first list position, record)",
             lambda c: (c[0] == fname and c[1] in comb_lines) or c[0].startswith("sm_")),
            ("loop control + prefetch", lambda c: True),
        ],
    }


def per_unit_budget(obj, kernel_match, src, first_marker, last_marker, unit_op, unit_name, out, extra_lines=(),
                    loop=False, unit_prefix=True):
    """Static SASS of the (unrolled) source lines [first_marker, last_marker] of
    `src`, divided by the number of `unit_op` instructions they contain (one per
    unit of work: a draw-test or a visited entry): lane-instructions per unit."""
    import collections
    f = os.path.join(CSRC, src)
    l0, l1 = line_of(f, first_marker), line_of(f, last_marker)
    lines = set(range(l0, l1 + 1)) | {line_of(f, m) for m in extra_lines}
    name, ins = disasm(os.path.join(BUILD, src + ".o"), kernel_match)
    marked = [x for x in ins if x[1] and x[1][0] == src and x[1][1] in lines]
    lo, hi = min(x[0] for x in marked), max(x[0] for x in marked)
    if loop:                       # the innermost natural loop around the marked lines
        best = None                # the back-edge enclosing the most marked instructions, then the tightest
        for addr, c, op in ins:
            m = re.match(r"(?:@!?U?P\w+\s+)?BRA(?:\.\w+)*\s+0x([0-9a-f]+)", op)
            if not m or int(m.group(1), 16) >= addr:
                continue
            t = int(m.group(1), 16)
            n_in = sum(1 for x in marked if t <= x[0] <= addr)
            key = (n_in, -(addr - t))
            if best is None or key > best[0]:
                best = (key, t, addr)
        lo, hi = best[1], best[2]
    # every instruction in the span (inlined helpers included)
    body = [x for x in ins if lo <= x[0] <= hi]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", op).split()[0] for _, _, op in body)
    units = sum(v for k, v in ops.items() if k == unit_op or (unit_prefix and k.startswith(unit_op + ".")))
    res = {"kernel": name.split(",")[0], "source": f"{src}:{l0}-{l1}", "span": [hex(lo), hex(hi)],
           "span_is": "innermost loop around the lines" if loop else "address span of the (unrolled) lines",
           "instructions": len(body),
           "units": units, "unit": unit_name, "unit_op": unit_op,
           "lane_instr_per_unit": len(body) / max(units, 1), "opcodes": dict(ops.most_common())}
    json.dump(res, open(out + ".json", "w"), indent=1)
    open(out + ".txt", "w").write("\n".join(f"/*{a:05x}*/ {op:60s} // {c[0]}:{c[1]}" for a, c, op in body) + "\n")
    print(json.dumps({k: v for k, v in res.items() if k != "opcodes"}, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["bitslice", "cm", "index", "simple"])
    ap.add_argument("--kernel-match", nargs="+", default=["bitslice_kernel", "ILi5ELi2ELb0ELi640"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_sass_bitslice"))
    a = ap.parse_args()
    if a.which == "cm":            # the byte tile's SWAR round: one LDS of a 4-row word per draw
        return per_unit_budget("hash_tiled_cm.cu", ["hash_tiled_cm_kernel", "ILi2ELi1ELi1ELi1E"], "hash_tiled_cm.cu",
                               "for (int u = PER - 1; u >= 0; u--) {",
                               "h4 = (h4 & ~m) | ((uint32_t)(part * PD + PER * i4 + u) * 0x01010101u & m);",
                               "LDS", "draw tested against a 4-row word (4 row-tests)",
                               os.path.join(ROOT, "profiles", "r2_sass_cm"), extra_lines=["const uint4 q4 = e4[i4];"],
                               unit_prefix=False)
    if a.which == "index":         # the INDEX rows kernel's entry walk: one global load of a filed draw per entry
        return per_unit_budget("hash_index.cu", ["hash_index_kernel", "ILi2ELb1ELi2EhE"], "hash_index.cu",
                               "v[u] = base + 32u * u + lane < lim ? __ldg(p.vals + addr[u]) : IX_NONE;",
                               "atomicMin(h + (v[u] >> 16), v[u] & 0xFFFFu);",
                               "LDG", "visited entry (filed draw) per lane",
                               os.path.join(ROOT, "profiles", "r2_sass_index"), loop=True)
    if a.which == "simple":        # the paper's loop: one cell load per draw
        return per_unit_budget("hash_simple.cu", ["hash_simple_kernel", "ILi1ELb0EhLb0E"], "hash_simple.cu",
                               "for (uint32_t t = 0; t < cap; t++) {",
                               "if (off < xv) { h = t + 1; found = true; break; }",
                               "LDG", "draw (the paper's per-row loop)",
                               os.path.join(ROOT, "profiles", "r2_sass_simple"), loop=True)
    spec = bitslice_regions()
    name, ins = disasm(os.path.join(BUILD, "hash_bitslice.cu.o"), a.kernel_match)
    fname, l0, l1 = spec["loop"]
    # the round loop = the innermost natural loop (a backward branch and its
    # target) that holds both test and combine instructions
    rp = dict(spec["regions"])
    test_pred = rp[[k for k in rp if k.startswith("test")][0]]
    comb_pred = rp[[k for k in rp if k.startswith("combine")][0]]
    scr_pred = rp[[k for k in rp if k.startswith("screen")][0]]
    loops = []                       # natural loops: (target, back-edge address)
    for addr, c, op in ins:
        m = re.match(r"(?:@!?U?P\w+\s+)?BRA(?:\.\w+)*\s+0x([0-9a-f]+)", op)
        if m and int(m.group(1), 16) < addr:
            loops.append((int(m.group(1), 16), addr))

    def innermost(*preds):
        best = None
        for tgt, addr in loops:
            body = [x for x in ins if tgt <= x[0] <= addr]
            if all(any(x[1] and pr(x[1]) for x in body) for pr in preds):
                if best is None or addr - tgt < best[1] - best[0]:
                    best = (tgt, addr)
        return best

    # the round loop holds the screen and the tests; the pass loop (inside it)
    # the tests and the first-green combine only
    rnd = innermost(test_pred, comb_pred, scr_pred)
    pas = innermost(test_pred, comb_pred)
    if rnd is None or pas is None or not (rnd[0] <= pas[0] and pas[1] <= rnd[1]):
        raise SystemExit(f"round/pass loops not found: {rnd} {pas}")
    cold = [rp[k] for k in rp if "cold" in k]
    counts = {r[0]: 0 for r in spec["regions"]}
    lines = []
    n_pass = n_round = 0
    for addr, c, op in [x for x in ins if rnd[0] <= x[0] <= rnd[1]]:
        c = c or ("?", 0)
        for rname, pred in spec["regions"]:
            if pred(c):
                counts[rname] += 1
                break
        hot = not any(pr(c) for pr in cold)
        in_pass = pas[0] <= addr <= pas[1]
        if hot:
            if in_pass:
                n_pass += 1
            else:
                n_round += 1
        lines.append(f"/*{addr:05x}*/ {op:60s} // {c[0]}:{c[1]}  [{rname.split(' ')[0]}{'' if hot else ' cold'}"
                     f"{' pass' if in_pass else ''}]")
    mt = re.search(r"ILi(\d+)ELi(\d+)ELb(\d)ELi(\d+)E", name)
    src = open(os.path.join(CSRC, "hash_bitslice.cu")).read()
    dpl = int(re.search(r"constexpr int BV_DPL = (\d+);", src).group(1))
    res = {"kernel": name.split(",")[0], "planes": int(mt.group(1)), "groups": int(mt.group(2)),
           "clamp": int(mt.group(3)), "threads": int(mt.group(4)),
           "loop_source": f"{fname}:{l0}-{l1}", "round_loop": [hex(rnd[0]), hex(rnd[1])],
           "pass_loop": [hex(pas[0]), hex(pas[1])], "by_region": counts,
           "draws_per_round": 32 * dpl, "entries_per_pass": 32,
           "round_instructions": n_round, "pass_instructions": n_pass,
           "lane_instr_per_screened_draw": 32.0 * n_round / (32 * dpl),
           "lane_instr_per_tested_entry": 32.0 * n_pass / 32,
           "note": "static SASS counts of the hot paths (cold regions excluded: late draws past the table, the cap, "
                   "the clamped top cells): per round (screen 32*BV_DPL draws, outside the pass loop) and per pass "
                   "(test up to 32 listed draws + first-green combine).  Counted on the unclamped variant: the "
                   "clamped one (c5's P = 5 of NB = 7) runs the same hot path plus the rare inline test of the "
                   "top cells, whose block layout the loop finder cannot separate"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".txt", "w").write("\n".join(lines) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
