#!/usr/bin/env python
"""SASS evidence for the shipped library:  python profiles/sass_summary.py > profiles/<tag>_sass.txt

Per kernel (template instances folded): counts of the opcodes that say what the code is built
from -- Blackwell packed FP32 (FFMA2 / FMUL2 / FADD2), cp.async (LDGSTS), MUFU, shared / global
atomics, warp collectives -- and of the ones it deliberately does not use (UTMALDG / UTCxMMA /
LDTM: no dense contraction on this path).  Then the first lines of the blend's packed loop."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_07967_b200/_lib/libflashgs_b200.so"
WATCH = ["FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "DFMA", "DMUL", "DADD", "MUFU", "LDGSTS", "LDG", "STG",
         "LDS", "STS", "ATOMS", "ATOMG", "RED", "REDUX", "SHFL", "MATCH", "VOTE", "BAR", "ACQBULK",
         "UTMALDG", "UTMASTG", "UTCHMMA", "UTCQMMA", "LDTM", "STTM", "HMMA"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
counts, order, fn = collections.defaultdict(collections.Counter), [], None
blend_lines = []
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        name = m.group(1)
        k = re.search(r"\d+(k_[a-z0-9_]+?)(I[LN]|E|P)", name)
        fn = k.group(1) if k else name
        full = name
        if fn not in order:
            order.append(fn)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", ln)
    if m and fn:
        counts[fn][m.group(1)] += 1
        counts[fn]["_all"] += 1
        if "k_blend2ILb1ELb0" in full and re.search(r"FFMA2|FMUL2|FADD2|LDGSTS|MUFU\.EX2", ln) and len(blend_lines) < 28:
            blend_lines.append(ln.rstrip())
print(f"# cuobjdump -sass {LIB}  (sm_100a; counts are static instructions, all template instances of a kernel summed)\n")
print("kernel".ljust(22) + "total".rjust(8) + "".join(o.rjust(8) for o in WATCH))
for fn in order:
    c = counts[fn]
    print(fn.ljust(22) + str(c["_all"]).rjust(8) + "".join((str(c[o]) if c[o] else ".").rjust(8) for o in WATCH))
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print("\nlibrary totals: " + ", ".join(f"{o} {tot[o]}" for o in WATCH))
print("\n# k_blend2<contrib, no extras>: first packed-FP32 / cp.async / ex2 instructions")
print("\n".join(blend_lines))
