#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of one kernel: joins the SASS view of an
ncu report with nvdisasm's line table of the library that was profiled.

    python tools/srcprof.py <rep.ncu-rep> <mangled-kernel-substring> [top=40] [lib.so]

Lines are the innermost frames inside this repo's csrc/ (inlined helpers count where they are
written, not where they are called)."""
import csv, glob, io, os, re, subprocess, sys, tempfile

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2408_07967_b200/_lib/libflashgs_b200.so"

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = None
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cub], capture_output=True, text=True).stdout
    cur, chain, tab, infn, last = None, [], [], False, ("?", 0)
    for ln in txt.splitlines():
        m = re.match(r"\.text\.(\S+):", ln)
        if m:
            if infn and tab: break
            infn = kern in m.group(1); tab = []; chain = []
            continue
        if not infn: continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            chain.append((m.group(1), int(m.group(2))))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            if chain:
                own = [c for c in chain if "/csrc/" in c[0]]
                if os.environ.get("SRCPROF_CALLSITE"):      # attribute inlined fgs_common.cuh helpers to their call site
                    cu = [c for c in own if c[0].endswith(".cu")]
                    own = cu or own
                last = own[0] if own else chain[0]
                chain = []
            tab.append((int(m.group(1), 16), last, m.group(2).strip()))
    if infn and tab:
        lines_of = tab
        break
if not lines_of:
    sys.exit(f"kernel {kern} not found in {lib}")

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if r and r[0].startswith("0x")]
base = int(data[0]["Address"], 16)
byoff = {o: (p, s) for o, p, s in lines_of}
agg, unk = {}, 0
STALLS = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for d in data:
    off = int(d["Address"], 16) - base
    p = byoff.get(off)
    if p is None: unk += 1; continue
    key = (os.path.basename(p[0][0]), p[0][1])
    a = agg.setdefault(key, [0, 0, {}])
    a[0] += int(d["Instructions Executed"] or 0)
    a[1] += int(d["# Samples"] or 0)
    for s in STALLS:
        v = int(d.get(s) or 0)
        if v: a[2][s] = a[2].get(s, 0) + v
ti = sum(a[0] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
src_cache = {}
def src(f, l):
    if f not in src_cache:
        p = os.path.join("paper_2408_07967_b200/csrc", f)
        src_cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
    L = src_cache[f]
    return L[l - 1].strip()[:100] if 0 < l <= len(L) else ""
if os.environ.get("SRCPROF_RANGES"):                # e.g. "geometry:907-1069,walk:722-813": sums per line range
    for spec in os.environ["SRCPROF_RANGES"].split(","):
        name, r = spec.split(":"); lo, hi = map(int, r.split("-"))
        ii = sum(a[0] for (f, l), a in agg.items() if f.endswith(".cu") and lo <= l <= hi)
        ss = sum(a[1] for (f, l), a in agg.items() if f.endswith(".cu") and lo <= l <= hi)
        print(f"range {name:12s} {lo:5d}-{hi:5d}: {100*ii/ti:5.1f}% inst {100*ss/ts:5.1f}% smp")
print(f"{kern}: {ti} warp instructions, {ts} samples, {unk} unmatched SASS rows")
tot_st = {}
for a in agg.values():
    for s, v in a[2].items(): tot_st[s] = tot_st.get(s, 0) + v
print("stall samples: " + ", ".join(f"{s[6:]} {100*v/ts:.1f}%" for s, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:8]))
for title, idx in (("by instructions", 0), ("by samples", 1)):
    print("--- " + title)
    for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][idx])[:top]:
        st = ",".join(f"{s[6:]}:{v}" for s, v in sorted(a[2].items(), key=lambda kv: -kv[1])[:2])
        print(f"{f}:{l:5d} {100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% smp [{st}] | {src(f, l)}")
