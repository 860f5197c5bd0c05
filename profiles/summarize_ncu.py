#!/usr/bin/env python
"""Turn ncu outputs (brought back under gpurun_out/) into a small tracked summary.

    python profiles/summarize_ncu.py <tag> <launches.csv> <rep1.ncu-rep> [...]  > profiles/<tag>.md

The launch list comes from
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file <launches.csv> python bench.py --steps 2 --warmup 3 --no-cpu
and each .ncu-rep from
    ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 8 -c 1 -o <rep> <same command>
"""
import csv
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 write sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "CTAs/SM (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__waves_per_multiprocessor", "waves / SM"),
    ("sm__cycles_elapsed.max", "cycles elapsed (max SM)"),
    ("smsp__cycles_active.avg", "cycles active (avg SMSP)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    print(f"# ncu summary `{tag}`\n")
    print("Numbers under ncu are cold-cache and serialised: compare SHARES, not absolutes.\n")
    agg = OrderedDict()
    total = 0.0
    with open(launches) as f:
        rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        ns = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
        total += ns
    print("## launch list (whole bench.py run: warm-up + timed + e2e frames)\n")
    print("| kernel | launches | total us | avg us | share |\n|---|---:|---:|---:|---:|")
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {ns / 1e3:.1f} | {ns / 1e3 / n:.2f} | {100 * ns / total:.1f}% |")
    for path in sys.argv[3:]:
        hdr, units, data = rep_rows(path)
        for vals in data:
            name = vals[hdr.index("Kernel Name")].split("(")[0]
            print(f"\n## `{name.strip()}`  ({path.split('/')[-1]})\n")
            print("| metric | value | unit |\n|---|---:|---|")
            for key, label in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    print(f"| {label} (`{key}`) | {vals[i]} | {units[i]} |")
            stalls = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                    try:
                        stalls.append((float(vals[i]), h.split("stalled_")[1].split("_per_issue")[0]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            print("\nTop warp stall reasons (warps stalled per issue-active cycle): "
                  + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]))


if __name__ == "__main__":
    main()
