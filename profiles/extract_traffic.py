#!/usr/bin/env python
"""ncu reports -> profiles/<tag>_traffic.json: per kernel DRAM bytes, duration, instruction
count and issue-slot utilisation of ONE launch (what bench.py's roofline.traffic cites).

    python profiles/extract_traffic.py <tag> <workload> <rep1.ncu-rep> [...]
"""
import csv
import json
import subprocess
import sys

WANT = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__time_duration.sum": "duration_ns",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_busy_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_busy_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_busy_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e3, "ms": 1e6, "ns": 1.0,
         "s": 1e9}


def main():
    tag, workload = sys.argv[1], sys.argv[2]
    out = {"workload": workload, "source": [], "kernels": {}}
    for path in sys.argv[3:]:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units = rows[0], rows[1]
        out["source"].append(path.split("/")[-1])
        for vals in rows[2:]:
            name = vals[hdr.index("Kernel Name")].split("(")[0].replace("void ", "") \
                .replace("<unnamed>::", "").strip()
            rec = {}
            for key, label in WANT.items():
                if key in hdr:
                    i = hdr.index(key)
                    rec[label] = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            rec["dram_bytes"] = rec.get("dram_read_bytes", 0.0) + rec.get("dram_write_bytes", 0.0)
            out["kernels"][name] = rec
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
