#!/usr/bin/env python
"""Print the per-kernel times of bench.py JSON lines (files given as arguments)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        line = [l for l in open(path).read().splitlines() if l.startswith("{")][-1]
    except (IndexError, OSError):
        print(f"{path}: no JSON line")
        continue
    d = json.loads(line)
    ks = " ".join(f"{k['name']}={k['ms'] * 1e3:.1f}" for k in d.get("kernels", []))
    e2e = d.get("e2e", {})
    print(f"{path}: {d.get("ms_per_step", 0) * 1e3:.1f} us/step lat {d.get("frame_latency_ms", 0) * 1e3:.1f} (prof {d.get("frame_latency_profiled_ms", 0) * 1e3:.1f})  e2e {e2e.get('ms_per_step', 0) * 1e3:.1f} us "
          f"pairs={d.get('config', {}).get('pairs')} clocks={d.get('clocks', {}).get('sm_mhz')} | {ks}")
