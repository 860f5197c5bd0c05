#!/usr/bin/env python
"""Probe: distribution of pairs per tile for a bench workload."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench
import paper_2408_07967_b200 as fgs

name = sys.argv[1] if len(sys.argv) > 1 else "c4-4k"
act, W, H, desc = bench.make_scene(fgs, name)
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
keys, vals, starts = fgs.sorted_pairs(pipe, cam)
n = np.diff(starts)
print(desc, "pairs", n.sum(), "tiles", n.size)
for lo, hi in ((0, 0), (1, 1024), (1025, 4096), (4097, 8192), (8193, 16384), (16385, 32768), (32769, 1 << 30)):
    m = (n >= lo) & (n <= hi)
    print(f"  {lo:6d}..{hi:10d}: {m.sum():6d} tiles, {n[m].sum():10d} pairs ({100.0 * n[m].sum() / n.sum():5.1f}%)")
print("  max", n.max())
