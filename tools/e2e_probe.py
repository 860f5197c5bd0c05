#!/usr/bin/env python
"""Probe (run under gpurun): views/s through Pipeline.render_iter for K = 20 and 100 frames."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2408_07967_b200 as fgs

name = sys.argv[1] if len(sys.argv) > 1 else "c4-4k"
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 3
act, W, H, desc = bench.make_scene(fgs, name)
cams = fgs.orbit_cameras(16, 24.0, W, H)
pipe = fgs.Pipeline(act)
for c in cams[:4]:
    pipe.render(c)
for fb, _ in pipe.render_iter([cams[i % 16] for i in range(12)], streams=streams):
    pass
for K in (20, 20, 100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    for fb, st in pipe.render_iter([cams[i % 16] for i in range(K)], streams=streams):
        n += 1
    dt = time.perf_counter() - t0
    print(f"{name} streams={streams} K={K}: {dt / K * 1e3:.3f} ms/view, {K / dt:.1f} views/s")
