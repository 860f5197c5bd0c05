#!/usr/bin/env python
"""Probe (run under gpurun): how many tiles of the small sort class are tiny?"""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import bench
import paper_2408_07967_b200 as fgs

for name in (sys.argv[1:] or ["c4-4k", "c4", "c3", "c2"]):
    act, W, H, desc = bench.make_scene(fgs, name)
    cam = fgs.orbit_cameras(16, 24.0, W, H)[0]
    pipe = fgs.Pipeline(act)
    pipe.render(cam, as_numpy=False)
    ws = pipe._free[(W, H)][-1]
    T = int(ws.lay.tiles)
    starts = ws.view(torch, ws.lay.off_starts, (T + 1) * 4, torch.int32).cpu().numpy().astype(np.int64)
    n = np.diff(starts)
    small = n[(n > 0) & (n <= 2048)]
    print(f"{name}: tiles {T}, empty {(n == 0).sum()}, small class {small.size} tiles / {small.sum()} pairs")
    for hi in (32, 64, 128, 256, 512, 1024, 2048):
        m = small <= hi
        print(f"   n <= {hi:4d}: {m.sum():6d} tiles ({100.0 * m.mean():5.1f} %), {small[m].sum():9d} pairs")
    del pipe
    torch.cuda.empty_cache()
