#!/usr/bin/env python
"""Probe (run under gpurun): candidate-rectangle sizes of K1's Gaussians, per Gaussian and per
warp (32 consecutive slots of the Morton-ordered scene), for one view of a bench workload."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch
import bench
import paper_2408_07967_b200 as fgs

name = sys.argv[1] if len(sys.argv) > 1 else "c4-4k"
act, W, H, desc = bench.make_scene(fgs, name)
cam = fgs.orbit_cameras(16, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
fb, st = pipe.render(cam, as_numpy=False)
ws = pipe._free[(W, H)][-1]
lay = ws.lay
P = act.count
rects = ws.view(torch, lay.off_rects, P * 8, torch.int16).cpu().numpy().view(np.uint16).reshape(P, 4).astype(np.int64)
flags = ws.view(torch, lay.off_flags, P, torch.uint8).cpu().numpy()
counts = ws.view(torch, lay.off_counts, P * 4, torch.int32).cpu().numpy()
ret = (flags & 1) != 0
nx = np.where(ret, rects[:, 2] - rects[:, 0] + 1, 0)
ny = np.where(ret, rects[:, 3] - rects[:, 1] + 1, 0)
print(desc, "retained", int(ret.sum()), "pairs", int(counts.sum()), "candidates", int((nx * ny).sum()))
tot = ret.sum()
for a in range(1, 5):
    print("  ny\\nx " + " ".join(f"{100.0 * ((nx == b) & (ny == a)).sum() / tot:6.2f}" for b in range(1, 5)) +
          f"   (row ny={a}, columns nx=1..4, % of retained)")
big = (nx > 3) | (ny > 3)
print(f"  beyond 3x3: {100.0 * big.sum() / tot:.2f} % of Gaussians, {100.0 * counts[big].sum() / counts.sum():.2f} % of pairs, "
      f"{100.0 * (nx * ny)[big].sum() / (nx * ny).sum():.2f} % of candidates")
Pw = (P // 32) * 32
mx = np.maximum(nx, ny)[:Pw].reshape(-1, 32)
wmax = mx.max(axis=1)
for k in (1, 2, 3):
    print(f"  warps with every rectangle <= {k}x{k}: {100.0 * (wmax <= k).mean():.2f} %")
cb = (nx * ny * big)[:Pw].reshape(-1, 32).sum(axis=1)
print(f"  cooperative-walk candidates per warp: mean {cb.mean():.1f}, p50 {np.percentile(cb, 50):.0f}, p90 {np.percentile(cb, 90):.0f}, "
      f"p99 {np.percentile(cb, 99):.0f}, max {cb.max()}; windows per warp mean {np.ceil(cb / 32).mean():.2f}")
cta = cb[: (cb.size // 8) * 8].reshape(-1, 8)
print(f"  per CTA (8 warps): windows max-over-warps mean {np.ceil(cta / 32).max(axis=1).mean():.2f}, "
      f"balanced (sum/8) mean {(np.ceil(cta.sum(axis=1) / 32) / 8).mean():.2f}")
small_cand = (nx * ny * (~big))[:Pw].reshape(-1, 32)
print(f"  small-walk: mean candidates per Gaussian {(nx * ny)[ret & ~big].mean():.2f}, pairs {counts[ret & ~big].mean():.2f}; "
      f"per warp max candidates mean {small_cand.max(axis=1).mean():.2f}")
