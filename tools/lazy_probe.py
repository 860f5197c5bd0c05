#!/usr/bin/env python
"""How deep does the blend reach into heavy tiles?  (run under gpurun)

    python tools/lazy_probe.py [workload ...]

Renders view 0 (and view 5) of the workload with contrib flags on and reads the frame's range
table and contrib flags back from the workspace: for every tile with more than 2048 pairs, the
position of its LAST contributing pair.  A front-only depth sort of such tiles (sort the
nearest F pairs, the rest only if the tile has not saturated by then) pays when that position
is almost always far below the tile's pair count."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2408_07967_b200 as fgs  # noqa: E402


def probe(name, views=(0, 5)):
    act, W, H, desc = bench.make_scene(fgs, name)
    cams = fgs.orbit_cameras(16, 24.0, W, H)
    pipe = fgs.Pipeline(act)
    for v in views:
        fb, st = pipe.render(cams[v], as_numpy=False)
        ws = pipe._free[(W, H)][-1]
        lay = ws.lay
        T = int(lay.tiles)
        starts = ws.view(torch, lay.off_starts, (T + 1) * 4, torch.int32).cpu().numpy().astype(np.int64)
        contrib = ws.view(torch, lay.off_contrib, int(starts[-1]), torch.uint8).cpu().numpy()
        n = np.diff(starts)
        heavy = np.nonzero(n > 2048)[0]
        idx = np.nonzero(contrib)[0]
        # last contributing position per tile
        tile_of = np.searchsorted(starts, idx, side="right") - 1
        last = np.full(T, -1, dtype=np.int64)
        np.maximum.at(last, tile_of, idx - starts[tile_of])
        lh, nh = last[heavy] + 1, n[heavy]
        print(f"{name} view {v}: M={int(starts[-1])} tiles={T} heavy(>2048)={heavy.size} "
              f"pairs in heavy={int(nh.sum())} ({100.0 * nh.sum() / max(1, starts[-1]):.1f} %)")
        if heavy.size == 0:
            continue
        for F in (512, 1024, 1536, 2048, 3072):
            deep = lh > F
            print(f"   last contributing pair beyond {F:5d}: {int(deep.sum()):6d} tiles "
                  f"({100.0 * deep.mean():5.2f} %), holding {int(nh[deep].sum()):9d} pairs")
        q = np.percentile(lh, [50, 90, 99, 100])
        print(f"   last contributing position: median {q[0]:.0f}, p90 {q[1]:.0f}, p99 {q[2]:.0f}, max {q[3]:.0f}; "
              f"reaches the end of the bucket in {int((lh >= nh).sum())} tiles")
    del pipe


if __name__ == "__main__":
    for w in (sys.argv[1:] or ["c4-4k", "c3", "c2-dense", "c4"]):
        probe(w)
        torch.cuda.empty_cache()
