"""Per-band device times of one 8K frame on ONE GPU (what each rank of a row-band job runs):
    python tools/band_probe.py [bands=8] [workload=c4]
Prints, per band, the stage times FrameStats reports (CUDA events around the stages) and the
projected multi-GPU frame time = slowest band (+ the NCCL gather, not measured here)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
import paper_2408_07967_b200 as fgs

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wl = sys.argv[2] if len(sys.argv) > 2 else "c4"
act, W, H, desc = bench.make_scene(fgs, wl)
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
gh = -(-H // 16)
from paper_2408_07967_b200 import sharding
split = sys.argv[3] if len(sys.argv) > 3 else "balanced"
if split == "balanced":
    rw = pipe.row_weights(cam)
    bands = sharding.balanced_band_partition(rw, nb, fixed_rows=0.3 * float(rw.mean()))
else:
    bands = sharding.band_partition(gh, nb)
print("split:", split, bands)
full, st = pipe.render(cam, as_numpy=False)
for _ in range(3):
    full, st = pipe.render(cam, as_numpy=False)
print(f"{desc}\nfull frame: total {st.total_ns / 1e6:.3f} ms  preprocess+bin {st.preprocess_bin_ns / 1e6:.3f}  "
      f"sort {st.sort_ns / 1e6:.3f}  render {st.render_ns / 1e6:.3f}  pairs {st.pairs_emitted}")
worst = 0.0
for b in range(nb):
    band = bands[b]
    for _ in range(3):
        fb, s = pipe.render(cam, band=band, as_numpy=False)
    worst = max(worst, s.total_ns / 1e6)
    print(f"band {b} rows {band}: total {s.total_ns / 1e6:.3f} ms  preprocess+bin {s.preprocess_bin_ns / 1e6:.3f}  "
          f"sort {s.sort_ns / 1e6:.3f}  render {s.render_ns / 1e6:.3f}  pairs {s.pairs_emitted}")
print(f"slowest band {worst:.3f} ms -> projected {nb}-GPU frame (before the gather): {worst:.3f} ms, "
      f"{st.total_ns / 1e6 / worst:.2f}x over one GPU")
