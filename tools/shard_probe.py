"""Gaussian-sharded row bands, projected from ONE GPU.

    python tools/shard_probe.py [ranks=8] [workload=c4]

Today's row-band frame (Pipeline.render_bands) replicates K1 on every rank.  The sharded
variant gives rank r the preprocess CTAs (256-slot blocks of the Morton-ordered scene)
b = r (mod N) for the WHOLE frame, then moves every pair's record and every needed splat row
to the rank that owns the band of its tile.  This probe times what one rank of such a job
would run, piece by piece, on a single B200:

  K1 + scan + emit over a 1/N shard, whole frame   (a Pipeline over the shard's Gaussians)
  sort + blend of one band                         (today's band render of the full scene)
  exchange                                         (bytes counted from the frame itself,
                                                    divided by an ASSUMED NVLink rate)

and prints the projected frame time = slowest shard + exchange + slowest band.  Nothing here
was measured on more than one GPU."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
import paper_2408_07967_b200 as fgs
from paper_2408_07967_b200 import sharding

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wl = sys.argv[2] if len(sys.argv) > 2 else "c4"
NVLINK_GBS = 700.0          # assumed achievable per-GPU unidirectional all-to-all rate (of 900 nominal)

act, W, H, desc = bench.make_scene(fgs, wl)
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
gh = -(-H // 16)
for _ in range(3):
    full, st = pipe.render(cam, as_numpy=False)
print(desc)
print(f"one GPU: total {st.total_ns / 1e6:.3f} ms = bin {st.preprocess_bin_ns / 1e6:.3f} + sort {st.sort_ns / 1e6:.3f} "
      f"+ blend {st.render_ns / 1e6:.3f}; pairs {st.pairs_emitted}")

# bands: balanced on the row histogram, as render_bands cuts them
rw = pipe.row_weights(cam)
bands = sharding.balanced_band_partition(rw, N, fixed_rows=0.3 * float(rw.mean()))
band_ms, band_pairs = [], []
for b in bands:
    for _ in range(3):
        fb, s = pipe.render(cam, band=b, as_numpy=False)
    band_ms.append((s.sort_ns + s.render_ns) / 1e6)
    band_pairs.append(s.pairs_emitted)
    rep_bin = s.preprocess_bin_ns / 1e6
print("band sort+blend ms:", " ".join(f"{v:.3f}" for v in band_ms), "| replicated bin stage of a band frame:", f"{rep_bin:.3f}")

# which Gaussians does each band need (rows to ship): tile-row span of every retained Gaussian
bo = fgs.preprocess_and_bin(pipe, cam)
ret = bo.retained & (bo.pair_counts > 0)
ty0, ty1 = bo.tile_rects[:, 1], bo.tile_rects[:, 3]
rows_needed = [int(np.count_nonzero(ret & (ty1 >= b0) & (ty0 <= b1))) for b0, b1 in bands]
del bo

# shards: preprocess CTAs (256 consecutive slots) dealt round-robin to the ranks
order = pipe.slot_order if pipe.slot_order is not None else np.arange(act.count)
blocks = np.arange(act.count) // 256
shard_ms = []
del pipe
for r in range(N):
    idx = order[blocks % N == r]
    sub = fgs.ActivatedScene(act.means[idx], act.opacities[idx], act.scales[idx], act.rotations[idx], act.sh[idx])
    sp = fgs.Pipeline(sub)
    for _ in range(3):
        fb, s = sp.render(cam, as_numpy=False)
    shard_ms.append(s.preprocess_bin_ns / 1e6)
    del sp, sub
    torch.cuda.empty_cache()
    if r >= 1 and N > 4:      # shards are statistically alike: two are enough for the estimate
        shard_ms += [max(shard_ms)] * (N - len(shard_ms))
        break
print("shard bin stage (K1 + scan + emit over 1/N of the Gaussians, whole frame) ms:", " ".join(f"{v:.3f}" for v in shard_ms))

# exchange: a band owner receives its pairs' 8-byte records and its Gaussians' 56-byte rows
# (48 B splat row + depth + index) from the other N-1 ranks
recv = [(8.0 * band_pairs[k] + 56.0 * rows_needed[k]) * (N - 1) / N for k in range(N)]
ex_ms = max(recv) / (NVLINK_GBS * 1e9) * 1e3
print(f"exchange: max {max(recv) / 1e6:.1f} MB into one rank -> {ex_ms:.3f} ms at an ASSUMED {NVLINK_GBS:.0f} GB/s")
gather_ms = 12.0 * W * H * (N - 1) / N / (NVLINK_GBS * 1e9) * 1e3
proj = max(shard_ms) + ex_ms + max(band_ms) + gather_ms
print(f"projected {N}-GPU frame: {max(shard_ms):.3f} + {ex_ms:.3f} + {max(band_ms):.3f} + gather {gather_ms:.3f} = {proj:.3f} ms "
      f"-> {st.total_ns / 1e6 / proj:.2f}x over one GPU")
print(f"today's replicated-K1 bands: {rep_bin:.3f} + {max(band_ms):.3f} + gather {gather_ms:.3f} = {rep_bin + max(band_ms) + gather_ms:.3f} ms "
      f"-> {st.total_ns / 1e6 / (rep_bin + max(band_ms) + gather_ms):.2f}x")
