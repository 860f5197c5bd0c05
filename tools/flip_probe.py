"""Probe: which pairs' contrib flags differ between the default and the exact blend, and why."""
import sys
import numpy as np
sys.path.insert(0, ".")
import bench
import paper_2408_07967_b200 as fgs

wl = sys.argv[1] if len(sys.argv) > 1 else "c4-4k"
act, W, H, desc = bench.make_scene(fgs, wl)
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
b = fgs.preprocess_and_bin(pipe, cam)
keys, vals, starts = fgs.sorted_pairs(pipe, cam)
img0, c0, _ = fgs.render_frame(b.splat, vals, starts, W, H, (0, 0, 0), 1 / 255)
img1, c1, _ = fgs.render_frame(b.splat, vals, starts, W, H, (0, 0, 0), 1 / 255, exact=True)
print("contrib default", int(c0.sum()), "exact", int(c1.sum()), "max abs", float(np.abs(img0 - img1).max()))
diff = np.nonzero(c0 != c1)[0]
print("differing pairs:", diff[:20], len(diff))
gw = -(-W // 16)
f32 = np.float32
import math
for i in diff[:5]:
    t = int(np.searchsorted(starts, i, side="right") - 1)
    ty, tx = divmod(t, gw)
    print(f"pair {i}: tile {t} ({tx},{ty}) range {starts[t]}..{starts[t+1]} pos {i - starts[t]} default={c0[i]} exact={c1[i]}")
    # replay the tile pixel by pixel (float32, reference order), track T at pair i
    for y in range(ty * 16, min(ty * 16 + 16, H)):
        for x in range(tx * 16, min(tx * 16 + 16, W)):
            fx, fy, T = f32(x) + f32(0.5), f32(y) + f32(0.5), f32(1.0)
            for j in range(int(starts[t]), int(i) + 1):
                r = b.splat[vals[j]]
                dx, dy = fx - r[0], fy - r[1]
                if abs(dx) > r[10] or abs(dy) > r[11]:
                    continue
                s = f32(0.5) * (r[2] * dx * dx + r[4] * dy * dy) + r[3] * dx * dy
                if s > f32(0.5) * r[6]:
                    continue
                al = min(f32(0.99), r[5] * f32(math.exp(-float(s))))
                if j == i:
                    print(f"   px ({x},{y}) T_before={T:.9g} alpha={al:.9g} tau={1/255:.9g} s={s:.7g} hk={0.5*r[6]:.7g}")
                if al < f32(1 / 255):
                    continue
                T = T * (f32(1.0) - al)
                if T < f32(1e-4):
                    break
