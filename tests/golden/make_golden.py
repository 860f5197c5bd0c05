"""Generate golden vectors by running the REFERENCE itself (tilesplat).

Run in the build container only (needs /root/reference; the GPU box has no
copy).  The reference tree is imported from a scratch copy so numba's cache
never lands in the read-only mount:

    rm -rf /tmp/ref && mkdir -p /tmp/ref && cp -r /root/reference/pkg/src /tmp/ref/
    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Each .npz holds the activated inputs, the camera fields, and the reference's
outputs at every stage boundary of SURVEY.md §8(c): splat rows, depth,
retained, tile rects, the SORTED (key, value) arrays (emission order is
unspecified in the reference, binning.py:19-21), the range table, the frame,
the contrib flags and the FrameStats counters.
"""

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/tmp/ref/src")
import tilesplat as ts  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cam_fields(cam, prefix):
    return {
        prefix + "wh": np.array([cam.width, cam.height], np.int32),
        prefix + "position": cam.position,
        prefix + "view": cam.world_to_camera,
        prefix + "proj": cam.full_projection,
        prefix + "intr": np.array([cam.tan_fovx, cam.tan_fovy, cam.focal_x, cam.focal_y],
                                  np.float64),
    }


def sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def run_case(name, act, cams, tau, bg, sh_degree, full_strategies=("precise",),
             store_inputs=True, store_splat=True):
    out = {"tau": np.float64(tau), "bg": np.asarray(bg, np.float32),
           "sh_degree": np.int32(sh_degree), "ncam": np.int32(len(cams))}
    if store_inputs:
        out.update(means=act.means, opacities=act.opacities, scales=act.scales,
                   rotations=act.rotations, sh=act.sh)
    k, keep = ts.power_cutoffs(act.opacities, tau)
    out["k"] = k
    pipe = ts.Pipeline(act, sh_degree=sh_degree)
    for ci, cam in enumerate(cams):
        p = f"c{ci}_"
        out.update(cam_fields(cam, p))
        for strat in ts.STRATEGIES:
            b = ts.preprocess_and_bin(act, cam, strat, tau, workers=8, sh_degree=sh_degree)
            out[p + strat + "_pairs"] = np.int64(b.emitted_count)
            if strat not in full_strategies:
                continue
            q = p + ("" if strat == "precise" else strat + "_")
            keys, vals = ts.sort_pairs(b.keys, b.values, 8, b.grid_w * b.grid_h,
                                       max(act.count, 1))
            starts = ts.tile_range_table(keys, b.grid_w, b.grid_h)
            img, contrib, nonempty = ts.render_frame(b.splat, vals, starts, cam.width,
                                                     cam.height, bg, tau, workers=8)
            fb, st = pipe.render(cam, strat, tau, bg, workers=8)
            assert np.array_equal(fb.image, img)
            out[q + "retained"] = np.packbits(b.retained)
            out[q + "depth"] = b.depth
            out[q + "rects"] = b.tile_rects.astype(np.int16)
            if store_splat and strat == "precise":
                out[q + "splat"] = b.splat
            out[q + "splat_sha"] = sha(b.splat)
            out[q + "keys"] = keys
            out[q + "values"] = vals
            out[q + "starts"] = starts.astype(np.int32)
            if strat == "precise":
                out[q + "image"] = img
            out[q + "image_sha"] = sha(img)
            out[q + "contrib"] = np.packbits(contrib)
            out[q + "stats"] = np.array([st.pairs_emitted, st.pairs_contributing,
                                         st.gaussians_retained, st.gaussians_degenerate,
                                         st.tiles_nonempty], np.int64)
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(name, os.path.getsize(path) // 1024, "KiB")


def main():
    # BASELINE config 1: the survey's fingerprinted case
    act = ts.activate(ts.gen_synthetic("mixed", 10_000, 1))
    cams = ts.orbit_cameras(1, 24.0, 256, 256)
    run_case("c1_mixed10k_256", act, cams, 1.0 / 255.0, (0, 0, 0), 3, store_splat=False)
    img = np.load(os.path.join(HERE, "c1_mixed10k_256.npz"))["c0_image"]
    assert hashlib.sha256(img.tobytes()).hexdigest()[:16] == "57807ea6520ab90c"

    # the reference's own session fixtures (tests/conftest.py:156-168), all
    # three strategy arms stored in full
    for preset, seed in (("mixed", 11), ("elongated", 5)):
        act = ts.activate(ts.gen_synthetic(preset, 800, seed))
        run_case(f"{preset}800_256x192", act, ts.orbit_cameras(3, 24.0, 256, 192),
                 1.0 / 255.0, (0, 0, 0), 3, full_strategies=ts.STRATEGIES)

    # edge tiles (70x42, test_render.py:188-192), close camera, tau above the
    # default, coloured background, lower SH degree
    act = ts.activate(ts.gen_synthetic("mixed", 3000, 9))
    run_case("edge3000_70x42", act, ts.orbit_cameras(2, 6.0, 70, 42), 0.01,
             (0.2, 0.5, 1.0), 2)


if __name__ == "__main__":
    main()
