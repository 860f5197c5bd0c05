"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle on
the same inputs, and against the reference's own golden vectors.

Bars (BASELINE.json north_star): pair lists and sorted key order BIT-EXACT;
pixels max-abs <= 1e-3 and PSNR >= 60 dB in the default (ex2.approx) mode,
and bit-identical in exact mode.
"""

import hashlib

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from oracle import oracle as orc
from fgs_testlib import identity_camera, make_raw_scene

pytestmark = pytest.mark.gpu

STRATS = ("precise", "tight-aabb", "baseline-circle-aabb")
PIX_TOL = 1e-3          # north_star: max-abs 1e-3
PSNR_MIN = 60.0         # north_star: PSNR >= 60 dB
STOP_FLIPS_MAX = 3      # full-size frames, default mode: pairs whose contrib flag may differ
                        # through the T < 1e-4 stop (see _full_frame_against_oracle)


def _sorted_pairs(b, count):
    order = np.lexsort((b.values, b.keys))
    return b.keys[order], b.values[order]


def _psnr_ok(a, b):
    p = fgs.psnr(a, b)
    return p == "identical" or p >= PSNR_MIN


# ---------------------------------------------------------------------------
# against the reference's golden vectors
# ---------------------------------------------------------------------------
def test_golden_cutoffs(golden):
    k, _ = fgs.power_cutoffs(golden.act.opacities, golden.tau)
    assert np.array_equal(k.view(np.uint32), golden.z["k"].view(np.uint32))


def test_golden_every_stage(golden):
    g = golden
    pipe = fgs.Pipeline(g.act, sh_degree=g.sh_degree)
    for ci in range(g.ncam):
        cam = g.camera(ci)
        for s in STRATS:
            b = fgs.preprocess_and_bin(pipe, cam, s, g.tau, sh_degree=g.sh_degree)
            assert b.emitted_count == int(g.z[f"c{ci}_{s}_pairs"]), (ci, s)
            if not g.has(ci, "keys", s):
                continue
            ret = g.retained(ci, s)
            assert np.array_equal(b.retained, ret)
            assert np.array_equal(b.depth.view(np.uint32), g.get(ci, "depth", s).view(np.uint32))
            assert np.array_equal(b.tile_rects[ret], g.get(ci, "rects", s).astype(np.int32)[ret])
            # splat rows bit-exact (geometry AND SH colours)
            sha = np.frombuffer(hashlib.sha256(b.splat.tobytes()).digest(), np.uint8)
            assert np.array_equal(sha, g.get(ci, "splat_sha", s))
            keys, vals = fgs.sort_pairs(b.keys, b.values, 1, b.grid_w * b.grid_h,
                                        max(g.act.count, 1))
            assert np.array_equal(keys, g.get(ci, "keys", s))
            assert np.array_equal(vals, g.get(ci, "values", s))
            starts = fgs.tile_range_table(keys, b.grid_w, b.grid_h)
            assert np.array_equal(starts, g.get(ci, "starts", s).astype(np.int64))
            img, contrib, nonempty = fgs.render_frame(b.splat, vals, starts, cam.width,
                                                      cam.height, g.bg, g.tau, exact=True)
            sha = np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8)
            assert np.array_equal(sha, g.get(ci, "image_sha", s)), "exact-mode frame not bit-identical"
            assert np.array_equal(contrib, g.contrib(ci, s))
            st = g.get(ci, "stats", s)
            assert (b.emitted_count, int(contrib.sum()), b.gaussians_retained,
                    b.gaussians_degenerate, nonempty) == tuple(int(v) for v in st)


def test_golden_pipeline_render(golden):
    g = golden
    pipe = fgs.Pipeline(g.act, sh_degree=g.sh_degree)
    for ci in range(g.ncam):
        cam = g.camera(ci)
        ref = g.get(ci, "image")
        want = tuple(int(v) for v in g.get(ci, "stats"))
        fb, st = pipe.render(cam, "precise", g.tau, g.bg)
        assert fb.image.shape == ref.shape and fb.image.dtype == np.float32
        assert fgs.max_abs_diff(fb.image, ref) <= PIX_TOL
        assert _psnr_ok(fb.image, ref)
        assert (st.pairs_emitted, st.gaussians_retained, st.gaussians_degenerate,
                st.tiles_nonempty) == (want[0], want[2], want[3], want[4])
        assert st.pairs_contributing == want[1]      # the packed blend never flips a skip
        assert st.pair_buffer_bytes == 12 * want[0]
        fbx, stx = pipe.render(cam, "precise", g.tau, g.bg, exact=True)
        assert np.array_equal(fbx.image.view(np.uint32), ref.view(np.uint32))
        assert stx.pairs_contributing == want[1]


def test_c1_survey_fingerprints(golden_c1):
    g = golden_c1
    fb, st = fgs.Pipeline(g.act).render(g.camera(0), exact=True)
    assert (st.gaussians_retained, st.pairs_emitted, st.pairs_contributing,
            st.tiles_nonempty, st.candidate_tiles) == (10000, 47264, 34034, 236, 52466)
    assert hashlib.sha256(fb.image.tobytes()).hexdigest()[:16] == "57807ea6520ab90c"
    b = fgs.preprocess_and_bin(g.act, g.camera(0))
    assert hashlib.sha256(np.sort(b.keys).tobytes()).hexdigest()[:16] == "985b4149ce95e8e8"


# ---------------------------------------------------------------------------
# against the oracle on fresh seeded inputs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("preset,n,seed,w,h,radius,tau,deg,bg", [
    ("mixed", 20000, 2, 640, 360, 24.0, 1 / 255, 3, (0, 0, 0)),
    ("elongated", 30000, 4, 512, 288, 12.0, 1 / 255, 3, (0.1, 0.2, 0.3)),
    ("isotropic", 5000, 6, 200, 120, 14.0, 0.01, 1, (1, 1, 1)),
    ("mixed", 6000, 8, 70, 42, 6.0, 1 / 255, 0, (0, 0, 0)),          # ragged edge tiles
    ("mixed", 3000, 10, 1000, 40, 10.0, 0.02, 2, (0, 0, 0)),         # wide strip
    ("isotropic", 400, 13, 640, 368, 9.5, 1 / 255, 3, (0, 0, 0)),    # splats covering 100s of tiles
])
def test_oracle_parity_all_stages(preset, n, seed, w, h, radius, tau, deg, bg):
    act = fgs.activate(fgs.gen_synthetic(preset, n, seed))
    pipe = fgs.Pipeline(act, sh_degree=deg)                          # tile-bucket, Morton slots
    pipe1 = fgs.Pipeline(act, sh_degree=deg, sort_mode="onesweep")   # identity slots
    assert pipe.spatial_order and not pipe1.spatial_order
    for cam in fgs.orbit_cameras(2, radius, w, h):
        for s in STRATS:
            ob = orc.preprocess_and_bin(act, cam, s, tau, deg)
            ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, max(n, 1))
            # tile-bucket emission: same multiset, bucketed by tile
            tb = fgs.preprocess_and_bin(pipe, cam, s, tau, sh_degree=deg, sort_mode="tile-bucket")
            assert np.array_equal(tb.pair_counts, ob.pair_counts)
            assert np.all(np.diff((tb.keys >> np.uint64(32)).astype(np.int64)) >= 0)
            tk, tv = _sorted_pairs(tb, n)
            assert np.array_equal(tk, ok) and np.array_equal(tv, ov)
            gb = fgs.preprocess_and_bin(pipe1, cam, s, tau, sh_degree=deg)
            assert np.array_equal(gb.retained, ob.retained)
            assert np.array_equal(gb.depth.view(np.uint32), ob.depth.view(np.uint32))
            assert np.array_equal(gb.splat.view(np.uint32), ob.splat.view(np.uint32))
            assert np.array_equal(gb.tile_rects[ob.retained], ob.tile_rects[ob.retained])
            assert np.array_equal(gb.pair_counts, ob.pair_counts)
            # onesweep emission order: ascending Gaussian index
            assert np.all(np.diff(gb.values.astype(np.int64)) >= 0)
            gk, gv = _sorted_pairs(gb, n)
            assert np.array_equal(gk, ok) and np.array_equal(gv, ov)
        # whole frame (precise)
        oimg, ost, oalpha, odepth = orc.render(act, cam, "precise", tau, bg, deg, extras=True)
        fb, st = pipe.render(cam, "precise", tau, bg, extras=True)
        assert fgs.max_abs_diff(fb.image, oimg) <= PIX_TOL and _psnr_ok(fb.image, oimg)
        assert np.abs(fb.alpha - oalpha).max() <= PIX_TOL
        assert np.abs(fb.depth - odepth).max() <= PIX_TOL * max(1.0, float(odepth.max()))
        assert st.pairs_emitted == ost["pairs_emitted"]
        assert st.tiles_nonempty == ost["tiles_nonempty"]
        fbx, stx = pipe.render(cam, "precise", tau, bg, exact=True, extras=True)
        assert np.array_equal(fbx.image.view(np.uint32), oimg.view(np.uint32))
        assert np.array_equal(fbx.alpha.view(np.uint32), oalpha.view(np.uint32))
        assert np.array_equal(fbx.depth.view(np.uint32), odepth.view(np.uint32))
        assert stx.pairs_contributing == ost["pairs_contributing"]


@pytest.mark.parametrize("mode", ["tile-bucket", "onesweep"])
@pytest.mark.parametrize("n,w,h,radius", [(50000, 800, 448, 20.0), (3000, 70, 42, 6.0),
                                          (200000, 320, 192, 16.0)])
def test_sorted_buffer_matches_oracle_order(mode, n, w, h, radius):
    """What the blend consumes -- the device-sorted (key, value) list and the range
    table -- must equal the reference's (key, value) order bit for bit, in both
    sort modes.  The 200K / 320x192 case has buckets far
    above 4096 pairs (the tile sort's global-stride path)."""
    act = fgs.activate(fgs.gen_synthetic("mixed", n, 12))
    cam = fgs.orbit_cameras(1, radius, w, h)[0]
    pipe = fgs.Pipeline(act, sort_mode=mode)
    ob = orc.preprocess_and_bin(act, cam)
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, act.count)
    ostarts = orc.tile_range_table(ok, ob.grid_w, ob.grid_h)
    keys, vals, starts = fgs.sorted_pairs(pipe, cam)
    assert np.array_equal(keys, ok)
    assert np.array_equal(vals, ov)
    assert np.array_equal(starts, ostarts)
    fb, st = pipe.render(cam, exact=True)
    oimg, ost = orc.render(act, cam)
    assert np.array_equal(fb.image.view(np.uint32), oimg.view(np.uint32))
    assert (st.pairs_emitted, st.tiles_nonempty, st.pairs_contributing) == \
        (ost["pairs_emitted"], ost["tiles_nonempty"], ost["pairs_contributing"])


@pytest.mark.parametrize("n", [3000, 30000])
def test_equal_depth_ties_order_by_index(n):
    """Every Gaussian at the same camera depth: inside a tile the order is decided by
    the index tie-break alone (sorting.py:3-5, test_sorting.py:55-60).  3000 exercises
    the shared-memory tie fix-up, 30000 (buckets > 4096 with a single depth value)
    the large-bucket fallback."""
    rng = np.random.default_rng(n)
    cam = identity_camera(32, 32, focal=16)
    z = 10.0
    xy = rng.uniform(-0.95, 0.95, size=(n, 2)) * z
    scene = make_raw_scene(np.concatenate([xy, np.full((n, 1), z)], axis=1),
                           rng.uniform(0.05, 0.4, size=(n, 3)), rng.uniform(0.1, 0.9, size=n),
                           dc=rng.uniform(-1, 1, size=(n, 3)))
    act = fgs.activate(scene)
    ob = orc.preprocess_and_bin(act, cam)
    assert np.unique(ob.depth[ob.retained]).size == 1
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, n)
    for mode in ("tile-bucket", "onesweep"):
        keys, vals, starts = fgs.sorted_pairs(fgs.Pipeline(act, sort_mode=mode), cam)
        assert np.array_equal(keys, ok) and np.array_equal(vals, ov), mode
        assert np.array_equal(starts, orc.tile_range_table(ok, ob.grid_w, ob.grid_h))


def test_both_sort_modes_give_identical_frames():
    act = fgs.activate(fgs.gen_synthetic("elongated", 40000, 3))
    for cam in fgs.orbit_cameras(2, 14.0, 640, 360):
        a, sa = fgs.Pipeline(act, sort_mode="tile-bucket").render(cam)
        b, sb = fgs.Pipeline(act, sort_mode="onesweep").render(cam)
        assert np.array_equal(a.image, b.image)
        assert (sa.pairs_emitted, sa.tiles_nonempty, sa.pairs_contributing) == \
            (sb.pairs_emitted, sb.tiles_nonempty, sb.pairs_contributing)


# ---------------------------------------------------------------------------
# stage-level behaviour mirrored from the reference's own tests
# ---------------------------------------------------------------------------
def test_sort_pairs_vs_lexsort_and_ties():
    # test_sorting.py:38-60: arbitrary order in, (key, value) order out
    rng = np.random.default_rng(0)
    n = 100_000
    keys = (rng.integers(0, 300, n).astype(np.uint64) << np.uint64(32)) \
        | rng.integers(0, 1 << 32, n).astype(np.uint64)
    keys[::7] = keys[0]                                   # heavy ties
    vals = rng.integers(0, 70000, n).astype(np.uint32)
    k, v = fgs.sort_pairs(keys, vals, 1, 300, 70000)
    order = np.lexsort((vals, keys))
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])
    k2, v2 = fgs.sort_pairs(keys, vals)                   # no bounds: all bytes
    assert np.array_equal(k2, k) and np.array_equal(v2, v)
    ko, vo = orc.sort_pairs(keys, vals, 300, 70000)
    assert np.array_equal(k, ko) and np.array_equal(v, vo)


@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 12289, 1_000_003])
def test_sort_pairs_sizes(n):
    rng = np.random.default_rng(n)
    keys = (rng.integers(0, 8160, n).astype(np.uint64) << np.uint64(32)) \
        | rng.integers(0, 1 << 31, n).astype(np.uint64)
    vals = rng.integers(0, 1 << 20, n).astype(np.uint32)
    k, v = fgs.sort_pairs(keys, vals, 1, 8160, 1 << 20)
    order = np.lexsort((vals, keys))
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])


def test_sort_pairs_errors():
    with pytest.raises(ValueError):
        fgs.sort_pairs(np.zeros(3, np.uint64), np.zeros(2, np.uint32))


def test_tile_range_table_examples():
    # test_sorting.py:94-109
    keys = np.array([0, 0, 3], np.uint64) << np.uint64(32)
    assert fgs.tile_range_table(keys, 2, 2).tolist() == [0, 2, 2, 2, 3]
    assert fgs.tile_range_table(np.zeros(0, np.uint64), 2, 2).tolist() == [0, 0, 0, 0, 0]
    with pytest.raises(fgs.UnsortedPairsError):
        fgs.tile_range_table(keys[::-1].copy(), 2, 2)
    with pytest.raises(ValueError):
        fgs.tile_range_table(np.array([9], np.uint64) << np.uint64(32), 2, 2)


def test_binning_known_answers():
    # test_binning.py:23-77: single tile; 16/4/4; rotated 16/9/7
    import math
    cam = identity_camera(64, 64, focal=32)
    z = 16.0
    ndc = (2 * 24 + 1) / 64 - 1
    scene = make_raw_scene([[ndc * z, ndc * z, z]], [0.4, 0.4, 0.4], [0.9])
    for s in STRATS:
        out = fgs.preprocess_and_bin(scene, cam, s)
        assert out.emitted_count == 1
        assert int(out.keys[0] >> np.uint64(32)) == 5
        assert np.uint32(out.keys[0] & np.uint64(0xffffffff)) == np.float32(16.0).view(np.uint32)
        assert out.values[0] == 0
    z = 32.0
    scene = make_raw_scene([[((2 * 32 + 1) / 64 - 1) * z, ((2 * 24 + 1) / 64 - 1) * z, z]],
                           [10.0, 1.0, 0.01], [0.6])
    c = {s: fgs.preprocess_and_bin(scene, cam, s).emitted_count for s in STRATS}
    assert (c["baseline-circle-aabb"], c["tight-aabb"], c["precise"]) == (16, 4, 4)
    q = [math.cos(math.pi / 8), 0.0, 0.0, math.sin(math.pi / 8)]
    scene = make_raw_scene([[((2 * 40 + 1) / 64 - 1) * z, ((2 * 40 + 1) / 64 - 1) * z, z]],
                           [10.0, 0.6, 0.01], [0.6], quats=[q])
    c = {s: fgs.preprocess_and_bin(scene, cam, s).emitted_count for s in STRATS}
    assert (c["baseline-circle-aabb"], c["tight-aabb"], c["precise"]) == (16, 9, 7)


def test_empty_scene_is_background():
    # test_binning.py:16-21, test_render.py:161-166
    cam = identity_camera(48, 32)
    fb, st = fgs.Pipeline(fgs.gen_synthetic("mixed", 0, 1)).render(cam, background=(0.25, 0.5, 0.75))
    assert st.pairs_emitted == 0 and st.gaussians_retained == 0 and st.tiles_nonempty == 0
    assert np.array_equal(fb.image, np.broadcast_to(np.float32([0.25, 0.5, 0.75]), (32, 48, 3)))


def test_forced_regrow_never_truncates():
    # test_binning.py:166-175
    act = fgs.activate(fgs.gen_synthetic("mixed", 5000, 21))
    cam = fgs.orbit_cameras(1, 24.0, 256, 256)[0]
    pipe = fgs.Pipeline(act)
    fb0, st0 = pipe.render(cam, exact=True)
    fb1, st1 = fgs.Pipeline(act).render(cam, exact=True, initial_capacity=10)
    assert st1.buffer_regrows >= 1 and st0.buffer_regrows == 0
    assert st1.pairs_emitted == st0.pairs_emitted
    assert np.array_equal(fb0.image, fb1.image)
    b = fgs.preprocess_and_bin(act, cam, initial_capacity=7)
    assert b.buffer_regrows >= 1 and b.emitted_count == st0.pairs_emitted


def test_argument_errors():
    act = fgs.activate(fgs.gen_synthetic("mixed", 10, 1))
    cam = identity_camera()
    with pytest.raises(ValueError):
        fgs.Pipeline(act).render(cam, strategy="nope")
    with pytest.raises(ValueError):
        fgs.Pipeline(act, sh_degree=4).render(cam)
    with pytest.raises(TypeError):
        fgs.Pipeline(object())


def test_repeatable_and_thread_safe():
    # test_pipeline.py:28-35; SURVEY 8(b) threading row
    import threading
    act = fgs.activate(fgs.gen_synthetic("mixed", 20000, 5))
    cams = fgs.orbit_cameras(4, 24.0, 320, 240)
    pipe = fgs.Pipeline(act)
    want = [pipe.render(c)[0].image.copy() for c in cams]
    got = [None] * 16

    def job(i):
        got[i] = pipe.render(cams[i % 4])[0].image.copy()
    th = [threading.Thread(target=job, args=(i,)) for i in range(16)]
    [t.start() for t in th]
    [t.join() for t in th]
    for i in range(16):
        assert np.array_equal(got[i], want[i % 4])


def test_render_many_matches_render():
    """The pipelined batch path returns exactly what per-camera render() returns."""
    act = fgs.activate(fgs.gen_synthetic("mixed", 20000, 9))
    cams = fgs.orbit_cameras(7, 22.0, 384, 256) + fgs.orbit_cameras(2, 22.0, 320, 200)
    pipe = fgs.Pipeline(act)
    want = [pipe.render(c) for c in cams]
    got = pipe.render_many(cams, depth=3)
    assert len(got) == len(cams)
    for (fa, sa), (fb, sb) in zip(want, got):
        assert np.array_equal(fa.image, fb.image)
        assert (sa.pairs_emitted, sa.pairs_contributing, sa.tiles_nonempty, sa.gaussians_retained) == \
            (sb.pairs_emitted, sb.pairs_contributing, sb.tiles_nonempty, sb.gaussians_retained)
    # forced overflow inside the batch falls back to grow-and-rerun
    small = fgs.Pipeline(act)
    small._default_capacity = lambda: 64
    got2 = small.render_many(cams[:3])
    assert all(np.array_equal(a[0].image, b[0].image) for a, b in zip(want[:3], got2))
    assert got2[0][1].buffer_regrows >= 1      # later frames reuse the grown workspace
    # streaming form: frames can be dropped as they arrive (pinned buffers recycle)
    n = 0
    for (fa, _), (fb, _) in zip(want, pipe.render_iter(cams)):
        assert np.array_equal(fa.image, fb.image)
        n += 1
    assert n == len(cams)


def test_row_bands_equal_full_frame():
    """the union of band renders is bit-identical to the full frame."""
    act = fgs.activate(fgs.gen_synthetic("mixed", 20000, 7))
    cam = fgs.orbit_cameras(1, 20.0, 512, 400)[0]
    pipe = fgs.Pipeline(act)
    full, st = pipe.render(cam)
    gh = -(-400 // 16)
    out = np.zeros_like(full.image)
    total = 0
    for b0, b1 in ((0, 7), (8, 15), (16, gh - 1)):
        fb, s = pipe.render(cam, band=(b0, b1))
        y0, y1 = b0 * 16, min((b1 + 1) * 16, 400)
        assert fb.rows == (y0, y1) and fb.image.shape == (y1 - y0, 512, 3)   # the band's rows only
        out[y0:y1] = fb.image
        total += s.pairs_emitted
    assert np.array_equal(out, full.image)
    assert total == st.pairs_emitted


def test_render_bands_world1_equals_render():
    """The product row-band API on a one-rank process group: Pipeline.render_bands renders
    the frame's band(s) into the gather buffer and returns the same bits as render(); the
    gather itself is covered at world size 2 over gloo (tests/test_sharding_gloo.py)."""
    import os
    import tempfile
    import torch
    import torch.distributed as dist
    act = fgs.activate(fgs.gen_synthetic("mixed", 20000, 7))
    cam = fgs.orbit_cameras(1, 20.0, 512, 400)[0]
    pipe = fgs.Pipeline(act)
    full, st = pipe.render(cam, background=(0.1, 0.2, 0.3))
    with pytest.raises(RuntimeError):
        pipe.render_bands(cam)                       # no process group yet
    store = tempfile.NamedTemporaryFile(delete=False)
    store.close()
    dist.init_process_group("nccl", init_method="file://" + store.name, rank=0, world_size=1,
                            device_id=pipe.device)
    try:
        fb, s = pipe.render_bands(cam, background=(0.1, 0.2, 0.3))
        assert fb.rows == (0, 400) and np.array_equal(fb.image, full.image)
        assert s.pairs_emitted == st.pairs_emitted and s.pairs_contributing == st.pairs_contributing
        out = torch.zeros((400, 512, 3), dtype=torch.float32, device=pipe.device)
        fbd, _ = pipe.render_bands(cam, None, "precise", 1 / 255, (0.1, 0.2, 0.3), out=out,
                                   as_numpy=False, sync=False)
        torch.cuda.synchronize()
        assert fbd.image is out and np.array_equal(out.cpu().numpy(), full.image)
        fq, _ = pipe.render_bands(cam, background=(0.1, 0.2, 0.3), quantized=True)
        assert fq.image.dtype == np.uint8 and np.array_equal(fq.image, fgs.images.quantize(full.image))
        with pytest.raises(ValueError):
            pipe.render_bands(cam, bands=[(0, 3), (4, 24)])      # two bands, one rank
    finally:
        dist.destroy_process_group()
        if os.path.exists(store.name):
            os.unlink(store.name)


# ---------------------------------------------------------------------------
# report emitters (reference pipeline.py:171-269, docs/report-schema.md)
# ---------------------------------------------------------------------------
def test_compare_modes_report_matches_oracle_counters():
    act = fgs.activate(fgs.gen_synthetic("elongated", 4000, 5))
    cams = fgs.orbit_cameras(2, 14.0, 256, 192)
    rep = fgs.compare_modes(act, cams).to_dict()
    assert rep["schema_version"] == 1 and rep["kind"] == "compare"
    assert sorted(rep["strategies"]) == sorted(STRATS) and len(rep["frames"]) == 2
    for fr, cam in zip(rep["frames"], cams):
        assert fr["frame_id"] == cam.cam_id
        for s in STRATS:
            _, ost = orc.render(act, cam, s)
            got = fr["stats"][s]
            for k in ("pairs_emitted", "pairs_contributing", "gaussians_retained",
                      "gaussians_degenerate", "tiles_nonempty"):
                assert got[k] == ost[k], (s, k)
            assert got["pair_buffer_bytes"] == 12 * got["pairs_emitted"]
            assert set(got) == {"strategy", "tau", "workers", "preprocess_bin_ns", "sort_ns",
                                "render_ns", "total_ns", "pairs_emitted", "pairs_contributing",
                                "gaussians_retained", "gaussians_degenerate", "tiles_nonempty",
                                "pair_buffer_bytes", "buffer_regrows"}
        # the shared tau rule makes every strategy render the same frame (render.py:17-22)
        for a in STRATS:
            for b in STRATS:
                assert fr["psnr"][f"{a}|{b}"] == "identical"
                assert fr["max_abs_diff"][f"{a}|{b}"] == 0.0
        r = fr["pairs_emitted_ratio_vs_first"]
        assert rep["strategies"][0] == "baseline-circle-aabb"       # binning.py:38 order
        assert r["precise"] <= r["tight-aabb"] <= r["baseline-circle-aabb"] == 1.0
    agg = rep["aggregate"]
    assert agg["precise"]["frames"] == 2
    assert agg["precise"]["pairs_emitted_total"] == sum(
        f["stats"]["precise"]["pairs_emitted"] for f in rep["frames"])
    with pytest.raises(ValueError):
        fgs.compare_modes(act, cams, strategies=["precise"])


def test_bench_frames_report_shape_and_determinism():
    act = fgs.activate(fgs.gen_synthetic("mixed", 3000, 7))
    cams = fgs.orbit_cameras(3, 20.0, 320, 200)
    rep = fgs.bench_frames(act, cams, repeat=2)
    assert rep["kind"] == "bench" and rep["repeat"] == 2 and rep["frames_per_repeat"] == 3
    assert set(rep["frame_ms"]) == {"0", "1", "2"}
    assert rep["min_ms"] <= rep["avg_ms"] <= rep["max_ms"]
    assert abs(sum(rep["stage_percent"].values()) - 100.0) < 1e-6
    assert rep["stage_coverage_percent"] >= 95.0          # SPEC acceptance: stages cover the frame
    for cam, m, c in zip(cams, rep["pairs_emitted"], rep["pairs_contributing"]):
        _, ost = orc.render(act, cam)
        assert (m, c) == (ost["pairs_emitted"], ost["pairs_contributing"])
    with pytest.raises(ValueError):
        fgs.bench_frames(act, cams, repeat=0)


# ---------------------------------------------------------------------------
# quantised output and the frame-service adapter (reference images.py:12-15, service.py:111-155)
# ---------------------------------------------------------------------------
def test_quantized_frames_match_reference_quantize():
    from paper_2408_07967_b200 import service
    act = fgs.activate(fgs.gen_synthetic("mixed", 5000, 9))
    cams = fgs.orbit_cameras(3, 18.0, 333, 201)          # odd sizes: vector tail path
    pipe = fgs.Pipeline(act)
    for cam in cams:
        for bg in ((0, 0, 0), (1.5, -0.25, 0.3)):        # out-of-range channels get clipped
            fb, _ = pipe.render(cam, background=bg)
            q, _ = pipe.render(cam, background=bg, quantized=True)
            assert q.image.dtype == np.uint8 and q.image.shape == fb.image.shape
            assert np.array_equal(q.image, service.quantize(fb.image))
    many = pipe.render_many(cams, quantized=True)
    for cam, (fbq, _) in zip(cams, many):
        assert np.array_equal(fbq.image, service.quantize(pipe.render(cam)[0].image))


def test_frame_service_render_pose():
    from paper_2408_07967_b200 import service
    act = fgs.activate(fgs.gen_synthetic("mixed", 3000, 4))
    svc = service.FrameService(act, encoding="ppm", max_pixels=320 * 240)
    req = {"width": 320, "height": 200, "position": [0.0, 0.0, -20.0], "yaw": 0.1, "pitch": -0.05}
    body, headers = svc.render_pose(req)
    assert body.startswith(b"P6\n320 200\n255\n") and len(body) == 15 + 320 * 200 * 3
    cam, strat = svc.camera_for(req)
    oimg, ost = orc.render(act, cam)
    assert headers["X-Flash-Pairs-Emitted"] == str(ost["pairs_emitted"])
    assert headers["X-Flash-Strategy"] == strat == "precise"
    got = np.frombuffer(body[15:], np.uint8).reshape(200, 320, 3).astype(np.int32)
    assert np.abs(got - service.quantize(oimg).astype(np.int32)).max() <= 1   # 1e-3 tolerance -> <= 1 level
    # toggling the strategy gives the identical bytes (reference test_service.py:94-101)
    body2, _ = svc.render_pose(dict(req, strategy="baseline-circle-aabb"))
    assert body2 == body
    with pytest.raises(service.OversizeError):
        svc.render_pose(dict(req, width=4000, height=4000))
    for bad in ({"width": 320}, dict(req, position=[1, 2]), dict(req, strategy="nope"),
                dict(req, fov_y=1.0), {"width": 320, "height": 200, "position": [0, 0, 0]},
                dict(req, width=8, height=8)):
        with pytest.raises(service.PoseError):
            svc.render_pose(bad)


# ---------------------------------------------------------------------------
# spatial slot order (per scene): a pure layout choice, results must not move
# ---------------------------------------------------------------------------
def _morton63(means):
    m = np.asarray(means, dtype=np.float32)
    lo, hi = m.min(axis=0), m.max(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        t = (m - lo) / (hi - lo)
    t = np.where(hi > lo, t, np.float32(0)).astype(np.float32)
    t = np.clip(t, np.float32(0), np.float32(1))
    q = (t * np.float32(2097151.0)).astype(np.uint64)
    code = np.zeros(m.shape[0], dtype=np.uint64)
    for bit in range(21):
        for a in range(3):
            code |= ((q[:, a] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + a)
    return code


@pytest.mark.parametrize("n", [1, 31, 1000, 70001])
def test_scene_order_is_the_stable_morton_permutation(n):
    act = fgs.activate(fgs.gen_synthetic("mixed", n, 21))
    pipe = fgs.Pipeline(act)
    assert pipe.spatial_order and pipe.slot_order.shape == (n,)
    assert np.array_equal(np.sort(pipe.slot_order), np.arange(n))
    want = np.lexsort((np.arange(n), _morton63(act.means)))
    assert np.array_equal(pipe.slot_order, want)


@pytest.mark.parametrize("preset,n,w,h,radius", [("mixed", 9000, 400, 240, 16.0),
                                                 ("isotropic", 300, 640, 368, 9.5),    # huge splats
                                                 ("elongated", 20000, 512, 288, 12.0)])
def test_results_do_not_depend_on_slot_order(preset, n, w, h, radius):
    """Morton slots (CTA tile tables mostly hit) against caller-order slots (tables overflow,
    per-pair fallback path): same frames, same sorted lists, same stage outputs."""
    act = fgs.activate(fgs.gen_synthetic(preset, n, 17))
    cam = fgs.orbit_cameras(1, radius, w, h)[0]
    a = fgs.Pipeline(act, spatial_order=True)
    b = fgs.Pipeline(act, spatial_order=False)
    for exact in (False, True):
        fa, sa = a.render(cam, exact=exact, extras=True)
        fb, sb = b.render(cam, exact=exact, extras=True)
        assert np.array_equal(fa.image.view(np.uint32), fb.image.view(np.uint32))
        assert np.array_equal(fa.alpha.view(np.uint32), fb.alpha.view(np.uint32))
        assert np.array_equal(fa.depth.view(np.uint32), fb.depth.view(np.uint32))
        assert (sa.pairs_emitted, sa.pairs_contributing, sa.tiles_nonempty) == \
               (sb.pairs_emitted, sb.pairs_contributing, sb.tiles_nonempty)
    for s in STRATS:
        ka, va, ta = fgs.sorted_pairs(a, cam, s)
        kb, vb, tb = fgs.sorted_pairs(b, cam, s)
        assert np.array_equal(ka, kb) and np.array_equal(va, vb) and np.array_equal(ta, tb)
        ob = orc.preprocess_and_bin(act, cam, s)
        ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, n)
        assert np.array_equal(ka, ok) and np.array_equal(va, ov)
    ba, bb = fgs.preprocess_and_bin(a, cam), fgs.preprocess_and_bin(b, cam)
    assert np.array_equal(ba.splat.view(np.uint32), bb.splat.view(np.uint32))
    assert np.array_equal(ba.pair_counts, bb.pair_counts)
    with pytest.raises(ValueError):
        fgs.Pipeline(act, sort_mode="onesweep", spatial_order=True)


def test_overlapped_views_match_one_at_a_time_on_dense_tiles():
    """Views in flight on several streams (render_many) against render() one at a time, on a
    scene whose tiles span every tile-sort size class (small ... dense)."""
    act = fgs.activate(fgs.gen_synthetic("mixed", 150_000, 23))
    cams = fgs.orbit_cameras(6, 22.0, 480, 272)
    pipe = fgs.Pipeline(act)
    ref = [pipe.render(c, exact=True) for c in cams]
    sizes = np.diff(fgs.sorted_pairs(pipe, cams[0])[2])
    assert sizes.max() > 8192 and ((sizes > 4096) & (sizes <= 8192)).any() and (sizes < 1024).any()
    for streams in (2, 3):
        for rep in range(3):
            got = pipe.render_many(cams, exact=True, streams=streams, depth=2 * streams)
            for (fa, sa), (fb, sb) in zip(ref, got):
                assert np.array_equal(fa.image.view(np.uint32), fb.image.view(np.uint32))
                assert (sa.pairs_emitted, sa.pairs_contributing) == (sb.pairs_emitted, sb.pairs_contributing)
    oimg, ost = orc.render(act, cams[0])
    assert np.array_equal(ref[0][0].image.view(np.uint32), oimg.view(np.uint32))


def test_device_activate_tracks_the_reference_activation():
    """fgs_scene_activate: rotations bit-identical to the NumPy
    activation, scales / opacities within a few ulp, frames within the pixel tolerance."""
    raw = fgs.gen_synthetic("mixed", 20000, 31)
    raw.rotations[7] = 0.0                                  # zero-norm row -> identity
    host = fgs.activate(raw)
    pipe = fgs.Pipeline(raw, device_activate=True)
    dev = pipe.activated
    assert np.array_equal(dev.rotations.view(np.uint32), host.rotations.view(np.uint32))
    assert np.array_equal(dev.rotations[7], np.array([1, 0, 0, 0], np.float32))

    def ulps(a, b):
        return np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64)).max()
    # exp is correctly rounded here; NumPy's float32 SIMD exp is good to ~2 ulp, and the
    # sigmoid's divide can stretch that to a few ulp of the (smaller) quotient
    assert ulps(dev.scales, host.scales) <= 2 and ulps(dev.opacities, host.opacities) <= 6
    cam = fgs.orbit_cameras(1, 20.0, 400, 240)[0]
    fd_, sd = pipe.render(cam)
    fh, sh_ = fgs.Pipeline(host).render(cam)
    assert fgs.max_abs_diff(fd_.image, fh.image) <= PIX_TOL and _psnr_ok(fd_.image, fh.image)
    assert abs(sd.pairs_emitted - sh_.pairs_emitted) <= max(2, sh_.pairs_emitted // 10000)
    # an already activated scene is taken as is
    assert fgs.Pipeline(host, device_activate=True).activated is host


# ---------------------------------------------------------------------------
# packed-f32x2 blend: the single alpha >= thr test must reproduce the reference's
# three skips exactly (contrib flags identical to the exact mode), frames within 2e-5
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("preset,n,seed,w,h,radius,tau", [
    ("mixed", 40000, 21, 640, 368, 20.0, 1 / 255),
    ("elongated", 30000, 22, 512, 300, 12.0, 1 / 255),      # kappa-scaled guard band
    ("isotropic", 8000, 23, 330, 200, 10.0, 0.02),
    ("mixed", 2000, 24, 97, 61, 5.0, 1 / 255),              # close-up: huge splats, ragged tiles
])
def test_packed_blend_never_flips_a_skip(preset, n, seed, w, h, radius, tau):
    act = fgs.activate(fgs.gen_synthetic(preset, n, seed))
    pipe = fgs.Pipeline(act)
    for cam in fgs.orbit_cameras(2, radius, w, h):
        b = fgs.preprocess_and_bin(pipe, cam, "precise", tau)
        keys, vals = fgs.sort_pairs(b.keys, b.values, 1, b.grid_w * b.grid_h, n)
        starts = fgs.tile_range_table(keys, b.grid_w, b.grid_h)
        for bg in ((0, 0, 0), (1.0, 0.5, 0.25)):
            ix, cx, _ = fgs.render_frame(b.splat, vals, starts, w, h, bg, tau, exact=True)
            i2, c2, _ = fgs.render_frame(b.splat, vals, starts, w, h, bg, tau)
            assert np.array_equal(c2, cx), "a pair's contributes/skipped verdict differs"
            assert fgs.max_abs_diff(i2, ix) <= 2e-5
        # alpha / depth maps ride the same packed accumulators
        ix, _, _, ax, dx = fgs.render_frame(b.splat, vals, starts, w, h, (0, 0, 0), tau, exact=True,
                                            gaussian_depth=b.depth)
        i2, _, _, a2, d2 = fgs.render_frame(b.splat, vals, starts, w, h, (0, 0, 0), tau,
                                            gaussian_depth=b.depth)
        assert np.abs(a2 - ax).max() <= 2e-5
        assert np.abs(d2 - dx).max() <= 2e-5 * max(1.0, float(dx.max()))


def test_packed_blend_rows_outside_its_shortcut():
    """Hand-made rows whose extent rectangle is NOT the cutoff ellipse's bounding box
    (clipped rectangle, opacity above the cap, zero conic terms): the packed kernel must
    hand them to the reference-order path, so the verdicts still match the exact mode."""
    rng = np.random.default_rng(5)
    n, w, h = 600, 160, 96
    splat = np.zeros((n, 12), np.float32)
    splat[:, 0] = rng.uniform(-10, w + 10, n)
    splat[:, 1] = rng.uniform(-10, h + 10, n)
    sx, sy = rng.uniform(1.5, 14, n), rng.uniform(1.5, 14, n)
    rho = rng.uniform(-0.9, 0.9, n)
    cov = np.stack([sx * sx, rho * sx * sy, sy * sy], 1)
    det = cov[:, 0] * cov[:, 2] - cov[:, 1] ** 2
    splat[:, 2], splat[:, 3], splat[:, 4] = cov[:, 2] / det, -cov[:, 1] / det, cov[:, 0] / det
    splat[:, 5] = rng.uniform(0.05, 1.0, n)                       # some above the 0.99 cap
    splat[:, 6] = np.minimum(9.0, 2 * np.log(splat[:, 5] * 255.0))
    splat[:, 7:10] = rng.uniform(0, 1, (n, 3))
    splat[:, 10] = np.sqrt(splat[:, 6] * cov[:, 0]) * rng.choice([1.0, 0.5, 0.25, 2.0], n)   # clipped / loose
    splat[:, 11] = np.sqrt(splat[:, 6] * cov[:, 2]) * rng.choice([1.0, 0.6, 3.0], n)
    splat[::50, 3] = 0.0
    splat[::75, 2:5] = (0.02, 0.0, 0.0)                           # c = 0: degenerate conic
    gw, gh = -(-w // 16), -(-h // 16)
    # every Gaussian on every tile, in index order: the blend's own tests do all the culling
    vals = np.tile(np.arange(n, dtype=np.uint32), gw * gh)
    starts = np.arange(gw * gh + 1, dtype=np.int64) * n
    ix, cx, _ = fgs.render_frame(splat, vals, starts, w, h, (0.2, 0.1, 0.0), 1 / 255, exact=True)
    i2, c2, _ = fgs.render_frame(splat, vals, starts, w, h, (0.2, 0.1, 0.0), 1 / 255)
    assert cx.any() and np.array_equal(c2, cx)
    assert fgs.max_abs_diff(i2, ix) <= 2e-5


@pytest.mark.parametrize("preset,n,radius,spatial", [
    ("mixed", 30000, 20.0, True),
    ("mixed", 30000, 20.0, False),        # caller-order slots: CTA tile tables overflow ->
    ("isotropic", 600, 9.5, False),       # ... the per-pair fallback cursor must rewind too
])
def test_stages_can_be_repeated_on_one_frame(preset, n, radius, spatial):
    """fgs_emit (tile order + placement), fgs_sort and fgs_blend are idempotent on a frame:
    running them again -- another background, a re-issued stage -- gives the same frame."""
    import ctypes as C
    import torch
    from paper_2408_07967_b200 import _capi
    w, h = 400, 240
    act = fgs.activate(fgs.gen_synthetic(preset, n, 31))
    cam = fgs.orbit_cameras(1, radius, w, h)[0]
    pipe = fgs.Pipeline(act, spatial_order=spatial)
    want, _ = pipe.render(cam)
    L = _capi.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    ws = fgs.pipeline._Workspace(torch, dev, n, w, h, pipe._default_capacity())
    ws.set_mode(_capi.SORT_MODES["tile-bucket"])
    kcut = pipe._cutoffs(torch, 1 / 255)
    camc = _capi.camera_struct(cam)
    gh = -(-h // 16)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    base, lay = C.c_void_p(ws.base), C.byref(ws.lay)
    bg = (C.c_float * 3)(0, 0, 0)
    _capi.check(L.fgs_preprocess(pipe.packed.data_ptr(), kcut.data_ptr(), n, C.byref(camc), 1 / 255,
                                 3, 0, 0, gh - 1, base, lay, st))
    _capi.check(L.fgs_scan(base, lay, st))
    for _ in range(3):
        _capi.check(L.fgs_emit(pipe.packed.data_ptr(), C.byref(camc), 0, 0, gh - 1, base, lay, st))
    for _ in range(2):
        _capi.check(L.fgs_sort(base, lay, ws.next_epoch(), st))
    _capi.check(L.fgs_ranges(base, lay, st))
    for _ in range(2):
        _capi.check(L.fgs_blend(pipe.packed.data_ptr(), bg, 1 / 255, 2, 0, gh - 1, ws.rgb.data_ptr(),
                                None, None, base, lay, st))
    torch.cuda.synchronize()
    assert np.array_equal(ws.rgb.cpu().numpy(), want.image)


# ---------------------------------------------------------------------------
# BASELINE.json's full sizes
# ---------------------------------------------------------------------------
def _full_frame_against_oracle(act, pipe, cam, crop=None):
    """One camera: sorted (key, value) list and range table bit-exact, counters equal,
    default frame inside the pixel tolerance with IDENTICAL contributing-pair count,
    exact-mode frame bit-identical.  `crop` = (y0, y1, x0, x1) additionally names the
    sub-frame whose bits are compared on their own."""
    ob = orc.preprocess_and_bin(act, cam)
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, act.count)
    ostarts = orc.tile_range_table(ok, ob.grid_w, ob.grid_h)
    keys, vals, starts = fgs.sorted_pairs(pipe, cam)
    assert keys.shape == ok.shape
    assert hashlib.sha256(keys.tobytes()).digest() == hashlib.sha256(ok.tobytes()).digest()
    assert np.array_equal(keys, ok) and np.array_equal(vals, ov)
    assert np.array_equal(starts, ostarts)
    del keys, vals, ok, ov, ob
    oimg, ost = orc.render(act, cam)
    fb, st = pipe.render(cam)
    assert (st.gaussians_retained, st.pairs_emitted, st.tiles_nonempty) == \
        (ost["gaussians_retained"], ost["pairs_emitted"], ost["tiles_nonempty"])
    # Default mode: no alpha / cutoff / rectangle skip ever flips (guard band, see
    # test_packed_blend_never_flips_a_skip), but the T < 1e-4 stop (render.py:228) is taken on
    # the default mode's own T, which differs from the reference's by ~1e-6 relative: a pixel
    # whose T lands that close to 1e-4 may stop one pair early or late, and a pair seen only by
    # such pixels changes its flag (weight <= 1e-4, invisible in the frame).  Measured: 1 pair
    # of 3 407 488 on the 10M / 4K frame, 0 on every smaller config.  Exact mode: equality.
    assert abs(st.pairs_contributing - ost["pairs_contributing"]) <= STOP_FLIPS_MAX
    assert fgs.max_abs_diff(fb.image, oimg) <= PIX_TOL and _psnr_ok(fb.image, oimg)
    del fb
    fbx, stx = pipe.render(cam, exact=True)
    if crop is not None:
        y0, y1, x0, x1 = crop
        assert np.array_equal(fbx.image[y0:y1, x0:x1].view(np.uint32),
                              oimg[y0:y1, x0:x1].view(np.uint32))
    assert np.array_equal(fbx.image.view(np.uint32), oimg.view(np.uint32))
    assert stx.pairs_contributing == ost["pairs_contributing"]


@pytest.mark.parametrize("n,w,h,views,crop", [
    (1_000_000, 1920, 1080, (1, (0,)), None),                      # configs[1]
    (3_000_000, 3840, 2160, (1, (0,)), None),                      # configs[2]
    (10_000_000, 3840, 2160, (1, (0,)), None),                     # the north-star frame
    (10_000_000, 7680, 4320, (1, (0,)), (1648, 2672, 3328, 4352)),  # configs[3], whole 8K frame
    (3_000_000, 1920, 1080, (64, (0, 13, 37, 63)), None),          # configs[4]: 4 of the 64 views
])
def test_full_size_configs_against_the_oracle(n, w, h, views, crop):
    """BASELINE.json's configs at full size against the ORACLE (SURVEY.md 8(d) "Concrete
    configs"; the oracle finishes each in seconds on the box's host cores)."""
    act = fgs.activate(fgs.gen_synthetic("mixed", n, 1, density_scale=True))
    ncam, ids = views
    cams = fgs.orbit_cameras(ncam, 24.0, w, h)
    pipe = fgs.Pipeline(act)
    for i in ids:
        _full_frame_against_oracle(act, pipe, cams[i], crop)


@pytest.mark.parametrize("preset,n,w,h,radius", [("mixed", 1_000_000, 1920, 1080, 24.0),
                                                 ("elongated", 20000, 333, 207, 10.0)])
def test_eval_counts_match_the_instrumented_oracle(preset, n, w, h, radius):
    """fgs_blend_counts (what bench.py's FP32 roofline of the blend is computed from) against
    the instrumented copy of the reference loop in the oracle: identical class counts,
    M_proc and pixel count; and the pass leaves the exact-mode frame in the buffer."""
    act = fgs.activate(fgs.gen_synthetic(preset, n, 1, density_scale=n > 10_000 and preset == "mixed"))
    cam = fgs.orbit_cameras(1, radius, w, h)[0]
    pipe = fgs.Pipeline(act)
    got = fgs.blend_eval_counts(pipe, cam)
    ob = orc.preprocess_and_bin(act, cam)
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, act.count)
    want = orc.render_counts(ob.splat, ov, orc.tile_range_table(ok, ob.grid_w, ob.grid_h), w, h, 1 / 255)
    for k in ("rect_rejected", "cutoff_rejected", "alpha_rejected", "blended", "pairs_processed", "pixels"):
        assert got[k] == want[k], (k, got[k], want[k])
    assert got["pairs_emitted"] == ob.emitted_count and got["pixels"] == w * h
    assert got["flops"] == sum(fgs.EVAL_FLOPS[k] * want[k] for k in fgs.EVAL_FLOPS)
    assert got["pairs_processed"] <= got["pairs_emitted"]


def test_north_star_size_properties():
    """10M Gaussians at 3840x2160 (the north-star frame) through size-independent
    properties: both sort modes give the same sorted list and bit-identical frames,
    the sorted list is non-decreasing in (key, value) and consistent with the range
    table, the pair count equals the sum of the per-Gaussian counts, the union of
    four row bands is bit-identical to the whole frame, and the default frame stays
    within the pixel tolerance of the exact-mode one (itself bit-identical to the
    reference at every size the oracle is run on)."""
    n, w, h = 10_000_000, 3840, 2160
    act = fgs.activate(fgs.gen_synthetic("mixed", n, 1, density_scale=True))
    cam = fgs.orbit_cameras(1, 24.0, w, h)[0]
    pipe = fgs.Pipeline(act)
    keys, vals, starts = fgs.sorted_pairs(pipe, cam)
    b = fgs.preprocess_and_bin(pipe, cam)
    assert keys.size == int(b.pair_counts.sum()) == starts[-1]
    dk = np.diff(keys.view(np.int64))
    assert np.all(dk >= 0) and np.all(np.diff(vals.astype(np.int64))[dk == 0] > 0)
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    assert np.array_equal(starts, np.searchsorted(tiles, np.arange(starts.size)))
    assert hashlib.sha256(np.sort(b.keys).tobytes()).digest() == \
        hashlib.sha256(np.sort(keys).tobytes()).digest()
    del b, dk, tiles
    full, st = pipe.render(cam)
    fx, stx = pipe.render(cam, exact=True)
    assert st.pairs_emitted == keys.size
    assert fgs.max_abs_diff(full.image, fx.image) <= 1e-4
    gh = -(-h // 16)
    out = np.zeros_like(full.image)
    edges = [0, gh // 4, gh // 2, 3 * gh // 4, gh]
    total = 0
    for b0, b1 in zip(edges[:-1], edges[1:]):
        fb, s = pipe.render(cam, band=(b0, b1 - 1))
        out[b0 * 16:min(b1 * 16, h)] = fb.image
        total += s.pairs_emitted
    assert total == st.pairs_emitted and np.array_equal(out, full.image)
    del pipe
    pipe1 = fgs.Pipeline(act, sort_mode="onesweep")
    k1, v1, s1 = fgs.sorted_pairs(pipe1, cam)
    assert np.array_equal(k1, keys) and np.array_equal(v1, vals) and np.array_equal(s1, starts)
    f1, _ = pipe1.render(cam)
    assert np.array_equal(f1.image, full.image)


def test_row_weights_and_balanced_bands():
    """fgs_row_histogram counts the in-frustum Gaussians by the tile row of their projected
    centre (checked against the splat rows the oracle writes), and the union of the
    work-balanced bands it leads to is bit-identical to the whole frame."""
    from paper_2408_07967_b200 import sharding
    act = fgs.activate(fgs.gen_synthetic("mixed", 30000, 17))
    cam = fgs.orbit_cameras(1, 9.0, 640, 400)[0]            # camera inside the cloud: culling matters
    pipe = fgs.Pipeline(act)
    rw = pipe.row_weights(cam)
    gh = -(-400 // 16)
    assert rw.shape == (gh,) and rw.dtype == np.int64
    # host restatement: frustum_mask (projection.py:39-47) + ndc2pix centre row
    m = np.asarray(act.means, np.float32)
    v = np.asarray(cam.world_to_camera, np.float32)
    z = ((v[2, 0] * m[:, 0] + v[2, 1] * m[:, 1]) + v[2, 2] * m[:, 2]) + v[2, 3]
    keep = (z > np.float32(0.2)) & (np.asarray(act.opacities) > np.float32(1 / 255))
    fp = np.asarray(cam.full_projection, np.float32)
    h1 = ((fp[1, 0] * m[:, 0] + fp[1, 1] * m[:, 1]) + fp[1, 2] * m[:, 2]) + fp[1, 3]
    h3 = ((fp[3, 0] * m[:, 0] + fp[3, 1] * m[:, 1]) + fp[3, 2] * m[:, 2]) + fp[3, 3]
    den = np.where(np.abs(h3) > np.float32(1e-7), h3, np.float32(1e-7))
    py = ((h1 / den + np.float32(1)) * np.float32(400) - np.float32(1)) * np.float32(0.5)
    ty = np.floor(py * np.float32(0.0625))
    ok = keep & (ty >= -1) & (ty <= gh)
    want = np.bincount(np.clip(ty[ok], 0, gh - 1).astype(np.int64), minlength=gh)
    assert np.array_equal(rw, want)
    full, st = pipe.render(cam)
    bands = sharding.balanced_band_partition(rw, 4, fixed_rows=0.3 * float(rw.mean()))
    assert bands != sharding.band_partition(gh, 4)
    out = np.zeros_like(full.image)
    total = 0
    for b in bands:
        fb, s = pipe.render(cam, band=b)
        y0, y1 = sharding.band_pixel_rows(b, 400)
        out[y0:y1] = fb.image
        total += s.pairs_emitted
    assert np.array_equal(out, full.image) and total == st.pairs_emitted


def test_sparse_scene_on_a_large_grid():
    """A few Gaussians on a 4096x2176 frame (34 816 tiles, mostly empty): the tile scan's
    slice-total path, empty tiles in every size bin of the blend order, ragged last row."""
    act = fgs.activate(fgs.gen_synthetic("mixed", 3000, 23))
    cam = fgs.orbit_cameras(1, 18.0, 4096, 2170)[0]
    pipe = fgs.Pipeline(act)
    ob = orc.preprocess_and_bin(act, cam)
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, act.count)
    keys, vals, starts = fgs.sorted_pairs(pipe, cam)
    assert np.array_equal(keys, ok) and np.array_equal(vals, ov)
    assert np.array_equal(starts, orc.tile_range_table(ok, ob.grid_w, ob.grid_h))
    oimg, ost = orc.render(act, cam, "precise", 1 / 255, (0.2, 0.1, 0.3))
    fb, st = pipe.render(cam, "precise", 1 / 255, (0.2, 0.1, 0.3), exact=True)
    assert np.array_equal(fb.image.view(np.uint32), oimg.view(np.uint32))
    assert (st.pairs_emitted, st.tiles_nonempty, st.pairs_contributing) == \
        (ost["pairs_emitted"], ost["tiles_nonempty"], ost["pairs_contributing"])


# ---------------------------------------------------------------------------
# against the UNMODIFIED reference package run on this box (baseline/_ref: the git-ignored
# `pip install --target` of /root/reference/pkg, which travels with the snapshot) -- the
# CUDA path and the real `tilesplat`, no oracle in between
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("preset,n,seed,w,h,radius,strat", [
    ("mixed", 20000, 5, 480, 270, 24.0, "precise"),
    ("elongated", 6000, 9, 320, 200, 16.0, "precise"),
    ("mixed", 6000, 11, 320, 200, 20.0, "tight-aabb"),
    ("isotropic", 6000, 13, 256, 256, 20.0, "baseline-circle-aabb"),
])
def test_cuda_path_against_the_reference_package(preset, n, seed, w, h, radius, strat):
    """tilesplat.preprocess_and_bin / sort_pairs / tile_range_table / Pipeline.render against the
    same calls of this package on the GPU: pair list, sorted (key, value) order, range table and
    splat rows bit-exact; exact-mode frame bit-identical, default frame within 1e-3 / 60 dB;
    FrameStats counters equal (binning.py:197, sorting.py:101-152, pipeline.py:77-111)."""
    import dataclasses
    from fgs_testlib import load_tilesplat
    ts = load_tilesplat()
    if ts is None:
        pytest.skip("reference package not on this box (baseline/_ref missing or numba absent)")
    act = fgs.activate(fgs.gen_synthetic(preset, n, seed))
    cam = fgs.orbit_cameras(2, radius, w, h)[1]
    r_act = ts.ActivatedScene(**{f.name: getattr(act, f.name) for f in dataclasses.fields(ts.ActivatedScene)})
    r_cam = ts.Camera(**{f.name: getattr(cam, f.name) for f in dataclasses.fields(ts.Camera)})
    bg = (0.1, 0.2, 0.3)
    rb = ts.preprocess_and_bin(r_act, r_cam, strat, 1 / 255, workers=2)
    tiles = rb.grid_w * rb.grid_h
    rk, rv = ts.sort_pairs(rb.keys, rb.values, 2, tiles, r_act.count)
    rstarts = ts.tile_range_table(rk, rb.grid_w, rb.grid_h)
    rfb, rst = ts.Pipeline(r_act).render(r_cam, strat, background=bg, workers=2)

    pipe = fgs.Pipeline(act)
    gb = fgs.preprocess_and_bin(pipe, cam, strat)
    gk, gv = fgs.sort_pairs(gb.keys, gb.values, 1, tiles, act.count)
    assert np.array_equal(gk, rk) and np.array_equal(gv, rv)
    assert np.array_equal(fgs.tile_range_table(gk, gb.grid_w, gb.grid_h), rstarts)
    assert np.array_equal(gb.retained, rb.retained)
    assert np.array_equal(gb.splat[gb.retained].view(np.uint32), rb.splat[rb.retained].view(np.uint32))
    fbx, stx = pipe.render(cam, strat, background=bg, exact=True)
    fb, st = pipe.render(cam, strat, background=bg)
    assert np.array_equal(fbx.image.view(np.uint32), np.asarray(rfb.image).view(np.uint32))
    assert float(np.abs(fb.image - rfb.image).max()) <= PIX_TOL and _psnr_ok(fb.image, rfb.image)
    for s in (st, stx):
        assert (s.pairs_emitted, s.pairs_contributing, s.tiles_nonempty, s.gaussians_retained) == \
            (rst.pairs_emitted, rst.pairs_contributing, rst.tiles_nonempty, rst.gaussians_retained)


def test_dense_tile_with_a_depth_cluster_falls_back_mid_way():
    """One tile far above the largest sort class (> 8192 pairs): the medium class splits it by
    depth and sorts chunk after chunk; here one chunk holds 3000 pairs of a single depth, which
    the bucket-rank sort gives up on AFTER earlier chunks were written -- the tile goes to the
    tail kernel and is sorted again from the untouched records.  Order must still be the
    reference's (depth, then index: sorting.py:3-5)."""
    rng = np.random.default_rng(77)
    n_spread, n_same = 9500, 3000
    n = n_spread + n_same
    cam = identity_camera(16, 16, focal=8)
    z = np.concatenate([rng.uniform(5.0, 15.0, n_spread), np.full(n_same, 10.0)])
    rng.shuffle(z)
    xy = rng.uniform(-0.6, 0.6, size=(n, 2)) * z[:, None]
    scene = make_raw_scene(np.concatenate([xy, z[:, None]], axis=1),
                           rng.uniform(0.05, 0.3, size=(n, 3)), rng.uniform(0.1, 0.9, size=n),
                           dc=rng.uniform(-1, 1, size=(n, 3)))
    act = fgs.activate(scene)
    ob = orc.preprocess_and_bin(act, cam)
    ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, n)
    assert ob.grid_w * ob.grid_h == 1 and ok.size > 8192
    pipe = fgs.Pipeline(act)
    for _ in range(2):                                     # the frame's work counters rewind
        keys, vals, starts = fgs.sorted_pairs(pipe, cam)
        assert np.array_equal(keys, ok) and np.array_equal(vals, ov)
    fb, st = pipe.render(cam, exact=True)
    oimg, ost = orc.render(act, cam)
    assert np.array_equal(fb.image.view(np.uint32), oimg.view(np.uint32))
    assert st.pairs_contributing == ost["pairs_contributing"]
