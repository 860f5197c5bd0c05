"""Pin the CPU oracle to the reference: every stage boundary of every golden
case (outputs of the reference itself, tests/golden/make_golden.py) must be
reproduced BIT-FOR-BIT by oracle/fgs_oracle.c.  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from fgs_testlib import GoldenCase

STRATS = ("precise", "tight-aabb", "baseline-circle-aabb")


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def test_cutoffs_match_reference(golden):
    k, _ = orc.power_cutoffs(golden.act.opacities, golden.tau)
    assert np.array_equal(k.view(np.uint32), golden.z["k"].view(np.uint32))


def test_pair_counts_all_strategies(golden):
    for ci in range(golden.ncam):
        cam = golden.camera(ci)
        counts = {}
        for s in STRATS:
            b = orc.preprocess_and_bin(golden.act, cam, s, golden.tau, golden.sh_degree)
            counts[s] = b.emitted_count
            assert b.emitted_count == int(golden.z[f"c{ci}_{s}_pairs"]), (ci, s)
        assert counts["precise"] <= counts["tight-aabb"] <= counts["baseline-circle-aabb"]


def test_every_stage_bit_exact(golden):
    g = golden
    for ci in range(g.ncam):
        cam = g.camera(ci)
        for s in STRATS:
            if not g.has(ci, "keys", s):
                continue
            b = orc.preprocess_and_bin(g.act, cam, s, g.tau, g.sh_degree)
            ret = g.retained(ci, s)
            assert np.array_equal(b.retained, ret)
            assert np.array_equal(b.depth.view(np.uint32), g.get(ci, "depth", s).view(np.uint32))
            assert np.array_equal(b.tile_rects[ret], g.get(ci, "rects", s).astype(np.int32)[ret])
            assert np.array_equal(_sha(b.splat), g.get(ci, "splat_sha", s))
            if g.has(ci, "splat", s):
                assert np.array_equal(b.splat.view(np.uint32), g.get(ci, "splat", s).view(np.uint32))
            keys, vals = orc.sort_pairs(b.keys, b.values, b.grid_w * b.grid_h, max(g.act.count, 1))
            assert np.array_equal(keys, g.get(ci, "keys", s))
            assert np.array_equal(vals, g.get(ci, "values", s))
            starts = orc.tile_range_table(keys, b.grid_w, b.grid_h)
            assert np.array_equal(starts, g.get(ci, "starts", s).astype(np.int64))
            img, contrib, nonempty = orc.render_frame(b.splat, vals, starts, cam.width,
                                                      cam.height, g.bg, g.tau)
            assert np.array_equal(_sha(img), g.get(ci, "image_sha", s))
            if g.has(ci, "image", s):
                assert np.array_equal(img.view(np.uint32), g.get(ci, "image", s).view(np.uint32))
            assert np.array_equal(contrib, g.contrib(ci, s))
            st = g.get(ci, "stats", s)
            assert (b.emitted_count, int(contrib.sum()), b.gaussians_retained,
                    b.gaussians_degenerate, nonempty) == tuple(int(v) for v in st)


def test_c1_survey_fingerprints(golden_c1):
    """10000 retained, 47264 pairs, 34034 contributing, 236 tiles,
    sha256(sorted keys)[:16] = 985b4149ce95e8e8, sha256(image)[:16] = 57807ea6520ab90c."""
    g = golden_c1
    img, st = orc.render(g.act, g.camera(0), "precise", g.tau, g.bg, g.sh_degree)
    assert (st["gaussians_retained"], st["pairs_emitted"], st["pairs_contributing"],
            st["tiles_nonempty"]) == (10000, 47264, 34034, 236)
    assert hashlib.sha256(img.tobytes()).hexdigest()[:16] == "57807ea6520ab90c"
    b = orc.preprocess_and_bin(g.act, g.camera(0))
    assert hashlib.sha256(np.sort(b.keys).tobytes()).hexdigest()[:16] == "985b4149ce95e8e8"
    assert int(b.tile_counts.sum()) == 52466


def test_sort_is_key_then_value_order():
    rng = np.random.default_rng(0)
    keys = (rng.integers(0, 50, 100_000).astype(np.uint64) << np.uint64(32)) \
        | rng.integers(0, 1 << 20, 100_000).astype(np.uint64)
    vals = rng.integers(0, 5000, 100_000).astype(np.uint32)
    k, v = orc.sort_pairs(keys, vals, 50, 5000)
    order = np.lexsort((vals, keys))
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])


def test_range_table_examples():
    keys = np.array([0, 0, 3], np.uint64) << np.uint64(32)
    assert orc.tile_range_table(keys, 2, 2).tolist() == [0, 2, 2, 2, 3]
    with pytest.raises(orc.UnsortedPairsError):
        orc.tile_range_table(keys[::-1].copy(), 2, 2)
    with pytest.raises(ValueError):
        orc.tile_range_table(np.array([9], np.uint64) << np.uint64(32), 2, 2)


def test_eval_counts_against_a_numpy_restatement():
    """The instrumented copy of the compositing loop (orc_render_counts, the source of the
    blend's FP32 roofline) against a plain NumPy/Python restatement of render.py:106-129 on a
    small golden case: class counts, M_proc and pixel count."""
    import math
    g = GoldenCase("edge3000_70x42")
    cam = g.camera(0)
    b = orc.preprocess_and_bin(g.act, cam, "precise", g.tau, g.sh_degree)
    keys, vals = orc.sort_pairs(b.keys, b.values, b.grid_w * b.grid_h, g.act.count)
    starts = orc.tile_range_table(keys, b.grid_w, b.grid_h)
    got = orc.render_counts(b.splat, vals, starts, cam.width, cam.height, g.tau)
    f32 = np.float32
    tau = f32(g.tau)
    want = dict(rect_rejected=0, cutoff_rejected=0, alpha_rejected=0, blended=0,
                pairs_processed=0, pixels=0)
    sp = b.splat
    for t in range(b.grid_w * b.grid_h):
        ty, tx = divmod(t, b.grid_w)
        deepest = 0
        for y in range(ty * 16, min(ty * 16 + 16, cam.height)):
            for x in range(tx * 16, min(tx * 16 + 16, cam.width)):
                fx, fy, T, seen = f32(x) + f32(0.5), f32(y) + f32(0.5), f32(1.0), 0
                for i in range(int(starts[t]), int(starts[t + 1])):
                    r = sp[vals[i]]
                    seen += 1
                    dx, dy = fx - r[0], fy - r[1]
                    if abs(dx) > r[10] or abs(dy) > r[11]:
                        want["rect_rejected"] += 1
                        continue
                    s = f32(0.5) * (r[2] * dx * dx + r[4] * dy * dy) + r[3] * dx * dy
                    if s > f32(0.5) * r[6]:
                        want["cutoff_rejected"] += 1
                        continue
                    al = min(f32(0.99), r[5] * f32(math.exp(-float(s))))
                    if al < tau:
                        want["alpha_rejected"] += 1
                        continue
                    want["blended"] += 1
                    T = T * (f32(1.0) - al)
                    if T < f32(1e-4):
                        break
                deepest = max(deepest, seen)
                want["pixels"] += 1
        want["pairs_processed"] += deepest
    # exp here is float64-rounded, the oracle's is glibc expf: a verdict can only differ when
    # alpha sits within an ulp of tau -- allow a handful of evaluations to change class
    assert got["pixels"] == want["pixels"] == cam.width * cam.height
    assert got["rect_rejected"] == want["rect_rejected"]
    assert got["cutoff_rejected"] == want["cutoff_rejected"]
    assert abs(got["alpha_rejected"] - want["alpha_rejected"]) <= 3
    assert abs(got["blended"] - want["blended"]) <= 3
    assert abs(got["pairs_processed"] - want["pairs_processed"]) <= 3
    assert got["blended"] >= int(np.count_nonzero(g.contrib(0)))
