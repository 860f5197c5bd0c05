"""Geometry and tile-test semantics of K1 on single-Gaussian scenes, observed through the pair
list (``preprocess_and_bin``) -- the cases the reference pins down in pkg/tests/test_intersect.py
(centre inside a tile, far miss, an ellipse that swallows every tile, translation by whole
tiles), test_projection.py (the z-near and opacity culls) and test_extent.py (the three
strategies nest).  Every case is also compared with the oracle's pair list.
"""

import math

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from oracle import oracle as orc
from fgs_testlib import identity_camera, make_raw_scene

pytestmark = pytest.mark.gpu

STRATS = ("precise", "tight-aabb", "baseline-circle-aabb")
W = H = 128
FOCAL = 64.0


def _at_pixel(px, py, z):
    """World position (camera at the origin looking down +z) that projects to pixel centre
    coordinates (px, py) of the W x H frame."""
    return [(px - W / 2) * z / FOCAL, (py - H / 2) * z / FOCAL, z]


def _tiles(scene, cam, strategy):
    out = fgs.preprocess_and_bin(scene, cam, strategy)
    ob = orc.preprocess_and_bin(fgs.activate(scene), cam, strategy)
    got = np.sort(out.keys >> np.uint64(32)).astype(np.int64)
    want = np.sort(ob.keys >> np.uint64(32)).astype(np.int64)
    assert np.array_equal(got, want), strategy                    # the oracle's tile set, exactly
    return set(got.tolist())


def test_centre_tile_is_always_hit_and_strategies_nest():
    cam = identity_camera(W, H, focal=FOCAL)
    rng = np.random.default_rng(3)
    for _ in range(12):
        px, py = rng.uniform(4, W - 4, 2)
        q = rng.normal(size=4)
        scene = make_raw_scene([_at_pixel(px, py, 12.0)], rng.uniform(0.05, 1.5, 3),
                               [rng.uniform(0.1, 0.95)], quats=[q / np.linalg.norm(q)])
        sets = {s: _tiles(scene, cam, s) for s in STRATS}
        centre = int(py // 16) * (W // 16) + int(px // 16)
        for s in STRATS:
            assert centre in sets[s]                                # intersect.py:84-86
        assert sets["precise"] <= sets["tight-aabb"] <= sets["baseline-circle-aabb"]


def test_far_miss_and_an_ellipse_that_covers_the_frame():
    cam = identity_camera(W, H, focal=FOCAL)
    # a small splat in the top-left corner never reaches the bottom-right tiles
    small = make_raw_scene([_at_pixel(8.0, 8.0, 10.0)], [0.05, 0.05, 0.05], [0.9])
    far = {7 * 8 + 7, 7 * 8 + 6, 6 * 8 + 7}
    for s in STRATS:
        assert not (_tiles(small, cam, s) & far)
    # a splat far larger than the frame hits every one of its 64 tiles under every strategy
    huge = make_raw_scene([_at_pixel(64.0, 64.0, 10.0)], [40.0, 40.0, 40.0], [0.9])
    for s in STRATS:
        assert _tiles(huge, cam, s) == set(range(64))


def test_translation_by_whole_tiles_shifts_the_tile_set():
    # intersect.py's predicate is translation-equivariant: moving the centre by 16 px moves the
    # set of hit tiles by one column (well inside the grid, so no clamping interferes)
    cam = identity_camera(W, H, focal=FOCAL)
    q = [math.cos(0.4), 0.0, 0.0, math.sin(0.4)]
    z = 16.0                                     # 16 px <-> 16 * z / FOCAL = 4 world units: exact
    a = make_raw_scene([_at_pixel(41.25, 52.5, z)], [1.6, 0.3, 0.2], [0.8], quats=[q])
    b = make_raw_scene([_at_pixel(41.25 + 16.0, 52.5 + 32.0, z)], [1.6, 0.3, 0.2], [0.8], quats=[q])
    for s in STRATS:
        ta, tb = _tiles(a, cam, s), _tiles(b, cam, s)
        assert len(ta) > 1
        assert tb == {t + 1 + 2 * (W // 16) for t in ta}, s


def test_near_plane_and_opacity_culls():
    # projection.py:39-47: kept iff z > 0.2 and opacity > the frustum threshold; binning.py then
    # drops what stays below tau (nothing can contribute)
    cam = identity_camera(W, H, focal=FOCAL)
    tau = 1.0 / 255.0
    zs = [0.19, 0.21, 5.0, -3.0, 5.0, 5.0]
    ops = [0.9, 0.9, 0.9, 0.9, tau * 0.9, tau * 1.5]
    scene = make_raw_scene([[0.0, 0.0, z] for z in zs], [0.02, 0.02, 0.02], ops)
    act = fgs.activate(scene)
    out = fgs.preprocess_and_bin(scene, cam)
    ob = orc.preprocess_and_bin(act, cam)
    assert np.array_equal(np.asarray(out.retained, bool), np.asarray(ob.retained, bool))
    assert np.asarray(out.retained, bool).tolist() == [False, True, True, False, False, True]
    assert sorted(out.values.tolist()) == sorted(ob.values.tolist())
    assert set(out.values.tolist()) == {1, 2, 5}
