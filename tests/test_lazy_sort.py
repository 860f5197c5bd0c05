"""lazy_sort (fgs_layout.lazy_sort): heavy tiles get only their nearest pairs sorted, the blend
re-does the tiles that were not saturated by then.  Whatever the guess, the frame, the
contributing-pair count and every other counter must be those of the full sort, i.e. the
reference's (sorting.py:101-136 + render.py:135-252) -- exact mode bit for bit.

Each case builds heavy tiles (> 4096 pairs) on purpose and checks which path they took:
  opaque       tiles saturate inside the front               -> no redo
  translucent  opacities just above tau: nothing saturates   -> every front is redone
  mixed        left half opaque, right half translucent      -> both at once
  near cluster thousands of pairs of ONE depth at the near end: the front gives up (F = 0)
  late cluster the cluster sits just behind 300 nearer pairs: the front is cut before it
"""

import ctypes as C

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from oracle import oracle as orc
from fgs_testlib import identity_camera, make_raw_scene

pytestmark = pytest.mark.gpu


SPREAD = 1.15        # the cloud overfills the 64 x 64 frame: border pixels are covered too


def _scene(kind, n=60000, seed=5):
    rng = np.random.default_rng(seed)
    z = rng.uniform(5.0, 15.0, n)
    xy = rng.uniform(-SPREAD, SPREAD, size=(n, 2)) * z[:, None]
    thick, thin = rng.uniform(0.6, 0.95, n), rng.uniform(0.005, 0.012, n)
    if kind == "opaque":
        op = thick
    elif kind == "translucent":
        op = thin
    elif kind == "mixed":
        op = np.where(xy[:, 0] < 0.0, thick, thin)
    elif kind == "near cluster":
        op = thin
        z[: n // 2] = 5.0                       # thousands of pairs of one depth per tile, all nearest
        xy[: n // 2] = rng.uniform(-SPREAD, SPREAD, size=(n // 2, 2)) * 5.0
        z[n // 2:] = rng.uniform(5.5, 15.0, n - n // 2)
        xy[n // 2:] = rng.uniform(-SPREAD, SPREAD, size=(n - n // 2, 2)) * z[n // 2:, None]
    elif kind == "late cluster":
        op = thin
        k = n // 18                              # ~400 pairs per tile in front of the cluster
        z[:k] = rng.uniform(4.0, 4.9, k)
        xy[:k] = rng.uniform(-SPREAD, SPREAD, size=(k, 2)) * z[:k, None]
        z[k: n // 2] = 5.0
        xy[k: n // 2] = rng.uniform(-SPREAD, SPREAD, size=(n // 2 - k, 2)) * 5.0
    else:
        raise AssertionError(kind)
    return fgs.activate(make_raw_scene(np.concatenate([xy, z[:, None]], axis=1),
                                       rng.uniform(0.2, 0.5, size=(n, 3)), op,
                                       dc=rng.uniform(-1, 1, size=(n, 3))))


@pytest.mark.parametrize("kind", ["opaque", "translucent", "mixed", "near cluster", "late cluster"])
def test_lazy_fronts_give_the_full_sort_frame(kind):
    n = 80000 if kind.endswith("cluster") else 60000
    act = _scene(kind, n)
    cam = identity_camera(64, 64, focal=32)
    ob = orc.preprocess_and_bin(act, cam)
    per_tile = np.bincount((ob.keys >> np.uint64(32)).astype(np.int64), minlength=16)
    assert (per_tile > 4096).sum() >= 8, per_tile          # the case is about heavy tiles
    oimg, ost = orc.render(act, cam)
    lazy, full = fgs.Pipeline(act), fgs.Pipeline(act, lazy_sort=False)
    for exact in (True, False):
        lazy.lazy_sort = True            # (a frame of failed fronts switches it off: keep it on)
        fl, sl = lazy.render(cam, exact=exact)
        ff, sf = full.render(cam, exact=exact)
        # (front_tiles counts the frame's heavy tiles with the option on or off)
        assert sf.redo_tiles == 0
        assert sl.front_tiles == sf.front_tiles == int((per_tile > 4096).sum())
        if kind == "opaque":
            assert sl.redo_tiles == 0
        elif kind == "mixed":
            assert 0 < sl.redo_tiles < sl.front_tiles
        else:
            assert sl.redo_tiles == sl.front_tiles
        # the lazy frame IS the full-sort frame, in both blend modes
        assert np.array_equal(fl.image.view(np.uint32), ff.image.view(np.uint32))
        assert (sl.pairs_contributing, sl.pairs_emitted, sl.tiles_nonempty) == \
            (sf.pairs_contributing, sf.pairs_emitted, sf.tiles_nonempty)
        if exact:                        # ... and the reference's
            assert np.array_equal(fl.image.view(np.uint32), oimg.view(np.uint32))
            assert sl.pairs_contributing == ost["pairs_contributing"]
    fresh = fgs.Pipeline(act)
    assert fresh.lazy_sort == 2
    fresh.render(cam)
    # the next frame's level follows this one: most fronts failed -> the pipeline stops
    # guessing for good; and 16 heavy tiles are too few to pay for the two extra launches
    assert fresh.lazy_sort == 0
    assert fresh._lazy_cap == (2 if kind == "opaque" else 0)  # (mixed: half of the fronts failed)


@pytest.mark.parametrize("kind", ["opaque", "translucent", "mixed"])
def test_lazy_level_2_takes_the_medium_tiles(kind):
    """Level 2: tiles of 2049..4096 pairs get a front too."""
    act = _scene(kind, 30000)
    cam = identity_camera(64, 64, focal=32)
    ob = orc.preprocess_and_bin(act, cam)
    per_tile = np.bincount((ob.keys >> np.uint64(32)).astype(np.int64), minlength=16)
    medium = (per_tile > 2048) & (per_tile <= 4096)
    assert medium.sum() >= 12, per_tile
    oimg, ost = orc.render(act, cam)
    lazy = fgs.Pipeline(act)
    assert lazy.lazy_sort == 2
    fl, sl = lazy.render(cam, exact=True)
    assert sl.front_tiles == int((per_tile > 4096).sum())
    if kind == "opaque":
        assert sl.redo_tiles == 0
    elif kind == "translucent":
        assert sl.redo_tiles == int((per_tile > 2048).sum())
    else:
        assert 0 < sl.redo_tiles < int((per_tile > 2048).sum())
    assert np.array_equal(fl.image.view(np.uint32), oimg.view(np.uint32))
    assert sl.pairs_contributing == ost["pairs_contributing"]
    lazy.lazy_sort = 1                    # level 1 leaves these tiles to the full sort
    f1, s1 = lazy.render(cam, exact=True)
    assert s1.redo_tiles == 0 or (per_tile > 4096).any()
    assert np.array_equal(f1.image.view(np.uint32), oimg.view(np.uint32))


def test_lazy_extras_and_bands():
    """alpha / depth maps and row-band renders through the lazy path (mixed: some tiles redone)."""
    act = _scene("mixed")
    cam = identity_camera(64, 64, focal=32)
    lazy, full = fgs.Pipeline(act), fgs.Pipeline(act, lazy_sort=False)
    fl, sl = lazy.render(cam, exact=True, extras=True)
    ff, _ = full.render(cam, exact=True, extras=True)
    assert 0 < sl.redo_tiles < sl.front_tiles
    for a, b in ((fl.image, ff.image), (fl.alpha, ff.alpha), (fl.depth, ff.depth)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    rows = []
    for band in ((0, 0), (1, 2), (3, 3)):
        lazy.lazy_sort = True
        fb, sb = lazy.render(cam, exact=True, band=band)
        assert sb.front_tiles > 0
        rows.append(fb.image)
    assert np.array_equal(np.concatenate(rows, axis=0).view(np.uint32), ff.image.view(np.uint32))


def test_lazy_stages_can_be_repeated_on_one_frame():
    """fgs_sort and fgs_blend re-issued on a lazy frame: the redo cursor rewinds, the frame and
    the counters repeat."""
    import torch
    from paper_2408_07967_b200 import _capi
    act = _scene("mixed")
    n = act.count
    cam = identity_camera(64, 64, focal=32)
    pipe = fgs.Pipeline(act)
    want, swant = pipe.render(cam)
    assert 0 < swant.redo_tiles < swant.front_tiles
    L = _capi.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    ws = fgs.pipeline._Workspace(torch, dev, n, 64, 64, pipe._default_capacity())
    ws.set_mode(_capi.SORT_MODES["tile-bucket"], lazy_sort=True)
    kcut = pipe._cutoffs(torch, 1 / 255)
    camc = _capi.camera_struct(cam)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    base, lay = C.c_void_p(ws.base), C.byref(ws.lay)
    bg = (C.c_float * 3)(0, 0, 0)
    _capi.check(L.fgs_preprocess(pipe.packed.data_ptr(), kcut.data_ptr(), n, C.byref(camc), 1 / 255,
                                 3, 0, 0, 3, base, lay, st))
    _capi.check(L.fgs_scan(base, lay, st))
    _capi.check(L.fgs_emit(pipe.packed.data_ptr(), C.byref(camc), 0, 0, 3, base, lay, st))
    for _ in range(2):
        _capi.check(L.fgs_sort(base, lay, ws.next_epoch(), st))
    for _ in range(3):
        _capi.check(L.fgs_blend(pipe.packed.data_ptr(), bg, 1 / 255, 2, 0, 3, ws.rgb.data_ptr(),
                                None, None, base, lay, st))
        torch.cuda.synchronize()
        s = np.frombuffer(ws.stats_tensor().cpu().numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
        assert int(s["redo_tiles"]) == swant.redo_tiles
        assert np.array_equal(ws.rgb.cpu().numpy(), want.image)


def test_lazy_with_caller_order_slots():
    """Slots in the caller's order: CTA tile tables overflow and the placement walk (k_place)
    fills the buckets the front kernel then reads -- same frame as the full sort's and the
    oracle's."""
    act = _scene("mixed")
    cam = identity_camera(64, 64, focal=32)
    oimg, ost = orc.render(act, cam)
    lazy = fgs.Pipeline(act, spatial_order=False)
    full = fgs.Pipeline(act, spatial_order=False, lazy_sort=False)
    for level in (2, 1):
        lazy.lazy_sort = level
        fl, sl = lazy.render(cam, exact=True)
        ff, sf = full.render(cam, exact=True)
        assert sl.front_tiles == sf.front_tiles > 0 and sl.redo_tiles > 0
        assert np.array_equal(fl.image.view(np.uint32), ff.image.view(np.uint32))
        assert np.array_equal(fl.image.view(np.uint32), oimg.view(np.uint32))
        assert sl.pairs_contributing == sf.pairs_contributing == ost["pairs_contributing"]
