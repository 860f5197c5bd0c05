"""Compositor semantics on hand-made splat tables, through the stand-alone blend entry point
(``fgs_blend_tiles`` = the reference's ``render_frame`` on caller-supplied arrays,
render.py:273-310).  The cases follow what the reference's own tests pin down
(pkg/tests/test_render.py: background of an empty range, a two-splat composite that is exact
in float32, the T < 1e-4 stop after two capped splats, the cutoff skip, energy bound, frames
that are not a multiple of the tile size) -- each checked here against a known answer, against
an independent per-pixel NumPy loop, or against the oracle, in BOTH blend modes (the packed
default kernel and the bit-exact one).
"""

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from oracle import oracle as orc
from fgs_testlib import identity_camera, make_raw_scene

pytestmark = pytest.mark.gpu

TAU = 1.0 / 255.0
F = np.float32


def row(cx, cy, conic=(1.0, 0.0, 1.0), opacity=0.5, k=9.0, rgb=(1.0, 1.0, 1.0), half=(1e6, 1e6)):
    """One splat row in the reference's layout (render.py:34-40)."""
    return np.array([cx, cy, conic[0], conic[1], conic[2], opacity, k, rgb[0], rgb[1], rgb[2],
                     half[0], half[1]], dtype=np.float32)


def blend_tile(rows, values, w=16, h=16, bg=(0.0, 0.0, 0.0), exact=False):
    splat = np.stack(rows) if len(rows) else np.zeros((1, 12), np.float32)
    gw, gh = -(-w // 16), -(-h // 16)
    assert gw * gh == 1
    img, contrib, _ = fgs.render_frame(splat, np.asarray(values, np.uint32), [0, len(values)], w, h,
                                       bg, TAU, exact=exact)
    return img, contrib


def loop_composite(rows, values, w, h, bg):
    """The documented per-pixel rule (render.py:106-129), one pixel at a time in float32 with the
    exponential in float64 rounded once -- good to 1 ulp of the library's expf, so compared with a
    tolerance, and exactly where the case makes alpha exact."""
    img = np.zeros((h, w, 3), np.float32)
    touched = np.zeros(len(values), bool)
    for py in range(h):
        for px in range(w):
            T, c = F(1.0), np.zeros(3, np.float32)
            for i, g in enumerate(values):
                r = rows[g]
                dx, dy = F(px) + F(0.5) - r[0], F(py) + F(0.5) - r[1]
                if abs(dx) > r[10] or abs(dy) > r[11]:
                    continue
                s = F(0.5) * (r[2] * dx * dx + r[4] * dy * dy) + r[3] * dx * dy
                if s > F(0.5) * r[6]:
                    continue
                al = min(F(r[5] * F(np.exp(-np.float64(s)))), F(0.99))
                if al < F(TAU):
                    continue
                touched[i] = True
                c = c + r[7:10] * (al * T)
                T = T * (F(1.0) - al)
                if T < F(1e-4):
                    break
            img[py, px] = c + T * np.asarray(bg, np.float32)
    return img, touched


@pytest.mark.parametrize("exact", [False, True])
def test_empty_range_is_the_background(exact):
    img, contrib = blend_tile([], [], bg=(0.25, 0.5, 0.75), exact=exact)
    assert np.all(img == np.asarray([0.25, 0.5, 0.75], np.float32))
    assert contrib.size == 0


@pytest.mark.parametrize("exact", [False, True])
def test_two_splats_on_a_pixel_centre(exact):
    # both centres on pixel (0, 0): s = 0, alpha = opacity = 0.5 exactly, so
    # C = 0.5 c1 + 0.25 c2 + 0.25 bg with every product exact in float32
    rows = [row(0.5, 0.5, rgb=(1, 0, 0)), row(0.5, 0.5, rgb=(0, 1, 0))]
    img, contrib = blend_tile(rows, [0, 1], bg=(0, 0, 1), exact=exact)
    assert img[0, 0].tolist() == [0.5, 0.25, 0.25]
    assert contrib.tolist() == [1, 1]
    want, _ = loop_composite(rows, [0, 1], 16, 16, (0, 0, 1))
    assert np.allclose(img, want, atol=2e-6)


@pytest.mark.parametrize("exact", [False, True])
def test_stop_after_two_capped_splats(exact):
    # alpha is capped at 0.99 (render.py:217-218): after two such splats T = 0.01^2, just below
    # the 1e-4 stop in float32 (render.py:228), so a third identical splat touches nothing
    r = row(0.5, 0.5, conic=(1000.0, 0.0, 1000.0), opacity=0.999, rgb=(1, 1, 1))
    rows = [r, r, r]
    want, touched = loop_composite(rows, [0, 1, 2], 2, 2, (0, 0, 0))
    assert touched.tolist() == [True, True, False]
    img, contrib = blend_tile(rows, [0, 1, 2], w=2, h=2, exact=exact)
    assert contrib.tolist() == [1, 1, 0]
    assert np.allclose(img, want, atol=2e-6)
    assert img[0, 0, 0] == F(0.99) + F(0.99) * (F(1.0) - F(0.99))   # alpha exact: pixel exact


@pytest.mark.parametrize("exact", [False, True])
def test_cutoff_skip_along_a_row(exact):
    # pixels whose alpha would still be >= tau but whose power is beyond k / 2 are skipped
    # (render.py:214, the rule shared with the extent stage): 0.08 dx^2 > 4  <=>  dx > 7.07
    r = row(0.5, 0.5, conic=(0.08, 0.0, 0.08), opacity=0.9, k=4.0)
    img, contrib = blend_tile([r], [0], w=16, h=1, exact=exact)
    for px in range(16):
        dx = F(px)
        q = F(0.08) * dx * dx
        al = min(F(0.9) * F(np.exp(-0.5 * float(q))), F(0.99))
        lit = q <= F(4.0) and al >= F(TAU)
        assert (img[0, px, 0] > 0) == lit, px
    assert contrib.tolist() == [1]


def _random_tile(rng, n_pairs, n_splats=64):
    """Random rows with their own cutoffs and extents (binning.py:176-194 rule), and a random
    front-to-back list for one tile."""
    s1, s2 = rng.uniform(0.8, 8.0, n_splats), rng.uniform(0.8, 8.0, n_splats)
    th = rng.uniform(0, np.pi, n_splats)
    ct, st = np.cos(th), np.sin(th)
    cov = np.stack([ct * ct * s1 * s1 + st * st * s2 * s2, ct * st * (s1 * s1 - s2 * s2),
                    st * st * s1 * s1 + ct * ct * s2 * s2], axis=1).astype(np.float32)
    det = cov[:, 0] * cov[:, 2] - cov[:, 1] * cov[:, 1]
    conic = np.stack([cov[:, 2] / det, -cov[:, 1] / det, cov[:, 0] / det], axis=1).astype(np.float32)
    op = rng.uniform(0.02, 0.995, n_splats).astype(np.float32)
    k = np.asarray(fgs.power_cutoffs(op, TAU)[0], np.float32)        # extent.py:19-30, on the GPU
    rows = np.zeros((n_splats, 12), np.float32)
    rows[:, 0], rows[:, 1] = rng.uniform(-10, 26, n_splats), rng.uniform(-10, 26, n_splats)
    rows[:, 2:5], rows[:, 5], rows[:, 6] = conic, op, k
    rows[:, 7:10] = rng.uniform(0, 1, (n_splats, 3))
    rows[:, 10], rows[:, 11] = np.sqrt(k * cov[:, 0]), np.sqrt(k * cov[:, 2])
    return rows, rng.integers(0, n_splats, n_pairs).astype(np.uint32)


def test_random_tiles_against_the_oracle_and_bounds():
    """150 random tiles of 0..40 pairs: exact mode bit-identical to the oracle (itself pinned to
    the reference), default mode within the pixel tolerance with identical contrib flags, white
    background never exceeded (energy bound: sum of weights + T = 1)."""
    rng = np.random.default_rng(12)
    for trial in range(150):
        rows, values = _random_tile(rng, int(rng.integers(0, 41)))
        oimg, ocon, _ = orc.render_frame(rows, values, np.array([0, values.size]), 16, 16, (1, 1, 1), TAU)
        ix, cx, _ = fgs.render_frame(rows, values, [0, values.size], 16, 16, (1, 1, 1), TAU, exact=True)
        i2, c2, _ = fgs.render_frame(rows, values, [0, values.size], 16, 16, (1, 1, 1), TAU)
        assert np.array_equal(ix.view(np.uint32), np.asarray(oimg, np.float32).view(np.uint32)), trial
        assert np.array_equal(cx.astype(bool), np.asarray(ocon).astype(bool)), trial
        assert np.array_equal(c2, cx), trial
        assert fgs.max_abs_diff(i2, ix) <= 1e-5, trial
        assert float(ix.max()) <= 1.0 + 1e-5 and float(i2.max()) <= 1.0 + 1e-5


def test_frame_that_is_not_a_multiple_of_the_tile():
    cam = identity_camera(70, 42)
    act = fgs.activate(fgs.gen_synthetic("mixed", 100, 2))
    fb, st = fgs.Pipeline(act).render(cam, exact=True)
    oimg, ost = orc.render(act, cam)
    assert fb.image.shape == (42, 70, 3) and np.all(np.isfinite(fb.image))
    assert np.array_equal(fb.image.view(np.uint32), oimg.view(np.uint32))
    assert st.pairs_contributing == ost["pairs_contributing"]


def test_brightest_pixel_sits_on_the_projected_centre():
    scene = make_raw_scene([[0.5, -0.25, 20.0]], [0.35, 0.35, 0.35], [0.98], dc=[[2.0, 2.0, 2.0]])
    cam = identity_camera(96, 96, focal=48)
    pipe = fgs.Pipeline(scene)
    fb, _ = pipe.render(cam)
    b = fgs.preprocess_and_bin(pipe, cam)
    cx, cy = (float(v) for v in np.asarray(b.splat).reshape(-1, 12)[0, :2])
    by, bx = np.unravel_index(np.argmax(fb.image.sum(axis=2)), (96, 96))
    assert abs(bx + 0.5 - cx) <= 1.0 and abs(by + 0.5 - cy) <= 1.0
