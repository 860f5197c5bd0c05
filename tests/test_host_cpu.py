"""CPU-side checks: the C-ABI library loads and exports what the header declares,
struct layouts agree with the C compiler, host logic (scene generator, cameras,
metrics, argument errors) behaves like the reference.  No GPU compute."""

import ctypes as C
import hashlib
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from paper_2408_07967_b200 import _capi, build as fgs_build
from fgs_testlib import identity_camera

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashgs_b200.h")


@pytest.fixture(scope="module")
def lib():
    fgs_build.build()
    return _capi.lib()


def test_library_exports_every_declared_symbol(lib):
    text = open(HEADER).read()
    declared = set(re.findall(r"\b(fgs_[a-z_0-9]+)\s*\(", text))
    assert declared == set(_capi.SYMBOLS), declared ^ set(_capi.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fgs_abi_version() == _capi.ABI_VERSION
    assert lib.fgs_error_string(-3) == b"unknown strategy"


def test_struct_layouts_match_the_c_compiler():
    src = '#include <stdio.h>\n#include "flashgs_b200.h"\nint main(){printf("%zu %zu %zu %zu %zu\\n",' \
          'sizeof(fgs_camera),sizeof(fgs_stats),sizeof(fgs_layout),' \
          '__builtin_offsetof(fgs_layout,gaussians),__builtin_offsetof(fgs_camera,tan_fovx));return 0;}'
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert got == [C.sizeof(_capi.FgsCamera), C.sizeof(_capi.FgsStats), C.sizeof(_capi.FgsLayout),
                   _capi.FgsLayout.gaussians.offset, _capi.FgsCamera.tan_fovx.offset]


def test_workspace_layout_is_host_only_and_consistent(lib):
    lay = _capi.layout(1_000_000, 1920, 1080, 8_000_000)
    assert (lay.grid_w, lay.grid_h, lay.tiles, lay.tile_bits) == (120, 68, 8160, 13)
    assert lay.sort_passes == 6 and lay.sort_mode == _capi.SORT_TILE_BUCKET
    assert (lay.sorted_keys_in, lay.sorted_vals_in) == (1, 0)
    one = _capi.layout(1_000_000, 1920, 1080, 8_000_000, _capi.SORT_ONESWEEP)
    assert (one.sort_mode, one.sorted_keys_in, one.sorted_vals_in) == (0, 0, 0)
    assert one.total_bytes == lay.total_bytes
    assert lay.preprocess_blocks == 3907
    assert lay.off_tilecount == lay.off_stats + 256        # one memset clears stats + histogram
    offs = [lay.off_stats, lay.off_tilecount, lay.off_cursor, lay.off_splat, lay.off_depth, lay.off_rects, lay.off_flags,
            lay.off_counts, lay.off_blocksums, lay.off_keys[0], lay.off_keys[1],
            lay.off_vals[0], lay.off_vals[1], lay.off_sortstate, lay.off_hist,
            lay.off_starts, lay.off_contrib]
    assert offs == sorted(offs) and all(o % 256 == 0 for o in offs)
    assert lay.total_bytes > lay.off_contrib + 8_000_000 - 256
    # keys[1] | vals[0] | vals[1] are contiguous: the (CTA, tile) table list lives there
    assert lay.off_vals[0] == lay.off_keys[1] + 8 * lay.capacity
    assert lay.off_vals[1] == lay.off_vals[0] + 4 * lay.capacity
    assert _capi.layout(10, 64, 64, 1000).capacity == 1024              # rounded up to 64
    assert _capi.layout(10_000_000, 7680, 4320, 1 << 20).sort_passes == 6   # 31 + 17 bits
    with pytest.raises(_capi.FgsError):
        _capi.layout(10, 64, 64, 1 << 31)                                   # FGS_E_SIZE
    with pytest.raises(_capi.FgsError):
        _capi.layout(-1, 64, 64, 10)
    assert lib.fgs_scene_bytes(1000) == 1024 * 248


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fgs.Pipeline(fgs.gen_synthetic("mixed", 10, 1))
    with pytest.raises(RuntimeError):
        fgs.sort_pairs(np.zeros(4, np.uint64), np.zeros(4, np.uint32))


def test_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2408_07967_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                bad = re.search(r"^\s*(from|import)\s+oracle|libfgs_oracle|oracle/|oracle\.", text, re.M)
                assert bad is None, (os.path.join(dirpath, f), bad.group(0))


def test_scene_generator_is_deterministic():
    a = fgs.gen_synthetic("mixed", 1000, 1)
    b = fgs.gen_synthetic("mixed", 1000, 1)
    assert all(np.array_equal(getattr(a, f), getattr(b, f))
               for f in ("means", "sh", "logit_opacities", "log_scales", "rotations"))
    # same scene the reference generator names (first rows pinned from the golden file)
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_mixed10k_256.npz"))
    act = fgs.activate(fgs.gen_synthetic("mixed", 10_000, 1))
    assert np.array_equal(act.means, g["means"]) and np.array_equal(act.sh, g["sh"])
    assert np.array_equal(act.rotations, g["rotations"])
    # exp-derived fields may differ in the last bit on a CPU with another SIMD exp
    assert np.allclose(act.opacities, g["opacities"], rtol=3e-7, atol=0)
    assert np.allclose(act.scales, g["scales"], rtol=3e-7, atol=0)
    d = fgs.gen_synthetic("mixed", 20_000, 1, density_scale=True)
    u = fgs.gen_synthetic("mixed", 20_000, 1)
    assert np.allclose(d.log_scales - u.log_scales, np.log(0.5 ** (1 / 3)), atol=1e-6)
    with pytest.raises(ValueError):
        fgs.gen_synthetic("nope", 1, 1)
    assert fgs.gen_synthetic("isotropic", 0, 1).count == 0


def test_activate_and_cameras():
    s = fgs.gen_synthetic("elongated", 50, 2)
    s.rotations[3] = 0
    act = fgs.activate(s)
    assert np.array_equal(act.rotations[3], [1, 0, 0, 0])
    assert np.allclose(np.linalg.norm(act.rotations, axis=1), 1, atol=1e-6)
    assert (act.opacities > 0).all() and (act.opacities < 1).all()
    cam = identity_camera(100, 100)
    assert cam.grid == (7, 7)
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_mixed10k_256.npz"))
    oc = fgs.orbit_cameras(1, 24.0, 256, 256)[0]
    assert np.array_equal(oc.world_to_camera, g["c0_view"])
    assert np.array_equal(oc.full_projection, g["c0_proj"])
    assert np.array_equal(oc.position, g["c0_position"])
    assert [oc.tan_fovx, oc.tan_fovy, oc.focal_x, oc.focal_y] == g["c0_intr"].tolist()
    with pytest.raises(fgs.CameraValidationError):
        fgs.make_camera(8, 64, (0, 0, 0), np.eye(3), 32, 32)
    with pytest.raises(fgs.CameraValidationError):
        fgs.make_camera(64, 64, (0, 0, 0), np.eye(3) * 1.1, 32, 32)


def test_psnr_known_answers():
    # reference tests/test_pipeline.py:38-58
    a = np.zeros((4, 4, 3), np.float32)
    assert fgs.psnr(a, a) == "identical"
    assert abs(fgs.psnr(a, a + np.float32(0.1)) - 20.0) < 1e-4
    assert abs(fgs.psnr(a, a + np.float32(1.0))) < 1e-9
    assert abs(fgs.max_abs_diff(a, a + np.float32(0.25)) - 0.25) < 1e-9
    with pytest.raises(ValueError):
        fgs.psnr(a, np.zeros((2, 2, 3), np.float32))


def test_integration_doc_structs_match_the_library():
    """INTEGRATION.md shows the reference-side ctypes binding; its struct mirrors must
    have the real field names and sizes."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "INTEGRATION.md")).read()
    ns = {"C": C}
    exec(src[src.index("class Cam(C.Structure):"):src.index("class Layout(C.Structure):")], ns)
    exec(src[src.index("class Layout(C.Structure):"):src.index("    # fill it with")], ns)
    assert C.sizeof(ns["Cam"]) == C.sizeof(_capi.FgsCamera)
    assert [f[0] for f in ns["Cam"]._fields_] == [f[0] for f in _capi.FgsCamera._fields_]
    assert C.sizeof(ns["Layout"]) == C.sizeof(_capi.FgsLayout)
    assert [f[0] for f in ns["Layout"]._fields_] == [f[0] for f in _capi.FgsLayout._fields_]


# ---------------------------------------------------------------------------
# INTEGRATION.md option A: the reference's own Scene / Camera objects go straight
# through the host boundary.  Needs the reference tree (this container only); it
# is imported from a scratch copy so nothing is written under /root/reference.
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def tilesplat():
    from fgs_testlib import load_tilesplat
    mod = load_tilesplat()
    if mod is None:
        pytest.skip("reference package not present / not importable on this box")
    return mod


def test_reference_objects_pass_the_boundary_unchanged(tilesplat):
    """The reference's Scene, ActivatedScene and Camera are accepted as they are: same
    field names, bit-identical activation, identical flattened camera."""
    from paper_2408_07967_b200 import scene as sc
    ts = tilesplat
    raw_ref = ts.gen_synthetic("mixed", 3000, 5)
    raw_own = fgs.gen_synthetic("mixed", 3000, 5)
    assert sc.is_raw_scene(raw_ref) and not sc.is_activated_scene(raw_ref)
    for f in ("means", "sh", "logit_opacities", "log_scales", "rotations"):
        assert np.array_equal(np.asarray(getattr(raw_ref, f)), np.asarray(getattr(raw_own, f))), f
    act_ref = ts.activate(raw_ref)
    assert sc.is_activated_scene(act_ref) and not sc.is_raw_scene(act_ref)
    act_own = fgs.activate(raw_ref)                 # our activate on THEIR object
    for f in ("means", "opacities", "scales", "rotations", "sh"):
        a, b = np.asarray(getattr(act_ref, f)), np.asarray(getattr(act_own, f))
        assert a.dtype == b.dtype == np.float32 and np.array_equal(a.view(np.uint32), b.view(np.uint32)), f
    cams_ref = ts.orbit_cameras(3, 24.0, 640, 360)
    cams_own = fgs.orbit_cameras(3, 24.0, 640, 360)
    for cr, co in zip(cams_ref, cams_own):
        a, b = _capi.camera_struct(cr), _capi.camera_struct(co)
        assert bytes(a) == bytes(b)
        assert cr.grid == co.grid
    # make_camera validation behaves like the reference's
    with pytest.raises(ts.model_io.CameraValidationError):
        ts.make_camera(8, 64, (0, 0, 0), np.eye(3), 32.0, 32.0)
    with pytest.raises(fgs.CameraValidationError):
        fgs.make_camera(8, 64, (0, 0, 0), np.eye(3), 32.0, 32.0)


def test_oracle_matches_the_reference_on_a_fresh_case(tilesplat):
    """The oracle against the reference run here, on a case that is not a committed fixture
    (pair list, sorted order, range table, frame bits, contrib flags, counters)."""
    from oracle import oracle as orc
    ts = tilesplat
    act = ts.activate(ts.gen_synthetic("elongated", 2500, 21))
    cam = ts.orbit_cameras(2, 15.0, 208, 120)[1]
    for strat in ("precise", "tight-aabb"):
        b = ts.preprocess_and_bin(act, cam, strat, 1 / 255, workers=2)
        keys, vals = ts.sort_pairs(b.keys, b.values, 2, b.grid_w * b.grid_h, act.count)
        ob = orc.preprocess_and_bin(act, cam, strat)
        ok, ov = orc.sort_pairs(ob.keys, ob.values, ob.grid_w * ob.grid_h, act.count)
        assert np.array_equal(keys, ok) and np.array_equal(vals, ov)
        assert np.array_equal(b.splat.view(np.uint32), ob.splat.view(np.uint32))
    fb, st = ts.Pipeline(act).render(cam, "precise", workers=2)
    oimg, ost = orc.render(act, cam)
    assert np.array_equal(fb.image.view(np.uint32), oimg.view(np.uint32))
    assert (st.pairs_emitted, st.pairs_contributing, st.tiles_nonempty) == \
        (ost["pairs_emitted"], ost["pairs_contributing"], ost["tiles_nonempty"])
