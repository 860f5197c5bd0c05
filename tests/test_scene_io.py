"""Scene / camera files either side of the path (paper_2408_07967_b200/scene_io.py), read
like the reference's own tests (tests/test_model_io.py:17-75, 100-140): round trips,
schema errors, and -- on the GPU -- that the device ingest moves every value bit for bit."""

import json

import numpy as np
import pytest

import paper_2408_07967_b200 as fgs
from paper_2408_07967_b200.scene_io import PLY_PROPERTIES, VERTEX_STRIDE


def _header(count, props=PLY_PROPERTIES, fmt="format binary_little_endian 1.0"):
    lines = ["ply", fmt, f"element vertex {count}"] + [f"property float {p}" for p in props]
    return ("\n".join(lines + ["end_header"]) + "\n").encode()


def test_vertex_stride_is_248():
    assert len(PLY_PROPERTIES) == 62 and VERTEX_STRIDE == 248


def test_zero_vertex_record(tmp_path):
    path = tmp_path / "one.ply"
    path.write_bytes(_header(1) + b"\x00" * VERTEX_STRIDE)
    scene = fgs.load_ply(path)
    assert scene.count == 1
    assert np.all(scene.means[0] == 0) and scene.logit_opacities[0] == 0
    assert scene.sh.shape == (1, 16, 3)


def test_ply_round_trip_bytes(tmp_path):
    scene = fgs.gen_synthetic("mixed", 64, 9)
    p1, p2 = tmp_path / "a.ply", tmp_path / "b.ply"
    fgs.save_ply(scene, p1)
    back = fgs.load_ply(p1)
    for name in ("means", "normals", "sh", "logit_opacities", "log_scales", "rotations"):
        assert np.array_equal(getattr(back, name), getattr(scene, name)), name
    fgs.save_ply(back, p2)
    assert p1.read_bytes() == p2.read_bytes()


def test_ply_sh_layout_is_channel_major_on_disk(tmp_path):
    """f_rest_k holds coefficient 1 + k % 15 of channel k // 15 (model_io.py:189-192)."""
    rec = np.arange(62, dtype="<f4")[None, :]
    path = tmp_path / "idx.ply"
    path.write_bytes(_header(1) + rec.tobytes())
    s = fgs.load_ply(path)
    assert s.sh[0, 0].tolist() == [6.0, 7.0, 8.0]
    for coef in range(1, 16):
        assert s.sh[0, coef].tolist() == [9.0 + coef - 1, 24.0 + coef - 1, 39.0 + coef - 1]
    assert s.logit_opacities[0] == 54.0 and s.log_scales[0].tolist() == [55.0, 56.0, 57.0]
    assert s.rotations[0].tolist() == [58.0, 59.0, 60.0, 61.0]


def test_ply_missing_property(tmp_path):
    path = tmp_path / "bad.ply"
    path.write_bytes(_header(0, [p for p in PLY_PROPERTIES if p != "opacity"]))
    with pytest.raises(fgs.PlySchemaError, match="opacity"):
        fgs.load_ply(path)


def test_ply_reordered_or_typed_properties(tmp_path):
    path = tmp_path / "bad.ply"
    path.write_bytes(_header(0, PLY_PROPERTIES[::-1]))
    with pytest.raises(fgs.PlySchemaError, match="canonical layout"):
        fgs.load_ply(path)
    path.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 0\n"
                     b"property double x\nend_header\n")
    with pytest.raises(fgs.PlySchemaError, match="unsupported property line"):
        fgs.load_ply(path)


def test_ply_malformed_header(tmp_path):
    path = tmp_path / "bad.ply"
    path.write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(fgs.PlyParseError, match="format ascii 1.0"):
        fgs.load_ply(path)
    path.write_bytes(b"plx\nend_header\n")
    with pytest.raises(fgs.PlyParseError, match="not a PLY file"):
        fgs.load_ply(path)
    path.write_bytes(b"ply\nformat binary_little_endian 1.0\n")
    with pytest.raises(fgs.PlyParseError, match="unexpected end of file"):
        fgs.load_ply(path)
    path.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement face 3\nend_header\n")
    with pytest.raises(fgs.PlyParseError, match="unsupported element line"):
        fgs.load_ply(path)
    path.write_bytes(b"ply\nformat binary_little_endian 1.0\nend_header\n")
    with pytest.raises(fgs.PlyParseError, match="no 'element vertex' line"):
        fgs.load_ply(path)


def test_ply_truncated_body(tmp_path):
    scene = fgs.gen_synthetic("isotropic", 4, 1)
    path = tmp_path / "t.ply"
    fgs.save_ply(scene, path)
    path.write_bytes(path.read_bytes()[:-100])
    with pytest.raises(fgs.PlyLengthError, match=r"expected 992 bytes, got 892"):
        fgs.load_ply(path)


def test_camera_json_round_trip_and_schema(tmp_path):
    cams = fgs.orbit_cameras(3, 10.0, 64, 48)
    path = tmp_path / "cams.json"
    fgs.save_cameras(cams, path)
    back = fgs.load_cameras(path)
    assert [c.cam_id for c in back] == [c.cam_id for c in cams]
    for a, b in zip(cams, back):
        assert (a.width, a.height, a.focal_x, a.focal_y) == (b.width, b.height, b.focal_x, b.focal_y)
        assert np.array_equal(a.position, b.position)
        assert np.allclose(a.full_projection, b.full_projection, atol=1e-6)
    entries = json.loads(path.read_text())
    del entries[1]["fx"]
    path.write_text(json.dumps(entries))
    with pytest.raises(fgs.CameraSchemaError, match=r"entry 1 missing fields: \['fx'\]"):
        fgs.load_cameras(path)
    path.write_text(json.dumps({"id": 0}))
    with pytest.raises(fgs.CameraSchemaError, match="JSON array"):
        fgs.load_cameras(path)


def test_device_ingest_fails_loudly_without_a_gpu(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA device present")
    path = tmp_path / "s.ply"
    fgs.save_ply(fgs.gen_synthetic("mixed", 8, 1), path)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fgs.load_ply_device(path)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 127, 128, 129, 50_000])
def test_device_ingest_is_bit_identical_to_the_host_loader(tmp_path, n):
    scene = fgs.gen_synthetic("mixed", n, 5) if n else fgs.gen_synthetic("mixed", 4, 5)
    path = tmp_path / "s.ply"
    if n == 0:
        path.write_bytes(_header(0))
    else:
        fgs.save_ply(scene, path)
    host = fgs.load_ply(path)
    dev = fgs.load_ply_device(path).to_host()
    assert dev.count == host.count == n
    for name in ("means", "sh", "logit_opacities", "log_scales", "rotations"):
        assert np.array_equal(getattr(dev, name).view(np.uint32), getattr(host, name).view(np.uint32)), name


@pytest.mark.gpu
def test_pipeline_from_ply_matches_device_activation_of_the_host_scene(tmp_path):
    """Pipeline.from_ply (header on the host, body split + activated + packed on the device)
    renders the frame Pipeline(load_ply(...), device_activate=True) renders, bit for bit.
    Against the HOST-activated scene the frame is not bit-comparable: the device's exp is
    correctly rounded, NumPy's float32 SIMD exp is not, and a 1-ulp opacity difference can
    flip one of the reference's hard skips (alpha < tau) for a pixel -- one contribution
    of at most ~tau * colour.  So: PSNR >= 60 dB, no pixel off by more than one such
    contribution, and almost all pixels within 1e-3."""
    scene = fgs.gen_synthetic("mixed", 20_000, 11)
    path = tmp_path / "s.ply"
    fgs.save_ply(scene, path)
    cam = fgs.orbit_cameras(1, 20.0, 480, 272)[0]
    a = fgs.Pipeline.from_ply(path)
    b = fgs.Pipeline(fgs.load_ply(path), device_activate=True)
    fa, sa = a.render(cam)
    fb, sb = b.render(cam)
    assert np.array_equal(fa.image, fb.image) and sa.pairs_emitted == sb.pairs_emitted
    for name in ("means", "opacities", "scales", "rotations", "sh"):
        assert np.array_equal(getattr(a.activated, name), getattr(b.activated, name)), name
    fh, _ = fgs.Pipeline(fgs.load_ply(path)).render(cam)
    d = np.abs(fa.image - fh.image)
    p = fgs.psnr(fa.image, fh.image)
    assert (p == "identical" or p >= 60.0) and d.max() <= 5e-3
    assert (d > 1e-3).any(axis=2).mean() <= 1e-4
    with pytest.raises(fgs.PlyLengthError):
        path.write_bytes(path.read_bytes()[:-8])
        fgs.load_ply_device(path)


# ---------------------------------------------------------------------------
# frame export (reference images.py:12-55, tests/test_images.py)
# ---------------------------------------------------------------------------
def test_quantize_rounds_half_away_from_zero_and_clips():
    img = np.array([[[0.0, 0.5 / 255.0, 1.0], [-0.2, 1.7, 254.5 / 255.0],
                     [0.499 / 255.0, 127.5 / 255.0, 0.25]]], dtype=np.float32)
    q = fgs.images.quantize(img)
    want = np.floor(np.clip(img.astype(np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    assert q.dtype == np.uint8 and np.array_equal(q, want)
    assert q[0, 0].tolist() == [0, 1, 255] and q[0, 1].tolist()[:2] == [0, 255]


def test_ppm_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    img = rng.random((37, 53, 3), dtype=np.float32)
    path = tmp_path / "f.ppm"
    fgs.write_ppm(img, path)
    raw = path.read_bytes()
    assert raw.startswith(b"P6\n53 37\n255\n") and len(raw) == len(b"P6\n53 37\n255\n") + 37 * 53 * 3
    back = fgs.read_ppm(path)
    assert np.array_equal(back, fgs.images.quantize(img))
    path.write_bytes(b"P5\n1 1\n255\n\x00")
    with pytest.raises(ValueError, match="not a P6"):
        fgs.read_ppm(path)
    path.write_bytes(b"P6\n1 1\n65535\n\x00\x00\x00")
    with pytest.raises(ValueError, match="maxval"):
        fgs.read_ppm(path)


def test_png_round_trip(tmp_path):
    Image = pytest.importorskip("PIL.Image")
    img = np.random.default_rng(4).random((20, 31, 3), dtype=np.float32)
    path = tmp_path / "f.png"
    fgs.write_png(img, path)
    assert np.array_equal(np.asarray(Image.open(path).convert("RGB")), fgs.images.quantize(img))


@pytest.mark.gpu
def test_device_frames_export_the_same_bytes(tmp_path):
    """A frame left on the device is quantised there; the PPM equals the one written
    from the host copy of the same frame."""
    act = fgs.activate(fgs.gen_synthetic("mixed", 5000, 2))
    cam = fgs.orbit_cameras(1, 16.0, 333, 210)[0]
    pipe = fgs.Pipeline(act)
    fb_dev, _ = pipe.render(cam, as_numpy=False)
    fb_host, _ = pipe.render(cam)
    assert fb_dev.image.is_cuda
    p1, p2 = tmp_path / "d.ppm", tmp_path / "h.ppm"
    fgs.write_ppm(fb_dev.image, p1)
    fgs.write_ppm(fb_host.image, p2)
    assert p1.read_bytes() == p2.read_bytes()
    assert np.array_equal(fgs.read_ppm(p1), fgs.images.quantize(fb_host.image))
