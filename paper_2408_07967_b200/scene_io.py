"""Scene / camera files either side of the path (scene ingest).

Mirrors the reference's file formats and error behaviour so a caller can swap
the import:

* ``load_ply`` / ``save_ply``          -> reference ``model_io.py:136-222``
  (binary little-endian PLY, 62 float32 properties per vertex, 248-byte stride;
  ``PlyParseError`` / ``PlySchemaError`` / ``PlyLengthError`` as ``model_io.py:22-31``)
* ``load_cameras`` / ``save_cameras``  -> reference ``model_io.py:311-343``
* ``load_ply_device``                  -> the B200 ingest: the header is parsed on the
  host (a few hundred bytes), the vertex body goes to the device in one pinned
  copy (248 B/Gaussian) and is split into the reference's arrays there
  (``fgs_scene_unpack_ply``); ``Pipeline(device_scene)`` then activates
  (``fgs_scene_activate``) and packs it without the scene ever being re-laid out
  on the host.  Values are moved bit for bit, so a device-ingested scene equals
  ``load_ply``'s arrays exactly.

No CPU fallback: ``load_ply_device`` needs the CUDA library and a device.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .scene import SH_BASIS, Scene, make_camera


class PlyParseError(ValueError):
    """Header is not the expected binary PLY structure (reference ``model_io.py:22``)."""


class PlySchemaError(ValueError):
    """Vertex properties do not match the schema (reference ``model_io.py:26``)."""


class PlyLengthError(ValueError):
    """Body shorter than the header promises (reference ``model_io.py:30``)."""


class CameraSchemaError(ValueError):
    """Camera JSON entry lacks a required field (reference ``model_io.py:34``)."""


# canonical property order (reference model_io.py:42-51); byte offsets depend on it
PLY_PROPERTIES = (["x", "y", "z", "nx", "ny", "nz"] + [f"f_dc_{i}" for i in range(3)]
                  + [f"f_rest_{i}" for i in range(45)] + ["opacity"]
                  + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)])
VERTEX_FLOATS = len(PLY_PROPERTIES)          # 62
VERTEX_STRIDE = 4 * VERTEX_FLOATS            # 248 bytes
_FORMAT_LINE = "format binary_little_endian 1.0"
_CAMERA_FIELDS = ("id", "width", "height", "position", "rotation", "fx", "fy")


def _parse_header(f) -> int:
    """Consumes the header of an open binary file, validates it the way
    ``model_io.py:136-186`` does (same exception types, same messages where the
    reference's tests match on them) and returns the vertex count."""
    lines = []
    while True:
        raw = f.readline()
        if not raw:
            raise PlyParseError("unexpected end of file inside header")
        try:
            lines.append(raw.decode("ascii").strip())
        except UnicodeDecodeError:
            raise PlyParseError(f"non-ascii header line: {raw[:40]!r}") from None
        if lines[-1] == "end_header":
            break
    if lines[0] != "ply":
        raise PlyParseError(f"not a PLY file, first line: {lines[0]!r}")
    formats = [ln for ln in lines if ln.startswith("format")]
    if not formats or formats[0] != _FORMAT_LINE:
        shown = formats[0] if formats else "<missing format line>"
        raise PlyParseError(f"unsupported format line: {shown!r}")
    count, props = None, []
    for ln in lines:
        words = ln.split()
        if ln.startswith("element "):
            if len(words) != 3 or words[1] != "vertex":
                raise PlyParseError(f"unsupported element line: {ln!r}")
            try:
                count = int(words[2])
            except ValueError:
                raise PlyParseError(f"bad vertex count line: {ln!r}") from None
        elif ln.startswith("property "):
            if len(words) != 3 or words[1] != "float":
                raise PlySchemaError(f"unsupported property line: {ln!r}")
            props.append(words[2])
    if count is None:
        raise PlyParseError("header has no 'element vertex' line")
    missing = [p for p in PLY_PROPERTIES if p not in props]
    if missing:
        raise PlySchemaError(f"missing vertex properties: {missing}")
    if props != PLY_PROPERTIES:
        extra = [p for p in props if p not in PLY_PROPERTIES]
        raise PlySchemaError("vertex properties deviate from the canonical layout "
                             f"(extra or reordered: {extra or props[:8]})")
    return count


def _check_body(nbytes: int, count: int) -> int:
    expected = count * VERTEX_STRIDE
    if nbytes < expected:
        raise PlyLengthError(f"vertex body truncated: expected {expected} bytes, got {nbytes}")
    return expected


def load_ply(path) -> Scene:
    """Host loader (``model_io.py:136-199``): raw values preserved exactly,
    activation is a separate step."""
    with open(path, "rb") as f:
        count = _parse_header(f)
        body = f.read()
    expected = _check_body(len(body), count)
    rec = np.frombuffer(body, dtype="<f4", count=expected // 4).reshape(count, VERTEX_FLOATS)
    sh = np.empty((count, SH_BASIS, 3), dtype=np.float32)
    sh[:, 0, :] = rec[:, 6:9]
    # the higher-order block is channel-major on disk: 15 red, 15 green, 15 blue
    sh[:, 1:, :] = rec[:, 9:54].reshape(count, 3, SH_BASIS - 1).transpose(0, 2, 1)
    col = lambda a, b: np.ascontiguousarray(rec[:, a:b])
    return Scene(means=col(0, 3), normals=col(3, 6), sh=sh,
                 logit_opacities=np.ascontiguousarray(rec[:, 54]),
                 log_scales=col(55, 58), rotations=col(58, 62))


def save_ply(scene, path) -> None:
    """Canonical binary PLY (``model_io.py:212-222``), round-trip exact."""
    n = int(np.asarray(scene.means).shape[0])
    rec = np.empty((n, VERTEX_FLOATS), dtype="<f4")
    sh = np.asarray(scene.sh, dtype=np.float32).reshape(n, SH_BASIS, 3)
    rec[:, 0:3] = scene.means
    rec[:, 3:6] = scene.normals
    rec[:, 6:9] = sh[:, 0, :]
    rec[:, 9:54] = sh[:, 1:, :].transpose(0, 2, 1).reshape(n, 45)
    rec[:, 54] = scene.logit_opacities
    rec[:, 55:58] = scene.log_scales
    rec[:, 58:62] = scene.rotations
    head = ["ply", _FORMAT_LINE, f"element vertex {n}"]
    head += [f"property float {p}" for p in PLY_PROPERTIES] + ["end_header"]
    with open(path, "wb") as f:
        f.write(("\n".join(head) + "\n").encode("ascii"))
        f.write(rec.tobytes())


@dataclass
class DeviceScene:
    """A raw scene whose arrays already live in device memory (torch tensors,
    float32, contiguous): what ``load_ply_device`` returns and ``Pipeline``
    accepts.  Field names follow ``Scene``; normals are dropped at ingest."""

    means: object            # (N, 3)
    sh: object               # (N, 48) = (N, 16, 3) flattened
    logit_opacities: object  # (N,)
    log_scales: object       # (N, 3)
    rotations: object        # (N, 4)

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    def to_host(self) -> Scene:
        n = self.count
        h = lambda t, shape: t.cpu().numpy().reshape(shape)
        return Scene(means=h(self.means, (n, 3)), normals=np.zeros((n, 3), np.float32),
                     sh=h(self.sh, (n, SH_BASIS, 3)), logit_opacities=h(self.logit_opacities, (n,)),
                     log_scales=h(self.log_scales, (n, 3)), rotations=h(self.rotations, (n, 4)))


def load_ply_device(path, device=None) -> DeviceScene:
    """Header on the host, body straight to the device (one pinned H2D copy of
    248 B/Gaussian), split into the reference's arrays by ``fgs_scene_unpack_ply``."""
    import torch
    from . import _capi
    if not torch.cuda.is_available():
        raise RuntimeError("load_ply_device needs a CUDA device (there is no CPU fallback); "
                           "use load_ply for a host Scene")
    L = _capi.lib()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with open(path, "rb") as f:
        count = _parse_header(f)
        start = f.tell()
        f.seek(0, 2)
        expected = _check_body(f.tell() - start, count)
        f.seek(start)
        pinned = torch.empty(max(expected, 4), dtype=torch.uint8, pin_memory=True)
        got = f.readinto(memoryview(pinned.numpy())[:expected]) if expected else 0
        if got != expected:
            raise PlyLengthError(f"vertex body truncated: expected {expected} bytes, got {got}")
    with torch.cuda.device(dev):
        payload = pinned.to(dev, non_blocking=True)
        f32 = lambda *shape: torch.empty(shape, dtype=torch.float32, device=dev)
        n = max(count, 1)
        out = DeviceScene(f32(n, 3)[:count], f32(n, 48)[:count], f32(n)[:count], f32(n, 3)[:count],
                          f32(n, 4)[:count])
        st = torch.cuda.current_stream(dev).cuda_stream
        _capi.check(L.fgs_scene_unpack_ply(payload.data_ptr(), count, out.means.data_ptr(),
                                           out.sh.data_ptr(), out.logit_opacities.data_ptr(),
                                           out.log_scales.data_ptr(), out.rotations.data_ptr(), st))
        torch.cuda.current_stream(dev).synchronize()      # `payload` and `pinned` die here
    return out


def load_cameras(path, near=0.01, far=100.0) -> list:
    """JSON camera list (``model_io.py:311-328``): entries with id, width, height,
    position (3), rotation (9, row-major world-to-camera), fx, fy."""
    with open(path, "r", encoding="utf-8") as f:
        entries = json.load(f)
    if not isinstance(entries, list):
        raise CameraSchemaError("camera file must contain a JSON array")
    cams = []
    for i, e in enumerate(entries):
        missing = [k for k in _CAMERA_FIELDS if k not in e]
        if missing:
            raise CameraSchemaError(f"camera entry {i} missing fields: {missing}")
        cams.append(make_camera(e["width"], e["height"], e["position"], e["rotation"], e["fx"],
                                e["fy"], near=near, far=far, cam_id=str(e["id"])))
    return cams


def save_cameras(cameras, path) -> None:
    """``model_io.py:331-343``."""
    out = [{"id": c.cam_id, "width": c.width, "height": c.height,
            "position": [float(v) for v in c.position],
            "rotation": [float(v) for v in np.asarray(c.world_to_camera)[:3, :3].reshape(9)],
            "fx": c.focal_x, "fy": c.focal_y} for c in cameras]
    with open(path, "w", encoding="utf-8") as f:
        json.dump(out, f, indent=2)
