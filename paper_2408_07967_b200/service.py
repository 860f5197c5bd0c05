"""Frame-service adapter on the GPU path.

What the reference's ``FrameService.render_pose`` does (``service.py:111-155``) --
validate a pose request, build a camera, call ``Pipeline.render``, encode the frame --
backed by the CUDA pipeline, with the 8-bit quantisation (``images.py:12-15``) done on the
device so only 3 bytes per pixel cross PCIe.  Request fields, defaults, limits, the error
classes and the ``X-Flash-*`` response headers are the reference's contract; the HTTP
server, static files and the viewer stay out of scope.
``render_pose`` is what a request handler calls.
"""

from __future__ import annotations

import math
import threading

import numpy as np

from .pipeline import STRATEGIES, TAU_DEFAULT, Pipeline
from .scene import CameraValidationError, make_camera

FOV_Y_DEFAULT, FOV_Y_RANGE = 60.0, (5.0, 175.0)          # degrees, service.py:134-136


class PoseError(ValueError):
    """Malformed pose request (the reference answers 400, ``service.py:33-34``)."""


class OversizeError(ValueError):
    """Requested frame exceeds ``max_pixels`` (413, ``service.py:37-38``)."""


def yaw_pitch_rotation(yaw: float, pitch: float) -> np.ndarray:
    """World-to-camera rotation for a yaw about world +y followed by a pitch about the
    camera's x axis (``service.py:43-54``): identity looks down +z, positive yaw turns the
    view toward +x, positive pitch tilts it up."""
    sy, cy = math.sin(yaw), math.cos(yaw)
    sp, cp = math.sin(pitch), math.cos(pitch)
    # R_x(pitch) @ R_y(yaw), written out
    return np.array([[cy, 0.0, -sy],
                     [sp * sy, cp, sp * cy],
                     [cp * sy, -sp, cp * cy]], dtype=np.float64)


def quantize(image) -> np.ndarray:
    """Host restatement of ``images.py:12-15`` for frames that are already on the host."""
    c = np.clip(np.asarray(image).astype(np.float64), 0.0, 1.0)
    return np.floor(c * 255.0 + 0.5).astype(np.uint8)


def ppm_bytes(rgb8: np.ndarray) -> bytes:
    """Binary P6, maxval 255 (``images.py:18-24``)."""
    h, w = rgb8.shape[:2]
    return f"P6\n{w} {h}\n255\n".encode("ascii") + np.ascontiguousarray(rgb8).tobytes()


def png_bytes(rgb8: np.ndarray) -> bytes:
    """PNG of an already quantised frame (``images.py:46-55``); needs Pillow."""
    import io

    from PIL import Image
    buf = io.BytesIO()
    Image.fromarray(np.ascontiguousarray(rgb8), mode="RGB").save(buf, format="PNG")
    return buf.getvalue()


def _number_list(req, key, count):
    """``req[key]`` as ``count`` floats, or PoseError."""
    try:
        vals = [float(v) for v in req[key]]
    except KeyError:
        raise PoseError(f"bad pose request: missing {key!r}") from None
    except (TypeError, ValueError) as e:
        raise PoseError(f"bad pose request: {key} is not a list of numbers ({e})") from e
    if len(vals) != count:
        raise PoseError(f"bad pose request: {key} must have {count} numbers")
    return vals


def _integer(req, key):
    try:
        return int(req[key])
    except KeyError:
        raise PoseError(f"bad pose request: missing {key!r}") from None
    except (TypeError, ValueError) as e:
        raise PoseError(f"bad pose request: {key}: {e}") from e


class FrameService:
    """Immutable scene + render configuration (``service.py:57-75``); safe to call
    from several request threads (``Pipeline.render`` takes a workspace per call)."""

    def __init__(self, scene, sh_degree=3, workers=1, default_strategy="precise",
                 tau=TAU_DEFAULT, background=(0.0, 0.0, 0.0), max_pixels=1920 * 1080,
                 max_inflight=4, encoding="png"):
        if encoding not in ("png", "ppm", "raw"):
            raise ValueError("encoding must be 'png', 'ppm' or 'raw'")
        self.pipeline = scene if isinstance(scene, Pipeline) else Pipeline(scene, sh_degree=sh_degree)
        self.workers = max(1, int(workers))
        self.default_strategy = default_strategy
        self.tau = float(tau)
        self.background = tuple(background)
        self.max_pixels = int(max_pixels)
        self.encoding = encoding
        self._inflight = threading.Semaphore(int(max_inflight))

    def camera_for(self, req: dict):
        """``(camera, strategy)`` for a pose request, or PoseError / OversizeError.

        The request carries ``width``, ``height``, ``position[3]`` and either a row-major
        ``rotation[9]`` or ``yaw`` / ``pitch`` in radians; optional ``fov_y`` (degrees,
        5..175, default 60) and ``strategy`` (``service.py:111-143``)."""
        size = (_integer(req, "width"), _integer(req, "height"))
        eye = _number_list(req, "position", 3)
        if size[0] * size[1] > self.max_pixels:
            raise OversizeError(f"{size[0]}x{size[1]} exceeds max pixels {self.max_pixels}")
        if "rotation" in req:
            rot = np.array(_number_list(req, "rotation", 9), dtype=np.float64).reshape(3, 3)
        elif "yaw" in req or "pitch" in req:
            try:
                rot = yaw_pitch_rotation(float(req.get("yaw", 0.0)), float(req.get("pitch", 0.0)))
            except (TypeError, ValueError) as e:
                raise PoseError(f"bad pose request: yaw / pitch: {e}") from e
        else:
            raise PoseError("pose needs either rotation[9] or yaw/pitch")
        strategy = req.get("strategy", self.default_strategy)
        if strategy not in STRATEGIES:
            raise PoseError(f"unknown strategy {strategy!r}")
        try:
            fov_y = float(req.get("fov_y", FOV_Y_DEFAULT))
        except (TypeError, ValueError) as e:
            raise PoseError(f"bad pose request: fov_y: {e}") from e
        if not FOV_Y_RANGE[0] <= fov_y <= FOV_Y_RANGE[1]:
            raise PoseError(f"fov_y {fov_y} out of range")
        # square pixels: one focal length from the vertical field of view
        focal = 0.5 * size[1] / math.tan(0.5 * math.radians(fov_y))
        try:
            camera = make_camera(size[0], size[1], eye, rot, fx=focal, fy=focal)
        except CameraValidationError as e:            # too small a frame, non-orthonormal rotation
            raise PoseError(str(e)) from e
        return camera, strategy

    def render_pose(self, req: dict):
        """(encoded frame, headers) for one pose request (``service.py:111-155``)."""
        camera, strategy = self.camera_for(req)
        with self._inflight:
            fb, stats = self.pipeline.render(camera, strategy, self.tau, self.background,
                                             self.workers, quantized=True)
        counters = (("Pairs-Emitted", stats.pairs_emitted),
                    ("Pairs-Contributing", stats.pairs_contributing),
                    ("Gaussians-Retained", stats.gaussians_retained))
        headers = {"X-Flash-Frame-Ms": f"{stats.total_ns / 1e6:.3f}"}
        headers.update({f"X-Flash-{name}": str(value) for name, value in counters})
        headers["X-Flash-Strategy"] = strategy
        if self.encoding == "raw":
            return fb.image, headers
        return (png_bytes if self.encoding == "png" else ppm_bytes)(fb.image), headers
