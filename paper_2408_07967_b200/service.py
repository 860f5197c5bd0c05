"""Frame-service adapter on the GPU path.

The reference's ``FrameService.render_pose`` (``service.py:111-155``) validates a
pose request, builds a camera, calls ``Pipeline.render`` and encodes the frame.
This module provides the same method backed by the CUDA pipeline, with the
8-bit quantisation (``images.py:12-15``) done on the device so only 3 bytes per
pixel cross PCIe.  The HTTP server, static files and the viewer stay out of
scope: ``render_pose`` is what a handler calls.
"""

from __future__ import annotations

import math
import threading

import numpy as np

from .pipeline import STRATEGIES, TAU_DEFAULT, Pipeline
from .scene import CameraValidationError, make_camera


class PoseError(ValueError):
    """Malformed pose request (the reference answers 400, ``service.py:33-34``)."""


class OversizeError(ValueError):
    """Requested frame exceeds ``max_pixels`` (413, ``service.py:37-38``)."""


def yaw_pitch_rotation(yaw: float, pitch: float) -> np.ndarray:
    """World-to-camera rotation: yaw about world y, then pitch (``service.py:43-54``);
    yaw 0 / pitch 0 looks down +z, positive yaw turns toward +x, positive pitch looks up."""
    cy, sy, cp, sp = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch)
    about_y = np.array([[cy, 0.0, -sy], [0.0, 1.0, 0.0], [sy, 0.0, cy]])
    about_x = np.array([[1.0, 0.0, 0.0], [0.0, cp, sp], [0.0, -sp, cp]])
    return about_x @ about_y


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
        """Validate a pose request and build its camera (``service.py:111-143``)."""
        try:
            width, height = int(req["width"]), int(req["height"])
            position = [float(v) for v in req["position"]]
            if len(position) != 3:
                raise ValueError("position must have 3 numbers")
        except (KeyError, TypeError, ValueError) as e:
            raise PoseError(f"bad pose request: {e}") from e
        if width * height > self.max_pixels:
            raise OversizeError(f"{width}x{height} exceeds max pixels {self.max_pixels}")
        if "rotation" in req:
            rotation = np.asarray(req["rotation"], dtype=np.float64)
            if rotation.size != 9:
                raise PoseError("rotation must have 9 numbers")
            rotation = rotation.reshape(3, 3)
        elif "yaw" in req or "pitch" in req:
            rotation = yaw_pitch_rotation(float(req.get("yaw", 0.0)), float(req.get("pitch", 0.0)))
        else:
            raise PoseError("pose needs either rotation[9] or yaw/pitch")
        strategy = req.get("strategy", self.default_strategy)
        if strategy not in STRATEGIES:
            raise PoseError(f"unknown strategy {strategy!r}")
        fov_y = float(req.get("fov_y", 60.0))
        if not 5.0 <= fov_y <= 175.0:
            raise PoseError(f"fov_y {fov_y} out of range")
        focal = height / (2.0 * math.tan(math.radians(fov_y) / 2.0))
        try:
            return make_camera(width, height, position, rotation, fx=focal, fy=focal), strategy
        except CameraValidationError as e:
            raise PoseError(str(e)) from e

    def render_pose(self, req: dict):
        """(encoded frame, headers) for one pose request (``service.py:111-155``)."""
        camera, strategy = self.camera_for(req)
        with self._inflight:
            fb, stats = self.pipeline.render(camera, strategy, self.tau, self.background,
                                             self.workers, quantized=True)
        headers = {
            "X-Flash-Frame-Ms": f"{stats.total_ns / 1e6:.3f}",
            "X-Flash-Pairs-Emitted": str(stats.pairs_emitted),
            "X-Flash-Pairs-Contributing": str(stats.pairs_contributing),
            "X-Flash-Gaussians-Retained": str(stats.gaussians_retained),
            "X-Flash-Strategy": strategy,
        }
        if self.encoding == "raw":
            return fb.image, headers
        return (png_bytes if self.encoding == "png" else ppm_bytes)(fb.image), headers
