"""Scene, camera and synthetic-scene inputs of the rasterizer hot path.

These are the *inputs* of the path, mirroring the
reference's types so a caller can hand either package the same objects:

* ``Scene`` / ``ActivatedScene`` / ``activate``  -> reference ``model_io.py:57-118``
* ``Camera`` / ``make_camera`` / ``look_at_camera`` / ``orbit_cameras``
                                              -> reference ``model_io.py:226-381``
* ``gen_synthetic``                            -> reference ``model_io.py:391-435``

Everything here is host-side NumPy and runs once per scene / per camera; the
per-frame work lives in the CUDA library.  ``Pipeline`` also accepts the
reference's own dataclasses (duck-typed on field names), so this module is
only needed when the reference package is not importable (e.g. on the GPU
box, where ``/root/reference`` does not exist).

PLY / JSON file I/O lives in ``scene_io.py``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TILE = 16
SH_BASIS = 16
PRESETS = ("elongated", "isotropic", "mixed")


class CameraValidationError(ValueError):
    """Camera values are inconsistent (reference ``model_io.py:39-40``)."""


# --------------------------------------------------------------------------
# scene containers
# --------------------------------------------------------------------------

@dataclass
class Scene:
    """Raw splat parameters as stored by trained checkpoints (pre-activation)."""

    means: np.ndarray            # (N, 3) f32
    normals: np.ndarray          # (N, 3) f32 (carried, unused)
    sh: np.ndarray               # (N, 16, 3) f32, coefficient-major, RGB innermost
    logit_opacities: np.ndarray  # (N,) f32
    log_scales: np.ndarray       # (N, 3) f32
    rotations: np.ndarray        # (N, 4) f32 (w, x, y, z), not normalised

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


@dataclass
class ActivatedScene:
    """Splat parameters after sigmoid / exp / quaternion normalisation."""

    means: np.ndarray      # (N, 3) f32
    opacities: np.ndarray  # (N,) f32
    scales: np.ndarray     # (N, 3) f32
    rotations: np.ndarray  # (N, 4) f32 unit (w, x, y, z)
    sh: np.ndarray         # (N, 16, 3) f32

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


def is_raw_scene(obj) -> bool:
    return all(hasattr(obj, f) for f in
               ("means", "sh", "logit_opacities", "log_scales", "rotations"))


def is_activated_scene(obj) -> bool:
    return all(hasattr(obj, f) for f in
               ("means", "sh", "opacities", "scales", "rotations"))


def activate(scene) -> ActivatedScene:
    """Raw -> activated parameters, same float32 NumPy arithmetic as the
    reference (``model_io.py:93-118``) so the arrays are bit-identical on the
    same host: sign-split sigmoid, ``exp`` of log-scales, quaternion
    normalisation with zero-norm rows mapped to identity."""
    f32 = np.float32
    x = np.asarray(scene.logit_opacities, dtype=f32)
    nonneg = x >= 0
    t = np.exp(np.where(nonneg, -x, x))          # never overflows
    denom = f32(1.0) + t
    opac = np.where(nonneg, f32(1.0) / denom, t / denom)

    q = np.asarray(scene.rotations, dtype=f32)
    qn = np.sqrt(np.sum(q * q, axis=1))
    good = qn > 0
    unit = np.empty_like(q)
    unit[good] = q[good] / qn[good, None]
    unit[~good] = np.array([1, 0, 0, 0], dtype=f32)

    return ActivatedScene(
        means=np.asarray(scene.means, dtype=f32),
        opacities=opac.astype(f32),
        scales=np.exp(np.asarray(scene.log_scales, dtype=f32)).astype(f32),
        rotations=unit,
        sh=np.asarray(scene.sh, dtype=f32),
    )


# --------------------------------------------------------------------------
# cameras
# --------------------------------------------------------------------------

@dataclass
class Camera:
    """Pose + intrinsics + pixel grid (field names follow the reference)."""

    width: int
    height: int
    position: np.ndarray         # (3,) f32
    world_to_camera: np.ndarray  # (4, 4) f32
    full_projection: np.ndarray  # (4, 4) f32 = projection @ view
    tan_fovx: float
    tan_fovy: float
    focal_x: float
    focal_y: float
    cam_id: str = "0"
    near: float = 0.01
    far: float = 100.0

    @property
    def grid(self) -> tuple:
        return (-(-self.width // TILE), -(-self.height // TILE))


def make_camera(width, height, position, rotation, fx, fy, near=0.01,
                far=100.0, cam_id="0", rotation_tol=1e-3) -> Camera:
    """Build a camera from a world-to-camera rotation and pixel focal lengths.

    Matrices are assembled in float64 and rounded once to float32, as the
    reference does (``model_io.py:268-305``); same validation errors.
    """
    width, height = int(width), int(height)
    if width < TILE or height < TILE:
        raise CameraValidationError(f"camera size {width}x{height} below 16x16")
    c = np.asarray(position, dtype=np.float64).reshape(3)
    r = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
    dev = np.abs(r @ r.T - np.eye(3)).max()
    if dev > rotation_tol:
        raise CameraValidationError(
            f"rotation not orthonormal: max |R R^T - I| = {dev:.2e}")
    v = np.eye(4)
    v[:3, :3] = r
    v[:3, 3] = -r @ c
    tx = width / (2.0 * fx)
    ty = height / (2.0 * fy)
    pm = np.zeros((4, 4))
    pm[0, 0] = 1.0 / tx
    pm[1, 1] = 1.0 / ty
    pm[2, 2] = far / (far - near)
    pm[2, 3] = -(far * near) / (far - near)
    pm[3, 2] = 1.0
    return Camera(width, height, c.astype(np.float32), v.astype(np.float32),
                  (pm @ v).astype(np.float32), float(tx), float(ty),
                  float(fx), float(fy), str(cam_id), float(near), float(far))


def look_at_camera(position, target, width, height, fov_y_deg=60.0,
                   near=0.01, far=100.0, cam_id="0") -> Camera:
    """Camera at ``position`` facing ``target``, image +y along world +y
    (reference ``model_io.py:343-366``)."""
    eye = np.asarray(position, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    n = np.linalg.norm(f)
    if n == 0:
        raise CameraValidationError("look_at target equals camera position")
    f /= n
    up = np.array([0.0, 1.0, 0.0])
    if abs(np.dot(up, f)) > 0.999:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(up, f)
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    fy = height / (2.0 * math.tan(math.radians(fov_y_deg) / 2.0))
    return make_camera(width, height, eye, np.stack([right, down, f]), fy, fy,
                       near=near, far=far, cam_id=cam_id)


def orbit_cameras(n, radius, width, height, fov_y_deg=60.0, target=(0, 0, 0),
                  elevation=0.35, near=0.01, far=100.0) -> list:
    """``n`` inward-looking cameras on a circle (reference ``model_io.py:369-381``)."""
    tgt = np.asarray(target, dtype=np.float64)
    out = []
    for i in range(n):
        a = 2.0 * math.pi * i / max(n, 1)
        eye = tgt + radius * np.array([math.cos(a), math.sin(elevation), math.sin(a)])
        out.append(look_at_camera(eye, tgt, width, height, fov_y_deg,
                                  near=near, far=far, cam_id=str(i)))
    return out


# --------------------------------------------------------------------------
# synthetic scenes (the benchmark workload)
# --------------------------------------------------------------------------

_STREAM = {"elongated": 1, "isotropic": 2, "mixed": 3}


def gen_synthetic(preset: str, count: int, seed: int, density_scale=False) -> Scene:
    """Deterministic synthetic scene; draws follow the reference generator's
    RNG order (``model_io.py:391-435``) so ``(preset, count, seed)`` names the
    same scene in both packages.

    ``density_scale=True`` applies SURVEY.md §8(d)'s rule for N > 1e4: add
    ``ln((1e4/N)^(1/3))`` to the log-scales so pairs per Gaussian stay at the
    10K-scene level instead of saturating the volume.
    """
    if preset not in PRESETS:
        raise ValueError(f"unknown preset {preset!r}, expected one of {PRESETS}")
    if count < 0:
        raise ValueError("count must be non-negative")
    n = int(count)
    rng = np.random.default_rng([int(seed), _STREAM[preset]])

    xyz = rng.uniform(-8.0, 8.0, size=(n, 3))

    low = int(round(0.68 * n))
    alpha = np.empty(n)
    alpha[:low] = rng.uniform(0.02, 0.35, size=low)
    alpha[low:] = rng.uniform(0.35, 0.98, size=n - low)
    rng.shuffle(alpha)

    major = np.exp(rng.normal(math.log(0.45), 0.35, size=n))
    if preset == "elongated":
        ratio = rng.uniform(10.0, 14.0, size=(n, 2))
    elif preset == "isotropic":
        ratio = np.ones((n, 2))
    else:
        round_ones = rng.random(n) < 0.5
        ratio = rng.uniform(2.0, 12.0, size=(n, 2))
        ratio[round_ones] = 1.0
    axes = np.stack([major, major / ratio[:, 0], major / ratio[:, 1]], axis=1)
    order = rng.random((n, 3)).argsort(axis=1)
    axes = np.take_along_axis(axes, order, axis=1)

    quat = rng.normal(size=(n, 4))

    coef = np.zeros((n, SH_BASIS, 3))
    coef[:, 0, :] = rng.normal(0.0, 0.35, size=(n, 3))
    coef[:, 1:, :] = rng.normal(0.0, 0.04, size=(n, SH_BASIS - 1, 3))

    log_scales = np.log(axes).astype(np.float32)
    if density_scale and n > 10_000:
        log_scales = log_scales + np.float32(math.log((1.0e4 / n) ** (1.0 / 3.0)))
    return Scene(
        means=xyz.astype(np.float32),
        normals=np.zeros((n, 3), dtype=np.float32),
        sh=coef.astype(np.float32),
        logit_opacities=np.log(alpha / (1.0 - alpha)).astype(np.float32),
        log_scales=log_scales.astype(np.float32),
        rotations=quat.astype(np.float32),
    )
