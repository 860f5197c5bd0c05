"""ctypes front end of the CPU oracle (``fgs_oracle.c``).

TEST INFRASTRUCTURE ONLY -- see the header of ``fgs_oracle.c``.  The product
package never imports this module; ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline legs do, as the checker / CPU arm.

The functions mirror the reference's stage entry points so tests read like
the reference's own:

    preprocess_and_bin -> binning.py:197     sort_pairs       -> sorting.py:101
    tile_range_table   -> sorting.py:139     render_frame     -> render.py:273
    render             -> pipeline.py:77 (bin -> sort -> render + stage timers)
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libfgs_oracle.so")

STRATEGIES = ("precise", "tight-aabb", "baseline-circle-aabb")
_STRAT_ID = {"precise": 0, "tight-aabb": 1, "baseline-circle-aabb": 2}


class UnsortedPairsError(ValueError):
    pass


class _Cam(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("view", C.c_float * 16), ("proj", C.c_float * 16),
                ("position", C.c_float * 3), ("_pad", C.c_float),
                ("tan_fovx", C.c_double), ("tan_fovy", C.c_double),
                ("focal_x", C.c_double), ("focal_y", C.c_double)]


def build(force=False) -> str:
    """Compile the oracle with the committed recipe (oracle/Makefile)."""
    src = os.path.join(_HERE, "fgs_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s", "-B"], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.orc_emit_pairs.restype = C.c_int64
        L.orc_render_frame.restype = C.c_int64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _cam_struct(cam) -> _Cam:
    s = _Cam()
    s.width, s.height = int(cam.width), int(cam.height)
    s.view[:] = np.asarray(cam.world_to_camera, dtype=np.float32).reshape(16).tolist()
    s.proj[:] = np.asarray(cam.full_projection, dtype=np.float32).reshape(16).tolist()
    s.position[:] = np.asarray(cam.position, dtype=np.float32).reshape(3).tolist()
    s.tan_fovx, s.tan_fovy = float(cam.tan_fovx), float(cam.tan_fovy)
    s.focal_x, s.focal_y = float(cam.focal_x), float(cam.focal_y)
    return s


def set_threads(n: int):
    lib().orc_set_threads(C.c_int(int(n)))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def power_cutoffs(alpha0, tau=1.0 / 255.0):
    a = np.ascontiguousarray(np.atleast_1d(alpha0), dtype=np.float32)
    k = np.empty_like(a)
    keep = np.empty(a.shape[0], dtype=np.uint8)
    lib().orc_power_cutoffs(_p(a), C.c_int64(a.shape[0]), C.c_double(tau), _p(k), _p(keep))
    return k, keep.astype(bool)


def tile_hits_ellipse(rect, center, conic, k) -> bool:
    L = lib()
    L.orc_tile_hits_ellipse.argtypes = [C.c_double] * 10
    return bool(L.orc_tile_hits_ellipse(*[float(v) for v in (*rect, *center, *conic, k)]))


@dataclass
class BinOutput:
    """Same fields as the reference's BinOutput (binning.py:150-173)."""
    splat: np.ndarray
    depth: np.ndarray
    retained: np.ndarray
    tile_rects: np.ndarray
    tile_counts: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    emitted_count: int
    gaussians_retained: int
    gaussians_degenerate: int
    buffer_regrows: int
    capacity: int
    grid_w: int
    grid_h: int
    strategy: str
    tau: float
    k_eff: np.ndarray = None
    pair_counts: np.ndarray = None

    @property
    def pair_buffer_bytes(self) -> int:
        return self.emitted_count * 12


def _scene_arrays(act):
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return f(act.means), f(act.opacities), f(act.scales), f(act.rotations), f(act.sh)


def preprocess_and_bin(act, camera, strategy="precise", tau=1.0 / 255.0,
                       sh_degree=3) -> BinOutput:
    if strategy not in _STRAT_ID:
        raise ValueError(f"unknown strategy {strategy!r}, expected one of {STRATEGIES}")
    if not 0 <= int(sh_degree) <= 3:
        raise ValueError("SH degree must be in 0..3")
    L = lib()
    means, opac, scales, rots, sh = _scene_arrays(act)
    P = means.shape[0]
    cam = _cam_struct(camera)
    splat = np.empty((P, 12), np.float32)
    depth = np.empty(P, np.float32)
    retained = np.empty(P, np.uint8)
    degenerate = np.empty(P, np.uint8)
    rects = np.empty((P, 4), np.int32)
    k_eff = np.empty(P, np.float32)
    sid = _STRAT_ID[strategy]
    rc = L.orc_preprocess(_p(means), _p(opac), _p(scales), _p(rots), _p(sh), C.c_int64(P),
                          C.byref(cam), C.c_double(tau), C.c_int(sh_degree), C.c_int(sid),
                          _p(splat), _p(depth), _p(retained), _p(degenerate), _p(rects),
                          _p(k_eff))
    if rc != 0:
        raise RuntimeError(f"orc_preprocess failed: {rc}")
    counts = np.empty(P, np.int64)
    args = (_p(splat), _p(depth), _p(retained), _p(rects), _p(k_eff), C.c_int64(P),
            C.c_int(camera.width), C.c_int(camera.height), C.c_int(sid))
    total = L.orc_emit_pairs(*args, _p(counts), None, None)
    keys = np.empty(total, np.uint64)
    values = np.empty(total, np.uint32)
    got = L.orc_emit_pairs(*args, _p(counts), _p(keys), _p(values))
    if got == -1:
        raise ValueError("depths must be positive and finite (cull failed upstream)")
    assert got == total
    nx = rects[:, 2] - rects[:, 0] + 1
    ny = rects[:, 3] - rects[:, 1] + 1
    ret = retained.astype(bool)
    gw, gh = -(-camera.width // 16), -(-camera.height // 16)
    return BinOutput(
        splat=splat, depth=depth, retained=ret, tile_rects=rects,
        tile_counts=np.where(ret, (nx * ny).astype(np.int64), 0),
        keys=keys, values=values, emitted_count=int(total),
        gaussians_retained=int(ret.sum()), gaussians_degenerate=int(degenerate.sum()),
        buffer_regrows=0, capacity=int(total), grid_w=gw, grid_h=gh,
        strategy=strategy, tau=float(tau), k_eff=k_eff, pair_counts=counts)


def sort_pairs(keys, values, grid_tiles=None, max_value=None):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    values = np.ascontiguousarray(values, dtype=np.uint32)
    if keys.shape[0] != values.shape[0]:
        raise ValueError("keys and values must have equal length")
    ok, ov = np.empty_like(keys), np.empty_like(values)
    rc = lib().orc_sort_pairs(_p(keys), _p(values), C.c_int64(keys.shape[0]),
                              C.c_int64(-1 if grid_tiles is None else int(grid_tiles)),
                              C.c_int64(-1 if max_value is None else int(max_value)),
                              _p(ok), _p(ov))
    if rc != 0:
        raise MemoryError("orc_sort_pairs")
    return ok, ov


def tile_range_table(sorted_keys, grid_w, grid_h):
    k = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
    tiles = int(grid_w) * int(grid_h)
    starts = np.empty(tiles + 1, np.int64)
    rc = lib().orc_tile_ranges(_p(k), C.c_int64(k.shape[0]), C.c_int64(tiles), _p(starts))
    if rc == -1:
        raise UnsortedPairsError("pair keys are not nondecreasing")
    if rc == -2:
        raise ValueError("tile index exceeds the grid")
    return starts


def render_frame(splat, sorted_values, starts, width, height, background, tau,
                 gaussian_depth=None, extras=False):
    """Returns (image, contrib, nonempty) or, with extras, also (alpha, depth)."""
    splat = np.ascontiguousarray(splat, dtype=np.float32)
    vals = np.ascontiguousarray(sorted_values, dtype=np.uint32)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float32).reshape(3))
    img = np.empty((height, width, 3), np.float32)
    contrib = np.zeros(vals.shape[0], np.uint8)
    alpha = np.empty((height, width), np.float32) if extras else None
    dmap = np.empty((height, width), np.float32) if extras else None
    gd = np.ascontiguousarray(gaussian_depth, dtype=np.float32) if extras else None
    n = lib().orc_render_frame(_p(splat), _p(vals), _p(st), C.c_int(width), C.c_int(height),
                               _p(bg), C.c_double(tau), _p(img), _p(contrib),
                               _p(gd), _p(alpha), _p(dmap))
    if extras:
        return img, contrib, int(n), alpha, dmap
    return img, contrib, int(n)


EVAL_CLASSES = ("rect_rejected", "cutoff_rejected", "alpha_rejected", "blended")


def render_counts(splat, sorted_values, starts, width, height, tau):
    """Instrumented copy of the naive compositing loop (render.py:106-129): evaluation
    counts by outcome, M_proc and the pixel count, as a dict."""
    splat = np.ascontiguousarray(splat, dtype=np.float32)
    vals = np.ascontiguousarray(sorted_values, dtype=np.uint32)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    out = np.zeros(8, np.uint64)
    lib().orc_render_counts(_p(splat), _p(vals), _p(st), C.c_int(width), C.c_int(height),
                            C.c_double(tau), _p(out))
    d = {k: int(out[i]) for i, k in enumerate(EVAL_CLASSES)}
    d["pairs_processed"], d["pixels"] = int(out[4]), int(out[5])
    return d


def render(act, camera, strategy="precise", tau=1.0 / 255.0,
           background=(0.0, 0.0, 0.0), sh_degree=3, extras=False):
    """Whole path with the reference's three stage timers (pipeline.py:84-102).

    Returns (image, stats dict[, alpha, depth])."""
    t0 = time.perf_counter_ns()
    out = preprocess_and_bin(act, camera, strategy, tau, sh_degree)
    t1 = time.perf_counter_ns()
    keys, values = sort_pairs(out.keys, out.values, out.grid_w * out.grid_h,
                              max(int(out.depth.shape[0]), 1))
    starts = tile_range_table(keys, out.grid_w, out.grid_h)
    t2 = time.perf_counter_ns()
    res = render_frame(out.splat, values, starts, camera.width, camera.height,
                       background, tau, out.depth, extras)
    t3 = time.perf_counter_ns()
    stats = dict(strategy=strategy, tau=float(tau), workers=max_threads(),
                 preprocess_bin_ns=t1 - t0, sort_ns=t2 - t1, render_ns=t3 - t2,
                 total_ns=t3 - t0, pairs_emitted=out.emitted_count,
                 pairs_contributing=int(res[1].sum()),
                 gaussians_retained=out.gaussians_retained,
                 gaussians_degenerate=out.gaussians_degenerate,
                 tiles_nonempty=res[2], pair_buffer_bytes=out.pair_buffer_bytes,
                 buffer_regrows=0)
    if extras:
        return res[0], stats, res[3], res[4]
    return res[0], stats
