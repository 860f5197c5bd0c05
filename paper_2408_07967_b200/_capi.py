"""ctypes binding of libflashgs_b200.so (include/flashgs_b200.h).

There is deliberately no fallback: if the library has not been built, or no
CUDA device is present, every product entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FGS_LIB selects another build of the same library (tuning variants, see build.py)
LIB_PATH = os.environ.get("FGS_LIB") or os.path.join(HERE, "_lib", "libflashgs_b200.so")

ABI_VERSION = 6
STRATEGIES = ("baseline-circle-aabb", "tight-aabb", "precise")   # binning.py:38 order
STRATEGY_ID = {"precise": 0, "tight-aabb": 1, "baseline-circle-aabb": 2}
BLEND_EXACT, BLEND_CONTRIB, BLEND_SCALAR = 1, 2, 4
SORT_ONESWEEP, SORT_TILE_BUCKET = 0, 1
SORT_MODES = {"onesweep": SORT_ONESWEEP, "tile-bucket": SORT_TILE_BUCKET}
SORT_TILE = 4096

# every symbol include/flashgs_b200.h declares (checked by the CPU test-suite)
SYMBOLS = (
    "fgs_abi_version", "fgs_error_string", "fgs_last_cuda_error", "fgs_scene_bytes",
    "fgs_scene_order_scratch_bytes", "fgs_scene_order", "fgs_scene_pack", "fgs_scene_activate", "fgs_scene_unpack_ply", "fgs_power_cutoffs", "fgs_workspace_layout", "fgs_layout_set_sort_mode",
    "fgs_workspace_init",
    "fgs_preprocess", "fgs_row_histogram", "fgs_scan", "fgs_emit", "fgs_sort", "fgs_ranges", "fgs_blend",
    "fgs_render", "fgs_sort_pairs_scratch_bytes", "fgs_sort_pairs", "fgs_tile_ranges",
    "fgs_blend_tiles", "fgs_blend_counts", "fgs_profile_begin", "fgs_profile_end", "fgs_quantize_rgb8",
)


class FgsCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("view", C.c_float * 16), ("proj", C.c_float * 16),
                ("position", C.c_float * 3), ("reserved0", C.c_float),
                ("tan_fovx", C.c_double), ("tan_fovy", C.c_double),
                ("focal_x", C.c_double), ("focal_y", C.c_double)]


class FgsStats(C.Structure):
    _fields_ = [("pairs_emitted", C.c_uint32), ("pairs_in_buffer", C.c_uint32),
                ("gaussians_retained", C.c_uint32), ("gaussians_degenerate", C.c_uint32),
                ("tiles_nonempty", C.c_uint32), ("pairs_contributing", C.c_uint32),
                ("overflow", C.c_uint32), ("bad_depth", C.c_uint32),
                ("unsorted", C.c_uint32), ("tile_out_of_grid", C.c_uint32),
                ("candidate_tiles_lo", C.c_uint32), ("candidate_tiles_hi", C.c_uint32),
                ("dense_tiles", C.c_uint32), ("medium_tiles", C.c_uint32),
                ("hard_tiles", C.c_uint32), ("list_used", C.c_uint32),
                ("front_tiles", C.c_uint32), ("redo_tiles", C.c_uint32),
                ("reserved_a", C.c_uint32), ("reserved_b", C.c_uint32)]


STATS_DTYPE = np.dtype([(n, np.uint32) for n, _ in FgsStats._fields_])
assert STATS_DTYPE.itemsize == C.sizeof(FgsStats) == 80
STATS_BYTES = STATS_DTYPE.itemsize


class FgsLayout(C.Structure):
    _fields_ = [("total_bytes", C.c_uint64), ("off_splat", C.c_uint64),
                ("off_depth", C.c_uint64), ("off_rects", C.c_uint64),
                ("off_flags", C.c_uint64), ("off_counts", C.c_uint64),
                ("off_passmask", C.c_uint64),
                ("off_blocksums", C.c_uint64), ("off_keys", C.c_uint64 * 2),
                ("off_vals", C.c_uint64 * 2), ("off_sortstate", C.c_uint64),
                ("off_hist", C.c_uint64), ("off_starts", C.c_uint64),
                ("off_contrib", C.c_uint64), ("off_stats", C.c_uint64),
                ("off_tilecount", C.c_uint64), ("off_cursor", C.c_uint64),
                ("off_ctainfo", C.c_uint64),
                ("off_tileorder", C.c_uint64),
                ("gaussians", C.c_int64), ("capacity", C.c_int64),
                ("width", C.c_int32), ("height", C.c_int32), ("grid_w", C.c_int32),
                ("grid_h", C.c_int32), ("tiles", C.c_int32), ("tile_bits", C.c_int32),
                ("preprocess_blocks", C.c_int32), ("sort_passes", C.c_int32),
                ("sort_mode", C.c_int32), ("sorted_keys_in", C.c_int32),
                ("sorted_vals_in", C.c_int32), ("keep_sorted_keys", C.c_int32),
                ("lazy_sort", C.c_int32), ("reserved0", C.c_int32),
                ("off_front", C.c_uint64)]


class FgsError(RuntimeError):
    def __init__(self, code, detail=""):
        self.code = int(code)
        super().__init__(f"libflashgs_b200 error {code}: {detail}")


_lib = None
_lock = threading.Lock()


def _declare(L):
    vp, i32, i64, u32, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
    cam_p, lay_p = C.POINTER(FgsCamera), C.POINTER(FgsLayout)
    f3 = C.POINTER(C.c_float)
    sig = {
        "fgs_abi_version": (C.c_int, []),
        "fgs_profile_begin": (None, [C.POINTER(C.c_void_p), i32]),
        "fgs_profile_end": (i32, []),
        "fgs_error_string": (C.c_char_p, [C.c_int]),
        "fgs_last_cuda_error": (C.c_char_p, []),
        "fgs_scene_bytes": (C.c_size_t, [i64]),
        "fgs_scene_activate": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
        "fgs_scene_unpack_ply": (C.c_int, [vp, i64, vp, vp, vp, vp, vp, vp]),
        "fgs_scene_order_scratch_bytes": (C.c_size_t, [i64]),
        "fgs_scene_order": (C.c_int, [vp, i64, vp, vp, C.c_size_t, vp]),
        "fgs_scene_pack": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, vp, vp]),
        "fgs_power_cutoffs": (C.c_int, [vp, i64, dbl, vp, vp]),
        "fgs_workspace_layout": (C.c_int, [i64, i32, i32, i64, lay_p]),
        "fgs_layout_set_sort_mode": (C.c_int, [lay_p, i32]),
        "fgs_workspace_init": (C.c_int, [vp, lay_p, vp]),
        "fgs_preprocess": (C.c_int, [vp, vp, i64, cam_p, dbl, i32, i32, i32, i32, vp, lay_p, vp]),
        "fgs_row_histogram": (C.c_int, [vp, i64, cam_p, dbl, vp, vp]),
        "fgs_scan": (C.c_int, [vp, lay_p, vp]),
        "fgs_emit": (C.c_int, [vp, cam_p, i32, i32, i32, vp, lay_p, vp]),
        "fgs_sort": (C.c_int, [vp, lay_p, u32, vp]),
        "fgs_ranges": (C.c_int, [vp, lay_p, vp]),
        "fgs_blend": (C.c_int, [vp, f3, dbl, i32, i32, i32, vp, vp, vp, vp, lay_p, vp]),
        "fgs_blend_counts": (C.c_int, [vp, f3, dbl, i32, i32, vp, vp, vp, lay_p, vp]),
        "fgs_render": (C.c_int, [vp, vp, i64, cam_p, dbl, i32, i32, f3, i32, i32, i32, u32,
                                 vp, vp, vp, vp, lay_p, vp]),
        "fgs_sort_pairs_scratch_bytes": (C.c_size_t, [i64]),
        "fgs_sort_pairs": (C.c_int, [vp, vp, i64, i32, i32, vp, vp, vp, C.c_size_t, u32, vp]),
        "fgs_tile_ranges": (C.c_int, [vp, i64, i32, vp, vp, vp]),
        "fgs_blend_tiles": (C.c_int, [vp, vp, vp, vp, i32, i32, f3, dbl, i32, i32, i32,
                                      vp, vp, vp, vp, vp, vp]),
        "fgs_quantize_rgb8": (C.c_int, [vp, i64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded CUDA library; raises if it is missing (no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_2408_07967_b200.build` (there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            _declare(L)
            if L.fgs_abi_version() != ABI_VERSION:
                raise RuntimeError("libflashgs_b200.so ABI version mismatch; rebuild it")
            _lib = L
    return _lib


def check(rc):
    if rc != 0:
        L = lib()
        msg = L.fgs_error_string(rc).decode()
        if rc == -4:
            msg += " (" + L.fgs_last_cuda_error().decode() + ")"
        raise FgsError(rc, msg)


def camera_struct(cam) -> FgsCamera:
    """Flatten a Camera (ours or the reference's; same field names)."""
    s = FgsCamera()
    s.width, s.height = int(cam.width), int(cam.height)
    s.view[:] = np.asarray(cam.world_to_camera, dtype=np.float32).reshape(16).tolist()
    s.proj[:] = np.asarray(cam.full_projection, dtype=np.float32).reshape(16).tolist()
    s.position[:] = np.asarray(cam.position, dtype=np.float32).reshape(3).tolist()
    s.tan_fovx, s.tan_fovy = float(cam.tan_fovx), float(cam.tan_fovy)
    s.focal_x, s.focal_y = float(cam.focal_x), float(cam.focal_y)
    return s


def layout(P, width, height, capacity, sort_mode=None) -> FgsLayout:
    out = FgsLayout()
    check(lib().fgs_workspace_layout(int(P), int(width), int(height), int(capacity), C.byref(out)))
    if sort_mode is not None:
        check(lib().fgs_layout_set_sort_mode(C.byref(out), int(sort_mode)))
    return out
