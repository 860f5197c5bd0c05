"""B200-native FlashGS forward rasterizer behind the reference's call surface.

``Pipeline.render`` (reference ``tilesplat/pipeline.py:77-111``) and its four
stages run as hand-written sm_100a CUDA kernels reached through the C ABI in
``include/flashgs_b200.h``.  Importing this package never touches the GPU;
the first call that needs it loads ``_lib/libflashgs_b200.so`` and raises if
it is absent -- there is no CPU fallback.
"""

from .pipeline import (EVAL_FLOPS, BinOutput, Framebuffer, FrameStats, Pipeline, STRATEGIES,
                       TAU_DEFAULT, TILE_SIZE, UnsortedPairsError, blend_eval_counts, max_abs_diff,
                       power_cutoffs, preprocess_and_bin, psnr, render_frame,
                       run_frame, sort_pairs, sorted_pairs, tile_range_table)
from .reports import REPORT_SCHEMA_VERSION, CompareReport, bench_frames, compare_modes
from . import images, service
from .images import read_ppm, write_png, write_ppm
from .scene import (ActivatedScene, Camera, CameraValidationError, Scene, activate,
                    gen_synthetic, look_at_camera, make_camera, orbit_cameras)

from .scene_io import (CameraSchemaError, DeviceScene, PlyLengthError, PlyParseError,
                       PlySchemaError, load_cameras, load_ply, load_ply_device, save_cameras,
                       save_ply)

__version__ = "0.1.0"

__all__ = [
    "CameraSchemaError", "DeviceScene", "PlyLengthError", "PlyParseError", "PlySchemaError",
    "load_cameras", "load_ply", "load_ply_device", "save_cameras", "save_ply",
    "ActivatedScene", "BinOutput", "Camera", "CameraValidationError", "CompareReport",
    "Framebuffer", "REPORT_SCHEMA_VERSION", "bench_frames", "compare_modes",
    "FrameStats", "Pipeline", "STRATEGIES", "Scene", "TAU_DEFAULT", "TILE_SIZE",
    "UnsortedPairsError", "EVAL_FLOPS", "blend_eval_counts", "activate", "gen_synthetic", "look_at_camera", "make_camera",
    "max_abs_diff", "orbit_cameras", "power_cutoffs", "preprocess_and_bin", "psnr",
    "read_ppm", "write_png", "write_ppm", "images",
    "render_frame", "run_frame", "service", "sort_pairs", "sorted_pairs", "tile_range_table",
]
