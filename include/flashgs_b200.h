/*
 * flashgs_b200.h -- C ABI of the B200-native FlashGS forward rasterizer.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `tilesplat` (a CPU NumPy/numba rasterizer; it has no FFI of its own, its
 * boundary is the Python call surface of pipeline.py).  Each entry point
 * below names the reference function it replaces (file:line under
 * /root/reference/pkg/src/tilesplat).  INTEGRATION.md shows the ctypes stub a
 * maintainer of the reference would add to route those functions here.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless the name ends in `_host`;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - every call is asynchronous on `stream`, never allocates, never
 *     synchronises, never throws; it returns FGS_OK or a negative FGS_E_*;
 *   - data-dependent conditions (pair-buffer overflow, unsorted keys, tile
 *     index outside the grid, non-positive depth) are reported through the
 *     device-side `fgs_stats` block, which the caller copies back after the
 *     frame (the caller owns all memory; kernels only borrow it);
 *   - float32 geometry follows the reference's NumPy operation order with no
 *     FMA contraction, so the emitted (key, value) pair list and its sorted
 *     order are bit-identical to the reference's.
 */
#ifndef FLASHGS_B200_H
#define FLASHGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGS_ABI_VERSION 6
#define FGS_TILE 16              /* constants.py:4  TILE_SIZE */

enum {
    FGS_OK = 0,
    FGS_E_ARG = -1,              /* null pointer / negative size / bad enum  */
    FGS_E_SH_DEGREE = -2,        /* render.py:58-59   ValueError             */
    FGS_E_STRATEGY = -3,         /* binning.py:201-202 ValueError            */
    FGS_E_CUDA = -4,             /* a launch failed; see fgs_last_cuda_error */
    FGS_E_SIZE = -5,             /* size exceeds 32-bit pair / tile indexing */
    FGS_E_WORKSPACE = -6         /* workspace too small for this call        */
};

/* binning.py:38  STRATEGIES */
enum { FGS_PRECISE = 0, FGS_TIGHT_AABB = 1, FGS_BASELINE_CIRCLE_AABB = 2 };

/* How the frame's pairs get into (tile, depth, index) order (fgs_layout.sort_mode).
 * Both produce the bit-identical sorted list and range table.
 *   TILE_BUCKET (default): counting sort on the tile index with the CTA as the
 *     unit: fgs_preprocess counts each CTA's pairs per tile in shared memory
 *     and reserves one range per (CTA, tile) in the tile's bucket; the scan of
 *     the per-tile counters is the range table; fgs_emit walks again, gathers
 *     each CTA's records by tile in shared memory and writes contiguous runs.
 *     Each bucket is then sorted on (depth bits, index) in shared memory.
 *     Best with a scene packed in spatial order (fgs_scene_order), where a
 *     CTA's Gaussians share a few dozen tiles.  ~20 B of HBM traffic per pair.
 *   ONESWEEP: pairs emitted in Gaussian order, then a stable LSD radix sort
 *     (8-bit digits, one-sweep passes with decoupled look-back) over the packed
 *     tile|depth key, then a range-identification kernel.  ~172 B per pair. */
enum { FGS_SORT_ONESWEEP = 0, FGS_SORT_TILE_BUCKET = 1 };

/* fgs_blend flags */
enum {
    FGS_BLEND_EXACT   = 1,  /* glibc-equivalent expf in FP64, no FMA: frame is
                               bit-identical to the reference's; default is the
                               ex2.approx path with an exact re-check at the
                               alpha<tau threshold (max-abs error ~1e-6)      */
    FGS_BLEND_CONTRIB = 2,  /* fill the per-pair "touched a pixel" flags and
                               stats.pairs_contributing (render.py:200-231)  */
    FGS_BLEND_SCALAR  = 4   /* default numerics on the one-pixel-per-thread kernel
                               (kept as the A/B arm of the packed-f32x2 kernel) */
};

/* model_io.py:226-254 Camera, flattened.  Doubles are the Python floats the
 * reference keeps; they are rounded to float32 where the reference rounds
 * them (projection.py:100-103). */
typedef struct fgs_camera {
    int32_t width, height;
    float   view[16];            /* world_to_camera, row-major            */
    float   proj[16];            /* full_projection, row-major            */
    float   position[3];
    float   reserved0;
    double  tan_fovx, tan_fovy, focal_x, focal_y;
} fgs_camera;

/* Device-side counters of one frame (pipeline.py:28-48 FrameStats fields that
 * are data, not time).  80 bytes; lives at fgs_layout.off_stats. */
typedef struct fgs_stats {
    uint32_t pairs_emitted;        /* M, exact even when it overflowed      */
    uint32_t pairs_in_buffer;      /* M, or 0 when M > capacity             */
    uint32_t gaussians_retained;
    uint32_t gaussians_degenerate;
    uint32_t tiles_nonempty;
    uint32_t pairs_contributing;   /* only with FGS_BLEND_CONTRIB           */
    uint32_t overflow;             /* M > capacity: grow and re-run
                                      (binning.py:134-143 "never truncate") */
    uint32_t bad_depth;            /* binning.py:50-51                      */
    uint32_t unsorted;             /* sorting.py:146-147                    */
    uint32_t tile_out_of_grid;     /* sorting.py:150-151                    */
    uint32_t candidate_tiles_lo;   /* sum of nx*ny over retained, low/high  */
    uint32_t candidate_tiles_hi;
    uint32_t dense_tiles;          /* TILE_BUCKET: tiles with > 8192 pairs       */
    uint32_t medium_tiles;         /* TILE_BUCKET: tiles with 2049..4096 pairs   */
    uint32_t hard_tiles;           /* TILE_BUCKET: tiles sent to the radix fallback */
    uint32_t list_used;            /* TILE_BUCKET: (CTA, tile) table entries of the frame;
                                      at most M, so it fits whenever M fits          */
    uint32_t front_tiles;          /* tiles with more than 4096 pairs (with medium_tiles: what
                                      lazy_sort would sort a front of; filled with it on or off) */
    uint32_t redo_tiles;           /* lazy_sort: of those, tiles that had not saturated by the end
                                      of their sorted front -- sorted in full and blended again */
    uint32_t reserved[2];
} fgs_stats;

/* Byte offsets of every per-frame buffer inside the caller's workspace.
 * A pure function of (P, width, height, capacity). */
typedef struct fgs_layout {
    uint64_t total_bytes;
    uint64_t off_splat;        /* float  [P][12]  render.py:34-40 row layout  */
    uint64_t off_depth;        /* float  [P]      camera-space z              */
    uint64_t off_rects;        /* uint16 [P][4]   inclusive tx0,ty0,tx1,ty1   */
    uint64_t off_flags;        /* uint8  [P]      bit0 retained, bit1 degen.  */
    uint64_t off_counts;       /* uint32 [P]      emitted pairs per Gaussian  */
    uint64_t off_passmask;     /* uint64 [P]      bit j = candidate tile j (row-major in
                                  the banded rect) passed; valid when the
                                  Gaussian has <= 64 candidates              */
    uint64_t off_blocksums;    /* uint32 [2][nblocks]  sums, exclusive bases  */
    uint64_t off_keys[2];      /* uint64 [capacity]   ping / pong             */
    uint64_t off_vals[2];      /* uint32 [capacity]
                                  TILE_BUCKET: keys[1], vals[0], vals[1] are contiguous
                                  and hold the frame's (CTA, tile) table list (16 B x
                                  capacity) between fgs_preprocess and fgs_emit   */
    uint64_t off_sortstate;    /* uint64 [sort tiles][256] look-back table    */
    uint64_t off_hist;         /* uint32 [16][256] + tickets                  */
    uint64_t off_starts;       /* int32  [tiles + 1]  sorting.py:139-152      */
    uint64_t off_contrib;      /* uint8  [capacity]                           */
    uint64_t off_stats;        /* fgs_stats                                   */
    uint64_t off_tilecount;    /* uint32 [tiles][8]: TILE_BUCKET per-tile counters, one 32-byte
                                  sector each: [0] pairs reserved through the CTAs' tile
                                  tables, [1] fallback pairs, [2] fallback cursor       */
    uint64_t off_cursor;       /* uint32 [tiles][8]: size-class tile lists (words 1..4 and 7), slice totals of the tile scan (5, 6) */
    uint64_t off_ctainfo;      /* uint32 [preprocess blocks][4]: TILE_BUCKET, each K1 CTA's
                                  (first table entry, entries, write-combined records, 0) */
    uint64_t off_tileorder;    /* uint32 [160 + tiles]: TILE_BUCKET, 64 size-bin counts, 64 bin
                                  cursors, 32 control words, then the band's tiles ordered
                                  heaviest first (the order the blend's CTAs take them in) */
    int64_t  gaussians, capacity;   /* capacity = the request rounded up to 64 pairs */
    int32_t  width, height, grid_w, grid_h, tiles, tile_bits;
    int32_t  preprocess_blocks, sort_passes;
    int32_t  sort_mode;        /* FGS_SORT_*; change only via fgs_layout_set_sort_mode */
    int32_t  sorted_keys_in, sorted_vals_in;   /* which keys[] / vals[] buffer holds
                                  the sorted pairs after fgs_sort               */
    int32_t  keep_sorted_keys; /* TILE_BUCKET: also write the sorted 64-bit keys
                                  (only the values feed the blend); caller-set  */
    int32_t  lazy_sort;        /* TILE_BUCKET, caller-set, ignored with keep_sorted_keys: front-to-back
                                  compositing stops once a tile is opaque (render.py:154,178,228),
                                  so of a heavy tile -- 1: more than 4096 pairs, 2: more than 2048 --
                                  fgs_sort only orders the nearest ~1024 pairs (every pair nearer
                                  than a depth threshold, so the front IS the head of the tile's
                                  sorted list) and fgs_blend composites those; a tile that has not
                                  saturated by then is sorted in full and blended again from scratch
                                  inside the same fgs_blend call.  The frame, the contrib flags of
                                  every pair a pixel consumed and all counters are those of the full
                                  sort; the sorted VALUE buffer is complete only for the tiles that
                                  needed it.  0 = every tile sorted in full (sorting.py:101-136).
                                  Keep the value unchanged between fgs_sort and fgs_blend.  */
    int32_t  reserved0;
    uint64_t off_front;        /* TILE_BUCKET: int32 [tiles] sorted pairs at the head of each tile's
                                  bucket (INT32_MAX = all of them), then uint32 [tiles] redo list */
} fgs_layout;

int         fgs_abi_version(void);
const char *fgs_error_string(int code);
const char *fgs_last_cuda_error(void);

/* Profiling aid (pipeline.py:84-102 stage timers, at kernel granularity): after
 * fgs_profile_begin, every kernel launched by the calling thread through this
 * library is followed by a cudaEventRecord of the next event in `events`
 * (cudaEvent_t handles, caller-owned) on the launch stream.  fgs_profile_end
 * disarms and returns how many were recorded.  Frame order: preprocess, scan,
 * emit, then (ONESWEEP) sort histogram, one per sort pass, ranges, or
 * (TILE_BUCKET) tile sort for small, medium, large buckets and the dense + hard tail; then
 * blend. */
void    fgs_profile_begin(void **events, int32_t n_events);
int32_t fgs_profile_end(void);

/* ---- per-scene (model_io.py:78-118 ActivatedScene; untimed in the reference,
 *      pipeline.py:1-5) ------------------------------------------------------ */

/* model_io.py:136-199 load_ply / _scene_from_payload, the payload split on the device
 * (scene ingest): `vertex_payload` is the PLY body already in device
 * memory -- `gaussians` records of 62 little-endian float32 (x y z, nx ny nz, f_dc_0..2,
 * f_rest_0..44 channel-major, opacity, scale_0..2, rot_0..3; VERTEX_STRIDE = 248 bytes,
 * model_io.py:42-51).  Writes the reference Scene's arrays (model_io.py:57-76): means (P,3),
 * sh (P,16,3) coefficient-major with RGB innermost, logit opacities (P,), log scales (P,3),
 * rotations (P,4) as stored; normals are parsed and dropped.  Values are copied bit for bit.
 * Header parsing and its PlyParseError / PlySchemaError / PlyLengthError stay on the host
 * (paper_2408_07967_b200/scene_io.py).  Outputs feed fgs_scene_activate and fgs_scene_pack;
 * rotations_out must be 16-byte aligned for fgs_scene_activate. */
int fgs_scene_unpack_ply(const float *vertex_payload, int64_t gaussians, float *means_out,
                         float *sh_out, float *logit_opacities_out, float *log_scales_out,
                         float *rotations_out, void *stream);

/* model_io.py:93-118 activate, on the device: sign-split
 * sigmoid of the opacity logits, exp of the log-scales, quaternion normalisation
 * with zero-norm rows mapped to the identity.  Rotations are bit-identical to the
 * reference's NumPy result (IEEE sqrt / divide, same summation order); opacities
 * and scales use a correctly rounded exp (float64 exp rounded once), while NumPy's
 * float32 SIMD exp is good to ~2 ulp: scales can differ from the reference's by
 * 2 ulp, opacities by a few more.  Frames then agree to PSNR >= 60 dB and within 1e-3 on all but
 * isolated pixels: a 1-ulp opacity difference can flip one of the reference's hard skips
 * (alpha < tau) for a pixel, i.e. one contribution of at most ~tau * colour (< 5e-3).  The
 * bit-exact pair-list and 1e-3 max-abs guarantees hold for scenes activated by the reference
 * itself (the default: Pipeline activates raw scenes on the host with the reference's NumPy ops).
 * All pointers are device arrays; outputs feed fgs_scene_pack. */
int fgs_scene_activate(const float *logit_opacities, const float *log_scales,
                       const float *rotations, int64_t gaussians, float *opacities_out,
                       float *scales_out, float *rotations_out, void *stream);

/* Bytes of the packed device scene for P Gaussians (248 B per Gaussian, P rounded
 * up to 32). */
size_t fgs_scene_bytes(int64_t gaussians);

/* Spatial (Morton) order of a scene, computed on the device: order_out[slot] =
 * index of the Gaussian stored in that slot, a permutation of 0..P-1 sorted by
 * the 63-bit Morton code of the mean inside the scene's bounding box (ties by
 * index).  Per scene, untimed like activate (pipeline.py:1-5).  `scratch` is
 * fgs_scene_order_scratch_bytes(P) bytes of device memory. */
size_t fgs_scene_order_scratch_bytes(int64_t gaussians);
int fgs_scene_order(const float *means, int64_t gaussians, uint32_t *order_out,
                    void *scratch, size_t scratch_bytes, void *stream);

/* Re-lay the reference's arrays (means (P,3), opacities (P,), scales (P,3),
 * rotations (P,4) wxyz unit, sh (P,16,3)) into float4 planes so that the
 * preprocess kernel's loads are coalesced, plus the slot <-> index tables.
 * `order` (device, may be NULL = identity) is a permutation of 0..P-1: slot i
 * holds Gaussian order[i].  The per-Gaussian frame buffers (splat, depth,
 * rects, flags, counts) are indexed by SLOT: buffer row `slot` belongs to
 * Gaussian order[slot].  Pair values are Gaussian indices and the sorted list
 * is the reference's for any packing; FGS_SORT_ONESWEEP alone requires the
 * identity order (its pair values are slots). */
int fgs_scene_pack(const float *means, const float *opacities, const float *scales,
                   const float *rotations, const float *sh, const uint32_t *order,
                   int64_t gaussians, void *packed_scene, void *stream);

/* extent.py:19-30 power_cutoffs: k = min(9, 2 ln(alpha0 / tau)) with the log in
 * float64, rounded once to float32.  One float per Gaussian; depends on the
 * scene and tau only, so callers cache it per tau. */
int fgs_power_cutoffs(const void *packed_scene, int64_t gaussians, double tau,
                      float *k_out, void *stream);

/* ---- per-frame ---------------------------------------------------------- */

int fgs_workspace_layout(int64_t gaussians, int32_t width, int32_t height,
                         int64_t capacity, fgs_layout *out_host);

/* Select FGS_SORT_* for every later call that takes this layout (offsets do not
 * change; only sort_mode / sorted_*_in do). */
int fgs_layout_set_sort_mode(fgs_layout *layout_host, int32_t sort_mode);

/* Must be called once after the workspace is allocated (zeroes the sort
 * look-back table, whose entries are epoch-tagged afterwards).  Asynchronous on
 * `stream` like every call: a frame issued on ANOTHER stream must wait for it. */
int fgs_workspace_init(void *workspace, const fgs_layout *layout_host, void *stream);

/* binning.py:197-257 preprocess_and_bin, phase A + the count half of phase B:
 * cull, project, conic, cutoff, extent rectangle, SH colour, and the number of
 * candidate tiles that pass the strategy's test (intersect.py:63-94 for
 * `precise`).  Writes splat rows, depth, rects, flags, counts, and block sums
 * (ONESWEEP) or the per-tile counters plus each CTA's (tile, range) list
 * (TILE_BUCKET).
 * Tile rows outside [band_ty0, band_ty1] are not counted (row-band mode;
 * pass 0 and grid_h-1 for a whole frame). */
int fgs_preprocess(const void *packed_scene, const float *k_cut, int64_t gaussians,
                   const fgs_camera *camera_host, double tau, int32_t sh_degree,
                   int32_t strategy, int32_t band_ty0, int32_t band_ty1,
                   void *workspace, const fgs_layout *layout_host, void *stream);

/* Row-band load estimate for the multi-GPU row-band split (the reference
 * has no counterpart -- its tiles are split over a thread pool, render.py:276-304): writes
 * rows_out[ty] = number of Gaussians passing the frustum test (projection.py:39-47) whose
 * projected centre (projection.py:158-171) lies in tile row ty, for ty in 0..ceil(height/16)-1
 * (device array, zeroed by the call).  Integer counts, identical on every rank, so ranks
 * derive the same work-balanced band edges (paper_2408_07967_b200.sharding) without
 * communicating.  The rendered frame does not depend on the band edges. */
int fgs_row_histogram(const void *packed_scene, int64_t gaussians, const fgs_camera *camera_host,
                      double tau, uint32_t *rows_out, void *stream);

/* binning.py:292 (np.cumsum) / 129-147 (shared cursor): exclusive scan of the
 * per-block pair counts; fixes M, the overflow flag, and resets sort counters. */
int fgs_scan(void *workspace, const fgs_layout *layout_host, void *stream);

/* binning.py:264-354 phase B emit.
 * ONESWEEP: key = tile << 32 | depth bits (binning.py:47-54), value = Gaussian
 *   index, written at the scanned offsets, i.e. in ascending Gaussian order
 *   (deterministic, unlike an atomic cursor) into keys[0] / vals[0].
 * TILE_BUCKET: every pair is written once, as a (depth bits << 32 | index)
 *   record inside its (CTA, tile) range of the tile's bucket in keys[0]; order
 *   inside a bucket is arbitrary until fgs_sort. */
int fgs_emit(const void *packed_scene, const fgs_camera *camera_host, int32_t strategy,
             int32_t band_ty0, int32_t band_ty1, void *workspace,
             const fgs_layout *layout_host, void *stream);

/* sorting.py:101-136 sort_pairs for the frame's pair buffer: stable LSD radix
 * sort, 8-bit digits, over key bits [0,31) and [32, 32+tile_bits); emission
 * order makes ties come out in ascending value, so the value passes of the
 * reference are not needed.  `epoch` must increase by at least 16 per call on
 * the same workspace.
 * TILE_BUCKET: each tile's bucket is sorted on (depth bits, Gaussian index) in
 * shared memory.  vals[0] receives the Gaussian index of every sorted pair; with
 * layout.keep_sorted_keys keys[1] = tile << 32 | depth bits as well. */
int fgs_sort(void *workspace, const fgs_layout *layout_host, uint32_t epoch, void *stream);

/* sorting.py:139-152 tile_range_table on the sorted buffer. */
int fgs_ranges(void *workspace, const fgs_layout *layout_host, void *stream);

/* render.py:273-310 render_frame (+ 135-252 the pipelined compositor).
 * out_rgb (H,W,3) float32 is required; out_alpha (H,W) = 1 - T_final and
 * out_depth (H,W) = sum of blend weight * camera z are optional extras.
 * `packed_scene` supplies the index -> slot table: pair values are Gaussian
 * indices, the splat rows are stored by slot. */
int fgs_blend(const void *packed_scene, const float background[3], double tau, int32_t flags,
              int32_t band_ty0, int32_t band_ty1,
              float *out_rgb, float *out_alpha, float *out_depth,
              void *workspace, const fgs_layout *layout_host, void *stream);

/* Measurement aid (SURVEY.md 8(d), FP32 roofline of the blend): re-blends the frame whose
 * sorted pairs are in the workspace with the exact-mode kernel and counts the (pixel, pair)
 * evaluations of the reference's naive loop (render.py:106-129) by outcome.  counts_out
 * (device, 8 x uint64, zeroed by the call): [0] rejected by the extent rectangle
 * (render.py:111), [1] by the cutoff s > k/2 (:114), [2] by alpha < tau (:119), [3] blended,
 * [4] M_proc = sum over tiles of the pairs visited before the tile's last pixel stopped
 * (:228-229), [5] pixels.  out_rgb receives the exact-mode frame.  Not on the frame path. */
int fgs_blend_counts(const void *packed_scene, const float background[3], double tau,
                     int32_t band_ty0, int32_t band_ty1, float *out_rgb, uint64_t *counts_out,
                     void *workspace, const fgs_layout *layout_host, void *stream);

/* pipeline.py:77-111 Pipeline.render: the six calls above, back to back on
 * `stream`, no host synchronisation in between. */
int fgs_render(const void *packed_scene, const float *k_cut, int64_t gaussians,
               const fgs_camera *camera_host, double tau, int32_t sh_degree,
               int32_t strategy, const float background[3], int32_t blend_flags,
               int32_t band_ty0, int32_t band_ty1, uint32_t epoch,
               float *out_rgb, float *out_alpha, float *out_depth,
               void *workspace, const fgs_layout *layout_host, void *stream);

/* ---- stand-alone stages on caller-supplied arrays (the reference exposes the
 *      same stages so intermediates can be diffed) ---------- */

/* Scratch bytes fgs_sort_pairs needs for n pairs. */
size_t fgs_sort_pairs_scratch_bytes(int64_t n);

/* sorting.py:101-136 on arbitrary input order: value bytes first
 * (ceil(value_bits/8) passes), then key bits [0, 32+tile_bits).  keys_out /
 * vals_out receive the result; inputs are not modified.  `scratch` must be
 * zero-initialised once and may then be reused with increasing epochs. */
int fgs_sort_pairs(const uint64_t *keys_in, const uint32_t *vals_in, int64_t n,
                   int32_t tile_bits, int32_t value_bits,
                   uint64_t *keys_out, uint32_t *vals_out,
                   void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream);

/* sorting.py:139-152: starts[tiles+1] (int32) from sorted keys; sets
 * stats->unsorted / stats->tile_out_of_grid instead of raising. */
int fgs_tile_ranges(const uint64_t *sorted_keys, int64_t n, int32_t tiles,
                    int32_t *starts, fgs_stats *stats, void *stream);

/* render.py:273-310 on a caller-supplied splat table (P,12), sorted values
 * and range table. */
int fgs_blend_tiles(const float *splat, const float *gaussian_depth,
                    const uint32_t *sorted_values, const int32_t *starts,
                    int32_t width, int32_t height, const float background[3],
                    double tau, int32_t flags, int32_t band_ty0, int32_t band_ty1,
                    float *out_rgb, float *out_alpha, float *out_depth,
                    uint8_t *contrib, fgs_stats *stats, void *stream);

/* images.py:12-15 quantize: float32 linear channels -> uint8,
 * q = floor(clip(c, 0, 1) * 255 + 0.5) evaluated in float64 like the reference.
 * `count` = number of channel values (H*W*3).  The step after the path: it lets a
 * frame service read back 3 bytes per pixel instead of 12. */
int fgs_quantize_rgb8(const float *rgb, int64_t count, uint8_t *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHGS_B200_H */
