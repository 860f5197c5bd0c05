// extern "C" entry points of libflashgs_b200.so (see include/flashgs_b200.h).
// Pure argument checking + stage launches; no allocation, no synchronisation.

#include <stdio.h>
#include <string.h>

#include "fgs_common.cuh"

static thread_local char g_cuda_err[256] = "";

void fgs_set_cuda_error(cudaError_t e)
{
    const char *n = cudaGetErrorName(e), *s = cudaGetErrorString(e);
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", n ? n : "?", s ? s : "?");
}

static thread_local void **g_prof_events = nullptr;
static thread_local int g_prof_cap = 0, g_prof_n = 0;

void fgs_prof_mark(cudaStream_t st)
{
    if (g_prof_events && g_prof_n < g_prof_cap)
        cudaEventRecord((cudaEvent_t)g_prof_events[g_prof_n++], st);
}

bool fgs_prof_armed() { return g_prof_events != nullptr; }

static CamDev make_cam(const fgs_camera *c)
{
    CamDev d;
    for (int i = 0; i < 12; ++i) d.v[i] = c->view[i];
    for (int i = 0; i < 4; ++i) {
        d.p0[i] = c->proj[i];
        d.p1[i] = c->proj[4 + i];
        d.p3[i] = c->proj[12 + i];
    }
    for (int i = 0; i < 3; ++i) d.pos[i] = c->position[i];
    d.limx = (float)(1.3 * c->tan_fovx);          // projection.py:100-101
    d.limy = (float)(1.3 * c->tan_fovy);
    d.fx = (float)c->focal_x;                     // projection.py:104-105
    d.fy = (float)c->focal_y;
    d.wf = (float)c->width;
    d.hf = (float)c->height;
    d.width = c->width;
    d.height = c->height;
    d.grid_w = (c->width + FGS_TILE - 1) / FGS_TILE;
    d.grid_h = (c->height + FGS_TILE - 1) / FGS_TILE;
    return d;
}

// lazy_sort as the launchers take it: 0 off, 1 / 2 = which tiles get a front only
static int fgs_lazy(const fgs_layout *L)
{
    if (L->lazy_sort <= 0 || L->keep_sorted_keys || L->sort_mode != FGS_SORT_TILE_BUCKET) return 0;
    return L->lazy_sort >= 2 ? 2 : 1;
}

// pair count beyond which lazy_sort sorts only a front of a tile (0: every tile in full)
static uint32_t fgs_heavy_thr(const fgs_layout *L)
{
    const int lazy = fgs_lazy(L);
    return lazy == 2 ? FGS_SMALL_TILE : lazy == 1 ? FGS_DENSE_TILE : 0u;
}

static int check_frame(const fgs_layout *L, const fgs_camera *c)
{
    if (!L) return FGS_E_ARG;
    if (c && (c->width != L->width || c->height != L->height)) return FGS_E_WORKSPACE;
    return FGS_OK;
}

extern "C" {

int fgs_abi_version(void) { return FGS_ABI_VERSION; }

const char *fgs_error_string(int code)
{
    switch (code) {
    case FGS_OK: return "ok";
    case FGS_E_ARG: return "invalid argument";
    case FGS_E_SH_DEGREE: return "SH degree must be in 0..3";
    case FGS_E_STRATEGY: return "unknown strategy";
    case FGS_E_CUDA: return "CUDA launch failed";
    case FGS_E_SIZE: return "size exceeds 32-bit pair/tile indexing";
    case FGS_E_WORKSPACE: return "workspace layout does not match this call";
    default: return "unknown error";
    }
}

const char *fgs_last_cuda_error(void) { return g_cuda_err; }

void fgs_profile_begin(void **events, int32_t n_events)
{
    g_prof_events = events;
    g_prof_cap = events ? n_events : 0;
    g_prof_n = 0;
}

int32_t fgs_profile_end(void)
{
    const int n = g_prof_n;
    g_prof_events = nullptr;
    g_prof_cap = g_prof_n = 0;
    return n;
}

size_t fgs_scene_bytes(int64_t P)
{
    if (P < 0) return 0;
    return (size_t)fgs_pad32(P) * (15 * sizeof(float4) + 2 * sizeof(uint32_t));
}

// scratch of fgs_scene_order: [bbox 256 B][codes u64][indices u32][sorted codes u64][sort scratch]
static inline uint64_t al256(uint64_t b) { return (b + 255) & ~(uint64_t)255; }

size_t fgs_scene_order_scratch_bytes(int64_t P)
{
    if (P < 0) return 0;
    const uint64_t p = (uint64_t)P;
    return (size_t)(256 + 2 * al256(p * 8) + al256(p * 4) + al256(fgs_sort_pairs_scratch_bytes(P)));
}

int fgs_scene_order(const float *means, int64_t P, uint32_t *order_out, void *scratch,
                    size_t scratch_bytes, void *stream)
{
    if (P < 0 || P > 0x3fffff00ll) return P < 0 ? FGS_E_ARG : FGS_E_SIZE;
    if (P == 0) return FGS_OK;
    if (!means || !order_out || !scratch) return FGS_E_ARG;
    if (scratch_bytes < fgs_scene_order_scratch_bytes(P)) return FGS_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t p = (uint64_t)P;
    char *b = (char *)scratch;
    float *bbox = (float *)b;            b += 256;
    uint64_t *codes = (uint64_t *)b;     b += al256(p * 8);
    uint32_t *idx = (uint32_t *)b;       b += al256(p * 4);
    uint64_t *codes_out = (uint64_t *)b; b += al256(p * 8);
    const size_t sort_bytes = fgs_sort_pairs_scratch_bytes(P);
    cudaError_t e = cudaMemsetAsync(b, 0, sort_bytes, st);     // look-back table starts clean
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    int rc = fgs_launch_morton_keys(means, P, bbox, codes, idx, st);
    if (rc) return rc;
    // stable LSD sort over code bits [0, 63): ties keep ascending index
    return fgs_sort_pairs(codes, idx, P, 31, 0, codes_out, order_out, b, sort_bytes, 1u, stream);
}

int fgs_scene_unpack_ply(const float *vertex_payload, int64_t P, float *means_out, float *sh_out,
                         float *logit_opacities_out, float *log_scales_out, float *rotations_out,
                         void *stream)
{
    if (P < 0) return FGS_E_ARG;
    if (P > 0x7fffff00ll) return FGS_E_SIZE;
    if (P && (!vertex_payload || !means_out || !sh_out || !logit_opacities_out || !log_scales_out ||
              !rotations_out))
        return FGS_E_ARG;
    return fgs_launch_unpack_ply(vertex_payload, P, means_out, sh_out, logit_opacities_out,
                                 log_scales_out, rotations_out, (cudaStream_t)stream);
}

int fgs_scene_activate(const float *logit_opacities, const float *log_scales, const float *rotations,
                       int64_t P, float *opacities_out, float *scales_out, float *rotations_out,
                       void *stream)
{
    if (P < 0) return FGS_E_ARG;
    if (P && (!logit_opacities || !log_scales || !rotations || !opacities_out || !scales_out ||
              !rotations_out))
        return FGS_E_ARG;
    if (((uintptr_t)rotations & 15) || ((uintptr_t)rotations_out & 15)) return FGS_E_ARG;
    return fgs_launch_activate(logit_opacities, log_scales, rotations, P, opacities_out, scales_out,
                               rotations_out, (cudaStream_t)stream);
}

int fgs_scene_pack(const float *means, const float *opacities, const float *scales,
                   const float *rotations, const float *sh, const uint32_t *order, int64_t P,
                   void *packed, void *stream)
{
    if (P < 0 || P > 0x7fffff00ll) return P < 0 ? FGS_E_ARG : FGS_E_SIZE;
    if (P && (!means || !opacities || !scales || !rotations || !sh || !packed)) return FGS_E_ARG;
    return fgs_launch_pack(means, opacities, scales, rotations, sh, order, P, packed,
                           (cudaStream_t)stream);
}

int fgs_power_cutoffs(const void *packed, int64_t P, double tau, float *k_out, void *stream)
{
    if (P < 0 || !(tau > 0.0)) return FGS_E_ARG;
    if (P && (!packed || !k_out)) return FGS_E_ARG;
    return fgs_launch_cutoffs(fgs_scene_view(packed, P), P, tau, k_out, (cudaStream_t)stream);
}

int fgs_workspace_layout(int64_t P, int32_t width, int32_t height, int64_t capacity,
                         fgs_layout *L)
{
    if (!L || P < 0 || width < 1 || height < 1 || capacity < 0) return FGS_E_ARG;
    // 30-bit pair counts in the sort look-back words; 31-bit Gaussian indices
    if (P > 0x7fffff00ll || capacity > 0x3fffffc0ll) return FGS_E_SIZE;
    memset(L, 0, sizeof(*L));
    const int64_t gw = (width + FGS_TILE - 1) / FGS_TILE, gh = (height + FGS_TILE - 1) / FGS_TILE;
    if (gw > 65535 || gh > 65535 || gw * gh > 0x7ffffff0ll) return FGS_E_SIZE;
    L->gaussians = P;
    capacity = (capacity + 63) & ~(int64_t)63;        // keys[1] | vals[0] | vals[1] contiguous
    L->capacity = capacity;
    L->width = width;
    L->height = height;
    L->grid_w = (int32_t)gw;
    L->grid_h = (int32_t)gh;
    L->tiles = (int32_t)(gw * gh);
    int tb = 0;
    while (((int64_t)1 << tb) < gw * gh) ++tb;        // bits to hold tile index < tiles
    L->tile_bits = tb;
    L->preprocess_blocks = (int32_t)((P + FGS_PRE_THREADS - 1) / FGS_PRE_THREADS);
    L->sort_passes = (31 + tb + 7) / 8;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t o = off;
        off += (bytes + 255) & ~(uint64_t)255;
        return o;
    };
    const uint64_t cap = (uint64_t)capacity, p = (uint64_t)P;
    const uint64_t sort_tiles = (cap + FGS_SORT_TILE - 1) / FGS_SORT_TILE;
    L->off_stats = take(sizeof(fgs_stats));          // stats and tilecount are contiguous:
    L->off_tilecount = take((uint64_t)L->tiles * 4 * FGS_CTR_STRIDE); // one memset clears both
    L->off_tileorder = take(((uint64_t)FGS_ORDER_HDR + L->tiles) * 4);  // ... and this header
    L->off_cursor = take((uint64_t)L->tiles * 4 * FGS_CTR_STRIDE);
    L->off_ctainfo = take((uint64_t)L->preprocess_blocks * 16 + 16);
    L->off_splat = take(p * 48);
    L->off_depth = take(p * 4);
    L->off_rects = take(p * 8);
    L->off_flags = take(p);
    L->off_counts = take(p * 4);
    L->off_passmask = take(p * 8);
    L->off_blocksums = take((uint64_t)L->preprocess_blocks * 8 + 8);
    L->off_keys[0] = take(cap * 8);
    L->off_keys[1] = take(cap * 8);
    L->off_vals[0] = take(cap * 4);
    L->off_vals[1] = take(cap * 4);
    L->off_sortstate = take(sort_tiles * 256 * 8);
    L->off_hist = take((FGS_SORT_MAXPASS * 256 + FGS_SORT_MAXPASS) * 4);
    L->off_starts = take(((uint64_t)L->tiles + 1) * 4);
    L->off_contrib = take(cap);
    L->off_front = take((uint64_t)L->tiles * 8);
    L->total_bytes = off;
    return fgs_layout_set_sort_mode(L, FGS_SORT_TILE_BUCKET);
}

int fgs_layout_set_sort_mode(fgs_layout *L, int32_t mode)
{
    if (!L || (mode != FGS_SORT_ONESWEEP && mode != FGS_SORT_TILE_BUCKET)) return FGS_E_ARG;
    L->sort_mode = mode;
    if (mode == FGS_SORT_TILE_BUCKET) {
        L->sorted_keys_in = 1;      // k_tile_sort: rec in keys[0] -> keys[1], vals[0]
        L->sorted_vals_in = 0;
    } else {
        L->sorted_keys_in = L->sorted_vals_in = L->sort_passes & 1;
    }
    return FGS_OK;
}

int fgs_workspace_init(void *ws, const fgs_layout *L, void *stream)
{
    if (!ws || !L) return FGS_E_ARG;
    const uint64_t sort_tiles = ((uint64_t)L->capacity + FGS_SORT_TILE - 1) / FGS_SORT_TILE;
    cudaError_t e = cudaMemsetAsync((char *)ws + L->off_sortstate, 0, sort_tiles * 256 * 8,
                                    (cudaStream_t)stream);
    if (e == cudaSuccess)
        e = cudaMemsetAsync((char *)ws + L->off_stats, 0, sizeof(fgs_stats), (cudaStream_t)stream);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    return FGS_OK;
}

int fgs_preprocess(const void *packed, const float *k_cut, int64_t P, const fgs_camera *cam,
                   double tau, int32_t sh_degree, int32_t strategy, int32_t band0, int32_t band1,
                   void *ws, const fgs_layout *L, void *stream)
{
    if (!cam || !ws || P < 0 || !(tau > 0.0)) return FGS_E_ARG;
    int rc = check_frame(L, cam);
    if (rc) return rc;
    if (P != L->gaussians) return FGS_E_WORKSPACE;
    if (P && (!packed || !k_cut)) return FGS_E_ARG;
    if (sh_degree < 0 || sh_degree > 3) return FGS_E_SH_DEGREE;
    if (strategy < 0 || strategy > 2) return FGS_E_STRATEGY;
    return fgs_launch_preprocess(fgs_scene_view(packed, P), k_cut, P, make_cam(cam), tau, sh_degree,
                                 strategy, band0, band1, L->sort_mode == FGS_SORT_TILE_BUCKET,
                                 L->tiles, fgs_frame_view(ws, L), (cudaStream_t)stream);
}

int fgs_row_histogram(const void *packed, int64_t P, const fgs_camera *cam, double tau,
                      uint32_t *rows_out, void *stream)
{
    if (!cam || !rows_out || P < 0 || !(tau > 0.0)) return FGS_E_ARG;
    if (cam->width < FGS_TILE || cam->height < FGS_TILE) return FGS_E_ARG;
    if (P && !packed) return FGS_E_ARG;
    return fgs_launch_row_histogram(fgs_scene_view(packed, P), P, make_cam(cam), tau, rows_out,
                                    (cudaStream_t)stream);
}

int fgs_scan(void *ws, const fgs_layout *L, void *stream)
{
    if (!ws || !L) return FGS_E_ARG;
    if (L->sort_mode == FGS_SORT_TILE_BUCKET)
        return fgs_launch_scan_tiles(fgs_frame_view(ws, L), L->tiles, L->capacity,
                                     (cudaStream_t)stream, fgs_heavy_thr(L));
    return fgs_launch_scan(fgs_frame_view(ws, L), L->preprocess_blocks, L->capacity,
                           (cudaStream_t)stream);
}

int fgs_emit(const void *packed, const fgs_camera *cam, int32_t strategy, int32_t band0,
             int32_t band1, void *ws, const fgs_layout *L, void *stream)
{
    if (!cam || !ws) return FGS_E_ARG;
    int rc = check_frame(L, cam);
    if (rc) return rc;
    if (L->gaussians && !packed) return FGS_E_ARG;
    if (strategy < 0 || strategy > 2) return FGS_E_STRATEGY;
    return fgs_launch_emit(fgs_scene_view(packed, L->gaussians), L->gaussians, make_cam(cam),
                           strategy, band0, band1,
                           L->sort_mode == FGS_SORT_TILE_BUCKET, fgs_frame_view(ws, L),
                           (cudaStream_t)stream, fgs_heavy_thr(L));
}

int fgs_sort(void *ws, const fgs_layout *L, uint32_t epoch, void *stream)
{
    if (!ws || !L || epoch == 0) return FGS_E_ARG;
    FrameDev f = fgs_frame_view(ws, L);
    if (L->sort_mode == FGS_SORT_TILE_BUCKET)
        return fgs_launch_tile_sort(f, L->tiles, L->keep_sorted_keys, fgs_lazy(L), (cudaStream_t)stream);
    const SortPlan plan = fgs_sort_plan(L->tile_bits, 0, 1);
    if (plan.npass != L->sort_passes) return FGS_E_WORKSPACE;
    return fgs_launch_sort(f.keys, f.vals, &f.stats->pairs_in_buffer, L->capacity, plan,
                           f.sortstate, f.hist, f.tickets, epoch, (cudaStream_t)stream);
}

int fgs_ranges(void *ws, const fgs_layout *L, void *stream)
{
    if (!ws || !L) return FGS_E_ARG;
    FrameDev f = fgs_frame_view(ws, L);
    if (L->sort_mode == FGS_SORT_TILE_BUCKET) return FGS_OK;   // k_scan_tiles already wrote it
    return fgs_launch_ranges(f.keys[L->sorted_keys_in], &f.stats->pairs_in_buffer, L->capacity,
                             L->tiles, f.starts, f.stats, (cudaStream_t)stream);
}

int fgs_blend(const void *packed, const float bg[3], double tau, int32_t flags, int32_t band0,
              int32_t band1, float *out_rgb, float *out_alpha, float *out_depth, void *ws,
              const fgs_layout *L, void *stream)
{
    if (!bg || !out_rgb || !ws || !L) return FGS_E_ARG;
    if (band0 < 0 || band1 >= L->grid_h) return FGS_E_ARG;
    if (L->gaussians && !packed) return FGS_E_ARG;
    FrameDev f = fgs_frame_view(ws, L);
    const int lazy = fgs_lazy(L);
    const uint32_t *inv = fgs_scene_view(packed, L->gaussians).inv;
    const uint32_t *order = L->sort_mode == FGS_SORT_TILE_BUCKET ? f.tileorder + FGS_ORDER_HDR : nullptr;
    int rc = fgs_launch_blend(f.splat, f.depth, f.vals[L->sorted_vals_in], inv, f.starts, order,
                              L->width, L->height, bg, tau, flags, band0, band1, out_rgb, out_alpha,
                              out_depth, f.contrib, f.stats, (cudaStream_t)stream,
                              lazy ? f.limit : nullptr, lazy ? f.redo_list : nullptr, 0);
    if (rc || !lazy) return rc;
    // the tiles that had not saturated at the end of their sorted front: full sort, blended again
    if ((rc = fgs_launch_tile_sort_redo(f, L->tiles, (cudaStream_t)stream))) return rc;
    return fgs_launch_blend(f.splat, f.depth, f.vals[L->sorted_vals_in], inv, f.starts, order,
                            L->width, L->height, bg, tau, flags, band0, band1, out_rgb, out_alpha,
                            out_depth, f.contrib, f.stats, (cudaStream_t)stream, nullptr, f.redo_list, 1);
}

int fgs_blend_counts(const void *packed, const float bg[3], double tau, int32_t band0, int32_t band1,
                     float *out_rgb, uint64_t *counts_out, void *ws, const fgs_layout *L, void *stream)
{
    if (!bg || !out_rgb || !counts_out || !ws || !L) return FGS_E_ARG;
    if (band0 < 0 || band1 >= L->grid_h) return FGS_E_ARG;
    if (L->gaussians && !packed) return FGS_E_ARG;
    FrameDev f = fgs_frame_view(ws, L);
    return fgs_launch_blend_counts(f.splat, f.vals[L->sorted_vals_in],
                                   fgs_scene_view(packed, L->gaussians).inv, f.starts, L->width,
                                   L->height, bg, tau, band0, band1, out_rgb, f.stats,
                                   (unsigned long long *)counts_out, (cudaStream_t)stream);
}

int fgs_render(const void *packed, const float *k_cut, int64_t P, const fgs_camera *cam, double tau,
               int32_t sh_degree, int32_t strategy, const float bg[3], int32_t blend_flags,
               int32_t band0, int32_t band1, uint32_t epoch, float *out_rgb, float *out_alpha,
               float *out_depth, void *ws, const fgs_layout *L, void *stream)
{
    int rc = fgs_preprocess(packed, k_cut, P, cam, tau, sh_degree, strategy, band0, band1, ws, L, stream);
    if (rc) return rc;
    if ((rc = fgs_scan(ws, L, stream))) return rc;
    if ((rc = fgs_emit(packed, cam, strategy, band0, band1, ws, L, stream))) return rc;
    if ((rc = fgs_sort(ws, L, epoch, stream))) return rc;
    if ((rc = fgs_ranges(ws, L, stream))) return rc;
    return fgs_blend(packed, bg, tau, blend_flags, band0, band1, out_rgb, out_alpha, out_depth, ws, L,
                     stream);
}

// ---- stand-alone stages ------------------------------------------------------

size_t fgs_sort_pairs_scratch_bytes(int64_t n)
{
    if (n < 0) return 0;
    const uint64_t nn = (uint64_t)n, tiles = (nn + FGS_SORT_TILE - 1) / FGS_SORT_TILE;
    auto al = [](uint64_t b) { return (b + 255) & ~(uint64_t)255; };
    // [n_dev + hist + tickets][state][keys ping][vals ping][keys pong][vals pong]
    return (size_t)(al(256 + (FGS_SORT_MAXPASS * 256 + FGS_SORT_MAXPASS) * 4) + al(tiles * 256 * 8) +
                    2 * al(nn * 8) + 2 * al(nn * 4));
}

int fgs_sort_pairs(const uint64_t *keys_in, const uint32_t *vals_in, int64_t n, int32_t tile_bits,
                   int32_t value_bits, uint64_t *keys_out, uint32_t *vals_out, void *scratch,
                   size_t scratch_bytes, uint32_t epoch, void *stream)
{
    if (n < 0 || tile_bits < 0 || tile_bits > 32 || value_bits < 0 || value_bits > 32 || epoch == 0)
        return FGS_E_ARG;
    if (n > 0x3fffffffll) return FGS_E_SIZE;
    if (n == 0) return FGS_OK;
    if (!keys_in || !vals_in || !keys_out || !vals_out || !scratch) return FGS_E_ARG;
    if (scratch_bytes < fgs_sort_pairs_scratch_bytes(n)) return FGS_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    auto al = [](uint64_t b) { return (b + 255) & ~(uint64_t)255; };
    const uint64_t nn = (uint64_t)n, tiles = (nn + FGS_SORT_TILE - 1) / FGS_SORT_TILE;
    char *b = (char *)scratch;
    uint32_t *n_dev = (uint32_t *)b;
    uint32_t *hist = (uint32_t *)(b + 256);
    uint32_t *tickets = hist + FGS_SORT_MAXPASS * 256;
    b += al(256 + (FGS_SORT_MAXPASS * 256 + FGS_SORT_MAXPASS) * 4);
    uint64_t *state = (uint64_t *)b;
    b += al(tiles * 256 * 8);
    uint64_t *keys[2];
    uint32_t *vals[2];
    keys[0] = (uint64_t *)b; b += al(nn * 8);
    vals[0] = (uint32_t *)b; b += al(nn * 4);
    keys[1] = (uint64_t *)b; b += al(nn * 8);
    vals[1] = (uint32_t *)b;
    const SortPlan plan = fgs_sort_plan(tile_bits, value_bits, 0);
    const uint32_t n32 = (uint32_t)n;
    cudaError_t e = cudaMemsetAsync(scratch, 0, 256 + (FGS_SORT_MAXPASS * 256 + FGS_SORT_MAXPASS) * 4, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(n_dev, &n32, 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(keys[0], keys_in, nn * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(vals[0], vals_in, nn * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    int rc = fgs_launch_sort(keys, vals, n_dev, n, plan, state, hist, tickets, epoch, st);
    if (rc) return rc;
    const int res = plan.npass & 1;
    e = cudaMemcpyAsync(keys_out, keys[res], nn * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(vals_out, vals[res], nn * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    return FGS_OK;
}

int fgs_tile_ranges(const uint64_t *sorted_keys, int64_t n, int32_t tiles, int32_t *starts,
                    fgs_stats *stats, void *stream)
{
    if (n < 0 || tiles < 1 || !starts || !stats || (n && !sorted_keys)) return FGS_E_ARG;
    if (n > 0x3fffffffll) return FGS_E_SIZE;
    cudaStream_t st = (cudaStream_t)stream;
    // stats->pairs_in_buffer doubles as the device-side n
    cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(fgs_stats), st);
    const uint32_t n32 = (uint32_t)n;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&stats->pairs_in_buffer, &n32, 4, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    return fgs_launch_ranges(sorted_keys, &stats->pairs_in_buffer, n, tiles, starts, stats, st);
}

int fgs_blend_tiles(const float *splat, const float *gaussian_depth, const uint32_t *sorted_values,
                    const int32_t *starts, int32_t width, int32_t height, const float bg[3],
                    double tau, int32_t flags, int32_t band0, int32_t band1, float *out_rgb,
                    float *out_alpha, float *out_depth, uint8_t *contrib, fgs_stats *stats,
                    void *stream)
{
    if (!starts || !bg || !out_rgb || width < 1 || height < 1) return FGS_E_ARG;
    if ((flags & FGS_BLEND_CONTRIB) && (!contrib || !stats)) return FGS_E_ARG;
    const int gh = (height + FGS_TILE - 1) / FGS_TILE;
    if (band0 < 0 || band1 >= gh) return FGS_E_ARG;
    return fgs_launch_blend(splat, gaussian_depth, sorted_values, nullptr, starts, nullptr, width, height, bg, tau,
                            flags, band0, band1, out_rgb, out_alpha, out_depth, contrib, stats,
                            (cudaStream_t)stream);
}

int fgs_quantize_rgb8(const float *rgb, int64_t count, uint8_t *out, void *stream)
{
    if (count < 0 || (count && (!rgb || !out))) return FGS_E_ARG;
    if (((uintptr_t)rgb & 15) || ((uintptr_t)out & 3)) return FGS_E_ARG;   // vector accesses
    return fgs_launch_quantize(rgb, count, out, (cudaStream_t)stream);
}

}  // extern "C"
