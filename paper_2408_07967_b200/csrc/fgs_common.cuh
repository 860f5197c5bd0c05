// Shared device/host definitions for the sm_100a rasterizer kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flashgs_b200.h"

#define FGS_WARP 32
#define FGS_FULL 0xffffffffu

// ---- constants.py:4-32, as float32 / float64 literals --------------------
#define FGS_Z_NEAR        0.2f
#define FGS_DILATION      0.3f
#define FGS_MAX_CUTOFF    9.0
#define FGS_ALPHA_CAP     0.99f
#define FGS_T_STOP        1e-4f
#define FGS_CUTOFF_SLACK  1.5e-6f

// ---- launch shapes ---------------------------------------------------------
#define FGS_PRE_THREADS   256      // K1 / K3: one Gaussian per thread
#ifndef FGS_PRE_MINBLOCKS
#define FGS_PRE_MINBLOCKS 4        // K1 resident CTAs per SM the register budget targets (64 registers; 5: 48 + 256 B of spills, slower)
#endif
#define FGS_SORT_THREADS  256
#define FGS_SORT_IPT      16
#define FGS_SORT_TILE     (FGS_SORT_THREADS * FGS_SORT_IPT)   // 4096 pairs per CTA pass
#define FGS_SORT_MAXPASS  16
#define FGS_BLEND_BATCH   256
#ifndef FGS_BLEND_UNROLL
#define FGS_BLEND_UNROLL  8        // survivor loop of the blend: pairs per unrolled block (8: 247 us on C2; 4: 251; 32: 276)
#endif
// per-tile atomic counters sit FGS_CTR_STRIDE words apart (one 32-byte sector each):
// thousands of L2 atomics on neighbouring words of one line serialise
#ifndef FGS_CTR_STRIDE
#define FGS_CTR_STRIDE    8
#endif
// tile-sort size classes: <= SMALL one CTA per tile; <= DENSE the medium list; beyond,
// the dense list.  The lists live in spare words of the cursor slots: dense entry i
// at cursor[i*FGS_CTR_STRIDE + 1], medium entry i at cursor[i*FGS_CTR_STRIDE + 2]
#define FGS_SMALL_TILE    2048
#define FGS_DENSE_TILE    4096      // medium: 2049..4096
#define FGS_LARGE_TILE    8192      // large: 4097..8192; beyond: dense (entry i of the large
                                    // list at cursor[i*FGS_CTR_STRIDE + 4])
// internal work counters live behind the public 80-byte stats block (the block is 256
// bytes in the workspace and zeroed with it at the start of every frame)
#define FGS_WORK_LARGE    0
#define FGS_WORK_MEDIUM_TICKET 2   // (+1: CTAs out) tile tickets of the persistent sort kernels
#define FGS_WORK_LARGE_TICKET  4   // (+1: CTAs out)
#define FGS_WORK_SORT_DONE     6   // bit 0: medium class finished, bit 1: large class, bit 2: small class
#define FGS_WORK_TAIL_OUT      7   // tail-kernel CTAs past their wait on FGS_WORK_SORT_DONE
#define FGS_WORK_STAGE_USED    8   // records the preprocess CTAs have reserved in the stage
#define FGS_WORK_FB_CTAS       9   // preprocess CTAs left to the placement walk (fallback list length)
#define FGS_WORK_DENSE0       10   // dense tiles the tile scan queued (the medium class splits them; later
                                   // entries of the dense list -- tiles a class gave up on -- are the tail's)
#define FGS_WORK_REDO     11   // lazy_sort: cursor of the redo list (tiles unsaturated at the end of their front)
#define FGS_WORK_REDO_OUT 12   // lazy_sort: CTAs of the second blend pass that have left
#define FGS_WORK_SMALL       13   // tiles of the small sort class (1..2048 pairs) the tile scan queued
#define FGS_WORK_SMALL_TICKET 14  // (+1: CTAs out)
#define FGS_CTA_NO_STAGE  0xffffffffu   // ctainfo.w of a CTA whose records were not staged
// blend tile order: tiles are binned by pair count (quarter-octave bins, heaviest = bin 0,
// empty = last) and the blend's CTAs take them in bin order, so the long tiles start first
// and the grid's tail is made of short ones
#define FGS_ORDER_BINS    64
#ifndef FGS_ORDER_MBITS
#define FGS_ORDER_MBITS   2        // mantissa bits of the size bins (2: quarter octaves)
#endif
#define FGS_ORDER_HDR     (2 * FGS_ORDER_BINS + 32)   // bin counts, bin cursors, [128] = CTAs done
static __host__ __device__ inline uint32_t *fgs_work(fgs_stats *s) { return (uint32_t *)(s + 1); }
static __host__ __device__ inline const uint32_t *fgs_work(const fgs_stats *s) { return (const uint32_t *)(s + 1); }

// Camera as the kernels see it (passed by value: lives in the constant bank).
struct CamDev {
    float v[12];          // world_to_camera rows 0..2
    float p0[4], p1[4], p3[4];   // full_projection rows 0, 1, 3
    float pos[3];
    float limx, limy;     // f32(1.3 * tan_fov)   projection.py:100-101
    float fx, fy;         // f32(focal)           projection.py:104-105
    float wf, hf;         // f32(width), f32(height)
    int   width, height, grid_w, grid_h;
};

// Packed device scene: float4 planes of stride `n` (P rounded up to 32), in SLOT order.
//   g0[i] = (mean.xyz, opacity)   g1[i] = (S00, S01, S02, S11)   g2[i] = (S12, S22, 0, 0)
//   with S the 3D covariance R diag(s^2) R^T evaluated once per scene (projection.py:59-85)
//   sh[j*n + i] = floats 4j..4j+3 of slot i's 48 SH coefficients
//   orig[i] = index the caller knows the Gaussian in slot i by;  inv[orig[i]] = i
// Slot order is the caller's order unless fgs_scene_pack was given a permutation (the
// Morton order of fgs_scene_order): neighbouring slots are then neighbours in space, so a
// CTA's Gaussians land on the same few tiles.  Every per-Gaussian frame buffer is indexed
// by slot; pair records carry `orig` (the reference's value and its tie-break), and the
// blend maps them back to slots through `inv` in its index prefetch.
struct SceneDev {
    const float4 *g0, *g1, *g2, *sh;
    const uint32_t *orig, *inv;
    int64_t n;
};

static inline int64_t fgs_pad32(int64_t p) { return (p + 31) & ~(int64_t)31; }

static inline SceneDev fgs_scene_view(const void *packed, int64_t P)
{
    SceneDev s;
    s.n = fgs_pad32(P);
    const float4 *b = (const float4 *)packed;
    s.g0 = b;
    s.g1 = b + s.n;
    s.g2 = b + 2 * s.n;
    s.sh = b + 3 * s.n;
    s.orig = (const uint32_t *)(b + 15 * s.n);
    s.inv = s.orig + s.n;
    return s;
}

// Frame buffers resolved from (workspace, layout).
struct FrameDev {
    float    *splat;
    float    *depth;
    ushort4  *rects;
    uint8_t  *flags;
    uint32_t *counts;
    uint64_t *passmask;     // [P]
    uint32_t *blocksums;    // [nblocks]
    uint32_t *blockbase;    // [nblocks]
    uint64_t *keys[2];
    uint32_t *vals[2];
    uint64_t *sortstate;
    uint32_t *hist;         // [FGS_SORT_MAXPASS][256]
    uint32_t *tickets;      // [FGS_SORT_MAXPASS]
    int32_t  *starts;
    uint8_t  *contrib;
    fgs_stats *stats;
    uint32_t *tilecount;    // [tiles]
    uint32_t *cursor;       // [tiles]
    uint4    *tablelist;    // TILE_BUCKET: (tile, range base, pairs, slot | record offset) per
                            // (CTA, tile); aliases vals[0] + vals[1] (8 B x capacity)
    uint64_t *stage;        // TILE_BUCKET: every preprocess CTA's records, grouped by table
                            // entry, between fgs_preprocess and fgs_emit; aliases keys[1]
    uint32_t *fb_list;      // TILE_BUCKET: preprocess CTAs left to the placement walk; aliases
                            // blockbase (ONESWEEP's scan output)
    uint4    *ctainfo;      // [preprocess blocks] (list base, entries, records, stage base or
                            // FGS_CTA_NO_STAGE)
    uint32_t *tileorder;    // [FGS_ORDER_HDR + tiles]: bin counts, bin cursors, blend tile order
    int32_t  *limit;        // [tiles] lazy_sort: sorted pairs at the head of each tile's bucket
    uint32_t *redo_list;    // [tiles] lazy_sort: tiles to sort in full and blend again
    uint32_t list_capacity;
};

static inline FrameDev fgs_frame_view(void *ws, const fgs_layout *L)
{
    char *b = (char *)ws;
    FrameDev f;
    f.splat = (float *)(b + L->off_splat);
    f.depth = (float *)(b + L->off_depth);
    f.rects = (ushort4 *)(b + L->off_rects);
    f.flags = (uint8_t *)(b + L->off_flags);
    f.counts = (uint32_t *)(b + L->off_counts);
    f.passmask = (uint64_t *)(b + L->off_passmask);
    f.blocksums = (uint32_t *)(b + L->off_blocksums);
    f.blockbase = f.blocksums + L->preprocess_blocks;
    f.keys[0] = (uint64_t *)(b + L->off_keys[0]);
    f.keys[1] = (uint64_t *)(b + L->off_keys[1]);
    f.vals[0] = (uint32_t *)(b + L->off_vals[0]);
    f.vals[1] = (uint32_t *)(b + L->off_vals[1]);
    f.sortstate = (uint64_t *)(b + L->off_sortstate);
    f.hist = (uint32_t *)(b + L->off_hist);
    f.tickets = f.hist + FGS_SORT_MAXPASS * 256;
    f.starts = (int32_t *)(b + L->off_starts);
    f.contrib = (uint8_t *)(b + L->off_contrib);
    f.stats = (fgs_stats *)(b + L->off_stats);
    f.tilecount = (uint32_t *)(b + L->off_tilecount);
    f.cursor = (uint32_t *)(b + L->off_cursor);
    f.tablelist = (uint4 *)(b + L->off_vals[0]);
    f.stage = f.keys[1];
    f.fb_list = f.blockbase;
    f.ctainfo = (uint4 *)(b + L->off_ctainfo);
    f.tileorder = (uint32_t *)(b + L->off_tileorder);
    f.limit = (int32_t *)(b + L->off_front);
    f.redo_list = (uint32_t *)(b + L->off_front) + L->tiles;
    f.list_capacity = (uint32_t)(L->capacity / 2);          // 16-byte entries in 8 B x capacity
    return f;
}

// Internal launchers (one translation unit per stage).
int  fgs_launch_pack(const float *means, const float *opac, const float *scales,
                     const float *rots, const float *sh, const uint32_t *order, int64_t P,
                     void *packed, cudaStream_t st);
int  fgs_launch_morton_keys(const float *means, int64_t P, float *bbox6, uint64_t *keys,
                            uint32_t *vals, cudaStream_t st);
int  fgs_launch_row_histogram(const SceneDev &sc, int64_t P, const CamDev &cam, double tau,
                              uint32_t *hist, cudaStream_t st);
int  fgs_launch_unpack_ply(const float *payload, int64_t P, float *means, float *sh, float *logit,
                           float *logs, float *rots, cudaStream_t st);
int  fgs_launch_activate(const float *logit, const float *log_scales, const float *rots, int64_t P,
                         float *opac, float *scales, float *unit, cudaStream_t st);
int  fgs_launch_cutoffs(const SceneDev &sc, int64_t P, double tau, float *k, cudaStream_t st);
int  fgs_launch_preprocess(const SceneDev &sc, const float *kcut, int64_t P, const CamDev &cam,
                           double tau, int sh_degree, int strategy, int band0, int band1,
                           int bucket, int tiles, const FrameDev &f, cudaStream_t st);
int  fgs_launch_scan(const FrameDev &f, int nblocks, int64_t capacity, cudaStream_t st);
int  fgs_launch_scan_tiles(const FrameDev &f, int tiles, int64_t capacity, cudaStream_t st,
                           uint32_t heavy_thr = 0);
int  fgs_launch_tile_order(const FrameDev &f, int grid_w, int band0, int band1, cudaStream_t st,
                           uint32_t heavy_thr = 0);
int  fgs_launch_emit(const SceneDev &sc, int64_t P, const CamDev &cam, int strategy, int band0,
                     int band1, int bucket, const FrameDev &f, cudaStream_t st, uint32_t heavy_thr = 0);
int  fgs_launch_tile_sort(const FrameDev &f, int tiles, int write_keys, int lazy, cudaStream_t st);
int  fgs_launch_tile_sort_redo(const FrameDev &f, int tiles, cudaStream_t st);
// (lazy: 0 off; 1 = tiles beyond FGS_DENSE_TILE pairs get a front only; 2 = beyond FGS_SMALL_TILE)

struct SortPlan {
    int npass;
    int on_value[FGS_SORT_MAXPASS];
    int shift[FGS_SORT_MAXPASS];
    int bits[FGS_SORT_MAXPASS];
    int compact;      // digits taken from ((key >> 32) << 31) | (key & 0x7fffffff)
};
SortPlan fgs_sort_plan(int tile_bits, int value_bits, int compact);
int  fgs_launch_sort(uint64_t *keys[2], uint32_t *vals[2], const uint32_t *n_dev, int64_t n_max,
                     const SortPlan &plan, uint64_t *state, uint32_t *hist, uint32_t *tickets,
                     uint32_t epoch, cudaStream_t st);
int  fgs_launch_ranges(const uint64_t *keys, const uint32_t *n_dev, int64_t n_max, int tiles,
                       int32_t *starts, fgs_stats *stats, cudaStream_t st);
// `limit` / `redo_list` (lazy_sort, both or neither): pairs sorted at the head of each tile;
// a tile unsaturated at the end of its front is appended to redo_list (cursor:
// stats->redo_tiles) and left unwritten.  `redo` = the second pass: the tiles of redo_list,
// in full, by persistent CTAs.
int  fgs_launch_blend(const float *splat, const float *gdepth, const uint32_t *vals,
                      const uint32_t *inv, const int32_t *starts, const uint32_t *order,
                      int width, int height,
                      const float bg[3],
                      double tau, int flags, int band0, int band1, float *rgb, float *alpha,
                      float *depth, uint8_t *contrib, fgs_stats *stats, cudaStream_t st,
                      const int32_t *limit = nullptr, uint32_t *redo_list = nullptr, int redo = 0);

int  fgs_launch_blend_counts(const float *splat, const uint32_t *vals, const uint32_t *inv,
                             const int32_t *starts, int width, int height, const float bg[3],
                             double tau, int band0, int band1, float *rgb, fgs_stats *stats,
                             unsigned long long *evals, cudaStream_t st);
int  fgs_launch_quantize(const float *rgb, int64_t count, uint8_t *out, cudaStream_t st);

void fgs_set_cuda_error(cudaError_t e);

// cudaFuncSetAttribute is per device: one flag per (call site, device), so a process that
// renders on several devices (one Pipeline per device) sets the attributes on each of them.
// Racing threads may both set them (idempotent).
struct FgsOncePerDevice {
    unsigned long long done = 0ull;
    __host__ bool need(int *dev_out)
    {
        int d = 0;
        cudaGetDevice(&d);
        *dev_out = d & 63;
        return !((__atomic_load_n(&done, __ATOMIC_ACQUIRE) >> (d & 63)) & 1ull);
    }
    __host__ void mark(int dev) { __atomic_fetch_or(&done, 1ull << dev, __ATOMIC_RELEASE); }
};
// Records the next caller-supplied profiling event on `st` (no-op unless
// fgs_profile_begin armed this thread).  Called after every kernel launch.
void fgs_prof_mark(cudaStream_t st);
bool fgs_prof_armed();

#define FGS_CHECK_LAUNCH()                                   \
    do {                                                     \
        cudaError_t e__ = cudaGetLastError();                \
        if (e__ != cudaSuccess) {                            \
            fgs_set_cuda_error(e__);                         \
            return FGS_E_CUDA;                               \
        }                                                    \
    } while (0)

// launch check + profiling mark, for the per-frame kernels
#define FGS_AFTER_LAUNCH(st) \
    do {                     \
        FGS_CHECK_LAUNCH();  \
        fgs_prof_mark(st);   \
    } while (0)

#ifdef __CUDACC__
// ---- programmatic dependent launch (PDL) -------------------------------------------------
// The kernels of a frame form a chain on one stream.  A kernel launched with programmatic
// stream serialization may be scheduled while its predecessor is still draining; it calls
// fgs_pdl_wait() before it touches global memory (blocks until the predecessor has completed
// and its writes are visible) and then fgs_pdl_trigger(), which lets ITS successor be
// scheduled the same way.  Wait-then-trigger keeps the chain transitive: when a kernel's wait
// returns, every earlier kernel of the frame has completed.  What is gained is the launch
// latency and the drain/fill bubble at every kernel boundary.  Both instructions are no-ops
// in a kernel launched the plain way (profiling passes launch everything the plain way).
__device__ __forceinline__ void fgs_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void fgs_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t fgs_launch_chain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                           cudaStream_t st, bool pdl, Args... args)
{
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}
#define FGS_CHAIN(kernel, grid, block, smem, st, ...)                                              \
    do {                                                                                           \
        const cudaError_t e__ = fgs_launch_chain(kernel, grid, block, smem, st, !fgs_prof_armed(), \
                                                 __VA_ARGS__);                                     \
        if (e__ != cudaSuccess) { fgs_set_cuda_error(e__); return FGS_E_CUDA; }                    \
    } while (0)

// Individually rounded float32 / float64 arithmetic: these intrinsics are never
// contracted into FMAs, which is what keeps the geometry bit-identical to the
// reference's NumPy ufunc chains.
__device__ __forceinline__ float  fm(float a, float b)   { return __fmul_rn(a, b); }
__device__ __forceinline__ float  fa(float a, float b)   { return __fadd_rn(a, b); }
__device__ __forceinline__ float  fs(float a, float b)   { return __fsub_rn(a, b); }
__device__ __forceinline__ float  fd(float a, float b)   { return __fdiv_rn(a, b); }
__device__ __forceinline__ float  fsq(float a)           { return __fsqrt_rn(a); }
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// size bin of a tile with v pairs: quarter-octave bins, heaviest first, empty last
// lazy_sort: the blend composites at most the sorted front of a heavy tile and usually stops
// after a few hundred pairs (the tile is opaque), so for its place in the blend order a tile
// beyond `heavy_thr` pairs weighs what it is expected to consume, not its pair count (0 = no
// threshold); a tile below the threshold may need all of its pairs and goes first.  Measured
// (blend, us): weight 1152 / 768 / 640 / 512 / 448 / 320 -> C2 170 / 157 / 151 / 144 / 144 / 148,
// 1M dense scene 211 / 198 / 190 / 185 / 183 / -, C5 217 at every weight (267 by pair count),
// no change where the blend is throughput-bound (10M / 4K, C3, 8K).
#ifndef FGS_FRONT_WEIGHT
#define FGS_FRONT_WEIGHT 448u
#endif
__device__ __forceinline__ uint32_t fgs_order_weight(uint32_t v, uint32_t heavy_thr)
{
    return (heavy_thr && v > heavy_thr) ? FGS_FRONT_WEIGHT : v;
}

__device__ __forceinline__ int fgs_order_bin(uint32_t v)
{
    if (v == 0) return FGS_ORDER_BINS - 1;
    int lb;
    if (v < 4) lb = (int)v;
    else {
        const int e = 31 - __clz(v);
        lb = e * 4 + (int)((v >> (e - 2)) & (3u & ~((1u << (2 - FGS_ORDER_MBITS)) - 1u))) - 4;   // v = 4 -> 4
    }
    lb = lb > FGS_ORDER_BINS - 2 ? FGS_ORDER_BINS - 2 : lb;
    return FGS_ORDER_BINS - 2 - lb;
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(FGS_FULL, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive scan over the 256 threads of a CTA; also returns the CTA total.
// `scratch` is 8 uint32 in shared memory.  Contains two barriers.
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t *scratch,
                                                        uint32_t &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(v, lane);
    if (lane == 31) scratch[w] = incl;
    __syncthreads();
    uint32_t wsum = lane < 8 ? scratch[lane] : 0u;
    uint32_t wincl = warp_incl_scan(wsum, lane);
    uint32_t wbase = __shfl_sync(FGS_FULL, wincl - wsum, w);
    total = __shfl_sync(FGS_FULL, wincl, 7);
    __syncthreads();
    return wbase + incl - v;
}
// The same for a 64-bit value (two packed counters share one pair of barriers).
// `scratch` is 8 uint64 in shared memory.
__device__ __forceinline__ unsigned long long block_excl_scan64_256(unsigned long long v,
                                                                    unsigned long long *scratch,
                                                                    unsigned long long &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(FGS_FULL, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) scratch[w] = incl;
    __syncthreads();
    unsigned long long wsum = lane < 8 ? scratch[lane] : 0ull, wincl = wsum;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(FGS_FULL, wincl, o);
        if (lane >= o) wincl += t;
    }
    const unsigned long long wbase = __shfl_sync(FGS_FULL, wincl - wsum, w);
    total = __shfl_sync(FGS_FULL, wincl, 7);
    __syncthreads();
    return wbase + incl - v;
}
#endif
