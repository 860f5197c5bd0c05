// K1 preprocess+count, K2 scan, K3 emit  (plus the per-scene pack / cutoff kernels).
//
// Replaces the reference's NumPy preprocessing and binning:
//   projection.py:19-47,59-121,139-171   extent.py:19-30,39-85
//   binning.py:176-194 (_candidate_rects), 217-249 (phase A), 259-354 (phase B)
//   intersect.py:25-43,63-94              render.py:52-86 (eval_sh_color)
//
// Numerics: every float32 / float64 operation is an explicitly rounded
// intrinsic in the reference's operation order, so the emitted pair list is
// bit-identical to the reference's (keys embed float32 depth bits and the pair
// set depends on float32 centres / conics / extents).  This file is also
// compiled with -fmad=false.
//
// Scheduling: one Gaussian per thread for the per-Gaussian math; the
// per-candidate-tile exact tests of a warp's 32 Gaussians are flattened into
// one work list and walked 32 candidates at a time, so a Gaussian covering 50
// tiles does not stall 31 lanes that cover one (the paper's "adaptive
// size-aware scheduling", generalised).  Emission is count -> scan -> emit:
// pairs land in ascending Gaussian order, which lets a stable sort on the key
// alone reproduce the reference's (key, value) order.

#include "fgs_common.cuh"

// ---------------------------------------------------------------------------
// per-scene kernels
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_scene_pack(const float *__restrict__ means, const float *__restrict__ opac,
             const float *__restrict__ scales, const float *__restrict__ rots,
             const float *__restrict__ sh, int64_t P, int64_t n, float4 *__restrict__ out)
{
    // One warp stages 32 Gaussians' 48 SH floats through shared memory so both
    // the AoS read and the plane-major write are coalesced.
    __shared__ float s_sh[4][32 * 48];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t g0 = ((int64_t)blockIdx.x * 4 + w) * 32;
    if (g0 >= n) return;
    const int64_t g = g0 + lane;
    const bool live = g < P;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = make_float4(1.f, 0.f, 0.f, 0.f);
    if (live) {
        a = make_float4(means[3 * g], means[3 * g + 1], means[3 * g + 2], opac[g]);
        b = make_float4(scales[3 * g], scales[3 * g + 1], scales[3 * g + 2], 0.f);
        c = make_float4(rots[4 * g], rots[4 * g + 1], rots[4 * g + 2], rots[4 * g + 3]);
    }
    out[g] = a;
    out[n + g] = b;
    out[2 * n + g] = c;
    const int64_t nlive = P - g0 < 32 ? P - g0 : 32;       // may be <= 0
    for (int i = lane; i < 32 * 48; i += 32)
        s_sh[w][i] = (i < nlive * 48) ? sh[g0 * 48 + i] : 0.f;
    __syncwarp();
    float4 *plane = out + 3 * n;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
        const float *r = &s_sh[w][lane * 48 + 4 * j];
        plane[(int64_t)j * n + g] = make_float4(r[0], r[1], r[2], r[3]);
    }
}

int fgs_launch_pack(const float *means, const float *opac, const float *scales,
                    const float *rots, const float *sh, int64_t P, void *packed, cudaStream_t st)
{
    const int64_t n = fgs_pad32(P);
    if (n == 0) return FGS_OK;
    const int64_t blocks = (n / 32 + 3) / 4;
    k_scene_pack<<<(unsigned)blocks, 128, 0, st>>>(means, opac, scales, rots, sh, P, n,
                                                   (float4 *)packed);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// extent.py:19-30
__global__ void __launch_bounds__(256)
k_power_cutoffs(const float4 *__restrict__ g0, int64_t P, double tau, float tau32,
                float *__restrict__ k_out)
{
    const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (g >= P) return;
    const float op = g0[g].w;
    const double safe = op > tau32 ? (double)op : 1.0;
    double k = dm(2.0, log(safe / tau));
    k_out[g] = (float)fmin(k, FGS_MAX_CUTOFF);
}

int fgs_launch_cutoffs(const SceneDev &sc, int64_t P, double tau, float *k, cudaStream_t st)
{
    if (P == 0) return FGS_OK;
    k_power_cutoffs<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(sc.g0, P, tau, (float)tau, k);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// ---------------------------------------------------------------------------
// exact ellipse / tile-rectangle test  (intersect.py:25-43, 63-94), float64
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool chord_hits(double A, double B, double C, double lo, double hi)
{
    const double delta = ds(dm(B, B), dm(dm(4.0, A), C));
    if (!(delta >= 0.0)) return false;
    const double twoA = dm(2.0, A);
    const double e1 = da(dm(twoA, lo), B);
    const double e2 = da(dm(twoA, hi), B);
    return ((e1 <= 0.0) || (dm(e1, e1) <= delta)) && ((e2 >= 0.0) || (dm(e2, e2) <= delta));
}

// Candidate tile (tx, ty) against the cutoff ellipse; rectangle clipped to the
// image as in binning.py:279-283.
__device__ __forceinline__ bool tile_hits(int tx, int ty, int width, int height, float cxf,
                                          float cyf, float af, float bf, float cf, float kf)
{
    const double x0 = (double)(tx * FGS_TILE), y0 = (double)(ty * FGS_TILE);
    const double x1 = fmin(x0 + FGS_TILE, (double)width);
    const double y1 = fmin(y0 + FGS_TILE, (double)height);
    const double cx = cxf, cy = cyf, a = af, b = bf, c = cf, k = kf;
    const double u0 = ds(x0, cx), u1 = ds(x1, cx), v0 = ds(y0, cy), v1 = ds(y1, cy);
    if ((u0 <= 0.0) && (u1 >= 0.0) && (v0 <= 0.0) && (v1 >= 0.0)) return true;
    const double b2 = dm(2.0, b);
    if (chord_hits(a, dm(b2, v0), ds(dm(dm(c, v0), v0), k), u0, u1)) return true;
    if (chord_hits(a, dm(b2, v1), ds(dm(dm(c, v1), v1), k), u0, u1)) return true;
    if (chord_hits(c, dm(b2, u0), ds(dm(dm(a, u0), u0), k), v0, v1)) return true;
    return chord_hits(c, dm(b2, u1), ds(dm(dm(a, u1), u1), k), v0, v1);
}

// float32 screening of the same predicate.  intersect.py:63-94 is true exactly when the
// cutoff ellipse a u^2 + 2 b u v + c v^2 <= k meets the (closed) tile rectangle, i.e. when
// the minimum of that convex form over the rectangle is <= k.  The minimum is 0 if the
// centre is inside; otherwise it lies on an edge the centre is outside of, where the form is
// a 1-D parabola.  Returns 1 (hit) or 0 (miss) when the float32 minimum is clear of k by
// more than 1e-4 of the largest term magnitude in the tile (1000x the rounding of this
// evaluation; the float64 reference is far more accurate still), and 2 when it is not --
// the caller then runs the float64 predicate, so the verdict is always the reference's.
__device__ __forceinline__ int tile_hits32(int tx, int ty, int width, int height, float cx,
                                           float cy, float a, float b, float c, float k)
{
    const float x0 = (float)(tx * FGS_TILE), y0 = (float)(ty * FGS_TILE);
    const float x1 = fminf(x0 + (float)FGS_TILE, (float)width);
    const float y1 = fminf(y0 + (float)FGS_TILE, (float)height);
    const float u0 = x0 - cx, u1 = x1 - cx, v0 = y0 - cy, v1 = y1 - cy;   // signs are exact
    const bool out_u = !(u0 <= 0.0f && u1 >= 0.0f), out_v = !(v0 <= 0.0f && v1 >= 0.0f);
    if (!out_u && !out_v) return 1;                       // intersect.py:84-86 centre in tile
    const float ue = u0 > 0.0f ? u0 : u1;                 // the edge facing the centre
    const float ve = v0 > 0.0f ? v0 : v1;
    float qmin = __int_as_float(0x7f800000);
    if (out_u) {                                          // edge u = ue, v in [v0, v1]
        const float bu = b * ue;
        const float vs = fminf(fmaxf(__fdividef(-bu, c), v0), v1);
        qmin = a * ue * ue + (c * vs * vs + 2.0f * bu * vs);
    }
    if (out_v) {                                          // edge v = ve, u in [u0, u1]
        const float bv = b * ve;
        const float us = fminf(fmaxf(__fdividef(-bv, a), u0), u1);
        qmin = fminf(qmin, c * ve * ve + (a * us * us + 2.0f * bv * us));
    }
    const float um = fmaxf(fabsf(u0), fabsf(u1)), vm = fmaxf(fabsf(v0), fabsf(v1));
    const float tol = 1e-4f * (fabsf(a) * um * um + fabsf(c) * vm * vm + 2.0f * fabsf(b) * um * vm
                               + fabsf(k));
    if (qmin < k - tol) return 1;
    if (qmin > k + tol) return 0;
    return 2;                                             // too close (or not finite): ask float64
}

// What a lane contributes to its warp's flattened candidate list.
struct TileJob {
    uint32_t cand;              // candidate tiles (0 = lane idle)
    float cx, cy, a, b, c, keff;
    int tx0, ty0, nx;
    uint64_t mask;              // K3: pass bits recorded by K1 (cand <= FGS_MASK_CAND)
};
#define FGS_MASK_CAND 64

// Walk the warp's candidate tiles 32 at a time.  Returns this lane's number of
// passing tiles.  MODE selects what happens to a passing (tile, Gaussian):
//   WALK_COUNT   nothing (count only)                                  (ONESWEEP, K1)
//   WALK_STAGE   take the pair's rank inside its tile from the tile's counter and
//                park (tile, rank, depth bits, index) in the stage     (TILE_BUCKET, K1)
//   WALK_EMIT    write (key, value) at out_base(owner) + rank          (ONESWEEP, K3)
// TILE_BUCKET: the counter's old value IS the pair's slot inside its bucket, so the
// histogram pass hands every pair its final position relative to the bucket start and K3
// is a plain placement (no second walk, no second round of atomics).  The atomic's return
// trip is hidden by parking each window's records in registers until the next window's
// tests are done.
enum { WALK_COUNT = 0, WALK_STAGE = 1, WALK_EMIT = 2 };

// Where WALK_STAGE parks its records: a chunk of `total candidates` records per warp,
// reserved with one atomic on stats->stage_used (passing pairs are packed at its front).
struct StageOut {
    uint4 *stage;               // (tile, rank in tile, depth bits, Gaussian index)
    uint32_t *tile_ctr;         // per-tile counters, FGS_CTR_STRIDE words apart
    fgs_stats *stats;
    uint32_t capacity;          // records the stage can hold
};

// The count walks (K1) also return, in `mask_out`, the pass bits of this lane's first 64
// candidates; the emit walks (K3) take them back through job.mask and only re-run the
// exact test for the rare Gaussian with more candidates than that.
template <bool PRECISE, int MODE>
__device__ __forceinline__ uint32_t warp_walk_tiles(const TileJob &job, int width, int height,
                                                    int grid_w, uint32_t out_base,
                                                    uint32_t depth_bits, uint32_t gid,
                                                    uint64_t *__restrict__ keys,
                                                    uint32_t *__restrict__ vals,
                                                    const StageOut *so = nullptr,
                                                    uint64_t *mask_out = nullptr)
{
    constexpr bool COUNTING = (MODE == WALK_COUNT || MODE == WALK_STAGE);
    const int lane = threadIdx.x & 31;
    const uint32_t incl = warp_incl_scan(job.cand, lane);
    const uint32_t total = __shfl_sync(FGS_FULL, incl, 31);
    const uint32_t excl = incl - job.cand;
    uint32_t mine = 0;
    uint64_t mymask = 0;
    // K3: does any lane of this warp need the exact test again?
    const bool any_big = !COUNTING && PRECISE && __any_sync(FGS_FULL, job.cand > FGS_MASK_CAND);
    // WALK_STAGE: the warp's chunk of the stage (lane 0 holds the raw reservation; it is
    // only broadcast when the first records are flushed, one window later)
    uint32_t chunk_raw = 0, staged = 0;
    bool pend = false;
    uint32_t pend_pos = 0, pend_tile = 0, pend_rank = 0, pend_bits = 0, pend_gid = 0;
    if (MODE == WALK_STAGE && lane == 0 && total)
        chunk_raw = atomicAdd(&so->stats->stage_used, total);
    // unrolled by two so a parked rank needs no register move right behind its atomic
    // (a move would wait for the return trip on the spot)
#pragma unroll 2
    for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t j = base + lane;
        // owner = first lane whose inclusive prefix exceeds j
        int o = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t v = __shfl_sync(FGS_FULL, incl, o + step - 1);
            if (v <= j) o += step;
        }
        const bool act = j < total;
        o = o > 31 ? 31 : o;
        const uint32_t excl_o = __shfl_sync(FGS_FULL, excl, o);
        const int tx0 = __shfl_sync(FGS_FULL, job.tx0, o);
        const int ty0 = __shfl_sync(FGS_FULL, job.ty0, o);
        const int nx = __shfl_sync(FGS_FULL, job.nx, o);
        const uint32_t local = act ? j - excl_o : 0u;
        const int ry = (int)(local / (uint32_t)(nx > 0 ? nx : 1));
        const int tx = tx0 + (int)local - ry * nx, ty = ty0 + ry;
        bool pass = act;
        if (PRECISE && !COUNTING) {
            // recorded bits of the owner (valid when it has <= 64 candidates)
            const uint32_t mlo = __shfl_sync(FGS_FULL, (uint32_t)job.mask, o);
            const uint32_t mhi = __shfl_sync(FGS_FULL, (uint32_t)(job.mask >> 32), o);
            const uint32_t word = local < 32u ? mlo : mhi;
            pass = act && ((word >> (local & 31u)) & 1u);
        }
        if (PRECISE && (COUNTING || any_big)) {
            const float cx = __shfl_sync(FGS_FULL, job.cx, o);
            const float cy = __shfl_sync(FGS_FULL, job.cy, o);
            const float a = __shfl_sync(FGS_FULL, job.a, o);
            const float b = __shfl_sync(FGS_FULL, job.b, o);
            const float c = __shfl_sync(FGS_FULL, job.c, o);
            const float ke = __shfl_sync(FGS_FULL, job.keff, o);
            if (COUNTING) {
                const int h = act ? tile_hits32(tx, ty, width, height, cx, cy, a, b, c, ke) : 0;
                pass = h == 1;
                if (h == 2) pass = tile_hits(tx, ty, width, height, cx, cy, a, b, c, ke);
            } else {
                const uint32_t cand_o = __shfl_sync(FGS_FULL, job.cand, o);
                if (cand_o > FGS_MASK_CAND)
                    pass = act && tile_hits(tx, ty, width, height, cx, cy, a, b, c, ke);
            }
        }
        const uint32_t ballot = __ballot_sync(FGS_FULL, pass);
        if (MODE == WALK_EMIT) {
            const uint32_t run_o = __shfl_sync(FGS_FULL, mine, o);
            const uint32_t base_o = __shfl_sync(FGS_FULL, out_base, o);
            const uint32_t bits_o = __shfl_sync(FGS_FULL, depth_bits, o);
            const uint32_t gid_o = __shfl_sync(FGS_FULL, gid, o);
            if (pass) {
                const int lo_o = excl_o > base ? (int)(excl_o - base) : 0;
                const uint32_t before = ballot & lanemask_lt() & ~((1u << lo_o) - 1u);
                const uint32_t slot = base_o + run_o + __popc(before);
                keys[slot] = ((uint64_t)(uint32_t)(ty * grid_w + tx) << 32) | bits_o;
                vals[slot] = gid_o;
            }
        }
        if (MODE == WALK_STAGE) {
            const uint32_t bits_o = __shfl_sync(FGS_FULL, depth_bits, o);
            const uint32_t gid_o = __shfl_sync(FGS_FULL, gid, o);
            const uint32_t tile = (uint32_t)(ty * grid_w + tx);
            uint32_t rank = 0;
            if (pass) rank = atomicAdd(&so->tile_ctr[(size_t)tile * FGS_CTR_STRIDE], 1u);
            // flush the previous window: its ranks have had a whole window to come back
            if (__any_sync(FGS_FULL, pend)) {
                const uint32_t cb = __shfl_sync(FGS_FULL, chunk_raw, 0);
                if (pend && cb + total <= so->capacity)
                    so->stage[cb + pend_pos] = make_uint4(pend_tile, pend_rank, pend_bits, pend_gid);
            }
            pend = pass;
            pend_pos = staged + __popc(ballot & lanemask_lt());
            pend_tile = tile;
            pend_rank = rank;
            pend_bits = bits_o;
            pend_gid = gid_o;
            staged += __popc(ballot);
        }
        // owner side: how many of my candidates in this window passed
        const int lo = excl > base ? (int)(excl - base) : 0;
        const int hi = incl - base < 32u ? (int)(incl - base) : 32;
        if (job.cand && incl > base && lo < hi) {
            const uint32_t m = (hi - lo == 32) ? FGS_FULL : (((1u << (hi - lo)) - 1u) << lo);
            mine += __popc(ballot & m);
            if (MODE == WALK_COUNT) {
                // my candidates in this window start at my local index base + lo - excl
                const uint32_t first = base + (uint32_t)lo - excl;
                if (first < 64u) mymask |= (uint64_t)((ballot & m) >> lo) << first;
            }
        }
    }
    if (MODE == WALK_STAGE && total) {
        const uint32_t cb = __shfl_sync(FGS_FULL, chunk_raw, 0);
        const bool fits = cb + total <= so->capacity;
        if (fits) {
            if (pend)
                so->stage[cb + pend_pos] = make_uint4(pend_tile, pend_rank, pend_bits, pend_gid);
            // the chunk was reserved by candidates: mark what the rejected ones left unused,
            // so the placement kernel can run flat over [0, stage_used)
            for (uint32_t i = staged + lane; i < total; i += 32) so->stage[cb + i].x = 0xffffffffu;
        } else if (lane == 0) {
            so->stats->overflow = 1u;                          // grow and re-run
        }
    }
    if (MODE == WALK_COUNT && mask_out) *mask_out = mymask;
    return mine;
}

// ---------------------------------------------------------------------------
// SH colour, render.py:52-86, for one channel triple
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sh_basis(float x, float y, float z, float *bz)
{
    const float C1 = 0.4886025119029199f;
    const float C2_0 = 1.0925484305920792f, C2_2 = 0.31539156525252005f,
                C2_4 = 0.5462742152960396f;
    const float C3_0 = -0.5900435899266435f, C3_1 = 2.890611442640554f,
                C3_2 = -0.4570457994644658f, C3_3 = 0.3731763325901154f,
                C3_5 = 1.445305721320277f;
    const float xx = fm(x, x), yy = fm(y, y), zz = fm(z, z);
    const float xy = fm(x, y), yz = fm(y, z), xz = fm(x, z);
    bz[1] = fm(C1, y);
    bz[2] = fm(C1, z);
    bz[3] = fm(C1, x);
    bz[4] = fm(C2_0, xy);
    bz[5] = fm(-C2_0, yz);
    bz[6] = fm(C2_2, fs(fs(fm(2.0f, zz), xx), yy));
    bz[7] = fm(-C2_0, xz);
    bz[8] = fm(C2_4, fs(xx, yy));
    bz[9] = fm(fm(C3_0, y), fs(fm(3.0f, xx), yy));
    bz[10] = fm(fm(C3_1, xy), z);
    bz[11] = fm(fm(C3_2, y), fs(fs(fm(4.0f, zz), xx), yy));
    bz[12] = fm(fm(C3_3, z), fs(fs(fm(2.0f, zz), fm(3.0f, xx)), fm(3.0f, yy)));
    bz[13] = fm(fm(C3_2, x), fs(fs(fm(4.0f, zz), xx), yy));
    bz[14] = fm(fm(C3_5, z), fs(xx, yy));
    bz[15] = fm(fm(C3_0, x), fs(xx, fm(3.0f, yy)));
}

// ---------------------------------------------------------------------------
// K1: preprocess + count
// ---------------------------------------------------------------------------
template <int STRAT, bool BUCKET>
__global__ void __launch_bounds__(FGS_PRE_THREADS, FGS_PRE_MINBLOCKS)
k_preprocess(SceneDev sc, const float *__restrict__ kcut, int P,
             const __grid_constant__ CamDev cam, float tau32, float frustum_thresh,
             int sh_degree, int band0, int band1, FrameDev f)
{
    __shared__ uint32_t s_red[8];
    const int g = blockIdx.x * FGS_PRE_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool live = g < P;

    TileJob job;
    job.cand = 0;
    job.cx = job.cy = job.a = job.b = job.c = job.keff = 0.f;
    job.tx0 = job.ty0 = 0;
    job.nx = 1;
    job.mask = 0;
    bool retained = false, degenerate = false;
    uint32_t full_cand = 0;
    float zcam = 0.0f;

    if (live) {
        const float4 m = sc.g0[g];
        const float x = m.x, y = m.y, z = m.z, op = m.w;
        // projection.py:19-26 view_points
        const float t0 = fa(fa(fa(fm(cam.v[0], x), fm(cam.v[1], y)), fm(cam.v[2], z)), cam.v[3]);
        const float t1 = fa(fa(fa(fm(cam.v[4], x), fm(cam.v[5], y)), fm(cam.v[6], z)), cam.v[7]);
        const float t2 = fa(fa(fa(fm(cam.v[8], x), fm(cam.v[9], y)), fm(cam.v[10], z)), cam.v[11]);
        f.depth[g] = t2;
        zcam = t2;
        ushort4 rect = make_ushort4(0, 0, 0, 0);
        // projection.py:39-47 frustum_mask
        if ((t2 > FGS_Z_NEAR) && (op > frustum_thresh)) {
            const float4 sc4 = sc.g1[g];
            const float4 q = sc.g2[g];
            const float k = kcut[g];
            // projection.py:59-76 quat_to_rotmat (w, x, y, z)
            const float qw = q.x, qx = q.y, qy = q.z, qz = q.w;
            float R[3][3];
            R[0][0] = fs(1.0f, fm(2.0f, fa(fm(qy, qy), fm(qz, qz))));
            R[0][1] = fm(2.0f, fs(fm(qx, qy), fm(qw, qz)));
            R[0][2] = fm(2.0f, fa(fm(qx, qz), fm(qw, qy)));
            R[1][0] = fm(2.0f, fa(fm(qx, qy), fm(qw, qz)));
            R[1][1] = fs(1.0f, fm(2.0f, fa(fm(qx, qx), fm(qz, qz))));
            R[1][2] = fm(2.0f, fs(fm(qy, qz), fm(qw, qx)));
            R[2][0] = fm(2.0f, fs(fm(qx, qz), fm(qw, qy)));
            R[2][1] = fm(2.0f, fa(fm(qy, qz), fm(qw, qx)));
            R[2][2] = fs(1.0f, fm(2.0f, fa(fm(qx, qx), fm(qy, qy))));
            // projection.py:79-85 compute_cov3d: M = R diag(s), S = M M^T
            const float s3[3] = {sc4.x, sc4.y, sc4.z};
            float M[3][3], S[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) M[i][j] = fm(R[i][j], s3[j]);
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int kx = 0; kx < 3; ++kx)
                    S[i][kx] = fa(fa(fm(M[i][0], M[kx][0]), fm(M[i][1], M[kx][1])),
                                  fm(M[i][2], M[kx][2]));
            // projection.py:88-121 compute_cov2d
            const float tz = t2 > 1e-3f ? t2 : 1e-3f;
            const float rx = fd(t0, tz), ry = fd(t1, tz);
            const float cxn = fminf(fmaxf(rx, -cam.limx), cam.limx);
            const float cyn = fminf(fmaxf(ry, -cam.limy), cam.limy);
            const float txc = fm(cxn, tz), tyc = fm(cyn, tz);
            const float inv_z = fd(1.0f, tz);
            const float inv_z2 = fm(inv_z, inv_z);
            const float J[2][3] = {{fm(cam.fx, inv_z), 0.0f, fm(-fm(cam.fx, txc), inv_z2)},
                                   {0.0f, fm(cam.fy, inv_z), fm(-fm(cam.fy, tyc), inv_z2)}};
            float T[2][3], M2[2][3];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int kx = 0; kx < 3; ++kx)
                    T[i][kx] = fa(fa(fm(J[i][0], cam.v[kx]), fm(J[i][1], cam.v[4 + kx])),
                                  fm(J[i][2], cam.v[8 + kx]));
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int kx = 0; kx < 3; ++kx)
                    M2[i][kx] = fa(fa(fm(T[i][0], S[0][kx]), fm(T[i][1], S[1][kx])),
                                   fm(T[i][2], S[2][kx]));
            const float c00 = fa(fa(fm(M2[0][0], T[0][0]), fm(M2[0][1], T[0][1])), fm(M2[0][2], T[0][2]));
            const float c01 = fa(fa(fm(M2[0][0], T[1][0]), fm(M2[0][1], T[1][1])), fm(M2[0][2], T[1][2]));
            const float c11 = fa(fa(fm(M2[1][0], T[1][0]), fm(M2[1][1], T[1][1])), fm(M2[1][2], T[1][2]));
            const float cxx = fa(c00, FGS_DILATION), cxy = c01, cyy = fa(c11, FGS_DILATION);
            // projection.py:139-155 conic_from_cov2d
            const float det = fs(fm(cxx, cyy), fm(cxy, cxy));
            const bool valid = det > 0.0f;
            const float inv = fd(1.0f, valid ? det : 1.0f);
            const float ca = fm(cyy, inv), cb = fm(-cxy, inv), cc = fm(cxx, inv);
            // projection.py:29-36 project_points, 158-171 ndc2pix
            const float h0 = fa(fa(fa(fm(cam.p0[0], x), fm(cam.p0[1], y)), fm(cam.p0[2], z)), cam.p0[3]);
            const float h1 = fa(fa(fa(fm(cam.p1[0], x), fm(cam.p1[1], y)), fm(cam.p1[2], z)), cam.p1[3]);
            const float h3 = fa(fa(fa(fm(cam.p3[0], x), fm(cam.p3[1], y)), fm(cam.p3[2], z)), cam.p3[3]);
            const float den = fabsf(h3) > 1e-7f ? h3 : 1e-7f;
            const float px = fm(fs(fm(fa(fd(h0, den), 1.0f), cam.wf), 1.0f), 0.5f);
            const float py = fm(fs(fm(fa(fd(h1, den), 1.0f), cam.hf), 1.0f), 0.5f);
            // binning.py:176-194 _candidate_rects
            const float hx = fsq(fmaxf(fm(k, cxx), 0.0f));
            const float hy = fsq(fmaxf(fm(k, cyy), 0.0f));
            float xmin, ymin, xmax, ymax;
            if (STRAT == FGS_BASELINE_CIRCLE_AABB) {
                // projection.py:124-136 eigenvalues_2x2 (float64), extent.py:55-66
                const double A = cxx, B = cxy, Cc = cyy;
                const double mid = dm(0.5, da(A, Cc));
                const double dd = ds(dm(A, Cc), dm(B, B));
                const double disc = __dsqrt_rn(fmax(ds(dm(mid, mid), dd), 0.0));
                const float lam1 = (float)da(mid, disc);
                const float r = ceilf(fm(3.0f, fsq(fmaxf(lam1, 0.0f))));
                xmin = fs(px, r); ymin = fs(py, r); xmax = fa(px, r); ymax = fa(py, r);
            } else {
                // extent.py:39-52 tight_aabb
                const float thx = fsq(fm(k, cxx)), thy = fsq(fm(k, cyy));
                xmin = fs(px, thx); ymin = fs(py, thy); xmax = fa(px, thx); ymax = fa(py, thy);
            }
            const float ex = fa(hx, 16.0f), ey = fa(hy, 16.0f);
            const float term = fa(fa(fm(fm(ca, ex), ex), fm(fm(fm(2.0f, fabsf(cb)), ex), ey)),
                                  fm(fm(cc, ey), ey));
            const float keff = fa(k, fm(FGS_CUTOFF_SLACK, term));
            // extent.py:69-85 tile_ranges: x/16 is exact in float32
            const float ftx0 = floorf(fm(xmin, 0.0625f)), fty0 = floorf(fm(ymin, 0.0625f));
            const float ftx1 = floorf(fm(xmax, 0.0625f)), fty1 = floorf(fm(ymax, 0.0625f));
            const float gwm = (float)(cam.grid_w - 1), ghm = (float)(cam.grid_h - 1);
            const bool nonempty = (ftx1 >= 0.0f) && (fty1 >= 0.0f) && (ftx0 <= gwm) && (fty0 <= ghm);
            degenerate = !valid;
            retained = valid && (op > tau32) && nonempty;
            if (retained) {
                const int tx0 = (int)fminf(fmaxf(ftx0, 0.0f), gwm);
                const int ty0 = (int)fminf(fmaxf(fty0, 0.0f), ghm);
                const int tx1 = (int)fminf(fmaxf(ftx1, 0.0f), gwm);
                const int ty1 = (int)fminf(fmaxf(fty1, 0.0f), ghm);
                rect = make_ushort4((unsigned short)tx0, (unsigned short)ty0,
                                    (unsigned short)tx1, (unsigned short)ty1);
                full_cand = (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1);
                const int by0 = ty0 > band0 ? ty0 : band0;
                const int by1 = ty1 < band1 ? ty1 : band1;
                if (by0 <= by1) {
                    job.cand = (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(by1 - by0 + 1);
                    job.cx = px; job.cy = py; job.a = ca; job.b = cb; job.c = cc;
                    job.keff = keff;
                    job.tx0 = tx0; job.ty0 = by0; job.nx = tx1 - tx0 + 1;
                }
                // binning.py:230-233 view direction, render.py:52-86 colour
                const float d0 = fs(x, cam.pos[0]), d1 = fs(y, cam.pos[1]), d2 = fs(z, cam.pos[2]);
                float nrm = fsq(fa(fa(fm(d0, d0), fm(d1, d1)), fm(d2, d2)));
                nrm = nrm > 0.0f ? nrm : 1.0f;
                float bz[16];
                sh_basis(fd(d0, nrm), fd(d1, nrm), fd(d2, nrm), bz);
                // 48 coefficients as 12 coalesced float4 loads: c[3*i + ch]
                float cf[48];
#pragma unroll
                for (int j = 0; j < 12; ++j) {
                    const float4 v = sc.sh[(int64_t)j * sc.n + g];
                    cf[4 * j] = v.x; cf[4 * j + 1] = v.y; cf[4 * j + 2] = v.z; cf[4 * j + 3] = v.w;
                }
                float rgb[3];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    float res = fm(0.28209479177387814f, cf[ch]);
                    if (sh_degree >= 1)
                        res = fs(fa(fs(res, fm(bz[1], cf[3 + ch])), fm(bz[2], cf[6 + ch])),
                                 fm(bz[3], cf[9 + ch]));
                    if (sh_degree >= 2) {
#pragma unroll
                        for (int i = 4; i < 9; ++i) res = fa(res, fm(bz[i], cf[3 * i + ch]));
                    }
                    if (sh_degree >= 3) {
#pragma unroll
                        for (int i = 9; i < 16; ++i) res = fa(res, fm(bz[i], cf[3 * i + ch]));
                    }
                    rgb[ch] = fmaxf(fa(res, 0.5f), 0.0f);
                }
                // render.py:34-40 splat row, binning.py:235-241
                float4 *row = (float4 *)(f.splat + (size_t)g * 12);
                row[0] = make_float4(px, py, ca, cb);
                row[1] = make_float4(cc, op, k, rgb[0]);
                row[2] = make_float4(rgb[1], rgb[2], hx, hy);
            }
        }
        f.rects[g] = rect;
        f.flags[g] = (uint8_t)((retained ? 1 : 0) | (degenerate ? 2 : 0));
    }

    uint32_t npairs;
    uint64_t passmask = 0;
    if (BUCKET) {
        const StageOut so{f.stage, f.tilecount, f.stats, f.stage_capacity};
        const float d = zcam;
        npairs = warp_walk_tiles<STRAT == FGS_PRECISE, WALK_STAGE>(
            job, cam.width, cam.height, cam.grid_w, 0, __float_as_uint(d), (uint32_t)g, nullptr,
            nullptr, &so);
        // binning.py:50-51: depths of emitted pairs must be positive and finite
        if (npairs && !(d < __int_as_float(0x7f800000))) f.stats->bad_depth = 1u;
    } else if (STRAT == FGS_PRECISE)
        npairs = warp_walk_tiles<true, WALK_COUNT>(job, cam.width, cam.height, cam.grid_w, 0, 0, 0,
                                                   nullptr, nullptr, nullptr, &passmask);
    else
        npairs = job.cand;
    if (live) {
        f.counts[g] = npairs;
        if (!BUCKET && STRAT == FGS_PRECISE && npairs) f.passmask[g] = passmask;
    }

    // block totals: pairs (-> blocksums), retained / degenerate / candidates (-> stats)
    uint32_t v0 = npairs, v1 = (retained ? 1u : 0u) | ((degenerate ? 1u : 0u) << 16), v2 = full_cand;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        v0 += __shfl_xor_sync(FGS_FULL, v0, o);
        v1 += __shfl_xor_sync(FGS_FULL, v1, o);
        v2 += __shfl_xor_sync(FGS_FULL, v2, o);
    }
    if (lane == 0) {
        s_red[threadIdx.x >> 5] = v0;
        if (v1 & 0xffffu) atomicAdd(&f.stats->gaussians_retained, v1 & 0xffffu);
        if (v1 >> 16) atomicAdd(&f.stats->gaussians_degenerate, v1 >> 16);
        if (v2) atomicAdd((unsigned long long *)&f.stats->candidate_tiles_lo, (unsigned long long)v2);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += s_red[i];
        f.blocksums[blockIdx.x] = t;
    }
}

static CamDev g_dummy_cam;   // keeps CamDev's layout in one place for sizeof checks
static_assert(sizeof(CamDev) % 4 == 0, "CamDev must be word-sized");

int fgs_launch_preprocess(const SceneDev &sc, const float *kcut, int64_t P, const CamDev &cam,
                          double tau, int sh_degree, int strategy, int band0, int band1,
                          int bucket, int tiles, const FrameDev &f, cudaStream_t st)
{
    (void)g_dummy_cam;
    // stats and (TILE_BUCKET) the per-tile histogram sit back to back: one memset
    const size_t zero_bytes = bucket ? (size_t)((char *)(f.tilecount + (size_t)tiles * FGS_CTR_STRIDE) - (char *)f.stats)
                                     : sizeof(fgs_stats);
    cudaError_t e = cudaMemsetAsync(f.stats, 0, zero_bytes, st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    if (P == 0) return FGS_OK;
    const double th = tau > 1.0 / 255.0 ? tau : 1.0 / 255.0;       // projection.py:46
    const unsigned blocks = (unsigned)((P + FGS_PRE_THREADS - 1) / FGS_PRE_THREADS);
    const float tau32 = (float)tau, fth = (float)th;
#define FGS_K1(S, B) k_preprocess<S, B><<<blocks, FGS_PRE_THREADS, 0, st>>>( \
        sc, kcut, (int)P, cam, tau32, fth, sh_degree, band0, band1, f)
    switch (strategy) {
    case FGS_PRECISE:
        if (bucket) FGS_K1(FGS_PRECISE, true); else FGS_K1(FGS_PRECISE, false);
        break;
    case FGS_TIGHT_AABB:
        if (bucket) FGS_K1(FGS_TIGHT_AABB, true); else FGS_K1(FGS_TIGHT_AABB, false);
        break;
    case FGS_BASELINE_CIRCLE_AABB:
        if (bucket) FGS_K1(FGS_BASELINE_CIRCLE_AABB, true); else FGS_K1(FGS_BASELINE_CIRCLE_AABB, false);
        break;
    default:
        return FGS_E_STRATEGY;
    }
#undef FGS_K1
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

// ---------------------------------------------------------------------------
// K2: exclusive scan of the per-block pair counts (one CTA; the table has
// P/256 entries).  Also fixes M, the overflow flag, and zeroes the sort
// histograms / tickets for this frame.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
k_scan_blocks(const uint32_t *__restrict__ sums, uint32_t *__restrict__ bases, int nblocks,
              unsigned long long capacity, uint32_t *__restrict__ hist_and_tickets,
              fgs_stats *__restrict__ stats)
{
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < FGS_SORT_MAXPASS * 256 + FGS_SORT_MAXPASS; i += 1024)
        hist_and_tickets[i] = 0u;
    if (threadIdx.x == 0) s_carry = 0ull;
    __syncthreads();
    for (int base = 0; base < nblocks; base += 1024) {
        const int i = base + threadIdx.x;
        const unsigned long long v = i < nblocks ? sums[i] : 0u;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(FGS_FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_w[w] = incl;
        __syncthreads();
        if (w == 0) {
            const unsigned long long ws = s_w[lane];
            unsigned long long wi = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(FGS_FULL, wi, o);
                if (lane >= o) wi += t;
            }
            s_w[lane] = wi - ws;
        }
        __syncthreads();
        const unsigned long long excl = s_carry + s_w[w] + incl - v;
        // offsets only matter when M fits; clamp so a 32-bit store never wraps silently
        if (i < nblocks) bases[i] = excl > 0xffffffffull ? 0xffffffffu : (uint32_t)excl;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const unsigned long long M = s_carry;
        const bool over = M > capacity;
        stats->pairs_emitted = M > 0xffffffffull ? 0xffffffffu : (uint32_t)M;
        stats->overflow = over ? 1u : 0u;
        stats->pairs_in_buffer = over ? 0u : (uint32_t)M;
    }
}

int fgs_launch_scan(const FrameDev &f, int nblocks, int64_t capacity, cudaStream_t st)
{
    k_scan_blocks<<<1, 1024, 0, st>>>(f.blocksums, f.blockbase, nblocks,
                                      (unsigned long long)capacity, f.hist, f.stats);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

// K2 (TILE_BUCKET): exclusive scan of the per-tile histogram.  The result IS the
// range table (sorting.py:139-152): starts[t] .. starts[t+1] is tile t's bucket.
// Also queues the tiles by size class, fixes M / overflow and counts non-empty tiles.
// One CTA per 1024 tiles; instead of a second kernel or a spin-wait, CTA b sums
// the (L2-resident) counts of all tiles before its own -- O(T^2/1024) reads, at
// most 33 MB for an 8K frame's 129600 tiles, and no inter-CTA dependency at all.
__global__ void __launch_bounds__(1024)
k_scan_tiles(const uint32_t *__restrict__ counts, int32_t *__restrict__ starts,
             uint32_t *__restrict__ cursor, int tiles, unsigned long long capacity,
             fgs_stats *__restrict__ stats)
{
    __shared__ unsigned long long s_w[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int first = blockIdx.x * 1024;
    // prefix of everything before this CTA's slice
    unsigned long long before = 0;
    for (int i = threadIdx.x; i < first; i += 1024) before += counts[(size_t)i * FGS_CTR_STRIDE];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) before += __shfl_xor_sync(FGS_FULL, before, o);
    if (lane == 0) s_w[w] = before;
    __syncthreads();
    unsigned long long carry = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) carry += s_w[i];
    __syncthreads();

    const int i = first + threadIdx.x;
    const unsigned long long v = i < tiles ? counts[(size_t)i * FGS_CTR_STRIDE] : 0u;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(FGS_FULL, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
        const unsigned long long ws = s_w[lane];
        unsigned long long wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(FGS_FULL, wi, o);
            if (lane >= o) wi += t;
        }
        s_w[lane] = wi - ws;
    }
    __syncthreads();
    const unsigned long long excl = carry + s_w[w] + incl - v;
    if (i < tiles) {
        const uint32_t e32 = excl > 0x7fffffffull ? 0x7fffffffu : (uint32_t)excl;
        starts[i] = (int32_t)e32;
        if (v > FGS_DENSE_TILE)     // queue the bucket for its tile-sort size class
            cursor[(size_t)atomicAdd(&stats->dense_tiles, 1u) * FGS_CTR_STRIDE + 1] = (uint32_t)i;
        else if (v > FGS_SMALL_TILE)
            cursor[(size_t)atomicAdd(&stats->medium_tiles, 1u) * FGS_CTR_STRIDE + 2] = (uint32_t)i;
    }
    const uint32_t nonempty = __reduce_add_sync(FGS_FULL, v ? 1u : 0u);
    if (lane == 0 && nonempty) atomicAdd(&stats->tiles_nonempty, nonempty);
    if (i == tiles - 1) {                       // the thread that owns the last tile knows M
        const unsigned long long M = excl + v;
        // K1 has already raised the flag if some warp's chunk did not fit the stage
        const bool over = M > capacity || stats->overflow != 0u;
        stats->pairs_emitted = M > 0xffffffffull ? 0xffffffffu : (uint32_t)M;
        stats->overflow = over ? 1u : 0u;       // later kernels of this frame see it and no-op
        stats->pairs_in_buffer = over ? 0u : (uint32_t)M;
        starts[tiles] = (int32_t)(M > 0x7fffffffull ? 0x7fffffffu : (uint32_t)M);
    }
}

int fgs_launch_scan_tiles(const FrameDev &f, int tiles, int64_t capacity, cudaStream_t st)
{
    k_scan_tiles<<<(unsigned)((tiles + 1023) / 1024), 1024, 0, st>>>(
        f.tilecount, f.starts, f.cursor, tiles, (unsigned long long)capacity, f.stats);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

// ---------------------------------------------------------------------------
// K3 (ONESWEEP): emit (key, value) pairs at the scanned offsets
// ---------------------------------------------------------------------------
template <int STRAT>
__global__ void __launch_bounds__(FGS_PRE_THREADS)
k_emit(int P, int width, int height, int grid_w, int band0, int band1, FrameDev f)
{
    __shared__ uint32_t s_scan[8];
    if (f.stats->overflow) return;                       // uniform: grow and re-run
    const int g = blockIdx.x * FGS_PRE_THREADS + threadIdx.x;
    const bool live = g < P;
    const uint32_t cnt = live ? f.counts[g] : 0u;
    uint32_t total;
    const uint32_t off = f.blockbase[blockIdx.x] + block_excl_scan_256(cnt, s_scan, total);
    if (total == 0) return;                              // uniform per block

    TileJob job;
    job.cand = 0;
    job.cx = job.cy = job.a = job.b = job.c = job.keff = 0.f;
    job.tx0 = job.ty0 = 0;
    job.nx = 1;
    job.mask = 0;
    uint32_t bits = 0;
    if (cnt) {
        const ushort4 r = f.rects[g];
        const int by0 = (int)r.y > band0 ? (int)r.y : band0;
        const int by1 = (int)r.w < band1 ? (int)r.w : band1;
        job.tx0 = r.x; job.ty0 = by0; job.nx = (int)r.z - (int)r.x + 1;
        job.cand = (uint32_t)job.nx * (uint32_t)(by1 - by0 + 1);
        if (STRAT == FGS_PRECISE) {
            if (job.cand <= FGS_MASK_CAND) {
                job.mask = f.passmask[g];                 // K1's verdicts, no test needed
            } else {
                const float4 *row = (const float4 *)(f.splat + (size_t)g * 12);
                const float4 r0 = row[0], r1 = row[1], r2 = row[2];
                const float k = r1.z, hx = r2.z, hy = r2.w;
                // binning.py:187-193 conservative cutoff for the exact test
                const float ex = fa(hx, 16.0f), ey = fa(hy, 16.0f);
                const float term = fa(fa(fm(fm(r0.z, ex), ex), fm(fm(fm(2.0f, fabsf(r0.w)), ex), ey)),
                                      fm(fm(r1.x, ey), ey));
                job.keff = fa(k, fm(FGS_CUTOFF_SLACK, term));
                job.cx = r0.x; job.cy = r0.y; job.a = r0.z; job.b = r0.w; job.c = r1.x;
            }
        }
        const float d = f.depth[g];
        bits = __float_as_uint(d);
        // binning.py:50-51: depths must be positive and finite
        if (!(d > 0.0f) || !(d < __int_as_float(0x7f800000))) f.stats->bad_depth = 1u;
    }
    warp_walk_tiles<STRAT == FGS_PRECISE, WALK_EMIT>(job, width, height, grid_w, off, bits,
                                                     (uint32_t)g, f.keys[0], f.vals[0]);
}

// ---------------------------------------------------------------------------
// K3 (TILE_BUCKET): place the staged pairs.  K1 parked (tile, rank, depth bits, index)
// per pair; the scan has since fixed every bucket's start, so a record goes to
// starts[tile] + rank.  Flat over the reserved part of the stage (unused slots carry
// tile = ~0), coalesced 16-byte reads, four records in flight per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_place(const uint4 *__restrict__ stage, const int32_t *__restrict__ starts,
        uint64_t *__restrict__ rec, const fgs_stats *__restrict__ stats)
{
    if (stats->overflow) return;                         // uniform: grow and re-run
    const uint32_t n = stats->stage_used;
    const uint32_t stride = gridDim.x * 256u;
    for (uint32_t i0 = blockIdx.x * 256u + threadIdx.x; i0 < n; i0 += 4u * stride) {
        uint4 r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = i0 + (uint32_t)k * stride;
            r[k] = i < n ? stage[i] : make_uint4(0xffffffffu, 0u, 0u, 0u);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (r[k].x != 0xffffffffu)
                rec[(uint32_t)starts[r[k].x] + r[k].y] = ((uint64_t)r[k].z << 32) | r[k].w;
    }
}

int fgs_launch_emit(int64_t P, const CamDev &cam, int strategy, int band0, int band1,
                    int bucket, const FrameDev &f, cudaStream_t st)
{
    if (P == 0) return FGS_OK;
    const unsigned blocks = (unsigned)((P + FGS_PRE_THREADS - 1) / FGS_PRE_THREADS);
    if (bucket) {
        // sized from the capacity (the record count lives on the device)
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t want = (f.stage_capacity + 1023) / 1024;
        const unsigned grid = (unsigned)(want < 1 ? 1 : (want > sms * 8 ? sms * 8 : want));
        k_place<<<grid, 256, 0, st>>>(f.stage, f.starts, f.keys[0], f.stats);
    } else if (strategy == FGS_PRECISE) {
        k_emit<FGS_PRECISE><<<blocks, FGS_PRE_THREADS, 0, st>>>(
            (int)P, cam.width, cam.height, cam.grid_w, band0, band1, f);
    } else {
        k_emit<FGS_TIGHT_AABB><<<blocks, FGS_PRE_THREADS, 0, st>>>(
            (int)P, cam.width, cam.height, cam.grid_w, band0, band1, f);
    }
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}
