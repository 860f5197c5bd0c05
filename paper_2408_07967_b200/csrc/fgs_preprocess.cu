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
#include <type_traits>

// ---------------------------------------------------------------------------
// per-scene kernels
// ---------------------------------------------------------------------------
// projection.py:59-76 quat_to_rotmat (w, x, y, z), 79-85 compute_cov3d: M = R diag(s),
// S = M M^T as left-to-right 3-term sums of individually rounded products.  S is bitwise
// symmetric (the products commute), so the six entries S00 S01 S02 S11 S12 S22 carry it.
__device__ __forceinline__ void fgs_cov3d(float sx, float sy, float sz, float qw, float qx,
                                          float qy, float qz, float *S6)
{
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
    const float s3[3] = {sx, sy, sz};
    float M[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[i][j] = fm(R[i][j], s3[j]);
    const int ii[6] = {0, 0, 0, 1, 1, 2}, kk[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e)
        S6[e] = fa(fa(fm(M[ii[e]][0], M[kk[e]][0]), fm(M[ii[e]][1], M[kk[e]][1])),
                   fm(M[ii[e]][2], M[kk[e]][2]));
}

__global__ void __launch_bounds__(128)
k_scene_pack(const float *__restrict__ means, const float *__restrict__ opac,
             const float *__restrict__ scales, const float *__restrict__ rots,
             const float *__restrict__ sh, const uint32_t *__restrict__ order, int64_t P,
             int64_t n, float4 *__restrict__ out)
{
    // One warp stages 32 Gaussians' 48 SH floats through shared memory so both
    // the AoS read and the plane-major write are coalesced.  Slot g holds the
    // caller's Gaussian order[g] (identity without an order).
    __shared__ float s_sh[4][32 * 48];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t g0 = ((int64_t)blockIdx.x * 4 + w) * 32;
    if (g0 >= n) return;
    const int64_t g = g0 + lane;
    const bool live = g < P;
    const int64_t src = live ? (order ? (int64_t)order[g] : g) : 0;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a;
    if (live) {
        a = make_float4(means[3 * src], means[3 * src + 1], means[3 * src + 2], opac[src]);
        // The 3D covariance is camera-independent (projection.py:59-85), so it is evaluated
        // once per scene, here, with the reference's individually rounded operations; K1
        // reads its six distinct entries instead of scale + quaternion (same 32 bytes).
        float S[6];
        fgs_cov3d(scales[3 * src], scales[3 * src + 1], scales[3 * src + 2], rots[4 * src],
                  rots[4 * src + 1], rots[4 * src + 2], rots[4 * src + 3], S);
        b = make_float4(S[0], S[1], S[2], S[3]);       // S00 S01 S02 S11
        c = make_float4(S[4], S[5], 0.f, 0.f);         // S12 S22
    }
    out[g] = a;
    out[n + g] = b;
    out[2 * n + g] = c;
    uint32_t *orig = (uint32_t *)(out + 15 * n), *inv = orig + n;
    orig[g] = live ? (uint32_t)src : 0xffffffffu;
    if (live) inv[src] = (uint32_t)g;     // `order` is a permutation: every index written once
    else inv[g] = 0xffffffffu;            // pad entries (g >= P is never a caller index)
    const int nlive = P - g0 < 32 ? (int)(P - g0) : 32;       // may be <= 0
    for (int k = 0; k < 32; ++k) {
        const int64_t srck = __shfl_sync(FGS_FULL, src, k);
        const bool lk = k < nlive;
        s_sh[w][k * 48 + lane] = lk ? sh[srck * 48 + lane] : 0.f;
        if (lane < 16) s_sh[w][k * 48 + 32 + lane] = lk ? sh[srck * 48 + 32 + lane] : 0.f;
    }
    __syncwarp();
    float4 *plane = out + 3 * n;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
        const float *r = &s_sh[w][lane * 48 + 4 * j];
        plane[(int64_t)j * n + g] = make_float4(r[0], r[1], r[2], r[3]);
    }
}

int fgs_launch_pack(const float *means, const float *opac, const float *scales,
                    const float *rots, const float *sh, const uint32_t *order, int64_t P,
                    void *packed, cudaStream_t st)
{
    const int64_t n = fgs_pad32(P);
    if (n == 0) return FGS_OK;
    const int64_t blocks = (n / 32 + 3) / 4;
    k_scene_pack<<<(unsigned)blocks, 128, 0, st>>>(means, opac, scales, rots, sh, order, P, n,
                                                   (float4 *)packed);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// ---- spatial order of a scene (per scene, untimed): 63-bit Morton codes of the means over
// their bounding box; the caller sorts (code, index) with the library's own radix sort.
__device__ __forceinline__ uint32_t f2ord(float f)
{
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);      // order-preserving float -> uint
}
__device__ __forceinline__ float ord2f(uint32_t u)
{
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void __launch_bounds__(256)
k_bbox(const float *__restrict__ means, int64_t P, uint32_t *__restrict__ box)
{
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x; g < P; g += (int64_t)gridDim.x * 256)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float v = means[3 * g + a];
            if (fabsf(v) <= 3.0e38f) {                       // skip NaN / inf
                const uint32_t o = f2ord(v);
                lo[a] = o < lo[a] ? o : lo[a];
                hi[a] = o > hi[a] ? o : hi[a];
            }
        }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(FGS_FULL, lo[a]);
        hi[a] = __reduce_max_sync(FGS_FULL, hi[a]);
    }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&box[a], lo[a]);
            atomicMax(&box[3 + a], hi[a]);
        }
}

__device__ __forceinline__ uint64_t spread21(uint32_t v)
{
    uint64_t x = v & 0x1fffffu;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

__global__ void __launch_bounds__(256)
k_morton_keys(const float *__restrict__ means, int64_t P, const uint32_t *__restrict__ box,
              uint64_t *__restrict__ keys, uint32_t *__restrict__ vals)
{
    const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (g >= P) return;
    uint32_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float lo = ord2f(box[a]), hi = ord2f(box[3 + a]);
        const float v = means[3 * g + a];
        float t = (hi > lo) ? fd(fs(v, lo), fs(hi, lo)) : 0.0f;
        t = (t >= 0.0f) ? t : 0.0f;                          // NaN -> 0
        t = t > 1.0f ? 1.0f : t;
        q[a] = (uint32_t)fm(t, 2097151.0f);
    }
    keys[g] = spread21(q[0]) | (spread21(q[1]) << 1) | (spread21(q[2]) << 2);
    vals[g] = (uint32_t)g;
}

int fgs_launch_morton_keys(const float *means, int64_t P, float *bbox6, uint64_t *keys,
                           uint32_t *vals, cudaStream_t st)
{
    if (P == 0) return FGS_OK;
    uint32_t *box = (uint32_t *)bbox6;
    cudaError_t e = cudaMemsetAsync(box, 0xff, 3 * sizeof(uint32_t), st);      // minima
    if (e == cudaSuccess) e = cudaMemsetAsync(box + 3, 0, 3 * sizeof(uint32_t), st);   // maxima
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    const int64_t want = (P + 255) / 256;
    k_bbox<<<(unsigned)(want > 1184 ? 1184 : want), 256, 0, st>>>(means, P, box);
    FGS_CHECK_LAUNCH();
    k_morton_keys<<<(unsigned)want, 256, 0, st>>>(means, P, box, keys, vals);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// model_io.py:93-118 activate
__global__ void __launch_bounds__(256)
k_activate(const float *__restrict__ logit, const float *__restrict__ log_scales,
           const float *__restrict__ rots, int64_t P, float *__restrict__ opac,
           float *__restrict__ scales, float *__restrict__ unit)
{
    const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (g >= P) return;
    // sign-split sigmoid: exp never overflows (model_io.py:101-105)
    const float x = logit[g];
    const bool nonneg = x >= 0.0f;
    const float t = (float)exp((double)(nonneg ? -x : x));
    const float denom = fa(1.0f, t);
    opac[g] = nonneg ? fd(1.0f, denom) : fd(t, denom);
#pragma unroll
    for (int a = 0; a < 3; ++a) scales[3 * g + a] = (float)exp((double)log_scales[3 * g + a]);
    const float4 q = reinterpret_cast<const float4 *>(rots)[g];
    const float nrm = fsq(fa(fa(fa(fm(q.x, q.x), fm(q.y, q.y)), fm(q.z, q.z)), fm(q.w, q.w)));
    reinterpret_cast<float4 *>(unit)[g] =
        nrm > 0.0f ? make_float4(fd(q.x, nrm), fd(q.y, nrm), fd(q.z, nrm), fd(q.w, nrm))
                   : make_float4(1.0f, 0.0f, 0.0f, 0.0f);
}

int fgs_launch_activate(const float *logit, const float *log_scales, const float *rots, int64_t P,
                        float *opac, float *scales, float *unit, cudaStream_t st)
{
    if (P == 0) return FGS_OK;
    k_activate<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(logit, log_scales, rots, P, opac, scales,
                                                            unit);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// model_io.py:167-199 (load_ply's payload split, _scene_from_payload) on the device: the
// PLY body is an array of 62-float vertex records (x y z, nx ny nz, f_dc_0..2, f_rest_0..44
// channel-major, opacity, scale_0..2, rot_0..3).  A CTA stages 128 records in shared memory
// with coalesced loads and writes the reference's arrays -- means (P,3), sh (P,16,3) with RGB
// innermost, logit opacities (P,), log scales (P,3), rotations (P,4) -- with coalesced
// stores.  Pure data movement (values bit-identical to the host loader's); normals are
// parsed and dropped as in the reference.  HBM-bound: 248 B read + 236 B written per vertex.
#define FGS_PLY_FLOATS 62
#define FGS_PLY_CHUNK  128
__global__ void __launch_bounds__(256)
k_unpack_ply(const float *__restrict__ payload, int64_t P, float *__restrict__ means,
             float *__restrict__ sh, float *__restrict__ logit, float *__restrict__ logs,
             float *__restrict__ rots)
{
    __shared__ float s[FGS_PLY_CHUNK * FGS_PLY_FLOATS];
    const int64_t v0 = (int64_t)blockIdx.x * FGS_PLY_CHUNK;
    const int nv = (int)(P - v0 < FGS_PLY_CHUNK ? P - v0 : FGS_PLY_CHUNK);
    const float *src = payload + v0 * FGS_PLY_FLOATS;
    for (int i = threadIdx.x; i < nv * FGS_PLY_FLOATS; i += 256) s[i] = src[i];
    __syncthreads();
    // record stride 62 is even: lanes reading consecutive vertices hit 2-way bank conflicts
    // at worst, which a bandwidth-bound copy does not notice
    for (int i = threadIdx.x; i < nv * 3; i += 256) {
        const int v = i / 3, c = i - v * 3;
        means[v0 * 3 + i] = s[v * FGS_PLY_FLOATS + c];
        logs[v0 * 3 + i] = s[v * FGS_PLY_FLOATS + 55 + c];
    }
    for (int i = threadIdx.x; i < nv; i += 256) logit[v0 + i] = s[i * FGS_PLY_FLOATS + 54];
    for (int i = threadIdx.x; i < nv * 4; i += 256) {
        const int v = i >> 2, c = i & 3;
        rots[v0 * 4 + i] = s[v * FGS_PLY_FLOATS + 58 + c];
    }
    for (int i = threadIdx.x; i < nv * 48; i += 256) {
        const int v = i / 48, r = i - v * 48, coef = r / 3, ch = r - coef * 3;
        // coefficient 0 = f_dc_ch; coefficient k >= 1 = f_rest_[ch * 15 + k - 1]
        const int off = coef == 0 ? 6 + ch : 9 + ch * 15 + coef - 1;
        sh[v0 * 48 + i] = s[v * FGS_PLY_FLOATS + off];
    }
}

int fgs_launch_unpack_ply(const float *payload, int64_t P, float *means, float *sh, float *logit,
                          float *logs, float *rots, cudaStream_t st)
{
    if (P == 0) return FGS_OK;
    k_unpack_ply<<<(unsigned)((P + FGS_PLY_CHUNK - 1) / FGS_PLY_CHUNK), 256, 0, st>>>(
        payload, P, means, sh, logit, logs, rots);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// Row-band load estimate (multi-GPU row bands): how many in-frustum Gaussians
// have their projected centre in each tile row.  Every rank of a band job runs it on the
// same scene and camera and gets the same integers, so the ranks agree on work-balanced band
// edges without talking to each other.  A proxy only (centres, not pairs) -- the frame does
// not depend on where the bands are cut.  16 B read per Gaussian.
#define FGS_ROWHIST_SMEM 4096
__global__ void __launch_bounds__(256)
k_row_histogram(const float4 *__restrict__ g0, int64_t P, const __grid_constant__ CamDev cam,
                float frustum_thresh, uint32_t *__restrict__ hist)
{
    __shared__ uint32_t s_h[FGS_ROWHIST_SMEM];
    const int gh = cam.grid_h;
    const bool in_smem = gh <= FGS_ROWHIST_SMEM;
    if (in_smem)
        for (int i = threadIdx.x; i < gh; i += 256) s_h[i] = 0u;
    __syncthreads();
    for (int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x; g < P; g += (int64_t)gridDim.x * 256) {
        const float4 m = g0[g];
        const float t2 = fa(fa(fa(fm(cam.v[8], m.x), fm(cam.v[9], m.y)), fm(cam.v[10], m.z)), cam.v[11]);
        if (!((t2 > FGS_Z_NEAR) && (m.w > frustum_thresh))) continue;
        const float h1 = fa(fa(fa(fm(cam.p1[0], m.x), fm(cam.p1[1], m.y)), fm(cam.p1[2], m.z)), cam.p1[3]);
        const float h3 = fa(fa(fa(fm(cam.p3[0], m.x), fm(cam.p3[1], m.y)), fm(cam.p3[2], m.z)), cam.p3[3]);
        const float den = fabsf(h3) > 1e-7f ? h3 : 1e-7f;
        const float py = fm(fs(fm(fa(fd(h1, den), 1.0f), cam.hf), 1.0f), 0.5f);
        const float ty = floorf(fm(py, 0.0625f));
        if (!(ty >= -1.0f && ty <= (float)gh)) continue;             // well outside the frame
        const int row = (int)fminf(fmaxf(ty, 0.0f), (float)(gh - 1));
        atomicAdd(in_smem ? &s_h[row] : &hist[row], 1u);
    }
    __syncthreads();
    if (in_smem)
        for (int i = threadIdx.x; i < gh; i += 256)
            if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

int fgs_launch_row_histogram(const SceneDev &sc, int64_t P, const CamDev &cam, double tau,
                             uint32_t *hist, cudaStream_t st)
{
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)cam.grid_h * sizeof(uint32_t), st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    if (P == 0) return FGS_OK;
    const double th = tau > 1.0 / 255.0 ? tau : 1.0 / 255.0;       // projection.py:46
    int64_t blocks = (P + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_row_histogram<<<(unsigned)blocks, 256, 0, st>>>(sc.g0, P, cam, (float)th, hist);
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
    // (this unit is compiled with -fmad=false for the reference-order geometry; the
    // screening is tolerance-guarded, so it uses explicit FMAs)
    float qmin = __int_as_float(0x7f800000);
    if (out_u) {                                          // edge u = ue, v in [v0, v1]
        const float bu = b * ue;
        const float vs = fminf(fmaxf(__fdividef(-bu, c), v0), v1);
        qmin = fmaf(a * ue, ue, fmaf(c * vs, vs, 2.0f * bu * vs));
    }
    if (out_v) {                                          // edge v = ve, u in [u0, u1]
        const float bv = b * ve;
        const float us = fminf(fmaxf(__fdividef(-bv, a), u0), u1);
        qmin = fminf(qmin, fmaf(c * ve, ve, fmaf(a * us, us, 2.0f * bv * us)));
    }
    const float um = fmaxf(fabsf(u0), fabsf(u1)), vm = fmaxf(fabsf(v0), fabsf(v1));
    const float tol = 1e-4f * fmaf(fabsf(a) * um, um, fmaf(fabsf(c) * vm, vm,
                                   fmaf(2.0f * fabsf(b) * um, vm, fabsf(k))));
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
//   WALK_COUNT   nothing (count + pass mask)                           (ONESWEEP, K1)
//   WALK_BIN     count + pass mask + the CTA's tile table              (TILE_BUCKET, K1)
//   WALK_EMIT    write (key, value) at out_base(owner) + rank          (ONESWEEP, K3)
//   WALK_PLACE   slot from the CTA's tile table, record into the CTA's
//                write-combining buffer (or straight to its bucket)    (TILE_BUCKET, K3)
//
// TILE_BUCKET binning is a counting sort on the tile index whose unit of work is the CTA,
// not the pair.  With the scene packed in spatial order a CTA's 256 Gaussians hit a few
// dozen tiles, so K1 counts pairs per tile in a shared-memory table and reserves ONE
// range per (CTA, tile) in the tile's bucket (one global atomic per table entry instead
// of one per pair; L2 serialises atomics per address).  After the scan has fixed the
// bucket starts, K3 walks again (K1's pass masks make that cheap), ranks each pair inside
// its (CTA, tile) range with a shared-memory atomic, gathers the CTA's records by tile in
// shared memory and writes them out as contiguous runs.  Tiles that do not fit the table
// (caller-order scenes, huge splats) fall back to per-pair global atomics.
enum { WALK_COUNT = 0, WALK_BIN = 1, WALK_EMIT = 2, WALK_PLACE = 3 };

// The CTA's tile table: open addressing, at most FGS_HT_PROBES probes.
#ifndef FGS_HT_BITS
#define FGS_HT_BITS   9             // 512 slots: a CTA of a spatially ordered scene fills ~30
#endif
#define FGS_HT_SIZE   (1 << FGS_HT_BITS)
#define FGS_HT_PER    (FGS_HT_SIZE / FGS_PRE_THREADS)   // slots a thread of the epilogue owns
#define FGS_HT_PROBES 16
#define FGS_HT_EMPTY  0xffffffffu
#ifndef FGS_WC_CAP
#define FGS_WC_CAP    3072          // records the placement walk's write-combining buffer holds
#endif
#ifndef FGS_BLOCK_CAP
#define FGS_BLOCK_CAP 4608          // records of a regular preprocess CTA (its block in the stage);
#endif                              // with rec_of and eoff it fills the 40 KB staging buffer it aliases
#ifndef FGS_PLACE_MINBLOCKS
#define FGS_PLACE_MINBLOCKS 4
#endif
#define FGS_WC_NONE   0xffffu       // table entry whose range is written directly
struct TileTable {
    uint32_t key[FGS_HT_SIZE];      // tile index, FGS_HT_EMPTY = free
    uint32_t val[FGS_HT_SIZE];      // K1: pairs of this CTA on the tile; K3: rank cursor
};

__device__ __forceinline__ uint32_t ht_hash(uint32_t tile)
{
    return (tile * 2654435761u) >> (32 - FGS_HT_BITS);
}
// slot of `tile`, inserting it if absent; -1 when FGS_HT_PROBES slots are taken by others
__device__ __forceinline__ int ht_insert(TileTable &T, uint32_t tile)
{
    uint32_t h = ht_hash(tile);
#pragma unroll 1
    for (int p = 0; p < FGS_HT_PROBES; ++p) {
        uint32_t k = T.key[h];
        if (k == FGS_HT_EMPTY) k = atomicCAS(&T.key[h], FGS_HT_EMPTY, tile);
        if (k == tile || k == FGS_HT_EMPTY) return (int)h;
        h = (h + 1) & (FGS_HT_SIZE - 1);
    }
    return -1;
}
// slot of `tile` in a finished table (same probe sequence), -1 if it never got one
__device__ __forceinline__ int ht_find(const TileTable &T, uint32_t tile)
{
    uint32_t h = ht_hash(tile);
#pragma unroll 1
    for (int p = 0; p < FGS_HT_PROBES; ++p) {
        const uint32_t k = T.key[h];
        if (k == tile) return (int)h;
        if (k == FGS_HT_EMPTY) return -1;
        h = (h + 1) & (FGS_HT_SIZE - 1);
    }
    return -1;
}

// K1 (TILE_BUCKET) work area; takes over the SH staging buffer once the colours are done.
// A "regular" CTA -- every pair found a table entry, at most FGS_BLOCK_CAP pairs, at most
// FGS_PARK_CAP of them from Gaussians on the cooperative walk -- leaves K1 with its records
// already grouped by (CTA, tile) run in the frame's stage, and K3 is a streaming copy of those
// runs into the tile buckets.  Any other CTA is put on the fallback list and placed by the
// second walk (k_place), exactly as every CTA was before the stage existed.
#ifndef FGS_PARK_CAP
#define FGS_PARK_CAP  2944          // pairs of cooperative-walk Gaussians a regular CTA can park
                                    // (1920: a quarter of the 8K frame's CTAs overflowed it)
#endif
#define FGS_ER_NONE   0xffffffffu
// What the walks write: its own shared memory (not the staging buffer), initialised when the
// CTA starts, so a warp goes from its colours straight into its walk -- no CTA barrier between
// the geometry and the binning (the warps of a CTA drift apart by then: that barrier held 11 %
// of the kernel's stall samples).
struct BinTable {
    TileTable tab;
    uint32_t park[FGS_PARK_CAP];    // entry | rank << 10 | owner thread << 20
    uint32_t npark, irregular;
};
// What the epilogue adds once every warp's walk is done (and with it every thread's use of the
// staging buffer, which this aliases).
struct BinSmem {
    uint64_t wc[FGS_BLOCK_CAP];     // the CTA's records in run order
    uint64_t rec_of[FGS_PRE_THREADS];   // each thread's record: depth bits << 32 | Gaussian index
    uint16_t eoff[FGS_HT_SIZE];     // offset of table entry e's run in the CTA's record block
};
struct BinNone {};

// What WALK_BIN / WALK_PLACE work on.
struct BinCtx {
    TileTable *table;
    uint32_t *tile_ctr;             // per tile, FGS_CTR_STRIDE words apart: [0] pairs reserved
                                    // through tables, [1] fallback pairs, [2] fallback cursor
    // WALK_BIN only
    uint32_t *park, *npark, *irregular;
    // WALK_PLACE only
    const uint32_t *gbase;          // [FGS_HT_SIZE] bucket position of the entry's range
    const uint16_t *wcoff;          // [FGS_HT_SIZE] offset in the write-combining buffer
    uint64_t *wcrec;                // [FGS_WC_CAP]
    uint32_t *wcdst;                // [FGS_WC_CAP]
    const int32_t *starts;
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
                                                    const BinCtx *bc = nullptr,
                                                    uint64_t *mask_out = nullptr)
{
    constexpr bool COUNTING = (MODE == WALK_COUNT || MODE == WALK_BIN);
    const int lane = threadIdx.x & 31;
    const uint32_t incl = warp_incl_scan(job.cand, lane);
    const uint32_t total = __shfl_sync(FGS_FULL, incl, 31);
    const uint32_t excl = incl - job.cand;
    // ceil(2^32 / nx), or 0 = "divide" for a rectangle so large the reciprocal is not exact
    const uint32_t rnx = (job.nx > 1 && (uint64_t)job.cand * (uint32_t)job.nx < (1ull << 32))
                             ? 0xffffffffu / (uint32_t)job.nx + 1u : 0u;
    uint32_t mine = 0;
    uint64_t mymask = 0;
    // K3: does any lane of this warp need the exact test again?
    const bool any_big = !COUNTING && PRECISE && __any_sync(FGS_FULL, job.cand > FGS_MASK_CAND);
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
        const uint32_t rnx_o = __shfl_sync(FGS_FULL, rnx, o);
        const uint32_t local = act ? j - excl_o : 0u;
        // local / nx by the owner's reciprocal ceil(2^32 / nx): exact while local * nx < 2^32
        // (a rectangle has at most grid tiles <= 2^31 candidates)
        const int ry = (int)(nx <= 1 ? local : rnx_o ? __umulhi(local, rnx_o) : local / (uint32_t)nx);
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
            const uint32_t cand_o = COUNTING ? 0u : __shfl_sync(FGS_FULL, job.cand, o);
            if (COUNTING || cand_o > FGS_MASK_CAND) {
                const int h = act ? tile_hits32(tx, ty, width, height, cx, cy, a, b, c, ke) : 0;
                pass = h == 1;
                if (h == 2) pass = tile_hits(tx, ty, width, height, cx, cy, a, b, c, ke);
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
        if (MODE == WALK_BIN) {
            // count the pair in the CTA's table; the atomic's return value is its rank in the
            // (CTA, tile) run, parked with the entry and the owner until the run offsets exist
            uint32_t word = FGS_ER_NONE;
            if (pass) {
                const uint32_t tile = (uint32_t)(ty * grid_w + tx);
                const int e = ht_insert(*bc->table, tile);
                if (e >= 0) {
                    const uint32_t r = atomicAdd(&bc->table->val[e], 1u);
                    word = (uint32_t)e | (r << 10) | ((uint32_t)((threadIdx.x & ~31) + o) << 20);
                } else {
                    atomicAdd(&bc->tile_ctr[(size_t)tile * FGS_CTR_STRIDE + 1], 1u);
                    *bc->irregular = 1u;
                }
            }
            const uint32_t parked = __ballot_sync(FGS_FULL, word != FGS_ER_NONE);
            if (parked) {
                uint32_t pbase = 0;
                if (lane == 0) pbase = atomicAdd(bc->npark, (uint32_t)__popc(parked));
                pbase = __shfl_sync(FGS_FULL, pbase, 0);
                if (word != FGS_ER_NONE) {
                    const uint32_t pos = pbase + __popc(parked & lanemask_lt());
                    if (pos < FGS_PARK_CAP) bc->park[pos] = word;
                    else *bc->irregular = 1u;
                }
            }
        }
        if (MODE == WALK_PLACE) {
            const uint32_t bits_o = __shfl_sync(FGS_FULL, depth_bits, o);
            const uint32_t gid_o = __shfl_sync(FGS_FULL, gid, o);
            if (pass) {
                const uint32_t tile = (uint32_t)(ty * grid_w + tx);
                const uint64_t rec = ((uint64_t)bits_o << 32) | gid_o;
                const int e = ht_find(*bc->table, tile);
                if (e >= 0) {
                    const uint32_t r = atomicAdd(&bc->table->val[e], 1u);
                    const uint32_t dst = bc->gbase[e] + r;
                    const uint32_t off = bc->wcoff[e];
                    if (off != FGS_WC_NONE) {
                        bc->wcrec[off + r] = rec;
                        bc->wcdst[off + r] = dst;
                    } else {
                        keys[dst] = rec;
                    }
                } else {
                    uint32_t *ctr = bc->tile_ctr + (size_t)tile * FGS_CTR_STRIDE;
                    keys[(uint32_t)bc->starts[tile] + ctr[0] + atomicAdd(&ctr[2], 1u)] = rec;
                }
            }
        }
        // owner side: how many of my candidates in this window passed
        const int lo = excl > base ? (int)(excl - base) : 0;
        const int hi = incl - base < 32u ? (int)(incl - base) : 32;
        if (job.cand && incl > base && lo < hi) {
            const uint32_t m = (hi - lo == 32) ? FGS_FULL : (((1u << (hi - lo)) - 1u) << lo);
            mine += __popc(ballot & m);
            if (COUNTING) {
                // my candidates in this window start at my local index base + lo - excl
                const uint32_t first = base + (uint32_t)lo - excl;
                if (first < 64u) mymask |= (uint64_t)((ballot & m) >> lo) << first;
            }
        }
    }
    if (COUNTING && mask_out) *mask_out = mymask;
    return mine;
}

// ---------------------------------------------------------------------------
// The lane-local walk for the common case: a Gaussian whose candidate rectangle is at most
// 3 x 3 tiles (95 % of them at 4-5 pairs per Gaussian) tests its own tiles, with no owner
// search and no operand shuffles.  What a column of tiles shares (the facing vertical edge
// ue, a ue^2, b ue, the unclamped minimiser -b ue / c) and what a row shares are evaluated
// once, so a tile costs two clamps, two Horner steps and the comparison.  Same screen as
// tile_hits32: the float32 minimum of the form over the tile decides unless it is within the
// guard band of keff, and then the reference's float64 predicate does.  The band here is
// 1e-4 of the Gaussian's own bound  a ex^2 + 2|b| ex ey + c ey^2 + |keff|  (ex = hx + 16,
// ey = hy + 16: every candidate tile lies inside the extent rectangle grown by one tile, so
// this bounds each tile's term magnitude) -- wider than tile_hits32's per-tile band, never
// narrower, so the verdict is the reference's all the same.
// Passing tiles are counted in the CTA's table; er[k] = entry | rank << 16 of tile
// k = row * 3 + col (FGS_ER_NONE: no pair).  Returns the pair count; `mask` gets the pass bits
// in the rectangle's own row-major order (what k_place expects).
// ---------------------------------------------------------------------------
template <bool PRECISE>
__device__ __forceinline__ uint32_t small_walk(bool mine, float cx, float cy, float a, float b,
                                               float c, float keff, float term, int tx0, int ty0,
                                               int nx, int ny, int width, int height, int grid_w,
                                               const BinCtx &bc, uint32_t (&er)[9], uint64_t &mask)
{
    uint32_t pass = 0;                                    // bit row * 3 + col
    if (mine) {
        if (PRECISE) {
            const float tol = 1e-4f * (term + fabsf(keff));
            const float klo = keff - tol, khi = keff + tol;
            const float rc = __fdividef(1.0f, c), ra = __fdividef(1.0f, a);
            const float xb = (float)(tx0 * FGS_TILE), yb = (float)(ty0 * FGS_TILE);
            const float wf = (float)width, hf = (float)height;
            float e0[3], e1[3], q2[3], lin[3], star[3];   // columns: u0 u1 a*ue^2 2*b*ue -b*ue/c
            bool inu[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const float x0 = xb + (float)(FGS_TILE * i);
                e0[i] = x0 - cx;
                e1[i] = fminf(x0 + (float)FGS_TILE, wf) - cx;
                inu[i] = e0[i] <= 0.0f && e1[i] >= 0.0f;
                const float ue = e0[i] > 0.0f ? e0[i] : e1[i];   // the edge facing the centre
                const float bu = b * ue;
                q2[i] = a * ue * ue;
                lin[i] = 2.0f * bu;
                star[i] = -bu * rc;
            }
            uint32_t amb = 0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                // the row's own terms: v0 v1, the facing edge ve, c*ve^2, 2*b*ve, -b*ve/a
                const float y0 = yb + (float)(FGS_TILE * j);
                const float f0 = y0 - cy, f1 = fminf(y0 + (float)FGS_TILE, hf) - cy;
                const bool inv = f0 <= 0.0f && f1 >= 0.0f;
                const float ve = f0 > 0.0f ? f0 : f1;
                const float bv = b * ve;
                const float r2 = c * ve * ve, rin = 2.0f * bv, rtar = -bv * ra;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    if (i < nx && j < ny) {
                        float q = __int_as_float(0x7f800000);
                        if (!inu[i]) {                    // edge u = ue, v in [v0, v1]
                            const float vs = fminf(fmaxf(star[i], f0), f1);
                            q = fmaf(fmaf(c, vs, lin[i]), vs, q2[i]);
                        }
                        if (!inv) {                       // edge v = ve, u in [u0, u1]
                            const float us = fminf(fmaxf(rtar, e0[i]), e1[i]);
                            q = fminf(q, fmaf(fmaf(a, us, rin), us, r2));
                        }
                        const uint32_t bit = 1u << (j * 3 + i);
                        if ((inu[i] && inv) || q < klo) pass |= bit;        // intersect.py:84-86 / clear hit
                        else if (!(q > khi)) amb |= bit;                    // too close (or not finite)
                    }
                }
            }
            while (amb) {                                 // rare: the reference's float64 predicate
                const int k = __ffs((int)amb) - 1;
                amb &= amb - 1u;
                if (tile_hits(tx0 + k % 3, ty0 + k / 3, width, height, cx, cy, a, b, c, keff))
                    pass |= 1u << k;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    if (i < nx && j < ny) pass |= 1u << (j * 3 + i);
        }
    }
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        er[k] = FGS_ER_NONE;
        if ((pass >> k) & 1u) {
            const int i = k % 3, j = k / 3;
            const uint32_t tile = (uint32_t)((ty0 + j) * grid_w + tx0 + i);
            // (electing one lane per tile with match.any to count its peers with a single
            // atomic was measured: 951 -> 1075 us on the 10M frame -- the match costs more
            // than the same-address atomics it saves)
            const int e = ht_insert(*bc.table, tile);
            if (e >= 0) {
                er[k] = (uint32_t)e | (atomicAdd(&bc.table->val[e], 1u) << 16);
            } else {
                atomicAdd(&bc.tile_ctr[(size_t)tile * FGS_CTR_STRIDE + 1], 1u);
                *bc.irregular = 1u;
            }
            m |= 1u << (j * nx + i);
        }
    }
    mask = m;
    return (uint32_t)__popc(pass);
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

#ifndef FGS_SH_STAGED
#define FGS_SH_STAGED 10          // SH float4 planes staged in shared memory (of 12): 40 KB, which
                                  // leaves 16 KB of the CTA's 56 for the tile table and the parked ranks
#endif
static_assert(FGS_SH_STAGED * FGS_PRE_THREADS * 16 >= (int)sizeof(BinSmem), "the binning work area aliases the staging buffer");
__device__ __forceinline__ void cp_async16_pre(void *smem, const void *gmem)
{
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem) : "memory");
}

#ifndef FGS_PLACE_PF_DIST
#define FGS_PLACE_PF_DIST 592    // K3: CTAs ahead for the L2 prefetch (4 per SM x 148; 0 = off)
#endif
// ---------------------------------------------------------------------------
// K1: preprocess + count
// ---------------------------------------------------------------------------
template <int STRAT, bool BUCKET, bool BANDED>
__global__ void __launch_bounds__(FGS_PRE_THREADS, FGS_PRE_MINBLOCKS)
k_preprocess(SceneDev sc, const float *__restrict__ kcut, int P,
             const __grid_constant__ CamDev cam, float tau32, float frustum_thresh,
             int sh_degree, int band0, int band1, FrameDev f)
{
    __shared__ uint32_t s_red[8], s_red1[8], s_red2[8];
    __shared__ uint32_t s_bin[4], s_scan[8];
    __shared__ unsigned long long s_scan64[8];
    // SH staging: plane j of thread t at s_sh[j * 256 + t] (48 KB, dynamic).  A thread's 12
    // cp.async gathers are issued as soon as its Gaussian passes the frustum test and land
    // while the covariance chain runs -- no registers held, one DRAM round trip hidden.
    extern __shared__ __align__(16) float4 s_sh[];
    fgs_pdl_trigger();                    // first kernel of the frame (plain launch): the tile
                                          // scan may be scheduled behind this grid's last wave
    const int g = blockIdx.x * FGS_PRE_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool live = g < P;
    BinSmem &B = *reinterpret_cast<BinSmem *>(s_sh);
    __shared__ typename std::conditional<BUCKET, BinTable, BinNone>::type s_bt_;
    BinTable &BT = *reinterpret_cast<BinTable *>(&s_bt_);
    TileTable &s_tab = BT.tab;
    if (BUCKET) {
        for (int i = threadIdx.x; i < FGS_HT_SIZE; i += FGS_PRE_THREADS) {
            s_tab.key[i] = FGS_HT_EMPTY;
            s_tab.val[i] = 0u;
        }
        if (threadIdx.x == 0) { BT.npark = 0u; BT.irregular = 0u; s_bin[2] = 0u; }
        __syncthreads();                  // (every warp arrives at once: the CTA has just started)
    }
    // TILE_BUCKET: this CTA's pairs per tile, their parked ranks and the record block.  The
    // work area takes over the SH staging buffer once every thread has consumed its
    // coefficients (the CTA then needs 48 KB, not 92).

    TileJob job;
    job.cand = 0;
    job.cx = job.cy = job.a = job.b = job.c = job.keff = 0.f;
    job.tx0 = job.ty0 = 0;
    job.nx = 1;
    job.mask = 0;
    bool retained = false, degenerate = false;
    uint32_t full_cand = 0, og = 0;
    float zcam = 0.0f, job_term = 0.0f;
    int job_ny = 0;

    if (live) {
        // all per-Gaussian geometry loads go out together (48 B; the culled ones waste 28)
        if (BUCKET) og = sc.orig[g];
        const float4 m = sc.g0[g];
        const float4 sc4 = sc.g1[g];
        const float4 q = sc.g2[g];
        const float k = kcut[g];
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
#ifndef FGS_PROBE_NO_SH     // (timing probe: K1 without the SH colours -- WRONG frames)
#pragma unroll
            for (int j = 0; j < FGS_SH_STAGED; ++j)
                cp_async16_pre(&s_sh[j * FGS_PRE_THREADS + threadIdx.x], &sc.sh[(int64_t)j * sc.n + g]);
            asm volatile("cp.async.commit_group;" ::: "memory");
#endif
            // projection.py:59-85: the 3D covariance, evaluated per scene by fgs_scene_pack
            float S[3][3];
            S[0][0] = sc4.x; S[0][1] = S[1][0] = sc4.y; S[0][2] = S[2][0] = sc4.z;
            S[1][1] = sc4.w; S[1][2] = S[2][1] = q.x;   S[2][2] = q.y;
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
                    job_ny = by1 - by0 + 1;
                    job_term = term;
                }
                // Row-band frames (multi-GPU): a Gaussian without candidate tiles in this
                // rank's band emits no pair here, so nothing reads its colour or splat row --
                // skip both (every rank walks all P Gaussians; this is most of them).  A
                // template flag: the whole-frame kernel is the same code as without it.
                if (!BANDED || by0 <= by1) {
                // binning.py:230-233 view direction, render.py:52-86 colour
                const float d0 = fs(x, cam.pos[0]), d1 = fs(y, cam.pos[1]), d2 = fs(z, cam.pos[2]);
                float nrm = fsq(fa(fa(fm(d0, d0), fm(d1, d1)), fm(d2, d2)));
                nrm = nrm > 0.0f ? nrm : 1.0f;
                float bz[16];
                sh_basis(fd(d0, nrm), fd(d1, nrm), fd(d2, nrm), bz);
                // The 48 coefficients c[3*i + ch] stream out of the staging buffer one float4 at
                // a time; every channel still accumulates its terms in the reference's order
                // (render.py:60-85), so the colours stay bit-exact, and only the running sums
                // are live (no 48-register coefficient array).
                asm volatile("cp.async.wait_group 0;" ::: "memory");   // own gathers: no barrier needed
                float rgb[3] = {0.0f, 0.0f, 0.0f};
#ifndef FGS_PROBE_NO_SH
                // planes beyond the staged ones come straight from global memory, issued here
                // and consumed last (the staging buffer is what caps the CTAs per SM)
                float4 late[12 - FGS_SH_STAGED + 1];
#pragma unroll
                for (int j = FGS_SH_STAGED; j < 12; ++j) late[j - FGS_SH_STAGED] = sc.sh[(int64_t)j * sc.n + g];
#pragma unroll
                for (int j = 0; j < 12; ++j) {
                    const float4 v4 = j < FGS_SH_STAGED ? s_sh[j * FGS_PRE_THREADS + threadIdx.x]
                                                        : late[j < FGS_SH_STAGED ? 0 : j - FGS_SH_STAGED];
                    const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int fi = 4 * j + u, i = fi / 3, ch = fi % 3;
                        const float v = vv[u];
                        if (i == 0) rgb[ch] = fm(0.28209479177387814f, v);
                        else if (i == 1 || i == 3) { if (sh_degree >= 1) rgb[ch] = fs(rgb[ch], fm(bz[i], v)); }
                        else if (i == 2) { if (sh_degree >= 1) rgb[ch] = fa(rgb[ch], fm(bz[i], v)); }
                        else if (i < 9) { if (sh_degree >= 2) rgb[ch] = fa(rgb[ch], fm(bz[i], v)); }
                        else { if (sh_degree >= 3) rgb[ch] = fa(rgb[ch], fm(bz[i], v)); }
                    }
                }
#else
                rgb[0] = bz[1]; rgb[1] = bz[2]; rgb[2] = bz[3];
#endif
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) rgb[ch] = fmaxf(fa(rgb[ch], 0.5f), 0.0f);
                // render.py:34-40 splat row, binning.py:235-241
                float4 *row = (float4 *)(f.splat + (size_t)g * 12);
                row[0] = make_float4(px, py, ca, cb);
                row[1] = make_float4(cc, op, k, rgb[0]);
                row[2] = make_float4(rgb[1], rgb[2], hx, hy);
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");       // culled after the frustum test
        }
        f.rects[g] = rect;
        f.flags[g] = (uint8_t)((retained ? 1 : 0) | (degenerate ? 2 : 0));
    }

    uint32_t npairs;
    uint64_t passmask = 0;
    uint32_t er[9];                       // small walk: entry | rank << 16 per tile of the 3 x 3
    const uint64_t rec = ((uint64_t)__float_as_uint(zcam) << 32) | og;
    if (BUCKET) {
        const BinCtx bc{&s_tab, f.tilecount, BT.park, &BT.npark, &BT.irregular,
                        nullptr, nullptr, nullptr, nullptr, nullptr};
        // rectangles of at most 3 x 3 tiles: each lane walks its own; the rest of the warp's
        // candidates (if any) go through the cooperative walk
        // (measured on the 10M frame: everything through the cooperative walk instead, with
        // the same parking, is 1021 us against 952)
        const bool small = job.cand != 0u && job.nx <= 3 && job_ny <= 3;
        npairs = small_walk<STRAT == FGS_PRECISE>(small, job.cx, job.cy, job.a, job.b, job.c, job.keff,
                                                  job_term, job.tx0, job.ty0, job.nx, job_ny,
                                                  cam.width, cam.height, cam.grid_w, bc, er, passmask);
        if (small) job.cand = 0u;
        if (__any_sync(FGS_FULL, job.cand != 0u)) {
            uint64_t bigmask = 0;
            const uint32_t nbig = warp_walk_tiles<STRAT == FGS_PRECISE, WALK_BIN>(
                job, cam.width, cam.height, cam.grid_w, 0, 0, 0, nullptr, nullptr, &bc, &bigmask);
            if (!small) { npairs = nbig; passmask = bigmask; }
        }
        // binning.py:50-51: depths of emitted pairs must be positive and finite
        if (npairs && !(zcam < __int_as_float(0x7f800000))) f.stats->bad_depth = 1u;
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
        s_red1[threadIdx.x >> 5] = v1;
        s_red2[threadIdx.x >> 5] = v2;
    }
    __syncthreads();                      // also: every warp's walk is done, the table is final,
                                          // and nobody reads the staging buffer any more
    if (BUCKET) B.rec_of[threadIdx.x] = rec;      // (read after the run-offset barrier)
    if (threadIdx.x == 0) {
        // one atomic per CTA and counter: every CTA of the grid hits the same three words,
        // and L2 serialises atomics on one address
        uint32_t t = 0, t1 = 0;
        unsigned long long t2 = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { t += s_red[i]; t1 += s_red1[i]; t2 += s_red2[i]; }
        f.blocksums[blockIdx.x] = t;
        if (t1 & 0xffffu) atomicAdd(&f.stats->gaussians_retained, t1 & 0xffffu);
        if (t1 >> 16) atomicAdd(&f.stats->gaussians_degenerate, t1 >> 16);
        if (t2) atomicAdd((unsigned long long *)&f.stats->candidate_tiles_lo, t2);
    }
    if (!BUCKET) return;

    // ---- TILE_BUCKET epilogue: one range per (CTA, tile) in the tile's bucket.  Thread t
    // owns table slots FGS_HT_PER t .. FGS_HT_PER (t + 1) - 1; entries go to the frame's table list in slot order, each
    // with the offset of its run in the CTA's record block.
    // The global round trips of this epilogue -- the bucket reservations (one atomic per
    // table entry, result needed for the list), the list reservation and the stage
    // reservation (thread 0) -- are issued as early as their operands exist and consumed
    // after the block scans / the placement, which hide them.
    uint32_t cnt[FGS_HT_PER], tl[FGS_HT_PER], gb[FGS_HT_PER], nent = 0, npr = 0;
#pragma unroll
    for (int k = 0; k < FGS_HT_PER; ++k) {
        const int e = threadIdx.x * FGS_HT_PER + k;
        tl[k] = s_tab.key[e];
        const bool used = tl[k] != FGS_HT_EMPTY;
        cnt[k] = used ? s_tab.val[e] : 0u;
        nent += used ? 1u : 0u;
        npr += cnt[k];
        // the counters always get the pairs, so M stays exact when the frame overflows
        gb[k] = used ? atomicAdd(&f.tilecount[(size_t)tl[k] * FGS_CTR_STRIDE], cnt[k]) : 0u;
    }
    // entries and pairs before this thread's slots: one scan of the packed pair
    unsigned long long tot2;
    const unsigned long long off2 =
        block_excl_scan64_256(((unsigned long long)nent << 40) | npr, s_scan64, tot2);
    const uint32_t tot_ent = (uint32_t)(tot2 >> 40), ent_off = (uint32_t)(off2 >> 40);
    const unsigned long long tot_pr64 = tot2 & ((1ull << 40) - 1ull);
    uint32_t pr_off = (uint32_t)(off2 & ((1ull << 40) - 1ull));
    // regular: every pair has a table entry and a parked rank, and the record block fits
    const bool regular = BT.irregular == 0u && tot_pr64 <= (unsigned long long)FGS_BLOCK_CAP;
    const uint32_t tot_pr = regular ? (uint32_t)tot_pr64 : 0u;
    uint32_t lb = 0, sb = FGS_CTA_NO_STAGE;
    if (threadIdx.x == 0) {
        if (tot_ent) lb = atomicAdd(&f.stats->list_used, tot_ent);
        if (regular && tot_pr) sb = atomicAdd(&fgs_work(f.stats)[FGS_WORK_STAGE_USED], tot_pr);
        if (!regular)                           // left to the placement walk (k_place)
            f.fb_list[atomicAdd(&fgs_work(f.stats)[FGS_WORK_FB_CTAS], 1u)] = blockIdx.x;
    }
    if (!regular) {
        // ---- the second walk places this CTA's pairs: its list says, per entry, where the
        // placement walk write-combines the run (a prefix of the runs fits its buffer)
        if (live && STRAT == FGS_PRECISE && npairs) f.passmask[g] = passmask;
        if (threadIdx.x == 0) {
            s_bin[0] = lb;
            s_bin[1] = (lb + tot_ent <= f.list_capacity) ? 1u : 0u;
            if (tot_ent && lb + tot_ent > f.list_capacity) f.stats->overflow = 1u;   // grow and re-run
        }
        __syncthreads();
        const uint32_t list_base = s_bin[0];
        const bool fits = s_bin[1] != 0u;
        uint32_t idx = list_base + ent_off, staged_end = 0;
#pragma unroll
        for (int k = 0; k < FGS_HT_PER; ++k) {
            const int e = threadIdx.x * FGS_HT_PER + k;
            if (tl[k] != FGS_HT_EMPTY) {
                const bool wc = (unsigned long long)pr_off + cnt[k] <= (unsigned long long)FGS_WC_CAP;
                if (wc) staged_end = pr_off + cnt[k];
                if (fits)
                    f.tablelist[idx++] = make_uint4(tl[k], gb[k], cnt[k],
                                                    ((uint32_t)e << 16) | (wc ? pr_off : FGS_WC_NONE));
            }
            pr_off += cnt[k];
        }
        if (staged_end) atomicMax(&s_bin[2], staged_end);
        __syncthreads();
        if (threadIdx.x == 0)
            f.ctainfo[blockIdx.x] = make_uint4(list_base, fits ? tot_ent : 0u, s_bin[2], FGS_CTA_NO_STAGE);
        return;
    }
    // ---- regular: run offsets, then every pair's record to its run, rank-th inside it
    {
        uint32_t o = pr_off;
#pragma unroll
        for (int k = 0; k < FGS_HT_PER; ++k) {
            if (tl[k] != FGS_HT_EMPTY) B.eoff[threadIdx.x * FGS_HT_PER + k] = (uint16_t)o;
            o += cnt[k];
        }
    }
    __syncthreads();                      // run offsets are in place
#pragma unroll
    for (int k = 0; k < 9; ++k)
        if (er[k] != FGS_ER_NONE) B.wc[B.eoff[er[k] & 0xffffu] + (er[k] >> 16)] = rec;
    for (uint32_t i = threadIdx.x; i < BT.npark; i += FGS_PRE_THREADS) {
        const uint32_t w = BT.park[i];
        B.wc[B.eoff[w & 1023u] + ((w >> 10) & 1023u)] = B.rec_of[w >> 20];
    }
    if (threadIdx.x == 0) {               // the two reservations have had the placement to arrive
        const bool fits = lb + tot_ent <= f.list_capacity;
        // M is exact either way (tile counters); a stage that does not fit means the pair
        // buffer does not either
        const bool stage_fits = !tot_pr || (uint64_t)sb + tot_pr <= (uint64_t)f.list_capacity * 2u;
        if ((tot_ent && !fits) || !stage_fits) f.stats->overflow = 1u;             // grow and re-run
        s_bin[0] = lb;
        s_bin[1] = fits ? 1u : 0u;
        s_bin[3] = stage_fits ? sb : FGS_CTA_NO_STAGE;
        f.ctainfo[blockIdx.x] = make_uint4(lb, fits ? tot_ent : 0u, tot_pr,
                                           tot_pr && stage_fits ? sb : FGS_CTA_NO_STAGE);
    }
    __syncthreads();
    if (s_bin[1]) {
        uint32_t idx = s_bin[0] + ent_off;
#pragma unroll
        for (int k = 0; k < FGS_HT_PER; ++k) {
            if (tl[k] != FGS_HT_EMPTY)
                f.tablelist[idx++] = make_uint4(tl[k], gb[k], cnt[k],
                                                ((uint32_t)(threadIdx.x * FGS_HT_PER + k) << 16) | pr_off);
            pr_off += cnt[k];
        }
    }
    const uint32_t stage_base = s_bin[3];
    if (tot_pr && stage_base != FGS_CTA_NO_STAGE)
        for (uint32_t i = threadIdx.x; i < tot_pr; i += FGS_PRE_THREADS)
            f.stage[stage_base + i] = B.wc[i];
}

static CamDev g_dummy_cam;   // keeps CamDev's layout in one place for sizeof checks
static_assert(sizeof(CamDev) % 4 == 0, "CamDev must be word-sized");

int fgs_launch_preprocess(const SceneDev &sc, const float *kcut, int64_t P, const CamDev &cam,
                          double tau, int sh_degree, int strategy, int band0, int band1,
                          int bucket, int tiles, const FrameDev &f, cudaStream_t st)
{
    (void)g_dummy_cam;
    // stats and (TILE_BUCKET) the per-tile histogram sit back to back: one memset
    // the stats block is 256 bytes in the workspace: public counters + internal work counters
    // (stats | tile counters | tile-order header) are contiguous in the workspace
    const size_t zero_bytes = bucket ? (size_t)((char *)(f.tileorder + FGS_ORDER_HDR) - (char *)f.stats)
                                     : 256;
    cudaError_t e = cudaMemsetAsync(f.stats, 0, zero_bytes, st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    if (P == 0) return FGS_OK;
    const double th = tau > 1.0 / 255.0 ? tau : 1.0 / 255.0;       // projection.py:46
    const unsigned blocks = (unsigned)((P + FGS_PRE_THREADS - 1) / FGS_PRE_THREADS);
    const float tau32 = (float)tau, fth = (float)th;
    constexpr int kShBytes = FGS_SH_STAGED * FGS_PRE_THREADS * 16; // SH staging, 4 KB per plane
    static FgsOncePerDevice attr_once;
    int attr_dev = 0;
    if (attr_once.need(&attr_dev)) {
        cudaError_t ea = cudaSuccess;
#define FGS_ATTR1(S, B, N) if (ea == cudaSuccess) ea = cudaFuncSetAttribute(k_preprocess<S, B, N>, \
        cudaFuncAttributeMaxDynamicSharedMemorySize, kShBytes)
#define FGS_ATTR(S, B) FGS_ATTR1(S, B, false); FGS_ATTR1(S, B, true)
        FGS_ATTR(FGS_PRECISE, true); FGS_ATTR(FGS_PRECISE, false);
        FGS_ATTR(FGS_TIGHT_AABB, true); FGS_ATTR(FGS_TIGHT_AABB, false);
        FGS_ATTR(FGS_BASELINE_CIRCLE_AABB, true); FGS_ATTR(FGS_BASELINE_CIRCLE_AABB, false);
#undef FGS_ATTR
#undef FGS_ATTR1
        if (ea != cudaSuccess) { fgs_set_cuda_error(ea); return FGS_E_CUDA; }
        attr_once.mark(attr_dev);
    }
    const bool banded = band0 > 0 || band1 < cam.grid_h - 1;
#define FGS_K1N(S, B, N) k_preprocess<S, B, N><<<blocks, FGS_PRE_THREADS, kShBytes, st>>>( \
        sc, kcut, (int)P, cam, tau32, fth, sh_degree, band0, band1, f)
#define FGS_K1(S, B) do { if (banded) FGS_K1N(S, B, true); else FGS_K1N(S, B, false); } while (0)
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
// For large grids (> FGS_SCAN_DIRECT_CTAS slices) the slices' totals are summed first by this
// kernel into the spare words 5/6 of the cursor slots, and k_scan_tiles adds up the totals
// before its slice instead of every count before it (8K frame: 127 slices, the last one would
// read 129 K counters through one SM: 41 us -> ~10).
#define FGS_SCAN_DIRECT_CTAS 12
__global__ void __launch_bounds__(1024)
k_tile_blocksums(const uint32_t *__restrict__ counts, uint32_t *__restrict__ cursor, int tiles)
{
    __shared__ unsigned long long s_w[32];
    fgs_pdl_wait();
    fgs_pdl_trigger();
    const int i = blockIdx.x * 1024 + threadIdx.x;
    unsigned long long v = i < tiles ? (unsigned long long)counts[(size_t)i * FGS_CTR_STRIDE] +
                                           counts[(size_t)i * FGS_CTR_STRIDE + 1] : 0ull;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FGS_FULL, v, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
#pragma unroll
        for (int k = 0; k < 32; ++k) t += s_w[k];
        cursor[(size_t)blockIdx.x * FGS_CTR_STRIDE + 5] = (uint32_t)t;
        cursor[(size_t)blockIdx.x * FGS_CTR_STRIDE + 6] = (uint32_t)(t >> 32);
    }
}

__global__ void __launch_bounds__(1024)
k_scan_tiles(const uint32_t *__restrict__ counts, int32_t *__restrict__ starts,
             uint32_t *__restrict__ cursor, uint32_t *__restrict__ bincount, int tiles,
             unsigned long long capacity, fgs_stats *__restrict__ stats, int use_sums,
             int32_t *__restrict__ limit, uint32_t heavy_thr)
{
    __shared__ unsigned long long s_w[32];
    __shared__ uint32_t s_bin[FGS_ORDER_BINS];
    fgs_pdl_wait();
    fgs_pdl_trigger();
    if (threadIdx.x < FGS_ORDER_BINS) s_bin[threadIdx.x] = 0u;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int first = blockIdx.x * 1024;
    // prefix of everything before this CTA's slice
    unsigned long long before = 0;
    if (use_sums) {
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += 1024)
            before += (unsigned long long)cursor[(size_t)j * FGS_CTR_STRIDE + 5] |
                      ((unsigned long long)cursor[(size_t)j * FGS_CTR_STRIDE + 6] << 32);
    } else {
        for (int i = threadIdx.x; i < first; i += 1024)
            before += counts[(size_t)i * FGS_CTR_STRIDE] + counts[(size_t)i * FGS_CTR_STRIDE + 1];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) before += __shfl_xor_sync(FGS_FULL, before, o);
    if (lane == 0) s_w[w] = before;
    __syncthreads();
    unsigned long long carry = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) carry += s_w[i];
    __syncthreads();

    const int i = first + threadIdx.x;
    // word 0: pairs reserved through the CTAs' tile tables, word 1: fallback pairs
    const unsigned long long v = i < tiles ? (unsigned long long)counts[(size_t)i * FGS_CTR_STRIDE] +
                                                 counts[(size_t)i * FGS_CTR_STRIDE + 1] : 0u;
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
    // size-bin histogram for the blend's tile order (placement: k_tile_order)
    if (i < tiles)
        atomicAdd(&s_bin[fgs_order_bin(fgs_order_weight(v > 0xffffffffull ? 0xffffffffu : (uint32_t)v, heavy_thr))], 1u);
    __syncthreads();
    if (threadIdx.x < FGS_ORDER_BINS && s_bin[threadIdx.x])
        atomicAdd(&bincount[threadIdx.x], s_bin[threadIdx.x]);
    if (i < tiles) {
        const uint32_t e32 = excl > 0x7fffffffull ? 0x7fffffffu : (uint32_t)excl;
        starts[i] = (int32_t)e32;
        if (v > FGS_LARGE_TILE) {   // queue the bucket for its tile-sort size class
            cursor[(size_t)atomicAdd(&stats->dense_tiles, 1u) * FGS_CTR_STRIDE + 1] = (uint32_t)i;
            atomicAdd(&fgs_work(stats)[FGS_WORK_DENSE0], 1u);
        }
        else if (v > FGS_DENSE_TILE)
            cursor[(size_t)atomicAdd(&fgs_work(stats)[FGS_WORK_LARGE], 1u) * FGS_CTR_STRIDE + 4] = (uint32_t)i;
        else if (v > FGS_SMALL_TILE)
            cursor[(size_t)atomicAdd(&stats->medium_tiles, 1u) * FGS_CTR_STRIDE + 2] = (uint32_t)i;
    }
    // the small class gets a list too (word 7 of the cursor slots): two thirds of a frame's
    // tiles are empty, and a sort kernel with one CTA per TILE spent most of its time starting
    // CTAs that found nothing to do.  One atomic per warp.
    {
        const bool is_small = i < tiles && v > 0ull && v <= (unsigned long long)FGS_SMALL_TILE;
        const uint32_t sm = __ballot_sync(FGS_FULL, is_small);
        if (sm) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&fgs_work(stats)[FGS_WORK_SMALL], (uint32_t)__popc(sm));
            base = __shfl_sync(FGS_FULL, base, 0);
            if (is_small)
                cursor[(size_t)(base + (uint32_t)__popc(sm & lanemask_lt())) * FGS_CTR_STRIDE + 7] = (uint32_t)i;
        }
        // lazy_sort: every pair of a tile counts as sorted unless the front kernel says otherwise
        if (i < tiles) limit[i] = 0x7fffffff;
    }
    const uint32_t nonempty = __reduce_add_sync(FGS_FULL, v ? 1u : 0u);
    if (lane == 0 && nonempty) atomicAdd(&stats->tiles_nonempty, nonempty);
    if (i == tiles - 1) {                       // the thread that owns the last tile knows M
        const unsigned long long M = excl + v;
        // K1 has already raised the flag if a CTA's table entries did not fit the list
        const bool over = M > capacity || stats->overflow != 0u;
        stats->pairs_emitted = M > 0xffffffffull ? 0xffffffffu : (uint32_t)M;
        stats->overflow = over ? 1u : 0u;       // later kernels of this frame see it and no-op
        stats->pairs_in_buffer = over ? 0u : (uint32_t)M;
        starts[tiles] = (int32_t)(M > 0x7fffffffull ? 0x7fffffffu : (uint32_t)M);
    }
}

int fgs_launch_scan_tiles(const FrameDev &f, int tiles, int64_t capacity, cudaStream_t st,
                          uint32_t heavy_thr)
{
    const unsigned slices = (unsigned)((tiles + 1023) / 1024);
    const int use_sums = slices > FGS_SCAN_DIRECT_CTAS ? 1 : 0;
    if (use_sums)
        FGS_CHAIN(k_tile_blocksums, dim3(slices), dim3(1024), 0, st, (const uint32_t *)f.tilecount,
                  f.cursor, tiles);
    FGS_CHAIN(k_scan_tiles, dim3(slices), dim3(1024), 0, st,
              f.tilecount, f.starts, f.cursor, f.tileorder, tiles, (unsigned long long)capacity, f.stats,
              use_sums, f.limit, heavy_thr);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

// Blend tile order: the band's tiles, heaviest size bin first.  Bin bases come from the
// histogram k_scan_tiles left in hdr[0..64); a CTA reserves its share of every bin with one
// atomic on the bin's cursor (hdr[64..128)) and ranks its tiles inside it in shared memory.
// Order inside a bin is arbitrary (every tile's output is independent of it).
__global__ void __launch_bounds__(1024)
k_tile_order(const int32_t *__restrict__ starts, uint32_t *__restrict__ hdr, int first_tile,
             int band_tiles, uint32_t *__restrict__ tile_ctr, const fgs_stats *__restrict__ stats,
             uint32_t heavy_thr)
{
    __shared__ uint32_t s_base[FGS_ORDER_BINS], s_cnt[FGS_ORDER_BINS], s_off[FGS_ORDER_BINS];
    fgs_pdl_wait();
    fgs_pdl_trigger();
    if (stats->overflow) return;
    const int t = threadIdx.x;
    if (t < FGS_ORDER_BINS) s_cnt[t] = 0u;
    if (t < 32) {                                   // exclusive scan of the 64 bin counts
        const uint32_t c0 = hdr[2 * t], c1 = hdr[2 * t + 1];
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(FGS_FULL, incl, o);
            if (t >= o) incl += u;
        }
        s_base[2 * t] = incl - c0 - c1;
        s_base[2 * t + 1] = incl - c1;
    }
    __syncthreads();
    const int i = blockIdx.x * 1024 + t;
    int bin = 0;
    uint32_t rank = 0;
    if (i < band_tiles) {
        const int tile = first_tile + i;
        bin = fgs_order_bin(fgs_order_weight((uint32_t)(starts[tile + 1] - starts[tile]), heavy_thr));
        rank = atomicAdd(&s_cnt[bin], 1u);
        // the placement kernel's per-pair fallback cursor (word 2) starts at zero every time
        // the stage is issued, not only on the frame's first pass (fgs_emit is idempotent)
        if (tile_ctr[(size_t)tile * FGS_CTR_STRIDE + 1]) tile_ctr[(size_t)tile * FGS_CTR_STRIDE + 2] = 0u;
    }
    __syncthreads();
    if (t < FGS_ORDER_BINS && s_cnt[t]) s_off[t] = atomicAdd(&hdr[FGS_ORDER_BINS + t], s_cnt[t]);
    __syncthreads();
    // Tiles outside the band are empty and were counted in the last bin by k_scan_tiles;
    // only the band's tiles are placed, so the first band_tiles entries are exactly the band.
    if (i < band_tiles) hdr[FGS_ORDER_HDR + s_base[bin] + s_off[bin] + rank] = (uint32_t)(first_tile + i);
    // the last CTA out rewinds the cursors, so running the stage again on the same frame
    // (fgs_emit is otherwise idempotent) rebuilds the same order instead of writing past it
    __syncthreads();
    if (t == 0 && atomicAdd(&hdr[2 * FGS_ORDER_BINS], 1u) == gridDim.x - 1) {
        for (int b = 0; b < FGS_ORDER_BINS; ++b) hdr[FGS_ORDER_BINS + b] = 0u;
        hdr[2 * FGS_ORDER_BINS] = 0u;
    }
}

int fgs_launch_tile_order(const FrameDev &f, int grid_w, int band0, int band1, cudaStream_t st,
                          uint32_t heavy_thr)
{
    if (band1 < band0) return FGS_OK;
    const int band_tiles = (band1 - band0 + 1) * grid_w;
    FGS_CHAIN(k_tile_order, dim3((unsigned)((band_tiles + 1023) / 1024)), dim3(1024), 0, st,
              f.starts, f.tileorder, band0 * grid_w, band_tiles, f.tilecount, f.stats, heavy_thr);
    FGS_CHECK_LAUNCH();
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
// K3 (TILE_BUCKET): the runs of every regular preprocess CTA, from the stage into the tile
// buckets.  One CTA per preprocess CTA: its table list gives, per run, the tile, the range
// reserved in the tile's bucket and the run's offset in the CTA's record block; the range
// table (k_scan_tiles) turns that into positions.  A pure streaming copy: coalesced reads of
// the block, runs written as contiguous segments.
// ---------------------------------------------------------------------------
#ifndef FGS_SCATTER_THREADS
#define FGS_SCATTER_THREADS 128
#endif
// One CTA of four warps per preprocess CTA; warp w takes the table entries w, w + 4, ...:
// lane l fetches entry 4 l + w (tile, bucket range, run offset) and the tile's bucket start --
// two round trips for up to 32 runs per warp -- and the warp then copies its runs one after
// the other, 32 records per step (a run of a Morton-ordered scene is ~30 records).  No shared
// memory, no barrier.
#ifndef FGS_SCATTER_MINB
#define FGS_SCATTER_MINB 12      // 40 registers: the copy is latency-bound, it wants the warps (47 registers: 178 -> 216 us)
#endif
__global__ void __launch_bounds__(FGS_SCATTER_THREADS, FGS_SCATTER_MINB)
k_scatter_runs(const uint4 *__restrict__ ctainfo, const uint4 *__restrict__ tablelist,
               const int32_t *__restrict__ starts, const uint64_t *__restrict__ stage,
               uint64_t *__restrict__ rec, const fgs_stats *__restrict__ stats)
{
    fgs_pdl_wait();
    fgs_pdl_trigger();
    constexpr uint32_t W = FGS_SCATTER_THREADS / 32;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t over = stats->overflow;
    const uint4 info = ctainfo[blockIdx.x];              // (list base, entries, records, stage base)
    if (over || info.w == FGS_CTA_NO_STAGE || info.z == 0u) return;
    const uint64_t *blk = stage + info.w;
    for (uint32_t eb = w; eb < info.y; eb += 32u * W) {  // this warp's entries eb, eb + W, ...
        uint32_t mydst = 0, myoff = 0, mycnt = 0;
        const uint32_t mine = eb + lane * W;
        if (mine < info.y) {
            const uint4 ent = tablelist[info.x + mine];  // (tile, range base, pairs, slot | offset)
            myoff = ent.w & 0xffffu;
            mycnt = ent.z;
            mydst = (uint32_t)starts[ent.x] + ent.y;
        }
        const uint32_t left = (info.y - eb + W - 1u) / W;
        const int n = left < 32u ? (int)left : 32;
        // four runs per step: their first 32 records are requested together, then stored
        for (int k0 = 0; k0 < n; k0 += 4) {
            uint32_t dst[4], off[4], cnt[4];
            uint64_t v[4], v2[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                dst[u] = __shfl_sync(FGS_FULL, mydst, (k0 + u) & 31);
                off[u] = __shfl_sync(FGS_FULL, myoff, (k0 + u) & 31);
                cnt[u] = k0 + u < n ? __shfl_sync(FGS_FULL, mycnt, (k0 + u) & 31) : 0u;
                v[u] = lane < cnt[u] ? blk[off[u] + lane] : 0ull;
                // (a run is ~33 records: its few records beyond 32 go out with the first 32,
                // not in a dependent second round trip)
                v2[u] = lane + 32u < cnt[u] ? blk[off[u] + lane + 32u] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (lane < cnt[u]) rec[dst[u] + lane] = v[u];
                if (lane + 32u < cnt[u]) rec[dst[u] + lane + 32u] = v2[u];
                for (uint32_t j = lane + 64u; j < cnt[u]; j += 32u) rec[dst[u] + j] = blk[off[u] + j];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3 fallback (TILE_BUCKET): the second walk, for the preprocess CTAs on the fallback list
// (a pair without a table entry, more pairs than the record block holds: caller-order scenes,
// huge splats, very dense scenes).  The CTA reloads its tile table from the frame's list (same
// slots, so lookups probe exactly as K1's inserts did), ranks every pair inside its
// (CTA, tile) range with a shared-memory atomic, gathers the records by tile in the
// write-combining buffer and writes them out as contiguous runs.  Persistent CTAs over the
// list; an empty list costs one launch.
// ---------------------------------------------------------------------------
struct PlaceSmem {
    TileTable tab;
    uint32_t gbase[FGS_HT_SIZE];
    uint16_t wcoff[FGS_HT_SIZE];
    uint32_t wcdst[FGS_WC_CAP];
    uint64_t wcrec[FGS_WC_CAP];
};

template <int STRAT>
__global__ void __launch_bounds__(FGS_PRE_THREADS, FGS_PLACE_MINBLOCKS)
k_place(int P, int width, int height, int grid_w, int band0, int band1,
        const uint32_t *__restrict__ orig, FrameDev f)
{
    extern __shared__ __align__(16) unsigned char place_raw[];
    PlaceSmem &S = *reinterpret_cast<PlaceSmem *>(place_raw);
    fgs_pdl_wait();
    fgs_pdl_trigger();
    if (f.stats->overflow) return;                       // uniform: grow and re-run
    const uint32_t nfb = fgs_work(f.stats)[FGS_WORK_FB_CTAS];
    for (uint32_t it = blockIdx.x; it < nfb; it += gridDim.x) {
    const int cta = (int)f.fb_list[it];
    const int g = cta * FGS_PRE_THREADS + threadIdx.x;
    const bool live = g < P;
    const uint32_t cnt = live ? f.counts[g] : 0u;
    const uint4 info = f.ctainfo[cta];                   // (list base, entries, staged records)
    // The Gaussian's own inputs are independent of the table: they go out with the first
    // round trip's successors (table list, bucket starts) instead of after the barriers.
    ushort4 r = make_ushort4(0, 0, 0, 0);
    uint64_t pm = 0;
    uint32_t bits = 0, og = 0;
    if (live) {                                          // not `if (cnt)`: that would chain them
        r = f.rects[g];                                  // behind the count's round trip
        if (STRAT == FGS_PRECISE) pm = f.passmask[g];    // (stale when cnt == 0, and unused)
        bits = __float_as_uint(f.depth[g]);
        og = orig[g];
    }
    __syncthreads();                                     // the previous CTA's flush is done
    if (__syncthreads_or(cnt != 0u) == 0) continue;      // uniform per block
    for (int i = threadIdx.x; i < FGS_HT_SIZE; i += FGS_PRE_THREADS) S.tab.key[i] = FGS_HT_EMPTY;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < info.y; i += FGS_PRE_THREADS) {
        const uint4 ent = f.tablelist[info.x + i];       // (tile, range base, pairs, slot | wc offset)
        const uint32_t e = ent.w >> 16;
        S.tab.key[e] = ent.x;
        S.tab.val[e] = 0u;
        S.gbase[e] = (uint32_t)f.starts[ent.x] + ent.y;
        S.wcoff[e] = (uint16_t)(ent.w & 0xffffu);
    }
    __syncthreads();

    TileJob job;
    job.cand = 0;
    job.cx = job.cy = job.a = job.b = job.c = job.keff = 0.f;
    job.tx0 = job.ty0 = 0;
    job.nx = 1;
    job.mask = 0;
    if (cnt) {
        const int by0 = (int)r.y > band0 ? (int)r.y : band0;
        const int by1 = (int)r.w < band1 ? (int)r.w : band1;
        job.tx0 = r.x; job.ty0 = by0; job.nx = (int)r.z - (int)r.x + 1;
        job.cand = (uint32_t)job.nx * (uint32_t)(by1 - by0 + 1);
        if (STRAT == FGS_PRECISE) {
            if (job.cand <= FGS_MASK_CAND) {
                job.mask = pm;                            // K1's verdicts, no test needed
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
    }
    const BinCtx bc{&S.tab, f.tilecount, nullptr, nullptr, nullptr,
                    S.gbase, S.wcoff, S.wcrec, S.wcdst, f.starts};
    // records carry the caller's Gaussian index: the reference's pair value and tie-break
    // (measured: letting each lane walk the set bits of its own mask instead -- no owner
    // search, no shuffles -- is 13 % slower: the divergence costs more than the walk)
    warp_walk_tiles<STRAT == FGS_PRECISE, WALK_PLACE>(job, width, height, grid_w, 0, bits,
                                                      og, f.keys[0], nullptr, &bc);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < info.z; i += FGS_PRE_THREADS) f.keys[0][S.wcdst[i]] = S.wcrec[i];
    }
}

int fgs_launch_emit(const SceneDev &sc, int64_t P, const CamDev &cam, int strategy, int band0,
                    int band1, int bucket, const FrameDev &f, cudaStream_t st, uint32_t heavy_thr)
{
    if (bucket) {                       // also for an empty scene: the blend reads the order
        const int rc = fgs_launch_tile_order(f, cam.grid_w, band0, band1, st, heavy_thr);
        if (rc) return rc;
    }
    if (P == 0) return FGS_OK;
    const unsigned blocks = (unsigned)((P + FGS_PRE_THREADS - 1) / FGS_PRE_THREADS);
    if (bucket) {
        static FgsOncePerDevice attr_once;
        int attr_dev = 0;
        if (attr_once.need(&attr_dev)) {
            cudaError_t e = cudaFuncSetAttribute(k_place<FGS_PRECISE>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)sizeof(PlaceSmem));
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k_place<FGS_TIGHT_AABB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(PlaceSmem));
            if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
            attr_once.mark(attr_dev);
        }
        FGS_CHAIN(k_scatter_runs, dim3(blocks), dim3(FGS_SCATTER_THREADS), 0, st,
                  (const uint4 *)f.ctainfo, (const uint4 *)f.tablelist, (const int32_t *)f.starts,
                  (const uint64_t *)f.stage, f.keys[0], (const fgs_stats *)f.stats);
        FGS_CHECK_LAUNCH();
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned pgrid = blocks < (unsigned)(FGS_PLACE_MINBLOCKS * sms) ? blocks
                                                                              : (unsigned)(FGS_PLACE_MINBLOCKS * sms);
        if (strategy == FGS_PRECISE)
            FGS_CHAIN(k_place<FGS_PRECISE>, dim3(pgrid), dim3(FGS_PRE_THREADS), sizeof(PlaceSmem), st,
                      (int)P, cam.width, cam.height, cam.grid_w, band0, band1, sc.orig, f);
        else
            FGS_CHAIN(k_place<FGS_TIGHT_AABB>, dim3(pgrid), dim3(FGS_PRE_THREADS), sizeof(PlaceSmem), st,
                      (int)P, cam.width, cam.height, cam.grid_w, band0, band1, sc.orig, f);
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
