// K6 per-tile alpha blending.
//
// Replaces render.py:135-252 (_composite_pipelined), 273-310 (render_frame).
//
// One CTA per 16x16 tile, one thread per pixel, one warp per 8x4 pixel block.
// Within a batch a warp first culls 32 pairs at a time against its block (one
// pair per lane, ballot) and only walks the survivors, so the per-pixel loop
// never spends issue slots on splats whose rectangle misses the whole block.
// The tile's sorted pair slice
// is consumed in batches of 256 through a two-step prefetch pipeline (the
// FlashGS scheme, at batch granularity): while batch i is
// blended out of shared memory, the 48-byte splat rows of batch i+1 are in
// flight as cp.async gathers (global -> shared, no register staging) and the
// pair indices of batch i+2 are in flight as plain loads.
//
// Numerics.  The three skips of the reference (extent rectangle, power
// cutoff, alpha < tau) are hard thresholds, so `s` is evaluated in the
// reference's exact float32 operation order with individually rounded
// operations (no FMA).  exp(-s):
//   EXACT  : double-precision port of the published expf algorithm glibc uses
//            (32-entry 2^(i/32) table + cubic), accumulations unfused: the
//            frame is bit-identical to the reference's.
//   default: ex2.approx.ftz.f32; when alpha lands within 1e-5 (relative) of
//            tau the exact path decides, so the alpha<tau skip never flips.
// Whole-tile early exit when every pixel's transmittance is below 1e-4
// (render.py:154,178,228-229) via __syncthreads_and; a warp whose 32 pixels
// are all finished skips the rest of a batch.

#include "fgs_common.cuh"
#include <stdlib.h>

namespace {

__device__ __constant__ unsigned long long c_exp2_tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

// expf as glibc computes it for |x| < 88 (sysdeps/ieee754/flt-32/e_expf.c,
// EXP2F_TABLE_BITS = 5): bit-equal to libm on 2e8 samples in [-11.5, 0.5].
__device__ __forceinline__ float expf_exact(float x, const unsigned long long *tab)
{
    const double InvLn2N = 0x1.71547652b82fep+0 * 32.0, Shift = 0x1.8p52;
    const double C0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
    const double C1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const double z = dm(InvLn2N, (double)x);
    double kd = da(z, Shift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = ds(kd, Shift);
    const double r = ds(z, kd);
    const unsigned long long t = tab[ki & 31ull] + (ki << 47);
    const double s = __longlong_as_double((long long)t);
    const double p = da(dm(C0, r), C1);
    const double r2 = dm(r, r);
    double y = da(dm(C2, r), 1.0);
    y = da(dm(p, r2), y);
    return (float)dm(y, s);
}

__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Second-level cull (after the extent rectangle): does the cutoff ellipse s <= k/2 of a
// pair miss the whole block of pixel centres [u0,u1] x [v0,v1] (offsets from the splat
// centre)?  s = (a u^2 + c v^2)/2 + b u v is convex, so over a rectangle that does not
// contain the centre its minimum lies on an edge the centre is outside of; each such edge
// is a 1-D parabola.  The comparison carries a margin of 1e-4 of the largest term
// magnitude in the block -- 100x the rounding of this float32 evaluation and of the
// per-pixel render.py:213 evaluation it stands in for -- so a pair is only dropped when
// every pixel of the block would have failed render.py:214 anyway.  NaNs keep the pair.
__device__ __forceinline__ bool ellipse_misses_block(float a, float b, float c, float k, float u0,
                                                     float u1, float v0, float v1)
{
    const bool out_u = u0 > 0.0f || u1 < 0.0f, out_v = v0 > 0.0f || v1 < 0.0f;
    if (!out_u && !out_v) return false;                   // centre inside the block
    const float ue = u0 > 0.0f ? u0 : u1;                 // the edge facing the centre
    const float ve = v0 > 0.0f ? v0 : v1;
    float qmin = __int_as_float(0x7f800000);
    if (out_u) {                                          // edge u = ue, v in [v0, v1]
        const float bu = b * ue;
        const float vs = fminf(fmaxf(__fdividef(-bu, c), v0), v1);
        qmin = fmaf(0.5f * a * ue, ue, fmaf(0.5f * c * vs, vs, bu * vs));
    }
    if (out_v) {                                          // edge v = ve, u in [u0, u1]
        const float bv = b * ve;
        const float us = fminf(fmaxf(__fdividef(-bv, a), u0), u1);
        qmin = fminf(qmin, fmaf(0.5f * c * ve, ve, fmaf(0.5f * a * us, us, bv * us)));
    }
    const float um = fmaxf(fabsf(u0), fabsf(u1)), vm = fmaxf(fabsf(v0), fabsf(v1));
    const float mag = fmaf(fabsf(a) * um, um, fmaf(fabsf(c) * vm, vm, 2.0f * fabsf(b) * um * vm));
    return qmin > fmaf(1e-4f, mag, 0.5f * k * 1.001f);
}

struct BlendSmem {
    float4 row[2][FGS_BLEND_BATCH][3];     // (cx,cy,a,b) (c,op,k,r) (g,b,hx,hy)
    float  z[2][FGS_BLEND_BATCH];          // camera depth of the pair's Gaussian (extras)
    uint32_t touched[2][FGS_BLEND_BATCH];  // contrib flags of the batch
    unsigned long long tab[32];
};

// COUNT (diagnostic, EXACT only): classify every (pixel, pair) evaluation the reference's
// naive loop performs (render.py:106-129) -- rejected by the extent rectangle (:111),
// by the cutoff (:114), by alpha < tau (:119), or blended -- and count, per tile, the
// pairs visited before the tile's last pixel stops (M_proc of SURVEY.md 8(d)).  The
// warp-level culls are switched off so that every live pixel classifies every pair
// itself.  evals[0..3] = the four classes, [4] = M_proc, [5] = pixels.
// lazy_sort (both blend kernels).  `limit` (first pass): only the first limit[tile] pairs of
// the tile's bucket are in order; a tile whose pixels are not all finished when that front is
// used up is appended to `redo_list` and NOT written (nor counted) -- the second pass, REDO,
// takes the tiles of that list in full with persistent CTAs after k_tile_sort_redo has sorted
// them.  The last CTA of the second pass publishes stats->redo_tiles and rewinds the cursor,
// so the stage can be re-issued on the frame.
template <typename Body>
__device__ __forceinline__ void blend_redo_pass(fgs_stats *stats, const uint32_t *redo_list, Body body)
{
    uint32_t *work = fgs_work(stats);
    const uint32_t cnt = work[FGS_WORK_REDO];
    for (uint32_t it = blockIdx.x; it < cnt; it += gridDim.x) {
        body((int)redo_list[it]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&work[FGS_WORK_REDO_OUT], 1u) == gridDim.x - 1u) {
            stats->redo_tiles = cnt;
            work[FGS_WORK_REDO] = 0u;
            work[FGS_WORK_REDO_OUT] = 0u;
        }
    }
}

template <bool EXACT, bool CONTRIB, bool EXTRAS, bool COUNT = false, bool REDO = false>
__global__ void __launch_bounds__(256)
k_blend(const float *__restrict__ splat, const float *__restrict__ gdepth,
        const uint32_t *__restrict__ vals, const uint32_t *__restrict__ inv,
        const int32_t *__restrict__ starts, const uint32_t *__restrict__ order, int width,
        int height, int grid_w, int first_tile, float bg0, float bg1, float bg2, float tau,
        float *__restrict__ rgb, float *__restrict__ alpha_out, float *__restrict__ depth_out,
        uint8_t *__restrict__ contrib, fgs_stats *__restrict__ stats,
        unsigned long long *__restrict__ evals = nullptr,
        const int32_t *__restrict__ limit = nullptr, uint32_t *__restrict__ redo_list = nullptr)
{
    __shared__ BlendSmem S;
    __shared__ uint32_t s_mproc;
    if (REDO) fgs_pdl_wait();
    if (COUNT && threadIdx.x == 0) s_mproc = 0u;
    if (stats != nullptr && stats->overflow) return;   // frame is re-run with a larger buffer
    const int tid = threadIdx.x;
    if (tid < 32) S.tab[tid] = c_exp2_tab[tid];
    const auto tile_body = [&](const int tile) {
    uint32_t ev_rect = 0, ev_cut = 0, ev_alpha = 0, ev_blend = 0, visited = 0;
    const int ty = tile / grid_w, tx = tile - ty * grid_w;
    // each warp owns an 8x4 pixel block (squarer than 16x2, so fewer splat
    // rectangles reach it); lanes run row-major inside the block
    const int lane = tid & 31, wq = tid >> 5;
    const int bx = tx * FGS_TILE + (wq & 1) * 8, by = ty * FGS_TILE + (wq >> 1) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    // pixel-centre bounds of the block, for the warp-level rectangle cull
    const float wx_lo = (float)bx + 0.5f, wx_hi = (float)bx + 7.5f;
    const float wy_lo = (float)by + 0.5f, wy_hi = (float)by + 3.5f;
    const bool inside = px < width && py < height;
    // A finished pixel (outside the image, or T < 1e-4) parks its x centre at +inf: every
    // later extent test then rejects it (render.py:203-204) without a separate flag.
    const float kInf = __int_as_float(0x7f800000);
    float fx = inside ? (float)px + 0.5f : kInf;
    const float fy = (float)py + 0.5f;
    // alpha within 1e-5 (relative) of tau <=> its bit pattern within [band_lo, band_lo+band_span]
    const uint32_t band_lo = __float_as_uint(tau * (1.0f - 1e-5f));
    const uint32_t band_span = __float_as_uint(tau * (1.0f + 1e-5f)) - band_lo;

    const int start = starts[tile];
    int n = starts[tile + 1] - start;
    bool cut = false, done_all = false;       // lazy_sort: only a sorted front of the tile exists
    if (!REDO && limit != nullptr) {
        const int l = limit[tile];
        cut = l < n;
        n = cut ? l : n;
    }

    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, dz = 0.0f;
    uint32_t ncontrib = 0;

    const int nb = (n + FGS_BLEND_BATCH - 1) / FGS_BLEND_BATCH;
    // A pair's value is the caller's Gaussian index; rows live at the Gaussian's slot
    // (inv: index -> slot, null = identity).  Three steps in flight: values of batch b+3,
    // their slots for batch b+2, row gathers of batch b+1.
    const auto slot_of = [&](uint32_t v) { return inv ? inv[v] : v; };
    // prologue: rows of batch 0 in flight, slots of batch 1, values of batch 2
    if (tid < n) {
        const uint32_t g = slot_of(vals[start + tid]);
        const float4 *src = (const float4 *)(splat + (size_t)g * 12);
        cp_async16(&S.row[0][tid][0], src);
        cp_async16(&S.row[0][tid][1], src + 1);
        cp_async16(&S.row[0][tid][2], src + 2);
        if (EXTRAS) S.z[0][tid] = gdepth ? gdepth[g] : 0.0f;
    }
    cp_async_commit();
    uint32_t idx_next = (FGS_BLEND_BATCH + tid < n) ? slot_of(vals[start + FGS_BLEND_BATCH + tid]) : 0u;
    uint32_t val_next2 = (2 * FGS_BLEND_BATCH + tid < n) ? vals[start + 2 * FGS_BLEND_BATCH + tid] : 0u;

    int b = 0;
    for (; b < nb; ++b) {
        const int cur = b & 1, nxt = cur ^ 1;
        // step 1: gather the rows of batch b+1 (their slots arrived during batch b-1)
        if ((b + 1) * FGS_BLEND_BATCH + tid < n) {
            const float4 *src = (const float4 *)(splat + (size_t)idx_next * 12);
            cp_async16(&S.row[nxt][tid][0], src);
            cp_async16(&S.row[nxt][tid][1], src + 1);
            cp_async16(&S.row[nxt][tid][2], src + 2);
            if (EXTRAS) S.z[nxt][tid] = gdepth ? gdepth[idx_next] : 0.0f;
        }
        cp_async_commit();
        // step 2: slots of batch b+2 (values arrived during batch b-1), values of batch b+3
        const uint32_t idx_next2 = ((b + 2) * FGS_BLEND_BATCH + tid < n) ? slot_of(val_next2) : 0u;
        const int i3 = (b + 3) * FGS_BLEND_BATCH + tid;
        val_next2 = i3 < n ? vals[start + i3] : 0u;
        if (CONTRIB) S.touched[cur][tid] = 0u;
        cp_async_wait<1>();
        __syncthreads();

        // step 3: blend batch b
        const int cnt = n - b * FGS_BLEND_BATCH < FGS_BLEND_BATCH ? n - b * FGS_BLEND_BATCH
                                                                  : FGS_BLEND_BATCH;
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            if (__all_sync(FGS_FULL, fx == kInf)) break;
            // warp-level cull, one pair per lane: a pair whose extent rectangle misses the
            // whole 8x4 block is rejected by every pixel's render.py:211 test (float32
            // subtraction is monotone, so testing the block's extreme centres is exact)
            const int jl = c0 + lane;
            bool keep = false;
            if (COUNT) keep = jl < cnt;
            else if (jl < cnt) {
                const float4 q0 = S.row[cur][jl][0];
                const float4 q1 = S.row[cur][jl][1];
                const float4 q2 = S.row[cur][jl][2];
                const float u0 = fs(wx_lo, q0.x), u1 = fs(wx_hi, q0.x);
                const float v0 = fs(wy_lo, q0.y), v1 = fs(wy_hi, q0.y);
                keep = !(u0 > q2.z || u1 < -q2.z || v0 > q2.w || v1 < -q2.w);
                if (keep) keep = !ellipse_misses_block(q0.z, q0.w, q1.x, q1.z, u0, u1, v0, v1);
            }
            const uint32_t live = __ballot_sync(FGS_FULL, keep);
            // Fixed trip count with a warp-uniform skip per pair, unrolled: a survivor's row
            // address and contrib slot are then immediate offsets from the chunk base.  (A
            // find-first-set loop over `live` spends ten uniform-datapath instructions per
            // survivor on bit scanning and address arithmetic, a fifth of the body.)
            constexpr int kUnroll = FGS_BLEND_UNROLL;
#pragma unroll kUnroll
            for (int jj = 0; jj < 32; ++jj) {
                if (!((live >> jj) & 1u)) continue;
                const int j = c0 + jj;
                // Straight-line body: a lane the reference would skip (render.py:211, 214,
                // 219) carries alpha = 0 through the blend, which leaves C and T bit-for-bit
                // unchanged.  With 18-28 of 32 lanes live per surviving pair, early-out
                // branches almost never skip work but cost reconvergence bookkeeping.
                const float4 r0 = S.row[cur][j][0];
                const float4 r1 = S.row[cur][j][1];
                const float4 r2 = S.row[cur][j][2];
                const float dx = fs(fx, r0.x), dy = fs(fy, r0.y);
                // render.py:213  s = 0.5*(a dx dx + c dy dy) + b dx dy, unfused
                const float s = fa(fm(0.5f, fa(fm(fm(r0.z, dx), dx), fm(fm(r1.x, dy), dy))),
                                   fm(fm(r0.w, dx), dy));
                // render.py:211 extent rectangle (exact float32 compares), :214 cutoff
                bool on = !(fabsf(dx) > r2.z) && !(fabsf(dy) > r2.w) && !(s > fm(0.5f, r1.z));
                const bool ev_live = COUNT && fx != kInf;             // render.py:108 pixel still open
                if (ev_live) {
                    if (fabsf(dx) > r2.z || fabsf(dy) > r2.w) ++ev_rect;
                    else if (!on) ++ev_cut;
                }
                float al;
                if (EXACT) {
                    al = on ? fm(r1.y, expf_exact(-s, S.tab)) : 0.0f;
                } else {
                    al = r1.y * ex2_approx(-s * 1.4426950408889634f);
                    if (on && __float_as_uint(al) - band_lo <= band_span)
                        al = fm(r1.y, expf_exact(-s, S.tab));
                }
                al = al > FGS_ALPHA_CAP ? FGS_ALPHA_CAP : al;     // render.py:217-218
                if (ev_live && on) { if (al < tau) ++ev_alpha; else ++ev_blend; }
                on = on && !(al < tau);                           // render.py:219
                al = on ? al : 0.0f;
                if (EXACT) {
                    const float wgt = fm(al, T);
                    cr = fa(cr, fm(r1.w, wgt));
                    cg = fa(cg, fm(r2.x, wgt));
                    cb = fa(cb, fm(r2.y, wgt));
                    if (EXTRAS) dz = fa(dz, fm(S.z[cur][j], wgt));
                    T = fm(T, fs(1.0f, al));
                } else {
                    const float wgt = al * T;
                    cr = fmaf(r1.w, wgt, cr);
                    cg = fmaf(r2.x, wgt, cg);
                    cb = fmaf(r2.y, wgt, cb);
                    if (EXTRAS) dz = fmaf(S.z[cur][j], wgt, dz);
                    T = T * (1.0f - al);
                }
                if (CONTRIB && on) S.touched[cur][j] = 1u;
                if (COUNT && ev_live && T < FGS_T_STOP) visited = (uint32_t)(b * FGS_BLEND_BATCH + j + 1);
                if (T < FGS_T_STOP) fx = kInf;                    // render.py:228
            }
        }
        const bool all_done = __syncthreads_and(fx == kInf);
        if (CONTRIB) {
            if (tid < cnt) {
                const uint32_t t = S.touched[cur][tid];
                contrib[start + b * FGS_BLEND_BATCH + tid] = (uint8_t)t;
                ncontrib += t;
            }
        }
        idx_next = idx_next2;
        if (all_done) { done_all = true; ++b; break; }
    }
    cp_async_wait<0>();
    if (cut && !done_all) {                   // uniform: the sorted front was not enough
        if (tid == 0) redo_list[atomicAdd(&fgs_work(stats)[FGS_WORK_REDO], 1u)] = (uint32_t)tile;
        return;
    }
    if (cut) n = starts[tile + 1] - start;
    if (CONTRIB)   // pairs behind a whole-tile early exit never touched a pixel
        for (int i = b * FGS_BLEND_BATCH + tid; i < n; i += FGS_BLEND_BATCH) contrib[start + i] = 0;

    if (inside) {
        const size_t o = (size_t)py * width + px;
        if (EXACT) {
            rgb[3 * o + 0] = fa(cr, fm(T, bg0));                  // render.py:250-252
            rgb[3 * o + 1] = fa(cg, fm(T, bg1));
            rgb[3 * o + 2] = fa(cb, fm(T, bg2));
        } else {
            rgb[3 * o + 0] = fmaf(T, bg0, cr);
            rgb[3 * o + 1] = fmaf(T, bg1, cg);
            rgb[3 * o + 2] = fmaf(T, bg2, cb);
        }
        if (EXTRAS) {
            if (alpha_out) alpha_out[o] = 1.0f - T;
            if (depth_out) depth_out[o] = dz;
        }
    }
    if (CONTRIB) {
        ncontrib = __reduce_add_sync(FGS_FULL, ncontrib);
        if ((tid & 31) == 0 && ncontrib) atomicAdd(&stats->pairs_contributing, ncontrib);
    }
    if (COUNT && evals != nullptr) {
        // a pixel that never stopped visited the whole list; pixels outside the image none
        if (inside && fx != kInf) visited = (uint32_t)n;
        if (!inside) visited = 0u;
        __syncthreads();                    // s_mproc's initial zero (an empty tile has no barrier before here)
        const uint32_t vmax = __reduce_max_sync(FGS_FULL, visited);
        if ((tid & 31) == 0) atomicMax(&s_mproc, vmax);
        const uint32_t c0 = __reduce_add_sync(FGS_FULL, ev_rect), c1 = __reduce_add_sync(FGS_FULL, ev_cut);
        const uint32_t c2 = __reduce_add_sync(FGS_FULL, ev_alpha), c3 = __reduce_add_sync(FGS_FULL, ev_blend);
        const uint32_t c5 = __reduce_add_sync(FGS_FULL, inside ? 1u : 0u);
        if ((tid & 31) == 0) {
            if (c0) atomicAdd(&evals[0], (unsigned long long)c0);
            if (c1) atomicAdd(&evals[1], (unsigned long long)c1);
            if (c2) atomicAdd(&evals[2], (unsigned long long)c2);
            if (c3) atomicAdd(&evals[3], (unsigned long long)c3);
            if (c5) atomicAdd(&evals[5], (unsigned long long)c5);
        }
        __syncthreads();
        if (tid == 0 && s_mproc) atomicAdd(&evals[4], (unsigned long long)s_mproc);
    }
    };  // tile_body
    if (REDO) {
        blend_redo_pass(stats, redo_list, tile_body);
    } else {
        // CTA i takes the i-th tile of the blend order (heaviest first), or of the band in
        // raster order when no order was built
        tile_body(order ? (int)order[blockIdx.x] : first_tile + (int)blockIdx.x);
    }
}

// ---------------------------------------------------------------------------------------
// k_blend2: the default-mode blend, two pixels per thread on Blackwell's packed float32
// pipe (FFMA2 / FMUL2 / FADD2: one issue slot for two lanes' worth of float32 work).
//
// One CTA of 128 threads per 16x16 tile; a warp owns an 8x8 pixel block and lane l the
// pixels (x, y) and (x, y+4), which share dx, so the quadratic form is a Horner chain in
// the packed dy:   -log2(e) * s = dy * (c2*dy + b2*dx) + a2*dx*dx   (a2 = -log2e/2 * a ...)
// = 4 scalar + 3 packed operations for two pixels against 22 scalar ones in k_blend.
//
// The reference's three skips (render.py:211 extent rectangle, :214 s > k/2, :219
// alpha < tau) collapse into ONE comparison, alpha >= thr with thr = max(tau, op*exp(-k/2)):
//   * s > k/2  <=>  op*exp(-s) < op*exp(-k/2)  (monotone), and
//   * the extent rectangle is the bounding box of the cutoff ellipse (binning.py:181-182),
//     so a pixel outside it has s > k/2 -- the transform pass below CHECKS that per pair
//     from the row itself (hx^2 >= k*c/det, hy^2 >= k*a/det); a row that does not satisfy
//     it (hand-made rows through fgs_blend_tiles) is blended by the exact path entirely.
// Those equivalences hold in real arithmetic.  In float32 the fused evaluation here and the
// reference's unfused one differ by at most ~1.3e-5*kappa relative in alpha
// (kappa = a*c/det bounds the cancellation between the three terms), so whenever alpha
// lands within eps = thr*(2e-5 + 2.5e-5*kappa) of thr the lane recomputes the pair the
// reference's way -- unfused s, the three tests in order, glibc-equivalent expf -- and that
// verdict (and alpha) is used.  Outside the band both evaluations agree on the verdict.
// A band hit is rare (~1e-4 of evaluations), the exact path is a warp-level branch.
//
// Pipeline: as k_blend, at 128 pairs per batch; the thread that gathered a pair's row also
// transforms it (a2, b2, c2, thr, eps) into the batch's fast-row table before the barrier.

typedef float2 pk2;                   // two float32 lanes: x = pixel (x, y), y = pixel (x, y+4)
__device__ __forceinline__ pk2 pk(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ void upk(pk2 v, float &lo, float &hi) { lo = v.x; hi = v.y; }
__device__ __forceinline__ pk2 mul2(pk2 a, pk2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ pk2 add2(pk2 a, pk2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ pk2 sub2(pk2 a, pk2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ pk2 fma2(pk2 a, pk2 b, pk2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ pk2 bc(float v) { return pk(v, v); }   // broadcast operand (R.F32 in SASS)

#define FGS_B2_THREADS 128
#define FGS_B2_BATCH   128
#ifndef FGS_B2_MINCTAS
#define FGS_B2_MINCTAS 9       // 56 registers, no spills: 36 warps/SM (10 = 48 registers + spills: slower)
#endif
#ifndef FGS_B2_UNROLL
#define FGS_B2_UNROLL  16
#endif

struct Blend2Smem {
    float4 row[2][FGS_B2_BATCH][3];    // reference rows (cp.async destination)
    float4 fast[FGS_B2_BATCH][3];      // (cx,cy,a2,b2) (c2,op,thr,eps) (r,g,b,z)
    float  z[2][FGS_B2_BATCH];
    uint32_t touched[FGS_B2_BATCH];
    unsigned long long tab[32];
};

// One pixel of a pair the reference's way (render.py:203-219): returns alpha, 0 if skipped.
__device__ __forceinline__ float alpha_exact(const float4 r0, const float4 r1, const float4 r2,
                                             float fx, float fy, float tau,
                                             const unsigned long long *tab)
{
    const float dx = fs(fx, r0.x), dy = fs(fy, r0.y);
    const float s = fa(fm(0.5f, fa(fm(fm(r0.z, dx), dx), fm(fm(r1.x, dy), dy))),
                       fm(fm(r0.w, dx), dy));
    if (fabsf(dx) > r2.z || fabsf(dy) > r2.w || s > fm(0.5f, r1.z)) return 0.0f;
    float al = fm(r1.y, expf_exact(-s, tab));
    al = al > FGS_ALPHA_CAP ? FGS_ALPHA_CAP : al;
    return al < tau ? 0.0f : al;
}

// The rare path of k_blend2, out of line so the unrolled survivor loop stays compact in the
// instruction cache (inlined it cost 5 us of 177 on C2): both pixels of a lane the
// reference's way.
__device__ __noinline__ float2 alpha_exact_pair(const float4 *row, float fx, float fy0, float fy1,
                                                float tau, const unsigned long long *tab)
{
    const float4 r0 = row[0], r1 = row[1], r2 = row[2];
    return make_float2(alpha_exact(r0, r1, r2, fx, fy0, tau, tab),
                       alpha_exact(r0, r1, r2, fx, fy1, tau, tab));
}

#ifndef FGS_B2_REDO_MINCTAS
#define FGS_B2_REDO_MINCTAS FGS_B2_MINCTAS
#endif
template <bool CONTRIB, bool EXTRAS, bool REDO = false>
__global__ void __launch_bounds__(FGS_B2_THREADS, REDO ? FGS_B2_REDO_MINCTAS : FGS_B2_MINCTAS)
k_blend2(const float *__restrict__ splat, const float *__restrict__ gdepth,
         const uint32_t *__restrict__ vals, const uint32_t *__restrict__ inv,
         const int32_t *__restrict__ starts, const uint32_t *__restrict__ order, int width,
         int height, int grid_w, int first_tile,
         float bg0, float bg1, float bg2, float tau, float *__restrict__ rgb,
         float *__restrict__ alpha_out, float *__restrict__ depth_out,
         uint8_t *__restrict__ contrib, fgs_stats *__restrict__ stats,
         const int32_t *__restrict__ limit, uint32_t *__restrict__ redo_list)
{
    __shared__ Blend2Smem S;
    fgs_pdl_wait();            // (the tail sort kernel before it is launched the plain way and
                               // waits for every size class)
    const uint32_t over = stats != nullptr ? stats->overflow : 0u;   // consumed below, after the
                                                                     // tile lookup is out too
    constexpr int B = FGS_B2_BATCH;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wq = tid >> 5;
    if (tid < 32) S.tab[tid] = c_exp2_tab[tid];
    // CTA i takes the i-th tile of the blend order (heaviest first: longest-first list
    // scheduling by the hardware's in-order CTA dispatch), or of the band in raster order.
    // (Persistent CTAs pulling tiles from a ticket counter were slower: 72 registers, and the
    // per-tile prologue no longer overlaps other CTAs' blending -- 197 us against 177 on C2.)
    const int tile0 = REDO ? 0 : (order ? (int)order[blockIdx.x] : first_tile + (int)blockIdx.x);
    if (over) return;                                    // uniform: grow and re-run
    const auto tile_body = [&](const int tile) {
    uint32_t ncontrib = 0;
    const int ty = tile / grid_w, tx = tile - ty * grid_w;
    const int bx = tx * FGS_TILE + (wq & 1) * 8, by = ty * FGS_TILE + (wq >> 1) * 8;
    const int px = bx + (lane & 7), py0 = by + (lane >> 3), py1 = py0 + 4;
    const float wx_lo = (float)bx + 0.5f, wx_hi = (float)bx + 7.5f;
    const float wy_lo = (float)by + 0.5f, wy_hi = (float)by + 7.5f;
    const bool inside0 = px < width && py0 < height, inside1 = px < width && py1 < height;
    // A finished pixel (outside the image, or T < 1e-4, render.py:228) parks its y centre at
    // +inf: dy = inf, c2 < 0 => -log2e*s = -inf, alpha = 0 < thr, and the exact path's extent
    // test rejects it too -- no separate "live" flag in the loop.
    const float kInf = __int_as_float(0x7f800000);
    const float fx = (float)px + 0.5f;
    float fy0 = inside0 ? (float)py0 + 0.5f : kInf, fy1 = inside1 ? (float)py1 + 0.5f : kInf;
    constexpr float kL = -1.4426950408889634f;       // -log2(e)

    const int start = starts[tile];
    int n = starts[tile + 1] - start;
    bool cut = false, done_all = false;       // lazy_sort: only a sorted front of the tile exists
    if (!REDO && limit != nullptr) {
        const int l = limit[tile];
        cut = l < n;
        n = cut ? l : n;
    }

    pk2 T2 = pk(1.0f, 1.0f), cr2 = pk(0.0f, 0.0f), cg2 = cr2, cb2 = cr2, dz2 = cr2;

    const int nb = (n + B - 1) / B;
    const auto slot_of = [&](uint32_t v) { return inv ? inv[v] : v; };
    if (tid < n) {
        const uint32_t g = slot_of(vals[start + tid]);
        const float4 *src = (const float4 *)(splat + (size_t)g * 12);
        cp_async16(&S.row[0][tid][0], src);
        cp_async16(&S.row[0][tid][1], src + 1);
        cp_async16(&S.row[0][tid][2], src + 2);
        if (EXTRAS) S.z[0][tid] = gdepth ? gdepth[g] : 0.0f;
    }
    cp_async_commit();
    uint32_t idx_next = (B + tid < n) ? slot_of(vals[start + B + tid]) : 0u;
    uint32_t val_next2 = (2 * B + tid < n) ? vals[start + 2 * B + tid] : 0u;

    int b = 0;
    for (; b < nb; ++b) {
        const int cur = b & 1, nxt = cur ^ 1;
        const int cnt = n - b * B < B ? n - b * B : B;
        // step 0: this thread's own gather of batch b has landed (its own cp.async group):
        // derive the pair's fast row.  fast[] is free: every warp passed the barrier that
        // ended batch b-1.
        cp_async_wait<0>();
        if (tid < cnt) {
            const float4 q0 = S.row[cur][tid][0], q1 = S.row[cur][tid][1], q2 = S.row[cur][tid][2];
            const float a = q0.z, bb = q0.w, c = q1.x, op = q1.y, k = q1.z;
            const float hk = 0.5f * k;
            const float thr = fmaxf(tau, op * ex2_approx(hk * kL));
            const float ac = a * c, det = fmaf(-bb, bb, ac);
            const float kap = ac / det;
            // extent rectangle contains the cutoff ellipse?  (x half-extent^2 = k*c/det)
            const float slack = 1.0f - 1e-6f * kap;
            const bool boxed = q2.z * q2.z * det >= k * c * slack && q2.w * q2.w * det >= k * a * slack;
            float eps = thr * fmaf(2.5e-5f, kap, 2e-5f);
            if (!(det > 0.0f) || !(kap < 400.0f) || !boxed || !(c > 0.0f) || !(a > 0.0f))
                eps = __int_as_float(0x7f800000);    // every evaluation takes the exact path
            S.fast[tid][0] = make_float4(q0.x, q0.y, a * (0.5f * kL), bb * kL);
            S.fast[tid][1] = make_float4(c * (0.5f * kL), op, thr, eps);
            S.fast[tid][2] = make_float4(q1.w, q2.x, q2.y, EXTRAS ? S.z[cur][tid] : 0.0f);
        }
        // step 1: gather the rows of batch b+1
        if ((b + 1) * B + tid < n) {
            const float4 *src = (const float4 *)(splat + (size_t)idx_next * 12);
            cp_async16(&S.row[nxt][tid][0], src);
            cp_async16(&S.row[nxt][tid][1], src + 1);
            cp_async16(&S.row[nxt][tid][2], src + 2);
            if (EXTRAS) S.z[nxt][tid] = gdepth ? gdepth[idx_next] : 0.0f;
        }
        cp_async_commit();
        // step 2: slots of batch b+2, values of batch b+3
        const uint32_t idx_next2 = ((b + 2) * B + tid < n) ? slot_of(val_next2) : 0u;
        const int i3 = (b + 3) * B + tid;
        val_next2 = i3 < n ? vals[start + i3] : 0u;
        if (CONTRIB) S.touched[tid] = 0u;
        __syncthreads();

        // step 3: blend batch b
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            if (__all_sync(FGS_FULL, fy0 == kInf && fy1 == kInf)) break;
            const int jl = c0 + lane;
            bool keep = false;
            if (jl < cnt) {
                const float4 q0 = S.row[cur][jl][0];
                const float4 q1 = S.row[cur][jl][1];
                const float4 q2 = S.row[cur][jl][2];
                const float u0 = fs(wx_lo, q0.x), u1 = fs(wx_hi, q0.x);
                const float v0 = fs(wy_lo, q0.y), v1 = fs(wy_hi, q0.y);
                keep = !(u0 > q2.z || u1 < -q2.z || v0 > q2.w || v1 < -q2.w);
                if (keep) keep = !ellipse_misses_block(q0.z, q0.w, q1.x, q1.z, u0, u1, v0, v1);
            }
            const uint32_t survivors = __ballot_sync(FGS_FULL, keep);
            constexpr int kUnroll2 = FGS_B2_UNROLL;
#pragma unroll kUnroll2
            for (int jj = 0; jj < 32; ++jj) {
                if (!((survivors >> jj) & 1u)) continue;
                const int j = c0 + jj;
                const float4 f0 = S.fast[j][0];
                const float4 f1 = S.fast[j][1];
                const float4 f2 = S.fast[j][2];
                const float dx = fx - f0.x;
                const pk2 ab = mul2(pk(f0.z, f0.w), bc(dx));         // (a2 dx, b2 dx): one FMUL2
                const float adx2 = ab.x * dx, bdx = ab.y;
                const pk2 dy2 = sub2(pk(fy0, fy1), bc(f0.y));
                const pk2 h2 = fma2(bc(f1.x), dy2, bc(bdx));
                const pk2 m2 = fma2(dy2, h2, bc(adx2));              // -log2(e) * s
                float m0, m1;
                upk(m2, m0, m1);
                pk2 al2 = mul2(bc(f1.y), pk(ex2_approx(m0), ex2_approx(m1)));
                const pk2 d2 = sub2(al2, bc(f1.z));
                float al0, al1, d0, d1;
                upk(d2, d0, d1);
                upk(al2, al0, al1);
                bool on0 = d0 >= 0.0f, on1 = d1 >= 0.0f;
                // one FMNMX with |.| on both operands + one compare for the two pixels (a NaN in
                // either means a NaN in both: the row's centre or conic is NaN, and eps = inf
                // sends rows with a degenerate conic here anyway).  The branch is taken by the
                // whole warp when any lane is in the band: a uniform branch needs no
                // reconvergence bookkeeping around the call, and the exact path gives the lanes
                // outside the band the verdict they already had.
                const bool band = !(fminf(fabsf(d0), fabsf(d1)) > f1.w);
                if (__any_sync(FGS_FULL, band)) {
                    // within eps of the threshold (or a row the shortcut does not cover):
                    // the reference's own evaluation decides, for both pixels
                    const float2 ax = alpha_exact_pair(&S.row[cur][j][0], fx, fy0, fy1, tau, S.tab);
                    al0 = ax.x;
                    al1 = ax.y;
                    on0 = al0 > 0.0f;
                    on1 = al1 > 0.0f;
                }
                al0 = fminf(al0, FGS_ALPHA_CAP);                     // render.py:217-218
                al1 = fminf(al1, FGS_ALPHA_CAP);
                al2 = pk(on0 ? al0 : 0.0f, on1 ? al1 : 0.0f);
                const pk2 w2 = mul2(al2, T2);
                cr2 = fma2(bc(f2.x), w2, cr2);
                cg2 = fma2(bc(f2.y), w2, cg2);
                cb2 = fma2(bc(f2.z), w2, cb2);
                if (EXTRAS) dz2 = fma2(bc(f2.w), w2, dz2);
                T2 = sub2(T2, w2);                                   // T (1 - alpha) = T - alpha T
                // (every lane stores the same word: marking with a register that happens to be
                // live saves the constant's MOV, but lanes then race with different values)
                if (CONTRIB && (on0 || on1)) S.touched[j] = 1u;
                float t0, t1;
                upk(T2, t0, t1);
                if (t0 < FGS_T_STOP) fy0 = kInf;                     // render.py:228
                if (t1 < FGS_T_STOP) fy1 = kInf;
            }
        }
        const bool all_done = __syncthreads_and(fy0 == kInf && fy1 == kInf);
        if (CONTRIB) {
            if (tid < cnt) {
                const uint32_t t = S.touched[tid];
                contrib[start + b * B + tid] = (uint8_t)t;
                ncontrib += t;
            }
        }
        idx_next = idx_next2;
        if (all_done) { done_all = true; ++b; break; }
    }
    cp_async_wait<0>();
    if (cut && !done_all) {                   // uniform: the sorted front was not enough
        if (tid == 0) redo_list[atomicAdd(&fgs_work(stats)[FGS_WORK_REDO], 1u)] = (uint32_t)tile;
        return;
    }
    if (cut) n = starts[tile + 1] - start;
    if (CONTRIB)
        for (int i = b * B + tid; i < n; i += B) contrib[start + i] = 0;

    float t0, t1, r0, r1, g0, g1, b0, b1, z0, z1;
    upk(T2, t0, t1);
    upk(cr2, r0, r1);
    upk(cg2, g0, g1);
    upk(cb2, b0, b1);
    upk(dz2, z0, z1);
    if (inside0) {
        const size_t o = (size_t)py0 * width + px;
        rgb[3 * o + 0] = fmaf(t0, bg0, r0);                          // render.py:250-252
        rgb[3 * o + 1] = fmaf(t0, bg1, g0);
        rgb[3 * o + 2] = fmaf(t0, bg2, b0);
        if (EXTRAS) {
            if (alpha_out) alpha_out[o] = 1.0f - t0;
            if (depth_out) depth_out[o] = z0;
        }
    }
    if (inside1) {
        const size_t o = (size_t)py1 * width + px;
        rgb[3 * o + 0] = fmaf(t1, bg0, r1);
        rgb[3 * o + 1] = fmaf(t1, bg1, g1);
        rgb[3 * o + 2] = fmaf(t1, bg2, b1);
        if (EXTRAS) {
            if (alpha_out) alpha_out[o] = 1.0f - t1;
            if (depth_out) depth_out[o] = z1;
        }
    }
    if (CONTRIB) {
        ncontrib = __reduce_add_sync(FGS_FULL, ncontrib);
        if (lane == 0 && ncontrib) atomicAdd(&stats->pairs_contributing, ncontrib);
    }
    };  // tile_body
    if (REDO) blend_redo_pass(stats, redo_list, tile_body);
    else tile_body(tile0);
}

template <bool CONTRIB, bool REDO>
int launch2(bool extras, dim3 grid, cudaStream_t st, const float *splat, const float *gdepth,
            const uint32_t *vals, const uint32_t *inv, const int32_t *starts, const uint32_t *order,
            int width, int height,
            int grid_w, int first_tile, const float bg[3], float tau, float *rgb, float *alpha,
            float *depth, uint8_t *contrib, fgs_stats *stats, const int32_t *limit, uint32_t *redo_list)
{
    if (extras)
        FGS_CHAIN((k_blend2<CONTRIB, true, REDO>), grid, dim3(FGS_B2_THREADS), 0, st, splat, gdepth, vals, inv,
                  starts, order, width, height, grid_w, first_tile, bg[0], bg[1], bg[2], tau, rgb, alpha,
                  depth, contrib, stats, limit, redo_list);
    else
        FGS_CHAIN((k_blend2<CONTRIB, false, REDO>), grid, dim3(FGS_B2_THREADS), 0, st, splat, gdepth, vals, inv,
                  starts, order, width, height, grid_w, first_tile, bg[0], bg[1], bg[2], tau, rgb, alpha,
                  depth, contrib, stats, limit, redo_list);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

template <bool EXACT, bool CONTRIB, bool REDO>
int launch(bool extras, dim3 grid, cudaStream_t st, const float *splat, const float *gdepth,
           const uint32_t *vals, const uint32_t *inv, const int32_t *starts, const uint32_t *order,
           int width, int height, int grid_w,
           int first_tile, const float bg[3], float tau, float *rgb, float *alpha, float *depth,
           uint8_t *contrib, fgs_stats *stats, const int32_t *limit, uint32_t *redo_list)
{
    unsigned long long *no_evals = nullptr;
    // (the second pass is chained: it starts with griddepcontrol.wait)
    if (extras)
        FGS_CHAIN((k_blend<EXACT, CONTRIB, true, false, REDO>), grid, dim3(256), 0, st, splat, gdepth, vals, inv,
                  starts, order, width, height, grid_w, first_tile, bg[0], bg[1], bg[2], tau, rgb, alpha,
                  depth, contrib, stats, no_evals, limit, redo_list);
    else
        FGS_CHAIN((k_blend<EXACT, CONTRIB, false, false, REDO>), grid, dim3(256), 0, st, splat, gdepth, vals, inv,
                  starts, order, width, height, grid_w, first_tile, bg[0], bg[1], bg[2], tau, rgb, alpha,
                  depth, contrib, stats, no_evals, limit, redo_list);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

}  // namespace

int fgs_launch_blend(const float *splat, const float *gdepth, const uint32_t *vals,
                     const uint32_t *inv, const int32_t *starts, const uint32_t *order,
                     int width, int height,
                     const float bg[3], double tau,
                     int flags, int band0, int band1, float *rgb, float *alpha, float *depth,
                     uint8_t *contrib, fgs_stats *stats, cudaStream_t st,
                     const int32_t *limit, uint32_t *redo_list, int redo)
{
    const int grid_w = (width + FGS_TILE - 1) / FGS_TILE;
    if (band1 < band0) return FGS_OK;
    if ((limit != nullptr || redo) && (redo_list == nullptr || stats == nullptr)) return FGS_E_ARG;
    dim3 grid((unsigned)(grid_w * (band1 - band0 + 1)));
    if (redo) {
        // persistent CTAs over the redo list (its length is only known on the device)
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned want = (unsigned)(4 * sms);
        grid = dim3(grid.x < want ? grid.x : want);
    }
    const int first_tile = band0 * grid_w;
    const bool exact = flags & FGS_BLEND_EXACT, want_contrib = (flags & FGS_BLEND_CONTRIB) && contrib;
    const bool extras = (alpha != nullptr) || (depth != nullptr && gdepth != nullptr);
    if (depth != nullptr && gdepth == nullptr) return FGS_E_ARG;
    const float tau32 = (float)tau;
#define FGS_ARGS extras, grid, st, splat, gdepth, vals, inv, starts, order, width, height, \
                 grid_w, first_tile, bg, tau32, rgb, alpha, depth, contrib, stats, limit, redo_list
#define FGS_GO(E, C) (redo ? launch<E, C, true>(FGS_ARGS) : launch<E, C, false>(FGS_ARGS))
    if (exact) return want_contrib ? FGS_GO(true, true) : FGS_GO(true, false);
    if (flags & FGS_BLEND_SCALAR) return want_contrib ? FGS_GO(false, true) : FGS_GO(false, false);
#undef FGS_GO
#define FGS_GO2(C) (redo ? launch2<C, true>(FGS_ARGS) : launch2<C, false>(FGS_ARGS))
    return want_contrib ? FGS_GO2(true) : FGS_GO2(false);
#undef FGS_GO2
#undef FGS_ARGS
}

// Diagnostic pass over a finished frame's sorted pairs: the exact-mode blend with the
// evaluation counters on (see k_blend, COUNT).  `evals` is zeroed here.
int fgs_launch_blend_counts(const float *splat, const uint32_t *vals, const uint32_t *inv,
                            const int32_t *starts, int width, int height, const float bg[3],
                            double tau, int band0, int band1, float *rgb, fgs_stats *stats,
                            unsigned long long *evals, cudaStream_t st)
{
    const int grid_w = (width + FGS_TILE - 1) / FGS_TILE;
    cudaError_t e = cudaMemsetAsync(evals, 0, 8 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
    if (band1 < band0) return FGS_OK;
    const dim3 grid((unsigned)(grid_w * (band1 - band0 + 1)));
    k_blend<true, false, false, true><<<grid, 256, 0, st>>>(
        splat, nullptr, vals, inv, starts, nullptr, width, height, grid_w, band0 * grid_w, bg[0],
        bg[1], bg[2], (float)tau, rgb, nullptr, nullptr, nullptr, stats, evals);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}

// images.py:12-15 quantize (float64 like the reference); four values per thread
__global__ void __launch_bounds__(256)
k_quantize_rgb8(const float *__restrict__ rgb, int64_t count, uint8_t *__restrict__ out)
{
    const int64_t i0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
    if (i0 >= count) return;
    auto q = [](float v) -> uint32_t {
        double c = (double)v;
        c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
        return (uint32_t)floor(da(dm(c, 255.0), 0.5));
    };
    if (i0 + 4 <= count) {
        const float4 v = *reinterpret_cast<const float4 *>(rgb + i0);
        *reinterpret_cast<uint32_t *>(out + i0) = q(v.x) | (q(v.y) << 8) | (q(v.z) << 16) | (q(v.w) << 24);
    } else {
        for (int64_t i = i0; i < count; ++i) out[i] = (uint8_t)q(rgb[i]);
    }
}

int fgs_launch_quantize(const float *rgb, int64_t count, uint8_t *out, cudaStream_t st)
{
    if (count == 0) return FGS_OK;
    const int64_t blocks = (count + 1023) / 1024;
    k_quantize_rgb8<<<(unsigned)blocks, 256, 0, st>>>(rgb, count, out);
    FGS_CHECK_LAUNCH();
    return FGS_OK;
}
