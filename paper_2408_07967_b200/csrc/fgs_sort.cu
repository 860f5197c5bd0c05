// K4 device radix sort and K5 tile-range identification.
//
// Replaces sorting.py:29-58 (numba histogram / scatter), 68-136 (sort_pairs)
// and 139-152 (tile_range_table).
//
// One-sweep LSD radix sort, 8-bit digits: one kernel reads the keys once and
// builds the digit histograms of every pass; then each pass is ONE kernel that
// ranks a 4096-pair tile in shared memory (warp match-any ranking, stable),
// obtains its global digit offsets from the preceding tiles with a decoupled
// look-back, and scatters.  Per pass the pairs are read once and written once
// (24 B per pair), which is the HBM floor for an out-of-place LSD pass.
//
// Order contract: stable.  The frame path emits pairs in ascending Gaussian
// index, so stability alone yields the reference's (key, value) order; the
// stand-alone fgs_sort_pairs prepends value-digit passes like the reference.
//
// The look-back table is never cleared: entries carry the 32-bit `epoch` of
// the pass that wrote them and are ignored unless it matches.

#include "fgs_common.cuh"

namespace {

struct PassArgs {
    int on_value, shift, bits, compact;
};

__device__ __forceinline__ uint64_t sort_word(uint64_t key, int compact)
{
    // depth > 0, so bit 31 of the key is always clear: squeeze it out
    return compact ? (((key >> 32) << 31) | (key & 0x7fffffffull)) : key;
}

__device__ __forceinline__ uint32_t digit_of(uint64_t key, uint32_t val, const PassArgs &a)
{
    const uint32_t mask = (1u << a.bits) - 1u;
    return a.on_value ? ((val >> a.shift) & mask)
                      : ((uint32_t)(sort_word(key, a.compact) >> a.shift) & mask);
}

struct HistArgs {
    int npass;
    PassArgs p[FGS_SORT_MAXPASS];
};

// ---- all digit histograms in one read of the pairs -------------------------
__global__ void __launch_bounds__(256)
k_sort_hist(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vals,
            const uint32_t *__restrict__ n_dev, const __grid_constant__ HistArgs ha,
            uint32_t *__restrict__ hist)
{
    extern __shared__ uint32_t s_h[];            // [npass][256]
    const uint32_t n = *n_dev;
    for (int i = threadIdx.x; i < ha.npass * 256; i += 256) s_h[i] = 0u;
    __syncthreads();
    bool need_val = false;
    for (int p = 0; p < ha.npass; ++p) need_val |= ha.p[p].on_value != 0;
    for (uint32_t i = blockIdx.x * 256u + threadIdx.x; i < n; i += gridDim.x * 256u) {
        const uint64_t k = keys[i];
        const uint32_t v = need_val ? vals[i] : 0u;
        for (int p = 0; p < ha.npass; ++p) atomicAdd(&s_h[p * 256 + digit_of(k, v, ha.p[p])], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ha.npass * 256; i += 256) {
        const uint32_t c = s_h[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// ---- one pass ---------------------------------------------------------------
constexpr uint32_t ST_AGG = 1u << 30, ST_INCL = 2u << 30, ST_MASK = 3u << 30;
constexpr int NW = FGS_SORT_THREADS / 32;       // 8 warps
constexpr int BINS = 257;                        // 256 digits + 1 bin for padding lanes

struct SortSmem {
    uint64_t keys[FGS_SORT_TILE];
    uint32_t vals[FGS_SORT_TILE];
    uint32_t whist[NW][BINS];
    uint32_t tile_excl[256];     // exclusive scan of this tile's digit counts
    int64_t  gbase[256];         // global output index of tile-sorted slot 0 of each digit
    uint32_t scan[8];
    uint32_t tile;
};

__global__ void __launch_bounds__(FGS_SORT_THREADS, 3)
k_sort_pass(const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
            uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
            const uint32_t *__restrict__ n_dev, PassArgs pa, const uint32_t *__restrict__ hist,
            uint64_t *state, uint32_t *ticket, uint32_t epoch)
{
    extern __shared__ __align__(16) unsigned char s_raw[];
    SortSmem &S = *reinterpret_cast<SortSmem *>(s_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t n = *n_dev;
    const uint32_t ntiles = (n + FGS_SORT_TILE - 1) / FGS_SORT_TILE;

    // global digit bases for this pass: exclusive scan of the 256-bin histogram
    uint32_t dtotal;
    const uint32_t dbase = block_excl_scan_256(hist[tid], S.scan, dtotal);

    for (;;) {
        if (tid == 0) S.tile = atomicAdd(ticket, 1u);
        for (int i = tid; i < NW * BINS; i += FGS_SORT_THREADS) (&S.whist[0][0])[i] = 0u;
        __syncthreads();
        const uint32_t tile = S.tile;
        if (tile >= ntiles) break;
        const uint32_t tbase = tile * FGS_SORT_TILE;
        const uint32_t nvalid = n - tbase < FGS_SORT_TILE ? n - tbase : FGS_SORT_TILE;

        // warp-striped load: item i of lane l sits at w*512 + i*32 + l
        uint64_t key[FGS_SORT_IPT];
        uint32_t val[FGS_SORT_IPT];
        uint16_t rank[FGS_SORT_IPT];
        const uint32_t wbase = w * (32 * FGS_SORT_IPT);
#pragma unroll
        for (int i = 0; i < FGS_SORT_IPT; ++i) {
            const uint32_t loc = wbase + i * 32 + lane;
            const bool ok = loc < nvalid;
            key[i] = ok ? keys_in[tbase + loc] : 0ull;
            val[i] = ok ? vals_in[tbase + loc] : 0u;
        }
        // stable in-warp ranking per digit
        uint32_t *wh = S.whist[w];
#pragma unroll
        for (int i = 0; i < FGS_SORT_IPT; ++i) {
            const bool ok = wbase + i * 32 + lane < nvalid;
            const uint32_t d = ok ? digit_of(key[i], val[i], pa) : 256u;
            const uint32_t prev = wh[d];
            __syncwarp();
            const uint32_t peers = __match_any_sync(FGS_FULL, d);
            const uint32_t before = __popc(peers & lanemask_lt());
            if (before == 0) wh[d] = prev + __popc(peers);
            __syncwarp();
            rank[i] = (uint16_t)(prev + before);
        }
        __syncthreads();

        // per digit (thread d): exclusive prefix over warps, tile count
        uint32_t cnt = 0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
            const uint32_t c = S.whist[ww][tid];
            S.whist[ww][tid] = cnt;
            cnt += c;
        }
        // publish, then look back over preceding tiles for this digit's prefix
        uint64_t *st = state + (size_t)tile * 256 + tid;
        const uint64_t tag = (uint64_t)epoch << 32;
        uint32_t excl = 0;
        if (tile == 0) {
            *(volatile uint64_t *)st = tag | ST_INCL | cnt;
        } else {
            *(volatile uint64_t *)st = tag | ST_AGG | cnt;
            // look back 8 predecessors per round trip (independent loads in flight);
            // tile 0 always carries an inclusive prefix, so the walk terminates
            int t = (int)tile - 1;
            for (bool found = false; !found;) {
                uint64_t v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    v[i] = (t - i >= 0) ? *(const volatile uint64_t *)(state + (size_t)(t - i) * 256 + tid)
                                        : 0ull;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (found || t - i < 0) continue;
                    const uint32_t lo = (uint32_t)v[i];
                    if ((uint32_t)(v[i] >> 32) != epoch || (lo & ST_MASK) == 0u) {
                        t -= i;                 // not published yet: poll again from here
                        goto next_round;
                    }
                    excl += lo & ~ST_MASK;
                    if ((lo & ST_MASK) == ST_INCL) found = true;
                }
                t -= 8;
            next_round:;
            }
            *(volatile uint64_t *)st = tag | ST_INCL | (excl + cnt);
        }
        uint32_t ttotal;
        const uint32_t texcl = block_excl_scan_256(cnt, S.scan, ttotal);
        S.tile_excl[tid] = texcl;
        S.gbase[tid] = (int64_t)dbase + excl - texcl;
        __syncthreads();

        // reorder the tile in shared memory by digit (stable)
#pragma unroll
        for (int i = 0; i < FGS_SORT_IPT; ++i) {
            const bool ok = wbase + i * 32 + lane < nvalid;
            if (ok) {
                const uint32_t d = digit_of(key[i], val[i], pa);
                const uint32_t pos = S.tile_excl[d] + S.whist[w][d] + rank[i];
                S.keys[pos] = key[i];
                S.vals[pos] = val[i];
            }
        }
        __syncthreads();
        // coalesced runs out: consecutive threads write consecutive addresses
#pragma unroll
        for (int i = 0; i < FGS_SORT_IPT; ++i) {
            const uint32_t idx = i * FGS_SORT_THREADS + tid;
            if (idx < nvalid) {
                const uint64_t k = S.keys[idx];
                const uint32_t v = S.vals[idx];
                const int64_t dst = S.gbase[digit_of(k, v, pa)] + idx;
                keys_out[dst] = k;
                vals_out[dst] = v;
            }
        }
        __syncthreads();
    }
}

// ---- K5: tile ranges --------------------------------------------------------
// starts[t] = first sorted index whose tile >= t  (np.searchsorted side="left").
__global__ void __launch_bounds__(256)
k_tile_ranges(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ n_dev, int tiles,
              int32_t *__restrict__ starts, fgs_stats *__restrict__ stats)
{
    const uint32_t n = *n_dev;
    const uint32_t stride = gridDim.x * 256u;
    uint32_t nonempty = 0;
    for (uint32_t i = blockIdx.x * 256u + threadIdx.x; i <= n; i += stride) {
        // boundary between sorted element i-1 and i (with virtual ends)
        long long prev = -1, cur = tiles;
        if (i > 0) {
            const uint64_t kp = keys[i - 1];
            prev = (long long)(kp >> 32);
            if (i < n && keys[i] < kp) stats->unsorted = 1u;           // sorting.py:146-147
        }
        if (i < n) cur = (long long)(keys[i] >> 32);
        if (i == n && n > 0 && prev >= tiles) stats->tile_out_of_grid = 1u;  // sorting.py:150-151
        if (cur > tiles) cur = tiles;
        if (cur > prev) {
            for (long long t = prev + 1; t <= cur; ++t)
                if (t <= tiles) starts[t] = (int32_t)i;
            if (i < n) ++nonempty;
        }
    }
    nonempty = __reduce_add_sync(FGS_FULL, nonempty);
    if ((threadIdx.x & 31) == 0 && nonempty) atomicAdd(&stats->tiles_nonempty, nonempty);
}

// ---- TILE_BUCKET: per-tile sort in shared memory ------------------------------
// After the MSD counting pass (k_preprocess histogram -> k_scan_tiles -> k_emit
// scatter) tile t's pairs sit, in arbitrary order, in rec[starts[t] .. starts[t+1])
// as (depth bits << 32 | Gaussian index).  One CTA sorts one bucket ascending on
// that 64-bit word, which is exactly the reference's (depth, then index) order
// inside a tile (sorting.py:3-5).  Records are unique.
//
// The sort is an LSD radix sort on the four depth bytes, entirely in shared
// memory (same stable warp-match ranking as k_sort_pass, local digit offsets
// instead of a look-back); equal-depth neighbours -- rare: two Gaussians with the
// same float32 depth in one tile -- are then put in index order by an odd-even
// pass.  This radix sort serves the dense buckets (> 4096 records, persistent CTAs
// over the list k_scan_tiles collected) and the rare buckets the faster
// bucket-rank sort below gives up on.  Buckets beyond 8192 first go through one counting
// pass on their top 8 varying depth bits (through L2); consecutive bins are then
// grouped into chunks of at most 8192 records, each sorted in shared memory.  A bitonic network (all-ascending form, so
// comparators touching an index >= n are simply skipped) is the last resort for
// pathological depth distributions.
template <int NT, int EMAX>
struct TileSortSmem {
    static constexpr int CAP = NT * EMAX;
    static constexpr int WARPS = NT / 32;
    uint64_t s[CAP];
    uint32_t whist[WARPS][BINS];
    uint32_t texcl[256];
    uint32_t scan[32];
    uint32_t sub[257];
    uint32_t grp[258];
    uint32_t mm[2];
    uint32_t ngroups;
};

// Exclusive scan of one value per thread over the first 256 threads of an NT-thread
// CTA (the other threads pass 0).  Two barriers.
template <int NT>
__device__ __forceinline__ uint32_t ts_scan256(uint32_t v, uint32_t *scratch)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(v, lane);
    if (lane == 31 && w < 8) scratch[w] = incl;
    __syncthreads();
    uint32_t wsum = lane < 8 ? scratch[lane] : 0u;
    uint32_t wincl = warp_incl_scan(wsum, lane);
    uint32_t wbase = __shfl_sync(FGS_FULL, wincl - wsum, w & 7);
    __syncthreads();
    return wbase + incl - v;
}

template <int NT>
__device__ __forceinline__ void ts_step_smem(uint64_t *s, int count, int mask, int hb)
{
    // compare-exchange (i, i ^ mask) for every i < count with bit `hb` clear
    for (int t = threadIdx.x; t < count / 2; t += NT) {
        const int i = ((t & ~(hb - 1)) << 1) | (t & (hb - 1));
        const int p = i ^ mask;
        const uint64_t a = s[i], b = s[p];
        if (a > b) { s[i] = b; s[p] = a; }
    }
    __syncthreads();
}

template <int NT>
__device__ __forceinline__ void ts_step_global(uint64_t *g, int n, int npad, int mask, int hb)
{
    for (int t = threadIdx.x; t < npad / 2; t += NT) {
        const int i = ((t & ~(hb - 1)) << 1) | (t & (hb - 1));
        const int p = i ^ mask;
        if (p < n) {
            const uint64_t a = g[i], b = g[p];
            if (a > b) { g[i] = b; g[p] = a; }
        }
    }
    __syncthreads();
}

template <int NT>
__device__ __forceinline__ void ts_bitonic_smem(uint64_t *s, int npad)
{
    for (int k = 2; k <= npad; k <<= 1) {
        ts_step_smem<NT>(s, npad, k - 1, k >> 1);
        for (int j = k >> 2; j > 0; j >>= 1) ts_step_smem<NT>(s, npad, j, j);
    }
}

// Sort m <= CAP records (src, global) ascending on (depth bits, index) into
// S.s[0..m): `npass` LSD byte passes starting at record bit 32, then the
// equal-depth fix-up.  Every thread of the CTA calls it with the same arguments.
template <int NT, int EMAX>
__device__ __forceinline__ void ts_sort_small(TileSortSmem<NT, EMAX> &S,
                                              const uint64_t *src, int m, int npass)
{
    constexpr int TS_E = EMAX;
    constexpr int WARPS = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint64_t *s = S.s;
    if (m <= 1) {
        if (tid == 0 && m == 1) s[0] = src[0];
        __syncthreads();
        return;
    }
    // records spread evenly over the warps: E per thread, warp-striped
    const int E = (m + NT - 1) / NT;
    const int wbase = w * 32 * E;
    uint64_t key[TS_E];
    uint16_t rank[TS_E];
#pragma unroll
    for (int i = 0; i < TS_E; ++i) {
        const int loc = wbase + i * 32 + lane;
        key[i] = (i < E && loc < m) ? src[loc] : ~0ull;
    }
    if (npass == 0) {                      // nothing to sort on: just stage the records
#pragma unroll
        for (int i = 0; i < TS_E; ++i) {
            const int loc = wbase + i * 32 + lane;
            if (i < E && loc < m) s[loc] = key[i];
        }
        __syncthreads();
    }
    uint32_t *wh = S.whist[w];
    for (int pass = 0; pass < npass; ++pass) {
        const int shift = 32 + 8 * pass;
        for (int i = tid; i < WARPS * BINS; i += NT) (&S.whist[0][0])[i] = 0u;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < TS_E; ++i) {
            if (i < E) {                                  // uniform
                const bool ok = wbase + i * 32 + lane < m;
                const uint32_t d = ok ? (uint32_t)(key[i] >> shift) & 0xffu : 256u;
                const uint32_t prev = wh[d];
                __syncwarp();
                const uint32_t peers = __match_any_sync(FGS_FULL, d);
                const uint32_t before = __popc(peers & lanemask_lt());
                if (before == 0) wh[d] = prev + __popc(peers);
                __syncwarp();
                rank[i] = (uint16_t)(prev + before);
            }
        }
        __syncthreads();
        uint32_t cnt = 0;
        if (tid < 256) {
#pragma unroll 8
            for (int ww = 0; ww < WARPS; ++ww) {
                const uint32_t c = S.whist[ww][tid];
                S.whist[ww][tid] = cnt;
                cnt += c;
            }
        }
        const uint32_t ex = ts_scan256<NT>(cnt, S.scan);
        if (tid < 256) S.texcl[tid] = ex;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < TS_E; ++i) {
            if (i < E && wbase + i * 32 + lane < m) {
                const uint32_t d = (uint32_t)(key[i] >> shift) & 0xffu;
                s[S.texcl[d] + wh[d] + rank[i]] = key[i];
            }
        }
        __syncthreads();
        if (pass + 1 < npass) {
#pragma unroll
            for (int i = 0; i < TS_E; ++i) {
                const int loc = wbase + i * 32 + lane;
                key[i] = (i < E && loc < m) ? s[loc] : ~0ull;
            }
        }
    }
    // equal depths: order by index (low word).  Odd-even transposition over
    // equal-depth neighbours; almost always zero or one round.
    for (int round = 0;; ++round) {
        bool swapped = false;
        for (int t = tid; 2 * t + 1 < m; t += NT) {
            const uint64_t a = s[2 * t], b = s[2 * t + 1];
            if ((a >> 32) == (b >> 32) && a > b) { s[2 * t] = b; s[2 * t + 1] = a; swapped = true; }
        }
        __syncthreads();
        for (int t = tid; 2 * t + 2 < m; t += NT) {
            const uint64_t a = s[2 * t + 1], b = s[2 * t + 2];
            if ((a >> 32) == (b >> 32) && a > b) { s[2 * t + 1] = b; s[2 * t + 2] = a; swapped = true; }
        }
        if (!__syncthreads_or(swapped)) break;
        if (round == 6) {           // long runs of one depth: finish with the network
            int npad = 2;
            while (npad < m) npad <<= 1;
            for (int i = m + tid; i < npad; i += NT) s[i] = ~0ull;
            __syncthreads();
            ts_bitonic_smem<NT>(s, npad);
            break;
        }
    }
}

// Bitonic sort of an arbitrarily large segment in global memory (strides >= CAP
// through L2, the rest chunk-wise in shared memory).  Last resort only.
template <int NT, int EMAX>
__device__ __noinline__ void ts_bitonic_global(TileSortSmem<NT, EMAX> &S, uint64_t *g, int n)
{
    constexpr int CAP = TileSortSmem<NT, EMAX>::CAP;
    const int tid = threadIdx.x;
    uint64_t *s = S.s;
    int npad = CAP;
    while (npad < n) npad <<= 1;
    const int nchunks = (n + CAP - 1) / CAP;
    for (int c = 0; c < nchunks; ++c) {
        const int cb = c * CAP;
        for (int i = tid; i < CAP; i += NT) s[i] = cb + i < n ? g[cb + i] : ~0ull;
        __syncthreads();
        ts_bitonic_smem<NT>(s, CAP);
        for (int i = tid; i < CAP; i += NT)
            if (cb + i < n) g[cb + i] = s[i];
        __syncthreads();
    }
    for (int k = 2 * CAP; k <= npad; k <<= 1) {
        ts_step_global<NT>(g, n, npad, k - 1, k >> 1);
        int j = k >> 2;
        for (; j >= CAP; j >>= 1) ts_step_global<NT>(g, n, npad, j, j);
        for (int c = 0; c < nchunks; ++c) {
            const int cb = c * CAP;
            for (int i = tid; i < CAP; i += NT) s[i] = cb + i < n ? g[cb + i] : ~0ull;
            __syncthreads();
            for (int jj = CAP >> 1; jj > 0; jj >>= 1) ts_step_smem<NT>(s, CAP, jj, jj);
            for (int i = tid; i < CAP; i += NT)
                if (cb + i < n) g[cb + i] = s[i];
            __syncthreads();
        }
    }
}

// ---- bucket-rank sort: the fast path for buckets of up to 4096 records -------------
// Depths inside a tile are spread fairly evenly between the tile's nearest and
// farthest splat, so a monotone linear map of the depth bits onto NB = CAP/4 bins
// leaves a handful of records per bin.  One shared-memory atomic per record builds
// the bin histogram (its return value is the record's slot inside the bin), a scan
// turns it into bin offsets, the records are scattered bin-contiguously, and each
// record then ranks itself inside its bin by comparing the full 64-bit word with
// the bin's few other members -- which also settles equal depths by index.  Six
// barriers per tile instead of twenty, no serial LDS -> match -> STS chains.
// A tile where some bin holds more than TB_MAXBIN records (many equal or tightly
// clustered depths) is pushed on the "hard" list and sorted by the radix kernel.
constexpr int TB_MAXBIN = 64;

// STAGE: keep a copy of the input records in shared memory (steps 2 and 4 read it);
// without it they re-read the bucket through L1/L2 and the capacity doubles.
template <int NT, int EMAX, bool STAGE = true, int NBDIV = 4>
struct BucketSmem {
    static constexpr int CAP = NT * EMAX;
    static constexpr int NB = CAP / NBDIV;                    // depth bins: NBDIV records per bin when full
    uint64_t a[STAGE ? CAP : 1];
    uint64_t b[CAP];
    uint32_t bin[NB + 1];
    uint32_t red[64];
};

// Sorts the n <= CAP records at g; the result goes to vals_out / keys_out [start, start+n).
// Returns false (nothing written) when the records have to go to the radix fallback.
// Every thread of the CTA calls it with the same arguments.
template <int NT, int EMAX, bool STAGE = true, int NBDIV = 4>
__device__ __forceinline__ bool tb_sort_range(BucketSmem<NT, EMAX, STAGE, NBDIV> &S, const uint64_t *g,
                                              int n, int start, uint64_t tile_hi,
                                              uint32_t *__restrict__ vals_out,
                                              uint64_t *__restrict__ keys_out, int write_keys)
{
    // (g is not __restrict__: a split bucket's chunks were written by this very CTA)
    constexpr int NB = BucketSmem<NT, EMAX, STAGE, NBDIV>::NB;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    // 1. stage the records, depth range of the tile
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int i = tid; i < n; i += NT) {
        const uint64_t r = g[i];
        if (STAGE) S.a[i] = r;
        const uint32_t d = (uint32_t)(r >> 32);
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
    }
    for (int i = tid; i <= NB; i += NT) S.bin[i] = 0u;
    lo = __reduce_min_sync(FGS_FULL, lo);
    hi = __reduce_max_sync(FGS_FULL, hi);
    if (lane == 0) { S.red[w] = lo; S.red[32 + w] = hi; }
    __syncthreads();
    lo = 0xffffffffu; hi = 0u;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        lo = S.red[i] < lo ? S.red[i] : lo;
        hi = S.red[32 + i] > hi ? S.red[32 + i] : hi;
    }
    const uint32_t range = hi - lo;
    const bool direct = range < (uint32_t)NB;                 // one depth value per bin
    const uint64_t inv = direct ? 0ull : ((uint64_t)NB << 32) / ((uint64_t)range + 1ull);
#define TB_BIN(d) (direct ? (d) - lo : (uint32_t)(((uint64_t)((d) - lo) * inv) >> 32))

    // 2. histogram; the atomic's return value is the record's slot inside its bin
    uint16_t slot[EMAX];
    bool too_big = false;
#pragma unroll
    for (int k = 0; k < EMAX; ++k) {
        const int i = tid + k * NT;
        if (i < n) {
            const uint32_t d = (uint32_t)((STAGE ? S.a[i] : g[i]) >> 32);
            const uint32_t sl = atomicAdd(&S.bin[1 + TB_BIN(d)], 1u);
            slot[k] = (uint16_t)sl;
            too_big |= sl >= (uint32_t)TB_MAXBIN;
        }
    }
    if (__syncthreads_or(too_big)) return false;

    // 3. bin offsets: inclusive scan of bin[1..NB] in place (bin[0] = 0)
    {
        constexpr int PER = (NB + NT - 1) / NT;               // consecutive bins per thread
        uint32_t v[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = 1 + tid * PER + k;
            v[k] = idx <= NB ? S.bin[idx] : 0u;
            sum += v[k];
        }
        uint32_t incl = warp_incl_scan(sum, lane);
        if (lane == 31) S.red[w] = incl;
        __syncthreads();
        uint32_t wsum = lane < NT / 32 ? S.red[lane] : 0u;
        uint32_t wincl = warp_incl_scan(wsum, lane);
        uint32_t run = __shfl_sync(FGS_FULL, wincl - wsum, w) + incl - sum;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = 1 + tid * PER + k;
            run += v[k];
            if (idx <= NB) S.bin[idx] = run;
        }
    }
    __syncthreads();

    // 4. scatter bin-contiguously
#pragma unroll
    for (int k = 0; k < EMAX; ++k) {
        const int i = tid + k * NT;
        if (i < n) {
            const uint64_t r = STAGE ? S.a[i] : g[i];
            S.b[S.bin[TB_BIN((uint32_t)(r >> 32))] + slot[k]] = r;
        }
    }
    __syncthreads();

    // 5. rank inside the bin by full-word comparison; write straight to the output
    for (int i = tid; i < n; i += NT) {
        const uint64_t r = S.b[i];
        const uint32_t bn = TB_BIN((uint32_t)(r >> 32));
        const int b0 = (int)S.bin[bn], b1 = (int)S.bin[bn + 1];
        int rank = 0;
        for (int j = b0; j < b1; ++j) rank += S.b[j] < r ? 1 : 0;
        vals_out[start + b0 + rank] = (uint32_t)r;
        if (write_keys) keys_out[start + b0 + rank] = tile_hi | (r >> 32);
    }
#undef TB_BIN
    return true;
}

template <int NT, int EMAX, bool STAGE = true, int NBDIV = 4>
__device__ __forceinline__ bool tb_sort_tile(BucketSmem<NT, EMAX, STAGE, NBDIV> &S, int tile,
                                             const uint64_t *__restrict__ rec,
                                             uint32_t *__restrict__ vals_out,
                                             uint64_t *__restrict__ keys_out,
                                             const int32_t *__restrict__ starts, int write_keys)
{
    const int start = starts[tile], n = starts[tile + 1] - start;
    return tb_sort_range<NT, EMAX, STAGE, NBDIV>(S, rec + start, n, start, (uint64_t)(uint32_t)tile << 32,
                                          vals_out, keys_out, write_keys);
}

// One bucket.  Every thread of the CTA calls it with the same arguments.  With
// SPLIT = false the caller guarantees n <= CAP (and the split code is not compiled
// in, which keeps the hot kernel inside the instruction cache).
template <int NT, int EMAX, bool SPLIT>
__device__ __forceinline__ void ts_sort_tile(TileSortSmem<NT, EMAX> &S, int tile,
                                             uint64_t *__restrict__ rec,
                                             uint64_t *__restrict__ alt, uint32_t *__restrict__ vals_out,
                                             uint64_t *__restrict__ keys_out,
                                             const int32_t *__restrict__ starts, int write_keys,
                                             BucketSmem<NT, EMAX> *B = nullptr)
{
    constexpr int CAP = TileSortSmem<NT, EMAX>::CAP;
    const int tid = threadIdx.x;
    const int start = starts[tile], n = starts[tile + 1] - start;
    if (n <= 0) return;
    uint64_t *g = rec + start;
    uint64_t *a = alt + start;
    uint64_t *s = S.s;
    const uint64_t tile_hi = (uint64_t)(uint32_t)tile << 32;
    const bool split = SPLIT && n > CAP;

    if (split) {
        // ---- bucket beyond the shared-memory capacity: one counting pass on the top 8
        // varying depth bits into `alt` (through L2).  Bins are in depth order, so runs
        // of consecutive bins are then grouped greedily into chunks of at most CAP
        // records and each chunk is sorted in shared memory on all four depth bytes.
        // keys_out may alias alt: a chunk is consumed before its slice is overwritten.
        if (tid == 0) { S.mm[0] = 0xffffffffu; S.mm[1] = 0u; }
        for (int i = tid; i < 257; i += NT) S.sub[i] = 0u;
        __syncthreads();
        uint32_t lo = 0xffffffffu, hi = 0u;
        for (int i = tid; i < n; i += NT) {
            const uint32_t d = (uint32_t)(g[i] >> 32);
            lo = d < lo ? d : lo;
            hi = d > hi ? d : hi;
        }
        lo = __reduce_min_sync(FGS_FULL, lo);
        hi = __reduce_max_sync(FGS_FULL, hi);
        if ((tid & 31) == 0) { atomicMin(&S.mm[0], lo); atomicMax(&S.mm[1], hi); }
        __syncthreads();
        const uint32_t diff = S.mm[0] ^ S.mm[1];
        const int top = diff ? 31 - __clz((int)diff) : 0;   // highest varying depth bit
        const int sh = top > 7 ? top - 7 : 0;                // bin = depth bits [sh, sh+8)
        for (int i = tid; i < n; i += NT)
            atomicAdd(&S.sub[1 + (((uint32_t)(g[i] >> 32) >> sh) & 0xffu)], 1u);
        __syncthreads();
        if (tid == 0) {
            uint32_t run = 0;
            for (int d = 0; d <= 256; ++d) { run += S.sub[d]; S.sub[d] = run; }
            uint32_t k = 0;
            S.grp[0] = 0;
            for (uint32_t d = 0; d < 256; ++d)
                if (S.sub[d + 1] - S.sub[S.grp[k]] > (uint32_t)CAP && d > S.grp[k]) S.grp[++k] = d;
            S.grp[++k] = 256;
            S.ngroups = k;
        }
        __syncthreads();
        if (tid < 256) S.texcl[tid] = S.sub[tid];            // scatter cursors
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            const uint64_t r = g[i];
            a[atomicAdd(&S.texcl[((uint32_t)(r >> 32) >> sh) & 0xffu], 1u)] = r;
        }
        __syncthreads();
    }
    const int ngroups = split ? (int)S.ngroups : 1;
    const uint64_t *src = split ? a : g;
    for (int k = 0; k < ngroups; ++k) {
        const int b0 = split ? (int)S.sub[S.grp[k]] : 0;
        const int m = split ? (int)S.sub[S.grp[k + 1]] - b0 : n;
        if (m == 0) continue;                                 // uniform
        if (!SPLIT || m <= CAP) {
            // chunks of a split bucket span a narrow depth range: the one-pass bucket-rank
            // sort almost always takes them; the four-pass radix is the fallback
            if (SPLIT && B != nullptr &&
                tb_sort_range<NT, EMAX>(*B, src + b0, m, start + b0, tile_hi, vals_out, keys_out,
                                        write_keys)) {
                __syncthreads();
                continue;
            }
            ts_sort_small<NT, EMAX>(S, src + b0, m, 4);
            for (int i = tid; i < m; i += NT) {
                const uint64_t r = s[i];
                vals_out[start + b0 + i] = (uint32_t)r;
                if (write_keys) keys_out[start + b0 + i] = tile_hi | (r >> 32);
            }
        } else {                                              // one bin alone exceeds CAP
            ts_bitonic_global<NT, EMAX>(S, a + b0, m);
            for (int i = tid; i < m; i += NT) {
                const uint64_t r = a[b0 + i];
                vals_out[start + b0 + i] = (uint32_t)r;
                if (write_keys) keys_out[start + b0 + i] = tile_hi | (r >> 32);
            }
        }
        if (split) __syncthreads();
    }
}

// A dense bucket (more records than any class's shared memory holds) inside a size-class
// kernel: the same split as ts_sort_tile's -- one counting pass on the top 8 varying depth bits
// into `alt` (through L2), consecutive bins grouped into chunks of at most CAP records -- with
// every chunk sorted by the class's own bucket-rank sort.  Returns false when a chunk cannot
// be (one bin alone beyond CAP, clustered depths): the caller queues the tile for the tail
// kernel, which sorts it again from `rec` (untouched here).
struct SplitSmem {
    uint32_t sub[257];
    uint32_t grp[258];
    uint32_t mm[2];
    uint32_t ngroups, bad;
};      // (2 KB: with it the medium class still fits 3 CTAs per SM)
template <int NT, int EMAX, bool STAGE, int NBDIV>
__device__ __forceinline__ bool tb_sort_dense(BucketSmem<NT, EMAX, STAGE, NBDIV> &B, SplitSmem &S, int tile,
                                              const uint64_t *__restrict__ rec, uint64_t *alt,
                                              uint32_t *__restrict__ vals_out, uint64_t *keys_out,
                                              const int32_t *__restrict__ starts, int write_keys)
{
    constexpr int CAP = BucketSmem<NT, EMAX, STAGE, NBDIV>::CAP;
    const int tid = threadIdx.x;
    const int start = starts[tile], n = starts[tile + 1] - start;
    if (n <= 0) return true;
    const uint64_t *g = rec + start;
    uint64_t *a = alt + start;
    if (tid == 0) { S.mm[0] = 0xffffffffu; S.mm[1] = 0u; S.bad = 0u; }
    for (int i = tid; i < 257; i += NT) S.sub[i] = 0u;
    __syncthreads();
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int i = tid; i < n; i += NT) {
        const uint32_t d = (uint32_t)(g[i] >> 32);
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
    }
    lo = __reduce_min_sync(FGS_FULL, lo);
    hi = __reduce_max_sync(FGS_FULL, hi);
    if ((tid & 31) == 0) { atomicMin(&S.mm[0], lo); atomicMax(&S.mm[1], hi); }
    __syncthreads();
    const uint32_t diff = S.mm[0] ^ S.mm[1];
    const int top = diff ? 31 - __clz((int)diff) : 0;        // highest varying depth bit
    const int sh = top > 7 ? top - 7 : 0;                     // bin = depth bits [sh, sh+8)
    for (int i = tid; i < n; i += NT)
        atomicAdd(&S.sub[1 + (((uint32_t)(g[i] >> 32) >> sh) & 0xffu)], 1u);
    __syncthreads();
    if (tid == 0) {
        uint32_t run = 0;
        for (int d = 0; d <= 256; ++d) { run += S.sub[d]; S.sub[d] = run; }
        uint32_t k = 0;
        S.grp[0] = 0;
        for (uint32_t d = 0; d < 256; ++d)
            if (S.sub[d + 1] - S.sub[S.grp[k]] > (uint32_t)CAP && d > S.grp[k]) S.grp[++k] = d;
        S.grp[++k] = 256;
        S.ngroups = k;
        for (uint32_t j = 0; j < k; ++j)
            if (S.sub[S.grp[j + 1]] - S.sub[S.grp[j]] > (uint32_t)CAP) S.bad = 1u;
    }
    __syncthreads();
    if (S.bad) return false;                                  // uniform
    uint32_t *cur = B.bin;                                    // scatter cursors (B is idle until the chunks)
    static_assert(BucketSmem<NT, EMAX, STAGE, NBDIV>::NB >= 256, "cursor array");
    if (tid < 256) cur[tid] = S.sub[tid];
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
        const uint64_t r = g[i];
        a[atomicAdd(&cur[((uint32_t)(r >> 32) >> sh) & 0xffu], 1u)] = r;
    }
    __syncthreads();
    const int ngroups = (int)S.ngroups;
    const uint64_t tile_hi = (uint64_t)(uint32_t)tile << 32;
    for (int k = 0; k < ngroups; ++k) {
        const int b0 = (int)S.sub[S.grp[k]];
        const int m = (int)S.sub[S.grp[k + 1]] - b0;
        if (m == 0) continue;                                 // uniform
        // keys_out may alias alt: a chunk is consumed (staged / scattered into shared memory)
        // before its slice is overwritten
        if (!tb_sort_range<NT, EMAX, STAGE, NBDIV>(B, a + b0, m, start + b0, tile_hi, vals_out, keys_out,
                                                   write_keys))
            return false;
        __syncthreads();
    }
    return true;
}

// Persistent size-class kernels: CTA b sorts list entry b first and then takes further
// entries from a ticket counter (the frame's zeroed work block: word `slot` = tickets drawn,
// word `slot + 1` = CTAs that have left) -- tiles of one class differ 2x in size, and a
// static stride leaves SMs idle behind the unlucky CTAs.  The next ticket is drawn before
// the current tile is sorted, so its round trip is hidden; CTAs without a first entry never
// touch the counter (L2 serialises same-address atomics: ~20 ns each).  The last working CTA
// out rewinds both words, so the stage can be re-issued on the frame.
struct TileTickets {
    uint32_t *ctr;
    uint32_t next, count;
    // false: this CTA has no work at all
    __device__ __forceinline__ bool open(fgs_stats *stats, int slot, uint32_t n)
    {
        ctr = fgs_work(stats) + slot;
        count = n;
        next = blockIdx.x;
        return blockIdx.x < n;
    }
    // returns the list entry this CTA sorts now (uniform; >= count: done), draws the one after
    __device__ __forceinline__ uint32_t take(uint32_t *bcast)
    {
        if (threadIdx.x == 0) {
            *bcast = next;
            if (next < count) next = gridDim.x + atomicAdd(ctr, 1u);
        }
        __syncthreads();
        const uint32_t i = *bcast;
        __syncthreads();
        return i;
    }
    // `done_bit`: raised in FGS_WORK_SORT_DONE by the last worker out, after every worker's
    // output is visible device-wide -- the tail kernel's explicit join with this class.  (The
    // classes are chained by launch_dependents WITHOUT a griddepcontrol.wait of their own, so
    // that they overlap; stream order alone then only promises the tail kernel its immediate
    // predecessor.)  The caller's loop ends with a barrier: every thread's stores precede this.
    __device__ __forceinline__ void close(fgs_stats *stats, uint32_t done_bit)
    {
        const uint32_t workers = count < gridDim.x ? count : gridDim.x;
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(ctr + 1, 1u) == workers - 1u) {
                ctr[0] = 0u;
                ctr[1] = 0u;
                __threadfence();
                atomicOr(fgs_work(stats) + FGS_WORK_SORT_DONE, done_bit);
            }
        }
    }
};

// Size classes (k_scan_tiles sorts the tiles into them):
//   small   n <= 2048   one CTA per tile, bucket-rank sort (4 or 8 records per thread)
//   medium  n <= 4096   persistent CTAs over the medium list, bucket-rank sort
//   large   n <= 8192   512 threads, bucket-rank sort without the staging copy
//   hard    n <= 4096   small / medium tiles the bucket-rank sort gave up on: radix sort
//   dense   n >  8192   (and large tiles that gave up) one counting pass on the top varying
//                       depth bits, then each chunk of <= 4096 by bucket-rank (radix fallback)
#ifndef FGS_MED_NBDIV
#define FGS_MED_NBDIV 2           // medium class: 2048 depth bins (rank loops half as long; 3 x 74 KB per SM)
#endif
#ifndef FGS_SMALL_NBDIV
#define FGS_SMALL_NBDIV 2         // small class: 512 / 1024 bins (37 KB, still 6 CTAs per SM)
#endif
__global__ void __launch_bounds__(256, 6)
k_tile_sort(const uint64_t *__restrict__ rec, uint32_t *__restrict__ vals_out,
            uint64_t *__restrict__ keys_out, const int32_t *__restrict__ starts,
            const uint32_t *__restrict__ small_list, uint32_t *__restrict__ hard_list,
            int write_keys, fgs_stats *__restrict__ stats)
{
    // one buffer, two instantiations: up to 1024 records with 4 per thread, up to 2048 with 8
    // (35 KB, 6 CTAs per SM).  Persistent CTAs over the list of small tiles the tile scan
    // queued (tickets: the tiles differ 1 : 2048 in size): two thirds of a frame's tiles are
    // empty and a sixth is heavy, and with one CTA per tile of the grid this kernel spent more
    // time starting CTAs that found nothing to do (10M / 4K: 55 -> 48 us, 8K frame:
    // 241 -> 184 us; C2, a grid of 8160 tiles: 24.5 -> 27 us -- the tickets cost a little).
    __shared__ __align__(16) unsigned char raw[sizeof(BucketSmem<256, 8, true, FGS_SMALL_NBDIV>)];
    __shared__ uint32_t s_ticket;
    if (stats->overflow) return;
    const uint32_t count = fgs_work(stats)[FGS_WORK_SMALL];
    TileTickets tk;
    if (!tk.open(stats, FGS_WORK_SMALL_TICKET, count)) return;
    for (uint32_t i = tk.take(&s_ticket); i < count; i = tk.take(&s_ticket)) {
        const int tile = (int)small_list[(size_t)i * FGS_CTR_STRIDE];
        const int n = starts[tile + 1] - starts[tile];
        const bool ok = n <= BucketSmem<256, 4>::CAP
            ? tb_sort_tile<256, 4, true, FGS_SMALL_NBDIV>(*reinterpret_cast<BucketSmem<256, 4, true, FGS_SMALL_NBDIV> *>(raw), tile, rec, vals_out,
                                   keys_out, starts, write_keys)
            : tb_sort_tile<256, 8, true, FGS_SMALL_NBDIV>(*reinterpret_cast<BucketSmem<256, 8, true, FGS_SMALL_NBDIV> *>(raw), tile, rec, vals_out,
                                   keys_out, starts, write_keys);
        if (!ok &&
            threadIdx.x == 0)
            hard_list[(size_t)atomicAdd(&stats->hard_tiles, 1u) * FGS_CTR_STRIDE] = (uint32_t)tile;
        __syncthreads();
    }
    tk.close(stats, 4u);
}

// medium class: threads per CTA x records per thread = 4096 (tuning knobs)
#ifndef FGS_MED_NT
#define FGS_MED_NT   512
#endif
#ifndef FGS_MED_MINB
#define FGS_MED_MINB 3
#endif
#ifndef FGS_MED_STAGE
#define FGS_MED_STAGE true       // records staged in shared memory (false: re-read from L2)
#endif
#ifndef FGS_LARGE_NT
#define FGS_LARGE_NT 512
#endif
#ifndef FGS_LARGE_MINB
#define FGS_LARGE_MINB 3       // 40 registers, 3 x 73 KB of shared memory per SM (2: 302 us at 10M@4K, 3: 256)
#endif
#define FGS_MED_EMAX (4096 / FGS_MED_NT)
__global__ void __launch_bounds__(FGS_MED_NT, FGS_MED_MINB)
k_tile_sort_medium(const uint64_t *__restrict__ rec, uint32_t *__restrict__ vals_out,
                   uint64_t *keys_out, const int32_t *__restrict__ starts,
                   const uint32_t *__restrict__ list, uint32_t *__restrict__ hard_list,
                   uint32_t *dense_list, int write_keys, fgs_stats *__restrict__ stats, int lazy)
{
    extern __shared__ __align__(16) unsigned char ts_raw[];
    using Smem = BucketSmem<FGS_MED_NT, FGS_MED_EMAX, FGS_MED_STAGE, FGS_MED_NBDIV>;
    Smem &S = *reinterpret_cast<Smem *>(ts_raw);
    // first of the size classes: waits for the placement kernel, then lets the next class
    // (disjoint tiles, launched without a wait of its own) start beside this one
    fgs_pdl_wait();
    fgs_pdl_trigger();
    if (stats->overflow) return;
    __shared__ uint32_t s_ticket;
    __shared__ SplitSmem s_split;
    // The dense tiles the scan queued come first (the longest jobs of the whole sort: split in
    // place, chunk by chunk, beside the other classes -- left to the tail kernel they were 61 us
    // of a mostly idle GPU on the 10M / 4K frame), then the medium list.
    // (lazy_sort: the dense tiles -- and with lazy == 2 the medium ones too -- are the front
    // kernel's; this kernel still opens the chain for the classes launched behind it)
    const uint32_t nd0 = lazy ? 0u : fgs_work(stats)[FGS_WORK_DENSE0];
    const uint32_t count = nd0 + (lazy == 2 ? 0u : stats->medium_tiles);
    TileTickets tk;
    if (!tk.open(stats, FGS_WORK_MEDIUM_TICKET, count)) return;
    for (uint32_t i = tk.take(&s_ticket); i < count; i = tk.take(&s_ticket)) {
        if (i < nd0) {
            const int tile = (int)dense_list[(size_t)i * FGS_CTR_STRIDE];
            if (!tb_sort_dense<FGS_MED_NT, FGS_MED_EMAX, FGS_MED_STAGE, FGS_MED_NBDIV>(
                    S, s_split, tile, rec, keys_out, vals_out, keys_out, starts, write_keys) &&
                threadIdx.x == 0)      // back of the dense list: the tail kernel's share
                dense_list[(size_t)atomicAdd(&stats->dense_tiles, 1u) * FGS_CTR_STRIDE] = (uint32_t)tile;
        } else {
            const int tile = (int)list[(size_t)(i - nd0) * FGS_CTR_STRIDE];
            if (!tb_sort_tile<FGS_MED_NT, FGS_MED_EMAX, FGS_MED_STAGE, FGS_MED_NBDIV>(S, tile, rec, vals_out, keys_out, starts, write_keys) &&
                threadIdx.x == 0)
                hard_list[(size_t)atomicAdd(&stats->hard_tiles, 1u) * FGS_CTR_STRIDE] = (uint32_t)tile;
        }
        __syncthreads();
    }
    tk.close(stats, 1u);
}

__global__ void __launch_bounds__(FGS_LARGE_NT, FGS_LARGE_MINB)
k_tile_sort_large(const uint64_t *__restrict__ rec, uint32_t *__restrict__ vals_out,
                  uint64_t *__restrict__ keys_out, const int32_t *__restrict__ starts,
                  const uint32_t *__restrict__ list, uint32_t *__restrict__ dense_list,
                  int write_keys, fgs_stats *__restrict__ stats)
{
    extern __shared__ __align__(16) unsigned char ts_raw[];
    using Smem = BucketSmem<FGS_LARGE_NT, 8192 / FGS_LARGE_NT, false>;
    Smem &S = *reinterpret_cast<Smem *>(ts_raw);
    fgs_pdl_trigger();      // no wait: released only after the medium class's wait returned
    if (stats->overflow) return;
    __shared__ uint32_t s_ticket;
    const uint32_t count = fgs_work(stats)[FGS_WORK_LARGE];
    TileTickets tk;
    if (!tk.open(stats, FGS_WORK_LARGE_TICKET, count)) return;
    for (uint32_t i = tk.take(&s_ticket); i < count; i = tk.take(&s_ticket)) {
        const int tile = (int)list[(size_t)i * FGS_CTR_STRIDE];
        if (!tb_sort_tile<FGS_LARGE_NT, 8192 / FGS_LARGE_NT, false>(S, tile, rec, vals_out, keys_out, starts, write_keys) &&
            threadIdx.x == 0)      // clustered depths: let the splitting kernel take it
            dense_list[(size_t)atomicAdd(&stats->dense_tiles, 1u) * FGS_CTR_STRIDE] = (uint32_t)tile;
        __syncthreads();
    }
    tk.close(stats, 2u);
}


// ---- lazy_sort: the front of a heavy tile ------------------------------------------------
// Front-to-back compositing stops once every pixel of a tile is opaque (render.py:154, 178,
// 228-229), and a tile holding thousands of pairs is opaque after a few hundred of them
// (measured on every benchmark frame: the last pair any pixel consumes sits at position
// 200-400 in the median heavy tile, beyond 1024 in at most 2 % of them -- tools/lazy_probe.py
// -- while heavy tiles hold 75-97 % of a frame's pairs).  So of a heavy tile only the nearest
// pairs are put in order: every record whose depth bin lies at or below the bin that takes the
// cumulative count past FGS_FRONT_MIN.  Bins are a monotone function of the depth bits, so this
// front is exactly the head of the tile's fully sorted list, F records long; limit[tile] = F
// tells the blend where the sorted part ends.  A tile that has not saturated by then goes on
// the redo list: k_tile_sort_redo sorts it in full and the blend composites it again from
// scratch (fgs_launch_blend_redo), so the frame never depends on the guess.
//
// Per tile: the depth range from a strided sample of 512 records (depths outside it clamp to
// the end bins, which keeps the map monotone), one pass that counts every record into 2048
// linear depth bins (shared-memory RED, no return value needed), a scan, one pass that
// scatters the front's records bin-contiguously into shared memory, and the in-bin ranking of
// those F records only.  Two reads of the bucket, ~17 instructions per record, against three
// reads and ~60 for the full bucket-rank sort; 33 KB of shared memory and 32 registers, so
// four 512-thread CTAs per SM hide the reads.
#ifndef FGS_FRONT_NT
#define FGS_FRONT_NT   512
#endif
#ifndef FGS_FRONT_MINB
#define FGS_FRONT_MINB 4         // 32 registers (the 16 depth words of a thread partly in local
                                 // memory, L1-resident): 134 us on the 10M / 4K frame against 138 at 3
#endif
#ifndef FGS_FRONT_CAP
#define FGS_FRONT_CAP  3072      // records a front may hold (24 KB)
#endif
#ifndef FGS_FRONT_MIN
#define FGS_FRONT_MIN  1024      // the front ends with the bin that takes it to at least this many
#endif
#ifndef FGS_FRONT_E
#define FGS_FRONT_E    16        // depth words a thread keeps in registers (one chunk = 8192 records)
#endif
#define FGS_FRONT_LOW  256       // a front cut short of a clustered bin must still hold this many
#define FGS_FRONT_NB   2048
struct FrontSmem {
    uint64_t b[FGS_FRONT_CAP];
    uint32_t bin[FGS_FRONT_NB + 1];
    uint32_t red[64];
    int32_t  pick[2];
};

// Returns F, the number of sorted records now at vals_out[start, start + F); 0 = gave up
// (one depth bin alone overflows the front: clustered depths -- the redo path sorts the tile).
// Every thread of the CTA calls it with the same arguments; n >= FGS_FRONT_NT.
//
// A bucket of up to NT * FGS_FRONT_E records (8192: the large class, 3/4 of the pairs of the
// 10M / 4K frame) is read ONCE: every thread keeps the depth words of its FGS_FRONT_E records
// in registers -- all their loads in flight together -- takes the exact depth range from them,
// counts them, and after the scan fetches the full record only of those that made the front.
// Larger buckets go through the same code chunk by chunk, twice (range from a strided sample).
__device__ __forceinline__ int front_sort_tile(FrontSmem &S, int tile, const uint64_t *__restrict__ rec,
                                               uint32_t *__restrict__ vals_out,
                                               const int32_t *__restrict__ starts)
{
    constexpr int NT = FGS_FRONT_NT, NB = FGS_FRONT_NB, E = FGS_FRONT_E, CH = NT * E;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int start = starts[tile], n = starts[tile + 1] - start;
    const uint64_t *g = rec + start;
    const uint32_t *gd = reinterpret_cast<const uint32_t *>(g) + 1;     // depth word of record i: gd[2 i]
    const bool one = n <= CH;                                 // uniform
    uint32_t dreg[E];
    const auto load_chunk = [&](int c0) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int i = c0 + tid + k * NT;
            dreg[k] = i < n ? gd[2 * i] : 0xffffffffu;
        }
    };

    // 1. depth range: exact from the registers, or of a strided sample (depths outside it
    // clamp to the end bins, which keeps the map monotone)
    {
        uint32_t lo = 0xffffffffu, hi = 0u;
        if (one) {
            load_chunk(0);
#pragma unroll
            for (int k = 0; k < E; ++k) {
                if (tid + k * NT < n) {
                    lo = dreg[k] < lo ? dreg[k] : lo;
                    hi = dreg[k] > hi ? dreg[k] : hi;
                }
            }
        } else {
            lo = hi = gd[2 * (int)(((int64_t)tid * n) / NT)];
        }
        lo = __reduce_min_sync(FGS_FULL, lo);
        hi = __reduce_max_sync(FGS_FULL, hi);
        if (lane == 0) { S.red[w] = lo; S.red[32 + w] = hi; }
    }
    for (int i = tid; i <= NB; i += NT) S.bin[i] = 0u;
    __syncthreads();
    uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        lo = S.red[i] < lo ? S.red[i] : lo;
        hi = S.red[32 + i] > hi ? S.red[32 + i] : hi;
    }
    // bin = (depth bits - lo) >> sh with the smallest shift that maps the range below NB:
    // monotone, one instruction, and between NB / 2 and NB bins in use
    const uint32_t range = hi - lo;
    const int sh = range < (uint32_t)NB ? 0 : 32 - __clz((int)(range >> 11));
    static_assert(FGS_FRONT_NB == 2048, "shift = bits of (range >> log2 NB)");
    const auto bin_of = [&](uint32_t d) -> uint32_t {
        return ((d < lo ? lo : (d > hi ? hi : d)) - lo) >> sh;
    };

    // 2. count every record into its bin
    for (int c0 = 0; c0 < n; c0 += CH) {
        if (!one) load_chunk(c0);
#pragma unroll
        for (int k = 0; k < E; ++k)
            if (c0 + tid + k * NT < n) atomicAdd(&S.bin[1 + bin_of(dreg[k])], 1u);
    }
    __syncthreads();

    // 3. bin offsets: inclusive scan of bin[1..NB] in place (bin[0] = 0), and the front's last bin
    {
        constexpr int PER = NB / NT;                          // consecutive bins per thread
        uint32_t v[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            v[k] = S.bin[1 + tid * PER + k];
            sum += v[k];
        }
        const uint32_t incl = warp_incl_scan(sum, lane);
        if (lane == 31) S.red[w] = incl;
        __syncthreads();
        const uint32_t wsum = lane < NT / 32 ? S.red[lane] : 0u;
        const uint32_t wincl = warp_incl_scan(wsum, lane);
        uint32_t run = __shfl_sync(FGS_FULL, wincl - wsum, w) + incl - sum;
        const uint32_t want = (uint32_t)(n < FGS_FRONT_MIN ? n : FGS_FRONT_MIN);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int bn = tid * PER + k;                     // bin bn = [run, run + v[k])
            const uint32_t end = run + v[k];
            if (run < want && end >= want) {                  // exactly one bin of the tile
                int bf = bn, F = (int)end;
                if (end > (uint32_t)FGS_FRONT_CAP) {
                    if (run >= (uint32_t)FGS_FRONT_LOW) { bf = bn - 1; F = (int)run; }
                    else { bf = -1; F = 0; }
                }
                S.pick[0] = bf;
                S.pick[1] = F;
            }
            S.bin[1 + bn] = end;
            run = end;
        }
    }
    __syncthreads();
    const int bf = S.pick[0], F = S.pick[1];
    if (bf < 0) return 0;                                      // uniform

    // 4. the front's records, bin-contiguous: bin[bn] is bin bn's cursor, and its end afterwards
    for (int c0 = 0; c0 < n; c0 += CH) {
        if (!one) load_chunk(c0);
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int i = c0 + tid + k * NT;
            if (i < n) {
                const uint32_t bn = bin_of(dreg[k]);
                if (bn <= (uint32_t)bf)
                    S.b[atomicAdd(&S.bin[bn], 1u)] = ((uint64_t)dreg[k] << 32) | (uint32_t)g[i];
            }
        }
    }
    __syncthreads();

    // 5. rank inside the bin by full-word comparison (settles equal depths by index)
    for (int i = tid; i < F; i += NT) {
        const uint64_t r = S.b[i];
        const uint32_t bn = bin_of((uint32_t)(r >> 32));
        const int b0 = bn ? (int)S.bin[bn - 1] : 0, b1 = (int)S.bin[bn];
        int rank = 0;
        for (int j = b0; j < b1; ++j) rank += S.b[j] < r ? 1 : 0;
        vals_out[start + b0 + rank] = (uint32_t)r;
    }
    return F;
}

__global__ void __launch_bounds__(FGS_FRONT_NT, FGS_FRONT_MINB)
k_tile_front(const uint64_t *__restrict__ rec, uint32_t *__restrict__ vals_out,
             const int32_t *__restrict__ starts, const uint32_t *__restrict__ dense_list,
             const uint32_t *__restrict__ large_list, const uint32_t *__restrict__ medium_list,
             int take_medium, int32_t *__restrict__ limit, fgs_stats *__restrict__ stats)
{
    extern __shared__ __align__(16) unsigned char ts_raw[];
    FrontSmem &S = *reinterpret_cast<FrontSmem *>(ts_raw);
    fgs_pdl_trigger();      // no wait, as the large class it stands in for: released only after
                            // the medium kernel's wait returned
    if (stats->overflow) return;
    __shared__ uint32_t s_ticket;
    const uint32_t nd0 = fgs_work(stats)[FGS_WORK_DENSE0], nl = fgs_work(stats)[FGS_WORK_LARGE];
    const uint32_t count = nd0 + nl + (take_medium ? stats->medium_tiles : 0u);
    TileTickets tk;
    if (!tk.open(stats, FGS_WORK_LARGE_TICKET, count)) return;
    for (uint32_t i = tk.take(&s_ticket); i < count; i = tk.take(&s_ticket)) {
        const int tile = (int)(i < nd0 ? dense_list[(size_t)i * FGS_CTR_STRIDE]
                               : i < nd0 + nl ? large_list[(size_t)(i - nd0) * FGS_CTR_STRIDE]
                                              : medium_list[(size_t)(i - nd0 - nl) * FGS_CTR_STRIDE]);
        const int F = front_sort_tile(S, tile, rec, vals_out, starts);
        if (threadIdx.x == 0) limit[tile] = F;
        __syncthreads();
    }
    tk.close(stats, 2u);
}

// The tail of the tile sort, one launch: the dense list (split path), then the hard list
// (small / medium buckets the bucket-rank sort gave up on: radix path, no second try).
__global__ void __launch_bounds__(256, 2)
k_tile_sort_tail(uint64_t *__restrict__ rec, uint64_t *__restrict__ alt,
                 uint32_t *__restrict__ vals_out, uint64_t *__restrict__ keys_out,
                 const int32_t *__restrict__ starts, const uint32_t *__restrict__ dense_list,
                 const uint32_t *__restrict__ hard_list, int write_keys,
                 fgs_stats *__restrict__ stats, int lazy)
{
    fgs_pdl_trigger();      // plain launch; the blend may queue up behind this grid

    extern __shared__ __align__(16) unsigned char ts_raw[];
    using Radix = TileSortSmem<256, 16>;
    Radix &S = *reinterpret_cast<Radix *>(ts_raw);
    // a bucket-rank work area behind the radix one, for the chunks of split buckets
    BucketSmem<256, 16> *B = reinterpret_cast<BucketSmem<256, 16> *>(
        ts_raw + ((sizeof(Radix) + 15) & ~size_t(15)));
    if (stats->overflow) return;
    // Explicit join with the medium and large classes (see TileTickets::close): they were
    // launched before this grid's stream predecessor and every CTA of theirs is resident,
    // so the flags arrive without this grid's help.  The wait is bounded: a frame that
    // never sees them is reported as unsorted instead of hanging the device.
    __shared__ uint32_t s_joined;
    if (threadIdx.x == 0) {
        uint32_t *work = fgs_work(stats);
        // (lazy_sort: bit 1 is the front kernel's, which takes the dense and large tiles and
        // with lazy == 2 the medium ones; the medium kernel keeps what is left)
        const uint32_t nmed = lazy == 2 ? 0u : stats->medium_tiles, nd = work[FGS_WORK_DENSE0];
        // the frame's heavy tiles -- those lazy_sort orders a front of -- reported either way:
        // the host arms lazy_sort only for frames that have enough of them to pay for its two
        // extra launches
        if (blockIdx.x == 0)
            stats->front_tiles = nd + work[FGS_WORK_LARGE];      // (level 2 adds stats->medium_tiles)
        const uint32_t need = (lazy ? ((nmed ? 1u : 0u) | ((nd | work[FGS_WORK_LARGE] | (stats->medium_tiles - nmed)) ? 2u : 0u))
                                    : (((nmed | nd) ? 1u : 0u) | (work[FGS_WORK_LARGE] ? 2u : 0u))) |
                              (work[FGS_WORK_SMALL] ? 4u : 0u);
        volatile uint32_t *done = work + FGS_WORK_SORT_DONE;
        uint32_t ok = 1u;
        for (uint32_t spin = 0; (*done & need) != need; ++spin) {
            if (spin > (1u << 23)) { ok = 0u; stats->unsorted = 1u; break; }
            __nanosleep(200);
        }
        __threadfence();
        s_joined = ok;
        // the last CTA past the join rewinds the flags (the stage may be re-issued on the frame)
        if (atomicAdd(work + FGS_WORK_TAIL_OUT, 1u) == gridDim.x - 1u) {
            work[FGS_WORK_SORT_DONE] = 0u;
            work[FGS_WORK_TAIL_OUT] = 0u;
        }
    }
    __syncthreads();
    if (!s_joined) return;
    // (the dense tiles the scan queued were split by the medium class; what it or the large
    // class could not sort sits behind them in the dense list)
    const uint32_t nd0 = fgs_work(stats)[FGS_WORK_DENSE0];
    const uint32_t ndense = stats->dense_tiles - nd0, nhard = stats->hard_tiles;
    for (uint32_t i = blockIdx.x; i < ndense + nhard; i += gridDim.x) {
        const bool dense = i < ndense;
        const int tile = (int)(dense ? dense_list[(size_t)(nd0 + i) * FGS_CTR_STRIDE]
                                     : hard_list[(size_t)(i - ndense) * FGS_CTR_STRIDE]);
        ts_sort_tile<256, 16, true>(S, tile, rec, alt, vals_out, keys_out, starts, write_keys,
                                    dense ? B : nullptr);
        __syncthreads();
    }
}


// lazy_sort: the tiles the blend found unsaturated at the end of their sorted front, sorted in
// full by the tail kernel's general path (any size: split on the top varying depth bits,
// bucket-rank per chunk, radix / bitonic fallbacks).  Rare by construction; rec is untouched
// by everything before, so the sort starts from the tile's bucket as the scatter left it.
__global__ void __launch_bounds__(256, 2)
k_tile_sort_redo(uint64_t *__restrict__ rec, uint64_t *__restrict__ alt,
                 uint32_t *__restrict__ vals_out, const int32_t *__restrict__ starts,
                 const uint32_t *__restrict__ redo_list, fgs_stats *__restrict__ stats)
{
    fgs_pdl_wait();
    fgs_pdl_trigger();
    extern __shared__ __align__(16) unsigned char ts_raw[];
    using Radix = TileSortSmem<256, 16>;
    Radix &S = *reinterpret_cast<Radix *>(ts_raw);
    BucketSmem<256, 16> *B = reinterpret_cast<BucketSmem<256, 16> *>(
        ts_raw + ((sizeof(Radix) + 15) & ~size_t(15)));
    if (stats->overflow) return;
    const uint32_t n = fgs_work(stats)[FGS_WORK_REDO];
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        ts_sort_tile<256, 16, true>(S, (int)redo_list[i], rec, alt, vals_out, alt, starts, 0, B);
        __syncthreads();
    }
}

}  // namespace

int fgs_launch_tile_sort(const FrameDev &f, int tiles, int write_keys, int lazy, cudaStream_t st)
{
    if (tiles <= 0) return FGS_OK;
    using MediumSmem = BucketSmem<FGS_MED_NT, FGS_MED_EMAX, FGS_MED_STAGE, FGS_MED_NBDIV>;
    using LargeSmem = BucketSmem<FGS_LARGE_NT, 8192 / FGS_LARGE_NT, false>;
    static_assert(LargeSmem::CAP == FGS_LARGE_TILE, "large class = large capacity");
    using TailRadix = TileSortSmem<256, 16>;
    constexpr size_t tail_bytes = ((sizeof(TailRadix) + 15) & ~size_t(15)) + sizeof(BucketSmem<256, 16>);
    static_assert(BucketSmem<256, 8>::CAP == FGS_SMALL_TILE, "small class = small capacity");
    static_assert(MediumSmem::CAP == FGS_DENSE_TILE && TailRadix::CAP == FGS_DENSE_TILE,
                  "medium capacity = radix capacity = chunk size of split buckets");
    static FgsOncePerDevice attr_once;
    int attr_dev = 0;
    if (attr_once.need(&attr_dev)) {
        cudaError_t e = cudaSuccess;
        auto prep = [&](const void *fn, size_t smem) {
            if (e == cudaSuccess && smem)
                e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            // largest shared-memory carve-out, or the occupancy the launch bounds assume
            // (6 x 17 KB, 3 x 69 KB, 3 x 73 KB, 2 x 112 KB per SM) is not reached
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared);
        };
        prep((const void *)k_tile_sort, 0);
        prep((const void *)k_tile_sort_medium, sizeof(MediumSmem));
        prep((const void *)k_tile_sort_large, sizeof(LargeSmem));
        prep((const void *)k_tile_sort_tail, tail_bytes);
        prep((const void *)k_tile_front, sizeof(FrontSmem));
        prep((const void *)k_tile_sort_redo, tail_bytes);
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        attr_once.mark(attr_dev);
    }
    int dev = 0, sms = 148;                 // per call: the persistent grids are sized for THIS device
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // lists in the spare words of the cursor slots: +1 dense, +2 medium, +3 hard
    uint32_t *dense_list = f.cursor + 1, *medium_list = f.cursor + 2, *hard_list = f.cursor + 3;
    uint32_t *large_list = f.cursor + 4;
    const unsigned mgrid = (unsigned)(tiles < FGS_MED_MINB * sms ? tiles : FGS_MED_MINB * sms);
    const unsigned dgrid = (unsigned)(tiles < FGS_LARGE_MINB * sms ? tiles : FGS_LARGE_MINB * sms);
    const unsigned tgrid = (unsigned)(tiles < 2 * sms ? tiles : 2 * sms);   // tail: 2 CTAs/SM, static stride
    // The small / medium / large classes sort disjoint tiles, so they may run side by side:
    // the persistent kernels go first (all their CTAs are resident at once and trigger
    // `griddepcontrol.launch_dependents` on entry), the next class is launched with
    // programmatic stream serialization and starts beside them instead of behind their tail.
    // None of them reads what another writes; the tail kernel (plain launch) waits for all.
    // With per-kernel profiling events armed the classes run back to back as before.
    const bool overlap = !fgs_prof_armed();
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = pdl;
    {
        FGS_CHAIN(k_tile_sort_medium, dim3(mgrid), dim3(FGS_MED_NT), sizeof(MediumSmem), st,
                  f.keys[0], f.vals[0], f.keys[1], f.starts, medium_list, hard_list, dense_list, write_keys, f.stats,
                  lazy);
        FGS_AFTER_LAUNCH(st);
    }
    if (lazy) {
        // the front kernel stands in for the large class (same place in the chain, same ticket
        // and done-flag words) and also takes the dense tiles
        cfg.gridDim = dim3((unsigned)(tiles < FGS_FRONT_MINB * sms ? tiles : FGS_FRONT_MINB * sms));
        cfg.blockDim = dim3(FGS_FRONT_NT);
        cfg.dynamicSmemBytes = sizeof(FrontSmem);
        cfg.numAttrs = overlap ? 1 : 0;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k_tile_front, (const uint64_t *)f.keys[0], f.vals[0],
            (const int32_t *)f.starts, (const uint32_t *)dense_list, (const uint32_t *)large_list,
            (const uint32_t *)medium_list, lazy == 2 ? 1 : 0, f.limit, f.stats);
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        FGS_AFTER_LAUNCH(st);
    } else {
        cfg.gridDim = dim3(dgrid);
        cfg.blockDim = dim3(FGS_LARGE_NT);
        cfg.dynamicSmemBytes = sizeof(LargeSmem);
        cfg.numAttrs = overlap ? 1 : 0;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k_tile_sort_large, (const uint64_t *)f.keys[0],
            f.vals[0], f.keys[1], (const int32_t *)f.starts, (const uint32_t *)large_list, dense_list,
            write_keys, f.stats);
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        FGS_AFTER_LAUNCH(st);
    }
    {
        cfg.gridDim = dim3((unsigned)(tiles < 6 * sms ? tiles : 6 * sms));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 0;
        cfg.numAttrs = overlap ? 1 : 0;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k_tile_sort, (const uint64_t *)f.keys[0],
            f.vals[0], f.keys[1], (const int32_t *)f.starts, (const uint32_t *)(f.cursor + 7), hard_list,
            write_keys, f.stats);
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        FGS_AFTER_LAUNCH(st);
    }
    k_tile_sort_tail<<<tgrid, 256, tail_bytes, st>>>(f.keys[0], f.keys[1], f.vals[0], f.keys[1],
                                                     f.starts, dense_list, hard_list, write_keys,
                                                     f.stats, lazy);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

// lazy_sort: full sort of the tiles on the redo list (behind the first blend pass)
int fgs_launch_tile_sort_redo(const FrameDev &f, int tiles, cudaStream_t st)
{
    if (tiles <= 0) return FGS_OK;
    using TailRadix = TileSortSmem<256, 16>;
    constexpr size_t tail_bytes = ((sizeof(TailRadix) + 15) & ~size_t(15)) + sizeof(BucketSmem<256, 16>);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)(tiles < 2 * sms ? tiles : 2 * sms);
    FGS_CHAIN(k_tile_sort_redo, dim3(grid), dim3(256), tail_bytes, st, f.keys[0], f.keys[1], f.vals[0],
              (const int32_t *)f.starts, (const uint32_t *)f.redo_list, f.stats);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}

SortPlan fgs_sort_plan(int tile_bits, int value_bits, int compact)
{
    SortPlan pl;
    pl.npass = 0;
    pl.compact = compact;
    for (int s = 0; s < value_bits; s += 8) {
        pl.on_value[pl.npass] = 1;
        pl.shift[pl.npass] = s;
        pl.bits[pl.npass] = value_bits - s < 8 ? value_bits - s : 8;
        ++pl.npass;
    }
    const int key_bits = (compact ? 31 : 32) + tile_bits;
    for (int s = 0; s < key_bits; s += 8) {
        pl.on_value[pl.npass] = 0;
        pl.shift[pl.npass] = s;
        pl.bits[pl.npass] = key_bits - s < 8 ? key_bits - s : 8;
        ++pl.npass;
    }
    return pl;
}

int fgs_launch_sort(uint64_t *keys[2], uint32_t *vals[2], const uint32_t *n_dev, int64_t n_max,
                    const SortPlan &plan, uint64_t *state, uint32_t *hist, uint32_t *tickets,
                    uint32_t epoch, cudaStream_t st)
{
    if (n_max <= 0 || plan.npass == 0) return FGS_OK;
    if (plan.npass > FGS_SORT_MAXPASS) return FGS_E_ARG;
    static FgsOncePerDevice attr_once;
    int attr_dev = 0;
    if (attr_once.need(&attr_dev)) {
        cudaError_t e = cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(SortSmem));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        attr_once.mark(attr_dev);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

    HistArgs ha;
    ha.npass = plan.npass;
    for (int p = 0; p < plan.npass; ++p)
        ha.p[p] = PassArgs{plan.on_value[p], plan.shift[p], plan.bits[p], plan.compact};
    const int64_t want = (n_max + 256 * 16 - 1) / (256 * 16);
    const unsigned hgrid = (unsigned)(want < 1 ? 1 : (want > sms * 8 ? sms * 8 : want));
    k_sort_hist<<<hgrid, 256, plan.npass * 256 * sizeof(uint32_t), st>>>(keys[0], vals[0], n_dev, ha, hist);
    FGS_AFTER_LAUNCH(st);

    const int64_t tiles_max = (n_max + FGS_SORT_TILE - 1) / FGS_SORT_TILE;
    const unsigned pgrid = (unsigned)(tiles_max < sms * 3 ? tiles_max : sms * 3);
    for (int p = 0; p < plan.npass; ++p) {
        const int src = p & 1, dst = src ^ 1;
        k_sort_pass<<<pgrid, FGS_SORT_THREADS, sizeof(SortSmem), st>>>(
            keys[src], vals[src], keys[dst], vals[dst], n_dev, ha.p[p], hist + p * 256, state,
            tickets + p, epoch + (uint32_t)p);
        FGS_AFTER_LAUNCH(st);
    }
    return FGS_OK;
}

int fgs_launch_ranges(const uint64_t *keys, const uint32_t *n_dev, int64_t n_max, int tiles,
                      int32_t *starts, fgs_stats *stats, cudaStream_t st)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n_max + 1 + 255) / 256;
    const unsigned grid = (unsigned)(want < 1 ? 1 : (want > sms * 16 ? sms * 16 : want));
    k_tile_ranges<<<grid, 256, 0, st>>>(keys, n_dev, tiles, starts, stats);
    FGS_AFTER_LAUNCH(st);
    return FGS_OK;
}
