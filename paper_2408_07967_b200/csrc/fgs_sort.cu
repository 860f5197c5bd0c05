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
// Buckets of up to 4096 records: LSD radix sort on the four depth bytes, entirely
// in shared memory (same stable warp-match ranking as k_sort_pass, local digit
// offsets instead of a look-back), then equal-depth neighbours -- rare: two
// Gaussians with the same float32 depth in one tile -- are put in index order by
// an odd-even pass.  Larger buckets (very dense scenes) use a bitonic network in
// its all-ascending form, long strides through L2 and the rest chunk-wise in
// shared memory; every comparator moves the larger element up, so comparators
// touching an index >= n are simply skipped and any n works without padding.
constexpr int TS_THREADS = 256;
constexpr int TS_CAP = 4096;
constexpr int TS_E = TS_CAP / TS_THREADS;       // max records per thread

struct TileSortSmem {
    uint64_t s[TS_CAP];
    uint32_t whist[NW][BINS];
    uint32_t texcl[256];
    uint32_t scan[8];
};

__device__ __forceinline__ void ts_step_smem(uint64_t *s, int count, int mask, int hb)
{
    // compare-exchange (i, i ^ mask) for every i < count with bit `hb` clear
    for (int t = threadIdx.x; t < count / 2; t += TS_THREADS) {
        const int i = ((t & ~(hb - 1)) << 1) | (t & (hb - 1));
        const int p = i ^ mask;
        const uint64_t a = s[i], b = s[p];
        if (a > b) { s[i] = b; s[p] = a; }
    }
    __syncthreads();
}

__device__ __forceinline__ void ts_step_global(uint64_t *g, int n, int npad, int mask, int hb)
{
    for (int t = threadIdx.x; t < npad / 2; t += TS_THREADS) {
        const int i = ((t & ~(hb - 1)) << 1) | (t & (hb - 1));
        const int p = i ^ mask;
        if (p < n) {
            const uint64_t a = g[i], b = g[p];
            if (a > b) { g[i] = b; g[p] = a; }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void ts_bitonic_smem(uint64_t *s, int npad)
{
    for (int k = 2; k <= npad; k <<= 1) {
        ts_step_smem(s, npad, k - 1, k >> 1);
        for (int j = k >> 2; j > 0; j >>= 1) ts_step_smem(s, npad, j, j);
    }
}

__global__ void __launch_bounds__(TS_THREADS, 4)
k_tile_sort(uint64_t *__restrict__ rec, uint32_t *__restrict__ vals_out,
            uint64_t *__restrict__ keys_out, const int32_t *__restrict__ starts, int write_keys,
            const fgs_stats *__restrict__ stats)
{
    __shared__ TileSortSmem S;
    if (stats->overflow) return;
    const int tile = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int start = starts[tile], n = starts[tile + 1] - start;
    if (n <= 0) return;
    uint64_t *g = rec + start;
    uint64_t *s = S.s;
    const uint64_t tile_hi = (uint64_t)(uint32_t)tile << 32;

    if (n <= TS_CAP) {
        if (n > 1) {
            // records spread evenly over the warps: E per thread, warp-striped
            const int E = (n + TS_THREADS - 1) / TS_THREADS;
            const int wbase = w * 32 * E;
            uint64_t key[TS_E];
            uint16_t rank[TS_E];
#pragma unroll
            for (int i = 0; i < TS_E; ++i) {
                const int loc = wbase + i * 32 + lane;
                key[i] = (i < E && loc < n) ? g[loc] : ~0ull;
            }
            uint32_t *wh = S.whist[w];
            for (int pass = 0; pass < 4; ++pass) {
                const int shift = 32 + 8 * pass;
                for (int i = tid; i < NW * BINS; i += TS_THREADS) (&S.whist[0][0])[i] = 0u;
                __syncthreads();
#pragma unroll
                for (int i = 0; i < TS_E; ++i) {
                    if (i < E) {                                  // uniform
                        const bool ok = wbase + i * 32 + lane < n;
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
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) {
                    const uint32_t c = S.whist[ww][tid];
                    S.whist[ww][tid] = cnt;
                    cnt += c;
                }
                uint32_t ttotal;
                S.texcl[tid] = block_excl_scan_256(cnt, S.scan, ttotal);
                __syncthreads();
#pragma unroll
                for (int i = 0; i < TS_E; ++i) {
                    if (i < E && wbase + i * 32 + lane < n) {
                        const uint32_t d = (uint32_t)(key[i] >> shift) & 0xffu;
                        s[S.texcl[d] + wh[d] + rank[i]] = key[i];
                    }
                }
                __syncthreads();
                if (pass < 3) {
#pragma unroll
                    for (int i = 0; i < TS_E; ++i) {
                        const int loc = wbase + i * 32 + lane;
                        key[i] = (i < E && loc < n) ? s[loc] : ~0ull;
                    }
                }
            }
            // equal depths: order by index (low word).  Odd-even transposition over
            // equal-depth neighbours; almost always zero or one round.
            for (int round = 0;; ++round) {
                bool swapped = false;
                for (int t = tid; 2 * t + 1 < n; t += TS_THREADS) {
                    const uint64_t a = s[2 * t], b = s[2 * t + 1];
                    if ((a >> 32) == (b >> 32) && a > b) { s[2 * t] = b; s[2 * t + 1] = a; swapped = true; }
                }
                __syncthreads();
                for (int t = tid; 2 * t + 2 < n; t += TS_THREADS) {
                    const uint64_t a = s[2 * t + 1], b = s[2 * t + 2];
                    if ((a >> 32) == (b >> 32) && a > b) { s[2 * t + 1] = b; s[2 * t + 2] = a; swapped = true; }
                }
                if (!__syncthreads_or(swapped)) break;
                if (round == 6) {           // long runs of one depth: finish with the network
                    int npad = 2;
                    while (npad < n) npad <<= 1;
                    for (int i = n + tid; i < npad; i += TS_THREADS) s[i] = ~0ull;
                    __syncthreads();
                    ts_bitonic_smem(s, npad);
                    break;
                }
            }
        } else {
            if (tid == 0) s[0] = g[0];
            __syncthreads();
        }
        for (int i = tid; i < n; i += TS_THREADS) {
            const uint64_t r = s[i];
            vals_out[start + i] = (uint32_t)r;
            if (write_keys) keys_out[start + i] = tile_hi | (r >> 32);
        }
        return;
    }

    // large bucket: chunk-wise in shared memory, long strides through L2
    int npad = TS_CAP;
    while (npad < n) npad <<= 1;
    const int nchunks = (n + TS_CAP - 1) / TS_CAP;
    for (int c = 0; c < nchunks; ++c) {
        const int cb = c * TS_CAP;
        for (int i = tid; i < TS_CAP; i += TS_THREADS) s[i] = cb + i < n ? g[cb + i] : ~0ull;
        __syncthreads();
        ts_bitonic_smem(s, TS_CAP);
        for (int i = tid; i < TS_CAP; i += TS_THREADS)
            if (cb + i < n) g[cb + i] = s[i];
        __syncthreads();
    }
    for (int k = 2 * TS_CAP; k <= npad; k <<= 1) {
        ts_step_global(g, n, npad, k - 1, k >> 1);
        int j = k >> 2;
        for (; j >= TS_CAP; j >>= 1) ts_step_global(g, n, npad, j, j);
        for (int c = 0; c < nchunks; ++c) {
            const int cb = c * TS_CAP;
            for (int i = tid; i < TS_CAP; i += TS_THREADS) s[i] = cb + i < n ? g[cb + i] : ~0ull;
            __syncthreads();
            for (int jj = TS_CAP >> 1; jj > 0; jj >>= 1) ts_step_smem(s, TS_CAP, jj, jj);
            for (int i = tid; i < TS_CAP; i += TS_THREADS)
                if (cb + i < n) g[cb + i] = s[i];
            __syncthreads();
        }
    }
    for (int i = tid; i < n; i += TS_THREADS) {
        const uint64_t r = g[i];
        vals_out[start + i] = (uint32_t)r;
        if (write_keys) keys_out[start + i] = tile_hi | (r >> 32);
    }
}

}  // namespace

int fgs_launch_tile_sort(const FrameDev &f, int tiles, int write_keys, cudaStream_t st)
{
    if (tiles <= 0) return FGS_OK;
    k_tile_sort<<<(unsigned)tiles, TS_THREADS, 0, st>>>(f.keys[0], f.vals[0], f.keys[1], f.starts,
                                                        write_keys, f.stats);
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(SortSmem));
        if (e != cudaSuccess) { fgs_set_cuda_error(e); return FGS_E_CUDA; }
        attr_set = true;
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
