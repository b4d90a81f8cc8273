// group.cu — fae_group_batches: the backward's sort-and-segment (a9) for every
// hot batch of a packed dataset, in bulk.
//
// The hot CSR is static for the whole run (the paper pre-processes once and
// stores the FAE format), so grouping each hot batch's lookups
// by hot id is hoisted out of the training step and done for all batches at
// once, as a SEGMENTED onesweep LSD radix sort over the whole hot CSR:
//   k_gs_init     tiles of 4096 lookups (never spanning two batches): (hot id,
//                 local bag) pairs + every pass's per-batch digit histogram
//   k_gs_pass     one 8-bit digit per pass, ceil(log2(H+1)/8) passes: warp
//                 match_any ranking, per-digit decoupled look-back restricted
//                 to the tiles of the same batch, stable scatter inside the
//                 batch (the last pass writes the bag ids straight to perm)
//   k_gs_segments runs of equal hot id -> segments; global numbering by a
//                 decoupled look-back
//   k_gs_records  one 16-byte SegRec per segment (batch-local indices), per
//                 batch stably partitioned: short segments (<= kPiece
//                 lookups, one lane group each) first, long ones (one CTA
//                 each) after
// Every pass streams its tile once (HBM-bound); no CTA-serial work per batch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kern_common.cuh"

namespace fae {

constexpr int kGSW = kGSThreads / 32;

__device__ __forceinline__ int32_t find_bag_g(const int64_t* __restrict__ off, int64_t n_bags,
                                              int64_t pos) {
    int64_t lo = 0, hi = n_bags - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= pos) lo = mid;
        else hi = mid - 1;
    }
    return (int32_t)lo;
}

// per-batch digit histograms of every pass (+ the bag ids, offsets input
// only): one block per batch (grid-stride over batches), 16 hot ids per
// thread per 4096-lookup chunk, match_any aggregation into shared memory, one
// plain store per bin at the end (the block owns the batch: no atomics)
__global__ void __launch_bounds__(kGSThreads)
k_gs_init(const int32_t* __restrict__ hot_idx, const int64_t* __restrict__ hot_off,
          const BatchDesc* __restrict__ desc, int64_t n_batches, int64_t H, int passes,
          int32_t* __restrict__ vals, uint32_t* __restrict__ ghist) {
    __shared__ uint32_t sh[kMaxSortPasses][kSortBins];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t b = blockIdx.x; b < n_batches; b += gridDim.x) {
        for (int i = tid; i < kMaxSortPasses * kSortBins; i += kGSThreads) (&sh[0][0])[i] = 0;
        __syncthreads();
        const BatchDesc d = desc[b];
        for (int64_t s0 = d.lk0; s0 < d.lk1; s0 += kGSTile) {
            const int64_t s1 = s0 + kGSTile < d.lk1 ? s0 + kGSTile : d.lk1;
            uint32_t key[kGSItems];
            const int64_t wb = s0 + (int64_t)warp * 32 * kGSItems;
#pragma unroll
            for (int r = 0; r < kGSItems; r++) {
                const int64_t j = wb + r * 32 + lane;
                if (j < s1) {
                    const int32_t hv = hot_idx[j];
                    key[r] = (uint32_t)hv >= (uint64_t)H ? (uint32_t)H : (uint32_t)hv;
                    if (hot_off) vals[j] = find_bag_g(hot_off + d.bag0, d.n_bags, j);
                } else {
                    key[r] = 0xFFFFFFFFu;
                }
            }
            for (int ps = 0; ps < passes; ps++) {
#pragma unroll
                for (int r = 0; r < kGSItems; r++) {
                    const bool ok = wb + r * 32 + lane < s1;
                    const uint32_t dg = ok ? ((key[r] >> (ps * kSortBits)) & (kSortBins - 1)) : (uint32_t)kSortBins + lane;
                    const uint32_t peers = match_label<kSortBits + 1>(dg);
                    if (ok && (__ffs(peers) - 1) == lane) atomicAdd(&sh[ps][dg], (uint32_t)__popc(peers));
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < kMaxSortPasses * kSortBins; i += kGSThreads)
            ghist[b * kMaxSortPasses * kSortBins + i] = (&sh[0][0])[i];
        __syncthreads();
    }
}

// status word: bits 31..30 flag (1 aggregate, 2 inclusive), 29..0 count.
// kin == nullptr: pass 0 reads the keys from the hot CSR (ids >= H map to
// H); vin == nullptr: the bag ids are (j - lk0) / P (fixed pooling).  The
// tile is ranked (warp match_any), staged in shared memory in local sorted
// order, and written with one contiguous run per digit (coalesced).
__global__ void __launch_bounds__(kGSThreads)
k_gs_pass(const uint32_t* __restrict__ kin, const int32_t* __restrict__ hot_idx, int64_t H,
          const int32_t* __restrict__ vin, int P, uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
          const int64_t* __restrict__ tile_start, const int32_t* __restrict__ tile_batch,
          const BatchDesc* __restrict__ desc, const uint32_t* __restrict__ ghist, int pass,
          uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr, uint32_t* err) {
    __shared__ uint32_t s_w[kGSW][kSortBins];
    __shared__ uint32_t s_goff[kSortBins];
    __shared__ uint32_t s_tds[kSortBins];
    __shared__ uint32_t s_ws[kGSW];
    __shared__ uint32_t s_k[kGSTile];
    __shared__ int32_t s_v[kGSTile];
    __shared__ int64_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int shift = pass * kSortBits;
    if (tid == 0) s_tile = (int64_t)atomicAdd(tile_ctr, 1u);
    for (int i = tid; i < kGSW * kSortBins; i += kGSThreads) (&s_w[0][0])[i] = 0;
    __syncthreads();
    const int64_t t = s_tile;
    const int64_t s0 = tile_start[t], s1 = tile_start[t + 1];
    const int n_tile = (int)(s1 - s0);
    const int32_t tb = tile_batch[t];
    const int b = tb & 0x7FFFFFFF;
    const bool first = tb < 0;
    const int64_t lk0 = desc[b].lk0;
    {   // batch digit starts: exclusive scan of the batch histogram
        const uint32_t v = ghist[((int64_t)b * kMaxSortPasses + pass) * kSortBins + tid];
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_ws[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; w++) wp += s_ws[w];
        s_goff[tid] = wp + x - v;
    }
    const int wl = warp * 32 * kGSItems;   // warp's first local position
    uint32_t k[kGSItems];
    int32_t v[kGSItems];
    uint16_t rk[kGSItems];
#pragma unroll
    for (int r = 0; r < kGSItems; r++) {
        const int li = wl + r * 32 + lane;
        const int64_t i = s0 + li;
        if (li < n_tile) {
            if (kin) {
                k[r] = kin[i];
            } else {
                const int32_t hv = hot_idx[i];
                if ((uint32_t)hv >= (uint64_t)H) {
                    atomicOr(err, kErrIndex);
                    k[r] = (uint32_t)H;
                } else {
                    k[r] = (uint32_t)hv;
                }
            }
            v[r] = vin ? vin[i] : (int32_t)((i - lk0) / P);
        } else {
            k[r] = 0u;
            v[r] = 0;
        }
    }
#pragma unroll
    for (int r = 0; r < kGSItems; r++) {
        const bool ok = wl + r * 32 + lane < n_tile;
        const uint32_t dg = ok ? ((k[r] >> shift) & (kSortBins - 1)) : (uint32_t)kSortBins;
        const uint32_t peers = match_label<kSortBits + 1>(dg);
        const uint32_t lt = __popc(peers & lanemask_lt());
        uint32_t cnt = 0;
        if (ok) cnt = s_w[warp][dg];
        __syncwarp();
        if (ok && lt == 0) s_w[warp][dg] = cnt + __popc(peers);
        __syncwarp();
        rk[r] = (uint16_t)(cnt + lt);
    }
    __syncthreads();
    const int d = tid;   // kGSThreads == kSortBins
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kGSW; w++) {
        const uint32_t c = s_w[w][d];
        s_w[w][d] = tot;
        tot += c;
    }
    // publish this tile's digit count early; finish the look-back later
    uint32_t* st = status + t * kSortBins + d;
    st_relaxed_u32(st, ((first ? 2u : 1u) << 30) | tot);
    {   // tile-local digit starts (exclusive scan of tot over digits)
        uint32_t x = tot;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __syncthreads();
        if (lane == 31) s_ws[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; w++) wp += s_ws[w];
        s_tds[d] = wp + x - tot;
    }
    __syncthreads();
    // stage the tile in local sorted order
#pragma unroll
    for (int r = 0; r < kGSItems; r++) {
        if (wl + r * 32 + lane < n_tile) {
            const uint32_t dg = (k[r] >> shift) & (kSortBins - 1);
            const uint32_t lp = s_tds[dg] + s_w[warp][dg] + rk[r];
            s_k[lp] = k[r];
            s_v[lp] = v[r];
        }
    }
    // look-back for digit d within the batch's tiles
    uint32_t excl = 0;
    if (!first) {
        int64_t q = t - 1;
        while (true) {
            uint32_t sv;
            do {
                sv = ld_relaxed_u32(status + q * kSortBins + d);
            } while ((sv >> 30) == 0);
            excl += sv & 0x3FFFFFFFu;
            if ((sv >> 30) == 2) break;
            --q;
        }
        st_relaxed_u32(st, (2u << 30) | (excl + tot));
    }
    s_goff[d] += excl;
    __syncthreads();
    // coalesced write-out: consecutive local positions of one digit are
    // consecutive output positions
    for (int i = tid; i < n_tile; i += kGSThreads) {
        const uint32_t kk = s_k[i];
        const uint32_t dg = (kk >> shift) & (kSortBins - 1);
        const int64_t pos = lk0 + s_goff[dg] + (i - s_tds[dg]);
        kout[pos] = kk;
        vout[pos] = s_v[i];
    }
}

// segments over the sorted keys; global numbering (look-back)
__global__ void __launch_bounds__(kGSThreads)
k_gs_segments(const uint32_t* __restrict__ keys, const int64_t* __restrict__ tile_start,
              const int32_t* __restrict__ tile_batch, BatchDesc* __restrict__ desc, int64_t n_tiles,
              int64_t H, int64_t L_total, uint64_t* __restrict__ status, uint32_t* __restrict__ tile_ctr,
              int64_t* __restrict__ seg_start, int32_t* __restrict__ seg_row, int64_t* __restrict__ totals) {
    __shared__ uint32_t s_ws[kGSW + 1];
    __shared__ uint64_t s_ex;
    __shared__ int64_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int64_t)atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t t = s_tile;
    const int64_t s0 = tile_start[t], s1 = tile_start[t + 1];
    const int32_t tb = tile_batch[t];
    const int b = tb & 0x7FFFFFFF;
    const int64_t lk0 = desc[b].lk0;
    const int64_t j0 = s0 + (int64_t)tid * kGSItems;
    uint32_t kk[kGSItems];
    uint32_t prev = (j0 > lk0 && j0 - 1 < s1) ? keys[j0 - 1] : 0xFFFFFFFFu;
    uint32_t fl = 0, cs = 0;
#pragma unroll
    for (int r = 0; r < kGSItems; r++) {
        const int64_t j = j0 + r;
        kk[r] = 0xFFFFFFFFu;
        if (j < s1) {
            kk[r] = keys[j];
            if (kk[r] < (uint64_t)H && (j == lk0 || prev != kk[r])) {
                fl |= 1u << r;
                cs++;
            }
            prev = kk[r];
        }
    }
    uint32_t x = cs;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_ws[warp] = x;
    __syncthreads();
    uint32_t wp = 0, tot = 0;
    for (int w = 0; w < kGSW; w++) {
        if (w < warp) wp += s_ws[w];
        tot += s_ws[w];
    }
    if (tid == 0) {
        const uint64_t ex = lookback_u64(status, t, tot);
        s_ex = ex;
        if (tb < 0) desc[b].sb0 = (int64_t)ex;   // first tile of batch b
        if (t == n_tiles - 1) {
            totals[0] = (int64_t)(ex + tot);
            seg_start[ex + tot] = L_total;
        }
    }
    __syncthreads();
    int64_t si = (int64_t)s_ex + wp + x - cs;
#pragma unroll
    for (int r = 0; r < kGSItems; r++) {
        if ((fl >> r) & 1u) {
            seg_start[si] = j0 + r;
            seg_row[si] = (int32_t)kk[r];
            si++;
        }
    }
}

// ---------------------------------------------------------------------------
// Fixed-pooling fast path (replaces k_gs_init + the k_gs_pass passes +
// k_gs_segments when every (batch, table) unit holds <= kUnitMax lookups).
// Hot ids are table-ordered (tables in order, R16), so a batch's stable sort
// by hot id is the concatenation over z of each unit's stable sort: unit
// (b, z) = the B_b*P lookups of table z in batch b, positions lk0 +
// (r*Tn + z)*P + p, bag id r*Tn + z.  One CTA per unit, in unit order:
//   1. keys into shared memory; the key range (min, max) of the unit;
//   2. stable LSD radix sort of (key - min, bag) in shared memory, 8-bit
//      digits, only ceil(bits(range)/8) passes (ballot ranking per warp,
//      items warp-strided in position order);
//   3. perm[lk0 + z*n + i] = bag of the i-th smallest (coalesced);
//   4. segments (runs of equal hot id; ids >= H make none): counted, the
//      global segment number by a decoupled look-back over units, seg_start
//      (= lk0 + z*n + i) / seg_row written; unit z = 0 sets desc[b].sb0.
// Same outputs as the generic path (perm, seg_start, seg_row, sb0, totals).
// ---------------------------------------------------------------------------
// resident unit CTAs per SM (launch bounds; measured)
#ifndef FAE_UNITS8_MB
#define FAE_UNITS8_MB 5
#endif
#ifndef FAE_UNITS16_MB
#define FAE_UNITS16_MB 4   // 4096-lookup units: 3.92 / 3.24 / 3.17 ms at 2 / 3 / 4 (Terabyte-shaped, 24M records)
#endif
constexpr int kUnitThreads = 256;
constexpr int kUnitIPT = 16;
constexpr int kUnitMax = kUnitThreads * kUnitIPT;   // 4096 lookups per unit
constexpr int kMaxUnitTables = 1024;                 // unit path: tables per batch

template <int IPT, bool kP1>
__global__ void __launch_bounds__(kUnitThreads, IPT <= 8 ? FAE_UNITS8_MB : FAE_UNITS16_MB)
k_gs_units(const int32_t* __restrict__ hot_idx, int64_t H, int Tn, int P_, const BatchDesc* __restrict__ desc,
           int32_t* __restrict__ perm, int32_t* __restrict__ useg_pos, int32_t* __restrict__ useg_row,
           uint32_t* __restrict__ ucnt, uint32_t* err) {
    constexpr int NW = kUnitThreads / 32;
    const int P = kP1 ? 1 : P_;   // single-lookup bags: no divisions below
    __shared__ uint32_t s_k[kUnitThreads * IPT];
    __shared__ int32_t s_v[kUnitThreads * IPT];
    __shared__ uint32_t s_w[NW][kSortBins];
    __shared__ uint32_t s_tds[kSortBins];
    __shared__ uint32_t s_ws[NW];
    __shared__ uint32_t s_mm[2][NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t u = blockIdx.x;
    const int64_t b = u / Tn;
    const int z = (int)(u - b * Tn);
    const BatchDesc d = desc[b];
    const int nrec = d.n_bags / Tn;
    const int n = nrec * P;
    const int64_t out0 = d.lk0 + (int64_t)z * n;
    // 1. keys (invalid ids -> 0xFFFFFFFF, sorted last, no segment)
    const int wl = warp * 32 * IPT;
    uint32_t k[IPT];
    uint32_t mn = 0xFFFFFFFFu, mx = 0u;
    bool bad = false;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int i = wl + r * 32 + lane;
        k[r] = 0xFFFFFFFFu;
        if (i < n) {
            const int rr = i / P, p = i - rr * P;
            const int32_t hv = hot_idx[d.lk0 + ((int64_t)rr * Tn + z) * P + p];
            if ((uint32_t)hv >= (uint64_t)H) {
                bad = true;
            } else {
                k[r] = (uint32_t)hv;
                mn = min(mn, k[r]);
                mx = max(mx, k[r]);
            }
        }
    }
    if (bad) atomicOr(err, kErrIndex);
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        s_mm[0][warp] = mn;
        s_mm[1][warp] = mx;
    }
    __syncthreads();
    mn = 0xFFFFFFFFu;
    mx = 0u;
#pragma unroll
    for (int w = 0; w < NW; w++) {
        mn = min(mn, s_mm[0][w]);
        mx = max(mx, s_mm[1][w]);
    }
    // local keys: valid ids -> id - mn in [0, range]; invalid -> range + 1
    const uint32_t range = mx >= mn ? mx - mn : 0u;
    const uint32_t top = range + 1u;
    int bits = 0;
    while (bits < 32 && (top >> bits) != 0u) bits++;
    const int passes = (bits + kSortBits - 1) / kSortBits;
    int32_t v[IPT];
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int i = wl + r * 32 + lane;
        k[r] = k[r] == 0xFFFFFFFFu ? top : k[r] - mn;
        v[r] = i < n ? (int32_t)((i / P) * Tn + z) : 0;
    }
    // 2. stable LSD passes; items stay warp-strided in position order
    for (int ps = 0; ps < passes; ps++) {
        const int shift = ps * kSortBits;
        for (int i = tid; i < NW * kSortBins; i += kUnitThreads) (&s_w[0][0])[i] = 0;
        __syncthreads();
        uint16_t rk[IPT];
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const bool ok = wl + r * 32 + lane < n;
            const uint32_t dg = ok ? ((k[r] >> shift) & (kSortBins - 1)) : (uint32_t)kSortBins;
            const uint32_t peers = match_label<kSortBits + 1>(dg);
            const uint32_t lt = __popc(peers & lanemask_lt());
            uint32_t cnt = 0;
            if (ok) cnt = s_w[warp][dg];
            __syncwarp();
            if (ok && lt == 0) s_w[warp][dg] = cnt + __popc(peers);
            __syncwarp();
            rk[r] = (uint16_t)(cnt + lt);
        }
        __syncthreads();
        {   // per digit: warp prefix (in place) and digit total; then the
            // exclusive scan of the totals over digits (kUnitThreads == bins)
            const int dg = tid;
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < NW; w++) {
                const uint32_t c = s_w[w][dg];
                s_w[w][dg] = tot;
                tot += c;
            }
            uint32_t x = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_ws[warp] = x;
            __syncthreads();
            uint32_t wp = 0;
            for (int w = 0; w < warp; w++) wp += s_ws[w];
            s_tds[dg] = wp + x - tot;
        }
        __syncthreads();
        // scatter (every thread finished reading the buffer before the syncs above)
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            if (wl + r * 32 + lane < n) {
                const uint32_t dg = (k[r] >> shift) & (kSortBins - 1);
                const uint32_t pos = s_tds[dg] + s_w[warp][dg] + rk[r];
                s_k[pos] = k[r];
                s_v[pos] = v[r];
            }
        }
        __syncthreads();
        if (ps + 1 < passes) {   // reload in position order for the next pass
#pragma unroll
            for (int r = 0; r < IPT; r++) {
                const int i = wl + r * 32 + lane;
                if (i < n) {
                    k[r] = s_k[i];
                    v[r] = s_v[i];
                }
            }
        }
    }
    if (passes == 0) {   // all keys equal: already in order
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const int i = wl + r * 32 + lane;
            if (i < n) {
                s_k[i] = k[r];
                s_v[i] = v[r];
            }
        }
        __syncthreads();
    }
    // 3. perm (coalesced)
    for (int i = tid; i < n; i += kUnitThreads) perm[out0 + i] = s_v[i];
    // 4. segments: thread-contiguous chunks of IPT positions
    const int j0 = tid * IPT;
    uint32_t fl = 0, cs = 0;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int i = j0 + r;
        if (i < n) {
            const uint32_t kk = s_k[i];
            if (kk != top && (i == 0 || s_k[i - 1] != kk)) {
                fl |= 1u << r;
                cs++;
            }
        }
    }
    uint32_t x = cs;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) s_ws[warp] = x;
    __syncthreads();
    uint32_t wp = 0, tot = 0;
    for (int w = 0; w < NW; w++) {
        if (w < warp) wp += s_ws[w];
        tot += s_ws[w];
    }
    // the unit's segments at its own lookup range (compacted by k_gs_ucompact)
    if (tid == 0) ucnt[u] = tot;
    (void)tot;
    int64_t si = out0 + wp + x - cs;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        if ((fl >> r) & 1u) {
            useg_pos[si] = (int32_t)(z * n + j0 + r);          // position in the batch
            useg_row[si] = (int32_t)(s_k[j0 + r] + mn);
            si++;
        }
    }
}

// Batch segment bases (one CTA): sb0/sb1 of every batch = prefix over
// batches of the sum of its Tn unit counts; totals[0] = S_total and the
// seg_start sentinel.  Units of batch b are b*Tn .. b*Tn + Tn - 1.
__global__ void __launch_bounds__(1024)
k_gs_ubase(BatchDesc* __restrict__ desc, int64_t nb, int Tn, const uint32_t* __restrict__ ucnt,
           int64_t* __restrict__ totals, int64_t* __restrict__ seg_start, int64_t L_total) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        const int64_t b = b0 + tid;
        int64_t c = 0;
        if (b < nb)
            for (int z = 0; z < Tn; z++) c += ucnt[b * Tn + z];
        int64_t x = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        int64_t wp = 0, tot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wp += s_w[w];
            tot += s_w[w];
        }
        const int64_t ex = s_carry + wp + x - c;
        if (b < nb) {
            desc[b].sb0 = ex;
            desc[b].sb1 = ex + c;
        }
        __syncthreads();
        if (tid == 0) s_carry += tot;
        __syncthreads();
    }
    if (tid == 0) {
        totals[0] = s_carry;
        seg_start[s_carry] = L_total;
    }
}

// Compaction: one CTA per batch (grid-stride); unit offsets by a scan of its
// Tn counts, then seg_start (global lookup position) / seg_row in unit order.
__global__ void __launch_bounds__(256)
k_gs_ucompact(const BatchDesc* __restrict__ desc, int64_t nb, int Tn, int P, const uint32_t* __restrict__ ucnt,
              const int32_t* __restrict__ useg_pos, const int32_t* __restrict__ useg_row,
              int64_t* __restrict__ seg_start, int32_t* __restrict__ seg_row) {
    __shared__ uint32_t s_off[kMaxUnitTables + 1];
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const BatchDesc d = desc[b];
        const int n = (d.n_bags / Tn) * P;
        __syncthreads();
        if (Tn <= 32) {   // the unit offsets by one warp scan (parallel count loads)
            if (threadIdx.x < 32) {
                const int z = threadIdx.x;
                const uint32_t v = z < Tn ? ucnt[b * Tn + z] : 0u;
                uint32_t x = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (z >= o) x += y;
                }
                if (z < Tn) s_off[z] = x - v;
                if (z == Tn - 1) s_off[Tn] = x;
            }
        } else if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int z = 0; z < Tn; z++) {
                s_off[z] = acc;
                acc += ucnt[b * Tn + z];
            }
            s_off[Tn] = acc;
        }
        __syncthreads();
        // all the batch's segments in one flat loop (unit of segment e: the
        // last z with s_off[z] <= e, a shared-memory binary search; empty
        // units share their offset with the next one and are skipped)
        const uint32_t total = s_off[Tn];
        for (uint32_t e = threadIdx.x; e < total; e += blockDim.x) {
            int lo = 0, hi = Tn - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_off[mid] <= e) lo = mid;
                else hi = mid - 1;
            }
            const int64_t src = d.lk0 + (int64_t)lo * n + (e - s_off[lo]);
            seg_start[d.sb0 + e] = d.lk0 + useg_pos[src];
            seg_row[d.sb0 + e] = useg_row[src];
        }
    }
}

// one block per batch b (grid-stride): link each segment t of batch b to
// the segment of batch b-1 with the same row (binary search in b-1's
// ascending rows): nxt[σ] = t; segments without one go to batch b's free
// list (stable order) and desc[b].n_free.
__global__ void __launch_bounds__(256)
k_gs_links(BatchDesc* __restrict__ desc, int64_t n_batches, const int64_t* __restrict__ seg_start,
           const int32_t* __restrict__ seg_row, int32_t* __restrict__ nxt, FreeRec* __restrict__ freer,
           int smem_rows) {
    extern __shared__ int32_t s_prev[];   // batch b-1's rows when they fit (smem_rows)
    __shared__ uint32_t s_w[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t b = blockIdx.x; b < n_batches; b += gridDim.x) {
        const BatchDesc d = desc[b];
        const int64_t S = d.sb1 - d.sb0;
        int64_t ps0 = 0, ps1 = 0;
        if (b > 0) {
            ps0 = desc[b - 1].sb0;
            ps1 = desc[b - 1].sb1;
        }
        uint32_t run = 0;
        // the previous batch's ascending rows in shared memory: the searches
        // then cost shared-memory latency instead of dependent L2 loads
        const bool staged = ps1 - ps0 <= (int64_t)smem_rows;
        __syncthreads();
        if (staged)
            for (int64_t i = tid; i < ps1 - ps0; i += 256) s_prev[i] = seg_row[ps0 + i];
        __syncthreads();
        // IPT consecutive segments per thread (blocked): one binary search for
        // the first, then a forward walk (both lists ascend); free segments
        // compacted in segment order by a block scan of the per-thread counts
        constexpr int IPT = 4;
        const int64_t np = ps1 - ps0;
        auto prow = [&](int64_t i) -> int32_t { return staged ? s_prev[i] : seg_row[ps0 + i]; };
        for (int64_t c0 = 0; c0 < S; c0 += 256 * IPT) {
            const int64_t q0 = c0 + (int64_t)tid * IPT;
            bool fr[IPT];
            int32_t row[IPT];
            uint32_t nf = 0;
            int64_t lo = 0;
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const int64_t q = q0 + i;
                fr[i] = false;
                row[i] = 0;
                if (q >= S) continue;
                row[i] = seg_row[d.sb0 + q];
                if (i == 0) {   // first position with prev row >= row
                    int64_t hi = np;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (prow(mid) < row[i]) lo = mid + 1;
                        else hi = mid;
                    }
                } else {   // a short walk, then a binary search over the rest
                    int steps = 0;
                    while (lo < np && steps < 8 && prow(lo) < row[i]) {
                        lo++;
                        steps++;
                    }
                    if (steps == 8 && lo < np && prow(lo) < row[i]) {
                        int64_t hi = np;
                        while (lo < hi) {
                            const int64_t mid = (lo + hi) >> 1;
                            if (prow(mid) < row[i]) lo = mid + 1;
                            else hi = mid;
                        }
                    }
                }
                if (lo < np && prow(lo) == row[i]) nxt[ps0 + lo] = (int32_t)q;
                else fr[i] = true;
                nf += fr[i];
            }
            uint32_t x = nf;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            __syncthreads();
            if (lane == 31) s_w[warp] = x;
            __syncthreads();
            uint32_t pre = 0, tot = 0;
            for (int w = 0; w < 8; w++) {
                if (w < warp) pre += s_w[w];
                tot += s_w[w];
            }
            uint32_t at = run + pre + x - nf;
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                if (!fr[i]) continue;
                const int64_t q = q0 + i;
                const int64_t s = d.sb0 + q;
                const int64_t st = seg_start[s];
                const int64_t e = q + 1 < S ? seg_start[s + 1] : d.lk1;
                FreeRec f;
                f.pos = (int32_t)(st - d.lk0);
                f.len = (int32_t)(e - st);
                f.row = row[i];
                f.pad = 0;
                freer[d.sb0 + at++] = f;
            }
            run += tot;
        }
        if (tid == 0) desc[b].n_free = (int32_t)run;
        __syncthreads();
    }
}

// one block per batch (grid-stride over batches): batch-local SegRecs,
// stably partitioned by length class (<= kTinySeg, <= kPiece, <= kMedium,
// longer), each class in ascending hot id; desc[b].n_tiny, n_short (tiny +
// small), n_med; long segments get their chunk range (c0, nc)
__global__ void __launch_bounds__(256)
k_gs_records(BatchDesc* __restrict__ desc, int64_t n_batches, const int64_t* __restrict__ seg_start,
             const int32_t* __restrict__ seg_row, const int32_t* __restrict__ nxt,
             SegRec* __restrict__ rec, int chunk, int32_t* __restrict__ lmap) {
    constexpr int NC = 4;
    __shared__ uint32_t s_w[NC][8];
    __shared__ uint32_t s_n[NC];
    __shared__ uint64_t s_w64[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t b = blockIdx.x; b < n_batches; b += gridDim.x) {
        const BatchDesc d = desc[b];
        const int64_t S = d.sb1 - d.sb0;
        const bool has_next = b + 1 < n_batches;
        BatchDesc dn{};
        if (has_next) dn = desc[b + 1];
        auto cls = [&](int64_t q, SegRec& r) -> int {
            const int64_t s = d.sb0 + q;
            const int64_t st = seg_start[s];
            const int64_t e = q + 1 < S ? seg_start[s + 1] : d.lk1;
            r.pos = (int32_t)(st - d.lk0);
            r.len = (int32_t)(e - st);
            r.row = seg_row[s];
            r.seg = (int32_t)q;
            r.npos = -1;
            r.nlen = 0;
            r.c0 = 0;
            r.nc = 1;
            const int32_t t = nxt ? nxt[s] : -1;
            if (t >= 0 && has_next) {
                const int64_t sn = dn.sb0 + t;
                const int64_t en = sn + 1 < dn.sb1 ? seg_start[sn + 1] : dn.lk1;
                r.npos = (int32_t)(seg_start[sn] - dn.lk0);
                r.nlen = (int32_t)(en - seg_start[sn]);
            }
            return r.len <= kTinySeg ? 0 : (r.len <= kPiece ? 1 : (r.len <= kMedium ? 2 : 3));
        };
        // pass 1: class sizes (the class depends on the length only); each
        // thread takes IPT consecutive segments per round
        constexpr int IPT = 4;
        constexpr int CHK = 256 * IPT;
        uint32_t nn[NC] = {0u, 0u, 0u, 0u};
        for (int64_t q0 = (int64_t)tid * IPT; q0 < S; q0 += CHK) {
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const int64_t q = q0 + i;
                if (q >= S) break;
                const int64_t s = d.sb0 + q;
                const int64_t len = (q + 1 < S ? seg_start[s + 1] : d.lk1) - seg_start[s];
                nn[0] += len <= kTinySeg;
                nn[1] += len > kTinySeg && len <= kPiece;
                nn[2] += len > kPiece && len <= kMedium;
                nn[3] += len > kMedium;
            }
        }
#pragma unroll
        for (int c = 0; c < NC; c++) {
            for (int o = 16; o; o >>= 1) nn[c] += __shfl_xor_sync(0xffffffffu, nn[c], o);
            if (lane == 0) s_w[c][warp] = nn[c];
        }
        __syncthreads();
        if (tid < NC) {
            uint32_t t = 0;
            for (int w = 0; w < 8; w++) t += s_w[tid][w];
            s_n[tid] = t;
        }
        __syncthreads();
        if (tid == 0) {
            desc[b].n_tiny = (int32_t)s_n[0];
            desc[b].n_short = (int32_t)(s_n[0] + s_n[1]);
            desc[b].n_med = (int32_t)s_n[2];
        }
        const uint32_t base[NC] = {0u, s_n[0], s_n[0] + s_n[1], s_n[0] + s_n[1] + s_n[2]};
        uint32_t run[NC] = {0u, 0u, 0u, 0u};
        __syncthreads();
        // pass 2: stable partition, rounds of CHK segments, IPT consecutive
        // segments per thread (blocked): the per-thread class counts (four
        // 16-bit fields, <= CHK each) are scanned across the block in thread
        // order, so the order inside a class is the segment order
        for (int64_t c0 = 0; c0 < S; c0 += CHK) {
            SegRec r[IPT];
            int k[IPT];
            uint64_t my = 0;
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const int64_t q = c0 + (int64_t)tid * IPT + i;
                k[i] = q < S ? cls(q, r[i]) : -1;
                if (k[i] >= 0) my += 1ull << (16 * k[i]);
            }
            uint64_t x = my;
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_w64[warp] = x;
            __syncthreads();
            uint64_t wp = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < 8; w++) {
                const uint64_t v = s_w64[w];
                if (w < warp) wp += v;
                tot += v;
            }
            const uint64_t ex = wp + x - my;
            uint32_t seen[NC] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                if (k[i] < 0) continue;
                const int c = k[i];
                const uint32_t pos = base[c] + run[c] + (uint32_t)((ex >> (16 * c)) & 0xFFFFu) + seen[c]++;
                rec[d.sb0 + pos] = r[i];
            }
#pragma unroll
            for (int c = 0; c < NC; c++) run[c] += (uint32_t)((tot >> (16 * c)) & 0xFFFFu);
            __syncthreads();   // s_w64 is rewritten by the next round
        }
        __syncthreads();
        {   // chunks of the long segments, in record order: block scan of nc
            int32_t* lm = lmap + lmap_base(d, b);
            uint32_t carry = 0;
            for (int64_t q0 = (int64_t)base[3]; q0 < S; q0 += 256) {
                const int64_t q = q0 + tid;
                uint32_t nc = 0;
                if (q < S) nc = (uint32_t)((rec[d.sb0 + q].len + chunk - 1) / chunk);
                uint32_t x = nc;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                __syncthreads();
                if (lane == 31) s_w[0][warp] = x;
                __syncthreads();
                uint32_t wp = 0, tot = 0;
                for (int w = 0; w < 8; w++) {
                    if (w < warp) wp += s_w[0][w];
                    tot += s_w[0][w];
                }
                if (q < S) {
                    const uint32_t c0 = carry + wp + x - nc;
                    SegRec& lr = rec[d.sb0 + q];
                    lr.c0 = (int32_t)c0;
                    lr.nc = (int32_t)nc;
                    for (uint32_t j = 0; j < nc; j++) lm[c0 + j] = (int32_t)(q - (int64_t)base[3]);
                }
                carry += tot;
            }
            if (tid == 0) desc[b].n_lchunk = (int32_t)carry;
        }
        __syncthreads();
    }
}

template <typename T>
static fae_status ensure(Ctx* c, T** p, int64_t* cap, int64_t need) {
    if (*p && *cap >= need) return FAE_OK;
    cudaFree(*p);
    *p = nullptr;
    const int64_t n = need + need / 8 + 256;
    FAE_CUDA(c, cudaMalloc(p, sizeof(T) * n));
    *cap = n;
    return FAE_OK;
}

void drop_graphs(Group& g);

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_group_info(const fae_ctx* h, int64_t* info) {
    if (!h || !info) return FAE_ERR_INVALID_ARG;
    const Group& g = h->c.grp;
    if (!g.valid) return FAE_ERR_NOT_INIT;
    info[0] = g.n_batches;
    info[1] = g.L_total;
    info[2] = g.n_long_total;
    info[3] = g.S_total;
    info[4] = g.max_long;
    info[5] = g.max_bags;
    int64_t nf = 0;
    for (const BatchDesc& d : g.hdesc) nf += d.n_free;
    info[6] = nf;
    info[7] = (g.P == 1 && !g.hot_off && h->c.world == 1) ? (h->c.persist ? 2 : (fused_step(&h->c) ? 1 : 0)) : 0;
    return FAE_OK;
}

extern "C" fae_status fae_group_batches(fae_ctx* h, const fae_tables* tabs, const fae_packed* pk,
                                        int32_t fixed_pool, int32_t batch, int64_t H) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_schema(c, tabs, "fae_group_batches");
    if (st != FAE_OK) return st;
    if (!pk || batch < 1 || fixed_pool < 0 || H < 0 || H >= (1ll << 31) - 1)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_group_batches: bad arguments");
    const int Tn = tabs->n_tables;
    const bool offs = fixed_pool == 0;
    if (pk->n_hot < 0 || pk->n_hot_lookups < 0 || (pk->n_hot_lookups > 0 && !pk->hot_idx) || (offs && !pk->hot_off))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_group_batches: bad packed dataset");
    if (pk->n_hot_lookups >= (1ll << 31) - 1)
        return set_err(c, FAE_ERR_CAPACITY, "fae_group_batches: >= 2^31 hot lookups");
    Group& g = c->grp;
    drop_graphs(g);
    g.valid = false;
    const bool verbose = getenv("FAE_VERBOSE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto stage = [&](const char* name) {
        if (!verbose) return;
        cudaStreamSynchronize(c->stream);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[fae_group_batches] %-10s %9.3f ms\n", name,
                std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const int64_t nb = cdiv(pk->n_hot, batch);
    g.n_batches = nb;
    g.Tn = Tn;
    g.P = fixed_pool;
    g.dim = tabs->dim;
    g.B = batch;
    g.H = H;
    g.hot_idx = pk->hot_idx;
    g.hot_off = offs ? pk->hot_off : nullptr;
    const int64_t L = pk->n_hot_lookups;
    g.L_total = L;
    // batch descriptors + tiles (host)
    g.hdesc.assign(nb, BatchDesc{});
    std::vector<int64_t> starts(nb + 1, 0);
    if (offs) {
        if (nb > 0) {
            FAE_CUDA(c, cudaMemcpy2DAsync(starts.data(), sizeof(int64_t), pk->hot_off,
                                          sizeof(int64_t) * batch * (int64_t)Tn, sizeof(int64_t), nb,
                                          cudaMemcpyDeviceToHost, c->stream));
            FAE_CUDA(c, cudaMemcpyAsync(&starts[nb], pk->hot_off + pk->n_hot * Tn, sizeof(int64_t),
                                        cudaMemcpyDeviceToHost, c->stream));
            FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        }
    } else {
        for (int64_t i = 0; i <= nb; i++)
            starts[i] = std::min<int64_t>(i * batch, pk->n_hot) * Tn * (int64_t)fixed_pool;
    }
    const int64_t n_units = nb * (int64_t)Tn;
    const bool unit_path = !c->gs_generic && !offs && fixed_pool > 0 && (int64_t)batch * fixed_pool <= kUnitMax &&
                           Tn <= kMaxUnitTables && n_units < (1ll << 31);
    std::vector<int64_t> tstart;   // radix-pass tiles (generic path only)
    std::vector<int32_t> tbatch;
    if (!unit_path) tstart.reserve(L / kGSTile + nb + 1);
    int64_t max_bags = 0, max_lk = 0;
    for (int64_t i = 0; i < nb; i++) {
        BatchDesc& d = g.hdesc[i];
        const int64_t r0 = i * batch, r1 = std::min<int64_t>((i + 1) * batch, pk->n_hot);
        d.lk0 = starts[i];
        d.lk1 = starts[i + 1];
        d.bag0 = r0 * Tn;
        d.n_bags = (int32_t)((r1 - r0) * Tn);
        max_bags = std::max<int64_t>(max_bags, d.n_bags);
        max_lk = std::max<int64_t>(max_lk, d.lk1 - d.lk0);
        if (!unit_path)
            for (int64_t s = d.lk0; s < d.lk1; s += kGSTile) {
                tstart.push_back(s);
                tbatch.push_back((int32_t)i | (s == d.lk0 ? (int32_t)0x80000000 : 0));
            }
    }
    if (max_lk >= (1ll << 30)) return set_err(c, FAE_ERR_CAPACITY, "fae_group_batches: batch too large");
    const int64_t nt = (int64_t)tbatch.size();
    stage("host");
    tstart.push_back(L);
    g.max_bags = max_bags;
    g.max_lookups = max_lk;
    int bits = 1;
    while (bits < 32 && ((uint64_t)1 << bits) <= (uint64_t)H) bits++;
    const int passes = (bits + kSortBits - 1) / kSortBits;
    // buffers
    int64_t k0cap = g.cap_L, k1cap = g.cap_L, vcap = g.cap_L, pcap = g.cap_L;
    if ((st = ensure(c, &g.keys[0], &k0cap, std::max<int64_t>(L, 1))) != FAE_OK) return st;
    if ((st = ensure(c, &g.keys[1], &k1cap, std::max<int64_t>(L, 1))) != FAE_OK) return st;
    if ((st = ensure(c, &g.vals, &vcap, std::max<int64_t>(L, 1))) != FAE_OK) return st;
    if ((st = ensure(c, &g.perm, &pcap, std::max<int64_t>(L, 1))) != FAE_OK) return st;
    g.cap_L = std::min(std::min(k0cap, k1cap), std::min(vcap, pcap));
    // segment arrays written before the segment count is known: capacity L
    // (records, free lists and links are sized by the count, below)
    int64_t c3 = g.cap_S, c4 = g.cap_S;
    if ((st = ensure(c, &g.seg_start, &c3, L + 2)) != FAE_OK) return st;
    if ((st = ensure(c, &g.seg_row, &c4, L + 2)) != FAE_OK) return st;
    g.cap_S = std::min(c3, c4);
    if ((st = ensure(c, &g.lmap, &g.cap_lmap, L / 64 + nb + 2)) != FAE_OK) return st;
    if ((st = ensure(c, &g.desc, &g.cap_B, std::max<int64_t>(nb, 1))) != FAE_OK) return st;
    int64_t t1 = g.cap_T, t2 = g.cap_T, t3 = g.cap_T * kSortBins, t4 = g.cap_T;
    if ((st = ensure(c, &g.tile_start, &t1, nt + 2)) != FAE_OK) return st;
    if ((st = ensure(c, &g.tile_batch, &t2, nt + 2)) != FAE_OK) return st;
    if ((st = ensure(c, &g.sstatus, &t3, (nt + 2) * kSortBins)) != FAE_OK) return st;
    if ((st = ensure(c, &g.pstatus, &t4, nt + 2)) != FAE_OK) return st;
    g.cap_T = std::min(std::min(t1, t2), std::min(t3 / kSortBins, t4));
    if ((st = ensure(c, &g.ghist, &g.cap_Hh, std::max<int64_t>(nb, 1) * kMaxSortPasses * kSortBins)) != FAE_OK)
        return st;
    if (!g.cursor) {
        FAE_CUDA(c, cudaMalloc(&g.cursor, sizeof(int64_t) * 8));
        g.run = g.cursor + 2;
        FAE_CUDA(c, cudaMalloc(&g.done_ctr, sizeof(uint32_t) * 16));
        FAE_CUDA(c, cudaMemset(g.done_ctr, 0, sizeof(uint32_t) * 16));
        FAE_CUDA(c, cudaMalloc(&g.pbar, sizeof(uint32_t) * (2 + 32 * kMaxPersistCtas)));
    }
    stage("alloc");
    g.S_total = 0;
    g.max_short = g.max_med = g.max_long = 0;
    g.max_free = 0;
    g.max_lchunk = 0;
    g.max_segs = 1;
    g.n_long_total = 0;
    if (nb > 0) {
        uint32_t* ctr = g.done_ctr + 8;   // tile counters (kept apart from the runner's)
        int64_t* totals = (int64_t*)scratch(c, 64);
        if (!totals) return set_err(c, FAE_ERR_CUDA, "fae_group_batches: scratch allocation failed");
        FAE_CUDA(c, cudaMemcpyAsync(g.desc, g.hdesc.data(), sizeof(BatchDesc) * nb, cudaMemcpyHostToDevice, c->stream));
        if (!unit_path) {
            FAE_CUDA(c, cudaMemcpyAsync(g.tile_start, tstart.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, c->stream));
            FAE_CUDA(c, cudaMemcpyAsync(g.tile_batch, tbatch.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, c->stream));
        }

        FAE_CUDA(c, cudaMemsetAsync(totals, 0, 64, c->stream));
        const int64_t gi = std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)sm_count(c) * 8));
        const int64_t gb = std::max<int64_t>(1, std::min<int64_t>(nb, (int64_t)sm_count(c) * 8));
        (void)gi;
        if (unit_path) {
            // fixed pooling, every (batch, table) unit <= kUnitMax lookups:
            // one in-shared-memory sort per unit (k_gs_units)
            const bool small_unit = (int64_t)batch * fixed_pool <= kUnitThreads * 8;
            auto ku = fixed_pool == 1 ? (small_unit ? k_gs_units<8, true> : k_gs_units<kUnitIPT, true>)
                                      : (small_unit ? k_gs_units<8, false> : k_gs_units<kUnitIPT, false>);
            ku<<<(unsigned)n_units, kUnitThreads, 0, c->stream>>>(g.hot_idx, H, Tn, fixed_pool, g.desc, g.perm,
                                                                  (int32_t*)g.keys[0], (int32_t*)g.keys[1],
                                                                  (uint32_t*)g.vals, c->d_err);
            FAE_LAUNCHED(c);
            k_gs_ubase<<<1, 1024, 0, c->stream>>>(g.desc, nb, Tn, (const uint32_t*)g.vals, totals, g.seg_start, L);
            FAE_LAUNCHED(c);
            const int64_t gc = std::max<int64_t>(1, std::min<int64_t>(nb, (int64_t)sm_count(c) * 8));
            k_gs_ucompact<<<(unsigned)gc, 256, 0, c->stream>>>(g.desc, nb, Tn, fixed_pool, (const uint32_t*)g.vals,
                                                               (const int32_t*)g.keys[0], (const int32_t*)g.keys[1],
                                                               g.seg_start, g.seg_row);
            FAE_LAUNCHED(c);
        } else {
            k_gs_init<<<(unsigned)gb, kGSThreads, 0, c->stream>>>(g.hot_idx, g.hot_off, g.desc, nb, H, passes, g.vals,
                                                                 g.ghist);
            FAE_LAUNCHED(c);
            stage("init");
            // passes: pass 0 reads the hot CSR (and, for fixed pooling, derives the
            // bag ids); the values ping-pong so that the last pass lands in perm
            uint32_t* kbuf[2] = {g.keys[0], g.keys[1]};
            int32_t* vbuf[2] = {g.vals, g.perm};
            int vo = (passes % 2 == 1) ? 1 : 0;          // value buffer written by pass 0
            const uint32_t* kin = nullptr;
            const int32_t* vin = offs ? g.vals : nullptr;
            if (offs && vo == 0) {                       // keep vals as pass 0's input
                FAE_CUDA(c, cudaMemcpyAsync(g.perm, g.vals, sizeof(int32_t) * L, cudaMemcpyDeviceToDevice, c->stream));
                vin = g.perm;
            }
            int ko = 0;
            for (int ps = 0; ps < passes; ps++) {
                FAE_CUDA(c, cudaMemsetAsync(g.sstatus, 0, sizeof(uint32_t) * nt * kSortBins, c->stream));
                FAE_CUDA(c, cudaMemsetAsync(ctr, 0, sizeof(uint32_t), c->stream));
                k_gs_pass<<<(unsigned)nt, kGSThreads, 0, c->stream>>>(kin, g.hot_idx, H, vin, fixed_pool, kbuf[ko],
                                                                      vbuf[vo], g.tile_start, g.tile_batch, g.desc,
                                                                      g.ghist, ps, g.sstatus, ctr, c->d_err);
                FAE_LAUNCHED(c);
                kin = kbuf[ko];
                vin = vbuf[vo];
                ko ^= 1;
                vo ^= 1;
            }
            // sorted keys in kin, bag ids in perm
            stage("passes");
            // sorted keys in kin, bag ids in perm
            FAE_CUDA(c, cudaMemsetAsync(g.pstatus, 0, sizeof(uint64_t) * nt, c->stream));
            FAE_CUDA(c, cudaMemsetAsync(ctr + 1, 0, sizeof(uint32_t), c->stream));
            k_gs_segments<<<(unsigned)nt, kGSThreads, 0, c->stream>>>(kin ? kin : (const uint32_t*)g.hot_idx, g.tile_start, g.tile_batch, g.desc, nt, H, L,
                                                                     g.pstatus, ctr + 1, g.seg_start, g.seg_row, totals);
            FAE_LAUNCHED(c);
        }
        stage("segments");
        int64_t tot = 0;
        FAE_CUDA(c, cudaMemcpyAsync(&tot, totals, sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaMemcpyAsync(g.hdesc.data(), g.desc, sizeof(BatchDesc) * nb, cudaMemcpyDeviceToHost, c->stream));
        st = read_latched(c);
        if (st != FAE_OK) return st;
        g.S_total = tot;
        // batches without lookups have no tile: take the next batch's base
        int64_t ns = g.S_total;
        for (int64_t i = nb - 1; i >= 0; i--) {
            BatchDesc& d = g.hdesc[i];
            if (d.lk1 == d.lk0) d.sb0 = ns;
            d.sb1 = ns;
            ns = d.sb0;
        }
        FAE_CUDA(c, cudaMemcpyAsync(g.desc, g.hdesc.data(), sizeof(BatchDesc) * nb, cudaMemcpyHostToDevice, c->stream));
        const int64_t gr = std::max<int64_t>(1, std::min<int64_t>(nb, (int64_t)sm_count(c) * 8));
        // the links to the next batch (SegRec npos/nlen) and the free lists are
        // read only by the fused one-kernel step (and the persistent kernel);
        // the two-kernel step (D > 16, multi-hot, world > 1) never needs them
        const bool links = fused_step(c) || (g.P == 1 && !g.hot_off && c->world == 1 && c->persist);
        if ((st = ensure(c, &g.rec, &g.cap_rec, g.S_total + 2)) != FAE_OK) return st;
        if (links) {
            if ((st = ensure(c, &g.freer, &g.cap_free, g.S_total + 2)) != FAE_OK) return st;
            if ((st = ensure(c, &g.nxt, &g.cap_nxt, g.S_total + 2)) != FAE_OK) return st;
        }
        if (links) {
            FAE_CUDA(c, cudaMemsetAsync(g.nxt, 0xFF, sizeof(int32_t) * std::max<int64_t>(g.S_total, 1), c->stream));
            int64_t ms = 0;
            for (const BatchDesc& d : g.hdesc) ms = std::max<int64_t>(ms, d.sb1 - d.sb0);
            const int smem_rows = (int)std::min<int64_t>(ms, 40 * 1024);   // <= 160 KB
            const size_t lsm = sizeof(int32_t) * std::max(smem_rows, 1);
            if (lsm > 48 * 1024)
                FAE_CUDA(c, cudaFuncSetAttribute(k_gs_links, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
            k_gs_links<<<(unsigned)gr, 256, lsm, c->stream>>>(g.desc, nb, g.seg_start, g.seg_row, g.nxt, g.freer,
                                                               smem_rows);
            FAE_LAUNCHED(c);
        }
        g.chunk = chunk_for_dim(tabs->dim);
        k_gs_records<<<(unsigned)gr, 256, 0, c->stream>>>(g.desc, nb, g.seg_start, g.seg_row, links ? g.nxt : nullptr,
                                                          g.rec, g.chunk, g.lmap);
        FAE_LAUNCHED(c);
        FAE_CUDA(c, cudaMemcpyAsync(g.hdesc.data(), g.desc, sizeof(BatchDesc) * nb, cudaMemcpyDeviceToHost, c->stream));
        st = read_latched(c);
        if (st != FAE_OK) return st;
        stage("records");
        for (const BatchDesc& d : g.hdesc) {
            const int64_t S = d.sb1 - d.sb0;
            const int64_t nl = S - d.n_short - d.n_med;
            g.max_short = std::max<int64_t>(g.max_short, d.n_short);
            g.max_med = std::max<int64_t>(g.max_med, d.n_med);
            g.max_long = std::max<int64_t>(g.max_long, nl);
            g.max_segs = std::max<int64_t>(g.max_segs, S);
            g.max_free = std::max<int64_t>(g.max_free, d.n_free);
            g.max_lchunk = std::max<int64_t>(g.max_lchunk, d.n_lchunk);
            g.n_long_total += S - d.n_short;
        }
        if (getenv("FAE_VERBOSE") && nb > 0) {
            double a[7] = {0, 0, 0, 0, 0, 0, 0};
            for (const BatchDesc& d : g.hdesc) {
                a[0] += d.n_tiny;
                a[1] += d.n_short - d.n_tiny;
                a[2] += d.n_med;
                a[3] += (d.sb1 - d.sb0) - d.n_short - d.n_med;
                a[4] += d.n_lchunk;
                a[5] += d.n_free;
                a[6] += (double)(d.lk1 - d.lk0);
            }
            fprintf(stderr, "[fae_group_batches] per batch: tiny %.0f short %.0f medium %.0f long %.0f (chunks %.0f) "
                            "free %.0f lookups %.0f\n", a[0] / nb, a[1] / nb, a[2] / nb, a[3] / nb, a[4] / nb,
                    a[5] / nb, a[6] / nb);
        }
    }
    if (g.max_segs > c->ws.cap_L) return set_err(c, FAE_ERR_CAPACITY, "fae_group_batches: batch segments exceed ctx capacity");
    {   // grow-only (cudaFree would synchronise the device on every call)
        const int64_t lc = std::max<int64_t>(g.max_lchunk, 1), ll = std::max<int64_t>(g.max_long, 1);
        const int64_t need_p = kUnroll * lc * 8 * c->cfg.max_dim, need_c = kUnroll * ll;
        if (g.cap_lpart < need_p) {
            cudaFree(g.lpart);
            g.lpart = nullptr;
            g.cap_lpart = need_p + need_p / 4;
            FAE_CUDA(c, cudaMalloc(&g.lpart, sizeof(float) * g.cap_lpart));
        }
        if (g.cap_lcnt < need_c) {
            cudaFree(g.lcnt);
            g.lcnt = nullptr;
            g.cap_lcnt = need_c + need_c / 4;
            FAE_CUDA(c, cudaMalloc(&g.lcnt, sizeof(uint32_t) * g.cap_lcnt));
            FAE_CUDA(c, cudaMemsetAsync(g.lcnt, 0, sizeof(uint32_t) * g.cap_lcnt, c->stream));
        }
    }
    st = read_latched(c);
    if (st != FAE_OK) return st;
    g.valid = true;
    return FAE_OK;
}

// Free the grouping's build-only scratch (sort keys / values, segment
// starts, links, tile state), keeping what the training loop reads (perm,
// records, free lists, chunk map, segment rows, descriptors).  The next
// fae_group_batches reallocates on demand.
extern "C" fae_status fae_release_scratch(fae_ctx* h) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    Group& g = c->grp;
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    void** ptrs[] = {(void**)&g.keys[0], (void**)&g.keys[1], (void**)&g.vals, (void**)&g.seg_start,
                     (void**)&g.nxt, (void**)&g.tile_start, (void**)&g.tile_batch, (void**)&g.sstatus,
                     (void**)&g.pstatus, (void**)&g.ghist};
    for (void** p : ptrs) {
        cudaFree(*p);
        *p = nullptr;
    }
    g.cap_L = 0;        // perm shares the lookup capacity with keys / vals
    g.cap_S = 0;        // seg_row shares it with seg_start
    g.cap_nxt = 0;
    g.cap_T = 0;
    g.cap_Hh = 0;
    return FAE_OK;
}
