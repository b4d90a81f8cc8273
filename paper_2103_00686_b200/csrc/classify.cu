// classify.cu — input classifier, mini-batch bundling and replicator extract
// (SURVEY §8(a) a5, a6, a7).
//
//  a5  P:L476-479 (§4.2): an input is hot iff all its lookups hit hot rows.
//  a6  P:L493-496: bundle hot / cold inputs into all-hot / all-cold batches;
//      emit the hot CSR in hot ids so hot batches run entirely on the GPU.
//  a7  P:L317, L502: extract the hot rows into the replicated hot table.
//
// B200 design: ONE pass over the sparse inputs.  Each CTA owns a tile of
// records; for every lookup it does one 128-bit rank-directory load (bit +
// hot id together, L2-resident), keeps the hot ids in shared memory, decides
// the records' class with a block vote, gets its output offsets from a
// decoupled look-back scan, and writes hot_ids / cold_ids / the hot CSR with
// coalesced stores.  The dataset (Kaggle-shaped: 4.7 GB) is read exactly once.
#include <algorithm>

#include "fae_internal.cuh"

namespace fae {

fae_status validate_schema(Ctx* c, const fae_tables* t, const char* who);
fae_status validate_csr(Ctx* c, const fae_tables* t, const fae_csr* d, const char* who);
fae_status upload_schema(Ctx* c, const fae_tables* t, std::vector<int64_t>& rowbase);

constexpr int kClsThreads = 256;
// fixed pooling: threads per tile (measured on B200, 45M Kaggle-shaped
// records: 256 threads 9.1 ms, 512 threads 10.3 ms)
constexpr int kClsFix = 256;
constexpr int kClsItems = 8192;      // lookups per tile kept in smem (fixed pooling)
constexpr int kRecBits = 28;         // look-back packing: records | lookups << 28
constexpr uint64_t kRecMask = (1ull << kRecBits) - 1;

// Fixed pooling, Tn*P <= kClsItems.  TR records per tile.
__global__ void __launch_bounds__(kClsFix)
k_classify_fixed(const int32_t* __restrict__ idx, int64_t n_rec, int Tn, int P, int TR,
                 const int64_t* __restrict__ rowbase, const uint4* __restrict__ dir,
                 int64_t* __restrict__ hot_ids, int64_t* __restrict__ cold_ids,
                 int32_t* __restrict__ hot_idx, uint64_t* __restrict__ status,
                 uint32_t* __restrict__ ctr, int64_t* __restrict__ result, uint32_t* err,
                 const int64_t* __restrict__ rows) {
    extern __shared__ int64_t s_dyn[];
    int64_t* s_rb = s_dyn;                               // [Tn+1]
    int64_t* s_rows = s_dyn + (Tn + 1);                  // [Tn]
    int32_t* s_hid = (int32_t*)(s_dyn + 2 * Tn + 1);     // [kClsItems]
    __shared__ int s_cold[kClsFix];
    __shared__ int s_list[kClsFix];
    __shared__ int s_wsum[kClsFix / 32];
    __shared__ int s_tile;
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int z = tid; z <= Tn; z += blockDim.x) s_rb[z] = rowbase[z];
    for (int z = tid; z < Tn; z += blockDim.x) s_rows[z] = rows[z];
    if (tid < TR) s_cold[tid] = 0;
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t r0 = tile * TR;
    if (r0 >= n_rec && tile != 0) return;
    const int nrec = (int)std::min<int64_t>(TR, std::max<int64_t>(0, n_rec - r0));
    const int TnP = Tn * P;
    const int nitems = nrec * TnP;
    const int32_t* src = idx + r0 * (int64_t)TnP;
    // 8 lookups per thread in flight: index loads, then the rank-directory
    // loads (L2-resident), then the tests; the next round's index loads are
    // issued before this round's directory loads (one dependent trip per round)
    int32_t jn[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int q = u * kClsFix + tid;
        jn[u] = q < nitems ? __ldg(src + q) : 0;
    }
    for (int q0 = 0; q0 < nitems; q0 += kClsFix * 8) {
        int32_t jv[8];
        int zv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int q = q0 + u * kClsFix + tid;
            jv[u] = jn[u];
            zv[u] = q < nitems ? (q % TnP) / P : -1;
        }
        if (q0 + kClsFix * 8 < nitems) {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int q = q0 + kClsFix * 8 + u * kClsFix + tid;
                jn[u] = q < nitems ? __ldg(src + q) : 0;
            }
        }
        uint4 e[8];
        int64_t gv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            gv[u] = -1;
            if (zv[u] >= 0) {
                if (jv[u] < 0 || (int64_t)jv[u] >= s_rows[zv[u]]) {
                    atomicOr(err, kErrIndex);
                } else {
                    gv[u] = s_rb[zv[u]] + jv[u];
                    e[u] = __ldg(dir + (gv[u] >> 6));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int q = q0 + u * kClsFix + tid;
            if (zv[u] < 0) continue;
            int32_t hid = -1;
            uint32_t rk;
            if (gv[u] >= 0 && hs_test(e[u], gv[u], &rk)) hid = (int32_t)rk;
            else s_cold[q / TnP] = 1;
            s_hid[q] = hid;
        }
    }
    __syncthreads();
    const bool hot = tid < nrec && !s_cold[tid];
    const uint32_t bal = __ballot_sync(0xffffffffu, hot);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int wp = 0, tot = 0;
    for (int w = 0; w < kClsFix / 32; w++) {
        if (w < warp) wp += s_wsum[w];
        tot += s_wsum[w];
    }
    const int rank = wp + __popc(bal & lanemask_lt());
    if (tid == 0) {
        s_ex = lookback_u64(status, tile, (uint64_t)tot);
        const int64_t last = n_rec > 0 ? (n_rec - 1) / TR : 0;
        if (tile == last) {
            result[0] = (int64_t)(s_ex + tot);
        }
    }
    __syncthreads();
    const int64_t ex = (int64_t)s_ex;
    if (tid < nrec) {
        if (hot) {
            hot_ids[ex + rank] = r0 + tid;
            s_list[rank] = tid;
        } else {
            cold_ids[(r0 - ex) + (tid - rank)] = r0 + tid;
        }
    }
    __syncthreads();
    int32_t* dst = hot_idx + ex * (int64_t)TnP;
    const int nout = tot * TnP;
    for (int jx = tid; jx < nout; jx += kClsFix) {
        const int k = jx / TnP;
        const int qq = jx - k * TnP;
        dst[jx] = s_hid[s_list[k] * TnP + qq];
    }
}

// Fixed pooling, persistent and TMA-staged (the default when idx is 16-byte
// aligned).  Each CTA loops over tiles of TR records claimed in order from a
// counter, through a 3-slot shared-memory ring: while it classifies tile i,
// the async (TMA) engine already holds the copy of tile i+1 in flight (one
// 1-D bulk copy of TR*Tn*P ids per tile), and tile i-1 waits, classified, for
// its output offsets.  One thread per record walks its Tn*P lookups in table
// order (table parameters are shared-memory broadcasts): a lookup into a
// table whose rows are ALL hot (the small tables) gets its hot id
// base_z + j without touching the rank directory; the others issue their
// 16-byte directory loads 8 at a time.  Hot ids overwrite the staged ids in
// place.  A tile publishes its hot-record count right after classifying and
// finishes its decoupled look-back one tile LATER (after classifying the
// next one), so the walk finds its predecessors already published instead of
// stalling the CTA; then its hot_ids / cold_ids and hot CSR are written with
// coalesced stores.
constexpr int kBulkRec = 256;          // threads per CTA (>= records per tile)
#ifndef FAE_CLS_L2HINT
#define FAE_CLS_L2HINT 1     // dataset tiles evict-first, rank directory evict-last, outputs streamed
#endif
constexpr int kBulkSlots = 3;
#ifndef FAE_CLS_MINB
#define FAE_CLS_MINB 4      // CTAs per SM (registers capped at 64)
#endif
#ifndef FAE_CLS_SMEM_KB
#define FAE_CLS_SMEM_KB 50  // the three tiles' shared memory per CTA
#endif
__global__ void __launch_bounds__(kBulkRec, FAE_CLS_MINB)
k_classify_bulk(const int32_t* __restrict__ idx, int64_t n_rec, int Tn, int P, int TR, int64_t n_tiles,
                const int64_t* __restrict__ rowbase, const int64_t* __restrict__ rows,
                const int64_t* __restrict__ hbase, const uint4* __restrict__ dir,
                int64_t* __restrict__ hot_ids, int64_t* __restrict__ cold_ids, int32_t* __restrict__ hot_idx,
                uint64_t* __restrict__ status, uint32_t* __restrict__ ctr, int64_t* __restrict__ result,
                uint32_t* err, uint32_t div_magic) {
    extern __shared__ __align__(128) unsigned char s_raw[];
    const int TnP = Tn * P;
    const int tile_items = TR * TnP;                      // multiple of 4 (TR % 32 == 0)
    int32_t* bufs = reinterpret_cast<int32_t*>(s_raw);     // [kBulkSlots][tile_items]
    int64_t* s_rb = reinterpret_cast<int64_t*>(bufs + kBulkSlots * tile_items);   // [Tn] global row base
    int64_t* s_hb = s_rb + Tn;                                       // [Tn] hot-id base, or -1
    int32_t* s_rows = reinterpret_cast<int32_t*>(s_hb + Tn);         // [Tn]
    int32_t* s_pq = s_rows + Tn;                                     // [TnP] items needing a probe
    __shared__ int s_np;
    __shared__ uint64_t s_bar[kBulkSlots];
    __shared__ int64_t s_tile[kBulkSlots];
    __shared__ int s_tot[kBulkSlots];
    __shared__ int s_rk[kBulkSlots][kBulkRec];             // rank among the tile's hot (>= 0) / cold (< 0) records
    __shared__ int s_list[kBulkSlots][kBulkRec];           // hot records of the tile, in order
    __shared__ int s_wsum[kBulkRec / 32];
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if FAE_CLS_L2HINT
    const uint64_t pol_dir = l2_policy_evict_last();
#endif
    for (int z = tid; z < Tn; z += blockDim.x) {
        s_rb[z] = rowbase[z];
        s_rows[z] = (int32_t)rows[z];
        s_hb[z] = hbase[z];
    }
    if (tid == 0) {   // the items of a record that probe the rank directory, in item order
        int np = 0;
        for (int q = 0; q < TnP; q++)
            if (hbase[q / P] < 0) s_pq[np++] = q;
        s_np = np;
    }
    const int64_t last_full = n_rec / TR;   // tiles [0, last_full) are full (bulk-copied)
    auto claim = [&](int slot) {            // thread 0
        const int64_t t = (int64_t)atomicAdd(ctr, 1u);
        s_tile[slot] = t;
        if (t < last_full) {
            fence_proxy_async_smem();
#if FAE_CLS_L2HINT
            bulk_load_hint(bufs + slot * tile_items, idx + t * tile_items, (uint32_t)tile_items * 4u, &s_bar[slot],
                           l2_policy_evict_first());
#else
            bulk_load(bufs + slot * tile_items, idx + t * tile_items, (uint32_t)tile_items * 4u, &s_bar[slot]);
#endif
        }
    };
    if (tid == 0) {
        for (int k = 0; k < kBulkSlots; k++) mbar_init(&s_bar[k], 1);
        mbar_init_fence();
        claim(0);
        claim(1);
    }
    __syncthreads();
    uint32_t phase_bits = 0u;                 // bit k: parity of slot k's next completion
    int prev = -1;                            // slot of the classified tile awaiting its writes
    for (int i = 0;; i++) {
        const int cur = i % kBulkSlots;
        const int64_t tile = s_tile[cur];
        const bool have = tile < n_tiles;
        if (have) {
            int32_t* buf = bufs + cur * tile_items;
            const int64_t r0 = tile * TR;
            const int nrec = (int)(n_rec - r0 < (int64_t)TR ? n_rec - r0 : (int64_t)TR);
            if (tile < last_full) {
                mbar_wait(&s_bar[cur], (phase_bits >> cur) & 1u);
                phase_bits ^= 1u << cur;
            } else {   // the partial last tile: plain loads
                const int32_t* src = idx + r0 * TnP;
                for (int q = tid; q < nrec * TnP; q += blockDim.x) buf[q] = __ldg(src + q);
                __syncthreads();
            }
            bool cold = true;
            if (tid < nrec) {
                cold = false;
                int32_t* my = buf + tid * TnP;
                // all-hot tables: hot id = base_z + j, no probe
                for (int q = 0; q < TnP; q++) {
                    const int z = P == 1 ? q : q / P;
                    if (s_hb[z] < 0) continue;
                    const int32_t j = my[q];
                    if (j < 0 || j >= s_rows[z]) {
                        atomicOr(err, kErrIndex);
                        cold = true;
                        my[q] = -1;
                    } else {
                        my[q] = (int32_t)(s_hb[z] + j);
                    }
                }
                // the others: rank-directory probes, 8 in flight
                const int np = s_np;
                for (int k0 = 0; k0 < np; k0 += 8) {
                    uint4 e[8];
                    int64_t gv[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        gv[u] = -1;
                        if (k0 + u < np) {
                            const int q = s_pq[k0 + u];
                            const int z = P == 1 ? q : q / P;
                            const int32_t j = my[q];
                            if (j < 0 || j >= s_rows[z]) {
                                atomicOr(err, kErrIndex);
                                cold = true;
                            } else {
                                gv[u] = s_rb[z] + j;
#if FAE_CLS_L2HINT
                                e[u] = ldg_hint_u4(dir + (gv[u] >> 6), pol_dir);
#else
                                e[u] = __ldg(dir + (gv[u] >> 6));
#endif
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        if (k0 + u >= np) break;
                        int32_t hid = -1;
                        if (gv[u] >= 0) {
                            uint32_t rk;
                            if (hs_test(e[u], gv[u], &rk)) hid = (int32_t)rk;
                            else cold = true;
                        }
                        my[s_pq[k0 + u]] = hid;
                    }
                }
            }
            const bool hot = tid < nrec && !cold;
            const uint32_t bal = __ballot_sync(0xffffffffu, hot);
            if (lane == 0) s_wsum[warp] = __popc(bal);
            __syncthreads();
            int wp = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kBulkRec / 32; w++) {
                if (w < warp) wp += s_wsum[w];
                tot += s_wsum[w];
            }
            const int rank = wp + __popc(bal & lanemask_lt());
            if (tid < nrec) {
                s_rk[cur][tid] = hot ? rank : -1 - (tid - rank);
                if (hot) s_list[cur][rank] = tid;
            }
            if (tid == 0) {
                s_tot[cur] = tot;
                lookback_publish(status, tile, (uint64_t)tot);
            }
        }
        __syncthreads();
        if (prev >= 0) {   // the previous tile: finish its look-back, write it out
            const int64_t pt = s_tile[prev];
            const int ptot = s_tot[prev];
            if (warp == 0) {
                const uint64_t ex = lookback_finish_warp(status, pt, (uint64_t)ptot);
                if (lane == 0) {
                    s_ex = ex;
                    if (pt == n_tiles - 1) result[0] = (int64_t)(ex + ptot);
                }
            }
            __syncthreads();
            const int64_t ex = (int64_t)s_ex;
            const int64_t r0 = pt * TR;
            const int nrec = (int)(n_rec - r0 < (int64_t)TR ? n_rec - r0 : (int64_t)TR);
            if (tid < nrec) {
                const int rk = s_rk[prev][tid];
                if (rk >= 0) __stcs(hot_ids + ex + rk, (int64_t)(r0 + tid));
                else __stcs(cold_ids + (r0 - ex) + (-1 - rk), (int64_t)(r0 + tid));
            }
            const int32_t* pbuf = bufs + prev * tile_items;
            int32_t* dst = hot_idx + ex * (int64_t)TnP;
            const int nout = ptot * TnP;
            for (int jx = tid; jx < nout; jx += blockDim.x) {
                const int k = (int)__umulhi((uint32_t)jx, div_magic);   // jx / TnP
                __stcs(dst + jx, pbuf[s_list[prev][k] * TnP + (jx - k * TnP)]);
            }
            __syncthreads();   // slot `prev` is free again
        }
        if (!have) break;
        if (tid == 0) claim((i + 2) % kBulkSlots);   // == prev (or the untouched third slot at i = 0)
        prev = cur;
    }
}

// General (offsets or large Tn*P): warp per record, hot ids recomputed in the
// write phase (L1/L2 hits).  Look-back value = records | lookups << 28.
constexpr int kGenRec = 64;   // records per tile
__global__ void __launch_bounds__(kClsThreads)
k_classify_general(const int32_t* __restrict__ idx, const int64_t* __restrict__ off, int P,
                   int64_t n_rec, int Tn, const int64_t* __restrict__ rowbase,
                   const int64_t* __restrict__ rows, const uint4* __restrict__ dir,
                   int64_t* __restrict__ hot_ids, int64_t* __restrict__ cold_ids,
                   int32_t* __restrict__ hot_idx, int64_t* __restrict__ hot_off,
                   uint64_t* __restrict__ status, uint32_t* __restrict__ ctr,
                   int64_t* __restrict__ result, uint32_t* err) {
    extern __shared__ int64_t s_dyn[];
    int64_t* s_rb = s_dyn;
    int64_t* s_rows = s_dyn + (Tn + 1);
    __shared__ int s_hot[kGenRec];
    __shared__ int64_t s_len[kGenRec];
    __shared__ int s_rank[kGenRec];
    __shared__ int64_t s_lpre[kGenRec];
    __shared__ int s_tile;
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kClsThreads / 32;
    for (int z = tid; z <= Tn; z += blockDim.x) s_rb[z] = rowbase[z];
    for (int z = tid; z < Tn; z += blockDim.x) s_rows[z] = rows[z];
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t r0 = tile * kGenRec;
    if (r0 >= n_rec && tile != 0) return;
    const int nrec = (int)std::min<int64_t>(kGenRec, std::max<int64_t>(0, n_rec - r0));
    auto bag_lo = [&](int64_t b) -> int64_t { return off ? off[b] : b * (int64_t)P; };
    for (int rl = warp; rl < nrec; rl += NW) {
        const int64_t r = r0 + rl;
        bool cold = false;
        for (int z = 0; z < Tn; z++) {
            const int64_t lo = bag_lo(r * Tn + z), hi = bag_lo(r * Tn + z + 1);
            for (int64_t p = lo + lane; p < hi; p += 32) {
                const int32_t j = __ldg(idx + p);
                if (j < 0 || (int64_t)j >= s_rows[z]) {
                    atomicOr(err, kErrIndex);
                    cold = true;
                } else {
                    const int64_t g = s_rb[z] + j;
                    uint32_t rk;
                    if (!hs_test(__ldg(dir + (g >> 6)), g, &rk)) cold = true;
                }
            }
        }
        cold = __any_sync(0xffffffffu, cold);
        if (lane == 0) {
            s_hot[rl] = !cold;
            s_len[rl] = bag_lo((r + 1) * Tn) - bag_lo(r * Tn);
        }
    }
    __syncthreads();
    if (warp == 0) {
        // scan over the tile's records of (hot, hot lookups), 2 records per lane
        uint64_t v0 = 0, v1 = 0;
        const int a = 2 * lane, b = 2 * lane + 1;
        if (a < nrec && s_hot[a]) v0 = 1ull | ((uint64_t)s_len[a] << kRecBits);
        if (b < nrec && s_hot[b]) v1 = 1ull | ((uint64_t)s_len[b] << kRecBits);
        const uint64_t pair = v0 + v1;
        uint64_t x = pair;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint64_t tot = __shfl_sync(0xffffffffu, x, 31);
        if (lane == 0) {
            s_ex = lookback_u64(status, tile, tot);
            const int64_t last = n_rec > 0 ? (n_rec - 1) / kGenRec : 0;
            if (tile == last) {
                const uint64_t inc = s_ex + tot;
                result[0] = (int64_t)(inc & kRecMask);
                result[1] = (int64_t)(inc >> kRecBits);
                if (off && hot_off) hot_off[(inc & kRecMask) * Tn] = (int64_t)(inc >> kRecBits);
            }
        }
        const uint64_t ex0 = x - pair;
        if (a < nrec) {
            s_rank[a] = (int)(ex0 & kRecMask);
            s_lpre[a] = (int64_t)(ex0 >> kRecBits);
        }
        if (b < nrec) {
            const uint64_t ex1 = ex0 + v0;
            s_rank[b] = (int)(ex1 & kRecMask);
            s_lpre[b] = (int64_t)(ex1 >> kRecBits);
        }
    }
    __syncthreads();
    const int64_t ex_rec = (int64_t)(s_ex & kRecMask);
    const int64_t ex_lk = (int64_t)(s_ex >> kRecBits);
    for (int rl = warp; rl < nrec; rl += NW) {
        const int64_t r = r0 + rl;
        if (!s_hot[rl]) {
            if (lane == 0) cold_ids[(r0 - ex_rec) + (rl - s_rank[rl])] = r;
            continue;
        }
        const int64_t h = ex_rec + s_rank[rl];
        if (lane == 0) hot_ids[h] = r;
        int64_t out = ex_lk + s_lpre[rl];
        const int64_t rbase = bag_lo(r * Tn);
        for (int z = 0; z < Tn; z++) {
            const int64_t lo = bag_lo(r * Tn + z), hi = bag_lo(r * Tn + z + 1);
            if (off && hot_off && lane == 0) hot_off[h * Tn + z] = out + (lo - rbase);
            for (int64_t p = lo + lane; p < hi; p += 32) {
                const int64_t g = s_rb[z] + __ldg(idx + p);
                uint32_t rk;
                hs_test(__ldg(dir + (g >> 6)), g, &rk);
                hot_idx[out + (p - rbase)] = (int32_t)rk;
            }
        }
    }
}

// extract: warp per 64-row word; lane l owns bits l (lo) and l (hi)
// kBack = false: W_hot[hot_id(g)] = W[g] (a7, extract); kBack = true:
// W[g] = W_hot[hot_id(g)] (the swap sync back to the master tables).
template <int NV4, bool kBack = false>
__global__ void __launch_bounds__(256)
k_extract(const uint4* __restrict__ dir, int64_t total, const float* W, int D, float* W_hot) {
    const int lane = threadIdx.x & 31;
    const int64_t wpb = blockDim.x >> 5;
    const int64_t words = (total + 63) >> 6;
    for (int64_t w = blockIdx.x * wpb + (threadIdx.x >> 5); w < words; w += (int64_t)gridDim.x * wpb) {
        const uint4 e = dir[w];
        const uint32_t lo = e.x, hi = e.y;
        const uint32_t lt = lanemask_lt();
        const int nd4 = D / 4;
        if ((lo >> lane) & 1u) {
            const int64_t g = w * 64 + lane;
            const int64_t hid = (int64_t)e.z + __popc(lo & lt);
            float4* s = reinterpret_cast<float4*>(const_cast<float*>(W) + g * D);
            float4* d = reinterpret_cast<float4*>(W_hot + hid * D);
            if (kBack) for (int k = 0; k < nd4; k++) s[k] = d[k];
            else for (int k = 0; k < nd4; k++) d[k] = s[k];
        }
        if ((hi >> lane) & 1u) {
            const int64_t g = w * 64 + 32 + lane;
            const int64_t hid = (int64_t)e.z + __popc(lo) + __popc(hi & lt);
            float4* s = reinterpret_cast<float4*>(const_cast<float*>(W) + g * D);
            float4* d = reinterpret_cast<float4*>(W_hot + hid * D);
            if (kBack) for (int k = 0; k < nd4; k++) s[k] = d[k];
            else for (int k = 0; k < nd4; k++) d[k] = s[k];
        }
    }
}

template <bool kBack = false>
__global__ void __launch_bounds__(256)
k_extract_scalar(const uint4* __restrict__ dir, int64_t total, const float* W, int D, float* W_hot) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        uint32_t rk;
        if (hs_test(dir[g >> 6], g, &rk))
            for (int d = 0; d < D; d++) {
                if (kBack) const_cast<float*>(W)[g * D + d] = W_hot[(int64_t)rk * D + d];
                else W_hot[(int64_t)rk * D + d] = W[g * D + d];
            }
    }
}

static int sms(Ctx* c) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, c->device);
    return n;
}

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_classify(fae_ctx* h, const fae_tables* tabs, const fae_csr* data, int32_t batch,
                                   uint64_t shuffle_seed, fae_packed* out) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_schema(c, tabs, "fae_classify");
    if (st != FAE_OK) return st;
    st = validate_csr(c, tabs, data, "fae_classify");
    if (st != FAE_OK) return st;
    if (!out || !out->hot_ids || !out->cold_ids || (!out->hot_idx && data->n_lookups > 0))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: null output buffer");
    if (data->off && !out->hot_off) return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: hot_off required with offsets");
    if (batch < 1) return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: batch must be >= 1");
    if (shuffle_seed != 0) return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: only the stable order (shuffle_seed 0) is implemented");
    HotSet& hs = c->hs;
    if (!hs.valid) return set_err(c, FAE_ERR_NOT_INIT, "fae_classify: no hot set (call fae_threshold first)");
    const int Tn = tabs->n_tables;
    if (Tn != hs.n_tables) return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: schema differs from the hot set's");
    for (int z = 0; z < Tn; z++)
        if (tabs->rows[z] != hs.rows[z]) return set_err(c, FAE_ERR_INVALID_ARG, "fae_classify: schema differs from the hot set's");
    const int64_t n = data->n_records;
    if (n >= (int64_t)kRecMask || data->n_lookups >= (1ll << 34))
        return set_err(c, FAE_ERR_CAPACITY, "fae_classify: > 2^28 records or > 2^34 lookups per shard");
    FAE_CUDA(c, cudaMemcpyAsync(c->d_rows_tmp, tabs->rows, sizeof(int64_t) * Tn, cudaMemcpyHostToDevice, c->stream));
    const int P = data->fixed_pool;
    // the persistent TMA-staged kernel: fixed pooling, 16-byte aligned ids,
    // two tiles of >= 32 records in shared memory
    const int64_t TnP64 = (int64_t)Tn * P;
    // three tiles in shared memory, <= 64 KB: 3 CTAs per SM (the register limit)
    int TRb = TnP64 > 0 ? (int)std::min<int64_t>(kBulkRec, (FAE_CLS_SMEM_KB * 1024 / 4 / kBulkSlots / TnP64) & ~31ll) : 0;
    const bool bulk = !data->off && TnP64 > 0 && TRb >= 32 && (((uintptr_t)data->idx) & 15) == 0 && n > 0 &&
                      !c->cls_legacy;
    if (bulk) {
        std::vector<int64_t> hb(Tn);
        for (int z = 0; z < Tn; z++)   // tables whose rows are all hot: hot id = base_z + j
            hb[z] = (hs.base[z + 1] - hs.base[z] == tabs->rows[z]) ? hs.base[z] : -1;
        const int64_t tiles = cdiv(n, TRb);
        size_t o = 0;
        auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
        const size_t o_st = take(sizeof(uint64_t) * tiles);
        const size_t o_ctr = take(sizeof(uint32_t) * 4);
        const size_t o_res = take(sizeof(int64_t) * 4);
        const size_t o_hb = take(sizeof(int64_t) * Tn);
        char* sc = (char*)scratch(c, o);
        if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_classify: scratch allocation failed");
        int64_t* d_res = (int64_t*)(sc + o_res);
        int64_t* d_hb = (int64_t*)(sc + o_hb);
        FAE_CUDA(c, cudaMemsetAsync(sc, 0, o_hb, c->stream));
        FAE_CUDA(c, cudaMemcpyAsync(d_hb, hb.data(), sizeof(int64_t) * Tn, cudaMemcpyHostToDevice, c->stream));
        const size_t smem = sizeof(int32_t) * kBulkSlots * (size_t)TRb * TnP64 + sizeof(int64_t) * 2 * Tn +
                            sizeof(int32_t) * (Tn + TnP64);
        FAE_CUDA(c, cudaFuncSetAttribute(k_classify_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 1;
        FAE_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_classify_bulk, kBulkRec, smem));
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms(c) * std::max(per_sm, 1)));
        const uint32_t magic = (uint32_t)((0xFFFFFFFFull + (uint64_t)TnP64) / (uint64_t)TnP64);   // ceil(2^32 / TnP)
        k_classify_bulk<<<(unsigned)grid, kBulkRec, smem, c->stream>>>(
            data->idx, n, Tn, P, TRb, tiles, hs.d_rowbase, c->d_rows_tmp, d_hb, hs.dir, out->hot_ids, out->cold_ids,
            out->hot_idx, (uint64_t*)(sc + o_st), (uint32_t*)(sc + o_ctr), d_res, c->d_err, magic);
        FAE_LAUNCHED(c);
        int64_t res[2] = {0, 0};
        FAE_CUDA(c, cudaMemcpyAsync(res, d_res, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, c->stream));
        st = read_latched(c);
        const int64_t nh = res[0];
        out->n_hot = nh;
        out->n_cold = n - nh;
        out->n_hot_lookups = nh * TnP64;
        out->n_hot_batches = cdiv(nh, batch);
        out->n_cold_batches = cdiv(n - nh, batch);
        return st;
    }
    const bool fast = !data->off && (int64_t)Tn * P <= kClsItems && Tn * P > 0;
    const int TR = fast ? std::min(kClsFix, std::max(1, kClsItems / (Tn * P))) : kGenRec;
    const int64_t tiles = std::max<int64_t>(1, cdiv(n, TR));
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
    const size_t o_st = take(sizeof(uint64_t) * tiles);
    const size_t o_ctr = take(sizeof(uint32_t) * 4);
    const size_t o_res = take(sizeof(int64_t) * 4);
    char* sc = (char*)scratch(c, o);
    if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_classify: scratch allocation failed");
    uint64_t* d_st = (uint64_t*)(sc + o_st);
    uint32_t* d_ctr = (uint32_t*)(sc + o_ctr);
    int64_t* d_res = (int64_t*)(sc + o_res);
    FAE_CUDA(c, cudaMemsetAsync(sc, 0, o, c->stream));
    const size_t rb_smem = sizeof(int64_t) * (2 * Tn + 1);
    if (fast) {
        const size_t smem = rb_smem + sizeof(int32_t) * kClsItems;
        if (smem > 48 * 1024)
            FAE_CUDA(c, cudaFuncSetAttribute(k_classify_fixed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_classify_fixed<<<(unsigned)tiles, kClsFix, smem, c->stream>>>(
            data->idx, n, Tn, P, TR, hs.d_rowbase, hs.dir, out->hot_ids, out->cold_ids, out->hot_idx, d_st, d_ctr,
            d_res, c->d_err, c->d_rows_tmp);
        FAE_LAUNCHED(c);
    } else {
        if (rb_smem > 48 * 1024)
            FAE_CUDA(c, cudaFuncSetAttribute(k_classify_general, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rb_smem));
        k_classify_general<<<(unsigned)tiles, kClsThreads, rb_smem, c->stream>>>(
            data->idx, data->off, P, n, Tn, hs.d_rowbase, c->d_rows_tmp, hs.dir, out->hot_ids, out->cold_ids,
            out->hot_idx, data->off ? out->hot_off : nullptr, d_st, d_ctr, d_res, c->d_err);
        FAE_LAUNCHED(c);
    }
    int64_t res[2] = {0, 0};
    FAE_CUDA(c, cudaMemcpyAsync(res, d_res, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, c->stream));
    st = read_latched(c);
    const int64_t nh = res[0];
    out->n_hot = nh;
    out->n_cold = n - nh;
    out->n_hot_lookups = fast ? nh * (int64_t)Tn * P : res[1];
    out->n_hot_batches = cdiv(nh, batch);
    out->n_cold_batches = cdiv(n - nh, batch);
    if (n == 0 && data->off && out->hot_off) {
        int64_t zero = 0;
        FAE_CUDA(c, cudaMemcpy(out->hot_off, &zero, sizeof(int64_t), cudaMemcpyHostToDevice));
    }
    return st;
}

extern "C" fae_status fae_extract(fae_ctx* h, const float* W, int32_t dim, float* W_hot) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    HotSet& hs = c->hs;
    if (!hs.valid) return set_err(c, FAE_ERR_NOT_INIT, "fae_extract: no hot set");
    if (!W || (!W_hot && hs.H_total > 0) || dim < 1) return set_err(c, FAE_ERR_INVALID_ARG, "fae_extract: bad arguments");
    if (hs.H_total == 0) return FAE_OK;
    const int64_t total = hs.total_rows;
    const bool vec = dim % 4 == 0 && (((uintptr_t)W | (uintptr_t)W_hot) & 15) == 0;
    if (vec) {
        const int64_t words = cdiv(total, 64);
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(words, 8), (int64_t)sms(c) * 16));
        k_extract<1><<<(unsigned)g, 256, 0, c->stream>>>(hs.dir, total, W, dim, W_hot);
    } else {
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), (int64_t)sms(c) * 8));
        k_extract_scalar<false><<<(unsigned)g, 256, 0, c->stream>>>(hs.dir, total, W, dim, W_hot);
    }
    FAE_LAUNCHED(c);
    return FAE_OK;
}

// cold CSR in global row ids (fixed pooling): out[k*TnP + q] = rowbase[z] +
// idx[cold[k]*TnP + q].  A cold id outside [0, n_rec) latches INDEX_RANGE and
// its lookups are written as row 0 (the call then fails).
__global__ void __launch_bounds__(256)
k_pack_cold(const int32_t* __restrict__ idx, const int64_t* __restrict__ cold_ids, int64_t n_cold, int64_t n_rec,
            int Tn, int P, const int64_t* __restrict__ rowbase, const int64_t* __restrict__ rows,
            int32_t* __restrict__ out, uint32_t* err) {
    const int64_t TnP = (int64_t)Tn * P;
    const int64_t n = n_cold * TnP;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / TnP, q = e - k * TnP;
        const int z = (int)(q / P);
        const int64_t r = cold_ids[k];
        const int32_t j = (r >= 0 && r < n_rec) ? idx[r * TnP + q] : -1;
        if (j < 0 || (int64_t)j >= rows[z]) {
            atomicOr(err, kErrIndex);
            out[e] = 0;
        } else {
            out[e] = (int32_t)(rowbase[z] + j);
        }
    }
}

// explicit offsets, pass 1: bag sizes of the cold records, sz[k*Tn + z]
__global__ void __launch_bounds__(256)
k_cold_sizes(const int64_t* __restrict__ off, const int64_t* __restrict__ cold_ids, int64_t n_cold, int64_t n_rec,
             int Tn, int64_t* __restrict__ sz, uint32_t* err) {
    const int64_t n = n_cold * Tn;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / Tn, z = e - k * Tn;
        const int64_t r = cold_ids[k];
        if (r < 0 || r >= n_rec) {
            atomicOr(err, kErrIndex);
            sz[e] = 0;
        } else {
            sz[e] = off[r * Tn + z + 1] - off[r * Tn + z];
        }
    }
}

// exclusive scan of n int64 values (< 2^62 in total) into out[0..n], out[n] =
// total: tiles of 256 x 16, block scan + decoupled look-back
constexpr int kScanItems = 16;
__global__ void __launch_bounds__(256)
k_scan_i64(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out, uint64_t* __restrict__ status,
           uint32_t* __restrict__ ctr) {
    __shared__ int s_tile;
    __shared__ uint64_t s_w[8];
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t i0 = tile * (256 * kScanItems) + (int64_t)tid * kScanItems;
    uint64_t v[kScanItems], sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        v[j] = i0 + j < n ? (uint64_t)in[i0 + j] : 0ull;
        sum += v[j];
    }
    uint64_t x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint64_t wp = 0, tot = 0;
    for (int w = 0; w < 8; w++) {
        if (w < warp) wp += s_w[w];
        tot += s_w[w];
    }
    if (tid == 0) {
        s_ex = lookback_u64(status, tile, tot);
        const int64_t last = n > 0 ? (n - 1) / (256 * kScanItems) : 0;
        if (tile == last) out[n] = (int64_t)(s_ex + tot);
    }
    __syncthreads();
    uint64_t run = s_ex + wp + x - sum;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (i0 + j < n) out[i0 + j] = (int64_t)run;
        run += v[j];
    }
}

// explicit offsets, pass 2: warp per cold record, lookups in global row ids
__global__ void __launch_bounds__(256)
k_pack_cold_off(const int32_t* __restrict__ idx, const int64_t* __restrict__ off,
                const int64_t* __restrict__ cold_ids, int64_t n_cold, int64_t n_rec, int Tn,
                const int64_t* __restrict__ rowbase, const int64_t* __restrict__ rows,
                const int64_t* __restrict__ cold_off, int32_t* __restrict__ out, uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const int64_t wpb = blockDim.x >> 5;
    for (int64_t k = blockIdx.x * wpb + (threadIdx.x >> 5); k < n_cold; k += (int64_t)gridDim.x * wpb) {
        const int64_t r = cold_ids[k];
        if (r < 0 || r >= n_rec) continue;   // latched by k_cold_sizes
        for (int z = 0; z < Tn; z++) {
            const int64_t lo = off[r * Tn + z], hi = off[r * Tn + z + 1];
            const int64_t o = cold_off[k * Tn + z];
            for (int64_t p = lo + lane; p < hi; p += 32) {
                const int32_t j = idx[p];
                if (j < 0 || (int64_t)j >= rows[z]) {
                    atomicOr(err, kErrIndex);
                    out[o + (p - lo)] = 0;
                } else {
                    out[o + (p - lo)] = (int32_t)(rowbase[z] + j);
                }
            }
        }
    }
}

extern "C" fae_status fae_pack_cold(fae_ctx* h, const fae_tables* tabs, const fae_csr* data,
                                    const int64_t* cold_ids, int64_t n_cold, int32_t* cold_idx,
                                    int64_t* cold_off) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_schema(c, tabs, "fae_pack_cold");
    if (st != FAE_OK) return st;
    st = validate_csr(c, tabs, data, "fae_pack_cold");
    if (st != FAE_OK) return st;
    if (n_cold < 0 || n_cold > data->n_records ||
        (n_cold > 0 && (!cold_ids || (!cold_idx && data->n_lookups > 0) || (data->n_lookups > 0 && !data->idx))))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_pack_cold: bad sizes or null buffers");
    if (data->off && !cold_off) return set_err(c, FAE_ERR_INVALID_ARG, "fae_pack_cold: cold_off required with offsets");
    int64_t total = 0;
    for (int z = 0; z < tabs->n_tables; z++) total += tabs->rows[z];
    // the same bound as the step calls that train the cold batches (H < 2^31 - 1)
    if (total >= (1ll << 31) - 1) return set_err(c, FAE_ERR_CAPACITY, "fae_pack_cold: global row ids >= 2^31 - 1");
    const int Tn = tabs->n_tables;
    if (n_cold == 0) {
        if (cold_off) FAE_CUDA(c, cudaMemsetAsync(cold_off, 0, sizeof(int64_t), c->stream));
        return read_latched(c);
    }
    std::vector<int64_t> rowbase;
    st = upload_schema(c, tabs, rowbase);
    if (st != FAE_OK) return st;
    if (!data->off) {
        const int64_t n = n_cold * Tn * (int64_t)data->fixed_pool;
        if (n > 0) {
            const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sms(c) * 16));
            k_pack_cold<<<(unsigned)g, 256, 0, c->stream>>>(data->idx, cold_ids, n_cold, data->n_records, Tn,
                                                            data->fixed_pool, c->d_rowbase_tmp, c->d_rows_tmp,
                                                            cold_idx, c->d_err);
            FAE_LAUNCHED(c);
        }
        return read_latched(c);
    }
    // explicit offsets: bag sizes -> exclusive scan (cold_off) -> copy
    const int64_t nb = n_cold * Tn;
    const int64_t tiles = cdiv(nb, 256 * kScanItems);
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
    const size_t o_sz = take(sizeof(int64_t) * nb);
    const size_t o_st = take(sizeof(uint64_t) * tiles);
    const size_t o_ctr = take(sizeof(uint32_t) * 4);
    char* sc = (char*)scratch(c, o);
    if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_pack_cold: scratch allocation failed");
    int64_t* d_sz = (int64_t*)(sc + o_sz);
    FAE_CUDA(c, cudaMemsetAsync(sc + o_st, 0, o - o_st, c->stream));
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(nb, 256), (int64_t)sms(c) * 16));
    k_cold_sizes<<<(unsigned)g, 256, 0, c->stream>>>(data->off, cold_ids, n_cold, data->n_records, Tn, d_sz,
                                                     c->d_err);
    FAE_LAUNCHED(c);
    k_scan_i64<<<(unsigned)tiles, 256, 0, c->stream>>>(d_sz, nb, cold_off, (uint64_t*)(sc + o_st),
                                                       (uint32_t*)(sc + o_ctr));
    FAE_LAUNCHED(c);
    const int64_t gw = std::max<int64_t>(1, std::min<int64_t>(cdiv(n_cold, 8), (int64_t)sms(c) * 16));
    k_pack_cold_off<<<(unsigned)gw, 256, 0, c->stream>>>(data->idx, data->off, cold_ids, n_cold, data->n_records, Tn,
                                                         c->d_rowbase_tmp, c->d_rows_tmp, cold_off, cold_idx,
                                                         c->d_err);
    FAE_LAUNCHED(c);
    return read_latched(c);
}

extern "C" fae_status fae_scatter_hot(fae_ctx* h, const float* W_hot, int32_t dim, float* W) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    HotSet& hs = c->hs;
    if (!hs.valid) return set_err(c, FAE_ERR_NOT_INIT, "fae_scatter_hot: no hot set");
    if (!W || (!W_hot && hs.H_total > 0) || dim < 1) return set_err(c, FAE_ERR_INVALID_ARG, "fae_scatter_hot: bad arguments");
    if (hs.H_total == 0) return FAE_OK;
    const int64_t total = hs.total_rows;
    const bool vec = dim % 4 == 0 && (((uintptr_t)W | (uintptr_t)W_hot) & 15) == 0;
    if (vec) {
        const int64_t words = cdiv(total, 64);
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(words, 8), (int64_t)sms(c) * 16));
        k_extract<1, true><<<(unsigned)g, 256, 0, c->stream>>>(hs.dir, total, W, dim, const_cast<float*>(W_hot));
    } else {
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), (int64_t)sms(c) * 8));
        k_extract_scalar<true><<<(unsigned)g, 256, 0, c->stream>>>(hs.dir, total, W, dim, const_cast<float*>(W_hot));
    }
    FAE_LAUNCHED(c);
    return FAE_OK;
}
