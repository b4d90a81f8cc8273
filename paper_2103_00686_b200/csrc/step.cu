// step.cu — the hot mini-batch embedding step.
//
//  a8  fae_emb_fwd         Y[b] = sum_{p in bag b} W_hot[idx[p]]
//  a9  fae_emb_bwd_update  G[r] = sum_{p: idx[p]=r} dY[bag(p)]      (sort-and-segment)
//  a10                     W_hot[r] -= lr * G[r]
//  a11 fae_sync_hot_grads  G_global = sum over ranks
//
// Kernels (no tensor cores: gather/scatter, HBM/L2 bound):
//  k_emb_fwd      sub-warp group of D/4 lanes per bag, 128-bit row loads,
//                 4 independent rows in flight per lane, streaming Y stores.
//  k_bwd_prep     (hot id, bag) pairs + all radix-digit histograms, one pass.
//  k_sort_pass    onesweep LSD radix pass: warp match_any ranking, per-digit
//                 decoupled look-back, stable scatter; ceil(log2(H+1)/8) passes.
//  k_pieces       run-length segments of equal hot id split into <= kPiece
//                 pieces (decoupled look-back over (pieces, segments)).
//  k_seg_reduce   one D/4-lane group per piece sums its dY rows; single-piece
//                 segments apply SGD directly, multi-piece segments combine
//                 their partials in piece order (last-arriver), so the sum
//                 order is fixed: results are deterministic run to run and
//                 identical on every rank.
#include <algorithm>

#include "kern_common.cuh"

namespace fae {

// ---------------------------------------------------------------------------
// a8 forward
// ---------------------------------------------------------------------------
template <int LPB, int NV>
__global__ void __launch_bounds__(256)
k_emb_fwd(const float* __restrict__ W, int64_t H, int D,
          const int32_t* __restrict__ idx, const int64_t* __restrict__ off,
          int P, int64_t n_bags, float* __restrict__ Y, uint32_t* err) {
    fwd_bags<LPB, NV>(W, H, D, idx, off, P, n_bags, Y, err);
}

// ---------------------------------------------------------------------------
// a9 backward: pairs + digit histograms
// scalars: [0] n_valid, [1] n_pieces, [2] n_segs, [3] n_items
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t find_bag(const int64_t* __restrict__ off, int64_t n_bags, int64_t pos) {
    // largest b in [0, n_bags) with off[b] <= pos
    int64_t lo = 0, hi = n_bags - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= pos) lo = mid;
        else hi = mid - 1;
    }
    return (int32_t)lo;
}

__global__ void __launch_bounds__(256)
k_bwd_prep(const int32_t* __restrict__ idx, const int64_t* __restrict__ off, int P,
           int64_t n_bags, int64_t H, int passes, int64_t cap, uint32_t* __restrict__ keys,
           int32_t* __restrict__ vals, uint32_t* __restrict__ ghist,
           int64_t* __restrict__ scalars, uint32_t* err) {
    __shared__ uint32_t sh[kMaxSortPasses][kSortBins];
    for (int i = threadIdx.x; i < kMaxSortPasses * kSortBins; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = off ? off[0] : 0;
    const int64_t n = off ? off[n_bags] - base : n_bags * (int64_t)P;
    // a multi-hot batch larger than the workspace (cap = the sort's tile
    // capacity, max_batch_lookups): latch CAPACITY and apply nothing (every
    // later kernel of the step sees n_items = 0), never write past the
    // workspace
    if (n > cap || n < 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            scalars[3] = 0;
            atomicOr(err, kErrOverflow);
        }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) scalars[3] = n;
    int nvalid = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = __ldg(idx + base + p);
        const int32_t bag = off ? find_bag(off, n_bags, base + p) : (int32_t)(p / P);
        uint32_t key;
        if ((uint32_t)r >= (uint64_t)H) {
            atomicOr(err, kErrIndex);
            key = (uint32_t)H;
        } else {
            key = (uint32_t)r;
            nvalid++;
        }
        keys[p] = key;
        vals[p] = bag;
        for (int ps = 0; ps < passes; ps++) atomicAdd(&sh[ps][(key >> (kSortBits * ps)) & (kSortBins - 1)], 1u);
    }
    // warp reduce nvalid
    for (int o = 16; o; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
    if ((threadIdx.x & 31) == 0 && nvalid) atomicAdd((unsigned long long*)&scalars[0], (unsigned long long)nvalid);
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kSortBins; i += blockDim.x) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

// Merge prep for a11: gathered per-rank lists (padded to cap per rank).
__global__ void __launch_bounds__(256)
k_merge_prep(const int32_t* __restrict__ g_rows, const int32_t* __restrict__ g_counts,
             int world, int64_t cap, int64_t H, int passes, uint32_t* __restrict__ keys,
             int32_t* __restrict__ vals, uint32_t* __restrict__ ghist,
             int64_t* __restrict__ scalars) {
    __shared__ uint32_t sh[kMaxSortPasses][kSortBins];
    for (int i = threadIdx.x; i < kMaxSortPasses * kSortBins; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int64_t n = (int64_t)world * cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) scalars[3] = n;
    int nvalid = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int rk = (int)(p / cap);
        const int64_t j = p - (int64_t)rk * cap;
        uint32_t key = (uint32_t)H;
        if (j < g_counts[rk]) {
            const int32_t r = g_rows[p];
            if ((uint32_t)r < (uint64_t)H) {
                key = (uint32_t)r;
                nvalid++;
            }
        }
        keys[p] = key;
        vals[p] = (int32_t)p;
        for (int ps = 0; ps < passes; ps++) atomicAdd(&sh[ps][(key >> (kSortBits * ps)) & (kSortBins - 1)], 1u);
    }
    for (int o = 16; o; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
    if ((threadIdx.x & 31) == 0 && nvalid) atomicAdd((unsigned long long*)&scalars[0], (unsigned long long)nvalid);
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kSortBins; i += blockDim.x) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

// ---------------------------------------------------------------------------
// onesweep LSD radix pass (stable)
// status word: bits 31..30 flag (1 aggregate, 2 inclusive), bits 29..0 count
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSortThreads)
k_sort_pass(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
            uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
            const int64_t* __restrict__ scalars, int shift,
            const uint32_t* __restrict__ ghist, uint32_t* __restrict__ status,
            uint32_t* __restrict__ tile_ctr) {
    constexpr int NW = kSortThreads / 32;
    __shared__ uint32_t s_w[NW][kSortBins];
    __shared__ uint32_t s_goff[kSortBins];
    __shared__ uint32_t s_wsum[NW];
    __shared__ int s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
    for (int i = tid; i < NW * kSortBins; i += kSortThreads) (&s_w[0][0])[i] = 0;
    const int64_t n = scalars[3];
    __syncthreads();
    const int tile = s_tile;
    const int64_t tbase = (int64_t)tile * kSortTile;
    if (tbase >= n) return;
    // global digit starts: exclusive scan of ghist over 256 digits
    {
        uint32_t v = ghist[tid];
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; w++) wp += s_wsum[w];
        s_goff[tid] = wp + x - v;
    }
    const int64_t wbase = tbase + (int64_t)warp * 32 * kSortItems;
    uint32_t k[kSortItems];
    int32_t v[kSortItems];
    uint32_t rk[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const int64_t i = wbase + j * 32 + lane;
        const bool ok = i < n;
        k[j] = ok ? kin[i] : 0u;
        v[j] = ok ? vin[i] : 0;
        const uint32_t d = ok ? ((k[j] >> shift) & (kSortBins - 1)) : kSortBins;
        const uint32_t peers = match_label<kSortBits + 1>(d);
        const uint32_t lt = __popc(peers & lanemask_lt());
        uint32_t cnt = 0;
        if (ok) cnt = s_w[warp][d];
        __syncwarp();
        if (ok && lt == 0) s_w[warp][d] = cnt + __popc(peers);
        __syncwarp();
        rk[j] = cnt + lt;
    }
    __syncthreads();
    {
        const int d = tid;  // kSortThreads == kSortBins
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) {
            const uint32_t c = s_w[w][d];
            s_w[w][d] = tot;
            tot += c;
        }
        uint32_t excl = 0;
        uint32_t* st = status + (int64_t)tile * kSortBins + d;
        if (tile == 0) {
            st_relaxed_u32(st, (2u << 30) | tot);
        } else {
            st_relaxed_u32(st, (1u << 30) | tot);
            int t = tile - 1;
            while (true) {
                uint32_t s;
                do {
                    s = ld_relaxed_u32(status + (int64_t)t * kSortBins + d);
                } while ((s >> 30) == 0);
                excl += s & 0x3FFFFFFFu;
                if ((s >> 30) == 2) break;
                --t;
            }
            st_relaxed_u32(st, (2u << 30) | (excl + tot));
        }
        s_goff[d] += excl;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const int64_t i = wbase + j * 32 + lane;
        if (i < n) {
            const uint32_t d = (k[j] >> shift) & (kSortBins - 1);
            const uint32_t pos = s_goff[d] + s_w[warp][d] + rk[j];
            kout[pos] = k[j];
            vout[pos] = v[j];
        }
    }
}

// ---------------------------------------------------------------------------
// pieces: segment heads and piece starts over the sorted keys
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSortThreads)
k_pieces(const uint32_t* __restrict__ keys, int64_t* __restrict__ scalars,
         uint64_t* __restrict__ status, uint32_t* __restrict__ tile_ctr,
         int32_t* __restrict__ piece_start, int32_t* __restrict__ piece_seg,
         int32_t* __restrict__ seg_first, int32_t* __restrict__ seg_row) {
    constexpr int NW = kSortThreads / 32;
    __shared__ uint64_t s_wsum[NW];
    __shared__ int64_t s_wmax[NW];
    __shared__ int64_t s_carry;
    __shared__ uint64_t s_texcl;
    __shared__ int s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int tile = s_tile;
    const int64_t nv = scalars[0];
    const int64_t tbase = (int64_t)tile * kSortTile;
    if (tbase >= nv && !(tile == 0 && nv == 0)) return;
    const int64_t i0 = tbase + (int64_t)tid * kSortItems;
    uint32_t kk[kSortItems + 1];
    kk[0] = (i0 > 0 && i0 - 1 < nv) ? keys[i0 - 1] : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) kk[j + 1] = (i0 + j < nv) ? keys[i0 + j] : 0xFFFFFFFFu;
    // pieces split relative to the segment start (see k_gs_pieces)
    if (tid == 0) {
        int64_t cs = tbase;
        if (tbase > 0 && tbase < nv && keys[tbase - 1] == keys[tbase]) {
            const uint32_t kv = keys[tbase];
            int64_t lo = 0, hi = tbase - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (keys[mid] < kv) lo = mid + 1;
                else hi = mid;
            }
            cs = lo;
        }
        s_carry = cs;
    }
    int64_t lasthead = -1;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const int64_t i = i0 + j;
        if (i < nv && (i == 0 || kk[j + 1] != kk[j])) lasthead = i;
    }
    {
        int64_t xm = lasthead;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, xm, o);
            if (lane >= o) xm = y > xm ? y : xm;
        }
        if (lane == 31) s_wmax[warp] = xm;
        __syncthreads();
        int64_t before = -1;
        for (int w = 0; w < warp; w++) before = s_wmax[w] > before ? s_wmax[w] : before;
        const int64_t xe = __shfl_up_sync(0xffffffffu, xm, 1);
        if (lane > 0) before = xe > before ? xe : before;
        lasthead = before >= 0 ? before : s_carry;
    }
    uint32_t np = 0, ns = 0;
    bool isps[kSortItems], ishd[kSortItems];
    {
        int64_t segstart = lasthead;
#pragma unroll
        for (int j = 0; j < kSortItems; j++) {
            const int64_t i = i0 + j;
            ishd[j] = isps[j] = false;
            if (i < nv) {
                const bool head = (i == 0) || (kk[j + 1] != kk[j]);
                if (head) segstart = i;
                ishd[j] = head;
                isps[j] = head || ((i - segstart) % kPiece == 0);
                ns += ishd[j];
                np += isps[j];
            }
        }
    }
    const uint64_t mine = ((uint64_t)np << 31) | ns;
    uint64_t x = mine;
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint64_t wp = 0, tot = 0;
    for (int w = 0; w < NW; w++) {
        if (w < warp) wp += s_wsum[w];
        tot += s_wsum[w];
    }
    if (tid == 0) {
        const uint64_t ex = lookback_u64(status, tile, tot);
        s_texcl = ex;
        const int64_t last_tile = nv > 0 ? (nv - 1) / kSortTile : 0;
        if (tile == last_tile) {
            const uint64_t inc = ex + tot;
            const int64_t P_total = (int64_t)(inc >> 31);
            const int64_t S_total = (int64_t)(inc & 0x7FFFFFFFu);
            scalars[1] = P_total;
            scalars[2] = S_total;
            piece_start[P_total] = (int32_t)nv;
            seg_first[S_total] = (int32_t)P_total;
        }
    }
    __syncthreads();
    const uint64_t ex = s_texcl + wp + x - mine;
    int64_t pb = (int64_t)(ex >> 31);
    int64_t sb = (int64_t)(ex & 0x7FFFFFFFu);
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const int64_t i = i0 + j;
        if (i < nv) {
            const bool head = ishd[j];
            const bool ps = isps[j];
            if (head) {
                seg_first[sb] = (int32_t)pb;
                seg_row[sb] = (int32_t)kk[j + 1];
                sb++;
            }
            if (ps) {
                piece_start[pb] = (int32_t)i;
                piece_seg[pb] = (int32_t)(sb - 1);
                pb++;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// segment reduce + SGD (or emit)
// ---------------------------------------------------------------------------
template <int LPB, int NV>
__global__ void __launch_bounds__(256)
k_seg_reduce(const int32_t* __restrict__ vals, const int64_t* __restrict__ scalars,
             const int32_t* __restrict__ piece_start, const int32_t* __restrict__ piece_seg,
             const int32_t* __restrict__ seg_first, const int32_t* __restrict__ seg_row,
             const float* __restrict__ src, int D, float* W, float lr, float* partial,
             uint32_t* seg_cnt, int emit, float* grad_out, uint32_t* err) {
    reduce_pieces<LPB, NV, int32_t>(0, scalars[1], 0, 0, vals, piece_start, piece_seg, seg_first,
                                    seg_row, src, D, W, lr, partial, seg_cnt, emit, grad_out, err);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <int LPB, int NV>
static void launch_fwd(Ctx* c, const float* W, int64_t H, int D, const int32_t* idx,
                       const int64_t* off, int P, int64_t n_bags, float* Y) {
    const int threads = 256;
    // bags per block: one per lane group, or one per warp for multi-hot bags
    const int64_t gpb = (off || P >= kWarpBagMinP) ? threads / 32 : threads / LPB;
    int64_t blocks = cdiv(n_bags, gpb);
    const int64_t maxb = (int64_t)sm_count(c) * 16;
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    k_emb_fwd<LPB, NV><<<(unsigned)blocks, threads, 0, c->stream>>>(W, H, D, idx, off, P, n_bags, Y, c->d_err);
}

template <int LPB, int NV>
static void launch_reduce(Ctx* c, int64_t n_items_hint, const float* src, int D, float* W,
                          float lr, bool emit) {
    StepWs& w = c->ws;
    const int threads = 256;
    const int64_t gpb = threads / LPB;
    const int64_t pieces_hint = n_items_hint + n_items_hint / kPiece + 1;
    int64_t blocks = cdiv(pieces_hint, gpb);
    const int64_t maxb = (int64_t)sm_count(c) * 16;
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    k_seg_reduce<LPB, NV><<<(unsigned)blocks, threads, 0, c->stream>>>(
        w.vals[0], w.scalars, w.piece_start, w.piece_seg, w.seg_first, w.seg_row, src, D, W, lr,
        w.partial, w.seg_cnt, emit ? 1 : 0, w.grad, c->d_err);
}

static int key_bits(int64_t H) {
    // keys in [0, H] (H marks invalid lookups)
    int b = 1;
    while (b < 32 && ((uint64_t)1 << b) <= (uint64_t)H) b++;
    return b;
}

// Sort (keys, vals) already in ws.keys[0]/vals[0] (prep done), then pieces and
// reduce.  Result of the sort lands back in buffer 0 (even passes) — we track
// which buffer holds it and swap pointers so vals[0] is sorted on exit.
static fae_status sort_pieces_reduce(Ctx* c, int64_t n_hint, int64_t H, int D, const float* src,
                                     float* W, float lr, bool emit) {
    StepWs& w = c->ws;
    const int passes = (key_bits(H) + kSortBits - 1) / kSortBits;
    const int64_t tiles = std::max<int64_t>(1, cdiv(n_hint, kSortTile));
    for (int ps = 0; ps < passes; ps++) {
        const int s = ps & 1;
        k_sort_pass<<<(unsigned)tiles, kSortThreads, 0, c->stream>>>(
            w.keys[s], w.vals[s], w.keys[s ^ 1], w.vals[s ^ 1], w.scalars, ps * kSortBits,
            w.ghist + ps * kSortBins, w.sort_status + (int64_t)ps * w.n_sort_tiles * kSortBins,
            w.tile_ctr + ps);
        FAE_LAUNCHED(c);
    }
    if (passes & 1) {
        std::swap(w.keys[0], w.keys[1]);
        std::swap(w.vals[0], w.vals[1]);
    }
    k_pieces<<<(unsigned)tiles, kSortThreads, 0, c->stream>>>(
        w.keys[0], w.scalars, w.piece_status, w.tile_ctr + 4, w.piece_start, w.piece_seg,
        w.seg_first, w.seg_row);
    FAE_LAUNCHED(c);
    FAE_DISPATCH_D(D, launch_reduce, c, n_hint, src, D, W, lr, emit);
    FAE_LAUNCHED(c);
    return FAE_OK;
}

static fae_status zero_ws(Ctx* c, int64_t n_hint) {
    StepWs& w = c->ws;
    // ghist, counters, scalars and the used look-back status prefix
    const int64_t tiles = std::max<int64_t>(1, cdiv(n_hint, kSortTile));
    FAE_CUDA(c, cudaMemsetAsync(w.ghist, 0, sizeof(uint32_t) * kMaxSortPasses * kSortBins, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(w.tile_ctr, 0, sizeof(uint32_t) * 8, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(w.scalars, 0, sizeof(int64_t) * 8, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(w.piece_status, 0, sizeof(uint64_t) * tiles, c->stream));
    for (int ps = 0; ps < kMaxSortPasses; ps++)
        FAE_CUDA(c, cudaMemsetAsync(w.sort_status + (int64_t)ps * w.n_sort_tiles * kSortBins, 0,
                                    sizeof(uint32_t) * tiles * kSortBins, c->stream));
    return FAE_OK;
}

fae_status bwd_group_and_reduce(Ctx* c, float* W_hot, int64_t H, int32_t D,
                                const uint32_t* /*unused*/, const int32_t* idx,
                                const int64_t* off, int32_t P, int64_t n_bags, int64_t n_hint,
                                const float* dY, float lr, bool emit) {
    StepWs& w = c->ws;
    fae_status st = zero_ws(c, n_hint);
    if (st != FAE_OK) return st;
    const int passes = (key_bits(H) + kSortBits - 1) / kSortBits;
    int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(n_hint, 256), (int64_t)sm_count(c) * 8));
    k_bwd_prep<<<(unsigned)blocks, 256, 0, c->stream>>>(idx, off, P, n_bags, H, passes,
                                                        std::min<int64_t>(n_hint, w.cap_L), w.keys[0],
                                                        w.vals[0], w.ghist, w.scalars, c->d_err);
    FAE_LAUNCHED(c);
    return sort_pieces_reduce(c, n_hint, H, D, dY, W_hot, lr, emit);
}

static fae_status validate_step(Ctx* c, const float* W, int64_t H, int32_t D, const int32_t* idx,
                                const int64_t* off, int32_t P, int64_t n_bags, const float* X,
                                const char* who) {
    if ((!W || !X || !idx) && n_bags > 0) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": null pointer");
    if (H < 0 || H >= (1ll << 31) - 1) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": H out of range");
    if (!dim_ok(D) || D > c->cfg.max_dim) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": unsupported dim");
    if (n_bags < 0 || (!off && P < 0)) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": bad sizes");
    if (n_bags > c->cfg.max_batch_bags) return set_err(c, FAE_ERR_CAPACITY, std::string(who) + ": n_bags > max_batch_bags");
    if (!off && n_bags * (int64_t)P > c->cfg.max_batch_lookups)
        return set_err(c, FAE_ERR_CAPACITY, std::string(who) + ": lookups > max_batch_lookups");
    if (n_bags > 0 && (((uintptr_t)W | (uintptr_t)X) & 15)) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": W/Y must be 16-byte aligned");
    return FAE_OK;
}

}  // namespace fae

using namespace fae;

extern "C" {

fae_status fae_emb_fwd(fae_ctx* h, const float* W_hot, int64_t H, int32_t D, const int32_t* idx,
                       const int64_t* off, int32_t fixed_pool, int64_t n_bags, float* Y) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_step(c, W_hot, H, D, idx, off, fixed_pool, n_bags, Y, "fae_emb_fwd");
    if (st != FAE_OK) return st;
    if (n_bags == 0) return FAE_OK;
    FAE_DISPATCH_D(D, launch_fwd, c, W_hot, H, D, idx, off, fixed_pool, n_bags, Y);
    FAE_LAUNCHED(c);
    return FAE_OK;
}

fae_status fae_emb_bwd_update(fae_ctx* h, float* W_hot, int64_t H, int32_t D, const int32_t* idx,
                              const int64_t* off, int32_t fixed_pool, int64_t n_bags,
                              const float* dY, float lr) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_step(c, W_hot, H, D, idx, off, fixed_pool, n_bags, dY, "fae_emb_bwd_update");
    if (st == FAE_OK && !(lr == lr)) st = set_err(c, FAE_ERR_INVALID_ARG, "fae_emb_bwd_update: lr is NaN");
    const bool multi = c->world > 1;
    if (multi) st = coll_agree(c, st, "fae_emb_bwd_update");   // no peer left blocked in the exchange
    if (st != FAE_OK) return st;
    const int64_t n_hint = off ? c->cfg.max_batch_lookups : n_bags * (int64_t)fixed_pool;
    if (n_bags == 0 && !multi) return FAE_OK;
    st = bwd_group_and_reduce(c, W_hot, H, D, nullptr, idx, off, fixed_pool, n_bags, n_hint, dY, lr, multi);
    if (st != FAE_OK || !multi) return st;
    // a11: exchange the local sparse gradient, merge deterministically, apply
    int64_t U = 0;
    FAE_CUDA(c, cudaMemcpyAsync(&U, c->ws.scalars + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    // rows are ws.seg_row[0..U), grads ws.grad[0..U)
    return sync_merge_apply(c, c->ws.seg_row, c->ws.grad, U, D, W_hot, H, lr, nullptr, nullptr, nullptr, 0);
}

}  // extern "C"

namespace fae {

// Rank-ordered merge of the gathered sorted lists (no re-sort): block r of
// g_rows / g_vals holds rank r's counts[r] (row, G) entries, rows ascending
// and unique within a rank.  The lane group of entry (r, j) owns row x iff no
// lower rank holds x (binary search in each lower list); the owner sums
// 0 + G_r + G_{r'} + ... over the ranks r' > r holding x, in rank order — the
// order the sort-based merge uses (one piece of <= world terms), so the
// result is identical on every rank and to the single-rank step — and
// applies W[x] = fmaf(-lr, G, W[x]).
__device__ __forceinline__ int64_t find_row(const int32_t* __restrict__ rows, int64_t n, int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(rows + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && __ldg(rows + lo) == x ? lo : -1;
}

template <int LPB, int NV>
__global__ void __launch_bounds__(256)
k_merge_apply(const int32_t* __restrict__ g_rows, const float* __restrict__ g_vals,
              const int32_t* __restrict__ counts, int world, int64_t cap, int D, float* W, float lr,
              uint32_t* err) {
    const int lane = threadIdx.x % LPB;
    const int64_t gpb = blockDim.x / LPB;
    const int64_t n = cap * world;
    for (int64_t e = blockIdx.x * gpb + threadIdx.x / LPB; e < n; e += (int64_t)gridDim.x * gpb) {
        const int r = (int)(e / cap);
        const int64_t j = e - (int64_t)r * cap;
        if (j >= counts[r]) continue;
        const int32_t x = __ldg(g_rows + e);
        bool owner = true;
        for (int q = 0; q < r && owner; q++)
            if (find_row(g_rows + (int64_t)q * cap, counts[q], x) >= 0) owner = false;
        if (!owner) continue;
        float4 acc[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = r; q < world; q++) {
            const int64_t t = q == r ? j : find_row(g_rows + (int64_t)q * cap, counts[q], x);
            if (t < 0) continue;
            const float4* v = reinterpret_cast<const float4*>(g_vals + ((int64_t)q * cap + t) * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) add4(acc[k], __ldg(v + k * LPB));
        }
        float4* w = reinterpret_cast<float4*>(W + (int64_t)x * D) + lane;
        bool bad = false;
#pragma unroll
        for (int k = 0; k < NV; k++) {
            float4 y = w[k * LPB];
            y.x = __fmaf_rn(-lr, acc[k].x, y.x);
            y.y = __fmaf_rn(-lr, acc[k].y, y.y);
            y.z = __fmaf_rn(-lr, acc[k].z, y.z);
            y.w = __fmaf_rn(-lr, acc[k].w, y.w);
            bad |= !(isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w));
            w[k * LPB] = y;
        }
        if (bad) atomicOr(err, kErrNonfinite);
    }
}

template <int LPB, int NV>
static fae_status launch_merge_apply(Ctx* c, const int32_t* counts, int64_t cap, int D, float* W, float lr) {
    const int64_t gpb = 256 / LPB;
    const int64_t n = cap * c->world;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, gpb), (int64_t)sm_count(c) * 16));
    k_merge_apply<LPB, NV><<<(unsigned)blocks, 256, 0, c->stream>>>(c->g_rows, c->g_vals, counts, c->world, cap, D,
                                                                    W, lr, c->d_err);
    FAE_LAUNCHED(c);
    return FAE_OK;
}

static fae_status merge_apply(Ctx* c, const int32_t* counts, int64_t cap, int D, float* W, float lr) {
    FAE_DISPATCH_D(D, return launch_merge_apply, c, counts, cap, D, W, lr);
    return FAE_OK;
}

// Gather every rank's sorted (row, G) list, merge in rank order and either
// apply SGD to W (W != nullptr) or write the merged list to out_rows/out_vals.
// known_counts (optional, device [world]) + known_cap: the per-rank counts of
// this exchange are already on the device and their maximum on the host (the
// training loop exchanges every step's counts once up front), so there is no
// count all-gather and no host synchronisation here when W != nullptr.
fae_status sync_merge_apply(Ctx* c, const int32_t* rows, const float* vals, int64_t U, int32_t D,
                            float* W, int64_t H, float lr, int32_t* out_rows, float* out_vals,
                            int64_t* out_count, int64_t out_cap, const int32_t* known_counts,
                            int64_t known_cap) {
    if (!has_comm(c)) return set_err(c, FAE_ERR_NOT_INIT, "sync: no communicator");
    const int world = c->world;
    int64_t cap = 0;
    const int32_t* dcounts = known_counts;
    if (!known_counts) {
        // 1. counts (a local U beyond capacity is exchanged as-is: every rank
        //    then sees the same maximum and returns the same error below)
        const int32_t Ui = (int32_t)std::min<int64_t>(U, INT32_MAX);
        FAE_CUDA(c, cudaMemcpyAsync(c->g_counts + c->rank, &Ui, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
        fae_status cs = coll_allgather(c, c->g_counts + c->rank, c->g_counts, 1, CollT::I32, "sync: allgather counts");
        if (cs != FAE_OK) return cs;
        std::vector<int32_t> counts(world);
        FAE_CUDA(c, cudaMemcpyAsync(counts.data(), c->g_counts, sizeof(int32_t) * world, cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        for (int i = 0; i < world; i++) cap = std::max<int64_t>(cap, counts[i]);
        dcounts = c->g_counts;
    } else {
        cap = known_cap;
    }
    if (cap == 0) {
        if (out_count) *out_count = 0;
        return FAE_OK;
    }
    if (cap > c->g_cap) return set_err(c, FAE_ERR_CAPACITY, "sync: a rank's U exceeds capacity");
    if (cap * world > c->ws.cap_L) return set_err(c, FAE_ERR_CAPACITY, "sync: gathered size exceeds workspace");
    // 2. padded payloads (rows, vals) — grouped all-gathers
    int32_t* my_rows = c->g_rows + (int64_t)c->rank * cap;
    float* my_vals = c->g_vals + (int64_t)c->rank * cap * D;
    if (U > 0) {
        FAE_CUDA(c, cudaMemcpyAsync(my_rows, rows, sizeof(int32_t) * U, cudaMemcpyDeviceToDevice, c->stream));
        FAE_CUDA(c, cudaMemcpyAsync(my_vals, vals, sizeof(float) * U * D, cudaMemcpyDeviceToDevice, c->stream));
    }
    {
        coll_group_start(c);
        fae_status a = coll_allgather(c, my_rows, c->g_rows, cap, CollT::I32, "sync: allgather rows");
        if (a == FAE_OK) a = coll_allgather(c, my_vals, c->g_vals, cap * D, CollT::F32, "sync: allgather grads");
        fae_status b = coll_group_end(c, "sync: allgather payload");
        if (a != FAE_OK) return a;
        if (b != FAE_OK) return b;
    }
    // 3. deterministic merge.  Applying to W: the rank-ordered merge of the
    //    sorted lists (one kernel).  Emitting the merged list: a stable sort by
    //    row over the rank-ordered concatenation, segment sums in fixed order.
    fae_status st = FAE_OK;
    if (W && !c->merge_sort) {
        st = merge_apply(c, dcounts, cap, D, W, lr);
        if (st != FAE_OK) return st;
        return coll_async_error(c, "sync");
    }
    const int64_t n = cap * world;
    st = zero_ws(c, n);
    if (st != FAE_OK) return st;
    int64_t Hk = H;
    if (!W) {
        // emit mode: key range from the rows themselves (< 2^31)
        Hk = (1ll << 31) - 2;
    }
    const int passes = (key_bits(Hk) + kSortBits - 1) / kSortBits;
    int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sm_count(c) * 8));
    k_merge_prep<<<(unsigned)blocks, 256, 0, c->stream>>>(c->g_rows, dcounts, world, cap, Hk, passes,
                                                          c->ws.keys[0], c->ws.vals[0], c->ws.ghist,
                                                          c->ws.scalars);
    FAE_LAUNCHED(c);
    st = sort_pieces_reduce(c, n, Hk, D, c->g_vals, W, lr, W == nullptr);
    if (st != FAE_OK) return st;
    if (!W) {
        int64_t Ug = 0;
        FAE_CUDA(c, cudaMemcpyAsync(&Ug, c->ws.scalars + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        if (Ug > out_cap) return set_err(c, FAE_ERR_CAPACITY, "sync: global U exceeds cap");
        FAE_CUDA(c, cudaMemcpyAsync(out_rows, c->ws.seg_row, sizeof(int32_t) * Ug, cudaMemcpyDeviceToDevice, c->stream));
        FAE_CUDA(c, cudaMemcpyAsync(out_vals, c->ws.grad, sizeof(float) * Ug * D, cudaMemcpyDeviceToDevice, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        *out_count = Ug;
    }
    return coll_async_error(c, "sync");
}

}  // namespace fae

extern "C" fae_status fae_sync_hot_grads(fae_ctx* h, int32_t* rows, float* vals, int64_t* count_host,
                                         int64_t cap, int32_t D) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    if (!rows || !vals || !count_host || cap < 0 || !dim_ok(D) || D > c->cfg.max_dim)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_sync_hot_grads: bad arguments");
    if (*count_host < 0 || *count_host > cap)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_sync_hot_grads: count outside [0, cap]");
    if (c->world == 1 && !has_comm(c)) return FAE_OK;   // identity
    return sync_merge_apply(c, rows, vals, *count_host, D, nullptr, 0, 0.f, rows, vals, count_host, cap);
}
