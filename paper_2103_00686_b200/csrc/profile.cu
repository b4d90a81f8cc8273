// profile.cu — input sampler + embedding logger.
//
//  a1  P:L358-363 (§4.1.1): x% of the records, uniform without replacement
//      (R6): the k = floor(R*x/100) records with the smallest
//      (key(seed, i), i), output in ascending record order.
//      B200 design: no sort of R keys.  An MSD radix SELECT over the 64-bit
//      keys (8-bit digits, one 256-bin histogram pass per level, keys
//      recomputed on the fly, nothing stored) finds the k-th smallest
//      (key, i) pair; a single look-back compaction pass then emits the
//      selected ids in ascending order.  With a comm the per-level
//      histograms are all-reduced, so a sharded profile selects exactly the
//      records an unsharded one would.
//  a2  P:L380-388 (§4.1.2 "Embedding Logger"): counts[rowbase_z + j] = number
//      of sampled lookups of row j of table z.  Warp per sampled record,
//      __match_any_sync aggregation of equal rows before one atomicAdd.
#include <algorithm>
#include <cmath>

#include "fae_internal.cuh"

namespace fae {

constexpr int kCandCap = 4096;
constexpr int kSelThreads = 256;
constexpr int kSelItems = 16;
constexpr int kSelTile = kSelThreads * kSelItems;

__global__ void __launch_bounds__(256)
k_sel_hist(int64_t n, int64_t gbase, uint64_t seed, uint64_t prefix, int pbits,
           uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[256];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const int shift = 56 - pbits;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = hash_key(seed, (uint64_t)(gbase + i));
        if (pbits == 0 || (k >> (64 - pbits)) == prefix) atomicAdd(&sh[(k >> shift) & 255], 1u);
    }
    __syncthreads();
    if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

// candidates: keys whose top pbits equal prefix -> (key, global id)
__global__ void __launch_bounds__(256)
k_sel_gather(int64_t n, int64_t gbase, uint64_t seed, uint64_t prefix, int pbits,
             unsigned long long* __restrict__ ck, long long* __restrict__ ci,
             uint32_t* __restrict__ cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = hash_key(seed, (uint64_t)(gbase + i));
        if (pbits == 0 || (pbits == 64 ? k == prefix : (k >> (64 - pbits)) == prefix)) {
            const uint32_t s = atomicAdd(cnt, 1u);
            if (s < kCandCap) {
                ck[s] = k;
                ci[s] = gbase + i;
            }
        }
    }
}

// one block: the candidate of rank `need-1` (0-based) among n_c candidates,
// ordered by (key, id).  O(n_c^2) rank counting — n_c <= kCandCap * world.
__global__ void __launch_bounds__(1024)
k_sel_pick(const unsigned long long* __restrict__ ck, const long long* __restrict__ ci, int n_c,
           int64_t need, unsigned long long* out_key, long long* out_id) {
    for (int a = threadIdx.x; a < n_c; a += blockDim.x) {
        const unsigned long long ka = ck[a];
        const long long ia = ci[a];
        int64_t r = 0;
        for (int b = 0; b < n_c; b++) {
            const unsigned long long kb = ck[b];
            r += (kb < ka) || (kb == ka && ci[b] < ia);
        }
        if (r == need - 1) {
            *out_key = ka;
            *out_id = ia;
        }
    }
}

// selected(i) <=> (key, gid) <= (tkey, tid); mode 0: none, 1: all, 2: threshold
__global__ void __launch_bounds__(kSelThreads)
k_sel_compact(int64_t n, int64_t gbase, uint64_t seed, const unsigned long long* tkey,
              const long long* tidp, int mode, uint64_t* __restrict__ status,
              uint32_t* __restrict__ ctr, int64_t* __restrict__ out_ids, int64_t* total) {
    __shared__ int s_tile;
    __shared__ uint32_t s_wsum[kSelThreads / 32];
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t tbase = tile * kSelTile;
    if (tbase >= n && !(tile == 0)) return;
    const unsigned long long tk = mode == 2 ? *tkey : 0ull;
    const long long ti = mode == 2 ? *tidp : 0ll;
    const int64_t i0 = tbase + (int64_t)tid * kSelItems;
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < kSelItems; j++) {
        const int64_t i = i0 + j;
        if (i < n) {
            bool sel;
            if (mode == 1) sel = true;
            else if (mode == 0) sel = false;
            else {
                const uint64_t k = hash_key(seed, (uint64_t)(gbase + i));
                sel = (k < tk) || (k == tk && (long long)(gbase + i) <= ti);
            }
            m |= (uint32_t)sel << j;
        }
    }
    const uint32_t c = __popc(m);
    uint32_t x = c;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t wp = 0, tot = 0;
    for (int w = 0; w < kSelThreads / 32; w++) {
        if (w < warp) wp += s_wsum[w];
        tot += s_wsum[w];
    }
    if (tid == 0) {
        s_ex = lookback_u64(status, tile, tot);
        const int64_t last = n > 0 ? (n - 1) / kSelTile : 0;
        if (tile == last) *total = (int64_t)(s_ex + tot);
    }
    __syncthreads();
    int64_t pos = (int64_t)s_ex + wp + x - c;
#pragma unroll
    for (int j = 0; j < kSelItems; j++)
        if ((m >> j) & 1u) out_ids[pos++] = i0 + j;
}

// warp per sampled record
__global__ void __launch_bounds__(256)
k_histogram(const int64_t* __restrict__ sampled, int64_t n_s, const int32_t* __restrict__ idx,
            const int64_t* __restrict__ off, int P, int Tn, const int64_t* __restrict__ rowbase,
            const int64_t* __restrict__ rows, uint32_t* __restrict__ counts, uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const int64_t wpb = blockDim.x >> 5;
    for (int64_t w = blockIdx.x * wpb + (threadIdx.x >> 5); w < n_s; w += (int64_t)gridDim.x * wpb) {
        const int64_t r = sampled[w];
        int64_t start, len;
        int64_t myoff = 0;
        if (off) {
            start = off[r * Tn];
            len = off[r * Tn + Tn] - start;
            if (Tn <= 31 && lane <= Tn) myoff = off[r * Tn + lane] - start;
        } else {
            start = r * (int64_t)Tn * P;
            len = (int64_t)Tn * P;
        }
        for (int64_t b0 = 0; b0 < len; b0 += 32) {
            const int64_t q = b0 + lane;
            const bool act = q < len;
            uint64_t key = ~(uint64_t)lane;   // unique sentinel
            int z = 0;
            if (!off) {
                z = act ? (int)(q / P) : 0;
            } else if (Tn <= 31) {
                // bag of lookup q: count bag starts (held by lanes 1..Tn-1) <= q
                for (int t = 1; t < Tn; t++) z += (__shfl_sync(0xffffffffu, myoff, t) <= q);
            } else if (act) {
                int lo = 0, hi = Tn - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (off[r * Tn + mid] - start <= q) lo = mid;
                    else hi = mid - 1;
                }
                z = lo;
            }
            if (act) {
                const int32_t j = idx[start + q];
                if (j < 0 || (int64_t)j >= __ldg(rows + z)) atomicOr(err, kErrIndex);
                else key = (uint64_t)(__ldg(rowbase + z) + j);
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            if (act && (key >> 63) == 0 && (__ffs(peers) - 1) == lane)
                atomicAdd(&counts[key], (uint32_t)__popc(peers));
        }
    }
}

// fixed pooling: thread per sampled lookup, 8 in flight; rows of tiny tables
// (tiny_off[z] >= 0) count in shared memory (one flush per block), the others
// in global memory with warp match_any aggregation.
constexpr int kTinySlots = 8192;
__global__ void __launch_bounds__(256)
k_histogram_fixed(const int64_t* __restrict__ sampled, int64_t n_s, const int32_t* __restrict__ idx,
                  int P, int Tn, const int64_t* __restrict__ rowbase, const int64_t* __restrict__ rows,
                  const int32_t* __restrict__ tiny_off, const int64_t* __restrict__ slot_row, int n_slots,
                  uint32_t* __restrict__ counts, uint32_t* err) {
    __shared__ uint32_t tiny[kTinySlots];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < n_slots; i += blockDim.x) tiny[i] = 0;
    __syncthreads();
    const int TnP = Tn * P;
    const int64_t n = n_s * TnP;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    // the sampled records are read once (evict-first): L2 keeps the counters
    // of the Zipf heads that the atomics hit again and again
    const uint64_t pol = l2_policy_evict_first();
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x * 8; i0 < n; i0 += stride) {
        int32_t jv[8];
        int zv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
            zv[u] = -1;
            jv[u] = 0;
            if (i < n) {
                const int64_t rs = i / TnP;
                const int qq = (int)(i - rs * TnP);
                zv[u] = qq / P;
                jv[u] = ldg_hint_i32(idx + __ldg(sampled + rs) * TnP + qq, pol);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            uint64_t key = ~(uint64_t)lane;   // unique sentinel: not counted globally
            const int z = zv[u];
            if (z >= 0) {
                const int32_t j = jv[u];
                if (j < 0 || (int64_t)j >= __ldg(rows + z)) {
                    atomicOr(err, kErrIndex);
                } else {
                    const int32_t to = __ldg(tiny_off + z);
                    if (to >= 0) atomicAdd(&tiny[to + j], 1u);
                    else key = (uint64_t)(__ldg(rowbase + z) + j);
                }
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            if ((key >> 63) == 0 && (__ffs(peers) - 1) == lane) atomicAdd(&counts[key], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_slots; i += blockDim.x)
        if (tiny[i]) atomicAdd(&counts[slot_row[i]], tiny[i]);
}

// T_z for offsets datasets: per-table lookup totals
__global__ void __launch_bounds__(256)
k_table_totals(const int64_t* __restrict__ off, int64_t n_bags, int Tn,
               unsigned long long* __restrict__ T) {
    extern __shared__ unsigned long long sT[];
    for (int z = threadIdx.x; z < Tn; z += blockDim.x) sT[z] = 0;
    __syncthreads();
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_bags;
         b += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&sT[b % Tn], (unsigned long long)(off[b + 1] - off[b]));
    __syncthreads();
    for (int z = threadIdx.x; z < Tn; z += blockDim.x)
        if (sT[z]) atomicAdd(&T[z], sT[z]);
}

static int sms(Ctx* c) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, c->device);
    return n;
}

fae_status upload_schema(Ctx* c, const fae_tables* t, std::vector<int64_t>& rowbase) {
    rowbase.assign(t->n_tables + 1, 0);
    for (int z = 0; z < t->n_tables; z++) rowbase[z + 1] = rowbase[z] + t->rows[z];
    FAE_CUDA(c, cudaMemcpyAsync(c->d_rowbase_tmp, rowbase.data(), sizeof(int64_t) * (t->n_tables + 1),
                                cudaMemcpyHostToDevice, c->stream));
    FAE_CUDA(c, cudaMemcpyAsync(c->d_rows_tmp, t->rows, sizeof(int64_t) * t->n_tables,
                                cudaMemcpyHostToDevice, c->stream));
    return FAE_OK;
}

fae_status validate_schema(Ctx* c, const fae_tables* t, const char* who) {
    if (!t || !t->rows || t->n_tables < 1) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": bad table schema");
    if (t->n_tables > c->cfg.max_tables) return set_err(c, FAE_ERR_CAPACITY, std::string(who) + ": n_tables > max_tables");
    int64_t tot = 0;
    for (int z = 0; z < t->n_tables; z++) {
        if (t->rows[z] < 1 || t->rows[z] >= (1ll << 31)) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": table rows out of range");
        tot += t->rows[z];
    }
    if (tot > c->cfg.max_rows) return set_err(c, FAE_ERR_CAPACITY, std::string(who) + ": sum of rows > max_rows");
    if (t->dim < 1) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": dim < 1");
    return FAE_OK;
}

fae_status validate_csr(Ctx* c, const fae_tables* t, const fae_csr* d, const char* who) {
    if (!d || d->n_records < 0 || (d->n_records > 0 && !d->idx && d->n_lookups > 0) ||
        (!d->off && d->fixed_pool < 0))
        return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": bad csr");
    if (!d->off && d->n_lookups != d->n_records * (int64_t)t->n_tables * d->fixed_pool)
        return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": n_lookups != n_records*n_tables*fixed_pool");
    if (d->record_base < 0 || d->n_records_global < d->record_base + d->n_records)
        return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": bad record_base/n_records_global");
    return FAE_OK;
}

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_profile(fae_ctx* h, const fae_tables* tabs, const fae_csr* data,
                                  double x_pct, uint64_t seed, uint32_t* counts, int64_t* T_host,
                                  int64_t* sampled_ids, int64_t* n_sampled) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    const bool multi = c->world > 1 && has_comm(c);
    fae_status st = validate_schema(c, tabs, "fae_profile");
    if (st == FAE_OK) st = validate_csr(c, tabs, data, "fae_profile");
    if (st == FAE_OK && !(x_pct > 0.0 && x_pct <= 100.0))
        st = set_err(c, FAE_ERR_INVALID_ARG, "fae_profile: x must be in (0, 100]");
    if (st == FAE_OK && (!counts || !T_host || !n_sampled))
        st = set_err(c, FAE_ERR_INVALID_ARG, "fae_profile: null output");
    // with a comm every rank must take the same early exit (no peer left
    // blocked in a collective)
    if (multi) st = coll_agree(c, st, "fae_profile");
    if (st != FAE_OK) return st;
    const int Tn = tabs->n_tables;
    std::vector<int64_t> rowbase;
    st = upload_schema(c, tabs, rowbase);
    if (st != FAE_OK) return st;
    const int64_t total_rows = rowbase[Tn];
    const int64_t n = data->n_records;
    const int64_t Rg = data->n_records_global;
    const int64_t gbase = data->record_base;
    const int64_t k = (int64_t)std::floor((double)Rg * x_pct / 100.0);

    // scratch layout
    const int64_t tiles = std::max<int64_t>(1, cdiv(n, kSelTile));
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
    const size_t o_ids = take(sizeof(int64_t) * std::max<int64_t>(1, n));
    const size_t o_hist = take(sizeof(uint32_t) * 256);
    const size_t o_ck = take(sizeof(unsigned long long) * kCandCap * std::max(1, c->world));
    const size_t o_ci = take(sizeof(long long) * kCandCap * std::max(1, c->world));
    const size_t o_cnt = take(sizeof(uint32_t) * 8);
    const size_t o_tk = take(sizeof(unsigned long long) * 2);
    const size_t o_st = take(sizeof(uint64_t) * tiles);
    const size_t o_tot = take(sizeof(int64_t) * 2);
    const size_t o_T = take(sizeof(unsigned long long) * Tn);
    const size_t o_toff = take(sizeof(int32_t) * Tn);
    const size_t o_srow = take(sizeof(int64_t) * kTinySlots);
    char* sc = (char*)scratch(c, o);
    if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_profile: scratch allocation failed");
    int64_t* ids = (int64_t*)(sc + o_ids);
    uint32_t* hist = (uint32_t*)(sc + o_hist);
    unsigned long long* ck = (unsigned long long*)(sc + o_ck);
    long long* ci = (long long*)(sc + o_ci);
    uint32_t* ccnt = (uint32_t*)(sc + o_cnt);
    unsigned long long* tkey = (unsigned long long*)(sc + o_tk);
    long long* tidp = (long long*)(sc + o_tk + sizeof(unsigned long long));
    uint64_t* status = (uint64_t*)(sc + o_st);
    int64_t* d_total = (int64_t*)(sc + o_tot);
    unsigned long long* dT = (unsigned long long*)(sc + o_T);

    const int64_t gridn = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sms(c) * 8));
    int mode = 2;
    if (k >= Rg) mode = 1;
    else if (k <= 0) mode = 0;
    if (mode == 2) {
        // MSD radix select of the k-th smallest (key, id)
        uint64_t prefix = 0;
        int pbits = 0;
        int64_t need = k;
        uint32_t h_hist[256];
        int64_t cnt = Rg;
        while (pbits < 64 && cnt > kCandCap) {
            FAE_CUDA(c, cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256, c->stream));
            k_sel_hist<<<(unsigned)gridn, 256, 0, c->stream>>>(n, gbase, seed, prefix, pbits, hist);
            FAE_LAUNCHED(c);
            if (multi) {
                st = coll_allreduce_sum(c, hist, 256, CollT::U32, "fae_profile: allreduce hist");
                if (st != FAE_OK) return st;
            }
            FAE_CUDA(c, cudaMemcpyAsync(h_hist, hist, sizeof(h_hist), cudaMemcpyDeviceToHost, c->stream));
            FAE_CUDA(c, cudaStreamSynchronize(c->stream));
            int64_t cum = 0;
            int d = 0;
            for (; d < 256; d++) {
                if (cum + h_hist[d] >= need) break;
                cum += h_hist[d];
            }
            need -= cum;
            prefix = (prefix << 8) | (uint64_t)d;
            pbits += 8;
            cnt = h_hist[d];
        }
        // candidates of this rank go to slot `rank` (padded with all-ones);
        // with a comm the slots are all-gathered in place.
        const int W = multi ? c->world : 1;
        const int me = multi ? c->rank : 0;
        unsigned long long* myk = ck + (int64_t)me * kCandCap;
        long long* myi = ci + (int64_t)me * kCandCap;
        FAE_CUDA(c, cudaMemsetAsync(ccnt, 0, sizeof(uint32_t) * 8, c->stream));
        FAE_CUDA(c, cudaMemsetAsync(myk, 0xFF, sizeof(unsigned long long) * kCandCap, c->stream));
        FAE_CUDA(c, cudaMemsetAsync(myi, 0xFF, sizeof(long long) * kCandCap, c->stream));
        k_sel_gather<<<(unsigned)gridn, 256, 0, c->stream>>>(n, gbase, seed, prefix, pbits, myk, myi, ccnt);
        FAE_LAUNCHED(c);
        uint32_t n_c = 0;
        FAE_CUDA(c, cudaMemcpyAsync(&n_c, ccnt, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        st = n_c > (uint32_t)kCandCap ? set_err(c, FAE_ERR_CAPACITY, "fae_profile: selection candidates overflow")
                                      : FAE_OK;
        if (multi) st = coll_agree(c, st, "fae_profile: candidates");
        if (st != FAE_OK) return st;
        if (multi) {
            coll_group_start(c);
            st = coll_allgather(c, myk, ck, kCandCap, CollT::U64, "fae_profile: allgather candidate keys");
            if (st == FAE_OK) st = coll_allgather(c, myi, ci, kCandCap, CollT::I64, "fae_profile: allgather candidate ids");
            fae_status st2 = coll_group_end(c, "fae_profile: allgather candidates");
            if (st != FAE_OK) return st;
            if (st2 != FAE_OK) return st2;
        }
        const int n_all = multi ? W * kCandCap : (int)n_c;
        const unsigned long long* pk = ck;
        const long long* pi = ci;
        k_sel_pick<<<1, 1024, 0, c->stream>>>(pk, pi, n_all, need, tkey, tidp);
        FAE_LAUNCHED(c);
    }
    FAE_CUDA(c, cudaMemsetAsync(ccnt + 2, 0, sizeof(uint32_t), c->stream));
    FAE_CUDA(c, cudaMemsetAsync(status, 0, sizeof(uint64_t) * tiles, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(d_total, 0, sizeof(int64_t), c->stream));
    k_sel_compact<<<(unsigned)tiles, kSelThreads, 0, c->stream>>>(n, gbase, seed, tkey, tidp, mode, status,
                                                                 ccnt + 2, ids, d_total);
    FAE_LAUNCHED(c);
    int64_t ns = 0;
    FAE_CUDA(c, cudaMemcpyAsync(&ns, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));

    // a2 histogram
    FAE_CUDA(c, cudaMemsetAsync(counts, 0, sizeof(uint32_t) * total_rows, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (ns > 0 && !data->off && data->fixed_pool > 0) {
        // tiny tables (<= 2048 rows) privatised in shared memory, up to kTinySlots
        std::vector<int32_t> toff(Tn, -1);
        std::vector<int64_t> srow;
        for (int z = 0; z < Tn; z++)
            if (tabs->rows[z] <= 2048 && (int64_t)srow.size() + tabs->rows[z] <= kTinySlots) {
                toff[z] = (int32_t)srow.size();
                for (int64_t j = 0; j < tabs->rows[z]; j++) srow.push_back(rowbase[z] + j);
            }
        int32_t* d_toff = (int32_t*)(sc + o_toff);
        int64_t* d_srow = (int64_t*)(sc + o_srow);
        FAE_CUDA(c, cudaMemcpyAsync(d_toff, toff.data(), sizeof(int32_t) * Tn, cudaMemcpyHostToDevice, c->stream));
        if (!srow.empty())
            FAE_CUDA(c, cudaMemcpyAsync(d_srow, srow.data(), sizeof(int64_t) * srow.size(), cudaMemcpyHostToDevice, c->stream));
        const int64_t items = ns * (int64_t)Tn * data->fixed_pool;
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(items, 256 * 8), (int64_t)sms(c) * 4));
        k_histogram_fixed<<<(unsigned)g, 256, 0, c->stream>>>(ids, ns, data->idx, data->fixed_pool, Tn,
                                                              c->d_rowbase_tmp, c->d_rows_tmp, d_toff, d_srow,
                                                              (int)srow.size(), counts, c->d_err);
        FAE_LAUNCHED(c);
    } else if (ns > 0) {
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(ns, 8), (int64_t)sms(c) * 16));
        k_histogram<<<(unsigned)g, 256, 0, c->stream>>>(ids, ns, data->idx, data->off, data->fixed_pool, Tn,
                                                        c->d_rowbase_tmp, c->d_rows_tmp, counts, c->d_err);
        FAE_LAUNCHED(c);
    }
    // T_z
    std::vector<int64_t> T(Tn, 0);
    if (data->off) {
        FAE_CUDA(c, cudaMemsetAsync(dT, 0, sizeof(unsigned long long) * Tn, c->stream));
        const int64_t nb = n * Tn;
        if (nb > 0) {
            const int64_t g = std::max<int64_t>(1, std::min<int64_t>(cdiv(nb, 256), (int64_t)sms(c) * 8));
            k_table_totals<<<(unsigned)g, 256, sizeof(unsigned long long) * Tn, c->stream>>>(data->off, nb, Tn, dT);
            FAE_LAUNCHED(c);
        }
        FAE_CUDA(c, cudaMemcpyAsync(T.data(), dT, sizeof(int64_t) * Tn, cudaMemcpyDeviceToHost, c->stream));
    } else {
        for (int z = 0; z < Tn; z++) T[z] = n * (int64_t)data->fixed_pool;
    }
    if (multi) {
        st = coll_allreduce_sum(c, counts, total_rows, CollT::U32, "fae_profile: allreduce counts");
        if (st != FAE_OK) return st;
        FAE_CUDA(c, cudaMemcpyAsync(dT, T.data(), sizeof(int64_t) * Tn, cudaMemcpyHostToDevice, c->stream));
        st = coll_allreduce_sum(c, dT, Tn, CollT::I64, "fae_profile: allreduce T");
        if (st != FAE_OK) return st;
        FAE_CUDA(c, cudaMemcpyAsync(T.data(), dT, sizeof(int64_t) * Tn, cudaMemcpyDeviceToHost, c->stream));
    }
    if (sampled_ids && ns > 0)
        FAE_CUDA(c, cudaMemcpyAsync(sampled_ids, ids, sizeof(int64_t) * ns, cudaMemcpyDeviceToDevice, c->stream));
    st = read_latched(c);   // synchronises
    for (int z = 0; z < Tn; z++) T_host[z] = T[z];
    *n_sampled = ns;
    return st;
}
