// threshold.cu — threshold knob, embedding classifier and hot-row remap
// (SURVEY §8(a) a3, a4).
//
//  Eq. 1   H_zt = t*T*x/100; large row hot iff k >= H_zt (Eq. 2's >=)
//  small tables < 1 MB are hot in full
//  BUDGET_EXACT smallest integer cutoff K whose hot set fits L
//  Eqs. 2-4 CLT estimate of the hot size per large table
//  remap hot_id(g) = #{hot g' < g}
//
// B200 design: the hot set is one bitmap over the concatenated rows plus an
// exclusive rank prefix per 64-row word, interleaved in 16-byte entries
// {lo, hi, prefix, 0} — a rank query is one 128-bit load (2 bits/row; the
// Kaggle-shaped hot set directory is 8.4 MB, L2-resident).  It is built in
// one pass over the loggers with a decoupled look-back scan.  The budget
// search evaluates 63 candidate cutoffs per pass over the loggers (binary
// search of each row's count in the sorted per-table candidate cutoffs ->
// 64-bin histogram), so it converges in ~log64(K_hi) passes.
#include <algorithm>
#include <cmath>

#include "fae_internal.cuh"

namespace fae {

fae_status upload_schema(Ctx* c, const fae_tables* t, std::vector<int64_t>& rowbase);
fae_status validate_schema(Ctx* c, const fae_tables* t, const char* who);

constexpr int kDirThreads = 256;
constexpr int kDirIters = 8;                       // rows per thread
constexpr int kDirTileRows = kDirThreads * kDirIters;   // 2048 rows = 32 words
constexpr int kNCand = 63;

__device__ __forceinline__ int table_of(const int64_t* s_rb, int Tn, int64_t g) {
    int lo = 0, hi = Tn - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_rb[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Per-table max count (large tables only matter; computed for all).  Each
// thread streams 4 consecutive loggers per 16-byte load; the table of a
// position is tracked incrementally (tables are contiguous), the running max
// kept in a register and flushed to shared memory only when the table
// changes, then one global atomic per table per block.
__device__ __forceinline__ int table_from(const int64_t* s_rb, int Tn, int64_t g, int z) {
    while (z + 1 < Tn && g >= s_rb[z + 1]) z++;
    return z;
}

__global__ void __launch_bounds__(256)
k_table_max(const uint32_t* __restrict__ counts, int64_t total, const int64_t* __restrict__ rowbase,
            int Tn, uint32_t* __restrict__ tmax) {
    extern __shared__ int64_t s_rb[];
    uint32_t* s_max = reinterpret_cast<uint32_t*>(s_rb + Tn + 1);
    for (int z = threadIdx.x; z <= Tn; z += blockDim.x) s_rb[z] = rowbase[z];
    for (int z = threadIdx.x; z < Tn; z += blockDim.x) s_max[z] = 0u;
    __syncthreads();
    const int64_t n4 = (((uintptr_t)counts & 15) == 0) ? total / 4 : 0;   // 16-byte loads when aligned
    const uint4* c4 = reinterpret_cast<const uint4*>(counts);
    int zc = -1;
    uint32_t m = 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4 + (total - 4 * n4);
         q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v[4];
        int64_t g0;
        int nv;
        if (q < n4) {
            const uint4 x = __ldcs(c4 + q);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
            g0 = q * 4;
            nv = 4;
        } else {   // the < 4 trailing loggers
            g0 = n4 * 4 + (q - n4);
            v[0] = counts[g0];
            nv = 1;
        }
        int z = table_of(s_rb, Tn, g0);
        for (int k = 0; k < nv; k++) {
            z = table_from(s_rb, Tn, g0 + k, z);
            if (z != zc) {
                if (zc >= 0 && m) atomicMax(&s_max[zc], m);
                zc = z;
                m = 0;
            }
            m = max(m, v[k]);
        }
    }
    if (zc >= 0 && m) atomicMax(&s_max[zc], m);
    __syncthreads();
    for (int z = threadIdx.x; z < Tn; z += blockDim.x)
        if (s_max[z]) atomicMax(&tmax[z], s_max[z]);
}

// For each large row: m = #{candidates c : cut[z][c] <= k}; hist[m]++ .
// cut is [Tn][kNCand] ascending in c (uint64; >= 1 for large tables, so a
// zero logger counts for no candidate); small tables have cut = 0 and are
// skipped via the `large` mask.  16-byte loads, incremental table tracking.
__global__ void __launch_bounds__(256)
k_count_ge_multi(const uint32_t* __restrict__ counts, int64_t total,
                 const int64_t* __restrict__ rowbase, int Tn,
                 const unsigned long long* __restrict__ cut, const uint8_t* __restrict__ large,
                 int ncand, unsigned long long* __restrict__ hist) {
    extern __shared__ int64_t s_rb[];
    __shared__ unsigned int sh[kNCand + 1];
    for (int z = threadIdx.x; z <= Tn; z += blockDim.x) s_rb[z] = rowbase[z];
    for (int i = threadIdx.x; i <= kNCand; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t n4 = (((uintptr_t)counts & 15) == 0) ? total / 4 : 0;   // 16-byte loads when aligned
    const uint4* c4 = reinterpret_cast<const uint4*>(counts);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4 + (total - 4 * n4);
         q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v[4];
        int64_t g0;
        int nv;
        if (q < n4) {
            const uint4 x = __ldcs(c4 + q);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
            g0 = q * 4;
            nv = 4;
        } else {
            g0 = n4 * 4 + (q - n4);
            v[0] = counts[g0];
            nv = 1;
        }
        if ((v[0] | (nv > 1 ? v[1] | v[2] | v[3] : 0u)) == 0u) continue;   // the common case
        int z = table_of(s_rb, Tn, g0);
        for (int k = 0; k < nv; k++) {
            z = table_from(s_rb, Tn, g0 + k, z);
            if (!v[k] || !large[z]) continue;
            const uint64_t vv = v[k];
            const unsigned long long* cz = cut + (int64_t)z * kNCand;
            int lo = 0, hi = ncand;   // first c with cut > v
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (cz[mid] <= vv) lo = mid + 1;
                else hi = mid;
            }
            if (lo) atomicAdd(&sh[lo], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= kNCand; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// Bitmap + rank directory.  kmin_eff[z] = 0 for small tables (all hot),
// else kmin_z >= 1.  dir[w] = {bits lo, bits hi, exclusive hot prefix, 0}.
__global__ void __launch_bounds__(kDirThreads)
k_build_dir(const uint32_t* __restrict__ counts, int64_t total, const int64_t* __restrict__ rowbase,
            int Tn, const unsigned long long* __restrict__ kmin_eff, uint4* __restrict__ dir,
            uint64_t* __restrict__ status, uint32_t* __restrict__ ctr, int64_t* __restrict__ H_out) {
    extern __shared__ int64_t s_rb[];
    __shared__ uint32_t s_half[kDirTileRows / 32];
    __shared__ int s_tile;
    __shared__ uint64_t s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int z = tid; z <= Tn; z += blockDim.x) s_rb[z] = rowbase[z];
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t tbase = tile * kDirTileRows;
    if (tbase >= total) return;
    const int zt = table_of(s_rb, Tn, tbase);   // tables are contiguous: track from the tile's first
    uint32_t cv[kDirIters];
#pragma unroll
    for (int it = 0; it < kDirIters; it++) {   // all loads in flight first
        const int64_t g = tbase + it * kDirThreads + tid;
        cv[it] = g < total ? __ldcs(counts + g) : 0u;
    }
    int z = zt;
#pragma unroll
    for (int it = 0; it < kDirIters; it++) {
        const int64_t g = tbase + it * kDirThreads + tid;
        bool hot = false;
        if (g < total) {
            z = table_from(s_rb, Tn, g, z);
            hot = (unsigned long long)cv[it] >= kmin_eff[z];
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hot);
        if (lane == 0) s_half[it * (kDirThreads / 32) + warp] = m;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t lo = s_half[2 * lane], hi = s_half[2 * lane + 1];
        const uint32_t pc = __popc(lo) + __popc(hi);
        uint32_t x = pc;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
        if (lane == 0) {
            s_ex = lookback_u64(status, tile, tot);
            const int64_t last = (total - 1) / kDirTileRows;
            if (tile == last) *H_out = (int64_t)(s_ex + tot);
        }
        __syncwarp();
        const uint64_t ex = s_ex;
        const int64_t w = tile * (kDirTileRows / 64) + lane;
        if (w * 64 < total) dir[w] = make_uint4(lo, hi, (uint32_t)(ex + x - pc), 0u);
    }
}

// rank at table boundaries: base[z] = hot_id(rowbase[z]); base[Tn] = H
__global__ void k_rank_at(const uint4* __restrict__ dir, const int64_t* __restrict__ rowbase, int Tn,
                          int64_t total, const int64_t* __restrict__ H, int64_t* __restrict__ base) {
    for (int z = threadIdx.x; z <= Tn; z += blockDim.x) {
        const int64_t g = rowbase[z];
        if (g >= total) {
            base[z] = *H;
        } else {
            uint32_t rk;
            hs_test(dir[g >> 6], g, &rk);
            base[z] = rk;
        }
    }
}

__global__ void __launch_bounds__(256)
k_remap(const uint4* __restrict__ dir, int64_t total, int32_t* __restrict__ remap) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        uint32_t rk;
        const bool b = hs_test(dir[g >> 6], g, &rk);
        remap[g] = b ? (int32_t)rk : -1;
    }
}

// Eqs. 2-4 for one large table per block.  out[z*6 + {0..5}] =
// {ybar, s, lo, hi, est, exact}.  fp64 with explicit round-to-nearest ops
// (no contraction) in the order the equations state.
__global__ void __launch_bounds__(1024)
k_estimate(const uint32_t* __restrict__ counts, const int64_t* __restrict__ rowbase,
           const int32_t* __restrict__ tables, const unsigned long long* __restrict__ kmin,
           int n, int m, uint64_t chunk_seed, double t_q, double* __restrict__ out) {
    __shared__ unsigned long long s_key[32];
    __shared__ long long s_idx[32];
    __shared__ long long s_chosen[256];
    __shared__ long long s_C[256];
    __shared__ unsigned long long s_cnt;
    const int z = tables[blockIdx.x];
    const int64_t g0 = rowbase[z];
    const int64_t Nz = rowbase[z + 1] - g0;
    const uint64_t km = kmin[z];
    const int64_t N = Nz / m;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double* o = out + (int64_t)z * 6;
    if (N < n) {
        if (tid == 0) s_cnt = 0;
        __syncthreads();
        unsigned long long c = 0;
        for (int64_t j = tid; j < Nz; j += blockDim.x) c += (counts[g0 + j] >= km);
        for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
        if (lane == 0) atomicAdd(&s_cnt, c);
        __syncthreads();
        if (tid == 0) {
            const double e = (double)s_cnt;
            o[0] = 0.0; o[1] = 0.0; o[2] = e; o[3] = e; o[4] = e; o[5] = 1.0;
        }
        return;
    }
    const uint64_t seed = chunk_seed ^ (uint64_t)z;
    unsigned long long pk = 0;
    long long pi = -1;   // previous selected pair; select pairs > (pk, pi)
    for (int r = 0; r < n; r++) {
        unsigned long long bk = ~0ull;
        long long bi = 0x7FFFFFFFFFFFFFFFll;
        for (int64_t cc = tid; cc < N; cc += blockDim.x) {
            const unsigned long long k = hash_key(seed, (uint64_t)cc);
            const bool gt = (k > pk) || (k == pk && cc > pi);
            if (gt && ((k < bk) || (k == bk && cc < bi))) {
                bk = k;
                bi = cc;
            }
        }
        for (int s = 16; s; s >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, s);
            const long long oi = __shfl_xor_sync(0xffffffffu, bi, s);
            if ((ok < bk) || (ok == bk && oi < bi)) {
                bk = ok;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_key[warp] = bk;
            s_idx[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nw; w++)
                if ((s_key[w] < s_key[0]) || (s_key[w] == s_key[0] && s_idx[w] < s_idx[0])) {
                    s_key[0] = s_key[w];
                    s_idx[0] = s_idx[w];
                }
            s_chosen[r] = s_idx[0];
        }
        __syncthreads();
        pk = s_key[0];
        pi = s_idx[0];
        __syncthreads();
    }
    if (tid == 0) {   // ascending chunk order
        for (int i = 1; i < n; i++) {
            const long long x = s_chosen[i];
            int j = i - 1;
            while (j >= 0 && s_chosen[j] > x) {
                s_chosen[j + 1] = s_chosen[j];
                j--;
            }
            s_chosen[j + 1] = x;
        }
    }
    __syncthreads();
    // Eq. 2: C_i, one warp per chunk
    for (int i = warp; i < n; i += nw) {
        const int64_t b = g0 + s_chosen[i] * (int64_t)m;
        long long c = 0;
        for (int j = lane; j < m; j += 32) c += (counts[b + j] >= km);
        for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
        if (lane == 0) s_C[i] = c;
    }
    __syncthreads();
    if (tid == 0) {
        double sum = 0.0;
        for (int i = 0; i < n; i++) sum = __dadd_rn(sum, (double)s_C[i]);
        const double ybar = __ddiv_rn(sum, (double)n);                       // Eq. 3
        double ss = 0.0;
        for (int i = 0; i < n; i++) {
            const double d = __dsub_rn((double)s_C[i], ybar);
            ss = __dadd_rn(ss, __dmul_rn(d, d));
        }
        const double s2 = n > 1 ? __ddiv_rn(ss, (double)(n - 1)) : 0.0;
        const double fpc = __ddiv_rn((double)(N - n), (double)N);
        const double hw = __dmul_rn(t_q, __dsqrt_rn(__dmul_rn(fpc, __ddiv_rn(s2, (double)n))));  // Eq. 4
        const double scale = __ddiv_rn((double)Nz, (double)m);
        double lo = __dmul_rn(__dsub_rn(ybar, hw), scale);
        double hi = __dmul_rn(__dadd_rn(ybar, hw), scale);
        if (lo < 0.0) lo = 0.0;
        if (hi > (double)Nz) hi = (double)Nz;
        o[0] = ybar;
        o[1] = __dsqrt_rn(s2);
        o[2] = lo;
        o[3] = hi;
        o[4] = __dmul_rn(ybar, scale);
        o[5] = 0.0;
    }
}

static int sms(Ctx* c) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, c->device);
    return n;
}

static uint64_t cut_of(uint64_t K, int64_t Tz, int64_t Tref) {
    // max(1, ceil(K*T_z/T_ref)), exact
    if (Tz <= 0) return ~0ull;
    const unsigned __int128 num = (unsigned __int128)K * (uint64_t)Tz;
    const unsigned __int128 q = (num + (uint64_t)(Tref - 1)) / (uint64_t)Tref;
    uint64_t v = q > (unsigned __int128)(~0ull) ? ~0ull : (uint64_t)q;
    return v < 1 ? 1 : v;
}

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_threshold(fae_ctx* h, const fae_tables* tabs, const uint32_t* counts,
                                    const int64_t* T_host, double x_pct, const fae_thresh_req* req,
                                    int32_t* remap_out, fae_thresh_result* res) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    fae_status st = validate_schema(c, tabs, "fae_threshold");
    if (st != FAE_OK) return st;
    if (!counts || !T_host || !req || !res) return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: null argument");
    if (!(x_pct > 0.0 && x_pct <= 100.0)) return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: x must be in (0, 100]");
    if (req->mode != FAE_THRESH_FIXED_T && req->mode != FAE_THRESH_BUDGET_EXACT &&
        req->mode != FAE_THRESH_CLT_SEARCH)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: bad mode");
    if (req->mode == FAE_THRESH_FIXED_T && !(req->t > 0.0 && req->t <= 1.0))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: t must be in (0, 1]");
    if (req->mode != FAE_THRESH_FIXED_T && req->budget_bytes < 0)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: negative budget");
    if ((req->want_estimate || req->mode == FAE_THRESH_CLT_SEARCH) &&
        (req->n_chunks < 2 || req->n_chunks > 256 || req->chunk_rows < 1))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_threshold: n must be in [2, 256] and m >= 1");
    const int Tn = tabs->n_tables;
    const int D = tabs->dim;
    std::vector<int64_t> rowbase;
    st = upload_schema(c, tabs, rowbase);
    if (st != FAE_OK) return st;
    const int64_t total = rowbase[Tn];
    std::vector<uint8_t> large(Tn);
    int64_t small_total = 0, Tref = 0;
    for (int z = 0; z < Tn; z++) {
        large[z] = !(tabs->rows[z] * (int64_t)D * 4 < req->small_table_bytes);
        if (!large[z]) small_total += tabs->rows[z] * (int64_t)D * 4;
        else Tref = std::max(Tref, T_host[z]);
    }
    // scratch
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
    const int64_t tiles = std::max<int64_t>(1, cdiv(total, kDirTileRows));
    const size_t o_cut = take(sizeof(unsigned long long) * Tn * kNCand);
    const size_t o_large = take(Tn);
    const size_t o_hist = take(sizeof(unsigned long long) * (kNCand + 1));
    const size_t o_tmax = take(sizeof(uint32_t) * Tn);
    const size_t o_kmin = take(sizeof(unsigned long long) * Tn);
    const size_t o_st = take(sizeof(uint64_t) * tiles);
    const size_t o_ctr = take(sizeof(uint32_t) * 4);
    const size_t o_H = take(sizeof(int64_t) * 2);
    const size_t o_base = take(sizeof(int64_t) * (Tn + 1));
    const size_t o_tab = take(sizeof(int32_t) * Tn);
    const size_t o_est = take(sizeof(double) * 6 * Tn);
    char* sc = (char*)scratch(c, o);
    if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_threshold: scratch allocation failed");
    unsigned long long* d_cut = (unsigned long long*)(sc + o_cut);
    uint8_t* d_large = (uint8_t*)(sc + o_large);
    unsigned long long* d_hist = (unsigned long long*)(sc + o_hist);
    uint32_t* d_tmax = (uint32_t*)(sc + o_tmax);
    unsigned long long* d_kmin = (unsigned long long*)(sc + o_kmin);
    uint64_t* d_status = (uint64_t*)(sc + o_st);
    uint32_t* d_ctr = (uint32_t*)(sc + o_ctr);
    int64_t* d_H = (int64_t*)(sc + o_H);
    int64_t* d_base = (int64_t*)(sc + o_base);
    int32_t* d_tab = (int32_t*)(sc + o_tab);
    double* d_est = (double*)(sc + o_est);
    FAE_CUDA(c, cudaMemcpyAsync(d_large, large.data(), Tn, cudaMemcpyHostToDevice, c->stream));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), (int64_t)sms(c) * 8));
    const size_t rb_smem = sizeof(int64_t) * (Tn + 1);

    std::vector<uint64_t> kmin(Tn, 0);
    uint64_t K = 0;
    int32_t slack = 0;
    double t_final = req->t;
    if (req->mode == FAE_THRESH_FIXED_T) {
        for (int z = 0; z < Tn; z++) {
            if (!large[z]) continue;
            const double H = ((req->t * (double)T_host[z]) * x_pct) / 100.0;   // Eq. 1 (R21)
            const double cc = std::ceil(H);
            kmin[z] = cc < 1.0 ? 1 : (cc >= 1.8e19 ? ~0ull : (uint64_t)cc);
        }
    } else if (req->mode == FAE_THRESH_CLT_SEARCH) {
        // Statistical optimizer (R27): geometric grid then 8
        // bisection steps on the Eq. 4 CI upper bound of the hot bytes; every
        // evaluation = Eq. 1 cutoffs + one k_estimate launch over the large
        // tables (Eqs. 2-4 on the device), summed here in table order
        std::vector<int32_t> tl;
        for (int z = 0; z < Tn; z++)
            if (large[z]) tl.push_back(z);
        if (!tl.empty())
            FAE_CUDA(c, cudaMemcpyAsync(d_tab, tl.data(), sizeof(int32_t) * tl.size(), cudaMemcpyHostToDevice, c->stream));
        std::vector<unsigned long long> km(Tn);
        std::vector<double> e(6 * Tn);
        auto kmin_at = [&](double t) {
            for (int z = 0; z < Tn; z++) {
                km[z] = 0ull;
                if (!large[z]) continue;
                const double H = ((t * (double)T_host[z]) * x_pct) / 100.0;   // Eq. 1 (R21)
                const double cc = std::ceil(H);
                km[z] = cc < 1.0 ? 1 : (cc >= 1.8e19 ? ~0ull : (uint64_t)cc);
            }
        };
        auto est_bytes = [&](double t, double* b) -> fae_status {
            kmin_at(t);
            if (!tl.empty()) {
                FAE_CUDA(c, cudaMemcpyAsync(d_kmin, km.data(), sizeof(unsigned long long) * Tn, cudaMemcpyHostToDevice,
                                            c->stream));
                k_estimate<<<(unsigned)tl.size(), 1024, 0, c->stream>>>(counts, c->d_rowbase_tmp, d_tab, d_kmin,
                                                                        req->n_chunks, req->chunk_rows,
                                                                        req->chunk_seed, req->t_quantile, d_est);
                FAE_LAUNCHED(c);
                FAE_CUDA(c, cudaMemcpyAsync(e.data(), d_est, sizeof(double) * 6 * Tn, cudaMemcpyDeviceToHost, c->stream));
                FAE_CUDA(c, cudaStreamSynchronize(c->stream));
            }
            double acc = 0.0;
            for (int z = 0; z < Tn; z++) {
                if (!large[z]) acc += (double)(tabs->rows[z] * (int64_t)D * 4);
                else acc += e[6 * z + 3] * (double)D * 4.0;
            }
            *b = acc;
            return FAE_OK;
        };
        const double L = (double)req->budget_bytes;
        double tg[29], b = 0.0;
        for (int j = 0; j <= 28; j++) tg[j] = std::pow(10.0, -8.0 + 0.25 * (double)j);
        int jstar = -1;
        for (int j = 0; j <= 28 && jstar < 0; j++) {
            if ((st = est_bytes(tg[j], &b)) != FAE_OK) return st;
            if (b <= L) jstar = j;
        }
        if (jstar < 0)
            return set_err(c, FAE_ERR_BUDGET_INFEASIBLE, "fae_threshold: the estimate at t = 0.1 exceeds the budget");
        t_final = tg[jstar];
        if (jstar == 0) {
            slack = 1;
        } else {
            double lo = tg[jstar - 1], hi = tg[jstar];
            for (int it = 0; it < 8; it++) {
                const double mid = (lo + hi) / 2.0;
                if ((st = est_bytes(mid, &b)) != FAE_OK) return st;
                if (b <= L) hi = mid;
                else lo = mid;
            }
            t_final = hi;
        }
        kmin_at(t_final);
        for (int z = 0; z < Tn; z++) kmin[z] = km[z];
    } else {
        if (small_total > req->budget_bytes)
            return set_err(c, FAE_ERR_BUDGET_INFEASIBLE, "fae_threshold: small tables alone exceed the budget");
        if (Tref == 0) Tref = 1;
        // K_hi: first K at which no large row can be hot
        FAE_CUDA(c, cudaMemsetAsync(d_tmax, 0, sizeof(uint32_t) * Tn, c->stream));
        k_table_max<<<(unsigned)grid, 256, rb_smem + sizeof(uint32_t) * Tn, c->stream>>>(counts, total,
                                                                                        c->d_rowbase_tmp, Tn, d_tmax);
        FAE_LAUNCHED(c);
        std::vector<uint32_t> tmax(Tn);
        FAE_CUDA(c, cudaMemcpyAsync(tmax.data(), d_tmax, sizeof(uint32_t) * Tn, cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        uint64_t Khi = 1;
        for (int z = 0; z < Tn; z++) {
            if (!large[z]) continue;
            const int64_t Tz = T_host[z] > 0 ? T_host[z] : 1;
            const unsigned __int128 need =
                ((unsigned __int128)((uint64_t)tmax[z] + 1) * (uint64_t)Tref + (uint64_t)Tz - 1) / (uint64_t)Tz;
            Khi = std::max<uint64_t>(Khi, (uint64_t)need);
        }
        // evaluate bytes() at a set of candidate K (ascending)
        auto eval = [&](const std::vector<uint64_t>& Ks, std::vector<int64_t>& bytes) -> fae_status {
            const int nc = (int)Ks.size();
            std::vector<unsigned long long> cut((size_t)Tn * kNCand, ~0ull);
            for (int z = 0; z < Tn; z++)
                for (int i = 0; i < nc; i++) cut[(size_t)z * kNCand + i] = large[z] ? cut_of(Ks[i], T_host[z], Tref) : 0ull;
            FAE_CUDA(c, cudaMemcpyAsync(d_cut, cut.data(), sizeof(unsigned long long) * cut.size(), cudaMemcpyHostToDevice, c->stream));
            FAE_CUDA(c, cudaMemsetAsync(d_hist, 0, sizeof(unsigned long long) * (kNCand + 1), c->stream));
            k_count_ge_multi<<<(unsigned)grid, 256, rb_smem, c->stream>>>(counts, total, c->d_rowbase_tmp, Tn, d_cut,
                                                                          d_large, nc, d_hist);
            FAE_LAUNCHED(c);
            std::vector<unsigned long long> hist(kNCand + 1);
            FAE_CUDA(c, cudaMemcpyAsync(hist.data(), d_hist, sizeof(unsigned long long) * (kNCand + 1), cudaMemcpyDeviceToHost, c->stream));
            FAE_CUDA(c, cudaStreamSynchronize(c->stream));
            // rows hot at candidate i = #{rows with m > i} = suffix sum of hist[i+1..]
            bytes.assign(nc, 0);
            unsigned long long suf = 0;
            for (int i = nc - 1; i >= 0; i--) {
                suf += hist[i + 1];
                bytes[i] = small_total + (int64_t)suf * D * 4;
            }
            return FAE_OK;
        };
        std::vector<int64_t> b;
        st = eval({1}, b);
        if (st != FAE_OK) return st;
        if (b[0] <= req->budget_bytes) {
            K = 1;
            slack = 1;
        } else {
            uint64_t lo = 1, hi = Khi;   // bytes(lo) > L >= bytes(hi)
            while (hi - lo > 1) {
                std::vector<uint64_t> Ks;
                const uint64_t span = hi - lo;
                for (int i = 1; i <= kNCand; i++) {
                    const uint64_t k = lo + (uint64_t)((unsigned __int128)span * i / (kNCand + 1));
                    if (k > lo && k < hi && (Ks.empty() || Ks.back() != k)) Ks.push_back(k);
                }
                if (Ks.empty()) break;
                st = eval(Ks, b);
                if (st != FAE_OK) return st;
                uint64_t nlo = lo, nhi = hi;
                for (size_t i = 0; i < Ks.size(); i++) {
                    if (b[i] <= req->budget_bytes) {
                        nhi = Ks[i];
                        break;
                    }
                    nlo = Ks[i];
                }
                lo = nlo;
                hi = nhi;
            }
            K = hi;
        }
        for (int z = 0; z < Tn; z++) kmin[z] = large[z] ? cut_of(K, T_host[z], Tref) : 0;
        t_final = (double)K / ((double)Tref * x_pct / 100.0);
    }
    // hot set: bitmap + rank directory.  The ctx's previous hot set is
    // invalid from here until every check below has passed: a
    // failure leaves no half-rebuilt set for fae_classify / fae_extract.
    HotSet& hs = c->hs;
    hs.valid = false;
    const int64_t words = cdiv(total, 64);
    if (hs.dir_cap < words) {
        cudaStreamSynchronize(c->stream);
        cudaFree(hs.dir);
        hs.dir = nullptr;
        hs.dir_cap = 0;
        FAE_CUDA(c, cudaMalloc(&hs.dir, sizeof(uint4) * (words + 32)));
        hs.dir_cap = words;
    }
    std::vector<unsigned long long> kmin_eff(Tn);
    for (int z = 0; z < Tn; z++) kmin_eff[z] = large[z] ? kmin[z] : 0ull;
    FAE_CUDA(c, cudaMemcpyAsync(d_kmin, kmin_eff.data(), sizeof(unsigned long long) * Tn, cudaMemcpyHostToDevice, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(d_status, 0, sizeof(uint64_t) * tiles, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(d_ctr, 0, sizeof(uint32_t) * 4, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(d_H, 0, sizeof(int64_t), c->stream));
    k_build_dir<<<(unsigned)tiles, kDirThreads, rb_smem, c->stream>>>(counts, total, c->d_rowbase_tmp, Tn, d_kmin,
                                                                     hs.dir, d_status, d_ctr, d_H);
    FAE_LAUNCHED(c);
    k_rank_at<<<1, 256, 0, c->stream>>>(hs.dir, c->d_rowbase_tmp, Tn, total, d_H, d_base);
    FAE_LAUNCHED(c);
    FAE_CUDA(c, cudaMemcpyAsync(hs.d_rowbase, c->d_rowbase_tmp, sizeof(int64_t) * (Tn + 1), cudaMemcpyDeviceToDevice, c->stream));
    if (remap_out) {
        k_remap<<<(unsigned)grid, 256, 0, c->stream>>>(hs.dir, total, remap_out);
        FAE_LAUNCHED(c);
    }
    std::vector<double> est(6 * Tn, 0.0);
    if (req->want_estimate) {
        std::vector<int32_t> tl;
        for (int z = 0; z < Tn; z++)
            if (large[z]) tl.push_back(z);
        if (!tl.empty()) {
            FAE_CUDA(c, cudaMemcpyAsync(d_tab, tl.data(), sizeof(int32_t) * tl.size(), cudaMemcpyHostToDevice, c->stream));
            FAE_CUDA(c, cudaMemsetAsync(d_est, 0, sizeof(double) * 6 * Tn, c->stream));
            k_estimate<<<(unsigned)tl.size(), 1024, 0, c->stream>>>(counts, c->d_rowbase_tmp, d_tab, d_kmin, req->n_chunks,
                                                                    req->chunk_rows, req->chunk_seed, req->t_quantile, d_est);
            FAE_LAUNCHED(c);
            FAE_CUDA(c, cudaMemcpyAsync(est.data(), d_est, sizeof(double) * 6 * Tn, cudaMemcpyDeviceToHost, c->stream));
        }
    }
    std::vector<int64_t> base(Tn + 1);
    FAE_CUDA(c, cudaMemcpyAsync(base.data(), d_base, sizeof(int64_t) * (Tn + 1), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    const int64_t H = base[Tn];
    if (H >= (1ll << 31) - 1) return set_err(c, FAE_ERR_CAPACITY, "fae_threshold: H_total >= 2^31");
    hs.valid = true;
    hs.n_tables = Tn;
    hs.dim = D;
    hs.total_rows = total;
    hs.H_total = H;
    hs.rows.assign(tabs->rows, tabs->rows + Tn);
    hs.rowbase = rowbase;
    hs.base = base;
    for (int z = 0; z < Tn; z++) {
        if (res->kmin) res->kmin[z] = (int64_t)std::min<uint64_t>(kmin[z], (uint64_t)INT64_MAX);
        if (res->hot_rows) res->hot_rows[z] = base[z + 1] - base[z];
        if (res->is_small) res->is_small[z] = !large[z];
        if (res->est_mean) res->est_mean[z] = est[6 * z + 0];
        if (res->est_sd) res->est_sd[z] = est[6 * z + 1];
        if (res->est_lo) res->est_lo[z] = est[6 * z + 2];
        if (res->est_hi) res->est_hi[z] = est[6 * z + 3];
        if (res->est_rows) res->est_rows[z] = est[6 * z + 4];
        if (res->est_exact) res->est_exact[z] = (int32_t)est[6 * z + 5];
    }
    if (res->base)
        for (int z = 0; z <= Tn; z++) res->base[z] = base[z];
    res->H_total = H;
    res->hot_bytes = H * (int64_t)D * 4;
    res->t_final = t_final;
    res->K = K;
    res->budget_slack = slack;
    return read_latched(c);
}
