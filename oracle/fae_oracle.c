/*
 * fae_oracle.c — plain, slow, obviously-correct CPU ORACLE for the FAE hot path
 * (Adnan et al., "Accelerating Recommendation System Training by Leveraging
 * Popular Choices", arXiv 2103.00686).
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2103_00686_b200/, include/fae.h) never calls, links or includes
 * anything here, and this file includes nothing from the product path.
 *
 * Citations: "P:Lnnn" = PAPER.md line nnn (section / equation in brackets);
 * the readings of silent or garbled passages are DESIGN.md "Readings" R1..R25.
 *
 * Floating point: every reduction is accumulated in fp64 in the order the
 * definition states and rounded once; compile with -ffp-contract=off.
 * Where the method is an exact result with a plain definition (counting,
 * membership, partition, pooling, gradient), the definition is written out.
 * Where the method approximates (Eqs. 2-4 CLT estimate), the steps follow the
 * paper's order and notation.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"): the Eq. 1 worked example
 * 302.5, brute force on tiny inputs, closed forms (A.W and A^T.dY
 * as sparse-dense products, p^B), invariants (partition, purity, conservation,
 * rank remap, monotonicity, untouched rows).  Parity unpinned: none.
 *
 * All-cores variant (the cpu_baseline's multi-thread figure):
 * the same file compiled with -fopenmp.  The pragmas only split loops whose
 * iterations are independent (keys, per-record classification, per-bag
 * forward) or integer counts (atomic increments); the backward splits by row
 * ownership (row r belongs to thread r mod nthreads, which scans the lookups
 * in ascending p), so every fp64 sum keeps its serial order and the results
 * are bit-identical to the serial build (tested).  Without -fopenmp the
 * pragmas are ignored.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
static int or_nthreads(void) { return omp_get_num_threads(); }
static int or_thread(void) { return omp_get_thread_num(); }
#else
static int or_nthreads(void) { return 1; }
static int or_thread(void) { return 0; }
#endif

/* status codes, same numeric meaning as the product ABI (documented, not shared) */
#define OR_OK 0
#define OR_INVALID_ARG 1
#define OR_BUDGET_INFEASIBLE 3
#define OR_INDEX_RANGE 4

/* ---------------------------------------------------------------------------
 * Counter hash (R6): splitmix64 finaliser of seed + (i+1)*golden.
 * ------------------------------------------------------------------------- */
uint64_t or_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

uint64_t or_key(uint64_t seed, uint64_t i)
{
    return or_mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

typedef struct { uint64_t key; int64_t i; } or_pair;

static int cmp_pair(const void* a, const void* b)
{
    const or_pair* p = (const or_pair*)a;
    const or_pair* q = (const or_pair*)b;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    if (p->i != q->i) return p->i < q->i ? -1 : 1;
    return 0;
}

/* ---------------------------------------------------------------------------
 * O1  Input sampler  (§4.1.1: "we sample x% of the input dataset
 * (D) ... obtains D-hat").  Uniform without replacement (R6): the k records
 * with the smallest (key(seed, i), i), k = floor(R*x/100), output in
 * ascending record id (original order kept).  Returns k, or -1 if x not in
 * (0, 100].
 * ------------------------------------------------------------------------- */
int64_t or_sample_count(int64_t R, double x_pct)
{
    if (!(x_pct > 0.0 && x_pct <= 100.0) || R < 0) return -1;
    return (int64_t)floor((double)R * x_pct / 100.0);
}

int64_t or_sample(int64_t R, double x_pct, uint64_t seed, int64_t* out_ids)
{
    int64_t k = or_sample_count(R, x_pct);
    if (k < 0) return -1;
    if (k == 0) return 0;
    or_pair* v = (or_pair*)malloc(sizeof(or_pair) * (size_t)R);
    uint8_t* chosen = (uint8_t*)calloc((size_t)R, 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < R; i++) { v[i].key = or_key(seed, (uint64_t)i); v[i].i = i; }
    qsort(v, (size_t)R, sizeof(or_pair), cmp_pair);
    for (int64_t j = 0; j < k; j++) chosen[v[j].i] = 1;
    int64_t w = 0;
    for (int64_t i = 0; i < R; i++) if (chosen[i]) out_ids[w++] = i;
    free(v); free(chosen);
    return k;
}

/* bag (r, z) = lookups [lo, hi) of the sample-major CSR (D1) */
static void bag_range(const int64_t* off, int32_t fixed_pool, int32_t n_tables,
                      int64_t r, int32_t z, int64_t* lo, int64_t* hi)
{
    int64_t b = r * n_tables + z;
    if (off) { *lo = off[b]; *hi = off[b + 1]; }
    else { *lo = b * fixed_pool; *hi = (b + 1) * fixed_pool; }
}

/* ---------------------------------------------------------------------------
 * O2  Embedding logger  (§4.1.2: "keep track of access counts
 * (denoted as k) of D-hat into each entry in E_z").  counts is the
 * concatenation of the per-table loggers (table z starts at sum_{z'<z} N_z').
 * Every lookup counts once (duplicates inside a bag count each time).
 * T_z = lookups into table z over ALL records (R3: "total number of accesses
 * into an embedding table").  Returns OR_INDEX_RANGE on a bad index.
 * ------------------------------------------------------------------------- */
int or_histogram(int32_t n_tables, const int64_t* rows, const int32_t* idx,
                 const int64_t* off, int32_t fixed_pool, int64_t n_records,
                 const int64_t* sampled, int64_t n_sampled,
                 uint32_t* counts, int64_t* T)
{
    int64_t total_rows = 0;
    int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tables + 1));
    for (int32_t z = 0; z < n_tables; z++) { base[z] = total_rows; total_rows += rows[z]; }
    base[n_tables] = total_rows;
    memset(counts, 0, sizeof(uint32_t) * (size_t)total_rows);
    int st = OR_OK;
    for (int32_t z = 0; z < n_tables; z++) T[z] = 0;
#pragma omp parallel for schedule(static) reduction(+ : T[:n_tables])
    for (int64_t r = 0; r < n_records; r++)
        for (int32_t z = 0; z < n_tables; z++) {
            int64_t lo, hi;
            bag_range(off, fixed_pool, n_tables, r, z, &lo, &hi);
            T[z] += hi - lo;
        }
#pragma omp parallel for schedule(static) reduction(max : st)
    for (int64_t s = 0; s < n_sampled; s++) {
        int64_t r = sampled[s];
        for (int32_t z = 0; z < n_tables; z++) {
            int64_t lo, hi;
            bag_range(off, fixed_pool, n_tables, r, z, &lo, &hi);
            for (int64_t p = lo; p < hi; p++) {
                int32_t j = idx[p];
                if (j < 0 || j >= rows[z]) { st = OR_INDEX_RANGE; continue; }
#pragma omp atomic
                counts[base[z] + j] += 1;
            }
        }
    }
    free(base);
    return st;
}

/* ---------------------------------------------------------------------------
 * Eq. 1:  H_zt = t * T * x / 100, evaluated as ((t*T)*x)/100 in
 * IEEE double (R21: this expression IS the definition).  A large-table row is
 * hot iff k >= H_zt (Eq. 2's ">=", R1), i.e. k >= kmin = ceil(H_zt); kmin is
 * clamped to >= 1 so that a row never seen in the sample is never hot (R25).
 * ------------------------------------------------------------------------- */
double or_cutoff(double t, int64_t T, double x_pct)
{
    return ((t * (double)T) * x_pct) / 100.0;
}

int64_t or_kmin_from_cutoff(double H)
{
    double c = ceil(H);
    if (c < 1.0) c = 1.0;
    return (int64_t)c;
}

/* small-table rule: tables < small_bytes (default 1 MB = 2^20 B,
 * R11) are hot in full.  Bytes = rows * dim * 4 (fp32, D2). */
static int is_small(int64_t rows, int32_t dim, int64_t small_bytes)
{
    return rows * (int64_t)dim * 4 < small_bytes;
}

/* Embedding classifier (§4.2: "tag (hot or cold) the embedding
 * table entries", one pass of each table).  hot[g] for every global row g. */
void or_tag_rows(int32_t n_tables, const int64_t* rows, int32_t dim,
                 int64_t small_bytes, const uint32_t* counts,
                 const int64_t* kmin, uint8_t* hot)
{
    int64_t g = 0;
    for (int32_t z = 0; z < n_tables; z++) {
        int small = is_small(rows[z], dim, small_bytes);
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < rows[z]; j++)
            hot[g + j] = small ? 1 : ((int64_t)counts[g + j] >= kmin[z] ? 1 : 0);
        g += rows[z];
    }
}

/* FIXED_T mode: kmin_z from Eq. 1 for every table (small tables report 0). */
void or_kmin_fixed_t(int32_t n_tables, const int64_t* rows, int32_t dim,
                     int64_t small_bytes, const int64_t* T, double t,
                     double x_pct, int64_t* kmin)
{
    for (int32_t z = 0; z < n_tables; z++)
        kmin[z] = is_small(rows[z], dim, small_bytes)
                      ? 0 : or_kmin_from_cutoff(or_cutoff(t, T[z], x_pct));
}

static int cmp_u32_desc(const void* a, const void* b)
{
    uint32_t p = *(const uint32_t*)a, q = *(const uint32_t*)b;
    return p < q ? 1 : (p > q ? -1 : 0);
}

/* #{j : k_j >= K} in a descending-sorted array (plain linear count). */
static int64_t count_ge(const uint32_t* sorted_desc, int64_t n, uint64_t K)
{
    int64_t c = 0;
    while (c < n && (uint64_t)sorted_desc[c] >= K) c++;
    return c;
}

/* K_z = max(1, ceil(K * T_z / T_ref)), exact integer arithmetic. */
static uint64_t table_cutoff(uint64_t K, int64_t Tz, int64_t Tref)
{
    unsigned __int128 num = (unsigned __int128)K * (unsigned __int128)(uint64_t)Tz;
    unsigned __int128 q = (num + (unsigned __int128)(uint64_t)(Tref - 1)) / (unsigned __int128)(uint64_t)Tref;
    uint64_t kz = (uint64_t)q;
    return kz < 1 ? 1 : kz;
}

/* ---------------------------------------------------------------------------
 * BUDGET_EXACT mode: the "naive mechanism" of P:L344-348 ("sorting all
 * embedding entries based on their access frequencies and classifying the top
 * h entries as hot", h = max hot entries that fit L), in Eq. 1 form (R10):
 * with T_ref = max over large tables of T_z and integer K >= 1, table z's
 * cutoff is K_z = ceil(K * T_z / T_ref) (= Eq. 1 at t = K / (T_ref x/100)).
 *   bytes(K) = sum_small N_z*D*4 + sum_large D*4*#{j : k_z[j] >= K_z}
 * Return the smallest K with bytes(K) <= L.  bytes() is non-increasing in K,
 * so the smallest feasible K is found by bisection over [1, K_hi], K_hi the
 * first K at which no large row can be hot.  Outputs kmin_z = K_z, K, t_final,
 * slack (K = 1 fits).  Returns OR_BUDGET_INFEASIBLE when even the
 * always-hot small tables exceed L.
 * ------------------------------------------------------------------------- */
int or_budget_exact(int32_t n_tables, const int64_t* rows, int32_t dim,
                    int64_t small_bytes, const uint32_t* counts,
                    const int64_t* T, double x_pct, int64_t budget_bytes,
                    int64_t* kmin, uint64_t* K_out, double* t_final,
                    int32_t* slack)
{
    int64_t small_total = 0, Tref = 0, g0 = 0;
    uint32_t** sorted = (uint32_t**)calloc((size_t)n_tables, sizeof(uint32_t*));
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tables + 1));
    for (int32_t z = 0; z < n_tables; z++) {
        start[z] = g0;
        if (is_small(rows[z], dim, small_bytes)) small_total += rows[z] * (int64_t)dim * 4;
        else if (T[z] > Tref) Tref = T[z];
        g0 += rows[z];
    }
    /* each large table's loggers sorted descending (independent per table) */
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t z = 0; z < n_tables; z++) {
        if (is_small(rows[z], dim, small_bytes)) continue;
        sorted[z] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)rows[z]);
        memcpy(sorted[z], counts + start[z], sizeof(uint32_t) * (size_t)rows[z]);
        qsort(sorted[z], (size_t)rows[z], sizeof(uint32_t), cmp_u32_desc);
    }
    free(start);
    *slack = 0;
    if (small_total > budget_bytes) {
        for (int32_t z = 0; z < n_tables; z++) free(sorted[z]);
        free(sorted);
        return OR_BUDGET_INFEASIBLE;
    }
    if (Tref == 0) Tref = 1;  /* no large table (or nothing accessed) */
    /* K_hi: every large table's cutoff exceeds its max count */
    uint64_t Khi = 1;
    for (int32_t z = 0; z < n_tables; z++) {
        if (!sorted[z] || rows[z] == 0) continue;
        uint64_t mk = sorted[z][0];
        int64_t Tz = T[z] > 0 ? T[z] : 1;
        unsigned __int128 need = ((unsigned __int128)(mk + 1) * (uint64_t)Tref + (uint64_t)Tz - 1) / (uint64_t)Tz;
        if ((uint64_t)need > Khi) Khi = (uint64_t)need;
    }
#define BYTES_AT(KK, OUT) do { \
        int64_t b_ = small_total; \
        for (int32_t z_ = 0; z_ < n_tables; z_++) if (sorted[z_]) { \
            uint64_t kz_ = T[z_] > 0 ? table_cutoff((KK), T[z_], Tref) : UINT64_MAX; \
            b_ += (int64_t)dim * 4 * count_ge(sorted[z_], rows[z_], kz_); } \
        (OUT) = b_; } while (0)
    int64_t b1;
    BYTES_AT(1, b1);
    uint64_t K;
    if (b1 <= budget_bytes) { K = 1; *slack = 1; }
    else {
        uint64_t lo = 1, hi = Khi;   /* bytes(lo) > L, bytes(hi) <= L */
        while (hi - lo > 1) {
            uint64_t mid = lo + (hi - lo) / 2;
            int64_t bm;
            BYTES_AT(mid, bm);
            if (bm <= budget_bytes) hi = mid; else lo = mid;
        }
        K = hi;
    }
#undef BYTES_AT
    for (int32_t z = 0; z < n_tables; z++)
        kmin[z] = sorted[z] ? (T[z] > 0 ? (int64_t)table_cutoff(K, T[z], Tref) : INT64_MAX) : 0;
    *K_out = K;
    *t_final = (double)K / ((double)Tref * x_pct / 100.0);
    for (int32_t z = 0; z < n_tables; z++) free(sorted[z]);
    free(sorted);
    return OR_OK;
}

/* bytes of the hot set for a given per-table kmin (used by tests as the
 * brute-force definition of bytes(K)). */
int64_t or_hot_bytes(int32_t n_tables, const int64_t* rows, int32_t dim,
                     int64_t small_bytes, const uint32_t* counts,
                     const int64_t* kmin)
{
    int64_t b = 0, g = 0;
    for (int32_t z = 0; z < n_tables; z++) {
        if (is_small(rows[z], dim, small_bytes)) b += rows[z] * (int64_t)dim * 4;
        else for (int64_t j = 0; j < rows[z]; j++)
            if ((int64_t)counts[g + j] >= kmin[z]) b += (int64_t)dim * 4;
        g += rows[z];
    }
    return b;
}

/* ---------------------------------------------------------------------------
 * ESTIMATE (§4.1.2, Eqs. 2-4) for ONE large table with logger
 * k[0..N_z) and cutoff kmin (= ceil(H_zt)):
 *  1. N = floor(N_z / m) full m-sized chunks (R7: aligned, disjoint).  If
 *     N < n: full scan, exact (flag = 1).
 *  2. pick the n chunks c in [0, N) with the smallest (key(chunk_seed, c), c)
 *     ("random chunks"), in ascending c.
 *  3. Eq. 2: C_i = #{j in chunk c_i : k_j >= H_zt}.
 *  4. Eq. 3: ybar = sum C_i / n (summed in ascending c, double).
 *  5. s^2 = sum (C_i - ybar)^2 / (n - 1) (R8, two-pass).
 *  6. Eq. 4: hw = t_q * sqrt(((N - n)/N) * (s^2 / n)); t_q = t_{alpha/2} with
 *     n-1 degrees of freedom, supplied by the caller (R9).
 *  7. est = ybar * N_z / m; lo/hi = (ybar -/+ hw) * N_z / m clamped [0, N_z].
 * out[0..5] = {ybar, s, lo_rows, hi_rows, est_rows, exact_flag};
 * C_out[n], chunk_out[n] receive C_i and the chosen chunk ids.
 * ------------------------------------------------------------------------- */
void or_estimate(const uint32_t* k, int64_t Nz, int64_t kmin, int32_t n,
                 int32_t m, uint64_t chunk_seed, double t_q, double* out,
                 int64_t* C_out, int64_t* chunk_out)
{
    int64_t N = Nz / m;
    if (N < n) {
        int64_t exact = 0;
        for (int64_t j = 0; j < Nz; j++) if ((int64_t)k[j] >= kmin) exact++;
        out[0] = 0.0; out[1] = 0.0;
        out[2] = (double)exact; out[3] = (double)exact; out[4] = (double)exact;
        out[5] = 1.0;
        return;
    }
    or_pair* v = (or_pair*)malloc(sizeof(or_pair) * (size_t)N);
    for (int64_t c = 0; c < N; c++) { v[c].key = or_key(chunk_seed, (uint64_t)c); v[c].i = c; }
    qsort(v, (size_t)N, sizeof(or_pair), cmp_pair);
    int64_t* chosen = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int32_t i = 0; i < n; i++) chosen[i] = v[i].i;
    /* ascending c */
    for (int32_t i = 1; i < n; i++) {
        int64_t x = chosen[i]; int32_t j = i - 1;
        while (j >= 0 && chosen[j] > x) { chosen[j + 1] = chosen[j]; j--; }
        chosen[j + 1] = x;
    }
    double sum = 0.0;
    for (int32_t i = 0; i < n; i++) {
        int64_t C = 0;
        for (int64_t j = chosen[i] * m; j < (chosen[i] + 1) * m; j++)
            if ((int64_t)k[j] >= kmin) C++;
        C_out[i] = C;
        chunk_out[i] = chosen[i];
        sum += (double)C;
    }
    double ybar = sum / (double)n;
    double ss = 0.0;
    for (int32_t i = 0; i < n; i++) {
        double d = (double)C_out[i] - ybar;
        ss += d * d;
    }
    double s2 = n > 1 ? ss / (double)(n - 1) : 0.0;
    double hw = t_q * sqrt(((double)(N - n) / (double)N) * (s2 / (double)n));
    double scale = (double)Nz / (double)m;
    double lo = (ybar - hw) * scale, hi = (ybar + hw) * scale;
    if (lo < 0.0) lo = 0.0;
    if (hi > (double)Nz) hi = (double)Nz;
    out[0] = ybar; out[1] = sqrt(s2); out[2] = lo; out[3] = hi;
    out[4] = ybar * scale; out[5] = 0.0;
    free(v); free(chosen);
}

/* ---------------------------------------------------------------------------
 * Statistical optimizer, CLT-driven (§4.1.3: "invokes the profiler
 * with varying t (interim thresholds) ... tunes the threshold to be higher or
 * lower than the previous one"; the search rule is unstated — R27 takes
 * SPEC's calibrate):
 *   est_bytes(t) = sum_small N_z*D*4 + sum_large D*4*hi_z(t)
 * with hi_z(t) the Eq. 4 CI upper bound (rows) of table z's Eqs. 2-4
 * estimate (or_estimate, chunk seed chunk_seed ^ z) at kmin_z(t) =
 * max(1, ceil(((t*T_z)*x)/100)) (Eq. 1).  t is fit iff est_bytes(t) <= L.
 *   1. grid t_j = 10^(-8 + j/4), j = 0..28 (ratio 10^(1/4) over [1e-8, 1e-1]);
 *   2. t_28 not fit -> OR_BUDGET_INFEASIBLE; j* = the smallest fit j;
 *   3. j* = 0 -> t = t_0, slack = 1;
 *   4. else bisection on [lo, hi] = [t_{j*-1}, t_{j*}] for 8 steps:
 *      mid = (lo + hi) / 2 (R27: arithmetic midpoint); fit(mid) ? hi = mid :
 *      lo = mid;  t = hi.
 * Outputs t_final, kmin_z(t_final) (0 for small tables), the estimated bytes
 * at t_final and the number of est_bytes evaluations.
 * ------------------------------------------------------------------------- */
static double est_bytes_at(int32_t n_tables, const int64_t* rows, int32_t dim,
                           int64_t small_bytes, const uint32_t* counts,
                           const int64_t* T, double t, double x_pct, int32_t n,
                           int32_t m, uint64_t chunk_seed, double t_q)
{
    double b = 0.0, out[6];
    int64_t g0 = 0;
    int64_t* C = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* ch = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int32_t z = 0; z < n_tables; z++) {
        if (is_small(rows[z], dim, small_bytes)) {
            b += (double)(rows[z] * (int64_t)dim * 4);
        } else {
            int64_t kmin = or_kmin_from_cutoff(or_cutoff(t, T[z], x_pct));
            or_estimate(counts + g0, rows[z], kmin, n, m, chunk_seed ^ (uint64_t)z, t_q, out, C, ch);
            b += out[3] * (double)dim * 4.0;
        }
        g0 += rows[z];
    }
    free(C); free(ch);
    return b;
}

int or_clt_search(int32_t n_tables, const int64_t* rows, int32_t dim,
                  int64_t small_bytes, const uint32_t* counts, const int64_t* T,
                  double x_pct, int64_t budget_bytes, int32_t n, int32_t m,
                  uint64_t chunk_seed, double t_q, int64_t* kmin,
                  double* t_final, double* bytes_final, int32_t* slack,
                  int32_t* evals)
{
    double L = (double)budget_bytes, tg[29], b;
    int32_t j, jstar = -1;
    *evals = 0; *slack = 0;
    for (j = 0; j <= 28; j++) tg[j] = pow(10.0, -8.0 + 0.25 * (double)j);
    for (j = 0; j <= 28; j++) {
        b = est_bytes_at(n_tables, rows, dim, small_bytes, counts, T, tg[j], x_pct, n, m, chunk_seed, t_q);
        (*evals)++;
        if (b <= L) { jstar = j; break; }
    }
    if (jstar < 0) return OR_BUDGET_INFEASIBLE;
    double t = tg[jstar];
    if (jstar == 0) {
        *slack = 1;
    } else {
        double lo = tg[jstar - 1], hi = tg[jstar];
        for (int32_t it = 0; it < 8; it++) {
            double mid = (lo + hi) / 2.0;
            b = est_bytes_at(n_tables, rows, dim, small_bytes, counts, T, mid, x_pct, n, m, chunk_seed, t_q);
            (*evals)++;
            if (b <= L) hi = mid; else lo = mid;
        }
        t = hi;
    }
    *t_final = t;
    *bytes_final = est_bytes_at(n_tables, rows, dim, small_bytes, counts, T, t, x_pct, n, m, chunk_seed, t_q);
    for (int32_t z = 0; z < n_tables; z++)
        kmin[z] = is_small(rows[z], dim, small_bytes) ? 0 : or_kmin_from_cutoff(or_cutoff(t, T[z], x_pct));
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * O4  Hot-row remap for the embedding replicator ("extracts hot
 * embedding entries and creates embedding bags").  Tables concatenated in
 * order, rows ascending within a table (R16):
 *   base_z = sum_{z'<z} hot_rows_z';  remap[g] = base_z + #{hot j' < j in z}
 * for hot rows, -1 for cold.  base has n_tables+1 entries (base[n] = H_total).
 * ------------------------------------------------------------------------- */
int64_t or_remap(int32_t n_tables, const int64_t* rows, const uint8_t* hot,
                 int32_t* remap, int64_t* base)
{
    int64_t g = 0, run = 0;
    for (int32_t z = 0; z < n_tables; z++) {
        base[z] = run;
        for (int64_t j = 0; j < rows[z]; j++, g++)
            remap[g] = hot[g] ? (int32_t)(run++) : -1;
    }
    base[n_tables] = run;
    return run;
}

/* ---------------------------------------------------------------------------
 * O5  Input classifier (§4.2: "A sparse-input is classified as
 * hot only if all its embedding table accesses are to hot entries").  An
 * empty bag is vacuously hot (R19).  flag[r] = 1 hot, 0 cold.
 * ------------------------------------------------------------------------- */
void or_classify(int32_t n_tables, const int64_t* rows, const int32_t* idx,
                 const int64_t* off, int32_t fixed_pool, int64_t n_records,
                 const int32_t* remap, uint8_t* flag)
{
    int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tables + 1));
    int64_t tot = 0;
    for (int32_t z = 0; z < n_tables; z++) { base[z] = tot; tot += rows[z]; }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n_records; r++) {
        int hotr = 1;
        for (int32_t z = 0; z < n_tables; z++) {
            int64_t lo, hi;
            bag_range(off, fixed_pool, n_tables, r, z, &lo, &hi);
            for (int64_t p = lo; p < hi; p++)
                if (remap[base[z] + idx[p]] < 0) hotr = 0;
        }
        flag[r] = (uint8_t)hotr;
    }
    free(base);
}

/* ---------------------------------------------------------------------------
 * O6  Mini-batch bundling ("bundles hot and cold inputs together
 * into mini-batches").  hot_ids / cold_ids ascending record id
 * (R17).  Hot batch i = hot_ids[iB, min((i+1)B, n_hot)), trailing partial kept
 * (R18) — batches are implicit slices, so nothing else is stored.
 * Remapped hot CSR: for each hot record in order, for z = 0..Tn-1, for each
 * index in bag order, emit remap[g]; hot_off (only if off != NULL) holds the
 * cumulative bag offsets, n_hot*Tn + 1 entries.
 * out_counts = {n_hot, n_cold, n_hot_lookups}.
 * ------------------------------------------------------------------------- */
void or_pack(int32_t n_tables, const int64_t* rows, const int32_t* idx,
             const int64_t* off, int32_t fixed_pool, int64_t n_records,
             const int32_t* remap, const uint8_t* flag, int64_t* hot_ids,
             int64_t* cold_ids, int32_t* hot_idx, int64_t* hot_off,
             int64_t* out_counts)
{
    int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tables + 1));
    int64_t tot = 0;
    for (int32_t z = 0; z < n_tables; z++) { base[z] = tot; tot += rows[z]; }
    int64_t nh = 0, nc = 0, nl = 0;
    if (off && hot_off) hot_off[0] = 0;
    for (int64_t r = 0; r < n_records; r++) {
        if (!flag[r]) { cold_ids[nc++] = r; continue; }
        for (int32_t z = 0; z < n_tables; z++) {
            int64_t lo, hi;
            bag_range(off, fixed_pool, n_tables, r, z, &lo, &hi);
            for (int64_t p = lo; p < hi; p++) hot_idx[nl++] = remap[base[z] + idx[p]];
            if (off && hot_off) hot_off[nh * n_tables + z + 1] = nl;
        }
        hot_ids[nh++] = r;
    }
    out_counts[0] = nh; out_counts[1] = nc; out_counts[2] = nl;
    free(base);
}

/* ---------------------------------------------------------------------------
 * O7  Replicator extract: W_hot[remap[g]] = W[g], bit copy.
 * ------------------------------------------------------------------------- */
void or_extract(int64_t total_rows, int32_t dim, const float* W,
                const int32_t* remap, float* W_hot)
{
    for (int64_t g = 0; g < total_rows; g++)
        if (remap[g] >= 0)
            memcpy(W_hot + (int64_t)remap[g] * dim, W + g * dim, sizeof(float) * (size_t)dim);
}

/* ---------------------------------------------------------------------------
 * Swap sync back to the master tables (P:L299-302,
 * L540: at a hot -> cold swap the hot rows trained on the GPU are written to
 * the CPU master copy): W[g] = W_hot[remap[g]] for every hot row g; cold rows
 * are not touched.  The inverse of or_extract.
 * ------------------------------------------------------------------------- */
void or_scatter_hot(int64_t total_rows, int32_t dim, const float* W_hot,
                    const int32_t* remap, float* W)
{
    for (int64_t g = 0; g < total_rows; g++)
        if (remap[g] >= 0)
            memcpy(W + g * dim, W_hot + (int64_t)remap[g] * dim, sizeof(float) * (size_t)dim);
}

/* ---------------------------------------------------------------------------
 * O8  Hot embedding-bag forward ("embedding bags"; sum
 * pooling, R12):  Y[b,:] = sum_{p in bag b} W_hot[idx[p], :], accumulated in
 * fp64 in bag order and rounded once.  Bag b = lookups [off[b], off[b+1])
 * (absolute positions in idx) or [b*P, (b+1)*P) when off == NULL.  An empty
 * bag gives a zero row.  Returns OR_INDEX_RANGE on idx outside [0, H).
 * ------------------------------------------------------------------------- */
int or_emb_fwd(const float* W_hot, int64_t H, int32_t dim, const int32_t* idx,
               const int64_t* off, int32_t fixed_pool, int64_t n_bags, float* Y)
{
    int st = OR_OK;
#pragma omp parallel reduction(max : st)
    {
        double* acc = (double*)malloc(sizeof(double) * (size_t)dim);
#pragma omp for schedule(static)
        for (int64_t b = 0; b < n_bags; b++) {
            int64_t lo = off ? off[b] : b * fixed_pool;
            int64_t hi = off ? off[b + 1] : (b + 1) * fixed_pool;
            for (int32_t d = 0; d < dim; d++) acc[d] = 0.0;
            for (int64_t p = lo; p < hi; p++) {
                int32_t r = idx[p];
                if (r < 0 || r >= H) { st = OR_INDEX_RANGE; continue; }
                for (int32_t d = 0; d < dim; d++) acc[d] += (double)W_hot[(int64_t)r * dim + d];
            }
            for (int32_t d = 0; d < dim; d++) Y[b * dim + d] = (float)acc[d];
        }
        free(acc);
    }
    return st;
}

/* ---------------------------------------------------------------------------
 * O9  Hot backward + SGD ("massively-parallel Stochastic Gradient
 * Descent"; plain SGD, R13; sum semantics, R14):
 *   G[r,:] = sum_{p : idx[p] = r} dY[bag(p), :]   (fp64, ascending p)
 *   W_hot[r,:] = (float)((double)W_hot[r,:] - (double)lr * G[r,:])
 * for every touched r; untouched rows are not written.
 * slot: caller scratch int32[H], all -1 on entry, restored to -1 on exit (a
 * plain map from row to its accumulator; not part of the definition).
 * ------------------------------------------------------------------------- */
int or_emb_bwd_sgd(float* W_hot, int64_t H, int32_t dim, const int32_t* idx,
                   const int64_t* off, int32_t fixed_pool, int64_t n_bags,
                   const float* dY, float lr, int32_t* slot)
{
    int64_t L = off ? off[n_bags] - off[0] : n_bags * fixed_pool;
    int64_t p0 = off ? off[0] : 0;
    int32_t* rowlist = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L > 0 ? L : 1));
    double* G = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1) * (size_t)dim);
    int64_t U = 0;
    int st = OR_OK;
    /* touched rows, in first-touch order (integer bookkeeping) */
    for (int64_t b = 0; b < n_bags; b++) {
        int64_t lo = off ? off[b] : b * fixed_pool;
        int64_t hi = off ? off[b + 1] : (b + 1) * fixed_pool;
        for (int64_t p = lo; p < hi; p++) {
            int32_t r = idx[p];
            if (r < 0 || r >= H) { st = OR_INDEX_RANGE; continue; }
            if (slot[r] < 0) {
                slot[r] = (int32_t)U;
                rowlist[U] = r;
                for (int32_t d = 0; d < dim; d++) G[U * dim + d] = 0.0;
                U++;
            }
        }
    }
    /* G[r] += dY[bag(p)] for p ascending; with OpenMP row r is summed by
     * thread r mod nthreads only, in the same ascending-p order */
#pragma omp parallel
    {
        const int nt = or_nthreads(), me = or_thread();
        for (int64_t b = 0; b < n_bags; b++) {
            int64_t lo = off ? off[b] : b * fixed_pool;
            int64_t hi = off ? off[b + 1] : (b + 1) * fixed_pool;
            for (int64_t p = lo; p < hi; p++) {
                int32_t r = idx[p];
                if (r < 0 || r >= H || r % nt != me) continue;
                double* g = G + (int64_t)slot[r] * dim;
                for (int32_t d = 0; d < dim; d++) g[d] += (double)dY[b * dim + d];
            }
        }
    }
    (void)p0;
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < U; u++) {
        int32_t r = rowlist[u];
        for (int32_t d = 0; d < dim; d++) {
            float* w = W_hot + (int64_t)r * dim + d;
            *w = (float)((double)*w - (double)lr * G[u * dim + d]);
        }
        slot[r] = -1;
    }
    free(rowlist); free(G);
    return st;
}

/* Sparse gradient of O9 without the update (rows ascending): used by the
 * sync tests (O10: sum over ranks == gradient of the concatenated batch).
 * Returns U; rows_out[U], G_out[U*dim] (fp64). */
int64_t or_emb_grad(int64_t H, int32_t dim, const int32_t* idx,
                    const int64_t* off, int32_t fixed_pool, int64_t n_bags,
                    const float* dY, int32_t* rows_out, double* G_out)
{
    int64_t U = 0;
    uint8_t* touched = (uint8_t*)calloc((size_t)(H > 0 ? H : 1), 1);
    for (int64_t b = 0; b < n_bags; b++) {
        int64_t lo = off ? off[b] : b * fixed_pool;
        int64_t hi = off ? off[b + 1] : (b + 1) * fixed_pool;
        for (int64_t p = lo; p < hi; p++)
            if (idx[p] >= 0 && idx[p] < H) touched[idx[p]] = 1;
    }
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(H > 0 ? H : 1));
    for (int64_t r = 0; r < H; r++) {
        if (touched[r]) { pos[r] = U; rows_out[U] = (int32_t)r; U++; }
        else pos[r] = -1;
    }
    for (int64_t u = 0; u < U * dim; u++) G_out[u] = 0.0;
    for (int64_t b = 0; b < n_bags; b++) {
        int64_t lo = off ? off[b] : b * fixed_pool;
        int64_t hi = off ? off[b + 1] : (b + 1) * fixed_pool;
        for (int64_t p = lo; p < hi; p++) {
            int32_t r = idx[p];
            if (r < 0 || r >= H) continue;
            for (int32_t d = 0; d < dim; d++) G_out[pos[r] * dim + d] += (double)dY[b * dim + d];
        }
    }
    free(touched); free(pos);
    return U;
}
