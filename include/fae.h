/*
 * fae.h — C ABI of the B200-native FAE hot path (libfae.so).
 *
 * FAE = "Frequently Accessed Embeddings", Adnan et al., "Accelerating
 * Recommendation System Training by Leveraging Popular Choices",
 * arXiv 2103.00686.  Citations "P:Lnnn" are PAPER.md line numbers with the
 * section / equation they fall in; "Rnn" are the readings in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Plain C, no exceptions across the ABI; every call returns fae_status.
 *    Host-side argument validation happens before any launch; the message is
 *    retrievable with fae_last_error().
 *  - Pointers marked "device" are CUDA device pointers on the ctx's device
 *    (torch tensors' data_ptr()); "host" pointers are ordinary host memory.
 *    The caller owns every input and output buffer.  The ctx owns only its
 *    scratch workspace and the current hot set (bitmap + rank directory).
 *  - Work is enqueued on the ctx stream (fae_set_stream).  Calls that return
 *    host values (fae_profile, fae_threshold, fae_classify, fae_check,
 *    fae_sync_hot_grads' count) synchronise that stream; the step calls
 *    fae_emb_fwd / fae_emb_bwd_update do not, allocate nothing, and are
 *    CUDA-graph capturable (world == 1).
 *  - Device-side errors (an index outside its table, a non-finite update)
 *    are latched in the ctx and reported by the next synchronising call or
 *    fae_check() as FAE_ERR_INDEX_RANGE / FAE_ERR_NONFINITE.
 *  - One ctx per GPU / rank; a ctx is not thread-safe.
 *
 * Data layout:
 *  - Tables z = 0..Tn-1 with N_z rows of D fp32 values, concatenated in table
 *    order: global row g = rowbase_z + j, rowbase_z = sum_{z'<z} N_z'.
 *  - Sparse inputs: sample-major CSR.  Record r, table z is bag b = r*Tn + z.
 *    idx[] holds int32 LOCAL row ids (j in [0, N_z)).  Bag b's lookups are
 *    idx[off[b] .. off[b+1]) when off != NULL (int64 absolute positions),
 *    else idx[b*P .. (b+1)*P) with P = fixed_pool.
 *  - Hot ids: the compact replicated hot table W_hot[H_total][D] holds the
 *    hot rows in global-row order (R16): hot_id(g) = #{hot g' < g}.
 */
#ifndef FAE_H
#define FAE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fae_status {
    FAE_OK = 0,
    FAE_ERR_INVALID_ARG = 1,       /* bad argument (message in fae_last_error) */
    FAE_ERR_CAPACITY = 2,          /* exceeds a capacity fixed at fae_create   */
    FAE_ERR_BUDGET_INFEASIBLE = 3, /* small tables alone exceed the budget     */
    FAE_ERR_INDEX_RANGE = 4,       /* an index outside its table (latched)     */
    FAE_ERR_NONFINITE = 5,         /* non-finite gradient/update (latched)     */
    FAE_ERR_CUDA = 6,              /* CUDA runtime error                        */
    FAE_ERR_NCCL = 7,              /* NCCL error / async error                  */
    FAE_ERR_NOT_INIT = 8           /* NULL ctx, or comm needed but not inited  */
} fae_status;

typedef struct fae_ctx fae_ctx;

/* Capacities, fixed at create time: all workspace is allocated by fae_create
 * (profile/classify scratch grows on demand inside those one-off calls). */
typedef struct fae_config {
    int32_t device;             /* CUDA device ordinal                          */
    int32_t max_tables;         /* Tn capacity (<= 4096)                        */
    int64_t max_rows;           /* sum_z N_z capacity (hot-set bitmap)          */
    int64_t max_batch_lookups;  /* L capacity of one step (< 2^30)              */
    int64_t max_batch_bags;     /* S capacity of one step                       */
    int32_t max_dim;            /* D capacity                                   */
    int32_t max_world;          /* ranks capacity for fae_sync_hot_grads        */
} fae_config;

/* Table schema (host). */
typedef struct fae_tables {
    int32_t n_tables;
    const int64_t* rows;        /* host [n_tables]: N_z                         */
    int32_t dim;                /* D (fp32 elements per row)                    */
} fae_tables;

/* Sparse-input CSR (D1).  For a record shard on rank g of a
 * sharded dataset, record_base is the global id of local record 0 and
 * n_records_global the total over ranks (sampling keys use global ids, so a
 * sharded profile equals the unsharded one).  Single GPU: 0 and n_records. */
typedef struct fae_csr {
    const int32_t* idx;         /* device [n_lookups] local row ids             */
    const int64_t* off;         /* device [n_records*n_tables+1] or NULL        */
    int32_t fixed_pool;         /* lookups per bag when off == NULL (>= 0)      */
    int64_t n_records;          /* records in this shard                        */
    int64_t n_lookups;          /* off[n_records*n_tables] or n_records*Tn*P    */
    int64_t record_base;        /* global id of local record 0                  */
    int64_t n_records_global;   /* records over all ranks                       */
} fae_csr;

/* --------------------------------------------------------------------------
 * Lifecycle
 * ------------------------------------------------------------------------ */
fae_status fae_create(const fae_config* cfg, fae_ctx** out);
void fae_destroy(fae_ctx* ctx);
/* stream: a cudaStream_t passed as void* (NULL = legacy default stream). */
fae_status fae_set_stream(fae_ctx* ctx, void* stream);
const char* fae_last_error(const fae_ctx* ctx);
/* Synchronise the ctx stream and report (and clear) latched device errors. */
fae_status fae_check(fae_ctx* ctx);
/* NCCL bootstrap: rank 0 calls fae_get_nccl_id, the caller broadcasts the
 * 128 bytes (torch.distributed), every rank calls fae_comm_init.  world == 1
 * needs no comm. */
fae_status fae_get_nccl_id(void* id128);
fae_status fae_comm_init(fae_ctx* ctx, const void* id128, int32_t rank,
                         int32_t world);
/* TEST-ONLY transport ("virtual ranks"): `world` ctxs of ONE process on ONE
 * GPU, each driven by its own host thread, join the loopback group
 * `group_key` as ranks 0..world-1.  Every collective of the library (the
 * sharded profile's select histograms / candidates / loggers / T, the a11
 * count and payload all-gathers) then runs as a host rendezvous plus device
 * copies and a rank-ordered integer sum, instead of NCCL; all other code is
 * the same as with fae_comm_init.  Collectives block the calling thread
 * (each synchronises the ctx stream), so the world > 1 step calls are not
 * graph-capturable on this transport.  A peer that does not arrive within
 * 120 s breaks the group (FAE_ERR_NCCL on every member).
 * Errors: INVALID_ARG unless the environment has FAE_LOOPBACK=1, or bad
 * rank/world (world <= cfg.max_world). */
fae_status fae_comm_init_loopback(fae_ctx* ctx, uint64_t group_key,
                                  int32_t rank, int32_t world);
/* Number of kernels this ctx has launched so far (bench evidence). */
int64_t fae_kernel_launches(const fae_ctx* ctx);

/* --------------------------------------------------------------------------
 * fae_profile — input sampler + embedding logger (a1 + a2).
 *  P:L358-363 (§4.1.1): sample x% of the dataset D -> D-hat; uniform without
 *    replacement (R6): the k = floor(R*x/100) records with the smallest
 *    (key(seed, i), i), key(seed, i) = splitmix64(seed + (i+1)*0x9E3779B97F4A7C15),
 *    i = global record id; original order kept.
 *  P:L380-388 (§4.1.2 "Embedding Logger"): k_z[j] = number of sampled lookups
 *    equal to row j of table z (duplicates count each time).
 *  T_z = lookups into table z over ALL records (R3).
 * Arguments:
 *  counts       device uint32 [sum N_z], overwritten (concatenated loggers).
 *  T_host       host int64 [n_tables], out.
 *  sampled_ids  device int64 [>= k] local record ids of the sample, ascending
 *               (optional, NULL to skip).
 *  n_sampled    host out: k (this shard's share when sharded).
 * With a comm (world > 1) every rank passes its record shard; the selection
 * is global, counts and T are summed over ranks (exact, ncclAllReduce).
 * Errors: INVALID_ARG if x not in (0, 100] or schema mismatch; INDEX_RANGE
 * (latched) if a sampled index >= N_z; CAPACITY if n_tables > max_tables or
 * sum N_z > max_rows.
 * ------------------------------------------------------------------------ */
fae_status fae_profile(fae_ctx* ctx, const fae_tables* tabs,
                       const fae_csr* data, double x_pct, uint64_t seed,
                       uint32_t* counts, int64_t* T_host,
                       int64_t* sampled_ids, int64_t* n_sampled);

/* --------------------------------------------------------------------------
 * fae_threshold — threshold knob, embedding classifier and hot-row remap
 * (a3 + a4).
 *  Small-table rule: N_z*D*4 < small_table_bytes => all hot.
 *  FIXED_T (Eq. 1): H_z = ((t*T_z)*x)/100 in IEEE double (R21);
 *    large row hot iff k >= H_z (Eq. 2's >=, R1), i.e. k >= kmin_z =
 *    max(1, ceil(H_z)) (R25).
 *  BUDGET_EXACT ("top h entries that fit L", in Eq. 1 form, R10):
 *    with T_ref = max_large T_z and integer K >= 1, kmin_z = max(1,
 *    ceil(K*T_z/T_ref)); bytes(K) = sum_small N_z*D*4 + sum_large D*4*
 *    #{j: k_z[j] >= kmin_z}; the smallest K with bytes(K) <= budget.
 *    t_final = K / (T_ref*x/100).  budget_slack = 1 when K = 1 fits.
 *  CLT_SEARCH (the statistical optimizer; search rule R27 =
 *    SPEC calibrate S:L191-199): est_bytes(t) = small-table bytes + D*4 *
 *    sum over large tables of the Eq. 4 CI upper bound (rows) of the Eqs. 2-4
 *    estimate at the Eq. 1 cutoff (n, m, t_quantile, chunk_seed as below);
 *    t fits iff est_bytes(t) <= budget_bytes.  Grid t_j = 10^(-8 + j/4),
 *    j = 0..28: the first fitting t_j, then 8 bisection steps between t_j
 *    and t_{j-1} (midpoint (lo + hi) / 2, keep the fitting side); t_final =
 *    the fitting end; rows are then tagged with the EXACT counts at
 *    t_final's Eq. 1 cutoffs.  budget_slack = 1 if t_0 = 1e-8 fits;
 *    BUDGET_INFEASIBLE if t = 0.1 does not.
 *  ESTIMATE (want_estimate, Eqs. 2-4) at the final cutoff, per
 *    large table: n chunks of m rows with the smallest (key(chunk_seed ^ z,
 *    c), c), C_i (Eq. 2), ybar (Eq. 3), s (n-1 denominator, R8), CI with the
 *    finite-population factor (Eq. 4) and caller-supplied t_quantile (R9);
 *    est rows = ybar*N_z/m, bounds clamped to [0, N_z]; tables with fewer
 *    than n full chunks are scanned exactly (est_exact = 1).
 *  Remap (R16): hot_id(g) = #{hot g' < g}; base_z = hot_id of
 *    table z's first row; H_total = number of hot rows.
 * The resulting hot set is kept in the ctx (1 bit/row + rank directory,
 * 2 bits/row in HBM) and used by fae_classify / fae_extract.
 * Arguments:
 *  counts     device uint32 [sum N_z] from fae_profile.
 *  T_host     host int64 [n_tables].
 *  remap_out  device int32 [sum N_z], optional: hot id or -1 per row.
 *  res        host struct with caller-owned host arrays (NULL to skip each).
 * Errors: INVALID_ARG (t not in (0,1], bad mode, x not in (0,100], n < 2 or
 * m < 1); BUDGET_INFEASIBLE; CAPACITY.
 * ------------------------------------------------------------------------ */
typedef enum fae_thresh_mode {
    FAE_THRESH_FIXED_T = 0,
    FAE_THRESH_BUDGET_EXACT = 1,
    FAE_THRESH_CLT_SEARCH = 2
} fae_thresh_mode;

typedef struct fae_thresh_req {
    int32_t mode;               /* fae_thresh_mode                            */
    double t;                   /* FIXED_T threshold, fraction in (0, 1] (R2) */
    int64_t budget_bytes;       /* BUDGET_EXACT / CLT_SEARCH: L              */
    int64_t small_table_bytes;  /* default 1 << 20 (R11)                     */
    int32_t want_estimate;      /* compute Eqs. 2-4 at the final cutoff      */
    int32_t n_chunks;           /* n (35)                             */
    int32_t chunk_rows;         /* m (1024)                           */
    double t_quantile;          /* t_{alpha/2}, n-1 dof: 3.6007 @ 99.9% (R9) */
    uint64_t chunk_seed;
} fae_thresh_req;

typedef struct fae_thresh_result {
    /* per-table host arrays [n_tables] (each may be NULL) */
    int64_t* kmin;              /* cutoff used (0 for small tables)          */
    int64_t* hot_rows;          /* exact hot rows per table                  */
    int64_t* base;              /* [n_tables + 1] hot-id base per table      */
    int32_t* is_small;
    double* est_mean;           /* ybar                                      */
    double* est_sd;             /* s                                         */
    double* est_lo;             /* CI lower bound, rows                      */
    double* est_hi;             /* CI upper bound, rows                      */
    double* est_rows;           /* point estimate, rows                      */
    int32_t* est_exact;         /* 1 if full-scan fallback                   */
    /* scalars (out) */
    int64_t H_total;
    int64_t hot_bytes;          /* H_total * D * 4                           */
    double t_final;
    uint64_t K;                 /* BUDGET_EXACT integer cutoff (0 otherwise) */
    int32_t budget_slack;
} fae_thresh_result;

fae_status fae_threshold(fae_ctx* ctx, const fae_tables* tabs,
                         const uint32_t* counts, const int64_t* T_host,
                         double x_pct, const fae_thresh_req* req,
                         int32_t* remap_out, fae_thresh_result* res);

/* --------------------------------------------------------------------------
 * fae_classify — input classifier + mini-batch bundling (a5 + a6).
 *  P:L476-479 (§4.2): a sparse input is hot iff ALL its lookups hit hot rows
 *    (empty bags are vacuously hot, R19).
 *  bundle hot and cold inputs into all-hot / all-cold
 *    mini-batches.  hot_ids / cold_ids are ascending local record ids (R17);
 *    hot batch i = hot_ids[i*B, min((i+1)*B, n_hot)), trailing partial batch
 *    kept (R18).  The remapped hot CSR lists, for each hot record in order,
 *    for z = 0..Tn-1, the bag's hot ids in bag order; with explicit offsets
 *    hot_off[n_hot*Tn + 1] holds its absolute bag offsets (fixed pooling:
 *    implicit, hot_off unused).
 * Uses the hot set of the last fae_threshold on this ctx.
 * Arguments (fae_packed, device buffers caller-sized):
 *  hot_ids, cold_ids  int64 [>= n_records] each.
 *  hot_idx            int32 [>= n_lookups].
 *  hot_off            int64 [>= n_records*Tn + 1] (offsets input only).
 *  batch              B >= 1 (INVALID_ARG otherwise; B larger than a kind's
 *                     count gives one partial batch, not an error).
 *  shuffle_seed       must be 0 (stable order); other values INVALID_ARG.
 * Outputs (host fields): n_hot, n_cold, n_hot_lookups, n_hot_batches,
 * n_cold_batches.  Errors: NOT_INIT if no hot set; INDEX_RANGE (latched).
 * ------------------------------------------------------------------------ */
typedef struct fae_packed {
    int64_t* hot_ids;
    int64_t* cold_ids;
    int32_t* hot_idx;
    int64_t* hot_off;
    int64_t n_hot;
    int64_t n_cold;
    int64_t n_hot_lookups;
    int64_t n_hot_batches;
    int64_t n_cold_batches;
} fae_packed;

fae_status fae_classify(fae_ctx* ctx, const fae_tables* tabs,
                        const fae_csr* data, int32_t batch,
                        uint64_t shuffle_seed, fae_packed* out);

/* --------------------------------------------------------------------------
 * fae_extract — embedding replicator (a7: "extracts hot
 * embedding entries and creates embedding bags replicated across GPUs"):
 *   W_hot[hot_id(g), :] = W[g, :] for every hot global row g (bit copy).
 *  W      [sum N_z][dim] fp32: device memory, or pinned host memory mapped
 *         into the device address space (only hot rows cross the link).
 *  W_hot  device [H_total][dim].
 * ------------------------------------------------------------------------ */
fae_status fae_extract(fae_ctx* ctx, const float* W, int32_t dim,
                       float* W_hot);

/* --------------------------------------------------------------------------
 * fae_scatter_hot — the hot/cold swap synchronisation back to the master
 * tables (at a swap from
 * hot to cold mini-batches the hot rows trained on the GPU are written back
 * to the CPU master copy, the "embedding sync"):
 *   W[g, :] = W_hot[hot_id(g), :] for every hot global row g (bit copy);
 *   cold rows of W are not touched.  The inverse of fae_extract.
 *  W_hot  device [H_total][dim].
 *  W      [sum N_z][dim] fp32: device memory, or pinned host memory mapped
 *         into the device address space (only hot rows cross the link).
 * Uses the hot set of the last fae_threshold.  Asynchronous on the ctx
 * stream.  Errors: NOT_INIT without a hot set, INVALID_ARG.
 * ------------------------------------------------------------------------ */
fae_status fae_scatter_hot(fae_ctx* ctx, const float* W_hot, int32_t dim,
                           float* W);

/* --------------------------------------------------------------------------
 * fae_pack_cold — the cold mini-batches' CSR in GLOBAL row ids (SURVEY §8(f)
 * NEXT-1, the cold-batch side; a cold input touches cold
 * rows, so its embeddings train against the full tables — here the
 * HBM-resident master tables, with the same step calls, H = sum N_z):
 *   for each cold record k in order, z = 0..Tn-1, each lookup p of bag
 *   (cold_ids[k], z) in bag order: cold_idx[...] = base_z + idx[p],
 *   base_z = sum_{z' < z} N_z'.
 *  data      fixed pooling (off == NULL) or explicit offsets; device idx/off.
 *  cold_ids  device int64 [n_cold] (fae_classify's cold_ids), each in
 *            [0, data->n_records) (else INDEX_RANGE).
 *  cold_idx  device int32 [>= cold lookups], caller-owned (fixed pooling:
 *            n_cold*Tn*P; offsets: n_lookups - n_hot_lookups suffices).
 *  cold_off  device int64 [n_cold*Tn + 1], caller-owned, offsets input only
 *            (NULL with fixed pooling): cold bag b's lookups are
 *            cold_idx[cold_off[b] .. cold_off[b+1]).
 * Cold batch i = records [i*B, min((i+1)*B, n_cold)); train it with
 * fae_emb_fwd / fae_emb_bwd_update on W (H = sum N_z) after the hot rows
 * were written back (fae_scatter_hot), and re-extract before the next hot
 * batch.  Errors: INVALID_ARG (null buffers, n_cold > n_records, offsets
 * without cold_off), CAPACITY (sum N_z >= 2^31 - 1, the step calls' bound),
 * INDEX_RANGE (latched: a cold id or an index outside its table).
 * Synchronises the stream.
 * ------------------------------------------------------------------------ */
fae_status fae_pack_cold(fae_ctx* ctx, const fae_tables* tabs,
                         const fae_csr* data, const int64_t* cold_ids,
                         int64_t n_cold, int32_t* cold_idx,
                         int64_t* cold_off);

/* --------------------------------------------------------------------------
 * fae_emb_fwd — hot embedding-bag forward (a8; sum
 * pooling, R12):
 *   Y[b, :] = sum_{p in bag b} W_hot[idx[p], :]           (fp32)
 *  W_hot  device [H][D];  idx device int32 hot ids in [0, H).
 *  off    device int64 [n_bags+1] absolute positions into idx, or NULL for
 *         fixed pooling (bag b = idx[b*P .. (b+1)*P)).
 *  Y      device [n_bags][D] (sample-major [B][Tn][D]).
 * D % 4 == 0, D <= max_dim, and D/4 a power of two or a multiple of 32.
 * Empty bag -> zero row.  Asynchronous; graph-capturable.
 * ------------------------------------------------------------------------ */
fae_status fae_emb_fwd(fae_ctx* ctx, const float* W_hot, int64_t H, int32_t D,
                       const int32_t* idx, const int64_t* off,
                       int32_t fixed_pool, int64_t n_bags, float* Y);

/* --------------------------------------------------------------------------
 * fae_emb_bwd_update — hot embedding backward + SGD (a9 + a10 [+ a11]):
 *   G[r, :] = sum_{p : idx[p] = r} dY[bag(p), :]   (sort-and-segment)
 *   W_hot[r, :] -= lr * G[r, :]  for every touched r; untouched rows are not
 *   written (bit-identical).  P:L230, L803 ("massively-parallel SGD"), plain
 *   SGD (R13), sum semantics (R14: the caller pre-scales dY for a mean).
 * With a comm of world > 1 the sparse G is summed over ranks first (a11,
 * P:L298-301), deterministically, so every replica applies identical bits.
 * Same argument conventions as fae_emb_fwd; dY device [n_bags][D].
 * n_lookups must fit max_batch_lookups.  Asynchronous; graph-capturable
 * when world == 1.
 * ------------------------------------------------------------------------ */
fae_status fae_emb_bwd_update(fae_ctx* ctx, float* W_hot, int64_t H,
                              int32_t D, const int32_t* idx,
                              const int64_t* off, int32_t fixed_pool,
                              int64_t n_bags, const float* dY, float lr);

/* --------------------------------------------------------------------------
 * fae_sync_hot_grads — hot-gradient synchronisation across GPUs (a11,
 * "hot embeddings are synchronized using the AllReduce
 * collectives over the fast NVlink"; P:L217-220 aggregated gradients).
 * In:  rows device int32 [cap] sorted ascending, unique; vals device fp32
 *      [cap][D]; *count_host = local U.
 * Out: rows/vals = the global sparse sum over ranks (sorted by row, summed
 *      in rank order: identical bits on every rank); *count_host = global U.
 * Errors: NOT_INIT without comm (world 1 is the identity); CAPACITY if the
 * global U or world*max(U) exceeds cap or the ctx capacity; NCCL.
 * ------------------------------------------------------------------------ */
fae_status fae_sync_hot_grads(fae_ctx* ctx, int32_t* rows, float* vals,
                              int64_t* count_host, int64_t cap, int32_t D);

/* --------------------------------------------------------------------------
 * fae_group_batches — the backward's sort-and-segment (a9) for EVERY hot
 * batch of a packed dataset, computed once.  The hot CSR is static for the
 * whole run (the paper pre-processes once and stores the FAE format,
 * P:L262, L496), so grouping each batch's lookups by hot id is hoisted out of
 * the training step.  Per batch: a stable sort of (hot id, bag) and the
 * run-length segments of equal hot id (split into pieces of <= 16 lookups;
 * long segments into chunks reduced by separate CTAs, 512 lookups at
 * D <= 16 and 256 above, so the chunking depends on tabs->dim).
 * The grouping is kept in the ctx and refers to pk->hot_idx / pk->hot_off,
 * which must stay valid and unchanged until the next fae_group_batches.
 *  pk          the fae_packed filled by fae_classify (device hot_idx, hot_off;
 *              host n_hot, n_hot_lookups).
 *  fixed_pool  P of the input (0 = explicit offsets, hot_off used).
 *  batch       B (records per hot batch).
 *  H           rows of the hot table (hot ids must be < H).
 * Errors: INVALID_ARG, CAPACITY (>= 2^31 hot lookups), INDEX_RANGE.
 * ------------------------------------------------------------------------ */
fae_status fae_group_batches(fae_ctx* ctx, const fae_tables* tabs,
                             const fae_packed* pk, int32_t fixed_pool,
                             int32_t batch, int64_t H);

/* --------------------------------------------------------------------------
 * fae_release_scratch — free the build-only scratch of the last
 * fae_group_batches (sort keys and values, segment starts, next-batch
 * links, tile state: about 20 bytes per grouped lookup), keeping what
 * fae_train_hot_batches reads.  For runs that keep two groupings alive
 * (hot and cold batches of a mixed epoch, NEXT-1).  The next
 * fae_group_batches reallocates on demand.  Synchronises the stream.
 * Errors: NOT_INIT (null ctx), CUDA.
 * ------------------------------------------------------------------------ */
fae_status fae_release_scratch(fae_ctx* ctx);

/* --------------------------------------------------------------------------
 * fae_train_hot_batches — the hot mini-batch training loop over grouped
 * batches [first, first + n): for each batch i in order,
 *   Y = fwd(batch i)                                  (a8, as fae_emb_fwd)
 *   W_hot[r] -= lr * sum_{p: idx[p]=r} dY_i[bag(p)]   (a9 + a10 [+ a11])
 * with dY_i = dY + (i % n_dy) * (B*Tn) * D (device [n_dy][B*Tn][D]; the
 * upstream gradient of each step, e.g. written by the MLP backward) and Y
 * device [B*Tn][D] (overwritten every step).  Sequential SGD semantics:
 * batch i+1 sees the rows batch i updated.  World 1: replays a captured
 * CUDA graph (no host work per step) of, per step, ONE fused kernel (part R:
 * backward + SGD of batch i-1, writing each updated row straight into the
 * Y of batch i; part F: the forward of batch i's remaining rows) for
 * single-lookup bags with D <= 16, else two kernels (forward, backward +
 * SGD), chained by programmatic dependent launch; bit-identical either way.
 * FAE_FUSED=0/1 forces the choice; FAE_PERSIST=1 selects a cooperative
 * persistent kernel with a grid barrier per step (single-lookup bags; slower
 * on B200, kept for measurement).  World > 1 (or FAE_FORCE_MERGE=1 on a
 * 1-rank communicator): the sparse gradient is exchanged every step
 * (fae_sync_hot_grads semantics): per step, the forward, a reduce that
 * writes this rank's (row, G) list straight into its slot of the exchange
 * buffer, an in-place NCCL all-gather of xcap entries per rank (xcap = the
 * call's largest per-step U over ranks, known after one up-front count
 * exchange), and a rank-ordered merge + SGD kernel (world > 2: via a
 * [world][H] int32 row-position table allocated here); replayed from a
 * captured graph of 128 steps (NCCL transport) or a host loop (loopback
 * test transport).  Every rank passes the same n; a rank with fewer
 * batches than first + n contributes empty gradients.
 * H must equal the H given to fae_group_batches and D the tabs->dim given
 * to it (the long-segment chunking is sized for that row width).
 * ------------------------------------------------------------------------ */
fae_status fae_train_hot_batches(fae_ctx* ctx, float* W_hot, int64_t H,
                                 int32_t D, int64_t first, int64_t n,
                                 const float* dY, int64_t n_dy, float* Y,
                                 float lr);

/* --------------------------------------------------------------------------
 * Live kernel timing of fae_train_hot_batches (bench evidence).  enable:
 *  0 off;
 *  1 in-kernel %globaltimer stamps (min CTA start / max CTA end per launch):
 *    keeps the programmatic-dependent-launch overlap; each kernel's time is
 *    its exclusive share of the step (fwd(s) from the end of reduce(s-1),
 *    reduce(s) from the end of fwd(s));
 *  2 CUDA event nodes around each kernel in the graph (serialises kernels).
 * ms[0]/n[0]: forward kernel (k_grp_fwd_pdl), ms[1]/n[1]: segment-reduce +
 * SGD kernel (k_grp_reduce_pdl); mode 1 also reports ms[2] = summed lead of
 * each reduce's entry over its forward's end and n[2] = steps where the
 * reduce entered before the forward ended (PDL overlap evidence); n[3] = 1
 * when the fused single-kernel step ran (its time is in ms[1]/n[1]); n[3] = 2
 * when the persistent epoch kernel ran (ms[1]/n[1] = its CUDA-event time and
 * launches, ms[3] = the batches those launches trained); ms, n have 4
 * entries.  Enabling resets the totals.
 * ------------------------------------------------------------------------ */
fae_status fae_set_kernel_timing(fae_ctx* ctx, int32_t enable);
/* Grouping summary: info[8] = {n_batches, hot lookups, segments of more
 * than 16 lookups, segments (distinct hot rows summed over batches), max
 * long segments per batch, max bags per batch, free segments (rows of a
 * batch absent from the previous batch, summed), fused step in use}. */
fae_status fae_group_info(const fae_ctx* ctx, int64_t* info);
fae_status fae_get_kernel_timing(const fae_ctx* ctx, double* ms, int64_t* n);
/* Exchange-loop timing (a11; world > 1 or FAE_FORCE_MERGE),
 * accumulated by fae_train_hot_batches under fae_set_kernel_timing(1) and
 * reset by it.  out[6] (host):
 *  out[0] ms in the all-gather: from this rank's reduce-emit end (or the
 *         previous merge's end on a step with no local batch) to the first
 *         merge CTA's start, summed over timed steps;
 *  out[1] ms in the rank-ordered merge + SGD kernel, summed;
 *  out[2] steps timed;
 *  out[3] bytes one rank contributes to the all-gathers, summed over the
 *         call's steps: xcap * (4 + 4D) per step (xcap = the largest U of
 *         any rank and step of the call; every rank receives (world-1) times
 *         this);
 *  out[4] steps run; out[5] xcap of the last call.
 * Errors: INVALID_ARG (null). */
fae_status fae_get_exchange_timing(const fae_ctx* ctx, double* out);

/* ==========================================================================
 * Scheduler (§4.3 "Communication Overheads",
 * P:L538-572, Eq. 5 `eqn:scheduler` P:L550-557): the interleaving of cold
 * and hot mini-batches of an epoch and its loss-feedback rate.  Host-only
 * state machine (no GPU work); the caller runs the phases (e.g. the hot
 * loop on W_hot, the cold loop on the master tables) and reports the test
 * loss at every swap boundary.  Readings R28-R31:
 *  - R(r): a phase issues ceil(r% * the kind's per-epoch batch count)
 *    batches (>= 1) of one kind; r in [1, 100].
 *  - cold first, start R(50); once a kind is drained the
 *    rest of the other kind is one phase.
 *  - Eq. 5 at each swap with the post-swap test loss L_i: L_i > L_{i-1}
 *    halves r (clamp 1); else if the last u losses each strictly decreased
 *    (sliding window, u = 4) r doubles (clamp 100); else
 *    unchanged.  The first loss changes nothing.
 *  - each swap logs n_devices sync events of hot_bytes.
 *  - the rate persists across epochs (fae_sched_new_epoch).
 * The struct is caller-owned plain data; fields are read-only to callers.
 * ========================================================================== */
#define FAE_SCHED_COLD 0
#define FAE_SCHED_HOT 1
#define FAE_SCHED_MAX_U 64
typedef struct fae_sched {
    int64_t n[2];            /* batches per epoch: [COLD], [HOT] */
    int64_t done[2];         /* issued this epoch */
    double r;                /* current rate r(i), percent */
    int32_t u;               /* successive-decrease window */
    int32_t next_kind;       /* kind the next phase prefers */
    int32_t last_kind;       /* kind of the last issued phase, -1 none */
    int32_t n_hist;          /* losses kept (<= u + 1) */
    double hist[FAE_SCHED_MAX_U + 1];   /* the last n_hist losses, oldest first */
    int64_t swaps;           /* swap boundaries recorded (all epochs) */
    int64_t sync_events;     /* n_devices per swap */
    int64_t sync_bytes;      /* hot_bytes * n_devices per swap */
} fae_sched;

/* n_cold / n_hot >= 0 batches per epoch, r_start in [1, 100], u in
 * [1, FAE_SCHED_MAX_U].  Errors: INVALID_ARG. */
fae_status fae_sched_init(fae_sched* s, int64_t n_cold, int64_t n_hot,
                          double r_start, int32_t u);
/* Next phase: *kind (FAE_SCHED_COLD / HOT), batches [*first, *first +
 * *count) of that kind; *count = 0 once both kinds are drained.
 * *swap_after = 1 when a phase of the other kind will follow, i.e. the
 * caller must synchronise the hot rows and call fae_sched_record_swap with
 * the post-swap test loss before the next fae_sched_next.
 * Errors: INVALID_ARG (null). */
fae_status fae_sched_next(fae_sched* s, int32_t* kind, int64_t* first,
                          int64_t* count, int32_t* swap_after);
/* Swap boundary: sync accounting, then Eq. 5 with test_loss (finite).
 * Errors: INVALID_ARG (null, non-finite loss, n_devices < 1, hot_bytes < 0). */
fae_status fae_sched_record_swap(fae_sched* s, double test_loss,
                                 int64_t hot_bytes, int32_t n_devices);
/* Restart the epoch's queues (rate, history and counters persist). */
fae_status fae_sched_new_epoch(fae_sched* s);

/* ==========================================================================
 * DLRM hot step: the model a hot mini-batch trains
 * "entirely on the GPU" — bottom MLP over the dense features,
 * the embedding bags (a8), "dot" feature interaction, top MLP, logarithmic
 * loss, backward, SGD; widths from tab:benchmarks
 * (e.g. RMC2 13-512-256-64-16 / 512-256-1) or SYN-M1..M4
 * (P:L892-914).  Readings R32-R34: ReLU after every bottom
 * layer and every top layer but the last (linear logit, sigmoid inside the
 * loss); interaction input T = [bottom output, Y_0 .. Y_{Tn-1}], output
 * [bottom output, <T_i, T_j> for i > j in row-major (i, j) order]; loss =
 * mean over the batch of the log loss; plain SGD of every weight and bias.
 * Parameters: ONE caller-owned device fp32 buffer, per layer (bottom
 * first, then top) W [out][ld] row-major (ld = in rounded up to a multiple
 * of 4 floats, so every GEMM operand is 16-byte aligned; the GEMMs run
 * over the padded width, so the pad entries MUST be zero — they are read as
 * zero weights and stay zero) followed by b [out]; fae_dlrm_param_count
 * gives the length.
 * GEMMs through cuBLAS (tf32 = 1: TF32 on the tensor cores; 0: pedantic
 * fp32); everything else hand-written kernels; no allocation after create.
 * ========================================================================== */
#define FAE_DLRM_MAX_LAYERS 8
typedef struct fae_dlrm_cfg {
    int32_t n_dense;                        /* dense features per sample */
    int32_t n_bottom;                       /* bottom layers */
    int32_t bottom[FAE_DLRM_MAX_LAYERS];    /* widths; the last == dim */
    int32_t n_top;                          /* top layers */
    int32_t top[FAE_DLRM_MAX_LAYERS];       /* widths; the last == 1 */
    int32_t n_tables;                       /* sparse features Tn */
    int32_t dim;                            /* embedding dim D */
    int32_t max_batch;                      /* samples per mini-batch */
    int32_t tf32;                           /* 1: TF32 tensor-core GEMMs */
} fae_dlrm_cfg;
typedef struct fae_dlrm fae_dlrm;

/* Parameter count of the flat buffer (-1: invalid configuration). */
int64_t fae_dlrm_param_count(const fae_dlrm_cfg* cfg);
/* Allocates the activations, gradients, interaction tables and a cuBLAS
 * handle on ctx's device; uses ctx's stream.  Errors: INVALID_ARG, CUDA. */
fae_status fae_dlrm_create(fae_ctx* ctx, const fae_dlrm_cfg* cfg,
                           fae_dlrm** out);
void fae_dlrm_destroy(fae_dlrm* m);
/* One DLRM step on a batch of B <= max_batch samples (device pointers):
 * dense [B][n_dense], label [B] (0 / 1), Y [B][Tn][D] (the a8 output);
 * train = 1: backward + SGD of params (lr) and dY [B][Tn][D] = dL/dY (the
 * a9 input; L = mean log loss); train = 0: forward only.  The summed
 * per-sample loss and the sample count accumulate on the device
 * (fae_dlrm_loss).  Asynchronous.  Errors: INVALID_ARG. */
fae_status fae_dlrm_step(fae_dlrm* m, float* params, int32_t B,
                         const float* dense, const float* label,
                         const float* Y, float* dY, float lr, int32_t train);
/* Host read of the accumulated {sum of per-sample losses, samples};
 * reset = 1 zeroes them.  Synchronises the stream. */
fae_status fae_dlrm_loss(fae_dlrm* m, double* sum_loss, double* n_samples,
                         int32_t reset);
/* The model's internal Y / dY batch buffers and loss accumulator (device),
 * for callers that run a8 / a9 themselves. */
fae_status fae_dlrm_buffers(fae_dlrm* m, float** Y, float** dY,
                            double** loss_acc);
/* The full hot step over grouped hot batches [first, first + n) (after
 * fae_group_batches), world 1: per batch, the a8 forward of the grouped
 * loop into the model's Y, the DLRM forward + backward + SGD (lr_mlp) of
 * the batch's records (dense / label gathered through hot_ids: device
 * int64 [n_hot], dense [n_records][n_dense], label [n_records], indexed by
 * record id), then a9 + a10 on W_hot with the model's dY (lr_emb);
 * replayed from a captured graph of 128 steps.  Sequential semantics.
 * World > 1 (data parallel, every rank the same n): the loss is averaged
 * over the GLOBAL batch of each step (every rank's records), the MLP
 * gradient is all-reduced in ONE collective group with the hot-gradient
 * all-gathers of a11, then every rank applies the merged hot rows and
 * params -= lr_mlp * (summed gradient): replicas stay identical.
 * Errors: NOT_INIT (no grouping, or world > 1 without a comm), INVALID_ARG
 * (shapes differ from the grouping / model). */
fae_status fae_train_dlrm_batches(fae_ctx* ctx, fae_dlrm* m, float* params,
                                  float* W_hot, int64_t H, int32_t D,
                                  int64_t first, int64_t n,
                                  const int64_t* hot_ids, const float* dense,
                                  const float* label, float lr_mlp,
                                  float lr_emb);

#ifdef __cplusplus
}
#endif
#endif /* FAE_H */
