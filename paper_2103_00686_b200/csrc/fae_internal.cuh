// fae_internal.cuh — private declarations of libfae (B200 / sm_100a).
// Nothing here is shared with oracle/ (the oracle is an independent C file).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/fae.h"

namespace fae {

constexpr int kMaxTables = 4096;
constexpr int kSortBits = 8;           // radix digit width
constexpr int kSortBins = 1 << kSortBits;
constexpr int kSortThreads = 256;
constexpr int kSortItems = 4;          // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kMaxSortPasses = 4;      // 32-bit keys
constexpr int kPiece = 16;             // max lookups per reduction piece
constexpr int kUnroll = 128;           // steps per captured epoch graph
constexpr int kMedium = 128;           // segments of (kPiece, kMedium] lookups: one warp
// Lookups per long-segment CTA (one CTA pass).  Measured on B200: at D = 16
// (LPB = 4) with the fused step, 1024-chunks 6.59, 512 6.65, 2048 7.62 us
// per step (Kaggle-shaped); at D = 64 (LPB = 16) 256-chunks beat 512
// (reduce 17.0 vs 20.0 us per batch).
#ifndef FAE_CHUNK_SMALL
#define FAE_CHUNK_SMALL 1024
#endif
__host__ __device__ constexpr int chunk_of_lpb(int lpb) { return lpb <= 4 ? FAE_CHUNK_SMALL : 256; }
inline int chunk_for_dim(int D) { return chunk_of_lpb(D / 4 < 32 ? D / 4 : 32); }
// reduce blocks of a batch's medium segments: one warp each when a warp holds
// >= 8 lane groups (LPB <= 4), else one CTA each (single-chunk long path)
__host__ __device__ inline int64_t med_blocks_for(int64_t n_med, int lpb) {
    return lpb <= 4 ? (n_med + 7) / 8 : n_med;
}
// the two-kernel reduce (reduce_segments): at LPB >= 8 a medium segment
// (<= kMedium lookups = 8 pieces) takes 8 lane groups, so a CTA holds
// 32 / LPB of them (FAE_MED_PACK=0: one CTA each, as the fused step)
#ifndef FAE_MED_PACK
#define FAE_MED_PACK 1
#endif
__host__ __device__ constexpr int med_per_cta(int lpb) { return (FAE_MED_PACK && lpb >= 8 && lpb < 32) ? 32 / lpb : 1; }
__host__ __device__ inline int64_t med_blocks_red(int64_t n_med, int lpb) {
    return lpb <= 4 ? (n_med + 7) / 8 : (n_med + med_per_cta(lpb) - 1) / med_per_cta(lpb);
}
constexpr int kStampSlots = 16;        // timing stamps per step (epoch runner)
constexpr int kMaxPersistCtas = 2048;  // persistent kernel: barrier flag slots
constexpr int kTinySeg = 4;            // segments of <= kTinySeg lookups: 4 per lane group
constexpr int kGSThreads = 256;        // grouping sort: threads per tile
constexpr int kGSItems = 16;           // grouping sort: items per thread
constexpr int kGSTile = kGSThreads * kGSItems;   // 4096 lookups per tile

// error latch bits (device word)
constexpr uint32_t kErrIndex = 1u;
constexpr uint32_t kErrNonfinite = 2u;
constexpr uint32_t kErrOverflow = 4u;
constexpr uint32_t kErrBarrier = 8u;    // persistent kernel: grid barrier timed out

// Look-back status words: 2 flag bits on top of the value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// Collectives (coll.cu): NCCL or the test-only loopback transport.
enum class CollT { U32, I32, I64, U64, F32 };
struct LbMember;

// Step workspace: everything fae_emb_bwd_update needs, allocated at create.
struct StepWs {
    int64_t cap_L = 0;                  // lookups capacity
    uint32_t* keys[2] = {nullptr, nullptr};
    int32_t* vals[2] = {nullptr, nullptr};
    // zeroed region (one memset per call): digit histograms, tile counters,
    // look-back status words, scalars.
    void* zero_base = nullptr;
    size_t zero_bytes = 0;
    uint32_t* ghist = nullptr;          // [kMaxSortPasses][256]
    uint32_t* tile_ctr = nullptr;       // [8]
    uint32_t* sort_status = nullptr;    // [kMaxSortPasses][tiles][256]
    uint64_t* piece_status = nullptr;   // [tiles]
    int64_t* scalars = nullptr;         // [0]=n_valid [1]=n_pieces [2]=n_segs
    // not zeroed per call
    int32_t* piece_start = nullptr;     // [cap_P + 1]
    int32_t* piece_seg = nullptr;       // [cap_P]
    int32_t* seg_first = nullptr;       // [cap_L + 1]
    int32_t* seg_row = nullptr;         // [cap_L]
    uint32_t* seg_cnt = nullptr;        // [cap_L], kept zero by the finisher
    float* partial = nullptr;           // [cap_P][max_dim]
    float* grad = nullptr;              // [cap_L][max_dim] emitted sparse G
    int64_t cap_P = 0;
    int64_t n_sort_tiles = 0;
    int64_t n_piece_tiles = 0;
};

// Hot set produced by fae_threshold: 16-byte entries per 64 rows
// {bits lo, bits hi, exclusive hot-rank prefix, unused}.
struct HotSet {
    bool valid = false;
    int32_t n_tables = 0;
    int32_t dim = 0;
    int64_t total_rows = 0;
    int64_t H_total = 0;
    std::vector<int64_t> rows, rowbase, base;   // host copies
    uint4* dir = nullptr;                       // device [ceil(total/64)]
    int64_t dir_cap = 0;
    int64_t* d_rowbase = nullptr;               // device [n_tables + 1]
};

// Grouping of a packed dataset's hot batches (fae_group_batches): the
// backward's sort-and-segment result per batch, computed once.
struct BatchDesc {
    int64_t lk0, lk1;      // lookups [lk0, lk1) of hot_idx (global positions)
    int64_t bag0;          // global bag index of the batch's first bag
    int64_t sb0, sb1;      // segments [sb0, sb1) (records: short first)
    int32_t n_short;       // segments of <= kPiece lookups (records first)
    int32_t n_med;         // then segments of <= kMedium lookups; then the long ones
    int32_t n_bags;
    int32_t n_free;        // segments whose row is not in batch b-1 (FreeRecs at sb0)
    int32_t n_lchunk;      // chunks of the long segments (one CTA each)
    int32_t n_tiny;        // leading segments of <= kTinySeg lookups (4 per lane group)
};

// One segment (a run of equal hot ids in a grouped batch), batch-local
// indices, 32 bytes.  Per batch the records are stably partitioned by length:
// <= kTinySeg lookups (4 per lane group), <= kPiece (one lane group each),
// <= kMedium (one warp each), longer (one CTA per chunk_for_dim lookups).
struct alignas(16) SegRec {
    int32_t pos;    // first position of the segment in the batch
    int32_t len;    // lookups of the segment
    int32_t row;    // hot id
    int32_t seg;    // segment index in the batch (ascending hot id)
    int32_t npos;   // same row in the NEXT batch: its first position, or -1
    int32_t nlen;   //   and its number of lookups (0 if absent)
    int32_t c0;     // long segments: index of its first chunk in the batch
    int32_t nc;     //   and its number of chunks (1 otherwise)
};

// A segment of batch b whose row is not in batch b-1 (the fused step gathers
// it for the forward of batch b); 16 bytes.
struct alignas(16) FreeRec {
    int32_t pos, len, row, pad;
};

// Long-chunk -> long-segment map (Group::lmap) of batch `bi`: its slice
// starts at lk0 / 64 + bi.  A batch has at most L_b / 128 chunks (every long
// segment has > kMedium = 128 lookups and a chunk >= 128), so the slices of
// consecutive batches never overlap; capacity L_total / 64 + n_batches + 1.
// the fused one-kernel step applies (single-lookup bags, world 1)
struct Ctx;
bool fused_step(const Ctx* c);

__host__ __device__ inline int64_t lmap_base(const BatchDesc& d, int64_t bi) { return d.lk0 / 64 + bi; }

struct Group {
    bool valid = false;
    int64_t n_batches = 0, L_total = 0, S_total = 0, n_long_total = 0;
    int32_t Tn = 0, P = 0, B = 0, dim = 0;
    int64_t H = 0;
    int64_t max_bags = 0, max_lookups = 0, max_short = 0, max_med = 0, max_long = 0, max_segs = 0;
    const int32_t* hot_idx = nullptr;
    const int64_t* hot_off = nullptr;
    BatchDesc* desc = nullptr;        // device [n_batches]
    std::vector<BatchDesc> hdesc;     // host copy
    int64_t cap_B = 0;
    // grouping result
    int32_t* perm = nullptr;          // [L_total] local bag index, grouped by hot id
    SegRec* rec = nullptr;            // [S_total]
    FreeRec* freer = nullptr;         // [S_total] (per batch at sb0, n_free entries)
    int32_t* nxt = nullptr;           // [S_total] link to the next batch's segment (local) or -1
    int64_t max_free = 0;
    int64_t max_lchunk = 0;
    int32_t chunk = 512;              // lookups per long-segment chunk (chunk_for_dim)
    float* lpart = nullptr;           // [kUnroll][max_lchunk][8][max_dim] chunk block sums
    uint32_t* lcnt = nullptr;         // [kUnroll][max_long] arrival counters (kept zero)
    int64_t cap_lpart = 0, cap_lcnt = 0;
    int64_t cap_L = 0, cap_R = 0;
    int64_t cap_rec = 0, cap_free = 0, cap_nxt = 0;   // sized by the segment count
    // grouping scratch (kept for reuse)
    uint32_t* keys[2] = {nullptr, nullptr};
    int32_t* vals = nullptr;          // [L_total] (second value buffer is perm)
    int64_t* seg_start = nullptr;     // [cap_S] global position of each segment
    int32_t* seg_row = nullptr;       // [cap_S] hot id of each segment (ascending per batch)
    int64_t cap_S = 0;
    int64_t* tile_start = nullptr;    // [n_tiles + 1] global positions
    int32_t* tile_batch = nullptr;    // [n_tiles] (bit 31: first tile of its batch)
    uint32_t* sstatus = nullptr;      // [n_tiles][256] digit look-back
    uint64_t* pstatus = nullptr;      // [n_tiles] segment look-back
    uint32_t* ghist = nullptr;        // [n_batches][kMaxSortPasses][256]
    int64_t cap_T = 0, cap_Hh = 0;
    // epoch runner
    int64_t* cursor = nullptr;        // device: [0] base / cursor, [2] first, [3] n, [4] exchange steps
    int64_t* run = nullptr;
    uint32_t* done_ctr = nullptr;
    int32_t* lmap = nullptr;          // long chunk -> long record index (lmap_base per batch)
    int32_t* xcnt = nullptr;          // world > 1: every step's per-rank gradient sizes
    int64_t cap_xcnt = 0;
    int32_t* ptab = nullptr;          // world > 2: [world][H] row -> position in a rank's gathered list
    int64_t cap_ptab = 0;
    cudaGraphExec_t xgraph = nullptr; // world > 1 (NCCL): kUnroll exchange steps
    uint64_t xgraph_key = 0;
    int64_t xcap_last = 0;            // entries per rank of the last call's exchange (padded)
    int64_t cap_lmap = 0;
    uint32_t* pbar = nullptr;         // persistent kernel: [0] arrivals, [1] abort, [2 + 32 c] CTA c's flag

    cudaGraphExec_t graph = nullptr;
    int graph_steps = 0;
    uint64_t graph_key = 0;
    cudaGraphExec_t tgraph[2] = {nullptr, nullptr};
    cudaEvent_t tev[2][3 * kUnroll] = {};
    uint64_t tgraph_key = 0;
    unsigned long long* stamps = nullptr;
    int64_t stamp_cap = 0;
    unsigned long long* h_stamps = nullptr;   // pinned: deferred harvest of the last timed call
    int64_t h_stamps_cap = 0;
    cudaEvent_t h_ev = nullptr;
    int64_t h_pending_n = 0;
    bool h_pending_fused = false;
};

struct Ctx {
    fae_config cfg{};
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint32_t* d_err = nullptr;                  // latched device error bits
    int64_t launches = 0;
    StepWs ws;
    HotSet hs;
    // grow-on-demand scratch for the one-off calls
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    int64_t* d_rowbase_tmp = nullptr;           // [max_tables+1]
    int64_t* d_rows_tmp = nullptr;              // [max_tables]
    // collectives: NCCL communicator or loopback virtual-rank group (tests)
    ncclComm_t comm = nullptr;
    LbMember* lb = nullptr;
    int rank = 0, world = 1;
    int64_t* g_flag = nullptr;                  // [2] coll_agree scratch
    // sync scratch
    int32_t* g_rows = nullptr;                  // [max_world * cap_L]
    float* g_vals = nullptr;                    // [max_world * cap_L * max_dim]
    // exchange loops: odd steps use a second slot set, so a step's reduce-emit
    // never waits for the previous step's merge (grown on demand)
    int32_t* g_rows2 = nullptr;
    float* g_vals2 = nullptr;
    int64_t g_cap2 = 0;                         // entries of g_rows2 (world * xcap)
    int32_t* g_counts = nullptr;                // [max_world]
    int64_t g_cap = 0;
    Group grp;
    // kernel timing (fae_set_kernel_timing): accumulated over timed calls
    int timing = 0;                   // 0 off, 1 in-kernel stamps, 2 graph events
    double t_ms[2] = {0.0, 0.0};      // [0] fwd kernel, [1] reduce kernel
    int64_t t_n[2] = {0, 0};
    int64_t t_overlap_n = 0;          // steps whose reduce entered before the fwd ended
    double t_red_entry_lead_ms = 0.0; // sum of (fwd end - reduce entry)
    double t_tier_ms[2] = {0.0, 0.0}; // reduce tiers' completion after fwd end
    double t_x_ms[2] = {0.0, 0.0};    // exchange loop: [0] all-gather (reduce end -> merge entry), [1] merge
    int64_t t_x_n = 0;                // steps timed by t_x_ms
    double t_x_bytes = 0.0;           // slot bytes one rank contributes, summed over timed steps
    int64_t t_x_steps = 0;
    bool no_pdl = false;              // FAE_NO_PDL=1: plain serialized launches
    int fused_mode = -1;              // FAE_FUSED: -1 auto (D <= 16), 1 on, 0 off (P = 1, world 1)
    bool t_fused = false;             // timing came from the fused kernel
    bool t_persist = false;           // timing came from the persistent kernel
    int64_t t_persist_batches = 0;    // batches trained by the timed persistent launches
    bool persist = false;             // FAE_PERSIST=1: the persistent grid-barrier kernel
    int persist_mb = 0;               // FAE_PERSIST_MB: CTAs per SM (0 = occupancy limit)
    bool merge_sort = false;          // FAE_MERGE_SORT=1: sort-based merge of the exchanged gradients
    int merge_table = -1;             // FAE_MERGE_TABLE: exchange merge by position table (1) / search (0) / auto
    bool force_merge = false;         // FAE_FORCE_MERGE=1: the multi-rank exchange loop even at world 1 (tests)
    bool gs_generic = false;          // FAE_GS_GENERIC=1: radix-pass grouping even where the unit path applies
    bool cls_legacy = false;          // FAE_CLS_LEGACY=1: the round-1 one-tile-per-CTA classify kernel
    int red_mb = 4;                   // FAE_RED_MB: min resident reduce CTAs per SM (4/6/8)
    int pdl_trig = 0;                 // FAE_PDL_TRIG bit0: reduce triggers after its wait, bit1: fwd too
};

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
fae_status set_err(Ctx* c, fae_status st, const std::string& msg);
fae_status cuda_err(Ctx* c, cudaError_t e, const char* where);
void* scratch(Ctx* c, size_t bytes);   // ctx-owned, grows; nullptr on failure
fae_status read_latched(Ctx* c);       // sync + read/clear device error word

#define FAE_CUDA(c, expr)                                                   \
    do {                                                                    \
        cudaError_t e_ = (expr);                                            \
        if (e_ != cudaSuccess) return ::fae::cuda_err((c), e_, #expr);      \
    } while (0)

#define FAE_LAUNCHED(c)                                                     \
    do {                                                                    \
        (c)->launches++;                                                    \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) return ::fae::cuda_err((c), e_, "launch");   \
    } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// collectives (coll.cu)
inline bool has_comm(const Ctx* c) { return c->comm != nullptr || c->lb != nullptr; }
fae_status coll_allreduce_sum(Ctx* c, void* buf, int64_t count, CollT t, const char* who);
fae_status coll_allgather(Ctx* c, const void* send, void* recv, int64_t count, CollT t, const char* who);
void coll_group_start(Ctx* c);
fae_status coll_group_end(Ctx* c, const char* who);
fae_status coll_async_error(Ctx* c, const char* who);
fae_status coll_agree(Ctx* c, fae_status local, const char* who);
fae_status comm_bufs(Ctx* c);
void coll_free(Ctx* c);

// step internals (step.cu), used by sync
fae_status bwd_group_and_reduce(Ctx* c, float* W_hot, int64_t H, int32_t D,
                                const uint32_t* keys_in_or_null,
                                const int32_t* idx, const int64_t* off,
                                int32_t fixed_pool, int64_t n_bags,
                                int64_t n_hint, const float* src, float lr,
                                bool emit);
fae_status sync_merge_apply(Ctx* c, const int32_t* rows, const float* vals, int64_t U, int32_t D,
                            float* W, int64_t H, float lr, int32_t* out_rows, float* out_vals,
                            int64_t* out_count, int64_t out_cap, const int32_t* known_counts = nullptr,
                            int64_t known_cap = 0);
fae_status step_ws_alloc(Ctx* c);
// persistent epoch kernel (persist.cu): batches [first, first + n) of the
// grouping, world 1, single-lookup bags; ev (optional) brackets the launch
fae_status launch_train_persist(Ctx* c, float* W, int D, const float* dY, int64_t n_dy, float* Y, float lr,
                                int64_t first, int64_t n, cudaEvent_t* ev);
void group_free(Ctx* c);
// exchange runs (epoch.cu): setup and the pieces the DLRM exchange step reuses
struct XPrep {
    int64_t xcap = 0;
    int32_t* per_step = nullptr;   // device [n][world] segment counts
    bool table = false;
};
fae_status x_prepare(Ctx* c, int64_t first, int64_t n, int64_t H, int32_t** rec_total, XPrep* out);
fae_status launch_grp_fwd_x(Ctx* c, cudaStream_t st, int s, float* W, int64_t H, int D, float* Y);
fae_status launch_xreduce_plain(Ctx* c, cudaStream_t st, int s, int D, const float* dY, int64_t xcap);
// the exchange slot set of replay step s (even: g_rows / g_vals, odd: g_rows2 / g_vals2)
inline int32_t* xrows_of(Ctx* c, int s) { return (s & 1) ? c->g_rows2 : c->g_rows; }
inline float* xvals_of(Ctx* c, int s) { return (s & 1) ? c->g_vals2 : c->g_vals; }
fae_status launch_xmerge_any(Ctx* c, cudaStream_t st, int s, int last, float* W, int64_t H, int D, float lr,
                             int64_t xcap, const int32_t* per_step, bool table);
fae_status validate_schema(Ctx* c, const fae_tables* t, const char* who);
void step_ws_free(Ctx* c);

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ uint64_t hash_key(uint64_t seed, uint64_t i) {
    return mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Decoupled look-back (single thread): publish this tile's aggregate, walk
// back to the nearest inclusive prefix, publish the inclusive prefix, return
// the exclusive prefix.  Values are < 2^62 and may be packed sums of
// non-overflowing fields.
__device__ __forceinline__ uint64_t lookback_u64(uint64_t* status, int64_t tile,
                                                 uint64_t agg) {
    if (tile == 0) {
        st_relaxed_u64(&status[0], kFlagPre | agg);
        return 0;
    }
    st_relaxed_u64(&status[tile], kFlagAgg | agg);
    uint64_t excl = 0;
    int64_t t = tile - 1;
    while (true) {
        uint64_t s;
        do {
            s = ld_relaxed_u64(&status[t]);
        } while ((s >> 62) == 0);
        excl += s & kValMask;
        if ((s >> 62) == 2) break;
        --t;
    }
    st_relaxed_u64(&status[tile], kFlagPre | (excl + agg));
    return excl;
}

// 1-D bulk copies global -> shared through the async (TMA) engine, completion
// counted on an mbarrier (cp.async.bulk ... mbarrier::complete_tx::bytes).
// dst / src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier inits visible to the async proxy
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's (and, after a __syncthreads, the block's) generic-proxy
// shared-memory accesses before later async-proxy writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// L2 eviction-priority policies (createpolicy) and their use on a bulk copy
// and on a read-only 16-byte load: a streamed operand marked evict-first
// keeps a small, reused structure (marked evict-last) resident in L2
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint4 ldg_hint_u4(const uint4* p, uint64_t policy) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ int32_t ldg_hint_i32(const int32_t* p, uint64_t policy) {
    int32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

// Split look-back: publish a tile's aggregate now (tile 0: its inclusive
// prefix), finish the walk later — a CTA can do other work in between, so by
// the time it walks, its predecessors have published.
__device__ __forceinline__ void lookback_publish(uint64_t* status, int64_t tile, uint64_t agg) {
    st_relaxed_u64(&status[tile], (tile == 0 ? kFlagPre : kFlagAgg) | agg);
}
__device__ __forceinline__ uint64_t lookback_finish(uint64_t* status, int64_t tile, uint64_t agg) {
    if (tile == 0) return 0;
    uint64_t excl = 0;
    int64_t t = tile - 1;
    while (true) {
        uint64_t s;
        do {
            s = ld_relaxed_u64(&status[t]);
        } while ((s >> 62) == 0);
        excl += s & kValMask;
        if ((s >> 62) == 2) break;
        --t;
    }
    st_relaxed_u64(&status[tile], kFlagPre | (excl + agg));
    return excl;
}

// lookback_finish by a whole warp: 32 predecessors per step (the walk from a
// tile back to the nearest published inclusive prefix is up to a few hundred
// tiles when hundreds of CTAs classify concurrently).  All 32 lanes call it;
// every lane returns the exclusive prefix.
__device__ __forceinline__ uint64_t lookback_finish_warp(uint64_t* status, int64_t tile, uint64_t agg) {
    if (tile == 0) return 0;
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t base = tile - 1;
    while (true) {
        const int64_t t = base - lane;
        uint64_t s = t >= 0 ? ld_relaxed_u64(&status[t]) : kFlagPre;   // before tile 0: inclusive 0
        while (__any_sync(0xffffffffu, (s >> 62) == 0))
            if ((s >> 62) == 0) s = ld_relaxed_u64(&status[t]);
        const uint32_t pm = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        uint64_t v = s & kValMask;
        const int first = pm ? __ffs(pm) - 1 : 32;   // nearest inclusive prefix in the window
        if (lane > first) v = 0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pm) break;
        base -= 32;
    }
    if (lane == 0) st_relaxed_u64(&status[tile], kFlagPre | (excl + agg));
    return excl;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Hot-set rank query: e = dir[g >> 6]; bit and rank of global row g.
__device__ __forceinline__ bool hs_test(const uint4& e, int64_t g, uint32_t* rank) {
    const uint32_t b = (uint32_t)(g & 63);
    const uint32_t lo = e.x, hi = e.y;
    bool bit;
    uint32_t below;
    if (b < 32) {
        bit = (lo >> b) & 1u;
        below = __popc(lo & ((1u << b) - 1u));
    } else {
        bit = (hi >> (b - 32)) & 1u;
        below = __popc(lo) + __popc(hi & ((1u << (b - 32)) - 1u));
    }
    *rank = e.z + below;
    return bit;
}

}  // namespace fae

struct fae_ctx {
    fae::Ctx c;
};
