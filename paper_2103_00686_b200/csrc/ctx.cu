// ctx.cu — lifecycle, errors, NCCL bootstrap and step workspace of libfae.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fae_internal.cuh"

namespace fae {

fae_status set_err(Ctx* c, fae_status st, const std::string& msg) {
    if (c) c->err = msg;
    return st;
}

fae_status cuda_err(Ctx* c, cudaError_t e, const char* where) {
    std::string m = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return set_err(c, FAE_ERR_CUDA, m);
}

void* scratch(Ctx* c, size_t bytes) {
    if (bytes <= c->scratch_bytes) return c->scratch;
    if (c->scratch) {
        cudaStreamSynchronize(c->stream);
        cudaFree(c->scratch);
        c->scratch = nullptr;
        c->scratch_bytes = 0;
    }
    size_t want = bytes + (bytes >> 3) + (1 << 20);
    if (cudaMalloc(&c->scratch, want) != cudaSuccess) {
        cudaGetLastError();
        c->scratch = nullptr;
        return nullptr;
    }
    c->scratch_bytes = want;
    return c->scratch;
}

fae_status read_latched(Ctx* c) {
    uint32_t bits = 0;
    FAE_CUDA(c, cudaMemcpyAsync(&bits, c->d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (bits) {
        FAE_CUDA(c, cudaMemsetAsync(c->d_err, 0, sizeof(uint32_t), c->stream));
        if (bits & kErrIndex) return set_err(c, FAE_ERR_INDEX_RANGE, "index outside its table (latched on device)");
        if (bits & kErrNonfinite) return set_err(c, FAE_ERR_NONFINITE, "non-finite value in update (latched on device)");
        if (bits & kErrOverflow) return set_err(c, FAE_ERR_CAPACITY, "capacity exceeded on device: counter overflow or a batch larger than max_batch_lookups (latched)");
        if (bits & kErrBarrier) return set_err(c, FAE_ERR_CUDA, "persistent kernel: grid barrier timed out (latched on device)");
    }
    return FAE_OK;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

fae_status step_ws_alloc(Ctx* c) {
    StepWs& w = c->ws;
    const int64_t world = c->cfg.max_world > 1 ? c->cfg.max_world : 1;
    const int64_t cap = c->cfg.max_batch_lookups * world;
    w.cap_L = cap;
    w.n_sort_tiles = cdiv(cap, kSortTile);
    w.n_piece_tiles = cdiv(cap, kSortTile);
    w.cap_P = cap + cap / kPiece + 2;
    const int D = c->cfg.max_dim;
    for (int i = 0; i < 2; i++) {
        FAE_CUDA(c, cudaMalloc(&w.keys[i], sizeof(uint32_t) * cap));
        FAE_CUDA(c, cudaMalloc(&w.vals[i], sizeof(int32_t) * cap));
    }
    size_t off = 0;
    const size_t o_ghist = off; off = align_up(off + sizeof(uint32_t) * kMaxSortPasses * kSortBins, 256);
    const size_t o_ctr = off; off = align_up(off + sizeof(uint32_t) * 8, 256);
    const size_t o_sst = off; off = align_up(off + sizeof(uint32_t) * kMaxSortPasses * w.n_sort_tiles * kSortBins, 256);
    const size_t o_pst = off; off = align_up(off + sizeof(uint64_t) * w.n_piece_tiles, 256);
    const size_t o_sc = off; off = align_up(off + sizeof(int64_t) * 8, 256);
    w.zero_bytes = off;
    FAE_CUDA(c, cudaMalloc(&w.zero_base, w.zero_bytes));
    FAE_CUDA(c, cudaMemset(w.zero_base, 0, w.zero_bytes));
    char* zb = (char*)w.zero_base;
    w.ghist = (uint32_t*)(zb + o_ghist);
    w.tile_ctr = (uint32_t*)(zb + o_ctr);
    w.sort_status = (uint32_t*)(zb + o_sst);
    w.piece_status = (uint64_t*)(zb + o_pst);
    w.scalars = (int64_t*)(zb + o_sc);
    FAE_CUDA(c, cudaMalloc(&w.piece_start, sizeof(int32_t) * (w.cap_P + 1)));
    FAE_CUDA(c, cudaMalloc(&w.piece_seg, sizeof(int32_t) * w.cap_P));
    FAE_CUDA(c, cudaMalloc(&w.seg_first, sizeof(int32_t) * (cap + 1)));
    FAE_CUDA(c, cudaMalloc(&w.seg_row, sizeof(int32_t) * cap));
    FAE_CUDA(c, cudaMalloc(&w.seg_cnt, sizeof(uint32_t) * cap));
    FAE_CUDA(c, cudaMemset(w.seg_cnt, 0, sizeof(uint32_t) * cap));
    FAE_CUDA(c, cudaMalloc(&w.partial, sizeof(float) * w.cap_P * D));
    FAE_CUDA(c, cudaMalloc(&w.grad, sizeof(float) * cap * D));
    return FAE_OK;
}

void step_ws_free(Ctx* c) {
    StepWs& w = c->ws;
    for (int i = 0; i < 2; i++) {
        cudaFree(w.keys[i]);
        cudaFree(w.vals[i]);
    }
    cudaFree(w.zero_base);
    cudaFree(w.piece_start);
    cudaFree(w.piece_seg);
    cudaFree(w.seg_first);
    cudaFree(w.seg_row);
    cudaFree(w.seg_cnt);
    cudaFree(w.partial);
    cudaFree(w.grad);
    w = StepWs{};
}

}  // namespace fae

using namespace fae;

extern "C" {

fae_status fae_create(const fae_config* cfg, fae_ctx** out) {
    if (!cfg || !out) return FAE_ERR_INVALID_ARG;
    *out = nullptr;
    if (cfg->max_tables < 1 || cfg->max_tables > kMaxTables || cfg->max_rows < 1 ||
        cfg->max_batch_lookups < 1 || cfg->max_batch_bags < 1 || cfg->max_dim < 4 ||
        cfg->max_dim % 4 != 0 || cfg->max_world < 1 ||
        cfg->max_batch_lookups * (int64_t)cfg->max_world >= (1ll << 30))
        return FAE_ERR_INVALID_ARG;
    fae_ctx* h = new fae_ctx();
    Ctx* c = &h->c;
    c->cfg = *cfg;
    c->device = cfg->device;
    {
        const char* e = getenv("FAE_NO_PDL");
        c->no_pdl = e && e[0] == '1';
        const char* t = getenv("FAE_PDL_TRIG");
        // default 0: each kernel triggers its dependent at entry, so the next
        // kernel's static prologue (indices, segment records, dY gathers)
        // overlaps this one; every kernel still reads/writes W only after its
        // griddepcontrol.wait, and consecutive steps use distinct lpart/lcnt
        // slots.  Measured on B200 (Kaggle-shaped): 11.4 vs 12.5 us per step
        // with 3 (trigger after the wait).
        c->pdl_trig = t ? atoi(t) : 0;
        // the fused one-kernel step (bit-identical): automatic for D <= 16
        // (measured on B200, Kaggle-shaped: 6.7 vs 9.1 us per step; at D = 64
        // the two-kernel step wins, 18 vs 30 us); FAE_FUSED=1 forces it on,
        // FAE_FUSED=0 off
        const char* f = getenv("FAE_FUSED");
        c->fused_mode = f ? (f[0] == '1' ? 1 : 0) : -1;
        const char* m = getenv("FAE_RED_MB");
        c->red_mb = m ? atoi(m) : 4;
        // the persistent grid-barrier kernel is opt-in (FAE_PERSIST=1): on
        // B200 a grid barrier costs more than a graph kernel boundary
        const char* pe = getenv("FAE_PERSIST");
        c->persist = pe && pe[0] == '1';
        const char* ms = getenv("FAE_MERGE_SORT");
        c->merge_sort = ms && ms[0] == '1';
        const char* fm = getenv("FAE_FORCE_MERGE");
        c->force_merge = fm && fm[0] == '1';
        const char* gg = getenv("FAE_GS_GENERIC");
        c->gs_generic = gg && gg[0] == '1';
        const char* cl = getenv("FAE_CLS_LEGACY");
        c->cls_legacy = cl && cl[0] == '1';
        // exchange merge: FAE_MERGE_TABLE=1 / 0 forces the row-position
        // table / the binary searches (default: table for world > 2)
        const char* mt = getenv("FAE_MERGE_TABLE");
        c->merge_table = mt ? (mt[0] == '1' ? 1 : 0) : -1;
        const char* pm = getenv("FAE_PERSIST_MB");
        c->persist_mb = pm ? atoi(pm) : 0;
    }
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) {
        delete h;
        return FAE_ERR_CUDA;
    }
    if (cudaMalloc(&c->d_err, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemset(c->d_err, 0, sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&c->d_rowbase_tmp, sizeof(int64_t) * (cfg->max_tables + 1)) != cudaSuccess ||
        cudaMalloc(&c->d_rows_tmp, sizeof(int64_t) * cfg->max_tables) != cudaSuccess ||
        cudaMalloc(&c->hs.d_rowbase, sizeof(int64_t) * (cfg->max_tables + 1)) != cudaSuccess ||
        step_ws_alloc(c) != FAE_OK) {
        fae_destroy(h);
        return FAE_ERR_CUDA;
    }
    *out = h;
    return FAE_OK;
}

void fae_destroy(fae_ctx* h) {
    if (!h) return;
    Ctx* c = &h->c;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    else cudaDeviceSynchronize();
    coll_free(c);
    step_ws_free(c);
    group_free(c);
    cudaFree(c->d_err);
    cudaFree(c->scratch);
    cudaFree(c->d_rowbase_tmp);
    cudaFree(c->d_rows_tmp);
    cudaFree(c->hs.dir);
    cudaFree(c->hs.d_rowbase);
    cudaFree(c->g_rows);
    cudaFree(c->g_vals);
    cudaFree(c->g_counts);
    cudaFree(c->g_flag);
    delete h;
}

fae_status fae_set_stream(fae_ctx* h, void* stream) {
    if (!h) return FAE_ERR_NOT_INIT;
    h->c.stream = (cudaStream_t)stream;
    return FAE_OK;
}

const char* fae_last_error(const fae_ctx* h) {
    if (!h) return "null ctx";
    return h->c.err.c_str();
}

fae_status fae_check(fae_ctx* h) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_err(c, e, "fae_check");
    return read_latched(c);
}

int64_t fae_kernel_launches(const fae_ctx* h) { return h ? h->c.launches : 0; }

fae_status fae_get_nccl_id(void* id128) {
    if (!id128) return FAE_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return FAE_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
    memcpy(id128, &id, sizeof(id));
    return FAE_OK;
}

fae_status fae_comm_init(fae_ctx* h, const void* id128, int32_t rank, int32_t world) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    if (!id128 || world < 1 || rank < 0 || rank >= world || world > c->cfg.max_world)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_comm_init: bad rank/world");
    cudaSetDevice(c->device);
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    coll_free(c);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess)
        return set_err(c, FAE_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    c->rank = rank;
    c->world = world;
    return comm_bufs(c);
}

}  // extern "C"
