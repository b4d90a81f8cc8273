// coll.cu — the collectives of the multi-GPU path (a11 and the global
// profile) behind one small interface, with two
// transports:
//
//  * NCCL (the product path): one communicator per rank, stream-ordered
//    ncclAllReduce / ncclAllGather over NVLink / NVSwitch.
//  * loopback "virtual ranks" (TEST ONLY, fae_comm_init_loopback, enabled by
//    FAE_LOOPBACK=1): W ctxs of ONE process on ONE GPU, each driven by its own
//    host thread, form a group; a collective is a host rendezvous plus device
//    copies / a rank-ordered sum kernel.  NCCL rejects two ranks on one
//    device and the test boxes have one GPU, so this is how every G > 1 code
//    path of the library (sharded sampling, global loggers, the sparse
//    gradient exchange and its rank-ordered merge) runs in the parity tests.
//    Only the transport differs; the calling code is the same.
//
// Semantics (both transports): allreduce = elementwise sum in place
// (integers: uint32 wraps mod 2^32 like ncclSum; fp32: the loopback sums in
// rank order, NCCL in its own fixed order — identical on every rank either
// way); allgather = rank r's `count`
// elements land at recv + r*count on every rank.
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "fae_internal.cuh"

namespace fae {

static size_t coll_size(CollT t) {
    switch (t) {
        case CollT::U32:
        case CollT::I32:
        case CollT::F32: return 4;
        default: return 8;
    }
}

static ncclDataType_t nccl_type(CollT t) {
    switch (t) {
        case CollT::U32: return ncclUint32;
        case CollT::I32: return ncclInt32;
        case CollT::F32: return ncclFloat32;
        case CollT::U64: return ncclUint64;
        default: return ncclInt64;
    }
}

// ---------------------------------------------------------------------------
// loopback group
// ---------------------------------------------------------------------------
struct LbGroup {
    uint64_t key = 0;
    int world = 0;
    int members = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<const void*> slot;
};

struct LbMember {
    std::shared_ptr<LbGroup> g;
    void* tmp = nullptr;             // device staging (grows)
    size_t tmp_bytes = 0;
    void** dptrs = nullptr;          // device [world] source pointers
};

static std::mutex g_reg_mu;
static std::map<uint64_t, std::weak_ptr<LbGroup>> g_reg;

// generation barrier with a timeout (a peer that errored out never arrives)
static bool lb_barrier(LbGroup& g) {
    std::unique_lock<std::mutex> lk(g.mu);
    if (g.broken) return false;
    const uint64_t my = g.gen;
    if (++g.arrived == g.world) {
        g.arrived = 0;
        g.gen++;
        g.cv.notify_all();
        return true;
    }
    const bool ok = g.cv.wait_for(lk, std::chrono::seconds(120), [&] { return g.gen != my || g.broken; });
    if (!ok || g.broken) {
        g.broken = true;
        g.cv.notify_all();
        return false;
    }
    return true;
}

static void* lb_tmp(Ctx* c, size_t bytes) {
    LbMember* m = c->lb;
    if (bytes <= m->tmp_bytes) return m->tmp;
    cudaStreamSynchronize(c->stream);
    cudaFree(m->tmp);
    m->tmp = nullptr;
    m->tmp_bytes = 0;
    if (cudaMalloc(&m->tmp, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    m->tmp_bytes = bytes;
    return m->tmp;
}

template <typename T>
__global__ void k_lb_sum(void* const* __restrict__ src, int world, int64_t n, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T acc = 0;
        for (int r = 0; r < world; r++) acc += reinterpret_cast<const T*>(src[r])[i];   // rank order
        out[i] = acc;
    }
}

static fae_status lb_fail(Ctx* c, const char* who) {
    return set_err(c, FAE_ERR_NCCL, std::string(who) + ": loopback group broken (a peer rank failed or timed out)");
}

// publish `src`, wait for every rank, run `body` (reads every rank's source),
// wait again, then copy the staged result into `dst`
static fae_status lb_collective(Ctx* c, const void* src, void* dst, size_t out_bytes, const char* who,
                                bool reduce, CollT t, int64_t count) {
    LbGroup& g = *c->lb->g;
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    g.slot[c->rank] = src;
    if (!lb_barrier(g)) return lb_fail(c, who);
    char* tmp = (char*)lb_tmp(c, std::max<size_t>(out_bytes, 16));
    if (!tmp) return set_err(c, FAE_ERR_CUDA, std::string(who) + ": loopback staging allocation failed");
    const size_t esz = coll_size(t);
    if (reduce) {
        FAE_CUDA(c, cudaMemcpyAsync(c->lb->dptrs, g.slot.data(), sizeof(void*) * g.world, cudaMemcpyHostToDevice,
                                    c->stream));
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(count, 256), 1184));
        if (count > 0) {
            if (t == CollT::F32) k_lb_sum<float><<<(unsigned)blocks, 256, 0, c->stream>>>(c->lb->dptrs, g.world, count,
                                                                                         (float*)tmp);
            else if (esz == 4) k_lb_sum<uint32_t><<<(unsigned)blocks, 256, 0, c->stream>>>(c->lb->dptrs, g.world, count,
                                                                                          (uint32_t*)tmp);
            else k_lb_sum<unsigned long long><<<(unsigned)blocks, 256, 0, c->stream>>>(c->lb->dptrs, g.world, count,
                                                                                      (unsigned long long*)tmp);
            FAE_LAUNCHED(c);
        }
    } else {
        const size_t per = (size_t)count * esz;
        for (int r = 0; r < g.world && per > 0; r++)
            FAE_CUDA(c, cudaMemcpyAsync(tmp + r * per, g.slot[r], per, cudaMemcpyDeviceToDevice, c->stream));
    }
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (!lb_barrier(g)) return lb_fail(c, who);   // every rank has read every source
    if (out_bytes > 0) FAE_CUDA(c, cudaMemcpyAsync(dst, tmp, out_bytes, cudaMemcpyDeviceToDevice, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    return FAE_OK;
}

void coll_free(Ctx* c) {
    cudaFree(c->g_rows2);
    cudaFree(c->g_vals2);
    c->g_rows2 = nullptr;
    c->g_vals2 = nullptr;
    c->g_cap2 = 0;
    if (c->comm) ncclCommDestroy(c->comm);
    c->comm = nullptr;
    if (c->lb) {
        LbGroup& g = *c->lb->g;
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.members--;
        }
        cudaFree(c->lb->tmp);
        cudaFree(c->lb->dptrs);
        delete c->lb;
        c->lb = nullptr;
    }
}

// ---------------------------------------------------------------------------
// the interface
// ---------------------------------------------------------------------------
fae_status coll_allreduce_sum(Ctx* c, void* buf, int64_t count, CollT t, const char* who) {
    if (c->lb) return lb_collective(c, buf, buf, (size_t)count * coll_size(t), who, true, t, count);
    if (!c->comm) return set_err(c, FAE_ERR_NOT_INIT, std::string(who) + ": no communicator");
    ncclResult_t r = ncclAllReduce(buf, buf, (size_t)count, nccl_type(t), ncclSum, c->comm, c->stream);
    if (r != ncclSuccess) return set_err(c, FAE_ERR_NCCL, std::string(who) + ": " + ncclGetErrorString(r));
    return FAE_OK;
}

fae_status coll_allgather(Ctx* c, const void* send, void* recv, int64_t count, CollT t, const char* who) {
    if (c->lb) return lb_collective(c, send, recv, (size_t)count * coll_size(t) * c->world, who, false, t, count);
    if (!c->comm) return set_err(c, FAE_ERR_NOT_INIT, std::string(who) + ": no communicator");
    ncclResult_t r = ncclAllGather(send, recv, (size_t)count, nccl_type(t), c->comm, c->stream);
    if (r != ncclSuccess) return set_err(c, FAE_ERR_NCCL, std::string(who) + ": " + ncclGetErrorString(r));
    return FAE_OK;
}

void coll_group_start(Ctx* c) {
    if (c->comm) ncclGroupStart();
}

fae_status coll_group_end(Ctx* c, const char* who) {
    if (!c->comm) return FAE_OK;
    ncclResult_t r = ncclGroupEnd();
    if (r != ncclSuccess) return set_err(c, FAE_ERR_NCCL, std::string(who) + ": " + ncclGetErrorString(r));
    return FAE_OK;
}

fae_status coll_async_error(Ctx* c, const char* who) {
    if (!c->comm) return FAE_OK;
    ncclResult_t ae;
    if (ncclCommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
        return set_err(c, FAE_ERR_NCCL, std::string(who) + ": nccl async: " + ncclGetErrorString(ae));
    return FAE_OK;
}

// Agree on a local status across ranks before any data-path collective: a
// rank whose host-side validation failed must not leave its peers blocked in
// the exchange.  Returns the local status if it failed, else
// INVALID_ARG when a peer failed, else OK.  Synchronises the stream.
fae_status coll_agree(Ctx* c, fae_status local, const char* who) {
    if (c->world <= 1 || !has_comm(c)) return local;
    int64_t* flag = c->g_flag;
    int64_t v = local != FAE_OK ? 1 : 0;
    FAE_CUDA(c, cudaMemcpyAsync(flag, &v, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    fae_status st = coll_allreduce_sum(c, flag, 1, CollT::I64, who);
    if (st != FAE_OK) return st;
    int64_t any = 0;
    FAE_CUDA(c, cudaMemcpyAsync(&any, flag, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (local != FAE_OK) return local;
    if (any) return set_err(c, FAE_ERR_INVALID_ARG, std::string(who) + ": a peer rank failed validation");
    return FAE_OK;
}

// g_rows / g_vals / g_counts sized by the ctx's max_world (never by the
// world of one init, so a later re-init with more ranks cannot overflow)
fae_status comm_bufs(Ctx* c) {
    if (c->g_rows) return FAE_OK;
    const int64_t capL = c->cfg.max_batch_lookups;
    const int64_t mw = c->cfg.max_world;
    c->g_cap = capL;
    FAE_CUDA(c, cudaMalloc(&c->g_rows, sizeof(int32_t) * capL * mw));
    FAE_CUDA(c, cudaMalloc(&c->g_vals, sizeof(float) * capL * mw * c->cfg.max_dim));
    FAE_CUDA(c, cudaMalloc(&c->g_counts, sizeof(int32_t) * mw));
    FAE_CUDA(c, cudaMalloc(&c->g_flag, sizeof(int64_t) * 2));
    return FAE_OK;
}

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_comm_init_loopback(fae_ctx* h, uint64_t group_key, int32_t rank, int32_t world) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    const char* e = getenv("FAE_LOOPBACK");
    if (!(e && e[0] == '1'))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_comm_init_loopback: test-only transport (set FAE_LOOPBACK=1)");
    if (world < 1 || rank < 0 || rank >= world || world > c->cfg.max_world)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_comm_init_loopback: bad rank/world");
    cudaSetDevice(c->device);
    coll_free(c);
    std::shared_ptr<LbGroup> g;
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        auto it = g_reg.find(group_key);
        if (it != g_reg.end()) g = it->second.lock();
        if (g && (g->world != world || g->broken || g->members >= world)) g.reset();
        if (!g) {
            g = std::make_shared<LbGroup>();
            g->key = group_key;
            g->world = world;
            g->slot.assign(world, nullptr);
            g_reg[group_key] = g;
        }
        std::lock_guard<std::mutex> lk2(g->mu);
        g->members++;
    }
    c->lb = new LbMember();
    c->lb->g = g;
    FAE_CUDA(c, cudaMalloc(&c->lb->dptrs, sizeof(void*) * world));
    c->rank = rank;
    c->world = world;
    return comm_bufs(c);
}
