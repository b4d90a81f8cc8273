// epoch.cu — grouped hot batches and the graph-replayed hot-training loop.
//
// The hot CSR emitted by fae_classify is static for the whole training run
// (the paper pre-processes once and stores the "FAE format"),
// so the backward's sort-and-segment (a9) of every hot batch can be computed
// ONCE, in bulk, instead of inside every training step:
//
//  fae_group_batches     persistent kernel, one 1024-thread CTA per batch at a
//                        time: stable LSD radix sort of (hot id, bag) in the
//                        CTA (8-bit digits, warp match_any ranking, no
//                        inter-CTA communication), then run-length segments
//                        split into <= kPiece pieces; batches are numbered
//                        globally through a decoupled look-back over batches.
//  fae_train_hot_batches a CUDA graph of kUnroll steps, each step = 2 kernels
//                        (k_grp_fwd: a8;  k_grp_reduce: a9 segment sums + a10
//                        SGD), replayed ceil(n / kUnroll) times.  Kernels read
//                        their batch from a device-side cursor that the last
//                        CTA of k_grp_reduce advances, so one captured graph
//                        serves every batch (no per-step host work).
#include <algorithm>
#include <cstring>

#include "kern_common.cuh"

namespace fae {

fae_status validate_schema(Ctx* c, const fae_tables* t, const char* who);

constexpr int kGT = 1024;
constexpr int kGW = kGT / 32;
constexpr int kGI = 4;
constexpr int kGChunk = kGT * kGI;
constexpr int kUnroll = 32;

__device__ __forceinline__ int32_t find_bag64(const int64_t* __restrict__ off, int64_t n_bags,
                                              int64_t pos) {
    int64_t lo = 0, hi = n_bags - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= pos) lo = mid;
        else hi = mid - 1;
    }
    return (int32_t)lo;
}

// block-wide exclusive scan of one uint32 per thread (kGT threads)
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kGW ? s_ws[lane] : 0u;
        uint32_t z = w;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < kGW) s_ws[lane] = z - w;
        if (lane == 31) s_ws[kGW] = z;
    }
    __syncthreads();
    const uint32_t r = s_ws[warp] + x - v;
    *total = s_ws[kGW];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kGT, 1)
k_group(const int32_t* __restrict__ hot_idx, const int64_t* __restrict__ hot_off, int P,
        BatchDesc* __restrict__ desc, int64_t n_batches, int64_t H, int passes,
        uint32_t* __restrict__ kbuf, int32_t* __restrict__ vbuf, int64_t slot_cap,
        uint32_t* __restrict__ batch_ctr, uint64_t* __restrict__ bstatus,
        int32_t* __restrict__ perm, int64_t* __restrict__ piece_start,
        int32_t* __restrict__ piece_seg, int32_t* __restrict__ seg_first,
        int32_t* __restrict__ seg_row, int64_t* __restrict__ totals, uint32_t* err) {
    __shared__ uint32_t s_wh[kGW][kSortBins];
    __shared__ uint32_t s_off[kSortBins];
    __shared__ uint32_t s_tot[kSortBins];
    __shared__ uint32_t s_ws[kGW + 1];
    __shared__ int64_t s_batch;
    __shared__ uint64_t s_base;
    __shared__ uint32_t s_run[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* kA = kbuf + (int64_t)blockIdx.x * 2 * slot_cap;
    uint32_t* kB = kA + slot_cap;
    int32_t* vA = vbuf + (int64_t)blockIdx.x * 2 * slot_cap;
    int32_t* vB = vA + slot_cap;
    while (true) {
        if (tid == 0) s_batch = (int64_t)atomicAdd(batch_ctr, 1u);
        __syncthreads();
        const int64_t bi = s_batch;
        if (bi >= n_batches) break;
        const BatchDesc d = desc[bi];
        const int64_t L = d.lk1 - d.lk0;
        // (hot id, local bag) pairs in CSR order
        for (int64_t j = tid; j < L; j += kGT) {
            const int32_t r = hot_idx[d.lk0 + j];
            uint32_t key;
            if ((uint32_t)r >= (uint64_t)H) {
                atomicOr(err, kErrIndex);
                key = (uint32_t)H;
            } else {
                key = (uint32_t)r;
            }
            kA[j] = key;
            vA[j] = hot_off ? find_bag64(hot_off + d.bag0, d.n_bags, d.lk0 + j) : (int32_t)(j / P);
        }
        __syncthreads();
        uint32_t *kin = kA, *kout = kB;
        int32_t *vin = vA, *vout = vB;
        for (int ps = 0; ps < passes; ps++) {
            const int shift = ps * kSortBits;
            if (tid < kSortBins) s_off[tid] = 0;
            __syncthreads();
            for (int64_t j0 = 0; j0 < L; j0 += kGT) {
                const int64_t j = j0 + tid;
                const uint32_t dg = j < L ? ((kin[j] >> shift) & (kSortBins - 1)) : (uint32_t)kSortBins + lane;
                const uint32_t peers = __match_any_sync(0xffffffffu, dg);
                if (dg < (uint32_t)kSortBins && (__ffs(peers) - 1) == lane) atomicAdd(&s_off[dg], (uint32_t)__popc(peers));
            }
            __syncthreads();
            if (warp < kSortBins / 32) {   // exclusive scan over 256 digits (warps 0..7)
                const uint32_t v = s_off[tid];
                uint32_t x = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) s_ws[warp] = x;
                s_tot[tid] = x - v;
            }
            __syncthreads();
            if (tid < kSortBins) {
                uint32_t wp = 0;
                for (int w = 0; w < (tid >> 5); w++) wp += s_ws[w];
                s_off[tid] = s_tot[tid] + wp;
            }
            __syncthreads();
            for (int64_t c0 = 0; c0 < L; c0 += kGChunk) {
                for (int i = tid; i < kGW * kSortBins; i += kGT) (&s_wh[0][0])[i] = 0;
                __syncthreads();
                uint32_t k[kGI];
                int32_t v[kGI];
                uint32_t rk[kGI];
                const int64_t wb = c0 + (int64_t)warp * 32 * kGI;
#pragma unroll
                for (int r = 0; r < kGI; r++) {
                    const int64_t i = wb + r * 32 + lane;
                    const bool ok = i < L;
                    k[r] = ok ? kin[i] : 0u;
                    v[r] = ok ? vin[i] : 0;
                    const uint32_t dg = ok ? ((k[r] >> shift) & (kSortBins - 1)) : (uint32_t)kSortBins;
                    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
                    const uint32_t lt = __popc(peers & lanemask_lt());
                    uint32_t cnt = 0;
                    if (ok) cnt = s_wh[warp][dg];
                    __syncwarp();
                    if (ok && lt == 0) s_wh[warp][dg] = cnt + __popc(peers);
                    __syncwarp();
                    rk[r] = cnt + lt;
                }
                __syncthreads();
                if (tid < kSortBins) {
                    uint32_t tot = 0;
                    for (int w = 0; w < kGW; w++) {
                        const uint32_t cc = s_wh[w][tid];
                        s_wh[w][tid] = tot;
                        tot += cc;
                    }
                    s_tot[tid] = tot;
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < kGI; r++) {
                    const int64_t i = wb + r * 32 + lane;
                    if (i < L) {
                        const uint32_t dg = (k[r] >> shift) & (kSortBins - 1);
                        const uint32_t pos = s_off[dg] + s_wh[warp][dg] + rk[r];
                        kout[pos] = k[r];
                        vout[pos] = v[r];
                    }
                }
                __syncthreads();
                if (tid < kSortBins) s_off[tid] += s_tot[tid];
                __syncthreads();
            }
            uint32_t* tk = kin; kin = kout; kout = tk;
            int32_t* tv = vin; vin = vout; vout = tv;
            __syncthreads();
        }
        // count pieces / segments of this batch (invalid keys == H excluded)
        uint32_t np = 0, ns = 0;
        for (int64_t j = tid; j < L; j += kGT) {
            const uint32_t kk = kin[j];
            if (kk >= (uint64_t)H) continue;
            const bool head = j == 0 || kin[j - 1] != kk;
            ns += head;
            np += head || (j % kPiece == 0);
        }
        uint32_t tnp, tns;
        block_excl_scan(np, s_ws, &tnp);
        block_excl_scan(ns, s_ws, &tns);
        if (tid == 0) {
            const uint64_t agg = ((uint64_t)tnp << 31) | tns;
            const uint64_t ex = lookback_u64(bstatus, bi, agg);
            s_base = ex;
            const int64_t pb0 = (int64_t)(ex >> 31), sb0 = (int64_t)(ex & 0x7FFFFFFFu);
            desc[bi].pb0 = pb0;
            desc[bi].pb1 = pb0 + tnp;
            desc[bi].sb0 = sb0;
            desc[bi].sb1 = sb0 + tns;
            if (bi == n_batches - 1) {
                totals[0] = pb0 + tnp;
                totals[1] = sb0 + tns;
                piece_start[pb0 + tnp] = d.lk1;
                seg_first[sb0 + tns] = (int32_t)(pb0 + tnp);
            }
            s_run[0] = 0;
            s_run[1] = 0;
        }
        __syncthreads();
        const int64_t pbase = (int64_t)(s_base >> 31), sbase = (int64_t)(s_base & 0x7FFFFFFFu);
        // ordered write pass, kGT positions per round
        for (int64_t j0 = 0; j0 < L; j0 += kGT) {
            const int64_t j = j0 + tid;
            uint32_t kk = 0;
            bool head = false, ps = false;
            if (j < L) {
                kk = kin[j];
                perm[d.lk0 + j] = vin[j];
                if (kk < (uint64_t)H) {
                    head = j == 0 || kin[j - 1] != kk;
                    ps = head || (j % kPiece == 0);
                }
            }
            uint32_t cps, chd;
            const uint32_t eps = block_excl_scan(ps ? 1u : 0u, s_ws, &cps);
            const uint32_t ehd = block_excl_scan(head ? 1u : 0u, s_ws, &chd);
            const int64_t pidx = pbase + s_run[0] + eps;
            const int64_t sidx = sbase + s_run[1] + ehd + (head ? 1 : 0) - 1;
            if (head) {
                seg_first[sidx] = (int32_t)pidx;
                seg_row[sidx] = (int32_t)kk;
            }
            if (ps) {
                piece_start[pidx] = d.lk0 + j;
                piece_seg[pidx] = (int32_t)sidx;
            }
            __syncthreads();
            if (tid == 0) {
                s_run[0] += cps;
                s_run[1] += chd;
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// epoch runner kernels (batch from the device cursor)
// run[0] = first batch, run[1] = number of batches in this call
// ---------------------------------------------------------------------------
template <int LPB, int NV>
__global__ void __launch_bounds__(256)
k_grp_fwd(const BatchDesc* __restrict__ desc, const int64_t* __restrict__ run,
          const int64_t* __restrict__ cursor, const int32_t* __restrict__ hot_idx,
          const int64_t* __restrict__ hot_off, int P, const float* __restrict__ W, int64_t H,
          int D, float* __restrict__ Y, uint32_t* err) {
    const int64_t i = *cursor;
    if (i >= run[1]) return;
    const BatchDesc d = desc[run[0] + i];
    if (hot_off) fwd_bags<LPB, NV>(W, H, D, hot_idx, hot_off + d.bag0, 0, d.n_bags, Y, err);
    else fwd_bags<LPB, NV>(W, H, D, hot_idx + d.lk0, nullptr, P, d.n_bags, Y, err);
}

template <int LPB, int NV>
__global__ void __launch_bounds__(256)
k_grp_reduce(const BatchDesc* __restrict__ desc, const int64_t* __restrict__ run,
             int64_t* cursor, uint32_t* done_ctr, const int32_t* __restrict__ perm,
             const int64_t* __restrict__ piece_start, const int32_t* __restrict__ piece_seg,
             const int32_t* __restrict__ seg_first, const int32_t* __restrict__ seg_row,
             const float* __restrict__ dY, int64_t n_dy, int64_t dy_stride, int D, float* W,
             float lr, float* partial, uint32_t* seg_cnt, int emit, float* grad_out,
             uint32_t* err) {
    const int64_t i = *cursor;
    if (i < run[1]) {
        const BatchDesc d = desc[run[0] + i];
        const float* src = dY + (i % n_dy) * dy_stride;
        reduce_pieces<LPB, NV, int64_t>(d.pb0, d.pb1, d.sb0, 0, perm, piece_start, piece_seg,
                                        seg_first, seg_row, src, D, W, lr, partial, seg_cnt, emit,
                                        grad_out, err);
    }
    // the last CTA to finish advances the cursor (every CTA read it above)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(done_ctr, 1u);
        if (old == gridDim.x - 1) {
            *done_ctr = 0u;
            *cursor = i + 1;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
template <typename T>
static fae_status grow(Ctx* c, T** p, int64_t* cap, int64_t need) {
    if (*cap >= need && *p) return FAE_OK;
    cudaFree(*p);
    *p = nullptr;
    const int64_t n = need + need / 8 + 64;
    FAE_CUDA(c, cudaMalloc(p, sizeof(T) * n));
    *cap = n;
    return FAE_OK;
}

static void drop_graph(Group& g) {
    if (g.graph) cudaGraphExecDestroy(g.graph);
    g.graph = nullptr;
    g.graph_key = 0;
    for (int v = 0; v < 2; v++) {
        if (g.tgraph[v]) cudaGraphExecDestroy(g.tgraph[v]);
        g.tgraph[v] = nullptr;
    }
    g.tgraph_key = 0;
}

template <int LPB, int NV>
static void launch_grp_step(Ctx* c, cudaStream_t s, float* W, int64_t H, int D, const float* dY,
                            int64_t n_dy, float* Y, float lr, int emit, cudaEvent_t mid) {
    Group& g = c->grp;
    const int threads = 256;
    const int64_t gpb = threads / LPB;
    const int64_t maxb = (int64_t)sm_count(c) * 16;
    const int64_t fb = std::max<int64_t>(1, std::min<int64_t>(cdiv(g.max_bags, gpb), maxb));
    k_grp_fwd<LPB, NV><<<(unsigned)fb, threads, 0, s>>>(g.desc, g.run, g.cursor, g.hot_idx, g.hot_off, g.P,
                                                       W, H, D, Y, c->d_err);
    if (mid) cudaEventRecordWithFlags(mid, s, cudaEventRecordExternal);
    const int64_t rb = std::max<int64_t>(1, std::min<int64_t>(cdiv(g.max_pieces, gpb), maxb));
    k_grp_reduce<LPB, NV><<<(unsigned)rb, threads, 0, s>>>(
        g.desc, g.run, g.cursor, g.done_ctr, g.perm, g.piece_start, g.piece_seg, g.seg_first, g.seg_row,
        dY, n_dy, g.max_bags * (int64_t)D, D, W, lr, g.partial, g.seg_cnt, emit, c->ws.grad, c->d_err);
}

static fae_status launch_step(Ctx* c, cudaStream_t s, float* W, int64_t H, int D, const float* dY,
                              int64_t n_dy, float* Y, float lr, int emit, cudaEvent_t mid = nullptr) {
    FAE_DISPATCH_D(D, launch_grp_step, c, s, W, H, D, dY, n_dy, Y, lr, emit, mid);
    return FAE_OK;
}

static fae_status launch_step_split(Ctx* c, cudaStream_t s, float* W, int64_t H, int D, const float* dY,
                                    int64_t n_dy, float* Y, float lr, int emit, cudaEvent_t mid) {
    return launch_step(c, s, W, H, D, dY, n_dy, Y, lr, emit, mid);
}

// Capture kUnroll steps into an executable graph; with `ev` the graph also
// records ev[3s], ev[3s+1], ev[3s+2] around step s's two kernels.
static fae_status capture(Ctx* c, cudaGraphExec_t* out, float* W, int64_t H, int D, const float* dY,
                          int64_t n_dy, float* Y, float lr, cudaEvent_t* ev) {
    cudaStream_t cs;
    FAE_CUDA(c, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    FAE_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    fae_status st = FAE_OK;
    for (int s = 0; s < kUnroll && st == FAE_OK; s++) {
        if (ev) cudaEventRecordWithFlags(ev[3 * s], cs, cudaEventRecordExternal);
        st = launch_step_split(c, cs, W, H, D, dY, n_dy, Y, lr, 0, ev ? ev[3 * s + 1] : nullptr);
        if (ev) cudaEventRecordWithFlags(ev[3 * s + 2], cs, cudaEventRecordExternal);
    }
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (st != FAE_OK) {
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        return st;
    }
    if (e != cudaSuccess) {
        cudaStreamDestroy(cs);
        return cuda_err(c, e, "cudaStreamEndCapture");
    }
    e = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess) return cuda_err(c, e, "cudaGraphInstantiate");
    return FAE_OK;
}

}  // namespace fae

using namespace fae;

extern "C" fae_status fae_set_kernel_timing(fae_ctx* h, int32_t enable) {
    if (!h) return FAE_ERR_NOT_INIT;
    h->c.timing = enable != 0;
    h->c.t_ms[0] = h->c.t_ms[1] = 0.0;
    h->c.t_n[0] = h->c.t_n[1] = 0;
    return FAE_OK;
}

extern "C" fae_status fae_get_kernel_timing(const fae_ctx* h, double* ms, int64_t* n) {
    if (!h || !ms || !n) return FAE_ERR_INVALID_ARG;
    ms[0] = h->c.t_ms[0];
    ms[1] = h->c.t_ms[1];
    n[0] = h->c.t_n[0];
    n[1] = h->c.t_n[1];
    return FAE_OK;
}

extern "C" fae_status fae_group_info(const fae_ctx* h, int64_t* info) {
    if (!h || !info) return FAE_ERR_INVALID_ARG;
    const Group& g = h->c.grp;
    if (!g.valid) return FAE_ERR_NOT_INIT;
    info[0] = g.n_batches;
    info[1] = g.L_total;
    info[2] = g.P_total;
    info[3] = g.S_total;
    info[4] = g.max_pieces;
    info[5] = g.max_bags;
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
    drop_graph(g);
    g.valid = false;
    const int64_t nb = cdiv(pk->n_hot, batch);
    g.n_batches = nb;
    g.Tn = Tn;
    g.P = fixed_pool;
    g.B = batch;
    g.H = H;
    g.hot_idx = pk->hot_idx;
    g.hot_off = offs ? pk->hot_off : nullptr;
    g.L_total = pk->n_hot_lookups;
    // host batch descriptors
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
    }
    if (max_lk >= (1ll << 30)) return set_err(c, FAE_ERR_CAPACITY, "fae_group_batches: batch too large");
    g.max_bags = max_bags;
    g.max_lookups = max_lk;
    const int64_t L = g.L_total;
    const int64_t capP = L + L / kPiece + nb + 2;
    if ((st = grow(c, &g.perm, &g.cap_L, std::max<int64_t>(L, 1))) != FAE_OK) return st;
    if (g.cap_P < capP + 1 || !g.piece_start || !g.piece_seg) {
        cudaFree(g.piece_start);
        cudaFree(g.piece_seg);
        g.piece_start = nullptr;
        g.piece_seg = nullptr;
        g.cap_P = capP + capP / 8 + 64;
        FAE_CUDA(c, cudaMalloc(&g.piece_start, sizeof(int64_t) * g.cap_P));
        FAE_CUDA(c, cudaMalloc(&g.piece_seg, sizeof(int32_t) * g.cap_P));
    }
    if (g.cap_S < L + 2 || !g.seg_first) {
        cudaFree(g.seg_first);
        cudaFree(g.seg_row);
        cudaFree(g.seg_cnt);
        g.seg_first = nullptr;
        g.seg_row = nullptr;
        g.seg_cnt = nullptr;
        g.cap_S = L + 2 + L / 8 + 64;
        FAE_CUDA(c, cudaMalloc(&g.seg_first, sizeof(int32_t) * g.cap_S));
        FAE_CUDA(c, cudaMalloc(&g.seg_row, sizeof(int32_t) * g.cap_S));
        FAE_CUDA(c, cudaMalloc(&g.seg_cnt, sizeof(uint32_t) * g.cap_S));
        FAE_CUDA(c, cudaMemsetAsync(g.seg_cnt, 0, sizeof(uint32_t) * g.cap_S, c->stream));
    }
    if ((st = grow(c, &g.desc, &g.cap_B, std::max<int64_t>(nb, 1))) != FAE_OK) return st;
    if (!g.cursor) {
        FAE_CUDA(c, cudaMalloc(&g.cursor, sizeof(int64_t) * 4));
        g.run = g.cursor + 2;
        FAE_CUDA(c, cudaMalloc(&g.done_ctr, sizeof(uint32_t) * 4));
        FAE_CUDA(c, cudaMemset(g.done_ctr, 0, sizeof(uint32_t) * 4));
    }
    // scratch: per-CTA (k, v) x 2 slots, batch status, counters
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nb, sm_count(c)));
    const int64_t slot = std::max<int64_t>(max_lk, 1);
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o = (o + b + 255) / 256 * 256; return r; };
    const size_t o_k = take(sizeof(uint32_t) * 2 * slot * grid);
    const size_t o_v = take(sizeof(int32_t) * 2 * slot * grid);
    const size_t o_st = take(sizeof(uint64_t) * std::max<int64_t>(nb, 1));
    const size_t o_ctr = take(sizeof(uint32_t) * 4);
    const size_t o_tot = take(sizeof(int64_t) * 2);
    char* sc = (char*)scratch(c, o);
    if (!sc) return set_err(c, FAE_ERR_CUDA, "fae_group_batches: scratch allocation failed");
    FAE_CUDA(c, cudaMemcpyAsync(g.desc, g.hdesc.data(), sizeof(BatchDesc) * nb, cudaMemcpyHostToDevice, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(sc + o_st, 0, (o_ctr - o_st) + 256, c->stream));
    FAE_CUDA(c, cudaMemsetAsync(sc + o_tot, 0, sizeof(int64_t) * 2, c->stream));
    int bits = 1;
    while (bits < 32 && ((uint64_t)1 << bits) <= (uint64_t)H) bits++;
    const int passes = (bits + kSortBits - 1) / kSortBits;
    if (nb > 0) {
        k_group<<<grid, kGT, 0, c->stream>>>(g.hot_idx, g.hot_off, fixed_pool, g.desc, nb, H, passes,
                                             (uint32_t*)(sc + o_k), (int32_t*)(sc + o_v), slot,
                                             (uint32_t*)(sc + o_ctr), (uint64_t*)(sc + o_st), g.perm,
                                             g.piece_start, g.piece_seg, g.seg_first, g.seg_row,
                                             (int64_t*)(sc + o_tot), c->d_err);
        FAE_LAUNCHED(c);
    }
    int64_t tot[2] = {0, 0};
    FAE_CUDA(c, cudaMemcpyAsync(tot, sc + o_tot, sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaMemcpyAsync(g.hdesc.data(), g.desc, sizeof(BatchDesc) * nb, cudaMemcpyDeviceToHost, c->stream));
    st = read_latched(c);
    if (st != FAE_OK) return st;
    g.P_total = tot[0];
    g.S_total = tot[1];
    int64_t mp = 0, ms = 0;
    for (const BatchDesc& d : g.hdesc) {
        mp = std::max<int64_t>(mp, d.pb1 - d.pb0);
        ms = std::max<int64_t>(ms, d.sb1 - d.sb0);
    }
    g.max_pieces = std::max<int64_t>(mp, 1);
    g.max_segs = ms;
    cudaFree(g.partial);
    g.partial = nullptr;
    FAE_CUDA(c, cudaMalloc(&g.partial, sizeof(float) * g.max_pieces * c->cfg.max_dim));
    if (ms > c->ws.cap_L) return set_err(c, FAE_ERR_CAPACITY, "fae_group_batches: batch segments exceed ctx capacity");
    g.valid = true;
    return FAE_OK;
}

extern "C" fae_status fae_train_hot_batches(fae_ctx* h, float* W_hot, int64_t H, int32_t D, int64_t first,
                                            int64_t n, const float* dY, int64_t n_dy, float* Y, float lr) {
    if (!h) return FAE_ERR_NOT_INIT;
    Ctx* c = &h->c;
    Group& g = c->grp;
    if (!g.valid) return set_err(c, FAE_ERR_NOT_INIT, "fae_train_hot_batches: no grouped batches (fae_group_batches)");
    if (!dim_ok(D) || D > c->cfg.max_dim) return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: unsupported dim");
    if (H != g.H) return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: H differs from the grouped H");
    if (first < 0 || n < 0 || n_dy < 1 || (c->world == 1 && first + n > g.n_batches))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: batch range outside the grouped batches");
    if (!(lr == lr)) return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: lr is NaN");
    if (n > 0 && (!W_hot || !dY || !Y)) return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: null pointer");
    if (((uintptr_t)W_hot | (uintptr_t)dY | (uintptr_t)Y) & 15)
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_train_hot_batches: buffers must be 16-byte aligned");
    if (n == 0) return FAE_OK;
    const int64_t hrun[4] = {0, 0, first, n};   // cursor, pad, run[0], run[1]
    FAE_CUDA(c, cudaMemcpyAsync(g.cursor, hrun, sizeof(hrun), cudaMemcpyHostToDevice, c->stream));
    if (c->world > 1) {
        // a11 each step: emit the local sparse gradient, exchange, merge, apply
        // ranks may hold different numbers of hot batches: a rank past its
        // last batch contributes an empty gradient to every remaining exchange
        for (int64_t i = 0; i < n; i++) {
            int64_t U = 0;
            const int32_t* rows = g.seg_row;
            if (first + i < g.n_batches) {
                fae_status st = launch_step(c, c->stream, W_hot, H, D, dY, n_dy, Y, lr, 1);
                if (st != FAE_OK) return st;
                FAE_LAUNCHED(c);
                c->launches++;
                const BatchDesc& d = g.hdesc[first + i];
                rows = g.seg_row + d.sb0;
                U = d.sb1 - d.sb0;
            }
            fae_status st = sync_merge_apply(c, rows, c->ws.grad, U, D, W_hot, H, lr, nullptr, nullptr, nullptr, 0);
            if (st != FAE_OK) return st;
        }
        return FAE_OK;
    }
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { key = (key ^ v) * 1099511628211ull; };
    mix((uint64_t)(uintptr_t)W_hot);
    mix((uint64_t)H);
    mix((uint64_t)D);
    mix((uint64_t)(uintptr_t)dY);
    mix((uint64_t)n_dy);
    mix((uint64_t)(uintptr_t)Y);
    uint32_t lb;
    memcpy(&lb, &lr, 4);
    mix(lb);
    mix((uint64_t)(uintptr_t)g.perm);
    mix((uint64_t)(uintptr_t)g.partial);
    mix((uint64_t)(uintptr_t)g.desc);
    mix((uint64_t)g.max_pieces);
    mix((uint64_t)g.max_bags);
    mix((uint64_t)(uintptr_t)c->d_err);
    const int64_t reps = cdiv(n, kUnroll);
    if (c->timing) {
        // two graph instances with their own events: replay r+1 runs while
        // the host reads replay r's events (no GPU bubble)
        if (g.tgraph_key != key || !g.tgraph[0]) {
            for (int v = 0; v < 2; v++) {
                if (g.tgraph[v]) cudaGraphExecDestroy(g.tgraph[v]);
                g.tgraph[v] = nullptr;
                for (int e = 0; e < 3 * kUnroll; e++)
                    if (!g.tev[v][e]) FAE_CUDA(c, cudaEventCreate(&g.tev[v][e]));
                fae_status st = capture(c, &g.tgraph[v], W_hot, H, D, dY, n_dy, Y, lr, g.tev[v]);
                if (st != FAE_OK) return st;
            }
            g.tgraph_key = key;
        }
        auto harvest = [&](int v, int64_t r) -> fae_status {
            FAE_CUDA(c, cudaEventSynchronize(g.tev[v][3 * kUnroll - 1]));
            const int64_t steps = std::min<int64_t>(kUnroll, n - r * kUnroll);
            for (int64_t s = 0; s < steps; s++) {
                float a = 0.f, b = 0.f;
                FAE_CUDA(c, cudaEventElapsedTime(&a, g.tev[v][3 * s], g.tev[v][3 * s + 1]));
                FAE_CUDA(c, cudaEventElapsedTime(&b, g.tev[v][3 * s + 1], g.tev[v][3 * s + 2]));
                c->t_ms[0] += a;
                c->t_ms[1] += b;
            }
            c->t_n[0] += steps;
            c->t_n[1] += steps;
            return FAE_OK;
        };
        for (int64_t r = 0; r < reps; r++) {
            const int v = (int)(r & 1);
            if (r >= 2) {
                fae_status st = harvest(v, r - 2);
                if (st != FAE_OK) return st;
            }
            FAE_CUDA(c, cudaGraphLaunch(g.tgraph[v], c->stream));
        }
        for (int64_t r = std::max<int64_t>(0, reps - 2); r < reps; r++) {
            fae_status st = harvest((int)(r & 1), r);
            if (st != FAE_OK) return st;
        }
        c->launches += 2 * reps * kUnroll;
        return FAE_OK;
    }
    if (!g.graph || g.graph_key != key) {
        if (g.graph) cudaGraphExecDestroy(g.graph);
        g.graph = nullptr;
        fae_status st = capture(c, &g.graph, W_hot, H, D, dY, n_dy, Y, lr, nullptr);
        if (st != FAE_OK) return st;
        g.graph_key = key;
        g.graph_steps = kUnroll;
    }
    for (int64_t r = 0; r < reps; r++) FAE_CUDA(c, cudaGraphLaunch(g.graph, c->stream));
    c->launches += 2 * reps * g.graph_steps;
    return FAE_OK;
}
