// persist.cu — the persistent epoch kernel of fae_train_hot_batches (world 1,
// single-lookup bags): ONE cooperative launch trains batches [first,
// first + n) of the grouped hot CSR (sequential SGD).
//
// Step rel = 0 .. n is the fused step of epoch.cu spread over the grid:
//   part R  a9 + a10 of batch a = rel - 1: per segment (run of equal hot id)
//           G[r] = sum_{p: idx[p] = r} dY_a[bag(p)], W[r] -= lr * G[r], and the
//           new row is written straight into Y_b for the bags of batch b = rel
//           that look up r (SegRec.npos/nlen);
//   part F  a8 of batch b for the rows part R does not produce (FreeRecs):
//           Y_b[bag] = W[row] (single-lookup bags: the pooled sum is the row).
// A grid-wide barrier separates steps; it is the only ordering the method
// needs (W of batch a updated before batch b gathers it; Y_a complete before
// dY_a is consumed).  The barrier is split: a CTA arrives, then loads the
// STATIC inputs of its next unit (batch descriptors, segment records, sorted
// bag ids, the long-chunk -> segment search) into registers, then waits.
// After the barrier only the dynamic data moves: dY rows and W rows are
// loaded together, reduced, W is written and Y scattered — two dependent
// memory trips per step instead of the five to ten of a cold kernel.
//
// Arithmetic order is exactly the standalone fae_emb_bwd_update's (R26):
// pieces of 16 lookups from the segment start summed in position order,
// piece partials summed in blocks of CH, block sums added in order, one
// fmaf(-lr, G, W) per element — results are bit-identical to the graph path.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kern_common.cuh"

namespace fae {
namespace {

constexpr int kThreads = 256;
constexpr unsigned long long kBarTimeoutNs = 2000000000ull;

// ---------------------------------------------------------------------------
// split grid barrier: bar[0] counts arrivals monotonically (step rel is
// complete when it reaches (rel + 1) * gridDim.x); bar[1] is an abort word so
// a CTA that waits longer than kBarTimeoutNs ends the kernel (and every
// other waiter with it) instead of hanging the GPU.
// ---------------------------------------------------------------------------
// Modes (FAE_BAR): 0 poll the counter; 1 poll it with a short backoff;
// 2 the last arriver (atomicAdd return) releases one flag per CTA,
// bar[2 + 32 * cta] (own 128-byte line), and each CTA polls its own flag.
__device__ __forceinline__ uint32_t bar_arrive(uint32_t* bar, int mode) {
    __syncthreads();
    uint32_t old = 0;
    if (threadIdx.x == 0) {
        // release: the CTA's writes (ordered before this thread by bar.sync)
        // become visible before the arrival (bit 2 of mode: a full SC fence)
        if (mode & 4) __threadfence();
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if ((mode & 3) == 2) old = atomicAdd(bar, 1u);
        else asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    }
    return old;   // consumed only in bar_wait: the arrival's round trip overlaps the prefetch
}

__device__ __forceinline__ bool bar_wait(uint32_t* bar, uint32_t step, uint32_t old, int mode, uint32_t* err) {
    __shared__ int s_ok;
    const uint32_t target = step * gridDim.x;
    if (threadIdx.x < 32) {
        uint32_t* poll = bar;
        uint32_t want = target;
        if ((mode & 3) == 2) {
            const bool last = __shfl_sync(0xffffffffu, old, 0) == target - 1;
            if (last) {
                for (uint32_t c = threadIdx.x; c < gridDim.x; c += 32)
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar + 2 + 32 * c), "r"(step) : "memory");
            }
            poll = bar + 2 + 32 * blockIdx.x;
            want = step;
        }
        if (threadIdx.x == 0) {
            int ok = 1;
            uint64_t t0 = 0;
            for (uint32_t it = 0;; it++) {
                uint32_t v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(poll) : "memory");
                if ((int32_t)(v - want) >= 0) break;
                if ((mode & 3) == 1) __nanosleep(32);
                if ((it & 255) == 255) {
                    uint32_t ab;
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(ab) : "l"(bar + 1) : "memory");
                    if (ab) {
                        ok = 0;
                        break;
                    }
                    const uint64_t t = gtimer();
                    if (t0 == 0) {
                        t0 = t;
                    } else if (t - t0 > kBarTimeoutNs) {
                        atomicExch(bar + 1, 1u);
                        atomicOr(err, kErrBarrier);
                        ok = 0;
                        break;
                    }
                }
            }
            // acquire side: later loads of the CTA see the step's writes
            if (mode & 4) __threadfence();
            else asm volatile("fence.acq_rel.gpu;" ::: "memory");
            s_ok = ok;
        }
    }
    __syncthreads();
    return s_ok != 0;
}

// ---------------------------------------------------------------------------
// one unit of a step, its static part held in registers across the barrier
// ---------------------------------------------------------------------------
enum : int { kIdle = 0, kCta = 1, kWarp = 2, kGroup = 3, kFwd = 4 };

struct Pre {
    int kind;
    int4 r;                  // pos, len, row, seg (kFwd: pos, len, row)
    int2 nx;                 // Y link into batch b: npos (< 0: none), nlen
    int c0, nc;              // kCta: first chunk of the segment, chunks
    int k;                   // kCta multi-chunk: long record index (lcnt slot)
    int lb;                  // kCta: chunk index in the batch (lpart slot)
    int cbeg, cend;          // kCta: this chunk's lookups [cbeg, cend) of the segment
    int pbeg, pn;            // this lane group's first piece: offset in the segment, lookups
    const int32_t* pa;       // sorted bag ids of batch a (perm + lk0)
    const int32_t* pb;       // of batch b
    const float* dy;         // dY of batch a
    int32_t bag[kPiece];     // pa[r.x + pbeg + u]
    int32_t bg[kPiece];      // first Y-link bags of this worker (-1 pad)
    int dbg;                 // diagnostics (FAE_PERSIST_DBG): bit0 skip Y writes, bit1 skip dY loads
};

__device__ __forceinline__ int64_t step_blocks(const BatchDesc* __restrict__ desc, int64_t first, int64_t rel,
                                               int64_t n, int lpb) {
    const int G = kThreads / lpb;
    int64_t nb = 0;
    if (rel >= 1) {
        const BatchDesc& da = desc[first + rel - 1];
        nb += da.n_lchunk + med_blocks_for(da.n_med, lpb) + (da.n_short + G - 1) / G;
    }
    if (rel < n) {
        const BatchDesc& db = desc[first + rel];
        nb += (rel >= 1 ? (int64_t)db.n_free + G - 1 : (db.sb1 - db.sb0) + G - 1) / G;
    }
    return nb;
}

// Y-link bags of worker w (of nw) in the run [npos, npos + nlen) of pb
__device__ __forceinline__ void load_links(Pre& p, int w, int nw) {
#pragma unroll
    for (int u = 0; u < kPiece; u++) {
        const int q = w + u * nw;
        p.bg[u] = (p.nx.x >= 0 && q < p.nx.y) ? __ldg(p.pb + p.nx.x + q) : -1;
    }
}

__device__ __forceinline__ void load_piece(Pre& p) {
#pragma unroll
    for (int u = 0; u < kPiece; u++) p.bag[u] = u < p.pn ? __ldg(p.pa + p.r.x + p.pbeg + u) : -1;
}

template <int LPB, int NV>
__device__ __forceinline__ void prefetch(Pre& p, const BatchDesc* __restrict__ desc, int64_t first, int64_t rel,
                                         int64_t n, int64_t vb, const SegRec* __restrict__ rec,
                                         const FreeRec* __restrict__ freer, const int32_t* __restrict__ perm,
                                         const int32_t* __restrict__ lmap, const float* __restrict__ dY,
                                         int64_t n_dy, int64_t dy_stride) {
    constexpr int G = kThreads / LPB;
    constexpr int GW = 32 / LPB;
    constexpr int CHUNK = chunk_of_lpb(LPB);
    const int grp = threadIdx.x / LPB;
    p.kind = kIdle;
    p.nx = make_int2(-1, 0);
    p.pn = 0;
    p.pb = nullptr;
    const bool has_a = rel >= 1, has_b = rel < n;
    BatchDesc db{};
    if (has_b) {
        db = desc[first + rel];
        p.pb = perm + db.lk0;
    }
    if (has_a) {
        const BatchDesc da = desc[first + rel - 1];
        p.pa = perm + da.lk0;
        p.dy = dY + ((rel - 1) % n_dy) * dy_stride;
        const SegRec* ra = rec + da.sb0;
        const int64_t n_long = (da.sb1 - da.sb0) - da.n_short - da.n_med;
        const int64_t med_blocks = med_blocks_for(da.n_med, LPB);
        const int64_t red_blocks = da.n_lchunk + med_blocks + (da.n_short + G - 1) / G;
        if (vb < red_blocks) {
            int64_t b = vb;
            bool cta = false, direct = false;
            const SegRec* rp = nullptr;
            int64_t lb = 0;
            if (b < da.n_lchunk) {
                // long chunk b: its segment from the grouping's chunk map
                const SegRec* lrec = ra + da.n_short + da.n_med;
                const int32_t lo = __ldg(lmap + lmap_base(da, first + rel - 1) + b);
                p.k = lo;
                rp = lrec + lo;
                lb = b;
                cta = true;
            } else {
                b -= da.n_lchunk;
                if (b < med_blocks) {
                    if (LPB > 4) {              // medium segment on a CTA (one chunk)
                        rp = ra + da.n_short + b;
                        cta = direct = true;
                        lb = b;
                        p.k = 0;
                    } else {                    // one warp per medium segment
                        const int64_t m = b * 8 + (threadIdx.x >> 5);
                        if (m < da.n_med) {
                            rp = ra + da.n_short + m;
                            p.kind = kWarp;
                        }
                    }
                } else {
                    b -= med_blocks;
                    const int64_t q = b * G + grp;
                    if (q < da.n_short) {
                        rp = ra + q;
                        p.kind = kGroup;
                    }
                }
            }
            if (rp) {
                p.r = __ldg(reinterpret_cast<const int4*>(rp));
                const int4 r2 = __ldg(reinterpret_cast<const int4*>(rp) + 1);
                p.nx = has_b ? make_int2(r2.x, r2.y) : make_int2(-1, 0);   // no link past the run
                if (cta) {
                    p.kind = kCta;
                    p.c0 = direct ? (int)lb : r2.z;
                    p.nc = direct ? 1 : r2.w;
                    p.lb = (int)lb;
                    const int cidx = (int)(lb - p.c0);
                    p.cbeg = cidx * CHUNK;
                    p.cend = min(p.r.y, p.cbeg + CHUNK);
                    const int pc = grp;   // first piece of this group in the chunk
                    p.pbeg = p.cbeg + pc * kPiece;
                    p.pn = pc < CHUNK / kPiece && p.pbeg < p.cend ? min(kPiece, p.cend - p.pbeg) : 0;
                    load_piece(p);
                    load_links(p, grp, G);
                } else if (p.kind == kWarp) {
                    const int gi = (threadIdx.x & 31) / LPB;
                    p.pbeg = gi * kPiece;
                    p.pn = p.pbeg < p.r.y ? min(kPiece, p.r.y - p.pbeg) : 0;
                    load_piece(p);
                    load_links(p, gi, GW);
                } else {
                    p.pbeg = 0;
                    p.pn = p.r.y;
                    load_piece(p);
                    load_links(p, 0, 1);
                }
            }
            return;
        }
        vb -= red_blocks;
    }
    if (!has_b) return;
    // forward-only rows of batch b: its free list when batch a is in the
    // step, else every segment of b
    const int64_t q = vb * G + grp;
    int4 f = make_int4(-1, 0, 0, 0);
    if (has_a) {
        if (q < db.n_free) f = __ldg(reinterpret_cast<const int4*>(freer + db.sb0 + q));
    } else if (q < db.sb1 - db.sb0) {
        f = __ldg(reinterpret_cast<const int4*>(rec + db.sb0 + q));
    }
    if (f.x >= 0) {
        p.kind = kFwd;
        p.r = f;
        p.nx = make_int2(f.x, f.y);
        load_links(p, 0, 1);
    }
}

// sum of the piece's dY rows in position order (bags prefetched); CR rows
// in flight per lane (the sum order does not depend on it)
template <int LPB, int NV>
__device__ __forceinline__ void piece_sum(const int32_t (&bag)[kPiece], const float* __restrict__ src, int D,
                                          int lane, float4 (&g)[NV], bool skip) {
    constexpr int CR = kPiece / NV > 4 ? kPiece / NV : 4;
#pragma unroll
    for (int k = 0; k < NV; k++) g[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (skip) return;
#pragma unroll
    for (int c0 = 0; c0 < kPiece; c0 += CR) {
        float4 v[CR][NV];
#pragma unroll
        for (int u = 0; u < CR; u++) {
            const int32_t b = bag[c0 + u];
            const float4* rp = reinterpret_cast<const float4*>(src + (int64_t)(b < 0 ? 0 : b) * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) v[u][k] = b < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(rp + k * LPB);
        }
#pragma unroll
        for (int u = 0; u < CR; u++)
#pragma unroll
            for (int k = 0; k < NV; k++)
                if (bag[c0 + u] >= 0) add4(g[k], v[u][k]);
    }
}

template <int LPB, int NV>
__device__ __forceinline__ void load_w(const float* W, int32_t row, int D, int lane, float4 (&w)[NV]) {
    const float4* p = reinterpret_cast<const float4*>(W + (int64_t)row * D) + lane;   // coherent loads
#pragma unroll
    for (int k = 0; k < NV; k++) w[k] = p[k * LPB];
}

// w = fmaf(-lr, g, w), stored to W[row]
template <int LPB, int NV>
__device__ __forceinline__ void sgd_store(float4 (&w)[NV], const float4 (&g)[NV], float* W, int32_t row, int D,
                                          int lane, float lr, uint32_t* err) {
    float4* p = reinterpret_cast<float4*>(W + (int64_t)row * D) + lane;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        w[k].x = __fmaf_rn(-lr, g[k].x, w[k].x);
        w[k].y = __fmaf_rn(-lr, g[k].y, w[k].y);
        w[k].z = __fmaf_rn(-lr, g[k].z, w[k].z);
        w[k].w = __fmaf_rn(-lr, g[k].w, w[k].w);
        bad |= !(isfinite(w[k].x) && isfinite(w[k].y) && isfinite(w[k].z) && isfinite(w[k].w));
        p[k * LPB] = w[k];
    }
    if (bad) atomicOr(err, kErrNonfinite);
}

// Y_b[bag] = v for the run's bags of worker w (of nw); the first kPiece bags
// are prefetched in p.bg
template <int LPB, int NV>
__device__ __forceinline__ void write_links(const Pre& p, const float4 (&v)[NV], float* __restrict__ Y, int D,
                                            int lane, int w, int nw) {
    if (p.nx.x < 0 || (p.dbg & 1)) return;
#pragma unroll
    for (int u = 0; u < kPiece; u++) {
        if (p.bg[u] >= 0) {
            float4* y = reinterpret_cast<float4*>(Y + (int64_t)p.bg[u] * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) __stcs(y + k * LPB, v[k]);
        }
    }
    for (int q = w + kPiece * nw; q < p.nx.y; q += nw) {
        float4* y = reinterpret_cast<float4*>(Y + (int64_t)__ldg(p.pb + p.nx.x + q) * D) + lane;
#pragma unroll
        for (int k = 0; k < NV; k++) __stcs(y + k * LPB, v[k]);
    }
}

template <int LPB, int NV>
__device__ __forceinline__ void execute(Pre& p, int D, float* W, float lr, float* lpart, uint32_t* lcnt,
                                        float* __restrict__ Y, uint32_t* err) {
    constexpr int G = kThreads / LPB;
    constexpr int GW = 32 / LPB;
    constexpr int CH = kPiece / NV > 4 ? kPiece / NV : 4;
    constexpr int CHUNK = chunk_of_lpb(LPB);
    constexpr int NPC = CHUNK / kPiece;              // pieces per chunk
    static_assert(NPC <= 2 * G, "a chunk is at most two pieces per lane group");
    __shared__ float4 s_part[NPC][NV * LPB];
    __shared__ int s_last;
    const int lane = threadIdx.x % LPB;
    const int grp = threadIdx.x / LPB;
    if (p.kind == kGroup) {
        float4 w[NV], g[NV];
        load_w<LPB, NV>(W, p.r.z, D, lane, w);
        piece_sum<LPB, NV>(p.bag, p.dy, D, lane, g, p.dbg & 2);
        sgd_store<LPB, NV>(w, g, W, p.r.z, D, lane, lr, err);
        write_links<LPB, NV>(p, w, Y, D, lane, 0, 1);
    } else if (p.kind == kFwd) {
        float4 w[NV];
        load_w<LPB, NV>(W, p.r.z, D, lane, w);
        write_links<LPB, NV>(p, w, Y, D, lane, 0, 1);
    } else if (p.kind == kWarp) {
        // medium segment: each lane group sums one piece; partials in piece
        // order through shuffles (PieceSum order), group 0 owns the row
        const int gi = (threadIdx.x & 31) / LPB;
        float4 w[NV], g[NV];
        if (gi == 0) load_w<LPB, NV>(W, p.r.z, D, lane, w);
        piece_sum<LPB, NV>(p.bag, p.dy, D, lane, g, p.dbg & 2);
        const int ng = (p.r.y + kPiece - 1) / kPiece;
        float4 tot[NV], sub[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) tot[k] = sub[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        int in_blk = 0;
        for (int j = 0; j < ng; j++) {
#pragma unroll
            for (int k = 0; k < NV; k++) {
                float4 q;
                q.x = __shfl_sync(0xffffffffu, g[k].x, j * LPB + lane);
                q.y = __shfl_sync(0xffffffffu, g[k].y, j * LPB + lane);
                q.z = __shfl_sync(0xffffffffu, g[k].z, j * LPB + lane);
                q.w = __shfl_sync(0xffffffffu, g[k].w, j * LPB + lane);
                if (in_blk == 0) sub[k] = q;
                else add4(sub[k], q);
            }
            if (++in_blk == CH) {
#pragma unroll
                for (int k = 0; k < NV; k++) add4(tot[k], sub[k]);
                in_blk = 0;
            }
        }
        if (in_blk)
#pragma unroll
            for (int k = 0; k < NV; k++) add4(tot[k], sub[k]);
        if (gi == 0) sgd_store<LPB, NV>(w, tot, W, p.r.z, D, lane, lr, err);
#pragma unroll
        for (int k = 0; k < NV; k++) {   // broadcast group 0's new row to the warp
            w[k].x = __shfl_sync(0xffffffffu, w[k].x, lane);
            w[k].y = __shfl_sync(0xffffffffu, w[k].y, lane);
            w[k].z = __shfl_sync(0xffffffffu, w[k].z, lane);
            w[k].w = __shfl_sync(0xffffffffu, w[k].w, lane);
        }
        write_links<LPB, NV>(p, w, Y, D, lane, gi, GW);
    }
    if (__syncthreads_or(p.kind == kCta) == 0) return;
    // kCta (uniform over the CTA): one chunk of a long segment, or a whole
    // medium segment when a warp holds fewer than 8 lane groups
    float4 w[NV];
    if (grp == 0) load_w<LPB, NV>(W, p.r.z, D, lane, w);
    {
        float4 g[NV];
        piece_sum<LPB, NV>(p.bag, p.dy, D, lane, g, p.dbg & 2);
        if (grp < NPC) {
#pragma unroll
            for (int k = 0; k < NV; k++) s_part[grp][k * LPB + lane] = g[k];
        }
        if (NPC > G) {   // second piece of the group
            const int pc = grp + G;
            if (pc < NPC) {
                const int pbeg = p.cbeg + pc * kPiece;
                const int pn = pbeg < p.cend ? min(kPiece, p.cend - pbeg) : 0;
                int32_t bag2[kPiece];
#pragma unroll
                for (int u = 0; u < kPiece; u++) bag2[u] = u < pn ? __ldg(p.pa + p.r.x + pbeg + u) : -1;
                piece_sum<LPB, NV>(bag2, p.dy, D, lane, g, p.dbg & 2);
#pragma unroll
                for (int k = 0; k < NV; k++) s_part[pc][k * LPB + lane] = g[k];
            }
        }
    }
    __syncthreads();
    const int np = (p.cend - p.cbeg + kPiece - 1) / kPiece;
    const int nblk = (np + CH - 1) / CH;
    {
        float4 sub[NV];
        if (grp < nblk) {
            const int q0 = grp * CH, q1 = min(np, q0 + CH);
#pragma unroll
            for (int k = 0; k < NV; k++) sub[k] = s_part[q0][k * LPB + lane];
            for (int q = q0 + 1; q < q1; q++)
#pragma unroll
                for (int k = 0; k < NV; k++) add4(sub[k], s_part[q][k * LPB + lane]);
        }
        __syncthreads();
        if (grp < nblk)
#pragma unroll
            for (int k = 0; k < NV; k++) s_part[grp][k * LPB + lane] = sub[k];
        __syncthreads();
    }
    float4 tot[NV];
#pragma unroll
    for (int k = 0; k < NV; k++) tot[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.nc == 1) {
        if (grp == 0)
            for (int j = 0; j < nblk; j++)
#pragma unroll
                for (int k = 0; k < NV; k++) add4(tot[k], s_part[j][k * LPB + lane]);
    } else {
        // publish this chunk's block sums; the last-arriving chunk adds all
        // block sums of the segment in order
        if (grp < nblk) {
            float4* pp = reinterpret_cast<float4*>(lpart + ((int64_t)p.lb * 8 + grp) * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) __stcg(pp + k * LPB, s_part[grp][k * LPB + lane]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const uint32_t old = atomicAdd(&lcnt[p.k], 1u);
            s_last = old == (uint32_t)(p.nc - 1);
            if (s_last) __threadfence();
        }
        __syncthreads();
        if (!s_last) return;
        if (grp == 0) {
            for (int cc = 0; cc < p.nc; cc++) {
                const int len_c = min(CHUNK, p.r.y - cc * CHUNK);
                const int nb = ((len_c + kPiece - 1) / kPiece + CH - 1) / CH;
                const int64_t base = (int64_t)(p.c0 + cc) * 8;
                for (int j = 0; j < nb; j++) {
                    const float4* rp = reinterpret_cast<const float4*>(lpart + (base + j) * D) + lane;
#pragma unroll
                    for (int k = 0; k < NV; k++) add4(tot[k], __ldcg(rp + k * LPB));
                }
            }
            if (threadIdx.x == 0) lcnt[p.k] = 0u;
        }
    }
    if (grp == 0) {
        sgd_store<LPB, NV>(w, tot, W, p.r.z, D, lane, lr, err);
#pragma unroll
        for (int k = 0; k < NV; k++) s_part[0][k * LPB + lane] = w[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) w[k] = s_part[0][k * LPB + lane];
    write_links<LPB, NV>(p, w, Y, D, lane, grp, G);
}

// stamps (diagnostics, FAE_PERSIST_STAMPS): per step [0] max work end,
// [1] max barrier exit, [2] min barrier exit, [3 + kind - 1] max time from a
// CTA's barrier exit to the end of its units, by its first unit's kind
template <int LPB, int NV>
__global__ void __launch_bounds__(kThreads, 2)
k_train_persist(const BatchDesc* __restrict__ desc, int64_t first, int64_t n, const SegRec* __restrict__ rec,
                const FreeRec* __restrict__ freer, const int32_t* __restrict__ perm,
                const float* __restrict__ dY, int64_t n_dy, int64_t dy_stride, int D, float* W, float lr,
                float* lpart, uint32_t* lcnt, const int32_t* __restrict__ lmap, float* __restrict__ Y,
                uint32_t* err, uint32_t* bar,
                unsigned long long* stamps, int barmode, int dbg) {
    Pre p;
    p.dbg = dbg;
    int64_t nb = step_blocks(desc, first, 0, n, LPB);
    if ((int64_t)blockIdx.x < nb)
        prefetch<LPB, NV>(p, desc, first, 0, n, blockIdx.x, rec, freer, perm, lmap, dY, n_dy, dy_stride);
    unsigned long long t_exit = stamps ? gtimer() : 0ull;
    for (int64_t rel = 0; rel <= n; rel++) {
        int kind0 = 0;
        for (int64_t vb = blockIdx.x; vb < nb; vb += gridDim.x) {
            if (vb != (int64_t)blockIdx.x)
                prefetch<LPB, NV>(p, desc, first, rel, n, vb, rec, freer, perm, lmap, dY, n_dy, dy_stride);
            else if (stamps)
                kind0 = __syncthreads_or(p.kind == kCta) ? kCta : __syncthreads_or(p.kind == kWarp) ? kWarp
                      : __syncthreads_or(p.kind == kGroup) ? kGroup : kFwd;
            execute<LPB, NV>(p, D, W, lr, lpart, lcnt, Y, err);
            __syncthreads();
        }
        if (stamps && threadIdx.x == 0) {
            const unsigned long long t = gtimer();
            atomicMax(&stamps[rel * 8 + 0], t);
            if (kind0) atomicMax(&stamps[rel * 8 + 2 + kind0], t - t_exit);
        }
        const uint32_t old = bar_arrive(bar, barmode);
        if (rel < n) {   // the static part of the next step, while the barrier fills
            nb = step_blocks(desc, first, rel + 1, n, LPB);
            if ((int64_t)blockIdx.x < nb)
                prefetch<LPB, NV>(p, desc, first, rel + 1, n, blockIdx.x, rec, freer, perm, lmap, dY, n_dy, dy_stride);
        }
        if (!bar_wait(bar, (uint32_t)(rel + 1), old, barmode, err)) return;
        if (stamps && threadIdx.x == 0) {
            t_exit = gtimer();
            atomicMax(&stamps[rel * 8 + 1], t_exit);
            atomicMin(&stamps[rel * 8 + 2], t_exit);
        }
    }
}

template <int LPB, int NV>
fae_status launch_t(Ctx* c, float* W, int D, const float* dY, int64_t n_dy, float* Y, float lr, int64_t first,
                    int64_t n, cudaEvent_t* ev) {
    Group& g = c->grp;
    auto kern = k_train_persist<LPB, NV>;
    int per_sm = 0;
    FAE_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0));
    if (c->persist_mb > 0) per_sm = std::min(per_sm, c->persist_mb);
    if (per_sm < 1) return set_err(c, FAE_ERR_CUDA, "persistent kernel: no resident CTA per SM");
    const unsigned grid = (unsigned)(per_sm * sm_count(c));
    if (grid > kMaxPersistCtas) return set_err(c, FAE_ERR_CUDA, "persistent kernel: grid exceeds the barrier flags");
    FAE_CUDA(c, cudaMemsetAsync(g.pbar, 0, sizeof(uint32_t) * (2 + 32 * grid), c->stream));
    static const int barmode = getenv("FAE_BAR") ? atoi(getenv("FAE_BAR")) : 0;
    static const bool diag = getenv("FAE_PERSIST_STAMPS") != nullptr;
    static const int dbg = getenv("FAE_PERSIST_DBG") ? atoi(getenv("FAE_PERSIST_DBG")) : 0;
    unsigned long long* stamps = nullptr;
    if (diag) {
        if (g.stamp_cap < n + 1) {
            cudaFree(g.stamps);
            g.stamps = nullptr;
            g.stamp_cap = n + n / 4 + 64;
            FAE_CUDA(c, cudaMalloc(&g.stamps, sizeof(unsigned long long) * kStampSlots * g.stamp_cap));
        }
        stamps = g.stamps;
        std::vector<unsigned long long> init(8 * (n + 1), 0ull);
        for (int64_t i = 0; i <= n; i++) init[8 * i + 2] = ~0ull;
        FAE_CUDA(c, cudaMemcpyAsync(stamps, init.data(), sizeof(unsigned long long) * 8 * (n + 1),
                                    cudaMemcpyHostToDevice, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    const BatchDesc* desc = g.desc;
    const SegRec* rec = g.rec;
    const FreeRec* freer = g.freer;
    const int32_t* perm = g.perm;
    int64_t dy_stride = g.max_bags * (int64_t)D;
    float* lpart = g.lpart;
    uint32_t* lcnt = g.lcnt;
    const int32_t* lmap = g.lmap;
    uint32_t* err = c->d_err;
    uint32_t* bar = g.pbar;
    void* args[] = {&desc, &first, &n, &rec, &freer, &perm, &dY, &n_dy, &dy_stride, &D, &W, &lr,
                    &lpart, &lcnt, &lmap, &Y, &err, &bar, &stamps, (void*)&barmode, (void*)&dbg};
    if (ev) FAE_CUDA(c, cudaEventRecord(ev[0], c->stream));
    FAE_CUDA(c, cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kThreads), args, 0, c->stream));
    FAE_LAUNCHED(c);
    if (ev) FAE_CUDA(c, cudaEventRecord(ev[1], c->stream));
    if (diag) {
        std::vector<unsigned long long> st(8 * (n + 1));
        FAE_CUDA(c, cudaMemcpyAsync(st.data(), stamps, sizeof(unsigned long long) * 8 * (n + 1),
                                    cudaMemcpyDeviceToHost, c->stream));
        FAE_CUDA(c, cudaStreamSynchronize(c->stream));
        double work = 0, bar_lat = 0, skew = 0, kind[4] = {0, 0, 0, 0};
        for (int64_t i = 1; i <= n; i++) {
            work += (double)(st[8 * i] - st[8 * (i - 1) + 2]);
            bar_lat += (double)(st[8 * i + 1] - st[8 * i]);
            skew += (double)(st[8 * i + 1] - st[8 * i + 2]);
            for (int t = 0; t < 4; t++) kind[t] += (double)st[8 * i + 3 + t];
        }
        const double s = n > 0 ? 1e-3 / (double)n : 0.0;
        fprintf(stderr,
                "[persist] grid %u x %d, %lld steps: per step work %.2f us, barrier (last arrival -> last exit) "
                "%.2f us, exit skew %.2f us; slowest CTA by first unit: cta %.2f warp %.2f group %.2f fwd %.2f us\n",
                grid, kThreads, (long long)n, work * s, bar_lat * s, skew * s, kind[0] * s, kind[1] * s,
                kind[2] * s, kind[3] * s);
    }
    return FAE_OK;
}

}  // namespace

fae_status launch_train_persist(Ctx* c, float* W, int D, const float* dY, int64_t n_dy, float* Y, float lr,
                                int64_t first, int64_t n, cudaEvent_t* ev) {
    FAE_DISPATCH_D(D, return launch_t, c, W, D, dY, n_dy, Y, lr, first, n, ev);
    return FAE_OK;
}

}  // namespace fae
