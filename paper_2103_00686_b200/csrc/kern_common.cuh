// kern_common.cuh — device bodies shared by the standalone step calls
// (step.cu) and the graph-replayed epoch runner (epoch.cu).
#pragma once

#include "fae_internal.cuh"

namespace fae {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// lanes of the warp holding the same NB-bit label as this lane: one ballot per
// label bit (bit-sliced match; cheaper than __match_any_sync for small NB)
template <int NB>
__device__ __forceinline__ uint32_t match_label(uint32_t v) {
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const uint32_t bit = (v >> b) & 1u;
        const uint32_t bb = __ballot_sync(0xffffffffu, bit);
        m &= bit ? bb : ~bb;
    }
    return m;
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// a8: Y[b] = sum_{p in bag b} W[idx[p]] for bags [0, n_bags) (grid-stride over
// bags, LPB lanes per bag, NV float4 per lane).  Lookups go in chunks of 8:
// the 8 indices are loaded first, then the 8 rows (8 rows in flight per lane);
// the sum order is fixed: acc += ((r0+r1)+(r2+r3)); acc += ((r4+r5)+(r6+r7)).
// kPDL: the indices of the first chunk are loaded before griddepcontrol.wait
// (they are static), the rows of W after it (written by the previous kernel).
template <int LPB, int NV, bool kPDL = false>
__device__ __forceinline__ void fwd_bags_group(const float* __restrict__ W, int64_t H, int D,
                                         const int32_t* __restrict__ idx,
                                         const int64_t* __restrict__ off, int P, int64_t n_bags,
                                         float* __restrict__ Y, uint32_t* err) {
    const int lane = threadIdx.x % LPB;
    const int64_t gpb = blockDim.x / LPB;
    const int64_t stride = (int64_t)gridDim.x * gpb;
    bool waited = !kPDL;
    for (int64_t b = blockIdx.x * gpb + threadIdx.x / LPB; b < n_bags; b += stride) {
        int64_t lo, hi;
        if (off) {
            lo = off[b];
            hi = off[b + 1];
        } else {
            lo = b * P;
            hi = lo + P;
        }
        float4 acc[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p = lo; p < hi; p += 8) {
            int32_t r[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                r[u] = p + u < hi ? __ldg(idx + p + u) : -1;
                if (p + u < hi && (uint32_t)r[u] >= (uint64_t)H) {
                    atomicOr(err, kErrIndex);
                    r[u] = -1;
                }
            }
            if (!waited) {
                pdl_wait();
                waited = true;
            }
            float4 v[8][NV];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const float4* row = reinterpret_cast<const float4*>(W + (int64_t)(r[u] < 0 ? 0 : r[u]) * D) + lane;
#pragma unroll
                for (int k = 0; k < NV; k++)
                    v[u][k] = r[u] < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(row + k * LPB);
            }
#pragma unroll
            for (int k = 0; k < NV; k++) {
#pragma unroll
                for (int h = 0; h < 8; h += 4) {
                    acc[k].x += (v[h][k].x + v[h + 1][k].x) + (v[h + 2][k].x + v[h + 3][k].x);
                    acc[k].y += (v[h][k].y + v[h + 1][k].y) + (v[h + 2][k].y + v[h + 3][k].y);
                    acc[k].z += (v[h][k].z + v[h + 1][k].z) + (v[h + 2][k].z + v[h + 3][k].z);
                    acc[k].w += (v[h][k].w + v[h + 1][k].w) + (v[h + 2][k].w + v[h + 3][k].w);
                }
            }
        }
        float4* y = reinterpret_cast<float4*>(Y + b * D) + lane;
#pragma unroll
        for (int k = 0; k < NV; k++) __stcs(y + k * LPB, acc[k]);
    }
}

// a8 for multi-hot bags (explicit offsets, or fixed P >= 8): one warp per
// bag; lane group j of the warp's GW = 32/LPB groups sums the bag's chunks of
// 8 lookups j, j+GW, ... (8 indices, then 8 rows in flight; chunk sum
// ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) as above), then the group partials
// are combined by a fixed xor tree (offsets 16 .. LPB): deterministic, the
// same bits in every caller.
template <int LPB, int NV, bool kPDL = false>
__device__ __forceinline__ void fwd_bags_warp(const float* __restrict__ W, int64_t H, int D,
                                              const int32_t* __restrict__ idx,
                                              const int64_t* __restrict__ off, int P, int64_t n_bags,
                                              float* __restrict__ Y, uint32_t* err) {
    constexpr int GW = 32 / LPB;
    const int lane = threadIdx.x % LPB;
    const int gi = (threadIdx.x & 31) / LPB;
    const int64_t wpb = blockDim.x / 32;
    const int64_t stride = (int64_t)gridDim.x * wpb;
    bool waited = !kPDL;
    for (int64_t b = blockIdx.x * wpb + threadIdx.x / 32; b < n_bags; b += stride) {
        int64_t lo, hi;
        if (off) {
            lo = off[b];
            hi = off[b + 1];
        } else {
            lo = b * P;
            hi = lo + P;
        }
        float4 acc[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p = lo + 8 * gi; p < hi; p += 8 * GW) {
            int32_t r[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                r[u] = p + u < hi ? __ldg(idx + p + u) : -1;
                if (p + u < hi && (uint32_t)r[u] >= (uint64_t)H) {
                    atomicOr(err, kErrIndex);
                    r[u] = -1;
                }
            }
            if (!waited) {
                pdl_wait();
                waited = true;
            }
            float4 v[8][NV];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const float4* row = reinterpret_cast<const float4*>(W + (int64_t)(r[u] < 0 ? 0 : r[u]) * D) + lane;
#pragma unroll
                for (int k = 0; k < NV; k++)
                    v[u][k] = r[u] < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(row + k * LPB);
            }
#pragma unroll
            for (int k = 0; k < NV; k++) {
#pragma unroll
                for (int h = 0; h < 8; h += 4) {
                    acc[k].x += (v[h][k].x + v[h + 1][k].x) + (v[h + 2][k].x + v[h + 3][k].x);
                    acc[k].y += (v[h][k].y + v[h + 1][k].y) + (v[h + 2][k].y + v[h + 3][k].y);
                    acc[k].z += (v[h][k].z + v[h + 1][k].z) + (v[h + 2][k].z + v[h + 3][k].z);
                    acc[k].w += (v[h][k].w + v[h + 1][k].w) + (v[h + 2][k].w + v[h + 3][k].w);
                }
            }
        }
        if (!waited) {   // a warp whose bags are all empty still orders after W
            pdl_wait();
            waited = true;
        }
#pragma unroll
        for (int o = 16; o >= LPB; o >>= 1)
#pragma unroll
            for (int k = 0; k < NV; k++) {
                acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
                acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
                acc[k].z += __shfl_xor_sync(0xffffffffu, acc[k].z, o);
                acc[k].w += __shfl_xor_sync(0xffffffffu, acc[k].w, o);
            }
        if (gi == 0) {
            float4* y = reinterpret_cast<float4*>(Y + b * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) __stcs(y + k * LPB, acc[k]);
        }
    }
}

// pooled forward: warp per bag for multi-hot bags (offsets or P >= 8), lane
// group per bag otherwise
constexpr int kWarpBagMinP = 8;
template <int LPB, int NV, bool kPDL = false>
__device__ __forceinline__ void fwd_bags(const float* __restrict__ W, int64_t H, int D,
                                         const int32_t* __restrict__ idx,
                                         const int64_t* __restrict__ off, int P, int64_t n_bags,
                                         float* __restrict__ Y, uint32_t* err) {
    if (off || P >= kWarpBagMinP) fwd_bags_warp<LPB, NV, kPDL>(W, H, D, idx, off, P, n_bags, Y, err);
    else fwd_bags_group<LPB, NV, kPDL>(W, H, D, idx, off, P, n_bags, Y, err);
}

// a8 for single-lookup bags (fixed pooling P = 1): Y[b] = W[idx[b]] — a row
// gather; each LPB-lane group moves U bags per iteration (U rows in flight).
template <int LPB, int NV, bool kPDL = false, int U = 4>
__device__ __forceinline__ void fwd_gather1(const float* __restrict__ W, int64_t H, int D,
                                            const int32_t* __restrict__ idx, int64_t n_bags,
                                            float* __restrict__ Y, uint32_t* err) {
    const int lane = threadIdx.x % LPB;
    const int64_t gpb = blockDim.x / LPB;
    const int64_t groups = (int64_t)gridDim.x * gpb;
    const int64_t g0 = blockIdx.x * gpb + threadIdx.x / LPB;
    bool waited = !kPDL;
    for (int64_t b0 = g0 * U; b0 < n_bags; b0 += groups * U) {
        int32_t r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            r[u] = b0 + u < n_bags ? __ldg(idx + b0 + u) : -1;
            if (b0 + u < n_bags && (uint32_t)r[u] >= (uint64_t)H) {
                atomicOr(err, kErrIndex);
                r[u] = -2;
            }
        }
        if (!waited) {
            pdl_wait();
            waited = true;
        }
        float4 v[U][NV];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const float4* row = reinterpret_cast<const float4*>(W + (int64_t)(r[u] < 0 ? 0 : r[u]) * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++)
                v[u][k] = r[u] < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(row + k * LPB);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (r[u] == -1) continue;
            float4* y = reinterpret_cast<float4*>(Y + (b0 + u) * D) + lane;
#pragma unroll
            for (int k = 0; k < NV; k++) __stcs(y + k * LPB, v[u][k]);
        }
    }
}

// a10 (or emit for a11): apply W[row] -= lr * G, or write G to grad_out.
template <int LPB, int NV, bool kPDL = false>
__device__ __forceinline__ void finish_segment(int64_t s, int64_t s_out, const float4 (&g)[NV],
                                               int lane, const int32_t* __restrict__ seg_row,
                                               float* W, int D, float lr, bool emit,
                                               float* grad_out, uint32_t* err) {
    if (kPDL) pdl_wait();   // W is read by the previous kernel (fwd of this batch)
    if (emit) {
        float4* o = reinterpret_cast<float4*>(grad_out + s_out * D) + lane;
#pragma unroll
        for (int k = 0; k < NV; k++) o[k * LPB] = g[k];
        return;
    }
    const int32_t row = seg_row[s];
    float4* w = reinterpret_cast<float4*>(W + (int64_t)row * D) + lane;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        float4 x = w[k * LPB];
        x.x = __fmaf_rn(-lr, g[k].x, x.x);
        x.y = __fmaf_rn(-lr, g[k].y, x.y);
        x.z = __fmaf_rn(-lr, g[k].z, x.z);
        x.w = __fmaf_rn(-lr, g[k].w, x.w);
        bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
        w[k * LPB] = x;
    }
    if (bad) atomicOr(err, kErrNonfinite);
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

// a9 + a10 over pieces [p_begin, p_end): each LPB-lane group sums the src rows
// vals[i] for positions i in [piece_start[pi], piece_start[pi+1]) in order.
// Single-piece segments finish directly; multi-piece segments publish their
// partial (partial[pi - p_begin]) and the last arriver of the segment sums the
// partials in piece order (blocks of 16), so the summation order is fixed.
template <int LPB, int NV, typename PosT, bool kPDL = false>
__device__ __forceinline__ void reduce_pieces(
    int64_t p_begin, int64_t p_end, int64_t s_out_base, int64_t /*unused*/,
    const int32_t* __restrict__ vals, const PosT* __restrict__ piece_start,
    const int32_t* __restrict__ piece_seg, const int32_t* __restrict__ seg_first,
    const int32_t* __restrict__ seg_row, const float* __restrict__ src, int D, float* W,
    float lr, float* partial, uint32_t* seg_cnt, int emit, float* grad_out, uint32_t* err) {
    constexpr int CH = kPiece / NV > 4 ? kPiece / NV : 4;   // rows in flight per lane
    const int lane = threadIdx.x % LPB;
    const int gw = (threadIdx.x & 31) / LPB;
    const uint32_t gmask = (LPB == 32) ? 0xffffffffu : (((1u << LPB) - 1u) << (gw * LPB));
    const int leader = (threadIdx.x & 31) & ~(LPB - 1);
    const int64_t gpb = blockDim.x / LPB;
    const int64_t stride = (int64_t)gridDim.x * gpb;
    for (int64_t pi = p_begin + blockIdx.x * gpb + threadIdx.x / LPB; pi < p_end; pi += stride) {
        const int64_t i0 = piece_start[pi], i1 = piece_start[pi + 1];
        const int64_t s = piece_seg[pi];
        const int64_t f0 = seg_first[s], f1 = seg_first[s + 1];
        float4 g[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) g[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        // phase 1: the piece's (<= kPiece) bag ids; phase 2: their rows, CH at
        // a time, summed in position order
        int32_t bag[kPiece];
#pragma unroll
        for (int u = 0; u < kPiece; u++) bag[u] = i0 + u < i1 ? __ldg(vals + i0 + u) : -1;
#pragma unroll
        for (int c0 = 0; c0 < kPiece; c0 += CH) {
            float4 v[CH][NV];
#pragma unroll
            for (int u = 0; u < CH; u++) {
                const float4* row = reinterpret_cast<const float4*>(src + (int64_t)(bag[c0 + u] < 0 ? 0 : bag[c0 + u]) * D) + lane;
#pragma unroll
                for (int k = 0; k < NV; k++)
                    v[u][k] = bag[c0 + u] < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(row + k * LPB);
            }
#pragma unroll
            for (int u = 0; u < CH; u++)
#pragma unroll
                for (int k = 0; k < NV; k++)
                    if (bag[c0 + u] >= 0) add4(g[k], v[u][k]);
        }
        if (f1 - f0 == 1) {
            finish_segment<LPB, NV, kPDL>(s, s - s_out_base, g, lane, seg_row, W, D, lr, emit, grad_out, err);
            continue;
        }
        float4* pp = reinterpret_cast<float4*>(partial + (pi - p_begin) * D) + lane;
#pragma unroll
        for (int k = 0; k < NV; k++) __stcg(pp + k * LPB, g[k]);
        // one fence per group: the group's stores are ordered before the
        // leader's fence by __syncwarp; the last arriver's leader fences again
        // before the group reads the partials (L2 loads)
        __syncwarp(gmask);
        uint32_t old = 0;
        if ((threadIdx.x & 31) == leader) {
            __threadfence();
            old = atomicAdd(&seg_cnt[s], 1u);
            if (old == (uint32_t)(f1 - f0 - 1)) __threadfence();
        }
        old = __shfl_sync(gmask, old, leader);
        if (old != (uint32_t)(f1 - f0 - 1)) continue;
        __syncwarp(gmask);
        float4 tot[NV];
#pragma unroll
        for (int k = 0; k < NV; k++) tot[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t q0 = f0; q0 < f1; q0 += CH) {
            float4 blk[CH][NV];
#pragma unroll
            for (int u = 0; u < CH; u++) {
                const float4* rp = reinterpret_cast<const float4*>(partial + (q0 + u - p_begin) * D) + lane;
#pragma unroll
                for (int k = 0; k < NV; k++)
                    blk[u][k] = q0 + u < f1 ? __ldcg(rp + k * LPB) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float4 sub[NV];
#pragma unroll
            for (int k = 0; k < NV; k++) {
                sub[k] = blk[0][k];
#pragma unroll
                for (int u = 1; u < CH; u++) add4(sub[k], blk[u][k]);
                add4(tot[k], sub[k]);
            }
        }
        finish_segment<LPB, NV, kPDL>(s, s - s_out_base, tot, lane, seg_row, W, D, lr, emit, grad_out, err);
        if ((threadIdx.x & 31) == leader) seg_cnt[s] = 0u;
    }
}

#define FAE_DISPATCH_D(D, FN, ...)                                             \
    do {                                                                       \
        switch ((D) / 4) {                                                     \
            case 1: FN<1, 1>(__VA_ARGS__); break;                              \
            case 2: FN<2, 1>(__VA_ARGS__); break;                              \
            case 4: FN<4, 1>(__VA_ARGS__); break;                              \
            case 8: FN<8, 1>(__VA_ARGS__); break;                              \
            case 16: FN<16, 1>(__VA_ARGS__); break;                            \
            case 32: FN<32, 1>(__VA_ARGS__); break;                            \
            case 64: FN<32, 2>(__VA_ARGS__); break;                            \
            case 96: FN<32, 3>(__VA_ARGS__); break;                            \
            case 128: FN<32, 4>(__VA_ARGS__); break;                           \
            default: return set_err(c, FAE_ERR_INVALID_ARG, "unsupported dim"); \
        }                                                                      \
    } while (0)

inline bool dim_ok(int D) {
    if (D < 4 || D % 4) return false;
    const int q = D / 4;
    if (q <= 32) return (q & (q - 1)) == 0;
    return q % 32 == 0 && q <= 128;
}

inline int sm_count(Ctx* c) {
    static int cached[64] = {0};
    const int d = c->device;
    if (d >= 0 && d < 64 && cached[d]) return cached[d];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (d >= 0 && d < 64) cached[d] = n;
    return n;
}

}  // namespace fae
