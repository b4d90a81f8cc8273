// dlrm.cu — the full DLRM hot step: the model FAE trains
// on every hot mini-batch "entirely on the GPU": bottom MLP over
// the dense features, the embedding bags of the sparse features (a8, from
// the hot table), "dot" feature interaction, top MLP, logarithmic loss
// (P:L559-560), backward, SGD — shapes from tab:benchmarks
// and SYN-M1..M4.  Readings R32-R34.
//
// B200 design: the MLP layers are plain GEMMs -> cuBLAS (TF32 on the tensor
// cores, or pedantic fp32); everything around them is hand-written: bias +
// ReLU, the pairwise-dot interaction and its backward (one warp per sample,
// the sample's F x D vectors in shared memory), the fused sigmoid / log-loss
// / dL/dz kernel with a deterministic single-CTA loss sum, the ReLU masks,
// and SGD fused into the weight-gradient GEMM (W += -lr * X^T dC, beta = 1)
// and the bias GEMV.  All buffers are allocated at create, every step is
// graph-capturable, and fae_train_dlrm_batches replays kUnroll steps of
// {a8 forward (grouped kernel), DLRM forward + backward + SGD, a9 + a10
// (grouped reduce kernel)} from one captured graph with the device batch
// cursor of the hot-embedding loop.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kern_common.cuh"

namespace fae {

constexpr int kDlrmMaxLayers = FAE_DLRM_MAX_LAYERS;

struct Dlrm {
    Ctx* c = nullptr;
    fae_dlrm_cfg cfg{};
    cublasHandle_t blas = nullptr;
    int n_layers = 0;                     // bottom then top
    int in_[2 * kDlrmMaxLayers], out_[2 * kDlrmMaxLayers];
    int ld_[2 * kDlrmMaxLayers];          // row stride of W_l and of the layer's input: in rounded up to 4
    int ld_dense = 0, ld_top = 0;         // strides of the dense input and of the interaction output
    int64_t woff[2 * kDlrmMaxLayers], boff[2 * kDlrmMaxLayers];
    int F = 0, P = 0, top_in = 0;
    int64_t n_params = 0;
    // activations [max_batch][width]; act[0] = dense (staged), act[l+1] = output of layer l
    std::vector<float*> act;
    float* grad_a = nullptr;              // [max_batch][max width] ping
    float* grad_b = nullptr;              // [max_batch][max width] pong
    float* ones = nullptr;                // [max_batch]
    float* label = nullptr;               // [max_batch] (staged)
    float* Y = nullptr;                   // [max_batch][Tn][D] pooled bags (the a8 output)
    float* dY = nullptr;                  // [max_batch][Tn][D] (the a9 input)
    int16_t* pairs = nullptr;             // [P][2] (i, j), i > j, row-major
    int32_t* pidx = nullptr;              // [F][F] pair index of (max, min), -1 on the diagonal
    int32_t* nb = nullptr;                // device: [0] samples of the current batch, [1] loss divisor
    float* gbuf = nullptr;                // [n_params] gradient (world > 1: all-reduced before SGD)
    double* acc = nullptr;                // device: [0] sum of losses, [1] samples
    void* ws = nullptr;                   // cuBLAS workspace (graph capture)
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_key = 0;
    cudaGraphExec_t xgraph = nullptr;     // world > 1 exchange loop
    uint64_t xgraph_key = 0;
    int max_w = 0;
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// C[b][j] = act(C[b][j] + bias[j]) for b < nb; rows >= nb zeroed
__global__ void k_bias_act(float* __restrict__ C, const float* __restrict__ bias, int rows, int cols,
                           const int32_t* __restrict__ nb, int relu) {
    const int n = *nb;
    const int64_t tot = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / cols), j = (int)(e - (int64_t)b * cols);
        float v = C[e] + __ldg(bias + j);
        if (relu) v = fmaxf(v, 0.f);
        C[e] = b < n ? v : 0.f;
    }
}

// the same, 4 columns per thread (cols % 4 == 0, 16-byte aligned C and
// bias; 32-bit indices: rows * cols < 2^31): same arithmetic per element
__global__ void k_bias_act4(float4* __restrict__ C, const float4* __restrict__ bias, int rows, int cols4,
                            const int32_t* __restrict__ nb, int relu) {
    const int n = *nb;
    const int tot = rows * cols4;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
        const int b = e / cols4, j = e - b * cols4;
        float4 v = C[e];
        const float4 w = __ldg(bias + j);
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
        if (relu) {
            v.x = fmaxf(v.x, 0.f);
            v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f);
            v.w = fmaxf(v.w, 0.f);
        }
        C[e] = b < n ? v : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// dX *= (X > 0)   (X: the ReLU output that fed the layer)
__global__ void k_relu_mask(float* __restrict__ dX, const float* __restrict__ X, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        if (!(X[e] > 0.f)) dX[e] = 0.f;
}

__global__ void k_relu_mask4(float4* __restrict__ dX, const float4* __restrict__ X, int n4) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += gridDim.x * blockDim.x) {
        const float4 x = X[e];
        float4 d = dX[e];
        if (!(x.x > 0.f)) d.x = 0.f;
        if (!(x.y > 0.f)) d.y = 0.f;
        if (!(x.z > 0.f)) d.z = 0.f;
        if (!(x.w > 0.f)) d.w = 0.f;
        dX[e] = d;
    }
}

// Interaction forward: one warp per sample.  T = [x (bottom output), Y_0 ..
// Y_{Tn-1}] in shared memory; out[b] = [x, <T_i, T_j> for (i, j) in pairs].
__global__ void k_interact_fwd(const float* __restrict__ xbot, const float* __restrict__ Y, int B, int Tn, int D,
                               const int16_t* __restrict__ pairs, int P, const int32_t* __restrict__ nb,
                               float* __restrict__ out, int ld) {
    extern __shared__ float s_T[];   // [warps][F][D]
    const int F = Tn + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= B) return;
    float* T = s_T + (int64_t)warp * F * D;
    const bool valid = b < *nb;
    for (int e = lane; e < F * D; e += 32) {
        const int i = e / D, d = e - i * D;
        float v = 0.f;
        if (valid) v = i == 0 ? xbot[(int64_t)b * D + d] : Y[((int64_t)b * Tn + (i - 1)) * D + d];
        T[e] = v;
    }
    __syncwarp();
    float* o = out + (int64_t)b * ld;
    for (int d = lane; d < D; d += 32) o[d] = T[d];
    for (int k = lane; k < P; k += 32) {
        const int i = pairs[2 * k], j = pairs[2 * k + 1];
        const float* ti = T + i * D;
        const float* tj = T + j * D;
        float s = 0.f;
        for (int d = 0; d < D; d++) s = fmaf(ti[d], tj[d], s);
        o[D + k] = s;
    }
}

// Interaction backward: one warp per sample.  din[b] = [dx, dZ]:
//   dT_i = sum_{j != i} dZ_{pair(i, j)} T_j   (j ascending)
//   dxbot = dx + dT_0 (then the bottom ReLU mask), dY_z = dT_{z+1}.
__global__ void k_interact_bwd(const float* __restrict__ xbot, const float* __restrict__ Y, int B, int Tn, int D,
                               const int32_t* __restrict__ pidx, int P, const int32_t* __restrict__ nb,
                               const float* __restrict__ din, float* __restrict__ dxbot, float* __restrict__ dY, int ld) {
    extern __shared__ float s_T[];   // [warps][F][D]
    const int F = Tn + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= B) return;
    float* T = s_T + (int64_t)warp * F * D;
    const bool valid = b < *nb;
    for (int e = lane; e < F * D; e += 32) {
        const int i = e / D, d = e - i * D;
        float v = 0.f;
        if (valid) v = i == 0 ? xbot[(int64_t)b * D + d] : Y[((int64_t)b * Tn + (i - 1)) * D + d];
        T[e] = v;
    }
    __syncwarp();
    const float* g = din + (int64_t)b * ld;
    for (int e = lane; e < F * D; e += 32) {
        const int i = e / D, d = e - i * D;
        float s = 0.f;
        if (valid)
            for (int j = 0; j < F; j++) {
                if (j == i) continue;
                s = fmaf(g[D + pidx[i * F + j]], T[j * D + d], s);
            }
        if (i == 0) {
            const float x = T[d];
            const float v = valid ? g[d] + s : 0.f;
            dxbot[(int64_t)b * D + d] = x > 0.f ? v : 0.f;   // bottom ReLU mask
        } else {
            dY[((int64_t)b * Tn + (i - 1)) * D + d] = s;
        }
    }
}

// Register versions (F <= 32, D in {8, 16, 32, 64}): lane i holds the row
// T_i of its sample (forward) or its gradient dT_i (backward); row j is
// broadcast from a per-warp shared-memory copy of the sample's rows (one
// wavefront per float4, no bank conflicts; it replaced per-element shuffles,
// D shuffles per row: RMC3 interaction forward 45.6 -> see DESIGN §8).  Forward: lane i computes <T_i, T_j> for
// every j < i (pair index i(i-1)/2 + j), staged in shared memory and stored
// coalesced.  Backward: lane i accumulates dT_i = sum_{j != i} dZ_(i,j) T_j
// in ascending j (dZ staged in shared memory).  Same arithmetic and order as
// the shared-memory kernels above.
// stage the F = Tn + 1 rows of sample b (row 0 = bottom output, rows 1..Tn
// = its Tn contiguous embedding rows) into the warp's shared rows [F][RS]
// with coalesced float4 loads; invalid samples stage zeros
template <int D, int RS>
__device__ __forceinline__ void stage_rows(float* rows, const float* __restrict__ xbot, const float* __restrict__ Y,
                                           int64_t b, int Tn, bool valid, int lane) {
    constexpr int Q = D / 4;
    const int nq = (Tn + 1) * Q;
    const float4* x4 = reinterpret_cast<const float4*>(xbot + b * D);
    const float4* y4 = reinterpret_cast<const float4*>(Y + b * Tn * D);
    for (int e = lane; e < nq; e += 32) {
        const int r = e / Q, q = e - r * Q;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) v = r == 0 ? __ldg(x4 + q) : __ldg(y4 + (e - Q));
        *reinterpret_cast<float4*>(rows + r * RS + 4 * q) = v;
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_interact_fwd_reg(const float* __restrict__ xbot, const float* __restrict__ Y,
                                                          int B, int Tn, int P, const int32_t* __restrict__ nb,
                                                          float* __restrict__ out, int ld) {
    extern __shared__ float s_dyn[];   // [warps][32][D + 4] rows, then [warps][P] pair dots
    constexpr int RS = D + 4;          // padded row stride: a lane's own-row reads hit distinct banks
    const int F = Tn + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int b = blockIdx.x * nw + warp;
    if (b >= B) return;
    const bool valid = b < *nb;
    float* rows = s_dyn + (int64_t)warp * 32 * RS;
    stage_rows<D, RS>(rows, xbot, Y, b, Tn, valid, lane);
    __syncwarp();
    float* z = s_dyn + (int64_t)nw * 32 * RS + (int64_t)warp * P;
    const int kb = lane * (lane - 1) / 2;
    // <T_lane, T_j>, d ascending; four rows j at a time (four independent
    // chains, each in the order of a single one); the lane's own row is
    // re-read from shared memory (conflict-free: padded stride), so no row
    // lives in registers and the loads are not hoisted into spills
    const float4* own = reinterpret_cast<const float4*>(rows + (lane < F ? lane : 0) * RS);
    int j = 0;
    for (; j + 4 <= F - 1; j += 4) {
        const float4* r0 = reinterpret_cast<const float4*>(rows + j * RS);
        const float4* r1 = r0 + RS / 4;
        const float4* r2 = r1 + RS / 4;
        const float4* r3 = r2 + RS / 4;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 2
        for (int q = 0; q < D / 4; q++) {
            const float4 t = own[q];
            const float4 a0 = r0[q], a1 = r1[q], a2 = r2[q], a3 = r3[q];
            s0 = fmaf(t.x, a0.x, s0);
            s1 = fmaf(t.x, a1.x, s1);
            s2 = fmaf(t.x, a2.x, s2);
            s3 = fmaf(t.x, a3.x, s3);
            s0 = fmaf(t.y, a0.y, s0);
            s1 = fmaf(t.y, a1.y, s1);
            s2 = fmaf(t.y, a2.y, s2);
            s3 = fmaf(t.y, a3.y, s3);
            s0 = fmaf(t.z, a0.z, s0);
            s1 = fmaf(t.z, a1.z, s1);
            s2 = fmaf(t.z, a2.z, s2);
            s3 = fmaf(t.z, a3.z, s3);
            s0 = fmaf(t.w, a0.w, s0);
            s1 = fmaf(t.w, a1.w, s1);
            s2 = fmaf(t.w, a2.w, s2);
            s3 = fmaf(t.w, a3.w, s3);
        }
        if (lane < F) {
            if (lane > j) z[kb + j] = s0;
            if (lane > j + 1) z[kb + j + 1] = s1;
            if (lane > j + 2) z[kb + j + 2] = s2;
            if (lane > j + 3) z[kb + j + 3] = s3;
        }
    }
    for (; j < F - 1; j++) {
        const float4* rj = reinterpret_cast<const float4*>(rows + j * RS);
        float s = 0.f;
#pragma unroll 2
        for (int q = 0; q < D / 4; q++) {
            const float4 t = own[q];
            const float4 r = rj[q];
            s = fmaf(t.x, r.x, s);
            s = fmaf(t.y, r.y, s);
            s = fmaf(t.z, r.z, s);
            s = fmaf(t.w, r.w, s);
        }
        if (lane > j && lane < F) z[kb + j] = s;
    }
    __syncwarp();
    float* o = out + (int64_t)b * ld;
    for (int d = lane; d < D; d += 32) o[d] = rows[d];
    for (int k = lane; k < P; k += 32) o[D + k] = z[k];
}

template <int D>
__global__ void __launch_bounds__(128) k_interact_bwd_reg(const float* __restrict__ xbot, const float* __restrict__ Y,
                                                          int B, int Tn, int P, const int32_t* __restrict__ nb,
                                                          const float* __restrict__ din, float* __restrict__ dxbot,
                                                          float* __restrict__ dY, int ld) {
    extern __shared__ float s_dyn[];   // [warps][32][D + 4] rows, then [warps][P] pair gradients
    constexpr int RS = D + 4;
    constexpr int Q = D / 4;
    const int F = Tn + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int b = blockIdx.x * nw + warp;
    if (b >= B) return;
    const bool valid = b < *nb;
    float* rows = s_dyn + (int64_t)warp * 32 * RS;
    stage_rows<D, RS>(rows, xbot, Y, b, Tn, valid, lane);
    const float* g = din + (int64_t)b * ld;
    float* z = s_dyn + (int64_t)nw * 32 * RS + (int64_t)warp * P;
    for (int k = lane; k < P; k += 32) z[k] = valid ? g[D + k] : 0.f;
    __syncwarp();
    // dT_lane[d] = sum_{j != lane} dZ(lane, j) T_j[d], j ascending for every
    // d; columns in chunks of CW (the j loop stays rolled: no hoisted rows)
    constexpr int CW = D < 16 ? D : 16;
    float a[D];
#pragma unroll
    for (int c = 0; c < D / CW; c++) {
#pragma unroll
        for (int k = 0; k < CW; k++) a[c * CW + k] = 0.f;
#pragma unroll 1
        for (int j = 0; j < F; j++) {
            if (lane == j) continue;
            const int ii = lane > j ? lane : j, jj = lane > j ? j : lane;
            const float w = lane < F ? z[ii * (ii - 1) / 2 + jj] : 0.f;
            const float4* rj = reinterpret_cast<const float4*>(rows + j * RS + c * CW);
#pragma unroll
            for (int q = 0; q < CW / 4; q++) {
                const float4 r = rj[q];
                a[c * CW + 4 * q] = fmaf(w, r.x, a[c * CW + 4 * q]);
                a[c * CW + 4 * q + 1] = fmaf(w, r.y, a[c * CW + 4 * q + 1]);
                a[c * CW + 4 * q + 2] = fmaf(w, r.z, a[c * CW + 4 * q + 2]);
                a[c * CW + 4 * q + 3] = fmaf(w, r.w, a[c * CW + 4 * q + 3]);
            }
        }
    }
    __syncwarp();   // every lane is done reading the rows: each overwrites its own with dT
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < Q; q++) {   // dxbot = dx + dT_0, then the bottom ReLU mask (row 0 = bottom output)
            float4 x = *reinterpret_cast<const float4*>(rows + 4 * q);
            float4 v;
            v.x = x.x > 0.f ? (valid ? g[4 * q] + a[4 * q] : 0.f) : 0.f;
            v.y = x.y > 0.f ? (valid ? g[4 * q + 1] + a[4 * q + 1] : 0.f) : 0.f;
            v.z = x.z > 0.f ? (valid ? g[4 * q + 2] + a[4 * q + 2] : 0.f) : 0.f;
            v.w = x.w > 0.f ? (valid ? g[4 * q + 3] + a[4 * q + 3] : 0.f) : 0.f;
            *reinterpret_cast<float4*>(rows + 4 * q) = v;
        }
    } else if (lane < F) {
#pragma unroll
        for (int q = 0; q < Q; q++)
            *reinterpret_cast<float4*>(rows + lane * RS + 4 * q) =
                make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
    }
    __syncwarp();
    float4* ox = reinterpret_cast<float4*>(dxbot + (int64_t)b * D);
    for (int q = lane; q < Q; q += 32) ox[q] = *reinterpret_cast<const float4*>(rows + 4 * q);
    float4* oy = reinterpret_cast<float4*>(dY + (int64_t)b * Tn * D);
    for (int e = lane; e < Tn * Q; e += 32) {
        const int r = e / Q + 1, q = e - (r - 1) * Q;
        oy[e] = *reinterpret_cast<const float4*>(rows + r * RS + 4 * q);
    }
}

// Loss: one CTA.  z[b] (+ bias c) -> s = sigmoid(z); loss_b = max(z,0) -
// z y + log1p(exp(-|z|)); dz[b] = (s - y) / nb (0 for padded rows);
// acc[0] += sum_b loss_b (fixed-order block reduction), acc[1] += nb.
__global__ void __launch_bounds__(1024) k_loss(float* __restrict__ z, const float* __restrict__ bias,
                                               const float* __restrict__ y, int B, const int32_t* __restrict__ nb,
                                               float* __restrict__ dz, double* __restrict__ acc, int train) {
    __shared__ double s_w[32];
    const int n = nb[0];
    const int ndiv = nb[1] > 0 ? nb[1] : 1;   // samples of the (global) batch the loss is the mean over
    double part = 0.0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        float d = 0.f;
        if (b < n) {
            const float v = z[b] + bias[0];
            const float yy = y[b];
            part += (double)(fmaxf(v, 0.f) - v * yy + log1pf(expf(-fabsf(v))));
            const float s = 1.f / (1.f + expf(-v));
            d = (s - yy) / (float)ndiv;
        }
        if (train) dz[b] = d;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        acc[0] += t;
        acc[1] += (double)n;
    }
}

// Stage hot batch rel = *base + s of the grouped loop: dense features and
// labels of its records (hot_ids order) into the fixed buffers, nb.
__global__ void k_dlrm_stage(const BatchDesc* __restrict__ desc, const int64_t* __restrict__ run,
                             const int64_t* __restrict__ base, int s, int Tn, const int64_t* __restrict__ hot_ids,
                             const float* __restrict__ dense, const float* __restrict__ label, int n_dense,
                             int ld_dense, int max_batch, float* __restrict__ sdense, float* __restrict__ slabel,
                             int32_t* __restrict__ nb, const int32_t* __restrict__ rec_total) {
    const int64_t rel = *base + s;
    int n = 0;
    int64_t r0 = 0;
    if (rel < run[1]) {
        const BatchDesc d = desc[run[0] + rel];
        n = d.n_bags / Tn;
        r0 = d.bag0 / Tn;
    }
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)max_batch * (n_dense + 1);
         e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / (n_dense + 1)), k = (int)(e - (int64_t)b * (n_dense + 1));
        const int64_t rec = b < n ? hot_ids[r0 + b] : 0;
        if (k < n_dense) sdense[(int64_t)b * ld_dense + k] = b < n ? dense[rec * n_dense + k] : 0.f;
        else slabel[b] = b < n ? label[rec] : 0.f;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        nb[0] = n;
        nb[1] = rec_total ? (rel < base[4] ? rec_total[rel] : 0) : n;   // world > 1: the global batch
    }
}

__global__ void k_set_nb(int32_t* nb, int v) {
    if (threadIdx.x == 0) nb[0] = nb[1] = v;
}

// p = fmaf(-lr, g, p) over the flat parameters (world > 1, after the all-reduce)
__global__ void k_mlp_sgd(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        p[e] = __fmaf_rn(-lr, g[e], p[e]);
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static fae_status blas_err(Ctx* c, cublasStatus_t s, const char* what) {
    return set_err(c, FAE_ERR_CUDA, std::string("cuBLAS ") + what + " failed (status " + std::to_string((int)s) + ")");
}

#define FAE_BLAS(c, expr)                                              \
    do {                                                               \
        cublasStatus_t s_ = (expr);                                    \
        if (s_ != CUBLAS_STATUS_SUCCESS) return blas_err((c), s_, #expr); \
    } while (0)

static unsigned grid_for(int64_t n, Ctx* c) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sm_count(c) * 8));
}

// One DLRM forward (+ backward + SGD when train) on the staged buffers of
// the dlrm (act[0] = dense, label, Y -> dY), batch size *nb <= max_batch.
static fae_status dlrm_run(Dlrm* m, float* params, float lr, bool train, cudaStream_t st, bool grad_only = false) {
    Ctx* c = m->c;
    const int B = m->cfg.max_batch, nbot = m->cfg.n_bottom, L = m->n_layers;
    const int Tn = m->cfg.n_tables, D = m->cfg.dim;
    FAE_BLAS(c, cublasSetStream(m->blas, st));
    const float one = 1.f, zero = 0.f, mlr = -lr;
    // forward
    for (int l = 0; l < L; l++) {
        const float* X = (l == nbot) ? m->act[nbot + 1] /* interaction output */ : m->act[l < nbot ? l : l + 1];
        float* C = m->act[l < nbot ? l + 1 : l + 2];
        const float* W = params + m->woff[l];
        // K over the padded width (pad entries of W and X are zero): every
        // GEMM dimension but B / out a multiple of 4, so cuBLAS takes its
        // 16-byte-aligned sm100 kernels (an odd K = 13 or 415 fell back to
        // align-1 sm80 kernels)
        FAE_BLAS(c, cublasSgemm(m->blas, CUBLAS_OP_T, CUBLAS_OP_N, m->out_[l], B, m->ld_[l], &one, W, m->ld_[l], X,
                                m->ld_[l], &zero, C, m->out_[l]));
        if (l == L - 1) break;   // the logit: bias inside the loss kernel
        const float* bvec = params + m->boff[l];
        if (m->out_[l] % 4 == 0 && ((uintptr_t)bvec & 15) == 0 && ((uintptr_t)C & 15) == 0 &&
            (int64_t)B * m->out_[l] < (1ll << 31))
            k_bias_act4<<<grid_for((int64_t)B * m->out_[l] / 4, c), 256, 0, st>>>(
                reinterpret_cast<float4*>(C), reinterpret_cast<const float4*>(bvec), B, m->out_[l] / 4, m->nb, 1);
        else
            k_bias_act<<<grid_for((int64_t)B * m->out_[l], c), 256, 0, st>>>(C, bvec, B, m->out_[l], m->nb, 1);
        FAE_LAUNCHED(c);
        if (l == nbot - 1) {     // interaction: act[nbot] = bottom output -> act[nbot + 1]
            const int wpb = 4;
            const bool reg = Tn + 1 <= 32 && (D == 8 || D == 16 || D == 32 || D == 64);
            if (reg) {
                const size_t sm = sizeof(float) * wpb * (32 * (D + 4) + m->P);
                auto kf = D == 8 ? k_interact_fwd_reg<8> : D == 16 ? k_interact_fwd_reg<16>
                        : D == 32 ? k_interact_fwd_reg<32> : k_interact_fwd_reg<64>;
                kf<<<(unsigned)cdiv(B, wpb), 32 * wpb, sm, st>>>(m->act[nbot], m->Y, B, Tn, m->P, m->nb,
                                                                 m->act[nbot + 1], m->ld_top);
            } else {
                const size_t sm = sizeof(float) * wpb * (Tn + 1) * D;
                k_interact_fwd<<<(unsigned)cdiv(B, wpb), 32 * wpb, sm, st>>>(m->act[nbot], m->Y, B, Tn, D, m->pairs,
                                                                             m->P, m->nb, m->act[nbot + 1], m->ld_top);
            }
            FAE_LAUNCHED(c);
        }
    }
    float* z = m->act[L + 1];
    k_loss<<<1, 1024, 0, st>>>(z, params + m->boff[L - 1], m->label, B, m->nb, m->grad_a, m->acc, train ? 1 : 0);
    FAE_LAUNCHED(c);
    if (!train) return FAE_OK;
    // backward + SGD, top layers: dC in grad_a (ping-pong with grad_b)
    float* dC = m->grad_a;
    float* dX = m->grad_b;
    for (int l = L - 1; l >= 0; l--) {
        const bool top = l >= nbot;
        const float* X = top ? (l == nbot ? m->act[nbot + 1] : m->act[l + 1]) : m->act[l];
        float* W = params + m->woff[l];
        float* bvec = params + m->boff[l];
        const int out = m->out_[l], ld = m->ld_[l];
        const int in = ld;   // padded width: the pad rows of dX / dW come out zero (zero pads of W and X)
        // dX = dC W  (old W), for every layer but the first bottom one
        if (l > 0)
            FAE_BLAS(c, cublasSgemm(m->blas, CUBLAS_OP_N, CUBLAS_OP_N, in, B, out, &one, W, ld, dC, out, &zero, dX,
                                    ld));
        if (grad_only) {   // world > 1: the gradient, all-reduced before the update
            FAE_BLAS(c, cublasSgemm(m->blas, CUBLAS_OP_N, CUBLAS_OP_T, in, out, B, &one, X, ld, dC, out, &zero,
                                    m->gbuf + m->woff[l], ld));
            FAE_BLAS(c, cublasSgemv(m->blas, CUBLAS_OP_N, out, B, &one, dC, out, m->ones, 1, &zero,
                                    m->gbuf + m->boff[l], 1));
        } else {
            // W += -lr * X^T dC ; b += -lr * dC^T 1
            FAE_BLAS(c, cublasSgemm(m->blas, CUBLAS_OP_N, CUBLAS_OP_T, in, out, B, &mlr, X, ld, dC, out, &one, W, ld));
            FAE_BLAS(c, cublasSgemv(m->blas, CUBLAS_OP_N, out, B, &mlr, dC, out, m->ones, 1, &one, bvec, 1));
        }
        if (l == 0) break;
        if (l == nbot) {
            // dX = d(interaction output) -> dT: bottom output gradient (masked) and dY
            const int wpb = 4;
            const bool reg = Tn + 1 <= 32 && (D == 8 || D == 16 || D == 32 || D == 64);
            if (reg) {
                const size_t sm = sizeof(float) * wpb * (32 * (D + 4) + m->P);
                auto kb = D == 8 ? k_interact_bwd_reg<8> : D == 16 ? k_interact_bwd_reg<16>
                        : D == 32 ? k_interact_bwd_reg<32> : k_interact_bwd_reg<64>;
                kb<<<(unsigned)cdiv(B, wpb), 32 * wpb, sm, st>>>(m->act[nbot], m->Y, B, Tn, m->P, m->nb, dX, dC,
                                                                 m->dY, m->ld_top);
            } else {
                const size_t sm = sizeof(float) * wpb * (Tn + 1) * D;
                k_interact_bwd<<<(unsigned)cdiv(B, wpb), 32 * wpb, sm, st>>>(m->act[nbot], m->Y, B, Tn, D, m->pidx,
                                                                             m->P, m->nb, dX, dC, m->dY, m->ld_top);
            }
            FAE_LAUNCHED(c);
            continue;            // dC now holds the bottom output's gradient
        }
        // ReLU of the layer below (its output is X)
        if (((uintptr_t)dX & 15) == 0 && ((uintptr_t)X & 15) == 0 && (int64_t)B * ld < (1ll << 31))
            k_relu_mask4<<<grid_for((int64_t)B * ld / 4, c), 256, 0, st>>>(
                reinterpret_cast<float4*>(dX), reinterpret_cast<const float4*>(X), B * ld / 4);
        else
            k_relu_mask<<<grid_for((int64_t)B * ld, c), 256, 0, st>>>(dX, X, (int64_t)B * ld);
        FAE_LAUNCHED(c);
        std::swap(dC, dX);
    }
    return FAE_OK;
}

static bool cfg_ok(const fae_dlrm_cfg* g) {
    if (!g || g->n_dense < 1 || g->n_bottom < 1 || g->n_top < 1 || g->n_bottom > kDlrmMaxLayers ||
        g->n_top > kDlrmMaxLayers || g->n_tables < 1 || g->dim < 4 || g->max_batch < 1)
        return false;
    if (g->bottom[g->n_bottom - 1] != g->dim || g->top[g->n_top - 1] != 1) return false;
    for (int i = 0; i < g->n_bottom; i++)
        if (g->bottom[i] < 1) return false;
    for (int i = 0; i < g->n_top; i++)
        if (g->top[i] < 1) return false;
    const int64_t F = (int64_t)g->n_tables + 1;
    return F <= 256 && (F * g->dim) * 4 * 4 <= 200 * 1024;
}

}  // namespace fae

using namespace fae;

struct fae_dlrm {
    Dlrm m;
};

extern "C" int64_t fae_dlrm_param_count(const fae_dlrm_cfg* g) {
    if (!cfg_ok(g)) return -1;
    auto ld4 = [](int64_t v) { return (v + 3) / 4 * 4; };
    int64_t n = 0, prev = g->n_dense;
    for (int i = 0; i < g->n_bottom; i++) {
        n += ld4(prev) * g->bottom[i] + g->bottom[i];
        prev = g->bottom[i];
    }
    const int64_t F = g->n_tables + 1;
    prev = g->dim + F * (F - 1) / 2;
    for (int i = 0; i < g->n_top; i++) {
        n += ld4(prev) * g->top[i] + g->top[i];
        prev = g->top[i];
    }
    return n;
}

extern "C" void fae_dlrm_destroy(fae_dlrm* h) {
    if (!h) return;
    Dlrm& m = h->m;
    if (m.graph) cudaGraphExecDestroy(m.graph);
    if (m.xgraph) cudaGraphExecDestroy(m.xgraph);
    if (m.blas) cublasDestroy(m.blas);
    for (float* p : m.act) cudaFree(p);
    void* ptrs[] = {m.grad_a, m.grad_b, m.ones, m.label, m.Y, m.dY, m.pairs, m.pidx, m.nb, m.acc, m.ws, m.gbuf};
    for (void* p : ptrs) cudaFree(p);
    delete h;
}

extern "C" fae_status fae_dlrm_create(fae_ctx* ctx, const fae_dlrm_cfg* g, fae_dlrm** out) {
    if (!ctx) return FAE_ERR_NOT_INIT;
    Ctx* c = &ctx->c;
    if (!out || !cfg_ok(g)) return set_err(c, FAE_ERR_INVALID_ARG, "fae_dlrm_create: bad configuration");
    cudaSetDevice(c->device);
    fae_dlrm* h = new fae_dlrm();
    Dlrm& m = h->m;
    m.c = c;
    m.cfg = *g;
    auto fail = [&](fae_status st) {
        fae_dlrm_destroy(h);
        return st;
    };
    const int B = g->max_batch, Tn = g->n_tables, D = g->dim;
    m.F = Tn + 1;
    m.P = m.F * (m.F - 1) / 2;
    m.top_in = D + m.P;
    int prev = g->n_dense;
    int64_t o = 0;
    for (int i = 0; i < g->n_bottom; i++) {
        m.in_[m.n_layers] = prev;
        m.out_[m.n_layers] = g->bottom[i];
        prev = g->bottom[i];
        m.n_layers++;
    }
    prev = m.top_in;
    for (int i = 0; i < g->n_top; i++) {
        m.in_[m.n_layers] = prev;
        m.out_[m.n_layers] = g->top[i];
        prev = g->top[i];
        m.n_layers++;
    }
    for (int l = 0; l < m.n_layers; l++) {
        m.ld_[l] = (m.in_[l] + 3) / 4 * 4;
        m.woff[l] = o;
        o += (int64_t)m.ld_[l] * m.out_[l];
        m.boff[l] = o;
        o += m.out_[l];
        m.max_w = std::max(m.max_w, std::max(m.in_[l], m.out_[l]));
    }
    m.n_params = o;
    // act[0] dense, act[1..nbot] bottom outputs, act[nbot+1] interaction,
    // act[nbot+2..] top outputs (last: the logit)
    m.ld_dense = (g->n_dense + 3) / 4 * 4;
    m.ld_top = (m.top_in + 3) / 4 * 4;
    std::vector<int> widths;
    widths.push_back(m.ld_dense);
    for (int i = 0; i < g->n_bottom; i++) widths.push_back(g->bottom[i]);
    widths.push_back(m.ld_top);
    for (int i = 0; i < g->n_top; i++) widths.push_back(g->top[i]);
    for (int w : widths) {
        float* p = nullptr;
        if (cudaMalloc(&p, sizeof(float) * (size_t)B * w) != cudaSuccess) return fail(cuda_err(c, cudaGetLastError(), "fae_dlrm_create"));
        m.act.push_back(p);
        // the pad columns (beyond the layer width) are never written: zero
        // once, so the padded-width GEMMs multiply zeros
        if (cudaMemset(p, 0, sizeof(float) * (size_t)B * w) != cudaSuccess)
            return fail(cuda_err(c, cudaGetLastError(), "fae_dlrm_create"));
    }
    m.max_w = std::max(m.max_w, m.ld_top);
    for (int l = 0; l < m.n_layers; l++) m.max_w = std::max(m.max_w, m.ld_[l]);
    bool ok = cudaMalloc(&m.grad_a, sizeof(float) * (size_t)B * m.max_w) == cudaSuccess &&
              cudaMalloc(&m.grad_b, sizeof(float) * (size_t)B * m.max_w) == cudaSuccess &&
              cudaMalloc(&m.ones, sizeof(float) * B) == cudaSuccess &&
              cudaMalloc(&m.label, sizeof(float) * B) == cudaSuccess &&
              cudaMalloc(&m.Y, sizeof(float) * (size_t)B * Tn * D) == cudaSuccess &&
              cudaMalloc(&m.dY, sizeof(float) * (size_t)B * Tn * D) == cudaSuccess &&
              cudaMalloc(&m.pairs, sizeof(int16_t) * 2 * std::max(m.P, 1)) == cudaSuccess &&
              cudaMalloc(&m.pidx, sizeof(int32_t) * m.F * m.F) == cudaSuccess &&
              cudaMalloc(&m.nb, sizeof(int32_t) * 2) == cudaSuccess && cudaMalloc(&m.acc, sizeof(double) * 2) == cudaSuccess &&
              cudaMalloc(&m.gbuf, sizeof(float) * std::max<int64_t>(m.n_params, 1)) == cudaSuccess &&
              cudaMalloc(&m.ws, 32u << 20) == cudaSuccess;
    if (!ok) return fail(cuda_err(c, cudaGetLastError(), "fae_dlrm_create: allocation"));
    std::vector<float> ones(B, 1.f);
    std::vector<int16_t> pr;
    std::vector<int32_t> pidx((size_t)m.F * m.F, -1);
    for (int i = 1; i < m.F; i++)
        for (int j = 0; j < i; j++) {
            pidx[(size_t)i * m.F + j] = pidx[(size_t)j * m.F + i] = (int32_t)(pr.size() / 2);
            pr.push_back((int16_t)i);
            pr.push_back((int16_t)j);
        }
    if (cudaMemcpy(m.ones, ones.data(), sizeof(float) * B, cudaMemcpyHostToDevice) != cudaSuccess ||
        (m.P && cudaMemcpy(m.pairs, pr.data(), sizeof(int16_t) * pr.size(), cudaMemcpyHostToDevice) != cudaSuccess) ||
        cudaMemcpy(m.pidx, pidx.data(), sizeof(int32_t) * pidx.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(m.acc, 0, sizeof(double) * 2) != cudaSuccess || cudaMemset(m.nb, 0, sizeof(int32_t) * 2) != cudaSuccess ||
        cudaMemset(m.dY, 0, sizeof(float) * (size_t)B * Tn * D) != cudaSuccess)
        return fail(cuda_err(c, cudaGetLastError(), "fae_dlrm_create: upload"));
    if (cublasCreate(&m.blas) != CUBLAS_STATUS_SUCCESS)
        return fail(set_err(c, FAE_ERR_CUDA, "fae_dlrm_create: cublasCreate failed"));
    cublasSetMathMode(m.blas, g->tf32 ? CUBLAS_TF32_TENSOR_OP_MATH : CUBLAS_PEDANTIC_MATH);
    cublasSetWorkspace(m.blas, m.ws, 32u << 20);
    cublasSetPointerMode(m.blas, CUBLAS_POINTER_MODE_HOST);
    *out = h;
    return FAE_OK;
}

extern "C" fae_status fae_dlrm_buffers(fae_dlrm* h, float** Y, float** dY, double** loss_acc) {
    if (!h) return FAE_ERR_NOT_INIT;
    if (Y) *Y = h->m.Y;
    if (dY) *dY = h->m.dY;
    if (loss_acc) *loss_acc = h->m.acc;
    return FAE_OK;
}

extern "C" fae_status fae_dlrm_step(fae_dlrm* h, float* params, int32_t B, const float* dense, const float* label,
                                    const float* Y, float* dY, float lr, int32_t train) {
    if (!h) return FAE_ERR_NOT_INIT;
    Dlrm& m = h->m;
    Ctx* c = m.c;
    if (!params || !dense || !label || !Y || (train && !dY) || B < 0 || B > m.cfg.max_batch || !(lr == lr))
        return set_err(c, FAE_ERR_INVALID_ARG, "fae_dlrm_step: bad arguments");
    const int Tn = m.cfg.n_tables, D = m.cfg.dim;
    cudaStream_t st = c->stream;
    FAE_CUDA(c, cudaMemsetAsync(m.act[0], 0, sizeof(float) * (size_t)m.cfg.max_batch * m.ld_dense, st));
    if (B > 0) {
        FAE_CUDA(c, cudaMemcpy2DAsync(m.act[0], sizeof(float) * m.ld_dense, dense, sizeof(float) * m.cfg.n_dense,
                                      sizeof(float) * m.cfg.n_dense, B, cudaMemcpyDeviceToDevice, st));
        FAE_CUDA(c, cudaMemcpyAsync(m.label, label, sizeof(float) * B, cudaMemcpyDeviceToDevice, st));
        FAE_CUDA(c, cudaMemcpyAsync(m.Y, Y, sizeof(float) * (size_t)B * Tn * D, cudaMemcpyDeviceToDevice, st));
    }
    k_set_nb<<<1, 32, 0, st>>>(m.nb, B);
    FAE_LAUNCHED(c);
    fae_status s = dlrm_run(&m, params, lr, train != 0, st);
    if (s != FAE_OK) return s;
    if (train && B > 0)
        FAE_CUDA(c, cudaMemcpyAsync(dY, m.dY, sizeof(float) * (size_t)B * Tn * D, cudaMemcpyDeviceToDevice, st));
    return FAE_OK;
}

extern "C" fae_status fae_dlrm_loss(fae_dlrm* h, double* sum_loss, double* n_samples, int32_t reset) {
    if (!h) return FAE_ERR_NOT_INIT;
    Dlrm& m = h->m;
    Ctx* c = m.c;
    double v[2];
    FAE_CUDA(c, cudaMemcpyAsync(v, m.acc, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    FAE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (sum_loss) *sum_loss = v[0];
    if (n_samples) *n_samples = v[1];
    if (reset) FAE_CUDA(c, cudaMemsetAsync(m.acc, 0, sizeof(double) * 2, c->stream));
    return FAE_OK;
}

namespace fae {
fae_status launch_set_run(Ctx* c, cudaStream_t st, int64_t first, int64_t n, int64_t n_total);
fae_status launch_grp_fwd_pdl_any(Ctx* c, cudaStream_t st, int s, float* W, int64_t H, int D, float* Y);
fae_status launch_grp_reduce_any(Ctx* c, cudaStream_t st, int s, int last, float* W, int64_t H, int D,
                                 const float* dY, float lr);
}

// World > 1 (or FAE_FORCE_MERGE): data-parallel DLRM hot step.  Per step:
// the a8 forward of this rank's batch, the DLRM forward + backward with the
// loss averaged over the GLOBAL batch (every rank's records of the step) and
// the MLP gradient kept in gbuf, the a9 sums emitted into this rank's slot,
// then ONE collective group — the MLP gradient all-reduce fused with the
// hot-gradient all-gathers — and the
// updates: the rank-ordered hot-row merge + SGD, and params -= lr * gbuf.
// Replicas stay identical: every rank applies the same all-reduced /
// merged bits.
static fae_status train_dlrm_exchange(Ctx* c, Dlrm& m, float* params, float* W_hot, int64_t H, int D, int64_t first,
                                      int64_t n, const int64_t* hot_ids, const float* dense, const float* label,
                                      float lr_mlp, float lr_emb) {
    Group& g = c->grp;
    if (!has_comm(c)) return set_err(c, FAE_ERR_NOT_INIT, "fae_train_dlrm_batches: world > 1 without a communicator");
    XPrep xp;
    int32_t* rtot = nullptr;
    fae_status st0 = x_prepare(c, first, n, H, &rtot, &xp);
    if (st0 != FAE_OK) return st0;
    const int64_t xcap = xp.xcap;
    auto step = [&](cudaStream_t st, int s, int last) -> fae_status {
        fae_status r = launch_grp_fwd_x(c, st, s, W_hot, H, D, m.Y);
        if (r != FAE_OK) return r;
        k_dlrm_stage<<<grid_for((int64_t)m.cfg.max_batch * (m.cfg.n_dense + 1), c), 256, 0, st>>>(
            g.desc, g.run, g.cursor, s, g.Tn, hot_ids, dense, label, m.cfg.n_dense, m.ld_dense, m.cfg.max_batch, m.act[0],
            m.label, m.nb, rtot);
        FAE_LAUNCHED(c);
        r = dlrm_run(&m, params, lr_mlp, true, st, true);
        if (r != FAE_OK) return r;
        r = launch_xreduce_plain(c, st, s, D, m.dY, xcap);
        if (r != FAE_OK) return r;
        {
            cudaStream_t keep = c->stream;
            c->stream = st;
            coll_group_start(c);
            fae_status a = coll_allreduce_sum(c, m.gbuf, m.n_params, CollT::F32, "dlrm exchange: MLP gradients");
            if (a == FAE_OK)
                a = coll_allgather(c, xrows_of(c, s) + (int64_t)c->rank * xcap, xrows_of(c, s), xcap, CollT::I32,
                                   "dlrm exchange: allgather rows");
            if (a == FAE_OK)
                a = coll_allgather(c, xvals_of(c, s) + (int64_t)c->rank * xcap * D, xvals_of(c, s), xcap * D, CollT::F32,
                                   "dlrm exchange: allgather grads");
            fae_status b = coll_group_end(c, "dlrm exchange");
            c->stream = keep;
            if (a != FAE_OK) return a;
            if (b != FAE_OK) return b;
        }
        r = launch_xmerge_any(c, st, s, last, W_hot, H, D, lr_emb, xcap, xp.per_step, xp.table);
        if (r != FAE_OK) return r;
        k_mlp_sgd<<<grid_for(m.n_params, c), 256, 0, st>>>(params, m.gbuf, m.n_params, lr_mlp);
        FAE_LAUNCHED(c);
        return FAE_OK;
    };
    if (c->lb) {   // loopback (tests): host loop of the same kernels, replay-shaped steps
        for (int64_t i = 0; i < n; i++) {
            const int s = (int)(i % kUnroll);
            fae_status r = step(c->stream, s, s == kUnroll - 1 ? kUnroll : 0);
            if (r != FAE_OK) return r;
        }
        return coll_async_error(c, "fae_train_dlrm_batches");
    }
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { key = (key ^ v) * 1099511628211ull; };
    for (uint64_t v : {(uint64_t)(uintptr_t)params, (uint64_t)(uintptr_t)W_hot, (uint64_t)H, (uint64_t)D,
                       (uint64_t)(uintptr_t)hot_ids, (uint64_t)(uintptr_t)dense, (uint64_t)(uintptr_t)label,
                       (uint64_t)(uintptr_t)g.desc, (uint64_t)(uintptr_t)g.perm, (uint64_t)(uintptr_t)g.rec,
                       (uint64_t)(uintptr_t)g.lmap, (uint64_t)(uintptr_t)g.lpart, (uint64_t)(uintptr_t)g.seg_row,
                       (uint64_t)g.max_bags, (uint64_t)g.max_lchunk, (uint64_t)g.max_long, (uint64_t)xcap,
                       (uint64_t)(uintptr_t)xp.per_step, (uint64_t)(uintptr_t)rtot, (uint64_t)xp.table,
                       (uint64_t)(uintptr_t)g.ptab, (uint64_t)(uintptr_t)c->comm, (uint64_t)c->rank, (uint64_t)c->world})
        mix(v);
    uint32_t a, b;
    memcpy(&a, &lr_mlp, 4);
    memcpy(&b, &lr_emb, 4);
    mix(a);
    mix(b);
    if (!m.xgraph || m.xgraph_key != key) {
        if (m.xgraph) cudaGraphExecDestroy(m.xgraph);
        m.xgraph = nullptr;
        cudaStream_t cs;
        FAE_CUDA(c, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t graph;
        const int64_t l0 = c->launches;
        FAE_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        fae_status st = FAE_OK;
        for (int s = 0; s < kUnroll && st == FAE_OK; s++) st = step(cs, s, s == kUnroll - 1 ? kUnroll : 0);
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        c->launches = l0;
        if (st != FAE_OK || e != cudaSuccess) {
            if (e == cudaSuccess) cudaGraphDestroy(graph);
            cudaStreamDestroy(cs);
            return st != FAE_OK ? st : cuda_err(c, e, "cudaStreamEndCapture (dlrm exchange)");
        }
        e = cudaGraphInstantiate(&m.xgraph, graph, 0);
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        if (e != cudaSuccess) return cuda_err(c, e, "cudaGraphInstantiate (dlrm exchange)");
        m.xgraph_key = key;
    }
    const int64_t reps = cdiv(n, kUnroll);
    for (int64_t r = 0; r < reps; r++) FAE_CUDA(c, cudaGraphLaunch(m.xgraph, c->stream));
    c->launches += reps * kUnroll * (int64_t)(8 + 6 * m.n_layers);
    return coll_async_error(c, "fae_train_dlrm_batches");
}

extern "C" fae_status fae_train_dlrm_batches(fae_ctx* ctx, fae_dlrm* h, float* params, float* W_hot, int64_t H,
                                             int32_t D, int64_t first, int64_t n, const int64_t* hot_ids,
                                             const float* dense, const float* label, float lr_mlp, float lr_emb) {
    if (!ctx || !h) return FAE_ERR_NOT_INIT;
    Ctx* c = &ctx->c;
    Dlrm& m = h->m;
    Group& g = c->grp;
    if (!g.valid) return set_err(c, FAE_ERR_NOT_INIT, "fae_train_dlrm_batches: no grouped batches");
    const bool xpath = c->world > 1 || c->force_merge;
    fae_status vst = FAE_OK;
    if (!params || !W_hot || !hot_ids || !dense || !label || first < 0 || n < 0 ||
        (!xpath && first + n > g.n_batches) || H != g.H || D != m.cfg.dim || D != g.dim ||
        g.Tn != m.cfg.n_tables || g.B > m.cfg.max_batch || !(lr_mlp == lr_mlp) || !(lr_emb == lr_emb))
        vst = set_err(c, FAE_ERR_INVALID_ARG, "fae_train_dlrm_batches: bad arguments");
    if (xpath && has_comm(c) && c->world > 1) vst = coll_agree(c, vst, "fae_train_dlrm_batches");
    if (vst != FAE_OK) return vst;
    if (n == 0) return FAE_OK;
    if (xpath) return train_dlrm_exchange(c, m, params, W_hot, H, D, first, n, hot_ids, dense, label, lr_mlp, lr_emb);
    fae_status rs = launch_set_run(c, c->stream, first, n, n);
    if (rs != FAE_OK) return rs;
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { key = (key ^ v) * 1099511628211ull; };
    for (uint64_t v : {(uint64_t)(uintptr_t)params, (uint64_t)(uintptr_t)W_hot, (uint64_t)H, (uint64_t)D,
                       (uint64_t)(uintptr_t)hot_ids, (uint64_t)(uintptr_t)dense, (uint64_t)(uintptr_t)label,
                       (uint64_t)(uintptr_t)g.desc, (uint64_t)(uintptr_t)g.perm, (uint64_t)(uintptr_t)g.rec,
                       (uint64_t)(uintptr_t)g.lmap, (uint64_t)(uintptr_t)g.lpart, (uint64_t)g.max_bags,
                       (uint64_t)g.max_lchunk, (uint64_t)g.max_long})
        mix(v);
    uint32_t a, b;
    memcpy(&a, &lr_mlp, 4);
    memcpy(&b, &lr_emb, 4);
    mix(a);
    mix(b);
    if (!m.graph || m.graph_key != key) {
        if (m.graph) cudaGraphExecDestroy(m.graph);
        m.graph = nullptr;
        cudaStream_t cs;
        FAE_CUDA(c, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t graph;
        const int64_t l0 = c->launches;
        FAE_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        fae_status st = FAE_OK;
        for (int s = 0; s < kUnroll && st == FAE_OK; s++) {
            st = launch_grp_fwd_pdl_any(c, cs, s, W_hot, H, D, m.Y);
            if (st != FAE_OK) break;
            k_dlrm_stage<<<grid_for((int64_t)m.cfg.max_batch * (m.cfg.n_dense + 1), c), 256, 0, cs>>>(
                g.desc, g.run, g.cursor, s, g.Tn, hot_ids, dense, label, m.cfg.n_dense, m.ld_dense, m.cfg.max_batch, m.act[0],
                m.label, m.nb, (const int32_t*)nullptr);
            if (cudaGetLastError() != cudaSuccess) {
                st = set_err(c, FAE_ERR_CUDA, "fae_train_dlrm_batches: stage launch");
                break;
            }
            st = dlrm_run(&m, params, lr_mlp, true, cs);
            if (st != FAE_OK) break;
            st = launch_grp_reduce_any(c, cs, s, s == kUnroll - 1 ? kUnroll : 0, W_hot, H, D, m.dY, lr_emb);
        }
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        c->launches = l0;
        if (st != FAE_OK || e != cudaSuccess) {
            if (e == cudaSuccess) cudaGraphDestroy(graph);
            cudaStreamDestroy(cs);
            return st != FAE_OK ? st : cuda_err(c, e, "cudaStreamEndCapture (dlrm)");
        }
        e = cudaGraphInstantiate(&m.graph, graph, 0);
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        if (e != cudaSuccess) return cuda_err(c, e, "cudaGraphInstantiate (dlrm)");
        m.graph_key = key;
    }
    const int64_t reps = cdiv(n, kUnroll);
    for (int64_t r = 0; r < reps; r++) FAE_CUDA(c, cudaGraphLaunch(m.graph, c->stream));
    c->launches += reps * kUnroll * (int64_t)(6 + 6 * m.n_layers);
    return FAE_OK;
}
