// persist_probe.cu — floor of one sequential-SGD step on B200, measured two
// ways (ground truth for the persistent epoch kernel's design; not libfae):
//   * a persistent kernel: per step each lane group gathers K random dY rows,
//     RMWs one random W row, scatters K random Y rows; grid barrier per step;
//   * the same work as one kernel launch per step (stream-ordered).
// Also: the bare barrier (no work) at several grid sizes and barrier styles.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

struct Args {
    const float* dY; int64_t dy_rows;     // pool
    float* W; int64_t w_rows;
    float* Y; int64_t y_rows;
    int D;                                // floats per row (16 / 64)
    int units;                            // lane groups with work per step
    int K;                                // dY rows per unit (and Y rows)
    int work;                             // bit0 dY, bit1 W, bit2 Y
    int mode;                             // barrier: 0 counter poll (acq_rel fences), 1 SC fences, 2 flags
    uint32_t* bar;
};

__device__ __forceinline__ void barrier(uint32_t* bar, uint32_t step, int mode) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t target = step * gridDim.x;
        if (mode == 1) __threadfence(); else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (mode == 2) {
            uint32_t old = atomicAdd(bar, 1u);
            if (old == target - 1)
                for (uint32_t c = 0; c < gridDim.x; c++)
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar + 32 + 32 * c), "r"(step) : "memory");
            uint32_t* f = bar + 32 + 32 * blockIdx.x;
            uint32_t v;
            do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory"); } while ((int)(v - step) < 0);
        } else {
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            uint32_t v;
            do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while ((int)(v - target) < 0);
        }
        if (mode == 1) __threadfence(); else asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

template <int LPB>
__device__ __forceinline__ void step_work(const Args& a, int s) {
    const int lane = threadIdx.x % LPB;
    const int gpb = blockDim.x / LPB;
    for (int u = blockIdx.x * gpb + threadIdx.x / LPB; u < a.units; u += gridDim.x * gpb) {
        const uint32_t h0 = hsh((uint32_t)u * 2654435761u ^ (uint32_t)s * 40503u);
        float4 acc = make_float4(0, 0, 0, 0);
        float4 w = make_float4(0, 0, 0, 0);
        const int64_t wr = (int64_t)(hsh(h0 ^ 0x1234567u) % (uint32_t)a.w_rows);
        float4* wp = reinterpret_cast<float4*>(a.W + wr * a.D) + lane;
        if (a.work & 2) w = *wp;
        if (a.work & 1) {
            float4 v[16];
#pragma unroll
            for (int k = 0; k < 16; k++) {
                const int64_t r = (int64_t)(hsh(h0 + 977u * k) % (uint32_t)a.dy_rows);
                v[k] = k < a.K ? __ldg(reinterpret_cast<const float4*>(a.dY + r * a.D) + lane) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 16; k++) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
        }
        if (a.work & 2) {
            w.x -= 0.01f * acc.x; w.y -= 0.01f * acc.y; w.z -= 0.01f * acc.z; w.w -= 0.01f * acc.w;
            *wp = w;
        }
        if (a.work & 4) {
            for (int k = 0; k < a.K; k++) {
                const int64_t r = (int64_t)(hsh(h0 + 31337u * k) % (uint32_t)a.y_rows);
                __stcs(reinterpret_cast<float4*>(a.Y + r * a.D) + lane, w);
            }
        }
    }
}

template <int LPB>
__global__ void __launch_bounds__(256) k_persist(Args a, int steps, unsigned long long* t) {
    uint64_t t0 = gt();
    for (int s = 0; s < steps; s++) {
        step_work<LPB>(a, s);
        barrier(a.bar, s + 1, a.mode);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) { t[0] = t0; t[1] = gt(); }
}

template <int LPB>
__global__ void __launch_bounds__(256) k_step(Args a, int s) { step_work<LPB>(a, s); }

template <int LPB>
void run(Args a, int grid, int steps, const char* tag) {
    int occ = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_persist<LPB>, 256, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (grid > occ * sms) { printf("%-34s grid=%d exceeds residency %d x %d: skipped\n", tag, grid, occ, sms); return; }
    unsigned long long* t; cudaMalloc(&t, 16);
    cudaMemset(a.bar, 0, 4 * 32 * 4096);
    k_persist<LPB><<<grid, 256>>>(a, 4, t);
    cudaMemset(a.bar, 0, 4 * 32 * 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_persist<LPB><<<grid, 256>>>(a, steps, t);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    // launch-per-step reference (a graph of `steps` launches)
    cudaStream_t st; cudaStreamCreate(&st);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    const int ggrid = (a.units + 256 / LPB - 1) / (256 / LPB);
    for (int s = 0; s < 256; s++) k_step<LPB><<<ggrid > 0 ? ggrid : 1, 256, 0, st>>>(a, s);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < steps / 256; r++) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("%-34s D=%2d grid=%4d units=%6d K=%2d work=%d mode=%d: persistent %6.2f us/step | graph %6.2f us/step %s\n",
           tag, a.D, grid, a.units, a.K, a.work, a.mode, ms * 1e3 / steps, ms2 * 1e3 / (steps / 256 * 256),
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(st); cudaFree(t);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *dY, *W, *Y; uint32_t* bar;
    cudaMalloc(&dY, 256ll << 20); cudaMemset(dY, 0, 256ll << 20);
    cudaMalloc(&W, 1ll << 30); cudaMemset(W, 0, 1ll << 30);
    cudaMalloc(&Y, 32ll << 20); cudaMemset(Y, 0, 32ll << 20);
    cudaMalloc(&bar, 4 * 32 * 4096);
    const int steps = 2048;
    for (int D : {16, 64}) {
        Args a{};
        a.D = D; a.dY = dY; a.dy_rows = (256ll << 20) / (D * 4); a.W = W; a.w_rows = (D == 16 ? 133ll << 20 : 1100ll << 20) / (D * 4);
        if (a.w_rows * D * 4 > (1ll << 30)) a.w_rows = (1ll << 30) / (D * 4);
        a.Y = Y; a.bar = bar;
        const int L = D == 16 ? 53248 : 106496;
        a.y_rows = L;
        for (int mode : {0, 1, 2})
            for (int g : {sms, sms * 2, sms * 3}) {
                a.work = 0; a.units = 0; a.K = 1; a.mode = mode;
                if (D == 16) run<4>(a, g, steps, "barrier only");
            }
        a.mode = 0;
        for (int K : {1, 4, 16}) {
            a.K = K; a.units = L / K;
            for (int work : {1, 2, 4, 7})
                for (int g : {sms * 2, sms * 4}) {
                    a.work = work;
                    if (D == 16) run<4>(a, g, steps, "work");
                    else run<16>(a, g, steps, "work");
                }
        }
    }
    return 0;
}
