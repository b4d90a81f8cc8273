// gather_probe.cu — measures random-row gather throughput on the GPU
// (ground truth for the hot-step kernels' design).  Not part of libfae.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// each group of LPB lanes gathers U rows (D floats) per iteration, idx from an index array
template <int LPB, int U>
__global__ void gather(const float* __restrict__ W, int64_t rows, int D, const int32_t* __restrict__ idx,
                       int64_t n, float* __restrict__ out) {
    const int lane = threadIdx.x % LPB;
    const int64_t gpb = blockDim.x / LPB;
    const int64_t groups = (int64_t)gridDim.x * gpb;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t b0 = (blockIdx.x * gpb + threadIdx.x / LPB) * U; b0 < n; b0 += groups * U) {
        int32_t r[U];
#pragma unroll
        for (int u = 0; u < U; u++) r[u] = b0 + u < n ? __ldg(idx + b0 + u) : 0;
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = __ldg(reinterpret_cast<const float4*>(W + (int64_t)r[u] * D) + lane);
#pragma unroll
        for (int u = 0; u < U; u++) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x == 1234.5f) out[0] = acc.y;
}

__global__ void fill_idx(int32_t* idx, int64_t n, int64_t rows, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        idx[i] = (int32_t)((((uint64_t)hsh((uint32_t)i ^ seed) << 32) | hsh((uint32_t)i * 7 + seed)) % rows);
}

template <int LPB, int U>
void run(const float* W, int64_t rows, int D, const int32_t* idx, int64_t n, float* out, int grid, const char* tag) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    gather<LPB, U><<<grid, 256>>>(W, rows, D, idx, n, out);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; i++) gather<LPB, U><<<grid, 256>>>(W, rows, D, idx, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    double bytes = (double)n * D * 4 + n * 4.0;
    printf("%-28s D=%3d n=%9lld grid=%5d U=%d: %8.2f us  %7.1f GB/s\n", tag, D, (long long)n, grid, U, ms * 1e3, bytes / ms / 1e6);
}

int main() {
    const int64_t bytesW = 1ll << 30;
    float* W; cudaMalloc(&W, bytesW); cudaMemset(W, 0, bytesW);
    float* out; cudaMalloc(&out, 64);
    int32_t* idx; cudaMalloc(&idx, sizeof(int32_t) * (64 << 20));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int D : {16, 64}) {
        const int64_t rows = bytesW / (D * 4);
        for (int64_t n : {(int64_t)53248, (int64_t)106496, (int64_t)(16 << 20)}) {
            fill_idx<<<1024, 256>>>(idx, n, rows, 12345);
            for (int g : {sms * 2, sms * 4, sms * 8}) {
                if (D == 16) { run<4, 1>(W, rows, D, idx, n, out, g, "LPB4"); run<4, 4>(W, rows, D, idx, n, out, g, "LPB4"); run<4, 16>(W, rows, D, idx, n, out, g, "LPB4"); }
                else { run<16, 1>(W, rows, D, idx, n, out, g, "LPB16"); run<16, 4>(W, rows, D, idx, n, out, g, "LPB16"); run<16, 16>(W, rows, D, idx, n, out, g, "LPB16"); }
            }
        }
    }
    // launch overhead: empty kernel back to back
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 1000; i++) gather<4, 1><<<sms, 256>>>(W, 1, 16, idx, 0, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel back-to-back: %.2f us each\n", ms);
    return 0;
}
