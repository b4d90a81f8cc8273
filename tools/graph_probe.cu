// graph_probe.cu — per-kernel cost of a CUDA graph of N tiny kernels as N
// grows, with and without programmatic dependent launch (PDL) edges and with
// a 64-byte by-value parameter (ground truth for the epoch runner; not libfae).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct P64 { int64_t a[8]; };

__global__ void k_small(int* x, int s) { if (threadIdx.x == 0 && blockIdx.x == 0 && s < 0) x[0] = s; }
__global__ void k_big(P64 p, int* x, int s) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.a[s & 7] < 0) x[0] = s;
}

float run(int N, bool pdl, bool big, int grid) {
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* x; cudaMalloc(&x, 4);
    P64 p{}; for (int i = 0; i < 8; i++) p.a[i] = i;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256); cfg.gridDim = dim3(grid); cfg.stream = st; cfg.attrs = attr; cfg.numAttrs = 1;
    for (int s = 0; s < N; s++) {
        if (big) cudaLaunchKernelEx(&cfg, k_big, p, x, s);
        else cudaLaunchKernelEx(&cfg, k_small, x, s);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = N >= 4096 ? 2 : 32;
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; r++) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(st); cudaFree(x);
    return ms * 1e3f / (reps * N);
}

int main() {
    for (int grid : {148, 400})
        for (int big : {0, 1})
            for (int pdl : {0, 1})
                for (int N : {256, 2048, 24000})
                    printf("grid=%3d big=%d pdl=%d N=%6d: %.3f us/kernel\n", grid, big, pdl, N, run(N, pdl, big, grid));
    return 0;
}
