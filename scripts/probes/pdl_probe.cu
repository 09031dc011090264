// Probe: per-boundary cost of a chain of small dependent kernels in a CUDA
// graph, with and without programmatic dependent launch (PDL).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pdl_probe pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(float* buf, int n, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = buf[i] * 0.999f + 1.0f;
}

int main() {
    const int n = 1 << 16, chain = 20, reps = 200;
    float* buf;
    cudaMalloc(&buf, n * sizeof(float));
    cudaMemset(buf, 0, n * sizeof(float));
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int blocks : {148, 1184}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < chain; ++k) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(256);
                cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                cudaLaunchKernelEx(&cfg, k_step, buf, n, pdl);
            }
            cudaStreamEndCapture(st, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, st);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
            for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("blocks %4d pdl %d: %.2f us per kernel in a %d-kernel graph (%s)\n", blocks, pdl,
                   ms * 1e3 / reps / chain, chain, cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    return 0;
}
