// ffma_forms.cu -- FP32 issue/throughput of FFMA forms on the box:
//   k_cc   fma(x, a, b) with a, b kernel parameters (bt_fp32_peak's form)
//   k_rrr  fma(x, y, z) with three lane-varying registers
//   k_f2   FFMA2 (fma.rn.f32x2): two FP32 FMAs per instruction
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/probes/ffma_forms.cu -o /tmp/ffma_forms && /tmp/ffma_forms
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_cc(float* out, int iters, float a, float b) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-7f + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_rrr(float* out, int iters, float a, float b) {
    float x[8], y[8], z[8];
    for (int k = 0; k < 8; ++k) {
        x[k] = threadIdx.x * 1e-7f + k;
        y[k] = a + threadIdx.x * 1e-9f * k;
        z[k] = b - threadIdx.x * 1e-9f * k;
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], y[k], z[(k + u) & 7]);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_f2(float* out, int iters, float a, float b) {
    unsigned long long x[8], y[8], z[8];
    for (int k = 0; k < 8; ++k) {
        float x0 = threadIdx.x * 1e-7f + k, x1 = x0 + 0.5f;
        float y0 = a + threadIdx.x * 1e-9f * k, z0 = b - threadIdx.x * 1e-9f * k;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[k]) : "f"(x0), "f"(x1));
        asm("mov.b64 %0, {%1, %2};" : "=l"(y[k]) : "f"(y0), "f"(y0));
        asm("mov.b64 %0, {%1, %2};" : "=l"(z[k]) : "f"(z0), "f"(z0));
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(y[k]), "l"(z[(k + u) & 7]));
    float s = 0;
    for (int k = 0; k < 8; ++k) {
        float a0, a1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x[k]));
        s += a0 + a1;
    }
    if (s == 1234.5f) out[0] = s;
}

template <class K> float run(K k, float* out, int sms, double flopsPerIter) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    k<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
    k<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return (float)(flopsPerIter * iters * blocks * threads / (ms * 1e-3) / 1e12);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    for (int rep = 0; rep < 2; ++rep) {
        printf("FFMA param-operand form: %.1f TFLOP/s\n", run(k_cc, out, sms, 2.0 * 8 * 16));
        printf("FFMA three-register form: %.1f TFLOP/s\n", run(k_rrr, out, sms, 2.0 * 8 * 16));
        printf("FFMA2 (fma.rn.f32x2):     %.1f TFLOP/s\n", run(k_f2, out, sms, 4.0 * 8 * 16));
    }
    return 0;
}
