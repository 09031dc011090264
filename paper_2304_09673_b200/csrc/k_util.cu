// k_util.cu -- measurement helpers.
//
// k_ffma_peak: FP32 roofline denominator for the field-evaluation kernel.
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only, so the
// non-tensor FP32 peak (SMs x 128 lanes x 2 flop x f_SM) is measured on the
// box: 8 independent FFMA chains per thread, full occupancy, timed with
// CUDA events.
#include <cuda_runtime.h>

#include "../../include/bt_cuda.h"

namespace {

__global__ void __launch_bounds__(256) k_ffma_peak(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x * 1e-7f, x1 = x0 + 1.0f, x2 = x0 + 2.0f, x3 = x0 + 3.0f;
    float x4 = x0 + 4.0f, x5 = x0 + 5.0f, x6 = x0 + 6.0f, x7 = x0 + 7.0f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b);
            x1 = fmaf(x1, a, b);
            x2 = fmaf(x2, a, b);
            x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b);
            x5 = fmaf(x5, a, b);
            x6 = fmaf(x6, a, b);
            x7 = fmaf(x7, a, b);
        }
    }
    const float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

// Gather-copy of up to 8 device segments (16-byte aligned) into one buffer,
// with the SMs: the G-buffer snapshot of the streamed download, kept off the
// copy engines that carry the D2H.
struct CopySegs {
    const uint4* src[8];
    uint4* dst[8];
    uint32_t n16[8];  // 16-byte units
    uint32_t count;
};

__global__ void __launch_bounds__(256) k_copy_segments(CopySegs segs) {
    for (uint32_t s = 0; s < segs.count; ++s) {
        const uint4* __restrict__ a = segs.src[s];
        uint4* __restrict__ b = segs.dst[s];
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < segs.n16[s]; i += gridDim.x * blockDim.x)
            b[i] = a[i];
    }
}

}  // namespace

namespace btk {
// src/dst pointers 16-byte aligned; bytes rounded up to 16 (the snapshot
// slots and the G-buffer planes are cudaMalloc'd and padded)
void launch_copy_segments(cudaStream_t st, const void* const* src, void* const* dst, const size_t* bytes, int n,
                          int smCount) {
    CopySegs segs{};
    segs.count = 0;
    for (int i = 0; i < n && segs.count < 8; ++i) {
        if (!src[i] || !dst[i] || bytes[i] == 0) continue;
        segs.src[segs.count] = static_cast<const uint4*>(src[i]);
        segs.dst[segs.count] = static_cast<uint4*>(dst[i]);
        segs.n16[segs.count] = (uint32_t)((bytes[i] + 15) / 16);
        segs.count++;
    }
    if (segs.count) k_copy_segments<<<smCount * 4, 256, 0, st>>>(segs);
}
}  // namespace btk

extern "C" BT_API int bt_fp32_peak(int device, float* tflops, float* ms_out) {
    if (cudaSetDevice(device) != cudaSuccess) return BT_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return BT_ENOMEM;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    k_ffma_peak<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);  // warm-up / clock ramp
    k_ffma_peak<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    k_ffma_peak<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    if (tflops) *tflops = (float)(flops / (ms * 1e-3) / 1e12);
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? BT_OK : BT_ECUDA;
}
