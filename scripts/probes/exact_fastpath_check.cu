// exact_fastpath_check.cu -- exhaustive bit check of ExactOps::rcp_mid
// (bt_core.cuh; the A-buffer's box slab test) against the intrinsic it
// replaces: rcp_mid(b) == __frcp_rn(b) for every b with 2^-126 <= |b| < 2^126.
// Measured on a B200: 0 mismatches over 4,227,858,432 inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -I paper_2304_09673_b200/csrc scripts/probes/exact_fastpath_check.cu -o /tmp/fpc && /tmp/fpc
#include <cstdio>
#include "bt_core.cuh"

__device__ unsigned long long g_bad[2], g_n[2];

__global__ void k_check(uint32_t base) {
    const uint32_t u = base + blockIdx.x * blockDim.x + threadIdx.x;  // sign bit clear
    const float a = __uint_as_float(u);
    // rcp_mid on both signs inside its range
    const uint32_t ex = (u >> 23) & 0xFFu;
    if (ex >= 1u && ex <= 252u) {
#pragma unroll
        for (int sgn = 0; sgn < 2; ++sgn) {
            const float b = sgn ? -a : a;
            if (__float_as_uint(__frcp_rn(b)) != __float_as_uint(btk::ExactOps::rcp_mid(b))) atomicAdd(&g_bad[1], 1ull);
        }
        if (threadIdx.x == 0) atomicAdd(&g_n[1], 2ull * blockDim.x);
    }
    if (threadIdx.x == 0) atomicAdd(&g_n[0], blockDim.x);
}

int main() {
    const uint32_t total = 0x80000000u, chunk = 1u << 28;
    for (uint32_t b = 0; b < total; b += chunk) k_check<<<chunk / 256, 256>>>(b);
    unsigned long long bad[2], n[2];
    cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
    cudaMemcpyFromSymbol(n, g_n, sizeof n);
    printf("rcp_mid: %llu mismatches over %llu inputs (%llu scanned)\n", bad[1], n[1], n[0]);
    return bad[1] ? 1 : 0;
}
