// bt_bulk.cuh -- the TMA bulk-copy engine (cp.async.bulk, non-tensor) for
// staging contiguous per-tile data into shared memory, with an mbarrier
// completion per warp.
//
// A tile's 64 pixel rays are stored tile-major (`tile * 64 + y % 8 * 8 +
// x % 8`, 16 B each): one contiguous, 16-byte aligned 1 KB block -- the one
// layout on this path that a single bulk copy moves as is.  One lane arms the
// warp's barrier with the byte count and issues the copy; the copy engine
// writes shared memory and completes the transaction on the barrier; the
// warp waits on the barrier's phase.  No register staging, two instructions
// per tile instead of two loads + two stores per lane.
//
// Used by k_march (neutral there: C3 march 334-340 us with and without).
// Measured and NOT used in k_tile_raster, which stages the same 1 KB per
// tile: a copy issued and awaited per tile 109 -> 118 us at C3 (the extra
// barrier state pushes the 80-register budget into spills), double-buffered
// with the next tile's copy in flight 109 -> 129 us (each warp then holds two
// tiles of the queue: a longer tail), with or without the proxy fence.
// The other staged data do not have this shape: the fast parameter blocks of
// a view are computed from gathered tree words (convert_node), the candidate
// volumes of a tile are gathered by index, the view's node records are 8 B
// entries at arbitrary offsets (bulk copies need 16 B alignment and size).
#pragma once

#include <stdint.h>

namespace btk {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one arrival (the lane that issues the copy); call from a single lane, then
// __syncwarp before any lane uses the barrier
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Single lane: `bytes` (multiple of 16, both addresses 16 B aligned) from
// global `src` into shared `dst`, completing on `bar`.  The caller has the
// warp's earlier accesses of `dst` ordered before this by a __syncwarp (the
// compiler barrier; no "memory" clobbers here -- they make nvcc spill in
// k_tile_raster), and the proxy fence orders them for the copy engine.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar)));
}

// Every lane: wait for the barrier's phase `parity` to complete.  Bounded: a
// copy that never lands traps (a launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    for (uint32_t spin = 0;; ++spin) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 26)) __trap();
    }
}

}  // namespace btk
