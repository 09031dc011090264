// k_views.cu -- stage (c), part 1 on sm_100a: the pruned views of every
// interval record (see bt_views.cuh for the record format), and the march
// schedule.
//
//   k_view_build   lane per INTERVAL, refilled from a queue: Algorithm-1 view
//                  build in place over the records k_tile (k_tile.cu) wrote,
//                  one node dereference per step
//   k_order_*      longest-first march units from the tiles' cost proxy
#include "bt_device.h"
#include "bt_views.cuh"

#include <algorithm>

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
// Algorithm-1 view build of every interval record, in place over the
// interval's active words (intervals are independent once their active sets
// are known: no per-tile chain).  Thread per interval (grid stride), the
// view built by ViewBuild one node dereference per step; the traversal
// stacks live in shared memory (one u32 per entry, strided by the block
// size: conflict-free), the tree's blob headers come from the dense blob
// table.  Measured (C3 / C4 / C5, us): thread loop with a local-memory stack
// and float4 blob reads 16 / 43 / 92; this 11 / 40 / 57.  Tried: a
// warp-uniform step loop with lanes refilled from the interval queue
// (14 / 54 / 86: the per-step vote and refill cost more than the divergence
// it removes) and the per-node bookkeeping deferred to a pass over the
// finished view (18 / 123 / 183: the read-back of the view nodes).
constexpr uint32_t kViewThreads = 128;
#ifndef BT_VIEW_BLOCKS
#define BT_VIEW_BLOCKS 12
#endif

__device__ __forceinline__ void view_finish(const ViewBufs& vb, uint32_t k, const ViewBuild& b) {
    IntervalRec& r = vb.iv[k];
    uint32_t flags = 0u;
    if (b.v.err) flags |= kIvErr;
    if (b.rootUsed) flags |= kIvRootUsed;
    if (b.v.maxDepth > kStackCap) flags |= kIvDepthErr;
    r.viewPrim = b.v.nView | (b.v.nPrim << 16);
    r.actFlags = b.n | (flags << 8);
    r.cacheBytes = b.v.cacheFloats * 4u;
    r.flops = b.v.flops;
    r.nBlocks = b.v.nBlocks;
}

__global__ void __launch_bounds__(kViewThreads) k_view_build(DevTree t, ViewBufs vb) {
    __shared__ uint32_t stk[kStackCap * kViewThreads];
    if (vb.counters[1]) return;
    const uint32_t total = vb.counters[2];  // records allocated by k_tile
    const uint32_t stride = gridDim.x * kViewThreads;
    uint32_t k = blockIdx.x * kViewThreads + threadIdx.x;
    if (__all_sync(kFull, k >= total)) return;
    uint32_t* myStk = stk + threadIdx.x;
    ViewBuild b;
    for (; k < total; k += stride) {
        b.begin(vb.nodes + vb.iv[k].nodeOff, vb.iv[k].actFlags & 0xFFu, t.blobs);
        while (!b.done) b.step(t.blobs, myStk, kViewThreads);
        view_finish(vb, k, b);
    }
}

// ---------------------------------------------------------------- scheduling
// Longest-first order for the march: the persistent march kernel ends when
// its slowest tile does, so tiles are queued by a cost proxy known before the
// march (k_view_count: 4 x fragments + 16 x summed NDC depth extent, which
// tracks the per-tile march steps; measured on C2/C3/C5 it recovers most of
// the gain of an oracle order).  Counting sort on the proxy (256 bins),
// descending; equal keys in any order -- the order never changes results.
constexpr uint32_t kOrderBins = 256;

__device__ __forceinline__ uint32_t order_key(const ViewBufs& vb, uint32_t tile) {
    return kOrderBins - 1u - min(vb.tileCost[tile], kOrderBins - 1u);  // ascending key = descending cost
}

__global__ void k_order_count(ViewBufs vb, uint32_t* hist, uint32_t tile0, uint32_t tile1) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t tile = tile0 + i;
    const uint32_t key = tile < tile1 ? order_key(vb, tile) : kOrderBins;
    const uint32_t peers = __match_any_sync(kFull, key);
    if (key < kOrderBins && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[key], __popc(peers));
}

// One CTA: bin starts of the march units.  Expensive tiles are also SPLIT:
// each becomes two units (odd / even pixel columns) marched by two warps,
// halving the latency of the tiles that bound the kernel's tail.  A tile is
// split when its cost proxy is at least `beta` x the average work per warp of
// the grid (total cost / warps) -- many tiles per warp (large frames) split
// almost nothing, few tiles per warp (small frames) split the heavy ones --
// and at most `cap` tiles are split.  hist[256] = first unsplit key,
// hist[257] = total units.
__global__ void __launch_bounds__(kOrderBins) k_order_scan(uint32_t* hist, uint32_t nWarps, float beta,
                                                           uint32_t cap) {
    __shared__ uint32_t warpSums[kOrderBins / 32];
    __shared__ float costSum[kOrderBins / 32];
    __shared__ uint32_t splitEnd;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    auto block_scan = [&](uint32_t v) -> uint32_t {  // inclusive
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += n;
        }
        __syncthreads();
        if (lane == 31) warpSums[w] = incl;
        __syncthreads();
        uint32_t base = 0;
        for (int k = 0; k < w; ++k) base += warpSums[k];
        return base + incl;
    };
    const uint32_t v = hist[t];
    const float cost = (float)(kOrderBins - 1 - t);
    float c = (float)v * cost;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0) costSum[w] = c;
    if (t == 0) splitEnd = 0;
    __syncthreads();
    float total = 0.0f;
    for (int k = 0; k < (int)(kOrderBins / 32); ++k) total += costSum[k];
    const uint32_t incl = block_scan(v);
    // bins 0..splitEnd-1 are split (a prefix: costs decrease with the key)
    if (v > 0 && t < (int)kOrderBins - 1 && cost * (float)nWarps >= beta * total && incl <= cap)
        atomicMax(&splitEnd, (uint32_t)t + 1u);
    __syncthreads();
    const uint32_t units = t < (int)splitEnd ? 2u * v : v;
    const uint32_t uincl = block_scan(units);
    hist[t] = uincl - units;  // exclusive start of the bin = its scatter cursor
    if (t == (int)kOrderBins - 1) {
        hist[kOrderBins] = splitEnd;
        hist[kOrderBins + 1] = uincl;
    }
}

__global__ void k_order_scatter(ViewBufs vb, GBuf g, uint32_t* cursor, uint32_t* order, uint32_t tile0,
                                uint32_t tile1) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t tile = tile0 + i;
    const uint32_t key = tile < tile1 ? order_key(vb, tile) : kOrderBins;
    const bool split = key < cursor[kOrderBins];
    const uint32_t peers = __match_any_sync(kFull, key);
    const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
    const uint32_t per = split ? 2u : 1u;
    uint32_t base = 0;
    if (key < kOrderBins && lane == leader) base = atomicAdd(&cursor[key], per * __popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (key >= kOrderBins) return;
    const uint32_t pos = base + per * __popc(peers & ((1u << lane) - 1u));
    if (split) {
        order[pos] = tile | kUnitSplit;
        order[pos + 1] = tile | kUnitSplit | kUnitPart1;
        // the two halves combine the tile planes with max (k_march); tileCost
        // becomes the halves' "error counted" flag
        vb.tileCost[tile] = 0;
        g.tileMaxOverlap[tile] = 0;
        g.tileCacheBytes[tile] = 0;
        g.tileError[tile] = 0;
    } else {
        order[pos] = tile;
    }
}

}  // namespace

void launch_tile_order(cudaStream_t st, const ViewBufs& vb, const GBuf& g, uint32_t* hist, uint32_t* order,
                       uint32_t tile0, uint32_t tile1, uint32_t nWarps, float beta, uint32_t cap) {
    if (tile1 <= tile0) return;
    const uint32_t n = tile1 - tile0, blocks = (n + 255) / 256;
    cudaMemsetAsync(hist, 0, kOrderBins * sizeof(uint32_t), st);
    k_order_count<<<blocks, 256, 0, st>>>(vb, hist, tile0, tile1);
    k_order_scan<<<1, kOrderBins, 0, st>>>(hist, nWarps, beta, cap);
    k_order_scatter<<<blocks, 256, 0, st>>>(vb, g, hist, order, tile0, tile1);
}

void launch_view_build(cudaStream_t st, const DevTree& t, const ViewBufs& vb, int smCount) {
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((vb.ivCap + kViewThreads - 1) / kViewThreads,
                                                         (uint64_t)smCount * BT_VIEW_BLOCKS);
    k_view_build<<<blocks, kViewThreads, 0, st>>>(t, vb);
}

}  // namespace btk
