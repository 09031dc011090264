// k_views.cu -- stage (c), part 1 on sm_100a: compile every tile's interval
// sequence and pruned views (see bt_views.cuh for the record format).
//
//   k_view_count   warp per tile (WarpFetch): runs fetch_interval over the
//                  tile's fragment list, counts intervals and bounds the view
//                  nodes (sum of 2 nAct - 1, the ViewOverflow capacity)
//   k_view_scan    single-pass exclusive scan of the (intervals, nodes) pairs
//   k_view_fetch   warp per tile: fetch_interval again, writing each
//                  interval's bounds and active words at the scanned offsets
//   k_view_build   thread per INTERVAL: Algorithm-1 view build in place
//
// The fetch loop is re-run instead of stored because it is a few compares per
// fragment, while storing the active sets would cost more traffic than it
// saves.  Tiles outside [tile0, tile1) get no intervals.
#include "bt_device.h"
#include "bt_views.cuh"

#include <algorithm>

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kViewWarps = 4;    // warps (tiles) per block of the fetch passes

__device__ __forceinline__ uint2 add2(uint2 a, uint2 b) { return make_uint2(a.x + b.x, a.y + b.y); }

// Warp per tile (WarpFetch): run the fetch sequence, count intervals and the
// view-node bound; lane 0 also records the scheduling cost proxy.
// Slab of one tile in the count pass's scratch: the intervals (zBegin, zEnd,
// nAct) and their sorted active words, so that the fetch pass can copy
// instead of replaying the fetch sequence.  Tiles that do not fit (more than
// kSlabIv intervals or kSlabWords active words in total) are replayed.
constexpr uint32_t kSlabIv = 32, kSlabWords = 192;
constexpr uint32_t kSlabStride = 1 + 3 * kSlabIv + kSlabWords;  // u32 per tile
constexpr uint32_t kSlabOverflow = 0xFFFFFFFFu;

// Warp per tile (WarpFetch): run the fetch sequence, count intervals and the
// view-node bound, and keep the intervals in the tile's slab; lane 0 also
// records the scheduling cost proxy.
#ifndef BT_VIEW_MINB
#define BT_VIEW_MINB 8  // CTAs per SM the register budget must fit (scripts/viewminb_ab.sh)
#endif
__global__ void __launch_bounds__(kViewWarps * 32, BT_VIEW_MINB) k_view_count(Cam cam, TraceParams tp, FrameBufs fb, ViewBufs vb,
                                                                uint32_t tile0, uint32_t tile1, uint32_t tiles) {
    __shared__ WarpFetchSmem sm[kViewWarps];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const uint32_t tile = blockIdx.x * kViewWarps + wid;
    if (tile >= tiles) return;
    uint2 c = make_uint2(0u, 0u);
    float wsum = 0.0f;  // scheduling cost of the tile's views (below)
    if (tile >= tile0 && tile < tile1) {
        const uint32_t off = fb.offsets[tile];
        const uint32_t cnt = fb.offsets[tile + 1] - off;
        uint32_t* slab = vb.slab + (size_t)tile * kSlabStride;
        if (cnt) {
            WarpFetch f;
            f.init(fb.frags + off, cnt, &sm[wid], lane);
            float zb;
            uint32_t words = 0;
            bool fits = true;
            while (f.next<true>(cam, tp, zb)) {
                const uint32_t n = f.n;
                if (fits && (c.x >= kSlabIv || words + n > kSlabWords)) fits = false;
                if (fits) {
                    if (lane == 0) {
                        slab[1 + 3 * c.x] = __float_as_uint(zb);
                        slab[2 + 3 * c.x] = __float_as_uint(f.zEnd);
                        slab[3 + 3 * c.x] = n;
                    }
#pragma unroll
                    for (int sl = 0; sl < 3; ++sl)
                        if (lane + 32u * sl < n) slab[1 + 3 * kSlabIv + words + lane + 32u * sl] = f.aW[sl];
                    words += n;
                }
                c.x += 1u;
                c.y += 2u * n - 1u;
                {  // view-node bound weighted by the interval's length in view z (fetch windows)
                    const float dvz = FastOps::rcp(cam.invNear - f.zEnd * FastOps::rcp(cam.invDepthRange)) -
                                      FastOps::rcp(cam.invNear - zb * FastOps::rcp(cam.invDepthRange));
                    const float rel = fmaxf(dvz, 0.0f) * FastOps::rcp(tp.window);
                    wsum += (float)(2u * n - 1u) * fminf(4.0f, 1.0f + 4.0f * rel);
                }
            }
            if (lane == 0) slab[0] = fits ? c.x : kSlabOverflow;
        }
        // march cost proxy for longest-first scheduling: 2 x fragments + the
        // view-node bound (2 nAct - 1 per interval) weighted by the interval's
        // view-z length in fetch windows (1x .. 4x) + 16 x the summed NDC depth
        // extent of the fragments (variants compared with scripts/proxy_ab.sh)
        float span = 0.0f;
        for (uint32_t i = lane; i < cnt; i += 32)
            span += __ldg(&fb.frags[off + i].zExit) - __ldg(&fb.frags[off + i].zEntry);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(kFull, span, o);
        if (lane == 0) vb.tileCost[tile] = min(255u, 2u * cnt + (uint32_t)wsum + (uint32_t)(16.0f * fmaxf(span, 0.0f)));
    }
    if (lane == 0) vb.count[tile] = c;
}

// Same single-pass structure as the A-buffer scan (k_frame.cu): each block
// scans 4096 pairs, the last block to finish scans the block sums.
__global__ void __launch_bounds__(1024) k_view_scan(ViewBufs vb, uint32_t tiles) {
    __shared__ uint2 warpSums[32];
    __shared__ bool amLast;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t base = blockIdx.x * kViewScanBlock + tid * 4;
    uint2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (base + k < tiles) ? vb.count[base + k] : make_uint2(0u, 0u);
    const uint2 local = add2(add2(v[0], v[1]), add2(v[2], v[3]));
    uint2 incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nx = __shfl_up_sync(kFull, incl.x, o), ny = __shfl_up_sync(kFull, incl.y, o);
        if (lane >= o) incl = add2(incl, make_uint2(nx, ny));
    }
    if (lane == 31) warpSums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint2 s = warpSums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nx = __shfl_up_sync(kFull, s.x, o), ny = __shfl_up_sync(kFull, s.y, o);
            if (lane >= o) s = add2(s, make_uint2(nx, ny));
        }
        warpSums[lane] = s;  // inclusive
    }
    __syncthreads();
    uint2 run = make_uint2(incl.x - local.x, incl.y - local.y);
    if (wid > 0) run = add2(run, warpSums[wid - 1]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < tiles) vb.local[base + k] = run;
        run = add2(run, v[k]);
    }
    if (tid == 0) {
        vb.blockSum[blockIdx.x] = warpSums[31];
        __threadfence();
        const uint32_t done = atomicAdd(&vb.counters[0], 1u);
        amLast = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (amLast && wid == 0) {
        __threadfence();
        uint2 carry = make_uint2(0u, 0u);
        for (uint32_t b0 = 0; b0 < gridDim.x; b0 += 32) {
            const uint32_t b = b0 + lane;
            uint2 s = make_uint2(0u, 0u);
            if (b < gridDim.x) {
                const volatile uint32_t* p = reinterpret_cast<const volatile uint32_t*>(&vb.blockSum[b]);
                s = make_uint2(p[0], p[1]);
            }
            uint2 inc = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nx = __shfl_up_sync(kFull, inc.x, o), ny = __shfl_up_sync(kFull, inc.y, o);
                if (lane >= o) inc = add2(inc, make_uint2(nx, ny));
            }
            if (b < gridDim.x) vb.blockPrefix[b] = make_uint2(carry.x + inc.x - s.x, carry.y + inc.y - s.y);
            carry.x += __shfl_sync(kFull, inc.x, 31);
            carry.y += __shfl_sync(kFull, inc.y, 31);
        }
        if (lane == 0) {
            vb.blockPrefix[gridDim.x] = carry;
            vb.counters[1] = ((uint64_t)carry.x > vb.ivCap || (uint64_t)carry.y > vb.nodeCap) ? 1u : 0u;
        }
    }
}

// Warp per tile: replay the fetch sequence and write, per interval, the
// partial record (zBegin, zEnd, node range, overlap) and its active words.
// The words go to the LAST nAct slots of the interval's 2 nAct - 1 node
// slots, so the in-place view build below never overwrites an active word
// before reading it (after active i at most 2i + 1 nodes are written).
__global__ void __launch_bounds__(kViewWarps * 32, BT_VIEW_MINB) k_view_fetch(Cam cam, TraceParams tp, FrameBufs fb, ViewBufs vb,
                                                                uint32_t tile0, uint32_t tile1) {
    __shared__ WarpFetchSmem sm[kViewWarps];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const uint32_t tile = tile0 + blockIdx.x * kViewWarps + wid;
    if (tile >= tile1) return;
    const uint2 c = vb.count[tile];
    if (c.x == 0 || vb.counters[1]) return;  // no intervals, or the frame overflowed (march flags it)
    const uint2 o = view_offset(vb, tile);
    const uint32_t* slab = vb.slab + (size_t)tile * kSlabStride;
    uint32_t nodeOff = o.y;
    if (slab[0] != kSlabOverflow) {  // copy the count pass's intervals
        uint32_t words = 0;
        for (uint32_t k = 0; k < c.x; ++k) {
            const uint32_t n = slab[3 + 3 * k];
            uint2* act = vb.nodes + nodeOff + n - 1u;
            for (uint32_t j = lane; j < n; j += 32) act[j].x = slab[1 + 3 * kSlabIv + words + j];
            if (lane == 0) {
                IntervalRec& r = vb.iv[o.x + k];
                r.zBegin = __uint_as_float(slab[1 + 3 * k]);
                r.zEnd = __uint_as_float(slab[2 + 3 * k]);
                r.nodeOff = nodeOff;
                r.actFlags = n;
            }
            words += n;
            nodeOff += 2u * n - 1u;
        }
        return;
    }
    const uint32_t off = fb.offsets[tile];
    const uint32_t cnt = fb.offsets[tile + 1] - off;
    WarpFetch f;
    f.init(fb.frags + off, cnt, &sm[wid], lane);
    float zb;
    for (uint32_t k = 0; k < c.x && f.next<true>(cam, tp, zb); ++k) {
        const uint32_t n = f.n;
        uint2* act = vb.nodes + nodeOff + n - 1u;
#pragma unroll
        for (int sl = 0; sl < 3; ++sl)
            if (lane + 32u * sl < n) act[lane + 32u * sl].x = f.aW[sl];
        if (lane == 0) {
            IntervalRec& r = vb.iv[o.x + k];
            r.zBegin = zb;
            r.zEnd = f.zEnd;
            r.nodeOff = nodeOff;
            r.actFlags = n;
        }
        nodeOff += 2u * n - 1u;
    }
}

// Thread per interval: Algorithm-1 view build over the interval's active
// words, written in place; completes the record.  Intervals are independent
// once their active sets are known, so this pass has no per-tile chain.
__global__ void __launch_bounds__(128) k_view_build(DevTree t, ViewBufs vb, uint32_t totalSlot) {
    if (vb.counters[1]) return;
    const uint32_t total = vb.blockPrefix[totalSlot].x;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        IntervalRec& r = vb.iv[k];
        const uint32_t n = r.actFlags & 0xFFu;
        ViewOut v;
        v.nodes = vb.nodes + r.nodeOff;
        const uint32_t rootUsed = build_view_inplace(v, n, t.words);
        uint32_t flags = 0u;
        if (v.err) flags |= kIvErr;
        if (rootUsed) flags |= kIvRootUsed;
        if (v.maxDepth > kStackCap) flags |= kIvDepthErr;
        r.viewPrim = v.nView | (v.nPrim << 16);
        r.actFlags = n | (flags << 8);
        r.cacheBytes = v.cacheFloats * 4u;
        r.flops = v.flops;
        r.nBlocks = v.nBlocks;
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

void launch_views(cudaStream_t st, const DevTree& t, const Cam& cam, const TraceParams& tp, const FrameBufs& fb,
                  const ViewBufs& vb, uint32_t tiles, uint32_t tile0, uint32_t tile1, bool build, bool zero) {
    if (!build) {
        if (zero) cudaMemsetAsync(vb.counters, 0, 2 * sizeof(uint32_t), st);
        k_view_count<<<(tiles + kViewWarps - 1) / kViewWarps, kViewWarps * 32, 0, st>>>(cam, tp, fb, vb, tile0,
                                                                                         tile1, tiles);
        const uint32_t nblocks = (tiles + kViewScanBlock - 1) / kViewScanBlock;
        k_view_scan<<<nblocks, 1024, 0, st>>>(vb, tiles);
        return;
    }
    if (tile1 > tile0)
        k_view_fetch<<<(tile1 - tile0 + kViewWarps - 1) / kViewWarps, kViewWarps * 32, 0, st>>>(cam, tp, fb, vb,
                                                                                                tile0, tile1);
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((vb.ivCap + 127) / 128, 148u * 16u);
    k_view_build<<<blocks, 128, 0, st>>>(t, vb, (tiles + kViewScanBlock - 1) / kViewScanBlock);
}

size_t view_slab_words(uint32_t tiles) { return (size_t)tiles * kSlabStride; }

uint32_t view_scan_blocks(uint32_t tiles) { return (tiles + kViewScanBlock - 1) / kViewScanBlock; }

}  // namespace btk
