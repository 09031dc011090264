// k_views.cu -- stage (c), part 1 on sm_100a: compile every tile's interval
// sequence and pruned views (see bt_views.cuh for the record format).
//
//   k_view_count   thread per tile: runs fetch_interval over the tile's
//                  fragment list, counts intervals and bounds the view nodes
//                  (sum of 2 nAct - 1, the ViewOverflow capacity)
//   k_view_scan    single-pass exclusive scan of the (intervals, nodes) pairs
//   k_view_build   thread per tile: fetch_interval again, Algorithm-1 view
//                  build per interval, records written at the scanned offsets
//
// The fetch loop is re-run instead of stored because it is a few compares per
// fragment, while storing the active sets would cost more traffic than it
// saves.  Tiles outside [tile0, tile1) get no intervals.
#include "bt_device.h"
#include "bt_views.cuh"

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kViewThreads = 64;      // small blocks: the tiles of a frame spread over all SMs

__device__ __forceinline__ uint2 add2(uint2 a, uint2 b) { return make_uint2(a.x + b.x, a.y + b.y); }

__global__ void __launch_bounds__(kViewThreads) k_view_count(Cam cam, TraceParams tp, FrameBufs fb, ViewBufs vb,
                                                             uint32_t tile0, uint32_t tile1, uint32_t tiles) {
    const uint32_t tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= tiles) return;
    uint2 c = make_uint2(0u, 0u);
    if (tile >= tile0 && tile < tile1) {
        const uint32_t off = fb.offsets[tile];
        const uint32_t cnt = fb.offsets[tile + 1] - off;
        if (cnt) {
            TileFetch s;
            fetch_init(s);
            float zb;
            while (fetch_next(s, fb.frags + off, cnt, cam, tp, zb)) {
                c.x += 1u;
                c.y += 2u * s.nAct - 1u;
            }
        }
    }
    vb.count[tile] = c;
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

__global__ void __launch_bounds__(kViewThreads) k_view_build(DevTree t, Cam cam, TraceParams tp, FrameBufs fb,
                                                             ViewBufs vb, uint32_t tile0, uint32_t tile1) {
    const uint32_t tile = tile0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= tile1) return;
    const uint2 c = vb.count[tile];
    if (c.x == 0 || vb.counters[1]) return;  // no intervals, or the frame overflowed (march flags it)
    const uint2 o = view_offset(vb, tile);
    const uint32_t off = fb.offsets[tile];
    const uint32_t cnt = fb.offsets[tile + 1] - off;
    TileFetch s;
    fetch_init(s);
    ViewOut v;
    uint32_t nodeOff = o.y;
    float zb;
    for (uint32_t k = 0; k < c.x && fetch_next(s, fb.frags + off, cnt, cam, tp, zb); ++k) {
        v.nodes = vb.nodes + nodeOff;
        const uint32_t rootUsed = build_view(v, s.actWord, s.nAct, t.words);
        uint32_t flags = 0u;
        if (v.err) flags |= kIvErr;
        if (rootUsed) flags |= kIvRootUsed;
        if (v.maxDepth > kStackCap) flags |= kIvDepthErr;
        IntervalRec r;
        r.zBegin = zb;
        r.zEnd = s.zEnd;
        r.nodeOff = nodeOff;
        r.viewPrim = v.nView | (v.nPrim << 16);
        r.actFlags = s.nAct | (flags << 8);
        r.cacheBytes = v.cacheFloats * 4u;
        r.flops = v.flops;
        r.nBlocks = v.nBlocks;
        uint4* dst = reinterpret_cast<uint4*>(vb.iv + o.x + k);
        const uint4* src = reinterpret_cast<const uint4*>(&r);
        dst[0] = src[0];
        dst[1] = src[1];
        nodeOff += 2u * s.nAct - 1u;
        if (v.err) break;  // the reference's tile loop ends at the first throw
    }
}

}  // namespace

void launch_views(cudaStream_t st, const DevTree& t, const Cam& cam, const TraceParams& tp, const FrameBufs& fb,
                  const ViewBufs& vb, uint32_t tiles, uint32_t tile0, uint32_t tile1, bool build) {
    if (!build) {
        cudaMemsetAsync(vb.counters, 0, 2 * sizeof(uint32_t), st);
        k_view_count<<<(tiles + kViewThreads - 1) / kViewThreads, kViewThreads, 0, st>>>(cam, tp, fb, vb, tile0,
                                                                                          tile1, tiles);
        const uint32_t nblocks = (tiles + kViewScanBlock - 1) / kViewScanBlock;
        k_view_scan<<<nblocks, 1024, 0, st>>>(vb, tiles);
        return;
    }
    if (tile1 > tile0)
        k_view_build<<<(tile1 - tile0 + kViewThreads - 1) / kViewThreads, kViewThreads, 0, st>>>(t, cam, tp, fb, vb,
                                                                                                 tile0, tile1);
}

uint32_t view_scan_blocks(uint32_t tiles) { return (tiles + kViewScanBlock - 1) / kViewScanBlock; }

}  // namespace btk
