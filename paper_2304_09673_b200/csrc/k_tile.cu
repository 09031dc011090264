// k_tile.cu -- the per-tile stage of the frame on sm_100a: one warp per 8x8
// tile carries the tile from its candidate volumes to its interval records.
//
//   raster  (abuffer.cpp:175-225)  the candidate volumes of the tile's
//           superblock (k_pairs / k_sb_scatter) go through the reference's
//           tile cone test and the tile's pixel-centre pyramid; every survivor
//           is intersected with the tile's 64 pixel rays EXACTLY (two per
//           lane, rays held in registers for the whole tile), clipped,
//           reduced to (zEntry, zExit) and mapped to NDC; the tile's
//           fragments are rank-sorted by (zEntry, word, volume) -- the
//           order insert_sorted builds (abuffer.cpp:166-173) -- and written
//           as the tile's list (bump-allocated, fb.tileFrag);
//   views   (tracer.cpp:50-103)    fetch_interval replayed over the list by
//           the warp (WarpFetch), the intervals and their active words kept
//           in shared memory, the tile's records bump-allocated and written
//           (IntervalRec + the active words in the last nAct of the
//           interval's 2 nAct - 1 node slots), and the march cost proxy.
//
// One warp holds the tile from its candidates to its records: the rays are
// loaded once per tile instead of once per (tile, volume) item, fragments
// never go through a global pool, scan, scatter and sort, and the interval
// sequence is replayed once, from the warp's own sorted list.  The views
// themselves are built by k_view_build (thread per interval, k_views.cu).
#include <algorithm>

#include "bt_cull.cuh"

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kTileWarps = 4;
#ifndef BT_RASTER_UNROLL
#define BT_RASTER_UNROLL 2
#endif
constexpr int kRasterUnroll = BT_RASTER_UNROLL;  // the two rays of a lane: interleaved (2) or in turn (1)
constexpr uint32_t kTileStage = 256;  // fragments of a tile sorted in shared memory (more: sorted from global)
// the intervals of a tile kept for the record pass: at most kSlabIv intervals
// and kSlabWords active words in total (more: the fetch is replayed)
constexpr uint32_t kSlabIv = 32, kSlabWords = 192;

constexpr uint32_t kSmallIv = 136;  // intervals of a <= 32-fragment tile kept: at most 4 F + 2 (k_tile_views)

struct TileSmem {  // views pass, per warp
    union {
        struct {  // WarpFetch path (tiles of more than 32 fragments)
            WarpFetchSmem wf;
            float ivZb[kSlabIv], ivZe[kSlabIv];
            uint32_t ivN[kSlabIv];
            uint32_t words[kSlabWords];
        } big;
        struct {  // lane-per-fragment path: an interval's active set is a lane mask
            float zb[kSmallIv], ze[kSmallIv];
            uint32_t act[kSmallIv];
        } small;
    };
};

// The exact interval of one volume over the tile's rays (abuffer.cpp:198-216):
// every hitting ray's [vz0, vz1] clipped to [near, far]; entry / exit are
// the min / max over the tile (warp reductions; finite values, order-free),
// mapped to NDC once (ndc_from_view_z is monotone: bit for bit the
// reference's per-ray min / max, two divisions per volume instead of two per ray).
template <bool Fm>
__device__ __forceinline__ bool raster_volume(const Cam& cam, const RasterVol& rv, const float4* rays, float& entryOut,
                                              float& exitOut) {
    // the ray-independent terms, once per volume and frame (k_pairs, raster_vol_make)
    const uint32_t family = raster_vol_family(rv);
    const F3 a{rv.q0.x, rv.q0.y, rv.q0.z};
    float entry = f_inf(), exitv = -f_inf();
    bool any = false;
#pragma unroll kRasterUnroll
    for (int h = 0; h < 2; ++h) {
        const float4 rd = rays[(threadIdx.x & 31u) + 32u * h];
        if (!(rd.w > 0.0f)) continue;  // a pixel outside the image (marked w = 0)
        const F3 d{rd.x, rd.y, rd.z};
        float t0, t1;
        bool hit;
        if (family == 0u)
            hit = ray_sphere_pre(a, rv.q0.w, d, t0, t1);
        else if (family == 1u)
            hit = ray_obb_local<Fm>(a, d, Q4{rv.q1.x, rv.q1.y, rv.q1.z, rv.q1.w}, F3{rv.q2.x, rv.q2.y, rv.q2.z}, t0, t1);
        else
            hit = ray_capsule_pre<Fm>(raster_vol_capsule(rv), d, t0, t1);
        if (!hit) continue;
        float vz0 = E::mul(t0, rd.w), vz1 = E::mul(t1, rd.w);
        if (vz1 < cam.nearZ || vz0 > cam.farZ) continue;
        vz0 = smax(vz0, cam.nearZ);
        vz1 = smin(vz1, cam.farZ);
        entry = tmin2<Fm>(entry, vz0);
        exitv = tmax2<Fm>(exitv, vz1);
        any = true;
    }
    if (!__any_sync(kFull, any)) return false;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        entry = tmin2<Fm>(entry, __shfl_xor_sync(kFull, entry, o));
        exitv = tmax2<Fm>(exitv, __shfl_xor_sync(kFull, exitv, o));
    }
    entryOut = ndc_from_view_z_uniform(cam, entry);
    exitOut = ndc_from_view_z_uniform(cam, exitv);
    return true;
}

// Candidates of the tile -> its fragments, fragment k written to sink[k] for
// k < sinkCap; returns the fragment count (warp-uniform).  `tested` counts
// the (tile, volume) pairs ray-tested.
constexpr uint32_t kCullList = 128;  // survivors of the tile cull kept per warp before the ray tests

template <bool Fm>
__device__ uint32_t raster_tile(const Cam& cam, const Voi* vois, const FrameBufs& fb, uint32_t tile, int tx, int ty,
                                int tilesX, uint32_t* list, RasterVol* vstage, float4* rays, uint4* sink,
                                uint32_t sinkCap, uint32_t& tested) {
    const uint32_t lane = threadIdx.x & 31u;
    // the tile's 64 rays, staged once for all its volumes (dot(dir, forward)
    // > 0 inside the image; 0 marks pixels outside it)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int pix = (int)lane + 32 * h;
        const int px = tx * kTile + (pix & 7), py = ty * kTile + (pix >> 3);
        rays[pix] = (px < cam.width && py < cam.height) ? fb.rays[(size_t)tile * 64 + pix] : make_float4(0.f, 0.f, 1.f, 0.f);
    }
    const int sbX = (tilesX + kSB - 1) / kSB;
    const uint32_t sb = (uint32_t)((ty / kSB) * sbX + tx / kSB);
    const uint32_t nCand = min(fb.sbCount[sb], fb.sbCap);
    uint32_t nf = 0;
    tested = 0;
    for (uint32_t base = 0; base < nCand;) {
        // 1. cull: the reference's tile cone (abuffer.cpp:193-196) and the
        // tile's pixel-centre pyramid, one candidate per lane, survivors
        // compacted into the warp's list (the cull state dies before the
        // ray tests: fewer registers live across them)
        uint32_t cnt = 0;
        {  // (re-read per chunk: nothing of the cull stays live across the ray tests)
        const float4 c4 = fb.cones[tile];
        Cone cone;
        cone.axis = F3{c4.x, c4.y, c4.z};
        cone.cosH = c4.w;
        cone.sinH = fb.coneSin[tile];
        const float4* pyramid = fb.tileFrustum + (size_t)tile * 4;
        const uint32_t* cand = fb.sbList + (size_t)sb * fb.sbCap;
        while (base < nCand && cnt + 32u <= kCullList) {
            const uint32_t j = base + lane;
            uint32_t vi = 0;
            bool pass = false;
            if (j < nCand) {
                vi = cand[j];
                const CullVol cv = fb.cullVols[vi];
                pass = cullvol_cone_may_touch(cone, cv) && cullvol_pyramid_may_touch(pyramid, cv);
            }
            const uint32_t m = __ballot_sync(kFull, pass);
            if (pass) list[cnt + __popc(m & ((1u << lane) - 1u))] = vi;
            cnt += __popc(m);
            base += 32;
        }
        }
        tested += cnt;
        __syncwarp();
        // 2. the survivors' exact ray tests, one volume at a time; the
        // volumes' records are gathered 32 at a time into shared memory (one
        // load per lane, all in flight together) instead of one dependent
        // load per volume
        for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
            const uint32_t nc = min(32u, cnt - c0);
            if (lane < nc) vstage[lane] = fb.rasterVols[list[c0 + lane]];
            __syncwarp();
            for (uint32_t i = 0; i < nc; ++i) {
                const RasterVol rv = vstage[i];
                float en, ex;
                if (raster_volume<Fm>(cam, rv, rays, en, ex)) {
                    if (lane == 0 && nf < sinkCap)
                        sink[nf] = make_uint4(raster_vol_word(rv), __float_as_uint(en), __float_as_uint(ex),
                                              list[c0 + i]);
                    ++nf;
                }
            }
            __syncwarp();
        }
    }
    return nf;
}

// rank sort of the tile's n fragment records (src) into its list (dst)
__device__ __forceinline__ void sort_tile(const uint4* src, uint32_t n, Frag* dst) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint4 me = src[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < n; ++j) rank += key_less(src[j], me) ? 1u : 0u;
        Frag f;
        f.word = me.x;
        f.zEntry = __uint_as_float(me.y);
        f.zExit = __uint_as_float(me.z);
        dst[rank] = f;
    }
}

// The march cost proxy of a tile (longest-first scheduling): 2 x fragments +
// the view-node bound (2 nAct - 1 per interval) weighted by the interval's
// view-z length in fetch windows (1x .. 4x) + 16 x the summed NDC depth
// extent of the fragments (variants compared with scripts/proxy_ab.sh)
__device__ __forceinline__ float interval_cost(const Cam& cam, const TraceParams& tp, float zb, float ze, uint32_t n) {
    const float dvz = FastOps::rcp(cam.invNear - ze * FastOps::rcp(cam.invDepthRange)) -
                      FastOps::rcp(cam.invNear - zb * FastOps::rcp(cam.invDepthRange));
    const float rel = fmaxf(dvz, 0.0f) * FastOps::rcp(tp.window);
    return (float)(2u * n - 1u) * fminf(4.0f, 1.0f + 4.0f * rel);
}

// The tile's interval sequence (WarpFetch over its sorted list) -> interval
// records + active words, bump-allocated; vb.count / vb.base / tileCost.
__device__ void views_tile(const Cam& cam, const TraceParams& tp, const FrameBufs& fb, const ViewBufs& vb,
                           TileSmem& S, uint32_t tile, uint32_t fbase, uint32_t cnt) {
    const uint32_t lane = threadIdx.x & 31u;
    uint2 c = make_uint2(0u, 0u);
    float wsum = 0.0f;
    bool kept = true;  // every interval of the tile fits the shared-memory slab
    uint32_t words = 0;
    const Frag* list = fb.frags + fbase;
    if (cnt) {
        WarpFetch f;
        f.init(list, cnt, &S.big.wf, lane);
        float zb;
        while (f.next<true>(cam, tp, zb)) {
            const uint32_t n = f.n;
            if (kept && (c.x >= kSlabIv || words + n > kSlabWords)) kept = false;
            if (kept) {
                if (lane == 0) {
                    S.big.ivZb[c.x] = zb;
                    S.big.ivZe[c.x] = f.zEnd;
                    S.big.ivN[c.x] = n;
                }
#pragma unroll
                for (int sl = 0; sl < 3; ++sl)
                    if (lane + 32u * sl < n) S.big.words[words + lane + 32u * sl] = f.aW[sl];
                words += n;
            }
            c.x += 1u;
            c.y += 2u * n - 1u;
            wsum += interval_cost(cam, tp, zb, f.zEnd, n);
        }
    }
    // march cost proxy for longest-first scheduling: 2 x fragments + the
    // view-node bound (2 nAct - 1 per interval) weighted by the interval's
    // view-z length in fetch windows (1x .. 4x) + 16 x the summed NDC depth
    // extent of the fragments (variants compared with scripts/proxy_ab.sh)
    float span = 0.0f;
    for (uint32_t i = lane; i < cnt; i += 32) span += list[i].zExit - list[i].zEntry;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(kFull, span, o);
    uint2 base = make_uint2(0u, 0u);
    if (lane == 0) {
        vb.tileCost[tile] = min(255u, 2u * cnt + (uint32_t)wsum + (uint32_t)(16.0f * fmaxf(span, 0.0f)));
        if (c.x) {
            base.x = atomicAdd(&vb.counters[2], c.x);
            base.y = atomicAdd(&vb.counters[3], c.y);
        }
    }
    base.x = __shfl_sync(kFull, base.x, 0);
    base.y = __shfl_sync(kFull, base.y, 0);
    const bool fits = (uint64_t)base.x + c.x <= vb.ivCap && (uint64_t)base.y + c.y <= vb.nodeCap;
    if (lane == 0) {
        vb.count[tile] = c;
        vb.base[tile] = base;
        if (c.x && !fits) atomicExch(&vb.counters[1], 1u);  // the march flags the frame's tiles
    }
    if (!c.x || !fits) return;
    uint32_t nodeOff = base.y;
    if (kept) {  // the intervals kept in shared memory
        __syncwarp();
        uint32_t w = 0;
        for (uint32_t k = 0; k < c.x; ++k) {
            const uint32_t n = S.big.ivN[k];
            uint2* act = vb.nodes + nodeOff + n - 1u;
            for (uint32_t j = lane; j < n; j += 32) act[j].x = S.big.words[w + j];
            if (lane == 0) {
                IntervalRec& r = vb.iv[base.x + k];
                r.zBegin = S.big.ivZb[k];
                r.zEnd = S.big.ivZe[k];
                r.nodeOff = nodeOff;
                r.actFlags = n;
            }
            w += n;
            nodeOff += 2u * n - 1u;
        }
        return;
    }
    WarpFetch f;  // too many intervals for the slab: replay the fetch sequence
    f.init(list, cnt, &S.big.wf, lane);
    float zb;
    for (uint32_t k = 0; k < c.x && f.next<true>(cam, tp, zb); ++k) {
        const uint32_t n = f.n;
        uint2* act = vb.nodes + nodeOff + n - 1u;
#pragma unroll
        for (int sl = 0; sl < 3; ++sl)
            if (lane + 32u * sl < n) act[lane + 32u * sl].x = f.aW[sl];
        if (lane == 0) {
            IntervalRec& r = vb.iv[base.x + k];
            r.zBegin = zb;
            r.zEnd = f.zEnd;
            r.nodeOff = nodeOff;
            r.actFlags = n;
        }
        nodeOff += 2u * n - 1u;
    }
}

// fetch_interval (tracer.cpp:50-103) for a tile of at most 32 fragments,
// lane j holding fragment j of the sorted list: the active set is a lane
// mask, expiry one ballot, the fetch one segmented prefix-max scan of the
// exits, and the word order of the actives a popcount against each lane's
// static "words below mine" mask.  The view z of every entry (the window
// test) is computed once per fragment.  Same compares and exact operations
// as WarpFetch (bt_views.cuh) -- bit-identical intervals and active sets.
struct LaneFetch {
    uint32_t w;
    float en, ex, vzEn;
    uint32_t cnt, lane, active, n, cursor;
    float zEnd;

    BT_DEV void init(const Frag* list, uint32_t count, const Cam& cam) {
        lane = threadIdx.x & 31u;
        cnt = count;
        w = 0xFFFFFFFFu;
        en = f_inf();
        ex = -f_inf();
        vzEn = 0.0f;
        if (lane < count) {
            const Frag f = list[lane];
            w = f.word;
            en = f.zEntry;
            ex = f.zExit;
            vzEn = view_z_from_ndc(cam, en);
        }
        active = 0u;
        n = 0u;
        cursor = 0u;
        zEnd = 0.0f;
    }

    BT_DEV bool next(const Cam& cam, const TraceParams& tp, float& zBeginOut) {
        constexpr uint32_t kF = 0xFFFFFFFFu;
        const float zEndPrev = zEnd;
        const bool mine = (active >> lane) & 1u;
        const uint32_t expMask = __ballot_sync(kF, mine && ex <= zEndPrev);
        const bool expired = expMask != 0u;
        active &= ~expMask;
        n = __popc(active);
        const bool hasNext = cursor < cnt;
        if (n == 0u && !hasNext) return false;
        float zBegin = zEndPrev;
        if (hasNext) zBegin = smax(zEndPrev, __shfl_sync(kF, en, cursor));
        const float zBeginView = view_z_from_ndc(cam, zBegin);
        float maxExit = ((active >> lane) & 1u) ? ex : -f_inf();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxExit = fmaxf(maxExit, __shfl_xor_sync(kF, maxExit, o));
        // candidates cursor .. cnt-1: inclusive prefix max of their exits
        const bool cand = lane >= cursor && lane < cnt;
        float inclMax = cand ? ex : -f_inf();
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float v = __shfl_up_sync(kF, inclMax, o);
            if (lane >= (uint32_t)o) inclMax = fmaxf(inclMax, v);
        }
        float exclMax = __shfl_up_sync(kF, inclMax, 1);
        if (lane == 0) exclMax = -f_inf();
        bool ok = false;
        if (cand) {
            const uint32_t fj = lane - cursor, nj = n + fj;
            const float mx = fmaxf(maxExit, exclMax);
            ok = nj == 0u || !(en > mx || fj >= tp.maxNew || nj >= tp.maxOverlap ||
                               E::sub(vzEn, zBeginView) >= tp.window);
        }
        const uint32_t okMask = __ballot_sync(kF, ok) >> cursor;  // candidates in list order
        const uint32_t fetched = okMask == 0xFFFFFFFFu ? 32u : (uint32_t)(__ffs(~okMask) - 1);
        if (fetched) {
            maxExit = fmaxf(maxExit, __shfl_sync(kF, inclMax, cursor + fetched - 1u));
            active |= (fetched >= 32u ? 0xFFFFFFFFu : ((1u << fetched) - 1u)) << cursor;
            n += fetched;
            cursor += fetched;
        }
        float zEndNew = maxExit;
        if (cursor < cnt) zEndNew = smin(__shfl_sync(kF, en, cursor), maxExit);
        if (zEndNew <= zBegin && fetched == 0u && !expired) {
            float minExit = ((active >> lane) & 1u) ? ex : f_inf();
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) minExit = fminf(minExit, __shfl_xor_sync(kF, minExit, o));
            zEndNew = minExit;
        }
        zEnd = zEndNew;
        zBeginOut = zBegin;
        return true;
    }
};

// views_tile for a tile of at most 32 fragments (LaneFetch)
__device__ void views_tile_small(const Cam& cam, const TraceParams& tp, const FrameBufs& fb, const ViewBufs& vb,
                                 TileSmem& S, uint32_t tile, uint32_t fbase, uint32_t cnt) {
    const uint32_t lane = threadIdx.x & 31u;
    const Frag* list = fb.frags + fbase;
    LaneFetch f;
    f.init(list, cnt, cam);
    // static word order: the lanes whose word is below mine (words are unique in a tile)
    uint32_t below = 0u;
    for (uint32_t k = 0; k < cnt; ++k) below |= (__shfl_sync(kFull, f.w, k) < f.w ? 1u : 0u) << k;
    uint2 c = make_uint2(0u, 0u);
    float wsum = 0.0f;
    bool kept = true;
    float zb;
    while (f.next(cam, tp, zb)) {
        if (c.x >= kSmallIv) kept = false;
        if (kept && lane == 0) {
            S.small.zb[c.x] = zb;
            S.small.ze[c.x] = f.zEnd;
            S.small.act[c.x] = f.active;
        }
        c.x += 1u;
        c.y += 2u * f.n - 1u;
        wsum += interval_cost(cam, tp, zb, f.zEnd, f.n);
    }
    float span = lane < cnt ? f.ex - f.en : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(kFull, span, o);
    uint2 base = make_uint2(0u, 0u);
    if (lane == 0) {
        vb.tileCost[tile] = min(255u, 2u * cnt + (uint32_t)wsum + (uint32_t)(16.0f * fmaxf(span, 0.0f)));
        if (c.x) {
            base.x = atomicAdd(&vb.counters[2], c.x);
            base.y = atomicAdd(&vb.counters[3], c.y);
        }
    }
    base.x = __shfl_sync(kFull, base.x, 0);
    base.y = __shfl_sync(kFull, base.y, 0);
    const bool fits = (uint64_t)base.x + c.x <= vb.ivCap && (uint64_t)base.y + c.y <= vb.nodeCap;
    if (lane == 0) {
        vb.count[tile] = c;
        vb.base[tile] = base;
        if (c.x && !fits) atomicExch(&vb.counters[1], 1u);  // the march flags the frame's tiles
    }
    if (!c.x || !fits) return;
    uint32_t nodeOff = base.y;
    auto emit = [&](uint32_t k, float zBegin, float zEnd, uint32_t act) {
        const uint32_t n = __popc(act);
        // active words in word order into the last n of the 2n - 1 node slots
        if ((act >> lane) & 1u) vb.nodes[nodeOff + n - 1u + __popc(act & below)].x = f.w;
        if (lane == 0) {
            IntervalRec& r = vb.iv[base.x + k];
            r.zBegin = zBegin;
            r.zEnd = zEnd;
            r.nodeOff = nodeOff;
            r.actFlags = n;
        }
        nodeOff += 2u * n - 1u;
    };
    if (kept) {
        __syncwarp();
        for (uint32_t k = 0; k < c.x; ++k) emit(k, S.small.zb[k], S.small.ze[k], S.small.act[k]);
        return;
    }
    f.init(list, cnt, cam);  // more intervals than kept: replay
    for (uint32_t k = 0; k < c.x && f.next(cam, tp, zb); ++k) emit(k, zb, f.zEnd, f.active);
}

// Persistent warps over the tiles of [tile0, tile1) (a work queue: tiles
// differ by orders of magnitude in candidates and fragments).  Raster and
// views are two kernels with their own register budgets (together in one
// they spill); the views pass reads the tile's list back from L2.
#ifndef BT_RASTER_FM
#define BT_RASTER_FM 1
#endif
#ifndef BT_TILE_MINB
#define BT_TILE_MINB 7  // CTAs per SM the register budget of k_tile_raster must fit (62 registers)
#endif
__device__ __forceinline__ uint32_t next_tile(uint32_t* queue, uint32_t tile0) {
    uint32_t q = 0;
    if ((threadIdx.x & 31u) == 0) q = atomicAdd(queue, 1u);
    return tile0 + __shfl_sync(kFull, q, 0);
}

template <bool Fm>
__global__ void __launch_bounds__(kTileWarps * 32, BT_TILE_MINB)
    k_tile_raster(Cam cam, const Voi* vois, FrameBufs fb, int tilesX, uint32_t tile0, uint32_t tile1) {
    __shared__ uint4 stage[kTileWarps][kTileStage];
    __shared__ uint32_t culled[kTileWarps][kCullList];
    __shared__ RasterVol vstaged[kTileWarps][32];
    __shared__ float4 tileRays[kTileWarps][64];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    // a superblock candidate list that outgrew its capacity: empty,
    // flagged A-buffer (the checked path grows the buffers and rebuilds)
    const bool pairsLost = fb.counters[kCntSbNeed] != 0u;
    uint32_t testedSum = 0;
    for (uint32_t tile = next_tile(&fb.counters[kCntTileQueue], tile0); tile < tile1;
         tile = next_tile(&fb.counters[kCntTileQueue], tile0)) {
        const int tx = (int)(tile % (uint32_t)tilesX), ty = (int)(tile / (uint32_t)tilesX);
        uint32_t fbase = 0, nf = 0;
        if (!pairsLost) {
            uint32_t tested = 0;
            nf = raster_tile<Fm>(cam, vois, fb, tile, tx, ty, tilesX, culled[wid], vstaged[wid], tileRays[wid], stage[wid], kTileStage, tested);
            testedSum += tested;
        }
        if (lane == 0 && nf) fbase = atomicAdd(&fb.counters[kCntFrags], nf);
        fbase = __shfl_sync(kFull, fbase, 0);
        if ((uint64_t)fbase + nf > fb.fragCap) {  // the fragment store outgrew its buffer
            if (lane == 0) atomicExch(&fb.counters[kCntOverflow], 1u);
            nf = 0;
        } else if (nf > kTileStage) {  // rare: too many fragments to sort in shared memory
            uint32_t tested = 0;
            raster_tile<Fm>(cam, vois, fb, tile, tx, ty, tilesX, culled[wid], vstaged[wid], tileRays[wid], fb.unsorted + fbase, nf, tested);
            __syncwarp();
            sort_tile(fb.unsorted + fbase, nf, fb.frags + fbase);
        } else if (nf) {
            __syncwarp();
            sort_tile(stage[wid], nf, fb.frags + fbase);
        }
        if (lane == 0) {
            fb.tileFrag[tile] = make_uint2(fbase, nf);
            if (pairsLost && tile == tile0) atomicExch(&fb.counters[kCntOverflow], 1u);
        }
        __syncwarp();
    }
    if (lane == 0 && testedSum) atomicAdd(&fb.counters[kCntPool], testedSum);
}

__global__ void __launch_bounds__(kTileWarps * 32, 7)
    k_tile_views(Cam cam, TraceParams tp, FrameBufs fb, ViewBufs vb, uint32_t tile0, uint32_t tile1) {
    __shared__ TileSmem sm[kTileWarps];
    TileSmem& S = sm[threadIdx.x >> 5];
    for (uint32_t tile = next_tile(&fb.counters[kCntTileQueue + 1], tile0); tile < tile1;
         tile = next_tile(&fb.counters[kCntTileQueue + 1], tile0)) {
        const uint2 tf = fb.tileFrag[tile];
        if (tf.y <= 32u) views_tile_small(cam, tp, fb, vb, S, tile, tf.x, tf.y);
        else views_tile(cam, tp, fb, vb, S, tile, tf.x, tf.y);
        __syncwarp();
    }
}

}  // namespace

void launch_tile_pass(cudaStream_t st, uint32_t mode, const Cam& cam, const TraceParams& tp, const Voi* vois,
                      const FrameBufs& fb, const ViewBufs& vb, int tilesX, int tilesY, uint32_t tile0,
                      uint32_t tile1, int smCount) {
    const uint32_t tiles = (uint32_t)(tilesX * tilesY);
    cudaMemsetAsync(fb.counters + kCntTileQueue, 0, 2 * sizeof(uint32_t), st);
    // tiles outside [tile0, tile1) keep empty lists / no records (a sharded
    // frame's normals read every tile's records); the passes write every
    // tile of their range, so a whole frame needs no clearing
    const bool partial = tile0 != 0u || tile1 < tiles;
    if ((mode & kTileRaster) && partial) cudaMemsetAsync(fb.tileFrag, 0, (size_t)tiles * sizeof(uint2), st);
    if (mode & kTileViews) {
        if (partial) cudaMemsetAsync(vb.count, 0, (size_t)tiles * sizeof(uint2), st);
        cudaMemsetAsync(vb.counters, 0, 4 * sizeof(uint32_t), st);
    }
    if (tile1 <= tile0) return;
    const uint32_t want = (tile1 - tile0 + kTileWarps - 1) / kTileWarps;
    if (mode & kTileRaster) {
        // FMNMX min / max where they are result-identical (bt_geom.cuh tmin2)
        auto* k = (BT_RASTER_FM && cam.nearZ > 0.0f) ? k_tile_raster<true> : k_tile_raster<false>;
        k<<<std::min<uint32_t>((uint32_t)smCount * BT_TILE_MINB, want), kTileWarps * 32, 0, st>>>(cam, vois, fb,
                                                                                              tilesX, tile0, tile1);
    }
    if (mode & kTileViews)
        k_tile_views<<<std::min<uint32_t>((uint32_t)smCount * 7u, want), kTileWarps * 32, 0, st>>>(cam, tp, fb, vb,
                                                                                                   tile0, tile1);
}

}  // namespace btk
