// bt_views.cuh -- stage (c), part 1: the interval sequence and the pruned
// views of every tile, compiled ahead of the march.
//
// The reference interleaves, per tile, a serial fetch_interval + view build
// (tracer.cpp:50-103, traversal.cpp:30-99) with the 64-ray march of each
// interval (tracer.cpp:155-232).  Neither the intervals nor the views depend
// on the march -- the march only decides how far down the list a tile goes
// (it stops once all 64 rays have hit).  So the serial part runs here as one
// THREAD per tile over the whole list (k_views.cu), 32 tiles per warp instead
// of one lane of a 32-lane warp, and the march kernel reads the compiled
// records:
//
//   IntervalRec (32 B)  zBegin/zEnd (NDC), the view's node range, overlap,
//                       cache bytes, flags, appendix-B flops, fast-block size
//   ViewNode    (8 B)   hdr = isPrim(1) op(5, possibly a reserved code) |
//                       float4 offset of the node's fast parameter block;
//                       word = tree word of the node's parameters
//
// Semantics carried per record so that the march reproduces the reference
// loop exactly (tracer.cpp:165-230): overlap -> tileMaxOverlap; an overflow
// (TraversalOverflow / ViewOverflow) ends the tile with tileError; cache
// bytes -> tileCacheBytes; !rootUsed or an empty interval is skipped; an
// evaluation stack deeper than 22 ends the tile with tileError.
#pragma once

#include "bt_tile.cuh"

namespace btk {

constexpr uint32_t kIvErr = 1u;       // view build threw (stack / view overflow, logic)
constexpr uint32_t kIvRootUsed = 2u;  // PrunedView::rootUsed
constexpr uint32_t kIvDepthErr = 4u;  // eval stack deeper than kStackCap

struct alignas(16) IntervalRec {
    float zBegin, zEnd;
    uint32_t nodeOff;    // absolute index of the first ViewNode
    uint32_t viewPrim;   // nView | nPrim << 16
    uint32_t actFlags;   // nAct | flags << 8
    uint32_t cacheBytes;
    uint32_t flops;      // appendix-B flops of one evaluation of the view
    uint32_t nBlocks;    // float4s of fast parameter blocks of the view
};
static_assert(sizeof(IntervalRec) == 32, "IntervalRec is two uint4");

struct ViewBufs {
    uint2* count = nullptr;        // [tiles] (intervals, node bound) from the count pass
    uint2* local = nullptr;        // [tiles] exclusive scan inside a scan block
    uint2* blockSum = nullptr;     // [scan blocks]
    uint2* blockPrefix = nullptr;  // [scan blocks + 1], total at the end
    IntervalRec* iv = nullptr;     // [ivCap]
    uint2* nodes = nullptr;        // [nodeCap] (hdr, word)
    uint32_t* counters = nullptr;  // [0] scan completion, [1] overflow flag
    const uint32_t* order = nullptr;  // optional march units in order (tile | kUnitSplit | kUnitPart1), else raster
    const uint32_t* unitCount = nullptr;  // number of entries of `order` (device)
    uint32_t* tileCost = nullptr;     // [tiles] march cost proxy 0..255 (k_view_count; scheduling)
    uint64_t ivCap = 0, nodeCap = 0;
};

constexpr uint32_t kViewScanBlock = 4096;
constexpr uint32_t kUnitSplit = 0x80000000u;  // march unit = half a tile (one pixel-column parity)
constexpr uint32_t kUnitPart1 = 0x40000000u;  // ... the odd columns
constexpr uint32_t kUnitTile = 0x3FFFFFFFu;  // tiles per scan block of k_view_scan

// exclusive (interval, node) offsets of a tile
BT_DEV uint2 view_offset(const ViewBufs& vb, uint32_t tile) {
    const uint2 l = vb.local[tile], p = vb.blockPrefix[tile / kViewScanBlock];
    return make_uint2(l.x + p.x, l.y + p.y);
}

// ---------------------------------------------------------------- fetch

// Per-tile fetch state (TileFetchState, tracer.hpp:62-84), thread-local.
struct TileFetch {
    uint32_t actWord[kMaxOverlap];
    float actEntry[kMaxOverlap];
    float actExit[kMaxOverlap];
    uint32_t nAct, cursor;
    float zEnd;
};

BT_DEV void fetch_init(TileFetch& s) {
    s.nAct = 0;
    s.cursor = 0;
    s.zEnd = 0.0f;
}

// fetch_interval (tracer.cpp:50-103).  Returns false once the list is
// exhausted.  Same float bits as the CPU: compares, std::min/max semantics,
// view_z_from_ndc in exact IEEE ops.
BT_DEV bool fetch_next(TileFetch& s, const Frag* list, uint32_t cnt, const Cam& cam, const TraceParams& tp,
                       float& zBeginOut) {
    // 1. expire actives whose exit lies behind the previous interval end
    uint32_t n = s.nAct, m = 0;
    const float zEndPrev = s.zEnd;
    for (uint32_t i = 0; i < n; ++i) {
        if (!(s.actExit[i] <= zEndPrev)) {
            s.actWord[m] = s.actWord[i];
            s.actEntry[m] = s.actEntry[i];
            s.actExit[m] = s.actExit[i];
            ++m;
        }
    }
    const bool expired = m != n;
    n = m;
    uint32_t cursor = s.cursor;
    const bool hasNext = cursor < cnt;
    if (n == 0 && !hasNext) {
        s.nAct = 0;
        return false;
    }
    float zBegin = zEndPrev;
    if (hasNext) zBegin = smax(zEndPrev, __ldg(&list[cursor].zEntry));
    const float zBeginView = view_z_from_ndc(cam, zBegin);
    float maxExit = -f_inf();
    for (uint32_t i = 0; i < n; ++i) maxExit = smax(maxExit, s.actExit[i]);

    uint32_t fetched = 0;
    while (cursor < cnt) {
        const Frag* f = list + cursor;
        const float ce = __ldg(&f->zEntry);
        if (n != 0) {
            if (ce > maxExit) break;
            if (fetched >= tp.maxNew) break;
            if (n >= tp.maxOverlap) break;
            if (E::sub(view_z_from_ndc(cam, ce), zBeginView) >= tp.window) break;
        }
        const uint32_t cw = __ldg(&f->word);
        const float cx = __ldg(&f->zExit);
        // insert keeping ascending word order (lower_bound position)
        uint32_t pos = n;
        while (pos > 0 && s.actWord[pos - 1] >= cw) {
            s.actWord[pos] = s.actWord[pos - 1];
            s.actEntry[pos] = s.actEntry[pos - 1];
            s.actExit[pos] = s.actExit[pos - 1];
            --pos;
        }
        s.actWord[pos] = cw;
        s.actEntry[pos] = ce;
        s.actExit[pos] = cx;
        ++n;
        maxExit = smax(maxExit, cx);
        ++cursor;
        ++fetched;
    }
    float zEndNew = maxExit;
    if (cursor < cnt) zEndNew = smin(__ldg(&list[cursor].zEntry), maxExit);
    if (zEndNew <= zBegin && fetched == 0 && !expired) {
        float minExit = f_inf();
        for (uint32_t i = 0; i < n; ++i) minExit = smin(minExit, s.actExit[i]);
        zEndNew = minExit;
    }
    s.nAct = n;
    s.cursor = cursor;
    s.zEnd = zEndNew;
    zBeginOut = zBegin;
    return true;
}

// ---------------------------------------------------------------- view build

BT_DEV uint32_t tree_blob(const float4* words, uint32_t w) { return __float_as_uint(__ldg(&words[w].x)); }

struct ViewOut {
    uint2* nodes;        // this view's node slots
    uint32_t capacity;   // 2n - 1 (ViewOverflow beyond)
    uint32_t nView, nPrim, nBlocks, cacheFloats, depth, maxDepth, flops, err;
};

BT_DEV void view_append(ViewOut& v, uint32_t blob, uint32_t word, bool copyParams) {
    if (v.err) return;
    if (v.nView >= v.capacity) {
        v.err = kErrView;
        return;
    }
    const uint32_t floats = copyParams ? param_floats(blob) : 0u;
    if (floats > 0u && v.cacheFloats + floats <= kCacheFloats) v.cacheFloats += floats;
    v.nodes[v.nView] = make_uint2((blob & 0xFC000000u) | v.nBlocks, word);
    v.nBlocks += fast_block_size(blob);
    v.nView++;
    // evaluation stack depth and appendix-B flops of one evaluation
    if (blob_is_prim(blob)) {
        v.depth++;
        v.maxDepth = v.depth > v.maxDepth ? v.depth : v.maxDepth;
        v.flops += prim_flops(blob_op(blob));
    } else {
        v.depth--;
        v.flops += op_flops(blob_op(blob));
    }
}

// sparse_traverse<uint8_t, ViewBuildVisitor> (traversal.hpp:41-117,
// traversal.cpp:30-99) over the n active words (ascending), which sit in the
// .x of v.nodes[n - 1 + i]; the view is written over the same 2n - 1 slots
// (node m goes to slot m <= 2i + 1 < n - 1 + (i + 1) while active i + 1 is
// still unread).  Returns rootUsed.
BT_DEV uint32_t build_view_inplace(ViewOut& v, uint32_t n, const float4* words) {
    v.nView = v.nPrim = v.nBlocks = v.cacheFloats = v.depth = v.maxDepth = v.err = 0;
    v.flops = 12u;
    if (n == 0) return 0u;
    v.capacity = 2u * n - 1u;
    const uint2* act2 = v.nodes + (n - 1u);
    uint32_t sBlob[kStackCap];
    uint8_t sUse[kStackCap];
    uint32_t sp = 0;
    for (uint32_t i = 0; i < n && !v.err; ++i) {
        const uint32_t w = act2[i].x;
        uint32_t nodeBlob = tree_blob(words, w);
        view_append(v, nodeBlob, w, true);  // visitor.primitive
        v.nPrim++;
        uint32_t data = 1u;
        if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), blob_anc(sBlob[sp - 1])));
        const uint32_t nextAct = (i + 1 < n) ? act2[i + 1].x : 0u;
        for (;;) {
            const uint32_t anc = blob_anc(nodeBlob);
            const bool shadowed = (i + 1 < n) && anc > nextAct;
            const bool lastDone = (i + 1 == n) && (sp == 0 && anc == kSentinel);
            if (shadowed || lastDone) break;
            if (anc == kSentinel) {  // "traversal walked past the root"
                v.err = kErrLogic;
                return 0u;
            }
            const uint32_t opWord = anc;
            const bool fromLeft = blob_is_left(nodeBlob);
            nodeBlob = tree_blob(words, opWord);
            bool combined = false;
            if (sp > 0) {
                const uint32_t cb = sBlob[sp - 1];
                const uint32_t ca = blob_anc(cb), na = blob_anc(nodeBlob);
                const bool pop = (opWord == ca) || (na >= ca && (na == kSentinel || blob_is_left(nodeBlob)));
                if (pop) {
                    // visitor.combine(left = stacked, right = current)
                    const uint32_t children = ((uint32_t)sUse[sp - 1] << 1) | data;
                    const uint32_t opType = ((~children & blob_ignore(nodeBlob)) & 3u) == 0u ? children : 0u;
                    uint32_t stored = nodeBlob;
                    if (opType != 3u) stored = blob_with_op(stored, opType);
                    view_append(v, stored, opWord, opType == 3u);
                    data = opType != 0u ? 1u : 0u;
                    --sp;
                    combined = true;
                }
            }
            if (!combined) {
                // visitor.pass: selector nodes only gate the usage bit
                const uint32_t mask = fromLeft ? 1u : 2u;
                if (blob_ignore(nodeBlob) & mask) data = 0u;
            }
            if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), blob_anc(sBlob[sp - 1])));
        }
        if (v.err) return 0u;
        if (sp >= kStackCap) {
            v.err = kErrStack;
            return 0u;
        }
        sBlob[sp] = nodeBlob;
        sUse[sp] = (uint8_t)data;
        ++sp;
    }
    if (v.err) return 0u;
    const uint32_t result = sUse[sp - 1];
    --sp;
    if (sp != 0) {
        v.err = kErrLogic;
        return 0u;
    }
    return result;
}

}  // namespace btk
