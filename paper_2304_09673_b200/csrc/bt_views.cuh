// bt_views.cuh -- stage (c), part 1: the interval sequence and the pruned
// views of every tile, compiled ahead of the march.
//
// The reference interleaves, per tile, a serial fetch_interval + view build
// (tracer.cpp:50-103, traversal.cpp:30-99) with the 64-ray march of each
// interval (tracer.cpp:155-232).  Neither the intervals nor the views depend
// on the march -- the march only decides how far down the list a tile goes
// (it stops once all 64 rays have hit).  So they are compiled ahead of the
// march (k_views.cu): a warp per tile replays the fetch sequence with the
// O(n) steps spread over its lanes, a thread per interval builds the view,
// and the march kernel reads the records:
//
//   IntervalRec (32 B)  zBegin/zEnd (NDC), the view's node range, overlap,
//                       cache bytes, flags, appendix-B flops, fast-block size
//   ViewNode    (8 B)   hdr = isPrim(1) op(5, possibly a reserved code) |
//                       byte offset (bits 0-15) of the node's fast parameter block;
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
    uint32_t* counters = nullptr;  // [1] overflow flag (see below)
    uint32_t* slab = nullptr;      // [tiles * slab stride] count-pass intervals (k_views.cu)
    const uint32_t* order = nullptr;  // optional march units in order (tile | kUnitSplit | kUnitPart1), else raster
    const uint32_t* unitCount = nullptr;  // number of entries of `order` (device)
    uint32_t* tileCost = nullptr;     // [tiles] march cost proxy 0..255 (k_tile; scheduling)
    uint2* base = nullptr;            // [tiles] (first interval record, first view node) of the tile
    uint64_t ivCap = 0, nodeCap = 0;
};
// vb.counters: [1] overflow flag, [2] interval records allocated, [3] view nodes allocated

constexpr uint32_t kViewScanBlock = 4096;
constexpr uint32_t kUnitSplit = 0x80000000u;  // march unit = half a tile (one pixel-column parity)
constexpr uint32_t kUnitPart1 = 0x40000000u;  // ... the odd columns
constexpr uint32_t kUnitTile = 0x3FFFFFFFu;  // tiles per scan block of k_view_scan

// (interval, node) offsets of a tile's records (bump-allocated by k_tile)
BT_DEV uint2 view_offset(const ViewBufs& vb, uint32_t tile) { return vb.base[tile]; }

// ---------------------------------------------------------------- warp fetch
// fetch_interval (tracer.cpp:50-103; TileFetchState, tracer.hpp:62-84),
// executed by a WARP on one tile: the active set
// (<= 96 entries, sorted by word) is spread over the lanes (slot k of lane l
// is active l + 32k), the tile's fragment list is staged in shared memory,
// and every O(n) step of the serial loop becomes a ballot / shuffle step:
//   expire   ballot + popc compaction
//   maxExit  butterfly max
//   fetch    candidates cursor..cursor+31 tested in parallel against the
//            prefix max of the exits before them (the loop's running maxExit);
//            the fetched count is the first failing candidate
//   insert   rank merge (words are unique within a tile's list)
// Bit-identical to the serial loop: same compares, same IEEE
// view_z_from_ndc, and max/min reductions over finite values.

constexpr uint32_t kWarpFragStage = 128;  // fragments of a tile list staged per warp

struct WarpFetchSmem {
    uint32_t fW[kWarpFragStage];
    float fEn[kWarpFragStage], fEx[kWarpFragStage];
    uint32_t tW[kMaxOverlap];  // compaction / merge staging
    float tEn[kMaxOverlap], tEx[kMaxOverlap];
};

struct WarpFetch {
    uint32_t aW[3];
    float aEn[3], aEx[3];
    uint32_t n, cursor, cnt, lane;
    float zEnd;
    const Frag* list;
    WarpFetchSmem* sm;

    BT_DEV void frag(uint32_t i, uint32_t& w, float& en, float& ex) const {
        if (i < kWarpFragStage) {
            w = sm->fW[i];
            en = sm->fEn[i];
            ex = sm->fEx[i];
        } else {
            w = __ldg(&list[i].word);
            en = __ldg(&list[i].zEntry);
            ex = __ldg(&list[i].zExit);
        }
    }
    BT_DEV float entry_at(uint32_t i) const { return i < kWarpFragStage ? sm->fEn[i] : __ldg(&list[i].zEntry); }

    BT_DEV void init(const Frag* l, uint32_t count, WarpFetchSmem* smem, uint32_t ln) {
        list = l;
        cnt = count;
        sm = smem;
        lane = ln;
        n = 0;
        cursor = 0;
        zEnd = 0.0f;
        for (uint32_t i = lane; i < count && i < kWarpFragStage; i += 32) {
            sm->fW[i] = __ldg(&l[i].word);
            sm->fEn[i] = __ldg(&l[i].zEntry);
            sm->fEx[i] = __ldg(&l[i].zExit);
        }
        __syncwarp();
    }

    // registers <- staging rows [0, m)
    BT_DEV void reload(uint32_t m) {
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t i = lane + 32u * k;
            if (i < m) {
                aW[k] = sm->tW[i];
                aEn[k] = sm->tEn[i];
                aEx[k] = sm->tEx[i];
            }
        }
        __syncwarp();
    }

    // Sorted = false keeps the actives in fetch order instead of word order:
    // the interval bounds and the active counts are the same (they depend
    // only on the set), which is all the count pass needs.
    template <bool Sorted>
    BT_DEV bool next(const Cam& cam, const TraceParams& tp, float& zBeginOut) {
        constexpr uint32_t kFullMask = 0xFFFFFFFFu;
        const uint32_t lt = (1u << lane) - 1u;
        // 1. expire actives whose exit lies behind the previous interval end
        const float zEndPrev = zEnd;
        uint32_t keep[3], m = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t i = lane + 32u * k;
            keep[k] = __ballot_sync(kFullMask, i < n && !(aEx[k] <= zEndPrev));
            m += __popc(keep[k]);
        }
        const bool expired = m != n;
        if (expired) {
            uint32_t before = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if ((keep[k] >> lane) & 1u) {
                    const uint32_t pos = before + __popc(keep[k] & lt);
                    sm->tW[pos] = aW[k];
                    sm->tEn[pos] = aEn[k];
                    sm->tEx[pos] = aEx[k];
                }
                before += __popc(keep[k]);
            }
            reload(m);
        }
        n = m;
        const bool hasNext = cursor < cnt;
        if (n == 0 && !hasNext) return false;
        float zBegin = zEndPrev;
        if (hasNext) zBegin = smax(zEndPrev, entry_at(cursor));
        const float zBeginView = view_z_from_ndc(cam, zBegin);
        float maxExit = -f_inf();
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (lane + 32u * k < n) maxExit = fmaxf(maxExit, aEx[k]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxExit = fmaxf(maxExit, __shfl_xor_sync(kFullMask, maxExit, o));

        // 2. fetch, 32 candidates at a time
        uint32_t fetchedTotal = 0;
        for (;;) {
            const uint32_t avail = cnt - cursor;
            const uint32_t K = avail < 32u ? avail : 32u;
            uint32_t cw = 0;
            float ce = 0.0f, cx = -f_inf();
            bool ok = false;
            float inclMax = -f_inf();
            if (lane < K) frag(cursor + lane, cw, ce, cx);
            // exclusive prefix max of the candidates' exits
            inclMax = lane < K ? cx : -f_inf();
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float v = __shfl_up_sync(kFullMask, inclMax, o);
                if (lane >= (uint32_t)o) inclMax = fmaxf(inclMax, v);
            }
            float exclMax = __shfl_up_sync(kFullMask, inclMax, 1);
            if (lane == 0) exclMax = -f_inf();
            if (lane < K) {
                const uint32_t nj = n + lane, fj = fetchedTotal + lane;
                const float mx = fmaxf(maxExit, exclMax);
                ok = nj == 0u || !(ce > mx || fj >= tp.maxNew || nj >= tp.maxOverlap ||
                                   E::sub(view_z_from_ndc(cam, ce), zBeginView) >= tp.window);
            }
            const uint32_t okMask = __ballot_sync(kFullMask, ok);
            const uint32_t fetched = (~okMask) ? (uint32_t)(__ffs(~okMask) - 1) : 32u;  // leading ok lanes
            if (fetched == 0u) break;
            if (!Sorted) {  // append in fetch order
                __syncwarp();
                if (lane < fetched) {
                    sm->tW[n + lane] = cw;
                    sm->tEn[n + lane] = ce;
                    sm->tEx[n + lane] = cx;
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const uint32_t i = lane + 32u * k;
                    if (i < n) {
                        sm->tW[i] = aW[k];
                        sm->tEn[i] = aEn[k];
                        sm->tEx[i] = aEx[k];
                    }
                }
                maxExit = fmaxf(maxExit, __shfl_sync(kFullMask, inclMax, fetched - 1u));
                n += fetched;
                cursor += fetched;
                fetchedTotal += fetched;
                reload(n);
                if (fetched < 32u || cursor >= cnt) break;
                continue;
            }
            // 3. merge the fetched candidates into the word-sorted active set
            uint32_t rankOld[3] = {0u, 0u, 0u}, rankNew = 0u;
            for (uint32_t j = 0; j < fetched; ++j) {
                const uint32_t wj = __shfl_sync(kFullMask, cw, j);
                uint32_t below = 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const bool valid = lane + 32u * k < n;
                    if (valid && aW[k] > wj) rankOld[k]++;
                    below += __popc(__ballot_sync(kFullMask, valid && aW[k] < wj));
                }
                if (lane == j) rankNew += below;
                if (lane < fetched && wj < cw) rankNew++;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t i = lane + 32u * k;
                if (i < n) {
                    const uint32_t pos = i + rankOld[k];
                    sm->tW[pos] = aW[k];
                    sm->tEn[pos] = aEn[k];
                    sm->tEx[pos] = aEx[k];
                }
            }
            if (lane < fetched) {
                sm->tW[rankNew] = cw;
                sm->tEn[rankNew] = ce;
                sm->tEx[rankNew] = cx;
            }
            maxExit = fmaxf(maxExit, __shfl_sync(kFullMask, inclMax, fetched - 1u));
            n += fetched;
            cursor += fetched;
            fetchedTotal += fetched;
            reload(n);
            if (fetched < 32u || cursor >= cnt) break;
        }
        // 4. interval end
        float zEndNew = maxExit;
        if (cursor < cnt) zEndNew = smin(entry_at(cursor), maxExit);
        if (zEndNew <= zBegin && fetchedTotal == 0u && !expired) {
            float minExit = f_inf();
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (lane + 32u * k < n) minExit = fminf(minExit, aEx[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) minExit = fminf(minExit, __shfl_xor_sync(kFullMask, minExit, o));
            zEndNew = minExit;
        }
        zEnd = zEndNew;
        zBeginOut = zBegin;
        return true;
    }
};

// ---------------------------------------------------------------- view build

BT_DEV uint32_t tree_blob(const uint32_t* blobs, uint32_t w) { return __ldg(&blobs[w]); }

// Per-node constants of a view entry, as packed-field lookups (a dynamically
// indexed table would land in local memory):
//   floats  parameters copied into the reference's cache (param_float_count,
//           traversal.cpp:24-28): 7 transform floats + the shape's (sphere 1,
//           ellipsoid 3, torus 2, box 3, sphere-cone 3, quadric 10); 2 for
//           smooth / compact operators (field.hpp:106-116), 0 otherwise;
//   blocks  float4s of the node's fast parameter block (convert_node,
//           bt_fast.cuh): sphere 1, ellipsoid 5, torus 4, box 4, sphere-cone 5,
//           quadric 6; smooth 1, compact 2;
//   flops   SURVEY.md appendix-B weights: sphere 40, ellipsoid 57, torus 43,
//           box 43, sphere-cone 52, quadric 85; smooth 8, compact 22.
BT_HD void view_node_info(uint32_t blob, uint32_t& floats, uint32_t& blocks, uint32_t& flops) {
    const uint32_t op = blob_op(blob);
    if (blob_is_prim(blob)) {
        floats = 7u + (op < 6u ? (0xA33231u >> (4u * op)) & 15u : 3u);  // shape floats 1 3 2 3 3 10
        blocks = op < 5u ? (0x54451u >> (4u * op)) & 15u : 6u;           // 1 5 4 4 5, quadric 6
        flops = op < 6u ? (uint32_t)((0x55342B2B3928ull >> (8u * op)) & 0xFFu) : 0u;  // 40 57 43 43 52 85
    } else {
        const bool smooth = op - 6u < 3u, compact = op - 9u < 3u;
        floats = (smooth || compact) ? 2u : 0u;
        blocks = smooth ? 1u : compact ? 2u : 0u;
        flops = smooth ? 8u : compact ? 22u : 0u;
    }
}

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
    uint32_t floats, blocks, flops;
    view_node_info(blob, floats, blocks, flops);
    if (!copyParams) floats = 0u;
    if (floats > 0u && v.cacheFloats + floats <= kCacheFloats) v.cacheFloats += floats;
    v.nodes[v.nView] = make_uint2((blob & 0xFC000000u) | (v.nBlocks << 4), word);  // byte offset of the block
    v.nBlocks += blocks;
    v.nView++;
    v.flops += flops;  // appendix-B flops of one evaluation
    // evaluation stack depth
    if (blob_is_prim(blob)) {
        v.depth++;
        v.maxDepth = v.depth > v.maxDepth ? v.depth : v.maxDepth;
    } else {
        v.depth--;
    }
}

// sparse_traverse<uint8_t, ViewBuildVisitor> (traversal.hpp:41-117,
// traversal.cpp:30-99) over the n active words (ascending), which sit in the
// .x of v.nodes[n - 1 + i]; the view is written over the same 2n - 1 slots
// (node m goes to slot m <= 2i + 1 < n - 1 + (i + 1) while active i + 1 is
// still unread).
//
// Restated as a state machine that advances ONE node dereference per call
// (one loop, not the reference's nested primitive / walk loops), with the
// next primitive's word and blob read one primitive ahead, off the walk's
// pointer-chasing chain.  The traversal stack lives in shared memory, one u32
// per entry: a stacked node is only ever consulted for its ancestor
// (pop_required, the min() of traversal.hpp:92,110) and its usage bit, so
// entry = ancestor | usage << 31.  Errors end the view at once: the reference
// throws, and every later step of the loop would leave the record unchanged
// (view_append is a no-op once err is set).
struct ViewBuild {
    ViewOut v;
    const uint2* act2;
    uint32_t n, i, sp, nodeBlob, data, nextAct;
    uint32_t w0, b0, w1;  // read ahead: the next primitive's word and blob, and the word after it
    bool start;      // the next step begins active primitive i
    bool done;
    uint32_t rootUsed;

    BT_DEV void begin(uint2* nodes, uint32_t count, const uint32_t* blobs) {
        v.nodes = nodes;
        v.nView = v.nPrim = v.nBlocks = v.cacheFloats = v.depth = v.maxDepth = v.err = 0;
        v.flops = 12u;
        v.capacity = count ? 2u * count - 1u : 0u;
        n = count;
        act2 = nodes + (count ? count - 1u : 0u);
        i = sp = 0;
        nodeBlob = data = 0;
        nextAct = 0u;
        w0 = count ? act2[0].x : 0u;
        b0 = count ? tree_blob(blobs, w0) : 0u;
        w1 = count > 1u ? act2[1].x : 0u;
        start = true;
        rootUsed = 0;
        done = count == 0u;
    }
    BT_DEV void fail(uint32_t e) {
        if (!v.err) v.err = e;
        rootUsed = 0;
        done = true;
    }
    // stk[k * stride]: entry k of this thread's stack
    BT_DEV void step(const uint32_t* blobs, uint32_t* stk, uint32_t stride) {
        if (start) {  // visitor.primitive: active i (w0, b0) and i + 1 (w1) were read ahead
            const uint32_t w = w0;
            nodeBlob = b0;
            view_append(v, nodeBlob, w, true);
            v.nPrim++;
            data = 1u;
            if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), stk[(sp - 1) * stride] & kSentinel));
            nextAct = (i + 1 < n) ? w1 : 0u;
            // read ahead, off the walk's dependency chain: active i + 1's blob, active i + 2's word
            // (slot n + 1 + i: only slots <= 2i have been written so far)
            if (i + 1 < n) {
                w0 = w1;
                b0 = tree_blob(blobs, w1);
            }
            if (i + 2 < n) w1 = act2[i + 2].x;
            start = false;
        }
        if (v.err) return fail(v.err);
        const uint32_t anc = blob_anc(nodeBlob);
        const bool shadowed = (i + 1 < n) && anc > nextAct;
        const bool lastDone = (i + 1 == n) && (sp == 0 && anc == kSentinel);
        if (shadowed || lastDone) {  // the walk of primitive i ends: push
            if (sp >= kStackCap) return fail(kErrStack);
            stk[sp * stride] = anc | (data << 31);
            ++sp;
            if (++i < n) {
                start = true;
                return;
            }
            const uint32_t result = stk[(sp - 1) * stride] >> 31;
            if (--sp != 0) return fail(kErrLogic);  // "traversal left values on the stack"
            rootUsed = result;
            done = true;
            return;
        }
        if (anc == kSentinel) return fail(kErrLogic);  // "traversal walked past the root"
        const uint32_t opWord = anc;
        const bool fromLeft = blob_is_left(nodeBlob);
        nodeBlob = tree_blob(blobs, opWord);
        bool combined = false;
        if (sp > 0) {
            const uint32_t top = stk[(sp - 1) * stride];
            const uint32_t ca = top & kSentinel, na = blob_anc(nodeBlob);
            const bool pop = (opWord == ca) || (na >= ca && (na == kSentinel || blob_is_left(nodeBlob)));
            if (pop) {
                // visitor.combine(left = stacked, right = current)
                const uint32_t children = ((top >> 31) << 1) | data;
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
        if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), stk[(sp - 1) * stride] & kSentinel));
        if (v.err) fail(v.err);
    }
};

}  // namespace btk
