// bt_tile.cuh -- per-tile machinery of stage (c), device side.
//
//  * FetchState / fetch_interval  : the subfrustum fetch heuristic
//                                   (reference src/tracer.cpp:50-103)
//  * build_view                   : Algorithm 1 sparse bottom-up traversal
//                                   with the view-building visitor
//                                   (include/blobtree/traversal.hpp:41-117,
//                                   src/traversal.cpp:30-99)
//  * eval_view                    : Algorithm 3 stack evaluation of the view
//                                   (src/traversal.cpp:101-124), NR points at
//                                   once for instruction-level parallelism
//  * March                        : the over-relaxed sphere trace of
//                                   include/blobtree/tracer.hpp:99-177
//                                   restated as a state machine that needs
//                                   exactly one field value per step, so the
//                                   64 rays of a tile evaluate in lockstep.
//
// A warp owns one 8x8 tile: lane l carries pixels l and l+32.  The serial
// parts (fetch and view build) run on lane 0 against per-warp shared memory
// and are published with __syncwarp.
#pragma once

#include "bt_geom.cuh"

namespace btk {

// float4 units of a view node's precomputed parameter block (tolerance
// path, see bt_fast.cuh): affine rows for rotated primitives, reciprocals,
// operator constants.
BT_HD uint32_t fast_block_size(uint32_t blob) {
    if (blob_is_prim(blob)) {
        const uint32_t k = blob_op(blob);
        return k == 0u ? 1u : k == 1u ? 5u : k == 2u ? 4u : k == 3u ? 4u : k == 4u ? 5u : 6u;
    }
    const uint32_t c = blob_op(blob);
    return (c >= 6u && c <= 8u) ? 1u : (c >= 9u && c <= 11u) ? 2u : 0u;
}

// Tile error codes (tileError is 1 for either, like the reference's catch).
constexpr uint32_t kErrStack = 1;
constexpr uint32_t kErrView = 2;
constexpr uint32_t kErrLogic = 3;

constexpr int kFragStage = 128;  // fragments of a tile list staged in shared memory
constexpr int kViewCap = 2 * kMaxOverlap - 1;
constexpr uint32_t kFastBlockCap = kViewCap * 6;  // float4s per warp

struct TraceParams {
    float L, invL, relax, minStep, hitEps;
    uint32_t maxOverlap, maxNew;
    float window;  // resolved fetch window in view-z units
};

struct Frag {
    uint32_t word;
    float zEntry, zExit;
};

struct WarpSmem {
    // fetch state
    uint32_t actWord[kMaxOverlap];
    float actEntry[kMaxOverlap];
    float actExit[kMaxOverlap];
    Frag stage[kFragStage];
    // pruned view: blob (op possibly rewritten) and the source word of params
    uint32_t vBlob[kViewCap];
    uint32_t vWord[kViewCap];
    uint32_t vHdr[kViewCap];  // fast path: isPrim(1) op(5) | float4 offset of the parameter block
    // view-build traversal stack
    uint32_t sBlob[kStackCap];
    uint8_t sUse[kStackCap];
    // published scalars
    uint32_t nAct, cursor, nView, nPrim, rootUsed, maxDepth, flops, cacheFloats, err, done, vEnd;
    float zBegin, zEnd;
};

// --------------------------------------------------------------------------
// fetch_interval (tracer.cpp:50-103), lane 0 only.  Returns false when the
// tile list is exhausted.  All comparisons are on the same float bits as the
// CPU; view_z_from_ndc uses exact IEEE ops.

BT_DEV const Frag& frag_at(const WarpSmem& s, const Frag* list, uint32_t i) {
    return i < (uint32_t)kFragStage ? s.stage[i] : list[i];
}

BT_DEV bool fetch_interval(WarpSmem& s, const Frag* list, uint32_t cnt, const Cam& cam,
                           const TraceParams& tp, uint32_t& fetchedOut) {
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
    if (hasNext) zBegin = smax(zEndPrev, frag_at(s, list, cursor).zEntry);
    const float zBeginView = view_z_from_ndc(cam, zBegin);
    float maxExit = -f_inf();
    for (uint32_t i = 0; i < n; ++i) maxExit = smax(maxExit, s.actExit[i]);

    uint32_t fetched = 0;
    while (cursor < cnt) {
        Frag c = frag_at(s, list, cursor);
        if (n != 0) {
            if (c.zEntry > maxExit) break;
            if (fetched >= tp.maxNew) break;
            if (n >= tp.maxOverlap) break;
            if (E::sub(view_z_from_ndc(cam, c.zEntry), zBeginView) >= tp.window) break;
        }
        // insert keeping ascending word order (lower_bound position)
        uint32_t pos = n;
        while (pos > 0 && s.actWord[pos - 1] >= c.word) {
            s.actWord[pos] = s.actWord[pos - 1];
            s.actEntry[pos] = s.actEntry[pos - 1];
            s.actExit[pos] = s.actExit[pos - 1];
            --pos;
        }
        s.actWord[pos] = c.word;
        s.actEntry[pos] = c.zEntry;
        s.actExit[pos] = c.zExit;
        ++n;
        maxExit = smax(maxExit, c.zExit);
        ++cursor;
        ++fetched;
    }
    float zEndNew = maxExit;
    if (cursor < cnt) zEndNew = smin(frag_at(s, list, cursor).zEntry, maxExit);
    if (zEndNew <= zBegin && fetched == 0 && !expired) {
        float minExit = f_inf();
        for (uint32_t i = 0; i < n; ++i) minExit = smin(minExit, s.actExit[i]);
        zEndNew = minExit;
    }
    s.nAct = n;
    s.cursor = cursor;
    s.zBegin = zBegin;
    s.zEnd = zEndNew;
    fetchedOut = fetched;
    return true;
}

// --------------------------------------------------------------------------
// Pruned view build: sparse_traverse<uint8_t, ViewBuildVisitor>, lane 0 only.
// Records per view node the (possibly rewritten) blob and the source word
// of its parameters; reproduces the reference's parameter-cache accounting
// (tileCacheBytes) and its failure modes (stack > 22 -> TraversalOverflow,
// > 2n-1 nodes -> ViewOverflow).  Also derives the evaluation stack depth and
// the appendix-B flop weight of one evaluation of the view.

BT_DEV uint32_t tree_blob(const float4* words, uint32_t w) { return __float_as_uint(__ldg(&words[w].x)); }

BT_DEV void view_append(WarpSmem& s, uint32_t blob, uint32_t word, bool copyParams,
                        uint32_t capacity) {
    if (s.err) return;
    if (s.nView >= capacity) {
        s.err = kErrView;
        return;
    }
    uint32_t floats = copyParams ? param_floats(blob) : 0u;
    if (floats > 0u && s.cacheFloats + floats <= kCacheFloats) s.cacheFloats += floats;
    s.vBlob[s.nView] = blob;
    s.vWord[s.nView] = word;
    s.vHdr[s.nView] = (blob & 0xFC000000u) | s.vEnd;
    s.vEnd += fast_block_size(blob);
    s.nView++;
}

BT_DEV void build_view(WarpSmem& s, const float4* words) {
    const uint32_t n = s.nAct;
    s.nView = 0;
    s.nPrim = 0;
    s.vEnd = 0;
    s.cacheFloats = 0;
    s.rootUsed = 0;
    s.maxDepth = 0;
    s.flops = 12u;
    if (n == 0) return;
    const uint32_t capacity = 2u * n - 1u;
    uint32_t sp = 0;
    for (uint32_t i = 0; i < n && !s.err; ++i) {
        const uint32_t w = s.actWord[i];
        uint32_t nodeBlob = tree_blob(words, w);
        // visitor.primitive
        view_append(s, nodeBlob, w, true, capacity);
        s.nPrim++;
        uint32_t data = 1u;
        if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), blob_anc(s.sBlob[sp - 1])));
        for (;;) {
            const uint32_t anc = blob_anc(nodeBlob);
            const bool shadowed = (i + 1 < n) && anc > s.actWord[i + 1];
            const bool lastDone = (i + 1 == n) && (sp == 0 && anc == kSentinel);
            if (shadowed || lastDone) break;
            if (anc == kSentinel) {  // "traversal walked past the root"
                s.err = kErrLogic;
                return;
            }
            const uint32_t opWord = anc;
            const bool fromLeft = blob_is_left(nodeBlob);
            nodeBlob = tree_blob(words, opWord);
            bool combined = false;
            if (sp > 0) {
                const uint32_t cb = s.sBlob[sp - 1];
                const uint32_t ca = blob_anc(cb), na = blob_anc(nodeBlob);
                const bool pop = (opWord == ca) || (na >= ca && (na == kSentinel || blob_is_left(nodeBlob)));
                if (pop) {
                    // visitor.combine(left = stacked, right = current)
                    const uint32_t children = ((uint32_t)s.sUse[sp - 1] << 1) | data;
                    const uint32_t opType = ((~children & blob_ignore(nodeBlob)) & 3u) == 0u ? children : 0u;
                    uint32_t stored = nodeBlob;
                    if (opType != 3u) stored = blob_with_op(stored, opType);
                    view_append(s, stored, opWord, opType == 3u, capacity);
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
            if (sp > 0) nodeBlob = blob_with_anc(nodeBlob, min(blob_anc(nodeBlob), blob_anc(s.sBlob[sp - 1])));
        }
        if (s.err) return;
        if (sp >= kStackCap) {
            s.err = kErrStack;
            return;
        }
        s.sBlob[sp] = nodeBlob;
        s.sUse[sp] = (uint8_t)data;
        ++sp;
    }
    if (s.err) return;
    const uint32_t result = s.sUse[sp - 1];
    --sp;
    if (sp != 0) {
        s.err = kErrLogic;
        return;
    }
    s.rootUsed = result;
    // evaluation stack depth and per-evaluation algorithmic flops
    uint32_t depth = 0, maxd = 0, fl = 12u;
    for (uint32_t i = 0; i < s.nView; ++i) {
        const uint32_t b = s.vBlob[i];
        if (blob_is_prim(b)) {
            ++depth;
            fl += prim_flops(blob_op(b));
        } else {
            --depth;
            fl += op_flops(blob_op(b));
        }
        maxd = depth > maxd ? depth : maxd;
    }
    s.maxDepth = maxd;
    s.flops = fl;
}

// --------------------------------------------------------------------------
// View evaluation.  Parameters are read straight from the tree words (L1
// resident, warp-uniform address -> broadcast).  The evaluation stack is a
// per-lane local array indexed by a warp-uniform stack pointer.

template <int N> struct ParamBlock {
    float v[4 * N];
};

template <int N> BT_DEV void load_params(float* dst, const float4* src) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float4 q = __ldg(&src[i]);
        dst[4 * i + 0] = q.x;
        dst[4 * i + 1] = q.y;
        dst[4 * i + 2] = q.z;
        dst[4 * i + 3] = q.w;
    }
}

// One field value of the view at p (Algorithm 3): primitives push, operators
// pop two and push one; the per-node parameter block is loaded as float4s.
template <class O>
BT_DEV float eval_view(const WarpSmem& s, const float4* words, F3 p) {
    float stk[kStackCap];
    uint32_t sp = 0;
    const uint32_t n = s.nView;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t b = s.vBlob[i];
        const float4* P4 = words + s.vWord[i] + 1;
        const uint32_t code = blob_op(b);
        if (blob_is_prim(b)) {
            float P[20];
            load_params<5>(P, P4);
            stk[sp++] = eval_primitive<O>(code, P, p);
        } else {
            float kd[2] = {0.0f, 0.0f};
            if (code >= 6u) {
                const float4 q = __ldg(P4);
                kd[0] = q.x;
                kd[1] = q.y;
            }
            const float right = stk[sp - 1], left = stk[sp - 2];
            stk[sp - 2] = eval_operator<O>(code, kd, left, right);
            --sp;
        }
    }
    return stk[0];
}

// --------------------------------------------------------------------------
// Sphere-trace state machine (tracer.hpp:99-177).  phase: 0 finished,
// 1 needs f(t0), 2 needs f(tn) (main step), 3 needs f(tb) (unrelaxed
// back-off after an overshoot).  March arithmetic is always exact.

// Compact march state: 6 floats + 2 words per ray (register pressure is
// what limits the trace kernel's occupancy).  `st` packs the phase and the
// flags; on completion `t` holds the hit position.  r = f / L is recomputed
// where the reference reuses it (f is unchanged in between, same bits).
constexpr uint32_t kPhaseMask = 3u;  // 0 done, 1 needs f(t0), 2 needs f(tn), 3 needs f(tb)
constexpr uint32_t kRelax = 4u, kSaved = 8u, kHitFlag = 16u, kSlot1 = 32u;

struct March {
    float t, f, t1, savedT, savedF, evalT;
    uint32_t st, evals;
};

BT_DEV uint32_t march_phase(const March& m) { return m.st & kPhaseMask; }
BT_DEV bool march_hit(const March& m) { return (m.st & kHitFlag) != 0u; }

BT_DEV void march_finish(March& m, bool hit, float t) {
    m.st = (m.st & kSlot1) | (hit ? kHitFlag : 0u);
    m.t = t;
}

BT_DEV void march_set_phase(March& m, uint32_t ph) { m.st = (m.st & ~kPhaseMask) | ph; }

// Advance without evaluating until a field value is needed (reference loop
// head, tracer.hpp:115-139: step, saved-sphere reuse, clamp to t1).  The
// common case is straight-line select code; reusing a saved sample is the
// rare case and loops.
BT_DEV void march_advance(March& m, const TraceParams& tp) {
    for (;;) {
        const float r = E::mul(m.f, tp.invL);
        float tn = E::add(m.t, smax((m.st & kRelax) ? E::mul(tp.relax, r) : r, tp.minStep));
        if (!is_finite(r)) {
            march_finish(m, false, 0.0f);
            return;
        }
        if ((m.st & kSaved) && tn >= m.savedT) {  // rare: reaching the remembered sphere
            const bool reuse = m.savedT >= E::add(m.t, tp.minStep) && m.savedT <= m.t1;
            m.st = (m.st & ~kSaved) | kRelax;
            if (reuse) {
                // reused sample: never an overshoot, never beyond t1
                const float fn = m.savedF;
                tn = m.savedT;
                if (fn <= tp.hitEps) {
                    march_finish(m, true, tn);
                    return;
                }
                if (tn >= m.t1) {
                    march_finish(m, false, 0.0f);
                    return;
                }
                m.t = tn;
                m.f = fn;
                continue;
            }
        }
        const bool beyond = tn > m.t1;
        if (beyond && m.t >= m.t1) {
            march_finish(m, false, 0.0f);
            return;
        }
        m.evalT = beyond ? m.t1 : tn;
        march_set_phase(m, 2u);
        return;
    }
}

BT_DEV void march_idle(March& m, uint32_t slot) {
    m.st = slot ? kSlot1 : 0u;
    m.evals = 0;
    m.t = 0.0f;
}

BT_DEV void march_begin(March& m, float t0, float t1, uint32_t slot) {
    m.evals = 0;
    m.st = (slot ? kSlot1 : 0u) | kRelax;
    m.t1 = t1;
    if (t0 > t1) {
        march_finish(m, false, 0.0f);
        return;
    }
    m.t = t0;
    m.evalT = t0;
    march_set_phase(m, 1u);
}

// One field value consumed (tracer.hpp:115-175).  In every non-overshoot
// case the march moves to the sample (evalT, v): hit if v <= eps, miss if a
// main step reached t1, else advance.  Only the overshoot back-off branches.
BT_DEV void march_consume(March& m, float v, const TraceParams& tp) {
    m.evals++;
    const bool step = march_phase(m) == 2u;
    const float tn = m.evalT;
    const bool overshoot = step && (m.st & kRelax) &&
                           (E::mul(E::sub(tn, m.t), tp.L) >= E::add(m.f, fabsf(v)) || v < -tp.hitEps);
    if (!overshoot) {
        const bool hit = v <= tp.hitEps;
        const bool end = step && tn >= m.t1;
        m.t = tn;
        m.f = v;
        if (hit) march_finish(m, true, tn);
        else if (end) march_finish(m, false, 0.0f);
        else march_advance(m, tp);
        return;
    }
    // remember the non-overlapping sphere, back off to the safe one
    m.savedT = tn;
    m.savedF = v;
    m.st = (m.st & ~kRelax) | kSaved;
    const float tb = E::add(m.t, smax(E::mul(m.f, tp.invL), tp.minStep));
    if (tb >= m.savedT) {
        m.t = m.savedT;
        m.f = m.savedF;
        m.st = (m.st & ~kSaved) | kRelax;
        if (m.f <= tp.hitEps) march_finish(m, true, m.t);
        else march_advance(m, tp);
    } else if (tb > m.t1) {
        march_finish(m, false, 0.0f);
    } else {
        m.evalT = tb;
        march_set_phase(m, 3u);
    }
}

}  // namespace btk
