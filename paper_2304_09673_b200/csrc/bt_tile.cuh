// bt_tile.cuh -- per-tile machinery of stage (c), device side.
//
//  * TraceParams, Frag            : render constants, A-buffer fragment
//  * eval_staged                  : Algorithm 3 stack evaluation of a pruned
//                                   view staged in shared memory (exact path,
//                                   raw parameters; src/traversal.cpp:101-124)
//  * March                        : the over-relaxed sphere trace of
//                                   include/blobtree/tracer.hpp:99-177
//                                   restated as a state machine that needs
//                                   exactly one field value per step, so the
//                                   rays of a tile evaluate in lockstep.
//
// The interval sequence and the views themselves are compiled ahead of the
// march, one thread per tile (bt_views.cuh, k_views.cu).
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

constexpr int kViewCap = 2 * kMaxOverlap - 1;
constexpr uint32_t kFastBlockCap = kViewCap * 6;  // float4s of the largest view's fast blocks

struct TraceParams {
    float L, invL, relax, minStep, hitEps;
    uint32_t maxOverlap, maxNew;
    float window;  // resolved fetch window in view-z units
};

struct Frag {
    uint32_t word;
    float zEntry, zExit;
};

// --------------------------------------------------------------------------
// View evaluation (exact path).  Parameters are read straight from the tree
// words (L1 resident, warp-uniform address -> broadcast).  The evaluation
// stack is a per-lane local array indexed by a warp-uniform stack pointer.

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

// One field value of the staged view at p (Algorithm 3): primitives push,
// operators pop two and push one.  hdr = isPrim(1) op(5) | block offset,
// word = the node's tree word.
template <class O>
BT_DEV float eval_staged(const uint32_t* hdr, const uint32_t* word, uint32_t n, const float4* words, F3 p) {
    float stk[kStackCap];
    uint32_t sp = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t b = hdr[i];
        const float4* P4 = words + word[i] + 1;
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

// One field value consumed (tracer.hpp:115-175), as straight-line selects.
//
// Every outcome of the reference loop body is one of:
//   accept   the sample (evalT, v) becomes (t, f): phase 1 (f(t0)), phase 3
//            (back-off sample), a trusted main step, or an overshoot whose
//            back-off point tb already reaches the saved sphere (then
//            t = savedT = tn, f = savedF = v and relaxation is back on -- the
//            same state as a trusted step); then hit if v <= eps, miss if a
//            main step reached t1, else advance: the next step from (t, f),
//            clamped to t1.  While backing off, an advance that reaches the
//            remembered sphere re-uses it (no evaluation): hit / miss tests on
//            (savedT, savedF), then one more relaxed advance from there.
//   back off an overshoot: save (tn, v), march unrelaxed from tb (phase 3),
//            or miss when tb lies beyond t1
// Everything is computed unconditionally and committed by predicates, so a
// warp whose lanes end, hit, overshoot, back off or re-use a sphere in the
// same iteration never diverges.  Arithmetic is the reference's, op for op.
BT_DEV void march_consume(March& m, float v, const TraceParams& tp) {
    m.evals++;
    const uint32_t ph = m.st & kPhaseMask;
    const float tn = m.evalT;
    const bool main = ph == 2u;
    const bool relax = (m.st & kRelax) != 0u;
    const bool saved = (m.st & kSaved) != 0u;
    const bool ovBase = main && relax && (E::mul(E::sub(tn, m.t), tp.L) >= E::add(m.f, fabsf(v)) || v < -tp.hitEps);
    const float tb = E::add(m.t, smax(E::mul(m.f, tp.invL), tp.minStep));
    const bool ov = ovBase && !(tb >= tn);
    const bool acc = !ov;
    const bool hitNow = acc && v <= tp.hitEps;
    const bool endNow = acc && !hitNow && main && tn >= m.t1;
    const bool stepOn = acc && !hitNow && !endNow;
    // advance from the accepted sample (tn, v) with the current relaxation
    const float r = E::mul(v, tp.invL);
    const bool fin = is_finite(r);
    const float tnA = E::add(tn, smax(relax ? E::mul(tp.relax, r) : r, tp.minStep));
    // ... reaching the remembered sphere while backing off
    const bool reach = stepOn && fin && saved && tnA >= m.savedT;
    const bool reuse = reach && m.savedT >= E::add(tn, tp.minStep) && m.savedT <= m.t1;
    const bool hit2 = reuse && m.savedF <= tp.hitEps;
    const bool end2 = reuse && !hit2 && m.savedT >= m.t1;
    const float r2 = E::mul(m.savedF, tp.invL);
    const float tn2 = E::add(m.savedT, smax(E::mul(tp.relax, r2), tp.minStep));  // relaxation is back on
    const bool miss2 = reuse && !hit2 && !end2 && !is_finite(r2);
    const bool step2 = reuse && !hit2 && !end2 && !miss2;
    const bool beyond = tnA > m.t1;
    const bool missAdv = stepOn && !reuse && (!fin || (beyond && tn >= m.t1));
    const bool step1 = stepOn && !reuse && !missAdv;
    const bool missOv = ov && tb > m.t1;
    if (acc) {
        m.t = tn;
        m.f = v;
    }
    if (reuse) {
        m.t = m.savedT;
        m.f = m.savedF;
    }
    if (ov) {  // back off (phase 3) -- the saved sphere is only used when not missing
        m.savedT = tn;
        m.savedF = v;
        m.evalT = tb;
        m.st = (m.st & ~(kRelax | kPhaseMask)) | kSaved | 3u;
    }
    if (reach) m.st = (m.st & ~kSaved) | kRelax;
    if (step1) {
        m.evalT = beyond ? m.t1 : tnA;
        m.st = (m.st & ~kPhaseMask) | 2u;
    }
    if (step2) {
        m.evalT = tn2 > m.t1 ? m.t1 : tn2;
        m.st = (m.st & ~kPhaseMask) | 2u;
    }
    if (hitNow || hit2) m.st = (m.st & kSlot1) | kHitFlag;  // t holds the hit (tn or savedT)
    if (endNow || missAdv || missOv || end2 || miss2) {
        m.st = m.st & kSlot1;
        m.t = 0.0f;
    }
}

}  // namespace btk
