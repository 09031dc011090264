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
    uint32_t viewLipschitz;  // step bound per view (bt_set_step_bound): 1-Lipschitz views march with L = 1
};

// A view whose field is 1-Lipschitz: exact signed distances (sphere, torus,
// box, sphere-cone: field.cpp:219-254 are the Euclidean distances) combined
// only by sharp CSG (min / max / max(a, -b)) and the reserved pass-through
// codes, all of which preserve the Lipschitz constant 1.  The ellipsoid and
// quadric are first-order approximations and the smooth / compact blends
// compress the field (the reason for the global bound L = 1.45, PAPER.md
// "Ray processing"), so any of them keeps the configured bound.
BT_HD bool node_is_one_lipschitz(uint32_t hdr) {
    const uint32_t op = blob_op(hdr);
    if (blob_is_prim(hdr)) return op == 0u || op == 2u || op == 3u || op == 4u;
    return op <= 5u;
}
// ... or becomes 1-Lipschitz where every compact operator (codes 9-11) is in
// its CSG branch: max(f0, f1) > d (field.cpp:424-440) -- the compact blends
// are exactly CSG outside their support, which is their point
BT_HD bool node_is_lipschitz_capable(uint32_t hdr) {
    return node_is_one_lipschitz(hdr) || (!blob_is_prim(hdr) && blob_op(hdr) >= 9u && blob_op(hdr) <= 11u);
}

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
// Sphere-trace state machine (tracer.hpp:99-177), restated so that a ray
// needs exactly one field value per lockstep step.  March arithmetic is
// always exact (IEEE op by op), in both modes.
//
// State: the accepted sample (t, f), the end t1, the saved sphere
// (savedT, savedF), the point being evaluated (evalT), and st:
//   kActive  the ray is marching (phase != 0); with kMain clear the sample
//            is ACCEPTed as is (f(t0), or a back-off sample), with kMain set
//            it is a MAIN step (overshoot-tested while relaxed);
//   kSaved   a saved sphere is pending -- relaxation is off exactly while one
//            is (relaxOn == !savedValid is an invariant of the reference loop,
//            so one flag carries both);
//   kTestOv  kMain and not kSaved: the step is overshoot-tested (kept as its
//            own bit so the test is one LOP3);
//   kHitFlag on completion: t holds the hit position.
constexpr uint32_t kActive = 1u, kMain = 2u, kSaved = 4u, kHitFlag = 8u, kTestOv = 64u;
// bt_set_step_bound(1), comb views with compact operators: the step from the
// accepted point t (kLipT) / from the saved sphere (kLipS) was bounded with
// L = 1 (see march_consume)
constexpr uint32_t kLipT = 16u, kLipS = 32u;

struct March {
    float t, f, t1, savedT, savedF, evalT;
    uint32_t st, evals;
};

BT_DEV uint32_t march_phase(const March& m) { return m.st & kActive; }
BT_DEV bool march_hit(const March& m) { return (m.st & kHitFlag) != 0u; }

BT_DEV void march_idle(March& m) {
    m.st = 0u;
    m.evals = 0;
    m.t = 0.0f;
}

BT_DEV void march_begin(March& m, float t0, float t1) {
    m.evals = 0;
    m.t1 = t1;
    m.t = 0.0f;
    m.evalT = t0;
    m.st = t0 > t1 ? 0u : kActive;  // ACCEPT f(t0); t0 > t1: an empty interval, a miss without evaluation
}

// One field value v = f(evalT) consumed.  The reference loop, per sample:
//   MAIN, relaxed, overshoot ((tn-t)L >= f+|v| or v < -eps) -> save (tn, v),
//        back off to tb = t + max(f/L, minStep): evaluate there (ACCEPT next),
//        or, when tb already reaches the saved sphere, accept (tn, v) with
//        relaxation on -- the same as a trusted step -- or miss beyond t1;
//   otherwise the sample is accepted as (t, f): hit if v <= eps, else
//   ADVANCE: miss if f/L is not finite; step = max(relaxed ? relax f/L : f/L,
//        minStep); a step that reaches the saved sphere drops it (relaxation
//        back on) and, when the sphere lies in [t + minStep, t1], RE-USES it
//        without an evaluation: hit test on (savedT, savedF), then one more
//        relaxed advance from there; finally the step is clamped to t1, and a
//        sample already at t1 ends the march (a miss).
// The reference's end test after a trusted main step (tn >= t1 -> miss) is
// the clamp's "already at t1" case of the advance that follows, with the
// same outcome and the same evaluation count.  Everything is computed
// unconditionally and committed by predicates: a warp whose lanes hit,
// miss, overshoot, back off or re-use a sphere in the same step never
// diverges.
// Lip = true (bt_set_step_bound(1) on a comb view with compact operators):
// the bound L of each step is chosen at the sample the step starts from --
// 1 when `lip1` (every compact operator of the view is in its CSG branch
// with a margin max(f0, f1) - d above the relaxed step length, and every
// primitive is an exact distance, so the field is 1-Lipschitz over the whole
// step: each operand moves by at most the step length), else tp.L -- and
// remembered for the overshoot test, the back-off and the saved sphere.
// Lip = false is the reference's loop with the global bound.
template <bool Lip = false>
BT_DEV void march_consume(March& m, float v, const TraceParams& tp, bool lip1 = false) {
    // Boolean algebra with & | (no short-circuit branches) and FMNMX for the
    // step maxima: max(x, minStep) with minStep > 0 equals std::max except
    // for a NaN x, and a NaN x only arises from a non-finite f/L, which ends
    // the march before the step is used.
    m.evals++;
    const float tn = m.evalT;
    const bool testOv = (m.st & kTestOv) != 0u;
    const bool sv = (m.st & kSaved) != 0u;
    const float sT = m.savedT, sF = m.savedF;
    const float Lt = Lip && (m.st & kLipT) ? 1.0f : tp.L, invLt = Lip && (m.st & kLipT) ? 1.0f : tp.invL;
    const float invLn = Lip && lip1 ? 1.0f : tp.invL, invLs = Lip && (m.st & kLipS) ? 1.0f : tp.invL;
    const bool ovT = testOv &
                     ((E::mul(E::sub(tn, m.t), Lt) >= E::add(m.f, fabsf(v))) | (v < -tp.hitEps));
    const float tb = E::add(m.t, fmaxf(E::mul(m.f, invLt), tp.minStep));
    const bool ov = ovT & !(tb >= tn);
    const bool hit1 = !ov & (v <= tp.hitEps);
    // advance from the accepted (tn, v)
    const float r = E::mul(v, invLn);
    const bool fin = is_finite(r);
    const float tnA = E::add(tn, fmaxf(sv ? r : E::mul(tp.relax, r), tp.minStep));
    const bool reach = sv & !hit1 & fin & (tnA >= sT);  // sv implies !ov
    const bool reuse = reach & (sT >= E::add(tn, tp.minStep)) & (sT <= m.t1);
    // ... re-using the saved sphere, then one relaxed advance from it
    const float r2 = E::mul(sF, invLs);
    const float tn2 = E::add(sT, fmaxf(E::mul(tp.relax, r2), tp.minStep));
    const bool hit2 = reuse & (sF <= tp.hitEps);
    const float T = reuse ? sT : tn;  // the accepted point the next step starts from
    const float En = reuse ? tn2 : tnA;
    const bool finN = is_finite(reuse ? r2 : r);
    const bool beyond = En > m.t1;
    const bool hit = hit1 | hit2;
    const bool miss = (!ov & !hit & (!fin | !finN | (beyond & (T >= m.t1)))) | (ov & (tb > m.t1));
    m.savedT = ov ? tn : sT;
    m.savedF = ov ? v : sF;
    m.t = ov ? m.t : T;
    m.f = ov ? m.f : (reuse ? sF : v);
    m.evalT = ov ? tb : (beyond ? m.t1 : En);
    const bool keepSaved = sv & !reach;
    uint32_t next = ov ? (kActive | kSaved) : (keepSaved ? (kActive | kMain | kSaved) : (kActive | kMain | kTestOv));
    if (Lip) {
        const uint32_t lipT = ov ? (m.st & kLipT) : ((reuse ? (m.st & kLipS) != 0u : lip1) ? kLipT : 0u);
        const uint32_t lipS = ov ? (lip1 ? kLipS : 0u) : ((sv & !reach) ? (m.st & kLipS) : 0u);
        next |= lipT | lipS;
    }
    m.st = hit ? kHitFlag : (miss ? 0u : next);
}

}  // namespace btk
