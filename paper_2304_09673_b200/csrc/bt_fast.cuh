// bt_fast.cuh -- tolerance-path field evaluation over precomputed parameter
// blocks (the paper's per-tile parameter cache, made GPU-native).
//
// Once per fetched interval the warp converts every node of the pruned view
// into an evaluation-ready block (lane-parallel, convert_node): the rigid
// transform rotate(conj(q), p - t) becomes three affine rows R p + c, radii
// become reciprocals, operators carry k/6, 1/k and 6/(6d-k).  The marching
// loop then spends its issue slots on FFMA/MUFU work instead of quaternion
// algebra and divisions.  Same formulas as the reference (field.cpp:219-454)
// up to FP32 rounding -- this is the FMA path whose parity contract is the
// tolerance one (hit mask >= 99.9 %, depth <= 2 minStep).  The exact path
// (IEEE op-by-op on the raw parameters) lives in bt_core.cuh.
#pragma once

#include "bt_tile.cuh"

namespace btk {

// ---------------------------------------------------------------- conversion

BT_DEV void affine_rows(const float* P, float4* B) {
    // rotate(conj(q), v) for unit q == R v with R the matrix of conj(q)
    const float w = P[3], x = -P[4], y = -P[5], z = -P[6];
    const float r00 = 1.f - 2.f * (y * y + z * z), r01 = 2.f * (x * y - w * z), r02 = 2.f * (x * z + w * y);
    const float r10 = 2.f * (x * y + w * z), r11 = 1.f - 2.f * (x * x + z * z), r12 = 2.f * (y * z - w * x);
    const float r20 = 2.f * (x * z - w * y), r21 = 2.f * (y * z + w * x), r22 = 1.f - 2.f * (x * x + y * y);
    const float tx = P[0], ty = P[1], tz = P[2];
    B[0] = make_float4(r00, r01, r02, -(r00 * tx + r01 * ty + r02 * tz));
    B[1] = make_float4(r10, r11, r12, -(r10 * tx + r11 * ty + r12 * tz));
    B[2] = make_float4(r20, r21, r22, -(r20 * tx + r21 * ty + r22 * tz));
}

// Writes the fast block of one view node (blob may carry a reserved code).
// Reciprocals and quotients use the approximate MUFU forms (rcp.approx,
// <= 1 ulp): this is the tolerance path, and IEEE division's slow-path
// check and call would cost more than the whole conversion.
BT_DEV void convert_node(uint32_t blob, const float4* raw, float4* B) {
    const uint32_t code = blob_op(blob);
    if (!blob_is_prim(blob)) {
        if (code < 6u || code > 11u) return;  // reserved / sharp: no parameters
        const float4 q = __ldg(raw);
        const float k = q.x, d = q.y;
        const float invk = FastOps::rcp(k), k6 = k * (1.0f / 6.0f);
        if (code <= 8u) {
            B[0] = make_float4(k, k6, invk, 0.0f);
        } else {
            B[0] = make_float4(k, d, k6, invk);
            B[1] = make_float4(FastOps::rcp(d - k6), 0.0f, 0.0f, 0.0f);  // 6 / (6d - k)
        }
        return;
    }
    float P[20];
    load_params<5>(P, raw);
    const float* s = P + 7;
    if (code == 0u) {  // sphere: rotation-invariant, keep the centre
        B[0] = make_float4(P[0], P[1], P[2], s[0]);
        return;
    }
    affine_rows(P, B);
    switch (code) {
        case 1: {  // ellipsoid
            const float i0 = FastOps::rcp(s[0]), i1 = FastOps::rcp(s[1]), i2 = FastOps::rcp(s[2]);
            B[3] = make_float4(i0, i1, i2, -smin(s[0], smin(s[1], s[2])));
            B[4] = make_float4(i0 * i0, i1 * i1, i2 * i2, 0.0f);
            break;
        }
        case 2:  // torus
            B[3] = make_float4(s[0], s[1], 0.0f, 0.0f);
            break;
        case 3:  // box
            B[3] = make_float4(s[0], s[1], s[2], 0.0f);
            break;
        case 4: {  // sphere-cone
            const float b = (s[0] - s[1]) * FastOps::rcp(s[2]);
            const float a = FastOps::sqrt(1.0f - b * b);
            B[3] = make_float4(s[0], s[1], s[2], b);
            B[4] = make_float4(a, a * s[2], 0.0f, 0.0f);
            break;
        }
        default:  // quadric
            B[3] = make_float4(s[0], s[1], s[2], s[3]);
            B[4] = make_float4(s[4], s[5], s[6], s[7]);
            B[5] = make_float4(s[8], s[9], 0.0f, 0.0f);
            break;
    }
}

// ---------------------------------------------------------------- evaluation

BT_DEV float fsqrt(float a) { return FastOps::sqrt(a); }

BT_DEV float nan_to_zero(float v) { return is_nan(v) ? 0.0f : v; }

BT_DEV float f_sphere(float4 c, F3 p) {
    const float dx = p.x - c.x, dy = p.y - c.y, dz = p.z - c.z;
    return fsqrt(dx * dx + dy * dy + dz * dz) - c.w;
}
// three FFMAs per row: the translation is the chain's seed
BT_DEV F3 f_affine(float4 r0, float4 r1, float4 r2, F3 p) {
    return F3{fmaf(r0.x, p.x, fmaf(r0.y, p.y, fmaf(r0.z, p.z, r0.w))),
              fmaf(r1.x, p.x, fmaf(r1.y, p.y, fmaf(r1.z, p.z, r1.w))),
              fmaf(r2.x, p.x, fmaf(r2.y, p.y, fmaf(r2.z, p.z, r2.w)))};
}
BT_DEV float f_box(float4 e, F3 l) {
    const float qx = fabsf(l.x) - e.x, qy = fabsf(l.y) - e.y, qz = fabsf(l.z) - e.z;
    const float ox = fmaxf(qx, 0.0f), oy = fmaxf(qy, 0.0f), oz = fmaxf(qz, 0.0f);
    return fsqrt(ox * ox + oy * oy + oz * oz) + fminf(fmaxf(qx, fmaxf(qy, qz)), 0.0f);
}
BT_DEV float f_torus(float4 e, F3 l) {
    const float qx = fsqrt(l.x * l.x + l.z * l.z) - e.x;
    return fsqrt(qx * qx + l.y * l.y) - e.y;
}
BT_DEV float f_ellipsoid(float4 e, float4 f, F3 l) {  // k0 (k0 - 1) / k1
    const float ax = l.x * e.x, ay = l.y * e.y, az = l.z * e.z;
    const float bx = l.x * f.x, by = l.y * f.y, bz = l.z * f.z;
    const float k0 = fsqrt(ax * ax + ay * ay + az * az);
    const float k1 = fsqrt(bx * bx + by * by + bz * bz);
    return k1 <= 0.0f ? e.w : k0 * (k0 - 1.0f) * FastOps::rcp(k1);
}
BT_DEV float f_cone(float4 e, float4 f, F3 l) {
    const float qx = fsqrt(l.x * l.x + l.z * l.z), qy = l.y;
    const float k = qy * f.x - qx * e.w;
    if (k < 0.0f) return fsqrt(qx * qx + qy * qy) - e.x;
    if (k > f.y) {
        const float dy = qy - e.z;
        return fsqrt(qx * qx + dy * dy) - e.y;
    }
    return qx * f.x + qy * e.w - e.x;
}
BT_DEV float f_quadric(float4 e, float4 g, float4 h, F3 l) {  // f0 / max(|grad f0|, 1e-4)
    const float x = l.x, y = l.y, z = l.z;
    const float u = e.x * x + e.w * y + g.x * z + g.z;  // c0 x + c3 y + c4 z + c6
    const float vv = e.y * y + g.y * z + g.w;           // c1 y + c5 z + c7
    const float w = e.z * z + h.x;                      // c2 z + c8
    const float gx = u + e.x * x;
    const float gy = vv + e.y * y + e.w * x;
    const float gz = w + e.z * z + g.x * x + g.y * y;
    const float f0 = x * u + y * vv + z * w + h.y;
    return f0 * FastOps::rcp(fmaxf(fsqrt(gx * gx + gy * gy + gz * gz), 1e-4f));
}

// One primitive at NP points; the parameter block is loaded once.
template <int NP>
BT_DEV void fast_primitive(uint32_t oh, const float4* B, const F3* p, float* v) {
    if (oh & 1u) {  // sqrt(x) - r of a finite point: never NaN (no filter needed)
        const float4 c = B[0];
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_sphere(c, p[i]);
        return;
    }
    const float4 r0 = B[0], r1 = B[1], r2 = B[2], e = B[3];
    F3 l[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) l[i] = f_affine(r0, r1, r2, p[i]);
    if (oh & 8u) {
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_box(e, l[i]);
    } else if (oh & 4u) {
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_torus(e, l[i]);
    } else if (oh & 2u) {
        const float4 f = B[4];
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_ellipsoid(e, f, l[i]);
    } else if (oh & 16u) {
        const float4 f = B[4];
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_cone(e, f, l[i]);
    } else {
        const float4 g = B[4], h = B[5];
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = f_quadric(e, g, h, l[i]);
    }
    // the reference's NaN -> 0 filter (field.cpp:283), where a finite point
    // can produce NaN (see fast_prim)
    if (oh & 18u) {
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = nan_to_zero(v[i]);
    }
}

// Operators on the fast path.  FMNMX-based min/max (fminf/fmaxf) instead of
// the reference's std::min/max select semantics: they differ only for NaN
// operands and signed zeros, which the tolerance path does not carry (field
// values here are never NaN).  disp = (k/6) max(1 - |a-b|/k, 0)^3 is written
// branch-free: |a-b| >= k gives t = 0, k = 0 gives t = 0 via fmaxf(NaN, 0).
BT_DEV float fast_disp(float a, float b, float k6, float invk) {
    const float t = fmaxf(fmaf(-fabsf(a - b), invk, 1.0f), 0.0f);
    return k6 * (t * t * t);
}

BT_DEV float fast_smooth(uint32_t fl, float f0, float f1, float k6, float invk) {
    if (fl == 0u) return fminf(f0, f1) - fast_disp(f0, f1, k6, invk);
    if (fl == 1u) return fmaxf(f0, f1) + fast_disp(f0, f1, k6, invk);
    return fmaxf(f0, -f1) + fast_disp(f0, -f1, k6, invk);
}

BT_DEV float fast_csg(uint32_t fl, float f0, float f1) {
    return fl == 0u ? fminf(f0, f1) : (fl == 1u ? fmaxf(f0, f1) : fmaxf(f0, -f1));
}

// compact_op (field.cpp:424-440): CSG outside the support d, else a smooth
// blend whose radius shrinks with the smoothed value (blend_range).
// B[0] = (k, d, k/6, 1/k), B[1].x = 6 / (6d - k).
BT_DEV float fast_compact(uint32_t fl, const float4* B, float f0, float f1) {
    const float4 b0 = B[0];
    if (fmaxf(f0, f1) > b0.y) return fast_csg(fl, f0, f1);
    const float g = fast_smooth(fl, f0, f1, b0.z, b0.w);
    const float x = fl == 2u ? fabsf(g) : g;
    const float br = b0.x * fmaxf(fmaf(-x, B[1].x, 1.0f), 0.0f);
    const float kp = fl == 0u ? br : fminf(br, b0.x);
    return fast_smooth(fl, f0, f1, kp * (1.0f / 6.0f), FastOps::rcp(kp));
}

// Operator by its one-hot code (bit `code` of `oh`): bit tests ordered by
// frequency (compact and sharp unions dominate blobtree views) -- nvcc turns
// an equality chain on the code into a jump table, which costs more.
BT_DEV float fast_operator(uint32_t oh, const float4* B, float f0, float f1) {
    if (oh & (1u << 9)) return fast_compact(0u, B, f0, f1);
    if (oh & (1u << 3)) return fminf(f0, f1);
    if (oh & (3u << 10)) return fast_compact((oh & (1u << 10)) ? 1u : 2u, B, f0, f1);
    if (oh & (7u << 6)) {
        const float4 b0 = B[0];
        return fast_smooth((oh & (1u << 6)) ? 0u : ((oh & (1u << 7)) ? 1u : 2u), f0, f1, b0.y, b0.z);
    }
    if (oh & (1u << 4)) return fmaxf(f0, f1);
    if (oh & (1u << 5)) return fmaxf(f0, -f1);
    return (oh & 1u) ? f_inf() : ((oh & 2u) ? f1 : f0);
}

// Header of a staged fast-path node: isPrim(1) | one-hot code (bits 16-27) |
// block byte offset (16 bits; the fast blocks of a view fit in 5 KB).
BT_DEV uint32_t fast_hdr(uint32_t hdr) {
    return (hdr & 0x80000000u) | ((1u << blob_op(hdr)) << 16) | (hdr & 0xFFF0u);
}
BT_DEV uint32_t fast_hdr_code(uint32_t fh) { return (fh >> 16) & 0xFFFu; }

// ---------------------------------------------------------------- view classes
//
// The interpreter below (eval_view_fast) pays per node for the header load,
// the block address, prim/op tests, the kind and operator dispatch chains and
// the two-register stack -- ~27 instructions per node, more than the field
// arithmetic of the node on the small views that dominate (SURVEY.md appendix
// C scenes: 98 % of C3's field evaluations are on views of <= 4 primitives).
// The march therefore classifies each interval's view ONCE, when it is
// staged, and runs a march loop specialised for its class:
//   single  one primitive (20 % of C3's evaluations, 48 % of C1's): its kind
//           and block live in registers for the whole interval;
//   comb    a left comb P (P O)* -- every operator's right operand is the
//           primitive just before it (78 % at C3): one 8-byte record per
//           primitive (kind + block, operator code + block), no stack;
//   general anything else: the interpreter.
// Same formulas, same order of operations: the class only removes decoding.

// A value every lane holds, made visibly warp-uniform: REDUX writes a
// uniform register, so branches on it need no reconvergence barrier.  Used
// once per interval (the single class's record), NOT per node: measured on
// the per-node header reads (alternating A/B, scripts/ab_multi.sh) the
// REDUX latency on the header -> block address -> parameter chain costs
// more than the BSSY/BSYNC pairs it removes (C3 march +2.5 %, C2 / C5 +20 %).
// All 32 lanes must call.
BT_DEV uint32_t warp_uniform(uint32_t v) { return __reduce_or_sync(0xFFFFFFFFu, v); }

// comb record of primitive j: x = block byte offset << 16 | 1 << kind,
// y = the operator's block byte offset << 16 | 1 << operator code (j >= 1).
// One shift gives the address; the kind and operator dispatch are bit tests
// (LOP3 + branch each), which nvcc cannot turn into a jump table -- an
// equality chain on a small integer becomes a BRX table whose index
// arithmetic and reconvergence barriers cost more than the tests.
// (Measured: one switch over (kind, operator class) per primitive instead
// of the two compare chains makes the C3 march 30 % slower.)
BT_DEV uint32_t comb_rec(uint32_t hdr) { return ((hdr & 0xFFF0u) << 16) | (1u << blob_op(hdr)); }
BT_DEV const float4* comb_rec_block(const float4* blk, uint32_t x) {
    return reinterpret_cast<const float4*>(reinterpret_cast<const unsigned char*>(blk) + (x >> 16));
}
constexpr uint32_t kRecSphere = 1u << 0, kRecEllipsoid = 1u << 1, kRecTorus = 1u << 2, kRecBox = 1u << 3,
                   kRecCone = 1u << 4;
constexpr uint32_t kRecCsgUnion = 1u << 3, kRecCompactUnion = 1u << 9, kRecCompact = 7u << 9;

// One primitive value at one point; `kind` is warp-uniform.  The rigid
// transform is shared by every rotated kind.
//
// The reference's NaN -> 0 filter (field.cpp:283) is applied where a NaN can
// arise from a finite point: the ellipsoid (1/r of a zero radius times a zero
// coordinate) and the sphere-cone (sqrt(1 - b^2) for |r0 - r1| >= h) when
// their parameters bypassed validate_primitive (a tree uploaded straight
// through the C-ABI).  Sphere, box, torus and quadric are closed forms of
// finite values with no 0 * inf, inf - inf or sqrt of a negative: for finite
// points and parameters (|.| < 1e18, no overflow) they never produce NaN, and
// the filter there would cost 1.3 % of the march (measured, alternating A/B).
// tests/test_gpu_reference_scale.py checks NaN-free FMA frames on every kind.
BT_DEV float fast_prim(uint32_t x, const float4* B, F3 p) {
    if (x & kRecSphere) return f_sphere(B[0], p);
    const F3 l = f_affine(B[0], B[1], B[2], p);
    const float4 e = B[3];
    if (x & kRecBox) return f_box(e, l);
    if (x & kRecTorus) return f_torus(e, l);
    if (x & kRecEllipsoid) return nan_to_zero(f_ellipsoid(e, B[4], l));
    if (x & kRecCone) return nan_to_zero(f_cone(e, B[4], l));
    return f_quadric(e, B[4], B[5], l);
}

// operator of a comb step: compact and sharp unions first (the blobtree
// generators' joins), the general chain otherwise
BT_DEV float comb_op(uint32_t y, const float4* B, float f0, float f1) {
    if (y & kRecCompactUnion) return fast_compact(0u, B, f0, f1);
    if (y & kRecCsgUnion) return fminf(f0, f1);
    return fast_operator(y & 0xFFFFu, B, f0, f1);
}

BT_DEV float eval_comb(const uint2* rec, uint32_t nPrims, const float4* blk, F3 p) {
    uint2 r = rec[0];
    float v = fast_prim(r.x, comb_rec_block(blk, r.x), p);
    for (uint32_t j = 1; j < nPrims; ++j) {
        r = rec[j];
        const float w = fast_prim(r.x, comb_rec_block(blk, r.x), p);
        v = comb_op(r.y, comb_rec_block(blk, r.y), v, w);
    }
    return v;
}

// eval_comb plus the CSG margin of its compact operators: min over them of
// max(f0, f1) - d (> 0: every one is in its CSG branch, field.cpp:431)
BT_DEV float eval_comb_margin(const uint2* rec, uint32_t nPrims, const float4* blk, F3 p, float& margin) {
    uint2 r = rec[0];
    float v = fast_prim(r.x, comb_rec_block(blk, r.x), p);
    float mg = f_inf();
    for (uint32_t j = 1; j < nPrims; ++j) {
        r = rec[j];
        const float4* Bo = comb_rec_block(blk, r.y);
        const float w = fast_prim(r.x, comb_rec_block(blk, r.x), p);
        if (r.y & kRecCompact) mg = fminf(mg, fmaxf(v, w) - Bo[0].y);
        v = comb_op(r.y, Bo, v, w);
    }
    margin = mg;
    return v;
}

constexpr uint32_t kNotAnOp = 0x80000000u;  // a primitive header: ends a fused primitive + operator pair

// Algorithm 3 over the fast blocks of a staged view (headers in fast_hdr
// form; `prm` = the blocks in
// this warp's shared memory), at NP points per lane.  The two top stack
// entries live in registers (t0 = top, t1 = second): a left comb -- the
// common blobtree shape -- never touches the local-memory part, deeper
// entries spill to it only when a third value is pushed.
template <int NP>
BT_DEV void eval_view_fast(const uint32_t* hdr, uint32_t n, const float4* prm, const F3* p, float* out) {
    float deep[NP][kStackCap];
    float t0[NP], t1[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) t0[k] = t1[k] = 0.0f;
    uint32_t sp = 0;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(prm);
    uint32_t b = n ? hdr[0] : 0u;  // the next node's header is carried from the previous iteration
    for (uint32_t i = 0; i < n;) {
        const float4* B = reinterpret_cast<const float4*>(base + (b & 0xFFFFu));
        const uint32_t bn = i + 1 < n ? hdr[i + 1] : kNotAnOp;
        if (blob_is_prim(b)) {
            float v[NP];
            fast_primitive<NP>(fast_hdr_code(b), B, p, v);
            // a primitive directly followed by an operator (every step of a
            // left comb, the common blobtree shape): combine with the stack top
            // in place, no push / pop
            if (sp >= 1u && !blob_is_prim(bn)) {
                const uint32_t code = fast_hdr_code(bn);
                const float4* Bo = reinterpret_cast<const float4*>(base + (bn & 0xFFFFu));
#pragma unroll
                for (int k = 0; k < NP; ++k) t0[k] = fast_operator(code, Bo, t0[k], v[k]);
                i += 2;
                b = i < n ? hdr[i] : 0u;
                continue;
            }
            if (sp >= 2u) {
#pragma unroll
                for (int k = 0; k < NP; ++k) deep[k][sp - 2u] = t1[k];
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                t1[k] = t0[k];
                t0[k] = v[k];
            }
            ++sp;
        } else {
            const uint32_t code = fast_hdr_code(b);
#pragma unroll
            for (int k = 0; k < NP; ++k) t0[k] = fast_operator(code, B, t1[k], t0[k]);
            --sp;
            if (sp >= 2u) {
#pragma unroll
                for (int k = 0; k < NP; ++k) t1[k] = deep[k][sp - 2u];
            }
        }
        ++i;
        b = bn;
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) out[k] = t0[k];
}

}  // namespace btk
