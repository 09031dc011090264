// bt_cull.cuh -- conservative volume culls of the A-buffer (device side):
// a volume's support against a pixel-centre pyramid, and the sort key of a
// tile's fragment list.  Shared by the superblock pass (k_frame.cu) and the
// per-tile pass (k_tile.cu).
#pragma once

#include "bt_device.h"

namespace btk {

// Conservative volume-vs-pyramid test with a relative + absolute pad that
// dominates every FP32 rounding on both sides.  Oriented boxes and capsules
// use their own support along each inward plane normal, not their bounding
// sphere's (19 % fewer (tile, volume) pairs to ray-test at C3).
// A box (centre c, half-axis vectors A_i = h_i rotate(q, e_i); q is a unit
// quaternion to 1e-6, validate_primitive) reaches n.(c - apex) + sum |n.A_i|;
// a capsule max(n.(a - apex), n.(b - apex)) + r.  Same relative + absolute pad
// as the sphere test, plus for capsules the cancellation error of the exact
// capsule quadratic (~ulp(dist^2) / r in distance).  A pixel ray that the
// exact test intersects lies inside the pyramid, so the volume reaches every
// plane: a rejected (tile, volume) pair cannot produce a fragment.
struct VolumeSupport {
    uint32_t family;
    F3 c, a0, a1, a2;  // box: centre, half-axis vectors; capsule: a0, a1 = ends
    float r, pad;
};

__device__ __forceinline__ VolumeSupport volume_support(const Voi& v, F3 apex) {
    VolumeSupport s;
    s.family = v.family;
    const Sphere bs = bounding_sphere(v);
    const float vx = bs.c.x - apex.x, vy = bs.c.y - apex.y, vz = bs.c.z - apex.z;
    const float dist = sqrtf(vx * vx + vy * vy + vz * vz);
    s.pad = 1e-4f * (dist + fabsf(bs.r)) + 1e-5f;
    if (v.family == 1u) {
        const float w = v.rot.w, x = v.rot.x, y = v.rot.y, z = v.rot.z;
        // columns of the rotation matrix of q, scaled by the half extents
        s.a0 = F3{(1.f - 2.f * (y * y + z * z)) * v.half.x, 2.f * (x * y + w * z) * v.half.x, 2.f * (x * z - w * y) * v.half.x};
        s.a1 = F3{2.f * (x * y - w * z) * v.half.y, (1.f - 2.f * (x * x + z * z)) * v.half.y, 2.f * (y * z + w * x) * v.half.y};
        s.a2 = F3{2.f * (x * z + w * y) * v.half.z, 2.f * (y * z - w * x) * v.half.z, (1.f - 2.f * (x * x + y * y)) * v.half.z};
        s.c = v.center;
        s.r = 0.0f;
    } else if (v.family == 2u) {
        s.a0 = v.center;
        s.a1 = v.axisEnd;
        s.r = v.radius;
        s.pad += 2.5e-7f * dist * dist / fmaxf(v.radius, 1e-6f);
    } else {
        s.c = bs.c;
        s.r = bs.r;
    }
    return s;
}

__device__ __forceinline__ bool volume_pyramid_may_touch(const float4* pl, F3 apex, const VolumeSupport& s) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float4 n = pl[e];
        float reach;
        if (s.family == 1u) {
            reach = n.x * (s.c.x - apex.x) + n.y * (s.c.y - apex.y) + n.z * (s.c.z - apex.z) +
                    fabsf(n.x * s.a0.x + n.y * s.a0.y + n.z * s.a0.z) +
                    fabsf(n.x * s.a1.x + n.y * s.a1.y + n.z * s.a1.z) +
                    fabsf(n.x * s.a2.x + n.y * s.a2.y + n.z * s.a2.z);
        } else if (s.family == 2u) {
            reach = fmaxf(n.x * (s.a0.x - apex.x) + n.y * (s.a0.y - apex.y) + n.z * (s.a0.z - apex.z),
                          n.x * (s.a1.x - apex.x) + n.y * (s.a1.y - apex.y) + n.z * (s.a1.z - apex.z)) + s.r;
        } else {
            reach = n.x * (s.c.x - apex.x) + n.y * (s.c.y - apex.y) + n.z * (s.c.z - apex.z) + s.r;
        }
        if (reach < -s.pad) return false;
    }
    return true;
}


// A volume ready for k_tile_raster's culls, for the frame's camera, built once
// per frame and volume (k_pairs) instead of once per (tile, candidate):
//   q0 = (bs.c - apex, |bs.c - apex|^2)   cone_may_touch's ray-independent
//        terms, exact ops as there (bit-identical cone test); for boxes and
//        spheres also the pyramid test's centre offset (the same single
//        rounded subtraction)
//   q1 = (bs.r, pad, family, support radius)
//   q2, q3, q4 = box: the half-axis vectors a0, a1, a2; capsule: a0 - apex,
//        a1 - apex (q4 unused)
struct CullVol {
    float4 q0, q1, q2, q3, q4;
};

__device__ __forceinline__ CullVol cull_vol_make(const Sphere& bs, const VolumeSupport& s, F3 apex) {
    CullVol r;
    const F3 cv = vsub<E>(bs.c, apex);
    r.q0 = make_float4(cv.x, cv.y, cv.z, vdot<E>(cv, cv));
    r.q1 = make_float4(bs.r, s.pad, __uint_as_float(s.family), s.r);
    if (s.family == 1u) {
        r.q2 = make_float4(s.a0.x, s.a0.y, s.a0.z, 0.0f);
        r.q3 = make_float4(s.a1.x, s.a1.y, s.a1.z, 0.0f);
        r.q4 = make_float4(s.a2.x, s.a2.y, s.a2.z, 0.0f);
    } else {
        r.q2 = make_float4(s.a0.x - apex.x, s.a0.y - apex.y, s.a0.z - apex.z, 0.0f);
        r.q3 = make_float4(s.a1.x - apex.x, s.a1.y - apex.y, s.a1.z - apex.z, 0.0f);
        r.q4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    return r;
}

// cone_may_touch (the reference's tile cone test, abuffer.cpp:140-149) with
// the volume's terms precomputed: bit-identical
__device__ __forceinline__ bool cullvol_cone_may_touch(const Cone& k, const CullVol& r) {
    const F3 v{r.q0.x, r.q0.y, r.q0.z};
    const float x = vdot<E>(v, k.axis);
    const float yy = E::sub(r.q0.w, E::mul(x, x));
    const float y = E::sqrt(smax(yy, 0.0f));
    return E::sub(E::mul(k.cosH, y), E::mul(k.sinH, x)) <= r.q1.x;
}

// volume_pyramid_may_touch with the apex already subtracted
__device__ __forceinline__ bool cullvol_pyramid_may_touch(const float4* pl, const CullVol& r) {
    const uint32_t family = __float_as_uint(r.q1.z);
    const float pad = r.q1.y;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float4 n = pl[e];
        float reach;
        if (family == 1u) {
            reach = n.x * r.q0.x + n.y * r.q0.y + n.z * r.q0.z + fabsf(n.x * r.q2.x + n.y * r.q2.y + n.z * r.q2.z) +
                    fabsf(n.x * r.q3.x + n.y * r.q3.y + n.z * r.q3.z) + fabsf(n.x * r.q4.x + n.y * r.q4.y + n.z * r.q4.z);
        } else if (family == 2u) {
            reach = fmaxf(n.x * r.q2.x + n.y * r.q2.y + n.z * r.q2.z, n.x * r.q3.x + n.y * r.q3.y + n.z * r.q3.z) + r.q1.w;
        } else {
            reach = n.x * r.q0.x + n.y * r.q0.y + n.z * r.q0.z + r.q1.w;
        }
        if (reach < -pad) return false;
    }
    return true;
}

// key order of insert_sorted (abuffer.cpp:166-173): (zEntry, word); equal
// keys keep volume order (upper_bound insertion in volume order), hence the
// volume index tiebreak.  Fragment records: (word, entry bits, exit bits, voi).
__device__ __forceinline__ bool key_less(const uint4& a, const uint4& b) {
    const float ea = __uint_as_float(a.y), eb = __uint_as_float(b.y);
    if (ea != eb) return ea < eb;
    if (a.x != b.x) return a.x < b.x;
    return a.w < b.w;
}

}  // namespace btk
