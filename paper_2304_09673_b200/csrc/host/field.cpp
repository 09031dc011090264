// host/field.cpp -- primitive/operator bookkeeping, validation and the
// single-point field helpers of the drop-in API.  The arithmetic itself is
// the shared host/device core (../bt_core.cuh, ../bt_geom.cuh) instantiated
// with IEEE-exact ops, i.e. the same code the kernels run.
//
// Reference: src/field.cpp:10-459 (names, validation messages, formulas).
#include "blobtree/field.hpp"

#include <cstring>

#include "../bt_geom.cuh"

namespace blobtree {

namespace {

struct KindInfo {
    const char* name;
    uint32_t shapeFloats;
};
constexpr KindInfo kPrimInfo[kPrimitiveKindCount] = {
    {"sphere", 1}, {"ellipsoid", 3}, {"torus", 2}, {"box", 3}, {"sphere_cone", 3}, {"quadric", 10},
};
constexpr const char* kOpNames[9] = {"csg_union",     "csg_intersect",    "csg_diff",
                                     "smooth_union",  "smooth_intersect", "smooth_diff",
                                     "compact_union", "compact_intersect", "compact_diff"};

inline uint32_t code(OperatorKind k) { return static_cast<uint32_t>(k); }
inline uint32_t flavour(OperatorKind k) { return btk::op_flavour(code(k)); }

bool is_pos(float v) { return std::isfinite(v) && v > 0.0f; }

PrimitiveParams make(PrimitiveKind kind, Transform frame, std::initializer_list<float> shape) {
    PrimitiveParams p;
    p.kind = kind;
    p.frame = frame;
    size_t i = 0;
    for (float v : shape) p.shape[i++] = v;
    validate_primitive(p);
    return p;
}

}  // namespace

uint32_t shape_float_count(PrimitiveKind kind) {
    const auto k = static_cast<uint32_t>(kind);
    return k < kPrimitiveKindCount ? kPrimInfo[k].shapeFloats : 0u;
}

const char* primitive_kind_name(PrimitiveKind kind) {
    const auto k = static_cast<uint32_t>(kind);
    return k < kPrimitiveKindCount ? kPrimInfo[k].name : "?";
}

bool primitive_kind_from_name(const char* name, PrimitiveKind& out) {
    for (uint32_t k = 0; k < kPrimitiveKindCount; ++k) {
        if (std::strcmp(kPrimInfo[k].name, name) != 0) continue;
        out = static_cast<PrimitiveKind>(k);
        return true;
    }
    return false;
}

PrimitiveParams PrimitiveParams::sphere(float r, Transform frame) { return make(PrimitiveKind::Sphere, frame, {r}); }
PrimitiveParams PrimitiveParams::ellipsoid(Vec3 radii, Transform frame) {
    return make(PrimitiveKind::Ellipsoid, frame, {radii.x, radii.y, radii.z});
}
PrimitiveParams PrimitiveParams::torus(float major, float minor, Transform frame) {
    return make(PrimitiveKind::Torus, frame, {major, minor});
}
PrimitiveParams PrimitiveParams::box(Vec3 h, Transform frame) { return make(PrimitiveKind::Box, frame, {h.x, h.y, h.z}); }
PrimitiveParams PrimitiveParams::sphere_cone(float r0, float r1, float h, Transform frame) {
    return make(PrimitiveKind::SphereCone, frame, {r0, r1, h});
}
PrimitiveParams PrimitiveParams::quadric(const std::array<float, 10>& coeffs, Transform frame) {
    PrimitiveParams p;
    p.kind = PrimitiveKind::Quadric;
    p.frame = frame;
    p.shape = coeffs;
    validate_primitive(p);
    return p;
}

QuadricInfo analyze_quadric(const std::array<float, 10>& c) {
    const btk::QuadricInfoK k = btk::analyze_quadric_k(c.data());
    QuadricInfo info;
    info.lambdaMin = k.lmin;
    info.lambdaMax = k.lmax;
    info.positiveDefinite = k.pd;
    if (!k.pd) return info;
    info.center = Vec3{k.center.x, k.center.y, k.center.z};
    info.isoLevel = k.iso;
    info.hasInterior = info.isoLevel > 0.0f;
    return info;
}

void validate_primitive(const PrimitiveParams& p) {
    if (!is_finite(p.frame.translate)) throw std::invalid_argument("primitive translation must be finite");
    if (std::fabs(length(p.frame.rotation) - 1.0f) > 1e-6f)
        throw std::invalid_argument("primitive rotation must be a unit quaternion");
    const auto& s = p.shape;
    switch (p.kind) {
        case PrimitiveKind::Sphere:
            if (!is_pos(s[0])) throw std::invalid_argument("sphere radius must be > 0");
            return;
        case PrimitiveKind::Ellipsoid:
            if (!(is_pos(s[0]) && is_pos(s[1]) && is_pos(s[2])))
                throw std::invalid_argument("ellipsoid radii must be > 0");
            return;
        case PrimitiveKind::Torus:
            if (!(is_pos(s[0]) && is_pos(s[1]))) throw std::invalid_argument("torus radii must be > 0");
            if (!(s[1] < s[0])) throw std::invalid_argument("torus minor radius must be below the major radius");
            return;
        case PrimitiveKind::Box:
            if (!(is_pos(s[0]) && is_pos(s[1]) && is_pos(s[2])))
                throw std::invalid_argument("box half extents must be > 0");
            return;
        case PrimitiveKind::SphereCone:
            if (!(is_pos(s[0]) && is_pos(s[1]) && is_pos(s[2])))
                throw std::invalid_argument("sphere-cone radii and height must be > 0");
            if (!(std::fabs(s[0] - s[1]) < s[2]))
                throw std::invalid_argument("sphere-cone height must exceed the radius difference");
            return;
        case PrimitiveKind::Quadric: {
            const QuadricInfo info = analyze_quadric(s);
            if (!info.positiveDefinite) throw std::invalid_argument("quadric matrix must be positive definite");
            if (!info.hasInterior) throw std::invalid_argument("quadric must enclose a non-empty volume");
            return;
        }
    }
}

FieldValue eval_primitive_raw(uint8_t kind, const float* params, Point3 point) {
    return btk::eval_primitive<btk::ExactOps>(kind, params, btk::F3{point.x, point.y, point.z});
}

FieldValue eval_primitive(const PrimitiveParams& p, Point3 point) {
    float raw[kTransformFloatCount + 10] = {};
    raw[0] = p.frame.translate.x;
    raw[1] = p.frame.translate.y;
    raw[2] = p.frame.translate.z;
    raw[3] = p.frame.rotation.w;
    raw[4] = p.frame.rotation.x;
    raw[5] = p.frame.rotation.y;
    raw[6] = p.frame.rotation.z;
    std::memcpy(raw + kTransformFloatCount, p.shape.data(), shape_float_count(p.kind) * sizeof(float));
    return eval_primitive_raw(static_cast<uint8_t>(p.kind), raw, point);
}

// ---------------------------------------------------------------- operators

const char* operator_kind_name(OperatorKind kind) {
    const uint32_t c = code(kind);
    return (c >= 3 && c <= 11) ? kOpNames[c - 3] : "?";
}

bool operator_kind_from_name(const char* name, OperatorKind& out) {
    for (uint32_t c = 3; c <= 11; ++c) {
        if (std::strcmp(kOpNames[c - 3], name) != 0) continue;
        out = static_cast<OperatorKind>(c);
        return true;
    }
    return false;
}

bool is_sharp(OperatorKind k) { return code(k) >= 3 && code(k) <= 5; }
bool is_smooth(OperatorKind k) { return code(k) >= 6 && code(k) <= 8; }
bool is_compact(OperatorKind k) { return code(k) >= 9 && code(k) <= 11; }
bool is_union_like(OperatorKind k) { return code(k) >= 3 && code(k) <= 11 && flavour(k) == 0; }
bool is_intersect_like(OperatorKind k) { return code(k) >= 3 && code(k) <= 11 && flavour(k) == 1; }
bool is_diff_like(OperatorKind k) { return code(k) >= 3 && code(k) <= 11 && flavour(k) == 2; }

uint8_t ignore_mode_for(OperatorKind kind) {
    if (is_intersect_like(kind)) return kIgnoreIfAnyAbsent;
    return is_diff_like(kind) ? kIgnoreIfLeftAbsent : kNeverIgnore;
}

OperatorParams OperatorParams::sharp(OperatorKind kind) {
    OperatorParams op;
    op.kind = kind;
    validate_operator(op);
    return op;
}
OperatorParams OperatorParams::smooth(OperatorKind kind, float k) {
    OperatorParams op;
    op.kind = kind;
    op.blend = k;
    validate_operator(op);
    return op;
}
OperatorParams OperatorParams::compact(OperatorKind kind, float k, float rangeUpper) {
    OperatorParams op;
    op.kind = kind;
    op.blend = k;
    op.range = rangeUpper;
    validate_operator(op);
    return op;
}

void validate_operator(const OperatorParams& op) {
    if (is_sharp(op.kind)) return;
    if (!(op.blend > 0.0f && std::isfinite(op.blend))) throw std::invalid_argument("blend parameter k must be > 0");
    if (is_compact(op.kind) && !(std::isfinite(op.range) && op.range > op.blend / 6.0f))
        throw std::invalid_argument("operator range d must exceed k/6");
}

FieldValue csg_op(OperatorKind kind, FieldValue f0, FieldValue f1) { return btk::csg_op(flavour(kind), f0, f1); }
FieldValue smooth_disp(FieldValue f0, FieldValue f1, float k) { return btk::smooth_disp<btk::ExactOps>(f0, f1, k); }
FieldValue smooth_op(OperatorKind kind, FieldValue f0, FieldValue f1, float k) {
    return btk::smooth_op<btk::ExactOps>(flavour(kind), f0, f1, k);
}
float blend_range(float x, float k, float d) { return btk::blend_range<btk::ExactOps>(x, k, d); }
FieldValue compact_op(OperatorKind kind, FieldValue f0, FieldValue f1, float k, float d) {
    return btk::compact_op<btk::ExactOps>(flavour(kind), f0, f1, k, d);
}
FieldValue eval_operator_raw(uint8_t nodeop, const float* params, FieldValue f0, FieldValue f1) {
    return btk::eval_operator<btk::ExactOps>(nodeop, params, f0, f1);
}
FieldValue eval_operator(const OperatorParams& op, FieldValue f0, FieldValue f1) {
    const float kd[2] = {op.blend, op.range};
    return eval_operator_raw(static_cast<uint8_t>(op.kind), kd, f0, f1);
}

}  // namespace blobtree
