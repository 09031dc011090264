// scenes.cpp -- workload recipes C1..C5 + reference test scenes, and a
// small extern "C" accessor layer (prefix SCENE_PREFIX: `sc_` for the
// product build, `ref_` for the oracle build).  See scenes.hpp.
#include "scenes.hpp"

#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>

#include "../../../include/bt_cuda.h"
#include "blobtree/scene_io.hpp"
#ifdef SCENE_PRODUCT
#include "blobtree/device.hpp"
#endif

namespace scenes {

using namespace blobtree;

namespace {

using NodePtr = std::unique_ptr<SceneNode>;

Camera look_at(Vec3 pos, Vec3 target, float nearZ, float farZ, int w, int h) {
    Camera c;
    c.position = pos;
    c.target = target;
    c.up = Vec3{0, 1, 0};
    c.fovDegrees = 45.0f;
    c.nearZ = nearZ;
    c.farZ = farZ;
    c.width = w;
    c.height = h;
    return c;
}

NodePtr prim(const PrimitiveParams& p) { return SceneNode::make_primitive(p); }
NodePtr op(const OperatorParams& o, NodePtr l, NodePtr r) {
    return SceneNode::make_operator(o, std::move(l), std::move(r));
}
OperatorParams cunion(float k, float d) { return OperatorParams::compact(OperatorKind::CompactUnion, k, d); }
OperatorParams cinter(float k, float d) { return OperatorParams::compact(OperatorKind::CompactIntersect, k, d); }
OperatorParams cdiff(float k, float d) { return OperatorParams::compact(OperatorKind::CompactDiff, k, d); }
OperatorParams sunion() { return OperatorParams::sharp(OperatorKind::CsgUnion); }

// explicit draw order everywhere (one draw per statement)
struct Rng {
    std::mt19937 g;
    explicit Rng(uint32_t s) : g(s) {}
    float uni(float lo, float hi) {
        std::uniform_real_distribution<float> d(lo, hi);
        return d(g);
    }
    Vec3 vec(float lo, float hi) {
        const float x = uni(lo, hi);
        const float y = uni(lo, hi);
        const float z = uni(lo, hi);
        return Vec3{x, y, z};
    }
    Quat rot() {
        const Vec3 axis = vec(-1.0f, 1.0f);
        const float ang = uni(0.0f, 6.2831853f);
        if (length(axis) < 1e-3f) return Quat{};
        return quat_from_axis_angle(axis, ang);
    }
};

// one random primitive of the generator's five kinds around `center`
PrimitiveParams cell_primitive(Rng& r, Vec3 center, float scale) {
    const Vec3 off = r.vec(-0.8f * scale, 0.8f * scale);
    const Quat q = r.rot();
    const Transform tf{center + off, q};
    const int kind = static_cast<int>(r.uni(0.0f, 1.0f) * 5.0f);
    switch (kind) {
        case 0: return PrimitiveParams::sphere(r.uni(0.45f * scale, 0.9f * scale), tf);
        case 1: {
            const Vec3 h = r.vec(0.36f * scale, 0.72f * scale);
            return PrimitiveParams::box(h, tf);
        }
        case 2: {
            const float major = r.uni(0.45f * scale, 0.9f * scale);
            return PrimitiveParams::torus(major, 0.35f * major, tf);
        }
        case 3: {
            const float a = r.uni(0.45f * scale, 0.9f * scale);
            const float b = r.uni(0.45f * scale, 0.9f * scale);
            const float c = r.uni(0.45f * scale, 0.9f * scale);
            return PrimitiveParams::ellipsoid(Vec3{a, 0.7f * b, 0.85f * c}, tf);
        }
        default: {
            const float r0 = r.uni(0.45f * scale, 0.9f * scale) * 0.7f;
            return PrimitiveParams::sphere_cone(r0, r0 * 0.45f, r0 * 1.6f, tf);
        }
    }
}

// random positive definite quadric (the reference helpers' recipe, own draws)
PrimitiveParams random_quadric(Rng& r, Transform tf) {
    const Quat rq = r.rot();
    const float l0 = r.uni(0.5f, 2.2f), l1 = r.uni(0.5f, 2.2f), l2 = r.uni(0.5f, 2.2f);
    const Vec3 ax = rotate(rq, Vec3{1, 0, 0}), ay = rotate(rq, Vec3{0, 1, 0}), az = rotate(rq, Vec3{0, 0, 1});
    const float L[3] = {l0, l1, l2};
    const Vec3 cols[3] = {ax, ay, az};
    auto comp = [](const Vec3& v, int n) { return n == 0 ? v.x : (n == 1 ? v.y : v.z); };
    auto A = [&](int i, int j) {
        float s = 0.0f;
        for (int n = 0; n < 3; ++n) s += L[n] * comp(cols[n], i) * comp(cols[n], j);
        return s;
    };
    const Vec3 m = r.vec(-0.3f, 0.3f);
    const float iso = r.uni(0.3f, 1.0f);
    const float a11 = A(0, 0), a22 = A(1, 1), a33 = A(2, 2), a12 = A(0, 1), a13 = A(0, 2), a23 = A(1, 2);
    const float bx = -2.0f * (a11 * m.x + 0.5f * a12 * m.y + 0.5f * a13 * m.z);
    const float by = -2.0f * (a22 * m.y + 0.5f * a12 * m.x + 0.5f * a23 * m.z);
    const float bz = -2.0f * (a33 * m.z + 0.5f * a13 * m.x + 0.5f * a23 * m.y);
    const float mAm = a11 * m.x * m.x + a22 * m.y * m.y + a33 * m.z * m.z + a12 * m.x * m.y + a13 * m.x * m.z +
                      a23 * m.y * m.z;
    return PrimitiveParams::quadric({a11, a22, a33, a12, a13, a23, bx, by, bz, mAm - iso}, tf);
}

PrimitiveParams any_primitive(Rng& r, float range) {
    const Vec3 pos = r.vec(-range, range);
    const Transform tf{pos, r.rot()};
    const int kind = static_cast<int>(r.uni(0.0f, 1.0f) * 6.0f);
    const float s = r.uni(0.3f, 1.0f);
    switch (kind) {
        case 0: return PrimitiveParams::sphere(s, tf);
        case 1: return PrimitiveParams::ellipsoid(Vec3{s, 0.6f * s + 0.2f, 0.8f * s}, tf);
        case 2: return PrimitiveParams::torus(s, 0.4f * s, tf);
        case 3: return PrimitiveParams::box(Vec3{s, 0.7f * s, 0.5f * s + 0.1f}, tf);
        case 4: return PrimitiveParams::sphere_cone(s, 0.5f * s, 1.2f * s, tf);
        default: return random_quadric(r, tf);
    }
}

// ---------------------------------------------------------------- configs

// C1: 10 primitives, spheres + capsules, compact union + difference, 512^2
NodePtr build_c1(uint32_t seed) {
    Rng r(seed ? seed : 1u);
    NodePtr comb;
    for (int i = 0; i < 8; ++i) {
        const Vec3 pos = r.vec(-1.2f, 1.2f);
        NodePtr leaf;
        if (i % 2 == 0) {
            leaf = prim(PrimitiveParams::sphere(i % 4 == 0 ? 0.6f : 0.5f, Transform{pos, Quat{}}));
        } else {
            const Quat q = r.rot();
            leaf = prim(PrimitiveParams::sphere_cone(0.3f, 0.3f, 1.0f, Transform{pos, q}));
        }
        comb = comb ? op(cunion(0.3f, 0.3f), std::move(comb), std::move(leaf)) : std::move(leaf);
    }
    const Vec3 p0 = r.vec(-1.2f, 1.2f);
    const Vec3 p1 = r.vec(-1.2f, 1.2f);
    const Quat q1 = r.rot();
    NodePtr cut = op(cunion(0.2f, 0.2f), prim(PrimitiveParams::sphere(0.4f, Transform{p0, Quat{}})),
                     prim(PrimitiveParams::sphere_cone(0.25f, 0.25f, 0.8f, Transform{p1, q1})));
    return op(cdiff(0.2f, 0.2f), std::move(comb), std::move(cut));
}

// C2: astronaut-scale character, 142 primitives: 11 compact-union clusters
// of 10 (110), 12 compact-intersect lens pairs (24), 8 compact-diff carvings.
NodePtr build_c2(uint32_t seed) {
    Rng r(seed ? seed : 2u);
    // body layout (x, y, z, spread): torso, pelvis, head, 2 upper arms,
    // 2 forearms, 2 thighs, 2 shins
    const float parts[11][4] = {{0.0f, 0.6f, 0.0f, 0.55f},   {0.0f, -0.3f, 0.0f, 0.45f}, {0.0f, 1.75f, 0.0f, 0.35f},
                                {-0.85f, 0.9f, 0.0f, 0.3f},  {0.85f, 0.9f, 0.0f, 0.3f},  {-1.25f, 0.1f, 0.1f, 0.28f},
                                {1.25f, 0.1f, 0.1f, 0.28f},  {-0.35f, -1.2f, 0.0f, 0.32f}, {0.35f, -1.2f, 0.0f, 0.32f},
                                {-0.4f, -2.1f, 0.05f, 0.3f}, {0.4f, -2.1f, 0.05f, 0.3f}};
    std::vector<NodePtr> pieces;
    for (int c = 0; c < 11; ++c) {
        const Vec3 center{parts[c][0], parts[c][1], parts[c][2]};
        const float spread = parts[c][3];
        const float k = r.uni(0.1f, 0.3f);
        NodePtr acc;
        for (int i = 0; i < 10; ++i) {
            const Vec3 off = r.vec(-spread, spread);
            const Quat q = r.rot();
            const float s = r.uni(0.18f, 0.34f);
            const int kind = i % 4;
            const Transform tf{center + off, q};
            PrimitiveParams p = kind == 0   ? PrimitiveParams::sphere(s, tf)
                                : kind == 1 ? PrimitiveParams::ellipsoid(Vec3{s, 0.7f * s, 0.9f * s}, tf)
                                : kind == 2 ? PrimitiveParams::sphere_cone(s, 0.6f * s, 1.5f * s, tf)
                                            : PrimitiveParams::box(Vec3{0.8f * s, 0.6f * s, 0.7f * s}, tf);
            acc = acc ? op(cunion(k, k), std::move(acc), prim(p)) : prim(p);
        }
        if (c < 8) {  // carving: subtract a small sphere near the cluster surface
            const Vec3 off = r.vec(-spread, spread);
            const float s = r.uni(0.12f, 0.2f);
            acc = op(cdiff(0.08f, 0.08f), std::move(acc),
                     prim(PrimitiveParams::sphere(s, Transform{center + off + Vec3{0, 0, -0.25f}, Quat{}})));
        }
        pieces.push_back(std::move(acc));
    }
    for (int i = 0; i < 12; ++i) {  // lens pairs (visor, buttons, joints)
        const int host = i % 11;
        const Vec3 center{parts[host][0], parts[host][1], parts[host][2] - 0.35f};
        const Vec3 off = r.vec(-0.25f, 0.25f);
        const float s = r.uni(0.18f, 0.28f);
        const Vec3 a = center + off + Vec3{-0.6f * s, 0, 0};
        const Vec3 b = center + off + Vec3{0.6f * s, 0, 0};
        pieces.push_back(op(cinter(0.05f, 0.05f), prim(PrimitiveParams::sphere(s, Transform{a, Quat{}})),
                            prim(PrimitiveParams::sphere(s, Transform{b, Quat{}}))));
    }
    NodePtr root;
    for (auto& p : pieces) root = root ? op(sunion(), std::move(root), std::move(p)) : std::move(p);
    return root;
}

// C3/C4: lattice of 4-primitive compact-union cells (k = d = 0.21) merged by
// a left comb of sharp unions (generate_synthetic's structure, 4 per cell)
NodePtr build_cells(uint32_t cells, uint32_t seed, float& diagOut) {
    Rng r(seed ? seed : 3u);
    uint32_t nx = 1, ny = 1, nz = 1;
    while (nx * ny * nz < cells) {
        if (nx <= ny && nx <= nz) ++nx;
        else if (ny <= nz) ++ny;
        else ++nz;
    }
    const float cell = 2.0f, scale = 0.42f;
    const Vec3 origin{-0.5f * cell * (nx - 1), -0.5f * cell * (ny - 1), -0.5f * cell * (nz - 1)};
    NodePtr root;
    uint32_t placed = 0;
    for (uint32_t z = 0; z < nz && placed < cells; ++z)
        for (uint32_t y = 0; y < ny && placed < cells; ++y)
            for (uint32_t x = 0; x < nx && placed < cells; ++x, ++placed) {
                const Vec3 center = origin + Vec3{cell * x, cell * y, cell * z};
                NodePtr sub = prim(cell_primitive(r, center, scale));
                for (int i = 1; i < 4; ++i) {
                    NodePtr next = prim(cell_primitive(r, center, scale));
                    sub = op(cunion(0.5f * scale, 0.5f * scale), std::move(sub), std::move(next));
                }
                root = root ? op(sunion(), std::move(root), std::move(sub)) : std::move(sub);
            }
    const float sx = cell * nx, sy = cell * ny, sz = cell * nz;
    diagOut = std::sqrt(sx * sx + sy * sy + sz * sz);
    return root;
}

// quad:N -- N lattice cells of 4 primitives, two of them random positive
// definite quadrics, joined by compact unions (k = d = 0.21); every 5th cell
// is carved by a compact difference with a quadric.  Cells merge by a left
// comb of sharp unions.  Puts quadrics (the costliest primitive) on every
// path of the tolerance-path parity tests at frame scale.
NodePtr build_quads(uint32_t cells, uint32_t seed, float& diagOut) {
    Rng r(seed ? seed : 11u);
    uint32_t nx = 1, ny = 1, nz = 1;
    while (nx * ny * nz < cells) {
        if (nx <= ny && nx <= nz) ++nx;
        else if (ny <= nz) ++ny;
        else ++nz;
    }
    const float cell = 2.0f, scale = 0.42f;
    const Vec3 origin{-0.5f * cell * (nx - 1), -0.5f * cell * (ny - 1), -0.5f * cell * (nz - 1)};
    NodePtr root;
    uint32_t placed = 0;
    for (uint32_t z = 0; z < nz && placed < cells; ++z)
        for (uint32_t y = 0; y < ny && placed < cells; ++y)
            for (uint32_t x = 0; x < nx && placed < cells; ++x, ++placed) {
                const Vec3 center = origin + Vec3{cell * x, cell * y, cell * z};
                NodePtr sub;
                for (int i = 0; i < 4; ++i) {
                    PrimitiveParams pp = (i % 2 == 0)
                                             ? random_quadric(r, Transform{center + r.vec(-0.3f, 0.3f), r.rot()})
                                             : cell_primitive(r, center, scale);
                    NodePtr next = prim(pp);
                    sub = sub ? op(cunion(0.5f * scale, 0.5f * scale), std::move(sub), std::move(next))
                              : std::move(next);
                }
                if (placed % 5 == 4)
                    sub = op(cdiff(0.1f, 0.1f), std::move(sub),
                             prim(random_quadric(r, Transform{center + Vec3{0.0f, 0.0f, -0.6f}, r.rot()})));
                root = root ? op(sunion(), std::move(root), std::move(sub)) : std::move(sub);
            }
    const float sx = cell * nx, sy = cell * ny, sz = cell * nz;
    diagOut = std::sqrt(sx * sx + sy * sy + sz * sz);
    return root;
}

// C5: 4,000 primitives, left-heavy spine of 64 groups (depth ~70), each a
// balanced compact-union tree (k = d = 0.08) with 25% compact-intersect
// pairs (k = d = 0.05); every 9th spine operator is a compact difference.
NodePtr balanced(std::vector<NodePtr>& units, size_t lo, size_t hi) {
    if (hi - lo == 1) return std::move(units[lo]);
    const size_t mid = (lo + hi + 1) / 2;
    NodePtr l = balanced(units, lo, mid);
    NodePtr rr = balanced(units, mid, hi);
    return op(cunion(0.08f, 0.08f), std::move(l), std::move(rr));
}

NodePtr build_c5(uint32_t seed) {
    Rng r(seed ? seed : 5u);
    NodePtr spine;
    for (int g = 0; g < 64; ++g) {
        const int prims = g < 32 ? 63 : 62;
        const Vec3 gc{0.9f * (g % 8) - 3.15f, 0.9f * (g / 8) - 3.15f, 0.0f};
        std::vector<NodePtr> units;
        int placed = 0;
        int u = 0;
        while (placed < prims) {
            const bool pair = (u % 4 == 3) && (prims - placed >= 2);
            const Vec3 off = r.vec(-0.45f, 0.45f);
            const float s = r.uni(0.1f, 0.2f);
            if (pair) {
                const Vec3 d = r.vec(-0.08f, 0.08f);
                units.push_back(op(cinter(0.05f, 0.05f),
                                   prim(PrimitiveParams::sphere(s, Transform{gc + off, Quat{}})),
                                   prim(PrimitiveParams::sphere(s, Transform{gc + off + d, Quat{}}))));
                placed += 2;
            } else {
                const Quat q = r.rot();
                const Transform tf{gc + off, q};
                units.push_back(prim(u % 2 ? PrimitiveParams::box(Vec3{s, 0.8f * s, 0.6f * s}, tf)
                                           : PrimitiveParams::sphere(s, tf)));
                placed += 1;
            }
            ++u;
        }
        NodePtr group = balanced(units, 0, units.size());
        if (!spine) {
            spine = std::move(group);
            continue;
        }
        const OperatorParams sop = (g % 9 == 0) ? cdiff(0.1f, 0.1f) : cunion(0.1f, 0.1f);
        spine = op(sop, std::move(spine), std::move(group));
    }
    return spine;
}

void collect_prims(const SceneNode& n, std::vector<PrimitiveParams>& out) {
    if (n.isPrimitive) {
        out.push_back(n.primitive);
        return;
    }
    collect_prims(*n.left, out);
    collect_prims(*n.right, out);
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    size_t b = 0;
    for (size_t i = 0; i <= s.size(); ++i)
        if (i == s.size() || s[i] == sep) {
            out.push_back(s.substr(b, i - b));
            b = i + 1;
        }
    return out;
}

}  // namespace

std::unique_ptr<Scene> build(const std::string& name, uint32_t seed, int width, int height) {
    auto sc = std::make_unique<Scene>();
    sc->name = name;
    NodePtr root;
    const Vec3 origin{0, 0, 0};
    if (name == "C1") {
        root = build_c1(seed);
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 512, 512);
    } else if (name == "C2") {
        root = build_c2(seed);
        sc->camera = look_at(Vec3{0.0f, 0.0f, -7.5f}, Vec3{0.0f, -0.15f, 0.0f}, 0.1f, 40.0f, 1920, 1080);
    } else if (name == "C3" || name == "C4") {
        float diag = 0.0f;
        root = build_cells(name == "C3" ? 250u : 2500u, seed, diag);
        const Vec3 dir = normalize(Vec3{0.9f, 0.55f, -1.25f});
        const float dist = 0.6f * (1.35f * diag + 1.0f);
        sc->camera = look_at(dir * dist, origin, 0.1f, 3.0f * diag + 4.0f, name == "C3" ? 1920 : 3840,
                             name == "C3" ? 1080 : 2160);
    } else if (name == "C5") {
        root = build_c5(seed);
        sc->camera = look_at(Vec3{0, 0, -11}, origin, 0.1f, 40.0f, 1920, 1080);
    } else if (name == "sphere") {
        root = prim(PrimitiveParams::sphere(1.0f));
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 128, 128);
    } else if (name == "csg") {  // test_tracer.cpp "pipeline matches oracle on a csg scene"
        root = op(cdiff(0.3f, 0.3f),
                  op(cunion(0.4f, 0.4f), prim(PrimitiveParams::sphere(1.0f, Transform{{-0.7f, 0, 0}, Quat{}})),
                     prim(PrimitiveParams::box({0.8f, 0.6f, 0.6f}, Transform{{0.8f, 0, 0}, Quat{}}))),
                  prim(PrimitiveParams::sphere(0.7f, Transform{{0, 0.6f, -0.8f}, Quat{}})));
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 128, 128);
    } else if (name == "slab") {
        root = prim(PrimitiveParams::box({6, 6, 0.5f}));
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 128, 128);
    } else if (name == "comb_error") {  // test_tracer.cpp "tile errors mark the tile"
        root = prim(PrimitiveParams::sphere(2.0f));
        for (int i = 0; i < 24; ++i)
            root = op(sunion(), prim(PrimitiveParams::sphere(2.0f + 0.01f * i)), std::move(root));
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 64, 64);
    } else if (name.rfind("gen:", 0) == 0) {
        const auto f = split(name, ':');
        if (f.size() != 5) throw std::invalid_argument("gen:<preset>:<n>:<kind>:<blend>");
        SceneDocument doc = generate_synthetic(f[1], static_cast<uint32_t>(std::stoul(f[2])), f[3], f[4], seed);
        root = std::move(doc.root);
        sc->camera = doc.camera;
    } else if (name.rfind("stack:", 0) == 0) {  // n nearly concentric spheres, balanced compact unions:
        // every tile on the silhouette sees n overlapping fragments (overlap saturation, view overflow)
        const uint32_t n = static_cast<uint32_t>(std::stoul(name.substr(6)));
        if (n == 0) throw std::invalid_argument("stack:<n> needs n >= 1");
        std::vector<NodePtr> units;
        for (uint32_t i = 0; i < n; ++i)
            units.push_back(prim(PrimitiveParams::sphere(1.0f + 0.002f * i, Transform{{0.001f * i, 0, 0}, Quat{}})));
        root = balanced(units, 0, units.size());
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 64, 64);
    } else if (name.rfind("quad:", 0) == 0) {
        const uint32_t n = static_cast<uint32_t>(std::stoul(name.substr(5)));
        if (n == 0) throw std::invalid_argument("quad:<cells> needs cells >= 1");
        float diag = 0.0f;
        root = build_quads(n, seed, diag);
        const Vec3 dir = normalize(Vec3{0.9f, 0.55f, -1.25f});
        const float dist = 0.6f * (1.35f * diag + 1.0f);
        sc->camera = look_at(dir * dist, origin, 0.1f, 3.0f * diag + 4.0f, 1920, 1080);
    } else if (name.rfind("random:", 0) == 0) {
        const uint32_t n = static_cast<uint32_t>(std::stoul(name.substr(7)));
        Rng r(seed ? seed : 7u);
        for (uint32_t i = 0; i < n; ++i) {
            NodePtr leaf = prim(any_primitive(r, 2.0f));
            root = root ? op(sunion(), std::move(root), std::move(leaf)) : std::move(leaf);
        }
        sc->camera = look_at(Vec3{0, 0, -6}, origin, 0.1f, 40.0f, 96, 96);
    } else {
        throw std::invalid_argument("unknown scene '" + name + "'");
    }
    if (width > 0) sc->camera.width = width;
    if (height > 0) sc->camera.height = height;
    sc->tree = compile(*root);
    compute_fast_indices(sc->tree);
    collect_prims(*root, sc->base);
    return sc;
}

PrimitiveParams perturbed(const PrimitiveParams& base, uint32_t frame, uint32_t i) {
    PrimitiveParams p = base;
    const float f = static_cast<float>(frame), fi = static_cast<float>(i);
    const Vec3 d{std::sin(0.7f * f + fi), std::cos(1.3f * f + 2.0f * fi), std::sin(0.9f * f + 3.0f * fi)};
    p.frame.translate = base.frame.translate + d * 0.05f;
    return p;
}

}  // namespace scenes

// ======================================================================== C accessors

#ifndef SCENE_PREFIX
#define SCENE_PREFIX sc_
#endif
#define SC_CAT2(a, b) a##b
#define SC_CAT(a, b) SC_CAT2(a, b)
#define SC_FN(name) SC_CAT(SCENE_PREFIX, name)

namespace {
thread_local std::string g_sceneError;
}

extern "C" {

__attribute__((visibility("default"))) const char* SC_FN(scene_error)(void) { return g_sceneError.c_str(); }

__attribute__((visibility("default"))) void* SC_FN(scene_new)(const char* name, uint32_t seed, int width, int height) {
    try {
        return scenes::build(name, seed, width, height).release();
    } catch (const std::exception& e) {
        g_sceneError = e.what();
        return nullptr;
    }
}

__attribute__((visibility("default"))) void SC_FN(scene_free)(void* h) { delete static_cast<scenes::Scene*>(h); }

__attribute__((visibility("default"))) void SC_FN(scene_info)(void* h, uint32_t* nwords, uint32_t* nnodes,
                                                              uint32_t* nprims, uint32_t* rootWord, int32_t* width,
                                                              int32_t* height) {
    const auto* s = static_cast<scenes::Scene*>(h);
    *nwords = s->tree.word_count();
    *nnodes = s->tree.node_count();
    *nprims = static_cast<uint32_t>(s->tree.primitiveWords.size());
    *rootWord = s->tree.rootWord;
    *width = s->camera.width;
    *height = s->camera.height;
}

__attribute__((visibility("default"))) void SC_FN(scene_tree)(void* h, float* data, bt_node* nodes, uint32_t* prims) {
    const auto* s = static_cast<scenes::Scene*>(h);
    std::memcpy(data, s->tree.data.data(), s->tree.data.size() * sizeof(float));
    for (size_t i = 0; i < s->tree.nodes.size(); ++i) {
        const auto& n = s->tree.nodes[i];
        bt_node& o = nodes[i];
        std::memset(&o, 0, sizeof(o));
        o.word = n.word;
        o.parentWord = n.parentWord;
        o.leftChild = n.leftChild;
        o.rightChild = n.rightChild;
        o.isPrimitive = n.isPrimitive ? 1 : 0;
        o.nodeOp = n.nodeOp;
    }
    std::memcpy(prims, s->tree.primitiveWords.data(), s->tree.primitiveWords.size() * sizeof(uint32_t));
}

// Camera as 14 floats: position[3] target[3] up[3] fov near far width height
__attribute__((visibility("default"))) void SC_FN(scene_camera)(void* h, float* out) {
    const auto& c = static_cast<scenes::Scene*>(h)->camera;
    const float v[14] = {c.position.x, c.position.y, c.position.z, c.target.x, c.target.y,
                         c.target.z,   c.up.x,       c.up.y,       c.up.z,     c.fovDegrees,
                         c.nearZ,      c.farZ,       (float)c.width, (float)c.height};
    std::memcpy(out, v, sizeof(v));
}

// Replace the camera (same 14 floats as scene_camera); validated like every
// camera.  Edge-case tests: cameras looking away from the scene, inside its
// volumes, with the scene beyond the far plane, sub-tile images.
__attribute__((visibility("default"))) int SC_FN(scene_set_camera)(void* h, const float* v) {
    blobtree::Camera c;
    c.position = blobtree::Vec3{v[0], v[1], v[2]};
    c.target = blobtree::Vec3{v[3], v[4], v[5]};
    c.up = blobtree::Vec3{v[6], v[7], v[8]};
    c.fovDegrees = v[9];
    c.nearZ = v[10];
    c.farZ = v[11];
    c.width = static_cast<int>(v[12]);
    c.height = static_cast<int>(v[13]);
    try {
        blobtree::validate_camera(c);
    } catch (const std::exception& e) {
        g_sceneError = e.what();
        return -1;
    }
    static_cast<scenes::Scene*>(h)->camera = c;
    return 0;
}

// Apply frame `frame` of the C3/C4 perturbation to the scene's own tree and
// emit the parameter deltas (stride 17 floats) for bt_params_update.
__attribute__((visibility("default"))) uint32_t SC_FN(scene_perturb)(void* h, uint32_t frame, uint32_t* words,
                                                                     float* params, uint32_t* counts) {
    auto* s = static_cast<scenes::Scene*>(h);
    const uint32_t n = static_cast<uint32_t>(s->base.size());
    for (uint32_t i = 0; i < n; ++i) {
        const blobtree::PrimitiveParams p = scenes::perturbed(s->base[i], frame, i);
        const uint32_t w = s->tree.primitiveWords[i];
        blobtree::update_primitive_params(s->tree, w, p);
        const uint32_t cnt = blobtree::kTransformFloatCount + blobtree::shape_float_count(p.kind);
        if (words) words[i] = w;
        if (counts) counts[i] = cnt;
        if (params) std::memcpy(params + (size_t)i * 17, s->tree.params_at(w), cnt * sizeof(float));
    }
    return n;
}

#ifdef SCENE_PRODUCT
// Device camera constants from this library's CameraFrame (host tan etc.).
__attribute__((visibility("default"))) void SC_FN(scene_device_camera)(void* h, bt_camera* out) {
    *out = blobtree::to_device_camera(blobtree::CameraFrame(static_cast<scenes::Scene*>(h)->camera));
}
#endif

}  // extern "C"
