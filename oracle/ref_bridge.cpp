// ref_bridge.cpp -- extern "C" bridge over the UNMODIFIED reference library
// (test infrastructure; CPU checker only).
//
// Compiled by oracle/Makefile together with the reference sources under
// /root/reference/proj/src and -Dblobtree=blobtree_ref, so every
// `blobtree::` below resolves to the reference's own implementation.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load this library.
//
// Stage functions follow the reference's canonical per-frame composition
// (proj/tests/test_tracer.cpp:25-31, pipeline_render):
//   propagate_roi -> build_volumes_of_interest(margin = cfg.hitEpsilon)
//   -> rasterize_volumes -> render_tiles -> compute_normals.
#include <chrono>
#include <cstring>

#include "../include/bt_cuda.h"
#include "../paper_2304_09673_b200/csrc/scenes/scenes.hpp"
#include "blobtree/abuffer.hpp"
#include "blobtree/image_io.hpp"
#include "blobtree/tracer.hpp"

using namespace blobtree;

namespace {

thread_local std::string g_err;

RenderConfig to_cfg(const bt_render_config* c, uint32_t threads) {
    RenderConfig r;
    r.lipschitz = c->lipschitz;
    r.relax = c->relax;
    r.minStep = c->minStep;
    r.hitEpsilon = c->hitEpsilon;
    r.maxOverlap = c->maxOverlap;
    r.maxNewPerFetch = c->maxNewPerFetch;
    r.fetchWindow = c->fetchWindow;
    r.normalsMode = c->normalsMode ? RenderConfig::NormalsMode::CentralDifference
                                   : RenderConfig::NormalsMode::DepthDifferential;
    r.threads = threads;
    return r;
}

void to_voi(const VolumeOfInterest& v, bt_voi& o) {
    std::memset(&o, 0, sizeof(o));
    o.family = static_cast<uint8_t>(v.family);
    o.primitiveWord = v.primitiveWord;
    o.center[0] = v.center.x;
    o.center[1] = v.center.y;
    o.center[2] = v.center.z;
    o.radius = v.radius;
    o.halfExtents[0] = v.halfExtents.x;
    o.halfExtents[1] = v.halfExtents.y;
    o.halfExtents[2] = v.halfExtents.z;
    o.rotation[0] = v.rotation.w;
    o.rotation[1] = v.rotation.x;
    o.rotation[2] = v.rotation.y;
    o.rotation[3] = v.rotation.z;
    o.axisEnd[0] = v.axisEnd.x;
    o.axisEnd[1] = v.axisEnd.y;
    o.axisEnd[2] = v.axisEnd.z;
}

VolumeOfInterest from_voi(const bt_voi& o) {
    VolumeOfInterest v;
    v.family = static_cast<VolumeOfInterest::Family>(o.family);
    v.primitiveWord = o.primitiveWord;
    v.center = Vec3{o.center[0], o.center[1], o.center[2]};
    v.radius = o.radius;
    v.halfExtents = Vec3{o.halfExtents[0], o.halfExtents[1], o.halfExtents[2]};
    v.rotation = Quat{o.rotation[0], o.rotation[1], o.rotation[2], o.rotation[3]};
    v.axisEnd = Vec3{o.axisEnd[0], o.axisEnd[1], o.axisEnd[2]};
    return v;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int flatten(const TileABuffer& ab, uint32_t* offsets, bt_fragment* frags, uint64_t cap, uint64_t* total) {
    uint64_t n = 0;
    for (size_t t = 0; t < ab.tiles.size(); ++t) {
        if (offsets) offsets[t] = static_cast<uint32_t>(n);
        for (const Fragment& f : ab.tiles[t]) {
            if (frags) {
                if (n >= cap) return 1;
                frags[n] = bt_fragment{f.primitiveWord, f.zEntry, f.zExit};
            }
            ++n;
        }
    }
    if (offsets) offsets[ab.tiles.size()] = static_cast<uint32_t>(n);
    if (total) *total = n;
    return 0;
}

TileABuffer unflatten(const CameraFrame& frame, const uint32_t* offsets, const bt_fragment* frags) {
    TileABuffer ab;
    ab.tilesX = frame.tiles_x();
    ab.tilesY = frame.tiles_y();
    ab.tiles.resize(static_cast<size_t>(ab.tilesX) * ab.tilesY);
    for (size_t t = 0; t < ab.tiles.size(); ++t)
        for (uint32_t i = offsets[t]; i < offsets[t + 1]; ++i)
            ab.tiles[t].push_back(Fragment{frags[i].primitiveWord, frags[i].zEntry, frags[i].zExit});
    return ab;
}

void write_gbuffer_out(const GBuffer& g, uint8_t* hit, float* depth, float* normal, uint32_t* evalCount,
                       uint32_t* tmo, uint32_t* tcb, uint8_t* te) {
    const size_t px = g.hit.size(), tiles = g.tileError.size();
    if (hit) std::memcpy(hit, g.hit.data(), px);
    if (depth) std::memcpy(depth, g.depth.data(), px * 4);
    if (normal) std::memcpy(normal, g.normal.data(), px * 12);
    if (evalCount) std::memcpy(evalCount, g.evalCount.data(), px * 4);
    if (tmo) std::memcpy(tmo, g.tileMaxOverlap.data(), tiles * 4);
    if (tcb) std::memcpy(tcb, g.tileCacheBytes.data(), tiles * 4);
    if (te) std::memcpy(te, g.tileError.data(), tiles);
}

void write_stats(const RenderStats& s, uint64_t* out) {
    if (!out) return;
    out[0] = s.fieldEvals;
    out[1] = s.retainedNodeVisits;
    out[2] = s.primitiveEvals;
    out[3] = s.treeNodeCount;
    out[4] = s.maxOverlap;
    out[5] = s.maxCacheBytes;
}

scenes::Scene* S(void* h) { return static_cast<scenes::Scene*>(h); }

}  // namespace

#define API extern "C" __attribute__((visibility("default")))

API const char* ref_error(void) { return g_err.c_str(); }

// propagate_roi (linear_tree.cpp:170-185); out: one float per node ordinal
API int ref_roi(void* h, float* out) {
    try {
        const auto roi = propagate_roi(S(h)->tree);
        std::memcpy(out, roi.data(), roi.size() * 4);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// build_volumes_of_interest(tree, propagate_roi(tree), margin)
API int ref_vois(void* h, float margin, bt_voi* out) {
    try {
        const auto& t = S(h)->tree;
        const auto v = build_volumes_of_interest(t, propagate_roi(t), margin);
        for (size_t i = 0; i < v.size(); ++i) to_voi(v[i], out[i]);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// rasterize_volumes on caller volumes (abuffer.cpp:175-225), CSR output.
// frags may be NULL to query the total first.
API int ref_rasterize(void* h, const bt_voi* vois, uint32_t n, uint32_t* offsets, bt_fragment* frags, uint64_t cap,
                      uint64_t* total, double* ms) {
    try {
        std::vector<VolumeOfInterest> v(n);
        for (uint32_t i = 0; i < n; ++i) v[i] = from_voi(vois[i]);
        const CameraFrame frame(S(h)->camera);
        const auto t0 = std::chrono::steady_clock::now();
        const TileABuffer ab = rasterize_volumes(v, frame);
        if (ms) *ms = ms_since(t0);
        return flatten(ab, offsets, frags, cap, total);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// render_tiles on a caller A-buffer (tracer.cpp:141-236), optional normals
API int ref_render_tiles(void* h, const bt_render_config* cfg, uint32_t threads, const uint32_t* offsets,
                         const bt_fragment* frags, int normals, uint8_t* hit, float* depth, float* normal,
                         uint32_t* evalCount, uint32_t* tmo, uint32_t* tcb, uint8_t* te, uint64_t* stats, double* ms) {
    try {
        const scenes::Scene& s = *S(h);
        const CameraFrame frame(s.camera);
        const RenderConfig rc = to_cfg(cfg, threads);
        const TileABuffer ab = unflatten(frame, offsets, frags);
        RenderStats st;
        auto t0 = std::chrono::steady_clock::now();
        GBuffer g = render_tiles(s.tree, ab, frame, rc, &st);
        if (ms) ms[0] = ms_since(t0);
        if (normals) {
            t0 = std::chrono::steady_clock::now();
            compute_normals(s.tree, g, frame, rc.normalsMode);
            if (ms) ms[1] = ms_since(t0);
        }
        write_gbuffer_out(g, hit, depth, normal, evalCount, tmo, tcb, te);
        write_stats(st, stats);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Whole frame through the reference: (a) roi+voi, (b) rasterize, (c) trace,
// normals.  stage_ms[4] = {roi+voi, rasterize, render_tiles, normals}.
API int ref_frame(void* h, const bt_render_config* cfg, uint32_t threads, uint8_t* hit, float* depth, float* normal,
                  uint32_t* evalCount, uint32_t* tmo, uint32_t* tcb, uint8_t* te, uint64_t* stats, double* stage_ms,
                  uint64_t* fragments) {
    try {
        const scenes::Scene& s = *S(h);
        const RenderConfig rc = to_cfg(cfg, threads);
        auto t0 = std::chrono::steady_clock::now();
        const CameraFrame frame(s.camera);
        const auto roi = propagate_roi(s.tree);
        const auto vols = build_volumes_of_interest(s.tree, roi, rc.hitEpsilon);
        if (stage_ms) stage_ms[0] = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        const TileABuffer ab = rasterize_volumes(vols, frame);
        if (stage_ms) stage_ms[1] = ms_since(t0);
        if (fragments) *fragments = ab.fragment_count();
        RenderStats st;
        t0 = std::chrono::steady_clock::now();
        GBuffer g = render_tiles(s.tree, ab, frame, rc, &st);
        if (stage_ms) stage_ms[2] = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        compute_normals(s.tree, g, frame, rc.normalsMode);
        if (stage_ms) stage_ms[3] = ms_since(t0);
        write_gbuffer_out(g, hit, depth, normal, evalCount, tmo, tcb, te);
        write_stats(st, stats);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// oracle_render (tracer.cpp:238-280): brute force over the full tree
API int ref_oracle(void* h, const bt_render_config* cfg, uint32_t threads, uint8_t* hit, float* depth,
                   uint32_t* evalCount, uint64_t* stats) {
    try {
        const scenes::Scene& s = *S(h);
        const CameraFrame frame(s.camera);
        RenderStats st;
        const GBuffer g = oracle_render(s.tree, frame, to_cfg(cfg, threads), &st);
        write_gbuffer_out(g, hit, depth, nullptr, evalCount, nullptr, nullptr, nullptr);
        write_stats(st, stats);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// compare_gbuffers (image_io.cpp:175-209) on two hit/depth planes
API int ref_compare(int w, int h, const uint8_t* hitA, const float* depthA, const uint8_t* hitB, const float* depthB,
                    float tol, double* out5) {
    GBuffer a, b;
    a.init(w, h);
    b.init(w, h);
    const size_t px = static_cast<size_t>(w) * h;
    std::memcpy(a.hit.data(), hitA, px);
    std::memcpy(b.hit.data(), hitB, px);
    std::memcpy(a.depth.data(), depthA, px * 4);
    std::memcpy(b.depth.data(), depthB, px * 4);
    const CompareReport r = compare_gbuffers(a, b, tol);
    out5[0] = r.hitAgreement;
    out5[1] = r.depthRms;
    out5[2] = r.depthMax;
    out5[3] = static_cast<double>(r.depthOutliers);
    out5[4] = static_cast<double>(r.hitMismatches);
    return 0;
}

// ---- single-point helpers for golden / property tests -------------------
API float ref_eval_primitive_raw(uint8_t kind, const float* params, float x, float y, float z) {
    return eval_primitive_raw(kind, params, Point3{x, y, z});
}
API float ref_eval_operator_raw(uint8_t code, const float* params, float f0, float f1) {
    return eval_operator_raw(code, params, f0, f1);
}
API float ref_eval_full(void* h, float x, float y, float z) { return eval_full(S(h)->tree, Point3{x, y, z}); }
