// host/tracer.cpp -- stage (c) entry points of the drop-in API.
//
// render_tiles, oracle_render and compute_normals run on the GPU
// (csrc/k_trace.cu) with IEEE-exact arithmetic and download the result into
// the reference's GBuffer layout.  fetch_interval stays a host helper with
// the reference's semantics (src/tracer.cpp:50-103).
#include "blobtree/tracer.hpp"

#include <algorithm>
#include <cstdlib>
#include <thread>

#include "blobtree/device.hpp"

namespace blobtree {

void validate_config(const RenderConfig& cfg) {
    if (!(cfg.relax >= 1.0f && cfg.relax < 2.0f)) throw std::invalid_argument("relaxation factor must lie in [1, 2)");
    if (!(cfg.lipschitz >= 1.0f)) throw std::invalid_argument("lipschitz bound must be at least 1");
    if (!(cfg.minStep > 0.0f)) throw std::invalid_argument("min step must be > 0");
    if (!(cfg.hitEpsilon > 0.0f)) throw std::invalid_argument("hit epsilon must be > 0");
    if (cfg.maxOverlap < 1 || cfg.maxOverlap > kMaxOverlapLimit)
        throw std::invalid_argument("max overlap must lie in [1, 96]");
}

void GBuffer::init(int w, int h) {
    width = w;
    height = h;
    tilesX = (w + kTileSize - 1) / kTileSize;
    tilesY = (h + kTileSize - 1) / kTileSize;
    const size_t px = static_cast<size_t>(w) * h, tiles = static_cast<size_t>(tilesX) * tilesY;
    hit.assign(px, 0);
    depth.assign(px, 0.0f);
    normal.assign(px, Vec3{});
    evalCount.assign(px, 0);
    tileMaxOverlap.assign(tiles, 0);
    tileCacheBytes.assign(tiles, 0);
    tileError.assign(tiles, 0);
}

uint32_t resolve_thread_count(uint32_t requested) {
    if (requested) return requested;
    if (const char* env = std::getenv("BLOBTREE_THREADS")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v > 0) return static_cast<uint32_t>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1u;
}

std::optional<FetchInterval> fetch_interval(TileFetchState& st, const CameraFrame& frame, const RenderConfig& cfg) {
    const size_t before = st.actives.size();
    const float prevEnd = st.zEnd;
    std::erase_if(st.actives, [prevEnd](const ActiveFragment& a) { return a.zExit <= prevEnd; });
    const bool expired = st.actives.size() != before;
    const size_t n = st.list.size();
    if (st.actives.empty() && st.cursor >= n) return std::nullopt;

    const float zBegin = st.cursor < n ? std::max(prevEnd, st.list[st.cursor].zEntry) : prevEnd;
    float window = cfg.fetchWindow;
    if (!(window > 0.0f)) window = (frame.camera().farZ - frame.camera().nearZ) / 20.0f;
    const float beginView = frame.view_z_from_ndc(zBegin);
    float maxExit = -kFieldInfinity;
    for (const auto& a : st.actives) maxExit = std::max(maxExit, a.zExit);

    uint32_t fetched = 0;
    for (; st.cursor < n; ++st.cursor, ++fetched) {
        const Fragment& f = st.list[st.cursor];
        if (!st.actives.empty()) {
            const bool gap = f.zEntry > maxExit;
            const bool budget = fetched >= cfg.maxNewPerFetch;
            const bool full = st.actives.size() >= cfg.maxOverlap;
            const bool far = frame.view_z_from_ndc(f.zEntry) - beginView >= window;
            if (gap || budget || full || far) break;
        }
        auto at = std::lower_bound(st.actives.begin(), st.actives.end(), f.primitiveWord,
                                   [](const ActiveFragment& a, uint32_t w) { return a.word < w; });
        st.actives.insert(at, ActiveFragment{f.primitiveWord, f.zEntry, f.zExit});
        maxExit = std::max(maxExit, f.zExit);
    }

    float zEnd = st.cursor < n ? std::min(st.list[st.cursor].zEntry, maxExit) : maxExit;
    if (zEnd <= zBegin && fetched == 0 && !expired) {
        // saturated with nothing expiring: advance to the earliest exit
        zEnd = kFieldInfinity;
        for (const auto& a : st.actives) zEnd = std::min(zEnd, a.zExit);
    }
    st.zEnd = zEnd;
    return FetchInterval{zBegin, zEnd};
}

// ---------------------------------------------------------------- GPU entry points

namespace {

void upload_tree(bt_ctx* ctx, const LinearTree& tree) {
    check_device(bt_tree_upload(ctx, tree.data.data(), tree.word_count(),
                                reinterpret_cast<const bt_node*>(tree.nodes.data()), tree.node_count(),
                                tree.primitiveWords.data(), static_cast<uint32_t>(tree.primitiveWords.size()),
                                tree.rootWord),
                 "bt_tree_upload");
}

GBuffer download_gbuffer(bt_ctx* ctx, int w, int h) {
    GBuffer g;
    g.init(w, h);
    check_device(bt_gbuffer_download(ctx, g.hit.data(), g.depth.data(), reinterpret_cast<float*>(g.normal.data()),
                                     g.evalCount.data(), g.tileMaxOverlap.data(), g.tileCacheBytes.data(),
                                     g.tileError.data()),
                 "bt_gbuffer_download");
    return g;
}

RenderStats download_stats(bt_ctx* ctx) {
    bt_stats s;
    check_device(bt_stats_download(ctx, &s), "bt_stats_download");
    RenderStats r;
    r.fieldEvals = s.fieldEvals;
    r.retainedNodeVisits = s.retainedNodeVisits;
    r.primitiveEvals = s.primitiveEvals;
    r.treeNodeCount = s.treeNodeCount;
    r.maxOverlap = s.maxOverlap;
    r.maxCacheBytes = s.maxCacheBytes;
    return r;
}

}  // namespace

GBuffer render_tiles(const LinearTree& tree, const TileABuffer& abuffer, const CameraFrame& frame,
                     const RenderConfig& cfg, RenderStats* stats) {
    validate_config(cfg);
    const Camera& cam = frame.camera();
    if (abuffer.tilesX != frame.tiles_x() || abuffer.tilesY != frame.tiles_y())
        throw std::invalid_argument("A-buffer tiling differs from the camera's");
    ContextLease ctx;
    upload_tree(ctx, tree);
    const size_t tiles = abuffer.tiles.size();
    std::vector<uint32_t> offsets(tiles + 1, 0);
    for (size_t t = 0; t < tiles; ++t) offsets[t + 1] = offsets[t] + static_cast<uint32_t>(abuffer.tiles[t].size());
    std::vector<bt_fragment> frags;
    frags.reserve(offsets[tiles]);
    for (const auto& list : abuffer.tiles)
        for (const Fragment& f : list) frags.push_back(bt_fragment{f.primitiveWord, f.zEntry, f.zExit});
    const bt_camera dcam = to_device_camera(frame);
    const bt_render_config dcfg = to_device_config(cfg);
    check_device(bt_abuffer_upload(ctx, &dcam, offsets.data(), frags.data()), "bt_abuffer_upload");
    check_device(bt_stats_reset(ctx), "bt_stats_reset");
    check_device(bt_trace(ctx, &dcam, &dcfg, 0, 0, 1), "bt_trace");
    GBuffer g = download_gbuffer(ctx, cam.width, cam.height);
    if (stats) *stats = download_stats(ctx);
    return g;
}

GBuffer oracle_render(const LinearTree& tree, const CameraFrame& frame, const RenderConfig& cfg, RenderStats* stats) {
    validate_config(cfg);
    const Camera& cam = frame.camera();
    ContextLease ctx;
    upload_tree(ctx, tree);
    const bt_camera dcam = to_device_camera(frame);
    const bt_render_config dcfg = to_device_config(cfg);
    check_device(bt_stats_reset(ctx), "bt_stats_reset");
    check_device(bt_oracle_render(ctx, &dcam, &dcfg, 1), "bt_oracle_render");
    GBuffer g = download_gbuffer(ctx, cam.width, cam.height);
    if (stats) {
        *stats = download_stats(ctx);
        stats->maxOverlap = 0;
        stats->maxCacheBytes = 0;
    }
    return g;
}

void compute_normals(const LinearTree& tree, GBuffer& g, const CameraFrame& frame, RenderConfig::NormalsMode mode) {
    const Camera& cam = frame.camera();
    if (g.width != cam.width || g.height != cam.height)
        throw std::invalid_argument("G-buffer size differs from the camera's");
    ContextLease ctx;
    upload_tree(ctx, tree);
    const bt_camera dcam = to_device_camera(frame);
    check_device(bt_gbuffer_upload(ctx, &dcam, g.hit.data(), g.depth.data()), "bt_gbuffer_upload");
    check_device(bt_normals(ctx, &dcam, mode == RenderConfig::NormalsMode::CentralDifference ? 1 : 0, 1),
                 "bt_normals");
    check_device(bt_gbuffer_download(ctx, nullptr, nullptr, reinterpret_cast<float*>(g.normal.data()), nullptr,
                                     nullptr, nullptr, nullptr),
                 "bt_gbuffer_download");
}

}  // namespace blobtree
