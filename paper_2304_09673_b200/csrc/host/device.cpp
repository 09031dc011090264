// host/device.cpp -- glue between the drop-in C++ API and the C-ABI:
// the process-wide default context, POD conversions, and the
// device-resident Renderer (include/blobtree/device.hpp).
#include "blobtree/device.hpp"

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

namespace blobtree {

void check_device(int rc, const char* what) {
    if (rc == BT_OK) return;
    throw DeviceError(std::string(what) + ": " + bt_last_error());
}

namespace {

int device_from_env() {
    if (const char* env = std::getenv("BLOBTREE_DEVICE")) return std::atoi(env);
    return 0;
}

struct DefaultCtx {
    bt_ctx* ctx = nullptr;
    ~DefaultCtx() {
        // intentionally leaked at exit: the CUDA runtime may already be torn down
    }
};

}  // namespace

bt_ctx* default_context() {
    static std::once_flag once;
    static DefaultCtx holder;
    static int rc = BT_OK;
    static std::string err;
    std::call_once(once, [] {
        rc = bt_ctx_create(device_from_env(), &holder.ctx);
        if (rc != BT_OK) err = bt_last_error();
    });
    if (rc != BT_OK)
        throw DeviceError("blobtree-b200 needs a CUDA device (no CPU fallback): " + err);
    return holder.ctx;
}

namespace {
std::mutex& default_context_mutex() {
    static std::mutex m;
    return m;
}
}  // namespace

ContextLease::ContextLease() : lock_(default_context_mutex()), ctx_(default_context()) {}

bt_camera to_device_camera(const CameraFrame& frame) {
    bt_camera c;
    std::memset(&c, 0, sizeof(c));
    const Camera& cam = frame.camera();
    const Vec3 f = frame.forward(), r = frame.right(), u = frame.up_vector();
    const float pos[3] = {cam.position.x, cam.position.y, cam.position.z};
    const float fw[3] = {f.x, f.y, f.z}, rt[3] = {r.x, r.y, r.z}, up[3] = {u.x, u.y, u.z};
    std::memcpy(c.position, pos, sizeof(pos));
    std::memcpy(c.forward, fw, sizeof(fw));
    std::memcpy(c.right, rt, sizeof(rt));
    std::memcpy(c.up, up, sizeof(up));
    c.tanHalf = frame.tan_half();
    c.aspect = frame.aspect();
    c.invNear = frame.inv_near();
    c.invDepthRange = frame.inv_depth_range();
    c.nearZ = cam.nearZ;
    c.farZ = cam.farZ;
    c.width = cam.width;
    c.height = cam.height;
    return c;
}

bt_render_config to_device_config(const RenderConfig& cfg) {
    bt_render_config d;
    std::memset(&d, 0, sizeof(d));
    d.lipschitz = cfg.lipschitz;
    d.relax = cfg.relax;
    d.minStep = cfg.minStep;
    d.hitEpsilon = cfg.hitEpsilon;
    d.maxOverlap = cfg.maxOverlap;
    d.maxNewPerFetch = cfg.maxNewPerFetch;
    d.fetchWindow = cfg.fetchWindow;
    d.normalsMode = cfg.normalsMode == RenderConfig::NormalsMode::CentralDifference ? 1 : 0;
    d.threads = cfg.threads;
    return d;
}

// ---------------------------------------------------------------- Renderer

Renderer::Renderer(int device) {
    check_device(bt_ctx_create(device < 0 ? device_from_env() : device, &ctx_), "bt_ctx_create");
}

Renderer::~Renderer() { bt_ctx_destroy(ctx_); }

void Renderer::upload(const LinearTree& tree) {
    static_assert(sizeof(NodeRecord) == sizeof(bt_node), "NodeRecord layout");
    check_device(bt_tree_upload(ctx_, tree.data.data(), tree.word_count(),
                                reinterpret_cast<const bt_node*>(tree.nodes.data()), tree.node_count(),
                                tree.primitiveWords.data(), static_cast<uint32_t>(tree.primitiveWords.size()),
                                tree.rootWord),
                 "bt_tree_upload");
    tree_ = &tree;
    stagedWords_.clear();
    stagedCounts_.clear();
    stagedParams_.clear();
}

void Renderer::update_primitive_params(uint32_t word, const PrimitiveParams& params) {
    if (!tree_) throw DeviceError("Renderer::update_primitive_params before upload");
    const Blob b = tree_->blob_at(word);
    if (!b.isPrimitive || b.nodeOp != static_cast<uint8_t>(params.kind))
        throw std::invalid_argument("in-place update must keep the primitive kind");
    validate_primitive(params);
    constexpr uint32_t kStride = 17;
    const uint32_t n = kTransformFloatCount + shape_float_count(params.kind);
    const size_t base = stagedParams_.size();
    stagedParams_.resize(base + kStride, 0.0f);
    float* dst = stagedParams_.data() + base;
    const float head[kTransformFloatCount] = {params.frame.translate.x, params.frame.translate.y,
                                              params.frame.translate.z, params.frame.rotation.w,
                                              params.frame.rotation.x,  params.frame.rotation.y,
                                              params.frame.rotation.z};
    std::memcpy(dst, head, sizeof(head));
    std::memcpy(dst + kTransformFloatCount, params.shape.data(), shape_float_count(params.kind) * sizeof(float));
    stagedWords_.push_back(word);
    stagedCounts_.push_back(n);
}

void Renderer::flush_params() {
    if (stagedWords_.empty()) return;
    check_device(bt_params_update(ctx_, stagedWords_.data(), stagedParams_.data(), stagedCounts_.data(),
                                  static_cast<uint32_t>(stagedWords_.size()), 17),
                 "bt_params_update");
    stagedWords_.clear();
    stagedCounts_.clear();
    stagedParams_.clear();
}

void Renderer::render(const CameraFrame& frame, const RenderConfig& cfg, bool exact, bool useGraph) {
    validate_config(cfg);
    flush_params();
    const bt_camera cam = to_device_camera(frame);
    const bt_render_config dc = to_device_config(cfg);
    check_device(bt_render_frame(ctx_, &cam, &dc, 0, 0, exact ? 1 : 0, useGraph ? BT_FRAME_GRAPH : 0), "bt_render_frame");
}

GBuffer Renderer::download() const {
    bt_gbuffer_view v;
    check_device(bt_gbuffer_device(ctx_, &v), "bt_gbuffer_device");
    GBuffer g;
    g.init(v.width, v.height);
    static_assert(sizeof(Vec3) == 12, "Vec3 layout");
    check_device(bt_gbuffer_download(ctx_, g.hit.data(), g.depth.data(), reinterpret_cast<float*>(g.normal.data()),
                                     g.evalCount.data(), g.tileMaxOverlap.data(), g.tileCacheBytes.data(),
                                     g.tileError.data()),
                 "bt_gbuffer_download");
    return g;
}

bt_stats Renderer::device_stats() const {
    bt_stats s;
    check_device(bt_stats_download(ctx_, &s), "bt_stats_download");
    return s;
}

RenderStats Renderer::stats() const {
    const bt_stats s = device_stats();
    RenderStats r;
    r.fieldEvals = s.fieldEvals;
    r.retainedNodeVisits = s.retainedNodeVisits;
    r.primitiveEvals = s.primitiveEvals;
    r.treeNodeCount = s.treeNodeCount;
    r.maxOverlap = s.maxOverlap;
    r.maxCacheBytes = s.maxCacheBytes;
    return r;
}

void Renderer::reset_stats() { check_device(bt_stats_reset(ctx_), "bt_stats_reset"); }

}  // namespace blobtree
