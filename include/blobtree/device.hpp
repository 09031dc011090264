// blobtree/device.hpp -- device-resident fast path (extension of the
// drop-in API; no reference counterpart).
//
// The reference's free functions (render_tiles, rasterize_volumes, ...)
// return host vectors and re-upload their inputs on every call.  A Renderer
// keeps the tree, volumes, A-buffer and G-buffer resident in HBM across
// frames: per frame only the edited primitive parameters cross PCIe, and
// the whole chain (a) -> (b) -> (c) -> normals replays from one CUDA graph.
#pragma once

#include <mutex>
#include <vector>

#include "../bt_cuda.h"
#include "blobtree/tracer.hpp"

namespace blobtree {

struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& msg) : std::runtime_error(msg) {}
};

// throws DeviceError carrying bt_last_error() when rc != BT_OK
void check_device(int rc, const char* what);

bt_camera to_device_camera(const CameraFrame& frame);
bt_render_config to_device_config(const RenderConfig& cfg);

class Renderer {
public:
    explicit Renderer(int device = -1);  // -1: $BLOBTREE_DEVICE or 0
    ~Renderer();
    Renderer(const Renderer&) = delete;
    Renderer& operator=(const Renderer&) = delete;

    void upload(const LinearTree& tree);
    // validated host-side, staged, applied by the next flush/render
    void update_primitive_params(uint32_t word, const PrimitiveParams& params);
    void flush_params();

    // one frame: VOIs (margin = cfg.hitEpsilon) -> A-buffer -> trace -> normals
    void render(const CameraFrame& frame, const RenderConfig& cfg, bool exact = true, bool useGraph = false);
    GBuffer download() const;
    RenderStats stats() const;
    bt_stats device_stats() const;
    void reset_stats();

    bt_ctx* handle() const { return ctx_; }

private:
    bt_ctx* ctx_ = nullptr;
    const LinearTree* tree_ = nullptr;
    std::vector<uint32_t> stagedWords_;
    std::vector<uint32_t> stagedCounts_;
    std::vector<float> stagedParams_;
};

// process-wide context used by the free functions of the drop-in API.  A
// bt_ctx is not thread-safe, while the reference's free functions are
// reentrant: each drop-in call holds a ContextLease for its whole
// upload -> launch -> download sequence, so calls from several host threads
// serialise instead of interleaving on the shared context.
bt_ctx* default_context();

class ContextLease {
public:
    ContextLease();
    operator bt_ctx*() const { return ctx_; }
    bt_ctx* get() const { return ctx_; }

private:
    std::unique_lock<std::mutex> lock_;
    bt_ctx* ctx_;
};

}  // namespace blobtree
