// capi.cu -- context management and the extern "C" boundary (include/bt_cuda.h).
//
// A bt_ctx owns every device buffer of the path and one CUDA stream:
//   tree      : the reference's 16-byte word array, uploaded bit for bit,
//               plus structure-only side tables (primitive ordinals, the
//               compact-ancestor chain for ROI, the post-order program).
//   (a)       : per-node ROI and per-primitive VOIs (64 B each).
//   (b)       : rays / cones (camera products), candidate pairs, fragment
//               pool, CSR offsets and the sorted fragment array.
//   (c)       : the G-buffer planes and device statistics.
// Buffers are sized lazily and grown on demand; a per-frame CUDA graph is
// re-captured whenever a buffer moves or the frame key changes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bt_cuda.h"
#include "bt_device.h"
#include "bt_cull.cuh"

using namespace btk;

namespace {

thread_local std::string g_lastError;

int fail(int code, const std::string& msg) {
    g_lastError = msg;
    return code;
}

// launch errors (bad configuration, missing attribute, ...) of the kernels
// just enqueued; checked at the end of every eager entry point
int launch_status() {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return 0;
    g_lastError = std::string("kernel launch: ") + cudaGetErrorString(e);
    return BT_ECUDA;
}

#define BT_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(e_ == cudaErrorMemoryAllocation ? BT_ENOMEM : BT_ECUDA,          \
                        std::string(#call) + ": " + cudaGetErrorString(e_));             \
    } while (0)

template <class T> struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    cudaError_t reserve(size_t n) {
        if (n <= cap && ptr) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

struct FrameKey {
    bt_camera cam;
    bt_render_config cfg;
    uint32_t tile0, tile1;
    int exact;
    uint64_t bufEpoch;
    bool operator==(const FrameKey& o) const { return std::memcmp(this, &o, sizeof(FrameKey)) == 0; }
};

}  // namespace

constexpr int kProfSlots = 6;

struct bt_ctx {
    int device = 0;
    int smCount = 148;
    int smClockKHz = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    // a captured frame forks independent stages onto `side` (camera || ROI + VOIs,
    // march ordering || view build) and joins them back
    cudaStream_t side = nullptr;
    cudaEvent_t evFork[2] = {}, evJoin[2] = {};
    bool prezeroed = false;  // enqueueing a captured frame whose counters were zeroed on `side`

    // tree
    DevBuf<float4> words;
    DevBuf<uint32_t> primWords, primOrd, nodeWord, fullProgram, upperProgram, blobs;
    DevBuf<uint2> frontier;
    uint32_t nFrontier = 0, nUpper = 0, upperIsChain = 0, upperIsMinChain = 0;
    DevBuf<int32_t> compactAnc, parentOrd, fastScratch;
    DevBuf<uint32_t> ancOff, ancIdx;  // compact-ancestor lists (k_roi_all)
    bool haveAncLists = false;
    DevBuf<float> roi;
    DevBuf<Voi> vois;
    DevBuf<CullVol> cullVols;      // [nvoi] the volumes' cull terms for the frame's camera (k_pairs)
    DevBuf<RasterVol> rasterVols;  // [nvoi] the volumes' ray-test terms for the frame's camera (k_pairs)
    uint32_t nwords = 0, nnodes = 0, nprims = 0, nvoi = 0, fullDepth = 0;
    bool haveTree = false;
    bool haveRoi = false;
    // host copy of the uploaded structure: a re-upload of the same structure
    // (the drop-in free functions upload on every call) only copies the words
    std::vector<bt_node> hostNodes;
    std::vector<uint32_t> hostPrimWords;
    // GPU compile (bt_tree_compile): the scene graph, scratch, node records
    DevBuf<SceneNodeK> cmpNodes;
    DevBuf<uint8_t> cmpScratch;
    DevBuf<CompileNodeRec> cmpRecords;
    bool treeFromDevice = false;  // node records live in cmpRecords, not hostNodes

    // parameter staging
    DevBuf<uint32_t> pWords, pCounts;
    DevBuf<float> pParams;

    // frame
    int width = 0, height = 0, tilesX = 0, tilesY = 0;
    DevBuf<float4> rays, cones, sbCones, tileFrustum, sbFrustum;
    DevBuf<float> coneSin;
    DevBuf<uint4> pool, unsorted;
    DevBuf<Frag> frags;
    DevBuf<uint32_t> tileCount, tileCursor, tileLocal, blockSum, blockPrefix, offsets, counters;
    // (volume, superblock) pairs grouped by superblock, per-tile fragment lists
    DevBuf<uint32_t> sbCount, sbList;
    uint32_t sbCap = 0;  // candidates per superblock list
    DevBuf<uint2> tileFrag;
    bool haveAbuffer = false;
    bool haveRays = false;
    bt_camera rayCam{};
    uint32_t rayT0 = 0, rayT1 = 0;  // tiles whose rays / cones are current (whole superblock rows)

    // G-buffer
    DevBuf<uint8_t> hit, tileError;
    DevBuf<float> depth, normal;
    DevBuf<uint32_t> evalCount, tileMaxOverlap, tileCacheBytes, fallback;
    bool haveGbuffer = false;

    // streaming download (bt_gbuffer_download_async): two device snapshot slots
    cudaStream_t copyStream = nullptr, copyStream2 = nullptr;  // one per snapshot slot
    DevBuf<uint8_t> snap[2];
    cudaEvent_t evSnap[2] = {}, evCopied[2] = {}, evCopied2[2] = {};
    bool dlPending[2] = {false, false};
    int dlSlot = 0;

    // fused gather (bt_gbuffer_import): the march writes its pixels and tile
    // planes straight into another context's G-buffer (CUDA IPC, peer memory)
    struct Remote {
        bool on = false;
        void* p[7] = {};  // hit, depth, evalCount, tileMaxOverlap, tileCacheBytes, tileError, normal
        int width = 0, height = 0;
    } remote;

    DevBuf<uint64_t> stats;
    // compiled intervals / pruned views of stage (c) (k_views.cu)
    DevBuf<uint2> vCount, vBase, vNodes;
    DevBuf<IntervalRec> vIv;
    DevBuf<uint32_t> vCounters;
    // march scheduling: 0 raster, 1 longest-first by cost proxy (default), 2 host order
    DevBuf<uint32_t> tileOrder, tileCost, orderHist, hostUnits;
    bool viewsFrame = false;  // the G-buffer came from a whole-frame FMA-path march (its records are valid)
    int schedMode = 1;
    int stepBound = 0;  // 0 reference (global L), 1 view-local Lipschitz bound (bt_set_step_bound)
    int depthSlabs = 1;  // > 1: frames rendered slab by slab in view depth (bt_set_depth_slabs)
    DevBuf<uint32_t> tileQueue;   // k_trace work queue head
    DevBuf<float> gradScratch;  // per-warp primitive values of the gradient fallback
    uint32_t gradWarps = 0;

    uint64_t bufEpoch = 1;
    cudaGraphExec_t graph = nullptr;
    uint32_t graphKernels = 0, graphNodes = 0;
    FrameKey graphKey{};
    bool haveGraph = false;

    // profiling (CUDA events around each stage)
    bool profiling = false;
    // slots: 0 roi+voi, 1 abuffer, 2 trace (all of stage c), 3 normals,
    //        4 k_view_* (interval/view compilation), 5 k_march (field evaluation)
    float profMs[kProfSlots] = {};
    uint32_t profLaunch[kProfSlots] = {};
    cudaEvent_t ev[6] = {};
};

namespace {

// Every entry point runs on its context's device: a process may hold
// contexts on several GPUs, and the caller's thread may have any device
// current.  The previous device is restored on return.
struct DevGuard {
    int prev = -1;
    explicit DevGuard(const bt_ctx* c) {
        if (!c) return;
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess)
            prev = cur;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard&) = delete;
    DevGuard& operator=(const DevGuard&) = delete;
};

DevTree dev_tree(const bt_ctx* c) {
    DevTree t;
    t.words = c->words.ptr;
    t.blobs = c->blobs.ptr;
    t.primWords = c->primWords.ptr;
    t.primOrd = c->primOrd.ptr;
    t.nodeWord = c->nodeWord.ptr;
    t.compactAnc = c->compactAnc.ptr;
    t.ancOff = c->haveAncLists ? c->ancOff.ptr : nullptr;
    t.ancIdx = c->haveAncLists ? c->ancIdx.ptr : nullptr;
    t.fullProgram = c->fullProgram.ptr;
    t.nwords = c->nwords;
    t.nnodes = c->nnodes;
    t.nprims = c->nprims;
    t.fullDepth = c->fullDepth;
    t.frontier = c->frontier.ptr;
    t.upperProgram = c->upperProgram.ptr;
    t.nFrontier = c->nFrontier;
    t.nUpper = c->nUpper;
    t.upperIsChain = c->upperIsChain;
    t.upperIsMinChain = c->upperIsMinChain;
    return t;
}

FrameBufs frame_bufs(const bt_ctx* c) {
    FrameBufs f;
    f.rays = c->rays.ptr;
    f.cones = c->cones.ptr;
    f.coneSin = c->coneSin.ptr;
    f.sbCones = c->sbCones.ptr;
    f.tileFrustum = c->tileFrustum.ptr;
    f.sbFrustum = c->sbFrustum.ptr;
    f.pool = c->pool.ptr;
    f.unsorted = c->unsorted.ptr;
    f.frags = c->frags.ptr;
    f.tileCount = c->tileCount.ptr;
    f.tileCursor = c->tileCursor.ptr;
    f.tileLocal = c->tileLocal.ptr;
    f.blockSum = c->blockSum.ptr;
    f.blockPrefix = c->blockPrefix.ptr;
    f.offsets = c->offsets.ptr;
    f.counters = c->counters.ptr;
    f.sbCount = c->sbCount.ptr;
    f.sbList = c->sbList.ptr;
    f.sbCap = c->sbCap;
    f.rasterVols = c->rasterVols.ptr;
    f.cullVols = c->cullVols.ptr;
    f.tileFrag = c->tileFrag.ptr;
    f.poolCap = c->frags.cap;
    f.fragCap = std::min(c->frags.cap, c->unsorted.cap);
    return f;
}

ViewBufs view_bufs(const bt_ctx* c) {
    ViewBufs v;
    v.count = c->vCount.ptr;
    v.base = c->vBase.ptr;
    v.iv = c->vIv.ptr;
    v.nodes = c->vNodes.ptr;
    v.counters = c->vCounters.ptr;
    v.order = nullptr;  // chosen per trace (do_trace)
    v.tileCost = c->tileCost.ptr;
    v.ivCap = c->vIv.cap;
    v.nodeCap = c->vNodes.cap;
    return v;
}

GBuf gbuf(const bt_ctx* c) {
    GBuf g;
    g.hit = c->hit.ptr;
    g.depth = c->depth.ptr;
    g.normal = c->normal.ptr;
    g.evalCount = c->evalCount.ptr;
    g.tileMaxOverlap = c->tileMaxOverlap.ptr;
    g.tileCacheBytes = c->tileCacheBytes.ptr;
    g.tileError = c->tileError.ptr;
    g.fallback = c->fallback.ptr;
    g.width = c->width;
    g.height = c->height;
    g.tilesX = c->tilesX;
    g.tilesY = c->tilesY;
    return g;
}

// G-buffer targets of the march: the context's own planes, or the imported
// planes of another context (fused gather) when the image size matches.
GBuf trace_gbuf(const bt_ctx* c) {
    GBuf g = gbuf(c);
    if (c->remote.on && c->remote.width == c->width && c->remote.height == c->height) {
        g.hit = static_cast<uint8_t*>(c->remote.p[0]);
        g.depth = static_cast<float*>(c->remote.p[1]);
        g.evalCount = static_cast<uint32_t*>(c->remote.p[2]);
        g.tileMaxOverlap = static_cast<uint32_t*>(c->remote.p[3]);
        g.tileCacheBytes = static_cast<uint32_t*>(c->remote.p[4]);
        g.tileError = static_cast<uint8_t*>(c->remote.p[5]);
        g.normal = static_cast<float*>(c->remote.p[6]);
        g.remote = 1;
    }
    return g;
}

void release_remote(bt_ctx* c) {
    if (!c->remote.on) return;
    for (void*& q : c->remote.p) {
        if (q) cudaIpcCloseMemHandle(q);
        q = nullptr;
    }
    c->remote.on = false;
    c->bufEpoch++;
}

Cam to_cam(const bt_camera& k) {
    return make_cam(k.position, k.forward, k.right, k.up, k.tanHalf, k.aspect, k.invNear,
                    k.invDepthRange, k.nearZ, k.farZ, k.width, k.height);
}

int check_camera(const bt_camera* cam) {
    if (!cam) return fail(BT_EINVAL, "camera is null");
    if (cam->width <= 0 || cam->height <= 0) return fail(BT_EINVAL, "camera image size must be positive");
    return BT_OK;
}

// (Re)size every per-image buffer for a camera.
int ensure_image(bt_ctx* c, const bt_camera& cam) {
    const int tx = (cam.width + kTile - 1) / kTile, ty = (cam.height + kTile - 1) / kTile;
    if (tx == c->tilesX && ty == c->tilesY && cam.width == c->width && cam.height == c->height) return BT_OK;
    c->width = cam.width;
    c->height = cam.height;
    c->tilesX = tx;
    c->tilesY = ty;
    const size_t tiles = (size_t)tx * ty;
    const size_t px = (size_t)cam.width * cam.height;
    const size_t nsb = (size_t)((tx + kSB - 1) / kSB) * ((ty + kSB - 1) / kSB);
    const size_t nscan = (tiles + 4095) / 4096;
    BT_CUDA(c->rays.reserve(tiles * 64));
    BT_CUDA(c->cones.reserve(tiles));
    BT_CUDA(c->coneSin.reserve(tiles));
    BT_CUDA(c->sbCones.reserve(nsb));
    BT_CUDA(c->tileFrustum.reserve(tiles * 4));
    BT_CUDA(c->sbFrustum.reserve(nsb * 4));
    BT_CUDA(c->tileCount.reserve(tiles));
    BT_CUDA(c->tileCursor.reserve(tiles));
    BT_CUDA(c->tileLocal.reserve(tiles));
    BT_CUDA(c->blockSum.reserve(nscan));
    BT_CUDA(c->blockPrefix.reserve(nscan + 1));
    BT_CUDA(c->offsets.reserve(tiles + 1));
    BT_CUDA(c->hit.reserve(px));
    BT_CUDA(c->depth.reserve(px));
    BT_CUDA(c->normal.reserve(px * 3));
    BT_CUDA(c->evalCount.reserve(px));
    BT_CUDA(c->fallback.reserve(px));
    BT_CUDA(c->tileMaxOverlap.reserve(tiles));
    BT_CUDA(c->tileCacheBytes.reserve(tiles));
    BT_CUDA(c->tileError.reserve(tiles));
    BT_CUDA(c->vCount.reserve(tiles));
    BT_CUDA(c->vBase.reserve(tiles));
    BT_CUDA(c->vCounters.reserve(4));
    BT_CUDA(c->sbCount.reserve(nsb));
    BT_CUDA(c->tileFrag.reserve(tiles));
    BT_CUDA(c->tileCost.reserve(tiles));
    BT_CUDA(c->tileOrder.reserve(tiles * 2));
    BT_CUDA(c->orderHist.reserve(258));
    BT_CUDA(c->hostUnits.reserve(1));
    if (c->schedMode == 2) c->schedMode = 1;  // a host order no longer matches the image
    c->haveAbuffer = false;
    c->haveRays = false;
    c->haveGbuffer = false;
    c->bufEpoch++;
    return BT_OK;
}

// sbCap: candidates per superblock list (k_pairs appends straight into them);
// poolCap: fragments
int ensure_frame_caps(bt_ctx* c, size_t sbCap, size_t poolCap) {
    bool moved = false;
    const size_t nsb = superblock_count(c->tilesX, c->tilesY);
    sbCap = std::max<size_t>(sbCap, c->sbCap);
    if (sbCap > c->sbCap || nsb * sbCap > c->sbList.cap) {
        BT_CUDA(c->sbList.reserve(nsb * sbCap));
        c->sbCap = (uint32_t)sbCap;
        moved = true;
    }
    if (poolCap > c->frags.cap) {  // the fragment store (and its CSR / overflow staging)
        BT_CUDA(c->unsorted.reserve(poolCap));
        BT_CUDA(c->frags.reserve(poolCap));
        moved = true;
    }
    if (moved) c->bufEpoch++;
    return BT_OK;
}

void prof_begin(bt_ctx* c) {
    if (c->profiling) cudaEventRecord(c->ev[0], c->stream);
}
void prof_end(bt_ctx* c, int slot) {
    if (!c->profiling) return;
    cudaEventRecord(c->ev[1], c->stream);
    cudaEventSynchronize(c->ev[1]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->profMs[slot] += ms;
    c->profLaunch[slot] += 1;
}

TraceParams trace_params(const bt_render_config& cfg, const bt_camera& cam, int stepBound = 0) {
    TraceParams tp;
    tp.viewLipschitz = stepBound == 1 ? 1u : 0u;
    tp.L = cfg.lipschitz;
    tp.invL = 1.0f / cfg.lipschitz;
    tp.relax = cfg.relax;
    tp.minStep = cfg.minStep;
    tp.hitEps = cfg.hitEpsilon;
    tp.maxOverlap = cfg.maxOverlap;
    tp.maxNew = cfg.maxNewPerFetch;
    float window = cfg.fetchWindow;
    if (!(window > 0.0f)) window = (cam.farZ - cam.nearZ) / 20.0f;
    tp.window = window;
    return tp;
}

int check_config(const bt_render_config* cfg) {
    if (!cfg) return fail(BT_EINVAL, "render config is null");
    if (!(cfg->relax >= 1.0f && cfg->relax < 2.0f)) return fail(BT_EINVAL, "relaxation factor must lie in [1, 2)");
    if (!(cfg->lipschitz >= 1.0f)) return fail(BT_EINVAL, "lipschitz bound must be at least 1");
    if (!(cfg->minStep > 0.0f)) return fail(BT_EINVAL, "min step must be > 0");
    if (!(cfg->hitEpsilon > 0.0f)) return fail(BT_EINVAL, "hit epsilon must be > 0");
    if (cfg->maxOverlap == 0 || cfg->maxOverlap > BT_MAX_OVERLAP) return fail(BT_EINVAL, "max overlap must lie in [1, 96]");
    return BT_OK;
}

// Rays, tile cones and pyramids for the superblock rows that meet
// [tile0, tile1) (tile1 == 0: the whole image).  A sharded rank that does not
// compute normals needs only its own rows.
int do_camera(bt_ctx* c, const bt_camera& cam, uint32_t tile0 = 0, uint32_t tile1 = 0, cudaStream_t st = nullptr) {
    int rc = ensure_image(c, cam);
    if (rc) return rc;
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    if (tile1 == 0 || tile1 > tiles) tile1 = tiles;
    if (tile0 > tile1) tile0 = tile1;
    launch_camera(st ? st : c->stream, to_cam(cam), frame_bufs(c), c->tilesX, c->tilesY, tile0, tile1);
    c->haveRays = true;
    c->rayCam = cam;
    c->rayT1 = camera_tile_cover(c->tilesX, c->tilesY, tile0, tile1, &c->rayT0);
    return BT_OK;
}

int ensure_side(bt_ctx* c) {
    if (c->side) return BT_OK;
    BT_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        BT_CUDA(cudaEventCreateWithFlags(&c->evFork[i], cudaEventDisableTiming));
        BT_CUDA(cudaEventCreateWithFlags(&c->evJoin[i], cudaEventDisableTiming));
    }
    return BT_OK;
}

// true when the current rays cover [tile0, tile1) for this camera
bool rays_cover(const bt_ctx* c, const bt_camera& cam, uint32_t tile0, uint32_t tile1) {
    return c->haveRays && std::memcmp(&c->rayCam, &cam, sizeof(bt_camera)) == 0 && c->rayT0 <= tile0 &&
           tile1 <= c->rayT1;
}

int resolve_tiles(bt_ctx* c, uint32_t& tile0, uint32_t& tile1) {
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    if (tile1 == 0 || tile1 > tiles) tile1 = tiles;
    if (tile0 > tile1) return fail(BT_EINVAL, "tile range is empty or inverted");
    return BT_OK;
}

int ensure_view_caps(bt_ctx* c) {
    if (c->vIv.cap == 0) {
        const size_t tiles = (size_t)c->tilesX * c->tilesY;
        BT_CUDA(c->vIv.reserve(std::max<size_t>(1u << 16, tiles * 2)));
        BT_CUDA(c->vNodes.reserve(std::max<size_t>(1u << 18, tiles * 8)));
        c->bufEpoch++;
    }
    return BT_OK;
}

// The A-buffer: superblock pairs, then the per-tile pass (k_tile) in `mode`
// (raster, or raster + the interval records of `tp` in a fused frame).  In
// `checked` mode the allocation counters are read back afterwards (one D2H)
// and the frame rebuilt after growing what overflowed; inside a graph replay
// an overflow degrades to an empty, flagged A-buffer / record set.
int do_abuffer(bt_ctx* c, const bt_camera& cam, uint32_t tile0, uint32_t tile1, bool checked,
               uint32_t mode = kTileRaster, const TraceParams* tp = nullptr) {
    {  // first frame: a guess of the superblock lists' size (the checked path grows them); an image
       // resize: the same capacity over the new superblock count
        const size_t nsb = std::max<size_t>(1, superblock_count(c->tilesX, c->tilesY));
        const size_t guess = c->sbCap ? c->sbCap : std::max<size_t>(256, 2 * (size_t)c->nvoi * 16 / nsb);
        int rc = ensure_frame_caps(c, guess, c->frags.cap ? c->frags.cap : (size_t)1u << 20);
        if (rc) return rc;
    }
    if (mode & kTileViews) {
        int rc = ensure_view_caps(c);
        if (rc) return rc;
    }
    const TraceParams tpv = tp ? *tp : TraceParams{};
    for (int attempt = 0; attempt < 8; ++attempt) {
        launch_abuffer(c->stream, to_cam(cam), c->vois.ptr, c->nvoi, frame_bufs(c), c->tilesX, c->tilesY,
                       tile0, tile1, c->smCount, !c->prezeroed);
        launch_tile_pass(c->stream, mode, to_cam(cam), tpv, c->vois.ptr, frame_bufs(c), view_bufs(c), c->tilesX,
                         c->tilesY, tile0, tile1, c->smCount);
        if (!checked) break;
        uint32_t cnt[kCntSlots];
        uint32_t vc[4] = {0u, 0u, 0u, 0u};
        BT_CUDA(cudaMemcpyAsync(cnt, c->counters.ptr, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
        if (mode & kTileViews)
            BT_CUDA(cudaMemcpyAsync(vc, c->vCounters.ptr, sizeof(vc), cudaMemcpyDeviceToHost, c->stream));
        BT_CUDA(cudaStreamSynchronize(c->stream));
        const bool pairOver = cnt[kCntSbNeed] != 0u;  // a superblock list overflowed
        const bool fragOver = !pairOver && cnt[kCntFrags] > frame_bufs(c).fragCap;
        const bool ivOver = !pairOver && !fragOver && (mode & kTileViews) && (vc[2] > c->vIv.cap || vc[3] > c->vNodes.cap);
        if (!pairOver && !fragOver && !ivOver) break;
        // (lost pairs also lose their fragments and records: grow one thing at a time)
        int rc = ensure_frame_caps(c, pairOver ? (size_t)cnt[kCntSbNeed] * 3 / 2 + 64 : c->sbCap,
                                   fragOver ? (size_t)cnt[kCntFrags] * 2 : c->frags.cap);
        if (rc) return rc;
        if (ivOver) {
            if (vc[2] > c->vIv.cap) BT_CUDA(c->vIv.reserve((size_t)vc[2] * 2));
            if (vc[3] > c->vNodes.cap) BT_CUDA(c->vNodes.reserve((size_t)vc[3] * 2));
            c->bufEpoch++;
        }
    }
    c->haveAbuffer = true;
    return BT_OK;
}

// The interval records of an A-buffer built without them (bt_abuffer_build
// or an uploaded A-buffer, then bt_trace): k_tile in views mode, checked.
int do_views(bt_ctx* c, const bt_camera& cam, const TraceParams& tp, uint32_t tile0, uint32_t tile1, bool checked) {
    int rc = ensure_view_caps(c);
    if (rc) return rc;
    for (int attempt = 0; attempt < 8; ++attempt) {
        launch_tile_pass(c->stream, kTileViews, to_cam(cam), tp, c->vois.ptr, frame_bufs(c), view_bufs(c), c->tilesX,
                         c->tilesY, tile0, tile1, c->smCount);
        if (!checked) break;
        uint32_t vc[4];
        BT_CUDA(cudaMemcpyAsync(vc, c->vCounters.ptr, sizeof(vc), cudaMemcpyDeviceToHost, c->stream));
        BT_CUDA(cudaStreamSynchronize(c->stream));
        if (vc[2] <= c->vIv.cap && vc[3] <= c->vNodes.cap) break;
        if (vc[2] > c->vIv.cap) BT_CUDA(c->vIv.reserve((size_t)vc[2] * 2));
        if (vc[3] > c->vNodes.cap) BT_CUDA(c->vNodes.reserve((size_t)vc[3] * 2));
        c->bufEpoch++;
    }
    return BT_OK;
}

// Half-tile split rule of the march scheduler: tiles whose cost proxy is at
// least beta x the average work per warp become two units ($BT_SPLIT_BETA,
// default kSplitBeta), at most 2x the grid's warps of them.
constexpr float kSplitBeta = 0.5f;
float split_beta() {
    static float beta = -1.0f;
    if (beta < 0.0f) {
        beta = kSplitBeta;
        if (const char* e = getenv("BT_SPLIT_BETA")) beta = (float)atof(e);
    }
    return beta;
}

// Stage (c): the interval records (unless the fused A-buffer pass already
// wrote them), the views (k_view_build) beside the march order, then the
// march.  In `checked` mode the record totals are read back and the buffers
// grown (2x headroom); inside a graph replay an overflow is flagged
// (bt_stats_download) and the tiles marked.
// `slab` >= 0: depth slab `slab` of a slab-by-slab frame (cam = the slab's
// camera, `window` the frame camera's fetch window; slabs after the first
// continue the G-buffer of the earlier ones, in raster order).
int do_trace(bt_ctx* c, const bt_camera& cam, const bt_render_config& cfg, uint32_t tile0, uint32_t tile1,
             int exact, bool checked, bool haveRecords = false, int slab = -1, float window = 0.0f) {
    if (c->tileQueue.cap == 0) {
        BT_CUDA(c->tileQueue.reserve(1));
        c->bufEpoch++;
    }
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    const DevTree t = dev_tree(c);
    const Cam k = to_cam(cam);
    TraceParams tp = trace_params(cfg, cam, c->stepBound);
    if (slab >= 0) tp.window = window;
    // stage events only in eager frames: synchronising on an event inside a
    // stream capture would invalidate the capture
    const bool prof = c->profiling && checked;
    if (prof) cudaEventRecord(c->ev[2], c->stream);
    if (!haveRecords) {
        int rc = do_views(c, cam, tp, tile0, tile1, checked);
        if (rc) return rc;
    }
    // longest-first march units from k_tile's cost proxy; in a captured frame
    // they are ordered on the side stream while the views are built
    auto order = [&](cudaStream_t st) {
        launch_tile_order(st, view_bufs(c), trace_gbuf(c), c->orderHist.ptr, c->tileOrder.ptr, tile0, tile1,
                          trace_grid_warps(c->smCount), split_beta(), 2u * trace_grid_warps(c->smCount));
    };
    // (a slab frame keeps raster order: the half-tile split would reset the
    // tile planes the earlier slabs wrote)
    const int sched = slab >= 0 ? 0 : c->schedMode;
    const bool forkOrder = sched == 1 && !checked;
    if (sched == 1 && checked) order(c->stream);
    if (prof) cudaEventRecord(c->ev[3], c->stream);
    if (forkOrder) {
        int rc = ensure_side(c);
        if (rc) return rc;
        BT_CUDA(cudaEventRecord(c->evFork[1], c->stream));
        BT_CUDA(cudaStreamWaitEvent(c->side, c->evFork[1], 0));
        order(c->side);
        BT_CUDA(cudaEventRecord(c->evJoin[1], c->side));
    }
    if (prof) cudaEventRecord(c->ev[4], c->stream);
    launch_view_build(c->stream, t, view_bufs(c), c->smCount);
    if (prof) cudaEventRecord(c->ev[5], c->stream);
    if (forkOrder) BT_CUDA(cudaStreamWaitEvent(c->stream, c->evJoin[1], 0));
    ViewBufs vbm = view_bufs(c);
    if (sched == 1) {
        vbm.order = c->tileOrder.ptr;
        vbm.unitCount = c->orderHist.ptr + 257;
    } else if (sched == 2 && tile0 == 0 && tile1 == tiles) {
        vbm.order = c->tileOrder.ptr;
        vbm.unitCount = c->hostUnits.ptr;
    }
    GBuf gm = trace_gbuf(c);
    gm.accumulate = slab > 0 ? 1 : 0;
    launch_trace(c->stream, exact != 0, t, k, tp, frame_bufs(c), vbm, gm, c->stats.ptr, tile0, tile1, c->smCount,
                 c->tileQueue.ptr, !c->prezeroed || slab > 0);
    if (prof) {  // sub-stage split: views (records, build) and the march alone
        cudaEventRecord(c->ev[1], c->stream);
        cudaEventSynchronize(c->ev[1]);
        float a = 0.f, b = 0.f, m = 0.f;
        cudaEventElapsedTime(&a, c->ev[2], c->ev[3]);
        cudaEventElapsedTime(&b, c->ev[4], c->ev[5]);
        cudaEventElapsedTime(&m, c->ev[5], c->ev[1]);
        c->profMs[4] += a + b;
        c->profMs[5] += m;
        c->profLaunch[4] += 1;
        c->profLaunch[5] += 1;
    }
    c->haveGbuffer = true;
    // (a slab frame's records cover its last slab only: normals' fallback over the full tree)
    c->viewsFrame = !exact && tile0 == 0 && tile1 == tiles && slab < 0;
    return BT_OK;
}

// The camera of depth slab s of n: view depth [near, far] cut into n equal
// slabs; the A-buffer of a slab clips its fragments to the slab (rasterize_
// volumes' near / far clip), and its NDC constants are the slab's own.
bt_camera slab_camera(const bt_camera& cam, int s, int n) {
    bt_camera k = cam;
    const float range = cam.farZ - cam.nearZ;
    k.nearZ = s == 0 ? cam.nearZ : cam.nearZ + range * (float)s / (float)n;
    k.farZ = s == n - 1 ? cam.farZ : cam.nearZ + range * (float)(s + 1) / (float)n;
    k.invNear = 1.0f / k.nearZ;
    k.invDepthRange = 1.0f / (k.invNear - 1.0f / k.farZ);
    return k;
}

// rows [y0, y1) of the image (y1 < 0: all); `target`: the planes to shade
// (this context's, or the root's over peer memory for a sharded rank)
int do_normals(bt_ctx* c, const bt_camera& cam, int mode, int exact, int y0 = 0, int y1 = -1, bool target = false) {
    if (c->fullDepth > 128) return fail(BT_EINVAL, "full-tree evaluation stack deeper than 128 entries");
    if (c->gradWarps == 0) {
        // one CTA per queued pixel; frontier values live in shared memory,
        // or (very large trees) in a per-CTA global scratch
        const size_t per = (size_t)c->nFrontier * 6;
        size_t ctas = (size_t)c->smCount * 2;
        if (per * 4 + (size_t)c->nUpper * 4 > kGradSmemBytes) {
            ctas = std::min<size_t>(ctas, std::max<size_t>(1, (256u << 20) / (per * 4)));
            BT_CUDA(c->gradScratch.reserve(ctas * per));
        } else {
            BT_CUDA(c->gradScratch.reserve(1));
        }
        c->gradWarps = (uint32_t)ctas;
        c->bufEpoch++;
    }
    const ViewBufs vb = view_bufs(c);
    launch_normals(c->stream, exact != 0, dev_tree(c), to_cam(cam), frame_bufs(c), target ? trace_gbuf(c) : gbuf(c),
                   mode, c->counters.ptr, c->stats.ptr, c->smCount, c->gradScratch.ptr, c->gradWarps,
                   (c->viewsFrame || target) && !exact ? &vb : nullptr, !c->prezeroed, y0, y1);
    return BT_OK;
}

}  // namespace

// ======================================================================== C-ABI

extern "C" {

const char* bt_last_error(void) { return g_lastError.c_str(); }

int bt_ctx_create(int device, bt_ctx** out) {
    if (!out) return fail(BT_EINVAL, "out is null");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(BT_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(BT_EINVAL, "device index out of range");
    BT_CUDA(cudaSetDevice(device));
    bt_ctx* c = new bt_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->smCount, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&c->smClockKHz, cudaDevAttrClockRate, device);
    e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(BT_ECUDA, cudaGetErrorString(e));
    }
    c->stream = c->own;
    for (auto& e : c->ev) cudaEventCreate(&e);
    if (c->stats.reserve(kStSlots) != cudaSuccess || c->counters.reserve(kCntSlots) != cudaSuccess) {
        delete c;
        return fail(BT_ENOMEM, "cannot allocate statistics");
    }
    cudaMemset(c->stats.ptr, 0, kStSlots * sizeof(uint64_t));
    cudaMemset(c->counters.ptr, 0, kCntSlots * sizeof(uint32_t));
    *out = c;
    return BT_OK;
}

int bt_ctx_destroy(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c) return BT_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    c->frontier.release();
    c->cmpNodes.release();
    c->cmpScratch.release();
    c->cmpRecords.release();
    for (auto* b : {&c->primWords, &c->primOrd, &c->nodeWord, &c->fullProgram, &c->upperProgram, &c->blobs, &c->pWords, &c->pCounts,
                    &c->tileCount, &c->tileCursor, &c->tileLocal, &c->blockSum, &c->blockPrefix, &c->offsets,
                    &c->counters, &c->evalCount, &c->tileMaxOverlap, &c->tileCacheBytes, &c->fallback})
        b->release();
    c->words.release();
    c->compactAnc.release();
    c->ancOff.release();
    c->ancIdx.release();
    c->parentOrd.release();
    c->fastScratch.release();
    c->roi.release();
    c->vois.release();
    c->rasterVols.release();
    c->cullVols.release();
    c->pParams.release();
    c->rays.release();
    c->cones.release();
    c->sbCones.release();
    c->tileFrustum.release();
    c->sbFrustum.release();
    c->coneSin.release();
    c->pool.release();
    c->unsorted.release();
    c->frags.release();
    c->hit.release();
    c->tileError.release();
    c->depth.release();
    c->normal.release();
    c->stats.release();
    c->gradScratch.release();
    for (auto* b : {&c->vCount, &c->vBase, &c->vNodes, &c->tileFrag}) b->release();
    for (auto* b : {&c->sbCount, &c->sbList}) b->release();
    c->vIv.release();
    c->vCounters.release();
    c->tileOrder.release();
    c->tileCost.release();
    c->hostUnits.release();
    c->orderHist.release();
    c->tileQueue.release();
    for (auto& e : c->ev) cudaEventDestroy(e);
    release_remote(c);
    if (c->copyStream) {
        cudaStreamSynchronize(c->copyStream);
        cudaStreamSynchronize(c->copyStream2);
        cudaStreamDestroy(c->copyStream);
        cudaStreamDestroy(c->copyStream2);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(c->evSnap[i]);
            cudaEventDestroy(c->evCopied[i]);
            cudaEventDestroy(c->evCopied2[i]);
            c->snap[i].release();
        }
    }
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(c->evFork[i]);
            cudaEventDestroy(c->evJoin[i]);
        }
    }
    cudaStreamDestroy(c->own);
    delete c;
    return BT_OK;
}

int bt_sync(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    BT_CUDA(cudaStreamSynchronize(c->stream));
    if (c->copyStream) BT_CUDA(cudaStreamSynchronize(c->copyStream));
    if (c->copyStream2) BT_CUDA(cudaStreamSynchronize(c->copyStream2));
    BT_CUDA(cudaGetLastError());
    return BT_OK;
}

int bt_set_stream(bt_ctx* c, void* s) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    c->stream = s ? (cudaStream_t)s : c->own;
    c->haveGraph = false;
    return BT_OK;
}

int bt_device_info(bt_ctx* c, int* sm, int* clk) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (sm) *sm = c->smCount;
    if (clk) *clk = c->smClockKHz;
    return BT_OK;
}

int bt_tree_upload(bt_ctx* c, const float* data, uint32_t nwords, const bt_node* nodes, uint32_t nnodes,
                   const uint32_t* primitiveWords, uint32_t nprims, uint32_t rootWord) {
    DevGuard dg_(c);
    if (!c || !data || !nodes || !primitiveWords) return fail(BT_EINVAL, "null tree buffer");
    if (nwords == 0 || nnodes == 0 || nprims == 0) return fail(BT_EINVAL, "empty tree");
    if (nwords >= BT_ANCESTOR_SENTINEL) return fail(BT_EINVAL, "tree exceeds the 23-bit node index space");
    (void)rootWord;
    // frame products of the previous tree must not be marched or shaded
    // against the new one (fragment words, view nodes index its words)
    c->haveAbuffer = false;
    c->haveGbuffer = false;
    c->viewsFrame = false;
    if (c->haveTree && !c->treeFromDevice && nwords == c->nwords && nnodes == c->nnodes && nprims == c->nprims &&
        c->hostNodes.size() == nnodes && c->hostPrimWords.size() == nprims &&
        std::memcmp(c->hostNodes.data(), nodes, (size_t)nnodes * sizeof(bt_node)) == 0 &&
        std::memcmp(c->hostPrimWords.data(), primitiveWords, (size_t)nprims * 4) == 0) {
        // same structure: the side tables stay valid, only parameters changed
        BT_CUDA(cudaMemcpyAsync(c->words.ptr, data, (size_t)nwords * 16, cudaMemcpyHostToDevice, c->stream));
        launch_blob_table(c->stream, c->words.ptr, c->nodeWord.ptr, nnodes, c->blobs.ptr);
        BT_CUDA(cudaStreamSynchronize(c->stream));
        c->haveRoi = false;
        c->nvoi = 0;
        return BT_OK;
    }
    c->haveTree = false;
    // structure-only side tables
    std::vector<uint32_t> nodeWord(nnodes), primOrd(nprims), program(nnodes);
    std::vector<int32_t> parentOrd(nnodes, -1), compactAnc(nnodes, -1);
    for (uint32_t i = 0; i < nnodes; ++i) {
        nodeWord[i] = nodes[i].word;
        if (nodes[i].word >= nwords) return fail(BT_EINVAL, "node word out of range");
        program[i] = ((uint32_t)(nodes[i].isPrimitive ? 1u : 0u) << 31) | ((uint32_t)(nodes[i].nodeOp & 0x1F) << 26) |
                     (nodes[i].word & BT_ANCESTOR_SENTINEL);
        if (!nodes[i].isPrimitive) {
            const int32_t l = nodes[i].leftChild, r = nodes[i].rightChild;
            if (l < 0 || r < 0 || (uint32_t)l >= nnodes || (uint32_t)r >= nnodes)
                return fail(BT_EINVAL, "operator child ordinal out of range");
            parentOrd[l] = (int32_t)i;
            parentOrd[r] = (int32_t)i;
        }
    }
    // compact ancestor chain: nodes are post-order, parents after children,
    // so a reverse sweep sees every parent first.
    for (int64_t i = (int64_t)nnodes - 1; i >= 0; --i) {
        const int32_t p = parentOrd[i];
        if (p < 0) continue;
        const uint8_t op = nodes[p].nodeOp;
        compactAnc[i] = (op >= 9 && op <= 11) ? p : compactAnc[p];
    }
    // the compact-ancestor chains as CSR lists of parameter words (capped:
    // a very deep all-compact comb keeps the chain walk)
    std::vector<uint32_t> ancOff(nnodes + 1, 0), ancIdx;
    bool ancLists = true;
    for (uint32_t i = 0; i < nnodes && ancLists; ++i) {
        for (int32_t a = compactAnc[i]; a >= 0; a = compactAnc[a]) ancIdx.push_back(nodes[a].word + 1);
        ancOff[i + 1] = (uint32_t)ancIdx.size();
        if (ancIdx.size() > (size_t)(1u << 24)) ancLists = false;
    }
    // map primitive words to ordinals (both ascending)
    {
        uint32_t k = 0;
        for (uint32_t i = 0; i < nnodes && k < nprims; ++i)
            if (nodes[i].isPrimitive && nodes[i].word == primitiveWords[k]) primOrd[k++] = i;
        if (k != nprims) return fail(BT_EINVAL, "primitiveWords do not match the node records");
    }
    // frontier decomposition: subtree sizes in post-order, frontier roots are
    // the maximal subtrees of <= cap nodes.  The cap is chosen per tree by a
    // small cost model of k_gradient: phase 1's critical path (the heaviest
    // thread's nodes, ~6 units each: parameter loads + 6 evaluations) plus
    // phase 2's serial length (one unit per upper entry; a left comb of sharp
    // unions reduces in log steps).
    std::vector<uint32_t> size(nnodes, 1);
    for (uint32_t i = 0; i < nnodes; ++i)
        if (!nodes[i].isPrimitive) size[i] = 1 + size[nodes[i].leftChild] + size[nodes[i].rightChild];
    std::vector<uint2> frontier;
    std::vector<uint32_t> upper;
    bool chain = false, minChain = false;
    double bestCost = 0.0;
    for (uint32_t cap : {4u, 8u, 16u, kFrontierMax}) {
        std::vector<uint2> f;
        std::vector<uint32_t> u;
        for (uint32_t i = 0; i < nnodes; ++i) {
            const int32_t p = parentOrd[i];
            if (size[i] <= cap && (p < 0 || size[p] > cap)) {
                u.push_back(0x80000000u | (uint32_t)f.size());
                f.push_back(make_uint2(i + 1 - size[i], i));
            } else if (size[i] > cap) {
                u.push_back(program[i]);  // operator (size > 1)
            }
        }
        // left comb: LOAD, then (LOAD, OP) pairs -- every operator folds the
        // running value with a fresh load
        bool ch = !u.empty() && (u[0] >> 31) && (u.size() % 2 == 1);
        for (size_t j = 1; ch && j < u.size(); j += 2) ch = (u[j] >> 31) && !(u[j + 1] >> 31);
        bool mc = ch;
        for (size_t j = 2; mc && j < u.size(); j += 2) mc = ((u[j] >> 26) & 0x1Fu) == 3u;
        std::vector<uint32_t> load(256, 0);
        for (size_t j = 0; j < f.size(); ++j) load[j % 256] += f[j].y - f[j].x + 1;
        const double phase1 = 6.0 * *std::max_element(load.begin(), load.end());
        const double phase2 = mc ? 10.0 + (double)(u.size() / 2 + 31) / 32 : (double)u.size();
        if (frontier.empty() || phase1 + phase2 < bestCost) {
            bestCost = phase1 + phase2;
            frontier.swap(f);
            upper.swap(u);
            chain = ch;
            minChain = mc;
        }
    }
    // full post-order stack depth
    uint32_t depth = 0, maxd = 0;
    for (uint32_t i = 0; i < nnodes; ++i) {
        if (nodes[i].isPrimitive) {
            ++depth;
        } else {
            if (depth < 2) return fail(BT_EINVAL, "node records are not a post-order binary tree");
            --depth;
        }
        maxd = std::max(maxd, depth);
    }
    BT_CUDA(cudaSetDevice(c->device));
    BT_CUDA(c->words.reserve(nwords + 8));
    BT_CUDA(c->primWords.reserve(nprims));
    BT_CUDA(c->primOrd.reserve(nprims));
    BT_CUDA(c->nodeWord.reserve(nnodes));
    BT_CUDA(c->blobs.reserve(nwords));
    BT_CUDA(c->compactAnc.reserve(nnodes));
    BT_CUDA(c->parentOrd.reserve(nnodes));
    BT_CUDA(c->fullProgram.reserve(nnodes));
    BT_CUDA(c->roi.reserve(nnodes));
    BT_CUDA(c->frontier.reserve(frontier.size()));
    BT_CUDA(c->upperProgram.reserve(upper.size()));
    BT_CUDA(c->vois.reserve(nprims));
    BT_CUDA(c->rasterVols.reserve(nprims));
    BT_CUDA(c->cullVols.reserve(nprims));
    BT_CUDA(cudaMemsetAsync(c->words.ptr, 0, (nwords + 8) * sizeof(float4), c->stream));
    BT_CUDA(cudaMemcpyAsync(c->words.ptr, data, (size_t)nwords * 16, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->primWords.ptr, primitiveWords, nprims * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->primOrd.ptr, primOrd.data(), nprims * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->nodeWord.ptr, nodeWord.data(), nnodes * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemsetAsync(c->blobs.ptr, 0, (size_t)nwords * 4, c->stream));
    launch_blob_table(c->stream, c->words.ptr, c->nodeWord.ptr, nnodes, c->blobs.ptr);
    BT_CUDA(cudaMemcpyAsync(c->compactAnc.ptr, compactAnc.data(), nnodes * 4, cudaMemcpyHostToDevice, c->stream));
    c->haveAncLists = ancLists;
    if (ancLists) {
        BT_CUDA(c->ancOff.reserve(nnodes + 1));
        BT_CUDA(c->ancIdx.reserve(std::max<size_t>(1, ancIdx.size())));
        BT_CUDA(cudaMemcpyAsync(c->ancOff.ptr, ancOff.data(), (nnodes + 1) * 4, cudaMemcpyHostToDevice, c->stream));
        if (!ancIdx.empty())
            BT_CUDA(cudaMemcpyAsync(c->ancIdx.ptr, ancIdx.data(), ancIdx.size() * 4, cudaMemcpyHostToDevice,
                                    c->stream));
    }
    BT_CUDA(cudaMemcpyAsync(c->parentOrd.ptr, parentOrd.data(), nnodes * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->fullProgram.ptr, program.data(), nnodes * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->frontier.ptr, frontier.data(), frontier.size() * sizeof(uint2), cudaMemcpyHostToDevice,
                            c->stream));
    BT_CUDA(cudaMemcpyAsync(c->upperProgram.ptr, upper.data(), upper.size() * 4, cudaMemcpyHostToDevice, c->stream));
    c->nFrontier = (uint32_t)frontier.size();
    c->nUpper = (uint32_t)upper.size();
    c->upperIsChain = chain ? 1u : 0u;
    c->upperIsMinChain = minChain ? 1u : 0u;
    BT_CUDA(cudaStreamSynchronize(c->stream));
    c->nwords = nwords;
    c->nnodes = nnodes;
    c->nprims = nprims;
    c->nvoi = 0;
    c->fullDepth = maxd;
    c->gradWarps = 0;  // re-sized for the new primitive count on first use
    c->hostNodes.assign(nodes, nodes + nnodes);
    c->hostPrimWords.assign(primitiveWords, primitiveWords + nprims);
    c->treeFromDevice = false;
    c->haveTree = true;
    c->haveRoi = false;
    c->bufEpoch++;
    return BT_OK;
}

int bt_tree_compile(bt_ctx* c, const bt_scene_node* nodes, uint32_t n, uint32_t root, int onDevice) {
    DevGuard dg_(c);
    static_assert(sizeof(bt_scene_node) == sizeof(SceneNodeK), "bt_scene_node layout");
    static_assert(sizeof(bt_node) == sizeof(CompileNodeRec), "bt_node layout");
    if (!c || !nodes) return fail(BT_EINVAL, "null scene graph");
    if (n == 0) return fail(BT_EINVAL, "empty scene graph");
    if (root >= n) return fail(BT_EINVAL, "root index out of range");
    if (n >= BT_ANCESTOR_SENTINEL) return fail(BT_EINVAL, "tree exceeds the 23-bit node index space");
    c->haveAbuffer = false;
    c->haveGbuffer = false;
    c->viewsFrame = false;
    const SceneNodeK* dn = reinterpret_cast<const SceneNodeK*>(nodes);
    if (!onDevice) {
        BT_CUDA(c->cmpNodes.reserve(n));
        BT_CUDA(cudaMemcpyAsync(c->cmpNodes.ptr, nodes, (size_t)n * sizeof(SceneNodeK), cudaMemcpyHostToDevice,
                                c->stream));
        dn = c->cmpNodes.ptr;
    }
    // scratch, carved 16-byte aligned
    const size_t nb = (n + 1023) / 1024 + 1;
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 15) & ~(size_t)15;
        return o;
    };
    const size_t oParent = carve(4 * (size_t)n), oLeft = carve(n), oLm0 = carve(4 * (size_t)n),
                 oLm1 = carve(4 * (size_t)n), oNx0 = carve(4 * (size_t)n), oNx1 = carve(4 * (size_t)n),
                 oV0 = carve(16 * (size_t)n), oV1 = carve(16 * (size_t)n), oTot = carve(16), oErr = carve(16),
                 oA0 = carve(8 * (size_t)n), oA1 = carve(8 * (size_t)n), oF = carve(4 * (size_t)n),
                 oU = carve(4 * (size_t)n), oFP = carve(4 * (size_t)n), oUP = carve(4 * (size_t)n),
                 oBS = carve(4 * nb), oCnt = carve(16), oSize = carve(4 * (size_t)n), oDepth = carve(16),
                 oFlags = carve(16);
    BT_CUDA(c->cmpScratch.reserve(off));
    uint8_t* b = c->cmpScratch.ptr;
    CompileScratch sc;
    sc.parent = reinterpret_cast<int32_t*>(b + oParent);
    sc.isLeft = b + oLeft;
    sc.lm[0] = reinterpret_cast<int32_t*>(b + oLm0);
    sc.lm[1] = reinterpret_cast<int32_t*>(b + oLm1);
    sc.next[0] = reinterpret_cast<int32_t*>(b + oNx0);
    sc.next[1] = reinterpret_cast<int32_t*>(b + oNx1);
    sc.val[0] = reinterpret_cast<uint4*>(b + oV0);
    sc.val[1] = reinterpret_cast<uint4*>(b + oV1);
    sc.totals = reinterpret_cast<uint4*>(b + oTot);
    sc.err = reinterpret_cast<uint32_t*>(b + oErr);
    sc.anc[0] = reinterpret_cast<int2*>(b + oA0);
    sc.anc[1] = reinterpret_cast<int2*>(b + oA1);
    sc.isF = reinterpret_cast<uint32_t*>(b + oF);
    sc.isU = reinterpret_cast<uint32_t*>(b + oU);
    sc.fPos = reinterpret_cast<uint32_t*>(b + oFP);
    sc.uPos = reinterpret_cast<uint32_t*>(b + oUP);
    sc.blockSum = reinterpret_cast<uint32_t*>(b + oBS);
    sc.counts = reinterpret_cast<uint32_t*>(b + oCnt);
    auto errText = [](uint32_t e) -> std::string {
        switch (e & 0xFFu) {
            case kCmpErrKind: return "node kind out of range";
            case kCmpErrChildren: return "operator node must have two children";
            case kCmpErrParents: return "scene graph is not a tree (a node has two parents)";
            case kCmpErrForest: return "scene graph is not one tree rooted at the given root";
            case kCmpErrWords: return "tree exceeds the 23-bit node index space";
            default: return "node parameters invalid (node " + std::to_string(e >> 8) + " in post-order)";
        }
    };
    // phase A: structure + list ranking
    BT_CUDA(cudaMemsetAsync(sc.err, 0xFF, 4, c->stream));
    launch_compile_rank(c->stream, dn, n, root, sc);
    uint32_t hdr[8];
    BT_CUDA(cudaMemcpyAsync(hdr, sc.totals, 32, cudaMemcpyDeviceToHost, c->stream));  // totals + err
    BT_CUDA(cudaStreamSynchronize(c->stream));
    BT_CUDA(cudaGetLastError());
    if (hdr[4] != 0xFFFFFFFFu) return fail(BT_EINVAL, errText(hdr[4]));
    const uint32_t nwords = hdr[0], nprims = hdr[2];
    // phase B: emit into the tree buffers + side tables
    c->haveTree = false;
    BT_CUDA(c->words.reserve(nwords + 8));
    BT_CUDA(c->primWords.reserve(nprims));
    BT_CUDA(c->primOrd.reserve(nprims));
    BT_CUDA(c->nodeWord.reserve(n));
    BT_CUDA(c->blobs.reserve(nwords));
    BT_CUDA(c->compactAnc.reserve(n));
    BT_CUDA(c->parentOrd.reserve(n));
    BT_CUDA(c->fullProgram.reserve(n));
    BT_CUDA(c->roi.reserve(n));
    BT_CUDA(c->frontier.reserve(n));
    BT_CUDA(c->upperProgram.reserve(n));
    BT_CUDA(c->vois.reserve(nprims));
    BT_CUDA(c->rasterVols.reserve(nprims));
    BT_CUDA(c->cullVols.reserve(nprims));
    BT_CUDA(c->cmpRecords.reserve(n));
    BT_CUDA(cudaMemsetAsync(c->words.ptr, 0, (nwords + 8) * sizeof(float4), c->stream));
    BT_CUDA(cudaMemsetAsync(b + oDepth, 0, 16, c->stream));
    CompileOut o;
    o.words = c->words.ptr;
    o.records = c->cmpRecords.ptr;
    o.nodeWord = c->nodeWord.ptr;
    o.program = c->fullProgram.ptr;
    o.size = reinterpret_cast<uint32_t*>(b + oSize);
    o.primWords = c->primWords.ptr;
    o.primOrd = c->primOrd.ptr;
    o.parentOrd = c->parentOrd.ptr;
    o.compactAnc = c->compactAnc.ptr;
    o.frontier = c->frontier.ptr;
    o.upper = c->upperProgram.ptr;
    o.maxDepth = reinterpret_cast<uint32_t*>(b + oDepth);
    constexpr uint32_t kCompileFrontierCap = 16;  // any cap gives the same gradient values (capi.cu upload)
    launch_compile_emit(c->stream, dn, n, sc, o, kCompileFrontierCap);
    uint32_t tail[4];  // err, nFrontier, nUpper, maxDepth
    BT_CUDA(cudaMemcpyAsync(&tail[0], sc.err, 4, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaMemcpyAsync(&tail[1], sc.counts, 8, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaMemcpyAsync(&tail[3], o.maxDepth, 4, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    BT_CUDA(cudaGetLastError());
    if (tail[0] != 0xFFFFFFFFu) return fail(BT_EINVAL, errText(tail[0]));
    uint32_t* flags = reinterpret_cast<uint32_t*>(b + oFlags);
    launch_compile_chain(c->stream, c->upperProgram.ptr, tail[2], flags);
    launch_blob_table(c->stream, c->words.ptr, c->nodeWord.ptr, n, c->blobs.ptr);
    uint32_t fl[2];
    BT_CUDA(cudaMemcpyAsync(fl, flags, 8, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    BT_CUDA(cudaGetLastError());
    c->nwords = nwords;
    c->nnodes = n;
    c->nprims = nprims;
    c->nvoi = 0;
    c->fullDepth = tail[3];
    c->nFrontier = tail[1];
    c->nUpper = tail[2];
    c->upperIsChain = (tail[2] && fl[0]) ? 1u : 0u;
    c->upperIsMinChain = (tail[2] && fl[1]) ? 1u : 0u;
    c->haveAncLists = false;  // k_roi_all walks the compact-ancestor chain
    c->gradWarps = 0;
    c->hostNodes.clear();
    c->hostPrimWords.clear();
    c->treeFromDevice = true;
    c->haveTree = true;
    c->haveRoi = false;
    c->bufEpoch++;
    return BT_OK;
}

int bt_tree_info(bt_ctx* c, uint32_t* nwords, uint32_t* nnodes, uint32_t* nprims) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (nwords) *nwords = c->nwords;
    if (nnodes) *nnodes = c->nnodes;
    if (nprims) *nprims = c->nprims;
    return BT_OK;
}

int bt_tree_nodes_download(bt_ctx* c, bt_node* nodes, uint32_t nnodes, uint32_t* primWords, uint32_t nprims) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (nnodes > c->nnodes || nprims > c->nprims) return fail(BT_EINVAL, "count exceeds the tree");
    if (nodes && nnodes) {
        if (c->treeFromDevice)
            BT_CUDA(cudaMemcpyAsync(nodes, c->cmpRecords.ptr, (size_t)nnodes * sizeof(bt_node), cudaMemcpyDeviceToHost,
                                    c->stream));
        else
            std::memcpy(nodes, c->hostNodes.data(), (size_t)nnodes * sizeof(bt_node));
    }
    if (primWords && nprims)
        BT_CUDA(cudaMemcpyAsync(primWords, c->primWords.ptr, (size_t)nprims * 4, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    return BT_OK;
}

int bt_tree_download(bt_ctx* c, float* data, uint32_t nwords) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (nwords > c->nwords) return fail(BT_EINVAL, "nwords exceeds the uploaded tree");
    BT_CUDA(cudaMemcpyAsync(data, c->words.ptr, (size_t)nwords * 16, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    return BT_OK;
}

int bt_tree_fast_indices(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    BT_CUDA(c->fastScratch.reserve((size_t)c->nnodes * 4));
    launch_fast_indices(c->stream, c->words.ptr, c->nodeWord.ptr, c->parentOrd.ptr, c->nnodes, c->fastScratch.ptr);
    launch_blob_table(c->stream, c->words.ptr, c->nodeWord.ptr, c->nnodes, c->blobs.ptr);
    BT_CUDA(cudaGetLastError());
    return BT_OK;
}

int bt_params_update_device(bt_ctx* c, const uint32_t* dw, const float* dp, const uint32_t* dc, uint32_t n,
                            uint32_t stride) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (n == 0) return BT_OK;
    launch_params_update(c->stream, c->words.ptr, dw, dp, dc, n, stride);
    return BT_OK;
}

int bt_params_update(bt_ctx* c, const uint32_t* words, const float* params, const uint32_t* counts, uint32_t n,
                     uint32_t stride) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (n == 0) return BT_OK;
    if (!words || !params || !counts) return fail(BT_EINVAL, "null parameter buffer");
    for (uint32_t i = 0; i < n; ++i) {
        if (words[i] + 1 + (counts[i] + 3) / 4 > c->nwords || counts[i] > stride)
            return fail(BT_EINVAL, "parameter update outside the tree");
    }
    {  // pinned host buffers: the update kernel reads them over PCIe (see bt_cuda.h)
        const void* host[3] = {words, params, counts};
        void* mapped[3] = {};
        bool ok = true;
        for (int i = 0; i < 3 && ok; ++i) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, host[i]) != cudaSuccess) {
                cudaGetLastError();  // clear the query's error: unregistered memory is not a failure
                ok = false;
                break;
            }
            ok = a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
            mapped[i] = a.devicePointer;
        }
        if (ok) {
            launch_params_update(c->stream, c->words.ptr, static_cast<const uint32_t*>(mapped[0]),
                                 static_cast<const float*>(mapped[1]), static_cast<const uint32_t*>(mapped[2]), n,
                                 stride);
            return BT_OK;
        }
    }
    const bool moved = n > c->pWords.cap || (size_t)n * stride > c->pParams.cap;
    BT_CUDA(c->pWords.reserve(n));
    BT_CUDA(c->pCounts.reserve(n));
    BT_CUDA(c->pParams.reserve((size_t)n * stride));
    if (moved) c->bufEpoch++;
    BT_CUDA(cudaMemcpyAsync(c->pWords.ptr, words, n * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->pCounts.ptr, counts, n * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->pParams.ptr, params, (size_t)n * stride * 4, cudaMemcpyHostToDevice, c->stream));
    launch_params_update(c->stream, c->words.ptr, c->pWords.ptr, c->pParams.ptr, c->pCounts.ptr, n, stride);
    return BT_OK;
}

int bt_roi(bt_ctx* c, float* out, uint32_t nnodes) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    prof_begin(c);
    launch_roi_all(c->stream, dev_tree(c), c->roi.ptr);
    prof_end(c, 0);
    c->haveRoi = true;
    if (out) {
        if (nnodes != c->nnodes) return fail(BT_EINVAL, "roi output size must equal the node count");
        BT_CUDA(cudaMemcpyAsync(out, c->roi.ptr, nnodes * 4, cudaMemcpyDeviceToHost, c->stream));
        BT_CUDA(cudaStreamSynchronize(c->stream));
    }
    return BT_OK;
}

int bt_roi_upload(bt_ctx* c, const float* roi, uint32_t nnodes) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (!roi || nnodes != c->nnodes) return fail(BT_EINVAL, "roi must hold one value per node ordinal");
    BT_CUDA(cudaMemcpyAsync(c->roi.ptr, roi, nnodes * 4, cudaMemcpyHostToDevice, c->stream));
    c->haveRoi = true;
    return BT_OK;
}

int bt_voi_build(bt_ctx* c, float margin) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    if (!c->haveRoi) return fail(BT_ESTATE, "no range of interest computed or uploaded");
    prof_begin(c);
    launch_voi(c->stream, dev_tree(c), c->roi.ptr, margin, c->vois.ptr);
    prof_end(c, 0);
    c->nvoi = c->nprims;
    return BT_OK;
}

int bt_voi_upload(bt_ctx* c, const bt_voi* v, uint32_t n) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (n && !v) return fail(BT_EINVAL, "null volume buffer");
    std::vector<Voi> h(n);
    for (uint32_t i = 0; i < n; ++i) {
        Voi& d = h[i];
        d.family = v[i].family;
        if (d.family > 2u) return fail(BT_EINVAL, "unknown volume family");
        d.word = v[i].primitiveWord;
        d.center = F3{v[i].center[0], v[i].center[1], v[i].center[2]};
        d.radius = v[i].radius;
        d.half = F3{v[i].halfExtents[0], v[i].halfExtents[1], v[i].halfExtents[2]};
        d.rot = Q4{v[i].rotation[0], v[i].rotation[1], v[i].rotation[2], v[i].rotation[3]};
        d.axisEnd = F3{v[i].axisEnd[0], v[i].axisEnd[1], v[i].axisEnd[2]};
    }
    if (n > c->vois.cap) {
        BT_CUDA(c->vois.reserve(n));
        BT_CUDA(c->rasterVols.reserve(n));
        BT_CUDA(c->cullVols.reserve(n));
        c->bufEpoch++;
    }
    if (n) BT_CUDA(cudaMemcpyAsync(c->vois.ptr, h.data(), n * sizeof(Voi), cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    c->nvoi = n;
    return BT_OK;
}

int bt_voi_download(bt_ctx* c, bt_voi* out, uint32_t n) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (n > c->nvoi) return fail(BT_EINVAL, "more volumes requested than built");
    std::vector<Voi> h(n);
    if (n) BT_CUDA(cudaMemcpyAsync(h.data(), c->vois.ptr, n * sizeof(Voi), cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    for (uint32_t i = 0; i < n; ++i) {
        std::memset(&out[i], 0, sizeof(bt_voi));
        out[i].family = (uint8_t)h[i].family;
        out[i].primitiveWord = h[i].word;
        out[i].center[0] = h[i].center.x;
        out[i].center[1] = h[i].center.y;
        out[i].center[2] = h[i].center.z;
        out[i].radius = h[i].radius;
        out[i].halfExtents[0] = h[i].half.x;
        out[i].halfExtents[1] = h[i].half.y;
        out[i].halfExtents[2] = h[i].half.z;
        out[i].rotation[0] = h[i].rot.w;
        out[i].rotation[1] = h[i].rot.x;
        out[i].rotation[2] = h[i].rot.y;
        out[i].rotation[3] = h[i].rot.z;
        out[i].axisEnd[0] = h[i].axisEnd.x;
        out[i].axisEnd[1] = h[i].axisEnd.y;
        out[i].axisEnd[2] = h[i].axisEnd.z;
    }
    return BT_OK;
}

int bt_abuffer_build(bt_ctx* c, const bt_camera* cam, uint32_t tile0, uint32_t tile1) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    int rc = check_camera(cam);
    if (rc) return rc;
    prof_begin(c);
    rc = ensure_image(c, *cam);
    if (rc) return rc;
    rc = resolve_tiles(c, tile0, tile1);
    if (rc) return rc;
    rc = do_camera(c, *cam, tile0, tile1);
    if (rc) return rc;
    rc = do_abuffer(c, *cam, tile0, tile1, true);
    prof_end(c, 1);
    return rc ? rc : launch_status();
}

// The A-buffer as CSR for a download: the per-tile lists (bump order in
// fb.frags) are compacted into tile order on the device (k_frag_csr).
int abuffer_csr(bt_ctx* c, std::vector<uint32_t>& off) {
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    launch_frag_csr(c->stream, frame_bufs(c), tiles, c->smCount);
    off.resize(tiles + 1);
    BT_CUDA(cudaMemcpyAsync(off.data(), c->offsets.ptr, (tiles + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    return launch_status();
}

int bt_abuffer_info(bt_ctx* c, uint64_t* fragments, int32_t* tilesX, int32_t* tilesY) {
    DevGuard dg_(c);
    if (!c || !c->haveAbuffer) return fail(BT_ESTATE, "no A-buffer built");
    std::vector<uint32_t> off;
    const int rc = abuffer_csr(c, off);
    if (rc) return rc;
    if (fragments) *fragments = off.back();
    if (tilesX) *tilesX = c->tilesX;
    if (tilesY) *tilesY = c->tilesY;
    return BT_OK;
}

int bt_abuffer_download(bt_ctx* c, uint32_t* offsets, bt_fragment* frags, uint64_t capacity) {
    DevGuard dg_(c);
    if (!c || !c->haveAbuffer) return fail(BT_ESTATE, "no A-buffer built");
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    std::vector<uint32_t> off;
    const int rc = abuffer_csr(c, off);
    if (rc) return rc;
    if (offsets) std::memcpy(offsets, off.data(), (tiles + 1) * 4);
    if (frags) {
        if (capacity < off[tiles]) return fail(BT_EINVAL, "fragment capacity too small");
        static_assert(sizeof(bt_fragment) == sizeof(Frag), "fragment layout");
        if (off[tiles])
            BT_CUDA(cudaMemcpyAsync(frags, c->unsorted.ptr, (size_t)off[tiles] * sizeof(Frag), cudaMemcpyDeviceToHost,
                                    c->stream));
        BT_CUDA(cudaStreamSynchronize(c->stream));
    }
    return BT_OK;
}

int bt_abuffer_upload(bt_ctx* c, const bt_camera* cam, const uint32_t* offsets, const bt_fragment* frags) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    int rc = check_camera(cam);
    if (rc) return rc;
    if (!offsets) return fail(BT_EINVAL, "null offsets");
    rc = do_camera(c, *cam);
    if (rc) return rc;
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    const uint32_t total = offsets[tiles];
    if (total && !frags) return fail(BT_EINVAL, "null fragments");
    for (uint32_t i = 0; i < tiles; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(BT_EINVAL, "offsets must be non-decreasing");
    rc = ensure_frame_caps(c, std::max<uint32_t>(c->sbCap, 256u), std::max<size_t>(total, 1u << 16));
    if (rc) return rc;
    BT_CUDA(cudaMemcpyAsync(c->offsets.ptr, offsets, (tiles + 1) * 4, cudaMemcpyHostToDevice, c->stream));
    if (total)
        BT_CUDA(cudaMemcpyAsync(c->frags.ptr, frags, (size_t)total * sizeof(Frag), cudaMemcpyHostToDevice, c->stream));
    launch_tile_frag_from_offsets(c->stream, frame_bufs(c), tiles);
    BT_CUDA(cudaMemcpyAsync(c->counters.ptr + kCntFrags, &total, 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    c->haveAbuffer = true;
    return launch_status();
}

int bt_trace(bt_ctx* c, const bt_camera* cam, const bt_render_config* cfg, uint32_t tile0, uint32_t tile1,
             int exact) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    int rc = check_camera(cam);
    if (rc) return rc;
    rc = check_config(cfg);
    if (rc) return rc;
    if (!c->haveAbuffer) return fail(BT_ESTATE, "no A-buffer built");
    if (cam->width != c->width || cam->height != c->height)
        return fail(BT_EINVAL, "camera image size differs from the A-buffer's");
    rc = resolve_tiles(c, tile0, tile1);
    if (rc) return rc;
    if (!rays_cover(c, *cam, tile0, tile1)) {
        rc = do_camera(c, *cam);
        if (rc) return rc;
    }
    if (rc) return rc;
    prof_begin(c);
    rc = do_trace(c, *cam, *cfg, tile0, tile1, exact, true);
    prof_end(c, 2);
    return rc ? rc : launch_status();
}

int bt_normals(bt_ctx* c, const bt_camera* cam, int mode, int exact) {
    DevGuard dg_(c);
    if (!c || !c->haveGbuffer) return fail(BT_ESTATE, "no G-buffer rendered");
    int rc = check_camera(cam);
    if (rc) return rc;
    if (mode != 0 && mode != 1) return fail(BT_EINVAL, "unknown normals mode");
    prof_begin(c);
    if (!rays_cover(c, *cam, 0, (uint32_t)(c->tilesX * c->tilesY))) {  // e.g. after a sharded, normal-less frame
        rc = do_camera(c, *cam);
        if (rc) return rc;
    }
    rc = do_normals(c, *cam, mode, exact);
    prof_end(c, 3);
    return rc ? rc : launch_status();
}

int bt_normals_rows(bt_ctx* c, const bt_camera* cam, int mode, int exact, uint32_t tile0, uint32_t tile1) {
    DevGuard dg_(c);
    if (!c || !c->haveGbuffer) return fail(BT_ESTATE, "no G-buffer rendered");
    int rc = check_camera(cam);
    if (rc) return rc;
    if (mode != 0 && mode != 1) return fail(BT_EINVAL, "unknown normals mode");
    rc = resolve_tiles(c, tile0, tile1);
    if (rc) return rc;
    if (tile1 <= tile0) return BT_OK;
    // the rows' pixels, plus one pixel row of halo on each side for the rays
    const uint32_t tx = (uint32_t)c->tilesX, tiles = (uint32_t)(c->tilesX * c->tilesY);
    const uint32_t r0 = tile0 / tx, r1 = (tile1 + tx - 1) / tx;
    const uint32_t h0 = r0 > 0 ? (r0 - 1) * tx : 0u, h1 = std::min(tiles, (r1 + 1) * tx);
    if (!rays_cover(c, *cam, h0, h1)) {
        rc = do_camera(c, *cam, h0, h1);
        if (rc) return rc;
    }
    prof_begin(c);
    rc = do_normals(c, *cam, mode, exact, (int)(r0 * kTile), std::min((int)(r1 * kTile), c->height), true);
    prof_end(c, 3);
    return rc ? rc : launch_status();
}

int bt_oracle_render(bt_ctx* c, const bt_camera* cam, const bt_render_config* cfg, int exact) {
    DevGuard dg_(c);
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    int rc = check_camera(cam);
    if (rc) return rc;
    rc = check_config(cfg);
    if (rc) return rc;
    if (c->fullDepth > 128) return fail(BT_EINVAL, "full-tree evaluation stack deeper than 128 entries");
    rc = do_camera(c, *cam);
    if (rc) return rc;
    launch_oracle(c->stream, exact != 0, dev_tree(c), to_cam(*cam), trace_params(*cfg, *cam), frame_bufs(c), gbuf(c),
                  c->stats.ptr);
    BT_CUDA(cudaMemsetAsync(c->tileMaxOverlap.ptr, 0, c->tileMaxOverlap.cap * 4, c->stream));
    BT_CUDA(cudaMemsetAsync(c->tileCacheBytes.ptr, 0, c->tileCacheBytes.cap * 4, c->stream));
    BT_CUDA(cudaMemsetAsync(c->tileError.ptr, 0, c->tileError.cap, c->stream));
    c->haveGbuffer = true;
    c->viewsFrame = false;
    return launch_status();
}

int bt_render_frame(bt_ctx* c, const bt_camera* cam, const bt_render_config* cfg, uint32_t tile0, uint32_t tile1,
                    int exact, int flags) {
    DevGuard dg_(c);
    const bool use_graph = (flags & BT_FRAME_GRAPH) != 0;
    const bool normals = (flags & BT_FRAME_NO_NORMALS) == 0;
    if (!c || !c->haveTree) return fail(BT_ESTATE, "no tree uploaded");
    int rc = check_camera(cam);
    if (rc) return rc;
    rc = check_config(cfg);
    if (rc) return rc;
    rc = ensure_image(c, *cam);
    if (rc) return rc;
    rc = resolve_tiles(c, tile0, tile1);
    if (rc) return rc;
    if (c->fullDepth > 128) return fail(BT_EINVAL, "full-tree evaluation stack deeper than 128 entries");
    const int mode = cfg->normalsMode;
    auto enqueue = [&](bool checked) -> int {
        struct Reset {
            bool& f;
            ~Reset() { f = false; }
        } reset{c->prezeroed};
        // normals need every ray of the image (they run over the assembled frame)
        const uint32_t c0 = normals ? 0u : tile0, c1 = normals ? 0u : tile1;
        int r = BT_OK;
        if (!checked) {  // captured frame: the camera pass runs beside ROI + VOIs
            r = ensure_side(c);
            if (r) return r;
            BT_CUDA(cudaEventRecord(c->evFork[0], c->stream));
            BT_CUDA(cudaStreamWaitEvent(c->side, c->evFork[0], 0));
            r = do_camera(c, *cam, c0, c1, c->side);
            if (r) return r;
            // the frame's counters and per-tile cursors, zeroed here instead of
            // in front of each stage
            const size_t nsb = superblock_count(c->tilesX, c->tilesY);
            BT_CUDA(cudaMemsetAsync(c->counters.ptr, 0, kCntSlots * sizeof(uint32_t), c->side));
            BT_CUDA(cudaMemsetAsync(c->sbCount.ptr, 0, nsb * sizeof(uint32_t), c->side));
            BT_CUDA(cudaMemsetAsync(c->tileQueue.ptr, 0, sizeof(uint32_t), c->side));
            BT_CUDA(cudaEventRecord(c->evJoin[0], c->side));
            c->prezeroed = true;
        }
        launch_roi_all(c->stream, dev_tree(c), c->roi.ptr);
        launch_voi(c->stream, dev_tree(c), c->roi.ptr, cfg->hitEpsilon, c->vois.ptr);
        c->haveRoi = true;
        c->nvoi = c->nprims;
        if (checked) r = do_camera(c, *cam, c0, c1);
        else BT_CUDA(cudaStreamWaitEvent(c->stream, c->evJoin[0], 0));
        if (r) return r;
        // one per-tile pass builds each tile's fragment list AND its interval records
        const TraceParams tp = trace_params(*cfg, *cam, c->stepBound);
        if (c->depthSlabs <= 1) {
            r = do_abuffer(c, *cam, tile0, tile1, checked, kTileRaster | kTileViews, &tp);
            if (r) return r;
            r = do_trace(c, *cam, *cfg, tile0, tile1, exact, checked, true);
            if (r) return r;
        } else {
            // depth slabs (PAPER.md "Conclusion": processing by depth slabs limits
            // the A-buffer's memory): A-buffer, records and march per slab, front
            // to back; rays that hit stay done
            for (int sl = 0; sl < c->depthSlabs; ++sl) {
                const bt_camera cs = slab_camera(*cam, sl, c->depthSlabs);
                TraceParams tps = trace_params(*cfg, cs, c->stepBound);
                tps.window = tp.window;
                if (sl > 0) c->prezeroed = false;  // the frame's counters, again for this slab
                r = do_abuffer(c, cs, tile0, tile1, checked, kTileRaster | kTileViews, &tps);
                if (r) return r;
                r = do_trace(c, cs, *cfg, tile0, tile1, exact, checked, true, sl, tp.window);
                if (r) return r;
            }
        }
        return normals ? do_normals(c, *cam, mode, exact) : BT_OK;
    };
    if (!use_graph) {
        rc = enqueue(true);
        return rc ? rc : launch_status();
    }

    FrameKey key;
    std::memset(&key, 0, sizeof(key));
    key.cam = *cam;
    key.cfg = *cfg;
    key.tile0 = tile0;
    key.tile1 = tile1;
    key.exact = exact | (normals ? 0 : 2);
    key.bufEpoch = c->bufEpoch;
    if (!c->haveGraph || !(key == c->graphKey)) {
        // eager, capacity-checked frame first (grows buffers), then capture
        rc = enqueue(true);
        if (!rc) rc = launch_status();
        if (rc) return rc;
        BT_CUDA(cudaStreamSynchronize(c->stream));
        key.bufEpoch = c->bufEpoch;
        if (c->graph) {
            cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
        }
        cudaGraph_t g = nullptr;
        BT_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        rc = enqueue(false);
        cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(BT_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        {
            size_t nn = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            cudaGraphGetNodes(g, nodes.data(), &nn);
            uint32_t kernels = 0;
            for (auto& n : nodes) {
                cudaGraphNodeType ty;
                cudaGraphNodeGetType(n, &ty);
                if (ty == cudaGraphNodeTypeKernel) ++kernels;
            }
            c->graphKernels = kernels;
            c->graphNodes = (uint32_t)nn;
        }
        ce = cudaGraphInstantiate(&c->graph, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return fail(BT_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
        c->graphKey = key;
        c->haveGraph = true;
        return BT_OK;  // the eager frame already produced this frame's output
    }
    BT_CUDA(cudaGraphLaunch(c->graph, c->stream));
    return BT_OK;
}

int bt_graph_kernel_count(bt_ctx* c, uint32_t* kernels, uint32_t* nodes) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (kernels) *kernels = c->haveGraph ? c->graphKernels : 0;
    if (nodes) *nodes = c->haveGraph ? c->graphNodes : 0;
    return BT_OK;
}

int bt_gbuffer_download(bt_ctx* c, uint8_t* hit, float* depth, float* normal, uint32_t* evalCount,
                        uint32_t* tileMaxOverlap, uint32_t* tileCacheBytes, uint8_t* tileError) {
    DevGuard dg_(c);
    if (!c || !c->haveGbuffer) return fail(BT_ESTATE, "no G-buffer rendered");
    const size_t px = (size_t)c->width * c->height, tiles = (size_t)c->tilesX * c->tilesY;
    cudaStream_t s = c->stream;
    if (hit) BT_CUDA(cudaMemcpyAsync(hit, c->hit.ptr, px, cudaMemcpyDeviceToHost, s));
    if (depth) BT_CUDA(cudaMemcpyAsync(depth, c->depth.ptr, px * 4, cudaMemcpyDeviceToHost, s));
    if (normal) BT_CUDA(cudaMemcpyAsync(normal, c->normal.ptr, px * 12, cudaMemcpyDeviceToHost, s));
    if (evalCount) BT_CUDA(cudaMemcpyAsync(evalCount, c->evalCount.ptr, px * 4, cudaMemcpyDeviceToHost, s));
    if (tileMaxOverlap)
        BT_CUDA(cudaMemcpyAsync(tileMaxOverlap, c->tileMaxOverlap.ptr, tiles * 4, cudaMemcpyDeviceToHost, s));
    if (tileCacheBytes)
        BT_CUDA(cudaMemcpyAsync(tileCacheBytes, c->tileCacheBytes.ptr, tiles * 4, cudaMemcpyDeviceToHost, s));
    if (tileError) BT_CUDA(cudaMemcpyAsync(tileError, c->tileError.ptr, tiles, cudaMemcpyDeviceToHost, s));
    BT_CUDA(cudaStreamSynchronize(s));
    BT_CUDA(cudaGetLastError());
    return BT_OK;
}

namespace {
// slab = true: the seven planes lie at bt_gbuffer_layout's offsets of ONE
// caller allocation, so adjacent planes may be copied as one range (a copy
// must never span two separately pinned allocations)
int download_async(bt_ctx* c, void* const* planes, bool slab) {
    void* hit = planes[0];
    void* depth = planes[1];
    void* normal = planes[2];
    void* evalCount = planes[3];
    void* tileMaxOverlap = planes[4];
    void* tileCacheBytes = planes[5];
    void* tileError = planes[6];
    const size_t px = (size_t)c->width * c->height, tiles = (size_t)c->tilesX * c->tilesY;
    // plane layout of a snapshot slot (16-byte aligned offsets)
    const size_t sz[7] = {px, px * 4, px * 12, px * 4, tiles * 4, tiles * 4, tiles};
    const void* src[7] = {c->hit.ptr, c->depth.ptr, c->normal.ptr, c->evalCount.ptr,
                          c->tileMaxOverlap.ptr, c->tileCacheBytes.ptr, c->tileError.ptr};
    void* dst[7] = {hit, depth, normal, evalCount, tileMaxOverlap, tileCacheBytes, tileError};
    size_t off[7], total = 0;
    for (int i = 0; i < 7; ++i) {
        off[i] = total;
        total += (sz[i] + 15) & ~(size_t)15;
    }
    if (!c->copyStream) {
        BT_CUDA(cudaStreamCreateWithFlags(&c->copyStream, cudaStreamNonBlocking));
        BT_CUDA(cudaStreamCreateWithFlags(&c->copyStream2, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            BT_CUDA(cudaEventCreateWithFlags(&c->evSnap[i], cudaEventDisableTiming));
            BT_CUDA(cudaEventCreateWithFlags(&c->evCopied[i], cudaEventDisableTiming));
            BT_CUDA(cudaEventCreateWithFlags(&c->evCopied2[i], cudaEventDisableTiming));
        }
    }
    const int slot = c->dlSlot;
    c->dlSlot ^= 1;
    if (c->dlPending[slot]) {  // the slot is free again once both halves of its last copy are done
        BT_CUDA(cudaStreamWaitEvent(c->stream, c->evCopied[slot], 0));
        BT_CUDA(cudaStreamWaitEvent(c->stream, c->evCopied2[slot], 0));
    }
    if (c->snap[slot].cap < total) {
        BT_CUDA(cudaStreamSynchronize(c->copyStream));
        BT_CUDA(cudaStreamSynchronize(c->copyStream2));
        BT_CUDA(c->snap[slot].reserve(total));
    }
    uint8_t* base = c->snap[slot].ptr;
    {  // snapshot with an SM copy kernel: the copy engines are busy with the D2H
        const void* s7[7];
        void* d7[7];
        for (int i = 0; i < 7; ++i) {
            s7[i] = dst[i] ? src[i] : nullptr;
            d7[i] = base + off[i];
        }
        launch_copy_segments(c->stream, s7, d7, sz, 7, c->smCount);
    }
    BT_CUDA(cudaEventRecord(c->evSnap[slot], c->stream));
    // Host planes laid out like the snapshot slot (bt_gbuffer_layout: one
    // pinned slab) merge into one contiguous run; the runs then go down split
    // by bytes over two copy streams -- one D2H stream reaches ~44 GB/s on
    // this PCIe link, two concurrent ones ~55 GB/s, and every extra copy
    // costs a few microseconds of DMA setup.
    struct Run {
        uint8_t* d;
        const uint8_t* s;
        size_t n;
    };
    Run runs[7];
    int nr = 0;
    size_t bytes = 0;
    for (int i = 0; i < 7; ++i) {
        if (!dst[i]) continue;
        uint8_t* d = static_cast<uint8_t*>(dst[i]);
        const uint8_t* sp = base + off[i];
        Run& last = runs[nr > 0 ? nr - 1 : 0];
        if (slab && nr > 0 && (last.n & 15) == 0 && last.d + last.n == d && last.s + last.n == sp) {
            last.n += sz[i];
        } else {
            // a run ending in a padded plane is closed: its padding is not the caller's memory
            runs[nr++] = Run{d, sp, sz[i]};
        }
        bytes += sz[i];
    }
    BT_CUDA(cudaStreamWaitEvent(c->copyStream, c->evSnap[slot], 0));
    BT_CUDA(cudaStreamWaitEvent(c->copyStream2, c->evSnap[slot], 0));
    const size_t half = (bytes / 2 + 15) & ~(size_t)15;
    size_t done = 0;
    for (int r = 0; r < nr; ++r) {
        const Run& u = runs[r];
        // bytes of this run that fall in the first half of the total
        const size_t first = done >= half ? 0 : std::min(u.n, half - done);
        if (first) BT_CUDA(cudaMemcpyAsync(u.d, u.s, first, cudaMemcpyDeviceToHost, c->copyStream));
        if (u.n > first)
            BT_CUDA(cudaMemcpyAsync(u.d + first, u.s + first, u.n - first, cudaMemcpyDeviceToHost, c->copyStream2));
        done += u.n;
    }
    BT_CUDA(cudaEventRecord(c->evCopied[slot], c->copyStream));
    BT_CUDA(cudaEventRecord(c->evCopied2[slot], c->copyStream2));
    c->dlPending[slot] = true;
    return BT_OK;
}
}  // namespace

int bt_gbuffer_download_async(bt_ctx* c, uint8_t* hit, float* depth, float* normal, uint32_t* evalCount,
                              uint32_t* tileMaxOverlap, uint32_t* tileCacheBytes, uint8_t* tileError) {
    DevGuard dg_(c);
    if (!c || !c->haveGbuffer) return fail(BT_ESTATE, "no G-buffer rendered");
    void* const planes[7] = {hit, depth, normal, evalCount, tileMaxOverlap, tileCacheBytes, tileError};
    return download_async(c, planes, false);
}

int bt_gbuffer_download_async_slab(bt_ctx* c, void* slab) {
    DevGuard dg_(c);
    if (!c || !c->haveGbuffer) return fail(BT_ESTATE, "no G-buffer rendered");
    if (!slab) return fail(BT_EINVAL, "slab is null");
    size_t off[7], total = 0;
    const int rc = bt_gbuffer_layout(c, off, &total);
    if (rc != BT_OK) return rc;
    void* planes[7];
    for (int i = 0; i < 7; ++i) planes[i] = static_cast<uint8_t*>(slab) + off[i];
    return download_async(c, planes, true);
}

int bt_gbuffer_layout(bt_ctx* c, size_t offsets[7], size_t* total) {
    DevGuard dg_(c);
    if (!c || !offsets || !total) return fail(BT_EINVAL, "null argument");
    if (c->width <= 0 || c->height <= 0) return fail(BT_ESTATE, "no image size yet (upload a camera or render first)");
    const size_t px = (size_t)c->width * c->height, tiles = (size_t)c->tilesX * c->tilesY;
    const size_t sz[7] = {px, px * 4, px * 12, px * 4, tiles * 4, tiles * 4, tiles};
    size_t t = 0;
    for (int i = 0; i < 7; ++i) {
        offsets[i] = t;
        t += (sz[i] + 15) & ~(size_t)15;
    }
    *total = t;
    return BT_OK;
}

int bt_set_tile_order(bt_ctx* c, const uint32_t* order, uint32_t n) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    const uint32_t tiles = (uint32_t)(c->tilesX * c->tilesY);
    if (n != tiles || !order) return fail(BT_EINVAL, "tile order must list every tile of the image once");
    std::vector<uint8_t> seen(tiles, 0);
    for (uint32_t i = 0; i < n; ++i) {
        if (order[i] >= tiles || seen[order[i]]) return fail(BT_EINVAL, "tile order is not a permutation");
        seen[order[i]] = 1;
    }
    BT_CUDA(cudaMemcpyAsync(c->tileOrder.ptr, order, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->hostUnits.ptr, &n, 4, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    c->schedMode = 2;
    c->bufEpoch++;
    return BT_OK;
}

int bt_set_step_bound(bt_ctx* c, int mode) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (mode != 0 && mode != 1) return fail(BT_EINVAL, "step bound mode must be 0 or 1");
    if (mode != c->stepBound) {
        c->stepBound = mode;
        c->bufEpoch++;  // re-capture the frame graph
    }
    return BT_OK;
}

int bt_set_depth_slabs(bt_ctx* c, int slabs) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (slabs < 1 || slabs > 64) return fail(BT_EINVAL, "depth slabs must lie in [1, 64]");
    if (slabs != c->depthSlabs) {
        c->depthSlabs = slabs;
        c->bufEpoch++;  // re-capture the frame graph
    }
    return BT_OK;
}

int bt_set_scheduling(bt_ctx* c, int mode) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (mode != 0 && mode != 1) return fail(BT_EINVAL, "scheduling mode must be 0 (raster) or 1 (longest-first)");
    c->schedMode = mode;
    c->bufEpoch++;
    return BT_OK;
}

int bt_gbuffer_export(bt_ctx* c, bt_ipc_handles* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(BT_EINVAL, "null argument");
    if (!c->hit.ptr) return fail(BT_ESTATE, "no G-buffer allocated (render a frame first)");
    void* planes[7] = {c->hit.ptr, c->depth.ptr, c->evalCount.ptr, c->tileMaxOverlap.ptr, c->tileCacheBytes.ptr,
                       c->tileError.ptr, c->normal.ptr};
    for (int i = 0; i < 7; ++i) {
        cudaIpcMemHandle_t h;
        BT_CUDA(cudaIpcGetMemHandle(&h, planes[i]));
        static_assert(sizeof(h) == sizeof(out->plane[0]), "IPC handle size");
        std::memcpy(out->plane[i], &h, sizeof(h));
    }
    out->width = c->width;
    out->height = c->height;
    return BT_OK;
}

int bt_gbuffer_import(bt_ctx* c, const bt_ipc_handles* in) {
    DevGuard dg_(c);
    if (!c || !in) return fail(BT_EINVAL, "null argument");
    release_remote(c);
    for (int i = 0; i < 7; ++i) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, in->plane[i], sizeof(h));
        void* q = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            release_remote(c);
            return fail(BT_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
        c->remote.p[i] = q;
    }
    c->remote.on = true;
    c->remote.width = in->width;
    c->remote.height = in->height;
    c->bufEpoch++;
    return BT_OK;
}

int bt_gbuffer_import_release(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    release_remote(c);
    return BT_OK;
}

int bt_download_wait(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    if (c->copyStream) BT_CUDA(cudaStreamSynchronize(c->copyStream));
    if (c->copyStream2) BT_CUDA(cudaStreamSynchronize(c->copyStream2));
    BT_CUDA(cudaGetLastError());
    return BT_OK;
}

int bt_gbuffer_device(bt_ctx* c, bt_gbuffer_view* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(BT_EINVAL, "null argument");
    out->hit = c->hit.ptr;
    out->depth = c->depth.ptr;
    out->normal = c->normal.ptr;
    out->evalCount = c->evalCount.ptr;
    out->tileMaxOverlap = c->tileMaxOverlap.ptr;
    out->tileCacheBytes = c->tileCacheBytes.ptr;
    out->tileError = c->tileError.ptr;
    out->width = c->width;
    out->height = c->height;
    out->tilesX = c->tilesX;
    out->tilesY = c->tilesY;
    return BT_OK;
}

int bt_gbuffer_upload(bt_ctx* c, const bt_camera* cam, const uint8_t* hit, const float* depth) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    int rc = check_camera(cam);
    if (rc) return rc;
    if (!hit || !depth) return fail(BT_EINVAL, "null G-buffer plane");
    rc = do_camera(c, *cam);
    if (rc) return rc;
    const size_t px = (size_t)c->width * c->height;
    BT_CUDA(cudaMemcpyAsync(c->hit.ptr, hit, px, cudaMemcpyHostToDevice, c->stream));
    BT_CUDA(cudaMemcpyAsync(c->depth.ptr, depth, px * 4, cudaMemcpyHostToDevice, c->stream));
    c->haveGbuffer = true;
    c->viewsFrame = false;
    return BT_OK;
}

int bt_stats_download(bt_ctx* c, bt_stats* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(BT_EINVAL, "null argument");
    uint64_t st[kStSlots];
    uint32_t cnt[kCntSlots];
    BT_CUDA(cudaMemcpyAsync(st, c->stats.ptr, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaMemcpyAsync(cnt, c->counters.ptr, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
    BT_CUDA(cudaStreamSynchronize(c->stream));
    std::memset(out, 0, sizeof(*out));
    out->fieldEvals = st[kStFieldEvals];
    out->retainedNodeVisits = st[kStRetained];
    out->primitiveEvals = st[kStPrimEvals];
    out->treeNodeCount = c->nnodes;
    out->maxOverlap = (uint32_t)st[kStMaxOverlap];
    out->maxCacheBytes = (uint32_t)st[kStMaxCache];
    out->fieldFlops = st[kStFlops];
    out->candidatePairs = cnt[kCntPool];
    out->tileErrors = st[kStTileErrors];
    out->normalFallbacks = st[kStFallbacks];
    out->warpSteps = st[kStWarpSteps];
    if (c->haveAbuffer) out->fragments = cnt[kCntFrags];  // the per-tile lists' total (k_tile)
    if (cnt[kCntOverflow] || cnt[kCntSbNeed])
        return fail(BT_ENOMEM, "A-buffer capacity overflowed during a graph replay; re-run eagerly");
    if (c->vCounters.ptr) {
        uint32_t vc[2] = {0u, 0u};
        BT_CUDA(cudaMemcpyAsync(vc, c->vCounters.ptr, sizeof(vc), cudaMemcpyDeviceToHost, c->stream));
        BT_CUDA(cudaStreamSynchronize(c->stream));
        if (vc[1]) return fail(BT_ENOMEM, "interval-record capacity overflowed during a graph replay; re-run eagerly");
    }
    return BT_OK;
}

int bt_stats_reset(bt_ctx* c) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    BT_CUDA(cudaMemsetAsync(c->stats.ptr, 0, kStSlots * sizeof(uint64_t), c->stream));
    return BT_OK;
}

int bt_profile_enable(bt_ctx* c, int on) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    c->profiling = on != 0;
    for (int i = 0; i < kProfSlots; ++i) {
        c->profMs[i] = 0.f;
        c->profLaunch[i] = 0;
    }
    return BT_OK;
}

int bt_profile_read(bt_ctx* c, float* ms4, uint32_t* l4) { return bt_profile_read_ex(c, ms4, l4, 4); }

int bt_profile_read_ex(bt_ctx* c, float* ms, uint32_t* launches, uint32_t nslots) {
    DevGuard dg_(c);
    if (!c) return fail(BT_EINVAL, "ctx is null");
    for (uint32_t i = 0; i < nslots && i < (uint32_t)kProfSlots; ++i) {
        if (ms) ms[i] = c->profMs[i];
        if (launches) launches[i] = c->profLaunch[i];
    }
    return BT_OK;
}

}  // extern "C"
