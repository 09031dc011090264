// bt_device.h -- kernel argument blocks and launchers (internal to
// libblobtree_b200.so; the public boundary is include/bt_cuda.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bt_views.cuh"

namespace btk {

// Superblock = 8x8 tiles (64x64 pixels): unit of the coarse cone cull.
constexpr int kSB = 8;
constexpr uint32_t kScanBlockElems = 4096;  // elements per block of the single-pass scan (k_frame.cu)

struct DevTree {
    const float4* words = nullptr;
    const uint32_t* blobs = nullptr;       // blob header of each node, indexed by its word (dense: the view
                                           // build's ancestor walks read 4 B per node instead of a float4's .x)
    const uint32_t* primWords = nullptr;   // ascending word of each primitive
    const uint32_t* primOrd = nullptr;     // node ordinal of each primitive
    const uint32_t* nodeWord = nullptr;    // word of each node ordinal
    const int32_t* compactAnc = nullptr;   // nearest strict compact ancestor ordinal, -1 none
    // every node's compact strict ancestors as a CSR list of their parameter
    // words (ancOff[nnodes + 1], ancIdx): ROI loads them independently instead
    // of walking the chain (deep trees); null when the lists would be too long
    const uint32_t* ancOff = nullptr;
    const uint32_t* ancIdx = nullptr;
    const uint32_t* fullProgram = nullptr; // post-order (isPrim<<31 | op<<26 | word)
    uint32_t nwords = 0, nnodes = 0, nprims = 0;
    uint32_t fullDepth = 0;                // max stack depth of a full post-order walk
    // frontier decomposition of the full tree (gradient-normal fallback):
    // subtrees of <= kFrontierMax nodes, evaluated in parallel, then the
    // remaining upper operators in post-order over their values
    const uint2* frontier = nullptr;       // ordinal range [lo, hi] per subtree
    const uint32_t* upperProgram = nullptr;// bit31 ? load frontier value : (op<<26 | word)
    uint32_t nFrontier = 0, nUpper = 0;
    uint32_t upperIsChain = 0;  // upper program = F0 (Fi op)*: left comb, register accumulator
    uint32_t upperIsMinChain = 0;  // ... and every op is a sharp union: exact parallel (value, index) min
};
constexpr uint32_t kFrontierMax = 32;
constexpr size_t kGradSmemBytes = 160 * 1024;  // frontier values kept in shared memory up to this size

struct FrameBufs {
    // camera products
    float4* rays = nullptr;      // [tiles*64] dir.xyz, dot(dir, forward); tile-major
    float4* cones = nullptr;     // [tiles] axis.xyz, cos
    float* coneSin = nullptr;    // [tiles]
    float4* sbCones = nullptr;   // [superblocks] axis.xyz, half-angle (rad, conservative)
    float4* tileFrustum = nullptr; // [tiles*4] inward unit normals of the pixel-centre pyramid
    float4* sbFrustum = nullptr;   // [superblocks*4] same for the superblock
    // A-buffer
    uint4* pool = nullptr;       // (tile, voi, entry bits, exit bits), unsorted
    uint4* unsorted = nullptr;   // CSR slots: (word, entry, exit, voi)
    Frag* frags = nullptr;       // CSR slots, sorted by (zEntry, word)
    uint32_t* tileCount = nullptr;
    uint32_t* tileCursor = nullptr;
    uint32_t* tileLocal = nullptr;   // exclusive scan inside a 4096-tile block
    uint32_t* blockSum = nullptr;    // per scan block
    uint32_t* blockPrefix = nullptr; // exclusive over scan blocks (+ total at [nblocks])
    uint32_t* offsets = nullptr;     // CSR [tiles+1] (built on demand for downloads, k_frag_csr)
    uint32_t* counters = nullptr;    // see kCnt*
    // (volume, superblock) pairs grouped by superblock (k_tile's candidates)
    uint32_t* sbCount = nullptr;     // [superblocks] pairs per superblock
    uint32_t* sbList = nullptr;      // [superblocks * sbCap] volume indices: superblock sb's candidates at sb * sbCap
    uint2* tileFrag = nullptr;       // [tiles] (first fragment, count) of each tile's sorted list in frags
    struct CullVol* cullVols = nullptr;  // [volumes] cull terms for the frame's camera (k_pairs -> k_tile_raster)
    RasterVol* rasterVols = nullptr; // [volumes] ray-test terms for the frame's camera (k_pairs -> k_tile_raster)
    uint64_t poolCap = 0, fragCap = 0;
    uint32_t sbCap = 0;              // candidates per superblock list (k_pairs fills them directly)
};

// device counters (uint32 slots)
enum : int {
    kCntPairs = 0,
    kCntPool = 1,
    kCntScanDone = 2,
    kCntCandidates = 3,
    kCntFallback = 4,
    kCntOverflow = 5,
    kCntFallbackHard = 6,  // fast-path fallbacks without a usable view (full-tree gradient)
    kCntFrags = 7,         // fragments allocated (k_tile bump allocator)
    kCntTileQueue = 9,     // k_tile work queue head
    kCntSbNeed = 11,       // a superblock list overflowed: the capacity it needed (0: none)
    kCntSlots = 12
};

// device statistics (uint64 slots)
enum : int {
    kStFieldEvals = 0,
    kStRetained,
    kStPrimEvals,
    kStFlops,
    kStMaxOverlap,
    kStMaxCache,
    kStTileErrors,
    kStFallbacks,
    kStWarpSteps,  // lockstep march iterations (x32 lanes = evaluation slots offered)
    kStSlots
};

struct GBuf {
    uint8_t* hit = nullptr;
    float* depth = nullptr;
    float* normal = nullptr;  // xyz interleaved
    uint32_t* evalCount = nullptr;
    uint32_t* tileMaxOverlap = nullptr;
    uint32_t* tileCacheBytes = nullptr;
    uint8_t* tileError = nullptr;
    uint32_t* fallback = nullptr;  // pixel indices needing the gradient normal
    int width = 0, height = 0, tilesX = 0, tilesY = 0;
    int remote = 0;  // the planes are another GPU's (fused gather): fence the writes system-wide
    int accumulate = 0;  // depth slab > 0: the march continues the planes of the earlier slabs
};

inline Cam make_cam(const float* pos, const float* fwd, const float* right, const float* up,
                    float tanHalf, float aspect, float invNear, float invDepthRange, float nearZ,
                    float farZ, int w, int h) {
    Cam c;
    c.pos = F3{pos[0], pos[1], pos[2]};
    c.fwd = F3{fwd[0], fwd[1], fwd[2]};
    c.right = F3{right[0], right[1], right[2]};
    c.up = F3{up[0], up[1], up[2]};
    c.tanHalf = tanHalf;
    c.aspect = aspect;
    c.invNear = invNear;
    c.invDepthRange = invDepthRange;
    c.nearZ = nearZ;
    c.farZ = farZ;
    c.width = w;
    c.height = h;
    return c;
}

// ---- launchers (k_frame.cu) -------------------------------------------
void launch_params_update(cudaStream_t st, float4* words, const uint32_t* dWords,
                          const float* dParams, const uint32_t* dCounts, uint32_t n,
                          uint32_t stride);
void launch_roi_all(cudaStream_t st, const DevTree& t, float* roi);
void launch_voi(cudaStream_t st, const DevTree& t, const float* roi, float margin, Voi* vois);
// rays, tile cones and pyramids of the superblock rows meeting [tile0, tile1)
void launch_camera(cudaStream_t st, const Cam& cam, const FrameBufs& fb, int tilesX, int tilesY, uint32_t tile0,
                   uint32_t tile1);
// tiles [*cover0, return) whose rays launch_camera(tile0, tile1) computes
uint32_t camera_tile_cover(int tilesX, int tilesY, uint32_t tile0, uint32_t tile1, uint32_t* cover0);
void launch_abuffer(cudaStream_t st, const Cam& cam, const Voi* vois, uint32_t nvoi,
                    const FrameBufs& fb, int tilesX, int tilesY, uint32_t tile0, uint32_t tile1,
                    int smCount, bool zero = true);
// k_tile, warp per tile of [tile0, tile1): raster (the tile's candidate
// volumes from its superblock's pair list, exact ray tests, sorted fragment
// list) and / or views (fetch sequence -> interval records + active words).
constexpr uint32_t kTileRaster = 1u, kTileViews = 2u;
void launch_tile_pass(cudaStream_t st, uint32_t mode, const Cam& cam, const TraceParams& tp, const Voi* vois,
                      const FrameBufs& fb, const ViewBufs& vb, int tilesX, int tilesY, uint32_t tile0,
                      uint32_t tile1, int smCount);
// the A-buffer's CSR (fb.offsets, fragments in tile order in fb.unsorted as Frag) for a download
void launch_frag_csr(cudaStream_t st, const FrameBufs& fb, uint32_t tiles, int smCount);
// tileFrag from CSR offsets (an uploaded A-buffer)
void launch_tile_frag_from_offsets(cudaStream_t st, const FrameBufs& fb, uint32_t tiles);
uint32_t superblock_count(int tilesX, int tilesY);

// ---- launchers (k_util.cu) -------------------------------------------
void launch_copy_segments(cudaStream_t st, const void* const* src, void* const* dst, const size_t* bytes, int n,
                          int smCount);

// ---- launchers (k_tree.cu) -------------------------------------------
// compute_fast_indices on the device words (scratch: 4 n int32)
// ---------------------------------------------------------------- GPU compile (k_compile.cu)
// bt_scene_node (bt_cuda.h), layout-identical
struct SceneNodeK {
    uint8_t isPrimitive, kind, pad_[2];
    int32_t left, right;
    float params[17];
};
constexpr uint32_t kCmpErrKind = 1, kCmpErrChildren = 2, kCmpErrParents = 3, kCmpErrForest = 4, kCmpErrWords = 5,
                   kCmpErrParams = 6;
struct CompileScratch {
    int32_t* parent;
    uint8_t* isLeft;
    int32_t* lm[2];
    int32_t* next[2];
    uint4* val[2];
    uint4* totals;  // (words, nodes, primitives)
    uint32_t* err;  // smallest (post-order position << 8 | code), or a structure code
    int2* anc[2];
    uint32_t *isF, *isU, *fPos, *uPos, *blockSum, *counts;  // counts: frontier, upper entries
};
struct CompileNodeRec {  // bt_node (bt_cuda.h), layout-identical
    uint32_t word, parentWord;
    int32_t leftChild, rightChild;
    uint8_t isPrimitive, nodeOp, pad_[2];
};
struct CompileOut {
    float4* words;
    CompileNodeRec* records;
    uint32_t *nodeWord, *program, *size, *primWords, *primOrd;
    int32_t *parentOrd, *compactAnc;
    uint2* frontier;
    uint32_t* upper;
    uint32_t* maxDepth;
};
void launch_compile_rank(cudaStream_t st, const SceneNodeK* nodes, uint32_t n, uint32_t root, CompileScratch s);
void launch_compile_emit(cudaStream_t st, const SceneNodeK* nodes, uint32_t n, CompileScratch s, CompileOut o,
                         uint32_t frontierCap);
void launch_compile_chain(cudaStream_t st, const uint32_t* upper, uint32_t m, uint32_t* flags);

void launch_blob_table(cudaStream_t st, const float4* words, const uint32_t* nodeWord, uint32_t n, uint32_t* blobs);
void launch_fast_indices(cudaStream_t st, float4* words, const uint32_t* nodeWord, const int32_t* parentOrd,
                         uint32_t n, int32_t* scratch);

// ---- launchers (k_views.cu) -------------------------------------------
// k_view_build over the records k_tile allocated (thread per interval)
void launch_view_build(cudaStream_t st, const DevTree& t, const ViewBufs& vb, int smCount);
// longest-first march units of [tile0, tile1) from vb.tileCost (hist: 258 words of
// scratch, [257] = unit count); tiles costing >= beta x the average work per
// warp (at most cap of them) become two half-tile units
void launch_tile_order(cudaStream_t st, const ViewBufs& vb, const GBuf& g, uint32_t* hist, uint32_t* order,
                       uint32_t tile0, uint32_t tile1, uint32_t nWarps, float beta, uint32_t cap);
uint32_t trace_grid_warps(int smCount);

// ---- launchers (k_trace.cu) -------------------------------------------
void launch_trace(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam, const TraceParams& tp,
                  const FrameBufs& fb, const ViewBufs& vb, const GBuf& g, uint64_t* stats, uint32_t tile0,
                  uint32_t tile1, int smCount, uint32_t* tileQueue, bool zero = true);
// vb: the interval records of the march that produced this G-buffer (whole
// frame, FMA path) -- the gradient fallback then evaluates the pruned view
// of the interval each ray hit in; nullptr: the full tree (reference)
// pixel rows [y0, y1) of the image (a sharded rank: its own tile rows)
void launch_normals(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam,
                    const FrameBufs& fb, const GBuf& g, int mode, uint32_t* counters,
                    uint64_t* stats, int smCount, float* scratch, uint32_t scratchWarps,
                    const ViewBufs* vb, bool zero = true, int y0 = 0, int y1 = -1);
void launch_oracle(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam,
                   const TraceParams& tp, const FrameBufs& fb, const GBuf& g, uint64_t* stats);

}  // namespace btk
