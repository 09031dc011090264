/*
 * bt_cuda.h -- C-ABI of the B200 synchronized-tracing library
 * (libblobtree_b200.so).  Plain C: POD structs, pointers and sizes, no C++
 * or torch types.  Every entry point returns BT_OK (0) or an error code and
 * leaves a human-readable reason in bt_last_error().
 *
 * This is the boundary the drop-in C++ API (include/blobtree/ headers) calls for
 * the per-frame hot path of arXiv 2304.09673; each group cites the reference
 * interface it replaces (paths relative to /root/reference/proj):
 *
 *   tree + per-frame params  <- compile/LinearTree  include/blobtree/linear_tree.hpp:43-67,75
 *                               update_primitive_params               linear_tree.hpp:88-90
 *   (a) ROI / VOI            <- propagate_roi                         linear_tree.hpp:83-86
 *                               build_volumes_of_interest             linear_tree.hpp:109-115
 *   (b) tile A-buffer        <- rasterize_volumes                     abuffer.hpp:37-42
 *   (c) synchronized tracing <- render_tiles                          tracer.hpp:181-189
 *       normals              <- compute_normals                       tracer.hpp:197-201
 *       brute-force oracle   <- oracle_render                         tracer.hpp:191-195
 *
 * Threading: one context per device, not thread-safe per context.  Calls
 * are stream-ordered on the context's stream and asynchronous until a
 * bt_*_download or bt_sync.  Results are deterministic run to run (sorted
 * lists, integer atomics only).
 */
#ifndef BT_CUDA_H
#define BT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BT_API __attribute__((visibility("default")))

enum {
    BT_OK = 0,
    BT_EINVAL = 1,  /* bad argument / state (validation happens in C++ first) */
    BT_ECUDA = 2,   /* CUDA runtime error or no device                        */
    BT_ENOMEM = 3,  /* device allocation failed                               */
    BT_ESTATE = 4,  /* call order violated (e.g. trace before tree upload)    */
};

/* Blob / word layout constants (linear_tree.hpp:13-25, traversal.hpp:10-13,
 * camera.hpp:9).  The tree is uploaded in the reference's own 16-byte word
 * layout, bit for bit. */
#define BT_ANCESTOR_SENTINEL 0x7FFFFFu
#define BT_STACK_CAPACITY 22u
#define BT_MAX_OVERLAP 96u
#define BT_CACHE_BYTES 3072u
#define BT_TILE 8

/* NodeRecord (linear_tree.hpp:43-50), identical layout: 20 bytes. */
typedef struct bt_node {
    uint32_t word;
    uint32_t parentWord;
    int32_t leftChild;
    int32_t rightChild;
    uint8_t isPrimitive;
    uint8_t nodeOp;
    uint8_t pad_[2];
} bt_node;

/* CameraFrame members (camera.hpp:56-62) computed once on the host by the
 * CameraFrame constructor, so ray generation on the device is bit-identical. */
typedef struct bt_camera {
    float position[3];
    float forward[3];
    float right[3];
    float up[3];
    float tanHalf, aspect;
    float invNear, invDepthRange;
    float nearZ, farZ;
    int32_t width, height;
} bt_camera;

/* RenderConfig (tracer.hpp:11-26). normalsMode: 0 depth-differential,
 * 1 central difference. threads is ignored on the device. */
typedef struct bt_render_config {
    float lipschitz, relax, minStep, hitEpsilon;
    uint32_t maxOverlap, maxNewPerFetch;
    float fetchWindow;
    int32_t normalsMode;
    uint32_t threads;
} bt_render_config;

/* VolumeOfInterest (linear_tree.hpp:95-107), identical 64-byte layout.
 * family: 0 sphere, 1 oriented box, 2 capsule. */
typedef struct bt_voi {
    uint8_t family;
    uint8_t pad_[3];
    uint32_t primitiveWord;
    float center[3];
    float radius;
    float halfExtents[3];
    float rotation[4]; /* w, x, y, z */
    float axisEnd[3];
} bt_voi;

/* Fragment (abuffer.hpp:13-17), identical 12-byte layout. */
typedef struct bt_fragment {
    uint32_t primitiveWord;
    float zEntry, zExit;
} bt_fragment;

/* RenderStats (tracer.hpp:45-57) plus device-side work accounting.
 * fieldFlops = algorithmic FP32 flops of field evaluation per SURVEY.md
 * appendix B (12 per eval + kind-weighted primitive/operator costs). */
typedef struct bt_stats {
    uint64_t fieldEvals;
    uint64_t retainedNodeVisits;
    uint64_t primitiveEvals;
    uint64_t treeNodeCount;
    uint32_t maxOverlap;
    uint32_t maxCacheBytes;
    uint64_t fieldFlops;
    uint64_t fragments;       /* A-buffer entries of the last build          */
    uint64_t candidatePairs;  /* (volume, tile) pairs ray-tested             */
    uint64_t tileErrors;      /* tiles flagged by the tracer                 */
    uint64_t normalFallbacks; /* pixels that took the 6-tap gradient path    */
    uint64_t warpSteps;       /* lockstep march iterations of k_trace; lane
                                 utilisation = fieldEvals / (32 * warpSteps) */
} bt_stats;

/* Device pointers of the context's G-buffer (for zero-copy gathers). */
typedef struct bt_gbuffer_view {
    void* hit;            /* uint8  [height*width]                */
    void* depth;          /* float  [height*width]                */
    void* normal;         /* float3 [height*width]                */
    void* evalCount;      /* uint32 [height*width]                */
    void* tileMaxOverlap; /* uint32 [tilesY*tilesX]               */
    void* tileCacheBytes; /* uint32 [tilesY*tilesX]               */
    void* tileError;      /* uint8  [tilesY*tilesX]               */
    int32_t width, height, tilesX, tilesY;
} bt_gbuffer_view;

typedef struct bt_ctx bt_ctx;

/* ---- lifecycle -------------------------------------------------------- */
BT_API int bt_ctx_create(int device, bt_ctx** out);
BT_API int bt_ctx_destroy(bt_ctx* ctx);
BT_API const char* bt_last_error(void);
BT_API int bt_sync(bt_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the context's own stream. */
BT_API int bt_set_stream(bt_ctx* ctx, void* cuda_stream);
BT_API int bt_device_info(bt_ctx* ctx, int* sm_count, int* sm_clock_khz);

/* ---- tree (compile output, linear_tree.hpp:43-75) ---------------------- */
BT_API int bt_tree_upload(bt_ctx* ctx, const float* data, uint32_t nwords,
                          const bt_node* nodes, uint32_t nnodes,
                          const uint32_t* primitiveWords, uint32_t nprims,
                          uint32_t rootWord);
/* compute_fast_indices (linear_tree.cpp:150-168) on the uploaded tree, in
 * place on the device: every blob's ancestor becomes its fast target.  A
 * tree uploaded with parent ancestors (compile() only) ends up bit-identical
 * to one compiled with compute_fast_indices on the host; pointer jumping,
 * O(n log n) work instead of O(n x chain length).  bt_tree_download reads it. */
BT_API int bt_tree_fast_indices(bt_ctx* ctx);
/* Per-frame parameter deltas (update_primitive_params, linear_tree.cpp:187-193
 * after host validation): entry i rewrites count[i] floats at
 * data[4*(words[i]+1)] from params[i*stride ...].
 * Host buffers: PINNED ones (cudaHostAlloc / cudaHostRegister) are read by
 * the update kernel itself over PCIe, in stream order -- no copy-engine
 * transfer that would queue behind a streamed G-buffer download -- so, as
 * with any asynchronous copy from pinned memory, they must not change until
 * the frame has been synchronised.  Pageable buffers are staged with
 * cudaMemcpyAsync.  The _device variant takes device buffers (resident fast
 * path). */
BT_API int bt_params_update(bt_ctx* ctx, const uint32_t* words, const float* params,
                            const uint32_t* counts, uint32_t n, uint32_t stride);
BT_API int bt_params_update_device(bt_ctx* ctx, const uint32_t* d_words, const float* d_params,
                                   const uint32_t* d_counts, uint32_t n, uint32_t stride);
BT_API int bt_tree_download(bt_ctx* ctx, float* data, uint32_t nwords);

/* GPU compile (replaces blobtree::compile, linear_tree.cpp:70-148, when the
 * tree STRUCTURE changes per frame).  The scene graph
 * is a flat node array in any order: operators name their children by index
 * (left, right), primitives have -1; `root` indexes the root.  Parameters as
 * in the tree words: primitive translate xyz, rotation wxyz, shape (1-10
 * floats); operator blend, range (smooth / compact kinds).  The context's
 * tree becomes the post-order compile of the graph -- words, node records
 * and primitive words bit-identical to the reference's compile of the same
 * graph -- with every side table built on the device; `onDevice` = 1 when
 * `nodes` is a device pointer (a graph edited on the GPU), 0 for host memory.
 * Errors (BT_EINVAL) mirror compile's: an operator without two children, a
 * graph that is not one tree rooted at `root`, the 23-bit word space, and
 * validate_primitive / validate_operator on every node. */
typedef struct bt_scene_node {
    uint8_t isPrimitive;
    uint8_t kind;      /* PrimitiveKind 0..5 or OperatorKind 3..11 */
    uint8_t pad_[2];
    int32_t left, right;
    float params[17];
} bt_scene_node;
BT_API int bt_tree_compile(bt_ctx* ctx, const bt_scene_node* nodes, uint32_t n, uint32_t root, int onDevice);
/* sizes of the context's tree, and its node records / primitive words
 * (LinearTree::nodes / primitiveWords) */
BT_API int bt_tree_info(bt_ctx* ctx, uint32_t* nwords, uint32_t* nnodes, uint32_t* nprims);
BT_API int bt_tree_nodes_download(bt_ctx* ctx, bt_node* nodes, uint32_t nnodes, uint32_t* primWords,
                                  uint32_t nprims);

/* ---- (a) ROI / VOI ----------------------------------------------------- */
/* roi per node ordinal (propagate_roi); out may be NULL (device only). */
BT_API int bt_roi(bt_ctx* ctx, float* out_roi, uint32_t nnodes);
/* caller-provided ROI per node ordinal (build_volumes_of_interest's roiUpper) */
BT_API int bt_roi_upload(bt_ctx* ctx, const float* roi, uint32_t nnodes);
/* VOIs from the context's per-node ROI (bt_roi or bt_roi_upload first) */
BT_API int bt_voi_build(bt_ctx* ctx, float margin);
BT_API int bt_voi_upload(bt_ctx* ctx, const bt_voi* vois, uint32_t n);
BT_API int bt_voi_download(bt_ctx* ctx, bt_voi* out, uint32_t n);

/* ---- (b) A-buffer ------------------------------------------------------ */
/* Bins the context's volumes into the 8x8 tiles [tile0, tile1) of the
 * camera's image (tile1 = 0 means all tiles). */
BT_API int bt_abuffer_build(bt_ctx* ctx, const bt_camera* cam, uint32_t tile0, uint32_t tile1);
/* fragments: total entries; offsets has tilesX*tilesY+1 entries (CSR). */
BT_API int bt_abuffer_info(bt_ctx* ctx, uint64_t* fragments, int32_t* tilesX, int32_t* tilesY);
BT_API int bt_abuffer_download(bt_ctx* ctx, uint32_t* offsets, bt_fragment* frags,
                               uint64_t capacity);
BT_API int bt_abuffer_upload(bt_ctx* ctx, const bt_camera* cam, const uint32_t* offsets,
                             const bt_fragment* frags);

/* ---- (c) tracing + normals -------------------------------------------- */
/* exact != 0: IEEE op-by-op arithmetic (bit-identical to the CPU
 * reference); exact == 0: FMA-contracted field evaluation (tolerance path). */
BT_API int bt_trace(bt_ctx* ctx, const bt_camera* cam, const bt_render_config* cfg,
                    uint32_t tile0, uint32_t tile1, int exact);
BT_API int bt_normals(bt_ctx* ctx, const bt_camera* cam, int mode, int exact);
/* compute_normals (tracer.cpp:296-350) for the pixels of the tile rows
 * covering [tile0, tile1) only: a sharded rank shades its own rows.  With an
 * imported G-buffer (bt_gbuffer_import) the depths -- its rows and the
 * neighbour rows of the halo -- are read from, and the normals written to,
 * the root's planes over peer memory; the gradient fallback uses this
 * context's own interval records and tree.  Every rank's trace must be
 * complete (e.g. a stream-ordered collective) before any rank calls it. */
BT_API int bt_normals_rows(bt_ctx* ctx, const bt_camera* cam, int mode, int exact, uint32_t tile0, uint32_t tile1);
BT_API int bt_oracle_render(bt_ctx* ctx, const bt_camera* cam, const bt_render_config* cfg,
                            int exact);

/* One whole frame: (a) -> (b) -> (c) -> normals.  flags: BT_FRAME_GRAPH
 * replays the frame from a CUDA graph (re-captured when the camera, config,
 * tile range or a buffer changes); BT_FRAME_NO_NORMALS stops after tracing
 * (multi-GPU ranks: normals run after the row gather). */
#define BT_FRAME_GRAPH 1
#define BT_FRAME_NO_NORMALS 2
BT_API int bt_render_frame(bt_ctx* ctx, const bt_camera* cam, const bt_render_config* cfg,
                           uint32_t tile0, uint32_t tile1, int exact, int flags);

/* Kernel nodes in the captured per-frame graph (0 before the first capture). */
BT_API int bt_graph_kernel_count(bt_ctx* ctx, uint32_t* kernels, uint32_t* nodes);

BT_API int bt_gbuffer_download(bt_ctx* ctx, uint8_t* hit, float* depth, float* normal,
                               uint32_t* evalCount, uint32_t* tileMaxOverlap,
                               uint32_t* tileCacheBytes, uint8_t* tileError);
/* Streaming download: snapshots the G-buffer on the device (in stream order,
 * ~15 us at 1080p) and copies the snapshot to the caller's PINNED host
 * buffers on the context's copy stream, so frame N's transfer overlaps frame
 * N+1's render.  Two snapshot slots are used alternately; the host buffers
 * hold the frame once bt_download_wait() (or bt_sync()) returns.  Same
 * arguments as bt_gbuffer_download; null planes are skipped. */
BT_API int bt_gbuffer_download_async(bt_ctx* ctx, uint8_t* hit, float* depth, float* normal,
                                     uint32_t* evalCount, uint32_t* tileMaxOverlap,
                                     uint32_t* tileCacheBytes, uint8_t* tileError);
BT_API int bt_download_wait(bt_ctx* ctx);
/* Byte offsets of the seven planes (hit, depth, normal, evalCount,
 * tileMaxOverlap, tileCacheBytes, tileError; 16-byte aligned) in one host
 * slab of `total` bytes for the context's current image size. */
BT_API int bt_gbuffer_layout(bt_ctx* ctx, size_t offsets[7], size_t* total);
/* bt_gbuffer_download_async into ONE pinned allocation of at least `total`
 * bytes, planes at bt_gbuffer_layout's offsets (padding bytes between planes
 * are not written): adjacent planes go down as one range, two copies per
 * frame instead of up to fourteen. */
BT_API int bt_gbuffer_download_async_slab(bt_ctx* ctx, void* slab);

/* Fused gather over peer memory (multi-GPU).  The root rank
 * exports its G-buffer planes as CUDA IPC handles; every other rank imports
 * them, after which its traces write their tiles' pixels (hit, depth,
 * evalCount) and tile planes straight into the root's G-buffer over
 * NVLink, while the march runs -- no separate gather.  The image size must
 * match; the root must not resize its image while handles are imported.
 * After the ranks' streams are done (a host barrier), the root computes the
 * normals of the assembled frame. */
typedef struct bt_ipc_handles {
    unsigned char plane[7][64]; /* hit, depth, evalCount, tileMaxOverlap, tileCacheBytes, tileError, normal */
    int32_t width, height;
} bt_ipc_handles;
BT_API int bt_gbuffer_export(bt_ctx* ctx, bt_ipc_handles* out);
BT_API int bt_gbuffer_import(bt_ctx* ctx, const bt_ipc_handles* in);
BT_API int bt_gbuffer_import_release(bt_ctx* ctx);
/* March scheduling.  The persistent march kernel ends with its slowest tile,
 * so by default (mode 1) the tiles are queued longest-first by a cost proxy
 * computed with the interval count (fragments and their depth extent;
 * counting sort on the device, 3 small kernels).  Mode 0: raster order.
 * bt_set_tile_order installs a fixed host-given permutation of all tiles
 * instead (mode 2, full frames).  Results never depend on the order. */
BT_API int bt_set_scheduling(bt_ctx* ctx, int mode);
/* Step bound of the sphere trace (tracer.hpp:99-177).  Mode 0 (default):
 * the reference's global Lipschitz bound cfg.lipschitz for every interval.
 * Mode 1 (extension, PAPER.md "Ray processing": "replacing sphere-tracing
 * with segment-tracing would provide a more robust solution"): a bound per
 * interval view -- a view made only of exact distances (sphere, torus, box,
 * sphere-cone) and sharp CSG is 1-Lipschitz and marches with L = 1; every
 * other view keeps cfg.lipschitz.  The trajectory changes, so mode 1 is
 * held to its own tolerance contract against the reference
 * (tests/test_gpu_step_bound.py), never to bit-exactness. */
BT_API int bt_set_step_bound(bt_ctx* ctx, int mode);
/* Depth slabs (extension, PAPER.md "Conclusion and Future work": "when
 * targeting higher resolution, using larger tiles and processing by depth
 * slabs could also limit memory usage").  slabs > 1: bt_render_frame cuts
 * the view depth [near, far] into `slabs` equal slabs and builds the A-buffer,
 * the interval records and the march one slab at a time, front to back; a ray
 * that hits in a slab is done, the others continue in the next.  The A-buffer
 * and record buffers then hold one slab's fragments.  Fragments crossing a
 * slab boundary are clipped to it, so the march restarts there: held to its
 * own tolerance contract against the reference (tests/test_gpu_depth_slabs.py),
 * never to bit-exactness.  1 (default): the reference's single pass. */
BT_API int bt_set_depth_slabs(bt_ctx* ctx, int slabs);
BT_API int bt_set_tile_order(bt_ctx* ctx, const uint32_t* order, uint32_t n);
BT_API int bt_gbuffer_device(bt_ctx* ctx, bt_gbuffer_view* out);
/* hit/depth planes from the host (compute_normals on a caller's G-buffer) */
BT_API int bt_gbuffer_upload(bt_ctx* ctx, const bt_camera* cam, const uint8_t* hit, const float* depth);
BT_API int bt_stats_download(bt_ctx* ctx, bt_stats* out);
BT_API int bt_stats_reset(bt_ctx* ctx);

/* ---- timing helpers (CUDA events on the context's stream) ------------- */
/* Records per-kernel-class device time (ms) accumulated since the last
 * reset when profiling is enabled: [roi_voi, abuffer, trace, normals]. */
BT_API int bt_profile_enable(bt_ctx* ctx, int on);
BT_API int bt_profile_read(bt_ctx* ctx, float* ms4, uint32_t* launches4);
/* Up to 6 slots: the 4 above, then the two halves of trace: [4] interval /
 * view compilation (k_view_count, k_view_scan, k_view_build), [5] the march
 * kernel alone (k_march: field evaluation -- the roofline kernel). */
BT_API int bt_profile_read_ex(bt_ctx* ctx, float* ms, uint32_t* launches, uint32_t nslots);
/* Measured non-tensor FP32 peak of `device` (FFMA microbenchmark, TFLOP/s):
 * the roofline denominator of the field-evaluation kernel. */
BT_API int bt_fp32_peak(int device, float* tflops, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* BT_CUDA_H */
