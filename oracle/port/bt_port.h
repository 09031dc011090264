/*
 * bt_port.h -- C restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * An independent, single-file C11 re-derivation of the per-frame pipeline of
 * /root/reference/proj (propagate_roi -> build_volumes_of_interest ->
 * rasterize_volumes -> render_tiles -> compute_normals, plus oracle_render),
 * operating on the same POD layouts as the C-ABI (include/bt_cuda.h).  Every
 * function cites the reference lines it restates.  It is compiled FMA-free
 * (-ffp-contract=off, x86-64 baseline) and is pinned against the reference
 * library itself (oracle/_ref) and the golden fixtures in tests/golden/ by
 * tests/test_oracle_port.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use it; the
 * product never links it.
 */
#ifndef BT_PORT_H
#define BT_PORT_H

#include "../../include/bt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* tree view over the compiled word array (compile(), linear_tree.cpp:70-148) */
typedef struct port_tree {
    const float* data;        /* 4 floats per word */
    uint32_t nwords;
    const bt_node* nodes;     /* post-order */
    uint32_t nnodes;
    const uint32_t* prims;    /* ascending primitive words */
    uint32_t nprims;
} port_tree;

BT_API void port_roi(const port_tree* t, float* out);
BT_API void port_vois(const port_tree* t, const float* roi, float margin, bt_voi* out);
BT_API int port_rasterize(const bt_voi* vois, uint32_t n, const bt_camera* cam, uint32_t* offsets,
                          bt_fragment* frags, uint64_t cap, uint64_t* total);
/* stats6: fieldEvals, retainedNodeVisits, primitiveEvals, treeNodeCount, maxOverlap, maxCacheBytes */
BT_API int port_render_tiles(const port_tree* t, const bt_camera* cam, const bt_render_config* cfg,
                             const uint32_t* offsets, const bt_fragment* frags, int threads, uint8_t* hit,
                             float* depth, uint32_t* evalCount, uint32_t* tileMaxOverlap,
                             uint32_t* tileCacheBytes, uint8_t* tileError, uint64_t* stats6);
BT_API void port_normals(const port_tree* t, const bt_camera* cam, int mode, const uint8_t* hit,
                         const float* depth, float* normal);
BT_API void port_oracle(const port_tree* t, const bt_camera* cam, const bt_render_config* cfg, int threads,
                        uint8_t* hit, float* depth, uint32_t* evalCount, uint64_t* stats6);
/* single-point helpers for golden vectors */
BT_API float port_eval_primitive(uint32_t kind, const float* params, float x, float y, float z);
BT_API float port_eval_operator(uint32_t code, const float* params, float f0, float f1);
BT_API float port_eval_full(const port_tree* t, float x, float y, float z);

#ifdef __cplusplus
}
#endif
#endif
