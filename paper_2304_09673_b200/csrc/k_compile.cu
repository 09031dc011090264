// k_compile.cu -- GPU tree compile (reference
// src/linear_tree.cpp:70-148, CompileCursor::emit): a scene graph given as a
// flat node array in ANY order (children by index, the root by index) becomes
// the post-order word array, node records and primitive words -- bit for bit
// what the reference's recursive compile emits for the same graph -- plus the
// side tables the frame kernels read (bt_tree_upload builds them on the host).
//
// The recursion is a list ranking:
//   * parents and sides from the child links (k_cmp_link);
//   * the leftmost leaf of every subtree by pointer jumping down left children
//     (its first node in post-order);
//   * the post-order successor of a node: its parent when it is a right child,
//     else the leftmost leaf of its right sibling (the root ends the list);
//   * Wyllie ranking along the successor list with three weights at once --
//     the node's word count, 1, and its primitive flag -- gives every node's
//     first word, post-order ordinal and primitive rank (suffix sums, turned
//     into exclusive prefixes by the totals at the list head);
//   * k_cmp_emit writes each node where the recursion would have put it.
// Validation mirrors emit's throws: operators need two children, the graph
// must be one tree (one parent per node, every node reachable from the
// root), the word space must fit 23 bits, and validate_primitive /
// validate_operator (field.cpp:174-213, 389-397) hold for every node; the
// error reported is the one at the smallest post-order position.
#include <cuda_runtime.h>

#include "bt_device.h"
#include "bt_geom.cuh"

namespace btk {

namespace {

constexpr uint32_t kT = 256;

__device__ __forceinline__ uint32_t node_words(const SceneNodeK& s) {
    if (s.isPrimitive) {
        const uint32_t k = s.kind;
        const uint32_t shape = k == 0u ? 1u : k == 2u ? 2u : k == 5u ? 10u : 3u;
        return 1u + (7u + shape + 3u) / 4u;  // primitive_word_count
    }
    return (s.kind >= 3u && s.kind <= 5u) ? 1u : 2u;  // operator_word_count: sharp 1, else 2
}

// 1. parents / sides / structure checks; leftmost-leaf seeds; weights
__global__ void k_cmp_link(const SceneNodeK* nodes, uint32_t n, uint32_t root, int32_t* parent, uint8_t* isLeft,
                           int32_t* lm, uint32_t* err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SceneNodeK s = nodes[i];
    if (s.isPrimitive) {
        if (s.kind > 5u) atomicMin(err, kCmpErrKind);
        lm[i] = (int32_t)i;
        return;
    }
    if (s.kind < 3u || s.kind > 11u) atomicMin(err, kCmpErrKind);
    const int32_t l = s.left, r = s.right;
    if (l < 0 || r < 0 || (uint32_t)l >= n || (uint32_t)r >= n || l == r || (uint32_t)l == i || (uint32_t)r == i) {
        atomicMin(err, kCmpErrChildren);  // "operator node must have two children"
        lm[i] = (int32_t)i;
        return;
    }
    if (atomicCAS(reinterpret_cast<unsigned int*>(&parent[l]), 0xFFFFFFFFu, i) != 0xFFFFFFFFu ||
        atomicCAS(reinterpret_cast<unsigned int*>(&parent[r]), 0xFFFFFFFFu, i) != 0xFFFFFFFFu)
        atomicMin(err, kCmpErrParents);  // a node with two parents: not a tree
    isLeft[l] = 1;
    isLeft[r] = 0;
    lm[i] = l;
    (void)root;
}

// the root has no parent, every other node has one
__global__ void k_cmp_roots(const int32_t* parent, uint32_t n, uint32_t root, uint8_t* isLeft, uint32_t* err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if ((parent[i] < 0) != (i == root)) atomicMin(err, kCmpErrForest);
    if (i == root) isLeft[i] = 1;  // emit(root, isLeft = true)
}

__global__ void k_cmp_jump_lm(const int32_t* in, int32_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[in[i]];
}

// 2. post-order successor and the ranking weights
__global__ void k_cmp_succ(const SceneNodeK* nodes, const int32_t* parent, const uint8_t* isLeft, const int32_t* lm,
                           uint32_t n, uint32_t root, int32_t* next, uint4* val) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t s = -1;
    if (i != root && parent[i] >= 0) {
        const int32_t p = parent[i];
        s = isLeft[i] ? lm[nodes[p].right] : p;
    }
    next[i] = s;
    const SceneNodeK nd = nodes[i];
    val[i] = make_uint4(node_words(nd), 1u, nd.isPrimitive ? 1u : 0u, 0u);
}

// Wyllie step: val(i) += val(next(i)), next(i) = next(next(i))
__global__ void k_cmp_rank(const int32_t* nextIn, const uint4* valIn, int32_t* nextOut, uint4* valOut, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t s = nextIn[i];
    uint4 v = valIn[i];
    if (s >= 0) {
        const uint4 w = valIn[s];
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        nextOut[i] = nextIn[s];
    } else {
        nextOut[i] = -1;
    }
    valOut[i] = v;
}

// totals at the list head (the leftmost leaf of the root); every node reached
__global__ void k_cmp_totals(const int32_t* lm, const uint4* val, uint32_t n, uint32_t root, uint4* totals,
                             uint32_t* err) {
    const uint4 t = val[lm[root]];
    *totals = t;
    if (t.y != n) atomicMin(err, kCmpErrForest);  // a cycle or a part unreachable from the root
    if (t.x >= kSentinel) atomicMin(err, kCmpErrWords);  // "tree exceeds the 23-bit node index space"
}

// validate_primitive / validate_operator (field.cpp:174-213, 389-397)
__device__ uint32_t validate_node(const SceneNodeK& s) {
    const float* P = s.params;
    if (s.isPrimitive) {
        if (!(isfinite(P[0]) && isfinite(P[1]) && isfinite(P[2]))) return kCmpErrParams;
        // length(Quat) = sqrt(w w + x x + y y + z z), FMA-free as in the reference build
        const float ql = __fsqrt_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(P[3], P[3]), __fmul_rn(P[4], P[4])),
                                                        __fmul_rn(P[5], P[5])),
                                              __fmul_rn(P[6], P[6])));
        if (fabsf(__fsub_rn(ql, 1.0f)) > 1e-6f) return kCmpErrParams;
        const float* sh = P + 7;
        auto pos = [](float v) { return isfinite(v) && v > 0.0f; };
        switch (s.kind) {
            case 0: return pos(sh[0]) ? 0u : kCmpErrParams;
            case 1: case 3: return pos(sh[0]) && pos(sh[1]) && pos(sh[2]) ? 0u : kCmpErrParams;
            case 2: return pos(sh[0]) && pos(sh[1]) && !(sh[1] >= sh[0]) ? 0u : kCmpErrParams;
            case 4:
                return pos(sh[0]) && pos(sh[1]) && pos(sh[2]) && !(fabsf(__fsub_rn(sh[0], sh[1])) >= sh[2])
                           ? 0u : kCmpErrParams;
            default: {
                const QuadricInfoK q = analyze_quadric_k(sh);
                return q.pd && q.iso > 0.0f ? 0u : kCmpErrParams;
            }
        }
    }
    if (s.kind >= 3u && s.kind <= 5u) return 0u;  // sharp
    if (!(P[0] > 0.0f) || !isfinite(P[0])) return kCmpErrParams;
    if (s.kind >= 9u && (!isfinite(P[1]) || !(P[1] > __fdiv_rn(P[0], 6.0f)))) return kCmpErrParams;
    return 0u;
}

// 3. emit: words, node records, primitive words, side tables
__global__ void k_cmp_emit(const SceneNodeK* nodes, const int32_t* parent, const uint8_t* isLeft, const int32_t* lm,
                           const uint4* suf, const uint4* totals, uint32_t n, CompileOut o, uint32_t* err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 T = *totals;
    const SceneNodeK s = nodes[i];
    auto word_of = [&](int32_t j) { return T.x - suf[j].x; };
    auto ord_of = [&](int32_t j) { return T.y - suf[j].y; };
    const uint32_t word = word_of(i), ord = ord_of(i), prank = T.z - suf[i].z;
    const int32_t p = parent[i];
    const uint32_t op = s.kind & 0x1Fu;
    const uint32_t ignore = s.isPrimitive ? 0u : (op == 4u || op == 7u || op == 10u) ? 3u
                                                 : (op == 5u || op == 8u || op == 11u) ? 2u : 0u;
    const uint32_t anc = p >= 0 ? word_of(p) : kSentinel;
    const uint32_t blob = ((s.isPrimitive ? 1u : 0u) << 31) | (op << 26) | (ignore << 24) |
                          ((isLeft[i] ? 1u : 0u) << 23) | (anc & kSentinel);
    float* w = reinterpret_cast<float*>(o.words + word);
    w[0] = __uint_as_float(blob);
    if (s.isPrimitive) {
        const uint32_t cnt = 7u + (op == 0u ? 1u : op == 2u ? 2u : op == 5u ? 10u : 3u);
        for (uint32_t k = 0; k < cnt; ++k) w[4 + k] = s.params[k];
    } else if (!(op >= 3u && op <= 5u)) {
        w[4] = s.params[0];  // blend
        w[5] = s.params[1];  // range
    }
    const uint32_t e = validate_node(s);
    if (e) atomicMin(err, (ord << 8) | e);
    CompileNodeRec rec;
    rec.word = word;
    rec.parentWord = anc;
    rec.leftChild = s.isPrimitive ? -1 : (int32_t)ord_of(s.left);
    rec.rightChild = s.isPrimitive ? -1 : (int32_t)ord_of(s.right);
    rec.isPrimitive = s.isPrimitive ? 1 : 0;
    rec.nodeOp = (uint8_t)op;
    rec.pad_[0] = rec.pad_[1] = 0;
    o.records[ord] = rec;
    o.nodeWord[ord] = word;
    o.parentOrd[ord] = p >= 0 ? (int32_t)ord_of(p) : -1;
    o.program[ord] = ((s.isPrimitive ? 1u : 0u) << 31) | (op << 26) | (word & kSentinel);
    // subtree size in post-order: [ord(leftmost leaf), ord]
    o.size[ord] = ord - ord_of(lm[i]) + 1u;
    if (s.isPrimitive) {
        o.primWords[prank] = word;
        o.primOrd[prank] = ord;
    }
    // post-order stack depth after this node: primitives minus operators so far
    const uint32_t primsIncl = prank + (s.isPrimitive ? 1u : 0u);
    const int32_t depth = (int32_t)primsIncl - (int32_t)(ord + 1u - primsIncl);
    if (depth > 0) atomicMax(o.maxDepth, (uint32_t)depth);
}

// 4. nearest strict compact ancestor (ordinals): pointer jumping over
//    non-compact parents.  st: .x = target / value, .y = 1 when resolved
__global__ void k_cmp_anc_init(const int32_t* parentOrd, const uint32_t* program, uint32_t n, int2* st) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int32_t p = parentOrd[o];
    if (p < 0) {
        st[o] = make_int2(-1, 1);
        return;
    }
    const uint32_t op = (program[p] >> 26) & 0x1Fu;
    st[o] = (op >= 9u && op <= 11u) ? make_int2(p, 1) : make_int2(p, 0);
}

__global__ void k_cmp_anc_jump(const int2* in, int2* out, uint32_t n) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    int2 s = in[o];
    if (!s.y) {
        const int2 t = in[s.x];
        s = t.y ? make_int2(t.x, 1) : make_int2(t.x, 0);
    }
    out[o] = s;
}

__global__ void k_cmp_anc_out(const int2* st, uint32_t n, int32_t* compactAnc) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < n) compactAnc[o] = st[o].x;
}

// 5. frontier decomposition of the full tree (gradient fallback, capi.cu
//    bt_tree_upload): maximal subtrees of <= cap nodes, and the upper program
__global__ void k_cmp_front_flags(const uint32_t* size, const int32_t* parentOrd, uint32_t n, uint32_t cap,
                                  uint32_t* isF, uint32_t* isU) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int32_t p = parentOrd[o];
    const bool f = size[o] <= cap && (p < 0 || size[p] > cap);
    isF[o] = f ? 1u : 0u;
    isU[o] = (f || size[o] > cap) ? 1u : 0u;
}

__global__ void k_cmp_front_emit(const uint32_t* size, const uint32_t* program, const uint32_t* isF,
                                 const uint32_t* isU, const uint32_t* fPos, const uint32_t* uPos, uint32_t n,
                                 uint2* frontier, uint32_t* upper) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n || !isU[o]) return;
    if (isF[o]) {
        frontier[fPos[o]] = make_uint2(o + 1u - size[o], o);
        upper[uPos[o]] = 0x80000000u | fPos[o];
    } else {
        upper[uPos[o]] = program[o];
    }
}

// left comb (LOAD, then (LOAD, OP) pairs) / and of sharp unions: flags[0], flags[1]
__global__ void k_cmp_chain(const uint32_t* u, uint32_t m, uint32_t* flags) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const bool load = (u[j] >> 31) != 0u;
    bool ch = (m % 2u == 1u) && (j == 0u ? load : ((j & 1u) ? load : !load));
    bool mc = ch && (j == 0u || (j & 1u) || ((u[j] >> 26) & 0x1Fu) == 3u);
    if (!ch) atomicAnd(&flags[0], 0u);
    if (!mc) atomicAnd(&flags[1], 0u);
}

// exclusive scan of u32 flags (n <= 2^23): per-block sums, one block over
// them, then the offsets
constexpr uint32_t kScanItems = 1024;  // per block: 256 threads x 4

__global__ void k_cmp_scan_block(const uint32_t* in, uint32_t n, uint32_t* out, uint32_t* blockSum) {
    __shared__ uint32_t warpSum[kT / 32];
    const uint32_t base = blockIdx.x * kScanItems + threadIdx.x * 4u;
    uint32_t v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = base + k < n ? in[base + k] : 0u;
        s += v[k];
    }
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t incl = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= (uint32_t)d) incl += t;
    }
    if (lane == 31) warpSum[w] = incl;
    __syncthreads();
    uint32_t pre = 0;
    for (uint32_t k = 0; k < w; ++k) pre += warpSum[k];
    uint32_t run = pre + incl - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == kT - 1) blockSum[blockIdx.x] = pre + incl;
}

__global__ void k_cmp_scan_sums(uint32_t* blockSum, uint32_t nb, uint32_t* total) {
    if (threadIdx.x != 0) return;
    uint32_t run = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        const uint32_t v = blockSum[b];
        blockSum[b] = run;
        run += v;
    }
    *total = run;
}

__global__ void k_cmp_scan_add(uint32_t* out, uint32_t n, const uint32_t* blockSum) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += blockSum[i / kScanItems];
}

void scan_u32(cudaStream_t st, const uint32_t* in, uint32_t n, uint32_t* out, uint32_t* blockSum, uint32_t* total) {
    const uint32_t nb = (n + kScanItems - 1) / kScanItems;
    k_cmp_scan_block<<<nb, kT, 0, st>>>(in, n, out, blockSum);
    k_cmp_scan_sums<<<1, 32, 0, st>>>(blockSum, nb, total);
    k_cmp_scan_add<<<(n + kT - 1) / kT, kT, 0, st>>>(out, n, blockSum);
}

uint32_t rounds_for(uint32_t n) {
    uint32_t r = 1;
    while ((1u << r) < n && r < 31) ++r;
    return r + 1;
}

}  // namespace

// Phase A: structure, ranking, totals (the caller reads totals / err back to
// size the outputs).  Scratch layout is the caller's (CompileScratch).
void launch_compile_rank(cudaStream_t st, const SceneNodeK* nodes, uint32_t n, uint32_t root, CompileScratch s) {
    const uint32_t g = (n + kT - 1) / kT;
    cudaMemsetAsync(s.parent, 0xFF, (size_t)n * sizeof(int32_t), st);
    cudaMemsetAsync(s.isLeft, 0, n, st);
    k_cmp_link<<<g, kT, 0, st>>>(nodes, n, root, s.parent, s.isLeft, s.lm[0], s.err);
    k_cmp_roots<<<g, kT, 0, st>>>(s.parent, n, root, s.isLeft, s.err);
    int cur = 0;
    const uint32_t R = rounds_for(n);
    for (uint32_t r = 0; r < R; ++r, cur ^= 1) k_cmp_jump_lm<<<g, kT, 0, st>>>(s.lm[cur], s.lm[cur ^ 1], n);
    if (cur) cudaMemcpyAsync(s.lm[0], s.lm[1], (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    k_cmp_succ<<<g, kT, 0, st>>>(nodes, s.parent, s.isLeft, s.lm[0], n, root, s.next[0], s.val[0]);
    cur = 0;
    for (uint32_t r = 0; r < R; ++r, cur ^= 1)
        k_cmp_rank<<<g, kT, 0, st>>>(s.next[cur], s.val[cur], s.next[cur ^ 1], s.val[cur ^ 1], n);
    if (cur) cudaMemcpyAsync(s.val[0], s.val[1], (size_t)n * sizeof(uint4), cudaMemcpyDeviceToDevice, st);
    k_cmp_totals<<<1, 1, 0, st>>>(s.lm[0], s.val[0], n, root, s.totals, s.err);
}

// Phase B: emit into the context's tree buffers (words zeroed by the caller)
// and build the side tables.
void launch_compile_emit(cudaStream_t st, const SceneNodeK* nodes, uint32_t n, CompileScratch s, CompileOut o,
                         uint32_t frontierCap) {
    const uint32_t g = (n + kT - 1) / kT;
    k_cmp_emit<<<g, kT, 0, st>>>(nodes, s.parent, s.isLeft, s.lm[0], s.val[0], s.totals, n, o, s.err);
    // compact ancestors
    k_cmp_anc_init<<<g, kT, 0, st>>>(o.parentOrd, o.program, n, s.anc[0]);
    int cur = 0;
    const uint32_t R = rounds_for(n);
    for (uint32_t r = 0; r < R; ++r, cur ^= 1) k_cmp_anc_jump<<<g, kT, 0, st>>>(s.anc[cur], s.anc[cur ^ 1], n);
    k_cmp_anc_out<<<g, kT, 0, st>>>(s.anc[cur], n, o.compactAnc);
    // frontier + upper program
    k_cmp_front_flags<<<g, kT, 0, st>>>(o.size, o.parentOrd, n, frontierCap, s.isF, s.isU);
    scan_u32(st, s.isF, n, s.fPos, s.blockSum, &s.counts[0]);
    scan_u32(st, s.isU, n, s.uPos, s.blockSum, &s.counts[1]);
    k_cmp_front_emit<<<g, kT, 0, st>>>(o.size, o.program, s.isF, s.isU, s.fPos, s.uPos, n, o.frontier, o.upper);
}

void launch_compile_chain(cudaStream_t st, const uint32_t* upper, uint32_t m, uint32_t* flags) {
    cudaMemsetAsync(flags, 0xFF, 2 * sizeof(uint32_t), st);
    if (m) k_cmp_chain<<<(m + kT - 1) / kT, kT, 0, st>>>(upper, m, flags);
}

}  // namespace btk
