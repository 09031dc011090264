// k_tree.cu -- GPU tree preprocessing: compute_fast_indices on the device
// (reference src/linear_tree.cpp:150-168).
//
// The reference walks, for every node, up its parent chain while the chain
// keeps the node's side (isLeft) and never bypasses a selector (ignore mode
// of the opposite side), and stores the last reached ancestor: O(n x chain)
// hops with a binary search per hop, 141 ms at 10k primitives on a deep comb.
// Here the chain is a pointer-jumping problem: with
//   next_s(u) = parent(u)  if side(u) == s, (ignore(u) & guard(s)) == 0 and
//                          u is not the root
//             = u          otherwise (u ends every chain of side s through it)
// the fast target of node i is the fixed point of next_{side(i)} from
// parent(i).  ceil(log2(n)) rounds of next <- next(next) reach every fixed
// point (two arrays, one per side); a final pass rewrites the ancestor
// field of each node's blob in the device words.  Bit-identical to the host
// compute_fast_indices (only the 23-bit ancestor field changes).
#include <cuda_runtime.h>

#include "bt_device.h"

namespace btk {

namespace {

constexpr uint32_t kIgnoreRightAbsent = 1u, kIgnoreLeftAbsent = 2u;

__global__ void k_fast_init(const float4* words, const uint32_t* nodeWord, const int32_t* parentOrd, uint32_t n,
                            int32_t* nextL, int32_t* nextR) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t p = parentOrd[u];
    const uint32_t b = __float_as_uint(words[nodeWord[u]].x);
    const bool left = blob_is_left(b);
    const uint32_t ign = blob_ignore(b);
    const bool up = p >= 0;  // the walk stops at the root
    nextL[u] = (up && left && !(ign & kIgnoreRightAbsent)) ? p : (int32_t)u;
    nextR[u] = (up && !left && !(ign & kIgnoreLeftAbsent)) ? p : (int32_t)u;
}

__global__ void k_fast_jump(const int32_t* inL, const int32_t* inR, int32_t* outL, int32_t* outR, uint32_t n) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    outL[u] = inL[inL[u]];
    outR[u] = inR[inR[u]];
}

__global__ void k_fast_write(float4* words, const uint32_t* nodeWord, const int32_t* parentOrd, uint32_t n,
                             const int32_t* nextL, const int32_t* nextR) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t p = parentOrd[i];
    if (p < 0) return;  // the root keeps the sentinel
    float4* w = words + nodeWord[i];
    const uint32_t b = __float_as_uint(w->x);
    const int32_t target = blob_is_left(b) ? nextL[p] : nextR[p];
    w->x = __uint_as_float(blob_with_anc(b, nodeWord[target]));
}

// the dense blob table (DevTree::blobs): every node's header word, at its word
__global__ void k_blob_table(const float4* words, const uint32_t* nodeWord, uint32_t n, uint32_t* blobs) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t w = nodeWord[i];
    blobs[w] = __float_as_uint(words[w].x);
}

}  // namespace

void launch_blob_table(cudaStream_t st, const float4* words, const uint32_t* nodeWord, uint32_t n, uint32_t* blobs) {
    if (n) k_blob_table<<<(n + 255) / 256, 256, 0, st>>>(words, nodeWord, n, blobs);
}

void launch_fast_indices(cudaStream_t st, float4* words, const uint32_t* nodeWord, const int32_t* parentOrd,
                         uint32_t n, int32_t* scratch) {
    if (n == 0) return;
    int32_t* a[2] = {scratch, scratch + 2 * (size_t)n};  // (L, R) ping-pong
    const uint32_t blocks = (n + 255) / 256;
    k_fast_init<<<blocks, 256, 0, st>>>(words, nodeWord, parentOrd, n, a[0], a[0] + n);
    int cur = 0;
    for (uint32_t span = 1; span < n; span <<= 1) {
        k_fast_jump<<<blocks, 256, 0, st>>>(a[cur], a[cur] + n, a[cur ^ 1], a[cur ^ 1] + n, n);
        cur ^= 1;
    }
    k_fast_write<<<blocks, 256, 0, st>>>(words, nodeWord, parentOrd, n, a[cur], a[cur] + n);
}

}  // namespace btk
