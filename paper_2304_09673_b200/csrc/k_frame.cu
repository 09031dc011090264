// k_frame.cu -- stages (a) and (b) on sm_100a.
//
//   k_params_update  per-frame primitive parameter rewrite      (linear_tree.cpp:187-193)
//   k_roi_all        range of interest per node                 (linear_tree.cpp:170-185)
//   k_voi            volume of interest per primitive           (linear_tree.cpp:216-283)
//   k_camera         pixel rays, tile cones, superblock cones   (camera.cpp:29-37, abuffer.cpp:117-149)
//   k_pairs          (volume, superblock) coarse cull           (superset of abuffer.cpp:193-196),
//                    counted per superblock
//   k_scan           single-pass exclusive scan (superblock pair counts; tile
//                    fragment counts for a CSR download)
//   k_sb_scatter     pairs -> per-superblock candidate lists
// The per-tile work -- the exact tile cone and pixel pyramid culls, the 64
// exact ray intervals per candidate, the sorted fragment list -- is one warp
// per tile in k_tile.cu.
//
// Everything on the A-buffer path is evaluated with ExactOps (no FMA, IEEE
// div/sqrt), so (tile, word) membership and (zEntry, zExit) are bit-exact
// with the reference's single-threaded rasterize_volumes.
#include <algorithm>

#include "bt_cull.cuh"

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kScanBlock = kScanBlockElems;  // per scan block (1024 threads x 4)

// ---------------------------------------------------------------- (a)

__global__ void k_params_update(float4* words, const uint32_t* dWords, const float* dParams,
                                const uint32_t* dCounts, uint32_t n, uint32_t stride) {
    const uint32_t i = blockIdx.x * blockDim.y + threadIdx.y;
    if (i >= n) return;
    const uint32_t w = dWords[i];
    const uint32_t cnt = dCounts[i];
    float* dst = reinterpret_cast<float*>(words + w + 1);
    for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) dst[k] = dParams[(size_t)i * stride + k];
}

// roi(n) = max(0, d of every compact strict ancestor): the top-down
// max-propagation of propagate_roi, unrolled along the compact-ancestor chain.
__device__ __forceinline__ float roi_of(const DevTree& t, uint32_t ord) {
    float r = 0.0f;
    int32_t a = t.compactAnc[ord];
    while (a >= 0) {
        const float d = __ldg(&t.words[t.nodeWord[a] + 1].y);
        r = smax(r, d);
        a = t.compactAnc[a];
    }
    return r;
}

__global__ void k_roi_all(DevTree t, float* roi) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.nnodes) return;
    if (!t.ancOff) {
        roi[i] = roi_of(t, i);
        return;
    }
    // the same maximum, over independent loads (max of finite values starting
    // from +0 does not depend on the order)
    float r = 0.0f;
    const uint32_t k1 = t.ancOff[i + 1];
    for (uint32_t k = t.ancOff[i]; k < k1; ++k) r = smax(r, __ldg(&t.words[t.ancIdx[k]].y));
    roi[i] = r;
}

__global__ void k_voi(DevTree t, const float* roi, float margin, Voi* vois) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.nprims) return;
    const uint32_t w = t.primWords[i];
    const uint32_t blob = __float_as_uint(__ldg(&t.words[w].x));
    float P[20];
    const float4* src = t.words + w + 1;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        float4 q = __ldg(&src[k]);
        P[4 * k] = q.x;
        P[4 * k + 1] = q.y;
        P[4 * k + 2] = q.z;
        P[4 * k + 3] = q.w;
    }
    vois[i] = make_voi(blob_op(blob), w, P, roi[t.primOrd[i]], margin);
}

// ---------------------------------------------------------------- camera

// Pyramid spanned by the pixel-centre rays of a pixel rectangle
// [x0, x1] x [y0, y1] (inclusive pixel indices).  Ray directions are affine
// in the pixel coordinates before normalisation, so every pixel ray of the
// rectangle lies inside the pyramid of its four corner rays: a volume that
// misses the pyramid cannot be hit by any of them.  Writes 4 inward unit
// plane normals (through the camera position).
__device__ void pixel_pyramid(const Cam& c, int x0, int y0, int x1, int y1, float4* out) {
    auto dir = [&](int px, int py) {
        const float sx = ((2.0f * (px + 0.5f)) / c.width - 1.0f) * c.tanHalf * c.aspect;
        const float sy = (1.0f - (2.0f * (py + 0.5f)) / c.height) * c.tanHalf;
        return F3{c.fwd.x + c.right.x * sx + c.up.x * sy, c.fwd.y + c.right.y * sx + c.up.y * sy,
                  c.fwd.z + c.right.z * sx + c.up.z * sy};
    };
    const F3 d[4] = {dir(x0, y0), dir(x1, y0), dir(x1, y1), dir(x0, y1)};
    const F3 mid{0.25f * (d[0].x + d[1].x + d[2].x + d[3].x), 0.25f * (d[0].y + d[1].y + d[2].y + d[3].y),
                 0.25f * (d[0].z + d[1].z + d[2].z + d[3].z)};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const F3 a = d[e], b = d[(e + 1) & 3];
        F3 n{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
        float len = sqrtf(n.x * n.x + n.y * n.y + n.z * n.z);
        if (len > 0.0f) {
            n = F3{n.x / len, n.y / len, n.z / len};
            if (n.x * mid.x + n.y * mid.y + n.z * mid.z < 0.0f) n = F3{-n.x, -n.y, -n.z};
        } else {
            n = F3{0.f, 0.f, 0.f};  // degenerate edge (1-pixel rectangle side): never rejects
        }
        out[e] = make_float4(n.x, n.y, n.z, 0.0f);
    }
}

#ifndef BT_RASTER_MINB
#define BT_RASTER_MINB 4  // CTAs per SM of k_camera / k_raster the register budget must fit (scripts/rasterminb_ab.sh)
#endif
// One CTA per superblock: 4096 rays, 64 tile cones, 1 conservative
// superblock cone containing all of its tile cones.
__global__ void __launch_bounds__(256, BT_RASTER_MINB) k_camera(Cam cam, FrameBufs fb, int tilesX, int tilesY, int sb0) {
    __shared__ float4 sCone[64];
    __shared__ float sSin[64];
    __shared__ int sValid[64];
    __shared__ float sScreen[2][kSB * kTile];  // screen offsets of the block's 64 columns and 64 rows
    const int sbX = (tilesX + kSB - 1) / kSB;
    const int sb = sb0 + (int)blockIdx.x;
    const int sx = sb % sbX, sy = sb / sbX;
    if (threadIdx.x < 2 * kSB * kTile) {
        const int j = threadIdx.x & (kSB * kTile - 1);
        sScreen[threadIdx.x >> 6][j] = threadIdx.x < kSB * kTile
                                           ? screen_x(cam, E::add((float)(sx * kSB * kTile + j), 0.5f))
                                           : screen_y(cam, E::add((float)(sy * kSB * kTile + j), 0.5f));
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 64 * 64; k += blockDim.x) {
        const int lt = k >> 6, pix = k & 63;
        const int tx = sx * kSB + (lt & 7), ty = sy * kSB + (lt >> 3);
        if (tx >= tilesX || ty >= tilesY) continue;
        const int px = tx * kTile + (pix & 7), py = ty * kTile + (pix >> 3);
        if (px >= cam.width || py >= cam.height) continue;
        const RayDir r = ray_from_screen(cam, sScreen[0][px - sx * kSB * kTile], sScreen[1][py - sy * kSB * kTile]);
        fb.rays[(size_t)(ty * tilesX + tx) * 64 + pix] = make_float4(r.dir.x, r.dir.y, r.dir.z, r.ddf);
    }
    if (threadIdx.x < 64) {
        const int lt = threadIdx.x;
        const int tx = sx * kSB + (lt & 7), ty = sy * kSB + (lt >> 3);
        const bool valid = tx < tilesX && ty < tilesY;
        sValid[lt] = valid;
        if (valid) {
            const int x1 = min(tx * kTile + kTile, cam.width) - 1, y1 = min(ty * kTile + kTile, cam.height) - 1;
            pixel_pyramid(cam, tx * kTile, ty * kTile, x1, y1, fb.tileFrustum + (size_t)(ty * tilesX + tx) * 4);
            const Cone c = tile_cone(cam, tx, ty);
            const float4 v = make_float4(c.axis.x, c.axis.y, c.axis.z, c.cosH);
            fb.cones[ty * tilesX + tx] = v;
            fb.coneSin[ty * tilesX + tx] = c.sinH;
            sCone[lt] = v;
            sSin[lt] = c.sinH;
        }
    }
    if (threadIdx.x == 64) {
        const int x0 = sx * kSB * kTile, y0 = sy * kSB * kTile;
        const int x1 = min(x0 + kSB * kTile, cam.width) - 1, y1 = min(y0 + kSB * kTile, cam.height) - 1;
        pixel_pyramid(cam, x0, y0, x1, y1, fb.sbFrustum + (size_t)sb * 4);
    }
    __syncthreads();
    // superblock cone: axis = normalized sum of tile axes, half-angle =
    // max over tiles of angle(axis, tile axis) + tile half-angle, padded.
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        float ax = 0.f, ay = 0.f, az = 0.f;
        for (int lt = l; lt < 64; lt += 32)
            if (sValid[lt]) {
                ax += sCone[lt].x;
                ay += sCone[lt].y;
                az += sCone[lt].z;
            }
        for (int o = 16; o > 0; o >>= 1) {
            ax += __shfl_xor_sync(kFull, ax, o);
            ay += __shfl_xor_sync(kFull, ay, o);
            az += __shfl_xor_sync(kFull, az, o);
        }
        const float inv = rsqrtf(ax * ax + ay * ay + az * az);
        ax *= inv;
        ay *= inv;
        az *= inv;
        float th = 0.f;
        for (int lt = l; lt < 64; lt += 32)
            if (sValid[lt]) {
                const float4 c = sCone[lt];
                const float cx = ay * c.z - az * c.y, cy = az * c.x - ax * c.z, cz = ax * c.y - ay * c.x;
                const float sn = sqrtf(cx * cx + cy * cy + cz * cz);
                const float cs = ax * c.x + ay * c.y + az * c.z;
                const float ang = atan2f(sn, cs) + atan2f(sSin[lt], c.w);
                th = fmaxf(th, ang);
            }
        for (int o = 16; o > 0; o >>= 1) th = fmaxf(th, __shfl_xor_sync(kFull, th, o));
        if (l == 0) {
            // absolute + relative padding: float rounding of the exact tile
            // test is ~1e-6 relative, the pad is two orders above it.
            th = th * 1.0001f + 2e-4f;
            fb.sbCones[sb] = make_float4(ax, ay, az, th);
        }
    }
}

// Conservative superblock test: true whenever cone_may_touch would be true
// for at least one of its tiles ("coarse cull").
__device__ __forceinline__ bool sb_may_touch(float4 sc, F3 apex, const Sphere& s) {
    const float th = sc.w;
    if (th >= 1.5f) return true;
    const float vx = s.c.x - apex.x, vy = s.c.y - apex.y, vz = s.c.z - apex.z;
    const float d2 = vx * vx + vy * vy + vz * vz;
    const float len = sqrtf(d2);
    const float pad = 1e-4f * len + 1e-5f * fabsf(s.r) + 1e-6f;
    if (len <= s.r + pad) return true;
    const float x = vx * sc.x + vy * sc.y + vz * sc.z;
    float sn, cs;
    sincosf(th, &sn, &cs);
    if (x < len * sn + pad) return true;  // wrap-around region behind the cone
    const float y = sqrtf(fmaxf(d2 - x * x, 0.0f));
    return cs * y - sn * x <= s.r + pad;
}

// Superblock rectangle [x0, x1) x [y0, y1) that contains the screen
// projection of a bounding sphere, conservatively: the tangent slopes of the
// sphere seen from the camera (in double, radius and rectangle padded far
// beyond float rounding of the pixel rays).  A sphere reaching the camera
// plane keeps the whole screen.  Only a superset filter: the per-superblock
// pyramid / cone culls and the exact tile tests decide.
__device__ void sphere_sb_rect(const Cam& c, const Sphere& s, int tilesX, int tilesY, int& x0, int& x1, int& y0,
                               int& y1) {
    const int sbX = (tilesX + kSB - 1) / kSB, sbY = (tilesY + kSB - 1) / kSB;
    x0 = 0, x1 = sbX, y0 = 0, y1 = sbY;
    const double vx = (double)s.c.x - c.pos.x, vy = (double)s.c.y - c.pos.y, vz = (double)s.c.z - c.pos.z;
    const double X = vx * c.right.x + vy * c.right.y + vz * c.right.z;
    const double Y = vx * c.up.x + vy * c.up.y + vz * c.up.z;
    const double Z = vx * c.fwd.x + vy * c.fwd.y + vz * c.fwd.z;
    const double R = fabs((double)s.r) * 1.001 + 1e-4 + 1e-4 * sqrt(X * X + Y * Y + Z * Z);
    if (!(Z > 1.01 * R + 1e-6)) return;
    const double den = Z * Z - R * R;
    const double dx = sqrt(X * X + den), dy = sqrt(Y * Y + den);
    const double ka = (double)c.tanHalf * c.aspect, kb = (double)c.tanHalf;
    const double pad = 2.0 * kTile;  // pixels
    const double px0 = ((X * Z - R * dx) / den / ka + 1.0) * 0.5 * c.width - 0.5 - pad;
    const double px1 = ((X * Z + R * dx) / den / ka + 1.0) * 0.5 * c.width - 0.5 + pad;
    const double py0 = (1.0 - (Y * Z + R * dy) / den / kb) * 0.5 * c.height - 0.5 - pad;
    const double py1 = (1.0 - (Y * Z - R * dy) / den / kb) * 0.5 * c.height - 0.5 + pad;
    const double sbPx = (double)(kSB * kTile);
    x0 = (int)fmax(0.0, floor(px0 / sbPx));
    x1 = (int)fmin((double)sbX, floor(px1 / sbPx) + 1.0);
    y0 = (int)fmax(0.0, floor(py0 / sbPx));
    y1 = (int)fmin((double)sbY, floor(py1 / sbPx) + 1.0);
}

// one warp per volume: near/far cull (abuffer.cpp:188-191), then the
// coarse superblock cull over the superblocks its bounding sphere projects
// onto; surviving (volume, superblock) pairs are appended.
__global__ void __launch_bounds__(256) k_pairs(Cam cam, const Voi* vois, uint32_t nvoi, FrameBufs fb,
                                                int tilesX, int tilesY, uint32_t tile0,
                                                uint32_t tile1, int sbLo, int sbHi) {
    // warp = (volume, chunk of 32 superblocks): grid.y runs over the chunks
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nvoi) return;
    const Voi v = vois[warp];
    const Sphere bs = bounding_sphere(v);
    const float vz = view_z(cam, bs.c);
    if (E::add(vz, bs.r) < cam.nearZ || E::sub(vz, bs.r) > cam.farZ) return;
    const VolumeSupport sup = volume_support(v, cam.pos);
    const int sbX = (tilesX + kSB - 1) / kSB;
    // the volume's ray-test terms for this camera, once per frame (k_tile_raster)
    if (blockIdx.y == 0 && lane == 0) {
        fb.rasterVols[warp] = raster_vol_make(v, cam.pos);
        fb.cullVols[warp] = cull_vol_make(bs, sup, cam.pos);
    }
    int rx0, rx1, ry0, ry1;
    sphere_sb_rect(cam, bs, tilesX, tilesY, rx0, rx1, ry0, ry1);
    // ... within the superblock rows [sbLo, sbHi) that meet [tile0, tile1)
    ry0 = max(ry0, sbLo / sbX);
    ry1 = min(ry1, sbHi / sbX);
    const int rw = rx1 - rx0, nrect = (rw > 0 && ry1 > ry0) ? rw * (ry1 - ry0) : 0;
    for (int base = 32 * (int)blockIdx.y; base < nrect; base += 32 * (int)gridDim.y) {
        const int idx = base + lane;
        bool pass = false;
        int sb = 0;
        if (idx < nrect) {
            const int sx = rx0 + idx % rw, sy = ry0 + idx / rw;
            sb = sy * sbX + sx;
            const uint32_t first = (uint32_t)(sy * kSB * tilesX + sx * kSB);
            const int lastTy = min(sy * kSB + kSB, tilesY) - 1, lastTx = min(sx * kSB + kSB, tilesX) - 1;
            const uint32_t last = (uint32_t)(lastTy * tilesX + lastTx);
            if (last >= tile0 && first < tile1)
                pass = volume_pyramid_may_touch(fb.sbFrustum + (size_t)sb * 4, cam.pos, sup) &&
                       sb_may_touch(fb.sbCones[sb], cam.pos, bs);
        }
        const uint32_t m = __ballot_sync(kFull, pass);
        if (m == 0u) continue;
        if (lane == 0) atomicAdd(&fb.counters[kCntPairs], (uint32_t)__popc(m));
        if (pass) {  // straight into the superblock's list (lanes of a warp hold distinct superblocks)
            const uint32_t slot = atomicAdd(&fb.sbCount[sb], 1u);
            if (slot < fb.sbCap) fb.sbList[(size_t)sb * fb.sbCap + slot] = warp;
            else atomicMax(&fb.counters[kCntSbNeed], slot + 1u);  // the checked path grows sbCap
        }
    }
}

// Single-pass exclusive scan of n counts: every 1024-thread block scans 4096
// counts locally and publishes its sum; the last block to finish scans the
// block sums.  offset(i) = local[i] + blockPrefix[i / 4096]; the total is
// blockPrefix[nblocks].
struct ScanArgs {
    const uint32_t* count;
    uint32_t* local;
    uint32_t* blockSum;
    uint32_t* blockPrefix;
    uint32_t* done;
};

__global__ void __launch_bounds__(1024) k_scan(ScanArgs a, uint32_t n) {
    __shared__ uint32_t warpSums[32];
    __shared__ bool amLast;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t base = blockIdx.x * kScanBlock + tid * 4;
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (base + k < n) ? a.count[base + k] : 0u;
    const uint32_t local = v[0] + v[1] + v[2] + v[3];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nb = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += nb;
    }
    if (lane == 31) warpSums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t sm = warpSums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nb = __shfl_up_sync(kFull, sm, o);
            if (lane >= o) sm += nb;
        }
        warpSums[lane] = sm;  // inclusive
    }
    __syncthreads();
    uint32_t run = incl - local + (wid > 0 ? warpSums[wid - 1] : 0u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < n) a.local[base + k] = run;
        run += v[k];
    }
    if (tid == 0) {
        a.blockSum[blockIdx.x] = warpSums[31];
        __threadfence();
        const uint32_t done = atomicAdd(a.done, 1u);
        amLast = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (amLast && wid == 0) {
        __threadfence();
        uint32_t carry = 0;
        for (uint32_t b0 = 0; b0 < gridDim.x; b0 += 32) {
            const uint32_t b = b0 + lane;
            const uint32_t sv = b < gridDim.x ? *((volatile uint32_t*)&a.blockSum[b]) : 0u;
            uint32_t inc = sv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nb = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += nb;
            }
            if (b < gridDim.x) a.blockPrefix[b] = carry + inc - sv;
            carry += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) {
            a.blockPrefix[gridDim.x] = carry;
            *a.done = 0u;  // ready for the next scan on this counter
        }
    }
}

// --- CSR of the A-buffer for a download (the frame itself never needs it)
__global__ void k_frag_counts(FrameBufs fb, uint32_t tiles) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tiles) fb.tileCount[t] = fb.tileFrag[t].y;
}

__global__ void k_frag_offsets(FrameBufs fb, uint32_t tiles) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > tiles) return;
    fb.offsets[t] = t < tiles ? fb.tileLocal[t] + fb.blockPrefix[t / kScanBlock]
                              : fb.blockPrefix[(tiles + kScanBlock - 1) / kScanBlock];
}

// warp per tile: the tile's sorted list -> its CSR slots (fb.unsorted as Frag)
__global__ void k_frag_copy(FrameBufs fb, uint32_t tiles) {
    const uint32_t lane = threadIdx.x & 31u;
    Frag* csr = reinterpret_cast<Frag*>(fb.unsorted);
    for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles; t += (gridDim.x * blockDim.x) >> 5) {
        const uint2 tf = fb.tileFrag[t];
        const uint32_t o = fb.offsets[t];
        for (uint32_t i = lane; i < tf.y; i += 32) csr[o + i] = fb.frags[tf.x + i];
    }
}

// an uploaded CSR A-buffer: every tile's list is its CSR range
__global__ void k_tile_frag_from_offsets(FrameBufs fb, uint32_t tiles) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tiles) fb.tileFrag[t] = make_uint2(fb.offsets[t], fb.offsets[t + 1] - fb.offsets[t]);
}

}  // namespace

// ---------------------------------------------------------------- launchers

void launch_params_update(cudaStream_t st, float4* words, const uint32_t* dWords,
                          const float* dParams, const uint32_t* dCounts, uint32_t n,
                          uint32_t stride) {
    if (n == 0) return;
    dim3 block(32, 8);
    k_params_update<<<(n + 7) / 8, block, 0, st>>>(words, dWords, dParams, dCounts, n, stride);
}

void launch_roi_all(cudaStream_t st, const DevTree& t, float* roi) {
    if (t.nnodes == 0) return;
    k_roi_all<<<(t.nnodes + 255) / 256, 256, 0, st>>>(t, roi);
}

void launch_voi(cudaStream_t st, const DevTree& t, const float* roi, float margin, Voi* vois) {
    if (t.nprims == 0) return;
    k_voi<<<(t.nprims + 127) / 128, 128, 0, st>>>(t, roi, margin, vois);
}

// Superblocks [sbLo, sbHi) whose rows meet the tile range [tile0, tile1).
static void sb_range(int tilesX, int tilesY, uint32_t tile0, uint32_t tile1, int& sbLo, int& sbHi) {
    const int sbX = (tilesX + kSB - 1) / kSB, sbY = (tilesY + kSB - 1) / kSB;
    if (tile1 <= tile0) {
        sbLo = sbHi = 0;
        return;
    }
    const int row0 = (int)(tile0 / (uint32_t)tilesX) / kSB, row1 = (int)((tile1 - 1) / (uint32_t)tilesX) / kSB + 1;
    sbLo = row0 * sbX;
    sbHi = std::min(row1, sbY) * sbX;
}

uint32_t camera_tile_cover(int tilesX, int tilesY, uint32_t tile0, uint32_t tile1, uint32_t* cover0) {
    int sbLo, sbHi;
    sb_range(tilesX, tilesY, tile0, tile1, sbLo, sbHi);
    const int sbX = (tilesX + kSB - 1) / kSB;
    const uint32_t tiles = (uint32_t)(tilesX * tilesY);
    *cover0 = std::min<uint32_t>(tiles, (uint32_t)(sbLo / sbX) * kSB * (uint32_t)tilesX);
    return std::min<uint32_t>(tiles, (uint32_t)(sbHi / sbX) * kSB * (uint32_t)tilesX);
}

void launch_camera(cudaStream_t st, const Cam& cam, const FrameBufs& fb, int tilesX, int tilesY, uint32_t tile0,
                   uint32_t tile1) {
    int sbLo, sbHi;
    sb_range(tilesX, tilesY, tile0, tile1, sbLo, sbHi);
    if (sbHi > sbLo) k_camera<<<sbHi - sbLo, 256, 0, st>>>(cam, fb, tilesX, tilesY, sbLo);
}

uint32_t superblock_count(int tilesX, int tilesY) {
    return (uint32_t)(((tilesX + kSB - 1) / kSB) * ((tilesY + kSB - 1) / kSB));
}

// Superblock stage of the A-buffer: (volume, superblock) pairs, grouped by
// superblock.  The per-tile stage is launch_tile_pass (k_tile.cu).
void launch_abuffer(cudaStream_t st, const Cam& cam, const Voi* vois, uint32_t nvoi,
                    const FrameBufs& fb, int tilesX, int tilesY, uint32_t tile0, uint32_t tile1,
                    int smCount, bool zero) {
    const uint32_t nsbAll = superblock_count(tilesX, tilesY);
    if (zero) {
        cudaMemsetAsync(fb.counters, 0, kCntSlots * sizeof(uint32_t), st);
        cudaMemsetAsync(fb.sbCount, 0, nsbAll * sizeof(uint32_t), st);
    }
    if (nvoi > 0) {
        int sbLo, sbHi;
        sb_range(tilesX, tilesY, tile0, tile1, sbLo, sbHi);
        const uint32_t nsb = (uint32_t)(sbHi - sbLo);
        // (volume, chunk) warps: a volume's superblock rectangle is usually a
        // few superblocks, so chunks only help when there are few volumes
        // (each chunk warp repeats the volume's setup and rectangle)
        const uint32_t chunks =
            std::max<uint32_t>(1u, std::min<uint32_t>((nsb + 31) / 32, std::max<uint32_t>(1u, 2048u / nvoi)));
        const dim3 grid((nvoi * 32 + 255) / 256, chunks);
        k_pairs<<<grid, 256, 0, st>>>(cam, vois, nvoi, fb, tilesX, tilesY, tile0, tile1, sbLo, sbHi);
    }
}

void launch_frag_csr(cudaStream_t st, const FrameBufs& fb, uint32_t tiles, int smCount) {
    k_frag_counts<<<(tiles + 255) / 256, 256, 0, st>>>(fb, tiles);
    ScanArgs a{fb.tileCount, fb.tileLocal, fb.blockSum, fb.blockPrefix, fb.counters + kCntScanDone};
    k_scan<<<(tiles + kScanBlock - 1) / kScanBlock, 1024, 0, st>>>(a, tiles);
    k_frag_offsets<<<(tiles + 256) / 256, 256, 0, st>>>(fb, tiles);
    k_frag_copy<<<smCount * 4, 256, 0, st>>>(fb, tiles);
}

void launch_tile_frag_from_offsets(cudaStream_t st, const FrameBufs& fb, uint32_t tiles) {
    k_tile_frag_from_offsets<<<(tiles + 255) / 256, 256, 0, st>>>(fb, tiles);
}

}  // namespace btk
