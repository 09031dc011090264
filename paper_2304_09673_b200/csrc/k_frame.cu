// k_frame.cu -- stages (a) and (b) on sm_100a.
//
//   k_params_update  per-frame primitive parameter rewrite      (linear_tree.cpp:187-193)
//   k_roi_all        range of interest per node                 (linear_tree.cpp:170-185)
//   k_voi            volume of interest per primitive           (linear_tree.cpp:216-283)
//   k_camera         pixel rays, tile cones, superblock cones   (camera.cpp:29-37, abuffer.cpp:117-149)
//   k_pairs          (volume, superblock) coarse cull           (superset of abuffer.cpp:193-196)
//   k_tiles          exact tile cone + pixel pyramid per tile   (abuffer.cpp:193-196)
//   k_raster         64 exact pixel-ray intervals per item      (abuffer.cpp:198-222)
//   k_scan           tile counts -> CSR offsets (single pass)
//   k_scatter        unsorted pool -> CSR slots
//   k_sort           per-tile rank sort by (zEntry, word)       (insert_sorted, abuffer.cpp:166-173)
//
// Everything on the A-buffer path is evaluated with ExactOps (no FMA, IEEE
// div/sqrt), so (tile, word) membership and (zEntry, zExit) are bit-exact
// with the reference's single-threaded rasterize_volumes.
#include <algorithm>

#include "bt_device.h"

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kScanBlock = 4096;  // tiles per scan block (1024 threads x 4)

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

// Conservative volume-vs-pyramid test with a relative + absolute pad that
// dominates every FP32 rounding on both sides.  Oriented boxes and capsules
// use their own support along each inward plane normal, not their bounding
// sphere's (19 % fewer (tile, volume) pairs to ray-test at C3).
// A box (centre c, half-axis vectors A_i = h_i rotate(q, e_i); q is a unit
// quaternion to 1e-6, validate_primitive) reaches n.(c - apex) + sum |n.A_i|;
// a capsule max(n.(a - apex), n.(b - apex)) + r.  Same relative + absolute pad
// as the sphere test, plus for capsules the cancellation error of the exact
// capsule quadratic (~ulp(dist^2) / r in distance).  A pixel ray that the
// exact test intersects lies inside the pyramid, so the volume reaches every
// plane: a rejected (tile, volume) pair cannot produce a fragment.
struct VolumeSupport {
    uint32_t family;
    F3 c, a0, a1, a2;  // box: centre, half-axis vectors; capsule: a0, a1 = ends
    float r, pad;
};

__device__ __forceinline__ VolumeSupport volume_support(const Voi& v, F3 apex) {
    VolumeSupport s;
    s.family = v.family;
    const Sphere bs = bounding_sphere(v);
    const float vx = bs.c.x - apex.x, vy = bs.c.y - apex.y, vz = bs.c.z - apex.z;
    const float dist = sqrtf(vx * vx + vy * vy + vz * vz);
    s.pad = 1e-4f * (dist + fabsf(bs.r)) + 1e-5f;
    if (v.family == 1u) {
        const float w = v.rot.w, x = v.rot.x, y = v.rot.y, z = v.rot.z;
        // columns of the rotation matrix of q, scaled by the half extents
        s.a0 = F3{(1.f - 2.f * (y * y + z * z)) * v.half.x, 2.f * (x * y + w * z) * v.half.x, 2.f * (x * z - w * y) * v.half.x};
        s.a1 = F3{2.f * (x * y - w * z) * v.half.y, (1.f - 2.f * (x * x + z * z)) * v.half.y, 2.f * (y * z + w * x) * v.half.y};
        s.a2 = F3{2.f * (x * z + w * y) * v.half.z, 2.f * (y * z - w * x) * v.half.z, (1.f - 2.f * (x * x + y * y)) * v.half.z};
        s.c = v.center;
        s.r = 0.0f;
    } else if (v.family == 2u) {
        s.a0 = v.center;
        s.a1 = v.axisEnd;
        s.r = v.radius;
        s.pad += 2.5e-7f * dist * dist / fmaxf(v.radius, 1e-6f);
    } else {
        s.c = bs.c;
        s.r = bs.r;
    }
    return s;
}

__device__ __forceinline__ bool volume_pyramid_may_touch(const float4* pl, F3 apex, const VolumeSupport& s) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float4 n = pl[e];
        float reach;
        if (s.family == 1u) {
            reach = n.x * (s.c.x - apex.x) + n.y * (s.c.y - apex.y) + n.z * (s.c.z - apex.z) +
                    fabsf(n.x * s.a0.x + n.y * s.a0.y + n.z * s.a0.z) +
                    fabsf(n.x * s.a1.x + n.y * s.a1.y + n.z * s.a1.z) +
                    fabsf(n.x * s.a2.x + n.y * s.a2.y + n.z * s.a2.z);
        } else if (s.family == 2u) {
            reach = fmaxf(n.x * (s.a0.x - apex.x) + n.y * (s.a0.y - apex.y) + n.z * (s.a0.z - apex.z),
                          n.x * (s.a1.x - apex.x) + n.y * (s.a1.y - apex.y) + n.z * (s.a1.z - apex.z)) + s.r;
        } else {
            reach = n.x * (s.c.x - apex.x) + n.y * (s.c.y - apex.y) + n.z * (s.c.z - apex.z) + s.r;
        }
        if (reach < -s.pad) return false;
    }
    return true;
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
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(&fb.counters[kCntPairs], (uint32_t)__popc(m));
        slot = __shfl_sync(kFull, slot, 0) + __popc(m & ((1u << lane) - 1u));
        if (pass && slot < fb.pairCap) fb.pairs[slot] = make_uint2(warp, (uint32_t)sb);
    }
}

// One warp per (volume, superblock) pair, grid-stride: every lane tests two of
// the superblock's 64 tiles with the exact reference cone (abuffer.cpp:193-196)
// and the tile's pixel-centre pyramid; surviving (tile, volume) items are
// appended with ONE warp-aggregated atomic per pair.
__global__ void __launch_bounds__(256) k_tiles(Cam cam, const Voi* vois, FrameBufs fb, int tilesX, int tilesY,
                                                uint32_t tile0, uint32_t tile1) {
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t npairs = min((uint64_t)fb.counters[kCntPairs], fb.pairCap);
    const int sbX = (tilesX + kSB - 1) / kSB;
    for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < npairs; p += nwarps) {
        const uint2 pr = fb.pairs[p];
        const Voi vol = vois[pr.x];
        const Sphere bs = bounding_sphere(vol);
        const VolumeSupport sup = volume_support(vol, cam.pos);
        const int sx = pr.y % sbX, sy = pr.y / sbX;
        bool pass[2];
        uint32_t tiles[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int lt = lane + 32 * h;
            const int tx = sx * kSB + (lt & 7), ty = sy * kSB + (lt >> 3);
            pass[h] = false;
            tiles[h] = (uint32_t)(ty * tilesX + tx);
            if (tx < tilesX && ty < tilesY && tiles[h] >= tile0 && tiles[h] < tile1) {
                const float4 c = fb.cones[tiles[h]];
                Cone k;
                k.axis = F3{c.x, c.y, c.z};
                k.cosH = c.w;
                k.sinH = fb.coneSin[tiles[h]];
                pass[h] = cone_may_touch(k, cam.pos, bs) &&
                          volume_pyramid_may_touch(fb.tileFrustum + (size_t)tiles[h] * 4, cam.pos, sup);
            }
        }
        const uint32_t m0 = __ballot_sync(kFull, pass[0]), m1 = __ballot_sync(kFull, pass[1]);
        const uint32_t n = __popc(m0) + __popc(m1);
        if (n == 0) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&fb.counters[kCntPool], n);
        base = __shfl_sync(kFull, base, 0);
        const uint32_t below = (1u << lane) - 1u;
        if (pass[0]) {
            const uint32_t slot = base + __popc(m0 & below);
            if (slot < fb.poolCap) fb.pool[slot] = make_uint4(tiles[0], pr.x, 0u, 0u);
        }
        if (pass[1]) {
            const uint32_t slot = base + __popc(m0) + __popc(m1 & below);
            if (slot < fb.poolCap) fb.pool[slot] = make_uint4(tiles[1], pr.x, 0u, 0u);
        }
    }
}

constexpr uint32_t kNoFragment = 0xFFFFFFFFu;

// One warp per (tile, volume) item, grid-stride: the tile's 64 pixel rays (two
// per lane) are intersected with the volume exactly (abuffer.cpp:200-216),
// clipped to [near, far], mapped to NDC and reduced with min/max (order-free
// on these finite values).  The fragment lands in the item's own slot, so no
// global append counter is contended; misses mark the slot empty.
__global__ void __launch_bounds__(256, BT_RASTER_MINB) k_raster(Cam cam, const Voi* vois, FrameBufs fb) {
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nitems = min((uint64_t)fb.counters[kCntPool], fb.poolCap);
    for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nitems; it += nwarps) {
        const uint4 item = fb.pool[it];
        const uint32_t tile = item.x;
        const Voi v = vois[item.y];
        const int tilesX = (cam.width + kTile - 1) / kTile;
        const int tx = (int)(tile % (uint32_t)tilesX), ty = (int)(tile / (uint32_t)tilesX);
        F3 ol{0.f, 0.f, 0.f};
        if (v.family == 1u) ol = qrotate<E>(qconj(v.rot), vsub<E>(cam.pos, v.center));
        float entry = f_inf(), exitv = -f_inf();
        bool any = false;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int pix = lane + 32 * h;
            const int px = tx * kTile + (pix & 7), py = ty * kTile + (pix >> 3);
            if (px >= cam.width || py >= cam.height) continue;
            const float4 rd = fb.rays[(size_t)tile * 64 + pix];
            const F3 d{rd.x, rd.y, rd.z};
            float t0, t1;
            bool hit;
            if (v.family == 0u)
                hit = ray_sphere(cam.pos, d, v.center, v.radius, t0, t1);
            else if (v.family == 1u)
                hit = ray_obb_local(ol, d, v.rot, v.half, t0, t1);
            else
                hit = ray_capsule(cam.pos, d, v.center, v.axisEnd, v.radius, t0, t1);
            if (!hit) continue;
            float vz0 = E::mul(t0, rd.w), vz1 = E::mul(t1, rd.w);
            if (vz1 < cam.nearZ || vz0 > cam.farZ) continue;
            vz0 = smax(vz0, cam.nearZ);
            vz1 = smin(vz1, cam.farZ);
            entry = smin(entry, vz0);  // view z for now: NDC is applied once per item below
            exitv = smax(exitv, vz1);
            any = true;
        }
        if (!__any_sync(kFull, any)) {
            if (lane == 0) fb.pool[it].x = kNoFragment;
            continue;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            entry = smin(entry, __shfl_xor_sync(kFull, entry, o));
            exitv = smax(exitv, __shfl_xor_sync(kFull, exitv, o));
        }
        // ndc_from_view_z is monotone non-decreasing in vz (correctly rounded
        // 1/vz, subtraction and scaling are each monotone), so the min / max
        // over the rays of ndc(vz) is ndc of the min / max vz -- bit for bit
        // the reference's per-ray min/max (abuffer.cpp:206-213), with two
        // divisions per item instead of two per ray.
        entry = ndc_from_view_z(cam, entry);
        exitv = ndc_from_view_z(cam, exitv);
        if (lane == 0) {
            fb.pool[it] = make_uint4(tile, item.y, __float_as_uint(entry), __float_as_uint(exitv));
            atomicAdd(&fb.tileCount[tile], 1u);
        }
    }
}

// Single-pass scan: every 1024-thread block scans 4096 tile counts locally
// and publishes its sum; the last block to finish scans the block sums.
// offset(tile) = tileLocal[tile] + blockPrefix[tile / 4096].
__global__ void __launch_bounds__(1024) k_scan(FrameBufs fb, uint32_t tiles) {
    __shared__ uint32_t warpSums[32];
    __shared__ bool amLast;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t base = blockIdx.x * kScanBlock + tid * 4;
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (base + k < tiles) ? fb.tileCount[base + k] : 0u;
    const uint32_t local = v[0] + v[1] + v[2] + v[3];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) warpSums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = warpSums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += n;
        }
        warpSums[lane] = s;  // inclusive
    }
    __syncthreads();
    uint32_t run = incl - local + (wid > 0 ? warpSums[wid - 1] : 0u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (base + k < tiles) fb.tileLocal[base + k] = run;
        run += v[k];
    }
    if (tid == 0) {
        fb.blockSum[blockIdx.x] = warpSums[31];
        __threadfence();
        const uint32_t done = atomicAdd(&fb.counters[kCntScanDone], 1u);
        amLast = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (amLast && wid == 0) {
        __threadfence();
        uint32_t carry = 0;
        for (uint32_t b0 = 0; b0 < gridDim.x; b0 += 32) {
            const uint32_t b = b0 + lane;
            const uint32_t s = b < gridDim.x ? *((volatile uint32_t*)&fb.blockSum[b]) : 0u;
            uint32_t inc = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t n = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += n;
            }
            if (b < gridDim.x) fb.blockPrefix[b] = carry + inc - s;
            carry += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) fb.blockPrefix[gridDim.x] = carry;
    }
}

__device__ __forceinline__ uint32_t tile_offset(const FrameBufs& fb, uint32_t tile) {
    return fb.tileLocal[tile] + fb.blockPrefix[tile / kScanBlock];
}

// true when this frame's fragments do not fit the pool (the host grows the
// buffers and rebuilds; in a graph replay the A-buffer degrades to empty)
__device__ __forceinline__ bool pool_overflowed(const FrameBufs& fb) {
    return (uint64_t)fb.counters[kCntPool] > fb.poolCap || (uint64_t)fb.counters[kCntPairs] > fb.pairCap;
}

__global__ void k_scatter(const Voi* vois, FrameBufs fb) {
    if (pool_overflowed(fb)) return;
    const uint32_t n = min((uint64_t)fb.counters[kCntPool], fb.poolCap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint4 r = fb.pool[i];
        if (r.x == kNoFragment) continue;
        const uint32_t slot = tile_offset(fb, r.x) + atomicAdd(&fb.tileCursor[r.x], 1u);
        fb.unsorted[slot] = make_uint4(vois[r.y].word, r.z, r.w, r.y);
    }
}

// key order of insert_sorted: (zEntry, word); equal keys keep volume order
// (upper_bound insertion in volume order), hence the volume index tiebreak.
__device__ __forceinline__ bool key_less(const uint4& a, const uint4& b) {
    const float ea = __uint_as_float(a.y), eb = __uint_as_float(b.y);
    if (ea != eb) return ea < eb;
    if (a.x != b.x) return a.x < b.x;
    return a.w < b.w;
}

constexpr int kSortStage = 256;

// Warp per tile of [first, last) (the frame's tile range).
__global__ void __launch_bounds__(128) k_sort(FrameBufs fb, uint32_t tiles, uint32_t first, uint32_t last) {
    __shared__ uint4 stage[4][kSortStage];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = first + blockIdx.x * 4 + wid;
    if (tile >= last) return;
    if (pool_overflowed(fb)) {  // never index past the pool: empty A-buffer, flagged
        if (lane == 0) {
            fb.offsets[tile] = 0;
            if (tile == tiles - 1) fb.offsets[tiles] = 0;
            if (tile == first) atomicExch(&fb.counters[kCntOverflow], 1u);
        }
        return;
    }
    const uint32_t n = fb.tileCount[tile];
    const uint32_t off = tile_offset(fb, tile);
    fb.offsets[tile] = off;
    if (tile == tiles - 1 && lane == 0) fb.offsets[tiles] = off + n;
    if (n == 0) return;
    const uint4* src = fb.unsorted + off;
    const bool staged = n <= (uint32_t)kSortStage;
    if (staged)
        for (uint32_t i = lane; i < n; i += 32) stage[wid][i] = src[i];
    __syncwarp();
    const uint4* keys = staged ? stage[wid] : src;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint4 me = keys[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < n; ++j) rank += key_less(keys[j], me) ? 1u : 0u;
        Frag f;
        f.word = me.x;
        f.zEntry = __uint_as_float(me.y);
        f.zExit = __uint_as_float(me.z);
        fb.frags[off + rank] = f;
    }
}

// CSR offsets of every tile, thread per tile: a sharded frame sorts only its
// own tile range, the other tiles are empty but keep valid offsets.
__global__ void k_offsets_all(FrameBufs fb, uint32_t tiles) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tiles) return;
    const bool ov = pool_overflowed(fb);
    const uint32_t off = ov ? 0u : tile_offset(fb, t);
    fb.offsets[t] = off;
    if (t == tiles - 1) fb.offsets[tiles] = ov ? 0u : off + fb.tileCount[t];
}

__global__ void k_offsets_from_counts(FrameBufs fb, uint32_t tiles) {
    // used when the A-buffer was uploaded: counts from CSR offsets
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < tiles) fb.tileCount[i] = fb.offsets[i + 1] - fb.offsets[i];
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

void launch_abuffer(cudaStream_t st, const Cam& cam, const Voi* vois, uint32_t nvoi,
                    const FrameBufs& fb, int tilesX, int tilesY, uint32_t tile0, uint32_t tile1,
                    int smCount, bool zero) {
    const uint32_t tiles = (uint32_t)(tilesX * tilesY);
    if (zero) {
        cudaMemsetAsync(fb.counters, 0, kCntSlots * sizeof(uint32_t), st);
        cudaMemsetAsync(fb.tileCount, 0, tiles * sizeof(uint32_t), st);
        cudaMemsetAsync(fb.tileCursor, 0, tiles * sizeof(uint32_t), st);
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
        k_tiles<<<smCount * 8, 256, 0, st>>>(cam, vois, fb, tilesX, tilesY, tile0, tile1);
        k_raster<<<smCount * 8, 256, 0, st>>>(cam, vois, fb);
    }
    const uint32_t nblocks = (tiles + kScanBlock - 1) / kScanBlock;
    k_scan<<<nblocks, 1024, 0, st>>>(fb, tiles);
    k_scatter<<<smCount * 4, 256, 0, st>>>(vois, fb);
    if (tile0 == 0 && tile1 >= tiles) {
        k_sort<<<(tiles + 3) / 4, 128, 0, st>>>(fb, tiles, 0u, tiles);
    } else {
        k_offsets_all<<<(tiles + 255) / 256, 256, 0, st>>>(fb, tiles);
        const uint32_t last = std::min(tile1, tiles);
        if (last > tile0) k_sort<<<(last - tile0 + 3) / 4, 128, 0, st>>>(fb, tiles, tile0, last);
    }
}

void launch_offsets_from_counts(cudaStream_t st, const FrameBufs& fb, uint32_t tiles) {
    k_offsets_from_counts<<<(tiles + 255) / 256, 256, 0, st>>>(fb, tiles);
}

}  // namespace btk
