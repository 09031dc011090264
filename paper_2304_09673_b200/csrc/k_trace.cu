// k_trace.cu -- stage (c) on sm_100a, part 2: synchronized sphere tracing
// over the compiled intervals (k_views.cu), normals, and the GPU brute-force
// oracle.
//
//   k_march<O>     one warp per 8x8 tile (persistent, tile queue).  Per
//                  interval record: stage the pruned view into this warp's
//                  shared memory (fast path: lane-parallel conversion into
//                  evaluation-ready parameter blocks), then march the tile's
//                  unfinished rays in lockstep.  Rays are served from a
//                  warp-synchronous queue: a lane whose ray finished takes the
//                  next pending ray of the interval (ballot + popc rank), so
//                  64 rays keep 32 lanes busy until the queue drains
//                  (render_tiles, tracer.cpp:141-236).
//   k_normals      depth-differential normals (tracer.cpp:296-350); pixels
//                  without usable neighbours are queued for k_gradient.
//   k_gradient<O>  6-tap eval_full fallback (traversal.cpp:126-141).
//   k_oracle<O>    oracle_render (tracer.cpp:238-280): every pixel marched
//                  over [near, far] on the full tree.
//
// O = ExactOps gives bit-identical results to the CPU reference; O = FastOps
// lets nvcc contract the field arithmetic into FFMA (tolerance path).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "bt_bulk.cuh"
#include "bt_device.h"
#include "bt_fast.cuh"
#include "bt_views.cuh"

namespace btk {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kTraceWarps = 4;
constexpr int kFullStackCap = 128;
#ifndef BT_MARCH_BLOCKS
#define BT_MARCH_BLOCKS 320
#endif
constexpr uint32_t kMarchBlocks = BT_MARCH_BLOCKS;  // float4s of fast parameter blocks kept in shared memory per warp
constexpr uint32_t kNoRay = 0xFFFFFFFFu;

template <class O> __device__ __forceinline__ F3 ray_point(F3 o, F3 d, float t) {
    return vadd<O>(o, vscale<O>(d, t));
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class O> struct IsFast {
    static constexpr bool value = false;
};
template <> struct IsFast<FastOps> {
    static constexpr bool value = true;
};

#ifdef BT_STEP_HIST
__device__ unsigned long long g_stepHist[33];
__device__ unsigned int g_stepDone;
#endif

// Per-warp shared memory of k_march.
struct MarchSmem {
    float4 blocks[kMarchBlocks];  // fast parameter blocks of the staged view
    float4 rays[64];              // dir.xyz, dot(dir, forward) of the tile's rays (one bulk copy)
    uint32_t hdr[kViewCap];       // staged view: isPrim(1) op(5) | block byte offset
    union {
        uint32_t word[kViewCap + 1];      // exact path / raw parameters: tree word of each node
        uint2 rec[(kViewCap + 1) / 2];    // fast path: comb records (bt_fast.cuh, comb_*_rec)
    };
    float depth[64];
    uint32_t evals[64];
    uint8_t hit[64];
    uint8_t pend[64];             // rays still to march in this interval, in order
    // per-tile accounting, kept here rather than in registers live across the march
    uint32_t accFe[32], accFl[32], accRnv[32], accPe[32];
    uint32_t tileMaxOv, tileCache, tileErr, steps;
    uint64_t rayBar;              // completion barrier of the rays' bulk copy
};

// Per-block work accounting, flushed to the device statistics once per CTA.
struct BlockStats {
    unsigned long long fe, rnv, pe, fl, steps, errs;
    unsigned int maxOv, maxCache;
};

// View classes of the march loop (bt_fast.cuh, "view classes"): chosen once
// per interval, so the per-step evaluation carries no class test.
constexpr int kClsRaw = 0;      // raw tree parameters (exact path, or a view too large for the blocks)
constexpr int kClsGeneral = 1;  // fast blocks, interpreter
constexpr int kClsSingle = 2;   // fast blocks, one primitive
constexpr int kClsComb = 3;     // fast blocks, left comb P (P O)*
constexpr int kClsCombLip = 4;  // ... with a step bound per sample (bt_set_step_bound(1), compact operators)

// March the pending rays of one interval over the staged view.  `aux`:
// single -> the primitive's comb record; comb -> the primitive count.
template <class O, int Cls>
__device__ __forceinline__ void march_interval(const DevTree& t, const Cam& cam, const TraceParams& tp, MarchSmem& s,
                                               uint32_t aux, uint32_t nView, uint32_t nPend, float vz0, float vz1,
                                               uint32_t lt, uint32_t& fe, uint32_t& fl, uint32_t& steps,
                                               uint32_t flops) {
    const uint32_t uaux = warp_uniform(aux);  // class operand in a uniform register for the whole interval
    uint32_t cursor = 0, ray = kNoRay;
    March m;
    march_idle(m);
    m.evalT = 0.0f;
    F3 dir{0.f, 0.f, 1.f};
    for (;;) {
        // finished lanes are recorded and refilled only in steps where some
        // lane is idle: while all 32 carry a ray, a step costs one ballot here
        const bool idle = march_phase(m) == 0u;
        const uint32_t idleMask = __ballot_sync(kFull, idle);
        if (idleMask != 0u) {
            if (idle && ray != kNoRay) {  // record the ray that just finished
                const uint32_t e = m.evals;
                s.evals[ray] += e;
                if (march_hit(m)) {
                    s.hit[ray] = 1;
                    s.depth[ray] = m.t;
                }
                fe += e;
                fl += e * flops;
                ray = kNoRay;
            }
            if (cursor < nPend) {  // refill idle lanes from the queue
                const uint32_t rank = cursor + __popc(idleMask & lt);
                if (idle && rank < nPend) {
                    ray = s.pend[rank];
                    const float4 r = s.rays[ray];
                    dir = F3{r.x, r.y, r.z};
                    if (IsFast<O>::value) {  // t = view z * (1 / dot(dir, forward))
                        const float iw = FastOps::rcp(r.w);
                        march_begin(m, vz0 * iw, vz1 * iw);
                    } else {
                        march_begin(m, E::div(vz0, r.w), E::div(vz1, r.w));
                    }
                }
                cursor += __popc(idleMask);
            } else if (idleMask == kFull) {
                break;  // queue drained, every lane recorded
            }
            // (a refill whose rays all start empty -- t0 > t1 -- leaves a
            // step with no active lane: it evaluates for nobody and the next
            // iteration records them; rare enough not to pay a second vote)
        }
        ++steps;
#ifdef BT_STEP_HIST
        {  // experiment (scripts/step_hist.sh): histogram of active lanes per lockstep step
            const uint32_t act = __ballot_sync(kFull, march_phase(m) != 0u);
            if ((threadIdx.x & 31) == 0) atomicAdd(&g_stepHist[__popc(act)], 1ull);
        }
#endif
        const F3 p = ray_point<O>(cam.pos, dir, m.evalT);
        float v;
        float margin = 0.0f;
        if constexpr (Cls == kClsSingle) v = fast_prim(uaux, comb_rec_block(s.blocks, uaux), p);
        else if constexpr (Cls == kClsComb) v = eval_comb(s.rec, uaux, s.blocks, p);
        else if constexpr (Cls == kClsCombLip) v = eval_comb_margin(s.rec, uaux, s.blocks, p, margin);
        else if constexpr (Cls == kClsGeneral) eval_view_fast<1>(s.hdr, nView, s.blocks, &p, &v);
        else v = eval_staged<O>(s.hdr, s.word, nView, t.words, p);  // exact path, or an oversized view
        if constexpr (Cls == kClsCombLip) {
            const bool lip1 = margin > fmaxf(tp.relax * v, tp.minStep);
            if (march_phase(m) != 0u) march_consume<true>(m, v, tp, lip1);
        } else {
            if (march_phase(m) != 0u) march_consume(m, v, tp);
        }
    }
}

// Rays of this unit that are inside the image: bit l of word j = ray l + 32j.
__device__ __forceinline__ void unit_rays(const GBuf& g, int tx, int ty, uint32_t mine, uint32_t& v0, uint32_t& v1) {
    const int lane = threadIdx.x & 31;
    const int px = tx * kTile + (lane & 7);
    const int py0 = ty * kTile + (lane >> 3), py1 = py0 + 4;
    v0 = __ballot_sync(kFull, px < g.width && py0 < g.height) & mine;
    v1 = __ballot_sync(kFull, px < g.width && py1 < g.height) & mine;
}

// One 8x8 tile: walk its compiled intervals until all 64 rays have hit
// (tracer.cpp:165-230), then write its pixels and tile planes.  The tile's
// bookkeeping lives in the warp's shared memory, not in registers that would
// stay live across the march loop.
template <class O, bool SB = false>
__device__ __forceinline__ void march_tile(const DevTree& t, const Cam& cam, const TraceParams& tp,
                                           const FrameBufs& fb, const ViewBufs& vb, const GBuf& g, MarchSmem& s,
                                           BlockStats& bs, int lane, uint32_t unit, uint32_t& rayPhase) {
    const uint32_t lt = lanemask_lt();
    // a unit is a whole tile, or half of one (the rays of one pixel-column parity)
    const uint32_t tile = unit & kUnitTile;
    const bool half = (unit & kUnitSplit) != 0u;
    const uint32_t mine = !half ? kFull : ((unit & kUnitPart1) ? 0xAAAAAAAAu : 0x55555555u);
    const int tx = (int)(tile % (uint32_t)g.tilesX), ty = (int)(tile / (uint32_t)g.tilesX);
    if (g.accumulate) {  // a later depth slab: the rays that hit in an earlier one are done
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int li = lane + 32 * j;
            const int px = tx * kTile + (li & 7), py = ty * kTile + (li >> 3);
            const bool in = px < g.width && py < g.height;
            const size_t p = in ? (size_t)py * g.width + px : 0;
            s.hit[li] = in ? g.hit[p] : 0;
            s.depth[li] = in ? g.depth[p] : 0.0f;
            s.evals[li] = in ? g.evalCount[p] : 0u;
        }
    } else {
        s.hit[lane] = 0;
        s.hit[lane + 32] = 0;
        s.evals[lane] = 0;
        s.evals[lane + 32] = 0;
    }
    s.accFe[lane] = s.accFl[lane] = s.accRnv[lane] = s.accPe[lane] = 0;
    if (lane == 0) s.tileMaxOv = s.tileCache = s.tileErr = s.steps = 0;
    __syncwarp();
    const uint2 c = vb.count[tile];
    if (c.x != 0u && vb.counters[1] != 0u) {
        if (lane == 0) s.tileErr = 1;  // interval records overflowed in a graph replay (flagged to the host)
    } else if (c.x != 0u) {
        // the tile's 64 rays: one 1 KB bulk copy (tile-major ray layout)
        if (lane == 0) bulk_load(s.rays, fb.rays + (size_t)tile * 64, 64 * sizeof(float4), &s.rayBar);
        const uint2 o = view_offset(vb, tile);
        mbar_wait(&s.rayBar, rayPhase);
        rayPhase ^= 1u;
        for (uint32_t k = 0; k < c.x; ++k) {
            uint32_t v0, v1;
            unit_rays(g, tx, ty, mine, v0, v1);
            const uint32_t found0 = ~v0 | __ballot_sync(kFull, s.hit[lane] != 0);
            const uint32_t found1 = ~v1 | __ballot_sync(kFull, s.hit[lane + 32] != 0);
            if ((found0 & found1) == kFull) break;
            const uint4* rp = reinterpret_cast<const uint4*>(vb.iv + o.x + k);
            const uint4 ra = rp[0], rb = rp[1];
            const uint32_t flags = rb.x >> 8;
            if (lane == 0) s.tileMaxOv = max(s.tileMaxOv, rb.x & 0xFFu);
            if (flags & kIvErr) {
                if (lane == 0) s.tileErr = 1;
                break;
            }
            if (lane == 0) s.tileCache = max(s.tileCache, rb.y);
            if (!(flags & kIvRootUsed)) continue;
            const float zb = __uint_as_float(ra.x), ze = __uint_as_float(ra.y);
            if (ze <= zb) continue;
            if (flags & kIvDepthErr) {  // eval_pruned would throw on first use
                if (lane == 0) s.tileErr = 1;
                break;
            }
            const uint32_t nView = ra.w & 0xFFFFu;
            // fast path: evaluation-ready parameter blocks in shared memory when
            // the view fits (the common case); otherwise raw parameters
            const bool fits = IsFast<O>::value && rb.w <= kMarchBlocks;
            bool notComb = false, notLip1 = false, notLipCap = false;
            for (uint32_t i = lane; i < nView; i += 32) {
                const uint2 nd = vb.nodes[ra.z + i];
                s.hdr[i] = fits ? fast_hdr(nd.x) : nd.x;
                if (SB) {
                    notLip1 |= !node_is_one_lipschitz(nd.x);
                    notLipCap |= !node_is_lipschitz_capable(nd.x);
                }
                if (fits) {
                    convert_node(nd.x, t.words + nd.y + 1, s.blocks + ((nd.x & 0xFFFFu) >> 4));
                    // left comb: node 0 and every odd node a primitive, every even node > 0 an operator
                    const bool pr = blob_is_prim(nd.x);
                    notComb |= i == 0u ? !pr : pr != ((i & 1u) != 0u);
                    if (pr) s.rec[(i + 1u) >> 1].x = comb_rec(nd.x);
                    else s.rec[i >> 1].y = comb_rec(nd.x);
                } else {
                    s.word[i] = nd.y;
                }
            }
            const bool comb = fits && !__any_sync(kFull, notComb) && (nView & 1u);
            // step bound of this interval: the configured L, or 1 for a
            // 1-Lipschitz view when the view-local bound is enabled
            TraceParams tpi = tp;
            bool combLip = false;  // a comb whose compact operators may leave it 1-Lipschitz, step by step
            if (SB && tp.viewLipschitz) {
                if (!__any_sync(kFull, notLip1)) {
                    tpi.L = 1.0f;
                    tpi.invL = 1.0f;
                } else {
                    combLip = comb && !__any_sync(kFull, notLipCap);
                }
            }
            // queue of this interval: the tile's unfinished rays, in ray order
            const uint32_t p0 = ~found0, p1 = ~found1;
            const uint32_t c0 = __popc(p0), nPend = c0 + __popc(p1);
            if ((p0 >> lane) & 1u) s.pend[__popc(p0 & lt)] = (uint8_t)lane;
            if ((p1 >> lane) & 1u) s.pend[c0 + __popc(p1 & lt)] = (uint8_t)(lane + 32);
            __syncwarp();
            const float vz0 = view_z_from_ndc(cam, zb), vz1 = view_z_from_ndc(cam, ze);
            uint32_t ife = 0, ifl = 0, isteps = 0;
            if constexpr (IsFast<O>::value) {
                if (nView == 1u && comb)
                    march_interval<O, kClsSingle>(t, cam, tpi, s, s.rec[0].x, nView, nPend, vz0, vz1, lt, ife, ifl,
                                                  isteps, rb.z);
                else if (SB && combLip)  // (the step-bound kernel only: keeps the default kernel's code small)
                    march_interval<O, SB ? kClsCombLip : kClsComb>(t, cam, tpi, s, (nView + 1u) >> 1, nView, nPend,
                                                                   vz0, vz1, lt, ife, ifl, isteps, rb.z);
                else if (comb)
                    march_interval<O, kClsComb>(t, cam, tpi, s, (nView + 1u) >> 1, nView, nPend, vz0, vz1, lt, ife,
                                                ifl, isteps, rb.z);
                else if (fits)
                    march_interval<O, kClsGeneral>(t, cam, tpi, s, 0u, nView, nPend, vz0, vz1, lt, ife, ifl, isteps,
                                                   rb.z);
                else
                    march_interval<O, kClsRaw>(t, cam, tpi, s, 0u, nView, nPend, vz0, vz1, lt, ife, ifl, isteps, rb.z);
            } else {
                march_interval<O, kClsRaw>(t, cam, tpi, s, 0u, nView, nPend, vz0, vz1, lt, ife, ifl, isteps, rb.z);
            }
            s.accFe[lane] += ife;
            s.accFl[lane] += ifl;
            s.accRnv[lane] += ife * nView;
            s.accPe[lane] += ife * (ra.w >> 16);
            if (lane == 0) s.steps += isteps;
            __syncwarp();
        }
    }
    __syncwarp();
    uint32_t v0, v1;
    unit_rays(g, tx, ty, mine, v0, v1);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        if (!(((j ? v1 : v0) >> lane) & 1u)) continue;
        const int li = lane + 32 * j;
        const size_t p = (size_t)(ty * kTile + (li >> 3)) * g.width + tx * kTile + (li & 7);
        const bool h = s.hit[li] != 0;
        g.hit[p] = h ? 1 : 0;
        g.depth[p] = h ? s.depth[li] : 0.0f;
        g.evalCount[p] = s.evals[li];
    }
    const uint64_t sfe = warp_sum_u64(s.accFe[lane]), srnv = warp_sum_u64(s.accRnv[lane]);
    const uint64_t spe = warp_sum_u64(s.accPe[lane]), sfl = warp_sum_u64(s.accFl[lane]);
    if (lane == 0) {
        const uint32_t tileMaxOv = s.tileMaxOv, tileCache = s.tileCache;
        uint32_t tileErr = s.tileErr;
        if (!half && !g.accumulate) {
            g.tileMaxOverlap[tile] = tileMaxOv;
            g.tileCacheBytes[tile] = tileCache;
            g.tileError[tile] = (uint8_t)tileErr;
        } else if (!half) {  // a later depth slab: the tile's planes over all slabs
            g.tileMaxOverlap[tile] = max(g.tileMaxOverlap[tile], tileMaxOv);
            g.tileCacheBytes[tile] = max(g.tileCacheBytes[tile], tileCache);
            if (tileErr) g.tileError[tile] = 1;
        } else {  // both halves walk a prefix of the same intervals: the tile's values are the max
            if (tileMaxOv) atomicMax(&g.tileMaxOverlap[tile], tileMaxOv);
            if (tileCache) atomicMax(&g.tileCacheBytes[tile], tileCache);
            if (tileErr) {
                g.tileError[tile] = 1;
                if (atomicExch(&vb.tileCost[tile], 1u) != 0u) tileErr = 0;  // count the tile once
            }
        }
        if (sfe) {
            atomicAdd(&bs.fe, (unsigned long long)sfe);
            atomicAdd(&bs.rnv, (unsigned long long)srnv);
            atomicAdd(&bs.pe, (unsigned long long)spe);
            atomicAdd(&bs.fl, (unsigned long long)sfl);
        }
        if (s.steps) atomicAdd(&bs.steps, (unsigned long long)s.steps);
        if (tileErr) atomicAdd(&bs.errs, 1ull);
        if (tileMaxOv) atomicMax(&bs.maxOv, tileMaxOv);
        if (tileCache) atomicMax(&bs.maxCache, tileCache);
    }
    __syncwarp();
}

// Persistent kernel: each warp pulls tiles from a queue (tiles differ wildly
// in cost -- empty tiles exit at once).
template <class O, int MinBlocks, bool SB = false>
__global__ void __launch_bounds__(kTraceWarps * 32, MinBlocks)
    k_march(DevTree t, Cam cam, TraceParams tp, FrameBufs fb, ViewBufs vb, GBuf g, uint64_t* stats, uint32_t tile0,
            uint32_t tile1, uint32_t* tileQueue) {
    extern __shared__ __align__(16) unsigned char smemRaw[];
    __shared__ BlockStats bs;
    MarchSmem* smem = reinterpret_cast<MarchSmem*>(smemRaw);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) bs = BlockStats{0, 0, 0, 0, 0, 0, 0u, 0u};
    __syncthreads();
    MarchSmem& s = smem[wid];
    if (lane == 0) mbar_init(&s.rayBar);
    __syncwarp();
    uint32_t rayPhase = 0;
    const uint32_t nUnits = vb.order ? *vb.unitCount : tile1 - tile0;
    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(tileQueue, 1u);
        q = __shfl_sync(kFull, q, 0);
        if (q >= nUnits) break;
        const uint32_t tile = vb.order ? vb.order[q] : tile0 + q;
        march_tile<O, SB>(t, cam, tp, fb, vb, g, s, bs, lane, tile, rayPhase);
    }
    // fused gather: this rank's pixels went to another GPU's planes; make
    // them visible system-wide before the kernel ends (the completion
    // collective that orders the root's normals follows on this stream)
    if (g.remote) __threadfence_system();
    __syncthreads();
#ifdef BT_STEP_HIST
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&g_stepDone, 1u) == gridDim.x - 1) {
            printf("STEPHIST");
            for (int k = 0; k <= 32; ++k) {
                printf(" %llu", g_stepHist[k]);
                g_stepHist[k] = 0;
            }
            printf("\n");
            g_stepDone = 0;
        }
    }
#endif
    if (threadIdx.x == 0) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(stats);
        if (bs.fe) {
            atomicAdd(&st[kStFieldEvals], bs.fe);
            atomicAdd(&st[kStRetained], bs.rnv);
            atomicAdd(&st[kStPrimEvals], bs.pe);
            atomicAdd(&st[kStFlops], bs.fl);
        }
        if (bs.steps) atomicAdd(&st[kStWarpSteps], bs.steps);
        if (bs.errs) atomicAdd(&st[kStTileErrors], bs.errs);
        if (bs.maxOv) atomicMax(&st[kStMaxOverlap], (unsigned long long)bs.maxOv);
        if (bs.maxCache) atomicMax(&st[kStMaxCache], (unsigned long long)bs.maxCache);
    }
}

// ---------------------------------------------------------------- full tree

template <class O> __device__ float eval_full(const DevTree& t, F3 p) {
    float stk[kFullStackCap];
    int sp = 0;
    for (uint32_t i = 0; i < t.nnodes; ++i) {
        const uint32_t e = __ldg(&t.fullProgram[i]);
        const uint32_t w = e & kSentinel;
        const float4* P4 = t.words + w + 1;
        if (e >> 31) {
            float P[20];
            const uint32_t kind = (e >> 26) & 0x1Fu;
            load_params<5>(P, P4);
            stk[sp++] = eval_primitive<O>(kind, P, p);
        } else {
            const uint32_t code = (e >> 26) & 0x1Fu;
            float kd[2] = {0.f, 0.f};
            if (code >= 6u) {
                const float4 q = __ldg(P4);
                kd[0] = q.x;
                kd[1] = q.y;
            }
            const float right = stk[sp - 1], left = stk[sp - 2];
            stk[sp - 2] = eval_operator<O>(code, kd, left, right);
            --sp;
        }
    }
    return stk[0];
}

__device__ __forceinline__ F3 ray_dir_at(const FrameBufs& fb, const GBuf& g, int x, int y) {
    const uint32_t tile = (uint32_t)((y >> 3) * g.tilesX + (x >> 3));
    const float4 r = fb.rays[(size_t)tile * 64 + ((y & 7) << 3) + (x & 7)];
    return F3{r.x, r.y, r.z};
}

__device__ __forceinline__ F3 position_at(const Cam& cam, const FrameBufs& fb, const GBuf& g, int x, int y) {
    const F3 d = ray_dir_at(fb, g, x, y);
    return vadd<E>(cam.pos, vscale<E>(d, g.depth[(size_t)y * g.width + x]));
}

__global__ void k_normals(Cam cam, FrameBufs fb, GBuf g, int mode, uint32_t* counters, int y0, int y1) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = y0 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
    if (x >= g.width || y >= y1) return;
    const size_t p = (size_t)y * g.width + x;
    float* nout = g.normal + 3 * p;
    if (!g.hit[p]) {
        nout[0] = nout[1] = nout[2] = 0.0f;
        return;
    }
    bool ok = false;
    F3 n{0.f, 0.f, 0.f};
    if (mode == 0) {
        auto hitAt = [&](int xx, int yy) {
            return xx >= 0 && xx < g.width && yy >= 0 && yy < g.height && g.hit[(size_t)yy * g.width + xx] != 0;
        };
        const F3 pc = position_at(cam, fb, g, x, y);
        const bool l = hitAt(x - 1, y), r = hitAt(x + 1, y), u = hitAt(x, y - 1), d = hitAt(x, y + 1);
        F3 ddx{0.f, 0.f, 0.f}, ddy{0.f, 0.f, 0.f};
        bool okX = true, okY = true;
        if (l && r) ddx = vsub<E>(position_at(cam, fb, g, x + 1, y), position_at(cam, fb, g, x - 1, y));
        else if (r) ddx = vsub<E>(position_at(cam, fb, g, x + 1, y), pc);
        else if (l) ddx = vsub<E>(pc, position_at(cam, fb, g, x - 1, y));
        else okX = false;
        if (u && d) ddy = vsub<E>(position_at(cam, fb, g, x, y + 1), position_at(cam, fb, g, x, y - 1));
        else if (d) ddy = vsub<E>(position_at(cam, fb, g, x, y + 1), pc);
        else if (u) ddy = vsub<E>(pc, position_at(cam, fb, g, x, y - 1));
        else okY = false;
        if (okX && okY) {
            n = vcross<E>(ddx, ddy);
            const float len = vlen<E>(n);
            if (len > 1e-12f) {
                n = vdivs<E>(n, len);
                if (vdot<E>(n, ray_dir_at(fb, g, x, y)) > 0.0f) n = vneg(n);
                ok = true;
            }
        }
    }
    if (ok) {
        nout[0] = n.x;
        nout[1] = n.y;
        nout[2] = n.z;
    } else {
        const uint32_t slot = atomicAdd(&counters[kCntFallback], 1u);
        g.fallback[slot] = (uint32_t)p;
    }
}

// gradient_normal (tracer.cpp:285-294): eval_full (traversal.cpp:126-141) at
// p +- h e_axis, h = max(1e-3, 1e-4 t).  One CTA per queued pixel:
//   phase 1  every (frontier subtree, tap) pair is evaluated by one thread
//            (post-order over <= 32 nodes) -- independent work;
//   phase 2  six threads run the upper operator program over those values;
//            a left comb of sharp unions is a (value, index) min-reduction
//            (one warp per tap), exact because std::min keeps the earliest.
// Each node still combines exactly the same operands in the same order as
// the reference's serial walk, so the exact variant stays bit-identical.
// One frontier subtree at the 6 gradient taps: parameters are loaded once per
// node and the 6 evaluations are independent (ILP).
template <class O>
__device__ __forceinline__ void eval_subtree6(const DevTree& t, uint2 range, const F3* taps, float* out) {
    float stk[6][kFrontierMax / 2 + 1];
    int sp = 0;
    for (uint32_t j = range.x; j <= range.y; ++j) {
        const uint32_t e = __ldg(&t.fullProgram[j]);
        const uint32_t code = (e >> 26) & 0x1Fu;
        const float4* P4 = t.words + (e & kSentinel) + 1;
        if (e >> 31) {
            float P[20];
            load_params<5>(P, P4);
#pragma unroll
            for (int k = 0; k < 6; ++k) stk[k][sp] = eval_primitive<O>(code, P, taps[k]);
            ++sp;
        } else {
            float kd[2] = {0.f, 0.f};
            if (code >= 6u) {
                const float4 q = __ldg(P4);
                kd[0] = q.x;
                kd[1] = q.y;
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) stk[k][sp - 2] = eval_operator<O>(code, kd, stk[k][sp - 2], stk[k][sp - 1]);
            --sp;
        }
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = stk[k][0];
}

template <class O>
__global__ void __launch_bounds__(1024) k_gradient(DevTree t, Cam cam, FrameBufs fb, GBuf g,
                                                  const uint32_t* counters, uint64_t* stats, float* scratch,
                                                  uint32_t useSmem, uint32_t hardList) {
    extern __shared__ float dyn[];
    __shared__ float res[6];
    // main list: fallback[0, n); the fast path's hard list: fallback[px - 1 - i]
    const uint32_t n = counters[hardList ? kCntFallbackHard : kCntFallback];
    const uint32_t px = (uint32_t)g.width * (uint32_t)g.height;
    if (threadIdx.x == 0 && blockIdx.x == 0 && !hardList)
        atomicAdd((unsigned long long*)&stats[kStFallbacks], (unsigned long long)n);
    float* vals = useSmem ? dyn : scratch + (size_t)blockIdx.x * t.nFrontier * 6;
    // the serial upper program is staged once into shared memory (its loads
    // would otherwise sit on the dependent chain of phase 2)
    const uint32_t* upper = t.upperProgram;
    if (useSmem && n > blockIdx.x) {
        uint32_t* su = reinterpret_cast<uint32_t*>(dyn + t.nFrontier * 6);
        for (uint32_t j = threadIdx.x; j < t.nUpper; j += blockDim.x) su[j] = __ldg(&t.upperProgram[j]);
        upper = su;
        __syncthreads();
    }
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        const uint32_t p = g.fallback[hardList ? px - 1u - i : i];
        const int x = (int)(p % (uint32_t)g.width), y = (int)(p / (uint32_t)g.width);
        const F3 pc = position_at(cam, fb, g, x, y);
        const float h = smax(1e-3f, E::mul(1e-4f, g.depth[p]));
        const F3 taps[6] = {{E::add(pc.x, h), pc.y, pc.z}, {E::sub(pc.x, h), pc.y, pc.z},
                            {pc.x, E::add(pc.y, h), pc.z}, {pc.x, E::sub(pc.y, h), pc.z},
                            {pc.x, pc.y, E::add(pc.z, h)}, {pc.x, pc.y, E::sub(pc.z, h)}};
        for (uint32_t f = threadIdx.x; f < t.nFrontier; f += blockDim.x) {
            float v6[6];
            eval_subtree6<O>(t, __ldg(&t.frontier[f]), taps, v6);
#pragma unroll
            for (int k = 0; k < 6; ++k) vals[f * 6u + k] = v6[k];
        }
        __syncthreads();
        if (t.upperIsMinChain) {
            // min over the chain's values in order (csg union == std::min, the
            // earliest minimum wins): exact as a (value, index) reduction --
            // warp w reduces tap w.
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
            if (w < 6) {
                const uint32_t m = (t.nUpper + 1) / 2;  // values in the chain
                float best = f_inf();
                uint32_t bestIdx = 0xFFFFFFFFu;
                for (uint32_t q = lane; q < m; q += 32) {
                    const float v = vals[(upper[q == 0 ? 0 : 2 * q - 1] & 0x7FFFFFFFu) * 6u + w];
                    if (!(v != v) && (bestIdx == 0xFFFFFFFFu || v < best)) {  // NaN never wins b < a
                        best = v;
                        bestIdx = q;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(kFull, best, o);
                    const uint32_t oi = __shfl_xor_sync(kFull, bestIdx, o);
                    const bool take = oi != 0xFFFFFFFFu &&
                                      (bestIdx == 0xFFFFFFFFu || ov < best || (!(best < ov) && oi < bestIdx));
                    if (take) {
                        best = ov;
                        bestIdx = oi;
                    }
                }
                if (lane == 0) {  // ... unless it is the accumulator's first value
                    const float v0 = vals[(upper[0] & 0x7FFFFFFFu) * 6u + w];
                    res[w] = (v0 != v0) ? v0 : best;
                }
            }
        } else if (threadIdx.x < 6 && t.upperIsChain) {
            // left comb: acc = F0; acc = op(acc, Fi) -- same operand order as the
            // post-order walk, no stack traffic on the serial dependency chain
            float acc = vals[(upper[0] & 0x7FFFFFFFu) * 6u + threadIdx.x];
            for (uint32_t j = 1; j < t.nUpper; j += 2) {
                const float right = vals[(upper[j] & 0x7FFFFFFFu) * 6u + threadIdx.x];
                const uint32_t e = upper[j + 1];
                const uint32_t code = (e >> 26) & 0x1Fu;
                float kd[2] = {0.f, 0.f};
                if (code >= 6u) {
                    const float4 q = __ldg(t.words + (e & kSentinel) + 1);
                    kd[0] = q.x;
                    kd[1] = q.y;
                }
                acc = eval_operator<O>(code, kd, acc, right);
            }
            res[threadIdx.x] = acc;
        } else if (threadIdx.x < 6) {
            float stk[kFullStackCap];
            int sp = 0;
            for (uint32_t j = 0; j < t.nUpper; ++j) {
                const uint32_t e = upper[j];
                if (e >> 31) {
                    stk[sp++] = vals[(e & 0x7FFFFFFFu) * 6u + threadIdx.x];
                } else {
                    const uint32_t code = (e >> 26) & 0x1Fu;
                    float kd[2] = {0.f, 0.f};
                    if (code >= 6u) {
                        const float4 q = __ldg(t.words + (e & kSentinel) + 1);
                        kd[0] = q.x;
                        kd[1] = q.y;
                    }
                    const float right = stk[sp - 1], left = stk[sp - 2];
                    stk[sp - 2] = eval_operator<O>(code, kd, left, right);
                    --sp;
                }
            }
            res[threadIdx.x] = stk[0];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const F3 dv{E::sub(res[0], res[1]), E::sub(res[2], res[3]), E::sub(res[4], res[5])};
            const F3 nn = vnormalize<E>(dv);
            g.normal[3 * p + 0] = nn.x;
            g.normal[3 * p + 1] = nn.y;
            g.normal[3 * p + 2] = nn.z;
        }
        __syncthreads();
    }
}

// Tolerance path of the gradient fallback: eval_full is replaced by the
// pruned view of the interval the ray hit in (the march's own records), one
// warp per pixel, lanes 0..5 one tap each.  Near the hit every primitive
// whose volume of interest reaches the point is in that view, so the field
// agrees with eval_full there to ~1 ulp (the reference's own pruned-vs-full
// bound, test_traversal.cpp:132-152) -- at the cost of one small view per
// tap instead of the whole tree.  Pixels without a usable interval go to the
// hard list (full tree).
constexpr int kGradViewWarps = 4;
__global__ void __launch_bounds__(kGradViewWarps * 32) k_gradient_view(DevTree t, Cam cam, FrameBufs fb, ViewBufs vb,
                                                                        GBuf g, uint32_t* counters, uint64_t* stats) {
    __shared__ uint32_t sh[kGradViewWarps][kViewCap], sw[kGradViewWarps][kViewCap];
    __shared__ float4 blk[kGradViewWarps][kMarchBlocks];  // fast parameter blocks, as in k_march
    __shared__ float res[kGradViewWarps][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t n = counters[kCntFallback];
    const uint32_t px = (uint32_t)g.width * (uint32_t)g.height;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        atomicAdd((unsigned long long*)&stats[kStFallbacks], (unsigned long long)n);
    const uint32_t nwarps = gridDim.x * kGradViewWarps;
    for (uint32_t i = blockIdx.x * kGradViewWarps + w; i < n; i += nwarps) {
        const uint32_t p = g.fallback[i];
        const int x = (int)(p % (uint32_t)g.width), y = (int)(p / (uint32_t)g.width);
        const uint32_t tile = (uint32_t)((y >> 3) * g.tilesX + (x >> 3));
        const float4 r = fb.rays[(size_t)tile * 64 + ((y & 7) << 3) + (x & 7)];
        const float depth = g.depth[p];
        const float z = ndc_from_view_z(cam, E::mul(depth, r.w));
        // the first usable interval containing the hit, else the last one starting before it
        const uint32_t cnt = vb.counters[1] ? 0u : vb.count[tile].x;
        const uint2 o = cnt ? view_offset(vb, tile) : make_uint2(0u, 0u);
        int first = -1, last = -1;
        for (uint32_t k0 = 0; k0 < cnt; k0 += 32) {
            const uint32_t k = k0 + lane;
            bool c1 = false, c2 = false;
            if (k < cnt) {
                const IntervalRec rec = vb.iv[o.x + k];
                const uint32_t fl = rec.actFlags >> 8;
                const bool ok = (fl & kIvRootUsed) && !(fl & (kIvErr | kIvDepthErr));
                c2 = ok && rec.zBegin <= z;
                c1 = c2 && z <= rec.zEnd;
            }
            const uint32_t m1 = __ballot_sync(kFull, c1), m2 = __ballot_sync(kFull, c2);
            if (m1 && first < 0) first = (int)k0 + __ffs(m1) - 1;
            if (m2) last = (int)k0 + 31 - __clz(m2);
        }
        const int sel = first >= 0 ? first : last;
        if (sel < 0) {  // no view: full tree (k_gradient, hard list)
            if (lane == 0) g.fallback[px - 1u - atomicAdd(&counters[kCntFallbackHard], 1u)] = p;
            continue;
        }
        const IntervalRec rec = vb.iv[o.x + (uint32_t)sel];
        const uint32_t nView = rec.viewPrim & 0xFFFFu;
        // the view's parameter blocks are converted lane-parallel (one round of
        // loads) instead of read node by node inside the evaluation
        const bool fits = rec.nBlocks <= kMarchBlocks;
        for (uint32_t j = lane; j < nView; j += 32) {
            const uint2 nd = vb.nodes[rec.nodeOff + j];
            sh[w][j] = fits ? fast_hdr(nd.x) : nd.x;
            sw[w][j] = nd.y;
            if (fits) convert_node(nd.x, t.words + nd.y + 1, blk[w] + ((nd.x & 0xFFFFu) >> 4));
        }
        __syncwarp();
        const F3 pc = vadd<E>(cam.pos, vscale<E>(F3{r.x, r.y, r.z}, depth));
        const float h = smax(1e-3f, E::mul(1e-4f, depth));
        {  // lanes 0-5 evaluate the six taps; the whole warp runs the evaluator
           // (its header reads are warp-uniform reductions: every lane must call)
            F3 tap = pc;
            const float s = (lane & 1) ? -h : h;
            if (lane < 2) tap.x = E::add(pc.x, s);
            else if (lane < 4) tap.y = E::add(pc.y, s);
            else if (lane < 6) tap.z = E::add(pc.z, s);
            float v;
            if (fits) eval_view_fast<1>(sh[w], nView, blk[w], &tap, &v);
            else v = eval_staged<FastOps>(sh[w], sw[w], nView, t.words, tap);
            if (lane < 6) res[w][lane] = v;
        }
        __syncwarp();
        if (lane == 0) {
            const F3 dv{E::sub(res[w][0], res[w][1]), E::sub(res[w][2], res[w][3]), E::sub(res[w][4], res[w][5])};
            const F3 nn = vnormalize<E>(dv);
            g.normal[3 * p + 0] = nn.x;
            g.normal[3 * p + 1] = nn.y;
            g.normal[3 * p + 2] = nn.z;
        }
        __syncwarp();
    }
}

// oracle_render: one thread per pixel over [near, far], full tree.
template <class O>
__global__ void k_oracle(DevTree t, Cam cam, TraceParams tp, FrameBufs fb, GBuf g, uint64_t* stats) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    uint64_t fe = 0;
    if (x < g.width && y < g.height) {
        const size_t p = (size_t)y * g.width + x;
        const uint32_t tile = (uint32_t)((y >> 3) * g.tilesX + (x >> 3));
        const float4 r = fb.rays[(size_t)tile * 64 + ((y & 7) << 3) + (x & 7)];
        const F3 d{r.x, r.y, r.z};
        March m;
        march_begin(m, E::div(cam.nearZ, r.w), E::div(cam.farZ, r.w));
        while (march_phase(m) != 0u) {
            const float v = eval_full<O>(t, ray_point<O>(cam.pos, d, m.evalT));
            march_consume(m, v, tp);
        }
        g.hit[p] = march_hit(m) ? 1 : 0;
        g.depth[p] = march_hit(m) ? m.t : 0.0f;
        g.evalCount[p] = m.evals;
        fe = m.evals;
    }
    // warp-aggregate the counters
    const uint64_t s = warp_sum_u64(fe);
    if ((threadIdx.x + threadIdx.y * blockDim.x) % 32 == 0 && s) {
        atomicAdd((unsigned long long*)&stats[kStFieldEvals], (unsigned long long)s);
        atomicAdd((unsigned long long*)&stats[kStRetained], (unsigned long long)(s * t.nnodes));
        atomicAdd((unsigned long long*)&stats[kStPrimEvals], (unsigned long long)(s * t.nprims));
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers

// Register budget of the FMA-path kernel (blocks of 4 warps per SM the
// compiler must fit): a compile-time variant selected once per process
// ($BT_TRACE_MINBLOCKS, default kDefaultMinBlocks) so the budget can be swept
// on the device without rebuilding.
constexpr int kDefaultMinBlocks = 6;  // measured best of {4,5,6,8} on C3 (C1, C2 agree; C5 prefers 5 by 2 %)

template <int MB> struct TraceVariant {
    static void* fn(bool exact) {
        return exact ? (void*)k_march<ExactOps, MB> : (void*)k_march<FastOps, MB>;
    }
};

int trace_min_blocks() {
    static int mb = 0;
    if (mb == 0) {
        mb = kDefaultMinBlocks;
        if (const char* e = getenv("BT_TRACE_MINBLOCKS")) {
            const int v = atoi(e);
            if (v >= 4 && v <= 8) mb = v;
        }
    }
    return mb;
}

void* trace_fn(bool exact, bool stepBound = false) {
    // the view-local step bound (bt_set_step_bound(1), FMA path) is its own
    // kernel, at the default register budget
    if (stepBound && !exact) return (void*)k_march<FastOps, kDefaultMinBlocks, true>;
    switch (trace_min_blocks()) {
        case 4: return TraceVariant<4>::fn(exact);
        case 5: return TraceVariant<5>::fn(exact);
        case 6: return TraceVariant<6>::fn(exact);
        case 7: return TraceVariant<7>::fn(exact);
        default: return TraceVariant<8>::fn(exact);
    }
}

// Function attributes and occupancy are per device: cached per device index
// (the C-ABI makes the context's device current before any launch).
constexpr int kMaxDevices = 64;
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 || d >= kMaxDevices ? 0 : d;
}

uint32_t trace_grid_blocks(int smCount) {
    static int perSMDev[kMaxDevices] = {};
    int& perSM = perSMDev[current_device()];
    if (perSM == 0) {
        const size_t smem = sizeof(MarchSmem) * kTraceWarps;
        int best = 1;
        for (int v = 0; v < 3; ++v) {
            const void* f = trace_fn(v == 1, v == 2);
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int a = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, f, kTraceWarps * 32, smem);
            if (v < 2) best = std::max(best, a);
        }
        perSM = best;
    }
    return (uint32_t)(perSM * smCount);
}

uint32_t trace_grid_warps(int smCount) { return trace_grid_blocks(smCount) * kTraceWarps; }

void launch_trace(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam, const TraceParams& tp,
                  const FrameBufs& fb, const ViewBufs& vb, const GBuf& g, uint64_t* stats, uint32_t tile0,
                  uint32_t tile1, int smCount, uint32_t* tileQueue, bool zero) {
    if (tile1 <= tile0) return;
    const size_t smem = sizeof(MarchSmem) * kTraceWarps;
    const uint32_t blocks =
        std::min<uint32_t>(trace_grid_blocks(smCount), (tile1 - tile0 + kTraceWarps - 1) / kTraceWarps);
    if (zero) cudaMemsetAsync(tileQueue, 0, sizeof(uint32_t), st);
    void* args[] = {(void*)&t,    (void*)&cam,   (void*)&tp,    (void*)&fb,          (void*)&vb,       (void*)&g,
                    (void*)&stats, (void*)&tile0, (void*)&tile1, (void*)&tileQueue};
    cudaLaunchKernel(trace_fn(exact, tp.viewLipschitz != 0), dim3(blocks), dim3(kTraceWarps * 32), args, smem, st);
}

void launch_normals(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam,
                    const FrameBufs& fb, const GBuf& g, int mode, uint32_t* counters,
                    uint64_t* stats, int smCount, float* scratch, uint32_t scratchWarps,
                    const ViewBufs* vb, bool zero, int y0, int y1) {
    if (zero) {
        cudaMemsetAsync(counters + kCntFallback, 0, sizeof(uint32_t), st);
        cudaMemsetAsync(counters + kCntFallbackHard, 0, sizeof(uint32_t), st);
    }
    if (y1 < 0 || y1 > g.height) y1 = g.height;
    if (y0 < 0) y0 = 0;
    if (y1 <= y0) return;
    dim3 block(16, 16), grid((g.width + 15) / 16, (y1 - y0 + 15) / 16);
    k_normals<<<grid, block, 0, st>>>(cam, fb, g, mode, counters, y0, y1);
    const size_t bytes = (size_t)t.nFrontier * 6 * sizeof(float) + (size_t)t.nUpper * sizeof(uint32_t);
    const uint32_t useSmem = bytes <= kGradSmemBytes ? 1u : 0u;
    const size_t smem = useSmem ? bytes : 0;
    static bool attrDev[kMaxDevices] = {};
    bool& attr = attrDev[current_device()];
    if (!attr) {
        cudaFuncSetAttribute(k_gradient<ExactOps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmemBytes);
        cudaFuncSetAttribute(k_gradient<FastOps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmemBytes);
        attr = true;
    }
    // one CTA per queued pixel: as many threads as frontier subtrees (phase 1
    // is one subtree per thread), at least 6 warps for the min-chain phase
    const uint32_t threads = std::min<uint32_t>(1024u, std::max<uint32_t>(256u, (t.nFrontier + 31u) & ~31u));
    if (exact) {
        k_gradient<ExactOps><<<scratchWarps, threads, smem, st>>>(t, cam, fb, g, counters, stats, scratch, useSmem, 0u);
    } else if (vb) {
        k_gradient_view<<<smCount * 2, kGradViewWarps * 32, 0, st>>>(t, cam, fb, *vb, g, counters, stats);
        k_gradient<FastOps><<<scratchWarps, threads, smem, st>>>(t, cam, fb, g, counters, stats, scratch, useSmem, 1u);
    } else {
        k_gradient<FastOps><<<scratchWarps, threads, smem, st>>>(t, cam, fb, g, counters, stats, scratch, useSmem, 0u);
    }
}

void launch_oracle(cudaStream_t st, bool exact, const DevTree& t, const Cam& cam,
                   const TraceParams& tp, const FrameBufs& fb, const GBuf& g, uint64_t* stats) {
    dim3 block(16, 8), grid((g.width + 15) / 16, (g.height + 7) / 8);
    if (exact)
        k_oracle<ExactOps><<<grid, block, 0, st>>>(t, cam, tp, fb, g, stats);
    else
        k_oracle<FastOps><<<grid, block, 0, st>>>(t, cam, tp, fb, g, stats);
}

}  // namespace btk
