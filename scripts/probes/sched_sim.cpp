// sched_sim.cpp -- lockstep-step counts of march schedules, from the
// UNMODIFIED reference's render loop (tracer.cpp:141-236) replayed on one
// thread with per-(interval, ray) evaluation counts.  Compares:
//   tile     one warp walks a tile's intervals, 32 lanes over a FIFO ray queue
//            (what k_march does);
//   lpt      the same with each interval's rays ordered longest first (an
//            upper bound: it needs the costs before marching);
//   pair     horizontally adjacent tiles (2i, 2i+1) walked by one warp; an
//            interval of each whose pruned views are identical (same active
//            words) is marched as ONE queue of both tiles' pending rays.
//   make -C oracle ref && g++ -std=c++20 -O2 -Dblobtree=blobtree_ref -I/root/reference/proj/include \
//     -I<json> scripts/probes/sched_sim.cpp paper_2304_09673_b200/csrc/scenes/scenes.cpp \
//     oracle/_ref/libblobtree_ref.a -o /tmp/sched_sim && /tmp/sched_sim C3
#include <algorithm>
#include <cstdio>
#include <queue>
#include <string>
#include <vector>

#include "blobtree/abuffer.hpp"
#include "blobtree/tracer.hpp"
#include "blobtree/traversal.hpp"
#include "../../paper_2304_09673_b200/csrc/scenes/scenes.hpp"

using namespace blobtree;

struct Iv {
    std::vector<uint32_t> key;   // active words (the view is a function of them)
    std::vector<uint32_t> cost;  // evals of each ray marched in this interval (ray order)
    std::vector<uint32_t> pred;  // predictor: active volumes the ray's interval segment intersects
    std::vector<uint32_t> ray;   // ray index (in the tile) of each cost entry
};

// queue order by a per-ray key, longest first; `buckets` > 0: only the class
// of the key relative to the tile's maximum (>= max/2, >= max/4, ...) counts
static uint64_t makespan_key(const Iv& iv, const std::vector<uint32_t>& key, int buckets) {
    std::vector<size_t> idx(iv.cost.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    uint32_t mx = 1;
    for (uint32_t k : key) mx = std::max(mx, k);
    auto cls = [&](size_t i) -> int64_t {
        const uint32_t k = key[iv.ray[i]];
        if (buckets <= 0) return k;
        int c = 0;
        for (int b = 1; b < buckets; ++b)
            if ((uint64_t)k << b >= mx) { c = buckets - b; break; }
        return c;
    };
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return cls(a) > cls(b); });
    std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> h;
    for (int i = 0; i < 32; ++i) h.push(0);
    uint64_t m = 0;
    for (size_t i : idx) {
        uint64_t t = h.top();
        h.pop();
        t += std::max<uint32_t>(iv.cost[i], 1u);
        m = std::max(m, t);
        h.push(t);
    }
    return m;
}

static uint64_t makespan_pred(const Iv& iv) {
    std::vector<size_t> idx(iv.cost.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return iv.pred[a] > iv.pred[b]; });
    std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> h;
    for (int i = 0; i < 32; ++i) h.push(0);
    uint64_t m = 0;
    for (size_t i : idx) {
        uint64_t t = h.top();
        h.pop();
        t += std::max<uint32_t>(iv.cost[i], 1u);
        m = std::max(m, t);
        h.push(t);
    }
    return m;
}

static uint64_t makespan(std::vector<uint32_t> c, bool lpt) {
    if (c.empty()) return 0;
    if (lpt) std::sort(c.rbegin(), c.rend());
    std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> h;
    for (int i = 0; i < 32; ++i) h.push(0);
    uint64_t m = 0;
    for (uint32_t x : c) {
        uint64_t t = h.top();
        h.pop();
        // a ray with 0 evals (empty interval) still takes its lane for a step in k_march
        t += std::max<uint32_t>(x, 1u);
        m = std::max(m, t);
        h.push(t);
    }
    return m;
}

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "C3";
    auto sc = scenes::build(name, 0, 0, 0);
    const LinearTree& tree = sc->tree;
    RenderConfig cfg;
    CameraFrame frame(sc->camera);
    auto roi = propagate_roi(tree);
    auto vois = build_volumes_of_interest(tree, roi, cfg.hitEpsilon);
    TileABuffer ab = rasterize_volumes(vois, frame);
    const int tilesX = frame.tiles_x(), tilesY = frame.tiles_y();
    std::vector<std::vector<Iv>> tiles(tilesX * tilesY);
    uint64_t evalsTotal = 0;
    for (int ty = 0; ty < tilesY; ++ty)
        for (int tx = 0; tx < tilesX; ++tx) {
            const auto& frags = ab.at(tx, ty);
            if (frags.empty()) continue;
            std::vector<Ray> rays;
            std::vector<char> found;
            for (int y = ty * 8; y < std::min((ty + 1) * 8, sc->camera.height); ++y)
                for (int x = tx * 8; x < std::min((tx + 1) * 8, sc->camera.width); ++x) {
                    rays.push_back(frame.pixel_ray(x, y));
                    found.push_back(0);
                }
            int remaining = (int)rays.size();
            TileFetchState fetch;
            fetch.list = frags;
            try {
                while (remaining > 0) {
                    auto iv = fetch_interval(fetch, frame, cfg);
                    if (!iv) break;
                    std::vector<uint32_t> act;
                    for (const auto& a : fetch.actives) act.push_back(a.word);
                    PrunedView view = build_pruned_view(tree, act);
                    if (!view.rootUsed || iv->zEnd <= iv->zBegin) continue;
                    const float vz0 = frame.view_z_from_ndc(iv->zBegin), vz1 = frame.view_z_from_ndc(iv->zEnd);
                    Iv rec;
                    rec.key = act;
                    for (size_t i = 0; i < rays.size(); ++i) {
                        if (found[i]) continue;
                        const Ray& ray = rays[i];
                        uint32_t evals = 0;
                        auto fieldAt = [&](float t) { return eval_pruned(view, ray.origin + ray.dir * t); };
                        TraceResult res =
                            sphere_trace_interval(fieldAt, ray.t_from_view_z(vz0), ray.t_from_view_z(vz1), cfg, evals);
                        rec.cost.push_back(evals);
                        rec.ray.push_back((uint32_t)i);
                        uint32_t np = 0;
                        const float ta = ray.t_from_view_z(vz0), tb = ray.t_from_view_z(vz1);
                        for (const auto& a : fetch.actives) {
                            for (const auto& v : vois)
                                if (v.primitiveWord == a.word) {
                                    auto r = ray_volume_intersect(ray, v);
                                    if (r && r->second >= ta && r->first <= tb) ++np;
                                    break;
                                }
                        }
                        rec.pred.push_back(np);
                        evalsTotal += evals;
                        if (res.hit) {
                            found[i] = 1;
                            --remaining;
                        }
                    }
                    tiles[ty * tilesX + tx].push_back(std::move(rec));
                }
            } catch (...) {
            }
        }
    uint64_t sTile = 0, sLpt = 0, sPair = 0, ivs = 0, merged = 0, sPred = 0, sTot = 0, sB2 = 0, sB4 = 0, sSoFar = 0;
    for (auto& t : tiles) {
        std::vector<uint32_t> tot(64, 0);
        for (auto& iv : t)
            for (size_t i = 0; i < iv.cost.size(); ++i) tot[iv.ray[i]] += iv.cost[i];
        std::vector<uint32_t> sofar(64, 0);
        for (auto& iv : t) {
            sSoFar += makespan_key(iv, sofar, 0);
            for (size_t i = 0; i < iv.cost.size(); ++i) sofar[iv.ray[i]] += iv.cost[i];
        }
        for (auto& iv : t) {
            sTot += makespan_key(iv, tot, 0);
            sB2 += makespan_key(iv, tot, 2);
            sB4 += makespan_key(iv, tot, 4);
        }
    }
    for (auto& t : tiles)
        for (auto& iv : t) {
            sPred += makespan_pred(iv);
            sTile += makespan(iv.cost, false);
            sLpt += makespan(iv.cost, true);
            ++ivs;
        }
    // pairs: greedy walk -- merge the heads when their keys match, else march
    // the head with fewer... (the one of the tile with more intervals left)
    for (int ty = 0; ty < tilesY; ++ty)
        for (int tx = 0; tx < tilesX; tx += 2) {
            auto& A = tiles[ty * tilesX + tx];
            static std::vector<Iv> empty;
            auto& B = tx + 1 < tilesX ? tiles[ty * tilesX + tx + 1] : empty;
            size_t a = 0, b = 0;
            while (a < A.size() || b < B.size()) {
                if (a < A.size() && b < B.size() && A[a].key == B[b].key) {
                    std::vector<uint32_t> c = A[a].cost;
                    c.insert(c.end(), B[b].cost.begin(), B[b].cost.end());
                    sPair += makespan(c, false);
                    ++merged;
                    ++a;
                    ++b;
                } else if (a < A.size() && (b >= B.size() || A.size() - a >= B.size() - b)) {
                    // look ahead: if B's head matches A's next, march A's head alone
                    sPair += makespan(A[a].cost, false);
                    ++a;
                } else {
                    sPair += makespan(B[b].cost, false);
                    ++b;
                }
            }
        }
    // runs of R horizontally adjacent tiles walked by one warp in waves: wave
    // k marches interval k of every tile of the run (the ones still having
    // one); consecutive items of a wave with identical views share one queue
    for (int R : {2, 4, 8, 16}) {
        uint64_t steps = 0, items = 0, groups = 0;
        for (int ty = 0; ty < tilesY; ++ty)
            for (int tx0 = 0; tx0 < tilesX; tx0 += R) {
                const int tx1 = std::min(tilesX, tx0 + R);
                size_t maxK = 0;
                for (int tx = tx0; tx < tx1; ++tx) maxK = std::max(maxK, tiles[ty * tilesX + tx].size());
                for (size_t k = 0; k < maxK; ++k) {
                    std::vector<uint32_t> q;
                    const std::vector<uint32_t>* key = nullptr;
                    for (int tx = tx0; tx < tx1; ++tx) {
                        auto& T = tiles[ty * tilesX + tx];
                        if (k >= T.size()) continue;
                        ++items;
                        if (key && *key == T[k].key) {
                            q.insert(q.end(), T[k].cost.begin(), T[k].cost.end());
                        } else {
                            steps += makespan(q, false);
                            if (!q.empty()) ++groups;
                            q = T[k].cost;
                            key = &T[k].key;
                        }
                    }
                    steps += makespan(q, false);
                    if (!q.empty()) ++groups;
                }
            }
        std::printf("  run%-2d %llu steps (util %.3f), %llu items in %llu queues\n", R, (unsigned long long)steps,
                    evalsTotal / (32.0 * steps), (unsigned long long)items, (unsigned long long)groups);
    }
    {  // pairs, only the first intervals merged
        uint64_t steps = 0, merged1 = 0;
        for (int ty = 0; ty < tilesY; ++ty)
            for (int tx = 0; tx < tilesX; tx += 2) {
                auto& A = tiles[ty * tilesX + tx];
                static std::vector<Iv> none;
                auto& B = tx + 1 < tilesX ? tiles[ty * tilesX + tx + 1] : none;
                size_t a = 0, b = 0;
                if (!A.empty() && !B.empty() && A[0].key == B[0].key) {
                    std::vector<uint32_t> q = A[0].cost;
                    q.insert(q.end(), B[0].cost.begin(), B[0].cost.end());
                    steps += makespan(q, false);
                    a = b = 1;
                    ++merged1;
                }
                for (; a < A.size(); ++a) steps += makespan(A[a].cost, false);
                for (; b < B.size(); ++b) steps += makespan(B[b].cost, false);
            }
        std::printf("  pair-first %llu steps (util %.3f), %llu merged\n", (unsigned long long)steps,
                    evalsTotal / (32.0 * steps), (unsigned long long)merged1);
    }
    std::printf("%s: evals %llu  intervals %llu  ideal steps %llu\n", name.c_str(), (unsigned long long)evalsTotal,
                (unsigned long long)ivs, (unsigned long long)((evalsTotal + 31) / 32));
    std::printf("  tile  %llu steps (util %.3f)\n", (unsigned long long)sTile, evalsTotal / (32.0 * sTile));
    std::printf("  lpt   %llu steps (util %.3f)\n", (unsigned long long)sLpt, evalsTotal / (32.0 * sLpt));
    std::printf("  total-key lpt %llu  2-class %llu  4-class %llu\n", (unsigned long long)sTot, (unsigned long long)sB2,
                (unsigned long long)sB4);
    std::printf("  so-far-key lpt %llu\n", (unsigned long long)sSoFar);
    std::printf("  pred  %llu steps (util %.3f)\n", (unsigned long long)sPred, evalsTotal / (32.0 * sPred));
    std::printf("  pair  %llu steps (util %.3f), %llu merged interval pairs\n", (unsigned long long)sPair,
                evalsTotal / (32.0 * sPair), (unsigned long long)merged);
}
