// bigtile_sim.cpp -- what larger march tiles would cost (PAPER.md:1204,
// "using larger tiles"), from the UNMODIFIED reference's render loop: the
// 8x8 A-buffer of rasterize_volumes is merged into GX x GY groups of tiles
// (a volume's fragment over the group spans its fragments' entry min / exit
// max), and tracer.cpp's per-tile loop (fetch_interval, pruned view, sphere
// trace) runs over each group's merged list and all of its rays.  Reports
// field evaluations, evaluation work (evaluations x view nodes), interval
// count and the lockstep steps of 32 lanes over a FIFO ray queue per
// interval -- against the 8x8 pass.
//   make -C oracle ref && g++ -std=c++20 -O2 -Dblobtree=blobtree_ref -I/root/reference/proj/include \
//     -I<json> scripts/probes/bigtile_sim.cpp paper_2304_09673_b200/csrc/scenes/scenes.cpp \
//     oracle/_ref/libblobtree_ref.a -o /tmp/bigtile_sim && /tmp/bigtile_sim C3 2 1
#include <algorithm>
#include <cstdio>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "blobtree/abuffer.hpp"
#include "blobtree/tracer.hpp"
#include "blobtree/traversal.hpp"
#include "../../paper_2304_09673_b200/csrc/scenes/scenes.hpp"

using namespace blobtree;

static uint64_t makespan(const std::vector<uint32_t>& c) {
    if (c.empty()) return 0;
    std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> h;
    for (int i = 0; i < 32; ++i) h.push(0);
    uint64_t m = 0;
    for (uint32_t x : c) {
        uint64_t t = h.top();
        h.pop();
        t += std::max<uint32_t>(x, 1u);
        m = std::max(m, t);
        h.push(t);
    }
    return m;
}

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "C3";
    const int GX = argc > 2 ? std::atoi(argv[2]) : 2, GY = argc > 3 ? std::atoi(argv[3]) : 1;
    auto sc = scenes::build(name, 0, 0, 0);
    const LinearTree& tree = sc->tree;
    RenderConfig cfg;
    CameraFrame frame(sc->camera);
    auto roi = propagate_roi(tree);
    auto vois = build_volumes_of_interest(tree, roi, cfg.hitEpsilon);
    TileABuffer ab = rasterize_volumes(vois, frame);
    const int tilesX = frame.tiles_x(), tilesY = frame.tiles_y();
    uint64_t evals = 0, work = 0, steps = 0, intervals = 0, hits = 0, groups = 0;
    for (int gy = 0; gy < tilesY; gy += GY)
        for (int gx = 0; gx < tilesX; gx += GX) {
            std::map<uint32_t, Fragment> merged;
            for (int ty = gy; ty < std::min(tilesY, gy + GY); ++ty)
                for (int tx = gx; tx < std::min(tilesX, gx + GX); ++tx)
                    for (const Fragment& f : ab.at(tx, ty)) {
                        auto it = merged.find(f.primitiveWord);
                        if (it == merged.end()) merged[f.primitiveWord] = f;
                        else {
                            it->second.zEntry = std::min(it->second.zEntry, f.zEntry);
                            it->second.zExit = std::max(it->second.zExit, f.zExit);
                        }
                    }
            if (merged.empty()) continue;
            std::vector<Fragment> list;
            for (auto& [w, f] : merged) list.push_back(f);
            std::stable_sort(list.begin(), list.end(), [](const Fragment& a, const Fragment& b) {
                return a.zEntry < b.zEntry || (a.zEntry == b.zEntry && a.primitiveWord < b.primitiveWord);
            });
            std::vector<Ray> rays;
            std::vector<char> found;
            for (int y = gy * 8; y < std::min((gy + GY) * 8, sc->camera.height); ++y)
                for (int x = gx * 8; x < std::min((gx + GX) * 8, sc->camera.width); ++x) {
                    rays.push_back(frame.pixel_ray(x, y));
                    found.push_back(0);
                }
            ++groups;
            int remaining = (int)rays.size();
            TileFetchState fetch;
            fetch.list = list;
            try {
                while (remaining > 0) {
                    auto iv = fetch_interval(fetch, frame, cfg);
                    if (!iv) break;
                    std::vector<uint32_t> act;
                    for (const auto& a : fetch.actives) act.push_back(a.word);
                    PrunedView view = build_pruned_view(tree, act);
                    if (!view.rootUsed || iv->zEnd <= iv->zBegin) continue;
                    ++intervals;
                    const float vz0 = frame.view_z_from_ndc(iv->zBegin), vz1 = frame.view_z_from_ndc(iv->zEnd);
                    std::vector<uint32_t> cost;
                    for (size_t i = 0; i < rays.size(); ++i) {
                        if (found[i]) continue;
                        const Ray& ray = rays[i];
                        uint32_t e = 0;
                        auto fieldAt = [&](float t) { return eval_pruned(view, ray.origin + ray.dir * t); };
                        TraceResult res = sphere_trace_interval(fieldAt, ray.t_from_view_z(vz0), ray.t_from_view_z(vz1), cfg, e);
                        cost.push_back(e);
                        evals += e;
                        work += (uint64_t)e * view.blobs.size();
                        if (res.hit) {
                            found[i] = 1;
                            --remaining;
                            ++hits;
                        }
                    }
                    steps += makespan(cost);
                }
            } catch (...) {
            }
        }
    std::printf("%s %dx%d tiles: groups %llu intervals %llu evals %llu work(evals x nodes) %llu steps %llu "
                "util %.3f hits %llu\n",
                name.c_str(), GX, GY, (unsigned long long)groups, (unsigned long long)intervals,
                (unsigned long long)evals, (unsigned long long)work, (unsigned long long)steps,
                evals / (32.0 * steps), (unsigned long long)hits);
}
