// view_shapes.cpp -- histogram of pruned-view shapes weighted by field
// evaluations, from the UNMODIFIED reference's render loop (tracer.cpp:141-236)
// replayed on one thread.  Guides which view classes the march specialises.
//   make -C oracle ref && g++ -std=c++20 -O2 -Dblobtree=blobtree_ref -I/root/reference/proj/include \
//     -I<json> scripts/probes/view_shapes.cpp paper_2304_09673_b200/csrc/scenes/scenes.cpp \
//     oracle/_ref/libblobtree_ref.a -o /tmp/view_shapes && /tmp/view_shapes C3
#include <algorithm>
#include <cstdio>
#include <map>
#include <string>

#include "blobtree/abuffer.hpp"
#include "blobtree/tracer.hpp"
#include "blobtree/traversal.hpp"
#include "../../paper_2304_09673_b200/csrc/scenes/scenes.hpp"

using namespace blobtree;

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "C3";
    auto sc = scenes::build(name, 0, 0, 0);
    const LinearTree& tree = sc->tree;
    RenderConfig cfg;
    CameraFrame frame(sc->camera);
    auto roi = propagate_roi(tree);
    auto vois = build_volumes_of_interest(tree, roi, cfg.hitEpsilon);
    TileABuffer ab = rasterize_volumes(vois, frame);
    std::map<std::string, uint64_t> bySig, byClass;
    std::map<uint32_t, uint64_t> byN;
    uint64_t total = 0;
    const int tilesX = frame.tiles_x(), tilesY = frame.tiles_y();
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
                    // signature: P<kind> / O<code>; class: comb if every operator follows a primitive
                    std::string sig, cls;
                    int depth = 0, maxDepth = 0;
                    for (const Blob& b : view.blobs) {
                        if (b.isPrimitive) {
                            sig += "P" + std::to_string(b.nodeOp);
                            ++depth;
                        } else {
                            sig += "O" + std::to_string(b.nodeOp);
                            --depth;
                        }
                        maxDepth = std::max(maxDepth, depth);
                    }
                    cls = "n=" + std::to_string(view.blobs.size()) + " depth" + std::to_string(maxDepth);
                    const float vz0 = frame.view_z_from_ndc(iv->zBegin), vz1 = frame.view_z_from_ndc(iv->zEnd);
                    uint64_t ev = 0;
                    for (size_t i = 0; i < rays.size(); ++i) {
                        if (found[i]) continue;
                        const Ray& ray = rays[i];
                        uint32_t evals = 0;
                        auto fieldAt = [&](float t) { return eval_pruned(view, ray.origin + ray.dir * t); };
                        TraceResult res = sphere_trace_interval(fieldAt, ray.t_from_view_z(vz0), ray.t_from_view_z(vz1), cfg, evals);
                        ev += evals;
                        if (res.hit) { found[i] = 1; --remaining; }
                    }
                    bySig[sig] += ev;
                    byClass[cls] += ev;
                    byN[view.primitiveCount] += ev;
                    total += ev;
                }
            } catch (...) {
            }
        }
    auto dump = [&](const char* title, auto& m, size_t top) {
        std::vector<std::pair<uint64_t, std::string>> v;
        for (auto& [k, c] : m) v.push_back({c, k});
        std::sort(v.rbegin(), v.rend());
        std::printf("== %s (%zu distinct)\n", title, v.size());
        double cum = 0;
        for (size_t i = 0; i < std::min(top, v.size()); ++i) {
            cum += 100.0 * v[i].first / total;
            std::printf("%6.2f%% %6.2f%%  %s\n", 100.0 * v[i].first / total, cum, v[i].second.c_str());
        }
    };
    std::printf("%s: %llu field evals\n", name.c_str(), (unsigned long long)total);
    dump("by class", byClass, 25);
    dump("by signature", bySig, 30);
    std::map<std::string, uint64_t> n2;
    for (auto& [k, c] : byN) n2["prims=" + std::to_string(k)] = c;
    dump("by primitive count", n2, 20);
}
