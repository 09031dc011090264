// blobtree_render -- the command-line harness specified by the reference
// (SPEC.md "cli-harness", render_command; the reference ships only a stub,
// proj/tools/blobtree_render.cpp:1), on the B200 library.
//
//   blobtree_render (--scene PATH | --generate preset:gridN:kind:blend [--seed N])
//                   [--width W] [--height H] [--out DIR] [--stats-dir DIR]
//                   [--oracle] [--compare DIR] [--lipschitz L] [--relax R]
//                   [--min-step S] [--max-overlap N] [--fetch-window Z]
//                   [--normals depth|grad] [--tile-size 8] [--bench [FRAMES]]
//                   [--fast] [--device D]
//
// The pipeline is compile -> compute_fast_indices -> (device) ROI/VOIs ->
// A-buffer -> synchronized tracing -> normals; --oracle swaps in the
// brute-force oracle_render.  --fast selects the FMA field evaluation (the
// tolerance path) instead of the IEEE-exact kernels.  Outputs follow the
// reference's image_io: --out writes the G-buffer directory (depth16.pgm,
// hits.pgm, normal.ppm, color.ppm, meta.txt), --stats-dir the diagnostic
// planes, --compare loads a G-buffer directory and prints the CompareReport.
// --bench reports per-frame device time and the instrumentation totals (field
// evaluations, retained-node visits, full-tree-equivalent visits).
// Errors (I/O, parse, validation, device) exit non-zero with a message.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "blobtree/camera.hpp"
#include "blobtree/device.hpp"
#include "blobtree/image_io.hpp"
#include "blobtree/linear_tree.hpp"
#include "blobtree/scene_io.hpp"
#include "blobtree/tracer.hpp"

using namespace blobtree;

namespace {

struct Args {
    std::string scene, generate, out, statsDir, compare;
    uint64_t seed = 1;
    int width = 512, height = 512, device = -1, tileSize = 8;
    bool oracle = false, fast = false;
    int bench = 0;
    RenderConfig cfg;
};

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr,
                 "error: %s\nusage: blobtree_render (--scene PATH | --generate preset:gridN:kind:blend [--seed N])\n"
                 "       [--width W] [--height H] [--out DIR] [--stats-dir DIR] [--oracle] [--compare DIR]\n"
                 "       [--lipschitz L] [--relax R] [--min-step S] [--max-overlap N] [--fetch-window Z]\n"
                 "       [--normals depth|grad] [--tile-size 8] [--bench [FRAMES]] [--fast] [--device D]\n",
                 msg);
    std::exit(2);
}

double number(const char* flag, const char* v) {
    char* end = nullptr;
    const double x = std::strtod(v, &end);
    if (!v[0] || *end) usage((std::string("bad number for ") + flag + ": " + v).c_str());
    return x;
}

Args parse(int argc, char** argv) {
    Args a;
    bool hitEpsSet = false;
    for (int i = 1; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> const char* {
            if (i + 1 >= argc) usage((f + " needs a value").c_str());
            return argv[++i];
        };
        if (f == "--scene") a.scene = val();
        else if (f == "--generate") a.generate = val();
        else if (f == "--seed") a.seed = (uint64_t)number("--seed", val());
        else if (f == "--width") a.width = (int)number("--width", val());
        else if (f == "--height") a.height = (int)number("--height", val());
        else if (f == "--out") a.out = val();
        else if (f == "--stats-dir") a.statsDir = val();
        else if (f == "--compare") a.compare = val();
        else if (f == "--oracle") a.oracle = true;
        else if (f == "--fast") a.fast = true;
        else if (f == "--device") a.device = (int)number("--device", val());
        else if (f == "--lipschitz") a.cfg.lipschitz = (float)number("--lipschitz", val());
        else if (f == "--relax") a.cfg.relax = (float)number("--relax", val());
        else if (f == "--min-step") a.cfg.minStep = (float)number("--min-step", val());
        else if (f == "--hit-epsilon") {
            a.cfg.hitEpsilon = (float)number("--hit-epsilon", val());
            hitEpsSet = true;
        } else if (f == "--max-overlap") a.cfg.maxOverlap = (uint32_t)number("--max-overlap", val());
        else if (f == "--fetch-window") a.cfg.fetchWindow = (float)number("--fetch-window", val());
        else if (f == "--tile-size") a.tileSize = (int)number("--tile-size", val());
        else if (f == "--normals") {
            const std::string m = val();
            if (m == "depth") a.cfg.normalsMode = RenderConfig::NormalsMode::DepthDifferential;
            else if (m == "grad") a.cfg.normalsMode = RenderConfig::NormalsMode::CentralDifference;
            else usage("--normals takes depth or grad");
        } else if (f == "--bench") {
            a.bench = 5;
            if (i + 1 < argc && argv[i + 1][0] != '-') a.bench = (int)number("--bench", argv[++i]);
        } else usage(("unknown flag " + f).c_str());
    }
    if (a.scene.empty() == a.generate.empty()) usage("exactly one of --scene or --generate is required");
    if (a.tileSize != 8) usage("--tile-size other than 8 is not supported in v1");
    if (a.width <= 0 || a.height <= 0) usage("--width and --height must be positive");
    if (!hitEpsSet) a.cfg.hitEpsilon = RenderConfig::default_hit_epsilon(a.cfg.minStep, a.cfg.lipschitz);
    return a;
}

SceneDocument load(const Args& a) {
    if (!a.scene.empty()) return load_scene_file(a.scene);
    // preset:gridN:kind:blend
    std::vector<std::string> part;
    size_t s = 0;
    for (;;) {
        const size_t e = a.generate.find(':', s);
        part.push_back(a.generate.substr(s, e == std::string::npos ? std::string::npos : e - s));
        if (e == std::string::npos) break;
        s = e + 1;
    }
    if (part.size() != 4) usage("--generate takes preset:gridN:kind:blend");
    return generate_synthetic(part[0], (uint32_t)number("gridN", part[1].c_str()), part[2], part[3], a.seed);
}

int run(const Args& a) {
    SceneDocument doc = load(a);
    Camera cam = doc.camera;
    cam.width = a.width;
    cam.height = a.height;
    validate_camera(cam);
    validate_config(a.cfg);
    LinearTree tree = compile(*doc.root);
    compute_fast_indices(tree);
    const CameraFrame frame(cam);

    GBuffer g;
    RenderStats st;
    double frameMs = 0.0;
    if (a.oracle) {
        const auto t0 = std::chrono::steady_clock::now();
        g = oracle_render(tree, frame, a.cfg, &st);
        compute_normals(tree, g, frame, a.cfg.normalsMode);
        frameMs = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } else {
        Renderer r(a.device);
        r.upload(tree);
        const bool exact = !a.fast;
        r.render(frame, a.cfg, exact, false);  // eager, capacity-checked frame
        const int frames = a.bench > 0 ? a.bench : 0;
        if (frames > 0) {
            check_device(bt_sync(r.handle()), "bt_sync");
            r.reset_stats();
            const auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < frames; ++i) r.render(frame, a.cfg, exact, true);  // graph replays
            check_device(bt_sync(r.handle()), "bt_sync");
            frameMs = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / frames;
        }
        g = r.download();
        st = r.stats();
        if (frames > 0) {  // per-frame totals
            st.fieldEvals /= (uint64_t)frames;
            st.retainedNodeVisits /= (uint64_t)frames;
            st.primitiveEvals /= (uint64_t)frames;
        }
    }
    size_t hits = 0;
    for (uint8_t h : g.hit) hits += h;
    std::printf("scene: %zu nodes, %zu primitives; image %dx%d, %zu hits; %s\n", tree.nodes.size(),
                tree.primitiveWords.size(), g.width, g.height, hits,
                a.oracle ? "oracle_render (full tree)" : (a.fast ? "pipeline, FMA field evaluation" : "pipeline, IEEE-exact"));
    if (a.bench > 0 || a.oracle) {
        std::printf("frame: %.4f ms (%.1f Mrays/s)\n", frameMs,
                    frameMs > 0.0 ? (double)g.width * g.height / (frameMs * 1e3) : 0.0);
        std::printf("field evals %llu, retained-node visits %llu (%.2f per eval), full-tree-equivalent visits %llu, "
                    "max overlap %u, max cache bytes %u\n",
                    (unsigned long long)st.fieldEvals, (unsigned long long)st.retainedNodeVisits,
                    st.mean_retained_per_eval(), (unsigned long long)st.full_tree_equivalent_visits(), st.maxOverlap,
                    st.maxCacheBytes);
    }
    if (!a.out.empty()) write_gbuffer(a.out, g, frame);
    if (!a.statsDir.empty()) write_stats_images(a.statsDir, g);
    if (!a.compare.empty()) {
        const GBuffer ref = load_gbuffer(a.compare);
        const CompareReport rep = compare_gbuffers(g, ref, 2.0f * a.cfg.minStep);
        std::printf("%s\n", format_report(rep).c_str());
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const Args a = parse(argc, argv);
    try {
        return run(a);
    } catch (const SceneError& e) {
        std::fprintf(stderr, "scene error: %s\n", e.what());
    } catch (const DeviceError& e) {
        std::fprintf(stderr, "device error: %s\n", e.what());
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "invalid argument: %s\n", e.what());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
    }
    return 1;
}
