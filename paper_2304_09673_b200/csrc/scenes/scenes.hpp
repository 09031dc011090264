// scenes.hpp -- synthetic workloads C1..C5 and the
// small scenes of the reference's own tests, built through the PUBLIC
// blobtree C++ API only.
//
// The same source is compiled twice: against this repo's drop-in headers
// (libbt_scenes.so, used by bench.py and the tests) and against the
// reference headers with -Dblobtree=blobtree_ref (oracle/_ref/libbt_ref.so,
// the CPU checker).  Identical source + identical RNG draws => identical
// scenes on both sides; tests/test_scenes.py checks the compiled word arrays
// bit for bit.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "blobtree/camera.hpp"
#include "blobtree/linear_tree.hpp"

namespace scenes {

struct Scene {
    blobtree::Camera camera;
    blobtree::LinearTree tree;
    std::vector<blobtree::PrimitiveParams> base;  // primitiveWords order
    std::string name;
};

// name grammar:
//   C1 | C2 | C3 | C4 | C5            benchmark configs
//   sphere | csg | slab | comb_error  reference test scenes
//   gen:<preset>:<n>:<kind>:<blend>   generate_synthetic (seed = `seed`)
//   random:<prims>                    random union comb of the 6 kinds
// width/height <= 0 keep the config's own resolution.
std::unique_ptr<Scene> build(const std::string& name, uint32_t seed, int width, int height);

// per-frame perturbation of C3/C4: translate = base + 0.05 (sin(0.7f+i),
// cos(1.3f+2i), sin(0.9f+3i)) for every primitive i
blobtree::PrimitiveParams perturbed(const blobtree::PrimitiveParams& base, uint32_t frame, uint32_t i);

}  // namespace scenes
