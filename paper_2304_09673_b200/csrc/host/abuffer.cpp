// host/abuffer.cpp -- stage (b) entry point of the drop-in API.
// rasterize_volumes bins the volumes on the GPU (csrc/k_frame.cu) and
// downloads the CSR result into per-tile vectors; ray_volume_intersect and
// insert_sorted remain host helpers with the reference's semantics
// (src/abuffer.cpp:18-225).
#include "blobtree/abuffer.hpp"

#include <algorithm>

#include "../bt_geom.cuh"
#include "blobtree/device.hpp"
#include "blobtree/image_io.hpp"

namespace blobtree {

size_t TileABuffer::fragment_count() const {
    size_t total = 0;
    for (const auto& list : tiles) total += list.size();
    return total;
}

std::optional<std::pair<float, float>> ray_volume_intersect(const Ray& ray, const VolumeOfInterest& v) {
    using namespace btk;
    const F3 o{ray.origin.x, ray.origin.y, ray.origin.z};
    const F3 d{ray.dir.x, ray.dir.y, ray.dir.z};
    const F3 c{v.center.x, v.center.y, v.center.z};
    float t0 = 0.0f, t1 = 0.0f;
    bool hit = false;
    switch (v.family) {
        case VolumeOfInterest::Family::Sphere:
            hit = ray_sphere(o, d, c, v.radius, t0, t1);
            break;
        case VolumeOfInterest::Family::OrientedBox: {
            const Q4 q{v.rotation.w, v.rotation.x, v.rotation.y, v.rotation.z};
            const F3 ol = qrotate<E>(qconj(q), vsub<E>(o, c));
            hit = ray_obb_local(ol, d, q, F3{v.halfExtents.x, v.halfExtents.y, v.halfExtents.z}, t0, t1);
            break;
        }
        case VolumeOfInterest::Family::Capsule:
            hit = ray_capsule(o, d, c, F3{v.axisEnd.x, v.axisEnd.y, v.axisEnd.z}, v.radius, t0, t1);
            break;
    }
    if (!hit) return std::nullopt;
    return std::make_pair(t0, t1);
}

void insert_sorted(std::vector<Fragment>& list, const Fragment& f) {
    auto before = [](const Fragment& a, const Fragment& b) {
        return a.zEntry < b.zEntry || (a.zEntry == b.zEntry && a.primitiveWord < b.primitiveWord);
    };
    list.insert(std::upper_bound(list.begin(), list.end(), f, before), f);
}

TileABuffer rasterize_volumes(std::span<const VolumeOfInterest> volumes, const CameraFrame& frame) {
    TileABuffer out;
    out.tilesX = frame.tiles_x();
    out.tilesY = frame.tiles_y();
    const size_t tiles = static_cast<size_t>(out.tilesX) * out.tilesY;
    out.tiles.resize(tiles);
    ContextLease ctx;
    static_assert(sizeof(VolumeOfInterest) == sizeof(bt_voi), "VolumeOfInterest layout");
    std::vector<bt_voi> raw(volumes.size());
    for (size_t i = 0; i < volumes.size(); ++i) {
        const VolumeOfInterest& v = volumes[i];
        bt_voi& r = raw[i];
        r = bt_voi{};
        r.family = static_cast<uint8_t>(v.family);
        r.primitiveWord = v.primitiveWord;
        r.center[0] = v.center.x, r.center[1] = v.center.y, r.center[2] = v.center.z;
        r.radius = v.radius;
        r.halfExtents[0] = v.halfExtents.x, r.halfExtents[1] = v.halfExtents.y, r.halfExtents[2] = v.halfExtents.z;
        r.rotation[0] = v.rotation.w, r.rotation[1] = v.rotation.x, r.rotation[2] = v.rotation.y,
        r.rotation[3] = v.rotation.z;
        r.axisEnd[0] = v.axisEnd.x, r.axisEnd[1] = v.axisEnd.y, r.axisEnd[2] = v.axisEnd.z;
    }
    check_device(bt_voi_upload(ctx, raw.data(), static_cast<uint32_t>(raw.size())), "bt_voi_upload");
    const bt_camera cam = to_device_camera(frame);
    check_device(bt_abuffer_build(ctx, &cam, 0, 0), "bt_abuffer_build");
    uint64_t total = 0;
    check_device(bt_abuffer_info(ctx, &total, nullptr, nullptr), "bt_abuffer_info");
    std::vector<uint32_t> offsets(tiles + 1);
    std::vector<bt_fragment> frags(total);
    check_device(bt_abuffer_download(ctx, offsets.data(), frags.data(), total), "bt_abuffer_download");
    for (size_t t = 0; t < tiles; ++t) {
        auto& list = out.tiles[t];
        list.reserve(offsets[t + 1] - offsets[t]);
        for (uint32_t i = offsets[t]; i < offsets[t + 1]; ++i)
            list.push_back(Fragment{frags[i].primitiveWord, frags[i].zEntry, frags[i].zExit});
    }
    return out;
}

void write_tile_counts_pgm(const TileABuffer& buffer, const char* path) {
    std::vector<uint16_t> counts(buffer.tiles.size());
    std::transform(buffer.tiles.begin(), buffer.tiles.end(), counts.begin(),
                   [](const std::vector<Fragment>& l) { return static_cast<uint16_t>(std::min<size_t>(l.size(), 65535)); });
    write_pgm16(path, buffer.tilesX, buffer.tilesY, counts);
}

}  // namespace blobtree
