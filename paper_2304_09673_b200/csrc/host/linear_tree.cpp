// host/linear_tree.cpp -- blob packing, post-order compilation, fast
// ancestor pointers (one-time host preprocessing) and the stage-(a) entry
// points, which run on the GPU.
//
// Reference: src/linear_tree.cpp:9-283.
#include "blobtree/linear_tree.hpp"

#include <algorithm>
#include <bit>
#include <cstring>
#include <stdexcept>

#include "blobtree/device.hpp"

namespace blobtree {

uint32_t pack_blob(const Blob& b) {
    if (b.nodeOp > 31) throw std::invalid_argument("nodeop exceeds 5 bits");
    if (b.ignoreMode > 3) throw std::invalid_argument("ignore mode exceeds 2 bits");
    if (b.ancestor > kAncestorSentinel) throw std::invalid_argument("ancestor exceeds 23 bits");
    uint32_t w = b.ancestor;
    w |= static_cast<uint32_t>(b.isLeft) << 23;
    w |= static_cast<uint32_t>(b.ignoreMode) << 24;
    w |= static_cast<uint32_t>(b.nodeOp) << 26;
    w |= static_cast<uint32_t>(b.isPrimitive) << 31;
    return w;
}

Blob unpack_blob(uint32_t w) {
    Blob b;
    b.ancestor = w & kAncestorSentinel;
    b.isLeft = (w >> 23) & 1u;
    b.ignoreMode = static_cast<uint8_t>((w >> 24) & 3u);
    b.nodeOp = static_cast<uint8_t>((w >> 26) & 31u);
    b.isPrimitive = (w >> 31) != 0u;
    return b;
}

Blob LinearTree::blob_at(uint32_t word) const { return unpack_blob(std::bit_cast<uint32_t>(data[4 * word])); }

void LinearTree::set_blob(uint32_t word, const Blob& b) { data[4 * word] = std::bit_cast<float>(pack_blob(b)); }

uint32_t LinearTree::ordinal_of_word(uint32_t word) const {
    size_t lo = 0, hi = nodes.size();
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (nodes[mid].word < word) lo = mid + 1;
        else hi = mid;
    }
    if (lo == nodes.size() || nodes[lo].word != word) throw std::out_of_range("no node starts at this word");
    return static_cast<uint32_t>(lo);
}

uint32_t primitive_word_count(PrimitiveKind kind) {
    return 1u + (kTransformFloatCount + shape_float_count(kind) + 3u) / 4u;
}
uint32_t operator_word_count(OperatorKind kind) { return is_sharp(kind) ? 1u : 2u; }

namespace {

void store_params(LinearTree& t, uint32_t word, const PrimitiveParams& p) {
    float* dst = t.data.data() + 4 * (word + 1);
    const float head[kTransformFloatCount] = {p.frame.translate.x, p.frame.translate.y, p.frame.translate.z,
                                              p.frame.rotation.w,  p.frame.rotation.x,  p.frame.rotation.y,
                                              p.frame.rotation.z};
    std::memcpy(dst, head, sizeof(head));
    std::memcpy(dst + kTransformFloatCount, p.shape.data(), shape_float_count(p.kind) * sizeof(float));
}

// Post-order emitter: children first (left, right), then the node itself;
// returns the node's ordinal.
class Emitter {
public:
    explicit Emitter(LinearTree& t) : t_(t) {}

    uint32_t emit(const SceneNode& n, bool isLeft) {
        if (!n.isPrimitive && !(n.left && n.right)) throw std::invalid_argument("operator node must have two children");
        int32_t lo = -1, ro = -1;
        if (!n.isPrimitive) {
            lo = static_cast<int32_t>(emit(*n.left, true));
            ro = static_cast<int32_t>(emit(*n.right, false));
        }
        const uint32_t word = cursor_;
        cursor_ += n.isPrimitive ? primitive_word_count(n.primitive.kind) : operator_word_count(n.op.kind);
        if (cursor_ >= kAncestorSentinel) throw std::invalid_argument("tree exceeds the 23-bit node index space");
        t_.data.resize(4 * static_cast<size_t>(cursor_), 0.0f);

        Blob b;
        b.isPrimitive = n.isPrimitive;
        b.isLeft = isLeft;
        b.ancestor = kAncestorSentinel;
        if (n.isPrimitive) {
            validate_primitive(n.primitive);
            b.nodeOp = static_cast<uint8_t>(n.primitive.kind);
            b.ignoreMode = kNeverIgnore;
            store_params(t_, word, n.primitive);
        } else {
            validate_operator(n.op);
            b.nodeOp = static_cast<uint8_t>(n.op.kind);
            b.ignoreMode = ignore_mode_for(n.op.kind);
            if (!is_sharp(n.op.kind)) {
                t_.data[4 * (word + 1)] = n.op.blend;
                t_.data[4 * (word + 1) + 1] = n.op.range;
            }
        }
        t_.set_blob(word, b);

        NodeRecord rec;
        rec.word = word;
        rec.isPrimitive = n.isPrimitive;
        rec.nodeOp = b.nodeOp;
        rec.leftChild = lo;
        rec.rightChild = ro;
        const uint32_t ordinal = static_cast<uint32_t>(t_.nodes.size());
        t_.nodes.push_back(rec);
        if (n.isPrimitive) {
            t_.primitiveWords.push_back(word);
        } else {
            for (int32_t c : {lo, ro}) link_parent(static_cast<uint32_t>(c), word);
            if (is_smooth(n.op.kind)) t_.hasUnboundedBlend = true;
        }
        return ordinal;
    }

private:
    void link_parent(uint32_t child, uint32_t parentWord) {
        NodeRecord& rec = t_.nodes[child];
        rec.parentWord = parentWord;
        Blob cb = t_.blob_at(rec.word);
        cb.ancestor = parentWord;
        t_.set_blob(rec.word, cb);
    }

    LinearTree& t_;
    uint32_t cursor_ = 0;
};

}  // namespace

LinearTree compile(const SceneNode& root) {
    LinearTree tree;
    Emitter em(tree);
    const uint32_t rootOrdinal = em.emit(root, true);
    tree.rootWord = tree.nodes[rootOrdinal].word;
    return tree;
}

void compute_fast_indices(LinearTree& tree) {
    // word -> ordinal lookup table (O(1) instead of a binary search per hop)
    std::vector<int32_t> ordOf(tree.word_count() + 1, -1);
    for (size_t i = 0; i < tree.nodes.size(); ++i) ordOf[tree.nodes[i].word] = static_cast<int32_t>(i);
    for (const NodeRecord& rec : tree.nodes) {
        if (!ancestor_valid(rec.parentWord)) continue;
        Blob self = tree.blob_at(rec.word);
        const bool side = self.isLeft;
        const uint8_t guard = side ? kIgnoreIfRightAbsent : kIgnoreIfLeftAbsent;
        uint32_t target = rec.parentWord;
        while (true) {
            const Blob up = tree.blob_at(target);
            if (up.isLeft != side || (up.ignoreMode & guard) != 0) break;
            const uint32_t next = tree.nodes[static_cast<size_t>(ordOf[target])].parentWord;
            if (!ancestor_valid(next)) break;
            target = next;
        }
        self.ancestor = target;
        tree.set_blob(rec.word, self);
    }
}

void update_primitive_params(LinearTree& tree, uint32_t word, const PrimitiveParams& params) {
    const Blob b = tree.blob_at(word);
    if (!b.isPrimitive || b.nodeOp != static_cast<uint8_t>(params.kind))
        throw std::invalid_argument("in-place update must keep the primitive kind");
    validate_primitive(params);
    store_params(tree, word, params);
}

bool VolumeOfInterest::contains(Point3 p) const {
    if (family == Family::Sphere) return length(p - center) <= radius;
    if (family == Family::OrientedBox) {
        const Vec3 l = abs(rotate(conjugate(rotation), p - center));
        return l.x <= halfExtents.x && l.y <= halfExtents.y && l.z <= halfExtents.z;
    }
    if (family == Family::Capsule) {
        const Vec3 ab = axisEnd - center;
        const float t = std::clamp(dot(p - center, ab) / std::max(length_sq(ab), 1e-20f), 0.0f, 1.0f);
        return length(p - (center + ab * t)) <= radius;
    }
    return false;
}

// ---------------------------------------------------------------- stage (a) on the GPU

namespace {

void upload_tree(bt_ctx* ctx, const LinearTree& tree) {
    static_assert(sizeof(NodeRecord) == sizeof(bt_node), "NodeRecord layout");
    check_device(bt_tree_upload(ctx, tree.data.data(), tree.word_count(),
                                reinterpret_cast<const bt_node*>(tree.nodes.data()), tree.node_count(),
                                tree.primitiveWords.data(), static_cast<uint32_t>(tree.primitiveWords.size()),
                                tree.rootWord),
                 "bt_tree_upload");
}

}  // namespace

std::vector<float> propagate_roi(const LinearTree& tree) {
    std::vector<float> roi(tree.nodes.size(), 0.0f);
    if (tree.nodes.empty()) return roi;
    ContextLease ctx;
    upload_tree(ctx, tree);
    check_device(bt_roi(ctx, roi.data(), tree.node_count()), "bt_roi");
    return roi;
}

std::vector<VolumeOfInterest> build_volumes_of_interest(const LinearTree& tree, std::span<const float> roiUpper,
                                                        float margin) {
    const uint32_t n = static_cast<uint32_t>(tree.primitiveWords.size());
    std::vector<VolumeOfInterest> out(n);
    if (n == 0) return out;
    // the reference reads roiUpper[ordinal] for every primitive
    std::vector<float> roi(tree.nodes.size(), 0.0f);
    for (uint32_t w : tree.primitiveWords) {
        const uint32_t o = tree.ordinal_of_word(w);
        if (o >= roiUpper.size()) throw std::out_of_range("roiUpper has no entry for a primitive ordinal");
        roi[o] = roiUpper[o];
    }
    ContextLease ctx;
    upload_tree(ctx, tree);
    check_device(bt_roi_upload(ctx, roi.data(), tree.node_count()), "bt_roi_upload");
    check_device(bt_voi_build(ctx, margin), "bt_voi_build");
    static_assert(sizeof(VolumeOfInterest) == sizeof(bt_voi), "VolumeOfInterest layout");
    std::vector<bt_voi> raw(n);
    check_device(bt_voi_download(ctx, raw.data(), n), "bt_voi_download");
    for (uint32_t i = 0; i < n; ++i) {
        VolumeOfInterest& v = out[i];
        v.family = static_cast<VolumeOfInterest::Family>(raw[i].family);
        v.primitiveWord = raw[i].primitiveWord;
        v.center = Vec3{raw[i].center[0], raw[i].center[1], raw[i].center[2]};
        v.radius = raw[i].radius;
        v.halfExtents = Vec3{raw[i].halfExtents[0], raw[i].halfExtents[1], raw[i].halfExtents[2]};
        v.rotation = Quat{raw[i].rotation[0], raw[i].rotation[1], raw[i].rotation[2], raw[i].rotation[3]};
        v.axisEnd = Vec3{raw[i].axisEnd[0], raw[i].axisEnd[1], raw[i].axisEnd[2]};
    }
    return out;
}

}  // namespace blobtree
