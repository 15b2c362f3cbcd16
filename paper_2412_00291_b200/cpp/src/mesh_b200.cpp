// semvox drop-in (B200): extract_mesh / IncrementalMesher / extract_vertex_cloud
// over the device mesher (svx_mesh_extract, svx_mesh.cu). Reference:
// proj/src/mesh.cpp:105-287.
#include "semvox/mesh.hpp"

#include "svx.h"

#include <algorithm>
#include <map>
#include <stdexcept>
#include <string>

namespace semvox {

namespace {

void check(svx_status s) {
    if (s == SVX_OK) return;
    char msg[1024];
    svx_last_error(msg, sizeof(msg));
    switch (s) {
        case SVX_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SVX_CAPACITY: throw CapacityError(msg);
        case SVX_DATA: throw DataError(msg);
        default: throw std::runtime_error(std::string("svx: ") + msg);
    }
}

// reserved_unlabeled_id (mesh.cpp:218-222)
int reserved_unlabeled(const LabelSet* labels) {
    if (labels && !labels->names.empty() && labels->names.back() == "unlabeled")
        return labels->size() - 1;
    return -1;
}

static_assert(sizeof(Vec3f) == 12 && sizeof(std::array<uint32_t, 3>) == 12);

LabeledMesh run(const VoxelStore& store, float min_weight, const LabelSet* labels,
                const std::vector<BlockCoord>* blocks) {
    store.flush_host_writes();  // host-mirrored blocks the caller mutated
    svx_map* m = store.device_map();
    uint64_t nv = 0, nf = 0;
    if (blocks)
        check(svx_mesh_extract(m, min_weight, reserved_unlabeled(labels),
                               reinterpret_cast<const int32_t*>(blocks->data()), blocks->size(),
                               &nv, &nf));
    else
        check(svx_mesh_extract(m, min_weight, reserved_unlabeled(labels), nullptr, 0, &nv, &nf));
    LabeledMesh mesh;
    mesh.vertices.resize(nv);
    mesh.vertex_normals.resize(nv);
    mesh.vertex_labels.resize(nv);
    mesh.faces.resize(nf);
    check(svx_mesh_read(m, reinterpret_cast<float*>(mesh.vertices.data()),
                        reinterpret_cast<float*>(mesh.vertex_normals.data()),
                        mesh.vertex_labels.data(), reinterpret_cast<uint32_t*>(mesh.faces.data())));
    mesh.vertex_colors.resize(nv);
    for (size_t i = 0; i < nv; ++i) {
        const uint8_t l = mesh.vertex_labels[i];
        mesh.vertex_colors[i] = labels && l != kUnlabeled ? labels->color_of_label(l) : Rgb{};
    }
    return mesh;
}

}  // namespace

LabeledMesh extract_mesh(const VoxelStore& store, float min_weight, const LabelSet* labels) {
    return run(store, min_weight, labels, nullptr);
}

VertexCloud extract_vertex_cloud(const LabeledMesh& mesh) {
    VertexCloud out;
    std::map<std::array<float, 3>, bool> seen;
    for (size_t i = 0; i < mesh.vertices.size(); ++i) {
        const Vec3f& v = mesh.vertices[i];
        if (!seen.emplace(std::array<float, 3>{v.x(), v.y(), v.z()}, true).second) continue;
        out.points.emplace_back(v.cast<double>());
        const uint8_t l = mesh.vertex_labels[i];
        out.labels.push_back(l == kUnlabeled ? -1 : int(l));
    }
    return out;
}

const LabeledMesh& IncrementalMesher::update(const VoxelStore& store,
                                             const std::vector<BlockCoord>& dirty) {
    // a cell based in block B reads B and its +1 neighbours: dirty D affects D - {0,1}^3
    std::vector<BlockCoord> affected;
    affected.reserve(8 * dirty.size());
    for (const BlockCoord& d : dirty)
        for (int dz = -1; dz <= 0; ++dz)
            for (int dy = -1; dy <= 0; ++dy)
                for (int dx = -1; dx <= 0; ++dx) affected.push_back({d.x + dx, d.y + dy, d.z + dz});
    std::sort(affected.begin(), affected.end());
    affected.erase(std::unique(affected.begin(), affected.end()), affected.end());
    std::vector<uint8_t> found(affected.size());
    if (!affected.empty())
        check(svx_has_blocks(store.device_map(), reinterpret_cast<const int32_t*>(affected.data()),
                             affected.size(), found.data()));
    last_remeshed_.clear();
    for (size_t i = 0; i < affected.size(); ++i) {
        if (found[i]) {
            cache_.insert(affected[i]);
            last_remeshed_.push_back(affected[i]);
        } else {
            cache_.erase(affected[i]);
        }
    }
    if (cache_.empty()) {
        stitched_ = LabeledMesh{};
        return stitched_;
    }
    const std::vector<BlockCoord> blocks(cache_.begin(), cache_.end());
    stitched_ = run(store, min_weight_, labels_, &blocks);
    return stitched_;
}

}  // namespace semvox
