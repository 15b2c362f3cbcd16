// TEST INFRASTRUCTURE ONLY (oracle/): a C-ABI driver over the reference's OWN
// classes (compiled unmodified from /root/reference/proj/src into
// oracle/_ref/libsemvox_ref.so). Lets tests/ and bench.py's cpu_baseline /
// --impl reference leg run the reference hot path on exactly the inputs the GPU
// path consumes. Structs are the svx.h ones; nothing here is product code.
#include "../include/svx.h"

#include "semvox/mesh.hpp"
#include "semvox/scan_projection.hpp"
#include "semvox/semantic_integrator.hpp"
#include "semvox/threading.hpp"
#include "semvox/tsdf_integrator.hpp"
#include "semvox/voxel_store.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

using namespace semvox;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* msg) {
    g_err = msg;
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const CapacityError& e) {
        return set_err(SVX_CAPACITY, e.what());
    } catch (const DataError& e) {
        return set_err(SVX_DATA, e.what());
    } catch (const std::invalid_argument& e) {
        return set_err(SVX_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return set_err(SVX_DATA, e.what());
    }
}

ProjectionModel to_model(const svx_lidar_model* m) {
    ProjectionModel pm;
    pm.width = m->width;
    pm.height_px = m->height_px;
    pm.delta_phi = m->delta_phi;
    pm.delta_theta = m->delta_theta;
    pm.theta0 = m->theta0;
    pm.scale_f = m->scale_f;
    pm.offset_o = m->offset_o;
    pm.min_range = m->min_range;
    return pm;
}

Pose to_pose(const svx_pose* p) {
    Pose T = Pose::Identity();
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) T.linear()(i, j) = p->R[3 * i + j];
        T.translation()[i] = p->t[i];
    }
    return T;
}

IntegratorConfig to_icfg(const svx_integrator_cfg* c) {
    IntegratorConfig ic;
    ic.mode = c->mode == SVX_PROJECTIVE ? DistanceMode::projective : DistanceMode::non_projective;
    ic.truncation = c->truncation;
    ic.max_range = c->max_range;
    ic.alpha_epsilon = c->alpha_epsilon;
    ic.min_weight_clamp = c->min_weight_clamp;
    ic.drop_unreliable = c->drop_unreliable != 0;
    return ic;
}

struct RefMap {
    std::unique_ptr<VoxelStore> store;
    std::unique_ptr<TsdfIntegrator> tsdf;
    std::unique_ptr<SemanticIntegrator> sem;
    std::unique_ptr<IncrementalMesher> mesher;
    LabelSet mesher_labels;
    LabeledMesh mesh;
};

// A LabelSet whose reserved_unlabeled_id (mesh.cpp:218-222) is `reserved` (-1: none).
LabelSet reserved_labels(int32_t reserved) {
    LabelSet ls;
    if (reserved < 0) return ls;
    for (int i = 0; i <= reserved; ++i) {
        ls.names.push_back(i == reserved ? "unlabeled" : "c" + std::to_string(i));
        ls.colors.push_back(Rgb{});
    }
    return ls;
}

void fill_report(const FrameReport& r, svx_frame_report* out) {
    out->frame = r.frame;
    out->updated_voxels = r.updated_voxels;
    out->new_blocks = r.new_blocks;
    out->elapsed_ms = r.elapsed_ms;
}

ScanImages make_images(const svx_lidar_model* model, const float* depth, const float* normals,
                       const uint8_t* valid) {
    ScanImages img;
    img.model = to_model(model);
    img.width = model->width;
    img.height_px = model->height_px;
    const size_t n = static_cast<size_t>(img.width) * img.height_px;
    img.depth.assign(depth, depth + n);
    img.height.assign(n, 0.f);
    if (normals) {
        img.normals.resize(n);
        for (size_t i = 0; i < n; ++i)
            img.normals[i] = Vec3f(normals[3 * i], normals[3 * i + 1], normals[3 * i + 2]);
        img.normal_valid.assign(valid, valid + n);
    }
    return img;
}

PosedCloud make_cloud(const float* pts, uint64_t n, int32_t stride, const svx_pose* pose) {
    PosedCloud cloud;
    cloud.pose = to_pose(pose);
    cloud.points.resize(n);
    for (uint64_t i = 0; i < n; ++i)
        cloud.points[i] = Vec3d(pts[i * stride], pts[i * stride + 1], pts[i * stride + 2]);
    return cloud;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_worker_count() { return worker_count(); }

int ref_lidar_spinning(int32_t w, int32_t h, double up, double down, svx_lidar_model* out) {
    return guarded([&] {
        const ProjectionModel m = ProjectionModel::spinning(w, h, up, down);
        out->width = m.width;
        out->height_px = m.height_px;
        out->delta_phi = m.delta_phi;
        out->delta_theta = m.delta_theta;
        out->theta0 = m.theta0;
        out->scale_f = m.scale_f;
        out->offset_o = m.offset_o;
        out->min_range = m.min_range;
    });
}

// VoxelStore::load (voxel_store.cpp:132-168) into a new driver map.
void* ref_map_load(const char* path) {
    RefMap* m = nullptr;
    const int st = guarded([&] {
        auto store = std::make_unique<VoxelStore>(VoxelStore::load(path));
        m = new RefMap{std::move(store), nullptr, nullptr};
    });
    return st == 0 ? m : nullptr;
}

void* ref_map_create(const svx_map_cfg* cfg) {
    RefMap* m = nullptr;
    const int st = guarded([&] {
        MapConfig mc;
        mc.voxel_size = cfg->voxel_size;
        mc.truncation = cfg->truncation;
        mc.num_labels = cfg->num_labels;
        mc.max_blocks = cfg->max_blocks;
        auto store = std::make_unique<VoxelStore>(mc);
        m = new RefMap{std::move(store), nullptr, nullptr};
    });
    return st == 0 ? m : nullptr;
}

void ref_map_destroy(void* h) { delete static_cast<RefMap*>(h); }

// project_cloud + compute_normal_image
int ref_project(const svx_lidar_model* model, const float* pts, uint64_t n, int32_t stride,
                const svx_pose* pose, float* depth, float* height, float* normals,
                uint8_t* valid, uint64_t* dropped) {
    return guarded([&] {
        const ProjectionModel pm = to_model(model);
        ScanImages img = project_cloud(make_cloud(pts, n, stride, pose), pm);
        compute_normal_image(img, pm);
        const size_t P = img.depth.size();
        std::memcpy(depth, img.depth.data(), P * sizeof(float));
        std::memcpy(height, img.height.data(), P * sizeof(float));
        for (size_t i = 0; i < P; ++i)
            for (int c = 0; c < 3; ++c) normals[3 * i + c] = img.normals[i][c];
        std::memcpy(valid, img.normal_valid.data(), P);
        *dropped = img.dropped;
    });
}

int ref_integrate(void* h, const svx_lidar_model* model, const float* depth, const float* normals,
                  const uint8_t* valid, const svx_pose* pose, const svx_integrator_cfg* cfg,
                  svx_frame_report* rep) {
    RefMap* m = static_cast<RefMap*>(h);
    return guarded([&] {
        if (!m->tsdf) m->tsdf = std::make_unique<TsdfIntegrator>(*m->store, to_icfg(cfg));
        fill_report(m->tsdf->integrate_frame(make_images(model, depth, normals, valid), to_pose(pose)),
                    rep);
    });
}

// The per-frame body of cmd_integrate (semvox_main.cpp:122-124) on one posed
// cloud; *wall_ms covers project_cloud + compute_normal_image + integrate_frame.
int ref_integrate_cloud(void* h, const svx_lidar_model* model, const float* pts, uint64_t n,
                        int32_t stride, const svx_pose* pose, const svx_integrator_cfg* cfg,
                        svx_frame_report* rep, double* wall_ms) {
    RefMap* m = static_cast<RefMap*>(h);
    return guarded([&] {
        if (!m->tsdf) m->tsdf = std::make_unique<TsdfIntegrator>(*m->store, to_icfg(cfg));
        const ProjectionModel pm = to_model(model);
        const PosedCloud cloud = make_cloud(pts, n, stride, pose);
        const auto t0 = std::chrono::steady_clock::now();
        ScanImages img = project_cloud(cloud, pm);
        compute_normal_image(img, pm);
        fill_report(m->tsdf->integrate_frame(img, cloud.pose), rep);
        *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

int ref_integrate_labels(void* h, const svx_label_image* li, const svx_semantic_cfg* cfg,
                         svx_frame_report* rep) {
    RefMap* m = static_cast<RefMap*>(h);
    return guarded([&] {
        if (!m->sem) {
            SemanticConfig sc;
            sc.use_bayes = cfg->use_bayes != 0;
            sc.likelihood_floor = cfg->likelihood_floor;
            sc.default_confidence = cfg->default_confidence;
            sc.occlusion = cfg->occlusion == SVX_OCCLUSION_RAYCAST ? OcclusionCheck::raycast
                                                                   : OcclusionCheck::surrogate;
            m->sem = std::make_unique<SemanticIntegrator>(*m->store, sc);
        }
        LabelImage img;
        img.width = li->width;
        img.height = li->height;
        const size_t P = static_cast<size_t>(li->width) * li->height;
        img.labels.assign(li->labels, li->labels + P);
        if (li->confidence) img.confidence.assign(li->confidence, li->confidence + P);
        if (li->prob_tensor)
            img.prob_tensor.assign(li->prob_tensor,
                                   li->prob_tensor + P * static_cast<size_t>(m->store->config().num_labels));
        img.fx = li->fx;
        img.fy = li->fy;
        img.cx = li->cx;
        img.cy = li->cy;
        img.pose = to_pose(&li->pose);
        img.max_depth = li->max_depth;
        fill_report(m->sem->integrate_labels(img), rep);
    });
}

int ref_save(void* h, const char* path) {
    return guarded([&] { static_cast<RefMap*>(h)->store->save(path); });
}

uint64_t ref_block_count(void* h) { return static_cast<RefMap*>(h)->store->block_count(); }

int ref_stats(void* h, svx_stats* out) {
    const StoreStats s = static_cast<RefMap*>(h)->store->stats();
    out->allocated_blocks = s.allocated_blocks;
    out->observed_voxels = s.observed_voxels;
    out->memory_bytes = s.memory_bytes;
    return 0;
}

int ref_get_or_allocate_block(void* h, const int32_t b[3]) {
    return guarded([&] { static_cast<RefMap*>(h)->store->get_or_allocate_block({b[0], b[1], b[2]}); });
}

int ref_block_write(void* h, const int32_t b[3], const svx_tsdf_voxel* tsdf, const float* sem,
                    int32_t has_sem) {
    RefMap* m = static_cast<RefMap*>(h);
    return guarded([&] {
        VoxelBlock& blk = m->store->get_or_allocate_block({b[0], b[1], b[2]});
        for (int i = 0; i < kBlockVoxels; ++i) {
            blk.tsdf[i].distance = tsdf[i].distance;
            blk.tsdf[i].weight = tsdf[i].weight;
            blk.tsdf[i].gradient = Vec3f(tsdf[i].gradient[0], tsdf[i].gradient[1], tsdf[i].gradient[2]);
        }
        if (has_sem) {
            const int K = m->store->config().num_labels;
            blk.ensure_semantics(K);
            if (sem) std::memcpy(blk.semantics.data(), sem, sizeof(float) * kBlockVoxels * K);
        }
    });
}

// found: 1/0. probs may be NULL.
int ref_lookup(void* h, const int32_t* v, uint64_t n, svx_tsdf_voxel* out, float* probs,
               uint8_t* found) {
    RefMap* m = static_cast<RefMap*>(h);
    const int K = m->store->config().num_labels;
    for (uint64_t i = 0; i < n; ++i) {
        const auto r = m->store->lookup_voxel({v[3 * i], v[3 * i + 1], v[3 * i + 2]});
        found[i] = r.has_value();
        if (!r) continue;
        out[i].distance = r->first.distance;
        out[i].weight = r->first.weight;
        for (int c = 0; c < 3; ++c) out[i].gradient[c] = r->first.gradient[c];
        if (probs)
            for (int k = 0; k < K; ++k) probs[i * K + k] = r->second.probs[k];
    }
    return 0;
}

uint64_t ref_take_dirty(void* h, int32_t which, int32_t* out, uint64_t cap) {
    RefMap* m = static_cast<RefMap*>(h);
    std::vector<BlockCoord> d;
    if (which == 0 && m->tsdf) d = m->tsdf->take_dirty_blocks();
    if (which == 1 && m->sem) d = m->sem->take_dirty_blocks();
    for (size_t i = 0; i < d.size() && i < cap; ++i) {
        out[3 * i] = d[i].x;
        out[3 * i + 1] = d[i].y;
        out[3 * i + 2] = d[i].z;
    }
    return d.size();
}

// extract_mesh (mesh.cpp:224-229); the mesh stays in the map for ref_mesh_read.
int ref_mesh_extract(void* h, float min_weight, int32_t reserved, uint64_t* nv, uint64_t* nf) {
    return guarded([&] {
        RefMap* m = static_cast<RefMap*>(h);
        const LabelSet ls = reserved_labels(reserved);
        m->mesh = extract_mesh(*m->store, min_weight, reserved >= 0 ? &ls : nullptr);
        *nv = m->mesh.vertices.size();
        *nf = m->mesh.faces.size();
    });
}

// IncrementalMesher::update (mesh.cpp:231-287) with a mesher kept in the map;
// remeshed (cap entries) receives last_remeshed(), *n_remeshed its size.
int ref_mesh_incremental(void* h, float min_weight, int32_t reserved, const int32_t* dirty,
                         uint64_t n, uint64_t* nv, uint64_t* nf, int32_t* remeshed, uint64_t cap,
                         uint64_t* n_remeshed) {
    return guarded([&] {
        RefMap* m = static_cast<RefMap*>(h);
        if (!m->mesher) {
            m->mesher_labels = reserved_labels(reserved);
            m->mesher = std::make_unique<IncrementalMesher>(
                min_weight, reserved >= 0 ? &m->mesher_labels : nullptr);
        }
        std::vector<BlockCoord> d(n);
        for (uint64_t i = 0; i < n; ++i) d[i] = {dirty[3 * i], dirty[3 * i + 1], dirty[3 * i + 2]};
        m->mesh = m->mesher->update(*m->store, d);
        *nv = m->mesh.vertices.size();
        *nf = m->mesh.faces.size();
        const auto& r = m->mesher->last_remeshed();
        *n_remeshed = r.size();
        for (size_t i = 0; i < r.size() && i < cap; ++i) {
            remeshed[3 * i] = r[i].x;
            remeshed[3 * i + 1] = r[i].y;
            remeshed[3 * i + 2] = r[i].z;
        }
    });
}

void ref_mesh_read(void* h, float* vertices, float* normals, uint8_t* labels, uint32_t* faces) {
    const LabeledMesh& mesh = static_cast<RefMap*>(h)->mesh;
    for (size_t i = 0; i < mesh.vertices.size(); ++i)
        for (int c = 0; c < 3; ++c) {
            if (vertices) vertices[3 * i + c] = mesh.vertices[i][c];
            if (normals) normals[3 * i + c] = mesh.vertex_normals[i][c];
        }
    if (labels && !mesh.vertex_labels.empty())
        std::memcpy(labels, mesh.vertex_labels.data(), mesh.vertex_labels.size());
    if (faces)
        for (size_t i = 0; i < mesh.faces.size(); ++i)
            for (int c = 0; c < 3; ++c) faces[3 * i + c] = mesh.faces[i][c];
}

}  // extern "C"
