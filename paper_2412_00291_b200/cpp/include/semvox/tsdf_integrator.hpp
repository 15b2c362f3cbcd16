// semvox drop-in (B200): TSDF integration with the reference's interface
// (proj/include/semvox/tsdf_integrator.hpp). integrate_frame runs the device
// pipeline (band raycast -> own-pixel measurement -> ordered fold, svx_tsdf.cu)
// through svx_integrate_scan; the scalar formulas below are the per-voxel
// definitions the kernels implement, kept on the host for callers and tests.
#pragma once

#include "semvox/scan_projection.hpp"
#include "semvox/types.hpp"
#include "semvox/voxel_store.hpp"

#include <cmath>
#include <limits>
#include <string>
#include <vector>

namespace semvox {

enum class DistanceMode { projective, non_projective };

struct IntegratorConfig {
    DistanceMode mode = DistanceMode::non_projective;
    float truncation = 0.f;  // <= 0: the map's truncation
    double max_range = 70.0;
    double alpha_epsilon = 1e-2;
    float min_weight_clamp = 0.01f;
    bool drop_unreliable = false;  // skip pixels without a valid normal
};

struct FrameReport {
    int frame = -1;
    size_t updated_voxels = 0;
    size_t new_blocks = 0;
    double elapsed_ms = 0.0;

    std::string json_line() const;
};

struct DistanceSample {
    double psi = 0.0;
    double theta = 0.0;
    double alpha = 0.0;
    double d = 0.0;
};

DistanceSample make_distance_sample(double psi, double theta, double alpha, double alpha_epsilon);
double projective_distance(const Vec3d& voxel_center, const Vec3d& sensor_origin,
                           const Vec3d& measured_point);
double nonprojective_distance(double psi, double theta, double alpha, double alpha_epsilon);
float observation_weight(double psi, double tau, float min_clamp);

inline float truncate_distance(double d, double tau) {
    if (d >= 0.0) return float(tau < d ? tau : d);
    return float(d < -tau ? -tau : d);
}

TsdfVoxel fuse_voxel(const TsdfVoxel& old, double d, float w_new, const Vec3f& n_measured, double tau);

// Voxels crossed by the segment [a, b], in order (amortised 3D DDA over cells
// centred on the voxel centres). Same visiting sequence as the device DDA.
template <typename Fn>
void traverse_segment(const Vec3d& a, const Vec3d& b, const MapConfig& cfg, Fn&& visit) {
    const double nu = double(cfg.voxel_size);
    VoxelCoord c = world_to_voxel(a, cfg);
    const VoxelCoord last = world_to_voxel(b, cfg);
    Vec3d dir = b - a;
    const double len = dir.norm();
    if (len < 1e-12) {
        visit(c);
        return;
    }
    dir /= len;
    int32_t* cc[3] = {&c.x, &c.y, &c.z};
    int32_t step[3];
    double next[3], inc[3];
    for (int k = 0; k < 3; ++k) {
        if (std::abs(dir[k]) < 1e-15) {
            step[k] = 0;
            next[k] = inc[k] = std::numeric_limits<double>::infinity();
            continue;
        }
        step[k] = dir[k] > 0 ? 1 : -1;
        next[k] = (nu * (*cc[k] + 0.5 * step[k]) - a[k]) / dir[k];
        inc[k] = nu / std::abs(dir[k]);
    }
    const size_t budget = size_t(3.0 * len / nu) + 8;
    for (size_t s = 0; s < budget; ++s) {
        visit(c);
        if (c == last) return;
        const int k = next[1] < next[0] ? (next[2] < next[1] ? 2 : 1) : (next[2] < next[0] ? 2 : 0);
        if (next[k] > len) return;
        *cc[k] += step[k];
        next[k] += inc[k];
    }
}

class TsdfIntegrator {
public:
    TsdfIntegrator(VoxelStore& store, const IntegratorConfig& cfg);

    FrameReport integrate_frame(const ScanImages& images, const Pose& pose);

    // B200 addition: project_cloud + compute_normal_image + integrate_frame in one
    // device pass (the per-frame body of cmd_integrate); the images never leave HBM.
    FrameReport integrate_cloud(const PosedCloud& cloud, const ProjectionModel& model);

    const IntegratorConfig& config() const { return cfg_; }

    std::vector<BlockCoord> take_dirty_blocks();

private:
    VoxelStore& store_;
    IntegratorConfig cfg_;
    int frame_counter_ = 0;  // the dirty set lives on the device (VoxelStore::take_dirty)
};

}  // namespace semvox
