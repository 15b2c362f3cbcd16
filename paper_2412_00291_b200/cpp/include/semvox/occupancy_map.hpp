// semvox drop-in (B200): C++ host API of the occupancy extension (include/svx.h
// "occupancy extension" and "pinhole depth images"): free-space carving, log-odds
// occupancy, hit/miss counters and integer class histograms for per-point labelled
// LiDAR and labelled pinhole depth images. The reference has no such component
// (SPEC.md:255 declines carving; BASELINE.json's north star asks for it), so this
// header is this project's own, in the reference's style (PosedCloud, Pose,
// VoxelCoord, the reference's exception classes); parity is unpinned and the C
// oracle (oracle/svx_oracle.c, svxo_occ_*) is its checker.
#pragma once

#include "semvox/scan_projection.hpp"
#include "semvox/types.hpp"

#include <cstdint>
#include <string>
#include <vector>

struct svx_occ;

namespace semvox {

struct OccupancyConfig {
    double voxel_size = 0.1;
    int num_labels = 20;            // K histogram classes, 1..64
    uint32_t max_blocks = 1u << 20;  // 8x8x8-voxel blocks
    float l_hit = 0.85f, l_miss = -0.4f, l_min = -2.0f, l_max = 3.5f;
    double min_range = 0.3, max_range = 70.0;
    bool carve = true;  // false: endpoints only
};

struct OccupancyReport {
    int frame = 0;
    uint64_t points = 0, rays = 0, hit_voxels = 0, miss_voxels = 0, new_blocks = 0;
    double elapsed_ms = 0.0;
};

// A labelled pinhole depth image (camera frame: x right, y down, z forward, the
// reference's LabelImage convention); depth in metres, 0 / non-finite = no return.
struct DepthImage {
    int width = 0, height = 0;
    std::vector<float> depth;            // [v][u]
    std::vector<uint16_t> labels;        // optional, [v][u]
    std::vector<float> confidence;       // optional, [v][u]
    double fx = 0, fy = 0, cx = 0, cy = 0;
    double max_depth = 30.0;
    Pose pose = Pose::Identity();        // camera -> world
};

struct OccupancyVoxel {
    bool found = false;   // false: the voxel's block was never allocated
    float log_odds = 0.f;
    uint32_t hits = 0, misses = 0;
    int32_t label = -1;   // first argmax of the class histogram, -1 when empty
};

class OccupancyMap {
public:
    explicit OccupancyMap(const OccupancyConfig& cfg = {}, int device = 0);
    ~OccupancyMap();
    OccupancyMap(const OccupancyMap&) = delete;
    OccupancyMap& operator=(const OccupancyMap&) = delete;
    OccupancyMap(OccupancyMap&& o) noexcept;
    OccupancyMap& operator=(OccupancyMap&& o) noexcept;

    // One scan; points are in the sensor frame and are converted to f32 (the KITTI
    // wire format). labels / confidence: one per point, or empty.
    OccupancyReport integrate(const PosedCloud& cloud, const std::vector<uint16_t>& labels = {},
                              const std::vector<float>& confidence = {});
    // Depth images, one scan each, in order.
    std::vector<OccupancyReport> integrate_depth(const std::vector<DepthImage>& images);

    OccupancyVoxel query(const VoxelCoord& v) const;
    std::vector<uint32_t> histogram(const VoxelCoord& v) const;  // K counts (q8 confidence sums)
    size_t block_count() const;
    std::vector<uint8_t> export_socc1() const;  // svx.h "SOCC1"
    void save(const std::string& path) const;
    const OccupancyConfig& config() const { return cfg_; }

private:
    OccupancyConfig cfg_;
    svx_occ* occ_ = nullptr;
};

}  // namespace semvox
