// semvox drop-in (B200): OccupancyMap over the device occupancy map (svx_occ_*,
// svx_occ.cu). Header: semvox/occupancy_map.hpp.
#include "semvox/occupancy_map.hpp"

#include "svx.h"

#include <fstream>
#include <stdexcept>
#include <string>
#include <utility>

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
        case SVX_NOT_FOUND: throw std::out_of_range(msg);
        default: throw std::runtime_error(std::string("svx: ") + msg);
    }
}

svx_pose to_svx(const Pose& p) {
    svx_pose o;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) o.R[3 * r + c] = p.linear()(r, c);
        o.t[r] = p.translation()(r);
    }
    return o;
}

OccupancyReport from_svx(const svx_occ_report& r) {
    return OccupancyReport{r.frame, r.points, r.rays, r.hit_voxels, r.miss_voxels, r.new_blocks, r.elapsed_ms};
}

}  // namespace

OccupancyMap::OccupancyMap(const OccupancyConfig& cfg, int device) : cfg_(cfg) {
    svx_occ_cfg c;
    svx_default_occ_cfg(&c);
    c.voxel_size = float(cfg.voxel_size);
    c.num_labels = cfg.num_labels;
    c.max_blocks = cfg.max_blocks;
    c.l_hit = cfg.l_hit;
    c.l_miss = cfg.l_miss;
    c.l_min = cfg.l_min;
    c.l_max = cfg.l_max;
    c.min_range = cfg.min_range;
    c.max_range = cfg.max_range;
    c.carve = cfg.carve ? 1 : 0;
    check(svx_occ_create(&c, device, &occ_));
}

OccupancyMap::~OccupancyMap() {
    if (occ_) svx_occ_destroy(occ_);
}

OccupancyMap::OccupancyMap(OccupancyMap&& o) noexcept : cfg_(o.cfg_), occ_(std::exchange(o.occ_, nullptr)) {}

OccupancyMap& OccupancyMap::operator=(OccupancyMap&& o) noexcept {
    if (this != &o) {
        if (occ_) svx_occ_destroy(occ_);
        cfg_ = o.cfg_;
        occ_ = std::exchange(o.occ_, nullptr);
    }
    return *this;
}

OccupancyReport OccupancyMap::integrate(const PosedCloud& cloud, const std::vector<uint16_t>& labels,
                                        const std::vector<float>& confidence) {
    const size_t n = cloud.points.size();
    if (!labels.empty() && labels.size() != n) throw std::invalid_argument("labels: one per point");
    if (!confidence.empty() && confidence.size() != n) throw std::invalid_argument("confidence: one per point");
    std::vector<float> pts(3 * n);
    for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) pts[3 * i + k] = float(cloud.points[i][k]);
    const svx_pose pose = to_svx(cloud.pose);
    svx_occ_report r{};
    check(svx_occ_integrate(occ_, pts.data(), labels.empty() ? nullptr : labels.data(),
                            confidence.empty() ? nullptr : confidence.data(), n, 3, 0, &pose, &r));
    return from_svx(r);
}

std::vector<OccupancyReport> OccupancyMap::integrate_depth(const std::vector<DepthImage>& images) {
    std::vector<svx_pinhole> cams;
    std::vector<svx_pose> poses;
    std::vector<float> depth, conf;
    std::vector<uint16_t> labels;
    bool has_labels = false, has_conf = false;
    for (const DepthImage& im : images) {
        has_labels |= !im.labels.empty();
        has_conf |= !im.confidence.empty();
    }
    for (const DepthImage& im : images) {
        const size_t n = size_t(im.width > 0 ? im.width : 0) * size_t(im.height > 0 ? im.height : 0);
        if (im.depth.size() != n) throw std::invalid_argument("depth: width * height values");
        if (has_labels && im.labels.size() != n)
            throw std::invalid_argument("labels: all images or none, width * height each");
        if (has_conf && im.confidence.size() != n)
            throw std::invalid_argument("confidence: all images or none, width * height each");
        cams.push_back(svx_pinhole{im.width, im.height, im.fx, im.fy, im.cx, im.cy, im.max_depth});
        poses.push_back(to_svx(im.pose));
        depth.insert(depth.end(), im.depth.begin(), im.depth.end());
        if (has_labels) labels.insert(labels.end(), im.labels.begin(), im.labels.end());
        if (has_conf) conf.insert(conf.end(), im.confidence.begin(), im.confidence.end());
    }
    std::vector<svx_occ_report> reps(images.size());
    check(svx_occ_integrate_depth(occ_, depth.data(), has_labels ? labels.data() : nullptr,
                                  has_conf ? conf.data() : nullptr, cams.data(), poses.data(),
                                  int32_t(images.size()), 0, reps.data()));
    std::vector<OccupancyReport> out;
    out.reserve(reps.size());
    for (const svx_occ_report& r : reps) out.push_back(from_svx(r));
    return out;
}

OccupancyVoxel OccupancyMap::query(const VoxelCoord& v) const {
    const int32_t c[3] = {v.x, v.y, v.z};
    OccupancyVoxel o;
    uint8_t found = 0;
    check(svx_occ_lookup(occ_, c, 1, &o.log_odds, &o.hits, &o.misses, nullptr, &o.label, &found));
    o.found = found != 0;
    return o;
}

std::vector<uint32_t> OccupancyMap::histogram(const VoxelCoord& v) const {
    const int32_t c[3] = {v.x, v.y, v.z};
    std::vector<uint32_t> h(size_t(cfg_.num_labels));
    check(svx_occ_lookup(occ_, c, 1, nullptr, nullptr, nullptr, h.data(), nullptr, nullptr));
    return h;
}

size_t OccupancyMap::block_count() const {
    uint64_t n = 0;
    check(svx_occ_block_count(occ_, &n));
    return size_t(n);
}

std::vector<uint8_t> OccupancyMap::export_socc1() const {
    uint64_t size = 0;
    check(svx_occ_save_mem(occ_, nullptr, 0, &size));
    std::vector<uint8_t> buf(size);
    check(svx_occ_save_mem(occ_, buf.data(), size, &size));
    buf.resize(size);
    return buf;
}

void OccupancyMap::save(const std::string& path) const {
    const std::vector<uint8_t> buf = export_socc1();
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    f.write(reinterpret_cast<const char*>(buf.data()), std::streamsize(buf.size()));
    if (!f) throw std::runtime_error("write failed: " + path);
}

}  // namespace semvox
