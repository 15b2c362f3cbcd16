// semvox drop-in (B200): the reference's C++ API over the C-ABI (include/svx.h).
//
// Hot path (device): project_cloud, compute_normal_image,
// TsdfIntegrator::integrate_frame / integrate_cloud,
// SemanticIntegrator::integrate_labels and the VoxelStore map of record.
// Host: the per-value formulas (project_point, back_project, fuse_voxel, ...),
// label-set files, and the block mirror described in voxel_store.hpp.
// Errors: svx_status -> the reference's exception classes (svx.h "Conventions").
#include "semvox/scan_projection.hpp"
#include "semvox/semantic_integrator.hpp"
#include "semvox/tsdf_integrator.hpp"
#include "semvox/voxel_store.hpp"

#include "svx.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <unordered_map>

namespace semvox {

namespace {

constexpr double kPi = std::numbers::pi;

[[noreturn]] void raise(svx_status s) {
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
inline void check(svx_status s) {
    if (s != SVX_OK) raise(s);
}

svx_pose to_svx(const Pose& p) {
    svx_pose o;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) o.R[3 * r + c] = p.linear()(r, c);
        o.t[r] = p.translation()(r);
    }
    return o;
}

svx_lidar_model to_svx(const ProjectionModel& m) {
    return svx_lidar_model{m.width,  m.height_px, m.delta_phi, m.delta_theta,
                           m.theta0, m.scale_f,   m.offset_o,  m.min_range};
}

bool same_model(const svx_lidar_model& a, const svx_lidar_model& b) {
    return a.width == b.width && a.height_px == b.height_px && a.delta_phi == b.delta_phi &&
           a.delta_theta == b.delta_theta && a.theta0 == b.theta0 && a.min_range == b.min_range;
}

const int32_t* key3(const BlockCoord& b) { return &b.x; }
static_assert(sizeof(BlockCoord) == 12 && offsetof(BlockCoord, z) == 8);
static_assert(sizeof(Vec3d) == 24 && sizeof(Vec3f) == 12);

// Device ScanImages of one map, one per projection model seen.
class ScanCache {
public:
    explicit ScanCache(svx_map* m) : map_(m) {}
    ~ScanCache() {
        for (auto& e : scans_) svx_scan_destroy(e.second);
    }
    svx_scan* get(const ProjectionModel& model) {
        const svx_lidar_model lm = to_svx(model);
        for (auto& e : scans_)
            if (same_model(e.first, lm)) return e.second;
        svx_scan* s = nullptr;
        check(svx_scan_create(map_, &lm, &s));
        scans_.emplace_back(lm, s);
        return s;
    }

private:
    svx_map* map_;
    std::vector<std::pair<svx_lidar_model, svx_scan*>> scans_;
};

// Device context of the store-less free functions (project_cloud,
// compute_normal_image): a one-block map on device 0 that only owns scans.
// Intentionally never destroyed (CUDA teardown order at exit).
struct FreeContext {
    std::mutex mu;
    svx_map* map = nullptr;
    std::unique_ptr<ScanCache> scans;
    FreeContext() {
        svx_map_cfg cfg{0.25f, 1.25f, 1, 1};
        check(svx_map_create(&cfg, 0, &map));
        scans = std::make_unique<ScanCache>(map);
    }
};
FreeContext& free_context() {
    static FreeContext* ctx = new FreeContext();
    return *ctx;
}

double elapsed_ms(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ===================================================================== types
LabelSet LabelSet::load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw DataError("cannot open labelset: " + path);
    LabelSet out;
    for (std::string line; std::getline(in, line);) {
        if (line.empty() || line.front() == '#') continue;
        std::istringstream fields(line);
        std::string name;
        int rgb[3];
        if (!(fields >> name >> rgb[0] >> rgb[1] >> rgb[2]))
            throw DataError("bad labelset line: \"" + line + "\" in " + path);
        out.names.push_back(std::move(name));
        out.colors.push_back(Rgb{uint8_t(rgb[0]), uint8_t(rgb[1]), uint8_t(rgb[2])});
    }
    if (out.names.empty()) throw DataError("empty labelset: " + path);
    return out;
}

void LabelSet::save(const std::string& path) const {
    std::ofstream out(path);
    if (!out) throw DataError("cannot open for writing: " + path);
    for (size_t i = 0; i < names.size(); ++i)
        out << names[i] << ' ' << unsigned(colors[i].r) << ' ' << unsigned(colors[i].g) << ' '
            << unsigned(colors[i].b) << '\n';
}

// ================================================================ VoxelStore
namespace {
struct Mirrored {
    std::unique_ptr<VoxelBlock> blk;
    std::array<TsdfVoxel, kBlockVoxels> synced_tsdf;  // bytes last exchanged with HBM
    std::vector<float> synced_sem;
    bool exposed = false;
};
}  // namespace

struct VoxelStore::Impl {
    MapConfig cfg;
    svx_map* map = nullptr;
    std::recursive_mutex mu;
    std::unordered_map<BlockCoord, Mirrored, SpatialHash> mirror;
    std::vector<BlockCoord> exposed;
    std::vector<BlockCoord> taken[2];  // device dirty lists consumed by refresh()
    std::unique_ptr<ScanCache> scans;

    ~Impl() {
        scans.reset();
        if (map) svx_map_destroy(map);
    }

    int K() const { return cfg.num_labels; }
    size_t layer_floats() const { return size_t(kBlockVoxels) * size_t(K()); }

    Mirrored& insert(const BlockCoord& bc, const TsdfVoxel* tsdf, const float* sem, bool has_sem) {
        Mirrored e;
        e.blk = std::make_unique<VoxelBlock>(bc);
        if (tsdf) std::memcpy(e.blk->tsdf.data(), tsdf, sizeof(e.blk->tsdf));
        if (has_sem) e.blk->semantics.assign(sem, sem + layer_floats());
        e.synced_tsdf = e.blk->tsdf;
        e.synced_sem = e.blk->semantics;
        return mirror.emplace(bc, std::move(e)).first->second;
    }

    // Block in the mirror, read from HBM on first use; nullptr when unallocated.
    Mirrored* materialize(const BlockCoord& bc) {
        auto it = mirror.find(bc);
        if (it != mirror.end()) return &it->second;
        std::array<TsdfVoxel, kBlockVoxels> tsdf;
        std::vector<float> sem(layer_floats());
        int32_t has_sem = 0;
        const svx_status s = svx_block_read(map, key3(bc), reinterpret_cast<svx_tsdf_voxel*>(tsdf.data()),
                                            sem.data(), &has_sem);
        if (s == SVX_NOT_FOUND) return nullptr;
        check(s);
        return &insert(bc, tsdf.data(), sem.data(), has_sem != 0);
    }

    void expose(const BlockCoord& bc, Mirrored& e) {
        if (e.exposed) return;
        e.exposed = true;
        exposed.push_back(bc);
    }

    // Reads blocks (all allocated) into their mirror entries, in batches.
    void read_into(const std::vector<BlockCoord>& keys) {
        constexpr size_t kBatch = 1024;
        std::vector<TsdfVoxel> tsdf;
        std::vector<float> sem;
        std::vector<uint8_t> has_sem;
        for (size_t lo = 0; lo < keys.size(); lo += kBatch) {
            const size_t n = std::min(kBatch, keys.size() - lo);
            tsdf.resize(n * kBlockVoxels);
            sem.resize(n * layer_floats());
            has_sem.assign(n, 0);
            check(svx_blocks_read(map, key3(keys[lo]), n, reinterpret_cast<svx_tsdf_voxel*>(tsdf.data()),
                                  sem.data(), has_sem.data()));
            for (size_t i = 0; i < n; ++i) {
                const TsdfVoxel* t = tsdf.data() + i * kBlockVoxels;
                const float* s = sem.data() + i * layer_floats();
                auto it = mirror.find(keys[lo + i]);
                if (it == mirror.end()) {
                    insert(keys[lo + i], t, s, has_sem[i] != 0);
                    continue;
                }
                Mirrored& e = it->second;
                std::memcpy(e.blk->tsdf.data(), t, sizeof(e.blk->tsdf));
                if (has_sem[i]) e.blk->semantics.assign(s, s + layer_floats());
                e.synced_tsdf = e.blk->tsdf;
                e.synced_sem = e.blk->semantics;
            }
        }
    }

    void flush() {
        for (const BlockCoord& bc : exposed) {
            Mirrored& e = mirror.at(bc);
            VoxelBlock& b = *e.blk;
            const bool tsdf_changed =
                std::memcmp(b.tsdf.data(), e.synced_tsdf.data(), sizeof(b.tsdf)) != 0;
            const bool sem_valid = b.semantics.size() == layer_floats();
            const bool sem_changed =
                sem_valid && (e.synced_sem.size() != b.semantics.size() ||
                              std::memcmp(b.semantics.data(), e.synced_sem.data(),
                                          4 * b.semantics.size()) != 0);
            if (!tsdf_changed && !sem_changed) continue;
            check(svx_block_write(map, key3(bc), reinterpret_cast<const svx_tsdf_voxel*>(b.tsdf.data()),
                                  sem_changed ? b.semantics.data() : nullptr, sem_changed ? 1 : 0));
            e.synced_tsdf = b.tsdf;
            if (sem_changed) e.synced_sem = b.semantics;
        }
    }

    std::vector<BlockCoord> device_dirty(int which) {
        uint64_t n = 0;
        check(svx_take_dirty_blocks(map, which, nullptr, 0, &n));
        std::vector<BlockCoord> out(n);
        if (n) check(svx_take_dirty_blocks(map, which, &out[0].x, n, &n));
        out.resize(n);
        return out;
    }

    void refresh(int which) {
        if (mirror.empty()) return;  // nothing mirrored: leave the dirty list on the device
        std::vector<BlockCoord> changed = device_dirty(which);
        std::vector<BlockCoord> mirrored;
        for (const BlockCoord& bc : changed)
            if (mirror.count(bc)) mirrored.push_back(bc);
        read_into(mirrored);
        auto& t = taken[which];
        t.insert(t.end(), changed.begin(), changed.end());
    }

    std::vector<BlockCoord> sorted_keys() {
        uint64_t n = 0;
        check(svx_block_keys_sorted(map, nullptr, 0, &n));
        std::vector<BlockCoord> keys(n);
        if (n) check(svx_block_keys_sorted(map, &keys[0].x, n, &n));
        keys.resize(n);
        return keys;
    }
};

namespace {
std::unique_ptr<VoxelStore::Impl> make_impl(svx_map* map) {
    auto impl = std::make_unique<VoxelStore::Impl>();
    impl->map = map;
    svx_map_cfg c{};
    check(svx_map_config(map, &c));
    impl->cfg = MapConfig{c.voxel_size, c.truncation, c.num_labels, c.max_blocks};
    impl->scans = std::make_unique<ScanCache>(map);
    return impl;
}
}  // namespace

VoxelStore::VoxelStore(const MapConfig& cfg, int device) {
    cfg.validate();
    const svx_map_cfg c{cfg.voxel_size, cfg.truncation, cfg.num_labels, cfg.max_blocks};
    svx_map* map = nullptr;
    check(svx_map_create(&c, device, &map));
    impl_ = make_impl(map);
}
VoxelStore::VoxelStore(std::unique_ptr<Impl> impl) : impl_(std::move(impl)) {}
VoxelStore::VoxelStore(VoxelStore&& other) noexcept : impl_(std::move(other.impl_)) {}
VoxelStore::~VoxelStore() = default;

const MapConfig& VoxelStore::config() const { return impl_->cfg; }
svx_map* VoxelStore::device_map() const { return impl_->map; }

VoxelBlock& VoxelStore::get_or_allocate_block(const BlockCoord& bc) {
    std::lock_guard lock(impl_->mu);
    auto it = impl_->mirror.find(bc);
    Mirrored* e = it != impl_->mirror.end() ? &it->second : nullptr;
    if (!e) {
        int32_t was_new = 0;
        check(svx_get_or_allocate_block(impl_->map, key3(bc), &was_new));
        e = was_new ? &impl_->insert(bc, nullptr, nullptr, false) : impl_->materialize(bc);
    }
    impl_->expose(bc, *e);
    return *e->blk;
}

VoxelBlock* VoxelStore::find_block(const BlockCoord& bc) {
    std::lock_guard lock(impl_->mu);
    Mirrored* e = impl_->materialize(bc);
    if (!e) return nullptr;
    impl_->expose(bc, *e);
    return e->blk.get();
}

const VoxelBlock* VoxelStore::find_block(const BlockCoord& bc) const {
    std::lock_guard lock(impl_->mu);
    Mirrored* e = impl_->materialize(bc);
    return e ? e->blk.get() : nullptr;
}

std::optional<std::pair<TsdfVoxel, SemanticVoxel>> VoxelStore::lookup_voxel(const VoxelCoord& v) const {
    std::lock_guard lock(impl_->mu);
    const Mirrored* e = impl_->materialize(block_of(v));
    if (!e) return std::nullopt;
    const VoxelBlock& b = *e->blk;
    const int li = local_index(v);
    const int K = impl_->K();
    SemanticVoxel sv;
    if (b.has_semantics())
        sv.probs.assign(b.probs_at(li, K), b.probs_at(li, K) + K);
    else
        sv = SemanticVoxel::uniform(K);
    return std::make_pair(b.tsdf[size_t(li)], std::move(sv));
}

const TsdfVoxel* VoxelStore::tsdf_at(const VoxelCoord& v) const {
    std::lock_guard lock(impl_->mu);
    const Mirrored* e = impl_->materialize(block_of(v));
    return e ? &e->blk->tsdf[size_t(local_index(v))] : nullptr;
}

StoreStats VoxelStore::stats() const {
    std::lock_guard lock(impl_->mu);
    impl_->flush();
    svx_stats s{};
    check(svx_stats_get(impl_->map, &s));
    return StoreStats{size_t(s.allocated_blocks), size_t(s.observed_voxels), size_t(s.memory_bytes)};
}

size_t VoxelStore::block_count() const {
    std::lock_guard lock(impl_->mu);
    uint64_t n = 0;
    check(svx_block_count(impl_->map, &n));
    return size_t(n);
}

std::vector<BlockCoord> VoxelStore::block_coords_sorted() const {
    std::lock_guard lock(impl_->mu);
    return impl_->sorted_keys();
}

std::vector<VoxelBlock*> VoxelStore::mirror_all(bool expose) const {
    std::lock_guard lock(impl_->mu);
    const std::vector<BlockCoord> keys = impl_->sorted_keys();
    std::vector<BlockCoord> missing;
    for (const BlockCoord& bc : keys)
        if (!impl_->mirror.count(bc)) missing.push_back(bc);
    impl_->read_into(missing);
    std::vector<VoxelBlock*> out;
    out.reserve(keys.size());
    for (const BlockCoord& bc : keys) {
        Mirrored& e = impl_->mirror.at(bc);
        if (expose) impl_->expose(bc, e);
        out.push_back(e.blk.get());
    }
    return out;
}

void VoxelStore::save(const std::string& path) const {
    std::lock_guard lock(impl_->mu);
    impl_->flush();
    check(svx_save(impl_->map, path.c_str()));
}

VoxelStore VoxelStore::load(const std::string& path, int device) {
    svx_map* map = nullptr;
    check(svx_load(path.c_str(), device, 0, &map));
    return VoxelStore(make_impl(map));
}

void VoxelStore::flush_host_writes() const {
    std::lock_guard lock(impl_->mu);
    impl_->flush();
}

void VoxelStore::refresh_after_device(int which) const {
    std::lock_guard lock(impl_->mu);
    impl_->refresh(which);
}

std::vector<BlockCoord> VoxelStore::take_dirty(int which) {
    std::lock_guard lock(impl_->mu);
    std::vector<BlockCoord> out = std::move(impl_->taken[which]);
    impl_->taken[which].clear();
    const std::vector<BlockCoord> rest = impl_->device_dirty(which);
    out.insert(out.end(), rest.begin(), rest.end());
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
}

size_t VoxelStore::mirrored_blocks() const {
    std::lock_guard lock(impl_->mu);
    return impl_->mirror.size();
}

// ============================================================ scan projection
ProjectionModel ProjectionModel::spinning(int width, int height_px, double fov_up_deg,
                                          double fov_down_deg) {
    svx_lidar_model lm{};
    check(svx_lidar_spinning(width, height_px, fov_up_deg, fov_down_deg, &lm));
    ProjectionModel m;
    m.width = lm.width;
    m.height_px = lm.height_px;
    m.delta_phi = lm.delta_phi;
    m.delta_theta = lm.delta_theta;
    m.theta0 = lm.theta0;
    m.validate();
    return m;
}

bool project_point(const Vec3d& p, const ProjectionModel& model, int& u, int& v, double& range) {
    range = p.norm();
    if (!std::isfinite(range) || range < model.min_range) return false;
    int col = int(std::floor((kPi - std::atan2(p.y(), p.x())) / model.delta_phi)) % model.width;
    if (col < 0) col += model.width;
    const double polar = std::acos(std::clamp(p.z() / range, -1.0, 1.0));
    const int row = int(std::floor((polar - model.theta0) / model.delta_theta));
    if (row < 0 || row >= model.height_px) return false;
    u = col;
    v = row;
    return true;
}

Vec3d back_project(int u, int v, double depth, const ProjectionModel& model) {
    if (!(depth > 0.0)) throw std::invalid_argument("back_project: depth must be > 0");
    const double az = kPi - (u + 0.5) * model.delta_phi;
    const double polar = model.theta0 + (v + 0.5) * model.delta_theta;
    const double sp = std::sin(polar);
    return depth * Vec3d(sp * std::cos(az), sp * std::sin(az), std::cos(polar));
}

ScanImages project_cloud(const PosedCloud& cloud, const ProjectionModel& model) {
    model.validate();
    cloud.validate_pose();
    FreeContext& ctx = free_context();
    std::lock_guard lock(ctx.mu);
    svx_scan* scan = ctx.scans->get(model);
    const svx_pose pose = to_svx(cloud.pose);
    check(svx_project_f64(scan, cloud.points.empty() ? nullptr : cloud.points[0].data(),
                          cloud.points.size(), 3, 0, &pose));
    ScanImages img;
    img.width = model.width;
    img.height_px = model.height_px;
    img.model = model;
    const size_t P = size_t(model.width) * size_t(model.height_px);
    img.depth.resize(P);
    img.height.resize(P);
    uint64_t dropped = 0;
    check(svx_scan_download(scan, img.depth.data(), img.height.data(), nullptr, nullptr, &dropped,
                            nullptr));
    img.dropped = size_t(dropped);
    return img;
}

void compute_normal_image(ScanImages& img, const ProjectionModel& model) {
    const size_t P = size_t(img.width) * size_t(img.height_px);
    if (img.width != model.width || img.height_px != model.height_px || img.depth.size() != P)
        throw std::invalid_argument("compute_normal_image: image does not match the model");
    FreeContext& ctx = free_context();
    std::lock_guard lock(ctx.mu);
    svx_scan* scan = ctx.scans->get(model);
    check(svx_scan_upload(scan, img.depth.data(), nullptr, nullptr, nullptr));
    check(svx_compute_normals(scan));
    img.normals.assign(P, Vec3f::Zero());
    img.normal_valid.assign(P, 0);
    check(svx_scan_download(scan, nullptr, nullptr, img.normals[0].data(), img.normal_valid.data(),
                            nullptr, nullptr));
}

// ============================================================ TSDF integrator
std::string FrameReport::json_line() const {
    char buf[192];
    std::snprintf(buf, sizeof(buf),
                  "{\"frame\":%d,\"updated_voxels\":%zu,\"new_blocks\":%zu,\"elapsed_ms\":%.3f}",
                  frame, updated_voxels, new_blocks, elapsed_ms);
    return std::string(buf);
}

double nonprojective_distance(double psi, double theta, double alpha, double alpha_epsilon) {
    const double ct = std::cos(theta);
    if (alpha < alpha_epsilon) return std::abs(ct) * psi;
    const double mag = std::abs((std::cos(alpha) - 1.0) * std::sin(theta) / std::sin(alpha)) +
                       std::abs(ct * psi);
    return psi >= 0.0 ? mag : -mag;
}

DistanceSample make_distance_sample(double psi, double theta, double alpha, double alpha_epsilon) {
    return DistanceSample{psi, theta, alpha, nonprojective_distance(psi, theta, alpha, alpha_epsilon)};
}

double projective_distance(const Vec3d& voxel_center, const Vec3d& sensor_origin,
                           const Vec3d& measured_point) {
    const Vec3d d = measured_point - sensor_origin;
    const double range = d.norm();
    if (!(range > 0.0)) throw std::invalid_argument("measured range must be > 0");
    return range - (voxel_center - sensor_origin).dot(d / range);
}

float observation_weight(double psi, double tau, float min_clamp) {
    return float(std::clamp((psi + tau) / (2.0 * tau), double(min_clamp), 1.0));
}

TsdfVoxel fuse_voxel(const TsdfVoxel& old, double d, float w_new, const Vec3f& n_measured, double tau) {
    if (w_new < 0.f) throw std::invalid_argument("fuse_voxel: negative weight");
    TsdfVoxel out = old;
    if (w_new == 0.f) return out;
    const float w = old.weight + w_new;
    out.distance = (old.weight * old.distance + w_new * truncate_distance(d, tau)) / w;
    out.weight = w;
    if (!(old.weight > 0.f)) {
        out.gradient = n_measured;
        return out;
    }
    const Vec3f g = old.weight * old.gradient + w_new * n_measured;
    const float len = g.norm();
    if (len > 1e-12f) out.gradient = g / len;
    return out;
}

namespace {
svx_integrator_cfg to_svx(const IntegratorConfig& c) {
    svx_integrator_cfg o;
    o.mode = c.mode == DistanceMode::projective ? SVX_PROJECTIVE : SVX_NON_PROJECTIVE;
    o.truncation = c.truncation;
    o.max_range = c.max_range;
    o.alpha_epsilon = c.alpha_epsilon;
    o.min_weight_clamp = c.min_weight_clamp;
    o.drop_unreliable = c.drop_unreliable ? 1 : 0;
    return o;
}
FrameReport from_svx(const svx_frame_report& r, int frame, double ms) {
    return FrameReport{frame, size_t(r.updated_voxels), size_t(r.new_blocks), ms};
}
}  // namespace

TsdfIntegrator::TsdfIntegrator(VoxelStore& store, const IntegratorConfig& cfg)
    : store_(store), cfg_(cfg) {
    if (cfg_.truncation <= 0.f) cfg_.truncation = store.config().truncation;
    if (!(cfg_.alpha_epsilon > 0.0)) throw std::invalid_argument("alpha_epsilon must be > 0");
}

FrameReport TsdfIntegrator::integrate_frame(const ScanImages& images, const Pose& pose) {
    const auto t0 = std::chrono::steady_clock::now();
    const int frame = frame_counter_++;
    if (cfg_.mode == DistanceMode::non_projective && !images.has_normals())
        throw std::invalid_argument("non-projective mode needs a normal image");
    const ProjectionModel& model = images.model;
    const size_t P = size_t(images.width) * size_t(images.height_px);
    if (images.width != model.width || images.height_px != model.height_px || images.depth.size() != P)
        throw std::invalid_argument("integrate_frame: images do not match their model");
    if (images.has_normals() && (images.normals.size() != P || images.normal_valid.size() != P))
        throw std::invalid_argument("integrate_frame: normal image size mismatch");
    VoxelStore::Impl& st = *store_.impl_;
    std::lock_guard lock(st.mu);
    st.flush();
    svx_scan* scan = st.scans->get(model);
    check(svx_scan_upload(scan, images.depth.data(), images.height.size() == P ? images.height.data() : nullptr,
                          images.has_normals() ? images.normals[0].data() : nullptr,
                          images.has_normals() ? images.normal_valid.data() : nullptr));
    const svx_pose sp = to_svx(pose);
    const svx_integrator_cfg c = to_svx(cfg_);
    svx_frame_report rep{};
    check(svx_integrate_scan(st.map, scan, &sp, &c, &rep));
    st.refresh(0);
    return from_svx(rep, frame, elapsed_ms(t0));
}

FrameReport TsdfIntegrator::integrate_cloud(const PosedCloud& cloud, const ProjectionModel& model) {
    const auto t0 = std::chrono::steady_clock::now();
    model.validate();
    cloud.validate_pose();
    const int frame = frame_counter_++;
    VoxelStore::Impl& st = *store_.impl_;
    std::lock_guard lock(st.mu);
    st.flush();
    svx_scan* scan = st.scans->get(model);
    const svx_pose sp = to_svx(cloud.pose);
    // projection leaves depth, height and normals in HBM for the integration pass
    check(svx_project_f64(scan, cloud.points.empty() ? nullptr : cloud.points[0].data(),
                          cloud.points.size(), 3, 0, &sp));
    const svx_integrator_cfg c = to_svx(cfg_);
    svx_frame_report rep{};
    check(svx_integrate_scan(st.map, scan, &sp, &c, &rep));
    st.refresh(0);
    return from_svx(rep, frame, elapsed_ms(t0));
}

std::vector<BlockCoord> TsdfIntegrator::take_dirty_blocks() { return store_.take_dirty(0); }

// ======================================================== semantic integrator
SemanticVoxel bayes_update(const SemanticVoxel& prior, std::span<const float> likelihood) {
    if (prior.probs.size() != likelihood.size())
        throw std::invalid_argument("bayes_update: size mismatch");
    SemanticVoxel post;
    post.probs.resize(likelihood.size());
    double z = 0.0;
    for (size_t k = 0; k < likelihood.size(); ++k) {
        post.probs[k] = prior.probs[k] * likelihood[k];
        z += post.probs[k];
    }
    for (float& p : post.probs) p = float(p / z);
    return post;
}

std::vector<float> label_to_likelihood(int label_id, float confidence, int num_labels, float floor) {
    if (confidence < 0.f || confidence > 1.f) throw std::invalid_argument("confidence must be in [0, 1]");
    const bool multi = num_labels > 1;
    std::vector<float> like(size_t(num_labels), multi ? (1.f - confidence) / float(num_labels - 1) : 1.f);
    if (label_id >= 0 && label_id < num_labels) like[size_t(label_id)] = multi ? confidence : 1.f;
    float sum = 0.f;
    for (float& x : like) {
        x = x < floor ? floor : x;
        sum += x;
    }
    for (float& x : like) x /= sum;
    return like;
}

SemanticIntegrator::SemanticIntegrator(VoxelStore& store, const SemanticConfig& cfg)
    : store_(store), cfg_(cfg) {}

FrameReport SemanticIntegrator::integrate_labels(const LabelImage& img) {
    const auto t0 = std::chrono::steady_clock::now();
    const int frame = frame_counter_++;
    if (img.width <= 0 || img.height <= 0) return FrameReport{frame, 0, 0, elapsed_ms(t0)};
    const size_t P = size_t(img.width) * size_t(img.height);
    const int K = store_.config().num_labels;
    if (img.labels.size() != P) throw std::invalid_argument("integrate_labels: label image size mismatch");
    if (!img.confidence.empty() && img.confidence.size() != P)
        throw std::invalid_argument("integrate_labels: confidence image size mismatch");
    svx_label_image li{};
    li.width = img.width;
    li.height = img.height;
    li.labels = img.labels.data();
    li.confidence = img.confidence.empty() ? nullptr : img.confidence.data();
    // a tensor of the wrong size is ignored, as in the reference
    li.prob_tensor = img.prob_tensor.size() == P * size_t(K) ? img.prob_tensor.data() : nullptr;
    li.fx = img.fx;
    li.fy = img.fy;
    li.cx = img.cx;
    li.cy = img.cy;
    li.pose = to_svx(img.pose);
    li.max_depth = img.max_depth;
    svx_semantic_cfg c{};
    c.use_bayes = cfg_.use_bayes ? 1 : 0;
    c.likelihood_floor = cfg_.likelihood_floor;
    c.default_confidence = cfg_.default_confidence;
    c.occlusion = cfg_.occlusion == OcclusionCheck::raycast ? SVX_OCCLUSION_RAYCAST : SVX_OCCLUSION_SURROGATE;
    VoxelStore::Impl& st = *store_.impl_;
    std::lock_guard lock(st.mu);
    st.flush();
    svx_frame_report rep{};
    check(svx_integrate_labels(st.map, &li, &c, &rep));
    st.refresh(1);
    return from_svx(rep, frame, elapsed_ms(t0));
}

std::vector<BlockCoord> SemanticIntegrator::take_dirty_blocks() { return store_.take_dirty(1); }

}  // namespace semvox
