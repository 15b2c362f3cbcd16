// C-ABI of the B200 semvox hot path (include/svx.h). Host code: validation,
// pool management, SVOX1 import/export, and orchestration of the kernels in
// svx_project.cu / svx_tsdf.cu / svx_semantic.cu / svx_store.cu. Errors are
// C++ exceptions internally and become svx_status + svx_last_error() here.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "svx_map.hpp"

namespace svx {

uint32_t get_or_alloc_block(svx_map* m, uint64_t key, bool* was_new);
uint32_t ensure_layer(svx_map* m, uint32_t idx);
void find_blocks(svx_map* m, const uint64_t* h_keys, uint32_t n, uint32_t* h_idx);

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

template <typename Fn>
svx_status guarded(Fn&& fn) {
    try {
        fn();
        return SVX_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SVX_DATA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SVX_DATA;
    }
}

void require(bool ok, svx_status s, const char* msg) {
    if (!ok) throw Error(s, msg);
}

void validate_cfg(const svx_map_cfg& c) {  // MapConfig::validate (types.hpp:103-111)
    require(c.voxel_size > 0.f, SVX_INVALID_ARGUMENT, "voxel_size must be > 0");
    require(c.truncation > 0.f, SVX_INVALID_ARGUMENT, "truncation must be > 0");
    require(!(c.truncation < c.voxel_size), SVX_INVALID_ARGUMENT, "truncation must be >= voxel_size");
    require(c.num_labels >= 1 && c.num_labels <= 64, SVX_INVALID_ARGUMENT,
            "num_labels must be in [1, 64]");
    require(c.max_blocks != 0, SVX_INVALID_ARGUMENT, "max_blocks must be > 0");
}

void validate_model(const svx_lidar_model& m) {  // ProjectionModel::validate (scan_projection.hpp:26-33)
    require(m.width > 0 && m.height_px > 0, SVX_INVALID_ARGUMENT, "projection model: empty image");
    require(!(std::abs(m.width * m.delta_phi - 2.0 * kPi) > 1e-6), SVX_INVALID_ARGUMENT,
            "projection model: width * delta_phi must equal 2*pi");
    require(m.delta_theta > 0.0, SVX_INVALID_ARGUMENT, "projection model: delta_theta must be > 0");
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SVX_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

uint64_t key_of(const int32_t b[3]) {
    require(key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2]), SVX_INVALID_ARGUMENT,
            "block coordinate outside the device key range [-2^20, 2^20)");
    return pack_key(b[0], b[1], b[2]);
}

template <typename T>
T* dmalloc(size_t n) {
    T* p = nullptr;
    SVX_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

void free_map(svx_map* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    if (m->stream) cudaStreamSynchronize(m->stream);
    for (void* p : {(void*)m->keys, (void*)m->vals, (void*)m->block_keys, (void*)m->sem_idx,
                    (void*)m->dirty, (void*)m->fbcnt, (void*)m->fbstart, (void*)m->fbfill, (void*)m->fbblocks, (void*)m->stamp, (void*)m->touched, (void*)m->fctr,
                    (void*)m->d_ctr})
        if (p) cudaFree(p);
    if (m->h_ctr) cudaFreeHost(m->h_ctr);
    if (m->h_fctr) cudaFreeHost(m->h_fctr);
    if (m->h_outs) cudaFreeHost(m->h_outs);
    if (m->h_xmeta) cudaFreeHost(m->h_xmeta);
    m->outs.release();
    m->bucket.release();
    m->bucket2.release();
    m->fb_tmp.release();
    m->fbdesc.release();
    m->xsend.release();
    m->xpack.release();
    m->xaux.release();
    m->xcnt.release();
    if (m->xstate && m->xstate_free) m->xstate_free(m->xstate);
    m->vlist.release();
    prof_resolve(m);
    for (cudaEvent_t e : m->prof_free) cudaEventDestroy(e);
    m->records.release();
    m->records_alt.release();
    m->sort_tmp.release();
    m->cand.release();
    m->lbl.release();
    m->conf.release();
    m->tensor.release();
    m->like_table.release();
    m->sem_out.release();
    m->q_keys.release();
    m->q_idx.release();
    m->mesh.release();
    if (m->mesh.host_stage) cudaFreeHost(m->mesh.host_stage);
    if (m->copy_stream) cudaStreamSynchronize(m->copy_stream);
    for (int i = 0; i < svx_map::kIngestSlots; ++i) {
        if (m->ingest_ready[i]) cudaEventDestroy(m->ingest_ready[i]);
        if (m->ingest_used[i]) cudaEventDestroy(m->ingest_used[i]);
        m->ingest[i].release();
    }
    for (cudaEvent_t e : m->label_events) cudaEventDestroy(e);
    if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
    if (m->stream && m->own_stream) cudaStreamDestroy(m->stream);
    delete m;
}

svx_map* create_map(const svx_map_cfg& cfg, int device) {
    validate_cfg(cfg);
    int ndev = 0;
    SVX_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, SVX_INVALID_ARGUMENT, "no such CUDA device");
    DeviceGuard g(device);
    svx_map* m = new svx_map();
    try {
        m->cfg = cfg;
        m->device = device;
        SVX_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
        uint64_t want = std::max<uint64_t>(2ull * cfg.max_blocks, 1024);
        m->log2cap = 0;
        while ((1ull << m->log2cap) < want) ++m->log2cap;
        // a fallback record holds a pool index in 22 bits (svx_tsdf.cu): max_blocks <= 2^22
        require(m->log2cap <= 23, SVX_INVALID_ARGUMENT, "max_blocks too large for the device hash (<= 2^22)");
        m->cap = uint32_t(1u << m->log2cap);
        m->keys = dmalloc<uint64_t>(m->cap);
        m->vals = dmalloc<uint32_t>(m->cap);
        m->stamp = dmalloc<uint32_t>(m->cap);
        m->touched = dmalloc<uint32_t>(m->cap);
        m->fctr = dmalloc<uint32_t>(kMaxG * kFC);
        m->block_keys = dmalloc<uint64_t>(cfg.max_blocks);
        m->sem_idx = dmalloc<uint32_t>(cfg.max_blocks);
        m->dirty = dmalloc<uint8_t>(2ull * cfg.max_blocks);
        m->fbcnt = dmalloc<uint32_t>(cfg.max_blocks);
        m->fbstart = dmalloc<uint32_t>(cfg.max_blocks);
        m->fbfill = dmalloc<uint32_t>(cfg.max_blocks);
        m->fbblocks = dmalloc<uint32_t>(cfg.max_blocks);
        m->d_ctr = dmalloc<uint32_t>(kNumCounters);
        // fallback records per group: sized by use (grown on overflow, the group retried);
        // the per-group sort covers the whole buffer
        uint32_t rec_cap = 1u << 16;
        // test hook: tiny buffers exercise the abort-and-resume paths
        if (const char* e = std::getenv("SVX_TEST_REC_CAP")) {
            rec_cap = uint32_t(std::max(1L, std::atol(e)));
            m->test_rec_cap = true;
        }
        if (const char* e = std::getenv("SVX_TEST_POOL_HEAD")) m->test_pool_head = uint64_t(std::max(1L, std::atol(e)));
        set_rec_cap(m, rec_cap);
        m->fb_global = m->fb_env = std::getenv("SVX_FB_GLOBAL") != nullptr;  // A/B: the global radix sort
        SVX_CUDA(cudaMallocHost(&m->h_ctr, sizeof(uint32_t) * kNumCounters));
        SVX_CUDA(cudaMallocHost(&m->h_fctr, sizeof(uint32_t) * kMaxG * kFC));
        std::memset(m->h_ctr, 0, sizeof(uint32_t) * kNumCounters);
        SVX_CUDA(cudaMemsetAsync(m->keys, 0xFF, 8ull * m->cap, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->vals, 0xFF, 4ull * m->cap, m->stream));  // kInvalid: no block yet
        SVX_CUDA(cudaMemsetAsync(m->stamp, 0, 4ull * m->cap, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fctr, 0, 4ull * kMaxG * kFC, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->sem_idx, 0xFF, 4ull * cfg.max_blocks, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->dirty, 0, 2ull * cfg.max_blocks, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fbcnt, 0, 4ull * cfg.max_blocks, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fbfill, 0, 4ull * cfg.max_blocks, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->d_ctr, 0, sizeof(uint32_t) * kNumCounters, m->stream));
        m->block_bytes = sizeof(svx_tsdf_voxel) * kBlockVoxels;
        m->layer_bytes = sizeof(float) * kBlockVoxels * size_t(cfg.num_labels);
        m->tsdf_pool.reserve(device, size_t(cfg.max_blocks) * m->block_bytes);
        m->mask_pool.reserve(device, size_t(cfg.max_blocks) * 4 * kMaskWords);
        m->sem_pool.reserve(device, size_t(cfg.max_blocks) * m->layer_bytes);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
    } catch (...) {
        free_map(m);
        throw;
    }
    return m;
}

// SVOX1 image (voxel_store.cpp:101-130) of the whole map.
std::vector<uint8_t> build_svox1(svx_map* m) {
    DeviceGuard g(m->device);
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    const uint64_t n = m->n_blocks;
    const int K = m->cfg.num_labels;
    std::vector<uint64_t> keys(n);
    std::vector<uint32_t> sid(n);
    std::vector<svx_tsdf_voxel> tsdf(n * kBlockVoxels);
    std::vector<float> sem(m->n_layers * uint64_t(kBlockVoxels) * K);
    if (n) {
        SVX_CUDA(cudaMemcpy(keys.data(), m->block_keys, 8 * n, cudaMemcpyDeviceToHost));
        SVX_CUDA(cudaMemcpy(sid.data(), m->sem_idx, 4 * n, cudaMemcpyDeviceToHost));
        SVX_CUDA(cudaMemcpy(tsdf.data(), tsdf_base(m), n * m->block_bytes, cudaMemcpyDeviceToHost));
    }
    if (!sem.empty())
        SVX_CUDA(cudaMemcpy(sem.data(), sem_base(m), sem.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return keys[a] < keys[b]; });
    uint64_t size = 5 + 4 + 4 + 4 + 8;
    for (uint64_t i = 0; i < n; ++i)
        size += 12 + m->block_bytes + 1 + (sid[i] != kInvalid ? m->layer_bytes : 0);
    std::vector<uint8_t> out(size);
    uint8_t* p = out.data();
    auto put = [&](const void* src, size_t len) {
        std::memcpy(p, src, len);
        p += len;
    };
    put("SVOX1", 5);
    put(&m->cfg.voxel_size, 4);
    put(&m->cfg.truncation, 4);
    const uint32_t k32 = uint32_t(K);
    put(&k32, 4);
    put(&n, 8);
    for (uint32_t i : order) {
        int32_t b[3];
        unpack_key(keys[i], b[0], b[1], b[2]);
        put(b, 12);
        put(&tsdf[uint64_t(i) * kBlockVoxels], m->block_bytes);
        const uint8_t hs = sid[i] != kInvalid ? 1 : 0;
        put(&hs, 1);
        if (hs) put(&sem[uint64_t(sid[i]) * kBlockVoxels * K], m->layer_bytes);
    }
    return out;
}

svx_map* load_svox1(const std::vector<uint8_t>& buf, int device, uint32_t max_blocks,
                    const std::string& origin) {
    size_t off = 0;
    auto get = [&](void* dst, size_t len) {
        if (off + len > buf.size()) throw Error(SVX_DATA, "truncated map snapshot");
        std::memcpy(dst, buf.data() + off, len);
        off += len;
    };
    char magic[5];
    if (buf.size() < 5 || std::memcmp(buf.data(), "SVOX1", 5) != 0)
        throw Error(SVX_DATA, "not a SVOX1 snapshot: " + origin);
    get(magic, 5);
    svx_map_cfg cfg{};
    get(&cfg.voxel_size, 4);
    get(&cfg.truncation, 4);
    uint32_t k32 = 0;
    get(&k32, 4);
    cfg.num_labels = int32_t(k32);
    cfg.max_blocks = max_blocks ? max_blocks : (1u << 20);  // MapConfig default, voxel_store.cpp:139
    uint64_t nb = 0;
    get(&nb, 8);
    svx_map* m = create_map(cfg, device);
    try {
        DeviceGuard g(device);
        const int K = cfg.num_labels;
        std::vector<uint64_t> keys;
        std::vector<uint32_t> sid;
        std::vector<svx_tsdf_voxel> tsdf;
        std::vector<float> sem;
        uint32_t layers = 0;
        // a repeated block coordinate is the SAME block (get_or_allocate_block,
        // voxel_store.cpp:145): its TSDF is overwritten by the later record, its
        // semantic layer by a later record that has one and kept otherwise; the
        // capacity check counts distinct blocks only
        std::unordered_map<uint64_t, uint32_t> seen;
        seen.reserve(size_t(std::min<uint64_t>(nb, cfg.max_blocks)) * 2);
        for (uint64_t i = 0; i < nb; ++i) {
            int32_t b[3];
            get(b, 12);
            const uint64_t key = key_of(b);
            auto it = seen.find(key);
            uint32_t at;
            if (it == seen.end()) {
                if (keys.size() >= cfg.max_blocks)
                    throw Error(SVX_CAPACITY, "block budget exhausted (max_blocks = " +
                                                  std::to_string(cfg.max_blocks) + ")");
                at = uint32_t(keys.size());
                seen.emplace(key, at);
                keys.push_back(key);
                tsdf.resize(tsdf.size() + kBlockVoxels);
                sid.push_back(kInvalid);
            } else {
                at = it->second;
            }
            get(&tsdf[uint64_t(at) * kBlockVoxels], m->block_bytes);
            uint8_t hs = 0;
            get(&hs, 1);
            if (hs) {
                if (sid[at] == kInvalid) {
                    sem.resize(sem.size() + size_t(kBlockVoxels) * K);
                    sid[at] = layers++;
                }
                if (off + m->layer_bytes > buf.size())
                    throw Error(SVX_DATA, "truncated semantic section: " + origin);
                get(&sem[uint64_t(sid[at]) * kBlockVoxels * K], m->layer_bytes);
            }
        }
        const uint64_t n = keys.size();
        ensure_blocks(m, n);
        ensure_layers(m, layers);
        if (n) {
            SVX_CUDA(cudaMemcpy(m->block_keys, keys.data(), 8 * n, cudaMemcpyHostToDevice));
            SVX_CUDA(cudaMemcpy(m->sem_idx, sid.data(), 4 * n, cudaMemcpyHostToDevice));
            SVX_CUDA(cudaMemcpy(tsdf_base(m), tsdf.data(), n * m->block_bytes, cudaMemcpyHostToDevice));
        }
        if (layers)
            SVX_CUDA(cudaMemcpy(sem_base(m), sem.data(), sem.size() * 4, cudaMemcpyHostToDevice));
        m->n_blocks = n;
        m->n_layers = layers;
        push_block_counters(m);
        rebuild_hash(m);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
    } catch (...) {
        free_map(m);
        throw;
    }
    return m;
}

}  // namespace

void set_last_error(const char* msg) { g_last_error = msg; }

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

Model make_model(const svx_lidar_model& lm) {
    Model m{};
    m.W = lm.width;
    m.H = lm.height_px;
    m.dphi = lm.delta_phi;
    m.dtheta = lm.delta_theta;
    m.theta0 = lm.theta0;
    m.min_range = lm.min_range;
    m.inv_dphi_f = float(1.0 / lm.delta_phi);
    m.inv_dtheta_f = float(1.0 / lm.delta_theta);
    m.theta0_f = float(lm.theta0);
    // FP32 pixel-coordinate error bound ("pixel decisions"): angle error of
    // fast_atan2f (<= 1.2e-7 + 2 ulp) + FP32 geometry (<= 2e-6 relative) is < 3e-6 rad;
    // budget 8e-6 rad, plus the relative rounding of the scaled coordinate.
    m.margin_u = float(8e-6 / lm.delta_phi + 5e-7 * lm.width + 1e-4);
    m.margin_v = float(8e-6 / lm.delta_theta + 5e-7 * lm.height_px + 1e-4);
    const double lo = lm.min_range * (1.0 - 1e-5), hi = lm.min_range * (1.0 + 1e-5);
    m.r2_lo = float(lo * lo);
    m.r2_hi = float(hi * hi);
    return m;
}

Pose to_pose(const svx_pose& p) {
    Pose T;
    std::memcpy(T.R, p.R, sizeof T.R);
    std::memcpy(T.t, p.t, sizeof T.t);
    return T;
}

// PosedCloud::validate_pose (scan_projection.hpp:65-69)
void validate_pose(const svx_pose& p) {
    double mx = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double rr = (p.R[i] * p.R[j] + p.R[3 + i] * p.R[3 + j]) + p.R[6 + i] * p.R[6 + j];
            const double e = std::abs(rr - (i == j ? 1.0 : 0.0));
            if (e > mx) mx = e;
        }
    require(!(mx > 1e-6), SVX_INVALID_ARGUMENT, "pose rotation is not orthonormal");
}

}  // namespace svx

using namespace svx;

extern "C" {

size_t svx_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        const size_t n = std::min(cap - 1, g_last_error.size());
        std::memcpy(buf, g_last_error.data(), n);
        buf[n] = 0;
    }
    return g_last_error.size();
}

const char* svx_status_name(svx_status s) {
    switch (s) {
        case SVX_OK: return "ok";
        case SVX_INVALID_ARGUMENT: return "invalid_argument";
        case SVX_CAPACITY: return "capacity";
        case SVX_DATA: return "data";
        case SVX_CUDA: return "cuda";
        case SVX_NOT_FOUND: return "not_found";
    }
    return "unknown";
}

uint64_t svx_kernel_launches(void) { return g_launches.load(); }

void svx_default_integrator_cfg(svx_integrator_cfg* c) {
    c->mode = SVX_NON_PROJECTIVE;
    c->truncation = 0.f;
    c->max_range = 70.0;
    c->alpha_epsilon = 1e-2;
    c->min_weight_clamp = 0.01f;
    c->drop_unreliable = 0;
}

void svx_default_semantic_cfg(svx_semantic_cfg* c) {
    c->use_bayes = 1;
    c->likelihood_floor = 1e-3f;
    c->default_confidence = 0.9f;
    c->occlusion = SVX_OCCLUSION_SURROGATE;
}

svx_status svx_lidar_spinning(int32_t width, int32_t height_px, double up, double down,
                              svx_lidar_model* out) {
    return guarded([&] {
        // ProjectionModel::spinning (scan_projection.cpp:9-19)
        svx_lidar_model m{};
        m.width = width;
        m.height_px = height_px;
        m.delta_phi = 2.0 * kPi / width;
        m.theta0 = (90.0 - up) * kPi / 180.0;
        m.delta_theta = (up + down) * kPi / 180.0 / height_px;
        m.scale_f = 256.0;
        m.offset_o = 0.0;
        m.min_range = 0.3;
        validate_model(m);
        *out = m;
    });
}

svx_status svx_map_create(const svx_map_cfg* cfg, int device, svx_map** out) {
    return guarded([&] {
        require(cfg && out, SVX_INVALID_ARGUMENT, "null argument");
        *out = create_map(*cfg, device);
    });
}

svx_status svx_map_destroy(svx_map* m) {
    return guarded([&] { free_map(m); });
}

svx_status svx_map_config(const svx_map* m, svx_map_cfg* out) {
    return guarded([&] { *out = m->cfg; });
}

svx_status svx_map_get_stream(svx_map* m, void** stream) {
    return guarded([&] { *stream = m->stream; });
}

svx_status svx_profile_enable(svx_map* m, int32_t on) {
    return guarded([&] {
        DeviceGuard g(m->device);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        prof_resolve(m);
        m->prof = on != 0;
        m->prof_mask = on == 1 ? 0xFFFFFFFFu : uint32_t(on);
        m->prof_acc = svx_profile{};
    });
}

svx_status svx_profile_read(svx_map* m, svx_profile* out) {
    return guarded([&] {
        DeviceGuard g(m->device);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        prof_resolve(m);
        *out = m->prof_acc;
    });
}

svx_status svx_map_set_shard(svx_map* m, int32_t rank, int32_t world) {
    return guarded([&] {
        require(world >= 1 && rank >= 0 && rank < world, SVX_INVALID_ARGUMENT, "bad shard");
        m->shard_rank = rank;
        m->shard_world = world;
    });
}

svx_status svx_map_reserve(svx_map* m, uint64_t blocks, uint64_t layers) {
    return guarded([&] {
        require(m != nullptr, SVX_INVALID_ARGUMENT, "null map");
        DeviceGuard g(m->device);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        ensure_blocks(m, std::max<uint64_t>(blocks, m->n_blocks), 0);
        ensure_layers(m, std::min<uint64_t>(layers, m->cfg.max_blocks));
    });
}

int32_t svx_block_owner(const int32_t b[3], int32_t world) {
    return owner_of(pack_key(b[0], b[1], b[2]), world);
}

svx_status svx_get_or_allocate_block(svx_map* m, const int32_t b[3], int32_t* was_new) {
    return guarded([&] {
        DeviceGuard g(m->device);
        bool nw = false;
        get_or_alloc_block(m, key_of(b), &nw);
        if (was_new) *was_new = nw;
    });
}

svx_status svx_has_block(svx_map* m, const int32_t b[3], int32_t* found) {
    return guarded([&] {
        DeviceGuard g(m->device);
        *found = 0;
        if (!(key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2]))) return;
        const uint64_t k = pack_key(b[0], b[1], b[2]);
        uint32_t idx = kInvalid;
        find_blocks(m, &k, 1, &idx);
        *found = idx != kInvalid;
    });
}

svx_status svx_has_blocks(svx_map* m, const int32_t* bxyz, uint64_t n, uint8_t* found) {
    return guarded([&] {
        require(m && (bxyz || !n) && (found || !n), SVX_INVALID_ARGUMENT, "null argument");
        require(n < (1ull << 31), SVX_INVALID_ARGUMENT, "too many blocks in one query");
        if (!n) return;
        DeviceGuard g(m->device);
        std::vector<uint64_t> keys(n);
        std::vector<uint8_t> in_range(n);
        for (uint64_t i = 0; i < n; ++i) {
            const int32_t* b = bxyz + 3 * i;
            in_range[i] = key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2]);
            keys[i] = in_range[i] ? pack_key(b[0], b[1], b[2]) : 0;
        }
        std::vector<uint32_t> idx(n);
        find_blocks(m, keys.data(), uint32_t(n), idx.data());
        for (uint64_t i = 0; i < n; ++i) found[i] = in_range[i] && idx[i] != kInvalid;
    });
}

svx_status svx_mesh_extract(svx_map* m, float min_weight, int32_t reserved, const int32_t* bxyz,
                            uint64_t n, uint64_t* n_vertices, uint64_t* n_faces) {
    return guarded([&] {
        require(m && n_vertices && n_faces && (bxyz || !n), SVX_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(m->device);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        if (!bxyz) {
            run_extract_mesh(m, min_weight, reserved, nullptr, 0, n_vertices, n_faces);
            return;
        }
        std::vector<uint64_t> keys;
        keys.reserve(n);
        for (uint64_t i = 0; i < n; ++i) {
            const int32_t* b = bxyz + 3 * i;
            if (key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2]))
                keys.push_back(pack_key(b[0], b[1], b[2]));
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        run_extract_mesh(m, min_weight, reserved, keys.data(), keys.size(), n_vertices, n_faces);
    });
}

// Mesh read-back: one D2H of every requested array into a pinned staging buffer
// (full copy-engine bandwidth), then a multi-threaded copy into the caller's
// (typically pageable) buffers. A pageable cudaMemcpy runs at single-thread memcpy
// speed and dominated the end-to-end extraction time.
svx_status svx_mesh_read(svx_map* m, float* vertices, float* normals, uint8_t* labels,
                         uint32_t* faces) {
    return guarded([&] {
        require(m != nullptr, SVX_INVALID_ARGUMENT, "null map");
        DeviceGuard g(m->device);
        MeshState& ms = m->mesh;
        const uint64_t V = ms.n_vertices, F = ms.n_faces;
        struct Part {
            void* dst;
            const void* src;
            uint64_t bytes;
        };
        std::vector<Part> parts;
        if (vertices && V) parts.push_back({vertices, ms.verts.p, 12 * V});
        if (normals && V) parts.push_back({normals, ms.normals.p, 12 * V});
        if (labels && V) parts.push_back({labels, ms.labels.p, V});
        if (faces && F) parts.push_back({faces, ms.faces.p, 12 * F});
        uint64_t total = 0;
        for (const Part& q : parts) total += (q.bytes + 255) & ~uint64_t(255);
        if (!total) return;
        if (ms.host_stage_bytes < total) {
            if (ms.host_stage) cudaFreeHost(ms.host_stage);
            ms.host_stage = nullptr;
            ms.host_stage_bytes = 0;
            SVX_CUDA(cudaMallocHost(&ms.host_stage, total + total / 4));
            ms.host_stage_bytes = total + total / 4;
        }
        uint8_t* stage = static_cast<uint8_t*>(ms.host_stage);
        std::vector<uint8_t*> at;
        uint64_t off = 0;
        for (const Part& q : parts) {
            at.push_back(stage + off);
            SVX_CUDA(cudaMemcpyAsync(stage + off, q.src, q.bytes, cudaMemcpyDeviceToHost, m->stream));
            off += (q.bytes + 255) & ~uint64_t(255);
        }
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        const uint64_t chunk = 1ull << 20;
        std::atomic<uint64_t> next{0};
        std::vector<std::pair<size_t, uint64_t>> work;  // (part, offset)
        for (size_t k = 0; k < parts.size(); ++k)
            for (uint64_t o = 0; o < parts[k].bytes; o += chunk) work.push_back({k, o});
        auto worker = [&] {
            for (uint64_t w; (w = next.fetch_add(1)) < work.size();) {
                const auto [k, o] = work[w];
                std::memcpy(static_cast<uint8_t*>(parts[k].dst) + o, at[k] + o,
                            std::min(chunk, parts[k].bytes - o));
            }
        };
        std::vector<std::thread> pool;
        for (unsigned i = 1; i < nt && i < work.size(); ++i) pool.emplace_back(worker);
        worker();
        for (std::thread& th : pool) th.join();
    });
}

svx_status svx_mesh_device(svx_map* m, const float** vertices, const float** normals,
                           const uint8_t** labels, const uint32_t** faces) {
    return guarded([&] {
        require(m != nullptr, SVX_INVALID_ARGUMENT, "null map");
        if (vertices) *vertices = m->mesh.verts.p;
        if (normals) *normals = m->mesh.normals.p;
        if (labels) *labels = m->mesh.labels.p;
        if (faces) *faces = m->mesh.faces.p;
    });
}

svx_status svx_block_count(svx_map* m, uint64_t* n) {
    return guarded([&] { *n = m->n_blocks; });
}

svx_status svx_block_keys_sorted(svx_map* m, int32_t* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        DeviceGuard g(m->device);
        *n = m->n_blocks;
        if (!out) return;
        std::vector<uint64_t> keys(m->n_blocks);
        if (!keys.empty())
            SVX_CUDA(cudaMemcpy(keys.data(), m->block_keys, 8 * keys.size(), cudaMemcpyDeviceToHost));
        std::sort(keys.begin(), keys.end());
        for (uint64_t i = 0; i < keys.size() && i < cap; ++i)
            unpack_key(keys[i], out[3 * i], out[3 * i + 1], out[3 * i + 2]);
    });
}

svx_status svx_block_read(svx_map* m, const int32_t b[3], svx_tsdf_voxel* tsdf, float* sem,
                          int32_t* has_sem) {
    return guarded([&] {
        DeviceGuard g(m->device);
        if (!(key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2])))
            throw Error(SVX_NOT_FOUND, "block not allocated");
        const uint64_t k = pack_key(b[0], b[1], b[2]);
        uint32_t idx = kInvalid;
        find_blocks(m, &k, 1, &idx);
        if (idx == kInvalid) throw Error(SVX_NOT_FOUND, "block not allocated");
        if (tsdf)
            SVX_CUDA(cudaMemcpy(tsdf, tsdf_base(m) + uint64_t(idx) * kBlockVoxels, m->block_bytes,
                                cudaMemcpyDeviceToHost));
        uint32_t sid = kInvalid;
        SVX_CUDA(cudaMemcpy(&sid, m->sem_idx + idx, 4, cudaMemcpyDeviceToHost));
        if (has_sem) *has_sem = sid != kInvalid;
        if (sem && sid != kInvalid)
            SVX_CUDA(cudaMemcpy(sem, sem_base(m) + uint64_t(sid) * kBlockVoxels * m->cfg.num_labels,
                                m->layer_bytes, cudaMemcpyDeviceToHost));
    });
}

svx_status svx_blocks_read(svx_map* m, const int32_t* bxyz, uint64_t n, svx_tsdf_voxel* tsdf,
                           float* sem, uint8_t* has_sem) {
    return guarded([&] {
        require(m && (bxyz || !n) && tsdf, SVX_INVALID_ARGUMENT, "null argument");
        require(!sem || has_sem, SVX_INVALID_ARGUMENT, "has_sem required with sem");
        require(n < (1ull << 31), SVX_INVALID_ARGUMENT, "too many blocks in one read");
        if (!n) return;
        DeviceGuard g(m->device);
        std::vector<uint64_t> keys(n);
        for (uint64_t i = 0; i < n; ++i) {
            const int32_t* b = bxyz + 3 * i;
            if (!(key_in_range(b[0]) && key_in_range(b[1]) && key_in_range(b[2])))
                throw Error(SVX_NOT_FOUND, "block not allocated");
            keys[i] = pack_key(b[0], b[1], b[2]);
        }
        std::vector<uint32_t> idx(n);
        find_blocks(m, keys.data(), uint32_t(n), idx.data());
        for (uint32_t i : idx)
            if (i == kInvalid) throw Error(SVX_NOT_FOUND, "block not allocated");
        const uint64_t nf = uint64_t(kBlockVoxels) * m->cfg.num_labels;
        DevBuf<uint32_t> di;
        DevBuf<svx_tsdf_voxel> dt;
        DevBuf<float> ds;
        DevBuf<uint8_t> dh;
        di.alloc(n);
        dt.alloc(n * kBlockVoxels);
        if (sem) {
            ds.alloc(n * nf);
            dh.alloc(n);
        }
        SVX_CUDA(cudaMemcpyAsync(di.p, idx.data(), 4 * n, cudaMemcpyHostToDevice, m->stream));
        gather_blocks(m, di.p, n, dt.p, sem ? ds.p : nullptr, sem ? dh.p : nullptr);
        SVX_CUDA(cudaMemcpyAsync(tsdf, dt.p, n * m->block_bytes, cudaMemcpyDeviceToHost, m->stream));
        if (sem) {
            SVX_CUDA(cudaMemcpyAsync(has_sem, dh.p, n, cudaMemcpyDeviceToHost, m->stream));
            SVX_CUDA(cudaMemcpyAsync(sem, ds.p, 4 * n * nf, cudaMemcpyDeviceToHost, m->stream));
        }
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        di.release();
        dt.release();
        ds.release();
        dh.release();
    });
}

svx_status svx_block_write(svx_map* m, const int32_t b[3], const svx_tsdf_voxel* tsdf,
                           const float* sem, int32_t has_sem) {
    return guarded([&] {
        DeviceGuard g(m->device);
        const uint32_t idx = get_or_alloc_block(m, key_of(b), nullptr);
        if (tsdf)
            SVX_CUDA(cudaMemcpy(tsdf_base(m) + uint64_t(idx) * kBlockVoxels, tsdf, m->block_bytes,
                                cudaMemcpyHostToDevice));
        if (has_sem) {
            const uint32_t sid = ensure_layer(m, idx);
            if (sem)
                SVX_CUDA(cudaMemcpy(sem_base(m) + uint64_t(sid) * kBlockVoxels * m->cfg.num_labels,
                                    sem, m->layer_bytes, cudaMemcpyHostToDevice));
        }
    });
}

svx_status svx_lookup(svx_map* m, const int32_t* v, uint64_t n, svx_tsdf_voxel* tsdf,
                      float* probs, uint8_t* found) {
    return guarded([&] {
        DeviceGuard g(m->device);
        if (!n) return;
        const int K = m->cfg.num_labels;
        DevBuf<int32_t> dv;
        DevBuf<svx_tsdf_voxel> dt;
        DevBuf<float> dp;
        DevBuf<uint8_t> df;
        dv.alloc(3 * n);
        dt.alloc(n);
        df.alloc(n);
        if (probs) dp.alloc(n * K);
        SVX_CUDA(cudaMemcpyAsync(dv.p, v, 12 * n, cudaMemcpyHostToDevice, m->stream));
        lookup_voxels(m, dv.p, n, dt.p, probs ? dp.p : nullptr, df.p);
        if (tsdf) SVX_CUDA(cudaMemcpyAsync(tsdf, dt.p, sizeof(svx_tsdf_voxel) * n, cudaMemcpyDeviceToHost, m->stream));
        if (probs) SVX_CUDA(cudaMemcpyAsync(probs, dp.p, 4 * n * K, cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaMemcpyAsync(found, df.p, n, cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        dv.release();
        dt.release();
        dp.release();
        df.release();
    });
}

svx_status svx_stats_get(svx_map* m, svx_stats* out) {
    return guarded([&] {
        DeviceGuard g(m->device);
        out->allocated_blocks = m->n_blocks;
        out->observed_voxels = count_observed(m);
        out->memory_bytes = m->tsdf_pool.mapped() + m->sem_pool.mapped() +
                            uint64_t(m->cap) * (8 + 4 + 4 + 4 + 128) +
                            uint64_t(m->cfg.max_blocks) * (8 + 4 + 2);
    });
}

svx_status svx_save(svx_map* m, const char* path) {
    return guarded([&] {
        const std::vector<uint8_t> img = build_svox1(m);
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Error(SVX_DATA, std::string("cannot open for writing: ") + path);
        os.write(reinterpret_cast<const char*>(img.data()), std::streamsize(img.size()));
        if (!os) throw Error(SVX_DATA, std::string("write failed: ") + path);
    });
}

svx_status svx_save_mem(svx_map* m, uint8_t* buf, uint64_t cap, uint64_t* size) {
    return guarded([&] {
        const std::vector<uint8_t> img = build_svox1(m);
        *size = img.size();
        if (buf) {
            require(cap >= img.size(), SVX_INVALID_ARGUMENT, "buffer too small");
            std::memcpy(buf, img.data(), img.size());
        }
    });
}

svx_status svx_load(const char* path, int device, uint32_t max_blocks, svx_map** out) {
    return guarded([&] {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw Error(SVX_DATA, std::string("cannot open: ") + path);
        std::vector<uint8_t> buf((std::istreambuf_iterator<char>(is)), {});
        *out = load_svox1(buf, device, max_blocks, path);
    });
}

svx_status svx_take_dirty_blocks(svx_map* m, int32_t which, int32_t* out, uint64_t cap,
                                 uint64_t* n) {
    return guarded([&] {
        DeviceGuard g(m->device);
        require(which == 0 || which == 1, SVX_INVALID_ARGUMENT, "which must be 0 or 1");
        const uint64_t nb = m->n_blocks;
        std::vector<uint8_t> flags(nb);
        std::vector<uint64_t> keys(nb);
        uint8_t* d = m->dirty + uint64_t(which) * m->cfg.max_blocks;
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        if (nb) {
            SVX_CUDA(cudaMemcpy(flags.data(), d, nb, cudaMemcpyDeviceToHost));
            SVX_CUDA(cudaMemcpy(keys.data(), m->block_keys, 8 * nb, cudaMemcpyDeviceToHost));
        }
        std::vector<uint64_t> sel;
        for (uint64_t i = 0; i < nb; ++i)
            if (flags[i]) sel.push_back(keys[i]);
        std::sort(sel.begin(), sel.end());
        *n = sel.size();
        if (!out) return;
        for (uint64_t i = 0; i < sel.size() && i < cap; ++i)
            unpack_key(sel[i], out[3 * i], out[3 * i + 1], out[3 * i + 2]);
        if (nb) SVX_CUDA(cudaMemset(d, 0, nb));
    });
}

svx_status svx_scan_create(svx_map* m, const svx_lidar_model* model, svx_scan** out) {
    return guarded([&] {
        require(m && model && out, SVX_INVALID_ARGUMENT, "null argument");
        validate_model(*model);
        const uint64_t P = uint64_t(model->width) * uint64_t(model->height_px);
        require(P <= (1ull << 23), SVX_INVALID_ARGUMENT, "scan image larger than 2^23 pixels");
        DeviceGuard g(m->device);
        svx_scan* s = new svx_scan();
        try {
            s->map = m;
            s->model = *model;
            s->dm = make_model(*model);
            s->P = int(P);
            // back_project directions with the host libm (scan_projection.cpp:78-84)
            std::vector<double> dirs(3 * P);
            for (int v = 0; v < model->height_px; ++v)
                for (int u = 0; u < model->width; ++u) {
                    const double az = kPi - (u + 0.5) * model->delta_phi;
                    const double polar = model->theta0 + (v + 0.5) * model->delta_theta;
                    const double sp = std::sin(polar);
                    const size_t i = size_t(v) * model->width + u;
                    dirs[3 * i] = sp * std::cos(az);
                    dirs[3 * i + 1] = sp * std::sin(az);
                    dirs[3 * i + 2] = std::cos(polar);
                }
            s->dirs.alloc(3 * P);
            SVX_CUDA(cudaMemcpy(s->dirs.p, dirs.data(), 8 * 3 * P, cudaMemcpyHostToDevice));
            s->VW = int((P + 31) / 32);
            ensure_scan_slots(s, 1, 0);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

svx_status svx_scan_destroy(svx_scan* s) {
    return guarded([&] {
        if (!s) return;
        DeviceGuard g(s->map->device);
        cudaStreamSynchronize(s->map->stream);
        s->dirs.release();
        s->depth.release();
        s->height.release();
        s->normals.release();
        s->valid.release();
        s->pixkey.release();
        s->lexkey.release();
        s->pixcache.release();
        s->rowdist.release();
        s->validbits.release();
        s->points64.release();
        s->tie.release();
        s->points.release();
        delete s;
    });
}

namespace {
// A standalone projection (slot 0): read its dropped count, clear the per-frame counters
// it used (a TSDF group resets them itself).
void finish_projection(svx_scan* s) {
    svx_map* m = s->map;
    uint32_t fc[kFC];
    SVX_CUDA(cudaMemcpyAsync(fc, m->fctr, sizeof fc, cudaMemcpyDeviceToHost, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fctr, 0, sizeof fc, m->stream));
    sync_counters(m);
    s->dropped = fc[FC_DROPPED];
}

const float* stage_points(svx_scan* s, const float* pts, uint64_t n, int32_t stride, int32_t is_dev) {
    require(stride >= 3, SVX_INVALID_ARGUMENT, "point stride must be >= 3");
    require(n < (1ull << 32), SVX_INVALID_ARGUMENT, "too many points in one cloud");
    if (is_dev || n == 0) return pts;
    s->points.alloc(n * stride);
    SVX_CUDA(cudaMemcpyAsync(s->points.p, pts, 4ull * n * stride, cudaMemcpyHostToDevice,
                             s->map->stream));
    return s->points.p;
}
}  // namespace

svx_status svx_project(svx_scan* s, const float* pts, uint64_t n, int32_t stride,
                       int32_t is_dev, const svx_pose* pose) {
    return guarded([&] {
        DeviceGuard g(s->map->device);
        validate_pose(*pose);
        const float* d = stage_points(s, pts, n, stride, is_dev);
        launch_project(s, d, n, stride, to_pose(*pose));
        finish_projection(s);
    });
}

svx_status svx_project_f64(svx_scan* s, const double* pts, uint64_t n, int32_t stride,
                           int32_t is_dev, const svx_pose* pose) {
    return guarded([&] {
        DeviceGuard g(s->map->device);
        validate_pose(*pose);
        require(stride >= 3, SVX_INVALID_ARGUMENT, "point stride must be >= 3");
        require(n < (1ull << 32), SVX_INVALID_ARGUMENT, "too many points in one cloud");
        const double* d = pts;
        if (!is_dev && n) {
            s->points64.alloc(n * stride);
            SVX_CUDA(cudaMemcpyAsync(s->points64.p, pts, 8ull * n * stride, cudaMemcpyHostToDevice,
                                     s->map->stream));
            d = s->points64.p;
        }
        launch_project(s, d, n, stride, to_pose(*pose));
        finish_projection(s);
    });
}

svx_status svx_compute_normals(svx_scan* s) {
    return guarded([&] {
        DeviceGuard g(s->map->device);
        launch_normals(s);
        SVX_CUDA(cudaStreamSynchronize(s->map->stream));
    });
}

svx_status svx_scan_upload(svx_scan* s, const float* depth, const float* height,
                           const float* normals, const uint8_t* valid) {
    return guarded([&] {
        DeviceGuard g(s->map->device);
        const size_t P = size_t(s->P);
        require(depth != nullptr, SVX_INVALID_ARGUMENT, "depth image required");
        s->last_slot = 0;
        SVX_CUDA(cudaMemcpy(s->depth.p, depth, 4 * P, cudaMemcpyHostToDevice));
        if (height) SVX_CUDA(cudaMemcpy(s->height.p, height, 4 * P, cudaMemcpyHostToDevice));
        s->has_normals = normals != nullptr;
        s->rowdist_fresh = false;
        if (normals) {
            require(valid != nullptr, SVX_INVALID_ARGUMENT, "normal_valid required with normals");
            SVX_CUDA(cudaMemcpy(s->normals.p, normals, 12 * P, cudaMemcpyHostToDevice));
            SVX_CUDA(cudaMemcpy(s->valid.p, valid, P, cudaMemcpyHostToDevice));
        }
    });
}

svx_status svx_scan_download(svx_scan* s, float* depth, float* height, float* normals,
                             uint8_t* valid, uint64_t* dropped, int32_t* has_normals) {
    return guarded([&] {
        DeviceGuard g(s->map->device);
        SVX_CUDA(cudaStreamSynchronize(s->map->stream));
        const size_t P = size_t(s->P), o = size_t(s->last_slot) * P;
        if (depth) SVX_CUDA(cudaMemcpy(depth, s->depth.p + o, 4 * P, cudaMemcpyDeviceToHost));
        if (height) SVX_CUDA(cudaMemcpy(height, s->height.p + o, 4 * P, cudaMemcpyDeviceToHost));
        if (normals) SVX_CUDA(cudaMemcpy(normals, s->normals.p + 3 * o, 12 * P, cudaMemcpyDeviceToHost));
        if (valid) SVX_CUDA(cudaMemcpy(valid, s->valid.p + o, P, cudaMemcpyDeviceToHost));
        if (dropped) *dropped = s->dropped;
        if (has_normals) *has_normals = s->has_normals;
    });
}

svx_status svx_integrate_scan(svx_map* m, svx_scan* s, const svx_pose* pose,
                              const svx_integrator_cfg* cfg, svx_frame_report* rep) {
    return guarded([&] {
        require(m && s && pose && cfg && rep, SVX_INVALID_ARGUMENT, "null argument");
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        const FrameJob job{s, to_pose(*pose), nullptr, 0, 3, false};
        run_frames(m, &job, 1, *cfg, rep);
        rep->elapsed_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

svx_status svx_integrate_cloud(svx_map* m, svx_scan* s, const float* pts, uint64_t n,
                               int32_t stride, int32_t is_dev, const svx_pose* pose,
                               const svx_integrator_cfg* cfg, svx_frame_report* rep) {
    return guarded([&] {
        require(m && s && pose && cfg && rep, SVX_INVALID_ARGUMENT, "null argument");
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        validate_pose(*pose);
        const float* d = stage_points(s, pts, n, stride, is_dev);
        const FrameJob job{s, to_pose(*pose), d, n, stride, true};
        run_frames(m, &job, 1, *cfg, rep);
        rep->elapsed_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

svx_status svx_integrate_clouds_device(svx_map* m, svx_scan* s, const float* d_points,
                                       const uint64_t* offsets, int32_t stride,
                                       const svx_pose* poses, int32_t n_frames,
                                       const svx_integrator_cfg* cfg, svx_frame_report* reports) {
    return guarded([&] {
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<FrameJob> jobs(size_t(std::max(n_frames, 0)));
        for (int32_t f = 0; f < n_frames; ++f) {
            validate_pose(poses[f]);
            require(offsets[f + 1] >= offsets[f], SVX_INVALID_ARGUMENT, "offsets must not decrease");
            jobs[f] = FrameJob{s, to_pose(poses[f]), d_points + offsets[f] * stride,
                               offsets[f + 1] - offsets[f], stride, true};
        }
        run_frames(m, jobs.data(), n_frames, *cfg, reports);
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        for (int32_t f = 0; f < n_frames; ++f) reports[f].elapsed_ms = ms / n_frames;
    });
}

svx_status svx_integrate_clouds(svx_map* m, svx_scan* s, const float* points, const uint64_t* offsets,
                                int32_t stride, const svx_pose* poses, int32_t n_frames,
                                const svx_integrator_cfg* cfg, svx_frame_report* reports) {
    return guarded([&] {
        require(m && s && cfg && reports && (points || n_frames <= 0), SVX_INVALID_ARGUMENT,
                "null argument");
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        require(stride >= 3, SVX_INVALID_ARGUMENT, "point stride must be >= 3");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<FrameJob> jobs(size_t(std::max(n_frames, 0)));
        for (int32_t f = 0; f < n_frames; ++f) {
            validate_pose(poses[f]);
            require(offsets[f + 1] >= offsets[f], SVX_INVALID_ARGUMENT, "offsets must not decrease");
            require(offsets[f + 1] - offsets[f] < (1ull << 32), SVX_INVALID_ARGUMENT,
                    "too many points in one cloud");
            jobs[f] = FrameJob{s, to_pose(poses[f]), points + offsets[f] * stride,
                               offsets[f + 1] - offsets[f], stride, true, true};
        }
        run_frames(m, jobs.data(), n_frames, *cfg, reports);
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        for (int32_t f = 0; f < n_frames; ++f) reports[f].elapsed_ms = ms / n_frames;
    });
}

svx_status svx_integrate_clouds_labels(svx_map* m, svx_scan* s, const float* points, const uint64_t* offsets,
                                       int32_t stride, int32_t points_on_device, const svx_pose* poses,
                                       int32_t n_frames, const svx_integrator_cfg* cfg, const svx_label_image* imgs,
                                       const int32_t* img_offsets, int32_t imgs_on_device,
                                       const svx_semantic_cfg* scfg, svx_frame_report* reports,
                                       svx_frame_report* label_reports) {
    return guarded([&] {
        require(m && s && cfg && scfg && reports && offsets && img_offsets && (points || n_frames <= 0),
                SVX_INVALID_ARGUMENT, "null argument");
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        require(stride >= 3, SVX_INVALID_ARGUMENT, "point stride must be >= 3");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        const int n_img = n_frames > 0 ? img_offsets[n_frames] : 0;
        require(n_frames <= 0 || img_offsets[0] == 0, SVX_INVALID_ARGUMENT, "img_offsets[0] must be 0");
        require(n_img == 0 || (imgs && label_reports), SVX_INVALID_ARGUMENT, "null label images");
        std::vector<FrameJob> jobs(size_t(std::max(n_frames, 0)));
        for (int32_t f = 0; f < n_frames; ++f) {
            validate_pose(poses[f]);
            require(offsets[f + 1] >= offsets[f] && img_offsets[f + 1] >= img_offsets[f], SVX_INVALID_ARGUMENT,
                    "offsets must not decrease");
            require(offsets[f + 1] - offsets[f] < (1ull << 32), SVX_INVALID_ARGUMENT, "too many points in one cloud");
            jobs[f] = FrameJob{s, to_pose(poses[f]), points + offsets[f] * stride, offsets[f + 1] - offsets[f],
                               stride, true, points_on_device == 0};
        }
        // a label pass that may throw (a confidence map, or an invalid default confidence)
        // must stop the sequence at its frame: those batches alternate frame by frame
        bool may_throw = scfg->default_confidence < 0.f || scfg->default_confidence > 1.f;
        for (int i = 0; i < n_img; ++i) may_throw |= imgs[i].confidence != nullptr;
        if (may_throw) {
            for (int32_t f = 0; f < n_frames; ++f) {
                run_frames(m, &jobs[size_t(f)], 1, *cfg, &reports[f]);
                const int a = img_offsets[f], b = img_offsets[f + 1];
                if (b > a) run_integrate_labels_batch(m, imgs + a, b - a, imgs_on_device != 0, *scfg, label_reports + a);
            }
        } else {
            // every block the batch can allocate lies below the mapped pool (the band aborts
            // otherwise): size the label passes' candidate list and layers for it
            const uint64_t head = std::max<uint64_t>(32768, uint64_t(2.0 * m->new_ema * n_frames));
            ensure_blocks(m, m->n_blocks + head, 4 * head);
            LabelBatch lb = labels_begin(m, imgs, n_img, imgs_on_device != 0, *scfg,
                                         std::max<uint64_t>(m->mapped_blocks, m->n_blocks + head));
            LabelHook hook{&lb, img_offsets};
            run_frames(m, jobs.data(), n_frames, *cfg, reports, &hook);
            labels_finish(m, lb, label_reports);
        }
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        for (int32_t f = 0; f < n_frames; ++f) reports[f].elapsed_ms = ms / n_frames;
    });
}

svx_status svx_integrate_clouds_xbegin(svx_map* m, svx_scan* s, const float* d_points, const uint64_t* offsets,
                                       int32_t stride, const svx_pose* poses, int32_t n_frames,
                                       const svx_integrator_cfg* cfg, uint64_t* send_meta, const void** d_send) {
    return guarded([&] {
        require(m && s && cfg && send_meta && d_send && poses && offsets, SVX_INVALID_ARGUMENT, "null argument");
        require(s->map == m, SVX_INVALID_ARGUMENT, "scan belongs to another map");
        require(stride >= 3, SVX_INVALID_ARGUMENT, "point stride must be >= 3");
        DeviceGuard g(m->device);
        std::vector<FrameJob> jobs(size_t(std::max(n_frames, 0)));
        for (int32_t f = 0; f < n_frames; ++f) {
            validate_pose(poses[f]);
            require(offsets[f + 1] >= offsets[f], SVX_INVALID_ARGUMENT, "offsets must not decrease");
            require(offsets[f + 1] - offsets[f] < (1ull << 32), SVX_INVALID_ARGUMENT, "too many points in one cloud");
            jobs[f] = FrameJob{s, to_pose(poses[f]), d_points + offsets[f] * stride, offsets[f + 1] - offsets[f],
                               stride, true};
        }
        run_group_xbegin(m, jobs.data(), n_frames, *cfg, send_meta, d_send);
    });
}

svx_status svx_integrate_clouds_xend(svx_map* m, const void* d_recv, const uint64_t* recv_meta,
                                     svx_frame_report* reports) {
    return guarded([&] {
        require(m && reports && recv_meta, SVX_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(m->device);
        run_group_xend(m, d_recv, recv_meta, reports);
    });
}

svx_status svx_integrate_labels(svx_map* m, const svx_label_image* img,
                                const svx_semantic_cfg* cfg, svx_frame_report* rep) {
    return guarded([&] {
        require(m && img && cfg && rep, SVX_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        run_integrate_labels(m, *img, *cfg, rep);
        rep->elapsed_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

svx_status svx_integrate_labels_batch(svx_map* m, const svx_label_image* imgs, int32_t n,
                                      int32_t ptr_is_device, const svx_semantic_cfg* cfg,
                                      svx_frame_report* reps) {
    return guarded([&] {
        require(m && cfg && reps && (imgs || n <= 0), SVX_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(m->device);
        const auto t0 = std::chrono::steady_clock::now();
        run_integrate_labels_batch(m, imgs, n, ptr_is_device != 0, *cfg, reps);
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        for (int32_t i = 0; i < n; ++i) reps[i].elapsed_ms = ms / n;
    });
}

}  // extern "C"
