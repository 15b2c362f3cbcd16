// Host-side objects behind the C-ABI: svx_map (one voxel map on one device)
// and svx_scan (device ScanImages for one ProjectionModel).
//
// HBM layout of a map:
//   keys[cap] u64 / vals[cap] u32      open-addressing block hash (linear probing,
//                                      cap = pow2 >= 2*max_blocks), key = packed (x,y,z)
//   tsdf pool   [max_blocks][512] x 20 B  AoS TsdfVoxel, exactly the SVOX1 block body;
//                                      virtual range reserved once, physical memory
//                                      mapped on demand (CUDA VMM) so addresses are stable
//   sem pool    [layers][512][K] f32   lazily allocated semantic layers (VMM as above)
//   block_keys[idx], sem_idx[idx], dirty flags[idx]   per pool block
//   mask pool  [blocks][kMaskWords] u32  per-block visit masks of the current frame group
//                                      (VMM, parallel to the TSDF pool, 1152 B per block)
//   group scratch: stamp[cap] u32 (first touch per group), touched[cap] u32, fallback
//                  records (sorted per group), the per-frame visited-voxel lists
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "../../include/svx.h"
#include "svx_common.cuh"

namespace svx {

struct Error : std::runtime_error {
    svx_status status;
    Error(svx_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void cuda_check(cudaError_t e, const char* what);
#define SVX_CUDA(call) ::svx::cuda_check((call), #call)

// Growable device array with a stable base address (CUDA virtual memory
// management): reserve once, map physical chunks as the high-water mark grows.
// Mapping physical memory costs milliseconds per call, so growth can also run
// ahead of need on a helper thread (prefetch); kernels only ever touch the
// published mapped() prefix.
class VmmArray {
public:
    VmmArray() = default;
    ~VmmArray();
    VmmArray(const VmmArray&) = delete;
    VmmArray& operator=(const VmmArray&) = delete;

    void reserve(int device, size_t max_bytes);
    // Ensures [0, bytes) is mapped (waits for a pending prefetch). Never shrinks.
    void ensure(size_t bytes);
    // Starts mapping up to >= bytes in the background (no-op if already mapped or a
    // growth is in flight). The caller learns about it through mapped().
    void prefetch(size_t bytes);
    void* base() const { return reinterpret_cast<void*>(base_); }
    size_t mapped() const { return mapped_.load(std::memory_order_acquire); }

private:
    void grow(size_t bytes);  // maps [mapped_, >= bytes); caller holds no worker
    void join();
    int device_ = 0;
    CUdeviceptr base_ = 0;
    size_t reserved_ = 0, gran_ = 0;
    std::atomic<size_t> mapped_{0};
    std::thread worker_;
    std::atomic<bool> worker_done_{true};
    std::exception_ptr worker_err_;
    std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks_;
};

// Records the message svx_last_error() returns on this thread (svx_capi.cu).
void set_last_error(const char* msg);

// Runs fn, mapping exceptions to svx_status + svx_last_error (the C-ABI contract).
template <typename Fn>
svx_status api_guard(Fn&& fn) {
    try {
        fn();
        return SVX_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SVX_DATA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SVX_DATA;
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    // Grows geometrically (x1.5): regrowing frees the old buffer, and cudaFree
    // synchronises the device, so per-frame growth must stay rare.
    void alloc(size_t count) {
        if (count <= n) return;
        if (n) count = std::max(count, n + n / 2);
        if (p) cudaFree(p);
        p = nullptr;
        SVX_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// Device state of the last mesh extraction (svx_mesh.cu): scratch + output.
struct MeshState {
    DevBuf<uint64_t> keys;            // mesh blocks, sorted (2R: sort scratch)
    DevBuf<uint32_t> pidx;            // their pool indices (2R)
    DevBuf<uint32_t> rank_of_pool;    // [max_blocks] pool index -> mesh rank, kInvalid outside
    DevBuf<uint32_t> nb_pool, nb_rank;  // [R][27] neighbour blocks
    DevBuf<uint8_t> cases;            // [R][512] cell case bytes
    DevBuf<uint8_t> block_active;     // [R] block has a cell with geometry
    DevBuf<uint32_t> cellinfo;        // [R][512] local vertex offset | owned-edge mask << 12
    DevBuf<uint4> active;             // cells with geometry: rank, lin | case << 9, cellinfo, face offset
    DevBuf<unsigned long long> counts;  // per-block vertex/face counts and their scans
    DevBuf<float> verts, normals;     // 3V
    DevBuf<uint8_t> labels;           // V
    DevBuf<uint32_t> faces;           // 3F
    uint64_t n_vertices = 0, n_faces = 0;
    void* host_stage = nullptr;       // pinned read-back staging (svx_mesh_read)
    uint64_t host_stage_bytes = 0;
    void release() {
        keys.release(); pidx.release(); rank_of_pool.release(); nb_pool.release();
        nb_rank.release(); cases.release(); block_active.release(); cellinfo.release(); active.release(); counts.release();
        verts.release(); normals.release(); labels.release(); faces.release();
    }
};

}  // namespace svx

// Device ScanImages of up to `slots` frames of one ProjectionModel (one frame group,
// svx_tsdf.cu): frame slot g of an image array starts at g * P (normals at 3 g P, pixel
// cache at g P entries, valid bits at g * VW words).
struct svx_scan {
    svx_map* map = nullptr;
    svx_lidar_model model{};
    svx::Model dm{};
    int P = 0;
    int VW = 0;                   // valid-bit words per frame slot
    int slots = 0;                // frame slots allocated
    svx::DevBuf<double> dirs;     // P x 3 back_project directions (host libm, bit-exact)
    svx::DevBuf<float> depth;     // slots x P
    svx::DevBuf<float> height;    // slots x P
    svx::DevBuf<float> normals;   // slots x 3P (sensor frame)
    svx::DevBuf<uint8_t> valid;   // slots x P
    svx::DevBuf<unsigned long long> pixkey;  // slots x 2P: double-buffered (range bits << 32) | point index
    int parity[svx::kMaxG] = {};             // which pixkey half a slot's next projection uses
    svx::DevBuf<uint8_t> pixcache;           // slots x P x 48 B: ray, range, world normal, flags
    svx::DevBuf<uint8_t> rowdist;            // slots x P: row distance to the nearest empty pixel
    svx::DevBuf<uint32_t> validbits;         // slots x VW: pixel has a return (bit per pixel)
    bool rowdist_fresh = false;              // slot 0's rowdist matches its depth (user images)
    svx::DevBuf<unsigned long long> lexkey;  // slots x tie_cap: tie lists
    uint64_t tie_cap = 0;                    // tie-list entries per slot
    svx::DevBuf<uint8_t> tie;     // slots x P: possible exact-range tie
    svx::DevBuf<float> points;    // staging for host points
    svx::DevBuf<double> points64; // staging for host FP64 points
    int last_slot = 0;            // slot holding the most recent ScanImages
    bool has_normals = false;
    uint64_t dropped = 0;
    uint64_t n_points = 0;
};

struct svx_map {
    svx_map_cfg cfg{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    int32_t shard_rank = 0, shard_world = 1;

    // hash
    int log2cap = 0;
    uint32_t cap = 0;
    uint64_t* keys = nullptr;
    uint32_t* vals = nullptr;
    // pool
    svx::VmmArray tsdf_pool;   // svx_tsdf_voxel[blocks][512]
    svx::VmmArray sem_pool;    // float[layers][512*K]
    size_t block_bytes = 0, layer_bytes = 0;
    uint64_t* block_keys = nullptr;  // [max_blocks]
    uint32_t* sem_idx = nullptr;     // [max_blocks]
    uint8_t* dirty = nullptr;        // [2][max_blocks]
    // frame-group scratch (svx_tsdf.cu)
    uint32_t* stamp = nullptr;       // [cap] group serial of a slot's first touch
    uint32_t* touched = nullptr;     // [cap] slots touched by the current group
    svx::VmmArray mask_pool;         // [blocks][kMaskWords] u32 visit masks, parallel to the pool
    uint64_t mask_zeroed = 0;        // blocks of mask_pool zero-filled so far
    uint32_t* fctr = nullptr;        // [kMaxG][kFC] per-frame counters of the current group
    uint32_t* h_fctr = nullptr;      // pinned mirror (exchange mode)
    // fallback stage (voxels whose own pixel has no return in some frame): the group's visit
    // records (block, voxel, frame, pixel; the unused tail holds ~0, the sort's padding key),
    // their sorted copy, the radix sort's scratch, one descriptor per (voxel, frame) run
    svx::DevBuf<unsigned long long> records;
    svx::DevBuf<unsigned long long> records_alt;  // capacity path: visited block keys
    svx::DevBuf<uint8_t> sort_tmp;
    svx::DevBuf<unsigned long long> bucket, bucket2;  // the records, sorted (+ merge scratch)
    // per-block ordering (the default): per pool block its record count, bucket start and
    // fill cursor, and the list of blocks holding records ([max_blocks] each)
    uint32_t* fbcnt = nullptr;
    uint32_t* fbstart = nullptr;
    uint32_t* fbfill = nullptr;
    uint32_t* fbblocks = nullptr;
    bool fb_global = false;          // order the records with the global radix sort (next batch)
    bool fb_env = false;             // SVX_FB_GLOBAL=1: always (A/B)
    int fb_global_left = 0;          // batches left in the global ordering before a re-probe
    svx::DevBuf<uint8_t> fb_tmp;
    svx::DevBuf<uint4> fbdesc;       // fallback voxels: pool idx, voxel | frame << 16, records start, count
    uint32_t rec_cap = 0;            // fallback records per group (the sort's size)
    bool test_rec_cap = false;       // SVX_TEST_REC_CAP: fixed (tests of the overflow path)
    svx::DevBuf<uint32_t> vlist;     // per frame of the group: its visited voxels, (pool idx << 9) | voxel
    uint32_t vox_cap = 0;            // entries per frame
    // exchange mode (multi-GPU data plane, svx_tsdf.cu): per-destination send lists of
    // 16-byte visit entries, the packed send buffer, the received entries' ingest scratch
    svx::DevBuf<uint4> xsend, xpack, xaux;
    svx::DevBuf<uint32_t> xcnt;      // [world] entries per destination
    uint32_t xcap = 0;               // send-list entries per destination
    void* xstate = nullptr;          // the group between svx_integrate_clouds_xbegin and _xend
    void (*xstate_free)(void*) = nullptr;
    // per-frame results of a batch
    svx::DevBuf<svx::FrameOut> outs;
    svx::FrameOut* h_outs = nullptr;
    size_t h_outs_n = 0;
    uint32_t* h_xmeta = nullptr;     // pinned: exchange-mode send metadata (world x (1 + kMaxG))
    uint64_t mapped_blocks = 0;      // host mirror of C_MAPPED
    double new_ema = 0.0;            // moving average of new blocks per frame
    uint64_t test_pool_head = 0;     // test hook (SVX_TEST_POOL_HEAD): fixed pool headroom
    // host ingest ring (svx_integrate_clouds): the points of the next frame group are
    // copied on `copy_stream` while the current group integrates
    static constexpr int kIngestSlots = 2;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ingest_ready[kIngestSlots] = {}, ingest_used[kIngestSlots] = {};
    // host label images staged on copy_stream ahead of their label passes (one event per pass)
    std::vector<cudaEvent_t> label_events;
    svx::DevBuf<float> ingest[kIngestSlots];
    svx::DevBuf<uint64_t> q_keys;    // scratch of host block queries (find / insert)
    svx::DevBuf<uint32_t> q_idx;
    svx::DevBuf<uint32_t> cand;      // semantic candidate blocks
    svx::DevBuf<uint16_t> lbl;
    svx::DevBuf<float> conf, tensor;
    svx::DevBuf<float> like_table;   // [K+1][K] label -> likelihood at default confidence
    svx::DevBuf<uint32_t> sem_out;   // per image of a label batch: candidates, updated voxels
    svx::MeshState mesh;             // last extract_mesh result (svx_mesh.cu)
    // counters
    uint32_t* d_ctr = nullptr;       // device
    uint32_t* h_ctr = nullptr;       // pinned mirror
    uint32_t frame_serial = 0;
    int32_t tsdf_frames = 0, sem_frames = 0;
    uint64_t n_blocks = 0;           // host copy of C_BLOCKS after the last sync
    uint64_t n_layers = 0;
    // profiling: event pairs recorded around kernel groups on `stream`,
    // resolved at the next host synchronisation point
    bool prof = false;
    uint32_t prof_mask = 0;  // kernel groups (bit = SVX_K_*) timed with events
    svx_profile prof_acc{};
    struct PendingEv {
        int kid;
        cudaEvent_t a, b;
    };
    std::vector<PendingEv> prof_pending;
    std::vector<cudaEvent_t> prof_free;
};

namespace svx {

// Pool growth policy: keep at least `blocks` blocks of TSDF mapped.
// Maps at least `blocks` blocks now and starts mapping `ahead` more in the background.
void ensure_blocks(svx_map* m, uint64_t blocks, uint64_t ahead = 65536);
void ensure_layers(svx_map* m, uint64_t layers);
// Copies counters to the pinned mirror and synchronises the map stream.
void sync_counters(svx_map* m);
void count_launch(uint64_t n = 1);
// Profiling marks (no-ops unless svx_profile_enable(map, 1)).
struct ProfMark {
    svx_map* m;
    int kid;
    int launches;  // kernel launches the mark spans
    cudaEvent_t a = nullptr;
    ProfMark(svx_map* map, int k, int n_launches = 1);
    ~ProfMark();
};
void prof_resolve(svx_map* m);

// Launch with programmatic stream serialization (see pdl_wait in svx_common.cuh).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVX_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
    static const bool debug_sync = std::getenv("SVX_DEBUG_SYNC") != nullptr;
    if (debug_sync) {  // debugging aid: attribute a device fault to its kernel
        const cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) {
            const char* name = "?";
            cudaFuncGetName(&name, reinterpret_cast<const void*>(kernel));
            throw Error(SVX_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
        }
    }
}

inline svx_tsdf_voxel* tsdf_base(svx_map* m) {
    return static_cast<svx_tsdf_voxel*>(m->tsdf_pool.base());
}
inline float* sem_base(svx_map* m) { return static_cast<float*>(m->sem_pool.base()); }
inline HashView hash_view(svx_map* m) { return HashView{m->keys, m->vals, m->log2cap, m->cap - 1}; }
inline uint32_t* mask_base(svx_map* m) { return static_cast<uint32_t*>(m->mask_pool.base()); }

Model make_model(const svx_lidar_model& lm);
Pose to_pose(const svx_pose& p);
void validate_pose(const svx_pose& p);

// kernels' host launchers (svx_project.cu, svx_tsdf.cu, svx_semantic.cu, svx_store.cu)
// Projection of a frame group: frame g's points (device) go to scan slot g.
void launch_project_group(svx_scan* s, const void* const* d_pts, const uint64_t* n, int G, int stride,
                          bool fp64, const Pose* poses);
void launch_project(svx_scan* s, const float* d_pts, uint64_t n, int stride, const Pose& pose);
void launch_project(svx_scan* s, const double* d_pts, uint64_t n, int stride, const Pose& pose);
void launch_normals(svx_scan* s);
// Frame slots of a scan for groups of G frames of up to max_points points each.
void ensure_scan_slots(svx_scan* s, int G, uint64_t max_points);
// One TSDF frame: project (optional) + integrate_frame.
struct FrameJob {
    svx_scan* scan;
    Pose pose;
    const float* pts;  // device pointer (when project); HOST pointer when host_ingest
    uint64_t n;
    int stride;
    bool project;
    bool host_ingest = false;  // pts are in host memory: staged through the ingest ring
};
// Runs the frames in groups of up to kMaxG on the map stream, synchronising once at
// the end (plus once per abort + retry, rare). Fills one report per frame.
struct LabelBatch;
// Label images interleaved with a TSDF batch: the images [img_off[f], img_off[f + 1]) of
// frame f run right after frame f's fold (cmd_integrate's integrate_frame +
// integrate_labels, semvox_main.cpp:122-143).
struct LabelHook {
    LabelBatch* lb;
    const int* img_off;  // [n_frames + 1]
};
void run_frames(svx_map* m, const FrameJob* jobs, int n, const svx_integrator_cfg& cfg,
                svx_frame_report* reps, LabelHook* labels = nullptr);
// Exchange mode (multi-GPU data plane): one frame group in two halves around
// the caller's all-to-all. xbegin projects the group and casts this rank's share of its
// rays; visits of blocks other ranks own are returned packed by destination (16-byte
// entries, send_counts[world]). xend applies the entries received from all ranks and folds
// this rank's blocks.
void run_group_xbegin(svx_map* m, const FrameJob* jobs, int G, const svx_integrator_cfg& cfg,
                      uint64_t* send_meta, const void** d_send);
void run_group_xend(svx_map* m, const void* d_recv, const uint64_t* recv_meta, svx_frame_report* reps);
void reset_frame_state(svx_map* m);
// Fallback record capacity per frame group (buffers sized, padding key written).
void set_rec_cap(svx_map* m, uint32_t cap);
// Writes the host's block/layer/mapping counts into the device counters.
void push_block_counters(svx_map* m);
unsigned persistent_grid(int device);
void run_integrate_labels(svx_map* m, const svx_label_image& img, const svx_semantic_cfg& cfg,
                          svx_frame_report* rep);
void run_integrate_labels_batch(svx_map* m, const svx_label_image* imgs, int n, bool on_device,
                                const svx_semantic_cfg& cfg, svx_frame_report* reps);
// The same split in three (svx_semantic.cu): stage a batch, enqueue the label passes of
// images [i0, i1) without synchronising (TSDF frame groups interleave them with their
// folds), read the reports after the stream synchronised.
constexpr int kMaxLabelImages = 8;  // label images fused in one pass over the map
struct LabelBatch {
    const svx_label_image* imgs = nullptr;
    int n = 0;
    bool on_device = false;
    svx_semantic_cfg cfg{};
    int passes = 0, max_passes = 0;
    std::vector<int> pass_first, pass_count;
    uint64_t lo = 0, co = 0, to = 0;  // host staging offsets
    size_t events_used = 0;           // label_events of this batch
    std::vector<const uint16_t*> staged_lbl;  // per image: its staged device copy
    std::vector<const float*> staged_conf, staged_ten;
};
LabelBatch labels_begin(svx_map* m, const svx_label_image* imgs, int n, bool on_device,
                        const svx_semantic_cfg& cfg, uint64_t max_blocks_seen);
void labels_enqueue(svx_map* m, LabelBatch& lb, int i0, int i1, uint32_t group_frame);
void labels_finish(svx_map* m, const LabelBatch& lb, svx_frame_report* reps);
uint64_t count_observed(svx_map* m);
void launch_zero_blocks(svx_map* m, uint64_t first, uint64_t count);
void rebuild_hash(svx_map* m);
// Copies pool blocks d_idx[0..n) to d_out (n x 512 voxels); with d_sem, also their
// semantic layers (n x 512*K, has_sem[i] = 0 when block i has none).
void gather_blocks(svx_map* m, const uint32_t* d_idx, uint64_t n, svx_tsdf_voxel* d_out,
                   float* d_sem, uint8_t* d_has_sem);
// extract_mesh (mesh.cpp:105-287) over the sorted unique packed keys h_keys[0..n)
// (every allocated block when h_keys == nullptr); result in m->mesh.
void run_extract_mesh(svx_map* m, float min_weight, int reserved, const uint64_t* h_keys,
                      uint64_t n_keys, uint64_t* n_vertices, uint64_t* n_faces);
void lookup_voxels(svx_map* m, const int32_t* d_v, uint64_t n, svx_tsdf_voxel* d_out,
                   float* d_probs, uint8_t* d_found);

}  // namespace svx
