/*
 * svx.h — C-ABI of the B200-native semvox voxel-integration hot path.
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, no
 * torch / Eigen / STL in any signature. The C++ mirror of the reference API
 * (the semvox headers under paper_2412_00291_b200/cpp/include) and the Python host mirror
 * (paper_2412_00291_b200/__init__.py) are thin layers over these entry points.
 * Every function names the reference interface it replaces (paths relative to
 * the reference repo, proj/...).
 *
 * Conventions
 *   - Every entry point returns svx_status. 0 = ok; otherwise the matching
 *     reference exception class (std::invalid_argument, CapacityError,
 *     DataError; proj/include/semvox/types.hpp:20-27) or a CUDA failure.
 *     svx_last_error() returns the message of the last failure on this thread.
 *   - Poses are double R[9] (row-major) + t[3], sensor->world (semvox::Pose,
 *     proj/include/semvox/types.hpp:16).
 *   - One map = one CUDA device + one stream. Calls on a map are serialised
 *     (the reference integrators are single-caller). Calls are
 *     synchronous unless the name ends in _async.
 *   - Host pointers are borrowed for the duration of the call.
 */
#ifndef SVX_H_
#define SVX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SVX_OK = 0,
    SVX_INVALID_ARGUMENT = 1, /* std::invalid_argument                          */
    SVX_CAPACITY = 2,         /* semvox::CapacityError (types.hpp:20-22)        */
    SVX_DATA = 3,             /* semvox::DataError (types.hpp:25-27)            */
    SVX_CUDA = 4,             /* CUDA / NCCL runtime failure (no reference analogue) */
    SVX_NOT_FOUND = 5         /* lookup of an unallocated block (find_block == nullptr) */
} svx_status;

/* semvox::MapConfig (proj/include/semvox/types.hpp:97-112); validated like
 * MapConfig::validate(). */
typedef struct {
    float voxel_size;
    float truncation;
    int32_t num_labels;
    uint32_t max_blocks;
} svx_map_cfg;

/* semvox::ProjectionModel (proj/include/semvox/scan_projection.hpp:16-38). */
typedef struct {
    int32_t width;
    int32_t height_px;
    double delta_phi;
    double delta_theta;
    double theta0;
    double scale_f;
    double offset_o;
    double min_range;
} svx_lidar_model;

/* semvox::Pose = Eigen::Isometry3d: R row-major, then translation. */
typedef struct {
    double R[9];
    double t[3];
} svx_pose;

/* semvox::IntegratorConfig (proj/include/semvox/tsdf_integrator.hpp:14-23). */
enum { SVX_PROJECTIVE = 0, SVX_NON_PROJECTIVE = 1 };
typedef struct {
    int32_t mode;            /* SVX_NON_PROJECTIVE by default */
    float truncation;        /* <= 0: use the map's truncation */
    double max_range;        /* 70 */
    double alpha_epsilon;    /* 1e-2 */
    float min_weight_clamp;  /* 0.01 */
    int32_t drop_unreliable; /* 0 */
} svx_integrator_cfg;

/* semvox::SemanticConfig (proj/include/semvox/semantic_integrator.hpp:31-38). */
enum { SVX_OCCLUSION_SURROGATE = 0, SVX_OCCLUSION_RAYCAST = 1 };
typedef struct {
    int32_t use_bayes;          /* 1 */
    float likelihood_floor;     /* 1e-3 */
    float default_confidence;   /* 0.9 */
    int32_t occlusion;          /* SVX_OCCLUSION_SURROGATE */
} svx_semantic_cfg;

/* semvox::FrameReport (proj/include/semvox/tsdf_integrator.hpp:25-32). */
typedef struct {
    int32_t frame;
    uint64_t updated_voxels;
    uint64_t new_blocks;
    double elapsed_ms;
} svx_frame_report;

/* semvox::LabelImage (proj/include/semvox/semantic_integrator.hpp:14-26).
 * confidence and prob_tensor may be NULL (absent). prob_tensor is [v][u][k]. */
typedef struct {
    int32_t width;
    int32_t height;
    const uint16_t* labels;
    const float* confidence;
    const float* prob_tensor;
    double fx, fy, cx, cy;
    svx_pose pose; /* camera -> world */
    double max_depth;
} svx_label_image;

/* semvox::StoreStats (proj/include/semvox/voxel_store.hpp:40-44). */
typedef struct {
    uint64_t allocated_blocks;
    uint64_t observed_voxels;
    uint64_t memory_bytes;
} svx_stats;

/* One voxel as stored (semvox::TsdfVoxel, types.hpp:115-121): 20 bytes. */
typedef struct {
    float distance;
    float weight;
    float gradient[3];
} svx_tsdf_voxel;

typedef struct svx_map svx_map;
typedef struct svx_scan svx_scan;

/* ------------------------------------------------------------------ errors */
/* Copies the last error message of this thread; returns its full length. */
size_t svx_last_error(char* buf, size_t cap);
const char* svx_status_name(svx_status s);
/* Number of hot-path kernel launches issued by this process so far (all maps). */
uint64_t svx_kernel_launches(void);

/* ------------------------------------------------------------- storage */
/* VoxelStore::VoxelStore(const MapConfig&) — voxel_store.hpp:51. */
svx_status svx_map_create(const svx_map_cfg* cfg, int device, svx_map** out);
svx_status svx_map_destroy(svx_map* map);
svx_status svx_map_config(const svx_map* map, svx_map_cfg* out);
/* The map's CUDA stream (cudaStream_t), for callers that time or order work
 * around svx calls (e.g. torch.cuda.ExternalStream). */
svx_status svx_map_get_stream(svx_map* map, void** stream);

/* VoxelStore::get_or_allocate_block — voxel_store.cpp:9-23. *was_new may be NULL. */
svx_status svx_get_or_allocate_block(svx_map* map, const int32_t bxyz[3], int32_t* was_new);
/* VoxelStore::find_block != nullptr — voxel_store.cpp:25-35. *found = 0/1. */
svx_status svx_has_block(svx_map* map, const int32_t bxyz[3], int32_t* found);
/* VoxelStore::block_count — voxel_store.hpp:76-79. */
svx_status svx_block_count(svx_map* map, uint64_t* n);
/* VoxelStore::block_coords_sorted — voxel_store.cpp:71-80. out = n*3 int32 (x,y,z),
 * sorted lexicographically. Pass out=NULL to query n. */
svx_status svx_block_keys_sorted(svx_map* map, int32_t* out, uint64_t cap, uint64_t* n);
/* Host mirror of one VoxelBlock (voxel_store.hpp:17-38): tsdf = 512 voxels
 * (10240 B), sem = 512*K floats (only when *has_sem). Returns SVX_NOT_FOUND for an
 * unallocated block. sem may be NULL. */
svx_status svx_block_read(svx_map* map, const int32_t bxyz[3], svx_tsdf_voxel* tsdf,
                          float* sem, int32_t* has_sem);
/* Batched svx_block_read for n blocks (bxyz = n*3): tsdf = n*512 voxels, sem (may be
 * NULL) = n*512*K floats, has_sem[i] = 0 for blocks without a semantic layer (their
 * sem rows are left untouched). SVX_NOT_FOUND if any block is unallocated. Used by
 * host mirrors that materialise many blocks at once (VoxelStore::for_each_block,
 * voxel_store.hpp:82-91). */
svx_status svx_blocks_read(svx_map* map, const int32_t* bxyz, uint64_t n, svx_tsdf_voxel* tsdf,
                           float* sem, uint8_t* has_sem);
/* Write-back of a host-mirrored block. has_sem=1 allocates the semantic layer if
 * needed and writes sem (VoxelBlock::ensure_semantics + direct mutation). */
svx_status svx_block_write(svx_map* map, const int32_t bxyz[3], const svx_tsdf_voxel* tsdf,
                           const float* sem, int32_t has_sem);
/* VoxelStore::lookup_voxel / tsdf_at — voxel_store.cpp:37-56. Batched: vxyz = n*3
 * voxel coords; found[i] = 0 when the block is absent. probs (n*K) may be NULL; a
 * block without a semantic layer yields the uniform distribution 1/K. */
svx_status svx_lookup(svx_map* map, const int32_t* vxyz, uint64_t n, svx_tsdf_voxel* tsdf,
                      float* probs, uint8_t* found);
/* VoxelStore::stats — voxel_store.cpp:58-69 (memory_bytes is the GPU footprint). */
svx_status svx_stats_get(svx_map* map, svx_stats* out);
/* VoxelStore::save / load (SVOX1) — voxel_store.cpp:101-168. Byte-identical to
 * the reference's snapshot of the same map. */
svx_status svx_save(svx_map* map, const char* path);
/* In-memory SVOX1 image; buf=NULL queries the size. */
svx_status svx_save_mem(svx_map* map, uint8_t* buf, uint64_t cap, uint64_t* size);
/* VoxelStore::load: creates a new map (max_blocks = cfg default 2^20 unless
 * max_blocks > 0 is given, mirroring voxel_store.cpp:139-152). */
svx_status svx_load(const char* path, int device, uint32_t max_blocks, svx_map** out);
/* TsdfIntegrator / SemanticIntegrator::take_dirty_blocks — tsdf_integrator.cpp:260-264,
 * semantic_integrator.cpp:167-171. which: 0 = TSDF pass, 1 = semantic pass.
 * Sorted, unique; the list is cleared. out=NULL queries n without clearing. */
svx_status svx_take_dirty_blocks(svx_map* map, int32_t which, int32_t* out, uint64_t cap,
                                 uint64_t* n);

/* --------------------------------------------------------- preprocessing */
/* ScanImages on the device for one ProjectionModel (scan_projection.hpp:44-58).
 * Validates the model like ProjectionModel::validate. The scan is bound to the
 * map's device and stream. */
svx_status svx_scan_create(svx_map* map, const svx_lidar_model* model, svx_scan** out);
svx_status svx_scan_destroy(svx_scan* scan);
/* project_cloud — scan_projection.cpp:39-76. points: n rows of `stride` floats
 * (3 = xyz, 4 = KITTI xyzi), sensor frame. ptr_is_device: points already in HBM.
 * Validates the pose (PosedCloud::validate_pose, scan_projection.hpp:65-69). */
svx_status svx_project(svx_scan* scan, const float* points, uint64_t n, int32_t stride,
                       int32_t ptr_is_device, const svx_pose* pose);
/* project_cloud for FP64 points (PosedCloud holds Eigen::Vector3d,
 * scan_projection.hpp:60-63): same semantics, n rows of `stride` doubles. */
svx_status svx_project_f64(svx_scan* scan, const double* points, uint64_t n, int32_t stride,
                           int32_t ptr_is_device, const svx_pose* pose);
/* compute_normal_image — scan_projection.cpp:86-109. */
svx_status svx_compute_normals(svx_scan* scan);
/* Upload host ScanImages (depth, and optionally normals n*3 + valid) — the
 * integrate_frame(const ScanImages&) entry when the caller built images on host. */
svx_status svx_scan_upload(svx_scan* scan, const float* depth, const float* height,
                           const float* normals, const uint8_t* normal_valid);
/* Download ScanImages; any output pointer may be NULL. */
svx_status svx_scan_download(svx_scan* scan, float* depth, float* height, float* normals,
                             uint8_t* normal_valid, uint64_t* dropped, int32_t* has_normals);

/* ------------------------------------------------------------ integration */
/* TsdfIntegrator::integrate_frame — tsdf_integrator.cpp:97-258 (band-limited
 * DDA, own-pixel rule, accumulate-then-merge fold). The frame counter lives in
 * the map (one TSDF integrator per map, as in cmd_integrate). */
svx_status svx_integrate_scan(svx_map* map, svx_scan* scan, const svx_pose* pose,
                              const svx_integrator_cfg* cfg, svx_frame_report* report);
/* project_cloud + compute_normal_image + integrate_frame for one posed cloud —
 * the per-frame body of cmd_integrate (semvox_main.cpp:122-124) in one call. */
svx_status svx_integrate_cloud(svx_map* map, svx_scan* scan, const float* points, uint64_t n,
                               int32_t stride, int32_t ptr_is_device, const svx_pose* pose,
                               const svx_integrator_cfg* cfg, svx_frame_report* report);
/* A sequence of posed clouds already resident in HBM: frame f uses points
 * [offsets[f], offsets[f+1]) and poses[f]. Frames are integrated in groups of up to
 * 16 (one launch sequence per group: results identical to one integrate_frame call per
 * frame); no host synchronisation inside the call unless a buffer or the pool must
 * grow; reports[f] filled at the end. */
svx_status svx_integrate_clouds_device(svx_map* map, svx_scan* scan, const float* d_points,
                                       const uint64_t* offsets, int32_t stride,
                                       const svx_pose* poses, int32_t n_frames,
                                       const svx_integrator_cfg* cfg, svx_frame_report* reports);
/* The same sequence with the points in HOST memory (pinned for full overlap): the
 * points of the next frame group are copied to the device on a copy stream while the
 * current group integrates — the per-frame body of cmd_integrate with its prefetcher
 * (semvox_main.cpp:30-76,121-124) in one call. */
svx_status svx_integrate_clouds(svx_map* map, svx_scan* scan, const float* points,
                                const uint64_t* offsets, int32_t stride, const svx_pose* poses,
                                int32_t n_frames, const svx_integrator_cfg* cfg,
                                svx_frame_report* reports);
/* cmd_integrate's per-frame body over a sequence (semvox_main.cpp:121-146):
 * project_cloud + compute_normal_image + integrate_frame of cloud f, then
 * integrate_labels of its label images imgs[img_offsets[f] .. img_offsets[f+1]) (one
 * SemanticIntegrator: frame numbers continue across the images). Clouds in device
 * memory (points_on_device) or pinned host memory; label images in device memory
 * (imgs_on_device) or host memory. Frames run in groups of up to 16 with each frame's
 * label pass right after its fold, so the result equals the per-frame calls; a batch whose
 * label images may throw (confidence maps, or an invalid default confidence) alternates
 * frame by frame instead. reports[n_frames], label_reports[img_offsets[n_frames]]. */
svx_status svx_integrate_clouds_labels(svx_map* map, svx_scan* scan, const float* points,
                                       const uint64_t* offsets, int32_t stride,
                                       int32_t points_on_device, const svx_pose* poses,
                                       int32_t n_frames, const svx_integrator_cfg* cfg,
                                       const svx_label_image* imgs, const int32_t* img_offsets,
                                       int32_t imgs_on_device, const svx_semantic_cfg* scfg,
                                       svx_frame_report* reports, svx_frame_report* label_reports);
/* Multi-GPU data plane (exchange mode, SURVEY.md 8(e) "ray-partitioned DDA + one
 * all-to-all visit exchange"; no reference analogue: the reference is single-process).
 * On a key-sharded map (svx_map_set_shard, world >= 2) one group of n_frames <= 16
 * clouds (device pointers; every rank passes the same clouds) is integrated in two calls
 * around the caller's all-to-all (NCCL):
 *   xbegin  projects the group and casts this rank's share of the rays (round robin over
 *           pixel tiles); visits of blocks another rank owns are returned as 16-byte
 *           entries packed by destination rank (*d_send: a device buffer valid until the
 *           next xbegin). send_meta[world][17]: per destination, the number of entries,
 *           then per frame of the group the number of voxel bits sent (sizes the
 *           receiver's lists without a synchronisation).
 *   xend    applies the entries received from all ranks (d_recv, device memory, in source
 *           rank order; recv_meta[world][17] = what each source's send_meta held for this
 *           rank) and folds this rank's blocks; reports[f] hold this rank's share
 *           (updated_voxels / new_blocks summed over ranks = the unsharded values).
 * The union of the ranks' maps equals the map one rank builds alone, byte for byte. */
svx_status svx_integrate_clouds_xbegin(svx_map* map, svx_scan* scan, const float* d_points,
                                       const uint64_t* offsets, int32_t stride,
                                       const svx_pose* poses, int32_t n_frames,
                                       const svx_integrator_cfg* cfg, uint64_t* send_meta,
                                       const void** d_send);
svx_status svx_integrate_clouds_xend(svx_map* map, const void* d_recv,
                                     const uint64_t* recv_meta, svx_frame_report* reports);
/* SemanticIntegrator::integrate_labels — semantic_integrator.cpp:91-165, with
 * exact block-level frustum culling (results identical to the O(map) sweep). */
svx_status svx_integrate_labels(svx_map* map, const svx_label_image* img,
                                const svx_semantic_cfg* cfg, svx_frame_report* report);

/* n label images applied in order (as n integrate_labels calls) with one
 * synchronisation: labels / confidence / prob_tensor of every image are read from
 * DEVICE memory when ptr_is_device, else copied from the host asynchronously.
 * An invalid confidence stops the batch with SVX_INVALID_ARGUMENT. */
svx_status svx_integrate_labels_batch(svx_map* map, const svx_label_image* imgs, int32_t n,
                                      int32_t ptr_is_device, const svx_semantic_cfg* cfg,
                                      svx_frame_report* reports);

/* ------------------------------------------------------------------ mesh */
/* extract_mesh / IncrementalMesher::update's re-mesh — proj/src/mesh.cpp:105-287.
 * Marching cubes over every cell whose base corner lies in one of the given blocks
 * (bxyz = n*3 block coords; bxyz = NULL meshes every allocated block, as
 * extract_mesh does). Blocks absent from the map are skipped; duplicates are
 * ignored. Corners are read from any allocated block. A cell is meshed when its 8
 * corners have !(weight < min_weight). reserved_unlabeled: the class id of a
 * trailing "unlabeled" class (its vertices get label 255), or -1. Output order and
 * values are those of the reference's stitched mesh: vertices in first-appearance
 * order, faces (i0, i2, i1) per table triangle. The mesh stays on the device until
 * the next extraction (svx_mesh_read / svx_mesh_device). */
svx_status svx_mesh_extract(svx_map* map, float min_weight, int32_t reserved_unlabeled,
                            const int32_t* bxyz, uint64_t n, uint64_t* n_vertices,
                            uint64_t* n_faces);
/* Copies the last extracted mesh to host buffers; any pointer may be NULL.
 * vertices / normals: 3V floats (LabeledMesh::vertices / vertex_normals), labels: V
 * bytes (255 = kUnlabeled), faces: 3F uint32. */
svx_status svx_mesh_read(svx_map* map, float* vertices, float* normals, uint8_t* labels,
                         uint32_t* faces);
/* Device pointers of the last extracted mesh (valid until the next extraction or
 * svx_map_destroy), for consumers that stay on the GPU. */
svx_status svx_mesh_device(svx_map* map, const float** vertices, const float** normals,
                           const uint8_t** labels, const uint32_t** faces);
/* VoxelStore::find_block != nullptr for n blocks at once (bxyz = n*3): found[i] = 0/1. */
svx_status svx_has_blocks(svx_map* map, const int32_t* bxyz, uint64_t n, uint8_t* found);

/* ------------------------------------------------- occupancy extension */
/* Free-space carving + log-odds occupancy + hit/miss counters + integer class
 * histograms for per-point labelled LiDAR: the north-star extension of BASELINE.json
 * (SURVEY.md 8(f) row 3). The reference declines carving, so there is
 * no reference implementation: the contract below is this project's own and the
 * oracle (oracle/svx_oracle.c, svxo_occ_*) restates it serially ("parity unpinned").
 *
 * Per scan, for every point p (sensor frame) with finite coordinates and
 * r = |p| >= min_range (Eigen order, FP64):
 *   q = pose * p; o = pose.t; if r <= max_range the ray HITS the voxel of q and its
 *   end is q, else it is cut at max_range (end = o + (q - o) * (max_range / r), no hit).
 *   carve: every voxel traverse_segment(o, end) visits (tsdf_integrator.hpp:93-135)
 *   is a MISS, except the hit voxel. Per scan a voxel is updated once: HIT if any ray
 *   hit it, else MISS if any ray traversed it (order-independent by construction).
 *   Update (f32): HIT: L = min(L + l_hit, l_max), hits += 1;
 *                 MISS: L = max(L + l_miss, l_min), misses += 1.   (L starts at 0)
 *   Labels: a hitting point with label l < K adds q8(conf) to hist[voxel][l], an
 *   integer (u32 atomics, exact in any order); q8(c) = (uint32)(clamp(c,0,1)*255 + 0.5f),
 *   255 without a confidence, 0 for a non-finite one. Label = first argmax of the
 *   histogram, -1 when it is all zero. */
typedef struct {
    float voxel_size;      /* metres */
    int32_t num_labels;    /* K histogram classes, 1..64 */
    uint32_t max_blocks;   /* 8x8x8-voxel blocks */
    float l_hit;           /* 0.85  (OctoMap p_hit 0.7)   */
    float l_miss;          /* -0.4  (p_miss 0.4)          */
    float l_min;           /* -2.0  (p 0.12)              */
    float l_max;           /* 3.5   (p 0.97)              */
    double min_range;      /* 0.3 */
    double max_range;      /* 70  */
    int32_t carve;         /* 1: free-space carving along the ray; 0: endpoints only */
} svx_occ_cfg;

typedef struct {
    int32_t frame;
    uint64_t points;       /* input points */
    uint64_t rays;         /* points kept (finite, >= min_range) */
    uint64_t hit_voxels;   /* voxels updated as HIT this scan */
    uint64_t miss_voxels;  /* voxels updated as MISS this scan */
    uint64_t new_blocks;
    double elapsed_ms;
} svx_occ_report;

typedef struct svx_occ svx_occ;

void svx_default_occ_cfg(svx_occ_cfg* cfg);
svx_status svx_occ_create(const svx_occ_cfg* cfg, int device, svx_occ** out);
svx_status svx_occ_destroy(svx_occ* occ);
svx_status svx_occ_get_stream(svx_occ* occ, void** stream);
/* Key sharding (as svx_map_set_shard): this map owns blocks with owner(b) == rank. */
/* Maps and zero-fills pool memory for `blocks` occupancy blocks and `layers` histogram
 * layers now, so that a growing map does not pay the mapping calls during a scan.
 * No effect on results. */
svx_status svx_occ_reserve(svx_occ* occ, uint64_t blocks, uint64_t layers);
svx_status svx_occ_set_shard(svx_occ* occ, int32_t rank, int32_t world);
/* One scan: n points of `stride` floats (xyz first), sensor frame; labels (u16 per
 * point) and conf (f32 per point) may be NULL; ptr_is_device: all three in HBM. */
svx_status svx_occ_integrate(svx_occ* occ, const float* points, const uint16_t* labels,
                             const float* conf, uint64_t n, int32_t stride,
                             int32_t ptr_is_device, const svx_pose* pose,
                             svx_occ_report* report);
/* A sequence of scans: scan f is rows [offsets[f], offsets[f+1]) of points / labels /
 * conf, posed by poses[f]. */
svx_status svx_occ_integrate_batch(svx_occ* occ, const float* points, const uint16_t* labels,
                                   const float* conf, const uint64_t* offsets, int32_t stride,
                                   int32_t ptr_is_device, const svx_pose* poses,
                                   int32_t n_frames, svx_occ_report* reports);
/* Pinhole depth images (BASELINE.json configs[2]: multi-camera semantic depth images;
 * no reference implementation, parity unpinned). Camera frame: x right, y down, z
 * forward, the reference's LabelImage convention (semantic_integrator.cpp:117-121:
 * u = floor(fx*x/z + cx)), so pixel (u, v) is back-projected through its centre:
 *   x = f32((u + 0.5 - cx) * z / fx),  y = f32((v + 0.5 - cy) * z / fy)   (FP64, that
 *   order), point = (x, y, z) for a finite depth 0 < z <= max_depth (metres, f32),
 * and the pixel is dropped otherwise. Each image is then one scan of the occupancy
 * contract above (ray from the camera centre, labels[pixel] / conf[pixel]), exactly as
 * svx_occ_integrate with that point cloud. */
typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
    double max_depth;
} svx_pinhole;
/* n_images images, row-major (v * width + u), concatenated in order in depth / labels /
 * conf (labels and conf may be NULL); cams[i] and cam_to_world[i] per image. */
svx_status svx_occ_integrate_depth(svx_occ* occ, const float* depth, const uint16_t* labels,
                                   const float* conf, const svx_pinhole* cams,
                                   const svx_pose* cam_to_world, int32_t n_images,
                                   int32_t ptr_is_device, svx_occ_report* reports);
/* Point query of n voxels (vxyz = n*3). Any output may be NULL; hist is n*K. label =
 * histogram argmax (-1: none). found[i] = 0 for a voxel of an unallocated block. */
svx_status svx_occ_lookup(svx_occ* occ, const int32_t* vxyz, uint64_t n, float* log_odds,
                          uint32_t* hits, uint32_t* misses, uint32_t* hist, int32_t* label,
                          uint8_t* found);
svx_status svx_occ_block_count(svx_occ* occ, uint64_t* n);
/* Map export "SOCC1": "SOCC1", f32 voxel_size, u32 K, f32 l_hit, l_miss, l_min, l_max,
 * u64 n_blocks, then per block in sorted key order: i32 x,y,z, f32 log_odds[512],
 * u32 hits[512], u32 misses[512], u8 has_hist, [u32 hist[512][K]]. buf=NULL -> size. */
svx_status svx_occ_save_mem(svx_occ* occ, uint8_t* buf, uint64_t cap, uint64_t* size);

/* ------------------------------------------------------------ profiling */
/* Per-kernel device time measured with CUDA events on the map's stream (the
 * launching stream), plus the algorithmic counters the roofline needs
 * (SURVEY.md 8(d)). Enabling resets the accumulators. */
enum {
    SVX_K_PROJECT = 0,   /* project_cloud + normals (K1/K2)            */
    SVX_K_RAYCAST = 1,   /* band DDA + block hash (K3/K4)              */
    SVX_K_FOLD = 2,      /* own-pixel measure + fold (K5)              */
    SVX_K_FALLBACK = 3,  /* fallback collect + sort + fold             */
    SVX_K_SEM_CULL = 4,  /* semantic frustum cull                      */
    SVX_K_SEM_UPDATE = 5,/* semantic Bayes update (K6)                 */
    SVX_K_COMPACT = 6,   /* reserved (the compaction is part of K3 now) */
    SVX_K_COUNT = 8
};
typedef struct {
    double ms[SVX_K_COUNT];         /* summed event time per kernel group */
    uint64_t launches[SVX_K_COUNT];
    uint64_t frames, points, rays;  /* TSDF frames, input points, band rays */
    uint64_t touched_blocks, new_blocks, updated_voxels, fallback_voxels;
    uint64_t sem_images, sem_candidates, sem_updated, sem_new_layers;
    double host_enqueue_ms; /* host time spent issuing the TSDF frame kernels (batched path) */
    double host_resume_ms;  /* host time spent handling aborts (pool growth, buffer growth) */
    double host_map_ms;     /* host time spent mapping pool memory (CUDA VMM) */
    uint64_t aborts[8];     /* batch aborts by reason bit: pool, capacity, key, hash, records,
                               big bucket, voxel list */
} svx_profile;
/* on: 0 off, 1 all kernel groups, otherwise a bitmask (1 << SVX_K_*) of the groups
 * to time (each timed group costs two event records per launch). Counters are
 * always accumulated while profiling is on. */
svx_status svx_profile_enable(svx_map* map, int32_t on);
svx_status svx_profile_read(svx_map* map, svx_profile* out);

/* ------------------------------------------------------------- defaults */
void svx_default_integrator_cfg(svx_integrator_cfg* cfg);
void svx_default_semantic_cfg(svx_semantic_cfg* cfg);
/* ProjectionModel::spinning — scan_projection.cpp:9-19. */
svx_status svx_lidar_spinning(int32_t width, int32_t height_px, double fov_up_deg,
                              double fov_down_deg, svx_lidar_model* out);

/* ------------------------------------------------------------- sharding */
/* Key sharding for multi-GPU: this map owns only blocks with
 * owner(b) == rank among world ranks. world=1 owns everything. */
svx_status svx_map_set_shard(svx_map* map, int32_t rank, int32_t world);
/* Maps physical memory for `blocks` TSDF blocks and `layers` semantic layers now
 * (CUDA VMM; addresses never move), so that a growing map does not pay the mapping
 * calls on its critical path. No effect on results. */
svx_status svx_map_reserve(svx_map* map, uint64_t blocks, uint64_t layers);
/* owner(bxyz) under the same hash, for host-side routing and tests. */
int32_t svx_block_owner(const int32_t bxyz[3], int32_t world);

#ifdef __cplusplus
}
#endif

#endif /* SVX_H_ */
