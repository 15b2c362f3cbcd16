/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * svx_oracle: a plain-C restatement of the reference's hot path
 * (project_cloud, compute_normal_image, TsdfIntegrator::integrate_frame,
 * SemanticIntegrator::integrate_labels, VoxelStore SVOX1 save), serial,
 * compiled with -ffp-contract=off so every double/float operation rounds
 * exactly like the reference's CMake Release build (-O3, no -march, no FMA).
 * Each function cites the reference file:line it follows. It is pinned against
 * the reference's own translation units (oracle/_ref/libsemvox_ref.so, built from
 * /root/reference by oracle/Makefile) and against the reference's golden vectors
 * (tests/test_oracle_golden.py).
 */
#ifndef SVX_ORACLE_H_
#define SVX_ORACLE_H_

#include "../include/svx.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct svxo_map svxo_map;

svxo_map* svxo_map_create(const svx_map_cfg* cfg, int* status);
void svxo_map_destroy(svxo_map* m);

/* project_cloud (scan_projection.cpp:39-76). depth/height: P floats. */
int svxo_project(const svx_lidar_model* model, const float* pts, uint64_t n, int32_t stride,
                 const svx_pose* pose, float* depth, float* height, uint64_t* dropped);
/* compute_normal_image (scan_projection.cpp:86-109). normals: 3P floats. */
int svxo_normals(const svx_lidar_model* model, const float* depth, float* normals,
                 uint8_t* valid);
/* TsdfIntegrator::integrate_frame (tsdf_integrator.cpp:97-258). normals/valid may
 * be NULL (images without normals). */
int svxo_integrate(svxo_map* m, const svx_lidar_model* model, const float* depth,
                   const float* normals, const uint8_t* valid, const svx_pose* pose,
                   const svx_integrator_cfg* cfg, svx_frame_report* rep);
/* SemanticIntegrator::integrate_labels (semantic_integrator.cpp:91-165). */
int svxo_integrate_labels(svxo_map* m, const svx_label_image* img, const svx_semantic_cfg* cfg,
                          svx_frame_report* rep);
/* VoxelStore::save (voxel_store.cpp:101-130) into memory; buf NULL -> size. */
uint64_t svxo_save_mem(svxo_map* m, uint8_t* buf, uint64_t cap);
uint64_t svxo_block_count(const svxo_map* m);
int svxo_get_or_allocate_block(svxo_map* m, const int32_t bxyz[3]);
int svxo_block_write(svxo_map* m, const int32_t bxyz[3], const svx_tsdf_voxel* tsdf,
                     const float* sem, int32_t has_sem);
int svxo_lookup(const svxo_map* m, const int32_t v[3], svx_tsdf_voxel* out, float* probs);
uint64_t svxo_observed(const svxo_map* m);
/* Sorted unique dirty blocks of pass `which` (0 tsdf, 1 semantic); clears. */
uint64_t svxo_take_dirty(svxo_map* m, int32_t which, int32_t* out, uint64_t cap);
/* extract_mesh (mesh.cpp:105-229) over the blocks bxyz (n*3; NULL = all blocks);
 * reserved: trailing "unlabeled" class id or -1. The result stays in the map. */
int svxo_mesh_extract(svxo_map* m, float min_weight, int32_t reserved, const int32_t* bxyz,
                      uint64_t n, uint64_t* n_vertices, uint64_t* n_faces);
void svxo_mesh_read(const svxo_map* m, float* vertices, float* normals, uint8_t* labels,
                    uint32_t* faces);
/* Occupancy extension (include/svx.h): PARITY UNPINNED, no reference implementation. */
typedef struct svxo_occ svxo_occ;
svxo_occ* svxo_occ_create(const svx_occ_cfg* cfg);
void svxo_occ_destroy(svxo_occ* m);
int svxo_occ_integrate(svxo_occ* m, const float* pts, const uint16_t* labels, const float* conf,
                       uint64_t n, int32_t stride, const svx_pose* pose, svx_occ_report* rep);
/* One pinhole depth image (svx.h svx_occ_integrate_depth): back-projection, then
 * svxo_occ_integrate of the cloud. */
int svxo_occ_integrate_depth(svxo_occ* m, const float* depth, const uint16_t* labels,
                             const float* conf, const svx_pinhole* cam, const svx_pose* pose,
                             svx_occ_report* rep);
uint64_t svxo_occ_save_mem(svxo_occ* m, uint8_t* buf, uint64_t cap);
const char* svxo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
