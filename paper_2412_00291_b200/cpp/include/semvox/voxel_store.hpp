// semvox drop-in (B200): VoxelStore with the reference's interface
// (proj/include/semvox/voxel_store.hpp) whose map of record lives in HBM.
//
// The device map (svx_map, include/svx.h) holds every block: the open-addressing
// block hash, the TSDF pool and the lazily allocated semantic layers. The
// reference API hands out VoxelBlock references that callers mutate in place, so
// the store keeps a host MIRROR of the blocks the caller has touched:
//   - a block enters the mirror when the host API reaches it (allocation,
//     find_block, lookup_voxel, tsdf_at, for_each_block); a store that is only
//     driven by the integrators has an empty mirror and never copies a block;
//   - blocks handed out through non-const paths are "exposed": before any
//     device operation (integration, stats, save) their host bytes are compared
//     with the last synchronised copy and changed blocks are written back;
//   - after a device operation the blocks it changed (the device dirty lists)
//     are re-read into the mirror, so references held by the caller stay
//     coherent. The dirty lists taken for this are kept for the integrators'
//     take_dirty_blocks().
// All public members lock one mutex, so concurrent callers are serialised
// (the reference allows concurrent lookups and allocation; results are the same).
#pragma once

#include "semvox/types.hpp"

#include <array>
#include <memory>
#include <optional>
#include <utility>
#include <vector>

struct svx_map;

namespace semvox {

struct VoxelBlock {
    BlockCoord coord;
    std::array<TsdfVoxel, kBlockVoxels> tsdf;
    std::vector<float> semantics;  // 512*K after ensure_semantics(), else empty

    explicit VoxelBlock(const BlockCoord& bc) : coord(bc) {}

    bool has_semantics() const { return !semantics.empty(); }
    void ensure_semantics(int num_labels) {
        if (!semantics.empty()) return;
        semantics.assign(size_t(kBlockVoxels) * size_t(num_labels), 1.f / float(num_labels));
    }
    float* probs_at(int linear, int num_labels) {
        return semantics.data() + size_t(linear) * size_t(num_labels);
    }
    const float* probs_at(int linear, int num_labels) const {
        return semantics.data() + size_t(linear) * size_t(num_labels);
    }
};
static_assert(sizeof(TsdfVoxel) == 20, "TsdfVoxel must match the 20-byte device voxel");

struct StoreStats {
    size_t allocated_blocks = 0;
    size_t observed_voxels = 0;
    size_t memory_bytes = 0;  // device footprint (pools, hash, per-block tables)
};

class VoxelStore {
public:
    // device: CUDA ordinal the map lives on.
    explicit VoxelStore(const MapConfig& cfg, int device = 0);
    VoxelStore(VoxelStore&& other) noexcept;
    VoxelStore& operator=(VoxelStore&&) = delete;
    VoxelStore(const VoxelStore&) = delete;
    VoxelStore& operator=(const VoxelStore&) = delete;
    ~VoxelStore();

    const MapConfig& config() const;

    VoxelBlock& get_or_allocate_block(const BlockCoord& bc);
    VoxelBlock* find_block(const BlockCoord& bc);
    const VoxelBlock* find_block(const BlockCoord& bc) const;
    std::optional<std::pair<TsdfVoxel, SemanticVoxel>> lookup_voxel(const VoxelCoord& v) const;
    const TsdfVoxel* tsdf_at(const VoxelCoord& v) const;
    StoreStats stats() const;
    size_t block_count() const;
    std::vector<BlockCoord> block_coords_sorted() const;

    // Visits every block (sorted order); materialises the whole map on the host.
    template <typename Fn>
    void for_each_block(Fn&& fn) const {
        for (const VoxelBlock* b : mirror_all(false)) fn(*b);
    }
    template <typename Fn>
    void for_each_block(Fn&& fn) {
        for (VoxelBlock* b : mirror_all(true)) fn(*b);
    }

    void save(const std::string& path) const;
    static VoxelStore load(const std::string& path, int device = 0);

    // ---- B200 additions (not in the reference interface) ----
    // The C-ABI handle of the device map (include/svx.h), for callers that mix
    // this API with direct svx_* calls.
    svx_map* device_map() const;
    // Writes host-side mutations of exposed blocks back to HBM.
    void flush_host_writes() const;
    // Re-reads blocks changed by a device pass into the mirror. which: 0 TSDF, 1 semantic.
    void refresh_after_device(int which) const;
    // Dirty blocks of pass `which` (sorted, unique), including any the mirror
    // refresh already took off the device; clears them.
    std::vector<BlockCoord> take_dirty(int which);
    // Blocks currently mirrored on the host.
    size_t mirrored_blocks() const;

    struct Impl;

private:
    friend class TsdfIntegrator;
    friend class SemanticIntegrator;
    explicit VoxelStore(std::unique_ptr<Impl> impl);
    std::vector<VoxelBlock*> mirror_all(bool expose) const;
    std::unique_ptr<Impl> impl_;
};

}  // namespace semvox
