// Occupancy extension (include/svx.h "occupancy extension"):
// free-space carving with the reference's 3D-DDA (traverse_segment,
// tsdf_integrator.hpp:93-135), per-scan HIT/MISS deduplication, f32 log-odds with
// clamping, hit/miss counters and u32 class histograms for per-point labels.
//
// Map: its own open-addressing block hash (16-byte slots: key + pool index) and a CUDA
// VMM pool of 8 KB occupancy blocks, SoA inside a block so the fold is coalesced:
//     u32 tag[512] | f32 log_odds[512] | u32 hits[512] | u32 misses[512]
// plus lazily allocated histogram layers [512][K] u32 for blocks that received a
// labelled hit.
//
// Per scan (one host synchronisation, which sizes the fold grid):
//   k_occ_visit  thread per point, the ray's DDA at voxel resolution: on each change
//                of block a hash find-or-insert (pool index from a counter, first
//                touch this scan marks the block); per voxel a RED.MAX (after a load
//                that skips it when the tag already holds this scan's value: every ray
//                crosses the voxels near the sensor) of tag = 4*S + kind with
//                HIT = 3 > MISS = 1, so HIT wins and the result does not depend on ray
//                order; labelled hits claim the block's histogram layer. Pool blocks
//                are mapped and zeroed ahead of need; a scan that outruns the mapping
//                is completed by a second launch for the blocks the first one skipped.
//   k_occ_touched  compacts the marked blocks into the scan's touched list.
//   k_occ_hist   labelled hits add to the class histograms (after the capacity check).
//   k_occ_fold   persistent CTAs over the touched list, thread per voxel: voxels whose
//                tag carries this scan's serial S get their one log-odds / counter update.
// Deduplication is per-voxel tag based (no sort): tags carry the scan serial, so no
// clearing pass is needed between scans.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "svx_map.hpp"

namespace svx {
namespace {

constexpr int kOccWords = 4 * kBlockVoxels;  // u32 words per occupancy block
constexpr size_t kOccBlockBytes = 4ull * kOccWords;
constexpr uint32_t kClaim = 0xFFFFFFFEu;     // histogram layer being allocated
constexpr uint32_t kOverflow = 0xFFFFFFFDu;  // block beyond max_blocks
constexpr int kHit = 3, kMiss = 1;

enum OccCounter : int {
    O_BLOCKS = 0, O_LAYERS, O_TOUCHED, O_ERR_CAP, O_ERR_KEY, O_ERR_HASH, O_ERR_MAP, O_RAYS, O_COUNT
};

struct OccParams {
    Pose T;
    double nu, inv_nu, min_r, max_r;
    const float* pts;
    const uint16_t* lbl;
    const float* conf;
    uint64_t n;
    int stride, carve, K;
    uint32_t serial, max_blocks;
    int32_t shard_rank, shard_world;
    uint32_t mapped_blocks;  // pool blocks mapped and zeroed
    uint32_t prev_blocks;    // redo launch: blocks the first launch already tagged
    int redo;
    const uint32_t* order;   // visit order of the points (longest rays first), or null
};

// Hash slot: key and pool index side by side, so one 16-byte load resolves a probe.
struct __align__(16) OccSlot {
    unsigned long long key;  // kEmptyKey = free
    uint32_t idx;            // kInvalid until the inserting thread publishes it
    uint32_t pad;
};

struct OccDev {
    OccSlot* slots;
    int log2cap;
    uint32_t mask;
    uint32_t* pool;       // [blocks][kOccWords]
    uint32_t* hist;       // [layers][512][K]
    uint64_t* block_keys;
    uint32_t* hist_idx;
    uint32_t* block_tag;
    uint32_t* touched;
    uint32_t* ctr;
    uint32_t* rep;  // per scan of the batch: HIT voxels, MISS voxels
};

// The ray of point i (svx.h contract): false when the point is dropped.
__device__ inline bool point_ray(const OccParams& p, uint64_t i, d3& o, d3& end, bool& hit) {
    const float* q = p.pts + i * uint64_t(p.stride);
    const float x = q[0], y = q[1], z = q[2];
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) return false;
    const d3 ps = mk(x, y, z);
    const double r = sqrt(dot3(ps, ps));
    if (r < p.min_r) return false;
    const d3 pw = xform(p.T, ps);
    o = mk(p.T.t[0], p.T.t[1], p.T.t[2]);
    hit = r <= p.max_r;
    end = hit ? pw : add3(o, scale3(p.max_r / r, sub3(pw, o)));
    return true;
}

__device__ inline uint32_t slot_idx(const OccSlot* sl) {
    volatile const uint32_t* v = &sl->idx;
    uint32_t idx;
    while ((idx = *v) == kInvalid) {  // inserted, index not yet published
    }
    return idx;
}

// Find-or-insert of a block.
__device__ inline uint32_t claim_block(const OccParams& p, const OccDev& d, uint64_t key) {
    uint32_t s = hash_slot(key, d.log2cap);
    uint32_t idx = kInvalid;
    for (uint32_t probe = 0; probe <= d.mask; ++probe) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(&d.slots[s]));
        const uint64_t k = uint64_t(v.x) | (uint64_t(v.y) << 32);
        if (k == key) {
            idx = v.z != kInvalid ? v.z : slot_idx(&d.slots[s]);
            break;
        }
        if (k == kEmptyKey) {
            const unsigned long long old = atomicCAS(&d.slots[s].key, kEmptyKey, key);
            if (old == kEmptyKey) {
                idx = atomicAdd(&d.ctr[O_BLOCKS], 1u);
                if (idx >= p.max_blocks) {
                    atomicAdd(&d.ctr[O_ERR_CAP], 1u);
                    idx = kOverflow;
                } else {
                    d.block_keys[idx] = key;
                }
                __threadfence();
                atomicExch(&d.slots[s].idx, idx);
                break;
            }
            if (old == key) {
                idx = slot_idx(&d.slots[s]);
                break;
            }
        }
        s = (s + 1) & d.mask;
    }
    if (idx == kInvalid) {
        atomicAdd(&d.ctr[O_ERR_HASH], 1u);
        return kInvalid;
    }
    if (idx == kOverflow) return kInvalid;
    return idx;  // the caller marks the block touched (block_tag = serial)
}

__device__ inline uint32_t find_block(const OccDev& d, uint64_t key) {
    uint32_t s = hash_slot(key, d.log2cap);
    for (uint32_t probe = 0; probe <= d.mask; ++probe) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(&d.slots[s]));
        const uint64_t k = uint64_t(v.x) | (uint64_t(v.y) << 32);
        if (k == key) return v.z;
        if (k == kEmptyKey) return kInvalid;
        s = (s + 1) & d.mask;
    }
    return kInvalid;
}

__device__ inline bool owned(const OccParams& p, uint64_t key) {
    return p.shard_world <= 1 || owner_of(key, p.shard_world) == p.shard_rank;
}

__device__ inline uint32_t label_of(const OccParams& p, uint64_t i) {
    return p.lbl ? uint32_t(p.lbl[i]) : 0xFFFFFFFFu;
}

__device__ inline uint32_t q8(const OccParams& p, uint64_t i) {
    if (!p.conf) return 255u;
    const float c = p.conf[i];
    if (!isfinite(c)) return 0u;
    const float cc = c < 0.f ? 0.f : (c > 1.f ? 1.f : c);
    return uint32_t(cc * 255.f + 0.5f);
}

// Visits the ray's voxels (carving) then the hit voxel; fn(x, y, z, kind).
template <typename Fn>
__device__ inline void for_each_ray_voxel(const OccParams& p, d3 o, d3 end, bool hit, Fn&& fn) {
    int32_t ev[3];
    world_to_voxel(end, p.inv_nu, ev);
    if (p.carve)
        traverse_segment(o, end, p.nu, p.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
            if (hit && x == ev[0] && y == ev[1] && z == ev[2]) return;
            fn(x, y, z, kMiss);
        });
    if (hit) fn(ev[0], ev[1], ev[2], kHit);
}

// Tag updates of one ray, issued kTagBatch at a time: the loads of a batch are in flight
// together (the DDA does not depend on them), then each RED.MAX is issued only where the
// tag does not already hold the value. Entries are tag addresses with the HIT flag in
// bit 1 (tags are 4-byte aligned); the window shifts so every index is static (registers).
constexpr int kTagBatch = 8;
// Only the first kNearVoxels cells of a ray (next to the sensor, where every ray of the
// scan passes) go through the load-then-RED batch; beyond them few rays share a voxel
// and the RED.MAX is issued directly (no load, nothing to wait for).
#ifndef SVX_OCC_SORT
#define SVX_OCC_SORT 1
#endif
#ifndef SVX_OCC_NEAR
#define SVX_OCC_NEAR 32
#endif
constexpr uint32_t kNearVoxels = SVX_OCC_NEAR;
struct TagBatch {
    uintptr_t q[kTagBatch];
    int n = 0;
    __device__ TagBatch() {
#pragma unroll
        for (int j = 0; j < kTagBatch; ++j) q[j] = 0;
    }
    __device__ void flush(uint32_t tag_base) {
        uint32_t cur[kTagBatch];
#pragma unroll
        for (int j = 0; j < kTagBatch; ++j)
            cur[j] = q[j] ? __ldcg(reinterpret_cast<const uint32_t*>(q[j] & ~uintptr_t(3))) : 0u;
#pragma unroll
        for (int j = 0; j < kTagBatch; ++j) {
            if (!q[j]) continue;
            const uint32_t want = tag_base + uint32_t((q[j] & 2) ? kHit : kMiss);
            if (cur[j] < want) atomicMax(reinterpret_cast<uint32_t*>(q[j] & ~uintptr_t(3)), want);
            q[j] = 0;
        }
        n = 0;
    }
    __device__ void push(uint32_t* tag, bool is_hit, uint32_t tag_base) {
#pragma unroll
        for (int j = 0; j + 1 < kTagBatch; ++j) q[j] = q[j + 1];
        q[kTagBatch - 1] = reinterpret_cast<uintptr_t>(tag) | (is_hit ? 2u : 0u);
        if (++n == kTagBatch) flush(tag_base);
    }
};

// Per-CTA cache of the near blocks' hash lookups (key -> pool index) in shared memory:
// every ray of the scan starts at the sensor, so the blocks there are looked up by
// every thread. Direct-mapped, first come keeps the slot: the key is claimed with a
// CAS, and its index is published (one 32-bit store) after the block has been marked
// touched, so a hit needs neither the global probe nor the mark; a reader that sees
// the key before the index falls back to the global path.
constexpr int kBlockCache = 2048;
#ifndef SVX_OCC_VB
#define SVX_OCC_VB 256
#endif
constexpr int kVisitThreads = SVX_OCC_VB;  // rays per CTA

#ifndef SVX_OCC_MINB
#define SVX_OCC_MINB 1
#endif
__global__ void __launch_bounds__(kVisitThreads, SVX_OCC_MINB) k_occ_visit(OccParams p, OccDev d) {
    __shared__ unsigned long long ckey[kBlockCache];
    __shared__ uint32_t cidx[kBlockCache];
    for (int j = threadIdx.x; j < kBlockCache; j += blockDim.x) {
        ckey[j] = kEmptyKey;
        cidx[j] = kInvalid;
    }
    __syncthreads();
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= p.n) return;
    const uint64_t i = p.order ? p.order[tid] : tid;
    d3 o, end;
    bool hit;
    if (!point_ray(p, i, o, end, hit)) return;
    if (!p.redo) atomicAdd(&d.ctr[O_RAYS], 1u);
    uint64_t last = kEmptyKey;
    uint32_t* base = nullptr;
    uint32_t idx = kInvalid;
    bool done_before = false;  // redo: this block's updates were applied by the first launch
    const uint32_t lab = label_of(p, i);
    const uint32_t tag_base = p.serial * 4u;
    TagBatch tb;
    uint32_t nv = 0;  // cells of this ray visited so far
    for_each_ray_voxel(p, o, end, hit, [&](int32_t x, int32_t y, int32_t z, int kind) {
        ++nv;
        const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
        if (!(key_in_range(bx) && key_in_range(by) && key_in_range(bz))) {
            atomicAdd(&d.ctr[O_ERR_KEY], 1u);
            return;
        }
        const uint64_t key = pack_key(bx, by, bz);
        if (key != last) {
            last = key;
            idx = kInvalid;
            if (owned(p, key)) {
                const bool near = nv <= kNearVoxels;
                const uint32_t h = uint32_t((key * 0x9E3779B97F4A7C15ull) >> 53) & (kBlockCache - 1);
                if (near && ckey[h] == key) idx = *reinterpret_cast<volatile uint32_t*>(&cidx[h]);
                if (idx == kInvalid) {
                    idx = claim_block(p, d, key);
                    if (idx != kInvalid) {
                        if (near) {  // hot block: read, not write (same-address writes serialise)
                            if (__ldcg(&d.block_tag[idx]) != p.serial) d.block_tag[idx] = p.serial;
                            if (ckey[h] == kEmptyKey && atomicCAS(&ckey[h], kEmptyKey, key) == kEmptyKey)
                                cidx[h] = idx;
                        } else {
                            atomicMax(&d.block_tag[idx], p.serial);  // RED: tags only grow
                        }
                    }
                }
            }
            base = nullptr;
            if (idx != kInvalid) {
                if (idx < p.mapped_blocks) base = d.pool + uint64_t(idx) * kOccWords;
                else atomicOr(&d.ctr[O_ERR_MAP], 1u);
            }
            done_before = p.redo && idx < p.prev_blocks;
        }
        if (!base) return;
        // hot voxels (near the sensor every ray crosses them) are read, not written:
        // same-address writes serialise in L2
        if (!done_before) {
            if (nv < kNearVoxels) tb.push(base + local_linear(x, y, z), kind == kHit, tag_base);
            else atomicMax(base + local_linear(x, y, z), tag_base + uint32_t(kind));  // RED
        }
        if (kind == kHit && lab < uint32_t(p.K) && __ldcg(&d.hist_idx[idx]) == kInvalid &&
            atomicCAS(&d.hist_idx[idx], kInvalid, kClaim) == kInvalid)  // histogram layer
            atomicExch(&d.hist_idx[idx], atomicAdd(&d.ctr[O_LAYERS], 1u));
    });
    tb.flush(tag_base);
}

// Pinhole depth image -> camera-frame points (svx.h "pinhole depth images"): thread per
// pixel, NaN for a dropped pixel (the scan then drops it like any non-finite point).
__global__ void __launch_bounds__(256) k_depth_points(const float* __restrict__ depth, int32_t w,
                                                      uint64_t n, svx_pinhole cam,
                                                      float* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float z = depth[i];
    float x = CUDART_NAN_F, y = CUDART_NAN_F, zz = CUDART_NAN_F;
    if (isfinite(z) && z > 0.f && double(z) <= cam.max_depth) {
        const uint32_t u = uint32_t(i % uint64_t(w)), v = uint32_t(i / uint64_t(w));
        const double zd = double(z);
        x = float((double(u) + 0.5 - cam.cx) * zd / cam.fx);
        y = float((double(v) + 0.5 - cam.cy) * zd / cam.fy);
        zz = z;
    }
    out[3 * i] = x;
    out[3 * i + 1] = y;
    out[3 * i + 2] = zz;
}

// Visit order: the ray's cell count estimate (L1 voxel distance origin -> end, the DDA
// visits about that many cells) as a descending sort key, so that the 32 rays of a warp
// have similar lengths (lanes do not idle behind one long ray) and the longest rays start
// first (the grid's tail is short rays). Dropped points sort last. Only the schedule
// changes: the result does not depend on which thread handles which ray.
__global__ void __launch_bounds__(256) k_occ_ray_keys(OccParams p, uint32_t* __restrict__ key,
                                                      uint32_t* __restrict__ idx) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    d3 o, end;
    bool hit;
    uint32_t len = 0;
    if (point_ray(p, i, o, end, hit)) {
        int32_t a[3], b[3];
        world_to_voxel(o, p.inv_nu, a);
        world_to_voxel(end, p.inv_nu, b);
        const uint32_t l = p.carve ? uint32_t(abs(b[0] - a[0])) + uint32_t(abs(b[1] - a[1])) +
                                         uint32_t(abs(b[2] - a[2])) + 1u
                                   : 1u;
        len = l > 0xFFFEu ? 0xFFFEu : l;
        len += 1;
    }
    key[i] = 0xFFFFu - len;
    idx[i] = uint32_t(i);
}

// Labelled hits -> class histograms, once the scan is accepted (the adds cannot be
// undone, so they wait for the capacity check) and every claimed layer is mapped.
__global__ void __launch_bounds__(256) k_occ_hist(OccParams p, OccDev d) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const uint32_t lab = label_of(p, i);
    if (lab >= uint32_t(p.K)) return;
    d3 o, end;
    bool hit;
    if (!point_ray(p, i, o, end, hit) || !hit) return;
    int32_t ev[3];
    world_to_voxel(end, p.inv_nu, ev);
    const int32_t bx = block_coord(ev[0]), by = block_coord(ev[1]), bz = block_coord(ev[2]);
    const uint64_t key = pack_key(bx, by, bz);
    if (!owned(p, key)) return;
    const uint32_t idx = find_block(d, key);
    const uint32_t layer = d.hist_idx[idx];
    atomicAdd(&d.hist[(uint64_t(layer) * kBlockVoxels + local_linear(ev[0], ev[1], ev[2])) * p.K + lab],
              q8(p, i));
}

struct FoldParams {
    uint32_t serial;
    float l_hit, l_miss, l_min, l_max;
};

// Touched-block list of the scan: the blocks whose mark carries its serial.
__global__ void k_occ_touched(OccDev d, uint32_t n_blocks, uint32_t serial) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool t = i < n_blocks && d.block_tag[i] == serial;
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, t);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&d.ctr[O_TOUCHED], uint32_t(__popc(ballot)));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (t) d.touched[base + __popc(ballot & ((1u << lane) - 1))] = i;
}

// Persistent CTAs over the touched list, thread per voxel. The tag, log-odds and
// both counters are loaded together (coalesced, no dependent round trip).
__global__ void __launch_bounds__(kBlockVoxels) k_occ_fold(FoldParams fp, OccDev d) {
    const uint32_t n = __ldcg(&d.ctr[O_TOUCHED]);
    const int v = threadIdx.x;
    uint32_t nh = 0, nm = 0;
    for (uint32_t j = blockIdx.x; j < n; j += gridDim.x) {
        uint32_t* base = d.pool + uint64_t(d.touched[j]) * kOccWords;
        const uint32_t tag = __ldcg(&base[v]);
        float l = __uint_as_float(__ldcg(&base[kBlockVoxels + v]));
        const uint32_t h = __ldcg(&base[2 * kBlockVoxels + v]);
        const uint32_t ms = __ldcg(&base[3 * kBlockVoxels + v]);
        if ((tag >> 2) != fp.serial) continue;
        if ((tag & 3u) == uint32_t(kHit)) {
            const float t = l + fp.l_hit;
            l = t > fp.l_max ? fp.l_max : t;
            base[2 * kBlockVoxels + v] = h + 1u;
            ++nh;
        } else {
            const float t = l + fp.l_miss;
            l = t < fp.l_min ? fp.l_min : t;
            base[3 * kBlockVoxels + v] = ms + 1u;
            ++nm;
        }
        base[kBlockVoxels + v] = __float_as_uint(l);
    }
    nh = __reduce_add_sync(0xFFFFFFFFu, nh);
    nm = __reduce_add_sync(0xFFFFFFFFu, nm);
    if ((threadIdx.x & 31) == 0) {
        if (nh) atomicAdd(&d.rep[0], nh);
        if (nm) atomicAdd(&d.rep[1], nm);
    }
}

// capacity rollback: histogram layers claimed by the rejected scan
__global__ void k_occ_unclaim(uint32_t* __restrict__ hist_idx, uint32_t n_blocks, uint32_t keep) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_blocks && hist_idx[i] != kInvalid && hist_idx[i] >= keep) hist_idx[i] = kInvalid;
}

__global__ void k_occ_rebuild(OccDev d, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t key = d.block_keys[i];
    uint32_t s = hash_slot(key, d.log2cap);
    while (atomicCAS(&d.slots[s].key, kEmptyKey, key) != kEmptyKey) s = (s + 1) & d.mask;
    d.slots[s].idx = i;
}

__global__ void k_occ_clear_slots(OccSlot* __restrict__ slots, uint32_t cap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) {
        slots[i].key = kEmptyKey;
        slots[i].idx = kInvalid;
    }
}

__global__ void k_occ_lookup(OccDev d, int K, const int32_t* __restrict__ v, uint64_t n,
                             float* __restrict__ lo, uint32_t* __restrict__ hits,
                             uint32_t* __restrict__ misses, uint32_t* __restrict__ hist,
                             int32_t* __restrict__ label, uint8_t* __restrict__ found) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t x = v[3 * i], y = v[3 * i + 1], z = v[3 * i + 2];
    const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
    uint32_t idx = kInvalid;
    if (key_in_range(bx) && key_in_range(by) && key_in_range(bz)) idx = find_block(d, pack_key(bx, by, bz));
    if (idx == kInvalid || idx == kOverflow) {
        if (found) found[i] = 0;
        if (label) label[i] = -1;
        return;
    }
    const int lin = local_linear(x, y, z);
    const uint32_t* b = d.pool + uint64_t(idx) * kOccWords;
    if (found) found[i] = 1;
    if (lo) lo[i] = __uint_as_float(b[kBlockVoxels + lin]);
    if (hits) hits[i] = b[2 * kBlockVoxels + lin];
    if (misses) misses[i] = b[3 * kBlockVoxels + lin];
    const uint32_t layer = d.hist_idx[idx];
    int best = -1;
    uint32_t best_c = 0;
    for (int k = 0; k < K; ++k) {
        const uint32_t c = layer == kInvalid ? 0u : d.hist[(uint64_t(layer) * kBlockVoxels + lin) * K + k];
        if (hist) hist[i * K + k] = c;
        if (c > best_c) {
            best_c = c;
            best = k;
        }
    }
    if (label) label[i] = best;
}

inline unsigned grid256(uint64_t n) { return unsigned((n + 255) / 256); }

template <typename T>
T* dmalloc(size_t n) {
    T* p = nullptr;
    SVX_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

void require(bool ok, svx_status s, const char* msg) {
    if (!ok) throw Error(s, msg);
}

struct DevGuard {
    int prev = 0;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SVX_CUDA(cudaSetDevice(dev));
    }
    ~DevGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace
}  // namespace svx

struct svx_occ {
    svx_occ_cfg cfg{};
    int device = 0;
    cudaStream_t stream = nullptr;
    int32_t shard_rank = 0, shard_world = 1;
    int log2cap = 0;
    uint32_t cap = 0;
    void* slots = nullptr;  // OccSlot[cap]
    svx::VmmArray pool;   // [blocks][4 x 512] u32
    svx::VmmArray hist;   // [layers][512][K] u32
    size_t layer_bytes = 0;
    uint64_t* block_keys = nullptr;
    uint32_t* hist_idx = nullptr;
    uint32_t* block_tag = nullptr;
    uint32_t* touched = nullptr;
    uint32_t* d_ctr = nullptr;
    uint32_t* h_ctr = nullptr;
    uint32_t serial = 0;
    int32_t frames = 0;
    uint64_t n_blocks = 0, n_layers = 0;
    uint64_t mapped_blocks = 0, mapped_layers = 0;  // mapped and zeroed
    uint64_t max_new_blocks = 0;                    // largest per-scan growth seen
    uint64_t min_headroom = 65536;                  // blocks mapped ahead of a scan
    svx::DevBuf<uint32_t> rep;                      // per scan of a batch: HIT, MISS voxels
    svx::DevBuf<float> pts;
    svx::DevBuf<uint16_t> lbl;
    svx::DevBuf<float> conf;
    svx::DevBuf<float> dep;  // staged depth images
    svx::DevBuf<uint32_t> ray_key, ray_idx;  // visit order (sort keys / point indices, x2)
    svx::DevBuf<uint8_t> sort_tmp;
};

namespace svx {
namespace {

OccDev occ_dev(svx_occ* m) {
    return OccDev{static_cast<OccSlot*>(m->slots), m->log2cap, m->cap - 1,
                  static_cast<uint32_t*>(m->pool.base()), static_cast<uint32_t*>(m->hist.base()),
                  m->block_keys, m->hist_idx, m->block_tag, m->touched, m->d_ctr, m->rep.p};
}

void free_occ(svx_occ* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    if (m->stream) cudaStreamSynchronize(m->stream);
    for (void* p : {m->slots, (void*)m->block_keys, (void*)m->hist_idx,
                    (void*)m->block_tag, (void*)m->touched, (void*)m->d_ctr})
        if (p) cudaFree(p);
    if (m->h_ctr) cudaFreeHost(m->h_ctr);
    m->rep.release();
    m->pts.release();
    m->lbl.release();
    m->conf.release();
    m->dep.release();
    m->ray_key.release();
    m->ray_idx.release();
    m->sort_tmp.release();
    if (m->stream) cudaStreamDestroy(m->stream);
    delete m;
}

void validate(const svx_occ_cfg& c) {
    require(c.voxel_size > 0.f, SVX_INVALID_ARGUMENT, "voxel_size must be > 0");
    require(c.num_labels >= 1 && c.num_labels <= 64, SVX_INVALID_ARGUMENT, "num_labels must be in [1, 64]");
    require(c.max_blocks != 0 && c.max_blocks < (1u << 25), SVX_INVALID_ARGUMENT,
            "max_blocks must be in [1, 2^25)");
    require(c.l_hit >= 0.f && c.l_miss <= 0.f && c.l_min <= 0.f && c.l_max >= 0.f,
            SVX_INVALID_ARGUMENT, "log-odds: need l_hit >= 0, l_miss <= 0, l_min <= 0 <= l_max");
    require(c.min_range >= 0.0 && c.max_range > c.min_range, SVX_INVALID_ARGUMENT,
            "ranges: need 0 <= min_range < max_range");
}

// Maps and zero-fills the pool so that `blocks` blocks are usable (new blocks must
// read as zero: tags 0 < every serial). Only the growth is zeroed; mapping ahead of
// need runs on the pool's background thread.
void map_blocks(svx_occ* m, uint64_t blocks) {
    blocks = std::min<uint64_t>(blocks, m->cfg.max_blocks);
    if (blocks <= m->mapped_blocks) return;
    m->pool.ensure(blocks * kOccBlockBytes);  // immediate when a prefetch already covers it
    SVX_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(m->pool.base()) + m->mapped_blocks * kOccBlockBytes, 0,
                             (blocks - m->mapped_blocks) * kOccBlockBytes, m->stream));
    m->mapped_blocks = blocks;
}

void map_layers(svx_occ* m, uint64_t layers) {
    if (layers <= m->mapped_layers) return;
    const uint64_t target = std::min<uint64_t>(m->cfg.max_blocks, std::max(layers, m->mapped_layers * 2));
    m->hist.ensure(target * m->layer_bytes);
    SVX_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(m->hist.base()) + m->mapped_layers * m->layer_bytes, 0,
                             (target - m->mapped_layers) * m->layer_bytes, m->stream));
    m->mapped_layers = target;
}

// One scan; points / labels / conf already on the device. rep_slot: this scan's
// HIT/MISS counters on the device (read at the end of the batch).
void occ_scan(svx_occ* m, const float* d_pts, const uint16_t* d_lbl, const float* d_conf, uint64_t n,
              int stride, const svx_pose& pose, uint32_t* rep_slot, svx_occ_report* rep) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t st = m->stream;
    require(m->serial + 1 < (1u << 30), SVX_INVALID_ARGUMENT, "too many scans for one occupancy map");
    m->serial += 1;
    OccParams p{};
    p.T = to_pose(pose);
    p.nu = double(m->cfg.voxel_size);
    p.inv_nu = 1.0 / double(m->cfg.voxel_size);
    p.min_r = m->cfg.min_range;
    p.max_r = m->cfg.max_range;
    p.pts = d_pts;
    p.lbl = d_lbl;
    p.conf = d_conf;
    p.n = n;
    p.stride = stride;
    p.carve = m->cfg.carve;
    p.K = m->cfg.num_labels;
    p.serial = m->serial;
    p.max_blocks = m->cfg.max_blocks;
    p.shard_rank = m->shard_rank;
    p.shard_world = m->shard_world;
    // headroom for this scan's new blocks, mapped and zeroed ahead of the launch
    const uint64_t head = std::max<uint64_t>(m->min_headroom, 2 * m->max_new_blocks);
    map_blocks(m, m->n_blocks + head);
    m->pool.prefetch(std::min<uint64_t>(m->cfg.max_blocks, m->n_blocks + 4 * head) * kOccBlockBytes);
    p.mapped_blocks = uint32_t(m->mapped_blocks);
    m->h_ctr[O_BLOCKS] = uint32_t(m->n_blocks);
    m->h_ctr[O_LAYERS] = uint32_t(m->n_layers);
    for (int c = O_TOUCHED; c < O_COUNT; ++c) m->h_ctr[c] = 0;
    SVX_CUDA(cudaMemcpyAsync(m->d_ctr, m->h_ctr, 4 * O_COUNT, cudaMemcpyHostToDevice, st));
    OccDev d = occ_dev(m);
    d.rep = rep_slot;
    if (n) {
#if SVX_OCC_SORT
        if (n >= 4096 && n < (1ull << 32)) {
            m->ray_key.alloc(2 * n);
            m->ray_idx.alloc(2 * n);
            k_occ_ray_keys<<<grid256(n), 256, 0, st>>>(p, m->ray_key.p, m->ray_idx.p);
            size_t bytes = 0;
            SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, m->ray_key.p, m->ray_key.p + n,
                                                     m->ray_idx.p, m->ray_idx.p + n, int(n), 0, 16, st));
            m->sort_tmp.alloc(bytes);
            SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->sort_tmp.p, bytes, m->ray_key.p, m->ray_key.p + n,
                                                     m->ray_idx.p, m->ray_idx.p + n, int(n), 0, 16, st));
            p.order = m->ray_idx.p + n;
            count_launch(2);
        }
#endif
        k_occ_visit<<<unsigned((n + kVisitThreads - 1) / kVisitThreads), kVisitThreads, 0, st>>>(p, d);
        count_launch();
    }
    SVX_CUDA(cudaMemcpyAsync(m->h_ctr, m->d_ctr, 4 * O_COUNT, cudaMemcpyDeviceToHost, st));
    SVX_CUDA(cudaStreamSynchronize(st));
    const uint64_t old_blocks = m->n_blocks, old_layers = m->n_layers;
    if (m->h_ctr[O_ERR_KEY] || m->h_ctr[O_ERR_HASH] || m->h_ctr[O_ERR_CAP]) {
        // reject the scan: drop its new blocks and histogram claims. Its tags carry a
        // serial no fold will look for; log-odds, counters and histograms are untouched.
        k_occ_clear_slots<<<grid256(m->cap), 256, 0, st>>>(d.slots, m->cap);
        count_launch();
        if (old_blocks) {
            k_occ_rebuild<<<grid256(old_blocks), 256, 0, st>>>(d, uint32_t(old_blocks));
            k_occ_unclaim<<<grid256(old_blocks), 256, 0, st>>>(m->hist_idx, uint32_t(old_blocks),
                                                               uint32_t(old_layers));
            count_launch(2);
        }
        const uint64_t over = std::min<uint64_t>(m->h_ctr[O_BLOCKS], m->cfg.max_blocks);
        if (over > old_blocks)
            SVX_CUDA(cudaMemsetAsync(m->hist_idx + old_blocks, 0xFF, 4 * (over - old_blocks), st));
        SVX_CUDA(cudaStreamSynchronize(st));
        if (m->h_ctr[O_ERR_KEY])
            throw Error(SVX_INVALID_ARGUMENT, "voxel outside the device key range [-2^23, 2^23)");
        if (m->h_ctr[O_ERR_HASH]) throw Error(SVX_CAPACITY, "occupancy block hash is full");
        throw Error(SVX_CAPACITY, "occupancy map: max_blocks reached");
    }
    m->n_blocks = m->h_ctr[O_BLOCKS];
    m->n_layers = m->h_ctr[O_LAYERS];
    if (m->min_headroom >= 65536) m->max_new_blocks = std::max(m->max_new_blocks, m->n_blocks - old_blocks);
    const uint64_t rays = m->h_ctr[O_RAYS];
    if (m->h_ctr[O_ERR_MAP]) {  // the scan outran the mapped pool: finish the skipped blocks
        map_blocks(m, m->n_blocks);
        p.redo = 1;
        p.prev_blocks = p.mapped_blocks;
        p.mapped_blocks = uint32_t(m->mapped_blocks);
        k_occ_visit<<<unsigned((n + kVisitThreads - 1) / kVisitThreads), kVisitThreads, 0, st>>>(p, d);
        count_launch();
        // it may claim histogram layers for the blocks it completes
        SVX_CUDA(cudaMemcpyAsync(&m->h_ctr[O_LAYERS], &m->d_ctr[O_LAYERS], 4, cudaMemcpyDeviceToHost, st));
        SVX_CUDA(cudaStreamSynchronize(st));
        m->n_layers = m->h_ctr[O_LAYERS];
    }
    map_layers(m, m->n_layers);
    d = occ_dev(m);
    d.rep = rep_slot;
    if (n && p.lbl) {
        k_occ_hist<<<grid256(n), 256, 0, st>>>(p, d);
        count_launch();
    }
    if (m->n_blocks) {
        k_occ_touched<<<grid256(m->n_blocks), 256, 0, st>>>(d, uint32_t(m->n_blocks), m->serial);
        const FoldParams fp{m->serial, m->cfg.l_hit, m->cfg.l_miss, m->cfg.l_min, m->cfg.l_max};
        const unsigned grid = unsigned(std::min<uint64_t>(m->n_blocks, 148ull * 4));
        k_occ_fold<<<grid, kBlockVoxels, 0, st>>>(fp, d);
        count_launch(2);
    }
    SVX_CUDA(cudaGetLastError());
    if (rep) {
        rep->frame = m->frames;
        rep->points = n;
        rep->rays = rays;
        rep->new_blocks = m->n_blocks - old_blocks;
        rep->elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    m->frames += 1;
}

template <typename T>
const T* stage(svx_occ* m, DevBuf<T>& buf, const T* src, uint64_t count) {
    if (!src) return nullptr;
    buf.alloc(std::max<uint64_t>(count, 1));
    SVX_CUDA(cudaMemcpyAsync(buf.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, m->stream));
    return buf.p;
}

}  // namespace
}  // namespace svx

using namespace svx;

extern "C" {

void svx_default_occ_cfg(svx_occ_cfg* c) {
    c->voxel_size = 0.1f;
    c->num_labels = 20;
    c->max_blocks = 1u << 20;
    c->l_hit = 0.85f;
    c->l_miss = -0.4f;
    c->l_min = -2.0f;
    c->l_max = 3.5f;
    c->min_range = 0.3;
    c->max_range = 70.0;
    c->carve = 1;
}

svx_status svx_occ_create(const svx_occ_cfg* cfg, int device, svx_occ** out) {
    return api_guard([&] {
        require(cfg && out, SVX_INVALID_ARGUMENT, "null argument");
        validate(*cfg);
        int ndev = 0;
        SVX_CUDA(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, SVX_INVALID_ARGUMENT, "no such CUDA device");
        DevGuard g(device);
        svx_occ* m = new svx_occ();
        try {
            m->cfg = *cfg;
            m->device = device;
            SVX_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
            const uint64_t want = std::max<uint64_t>(2ull * cfg->max_blocks, 1024);
            while ((1ull << m->log2cap) < want) ++m->log2cap;
            m->cap = uint32_t(1u << m->log2cap);
            m->slots = dmalloc<OccSlot>(m->cap);
            m->block_keys = dmalloc<uint64_t>(cfg->max_blocks);
            m->hist_idx = dmalloc<uint32_t>(cfg->max_blocks);
            m->block_tag = dmalloc<uint32_t>(cfg->max_blocks);
            m->touched = dmalloc<uint32_t>(cfg->max_blocks);
            m->d_ctr = dmalloc<uint32_t>(O_COUNT);
            SVX_CUDA(cudaMallocHost(&m->h_ctr, 4 * O_COUNT));
            std::memset(m->h_ctr, 0, 4 * O_COUNT);
            k_occ_clear_slots<<<grid256(m->cap), 256, 0, m->stream>>>(static_cast<OccSlot*>(m->slots), m->cap);
            count_launch();
            SVX_CUDA(cudaMemsetAsync(m->hist_idx, 0xFF, 4ull * cfg->max_blocks, m->stream));
            SVX_CUDA(cudaMemsetAsync(m->block_tag, 0, 4ull * cfg->max_blocks, m->stream));
            m->layer_bytes = 4ull * kBlockVoxels * uint64_t(cfg->num_labels);
            // test hook: a tiny mapping headroom exercises the scan-completion launch
            if (const char* e = std::getenv("SVX_TEST_OCC_HEADROOM")) {
                m->min_headroom = uint64_t(std::max(0L, std::atol(e)));
                m->max_new_blocks = 0;
            }
            m->pool.reserve(device, size_t(cfg->max_blocks) * kOccBlockBytes);
            m->hist.reserve(device, size_t(cfg->max_blocks) * m->layer_bytes);
            SVX_CUDA(cudaStreamSynchronize(m->stream));
        } catch (...) {
            free_occ(m);
            throw;
        }
        *out = m;
    });
}

svx_status svx_occ_destroy(svx_occ* m) {
    return api_guard([&] { free_occ(m); });
}

svx_status svx_occ_get_stream(svx_occ* m, void** stream) {
    return api_guard([&] {
        require(m && stream, SVX_INVALID_ARGUMENT, "null argument");
        *stream = m->stream;
    });
}

svx_status svx_occ_reserve(svx_occ* m, uint64_t blocks, uint64_t layers) {
    return api_guard([&] {
        require(m != nullptr, SVX_INVALID_ARGUMENT, "null map");
        DevGuard g(m->device);
        map_blocks(m, blocks);
        map_layers(m, std::min<uint64_t>(layers, m->cfg.max_blocks));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
    });
}

svx_status svx_occ_set_shard(svx_occ* m, int32_t rank, int32_t world) {
    return api_guard([&] {
        require(m && world >= 1 && rank >= 0 && rank < world, SVX_INVALID_ARGUMENT, "bad shard");
        require(m->n_blocks == 0, SVX_INVALID_ARGUMENT, "set the shard before the first scan");
        m->shard_rank = rank;
        m->shard_world = world;
    });
}

svx_status svx_occ_integrate(svx_occ* m, const float* points, const uint16_t* labels,
                             const float* conf, uint64_t n, int32_t stride, int32_t on_device,
                             const svx_pose* pose, svx_occ_report* rep) {
    const uint64_t offs[2] = {0, n};
    return svx_occ_integrate_batch(m, points, labels, conf, offs, stride, on_device, pose, 1, rep);
}

svx_status svx_occ_integrate_batch(svx_occ* m, const float* points, const uint16_t* labels,
                                   const float* conf, const uint64_t* offs, int32_t stride,
                                   int32_t on_device, const svx_pose* poses, int32_t n_frames,
                                   svx_occ_report* reps) {
    return api_guard([&] {
        require(m && offs && poses && n_frames >= 0, SVX_INVALID_ARGUMENT, "null argument");
        require(stride >= 3, SVX_INVALID_ARGUMENT, "stride must be >= 3");
        DevGuard g(m->device);
        m->rep.alloc(2ull * std::max(n_frames, 1));
        SVX_CUDA(cudaMemsetAsync(m->rep.p, 0, 8ull * std::max(n_frames, 1), m->stream));
        for (int f = 0; f < n_frames; ++f) {
            require(offs[f + 1] >= offs[f], SVX_INVALID_ARGUMENT, "offsets must be non-decreasing");
            require(offs[f + 1] == offs[f] || points, SVX_INVALID_ARGUMENT, "null points");
            validate_pose(poses[f]);
            const uint64_t a = offs[f], n = offs[f + 1] - a;
            const float* dp = points ? points + a * uint64_t(stride) : nullptr;
            const uint16_t* dl = labels ? labels + a : nullptr;
            const float* dc = conf ? conf + a : nullptr;
            if (!on_device && n) {
                dp = stage(m, m->pts, dp, n * uint64_t(stride));
                dl = stage(m, m->lbl, dl, n);
                dc = stage(m, m->conf, dc, n);
            }
            occ_scan(m, dp, dl, dc, n, stride, poses[f], m->rep.p + 2 * f, reps ? reps + f : nullptr);
        }
        std::vector<uint32_t> hm(2ull * std::max(n_frames, 1));
        SVX_CUDA(cudaMemcpyAsync(hm.data(), m->rep.p, 4 * hm.size(), cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        for (int f = 0; reps && f < n_frames; ++f) {
            reps[f].hit_voxels = hm[2 * f];
            reps[f].miss_voxels = hm[2 * f + 1];
        }
    });
}

svx_status svx_occ_integrate_depth(svx_occ* m, const float* depth, const uint16_t* labels,
                                   const float* conf, const svx_pinhole* cams,
                                   const svx_pose* poses, int32_t n_images, int32_t on_device,
                                   svx_occ_report* reps) {
    return api_guard([&] {
        require(m && cams && poses && n_images >= 0, SVX_INVALID_ARGUMENT, "null argument");
        DevGuard g(m->device);
        uint64_t a = 0;
        for (int f = 0; f < n_images; ++f) {
            const svx_pinhole& c = cams[f];
            require(c.width > 0 && c.height > 0, SVX_INVALID_ARGUMENT, "image size must be positive");
            require(std::isfinite(c.fx) && std::isfinite(c.fy) && c.fx != 0.0 && c.fy != 0.0 &&
                        std::isfinite(c.cx) && std::isfinite(c.cy),
                    SVX_INVALID_ARGUMENT, "bad intrinsics");
            require(c.max_depth > 0.0, SVX_INVALID_ARGUMENT, "max_depth must be positive");
            validate_pose(poses[f]);
            a += uint64_t(c.width) * uint64_t(c.height);
        }
        require(a == 0 || depth, SVX_INVALID_ARGUMENT, "null depth");
        m->rep.alloc(2ull * std::max(n_images, 1));
        SVX_CUDA(cudaMemsetAsync(m->rep.p, 0, 8ull * std::max(n_images, 1), m->stream));
        a = 0;
        for (int f = 0; f < n_images; ++f) {
            const uint64_t n = uint64_t(cams[f].width) * uint64_t(cams[f].height);
            const float* dd = depth + a;
            const uint16_t* dl = labels ? labels + a : nullptr;
            const float* dc = conf ? conf + a : nullptr;
            if (!on_device) {
                dd = stage(m, m->dep, dd, n);
                dl = stage(m, m->lbl, dl, n);
                dc = stage(m, m->conf, dc, n);
            }
            m->pts.alloc(3 * n);
            k_depth_points<<<grid256(n), 256, 0, m->stream>>>(dd, cams[f].width, n, cams[f], m->pts.p);
            count_launch();
            occ_scan(m, m->pts.p, dl, dc, n, 3, poses[f], m->rep.p + 2 * f, reps ? reps + f : nullptr);
            a += n;
        }
        std::vector<uint32_t> hm(2ull * std::max(n_images, 1));
        SVX_CUDA(cudaMemcpyAsync(hm.data(), m->rep.p, 4 * hm.size(), cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        for (int f = 0; reps && f < n_images; ++f) {
            reps[f].hit_voxels = hm[2 * f];
            reps[f].miss_voxels = hm[2 * f + 1];
        }
    });
}

svx_status svx_occ_lookup(svx_occ* m, const int32_t* vxyz, uint64_t n, float* log_odds,
                          uint32_t* hits, uint32_t* misses, uint32_t* hist, int32_t* label,
                          uint8_t* found) {
    return api_guard([&] {
        require(m && (vxyz || !n), SVX_INVALID_ARGUMENT, "null argument");
        if (!n) return;
        DevGuard g(m->device);
        const int K = m->cfg.num_labels;
        DevBuf<int32_t> dv;
        DevBuf<uint8_t> out;
        dv.alloc(3 * n);
        // outputs packed in one device buffer: lo | hits | misses | label | hist | found
        const uint64_t b_lo = 0, b_h = b_lo + 4 * n, b_m = b_h + 4 * n, b_l = b_m + 4 * n,
                       b_hist = b_l + 4 * n, b_f = b_hist + 4 * n * K, total = b_f + n;
        out.alloc(total);
        SVX_CUDA(cudaMemcpyAsync(dv.p, vxyz, 12 * n, cudaMemcpyHostToDevice, m->stream));
        k_occ_lookup<<<grid256(n), 256, 0, m->stream>>>(
            occ_dev(m), K, dv.p, n, reinterpret_cast<float*>(out.p + b_lo),
            reinterpret_cast<uint32_t*>(out.p + b_h), reinterpret_cast<uint32_t*>(out.p + b_m),
            reinterpret_cast<uint32_t*>(out.p + b_hist), reinterpret_cast<int32_t*>(out.p + b_l),
            out.p + b_f);
        count_launch();
        std::vector<uint8_t> h(total);
        SVX_CUDA(cudaMemcpyAsync(h.data(), out.p, total, cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        if (log_odds) std::memcpy(log_odds, h.data() + b_lo, 4 * n);
        if (hits) std::memcpy(hits, h.data() + b_h, 4 * n);
        if (misses) std::memcpy(misses, h.data() + b_m, 4 * n);
        if (label) std::memcpy(label, h.data() + b_l, 4 * n);
        if (hist) std::memcpy(hist, h.data() + b_hist, 4 * n * K);
        if (found) std::memcpy(found, h.data() + b_f, n);
        dv.release();
        out.release();
    });
}

svx_status svx_occ_block_count(svx_occ* m, uint64_t* n) {
    return api_guard([&] {
        require(m && n, SVX_INVALID_ARGUMENT, "null argument");
        *n = m->n_blocks;
    });
}

svx_status svx_occ_save_mem(svx_occ* m, uint8_t* buf, uint64_t cap, uint64_t* size) {
    return api_guard([&] {
        require(m && size, SVX_INVALID_ARGUMENT, "null argument");
        DevGuard g(m->device);
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        const uint64_t nb = m->n_blocks;
        const int K = m->cfg.num_labels;
        std::vector<uint32_t> hidx(nb);
        if (nb) SVX_CUDA(cudaMemcpy(hidx.data(), m->hist_idx, 4 * nb, cudaMemcpyDeviceToHost));
        uint64_t with_hist = 0;
        for (uint32_t h : hidx) with_hist += h != kInvalid;
        const uint64_t per_block = 12 + 3 * 4 * kBlockVoxels + 1;
        const uint64_t total = 5 + 4 + 4 + 16 + 8 + nb * per_block + with_hist * m->layer_bytes;
        *size = total;
        if (!buf) return;
        require(cap >= total, SVX_INVALID_ARGUMENT, "buffer too small");
        std::vector<uint64_t> keys(nb);
        std::vector<uint32_t> pool(nb * kOccWords);
        std::vector<uint32_t> hist(m->n_layers * kBlockVoxels * uint64_t(K));
        if (nb) {
            SVX_CUDA(cudaMemcpy(keys.data(), m->block_keys, 8 * nb, cudaMemcpyDeviceToHost));
            SVX_CUDA(cudaMemcpy(pool.data(), m->pool.base(), nb * kOccBlockBytes, cudaMemcpyDeviceToHost));
        }
        if (!hist.empty())
            SVX_CUDA(cudaMemcpy(hist.data(), m->hist.base(), 4 * hist.size(), cudaMemcpyDeviceToHost));
        std::vector<uint64_t> order(nb);
        for (uint64_t i = 0; i < nb; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return keys[a] < keys[b]; });
        uint8_t* p = buf;
        auto put = [&](const void* src, size_t len) {
            std::memcpy(p, src, len);
            p += len;
        };
        put("SOCC1", 5);
        put(&m->cfg.voxel_size, 4);
        const uint32_t k32 = uint32_t(K);
        put(&k32, 4);
        put(&m->cfg.l_hit, 4);
        put(&m->cfg.l_miss, 4);
        put(&m->cfg.l_min, 4);
        put(&m->cfg.l_max, 4);
        put(&nb, 8);
        for (uint64_t i : order) {
            int32_t b[3];
            unpack_key(keys[i], b[0], b[1], b[2]);
            put(b, 12);
            put(&pool[i * kOccWords + kBlockVoxels], 3 * 4 * kBlockVoxels);  // L, hits, misses
            const uint8_t hs = hidx[i] != kInvalid;
            put(&hs, 1);
            if (hs) put(&hist[uint64_t(hidx[i]) * kBlockVoxels * K], m->layer_bytes);
        }
    });
}

}  // extern "C"
