// Map export to a labelled triangle mesh on the device: extract_mesh and the
// IncrementalMesher's re-mesh (proj/src/mesh.cpp:105-287), bit-identical output.
//
// The reference meshes each block on a CPU thread (marching cubes over the 512
// cells whose base corner lies in the block, a per-block edge -> vertex hash), then
// stitches the blocks in sorted order through a global edge hash, so a vertex's
// global index is its FIRST appearance in the traversal
//     blocks in sorted key order  >  cells in linear (z, y, x) order  >  edges 0..11.
// Here no hash is needed. A lattice edge with a sign change is referenced by the
// usable cells among the (up to) 4 cells that share it, and every one of them has
// it in its edge mask (the mask bit only depends on the two endpoint signs). Its
// vertex therefore belongs to the referencing cell with the smallest traversal index
// T = rank(block) * 512 + linear, and vertices sort by (T, edge). So:
//   k_mesh_nbr    per (mesh block, 27 neighbours): pool index and mesh rank of each
//                 neighbour block (one hash probe each).
//   k_mesh_case   CTA per mesh block: stages the 9x9x9 corner lattice (D and the
//                 weight test) of the block and its 7 upper neighbours in shared
//                 memory; cell case bytes (0 = unusable or no crossing).
//   k_mesh_own    CTA per mesh block: which of a cell's crossing edges it owns (no
//                 referencing candidate with a smaller T), CTA scan of owned-edge
//                 counts -> per-cell (local vertex offset | owned mask); per-block
//                 vertex and face totals.
//   (device exclusive scans of the per-block totals; one host sync sizes the output)
//   k_mesh_emit   CTA per mesh block: owned vertices (make_edge_vertex, mesh.cpp:52-95:
//                 position, normal, label) and faces (the case's triangles with each
//                 edge resolved to its owner's vertex index, emitted i0, i2, i1).
// Traffic: the TSDF pool is read once (plus the neighbour faces), intermediates are
// 5 B per cell; output is 25 B per vertex + 12 B per face.
#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "svx_map.hpp"
#include "svx_mc_tables.h"

namespace svx {

namespace {

constexpr int kCells = 512;
constexpr uint8_t kUnlabeledLabel = 255;  // kUnlabeled, types.hpp:32

__constant__ uint16_t c_edge_mask[256];
__constant__ int8_t c_tris[256][16];
__constant__ uint8_t c_ntri[256];

struct MeshTables {
    uint16_t edge_mask[256];
    int8_t tris[256][16];
    uint8_t ntri[256];
};

void upload_tables(int device) {
    static bool done[64] = {};
    if (device < 64 && done[device]) return;
    MeshTables t{};
    for (int c = 0; c < 256; ++c) {
        t.edge_mask[c] = mc_edge_mask(c);
        const char* s = kMcTris[c];
        int n = 0;
        for (; s[n]; ++n) t.tris[c][n] = int8_t(s[n] <= '9' ? s[n] - '0' : s[n] - 'a' + 10);
        for (int i = n; i < 16; ++i) t.tris[c][i] = -1;
        t.ntri[c] = uint8_t(n / 3);
    }
    SVX_CUDA(cudaMemcpyToSymbol(c_edge_mask, t.edge_mask, sizeof t.edge_mask));
    SVX_CUDA(cudaMemcpyToSymbol(c_tris, t.tris, sizeof t.tris));
    SVX_CUDA(cudaMemcpyToSymbol(c_ntri, t.ntri, sizeof t.ntri));
    if (device < 64) done[device] = true;
}

// neighbour index of a block offset in {-1, 0, 1}^3
__host__ __device__ inline int nb27(int ox, int oy, int oz) { return (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1); }

// Lattice edge of cell-local edge e: base corner offset (the lower endpoint) and
// axis, packed 5 bits per edge at compile time from the host tables.
constexpr uint64_t pack_edge_geom() {
    uint64_t g = 0;
    for (int e = 0; e < 12; ++e) {
        const int a = kMcEdge[e][0], b = kMcEdge[e][1];
        const int ax = kMcCorner[a][0] < kMcCorner[b][0] ? kMcCorner[a][0] : kMcCorner[b][0];
        const int ay = kMcCorner[a][1] < kMcCorner[b][1] ? kMcCorner[a][1] : kMcCorner[b][1];
        const int az = kMcCorner[a][2] < kMcCorner[b][2] ? kMcCorner[a][2] : kMcCorner[b][2];
        const int axis = kMcCorner[a][0] != kMcCorner[b][0] ? 0 : (kMcCorner[a][1] != kMcCorner[b][1] ? 1 : 2);
        g |= uint64_t(ax | ay << 1 | az << 2 | axis << 3) << (5 * e);
    }
    return g;
}
constexpr uint64_t kEdgeGeom = pack_edge_geom();
__device__ inline void edge_geom(int e, int& bx, int& by, int& bz, int& axis) {
    const uint32_t g = uint32_t(kEdgeGeom >> (5 * e)) & 31u;
    bx = g & 1;
    by = (g >> 1) & 1;
    bz = (g >> 2) & 1;
    axis = int(g >> 3);
}
// corner c of a cell: offsets (0,0,0) (1,0,0) (1,1,0) (0,1,0) (0,0,1) (1,0,1) (1,1,1) (0,1,1)
__host__ __device__ constexpr int corner_x(int c) { return (c ^ (c >> 1)) & 1; }
__host__ __device__ constexpr int corner_y(int c) { return (c >> 1) & 1; }
__host__ __device__ constexpr int corner_z(int c) { return (c >> 2) & 1; }
static_assert(corner_x(2) == kMcCorner[2][0] && corner_x(7) == kMcCorner[7][0] &&
                  corner_x(5) == kMcCorner[5][0] && corner_y(3) == kMcCorner[3][1] &&
                  corner_z(4) == kMcCorner[4][2],
              "corner numbering");
// Cell-local edge id of the lattice edge along `axis` whose base is at offset
// (ox, oy, oz) in {0,1}^3 (0 along axis) from the cell base.
__device__ inline int edge_id(int axis, int ox, int oy, int oz) {
    if (axis == 0) return oy ? (oz ? 6 : 2) : (oz ? 4 : 0);
    if (axis == 1) return ox ? (oz ? 5 : 1) : (oz ? 7 : 3);
    return ox ? (oy ? 10 : 9) : (oy ? 11 : 8);
}

struct MeshParams {
    uint32_t R;  // mesh blocks
    float min_weight;
    int reserved;  // reserved "unlabeled" class id or -1
    int K;
    double nu;
};

__global__ void k_mesh_setrank(const uint32_t* __restrict__ pidx, uint32_t R,
                               uint32_t* __restrict__ rank_of_pool, uint32_t value_or_rank) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const uint32_t p = pidx[r];
    if (p != kInvalid) rank_of_pool[p] = value_or_rank == 0 ? r : kInvalid;
}

__global__ void k_mesh_nbr(HashView h, const uint64_t* __restrict__ keys, uint32_t R,
                           const uint32_t* __restrict__ rank_of_pool, uint32_t* __restrict__ nb_pool,
                           uint32_t* __restrict__ nb_rank) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= uint64_t(R) * 27) return;
    const uint32_t r = uint32_t(i / 27);
    const int n = int(i % 27);
    int32_t bx, by, bz;
    unpack_key(keys[r], bx, by, bz);
    bx += n % 3 - 1;
    by += (n / 3) % 3 - 1;
    bz += n / 9 - 1;
    uint32_t p = kInvalid;
    if (key_in_range(bx) && key_in_range(by) && key_in_range(bz)) {
        const uint32_t s = hash_find(h, pack_key(bx, by, bz));
        if (s != kInvalid) p = h.vals[s];
    }
    nb_pool[i] = p;
    nb_rank[i] = p == kInvalid ? kInvalid : rank_of_pool[p];
}

constexpr int kWarpsPerCta = 8;  // mesh blocks per CTA in the warp-per-block kernels

// Case byte of every cell (mesh.cpp:143-160), one WARP per mesh block: the warp
// stages the block's 9x9x9 corner lattice (D and the weight test; the block and its
// 7 upper neighbours) in shared memory, then each lane classifies 16 cells. A cell is
// usable when all 8 corners exist with !(weight < min_weight); bit c set when corner
// c has distance < 0; 0 = no geometry (unusable, or edge mask empty). No CTA-wide
// barrier: blocks are independent, and at ~50k blocks per map the per-CTA cost of a
// 512-thread block-per-CTA layout dominated.
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_mesh_case(MeshParams mp, const uint32_t* __restrict__ nb_pool,
                                                                  const svx_tsdf_voxel* __restrict__ pool,
                                                                  uint8_t* __restrict__ cases,
                                                                  uint8_t* __restrict__ block_active) {
    __shared__ float sd[kWarpsPerCta][9 * 9 * 9];
    __shared__ uint8_t sok[kWarpsPerCta][9 * 9 * 9 + 7];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = blockIdx.x * kWarpsPerCta + w;
    if (r >= mp.R) return;
    uint32_t nbp = kInvalid;  // lane c < 8: pool index of upper neighbour c
    if (lane < 8) nbp = nb_pool[uint64_t(r) * 27 + nb27(lane & 1, (lane >> 1) & 1, lane >> 2)];
    const uint32_t own = __shfl_sync(0xFFFFFFFFu, nbp, 0);
    uint8_t* out = cases + uint64_t(r) * kCells;
    if (own == kInvalid) {  // block absent from the map: no cells
        reinterpret_cast<uint4*>(out)[lane] = make_uint4(0, 0, 0, 0);
        if (lane == 0) block_active[r] = 0;
        return;
    }
    for (int q = lane; q < 729; q += 32) {
        const int x = q % 9, y = (q / 9) % 9, z = q / 81;
        const uint32_t p = __shfl_sync(__activemask(), nbp, (x >> 3) | ((y >> 3) << 1) | ((z >> 3) << 2));
        float d = 0.f;
        uint8_t ok = 0;
        if (p != kInvalid) {
            const svx_tsdf_voxel* v = pool + uint64_t(p) * kBlockVoxels + ((x & 7) + 8 * (y & 7) + 64 * (z & 7));
            d = __ldg(&v->distance);  // 20-byte voxels: 4-byte aligned only
            ok = !(__ldg(&v->weight) < mp.min_weight);
        }
        sd[w][q] = d;
        sok[w][q] = ok;
    }
    __syncwarp();
    bool any = false;
    uint32_t word[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // cells 16*lane .. 16*lane+15
        const int c = 16 * lane + j;
        const int x = c & 7, y = (c >> 3) & 7, z = c >> 6;
        int cube = 0;
        bool usable = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int q = (x + corner_x(k)) + 9 * (y + corner_y(k)) + 81 * (z + corner_z(k));
            usable = usable && sok[w][q];
            if (sd[w][q] < 0.f) cube |= 1 << k;
        }
        const uint32_t b = (usable && c_edge_mask[cube]) ? uint32_t(cube) : 0u;
        any = any || b;
        word[j >> 2] |= b << (8 * (j & 3));
    }
    reinterpret_cast<uint4*>(out)[lane] = make_uint4(word[0], word[1], word[2], word[3]);
    const bool act = __any_sync(0xFFFFFFFFu, any);
    if (lane == 0) block_active[r] = act;
}

// Smallest traversal index among the cells referencing cell-local edge e of the cell
// (lx, ly, lz) of block r (the cell itself included; its T is `self_t`). Also returns
// the owner's rank, linear and its local id of the edge.
struct Owner {
    uint64_t t;
    uint32_t rank;
    int lin, e;
};
__device__ inline Owner edge_owner(int e, int lx, int ly, int lz, uint32_t r, const uint32_t* snr,
                                   const uint8_t* __restrict__ cases) {
    int ox, oy, oz, axis;
    edge_geom(e, ox, oy, oz, axis);
    Owner best{uint64_t(r) * kCells + (lx + 8 * ly + 64 * lz), r, lx + 8 * ly + 64 * lz, e};
    // candidate cells: base = edge base - d, d in {0,1} on the two other axes
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int d1 = k & 1, d2 = k >> 1;
        int dx = 0, dy = 0, dz = 0;
        if (axis == 0) { dy = d1; dz = d2; }
        else if (axis == 1) { dx = d1; dz = d2; }
        else { dx = d1; dy = d2; }
        const int cx = lx + ox - dx, cy = ly + oy - dy, cz = lz + oz - dz;  // in [-1, 8]
        if (cx == lx && cy == ly && cz == lz) continue;
        const int bx = cx < 0 ? -1 : (cx > 7 ? 1 : 0);
        const int by = cy < 0 ? -1 : (cy > 7 ? 1 : 0);
        const int bz = cz < 0 ? -1 : (cz > 7 ? 1 : 0);
        const uint32_t cr = snr[nb27(bx, by, bz)];
        if (cr == kInvalid) continue;
        const int clin = (cx & 7) + 8 * (cy & 7) + 64 * (cz & 7);
        if (!cases[uint64_t(cr) * kCells + clin]) continue;
        const uint64_t ct = uint64_t(cr) * kCells + clin;
        if (ct < best.t) best = Owner{ct, cr, clin, edge_id(axis, ox + (lx - cx), oy + (ly - cy), oz + (lz - cz))};
    }
    return best;
}

// Per cell: owned-edge mask and face count; one CTA scan of (owned << 16 | faces)
// gives the cell's local vertex and face offsets. Cells with geometry are appended to
// the active-cell list (any order: an entry carries its own offsets). Blocks without
// geometry (k_mesh_case's flag) leave at once.
__global__ void __launch_bounds__(kCells) k_mesh_own(const uint32_t* __restrict__ nb_rank,
                                                    const uint8_t* __restrict__ cases,
                                                    const uint8_t* __restrict__ block_active,
                                                    uint32_t* __restrict__ cellinfo,
                                                    unsigned long long* __restrict__ vcount,
                                                    unsigned long long* __restrict__ fcount,
                                                    uint4* __restrict__ active, uint32_t active_cap,
                                                    uint32_t* __restrict__ n_active) {
    using Scan = cub::BlockScan<uint32_t, kCells>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t snr[27];
    const uint32_t r = blockIdx.x;
    const int t = threadIdx.x;
    if (!block_active[r]) {
        if (t == 0) vcount[r] = fcount[r] = 0;
        return;
    }
    if (t < 27) snr[t] = nb_rank[uint64_t(r) * 27 + t];
    __syncthreads();
    const int cube = cases[uint64_t(r) * kCells + t];
    uint32_t mask = 0;
    if (cube) {
        const uint64_t self = uint64_t(r) * kCells + t;
        const int lx = t & 7, ly = (t >> 3) & 7, lz = t >> 6;
        uint32_t em = c_edge_mask[cube];
        while (em) {
            const int e = __ffs(em) - 1;
            em &= em - 1;
            if (edge_owner(e, lx, ly, lz, r, snr, cases).t == self) mask |= 1u << e;
        }
    }
    const uint32_t nf = cube ? c_ntri[cube] : 0u;
    uint32_t off, total;
    Scan(tmp).ExclusiveSum((uint32_t(__popc(mask)) << 16) | nf, off, total);
    if (t == 0) {
        vcount[r] = total >> 16;
        fcount[r] = total & 0xFFFFu;
    }
    cellinfo[uint64_t(r) * kCells + t] = (off >> 16) | (mask << 12);
    const bool act = cube != 0;
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, act);
    if (!ballot) return;
    const int lane = t & 31;
    uint32_t pos = 0;
    if (lane == 0) pos = atomicAdd(n_active, uint32_t(__popc(ballot)));
    pos = __shfl_sync(0xFFFFFFFFu, pos, 0) + __popc(ballot & ((1u << lane) - 1));
    if (act && pos < active_cap)
        active[pos] = make_uint4(r, uint32_t(t) | (uint32_t(cube) << 9), (off >> 16) | (mask << 12),
                                 off & 0xFFFFu);
}

struct MeshOut {
    float* verts;
    float* normals;
    uint8_t* labels;
    uint32_t* faces;
};

__device__ inline float nonzero_distance(float d) {  // mesh.cpp:44-48
    constexpr float eps = 1e-5f;
    if (d > -eps && d < eps) return d < 0.f ? -eps : eps;
    return d;
}

// Thread per active cell: its owned vertices (make_edge_vertex, mesh.cpp:52-95:
// position, normal, label) and its faces (table triangles, each edge resolved to its
// owner cell's vertex index, emitted i0, i2, i1: mesh.cpp:179-189).
__global__ void __launch_bounds__(256) k_mesh_emit(
    MeshParams mp, const uint4* __restrict__ active, uint32_t n_active,
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ nb_pool,
    const uint32_t* __restrict__ nb_rank, const uint8_t* __restrict__ cases,
    const uint32_t* __restrict__ cellinfo, const unsigned long long* __restrict__ vbase,
    const unsigned long long* __restrict__ fbase, const svx_tsdf_voxel* __restrict__ pool,
    const float* __restrict__ sem, const uint32_t* __restrict__ sem_idx, MeshOut out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_active) return;
    const uint4 a = active[i];
    const uint32_t r = a.x;
    const int t = int(a.y & 511u), cube = int(a.y >> 9);
    const uint32_t loff = a.z & 0xFFFu, mask = a.z >> 12, foff = a.w;
    const uint32_t* snr = nb_rank + uint64_t(r) * 27;
    const uint32_t* snp = nb_pool + uint64_t(r) * 27;
    const int lx = t & 7, ly = (t >> 3) & 7, lz = t >> 6;
    int32_t kx, ky, kz;
    unpack_key(keys[r], kx, ky, kz);
    const int32_t gx = kx * kBlockSide + lx, gy = ky * kBlockSide + ly, gz = kz * kBlockSide + lz;
    const uint64_t vb = vbase[r] + loff;

    // ---- owned vertices, in edge order
    uint32_t om = mask;
    uint32_t j = 0;
    while (om) {
        const int e = __ffs(om) - 1;
        om &= om - 1;
        int ox, oy, oz, axis;
        edge_geom(e, ox, oy, oz, axis);
        // lower endpoint a (the edge base) and upper endpoint b, cell-relative in [0, 8]
        const int ax = lx + ox, ay = ly + oy, az = lz + oz;
        const int bx2 = ax + (axis == 0), by2 = ay + (axis == 1), bz2 = az + (axis == 2);
        const uint32_t pa = __ldg(&snp[nb27(ax >> 3, ay >> 3, az >> 3)]);
        const uint32_t pb = __ldg(&snp[nb27(bx2 >> 3, by2 >> 3, bz2 >> 3)]);
        const int la = (ax & 7) + 8 * (ay & 7) + 64 * (az & 7);
        const int lb = (bx2 & 7) + 8 * (by2 & 7) + 64 * (bz2 & 7);
        const svx_tsdf_voxel va = pool[uint64_t(pa) * kBlockVoxels + la];
        const svx_tsdf_voxel vbx = pool[uint64_t(pb) * kBlockVoxels + lb];
        const float dl = nonzero_distance(va.distance);
        const float dh = nonzero_distance(vbx.distance);
        const float tt = dl / (dl - dh);
        const int32_t A[3] = {gx + ox, gy + oy, gz + oz};
        const int32_t B[3] = {A[0] + (axis == 0), A[1] + (axis == 1), A[2] + (axis == 2)};
        const uint64_t vi = vb + j;
        float n[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float cl = float(mp.nu * double(A[c]));  // voxel_center(...).cast<float>()
            const float ch = float(mp.nu * double(B[c]));
            out.verts[3 * vi + c] = cl + tt * (ch - cl);
            n[c] = (1.f - tt) * va.gradient[c] + tt * vbx.gradient[c];
        }
        const float norm = sqrtf((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out.normals[3 * vi + c] = norm > 1e-8f ? n[c] / norm : (c == 2 ? 1.f : 0.f);
        uint8_t label = kUnlabeledLabel;
        const uint32_t sa = sem_idx[pa], sb = sem_idx[pb];
        if (sa != kInvalid && sb != kInvalid) {
            const int K = mp.K;
            const float* pl = sem + (uint64_t(sa) * kBlockVoxels + la) * K;
            const float* ph = sem + (uint64_t(sb) * kBlockVoxels + lb) * K;
            const float prior = 1.f / float(K);
            bool lp = true, hp = true;
            for (int k = 0; k < K; ++k) {
                lp = lp && pl[k] == prior;
                hp = hp && ph[k] == prior;
            }
            if (!lp && !hp) {
                int best = 0;
                float best_p = -1.f;
                for (int k = 0; k < K; ++k) {
                    const float p = (1.f - tt) * pl[k] + tt * ph[k];
                    if (p > best_p) {  // tie -> lower class id
                        best_p = p;
                        best = k;
                    }
                }
                label = best == mp.reserved ? kUnlabeledLabel : uint8_t(best);
            }
        }
        out.labels[vi] = label;
        ++j;
    }

    // ---- faces
    uint32_t vid[12];
    uint32_t em = c_edge_mask[cube];
    while (em) {
        const int e = __ffs(em) - 1;
        em &= em - 1;
        if (mask >> e & 1) {
            vid[e] = uint32_t(vb + __popc(mask & ((1u << e) - 1)));
        } else {
            const Owner o = edge_owner(e, lx, ly, lz, r, snr, cases);
            const uint32_t oi = cellinfo[uint64_t(o.rank) * kCells + o.lin];
            vid[e] = uint32_t(vbase[o.rank] + (oi & 0xFFFu) + __popc((oi >> 12) & ((1u << o.e) - 1)));
        }
    }
    const uint64_t fb = fbase[r] + foff;
    const uint32_t nf = c_ntri[cube];
    for (uint32_t k = 0; k < nf; ++k) {
        const uint32_t i0 = vid[c_tris[cube][3 * k]], i1 = vid[c_tris[cube][3 * k + 1]],
                       i2 = vid[c_tris[cube][3 * k + 2]];
        out.faces[3 * (fb + k) + 0] = i0;
        out.faces[3 * (fb + k) + 1] = i2;
        out.faces[3 * (fb + k) + 2] = i1;
    }
}

__global__ void k_mesh_keys_pidx(HashView h, const uint64_t* __restrict__ keys, uint32_t n,
                                 uint32_t* __restrict__ pidx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = hash_find(h, keys[i]);
    pidx[i] = s == kInvalid ? kInvalid : h.vals[s];
}

__global__ void k_iota(uint32_t* __restrict__ p, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

inline unsigned grid256(uint64_t n) { return unsigned((n + 255) / 256); }

}  // namespace

// extract_mesh over the mesh blocks (h_keys sorted unique packed keys, or all
// allocated blocks when h_keys == nullptr). Result left in m->mesh_*.
void run_extract_mesh(svx_map* m, float min_weight, int reserved, const uint64_t* h_keys,
                      uint64_t n_keys, uint64_t* n_vertices, uint64_t* n_faces) {
    upload_tables(m->device);
    MeshState& ms = m->mesh;
    const uint64_t R64 = h_keys ? n_keys : m->n_blocks;
    if (R64 >= (1ull << 31) / 27) throw Error(SVX_INVALID_ARGUMENT, "too many blocks to mesh");
    const uint32_t R = uint32_t(R64);
    ms.n_vertices = ms.n_faces = 0;
    *n_vertices = *n_faces = 0;
    if (R == 0) return;
    cudaStream_t st = m->stream;
    const HashView h = hash_view(m);
    ms.keys.alloc(2 * uint64_t(R));
    ms.pidx.alloc(2 * uint64_t(R));
    uint64_t* keys = ms.keys.p;
    uint32_t* pidx = ms.pidx.p;
    if (h_keys) {
        SVX_CUDA(cudaMemcpyAsync(keys, h_keys, 8 * R64, cudaMemcpyHostToDevice, st));
        k_mesh_keys_pidx<<<grid256(R), 256, 0, st>>>(h, keys, R, pidx);
        count_launch();
    } else {
        // every allocated block, sorted by key (packed key order = BlockCoord order)
        k_iota<<<grid256(R), 256, 0, st>>>(pidx + R, R);
        count_launch();
        size_t bytes = 0;
        SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, m->block_keys, keys, pidx + R, pidx,
                                                 int(R), 0, 3 * kKeyBits, st));
        m->sort_tmp.alloc(bytes);
        SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->sort_tmp.p, bytes, m->block_keys, keys, pidx + R,
                                                 pidx, int(R), 0, 3 * kKeyBits, st));
    }
    if (!ms.rank_of_pool.p || ms.rank_of_pool.n < m->cfg.max_blocks) {
        ms.rank_of_pool.release();
        ms.rank_of_pool.alloc(m->cfg.max_blocks);
        SVX_CUDA(cudaMemsetAsync(ms.rank_of_pool.p, 0xFF, 4ull * m->cfg.max_blocks, st));
    }
    k_mesh_setrank<<<grid256(R), 256, 0, st>>>(pidx, R, ms.rank_of_pool.p, 0);
    count_launch();
    ms.nb_pool.alloc(27ull * R);
    ms.nb_rank.alloc(27ull * R);
    k_mesh_nbr<<<grid256(27ull * R), 256, 0, st>>>(h, keys, R, ms.rank_of_pool.p, ms.nb_pool.p,
                                                   ms.nb_rank.p);
    count_launch();
    k_mesh_setrank<<<grid256(R), 256, 0, st>>>(pidx, R, ms.rank_of_pool.p, 1);  // restore kInvalid
    count_launch();

    MeshParams mp{R, min_weight, reserved, m->cfg.num_labels, double(m->cfg.voxel_size)};
    ms.cases.alloc(uint64_t(R) * kCells);
    ms.cellinfo.alloc(uint64_t(R) * kCells);
    ms.counts.alloc(4ull * (R + 1) + 1);
    unsigned long long* vcount = ms.counts.p;
    unsigned long long* fcount = vcount + (R + 1);
    unsigned long long* vbase = fcount + (R + 1);
    unsigned long long* fbase = vbase + (R + 1);
    ms.block_active.alloc(R);
    const unsigned wgrid = (R + kWarpsPerCta - 1) / kWarpsPerCta;
    k_mesh_case<<<wgrid, 32 * kWarpsPerCta, 0, st>>>(mp, ms.nb_pool.p, tsdf_base(m), ms.cases.p,
                                                     ms.block_active.p);
    count_launch();
    if (!ms.active.p) ms.active.alloc(std::max<uint64_t>(1u << 20, uint64_t(R) * 32));
    SVX_CUDA(cudaMemsetAsync(ms.counts.p + 4ull * (R + 1), 0, 8, st));  // active-cell counter
    uint32_t* n_active = reinterpret_cast<uint32_t*>(ms.counts.p + 4ull * (R + 1));
    k_mesh_own<<<R, kCells, 0, st>>>(ms.nb_rank.p, ms.cases.p, ms.block_active.p, ms.cellinfo.p, vcount,
                                     fcount, ms.active.p,
                                     uint32_t(std::min<uint64_t>(ms.active.n, 0xFFFFFFFFu)), n_active);
    count_launch();
    SVX_CUDA(cudaMemsetAsync(vcount + R, 0, 8, st));
    SVX_CUDA(cudaMemsetAsync(fcount + R, 0, 8, st));
    size_t bytes = 0;
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, vcount, vbase, int(R + 1), st));
    m->sort_tmp.alloc(bytes);
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(m->sort_tmp.p, bytes, vcount, vbase, int(R + 1), st));
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(m->sort_tmp.p, bytes, fcount, fbase, int(R + 1), st));
    unsigned long long tot[3];
    SVX_CUDA(cudaMemcpyAsync(&tot[0], vbase + R, 8, cudaMemcpyDeviceToHost, st));
    SVX_CUDA(cudaMemcpyAsync(&tot[1], fbase + R, 8, cudaMemcpyDeviceToHost, st));
    SVX_CUDA(cudaMemcpyAsync(&tot[2], n_active, 8, cudaMemcpyDeviceToHost, st));
    SVX_CUDA(cudaStreamSynchronize(st));
    if (tot[0] >= (1ull << 32)) throw Error(SVX_CAPACITY, "mesh has more than 2^32 vertices");
    const uint32_t na = uint32_t(tot[2] & 0xFFFFFFFFu);
    if (na > ms.active.n) {  // list too small: grow and redo the (idempotent) ownership pass
        ms.active.release();
        ms.active.alloc(na + na / 4);
        SVX_CUDA(cudaMemsetAsync(n_active, 0, 4, st));
        k_mesh_own<<<R, kCells, 0, st>>>(ms.nb_rank.p, ms.cases.p, ms.block_active.p, ms.cellinfo.p,
                                         vcount, fcount, ms.active.p, uint32_t(ms.active.n), n_active);
        count_launch();
    }
    ms.verts.alloc(3 * tot[0] + 1);
    ms.normals.alloc(3 * tot[0] + 1);
    ms.labels.alloc(tot[0] + 1);
    ms.faces.alloc(3 * tot[1] + 1);
    if (na)
        k_mesh_emit<<<(na + 255) / 256, 256, 0, st>>>(
            mp, ms.active.p, na, keys, ms.nb_pool.p, ms.nb_rank.p, ms.cases.p, ms.cellinfo.p, vbase,
            fbase, tsdf_base(m), sem_base(m), m->sem_idx,
            MeshOut{ms.verts.p, ms.normals.p, ms.labels.p, ms.faces.p});
    count_launch();
    SVX_CUDA(cudaStreamSynchronize(st));
    ms.n_vertices = tot[0];
    ms.n_faces = tot[1];
    *n_vertices = tot[0];
    *n_faces = tot[1];
}

}  // namespace svx
