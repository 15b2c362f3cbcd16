// K3-K5: TsdfIntegrator::integrate_frame on the device (tsdf_integrator.cpp:97-258).
//
//   k_raycast_band   K3+K4. One thread per pixel: q = pose * back_project(u,v,r)
//                    (direction table => bit-exact), band [q - tau r^, q + tau r^],
//                    amortised DDA (tsdf_integrator.hpp:93-135). Per block crossing:
//                    find-or-insert in the open-addressing hash (new block => pool
//                    index from a bump counter), first touch this frame => append
//                    the slot to the frame's touched list. Per visit: set the voxel
//                    bit in the slot's 512-bit mask (RED.OR, consecutive visits in
//                    one 32-voxel word are merged in registers first). This is the
//                    per-scan dedup: visits collapse onto distinct voxels in L2.
//   k_fold           K5. Persistent warps, one touched block per warp iteration,
//                    lane = voxel (coalesced AoS access). For every touched voxel:
//                    own pixel = project_point(T_ws * centre); if it holds a return,
//                    measure that pixel only and fold (Eq. 4-5 accumulate-then-merge,
//                    .cpp:170-248); otherwise flag the voxel for the fallback. New
//                    blocks are written in full (zero-fill fused with the update).
//   k_collect_fb     Fallback voxels only: re-walk the rays, emit (slot, linear,
//   + radix sort     pixel) records for flagged voxels, sort => per-voxel visits in
//   k_fold_fb        ascending (v, u) pixel order, exactly the reference's order
//                    after its chunk-order merge + stable_sort; sequential fold.
#include <cub/device/device_radix_sort.cuh>
#include <math_constants.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "svx_map.hpp"

namespace svx {

struct FrameParams {
    Model m;
    Pose pose, w2s;
    d3 origin;
    double tau, max_range, alpha_eps, nu, inv_nu;
    float min_clamp;
    int nonproj, drop_unreliable, has_normals;
    int32_t shard_rank, shard_world;
    uint32_t frame_serial;
    uint32_t blocks_before;
    uint32_t max_blocks;
    uint32_t rec_cap;
};

namespace {

constexpr int kThreads = 256;

__device__ inline d3 dir_at(const double* __restrict__ dirs, uint32_t p) {
    return mk(__ldg(&dirs[3 * p]), __ldg(&dirs[3 * p + 1]), __ldg(&dirs[3 * p + 2]));
}

// traverse_segment (tsdf_integrator.hpp:93-135); visit(x, y, z) per cell.
template <typename Visit>
__device__ inline void traverse_segment(d3 a, d3 b, double nu, double inv, Visit&& visit) {
    int32_t cur[3], end[3];
    world_to_voxel(a, inv, cur);
    world_to_voxel(b, inv, end);
    d3 dir = sub3(b, a);
    const double len = sqrt(dot3(dir, dir));
    if (len < 1e-12) {
        visit(cur[0], cur[1], cur[2]);
        return;
    }
    dir = div3(dir, len);
    const double dv[3] = {dir.x, dir.y, dir.z};
    const double av[3] = {a.x, a.y, a.z};
    int32_t step[3];
    double t_max[3], t_delta[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (fabs(dv[i]) < 1e-15) {
            step[i] = 0;
            t_max[i] = CUDART_INF;
            t_delta[i] = CUDART_INF;
        } else {
            step[i] = dv[i] > 0 ? 1 : -1;
            const double boundary = nu * (double(cur[i]) + 0.5 * step[i]);
            t_max[i] = (boundary - av[i]) / dv[i];
            t_delta[i] = nu / fabs(dv[i]);
        }
    }
    const uint64_t max_steps = uint64_t(3.0 * len / nu) + 8;
    for (uint64_t n = 0; n < max_steps; ++n) {
        visit(cur[0], cur[1], cur[2]);
        if (cur[0] == end[0] && cur[1] == end[1] && cur[2] == end[2]) return;
        int m = 0;
        if (t_max[1] < t_max[m]) m = 1;
        if (t_max[2] < t_max[m]) m = 2;
        if (t_max[m] > len) return;
        cur[m] += step[m];
        t_max[m] += t_delta[m];
    }
}

// Ray of pixel p through the band (tsdf_integrator.cpp:123-131). Returns false
// when the pixel is skipped.
__device__ inline bool band_of(const FrameParams& f, const float* __restrict__ depth,
                               const uint8_t* __restrict__ valid,
                               const double* __restrict__ dirs, uint32_t p, d3& a, d3& b) {
    const float r = depth[p];
    if (r == 0.f || double(r) > f.max_range) return false;
    if (f.drop_unreliable && f.has_normals && !valid[p]) return false;
    const d3 q = xform(f.pose, scale3(double(r), dir_at(dirs, p)));
    const d3 dq = sub3(q, f.origin);
    const double z = dot3(dq, dq);
    const d3 ray = z > 0.0 ? div3(dq, sqrt(z)) : dq;
    const d3 tr = scale3(f.tau, ray);
    a = sub3(q, tr);
    b = add3(q, tr);
    return true;
}

__global__ void __launch_bounds__(kThreads)
k_raycast_band(FrameParams f, const float* __restrict__ depth, const uint8_t* __restrict__ valid,
               const double* __restrict__ dirs, HashView h, uint64_t* __restrict__ block_keys,
               uint32_t* __restrict__ stamp, uint32_t* __restrict__ touched,
               uint32_t* __restrict__ vmask, uint32_t* __restrict__ ctr) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(f.m.W) * uint32_t(f.m.H)) return;
    d3 a, b;
    if (!band_of(f, depth, valid, dirs, p, a, b)) return;
    warp_agg_inc(&ctr[C_RAYS]);

    uint64_t cur_key = kEmptyKey;
    uint32_t cur_slot = kInvalid;
    uint32_t pend_word = kInvalid, pend_bits = 0;

    traverse_segment(a, b, f.nu, f.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
        const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
        if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) {
            atomicAdd(&ctr[C_ERR_KEY], 1u);
            return;
        }
        const uint64_t key = pack_key(bx, by, bz);
        if (key != cur_key) {
            cur_key = key;
            if (f.shard_world > 1 && owner_of(key, f.shard_world) != f.shard_rank) {
                cur_slot = kInvalid;
            } else {
                int ins = 0;
                cur_slot = hash_insert(h, key, &ins);
                if (cur_slot == kInvalid) {
                    atomicAdd(&ctr[C_ERR_HASH], 1u);
                } else {
                    if (ins) {
                        const uint32_t idx = atomicAdd(&ctr[C_BLOCKS], 1u);
                        h.vals[cur_slot] = idx;
                        if (idx < f.max_blocks) block_keys[idx] = key;
                    }
                    if (atomicExch(&stamp[cur_slot], f.frame_serial) != f.frame_serial) {
                        const uint32_t t = atomicAdd(&ctr[C_TOUCHED], 1u);
                        touched[t] = cur_slot;
                    }
                }
            }
        }
        if (cur_slot == kInvalid) return;
        const int lin = local_linear(x, y, z);
        const uint32_t word = cur_slot * 32u + uint32_t(lin >> 5);
        const uint32_t bit = 1u << (lin & 31);
        if (word == pend_word) {
            pend_bits |= bit;
        } else {
            if (pend_word != kInvalid) atomicOr(&vmask[pend_word], pend_bits);
            pend_word = word;
            pend_bits = bit;
        }
    });
    if (pend_word != kInvalid) atomicOr(&vmask[pend_word], pend_bits);
}

struct Accum {
    double wd, w, wx, wy, wz;
};

// nonprojective_distance (tsdf_integrator.cpp:39-46)
__device__ inline double nonprojective_distance(double psi, double theta, double alpha,
                                                double eps) {
    const double ct = cos(theta);
    if (alpha < eps) return fabs(ct) * psi;
    const double mag = fabs((cos(alpha) - 1.0) * sin(theta) / sin(alpha)) + fabs(ct * psi);
    return psi >= 0.0 ? mag : -mag;
}

// measure lambda (tsdf_integrator.cpp:172-205) for pixel p.
__device__ inline bool measure(const FrameParams& f, const float* __restrict__ depth,
                               const float* __restrict__ normals,
                               const uint8_t* __restrict__ valid, const double* __restrict__ dirs,
                               uint32_t p, d3 center, const svx_tsdf_voxel& vox, Accum& acc) {
    const float dep = depth[p];
    if (dep == 0.f || double(dep) > f.max_range) return false;
    const bool have_normal = f.has_normals && valid[p];
    if (!have_normal && f.drop_unreliable) return false;
    const d3 q = xform(f.pose, scale3(double(dep), dir_at(dirs, p)));
    const d3 qo = sub3(q, f.origin);
    const double range = sqrt(dot3(qo, qo));
    const d3 ray = div3(qo, range);
    const double psi = range - dot3(sub3(center, f.origin), ray);
    if (fabs(psi) > f.tau) return false;
    float nw[3] = {0.f, 0.f, 0.f};
    if (have_normal) {
        const d3 r = matvec(f.pose.R, mk(normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]));
        nw[0] = float(r.x);
        nw[1] = float(r.y);
        nw[2] = float(r.z);
    }
    double d = psi;
    if (f.nonproj && have_normal) {
        float g[3] = {nw[0], nw[1], nw[2]};
        const float gsq = (vox.gradient[0] * vox.gradient[0] + vox.gradient[1] * vox.gradient[1]) +
                          vox.gradient[2] * vox.gradient[2];
        if (vox.weight > 0.f && gsq > 1e-12f) {
            g[0] = vox.gradient[0];
            g[1] = vox.gradient[1];
            g[2] = vox.gradient[2];
        }
        d3 gd = mk(g[0], g[1], g[2]);
        const double gz = dot3(gd, gd);
        if (gz > 0.0) gd = div3(gd, sqrt(gz));
        double ct = dot3(neg3(ray), gd);
        ct = ct < -1.0 ? -1.0 : (1.0 < ct ? 1.0 : ct);
        double ca = dot3(gd, mk(nw[0], nw[1], nw[2]));
        ca = ca < -1.0 ? -1.0 : (1.0 < ca ? 1.0 : ca);
        d = nonprojective_distance(psi, acos(ct), acos(ca), f.alpha_eps);
    }
    // observation_weight (tsdf_integrator.cpp:48-51)
    double wr = (psi + f.tau) / (2.0 * f.tau);
    const double lo = double(f.min_clamp);
    wr = wr < lo ? lo : (1.0 < wr ? 1.0 : wr);
    const float w_obs = float(wr);
    // truncate_distance (tsdf_integrator.hpp:57-59)
    const float gamma = float(d >= 0.0 ? (f.tau < d ? f.tau : d) : (d < -f.tau ? -f.tau : d));
    acc.wd += double(w_obs * gamma);
    acc.w += double(w_obs);
    if (have_normal) {
        acc.wx += double(w_obs * nw[0]);
        acc.wy += double(w_obs * nw[1]);
        acc.wz += double(w_obs * nw[2]);
    }
    return true;
}

// accumulate-then-merge fold (tsdf_integrator.cpp:239-247)
__device__ inline void fold(svx_tsdf_voxel& vox, const Accum& acc) {
    const double w_old = double(vox.weight);
    vox.distance = float((w_old * double(vox.distance) + acc.wd) / (w_old + acc.w));
    vox.weight = float(w_old + acc.w);
    const d3 bl = mk(w_old * double(vox.gradient[0]) + acc.wx, w_old * double(vox.gradient[1]) + acc.wy,
                     w_old * double(vox.gradient[2]) + acc.wz);
    const double nrm = sqrt(dot3(bl, bl));
    if (nrm > 1e-12) {
        vox.gradient[0] = float(bl.x / nrm);
        vox.gradient[1] = float(bl.y / nrm);
        vox.gradient[2] = float(bl.z / nrm);
    }
}

__device__ inline d3 center_of(uint64_t key, int linear, double nu) {
    int32_t bx, by, bz;
    unpack_key(key, bx, by, bz);
    const int32_t x = bx * kBlockSide + linear % kBlockSide;
    const int32_t y = by * kBlockSide + (linear / kBlockSide) % kBlockSide;
    const int32_t z = bz * kBlockSide + linear / (kBlockSide * kBlockSide);
    return mk(nu * x, nu * y, nu * z);
}

__device__ inline svx_tsdf_voxel load_voxel(const svx_tsdf_voxel* p) {
    svx_tsdf_voxel v;
    const float* s = reinterpret_cast<const float*>(p);
    v.distance = s[0];
    v.weight = s[1];
    v.gradient[0] = s[2];
    v.gradient[1] = s[3];
    v.gradient[2] = s[4];
    return v;
}
__device__ inline void store_voxel(svx_tsdf_voxel* p, const svx_tsdf_voxel& v) {
    float* d = reinterpret_cast<float*>(p);
    d[0] = v.distance;
    d[1] = v.weight;
    d[2] = v.gradient[0];
    d[3] = v.gradient[1];
    d[4] = v.gradient[2];
}

__global__ void __launch_bounds__(kThreads)
k_fold(FrameParams f, const float* __restrict__ depth, const float* __restrict__ normals,
       const uint8_t* __restrict__ valid, const double* __restrict__ dirs, HashView h,
       svx_tsdf_voxel* __restrict__ pool, const uint32_t* __restrict__ touched,
       uint32_t* __restrict__ vmask, uint8_t* __restrict__ dirty, uint32_t* __restrict__ ctr) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_touched = ctr[C_TOUCHED];
    uint32_t n_upd = 0, n_fb = 0;
    for (uint32_t t = warp; t < n_touched; t += nwarps) {
        const uint32_t slot = touched[t];
        const uint32_t idx = h.vals[slot];
        const uint64_t key = h.keys[slot];
        const bool is_new = idx >= f.blocks_before;
        svx_tsdf_voxel* blk = pool + uint64_t(idx) * kBlockVoxels;
        uint32_t* mw = vmask + uint64_t(slot) * 32;
        for (int j = 0; j < 16; ++j) {
            const uint32_t word = mw[j];
            const int linear = j * 32 + lane;
            const bool hit = (word >> lane) & 1u;
            svx_tsdf_voxel vox;
            if (is_new) {
                vox = svx_tsdf_voxel{0.f, 0.f, {0.f, 0.f, 0.f}};
            } else if (word) {
                vox = load_voxel(blk + linear);
            }
            bool write = is_new, fb = false;
            if (hit) {
                const d3 c = center_of(key, linear, f.nu);
                int ou, ov;
                double orr;
                if (project_point(xform(f.w2s, c), f.m, ou, ov, orr) &&
                    depth[uint32_t(ov) * f.m.W + ou] != 0.f) {
                    Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
                    if (measure(f, depth, normals, valid, dirs, uint32_t(ov) * f.m.W + ou, c, vox,
                                acc)) {
                        fold(vox, acc);
                        write = true;
                        ++n_upd;
                    }
                } else {
                    fb = true;
                }
            }
            const uint32_t fbw = __ballot_sync(0xFFFFFFFFu, fb);
            n_fb += fb ? 1 : 0;
            if (write) store_voxel(blk + linear, vox);
            if (lane == 0) {
                mw[j] = 0u;
                mw[16 + j] = fbw;
            }
        }
        if (lane == 0) dirty[idx] = 1;
    }
    for (int o = 16; o; o >>= 1) {
        n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
        n_fb += __shfl_xor_sync(0xFFFFFFFFu, n_fb, o);
    }
    if (lane == 0) {
        if (n_upd) atomicAdd(&ctr[C_UPDATED], n_upd);
        if (n_fb) atomicAdd(&ctr[C_FALLBACK], n_fb);
    }
}

// Fallback visit records: (slot << 32) | (linear << 23) | pixel.
__global__ void __launch_bounds__(kThreads)
k_collect_fb(FrameParams f, const float* __restrict__ depth, const uint8_t* __restrict__ valid,
             const double* __restrict__ dirs, HashView h, const uint32_t* __restrict__ vmask,
             unsigned long long* __restrict__ rec, uint32_t* __restrict__ ctr) {
    if (ctr[C_FALLBACK] == 0) return;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(f.m.W) * uint32_t(f.m.H)) return;
    d3 a, b;
    if (!band_of(f, depth, valid, dirs, p, a, b)) return;
    uint64_t cur_key = kEmptyKey;
    uint32_t cur_slot = kInvalid;
    traverse_segment(a, b, f.nu, f.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
        const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
        if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) return;
        const uint64_t key = pack_key(bx, by, bz);
        if (key != cur_key) {
            cur_key = key;
            cur_slot = (f.shard_world > 1 && owner_of(key, f.shard_world) != f.shard_rank)
                           ? kInvalid
                           : hash_find(h, key);
        }
        if (cur_slot == kInvalid) return;
        const int lin = local_linear(x, y, z);
        if (!((vmask[uint64_t(cur_slot) * 32 + 16 + (lin >> 5)] >> (lin & 31)) & 1u)) return;
        const uint32_t pos = atomicAdd(&ctr[C_RECORDS], 1u);
        if (pos < f.rec_cap)
            rec[pos] = (static_cast<unsigned long long>(cur_slot) << 32) |
                       (static_cast<unsigned long long>(lin) << 23) | p;
    });
}

__global__ void __launch_bounds__(kThreads)
k_fold_fb(FrameParams f, const float* __restrict__ depth, const float* __restrict__ normals,
          const uint8_t* __restrict__ valid, const double* __restrict__ dirs, HashView h,
          svx_tsdf_voxel* __restrict__ pool, const unsigned long long* __restrict__ rec,
          uint32_t n, uint32_t* __restrict__ ctr) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t upd = 0;
    if (i < n && (i == 0 || (rec[i - 1] >> 23) != (rec[i] >> 23))) {
        const unsigned long long head = rec[i] >> 23;
        const uint32_t slot = uint32_t(head >> 9);
        const int linear = int(head & 511);
        const uint32_t idx = h.vals[slot];
        const d3 c = center_of(h.keys[slot], linear, f.nu);
        svx_tsdf_voxel* vp = pool + uint64_t(idx) * kBlockVoxels + linear;
        svx_tsdf_voxel vox = load_voxel(vp);
        Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
        bool measured = false;
        for (uint32_t j = i; j < n && (rec[j] >> 23) == head; ++j)
            measured |= measure(f, depth, normals, valid, dirs, uint32_t(rec[j] & 0x7FFFFF), c,
                                vox, acc);
        if (measured) {
            fold(vox, acc);
            store_voxel(vp, vox);
            upd = 1;
        }
    }
    const unsigned any = __ballot_sync(0xFFFFFFFFu, upd);
    if ((threadIdx.x & 31) == 0 && any) atomicAdd(&ctr[C_UPDATED], uint32_t(__popc(any)));
}

// Capacity path: every visited block key of the frame (duplicates allowed).
__global__ void __launch_bounds__(kThreads)
k_collect_keys(FrameParams f, const float* __restrict__ depth, const uint8_t* __restrict__ valid,
               const double* __restrict__ dirs, unsigned long long* __restrict__ out,
               uint32_t cap, uint32_t* __restrict__ ctr) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(f.m.W) * uint32_t(f.m.H)) return;
    d3 a, b;
    if (!band_of(f, depth, valid, dirs, p, a, b)) return;
    uint64_t cur_key = kEmptyKey;
    traverse_segment(a, b, f.nu, f.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
        const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
        if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) return;
        const uint64_t key = pack_key(bx, by, bz);
        if (key == cur_key) return;
        cur_key = key;
        if (f.shard_world > 1 && owner_of(key, f.shard_world) != f.shard_rank) return;
        const uint32_t pos = atomicAdd(&ctr[C_RECORDS], 1u);
        if (pos < cap) out[pos] = key;
    });
}

__global__ void k_mark_dirty(const uint64_t* __restrict__ keys_sorted, uint32_t n, HashView h,
                             uint8_t* __restrict__ dirty) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = hash_find(h, keys_sorted[i]);
    if (s != kInvalid) dirty[h.vals[s]] = 1;
}

inline unsigned grid_for(uint64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

unsigned persistent_grid(int device) {
    static int sms[64] = {0};
    if (!sms[device]) cudaDeviceGetAttribute(&sms[device], cudaDevAttrMultiProcessorCount, device);
    return unsigned(sms[device] * 8);  // 8 CTAs x 8 warps per SM
}

void sort_u64(svx_map* m, unsigned long long* in, unsigned long long* out, uint32_t n) {
    size_t bytes = 0;
    SVX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, in, out, int(n), 0, 64, m->stream));
    m->sort_tmp.alloc(bytes ? bytes : 1);
    SVX_CUDA(cub::DeviceRadixSort::SortKeys(m->sort_tmp.p, bytes, in, out, int(n), 0, 64, m->stream));
}

// CapacityError path (tsdf_integrator.cpp:160-168 + voxel_store.cpp:18-20):
// blocks are allocated in sorted key order until max_blocks is reached; every
// block before the failing one is marked dirty; no voxel is updated.
void capacity_path(svx_map* m, const FrameParams& f0, svx_scan* s) {
    FrameParams f = f0;
    const uint32_t before = f.blocks_before;
    // 1. all visited keys of the frame
    uint32_t cap = uint32_t(std::min<uint64_t>(uint64_t(s->P) * 64, 1u << 30));
    for (;;) {
        m->records.alloc(cap);
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_RECORDS, 0, 4, m->stream));
        k_collect_keys<<<grid_for(s->P), kThreads, 0, m->stream>>>(f, s->depth.p, s->valid.p,
                                                                   s->dirs.p, m->records.p, cap,
                                                                   m->d_ctr);
        count_launch();
        sync_counters(m);
        if (m->h_ctr[C_RECORDS] <= cap) break;
        cap = m->h_ctr[C_RECORDS];
    }
    const uint32_t n = m->h_ctr[C_RECORDS];
    std::vector<unsigned long long> keys(n);
    SVX_CUDA(cudaMemcpy(keys.data(), m->records.p, sizeof(unsigned long long) * n,
                        cudaMemcpyDeviceToHost));
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    // 2. existing blocks (pool [0, before)) keep their indices
    std::vector<unsigned long long> existing(before);
    if (before)
        SVX_CUDA(cudaMemcpy(existing.data(), m->block_keys, sizeof(unsigned long long) * before,
                            cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> ex_sorted = existing;
    std::sort(ex_sorted.begin(), ex_sorted.end());
    std::vector<unsigned long long> alloc_new, dirty_keys;
    uint64_t room = m->cfg.max_blocks > before ? m->cfg.max_blocks - before : 0;
    for (unsigned long long k : keys) {
        const bool exists = std::binary_search(ex_sorted.begin(), ex_sorted.end(), k);
        if (!exists) {
            if (room == 0) break;  // get_or_allocate_block throws here
            alloc_new.push_back(k);
            --room;
        }
        dirty_keys.push_back(k);
    }
    // 3. rebuild the hash from the surviving key set
    const uint64_t total = before + alloc_new.size();
    ensure_blocks(m, total);
    if (!alloc_new.empty())
        SVX_CUDA(cudaMemcpy(m->block_keys + before, alloc_new.data(),
                            sizeof(unsigned long long) * alloc_new.size(), cudaMemcpyHostToDevice));
    m->h_ctr[C_BLOCKS] = uint32_t(total);
    SVX_CUDA(cudaMemcpy(m->d_ctr + C_BLOCKS, &m->h_ctr[C_BLOCKS], 4, cudaMemcpyHostToDevice));
    m->n_blocks = total;
    rebuild_hash(m);
    launch_zero_blocks(m, before, alloc_new.size());
    SVX_CUDA(cudaMemsetAsync(m->vmask, 0, sizeof(uint32_t) * 32ull * m->cap, m->stream));
    if (!dirty_keys.empty()) {
        m->records.alloc(dirty_keys.size());
        SVX_CUDA(cudaMemcpy(m->records.p, dirty_keys.data(),
                            sizeof(unsigned long long) * dirty_keys.size(), cudaMemcpyHostToDevice));
        k_mark_dirty<<<grid_for(dirty_keys.size()), kThreads, 0, m->stream>>>(
            reinterpret_cast<const uint64_t*>(m->records.p), uint32_t(dirty_keys.size()),
            hash_view(m), m->dirty);
        count_launch();
    }
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    throw Error(SVX_CAPACITY, "block budget exhausted (max_blocks = " +
                                  std::to_string(m->cfg.max_blocks) + ")");
}

}  // namespace

void run_integrate(svx_map* m, svx_scan* s, const Pose& pose, const svx_integrator_cfg& cfg,
                   svx_frame_report* rep) {
    rep->frame = m->tsdf_frames++;
    rep->updated_voxels = 0;
    rep->new_blocks = 0;
    if (!(cfg.alpha_epsilon > 0.0)) throw Error(SVX_INVALID_ARGUMENT, "alpha_epsilon must be > 0");
    if (cfg.mode == SVX_NON_PROJECTIVE && !s->has_normals)
        throw Error(SVX_INVALID_ARGUMENT, "non-projective mode needs a normal image");

    FrameParams f{};
    f.m = s->dm;
    f.pose = pose;
    f.w2s = inverse_pose(pose);
    f.origin = mk(pose.t[0], pose.t[1], pose.t[2]);
    f.tau = cfg.truncation > 0.f ? double(cfg.truncation) : double(m->cfg.truncation);
    f.max_range = cfg.max_range;
    f.alpha_eps = cfg.alpha_epsilon;
    f.min_clamp = cfg.min_weight_clamp;
    f.nonproj = cfg.mode == SVX_NON_PROJECTIVE;
    f.drop_unreliable = cfg.drop_unreliable != 0;
    f.has_normals = s->has_normals;
    f.nu = double(m->cfg.voxel_size);
    f.inv_nu = 1.0 / double(m->cfg.voxel_size);
    f.shard_rank = m->shard_rank;
    f.shard_world = m->shard_world;
    f.frame_serial = ++m->frame_serial;
    f.blocks_before = uint32_t(m->n_blocks);
    f.max_blocks = m->cfg.max_blocks;

    const uint32_t P = uint32_t(s->P);
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_TOUCHED, 0, sizeof(uint32_t) * (C_ERR_HASH - C_TOUCHED + 1),
                             m->stream));
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_RAYS, 0, sizeof(uint32_t), m->stream));
    HashView hv = hash_view(m);
    ProfMark* pm = new ProfMark(m, SVX_K_RAYCAST);
    k_raycast_band<<<grid_for(P), kThreads, 0, m->stream>>>(f, s->depth.p, s->valid.p, s->dirs.p,
                                                            hv, m->block_keys, m->stamp,
                                                            m->touched, m->vmask, m->d_ctr);
    count_launch();
    delete pm;
    SVX_CUDA(cudaGetLastError());
    sync_counters(m);
    const uint32_t* c = m->h_ctr;
    if (c[C_ERR_KEY])
        throw Error(SVX_INVALID_ARGUMENT, "block coordinate outside the device key range [-2^20, 2^20)");
    if (c[C_BLOCKS] > m->cfg.max_blocks || c[C_ERR_HASH]) capacity_path(m, f, s);
    ensure_blocks(m, c[C_BLOCKS]);

    {
        ProfMark pf(m, SVX_K_FOLD);
        k_fold<<<persistent_grid(m->device), kThreads, 0, m->stream>>>(
            f, s->depth.p, s->normals.p, s->valid.p, s->dirs.p, hv, tsdf_base(m), m->touched,
            m->vmask, m->dirty, m->d_ctr);
        count_launch();
    }
    SVX_CUDA(cudaGetLastError());
    sync_counters(m);
    if (c[C_FALLBACK]) {
        ProfMark pb(m, SVX_K_FALLBACK);
        uint32_t cap = std::max<uint32_t>(c[C_FALLBACK] * 16u, 1u << 16);
        for (;;) {
            m->records.alloc(cap);
            f.rec_cap = cap;
            SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_RECORDS, 0, 4, m->stream));
            k_collect_fb<<<grid_for(P), kThreads, 0, m->stream>>>(f, s->depth.p, s->valid.p,
                                                                  s->dirs.p, hv, m->vmask,
                                                                  m->records.p, m->d_ctr);
            count_launch();
            sync_counters(m);
            if (c[C_RECORDS] <= cap) break;
            cap = c[C_RECORDS];
        }
        const uint32_t n = c[C_RECORDS];
        if (n) {
            m->records_alt.alloc(n);
            sort_u64(m, m->records.p, m->records_alt.p, n);
            k_fold_fb<<<grid_for(n), kThreads, 0, m->stream>>>(f, s->depth.p, s->normals.p,
                                                               s->valid.p, s->dirs.p, hv,
                                                               tsdf_base(m), m->records_alt.p, n,
                                                               m->d_ctr);
            count_launch();
            SVX_CUDA(cudaGetLastError());
            sync_counters(m);
        }
    }
    m->prof_acc.frames += 1;
    m->prof_acc.rays += c[C_RAYS];
    m->prof_acc.touched_blocks += c[C_TOUCHED];
    m->prof_acc.new_blocks += c[C_BLOCKS] - f.blocks_before;
    m->prof_acc.updated_voxels += c[C_UPDATED];
    m->prof_acc.fallback_voxels += c[C_FALLBACK];
    rep->updated_voxels = c[C_UPDATED];
    rep->new_blocks = c[C_BLOCKS] - f.blocks_before;
    m->n_blocks = c[C_BLOCKS];
}

}  // namespace svx
