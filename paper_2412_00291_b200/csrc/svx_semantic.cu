// K6: SemanticIntegrator::integrate_labels on the device
// (semantic_integrator.cpp:91-165).
//
// The reference sweeps EVERY allocated block per image (O(map)). Here:
//   k_sem_cull    one thread per allocated block: the block's voxel-centre box is
//                 tested against the camera's half-spaces (z > 0, z <= max_depth,
//                 0 <= u < W, 0 <= v < H, each as an affine function of the
//                 centre) with a conservative margin. A block is dropped only if
//                 all 8 corners are outside one half-space, so no voxel the
//                 reference would update is lost: results are identical.
//   k_sem_update  persistent warps, one candidate block per iteration, lane =
//                 voxel. Per voxel exactly the reference test sequence (observed,
//                 D >= -tau/2, 0 < z <= max_depth, pixel in bounds, optional
//                 raycast occlusion), then likelihood (tensor or label +
//                 confidence, floored and renormalised in f32) and the Bayes
//                 step (f32 products, f64 normaliser, f32 inverse) or the
//                 latest-argmax ablation. The semantic layer of a block is
//                 allocated on first update (ensure_semantics) and filled 1/K.
#include <algorithm>
#include <chrono>

#include "svx_map.hpp"

namespace svx {

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(uint64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

struct SemParams {
    Pose w2c;
    d3 cam_o;
    double fx, fy, cx, cy, max_depth;
    int32_t W, H;
    int K;
    double nu, inv_nu, occ_floor;
    int use_bayes, raycast, has_tensor, has_conf;
    float floor_v, default_conf;
    uint32_t n_blocks;
};

__device__ inline d3 center_of(uint64_t key, int linear, double nu) {
    int32_t bx, by, bz;
    unpack_key(key, bx, by, bz);
    return mk(nu * (bx * kBlockSide + linear % kBlockSide),
              nu * (by * kBlockSide + (linear / kBlockSide) % kBlockSide),
              nu * (bz * kBlockSide + linear / (kBlockSide * kBlockSide)));
}

__global__ void k_sem_cull(SemParams sp, const uint64_t* __restrict__ block_keys,
                           uint32_t* __restrict__ cand, uint32_t* __restrict__ ctr) {
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= sp.n_blocks) return;
    const uint64_t key = block_keys[idx];
    int32_t bx, by, bz;
    unpack_key(key, bx, by, bz);
    // half-space values at the 8 corners of the voxel-centre box
    bool out_zlo = true, out_zhi = true, out_ulo = true, out_uhi = true, out_vlo = true,
         out_vhi = true;
    const bool planes = sp.fx > 0.0 && sp.fy > 0.0;
    for (int c = 0; c < 8; ++c) {
        const int32_t vx = bx * 8 + ((c & 1) ? 7 : 0);
        const int32_t vy = by * 8 + ((c & 2) ? 7 : 0);
        const int32_t vz = bz * 8 + ((c & 4) ? 7 : 0);
        const d3 p = xform(sp.w2c, mk(sp.nu * vx, sp.nu * vy, sp.nu * vz));
        const double mag = fabs(p.x) + fabs(p.y) + fabs(p.z) + 1.0;
        const double eps = 1e-9 * mag;
        if (!(p.z < -eps)) out_zlo = false;
        if (!(p.z > sp.max_depth + eps)) out_zhi = false;
        if (planes) {
            const double su = sp.fx * p.x + sp.cx * p.z;          // u >= 0  <=>  su >= 0
            const double tu = sp.fx * p.x + (sp.cx - sp.W) * p.z;  // u < W   <=>  tu < 0
            const double sv = sp.fy * p.y + sp.cy * p.z;
            const double tv = sp.fy * p.y + (sp.cy - sp.H) * p.z;
            const double e2 = 1e-9 * (fabs(sp.fx * p.x) + (fabs(sp.cx) + sp.W) * fabs(p.z) +
                                      fabs(sp.fy * p.y) + (fabs(sp.cy) + sp.H) * fabs(p.z) + 1.0);
            if (!(su < -e2)) out_ulo = false;
            if (!(tu > e2)) out_uhi = false;
            if (!(sv < -e2)) out_vlo = false;
            if (!(tv > e2)) out_vhi = false;
        } else {
            out_ulo = out_uhi = out_vlo = out_vhi = false;
        }
    }
    if (out_zlo || out_zhi || out_ulo || out_uhi || out_vlo || out_vhi) return;
    cand[warp_agg_inc(&ctr[C_CAND])] = idx;
}

// occluded_along_ray (semantic_integrator.cpp:64-84), TSDF read through the hash.
__device__ bool occluded_along_ray(const SemParams& sp, HashView h,
                                   const svx_tsdf_voxel* __restrict__ pool, d3 center) {
    const d3 dc = sub3(center, sp.cam_o);
    const double voxel_depth = sqrt(dot3(dc, dc));
    const double step = sp.nu;
    const double stop = voxel_depth - 2.5 * sp.nu;
    if (stop <= 2.0 * step) return false;
    const double z = dot3(dc, dc);
    const d3 ray = z > 0.0 ? div3(dc, sqrt(z)) : dc;
    float prev = 0.f;
    bool prev_valid = false;
    for (double t = 2.0 * step; t < stop; t += step) {
        int32_t vc[3];
        world_to_voxel(add3(sp.cam_o, scale3(t, ray)), sp.inv_nu, vc);
        const int32_t bx = block_coord(vc[0]), by = block_coord(vc[1]), bz = block_coord(vc[2]);
        uint32_t s = kInvalid;
        if (key_in_range(bx) && key_in_range(by) && key_in_range(bz))
            s = hash_find(h, pack_key(bx, by, bz));
        if (s == kInvalid) {
            prev_valid = false;
            continue;
        }
        const svx_tsdf_voxel& vox =
            pool[uint64_t(h.vals[s]) * kBlockVoxels + local_linear(vc[0], vc[1], vc[2])];
        if (!(vox.weight > 0.f)) {
            prev_valid = false;
            continue;
        }
        if (prev_valid && prev > 0.f && vox.distance <= 0.f) return true;
        prev = vox.distance;
        prev_valid = true;
    }
    return false;
}

__global__ void __launch_bounds__(kThreads)
k_sem_update(SemParams sp, HashView h, const uint64_t* __restrict__ block_keys,
             const svx_tsdf_voxel* __restrict__ pool, float* __restrict__ sem,
             uint32_t* __restrict__ sem_idx, const uint32_t* __restrict__ cand,
             const uint16_t* __restrict__ labels, const float* __restrict__ conf,
             const float* __restrict__ tensor, uint8_t* __restrict__ dirty_sem,
             uint32_t* __restrict__ ctr) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (ctr[C_ERR_CONF]) return;  // invalid confidence: no voxel is touched
    const uint32_t n_cand = ctr[C_CAND];
    const int K = sp.K;
    uint32_t n_upd = 0;
    for (uint32_t t = warp; t < n_cand; t += nwarps) {
        const uint32_t idx = cand[t];
        const uint64_t key = block_keys[idx];
        const svx_tsdf_voxel* blk = pool + uint64_t(idx) * kBlockVoxels;
        uint32_t pix[16];
        uint32_t pass = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            pix[j] = 0;
            const int linear = j * 32 + lane;
            const float w = blk[linear].weight;
            const float dist = blk[linear].distance;
            if (!(w > 0.f)) continue;
            if (double(dist) < sp.occ_floor) continue;
            const d3 c = center_of(key, linear, sp.nu);
            const d3 pc = xform(sp.w2c, c);
            if (pc.z <= 0.0 || pc.z > sp.max_depth) continue;
            const int u = int(floor(sp.fx * pc.x / pc.z + sp.cx));
            const int v = int(floor(sp.fy * pc.y / pc.z + sp.cy));
            if (u < 0 || u >= sp.W || v < 0 || v >= sp.H) continue;
            if (sp.raycast && occluded_along_ray(sp, h, pool, c)) continue;
            pix[j] = uint32_t(v) * uint32_t(sp.W) + uint32_t(u);
            pass |= 1u << j;
        }
        if (!__any_sync(0xFFFFFFFFu, pass != 0)) continue;
        uint32_t sid = sem_idx[idx];
        if (sid == kInvalid) {
            if (lane == 0) {
                sid = atomicAdd(&ctr[C_SEM], 1u);
                sem_idx[idx] = sid;
            }
            sid = __shfl_sync(0xFFFFFFFFu, sid, 0);
            float* layer = sem + uint64_t(sid) * kBlockVoxels * K;
            const float u0 = 1.f / float(K);
            for (int i = lane; i < kBlockVoxels * K; i += 32) layer[i] = u0;
            __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (!((pass >> j) & 1u)) continue;
            const int linear = j * 32 + lane;
            float* probs = sem + (uint64_t(sid) * kBlockVoxels + linear) * K;
            const uint32_t px = pix[j];
            // likelihood: two closed forms so no K-array lives in registers
            float base = 0.f, top = 0.f, sum = 0.f;
            int label = -1;
            const float* tp = nullptr;
            if (sp.has_tensor) {
                tp = tensor + uint64_t(px) * K;
                for (int k = 0; k < K; ++k) {
                    const float tk = tp[k];
                    sum += tk < sp.floor_v ? sp.floor_v : tk;
                }
            } else {
                // label_to_likelihood (semantic_integrator.cpp:24-39)
                const float cf = sp.has_conf ? conf[px] : sp.default_conf;
                label = int(labels[px]);
                base = K > 1 ? (1.f - cf) / float(K - 1) : 1.f;
                top = K > 1 ? cf : 1.f;
                if (!(label >= 0 && label < K)) label = -1;
                base = base < sp.floor_v ? sp.floor_v : base;
                top = top < sp.floor_v ? sp.floor_v : top;
                for (int k = 0; k < K; ++k) sum += (k == label) ? top : base;
            }
            if (sp.use_bayes) {
                // apply_likelihood (semantic_integrator.cpp:44-52)
                double z = 0.0;
                for (int k = 0; k < K; ++k) {
                    float lk;
                    if (tp) {
                        const float tk = tp[k];
                        lk = (tk < sp.floor_v ? sp.floor_v : tk) / sum;
                    } else {
                        lk = ((k == label) ? top : base) / sum;
                    }
                    const float pk = probs[k] * lk;
                    probs[k] = pk;
                    z += double(pk);
                }
                const float inv = float(1.0 / z);
                for (int k = 0; k < K; ++k) probs[k] = probs[k] * inv;
            } else {
                // apply_latest_argmax (semantic_integrator.cpp:54-59)
                int best = 0;
                float bl = 0.f;
                for (int k = 0; k < K; ++k) {
                    float lk;
                    if (tp) {
                        const float tk = tp[k];
                        lk = (tk < sp.floor_v ? sp.floor_v : tk) / sum;
                    } else {
                        lk = ((k == label) ? top : base) / sum;
                    }
                    if (k == 0 || lk > bl) {  // tie -> lower id
                        best = k;
                        bl = lk;
                    }
                }
                for (int k = 0; k < K; ++k) probs[k] = k == best ? 1.f : 0.f;
            }
            ++n_upd;
        }
        if (lane == 0) dirty_sem[idx] = 1;
    }
    for (int o = 16; o; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
    if (lane == 0 && n_upd) atomicAdd(&ctr[C_SEM_UPDATED], n_upd);
}

__global__ void k_check_conf(const float* __restrict__ conf, uint64_t n, uint32_t* __restrict__ ctr) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float c = conf[i];
    if (c < 0.f || c > 1.f) atomicAdd(&ctr[C_ERR_CONF], 1u);
}

}  // namespace

void run_integrate_labels(svx_map* m, const svx_label_image& img, const svx_semantic_cfg& cfg,
                          svx_frame_report* rep) {
    rep->frame = m->sem_frames++;
    rep->updated_voxels = 0;
    rep->new_blocks = 0;
    const int K = m->cfg.num_labels;
    if (img.width <= 0 || img.height <= 0 || !img.labels)
        throw Error(SVX_INVALID_ARGUMENT, "label image is empty");
    const uint64_t P = uint64_t(img.width) * uint64_t(img.height);
    SemParams sp{};
    const Pose cp = to_pose(img.pose);
    sp.w2c = inverse_pose(cp);
    sp.cam_o = mk(cp.t[0], cp.t[1], cp.t[2]);
    sp.fx = img.fx;
    sp.fy = img.fy;
    sp.cx = img.cx;
    sp.cy = img.cy;
    sp.max_depth = img.max_depth;
    sp.W = img.width;
    sp.H = img.height;
    sp.K = K;
    sp.nu = double(m->cfg.voxel_size);
    sp.inv_nu = 1.0 / double(m->cfg.voxel_size);
    sp.occ_floor = -0.5 * double(m->cfg.truncation);
    sp.use_bayes = cfg.use_bayes != 0;
    sp.raycast = cfg.occlusion == SVX_OCCLUSION_RAYCAST;
    sp.has_tensor = img.prob_tensor != nullptr;
    sp.has_conf = img.confidence != nullptr;
    sp.floor_v = cfg.likelihood_floor;
    sp.default_conf = cfg.default_confidence;
    sp.n_blocks = uint32_t(m->n_blocks);
    if (!sp.has_tensor && !sp.has_conf &&
        (cfg.default_confidence < 0.f || cfg.default_confidence > 1.f))
        throw Error(SVX_INVALID_ARGUMENT, "confidence must be in [0, 1]");

    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_CAND, 0, 4, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_ERR_CONF, 0, 4, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_SEM_UPDATED, 0, 4, m->stream));
    m->lbl.alloc(P);
    SVX_CUDA(cudaMemcpyAsync(m->lbl.p, img.labels, 2 * P, cudaMemcpyHostToDevice, m->stream));
    if (sp.has_conf) {
        m->conf.alloc(P);
        SVX_CUDA(cudaMemcpyAsync(m->conf.p, img.confidence, 4 * P, cudaMemcpyHostToDevice, m->stream));
        if (!sp.has_tensor) {
            k_check_conf<<<grid_for(P), kThreads, 0, m->stream>>>(m->conf.p, P, m->d_ctr);
            count_launch();
        }
    }
    if (sp.has_tensor) {
        m->tensor.alloc(P * K);
        SVX_CUDA(cudaMemcpyAsync(m->tensor.p, img.prob_tensor, 4 * P * K, cudaMemcpyHostToDevice,
                                 m->stream));
    }
    m->cand.alloc(std::max<uint64_t>(m->n_blocks, 1));
    // a block owns at most one layer: map as many layers as there are blocks, so the
    // update kernel never outgrows the pool and no mid-pass synchronisation is needed
    ensure_layers(m, m->n_blocks);
    if (m->n_blocks) {
        {
            ProfMark pm(m, SVX_K_SEM_CULL);
            k_sem_cull<<<grid_for(m->n_blocks), kThreads, 0, m->stream>>>(sp, m->block_keys,
                                                                          m->cand.p, m->d_ctr);
            count_launch();
        }
        {
            ProfMark pm(m, SVX_K_SEM_UPDATE);
            k_sem_update<<<persistent_grid(m->device), kThreads, 0, m->stream>>>(
                sp, hash_view(m), m->block_keys, tsdf_base(m), sem_base(m), m->sem_idx, m->cand.p,
                m->lbl.p, sp.has_conf ? m->conf.p : nullptr, sp.has_tensor ? m->tensor.p : nullptr,
                m->dirty + m->cfg.max_blocks, m->d_ctr);
            count_launch();
        }
        SVX_CUDA(cudaGetLastError());
    }
    sync_counters(m);
    if (m->h_ctr[C_ERR_CONF]) throw Error(SVX_INVALID_ARGUMENT, "confidence must be in [0, 1]");
    const uint32_t n_cand = m->h_ctr[C_CAND];
    rep->updated_voxels = m->h_ctr[C_SEM_UPDATED];
    m->prof_acc.sem_images += 1;
    m->prof_acc.sem_candidates += n_cand;
    m->prof_acc.sem_updated += m->h_ctr[C_SEM_UPDATED];
    m->prof_acc.sem_new_layers += m->h_ctr[C_SEM] - m->n_layers;
    m->n_layers = m->h_ctr[C_SEM];
}

}  // namespace svx
