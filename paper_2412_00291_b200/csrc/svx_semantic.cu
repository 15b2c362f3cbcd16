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
//   k_sem_update  persistent warps (grid = the resident CTAs), one eighth of a
//                 candidate block per task (2 voxels per lane: short chains of
//                 dependent loads), lane = voxel. Per voxel exactly the reference test sequence (observed,
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

// The voxel's K class probabilities in registers (compile-time K) or in place.
template <int KC>
struct Probs {
    float v[KC];
    __device__ inline void load(const float* p) {
        if constexpr (KC % 4 == 0) {
#pragma unroll
            for (int i = 0; i < KC / 4; ++i) {
                const float4 q = reinterpret_cast<const float4*>(p)[i];
                v[4 * i] = q.x;
                v[4 * i + 1] = q.y;
                v[4 * i + 2] = q.z;
                v[4 * i + 3] = q.w;
            }
        } else if constexpr (KC % 2 == 0) {
#pragma unroll
            for (int i = 0; i < KC / 2; ++i) {
                const float2 q = reinterpret_cast<const float2*>(p)[i];
                v[2 * i] = q.x;
                v[2 * i + 1] = q.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < KC; ++i) v[i] = p[i];
        }
    }
    __device__ inline void store(float* p) const {
        if constexpr (KC % 4 == 0) {
#pragma unroll
            for (int i = 0; i < KC / 4; ++i)
                reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else if constexpr (KC % 2 == 0) {
#pragma unroll
            for (int i = 0; i < KC / 2; ++i) reinterpret_cast<float2*>(p)[i] = make_float2(v[2 * i], v[2 * i + 1]);
        } else {
#pragma unroll
            for (int i = 0; i < KC; ++i) p[i] = v[i];
        }
    }
};

// Likelihood of class k for one pixel (label_to_likelihood / the floored tensor,
// semantic_integrator.cpp:24-39,130-145), divided by its f32 sum as the
// reference does. A label likelihood has two distinct values, so two divisions
// replace K (same quotients).
struct Like {
    const float* tp;  // tensor row or nullptr
    float floor_v, inv_src, lb, lt;
    int label;
    float sum;
    __device__ inline float operator()(int k) const {
        if (tp) {
            const float tk = tp[k];
            return (tk < floor_v ? floor_v : tk) / sum;
        }
        return k == label ? lt : lb;
    }
};

template <int KC>
__device__ inline void bayes_step(float* probs, const Like& like, int K, bool use_bayes) {
    if constexpr (KC > 0) {
        Probs<KC> p;
        p.load(probs);
        if (use_bayes) {  // apply_likelihood (semantic_integrator.cpp:44-52)
            double z = 0.0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                p.v[k] = p.v[k] * like(k);
                z += double(p.v[k]);
            }
            const float inv = float(1.0 / z);
#pragma unroll
            for (int k = 0; k < KC; ++k) p.v[k] = p.v[k] * inv;
        } else {  // apply_latest_argmax (semantic_integrator.cpp:54-59)
            int best = 0;
            float bl = like(0);
            for (int k = 1; k < KC; ++k) {
                const float lk = like(k);
                if (lk > bl) {  // tie -> lower id
                    best = k;
                    bl = lk;
                }
            }
#pragma unroll
            for (int k = 0; k < KC; ++k) p.v[k] = k == best ? 1.f : 0.f;
        }
        p.store(probs);
    } else {
        if (use_bayes) {
            double z = 0.0;
            for (int k = 0; k < K; ++k) {
                const float pk = probs[k] * like(k);
                probs[k] = pk;
                z += double(pk);
            }
            const float inv = float(1.0 / z);
            for (int k = 0; k < K; ++k) probs[k] = probs[k] * inv;
        } else {
            int best = 0;
            float bl = like(0);
            for (int k = 1; k < K; ++k) {
                const float lk = like(k);
                if (lk > bl) {
                    best = k;
                    bl = lk;
                }
            }
            for (int k = 0; k < K; ++k) probs[k] = k == best ? 1.f : 0.f;
        }
    }
}

#ifndef SVX_SEM_PARTS
#define SVX_SEM_PARTS 8
#endif
constexpr int kParts = SVX_SEM_PARTS;  // warp tasks per candidate block
constexpr uint32_t kLayerClaim = 0xFFFFFFFEu;  // semantic layer being allocated

template <int KC>
__global__ void __launch_bounds__(kThreads)
k_sem_update(SemParams sp, HashView h, const uint64_t* __restrict__ block_keys,
             const svx_tsdf_voxel* __restrict__ pool, float* __restrict__ sem,
             uint32_t* __restrict__ sem_idx, const uint32_t* __restrict__ cand,
             const uint16_t* __restrict__ labels, const float* __restrict__ conf,
             const float* __restrict__ tensor, uint8_t* __restrict__ dirty_sem,
             int check, uint32_t* __restrict__ ctr) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    // an image that throws (a voxel passing every test reads a confidence outside
    // [0, 1], label_to_likelihood, semantic_integrator.cpp:24-27,140-142) updates
    // nothing, and no later image of the batch runs
    if (ctr[C_ERR_CONF]) return;
    // check pass: runs only when the image holds such a confidence (or the default is
    // one); evaluates the reference's test sequence and flags, writes nothing else
    if (check && !ctr[C_CONF_MAYBE]) return;
    const uint32_t n_cand = ctr[C_CAND];
    const int K = KC > 0 ? KC : sp.K;
    uint32_t n_upd = 0;
    // task = (candidate block, quarter): 4 voxels per lane keeps each warp's chain of
    // dependent loads short; the grid is sized to the resident CTAs
    for (uint32_t t = warp; t < kParts * n_cand; t += nwarps) {
        const uint32_t idx = cand[t / kParts];
        const int part = int(t % kParts);
        const uint64_t key = block_keys[idx];
        const svx_tsdf_voxel* blk = pool + uint64_t(idx) * kBlockVoxels;
        constexpr int kPer = kBlockVoxels / 32 / kParts;
        uint32_t pix[kPer];
        uint32_t pass = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            pix[j] = 0;
            const int linear = (part * kPer + j) * 32 + lane;
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
        if (check) {
            if (!sp.has_tensor) {
#pragma unroll
                for (int j = 0; j < kPer; ++j) {
                    if (!((pass >> j) & 1u)) continue;
                    const float cf = sp.has_conf ? conf[pix[j]] : sp.default_conf;
                    if (cf < 0.f || cf > 1.f) atomicOr(&ctr[C_ERR_CONF], 1u);
                }
            }
            continue;
        }
        // the block's semantic layer (ensure_semantics): the first part to need it
        // claims it, fills it with 1/K and publishes its index; other parts wait
        uint32_t sid = __ldcg(&sem_idx[idx]);
        if (sid == kInvalid || sid == kLayerClaim) {
            uint32_t claimed = 0;
            if (lane == 0) {
                const uint32_t old = atomicCAS(&sem_idx[idx], kInvalid, kLayerClaim);
                if (old == kInvalid) {
                    sid = atomicAdd(&ctr[C_SEM], 1u);
                    claimed = 1;
                } else {
                    volatile uint32_t* vs = sem_idx + idx;
                    while ((sid = *vs) == kLayerClaim) {
                    }
                }
            }
            sid = __shfl_sync(0xFFFFFFFFu, sid, 0);
            claimed = __shfl_sync(0xFFFFFFFFu, claimed, 0);
            if (claimed) {
                float* layer = sem + uint64_t(sid) * kBlockVoxels * K;
                const float u0 = 1.f / float(K);
                for (int i = lane; i < kBlockVoxels * K; i += 32) layer[i] = u0;
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicExch(&sem_idx[idx], sid);
            }
        }
#pragma unroll 1
        for (int j = 0; j < kPer; ++j) {
            if (!((pass >> j) & 1u)) continue;
            const int linear = (part * kPer + j) * 32 + lane;
            const uint32_t px = pix[j];
            Like like{nullptr, sp.floor_v, 0.f, 0.f, 0.f, -1, 0.f};
            if (sp.has_tensor) {
                like.tp = tensor + uint64_t(px) * K;
                for (int k = 0; k < K; ++k) {
                    const float tk = like.tp[k];
                    like.sum += tk < sp.floor_v ? sp.floor_v : tk;
                }
            } else {
                // label_to_likelihood (semantic_integrator.cpp:24-39): floored, f32 sum in k order
                const float cf = sp.has_conf ? conf[px] : sp.default_conf;
                int label = int(labels[px]);
                float base = K > 1 ? (1.f - cf) / float(K - 1) : 1.f;
                float top = K > 1 ? cf : 1.f;
                if (!(label >= 0 && label < K)) label = -1;
                base = base < sp.floor_v ? sp.floor_v : base;
                top = top < sp.floor_v ? sp.floor_v : top;
                for (int k = 0; k < K; ++k) like.sum += (k == label) ? top : base;
                like.label = label;
                like.lb = base / like.sum;
                like.lt = top / like.sum;
            }
            bayes_step<KC>(sem + (uint64_t(sid) * kBlockVoxels + linear) * K, like, K, sp.use_bayes != 0);
            ++n_upd;
        }
        if (lane == 0) dirty_sem[idx] = 1;
    }
    for (int o = 16; o; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
    if (lane == 0 && n_upd) atomicAdd(&ctr[C_SEM_UPDATED], n_upd);
}

// Flags an image whose confidence image holds a value outside [0, 1] (NaN passes,
// as in the reference's comparison); the check pass of k_sem_update then decides
// whether a voxel actually reads one.
__global__ void k_check_conf(const float* __restrict__ conf, uint64_t n, uint32_t* __restrict__ ctr) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float c = conf[i];
    if (c < 0.f || c > 1.f) ctr[C_CONF_MAYBE] = 1u;
}

}  // namespace

// A sequence of label images, enqueued back to back on the map stream with one
// synchronisation at the end (images are applied in order, each seeing the
// previous ones' updates, exactly as successive integrate_labels calls).
// Labels / confidences / tensors are read from device memory when on_device,
// else copied from the host (asynchronously; pinned memory overlaps).
void run_integrate_labels_batch(svx_map* m, const svx_label_image* imgs, int n, bool on_device,
                                const svx_semantic_cfg& cfg, svx_frame_report* reps) {
    const int K = m->cfg.num_labels;
    for (int i = 0; i < n; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
        if (imgs[i].width <= 0 || imgs[i].height <= 0 || !imgs[i].labels)
            throw Error(SVX_INVALID_ARGUMENT, "label image is empty");
    }
    const bool bad_default = cfg.default_confidence < 0.f || cfg.default_confidence > 1.f;
    if (n <= 0) return;
    // staging for host images: every image of the batch gets its own slice
    uint64_t lbl_n = 0, conf_n = 0, ten_n = 0;
    for (int i = 0; i < n; ++i) {
        const uint64_t P = uint64_t(imgs[i].width) * uint64_t(imgs[i].height);
        lbl_n += P;
        if (imgs[i].confidence) conf_n += P;
        if (imgs[i].prob_tensor) ten_n += P * K;
    }
    if (!on_device) {
        m->lbl.alloc(lbl_n);
        if (conf_n) m->conf.alloc(conf_n);
        if (ten_n) m->tensor.alloc(ten_n);
    }
    m->cand.alloc(std::max<uint64_t>(m->n_blocks, 1));
    m->sem_out.alloc(3ull * n);
    // a block owns at most one layer: map as many layers as there are blocks, so the
    // update kernel never outgrows the pool and no mid-pass synchronisation is needed
    ensure_layers(m, m->n_blocks);
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_ERR_CONF, 0, 4, m->stream));
    uint64_t lo = 0, co = 0, to = 0;
    for (int i = 0; i < n; ++i) {
        const svx_label_image& img = imgs[i];
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
        const uint16_t* lbl = img.labels;
        const float* conf = img.confidence;
        const float* ten = img.prob_tensor;
        if (!on_device) {
            SVX_CUDA(cudaMemcpyAsync(m->lbl.p + lo, img.labels, 2 * P, cudaMemcpyHostToDevice, m->stream));
            lbl = m->lbl.p + lo;
            lo += P;
            if (conf) {
                SVX_CUDA(cudaMemcpyAsync(m->conf.p + co, img.confidence, 4 * P, cudaMemcpyHostToDevice,
                                         m->stream));
                conf = m->conf.p + co;
                co += P;
            }
            if (ten) {
                SVX_CUDA(cudaMemcpyAsync(m->tensor.p + to, img.prob_tensor, 4 * P * K,
                                         cudaMemcpyHostToDevice, m->stream));
                ten = m->tensor.p + to;
                to += P * K;
            }
        }
        // confidence validity: only a voxel that passes every test reads one
        const bool conf_check = !ten && (conf || bad_default);
        if (conf_check) {
            if (conf) {
                SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_CONF_MAYBE, 0, 4, m->stream));
                k_check_conf<<<grid_for(P), kThreads, 0, m->stream>>>(conf, P, m->d_ctr);
                count_launch();
            } else {
                SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_CONF_MAYBE, 0x01, 1, m->stream));
            }
        }
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_CAND, 0, 4, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_SEM_UPDATED, 0, 4, m->stream));
        if (m->n_blocks) {
            {
                ProfMark pm(m, SVX_K_SEM_CULL);
                k_sem_cull<<<grid_for(m->n_blocks), kThreads, 0, m->stream>>>(sp, m->block_keys, m->cand.p,
                                                                              m->d_ctr);
                count_launch();
            }
            {
                ProfMark pm(m, SVX_K_SEM_UPDATE);
                // compile-time class counts keep a voxel's probabilities in registers
                auto kern = &k_sem_update<0>;
                switch (K) {
                    case 2: kern = &k_sem_update<2>; break;
                    case 4: kern = &k_sem_update<4>; break;
                    case 8: kern = &k_sem_update<8>; break;
                    case 10: kern = &k_sem_update<10>; break;
                    case 16: kern = &k_sem_update<16>; break;
                    case 19: kern = &k_sem_update<19>; break;
                    case 20: kern = &k_sem_update<20>; break;
                    case 32: kern = &k_sem_update<32>; break;
                    default: break;
                }
                int per_sm = 0;
                SVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0));
                const unsigned grid = std::max(1u, unsigned(per_sm)) * (persistent_grid(m->device) / 8);
                for (int check = conf_check ? 1 : 0; check >= 0; --check) {
                    kern<<<grid, kThreads, 0, m->stream>>>(
                        sp, hash_view(m), m->block_keys, tsdf_base(m), sem_base(m), m->sem_idx, m->cand.p,
                        lbl, conf, ten, m->dirty + m->cfg.max_blocks, check, m->d_ctr);
                    count_launch();
                }
            }
            SVX_CUDA(cudaGetLastError());
        }
        // per-image results: candidates and updated voxels
        SVX_CUDA(cudaMemcpyAsync(m->sem_out.p + 3 * i, m->d_ctr + C_CAND, 4, cudaMemcpyDeviceToDevice,
                                 m->stream));
        SVX_CUDA(cudaMemcpyAsync(m->sem_out.p + 3 * i + 1, m->d_ctr + C_SEM_UPDATED, 4,
                                 cudaMemcpyDeviceToDevice, m->stream));
        SVX_CUDA(cudaMemcpyAsync(m->sem_out.p + 3 * i + 2, m->d_ctr + C_ERR_CONF, 4,
                                 cudaMemcpyDeviceToDevice, m->stream));
    }
    std::vector<uint32_t> outs(3ull * n);
    SVX_CUDA(cudaMemcpyAsync(outs.data(), m->sem_out.p, 12ull * n, cudaMemcpyDeviceToHost, m->stream));
    sync_counters(m);
    if (m->h_ctr[C_ERR_CONF]) {
        // images before the failing one are complete; the failing one is numbered (the
        // reference numbers a frame before it can throw, semantic_integrator.cpp:93-94)
        // and updated nothing; later images did not run
        int fail = 0;
        while (fail < n && !outs[3 * fail + 2]) ++fail;
        for (int i = 0; i < fail && i < n; ++i) {
            reps[i].frame = m->sem_frames++;
            reps[i].updated_voxels = outs[3 * i + 1];
        }
        m->sem_frames++;
        m->n_layers = m->h_ctr[C_SEM];
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_ERR_CONF, 0, 4, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        throw Error(SVX_INVALID_ARGUMENT, "confidence must be in [0, 1]");
    }
    for (int i = 0; i < n; ++i) {
        reps[i].frame = m->sem_frames++;
        reps[i].updated_voxels = outs[3 * i + 1];
        m->prof_acc.sem_images += 1;
        m->prof_acc.sem_candidates += outs[3 * i];
        m->prof_acc.sem_updated += outs[3 * i + 1];
    }
    m->prof_acc.sem_new_layers += m->h_ctr[C_SEM] - m->n_layers;
    m->n_layers = m->h_ctr[C_SEM];
}

void run_integrate_labels(svx_map* m, const svx_label_image& img, const svx_semantic_cfg& cfg,
                          svx_frame_report* rep) {
    run_integrate_labels_batch(m, &img, 1, false, cfg, rep);
}

}  // namespace svx
