// K6: SemanticIntegrator::integrate_labels on the device
// (semantic_integrator.cpp:91-165), for a BATCH of label images (e.g. the 6 cameras of a
// cfg3 frame) fused into one pass over the map.
//
// The reference sweeps every allocated block once per image and, per voxel, multiplies
// the image's likelihood into the voxel's class probabilities. A voxel's result depends
// only on its own state (W, D read, probabilities updated) and the images in their order,
// so a batch of images is applied voxel by voxel: each voxel's TSDF state is read once,
// tested against every image of the batch (the reference's test sequence per image),
// and its probabilities are loaded once, multiplied by the passing images' likelihoods in
// image order and stored once - identical to successive integrate_labels calls.
//   k_sem_cull    one thread per allocated block (the device block count): the block's
//                 voxel-centre box is tested against each image's half-spaces (z > 0,
//                 z <= max_depth, 0 <= u < W, 0 <= v < H, each as an affine function of
//                 the centre) with a conservative margin; a block is a candidate for the
//                 images whose frustum it may touch (bit mask), dropped only when all 8
//                 corners are outside one half-space of every image.
//   k_sem_update  persistent warps, one sixteenth of a candidate block per task, lane =
//                 voxel: observed and D >= -tau/2 (surrogate occlusion), then per image of
//                 the mask: 0 < z <= max_depth, pixel in bounds, optional raycast
//                 occlusion; then the layer (ensure_semantics: allocated on first update
//                 and filled 1/K) and the Bayes steps (f32 products, f64 normaliser, f32
//                 inverse) or the latest-argmax ablation, image by image.
//                 A check pass (same kernel) runs first when an image may read a
//                 confidence outside [0, 1]: label_to_likelihood throws only for a pixel a
//                 passing voxel reads (semantic_integrator.cpp:24-27,140-142), so the pass
//                 flags the first such image; images from it on are not applied.
#include <algorithm>
#include <chrono>
#include <cmath>

#include "svx_map.hpp"

#ifndef SVX_SEM_PREFETCH
#define SVX_SEM_PREFETCH 2
#endif
#ifndef SVX_SEM_PF_LAYER
#define SVX_SEM_PF_LAYER 1
#endif

namespace svx {

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(uint64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

constexpr int kMaxImg = kMaxLabelImages;  // label images fused in one pass
constexpr int kSemOut = 3 * kMaxImg + 1;    // per pass: confidence-map flags, errors, updates; candidates

// One label image (LabelImage, semantic_integrator.hpp:14-26) of a pass.
struct ImgParams {
    Pose w2c;
    d3 cam_o;
    double fx, fy, cx, cy, max_depth;
    int32_t W, H;
    const uint16_t* labels;
    const float* conf;
    const float* tensor;
    int has_tensor, has_conf, conf_maybe;  // conf_maybe: may read a confidence outside [0, 1]
    float reach;  // no voxel farther from the camera than this can pass 0 < z <= max_depth and the bounds
};

struct SemBatch {
    ImgParams img[kMaxImg];
    int n;  // images in this pass
    int K;
    double nu, inv_nu, occ_floor;
    int use_bayes, raycast, any_check;
    float floor_v, default_conf;
    uint32_t pass_id;  // 1-based index of this pass in the batch (confidence errors)
    uint32_t group_frame;  // inside a TSDF frame group: the frame this pass follows, else ~0
};

__device__ inline d3 center_of(uint64_t key, int linear, double nu) {
    int32_t bx, by, bz;
    unpack_key(key, bx, by, bz);
    return mk(nu * (bx * kBlockSide + linear % kBlockSide),
              nu * (by * kBlockSide + (linear / kBlockSide) % kBlockSide),
              nu * (bz * kBlockSide + linear / (kBlockSide * kBlockSide)));
}

// Per block: bit i set when the block may hold a voxel image i can update.
__global__ void __launch_bounds__(kThreads)
k_sem_cull(const __grid_constant__ SemBatch sb, const uint64_t* __restrict__ block_keys,
           const uint32_t* __restrict__ fm, uint2* __restrict__ cand, uint32_t* __restrict__ ctr) {
    if (ctr[C_ABORT]) return;  // the frame group these images follow is rolled back
    const uint32_t nb = ctr[C_BLOCKS];
    // inside a frame group, blocks its later frames allocated do not exist yet for this pass
    // (their voxels are unobserved anyway): skipped without reading them
    const uint32_t before = sb.group_frame == ~0u ? nb : ctr[C_BLOCKS_BEFORE];
    const uint32_t seen = sb.group_frame == ~0u ? 0u : (2u << sb.group_frame) - 1u;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nb; idx += gridDim.x * blockDim.x) {
        if (idx >= before && !(fm[uint64_t(idx) * kMaskWords + kHdrRow * 16] & seen)) continue;
        const uint64_t key = block_keys[idx];
        int32_t bx, by, bz;
        unpack_key(key, bx, by, bz);
        // block centre and half diagonal (of the voxel-centre box): a block farther than
        // the image's reach (a passing voxel has 0 < z <= max_depth and |x / z|, |y / z|
        // within the image, so distance <= max_depth sqrt(1 + ax^2 + ay^2)) cannot hold a
        // voxel it updates: most of the map costs one distance test per image
        const float bcx = float(sb.nu * (bx * 8 + 3.5)), bcy = float(sb.nu * (by * 8 + 3.5)),
                    bcz = float(sb.nu * (bz * 8 + 3.5));
        const float rad = float(sb.nu * 6.07) + 1e-3f;  // sqrt(3) * 3.5 voxels + slack
        uint32_t mask = 0;
        for (int i = 0; i < sb.n; ++i) {
            const ImgParams& ip = sb.img[i];
            {
                const float dx = bcx - float(ip.cam_o.x), dy = bcy - float(ip.cam_o.y), dz = bcz - float(ip.cam_o.z);
                const float reach = ip.reach + rad;
                if (dx * dx + dy * dy + dz * dz > reach * reach) continue;
            }
            // half-space values at the 8 corners of the voxel-centre box
            bool out_zlo = true, out_zhi = true, out_ulo = true, out_uhi = true, out_vlo = true, out_vhi = true;
            const bool planes = ip.fx > 0.0 && ip.fy > 0.0;
            for (int c = 0; c < 8; ++c) {
                const int32_t vx = bx * 8 + ((c & 1) ? 7 : 0);
                const int32_t vy = by * 8 + ((c & 2) ? 7 : 0);
                const int32_t vz = bz * 8 + ((c & 4) ? 7 : 0);
                const d3 p = xform(ip.w2c, mk(sb.nu * vx, sb.nu * vy, sb.nu * vz));
                const double mag = fabs(p.x) + fabs(p.y) + fabs(p.z) + 1.0;
                const double eps = 1e-9 * mag;
                if (!(p.z < -eps)) out_zlo = false;
                if (!(p.z > ip.max_depth + eps)) out_zhi = false;
                if (planes) {
                    const double su = ip.fx * p.x + ip.cx * p.z;          // u >= 0  <=>  su >= 0
                    const double tu = ip.fx * p.x + (ip.cx - ip.W) * p.z;  // u < W   <=>  tu < 0
                    const double sv = ip.fy * p.y + ip.cy * p.z;
                    const double tv = ip.fy * p.y + (ip.cy - ip.H) * p.z;
                    const double e2 = 1e-9 * (fabs(ip.fx * p.x) + (fabs(ip.cx) + ip.W) * fabs(p.z) +
                                              fabs(ip.fy * p.y) + (fabs(ip.cy) + ip.H) * fabs(p.z) + 1.0);
                    if (!(su < -e2)) out_ulo = false;
                    if (!(tu > e2)) out_uhi = false;
                    if (!(sv < -e2)) out_vlo = false;
                    if (!(tv > e2)) out_vhi = false;
                } else {
                    out_ulo = out_uhi = out_vlo = out_vhi = false;
                }
            }
            if (!(out_zlo || out_zhi || out_ulo || out_uhi || out_vlo || out_vhi)) mask |= 1u << i;
        }
        if (mask) cand[warp_agg_inc(&ctr[C_CAND])] = make_uint2(idx, mask);
    }
}

// occluded_along_ray (semantic_integrator.cpp:64-84), TSDF read through the hash.
__device__ bool occluded_along_ray(const SemBatch& sb, d3 cam_o, HashView h, const svx_tsdf_voxel* __restrict__ pool,
                                   d3 center) {
    const d3 dc = sub3(center, cam_o);
    const double voxel_depth = sqrt(dot3(dc, dc));
    const double step = sb.nu;
    const double stop = voxel_depth - 2.5 * sb.nu;
    if (stop <= 2.0 * step) return false;
    const double z = dot3(dc, dc);
    const d3 ray = z > 0.0 ? div3(dc, sqrt(z)) : dc;
    float prev = 0.f;
    bool prev_valid = false;
    for (double t = 2.0 * step; t < stop; t += step) {
        int32_t vc[3];
        world_to_voxel(add3(cam_o, scale3(t, ray)), sb.inv_nu, vc);
        const int32_t bx = block_coord(vc[0]), by = block_coord(vc[1]), bz = block_coord(vc[2]);
        uint32_t s = kInvalid;
        if (key_in_range(bx) && key_in_range(by) && key_in_range(bz)) s = hash_find(h, pack_key(bx, by, bz));
        if (s == kInvalid) {
            prev_valid = false;
            continue;
        }
        const svx_tsdf_voxel& vox = pool[uint64_t(h.vals[s]) * kBlockVoxels + local_linear(vc[0], vc[1], vc[2])];
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

// The voxel's K class probabilities in registers (compile-time K).
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
// semantic_integrator.cpp:24-39,130-145), divided by its f32 sum as the reference does.
// A label likelihood has two distinct values, so two divisions replace K (same quotients).
struct Like {
    const float* tp;  // tensor row or nullptr
    float floor_v, lb, lt;
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

// label_to_likelihood's two quotients for every label of an image without a confidence
// map or a tensor (they depend on the label only): lut[1 + l] = (lb, lt) for l in [-1, K),
// l = -1 for a label outside [0, K). The same f32 operations as make_like.
constexpr int kLutK = 32;  // classes covered by the shared-memory table
__device__ inline float2 label_quotients(const SemBatch& sb, float cf, int label, int K) {
    float base = K > 1 ? (1.f - cf) / float(K - 1) : 1.f;
    float top = K > 1 ? cf : 1.f;
    base = base < sb.floor_v ? sb.floor_v : base;
    top = top < sb.floor_v ? sb.floor_v : top;
    float sum = 0.f;
    for (int k = 0; k < K; ++k) sum += (k == label) ? top : base;
    return make_float2(base / sum, top / sum);
}

__device__ inline Like make_like(const SemBatch& sb, const ImgParams& ip, uint32_t px, int K,
                                 const float2* __restrict__ lut) {
    Like like{nullptr, sb.floor_v, 0.f, 0.f, -1, 0.f};
    if (lut) {
        int label = int(ip.labels[px]);
        if (!(label < K)) label = -1;
        const float2 q = lut[1 + label];
        like.label = label;
        like.lb = q.x;
        like.lt = q.y;
        return like;
    }
    if (ip.has_tensor) {
        like.tp = ip.tensor + uint64_t(px) * K;
        for (int k = 0; k < K; ++k) {
            const float tk = like.tp[k];
            like.sum += tk < sb.floor_v ? sb.floor_v : tk;
        }
    } else {
        // label_to_likelihood (semantic_integrator.cpp:24-39): floored, f32 sum in k order
        const float cf = ip.has_conf ? ip.conf[px] : sb.default_conf;
        int label = int(ip.labels[px]);
        float base = K > 1 ? (1.f - cf) / float(K - 1) : 1.f;
        float top = K > 1 ? cf : 1.f;
        if (!(label >= 0 && label < K)) label = -1;
        base = base < sb.floor_v ? sb.floor_v : base;
        top = top < sb.floor_v ? sb.floor_v : top;
        for (int k = 0; k < K; ++k) like.sum += (k == label) ? top : base;
        like.label = label;
        like.lb = base / like.sum;
        like.lt = top / like.sum;
    }
    return like;
}

// apply_likelihood / apply_latest_argmax (semantic_integrator.cpp:44-59) on registers
template <int KC>
__device__ inline void bayes_regs(Probs<KC>& p, const Like& like, bool use_bayes) {
    if (use_bayes) {
        double z = 0.0;
        if (like.tp) {
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                p.v[k] = p.v[k] * like(k);
                z += double(p.v[k]);
            }
        } else {  // a label likelihood: lt at the label, lb elsewhere (the same products)
            const float lt = like.lt, lb = like.lb;
            const int label = like.label;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                p.v[k] = p.v[k] * (k == label ? lt : lb);
                z += double(p.v[k]);
            }
        }
        // float(1 / z) from the reciprocal estimate when it decides the float
        float inv;
        if (!(z > 1e-300 && z < 1e300 && f32_of_est(rcp_est(z), inv))) inv = float(1.0 / z);
#pragma unroll
        for (int k = 0; k < KC; ++k) p.v[k] = p.v[k] * inv;
    } else {
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
}

// the same in place (class counts without a compile-time specialisation)
__device__ inline void bayes_mem(float* probs, const Like& like, int K, bool use_bayes) {
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

constexpr int kParts = 16;  // warp tasks per candidate block: lane = voxel
constexpr uint32_t kLayerClaim = 0xFFFFFFFEu;  // semantic layer being allocated

// Whether the check pass must evaluate image i: it may read an invalid confidence (an
// invalid default without a map, or a map k_check_conf flagged).
__device__ inline bool needs_check(const ImgParams& ip, const uint32_t* xconf, int i) {
    return ip.conf_maybe && (!ip.has_conf || xconf[i]);
}

// The Bayes steps of one queued voxel (k_sem_update): its probabilities in registers (or in
// place without a compile-time K), the passing images in order.
constexpr uint32_t kQueue = 64;  // voxels per warp queue (a ring: < 32 waiting + one task's 32)
template <int KC>
__device__ inline void bayes_queued(const SemBatch& sb, float* __restrict__ sem, int K, const uint32_t* q_sid,
                                    const uint32_t* q_lp, const uint32_t (*q_pix)[kQueue], uint32_t e, bool lut_ok,
                                    const float2 (*s_lut)[kLutK + 1]) {
    const uint32_t lp = q_lp[e], pass = lp & 0xFFu, linear = lp >> 8;
    float* probs = sem + (uint64_t(q_sid[e]) * kBlockVoxels + linear) * K;
    if constexpr (KC > 0) {
        Probs<KC> p;
        p.load(probs);
#pragma unroll 1
        for (uint32_t r = pass; r; r &= r - 1) {
            const int i = __ffs(r) - 1;
            const ImgParams& ip = sb.img[i];
            const float2* lut = (lut_ok && !ip.has_tensor && !ip.has_conf) ? s_lut[i] : nullptr;
            bayes_regs<KC>(p, make_like(sb, ip, q_pix[i][e], K, lut), sb.use_bayes != 0);
        }
        p.store(probs);
    } else {
#pragma unroll 1
        for (uint32_t r = pass; r; r &= r - 1) {
            const int i = __ffs(r) - 1;
            const ImgParams& ip = sb.img[i];
            const float2* lut = (lut_ok && !ip.has_tensor && !ip.has_conf) ? s_lut[i] : nullptr;
            bayes_mem(probs, make_like(sb, ip, q_pix[i][e], K, lut), K, sb.use_bayes != 0);
        }
    }
}

// xconf[i]: image i's confidence map holds an invalid value; xerr[i]: image i reads one
// (check pass); xupd[i]: voxels image i updated.
template <int KC>
__global__ void __launch_bounds__(kThreads)
k_sem_update(const __grid_constant__ SemBatch sb, HashView h, const uint64_t* __restrict__ block_keys,
             const svx_tsdf_voxel* __restrict__ pool, float* __restrict__ sem, uint32_t* __restrict__ sem_idx,
             const uint2* __restrict__ cand, uint8_t* __restrict__ dirty_sem, int check,
             const uint32_t* __restrict__ xconf, uint32_t* __restrict__ xerr, uint32_t* __restrict__ xupd,
             uint32_t* __restrict__ ctr) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (ctr[C_ABORT]) return;  // the frame group these images follow is rolled back
    // a confidence error of an earlier pass of the batch: nothing more is applied
    const uint32_t err = ctr[C_ERR_CONF];
    if (err && err != sb.pass_id) return;
    int n_apply = sb.n;
    if (check) {
        bool any = false;
        for (int i = 0; i < sb.n; ++i) any |= needs_check(sb.img[i], xconf, i);
        if (!any) return;
    } else {
        // images applied: up to the first one whose check failed (the reference throws in it)
        for (int i = 0; i < sb.n; ++i)
            if (xerr[i]) {
                n_apply = i;
                break;
            }
        if (n_apply == 0) return;
    }
    const uint32_t n_cand = ctr[C_CAND];
    const int K = KC > 0 ? KC : sb.K;
    // the pixel of each (image, voxel) of a warp's task in shared memory: the image loops
    // stay rolled (one copy of the likelihood / Bayes code: unrolled over 8 images the
    // kernel outgrows the instruction cache)
    __shared__ uint32_t s_pix[kThreads / 32][kMaxImg][32];
    uint32_t (*pix)[32] = s_pix[threadIdx.x >> 5];
    // label-only likelihood quotients per image (no confidence map, no tensor)
    __shared__ float2 s_lut[kMaxImg][kLutK + 1];
    const bool lut_ok = K <= kLutK;
    if (lut_ok) {
        for (int e = threadIdx.x; e < n_apply * (K + 1); e += blockDim.x) {
            const int i = e / (K + 1), l = e % (K + 1) - 1;
            s_lut[i][l + 1] = label_quotients(sb, sb.default_conf, l, K);
        }
    }
    __syncthreads();
    // per warp: a ring of voxels waiting for their Bayes steps (layer, voxel | images, pixels)
    __shared__ uint32_t q_sid[kThreads / 32][kQueue], q_lp[kThreads / 32][kQueue];
    __shared__ uint32_t q_pix[kThreads / 32][kMaxImg][kQueue];
    const int wq = threadIdx.x >> 5;
    uint32_t q_head = 0, q_tail = 0;
    uint32_t n_upd = 0;  // lane i < n_apply: voxels image i updated
    const uint32_t n_tasks = kParts * n_cand;
#if SVX_SEM_PREFETCH == 1
    // the next task's candidate, block key and TSDF weight / distance are loaded one
    // iteration ahead (their dependent chain overlaps this task's projections)
    uint2 cd_n = make_uint2(0u, 0u);
    uint64_t key_n = 0;
    float w_n = 0.f, dist_n = 0.f;
    auto fetch = [&](uint32_t tt) {
        if (tt >= n_tasks) return;
        cd_n = cand[tt / kParts];
        key_n = block_keys[cd_n.x];
        const svx_tsdf_voxel* vn = pool + uint64_t(cd_n.x) * kBlockVoxels + int(tt % kParts) * 32 + lane;
        w_n = vn->weight;
        dist_n = vn->distance;
    };
    fetch(warp);
#elif SVX_SEM_PREFETCH == 2
    // the next task's candidate entry is loaded one iteration ahead, and its block key and
    // TSDF voxel are prefetched into L2 once this task's projections are issued
    uint2 cd_n = warp < n_tasks ? cand[warp / kParts] : make_uint2(0u, 0u);
#endif
    for (uint32_t t = warp; t < n_tasks; t += nwarps) {
#if SVX_SEM_PREFETCH == 1
        const uint2 cd = cd_n;
        const uint64_t key = key_n;
        const float w = w_n, dist = dist_n;
        fetch(t + nwarps);
#elif SVX_SEM_PREFETCH == 2
        const uint2 cd = cd_n;
        if (t + nwarps < n_tasks) cd_n = cand[(t + nwarps) / kParts];
        const uint64_t key = block_keys[cd.x];
        const svx_tsdf_voxel* v = pool + uint64_t(cd.x) * kBlockVoxels + int(t % kParts) * 32 + lane;
        const float w = v->weight, dist = v->distance;
#else
        const uint2 cd = cand[t / kParts];
        const uint64_t key = block_keys[cd.x];
        const svx_tsdf_voxel* v = pool + uint64_t(cd.x) * kBlockVoxels + int(t % kParts) * 32 + lane;
        const float w = v->weight, dist = v->distance;
#endif
        const uint32_t idx = cd.x;
        const int linear = int(t % kParts) * 32 + lane;
        uint32_t pass = 0;
        if (w > 0.f && !(double(dist) < sb.occ_floor)) {
            const d3 c = center_of(key, linear, sb.nu);
#pragma unroll 1
            for (int i = 0; i < n_apply; ++i) {
                if (!((cd.y >> i) & 1u)) continue;
                const ImgParams& ip = sb.img[i];
                const d3 pc = xform(ip.w2c, c);
                if (pc.z <= 0.0 || pc.z > ip.max_depth) continue;
                // u = floor(fx x / z + cx), v = floor(fy y / z + cy) (semantic_integrator.cpp:
                // 117-121) from one reciprocal of z: the estimates are within ~3 ulp of the
                // reference's quotients, so floor() is decided unless an estimate lies within
                // the bound of an integer; then the reference's divisions are evaluated
                int u, vv;
                {
                    const double rz = rcp_est(pc.z);
                    const double bu = ip.fx * pc.x * rz, bv = ip.fy * pc.y * rz;
                    const double cu = bu + ip.cx, cv = bv + ip.cy;
                    const double eu = 1e-15 * (fabs(bu) + fabs(cu)) + 1e-300;
                    const double ev = 1e-15 * (fabs(bv) + fabs(cv)) + 1e-300;
                    const double fu = floor(cu), fv = floor(cv);
                    if (cu - eu >= fu && cu + eu < fu + 1.0) u = int(fu);
                    else u = int(floor(ip.fx * pc.x / pc.z + ip.cx));
                    if (cv - ev >= fv && cv + ev < fv + 1.0) vv = int(fv);
                    else vv = int(floor(ip.fy * pc.y / pc.z + ip.cy));
                }
                if (u < 0 || u >= ip.W || vv < 0 || vv >= ip.H) continue;
                if (sb.raycast && occluded_along_ray(sb, ip.cam_o, h, pool, c)) continue;
                pix[i][lane] = uint32_t(vv) * uint32_t(ip.W) + uint32_t(u);
                pass |= 1u << i;
            }
        }
#if SVX_SEM_PREFETCH == 2
        if (t + nwarps < n_tasks) {
            const svx_tsdf_voxel* vn = pool + uint64_t(cd_n.x) * kBlockVoxels + int((t + nwarps) % kParts) * 32 + lane;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vn));
            if (lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(block_keys + cd_n.x));
        }
#endif
        if (!__any_sync(0xFFFFFFFFu, pass != 0)) continue;
        if (check) {  // flag images whose passing voxels read an invalid confidence
#pragma unroll 1
            for (int i = 0; i < n_apply; ++i) {
                if (!((pass >> i) & 1u) || !needs_check(sb.img[i], xconf, i) || sb.img[i].has_tensor) continue;
                const float cf = sb.img[i].has_conf ? sb.img[i].conf[pix[i][lane]] : sb.default_conf;
                if (cf < 0.f || cf > 1.f) atomicOr(&xerr[i], 1u);
            }
            continue;
        }
        // the block's semantic layer (ensure_semantics): the first task to need it claims
        // it, fills it with 1/K and publishes its index; other tasks wait
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
        // the passing voxels join the warp's queue; the Bayes steps run 32 queued voxels at
        // a time on full warps (a task's voxels fail the W / D / frustum tests unevenly)
        {
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, pass != 0u);
            if (pass) {
                const uint32_t e = (q_tail + uint32_t(__popc(m & ((1u << lane) - 1u)))) & (kQueue - 1u);
                q_sid[wq][e] = sid;
                q_lp[wq][e] = (uint32_t(linear) << 8) | pass;
#if SVX_SEM_PF_LAYER
                {  // the voxel's probabilities, read when the queue next runs its Bayes steps
                    const char* pr = reinterpret_cast<const char*>(sem + (uint64_t(sid) * kBlockVoxels + linear) * K);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pr));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pr + 4 * K - 4));
                }
#endif
                for (uint32_t r = pass; r; r &= r - 1) {
                    const int i = __ffs(r) - 1;
                    q_pix[wq][i][e] = pix[i][lane];
                }
            }
            q_tail += uint32_t(__popc(m));
            __syncwarp();
            if (q_tail - q_head >= 32u) {
                bayes_queued<KC>(sb, sem, K, q_sid[wq], q_lp[wq], q_pix[wq], (q_head + lane) & (kQueue - 1u), lut_ok,
                                 s_lut);
                q_head += 32u;
                __syncwarp();
            }
        }
        __syncwarp();
        // per image, the warp's updated voxels: lane i keeps image i's count
        for (int i = 0; i < n_apply; ++i) {
            const uint32_t nu = __reduce_add_sync(0xFFFFFFFFu, (pass >> i) & 1u);
            if (lane == i) n_upd += nu;
        }
        if (lane == 0) dirty_sem[idx] = 1;
    }
    if (!check && q_tail > q_head && uint32_t(lane) < q_tail - q_head)  // the queue's rest
        bayes_queued<KC>(sb, sem, K, q_sid[wq], q_lp[wq], q_pix[wq], (q_head + lane) & (kQueue - 1u), lut_ok, s_lut);
    if (lane < n_apply && n_upd) atomicAdd(&xupd[lane], n_upd);
}

// Flags an image whose confidence map holds a value outside [0, 1] (NaN passes, as in the
// reference's comparison); the check pass of k_sem_update then decides whether a voxel
// actually reads one.
__global__ void k_check_conf(const float* __restrict__ conf, uint64_t n, uint32_t* __restrict__ flag) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float c = conf[i];
    if (c < 0.f || c > 1.f) *flag = 1u;
}

// A check pass that found a failing image makes its error sticky for the batch.
__global__ void k_conf_verdict(const uint32_t* __restrict__ xerr, int n, uint32_t pass_id, uint32_t* __restrict__ ctr) {
    for (int i = 0; i < n; ++i)
        if (xerr[i]) {
            atomicCAS(&ctr[C_ERR_CONF], 0u, pass_id);
            return;
        }
}

template <int KC>
void launch_update(const SemBatch& sb, svx_map* m, const uint2* cand, int check, const uint32_t* xconf,
                   uint32_t* xerr, uint32_t* xupd) {
    static int per_sm = 0;
    if (!per_sm) SVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sem_update<KC>, kThreads, 0));
    const unsigned grid = std::max(1u, unsigned(per_sm)) * (persistent_grid(m->device) / 8);
    k_sem_update<KC><<<grid, kThreads, 0, m->stream>>>(sb, hash_view(m), m->block_keys, tsdf_base(m), sem_base(m),
                                                       m->sem_idx, cand, m->dirty + m->cfg.max_blocks, check, xconf,
                                                       xerr, xupd, m->d_ctr);
    count_launch();
}

}  // namespace

// A sequence of label images, applied in passes of up to kMaxImg images (one map sweep
// per pass): the result equals successive integrate_labels calls (each voxel sees the
// images in order). Labels / confidences / tensors are read from device memory when
// on_device, else copied from the host (asynchronously; pinned memory overlaps).
// labels_begin stages the batch, labels_enqueue launches the passes of images [i0, i1)
// on the map stream (no synchronisation: a TSDF frame group interleaves them with its
// folds), labels_finish reads the per-image results after the stream synchronised.
LabelBatch labels_begin(svx_map* m, const svx_label_image* imgs, int n, bool on_device,
                        const svx_semantic_cfg& cfg, uint64_t max_blocks_seen) {
    const int K = m->cfg.num_labels;
    for (int i = 0; i < n; ++i)
        if (imgs[i].width <= 0 || imgs[i].height <= 0 || !imgs[i].labels)
            throw Error(SVX_INVALID_ARGUMENT, "label image is empty");
    LabelBatch lb;
    lb.imgs = imgs;
    lb.n = n;
    lb.on_device = on_device;
    lb.cfg = cfg;
    if (n <= 0) return lb;
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
        lb.staged_lbl.assign(size_t(n), nullptr);
        lb.staged_conf.assign(size_t(n), nullptr);
        lb.staged_ten.assign(size_t(n), nullptr);
    }
    // passes: at most one per image (ranges may split the batch anywhere), and a frame
    // group that is rolled back and retried enqueues its images' passes again
    lb.max_passes = 3 * n + 16;
    m->sem_out.alloc(uint64_t(kSemOut) * lb.max_passes);
    SVX_CUDA(cudaMemsetAsync(m->sem_out.p, 0, 4ull * kSemOut * lb.max_passes, m->stream));
    m->cand.alloc(2 * std::max<uint64_t>(max_blocks_seen, 1));  // uint2 per candidate block
    // a block owns at most one layer: map as many layers as there can be blocks, so the
    // update kernel never outgrows the pool and no mid-pass synchronisation is needed
    ensure_layers(m, max_blocks_seen);
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_ERR_CONF, 0, 4, m->stream));
    return lb;
}

void labels_enqueue(svx_map* m, LabelBatch& lb, int i0, int i1, uint32_t group_frame) {
    const int K = m->cfg.num_labels;
    const svx_semantic_cfg& cfg = lb.cfg;
    const bool bad_default = cfg.default_confidence < 0.f || cfg.default_confidence > 1.f;
    uint2* cand = reinterpret_cast<uint2*>(m->cand.p);
    for (int a = i0; a < i1; a += kMaxImg) {
        if (lb.passes >= lb.max_passes) throw Error(SVX_DATA, "label passes: too many retries");
        const int ps = lb.passes++;
        const int ni = std::min(kMaxImg, i1 - a);
        lb.pass_first.push_back(a);
        lb.pass_count.push_back(ni);
        uint32_t* out = m->sem_out.p + uint64_t(kSemOut) * ps;
        uint32_t *xconf = out, *xerr = out + kMaxImg, *xupd = out + 2 * kMaxImg;
        SemBatch sb{};
        sb.n = ni;
        sb.K = K;
        sb.nu = double(m->cfg.voxel_size);
        sb.inv_nu = 1.0 / double(m->cfg.voxel_size);
        sb.occ_floor = -0.5 * double(m->cfg.truncation);
        sb.use_bayes = cfg.use_bayes != 0;
        sb.raycast = cfg.occlusion == SVX_OCCLUSION_RAYCAST;
        sb.floor_v = cfg.likelihood_floor;
        sb.default_conf = cfg.default_confidence;
        sb.pass_id = uint32_t(ps + 1);
        sb.group_frame = group_frame;
        // host images go up on the copy stream when there is one (the TSDF ingest ring's):
        // they overlap the frame's TSDF kernels, and the map stream waits for them only
        // before this pass
        cudaStream_t cs = m->copy_stream ? m->copy_stream : m->stream;
        bool staged_now = false;
        for (int k = 0; k < ni; ++k) {
            const svx_label_image& img = lb.imgs[a + k];
            const uint64_t P = uint64_t(img.width) * uint64_t(img.height);
            ImgParams& ip = sb.img[k];
            const Pose cp = to_pose(img.pose);
            ip.w2c = inverse_pose(cp);
            ip.cam_o = mk(cp.t[0], cp.t[1], cp.t[2]);
            ip.fx = img.fx;
            ip.fy = img.fy;
            ip.cx = img.cx;
            ip.cy = img.cy;
            ip.max_depth = img.max_depth;
            ip.W = img.width;
            ip.H = img.height;
            ip.has_tensor = img.prob_tensor != nullptr;
            ip.has_conf = img.confidence != nullptr;
            ip.labels = img.labels;
            ip.conf = img.confidence;
            ip.tensor = img.prob_tensor;
            if (!lb.on_device) {  // staged once (a retried frame group reuses the copy)
                const size_t ii = size_t(a + k);
                if (!lb.staged_lbl[ii]) {
                    staged_now = true;
                    SVX_CUDA(cudaMemcpyAsync(m->lbl.p + lb.lo, img.labels, 2 * P, cudaMemcpyHostToDevice, cs));
                    lb.staged_lbl[ii] = m->lbl.p + lb.lo;
                    lb.lo += P;
                    if (img.confidence) {
                        SVX_CUDA(cudaMemcpyAsync(m->conf.p + lb.co, img.confidence, 4 * P, cudaMemcpyHostToDevice,
                                                 cs));
                        lb.staged_conf[ii] = m->conf.p + lb.co;
                        lb.co += P;
                    }
                    if (img.prob_tensor) {
                        SVX_CUDA(cudaMemcpyAsync(m->tensor.p + lb.to, img.prob_tensor, 4 * P * K,
                                                 cudaMemcpyHostToDevice, cs));
                        lb.staged_ten[ii] = m->tensor.p + lb.to;
                        lb.to += P * K;
                    }
                }
                ip.labels = lb.staged_lbl[ii];
                ip.conf = lb.staged_conf[ii];
                ip.tensor = lb.staged_ten[ii];
            }
            if (img.fx > 0.0 && img.fy > 0.0 && img.max_depth < 1e30) {
                const double ax = std::max(std::fabs(img.cx), std::fabs(img.width - img.cx)) / img.fx;
                const double ay = std::max(std::fabs(img.cy), std::fabs(img.height - img.cy)) / img.fy;
                ip.reach = float(img.max_depth * std::sqrt(1.0 + ax * ax + ay * ay) * (1.0 + 1e-5) + 1e-3);
            } else {
                ip.reach = 3e38f;  // no finite bound: the half-space tests decide
            }
            // confidence validity: only a voxel that passes every test reads one
            ip.conf_maybe = !ip.has_tensor && (ip.has_conf || bad_default);
            if (ip.conf_maybe) sb.any_check = 1;
        }
        if (staged_now && cs != m->stream) {
            if (lb.events_used == m->label_events.size()) {
                cudaEvent_t e;
                SVX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                m->label_events.push_back(e);
            }
            cudaEvent_t e = m->label_events[lb.events_used++];
            SVX_CUDA(cudaEventRecord(e, cs));
            SVX_CUDA(cudaStreamWaitEvent(m->stream, e, 0));
        }
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_CAND, 0, 4, m->stream));
        {
            ProfMark pm(m, SVX_K_SEM_CULL);
            k_sem_cull<<<persistent_grid(m->device), kThreads, 0, m->stream>>>(sb, m->block_keys, mask_base(m), cand,
                                                                              m->d_ctr);
            count_launch();
        }
        SVX_CUDA(cudaMemcpyAsync(out + 3 * kMaxImg, m->d_ctr + C_CAND, 4, cudaMemcpyDeviceToDevice, m->stream));
        {
            ProfMark pm(m, SVX_K_SEM_UPDATE);
            for (int check = sb.any_check ? 1 : 0; check >= 0; --check) {
                if (check)
                    for (int k = 0; k < ni; ++k)
                        if (sb.img[k].conf_maybe && sb.img[k].has_conf) {
                            const uint64_t P = uint64_t(sb.img[k].W) * uint64_t(sb.img[k].H);
                            k_check_conf<<<grid_for(P), kThreads, 0, m->stream>>>(sb.img[k].conf, P, xconf + k);
                            count_launch();
                        }
                switch (K) {  // compile-time class counts keep a voxel's probabilities in registers
                    case 2: launch_update<2>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 4: launch_update<4>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 8: launch_update<8>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 10: launch_update<10>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 16: launch_update<16>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 19: launch_update<19>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 20: launch_update<20>(sb, m, cand, check, xconf, xerr, xupd); break;
                    case 32: launch_update<32>(sb, m, cand, check, xconf, xerr, xupd); break;
                    default: launch_update<0>(sb, m, cand, check, xconf, xerr, xupd); break;
                }
                if (check) {
                    k_conf_verdict<<<1, 1, 0, m->stream>>>(xerr, ni, sb.pass_id, m->d_ctr);
                    count_launch();
                }
            }
        }
        SVX_CUDA(cudaGetLastError());
    }
}

// After the stream synchronised (sync_counters): reports of images [0, lb.n) in order.
void labels_finish(svx_map* m, const LabelBatch& lb, svx_frame_report* reps) {
    for (int i = 0; i < lb.n; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
    }
    std::vector<uint32_t> outs(size_t(kSemOut) * lb.passes);
    if (lb.passes)
        SVX_CUDA(cudaMemcpy(outs.data(), m->sem_out.p, 4ull * kSemOut * lb.passes, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> upd(lb.n, 0), err(lb.n, 0);
    for (int ps = 0; ps < lb.passes; ++ps) {
        for (int k = 0; k < lb.pass_count[ps]; ++k) {
            upd[lb.pass_first[ps] + k] = outs[size_t(kSemOut) * ps + 2 * kMaxImg + k];
            err[lb.pass_first[ps] + k] = outs[size_t(kSemOut) * ps + kMaxImg + k];
        }
        m->prof_acc.sem_candidates += outs[size_t(kSemOut) * ps + 3 * kMaxImg];
    }
    int fail = lb.n;  // the first image that reads an invalid confidence
    for (int i = 0; i < lb.n && fail == lb.n; ++i)
        if (err[i]) fail = i;
    for (int i = 0; i < fail; ++i) {
        reps[i].frame = m->sem_frames++;
        reps[i].updated_voxels = upd[i];
        m->prof_acc.sem_images += 1;
        m->prof_acc.sem_updated += upd[i];
    }
    m->prof_acc.sem_new_layers += m->h_ctr[C_SEM] - m->n_layers;
    m->n_layers = m->h_ctr[C_SEM];
    if (fail < lb.n) {
        // images before the failing one are complete; the failing one is numbered (the
        // reference numbers a frame before it can throw, semantic_integrator.cpp:93-94)
        // and updated nothing; later images did not run
        m->sem_frames++;
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_ERR_CONF, 0, 4, m->stream));
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        throw Error(SVX_INVALID_ARGUMENT, "confidence must be in [0, 1]");
    }
}

void run_integrate_labels_batch(svx_map* m, const svx_label_image* imgs, int n, bool on_device,
                                const svx_semantic_cfg& cfg, svx_frame_report* reps) {
    for (int i = 0; i < n; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
    }
    if (n <= 0) return;
    LabelBatch lb = labels_begin(m, imgs, n, on_device, cfg, m->n_blocks);
    if (m->n_blocks) labels_enqueue(m, lb, 0, n, ~0u);
    sync_counters(m);
    labels_finish(m, lb, reps);
}

void run_integrate_labels(svx_map* m, const svx_label_image& img, const svx_semantic_cfg& cfg,
                          svx_frame_report* rep) {
    run_integrate_labels_batch(m, &img, 1, false, cfg, rep);
}

}  // namespace svx
