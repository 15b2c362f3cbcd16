// K3-K5: TsdfIntegrator::integrate_frame on the device (tsdf_integrator.cpp:97-258).
//
// Three kernels per frame on the map stream, no host synchronisation (a batch of
// frames is synchronised once at its end):
//   k_raycast_band  K3+K4. CTA = 32 x 8 pixel tile, one thread per pixel. Writes the
//                   pixel cache (ray, range, world normal: the measurement inputs of
//                   tsdf_integrator.cpp:178-186, once per pixel instead of once per
//                   (pixel, voxel)). Band [q - tau r^, q + tau r^], amortised DDA
//                   (tsdf_integrator.hpp:93-135) into a shared-memory table of the
//                   tile's blocks and their 512-bit voxel masks. Per visit, the
//                   own-pixel test of the voxel (FP32, sensor-frame offset updated
//                   incrementally along the DDA, exact decision via error margins): a
//                   voxel whose own pixel has no return is measured by every visiting
//                   ray in the reference (.cpp:232-238), so the visit becomes a
//                   fallback record, measured right away. Tile epilogue: one hash
//                   find-or-insert per distinct block (new block => next pool index,
//                   zero-filled by the tile), dirty flag, touched list; the masks are
//                   ORed into the frame's half of the global mask words and the bits a
//                   tile sets first become the frame's touched-voxel list (each voxel
//                   exactly once).
//   k_fold          K5, one thread per touched voxel (flat, load-balanced): own pixel,
//                   measure, accumulate-then-merge fold (Eq. 4-5, .cpp:170-248). Also
//                   clears the previous frame's half of the mask words and moves the
//                   fallback records into per-block buckets.
//   k_fb_fold       CTA per block with fallback records: orders its bucket by (voxel,
//                   pixel) => per-voxel visits in ascending (v, u) order, exactly the
//                   reference's order after its chunk-order merge + stable_sort; sums
//                   the terms strictly in that order; fold. Its last CTA writes the
//                   frame report and resets the per-frame counters.
// Every kernel first checks the abort word: after an abort (pool growth, buffer
// growth, capacity) the rest of the batch no-ops and the host resumes it.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <vector>

#include "svx_map.hpp"

namespace svx {

struct FrameParams {
    Model m;
    Pose pose, w2s;
    d3 origin;
    float col[3][3];  // nu * (R^T e_m): sensor-frame step of +1 voxel along world axis m
    double tau, max_range, alpha_eps, nu, inv_nu;
    double ca_hi, ca_lo;  // cos(alpha_eps) +- 1e-12: margins of the alpha < eps branch
    float min_clamp;
    // band_all_own(): half voxel diagonal, safe min range, min sin(polar) over the
    // vertical field of view, pixel pitches
    float delta, min_range_safe, sin_min, dphi_f, dtheta_f;
    int nonproj, drop_unreliable, has_normals;
    int32_t shard_rank, shard_world;
    uint32_t frame_serial;
    uint32_t parity;  // which half of each block's 32 mask words this frame uses
    uint32_t max_blocks;
    uint32_t rec_cap, vox_cap;
};

struct PixCache {
    double ray[3];
    double range;
    float n[3];
    uint32_t flags;  // bit0: measurable, bit1: has normal
};
static_assert(sizeof(PixCache) == 48, "PixCache layout");

struct Term {  // one (pixel, voxel) measurement of the fallback path
    float wg, w, nx, ny, nz;
    uint32_t flags;  // bit0: measured, bit1: has normal
};

namespace {

constexpr int kThreads = 256;
constexpr int kFbThreads = 256;
constexpr int kFbMax = 4096;  // fallback records of one block ordered in shared memory

__device__ inline d3 dir_at(const double* __restrict__ dirs, uint32_t p) {
    return mk(__ldg(&dirs[3 * p]), __ldg(&dirs[3 * p + 1]), __ldg(&dirs[3 * p + 2]));
}

__device__ inline d3 voxel_center(int32_t x, int32_t y, int32_t z, double nu) {
    return mk(nu * x, nu * y, nu * z);
}

__device__ inline d3 center_of(uint64_t key, int linear, double nu) {
    int32_t bx, by, bz;
    unpack_key(key, bx, by, bz);
    return voxel_center(bx * kBlockSide + linear % kBlockSide,
                        by * kBlockSide + (linear / kBlockSide) % kBlockSide,
                        bz * kBlockSide + linear / (kBlockSide * kBlockSide), nu);
}

// Own pixel of a voxel centre c: project_point(world_to_sensor * c)
// (tsdf_integrator.cpp:232). pc is world_to_sensor * c in FP64 (reference formula).
__device__ inline uint32_t own_pixel(const FrameParams& f, d3 pc) {
    const uint32_t q = pixel_fast(float(pc.x), float(pc.y), float(pc.z), f.m, f.m.r2_lo, f.m.r2_hi);
    return q == kNeedFp64 ? pixel_fp64(pc, f.m) : q;
}

// Row distance (columns, azimuth wraps) from each pixel to the nearest pixel of
// its row without a return, capped at kRmax + 1.
constexpr int kRmax = kRowDistMax;
__global__ void __launch_bounds__(kThreads)
k_row_dist(const float* __restrict__ depth, int W, int H, uint8_t* __restrict__ hd,
           uint32_t* __restrict__ validbits, const uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool inside = p < uint32_t(W) * H;
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, inside && depth[inside ? p : 0] != 0.f);
    if ((threadIdx.x & 31) == 0 && p < uint32_t(W) * H) validbits[p >> 5] = bits;
    if (!inside) return;
    const int u = int(p % W);
    const float* row = depth + (p - u);
    int d = 0;
    for (; d <= kRmax; ++d) {
        int a = u + d, b = u - d;
        a -= a >= W ? W : 0;
        b += b < 0 ? W : 0;
        if (row[a] == 0.f || row[b] == 0.f) break;
    }
    hd[p] = uint8_t(d);
}

// Chebyshev distance from pixel p to the nearest pixel without a return or to
// the top/bottom image edge, capped at kRmax + 1: every pixel closer than that
// holds a return.
__device__ inline int valid_radius(const uint8_t* __restrict__ hd, int W, int H, uint32_t p) {
    const int u = int(p % W), v = int(p / W);
    int r = kRmax + 1;
    for (int dy = -kRmax; dy <= kRmax; ++dy) {
        const int ady = dy < 0 ? -dy : dy;
        if (ady >= r) continue;
        const int v2 = v + dy;
        const int h = (v2 < 0 || v2 >= H) ? 0 : int(hd[uint32_t(v2) * W + u]);
        r = min(r, max(ady, h));
    }
    return r;
}

// True when no voxel visited by the band of this ray can have its own pixel
// without a return: the voxel centre lies within delta = sqrt(3)/2 nu of the ray,
// so its direction is within angle a <= 1.1 delta / d_min of the pixel-centre
// direction, i.e. within k pixels; every pixel within k of p holds a return.
__device__ inline bool band_all_own(const FrameParams& f, const uint8_t* __restrict__ hd,
                                    uint32_t p, float r) {
    const float dmin = r - float(f.tau) - f.delta;
    if (!(dmin > f.min_range_safe)) return false;
    const float x = f.delta / dmin;
    if (x > 0.3f) return false;
    const float a = 1.1f * x;  // asin(x) <= 1.1 x for x <= 0.3
    const float s = f.sin_min - a;
    if (s < 0.1f || a > s * (1.f / 3.f)) return false;
    // azimuth offset <= 2 asin(sin(a/2) / s) <= 1.05 a / s for a / s <= 1/3
    const int ku = int(floorf(1.05f * a / (s * f.dphi_f) + 0.5f)) + 1;
    const int kv = int(floorf(a / f.dtheta_f + 0.5f)) + 1;
    const int k = max(ku, kv);
    if (k > kRmax) return false;
    return valid_radius(hd, f.m.W, f.m.H, p) > k;
}

struct Accum {
    double wd, w, wx, wy, wz;
};

// nonprojective_distance (tsdf_integrator.cpp:39-46)
__device__ inline double nonprojective_distance(double psi, double theta, double alpha,
                                                double eps) {
    double st, ct;
    sincos(theta, &st, &ct);  // same values as sin()/cos(), one shared range reduction
    if (alpha < eps) return fabs(ct) * psi;
    double sa, ca;
    sincos(alpha, &sa, &ca);
    const double mag = fabs((ca - 1.0) * st / sa) + fabs(ct * psi);
    return psi >= 0.0 ? mag : -mag;
}

// truncate_distance (tsdf_integrator.hpp:57-59)
__device__ inline float truncate_f(double d, double tau) {
    return float(d >= 0.0 ? (tau < d ? tau : d) : (d < -tau ? -tau : d));
}

// Gamma(d) of the non-projective distance from the clamped cosines ct = cos(theta)
// and ca = cos(alpha). The reference evaluates theta = acos(ct), alpha = acos(ca)
// and then cos/sin of both with libm (tsdf_integrator.cpp:39-46,195-196).
// Fast path without transcendentals: cos(acos(x)) = x and sin(acos(x)) =
// sqrt((1-x)(1+x)) up to |err| <= 2e-15 (1-ulp libm acos/cos/sin: pi * 2^-52 + 2^-52),
// an absolute bound E on the resulting d, and the f32 value the reference stores,
// float(clamp(d, +-tau)), accepted only when all of [d - E, d + E] rounds to it.
// The branch alpha < eps is decided on ca against cos(eps) with a 1e-12 margin
// (acos is strictly decreasing). Otherwise (ca near cos(eps), sin(alpha) < 1e-6,
// or an interval straddling a float boundary: ~1e-4 of the voxels) the reference
// formula is evaluated with CUDA's FP64 acos/sincos.
__device__ inline float gamma_nonprojective(const FrameParams& f, double psi, double ct, double ca) {
    constexpr double kAbs = 2e-15, kRel = 2e-15;
    bool fast = false;
    double d = 0.0, e = 0.0;
    if (ca > f.ca_hi) {  // alpha < eps: |cos theta| * psi
        d = fabs(ct) * psi;
        e = fabs(psi) * (kAbs + kRel * fabs(ct)) + 1e-15 * fabs(d);
        fast = true;
    } else if (ca < f.ca_lo) {
        const double st = sqrt((1.0 - ct) * (1.0 + ct));
        const double sa = sqrt((1.0 - ca) * (1.0 + ca));
        if (sa > 1e-6) {
            const double a = ca - 1.0;
            const double t1 = fabs(a * st / sa), t2 = fabs(ct * psi);
            const double mag = t1 + t2;
            d = psi >= 0.0 ? mag : -mag;
            const double da = kAbs + kRel * fabs(a), dst = kAbs + kRel * st, dsa = kAbs + kRel * sa;
            e = 1.01 * ((fabs(a) * dst + st * da) / sa + t1 * dsa / sa +
                        fabs(psi) * (kAbs + kRel * fabs(ct))) +
                1e-15 * mag;
            fast = true;
        }
    }
    if (fast) {
        const float lo = truncate_f(d - e, f.tau), hi = truncate_f(d + e, f.tau);
        if (lo == hi && __float_as_uint(lo) == __float_as_uint(hi)) return lo;
    }
    return truncate_f(nonprojective_distance(psi, acos(ct), acos(ca), f.alpha_eps), f.tau);
}

// measure lambda (tsdf_integrator.cpp:172-205) for pixel p, from the pixel cache:
// the contribution (w * Gamma(d), w, w * n) as the reference forms it, in f32.
__device__ inline Term measure_term(const FrameParams& f, const PixCache* __restrict__ cache,
                                    uint32_t p, d3 center, const svx_tsdf_voxel& vox) {
    Term t{0.f, 0.f, 0.f, 0.f, 0.f, 0u};
    const PixCache& pc = cache[p];
    const uint32_t flags = pc.flags;
    if (!(flags & 1u)) return t;
    const bool have_normal = flags & 2u;
    const d3 ray = mk(pc.ray[0], pc.ray[1], pc.ray[2]);
    const double psi = pc.range - dot3(sub3(center, f.origin), ray);
    if (fabs(psi) > f.tau) return t;
    const float nw[3] = {pc.n[0], pc.n[1], pc.n[2]};
    float gamma;
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
        gamma = gamma_nonprojective(f, psi, ct, ca);
    } else {
        gamma = truncate_f(psi, f.tau);
    }
    // observation_weight (tsdf_integrator.cpp:48-51)
    double wr = (psi + f.tau) / (2.0 * f.tau);
    const double lo = double(f.min_clamp);
    wr = wr < lo ? lo : (1.0 < wr ? 1.0 : wr);
    const float w_obs = float(wr);
    t.wg = w_obs * gamma;
    t.w = w_obs;
    if (have_normal) {
        t.nx = w_obs * nw[0];
        t.ny = w_obs * nw[1];
        t.nz = w_obs * nw[2];
    }
    t.flags = 1u | (have_normal ? 2u : 0u);
    return t;
}

// acc += term, in the reference's operation order (tsdf_integrator.cpp:201-203)
__device__ inline void accumulate(Accum& acc, const Term& t) {
    acc.wd += double(t.wg);
    acc.w += double(t.w);
    if (t.flags & 2u) {
        acc.wx += double(t.nx);
        acc.wy += double(t.ny);
        acc.wz += double(t.nz);
    }
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

// A fallback record: one (visiting ray, voxel) measurement of a voxel whose own
// pixel has no return, measured where the visit is found (band kernel) and
// summed later in pixel order (k_fb_fold). The voxel's state cannot change in
// between: fallback voxels are only written by k_fb_fold.
struct FbRec {
    uint32_t key;   // linear << 23 | pixel
    uint32_t slot;  // hash slot of the block
    Term t;
};
static_assert(sizeof(FbRec) == 32, "FbRec layout");

// Hash find-or-insert of a block key; a new block takes the next pool index.
struct SlotRef {
    uint32_t slot, idx;
    bool inserted;
};

// Pool index of an existing slot. A slot inserted concurrently by another CTA
// gets its index right after the key (find_or_insert): wait for it.
__device__ inline uint32_t block_index(HashView h, uint32_t slot) {
    uint32_t idx = __ldcg(&h.vals[slot]);
    while (idx == kInvalid) {
        __nanosleep(64);
        idx = *reinterpret_cast<volatile uint32_t*>(&h.vals[slot]);
    }
    return idx;
}

__device__ inline SlotRef find_or_insert(const FrameParams& f, HashView h,
                                         uint64_t* __restrict__ block_keys,
                                         uint32_t* __restrict__ ctr, uint64_t key) {
    SlotRef r{kInvalid, kInvalid, false};
    int ins = 0;
    r.slot = hash_insert(h, key, &ins);
    if (r.slot == kInvalid) {
        atomicOr(&ctr[C_ABORT], kAbortHash | kAbortCapacity);
        return r;
    }
    if (ins) {
        r.inserted = true;
        r.idx = atomicAdd(&ctr[C_BLOCKS], 1u);
        if (r.idx < f.max_blocks) block_keys[r.idx] = key;
        __threadfence();
        atomicExch(&h.vals[r.slot], r.idx);
        if (r.idx >= f.max_blocks) atomicOr(&ctr[C_ABORT], kAbortCapacity);
        else if (r.idx >= ctr[C_MAPPED]) raise_frame_abort(ctr, kAbortPool, f.frame_serial);
    } else {
        r.idx = block_index(h, r.slot);
    }
    return r;
}

__device__ inline void zero_block(svx_tsdf_voxel* __restrict__ pool, uint32_t idx, int lane, int lanes) {
    float4* z = reinterpret_cast<float4*>(pool + uint64_t(idx) * kBlockVoxels);
    for (int i = lane; i < kBlockVoxels * 5 / 4; i += lanes) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Measurement of fallback visit (slot, lin) by the ray of pixel p. A block
// created in this frame (pool index unset yet or >= the frame's first new index)
// is all-zero; its pool memory may not be zero-filled yet (tile epilogues).
__device__ inline Term fallback_term(const FrameParams& f, HashView h,
                                     const svx_tsdf_voxel* __restrict__ pool,
                                     const PixCache* __restrict__ cache, uint32_t blocks_before,
                                     uint32_t slot, uint64_t key, int lin, uint32_t p) {
    const uint32_t idx = __ldcg(&h.vals[slot]);
    svx_tsdf_voxel vox{0.f, 0.f, {0.f, 0.f, 0.f}};
    if (idx != kInvalid && idx < blocks_before) vox = load_voxel(pool + uint64_t(idx) * kBlockVoxels + lin);
    return measure_term(f, cache, p, center_of(key, lin, f.nu), vox);
}

__device__ inline void store_record(FbRec* __restrict__ rec, uint32_t pos, const FbRec& r) {
    uint4* d = reinterpret_cast<uint4*>(rec + pos);
    const uint4* s = reinterpret_cast<const uint4*>(&r);
    d[0] = s[0];
    d[1] = s[1];
}

// Per-visit work on global state (no tile staging): the path a visit takes when
// its tile's shared tables are full. Same effect as the staged path.
__device__ void visit_global(const FrameParams& f, HashView h, uint64_t* __restrict__ block_keys,
                             uint32_t* __restrict__ stamp, uint32_t* __restrict__ touched,
                             uint32_t* __restrict__ vmask, uint32_t* __restrict__ fbcnt,
                             FbRec* __restrict__ rec, svx_tsdf_voxel* __restrict__ pool,
                             const PixCache* __restrict__ cache, uint8_t* __restrict__ dirty,
                             unsigned long long* __restrict__ vlist, uint32_t blocks_before,
                             uint32_t* __restrict__ ctr, uint64_t key, int lin, bool fb, uint32_t p) {
    const SlotRef r = find_or_insert(f, h, block_keys, ctr, key);
    if (r.slot == kInvalid) return;
    if (atomicExch(&stamp[r.slot], f.frame_serial) != f.frame_serial)
        touched[atomicAdd(&ctr[C_TOUCHED], 1u)] = r.slot;
    if (r.idx >= f.max_blocks) return;
    if (r.inserted && r.idx < ctr[C_MAPPED]) zero_block(pool, r.idx, 0, 1);
    dirty[r.idx] = 1;
    const uint32_t bit = 1u << (lin & 31);
    if (!(atomicOr(&vmask[uint64_t(r.slot) * 32 + f.parity * 16 + (lin >> 5)], bit) & bit)) {
        const uint32_t pos = atomicAdd(&ctr[C_VOXLIST], 1u);
        if (pos < f.vox_cap) vlist[pos] = (static_cast<unsigned long long>(r.idx) << 9) | uint32_t(lin);
        else atomicOr(&ctr[C_ABORT], kAbortVoxList);
    }
    if (!fb) return;
    const Term t = fallback_term(f, h, pool, cache, blocks_before, r.slot, key, lin, p);
    if (!(t.flags & 1u)) return;  // no contribution
    atomicAdd(&fbcnt[r.slot], 1u);
    const uint32_t pos = atomicAdd(&ctr[C_RECORDS], 1u);
    if (pos < f.rec_cap)
        store_record(rec, pos, FbRec{(uint32_t(lin) << 23) | p, r.slot, t});
    else
        atomicOr(&ctr[C_ABORT], kAbortRecords);
}

// CTA = 32 x 8 pixel tile. The tile's rays run their DDA into shared memory: a
// local table of the distinct blocks they visit, the visit records and per-block
// voxel masks (smem atomics). Global work is then one hash find-or-insert per
// distinct block (in parallel across threads) and one RED.OR per non-empty mask
// word, instead of serialized global round trips per ray.
#ifndef SVX_TILE_U
#define SVX_TILE_U 32
#endif
constexpr int kTileU = SVX_TILE_U, kTileV = 256 / SVX_TILE_U;
constexpr int kLocalKeys = 256;
#ifndef SVX_TILE_FB
#define SVX_TILE_FB 1024
#endif
constexpr int kTileFb = SVX_TILE_FB;  // staged fallback visits per tile

__global__ void __launch_bounds__(kTileU * kTileV, 4)
k_raycast_band(FrameParams f, const float* __restrict__ depth, const float* __restrict__ normals,
               const uint8_t* __restrict__ valid, const double* __restrict__ dirs,
               const uint8_t* __restrict__ hd, const uint32_t* __restrict__ validbits,
               PixCache* __restrict__ cache, HashView h,
               uint64_t* __restrict__ block_keys, uint32_t* __restrict__ stamp,
               uint32_t* __restrict__ touched, uint32_t* __restrict__ vmask,
               uint32_t* __restrict__ fbcnt, FbRec* __restrict__ rec,
               svx_tsdf_voxel* __restrict__ pool, uint8_t* __restrict__ dirty,
               unsigned long long* __restrict__ vlist, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    // pool exhaustion raised by this frame does not stop its band: the frame
    // resumes after its band
    if (cta_aborted_for(ctr, kAbortPool, f.frame_serial)) return;
    __shared__ unsigned long long lkey[kLocalKeys];
    __shared__ uint32_t lslot[kLocalKeys];
    __shared__ uint32_t lidx[kLocalKeys];
    __shared__ uint32_t lmask[kLocalKeys][16];
    __shared__ uint32_t lfb[kTileFb];
    __shared__ uint32_t lcnt[kLocalKeys];  // kept fallback records per local block
    __shared__ uint32_t lnew[kLocalKeys];  // pool indices of blocks this tile created
    __shared__ uint32_t nfb, nnew;
    const int tid = threadIdx.x;
    const uint32_t blocks_before = ctr[C_BLOCKS_BEFORE];
    lkey[tid] = kEmptyKey;
    lcnt[tid] = 0u;
#pragma unroll
    for (int w = 0; w < 16; ++w) lmask[tid][w] = 0u;
    if (tid == 0) nfb = nnew = 0;
    __syncthreads();

    const int tiles_u = (f.m.W + kTileU - 1) / kTileU;
    const int tu = int(blockIdx.x) % tiles_u, tv = int(blockIdx.x) / tiles_u;
    const int u = tu * kTileU + (tid % kTileU);
    const int v = tv * kTileV + (tid / kTileU);
    const uint32_t tile_p0 = uint32_t(tv * kTileV) * uint32_t(f.m.W) + uint32_t(tu * kTileU);
    const bool has_pix = u < f.m.W && v < f.m.H;
    const uint32_t p = has_pix ? uint32_t(v) * uint32_t(f.m.W) + uint32_t(u) : 0u;
    const float r = has_pix ? depth[p] : 0.f;
    const bool in_range = has_pix && !(r == 0.f || double(r) > f.max_range);
    const bool have_normal = has_pix && f.has_normals && valid[p];
    // pixel cache (measure lambda inputs, tsdf_integrator.cpp:173-186)
    d3 q = mk(0, 0, 0), ray = mk(0, 0, 0);
    if (has_pix) {
        PixCache pc{};
        if (in_range) {
            q = xform(f.pose, scale3(double(r), dir_at(dirs, p)));
            const d3 dq = sub3(q, f.origin);
            const double range = sqrt(dot3(dq, dq));
            ray = div3(dq, range);
            pc.ray[0] = ray.x;
            pc.ray[1] = ray.y;
            pc.ray[2] = ray.z;
            pc.range = range;
            if (have_normal) {
                const d3 n = matvec(f.pose.R, mk(normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]));
                pc.n[0] = float(n.x);
                pc.n[1] = float(n.y);
                pc.n[2] = float(n.z);
            }
            pc.flags = ((have_normal || !f.drop_unreliable) ? 1u : 0u) | (have_normal ? 2u : 0u);
        }
        cache[p] = pc;
    }
    // band ray (tsdf_integrator.cpp:123-131)
#ifdef SVX_DIAG_NODDA  // timing diagnostic builds only (results invalid)
    const bool cast = false;
#else
    const bool cast = in_range && !(f.drop_unreliable && f.has_normals && !valid[p]);
#endif
#ifdef SVX_DIAG_NOVISIT
    uint32_t diag_sink = 0;
#endif
    if (cast) {
        warp_agg_inc(&ctr[C_RAYS]);
        const d3 tr = scale3(f.tau, ray);  // (q - o).normalized() == (q - o) / range
        const d3 a = sub3(q, tr), b = add3(q, tr);
        uint64_t cur_key = kEmptyKey;
        int cur_li = -1;
        bool cur_own = true;
        int pend_word = -1;
        uint32_t pend_bits = 0;
        int32_t x0 = 0, y0 = 0, z0 = 0;
        float p0x = 0.f, p0y = 0.f, p0z = 0.f;
        bool first = true;
        const bool all_own = band_all_own(f, hd, p, r);
        traverse_segment<true>(a, b, f.nu, f.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
#ifdef SVX_DIAG_NOVISIT
            diag_sink += uint32_t(x ^ y ^ z);
            return;
#endif
            const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
            if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) {
                atomicOr(&ctr[C_ABORT], kAbortKey);
                return;
            }
            const uint64_t key = pack_key(bx, by, bz);
            if (key != cur_key) {
                cur_key = key;
                cur_own = !(f.shard_world > 1 && owner_of(key, f.shard_world) != f.shard_rank);
                cur_li = -1;
                if (cur_own) {  // local table insert (open addressing in smem)
                    uint32_t s = hash_slot(key, 8);
                    for (int probe = 0; probe < kLocalKeys; ++probe) {
                        const unsigned long long old = atomicCAS(&lkey[s], kEmptyKey, key);
                        if (old == kEmptyKey || old == key) {
                            cur_li = int(s);
                            break;
                        }
                        s = (s + 1) & (kLocalKeys - 1);
                    }
                }
            }
            if (!cur_own) return;
            const int lin = local_linear(x, y, z);
            // own-pixel test of the visited voxel
            bool fb = false;
            if (!all_own) {
                if (first) {
                    const d3 pc0 = xform(f.w2s, voxel_center(x, y, z, f.nu));
                    p0x = float(pc0.x);
                    p0y = float(pc0.y);
                    p0z = float(pc0.z);
                    x0 = x;
                    y0 = y;
                    z0 = z;
                    first = false;
                }
                const float kx = float(x - x0), ky = float(y - y0), kz = float(z - z0);
                const float px = p0x + kx * f.col[0][0] + ky * f.col[1][0] + kz * f.col[2][0];
                const float py = p0y + kx * f.col[0][1] + ky * f.col[1][1] + kz * f.col[2][1];
                const float pz = p0z + kx * f.col[0][2] + ky * f.col[1][2] + kz * f.col[2][2];
                uint32_t own = pixel_fast(px, py, pz, f.m, f.m.r2_lo, f.m.r2_hi);
                if (own == kNeedFp64) own = pixel_fp64(xform(f.w2s, voxel_center(x, y, z, f.nu)), f.m);
                fb = own == kInvalid || !pixel_has_return(validbits, own);
            }
            if (cur_li < 0) {  // local table full: straight to global state
#ifdef SVX_DIAG_NOGLOBAL
                return;  // diagnostic build only: drop table-overflow visits
#endif
                visit_global(f, h, block_keys, stamp, touched, vmask, fbcnt, rec, pool, cache, dirty,
                             vlist, blocks_before, ctr, key, lin, fb, p);
                return;
            }
            const int word = cur_li * 16 + (lin >> 5);
            if (word != pend_word) {
                if (pend_word >= 0) atomicOr(&lmask[0][0] + pend_word, pend_bits);
                pend_word = word;
                pend_bits = 0u;
            }
            pend_bits |= 1u << (lin & 31);
            if (fb) {
                const uint32_t pos = atomicAdd(&nfb, 1u);
                if (pos < uint32_t(kTileFb))
                    lfb[pos] = (uint32_t(cur_li) << 24) | (uint32_t(lin) << 15) | uint32_t(tid);
                else
                    visit_global(f, h, block_keys, stamp, touched, vmask, fbcnt, rec, pool, cache,
                                 dirty, vlist, blocks_before, ctr, key, lin, true, p);
            }
        });
        if (pend_word >= 0) atomicOr(&lmask[0][0] + pend_word, pend_bits);
#ifdef SVX_DIAG_NOVISIT
        if (diag_sink == 0xFFFFFFFFu) atomicOr(&ctr[C_ABORT], 0u);
#endif
    }
    __syncthreads();
    // one global hash operation per distinct block of the tile; first touches of
    // the frame are appended to the touched list with one atomic per tile
    constexpr int kW = kTileU * kTileV / 32;
    __shared__ uint32_t s_w[2 * kW];
    uint32_t slot = kInvalid;
    bool first_touch = false;
    if (lkey[tid] != kEmptyKey) {
        const SlotRef r = find_or_insert(f, h, block_keys, ctr, lkey[tid]);
        slot = r.slot;
        if (slot != kInvalid) {
            first_touch = atomicExch(&stamp[slot], f.frame_serial) != f.frame_serial;
            lidx[tid] = r.idx;
            if (r.idx < f.max_blocks) {
                dirty[r.idx] = 1;
                if (r.inserted && r.idx < ctr[C_MAPPED]) lnew[atomicAdd(&nnew, 1u)] = r.idx;
            } else {
                slot = kInvalid;  // capacity abort is set; nothing below may touch the pool
                first_touch = false;
            }
        }
    }
    lslot[tid] = slot;
    const uint32_t tpos = cta_append<kW>(first_touch, &ctr[C_TOUCHED], s_w);
    if (first_touch) touched[tpos] = slot;
    // zero-fill the blocks this tile created (read from the next kernel on)
    for (uint32_t j = 0; j < nnew; ++j) zero_block(pool, lnew[j], tid, kTileU * kTileV);
    // fallback visits: measured here (the rays' pixel cache entries were written
    // above by this CTA); records that contribute are appended with one atomic per
    // round, and counted per block with one atomic per block
    const uint32_t nf = min(nfb, uint32_t(kTileFb));
    for (uint32_t i0 = 0; i0 < nf; i0 += kTileU * kTileV) {
        const uint32_t i = i0 + uint32_t(tid);
        FbRec r{};
        bool keep = false;
        uint32_t li = 0;
        if (i < nf) {
            const uint32_t e = lfb[i];
            li = e >> 24;
            r.slot = lslot[li];
            if (r.slot != kInvalid) {
                const uint32_t t = e & 255u;
                const uint32_t px = tile_p0 + (t / kTileU) * uint32_t(f.m.W) + (t % kTileU);
                const int lin = int((e >> 15) & 511u);
                r.t = fallback_term(f, h, pool, cache, blocks_before, r.slot, lkey[li], lin, px);
                r.key = (uint32_t(lin) << 23) | px;
                keep = r.t.flags & 1u;
            }
        }
        const uint32_t pos = cta_append<kW>(keep, &ctr[C_RECORDS], s_w);
        if (keep) {
            atomicAdd(&lcnt[li], 1u);
            if (pos < f.rec_cap) store_record(rec, pos, r);
            else atomicOr(&ctr[C_ABORT], kAbortRecords);
        }
    }
    // voxel masks -> this frame's half of the global mask words; the bits a tile
    // sets first (atomicOr returns them clear) are its voxels' single entries in
    // the frame's touched-voxel list
    uint32_t nv = 0;
    for (int i = tid; i < kLocalKeys * 16; i += kTileU * kTileV) {
        const int li = i >> 4, w = i & 15;
        uint32_t bits = lmask[li][w];
        if (bits && lslot[li] != kInvalid) {
            const uint32_t old = atomicOr(&vmask[uint64_t(lslot[li]) * 32 + f.parity * 16 + w], bits);
            bits &= ~old;
        } else {
            bits = 0u;
        }
        lmask[li][w] = bits;
        nv += __popc(bits);
    }
    uint32_t pos = cta_reserve<kW>(nv, &ctr[C_VOXLIST], s_w);
    if (nv && pos + nv > f.vox_cap) atomicOr(&ctr[C_ABORT], kAbortVoxList);
    for (int i = tid; i < kLocalKeys * 16 && nv; i += kTileU * kTileV) {
        const int li = i >> 4, w = i & 15;
        const unsigned long long hi = static_cast<unsigned long long>(lidx[li]) << 9;
        for (uint32_t bits = lmask[li][w]; bits; bits &= bits - 1, ++pos)
            if (pos < f.vox_cap) vlist[pos] = hi | (uint32_t(w) * 32u + uint32_t(__ffs(bits) - 1));
    }
    __syncthreads();  // lcnt complete
    if (lcnt[tid]) atomicAdd(&fbcnt[lslot[tid]], lcnt[tid]);
}

// One thread per touched voxel: own pixel, measure, fold. A list entry holds the
// pool index and the voxel, so the voxel and its block key load in parallel.
// The same kernel clears the previous frame's half of the mask words (the next
// frame uses it) and moves the fallback records into per-block buckets; a
// block's bucket is allocated by the first of its records to arrive.
__global__ void __launch_bounds__(kThreads)
k_fold(FrameParams f, const uint32_t* __restrict__ validbits, const PixCache* __restrict__ cache,
       const uint64_t* __restrict__ block_keys, svx_tsdf_voxel* __restrict__ pool,
       const unsigned long long* __restrict__ vlist, const uint32_t* __restrict__ touched_prev,
       uint32_t* __restrict__ vmask, const FbRec* __restrict__ rec,
       const uint32_t* __restrict__ fbcnt, uint32_t* __restrict__ fbstart,
       uint32_t* __restrict__ fbclaim, uint32_t* __restrict__ fbfill,
       uint32_t* __restrict__ fbslots, FbRec* __restrict__ bucket, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    {
        const uint32_t n_prev = ctr[C_TOUCHED_PREV];
        const uint32_t other = (f.parity ^ 1u) * 16u;
        for (uint32_t i = gtid; i < n_prev * 16u; i += stride)
            vmask[uint64_t(touched_prev[i >> 4]) * 32 + other + (i & 15u)] = 0u;
    }
    const uint32_t nv = min(ctr[C_VOXLIST], f.vox_cap);
    uint32_t n_upd = 0;
    for (uint32_t i = gtid; i < nv; i += stride) {
        const unsigned long long v = vlist[i];
        const uint64_t idx = v >> 9;
        const int linear = int(v & 511u);
        svx_tsdf_voxel* vp = pool + idx * kBlockVoxels + linear;
        const uint64_t key = block_keys[idx];
        svx_tsdf_voxel vox = load_voxel(vp);
        const d3 c = center_of(key, linear, f.nu);
        const uint32_t own = own_pixel(f, xform(f.w2s, c));
        if (own == kInvalid || !pixel_has_return(validbits, own)) continue;  // fallback path
        const Term t = measure_term(f, cache, own, c, vox);
        if (t.flags & 1u) {
            Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
            accumulate(acc, t);
            fold(vox, acc);
            store_voxel(vp, vox);
            ++n_upd;
        }
    }
    const uint32_t nr = min(ctr[C_RECORDS], f.rec_cap);
    for (uint32_t i = gtid; i < nr; i += stride) {
        const uint4* src = reinterpret_cast<const uint4*>(rec + i);
        const uint4 a = src[0], b = src[1];
        const uint32_t slot = a.y;
        uint32_t start = __ldcg(&fbstart[slot]);
        if (start == kInvalid) {
            if (atomicCAS(&fbclaim[slot], 0u, 1u) == 0u) {  // this record allocates the bucket
                start = atomicAdd(&ctr[C_BUCKET_TOP], fbcnt[slot]);
                fbslots[atomicAdd(&ctr[C_FB_BLOCKS], 1u)] = slot;
                atomicExch(&fbstart[slot], start);
            } else {
                while ((start = *reinterpret_cast<volatile uint32_t*>(&fbstart[slot])) == kInvalid)
                    __nanosleep(32);
            }
        }
        const uint32_t pos = start + atomicAdd(&fbfill[slot], 1u);
        uint4* dst = reinterpret_cast<uint4*>(bucket + pos);
        dst[0] = a;
        dst[1] = b;
    }
    for (int o = 16; o; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
    if ((threadIdx.x & 31) == 0 && n_upd) atomicAdd(&ctr[C_UPDATED], n_upd);
}

__device__ void write_frame_end(FrameOut* __restrict__ out, uint32_t* __restrict__ ctr) {
    FrameOut o;
    o.updated = ctr[C_UPDATED];
    o.new_blocks = ctr[C_BLOCKS] - ctr[C_BLOCKS_BEFORE];
    o.touched = ctr[C_TOUCHED];
    o.records = ctr[C_RECORDS];
    o.rays = ctr[C_RAYS];
    o.dropped = ctr[C_DROPPED];
    o.fb_voxels = ctr[C_FB_VOXELS];
    o.ok = 1;
    *out = o;
    ctr[C_TOUCHED_PREV] = ctr[C_TOUCHED];
    ctr[C_TOUCHED] = ctr[C_UPDATED] = ctr[C_RECORDS] = ctr[C_RAYS] = 0;
    ctr[C_DROPPED] = ctr[C_TIES] = ctr[C_FB_BLOCKS] = ctr[C_FB_VOXELS] = ctr[C_FB_BIG] = 0;
    ctr[C_VOXLIST] = ctr[C_BUCKET_TOP] = 0;
    ctr[C_BLOCKS_BEFORE] = ctr[C_BLOCKS];
}

__device__ inline Term record_term(const FbRec* __restrict__ r) {
    const uint4* q = reinterpret_cast<const uint4*>(r);
    const uint4 a = q[0], b = q[1];
    Term t;
    t.wg = __uint_as_float(a.z);
    t.w = __uint_as_float(a.w);
    t.nx = __uint_as_float(b.x);
    t.ny = __uint_as_float(b.y);
    t.nz = __uint_as_float(b.z);
    t.flags = b.w;
    return t;
}

// Ordered fold of one fallback voxel: the terms of records bucket[src[i..end)],
// summed in that order (ascending pixel). Loads are issued four at a time so the
// sequential sum does not pay one L2 round trip per record.
template <typename Src>
__device__ inline bool fold_records(svx_tsdf_voxel* vp, const FbRec* __restrict__ bucket,
                                    const Src* __restrict__ src, uint32_t i, uint32_t end) {
    if (i == end) return false;
    Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
    uint32_t j = i;
    for (; j + 4 <= end; j += 4) {
        const Term t0 = record_term(bucket + src[j]), t1 = record_term(bucket + src[j + 1]);
        const Term t2 = record_term(bucket + src[j + 2]), t3 = record_term(bucket + src[j + 3]);
        accumulate(acc, t0);
        accumulate(acc, t1);
        accumulate(acc, t2);
        accumulate(acc, t3);
    }
    for (; j < end; ++j) accumulate(acc, record_term(bucket + src[j]));
    svx_tsdf_voxel vox = load_voxel(vp);
    fold(vox, acc);
    store_voxel(vp, vox);
    return true;
}

// CTA per block with fallback records (the records cluster on few blocks, e.g. on
// the ring where the lowest beam meets the ground). Records arrive measured; the
// bucket is ordered by (voxel, pixel) in shared memory: counting sort by voxel
// (histogram, scan, scatter), then inside each voxel's segment a rank sort (the
// rank of a record is the number of smaller keys in its segment; keys are unique,
// a ray visits a voxel once), all in parallel. One thread per voxel then folds it
// with the terms summed strictly in that order.
__global__ void __launch_bounds__(kFbThreads)
k_fb_fold(HashView h, svx_tsdf_voxel* __restrict__ pool, const uint32_t* __restrict__ fbslots,
          uint32_t* __restrict__ fbcnt, uint32_t* __restrict__ fbstart,
          uint32_t* __restrict__ fbclaim, uint32_t* __restrict__ fbfill,
          const FbRec* __restrict__ bucket, uint32_t* __restrict__ bigslots,
          FrameOut* __restrict__ out, uint32_t serial, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    // a big bucket (host-sorted afterwards) of this frame must not stop its other buckets
    if (cta_aborted_for(ctr, kAbortBigBucket, serial)) return;
    using Scan = cub::BlockScan<uint32_t, kFbThreads>;
    constexpr int kPer = kBlockVoxels / kFbThreads;  // voxels per thread in the scan
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint32_t keys[kFbMax];   // grouped by voxel
    __shared__ uint16_t src1[kFbMax];   // record index of keys[i]
    __shared__ uint16_t src2[kFbMax];   // record indices in (voxel, pixel) order
    __shared__ uint32_t seg_start[kBlockVoxels], seg_cnt[kBlockVoxels], cursor[kBlockVoxels];
    __shared__ bool last;
    const uint32_t nb = ctr[C_FB_BLOCKS];
    uint32_t n_upd = 0;
    for (uint32_t t = blockIdx.x; t < nb; t += gridDim.x) {
        const uint32_t slot = fbslots[t];
        const uint32_t cnt = fbcnt[slot];
        const uint32_t start = fbstart[slot];
        if (cnt > uint32_t(kFbMax)) {
            if (threadIdx.x == 0) {
                bigslots[atomicAdd(&ctr[C_FB_BIG], 1u)] = slot;
                raise_frame_abort(ctr, kAbortBigBucket, serial);
            }
            continue;
        }
#ifdef SVX_DEBUG_CHECKS
        if (threadIdx.x == 0 && (start == kInvalid || slot > h.mask || start + cnt > ctr[C_BUCKET_TOP] ||
                                 h.vals[slot] == kInvalid)) {
            printf("k_fb_fold: t %u/%u slot %u cnt %u start %u top %u val %u serial %u\n", t, nb, slot, cnt,
                   start, ctr[C_BUCKET_TOP], h.vals[slot], serial);
            __trap();
        }
#endif
        const FbRec* bk = bucket + start;
        for (int v = threadIdx.x; v < kBlockVoxels; v += kFbThreads) seg_cnt[v] = 0u;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += kFbThreads) atomicAdd(&seg_cnt[bk[i].key >> 23], 1u);
        __syncthreads();
        {   // exclusive scan of the per-voxel counts -> segment starts
            uint32_t c[kPer];
#pragma unroll
            for (int j = 0; j < kPer; ++j) c[j] = seg_cnt[threadIdx.x * kPer + j];
            Scan(scan_tmp).ExclusiveSum(c, c);
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                seg_start[threadIdx.x * kPer + j] = c[j];
                cursor[threadIdx.x * kPer + j] = c[j];
            }
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += kFbThreads) {
            const uint32_t k = bk[i].key;
            const uint32_t d = atomicAdd(&cursor[k >> 23], 1u);
            keys[d] = k;
            src1[d] = uint16_t(i);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += kFbThreads) {
            const uint32_t k = keys[i], v = k >> 23;
            const uint32_t b = seg_start[v], e = b + seg_cnt[v];
            uint32_t r = 0;
            for (uint32_t j = b; j < e; ++j) r += keys[j] < k ? 1u : 0u;
            src2[b + r] = src1[i];
        }
        __syncthreads();
        svx_tsdf_voxel* blk = pool + uint64_t(h.vals[slot]) * kBlockVoxels;
        for (int v = threadIdx.x; v < kBlockVoxels; v += kFbThreads) {
            const uint32_t b = seg_start[v];
            n_upd += fold_records(blk + v, bk, src2, b, b + seg_cnt[v]) ? 1u : 0u;
        }
        if (threadIdx.x == 0) {  // per-slot fallback state, clean for the next frame
            fbcnt[slot] = 0u;
            fbstart[slot] = kInvalid;
            fbclaim[slot] = 0u;
            fbfill[slot] = 0u;
        }
        __syncthreads();  // shared arrays are reused by the next bucket
    }
    for (int o = 16; o; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
    if ((threadIdx.x & 31) == 0 && n_upd) {
        atomicAdd(&ctr[C_UPDATED], n_upd);
        atomicAdd(&ctr[C_FB_VOXELS], n_upd);
    }
    // the last CTA to finish writes the frame report
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&ctr[C_DONE], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        ctr[C_DONE] = 0;
        if (!atomicAdd(&ctr[C_ABORT], 0u)) write_frame_end(out, ctr);
    }
}

// Big buckets (more records than k_fb_fold orders in shared memory): keys and
// record indices sorted by CUB on the device, then one thread per voxel segment.
__global__ void k_fb_extract(const FbRec* __restrict__ bk, uint32_t cnt, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ idx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    keys[i] = bk[i].key;
    idx[i] = i;
}

__global__ void k_fb_fold_sorted(HashView h, svx_tsdf_voxel* __restrict__ pool, uint32_t slot,
                                 const FbRec* __restrict__ bk, const uint32_t* __restrict__ keys,
                                 const uint32_t* __restrict__ idx, uint32_t cnt,
                                 uint32_t* __restrict__ ctr) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt || !(i == 0 || (keys[i] >> 23) != (keys[i - 1] >> 23))) return;
    uint32_t end = i + 1;
    while (end < cnt && (keys[end] >> 23) == (keys[i] >> 23)) ++end;
    svx_tsdf_voxel* blk = pool + uint64_t(h.vals[slot]) * kBlockVoxels;
    if (fold_records(blk + (keys[i] >> 23), bk, idx, i, end)) {
        atomicAdd(&ctr[C_UPDATED], 1u);
        atomicAdd(&ctr[C_FB_VOXELS], 1u);
    }
}

__global__ void k_frame_end(FrameOut* __restrict__ out, uint32_t* __restrict__ ctr) {
    // trigger first: the next frame's projection may launch (its pre-wait part reads
    // only its own points) while this frame's last kernel drains
    pdl_trigger();
    pdl_wait();
    if (ctr[C_ABORT]) return;
    write_frame_end(out, ctr);
}

// Undo the per-frame record state before re-running the band kernel of a frame.
// (fallback counts and this frame's half of the mask words of its touched blocks)
__global__ void k_reset_fb(const uint32_t* __restrict__ touched, uint32_t* __restrict__ fbcnt,
                           uint32_t* __restrict__ vmask, uint32_t parity, uint32_t* __restrict__ ctr) {
    const uint32_t n = ctr[C_TOUCHED];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n * 16u; i += gridDim.x * blockDim.x) {
        const uint32_t slot = touched[i >> 4];
        if ((i & 15u) == 0) fbcnt[slot] = 0;
        vmask[uint64_t(slot) * 32 + parity * 16 + (i & 15u)] = 0u;
    }
}

// Capacity path: every visited block key of the frame (duplicates allowed).
__global__ void __launch_bounds__(kThreads)
k_collect_keys(FrameParams f, const float* __restrict__ depth, const uint8_t* __restrict__ valid,
               const double* __restrict__ dirs, unsigned long long* __restrict__ out,
               uint32_t cap, uint32_t* __restrict__ ctr) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(f.m.W) * uint32_t(f.m.H)) return;
    const float r = depth[p];
    if (r == 0.f || double(r) > f.max_range) return;
    if (f.drop_unreliable && f.has_normals && !valid[p]) return;
    const d3 q = xform(f.pose, scale3(double(r), dir_at(dirs, p)));
    const d3 dq = sub3(q, f.origin);
    const d3 ray = div3(dq, sqrt(dot3(dq, dq)));
    const d3 tr = scale3(f.tau, ray);
    uint64_t cur_key = kEmptyKey;
    traverse_segment(sub3(q, tr), add3(q, tr), f.nu, f.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
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

FrameParams make_params(svx_map* m, svx_scan* s, const Pose& pose, const svx_integrator_cfg& cfg,
                        uint32_t parity) {
    FrameParams f{};
    f.parity = parity & 1u;
    f.m = s->dm;
    f.pose = pose;
    f.w2s = inverse_pose(pose);
    f.origin = mk(pose.t[0], pose.t[1], pose.t[2]);
    const double nu = double(m->cfg.voxel_size);
    for (int a = 0; a < 3; ++a)        // world axis
        for (int i = 0; i < 3; ++i)    // sensor component: (R^T)_{i a} = R_{a i}
            f.col[a][i] = float(nu * pose.R[3 * a + i]);
    f.tau = cfg.truncation > 0.f ? double(cfg.truncation) : double(m->cfg.truncation);
    f.max_range = cfg.max_range;
    f.alpha_eps = cfg.alpha_epsilon;
    if (!(cfg.alpha_epsilon > 0.0)) {  // alpha < eps never holds
        f.ca_hi = f.ca_lo = 2.0;
    } else if (cfg.alpha_epsilon > kPi) {  // always holds (alpha <= pi)
        f.ca_hi = f.ca_lo = -2.0;
    } else {
        f.ca_hi = std::cos(cfg.alpha_epsilon) + 1e-12;
        f.ca_lo = std::cos(cfg.alpha_epsilon) - 1e-12;
    }
    f.min_clamp = cfg.min_weight_clamp;
    f.nonproj = cfg.mode == SVX_NON_PROJECTIVE;
    f.drop_unreliable = cfg.drop_unreliable != 0;
    f.has_normals = s->has_normals;
    f.nu = nu;
    f.inv_nu = 1.0 / nu;
    f.delta = float(0.8660254037844386 * nu * (1.0 + 1e-6)) + 1e-6f;
    f.min_range_safe = float(s->model.min_range * (1.0 + 1e-4)) + 1e-4f;
    {
        const double t0 = s->model.theta0, t1 = s->model.theta0 + s->model.height_px * s->model.delta_theta;
        // polar range inside (0, pi): sin is smallest at an end of the range
        f.sin_min = (t0 > 0.0 && t1 < kPi) ? float(std::min(std::sin(t0), std::sin(t1)) - 1e-6) : 0.f;
    }
    f.dphi_f = float(s->model.delta_phi * (1.0 - 1e-6));
    f.dtheta_f = float(s->model.delta_theta * (1.0 - 1e-6));
    f.shard_rank = m->shard_rank;
    f.shard_world = m->shard_world;
    f.frame_serial = ++m->frame_serial;
    f.max_blocks = m->cfg.max_blocks;
    f.rec_cap = m->rec_cap;
    f.vox_cap = m->vox_cap;
    return f;
}

// Stages of one frame: 0 band, 1 fold, 2 fallback (+ report), 3 report only.
enum { kStageBand = 0, kStageFold = 1, kStageFallback = 2, kStageReport = 3 };

// k_fold's grid: exactly one wave of resident CTAs (register-limited to 4 per SM),
// each thread striding over ~4 listed voxels. Measured on cfg2: 41 -> 37 us per frame
// against two waves (persistent_grid), 43 us at 2/3 of a wave, 49 us at half a wave.
unsigned fold_grid(int device) {
    static int grid[64] = {0};
    if (!grid[device]) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        SVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fold, kThreads, 0));
        grid[device] = std::max(1, sms * per_sm);
    }
    return unsigned(grid[device]);
}

void launch_stages(svx_map* m, svx_scan* s, const FrameParams& f, int from, FrameOut* out) {
    const uint32_t P = uint32_t(s->P);
    HashView hv = hash_view(m);
    const PixCache* cache = reinterpret_cast<const PixCache*>(s->pixcache.p);
    const unsigned pg = persistent_grid(m->device);
    uint32_t* touched_cur = m->touched + uint64_t(f.parity) * m->cap;
    uint32_t* touched_prev = m->touched + uint64_t(f.parity ^ 1u) * m->cap;
    if (from <= kStageBand) {
        ProfMark pm(m, SVX_K_RAYCAST);
        if (!s->rowdist_fresh) {  // host-provided depth: the projection did not build it
            launch_pdl(k_row_dist, grid_for(P), kThreads, m->stream, s->depth.p, s->dm.W, s->dm.H,
                       s->rowdist.p, s->validbits.p, m->d_ctr);
            count_launch();
            s->rowdist_fresh = true;
        }
        const unsigned tiles = unsigned(((s->dm.W + kTileU - 1) / kTileU) * ((s->dm.H + kTileV - 1) / kTileV));
        launch_pdl(k_raycast_band, tiles, 256, m->stream, f, s->depth.p, s->normals.p, s->valid.p,
                   s->dirs.p, s->rowdist.p, s->validbits.p, reinterpret_cast<PixCache*>(s->pixcache.p), hv,
                   m->block_keys,
                   m->stamp, touched_cur, m->vmask, m->fbcnt, reinterpret_cast<FbRec*>(m->records.p),
                   tsdf_base(m), m->dirty, m->vlist.p, m->d_ctr);
        count_launch();
    }
    if (from <= kStageFold) {
        ProfMark pm(m, SVX_K_FOLD);
        launch_pdl(k_fold, fold_grid(m->device), kThreads, m->stream, f, s->validbits.p, cache,
                   m->block_keys, tsdf_base(m),
                   m->vlist.p, touched_prev, m->vmask, reinterpret_cast<const FbRec*>(m->records.p),
                   m->fbcnt, m->fbstart, m->fbclaim, m->fbfill, m->fbslots,
                   reinterpret_cast<FbRec*>(m->bucket.p), m->d_ctr);
        count_launch();
    }
    if (from <= kStageFallback) {
        ProfMark pm(m, SVX_K_FALLBACK);
        // pg / 2 CTAs: measured on cfg2, pg / 4 is equal, pg, pg / 8 and pg / 16 are slower
        launch_pdl(k_fb_fold, pg / 2, kFbThreads, m->stream, hv, tsdf_base(m), m->fbslots, m->fbcnt,
                   m->fbstart, m->fbclaim, m->fbfill, reinterpret_cast<const FbRec*>(m->bucket.p),
                   m->bigslots, out, f.frame_serial, m->d_ctr);
        count_launch();
    } else {
        launch_pdl(k_frame_end, 1, 1, m->stream, out, m->d_ctr);
        count_launch();
    }
    SVX_CUDA(cudaGetLastError());
}

// CapacityError path (tsdf_integrator.cpp:160-168 + voxel_store.cpp:18-20):
// blocks are allocated in sorted key order until max_blocks is reached; every
// block before the failing one is marked dirty; no voxel is updated.
[[noreturn]] void capacity_path(svx_map* m, const FrameParams& f, svx_scan* s, uint32_t before) {
    uint32_t cap = uint32_t(std::min<uint64_t>(uint64_t(s->P) * 64, 1u << 30));
    for (;;) {
        m->records_alt.alloc(cap);
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_RECORDS, 0, 4, m->stream));
        k_collect_keys<<<grid_for(s->P), kThreads, 0, m->stream>>>(f, s->depth.p, s->valid.p,
                                                                   s->dirs.p, m->records_alt.p,
                                                                   cap, m->d_ctr);
        count_launch();
        sync_counters(m);
        if (m->h_ctr[C_RECORDS] <= cap) break;
        cap = m->h_ctr[C_RECORDS];
    }
    const uint32_t n = m->h_ctr[C_RECORDS];
    std::vector<unsigned long long> keys(n);
    SVX_CUDA(cudaMemcpy(keys.data(), m->records_alt.p, sizeof(unsigned long long) * n,
                        cudaMemcpyDeviceToHost));
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::vector<unsigned long long> existing(before);
    if (before)
        SVX_CUDA(cudaMemcpy(existing.data(), m->block_keys, sizeof(unsigned long long) * before,
                            cudaMemcpyDeviceToHost));
    std::sort(existing.begin(), existing.end());
    std::vector<unsigned long long> alloc_new, dirty_keys;
    uint64_t room = m->cfg.max_blocks > before ? m->cfg.max_blocks - before : 0;
    for (unsigned long long k : keys) {
        if (!std::binary_search(existing.begin(), existing.end(), k)) {
            if (room == 0) break;  // get_or_allocate_block throws here
            alloc_new.push_back(k);
            --room;
        }
        dirty_keys.push_back(k);
    }
    const uint64_t total = before + alloc_new.size();
    ensure_blocks(m, total);
    if (!alloc_new.empty())
        SVX_CUDA(cudaMemcpy(m->block_keys + before, alloc_new.data(),
                            sizeof(unsigned long long) * alloc_new.size(), cudaMemcpyHostToDevice));
    m->n_blocks = total;
    rebuild_hash(m);
    launch_zero_blocks(m, before, alloc_new.size());
    reset_frame_state(m);
    if (!dirty_keys.empty()) {
        m->records_alt.alloc(dirty_keys.size());
        SVX_CUDA(cudaMemcpy(m->records_alt.p, dirty_keys.data(),
                            sizeof(unsigned long long) * dirty_keys.size(), cudaMemcpyHostToDevice));
        k_mark_dirty<<<grid_for(dirty_keys.size()), kThreads, 0, m->stream>>>(
            reinterpret_cast<const uint64_t*>(m->records_alt.p), uint32_t(dirty_keys.size()),
            hash_view(m), m->dirty);
        count_launch();
    }
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    throw Error(SVX_CAPACITY, "block budget exhausted (max_blocks = " +
                                  std::to_string(m->cfg.max_blocks) + ")");
}

// Host side of kAbortBigBucket: each oversized bucket is ordered by a CUB pair
// sort (key, record index) on the device and folded per voxel segment.
void big_buckets(svx_map* m) {
    const uint32_t nbig = m->h_ctr[C_FB_BIG];
    std::vector<uint32_t> slots(nbig), cnt(nbig), start(nbig);
    SVX_CUDA(cudaMemcpy(slots.data(), m->bigslots, 4 * nbig, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < nbig; ++i) {
        SVX_CUDA(cudaMemcpy(&cnt[i], m->fbcnt + slots[i], 4, cudaMemcpyDeviceToHost));
        SVX_CUDA(cudaMemcpy(&start[i], m->fbstart + slots[i], 4, cudaMemcpyDeviceToHost));
    }
    const FbRec* bucket = reinterpret_cast<const FbRec*>(m->bucket.p);
    DevBuf<uint32_t> buf;
    for (uint32_t i = 0; i < nbig; ++i) {
        const uint32_t n = cnt[i];
        buf.alloc(4ull * n);
        uint32_t *k_in = buf.p, *k_out = buf.p + n, *i_in = buf.p + 2ull * n, *i_out = buf.p + 3ull * n;
        k_fb_extract<<<grid_for(n), kThreads, 0, m->stream>>>(bucket + start[i], n, k_in, i_in);
        size_t bytes = 0;
        SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k_in, k_out, i_in, i_out, int(n), 0, 32,
                                                 m->stream));
        m->sort_tmp.alloc(bytes ? bytes : 1);
        SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->sort_tmp.p, bytes, k_in, k_out, i_in, i_out, int(n),
                                                 0, 32, m->stream));
        k_fb_fold_sorted<<<grid_for(n), kThreads, 0, m->stream>>>(
            hash_view(m), tsdf_base(m), slots[i], bucket + start[i], k_out, i_out, n, m->d_ctr);
        count_launch(2);
        SVX_CUDA(cudaMemsetAsync(m->fbcnt + slots[i], 0, 4, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fbclaim + slots[i], 0, 4, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fbfill + slots[i], 0, 4, m->stream));
        SVX_CUDA(cudaMemsetAsync(m->fbstart + slots[i], 0xFF, 4, m->stream));
    }
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    buf.release();
}

}  // namespace

unsigned persistent_grid(int device) {
    static int sms[64] = {0};
    if (!sms[device]) cudaDeviceGetAttribute(&sms[device], cudaDevAttrMultiProcessorCount, device);
    return unsigned(sms[device] * 8);  // 8 CTAs x 8 warps per SM
}

// Clears the frame scratch (masks, fallback counts, per-frame counters) after a
// host-side intervention, and re-arms the device block counters.
void reset_frame_state(svx_map* m) {
    SVX_CUDA(cudaMemsetAsync(m->vmask, 0, sizeof(uint32_t) * 32ull * m->cap, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fbcnt, 0, sizeof(uint32_t) * m->cap, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fbclaim, 0, sizeof(uint32_t) * m->cap, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fbfill, 0, sizeof(uint32_t) * m->cap, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fbstart, 0xFF, sizeof(uint32_t) * m->cap, m->stream));
    for (int c : {C_TOUCHED, C_UPDATED, C_RECORDS, C_RAYS, C_DROPPED, C_TIES, C_FB_BLOCKS,
                  C_FB_VOXELS, C_FB_BIG, C_ABORT, C_VOXLIST, C_BUCKET_TOP, C_DONE, C_TOUCHED_PREV})
        m->h_ctr[c] = 0;
    m->h_ctr[C_BLOCKS] = m->h_ctr[C_BLOCKS_BEFORE] = uint32_t(m->n_blocks);
    m->h_ctr[C_MAPPED] = uint32_t(m->mapped_blocks);
    SVX_CUDA(cudaMemcpyAsync(m->d_ctr, m->h_ctr, sizeof(uint32_t) * kNumCounters,
                             cudaMemcpyHostToDevice, m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
}

namespace {
void put_ctr(svx_map* m, int c, uint32_t v) {
    m->h_ctr[c] = v;
    SVX_CUDA(cudaMemcpyAsync(m->d_ctr + c, &m->h_ctr[c], 4, cudaMemcpyHostToDevice, m->stream));
}
}  // namespace

void run_frames(svx_map* m, const FrameJob* jobs, int n, const svx_integrator_cfg& cfg,
                svx_frame_report* reps) {
    if (!(cfg.alpha_epsilon > 0.0)) throw Error(SVX_INVALID_ARGUMENT, "alpha_epsilon must be > 0");
    if (n <= 0) return;
    for (int i = 0; i < n; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
        if (!jobs[i].project && !jobs[i].scan->has_normals && cfg.mode == SVX_NON_PROJECTIVE)
            throw Error(SVX_INVALID_ARGUMENT, "non-projective mode needs a normal image");
    }
    m->outs.alloc(size_t(n));
    // frame reports start "not done": the resume logic finds the aborted frame as the
    // first report without ok (stale reports of an earlier batch must not count)
    SVX_CUDA(cudaMemsetAsync(m->outs.p, 0, sizeof(FrameOut) * size_t(n), m->stream));
    if (m->h_outs_n < size_t(n)) {
        if (m->h_outs) cudaFreeHost(m->h_outs);
        SVX_CUDA(cudaMallocHost(&m->h_outs, sizeof(FrameOut) * n));
        m->h_outs_n = size_t(n);
    }
    // per-frame buffers sized for the largest scan of the batch
    uint64_t pmax = 0, nmax = 0;
    for (int i = 0; i < n; ++i) {
        pmax = std::max<uint64_t>(pmax, uint64_t(jobs[i].scan->P));
        nmax = std::max<uint64_t>(nmax, jobs[i].n);
        if (jobs[i].project) jobs[i].scan->lexkey.alloc(std::min<uint64_t>(2 * jobs[i].n + 2, 0xFFFFFFF0ull));
    }
    if (m->vox_cap < 16 * pmax) {
        m->vox_cap = uint32_t(std::min<uint64_t>(16 * pmax, 0xFFFFFFF0ull));
        m->vlist.alloc(m->vox_cap);
    }
    // pool headroom for the whole batch (an overflow aborts and resumes below)
    // (an exhausted headroom costs one abort + resume; over-mapping costs physical
    // memory and cuMemCreate time, so size it from the recent new-block rate)
    const uint64_t head = m->test_pool_head ? m->test_pool_head
                                            : std::max<uint64_t>(32768, uint64_t(2.0 * m->new_ema * n));
    ensure_blocks(m, m->n_blocks + head, 4 * head);
    std::vector<FrameParams> fps(n);
    std::vector<int> parity(n, 0);
    std::vector<char> launched(n, 0);
    // host ingest ring: frame i's points go to slot i % R on the copy stream, at most
    // R - 1 frames ahead of the frame being launched; a slot is refilled only after
    // the projection of the frame that used it (event ingest_used)
    constexpr int R = svx_map::kIngestSlots;
    const bool ingest = jobs[0].host_ingest;
    if (ingest) {
        if (!m->copy_stream) {
            SVX_CUDA(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
            for (int r = 0; r < R; ++r) {
                SVX_CUDA(cudaEventCreateWithFlags(&m->ingest_ready[r], cudaEventDisableTiming));
                SVX_CUDA(cudaEventCreateWithFlags(&m->ingest_used[r], cudaEventDisableTiming));
            }
        }
        uint64_t most = 1;
        for (int i = 0; i < n; ++i) most = std::max<uint64_t>(most, jobs[i].n * uint64_t(jobs[i].stride));
        for (int r = 0; r < R; ++r) {
            m->ingest[r].alloc(most);
            SVX_CUDA(cudaEventRecord(m->ingest_used[r], m->stream));
        }
    }
    // fills the report of completed frame i (its FrameOut is final) and numbers it
    auto commit = [&](int i) {
        const FrameOut& o = m->h_outs[i];
        reps[i].frame = m->tsdf_frames++;
        reps[i].updated_voxels = o.updated;
        reps[i].new_blocks = o.new_blocks;
        m->new_ema = m->new_ema == 0.0 ? double(o.new_blocks) : 0.9 * m->new_ema + 0.1 * double(o.new_blocks);
        jobs[i].scan->dropped = o.dropped;
        m->prof_acc.frames += 1;
        m->prof_acc.rays += o.rays;
        m->prof_acc.touched_blocks += o.touched;
        m->prof_acc.new_blocks += o.new_blocks;
        m->prof_acc.updated_voxels += o.updated;
        m->prof_acc.fallback_voxels += o.fb_voxels;
    };
    int f0 = 0, stage0 = 0;
    for (;;) {
        const auto te0 = std::chrono::steady_clock::now();
        int next_copy = f0;
        for (int i = f0; i < n; ++i) {
            const FrameJob& j = jobs[i];
            const int from = i == f0 ? stage0 : 0;
            const float* pts = j.pts;
            if (ingest) {
                for (; next_copy < n && next_copy < i + R; ++next_copy) {
                    const FrameJob& c = jobs[next_copy];
                    const int r = next_copy % R;
                    SVX_CUDA(cudaStreamWaitEvent(m->copy_stream, m->ingest_used[r], 0));
                    if (c.n)
                        SVX_CUDA(cudaMemcpyAsync(m->ingest[r].p, c.pts, 4ull * c.n * c.stride,
                                                 cudaMemcpyHostToDevice, m->copy_stream));
                    SVX_CUDA(cudaEventRecord(m->ingest_ready[r], m->copy_stream));
                }
                SVX_CUDA(cudaStreamWaitEvent(m->stream, m->ingest_ready[i % R], 0));
                pts = m->ingest[i % R].p;
            }
            if (!launched[i] || (i > f0)) {
                if (j.project) {
                    if (launched[i]) j.scan->parity = parity[i];
                    parity[i] = j.scan->parity;
                    launch_project(j.scan, pts, j.n, j.stride, j.pose);
                    if (ingest) SVX_CUDA(cudaEventRecord(m->ingest_used[i % R], m->stream));
                }
                fps[i] = make_params(m, j.scan, j.pose, cfg, uint32_t(m->tsdf_frames + i));
                launched[i] = 1;
            }
            launch_stages(m, j.scan, fps[i], from, m->outs.p + i);
        }
        if (m->prof)
            m->prof_acc.host_enqueue_ms +=
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
        SVX_CUDA(cudaMemcpyAsync(m->h_outs, m->outs.p, sizeof(FrameOut) * n,
                                 cudaMemcpyDeviceToHost, m->stream));
        sync_counters(m);
        if (ingest) SVX_CUDA(cudaStreamSynchronize(m->copy_stream));
        const uint32_t abort = m->h_ctr[C_ABORT];
        if (!abort) break;
        const auto tr0 = std::chrono::steady_clock::now();
        for (int b = 0; b < 8; ++b) m->prof_acc.aborts[b] += (abort >> b) & 1u;
#ifdef SVX_DEBUG_CHECKS
        std::fprintf(stderr, "abort %#x f0 %d blocks %u before %u mapped %u records %u rec_cap %u touched %u fbb %u top %u\n",
                     abort, f0, m->h_ctr[C_BLOCKS], m->h_ctr[C_BLOCKS_BEFORE], m->h_ctr[C_MAPPED],
                     m->h_ctr[C_RECORDS], m->rec_cap, m->h_ctr[C_TOUCHED], m->h_ctr[C_FB_BLOCKS],
                     m->h_ctr[C_BUCKET_TOP]);
#endif
        // the first frame of this pass without a report is the one that aborted
        int fa = f0;
        while (fa < n && m->h_outs[fa].ok) ++fa;
        if (fa >= n) fa = n - 1;
        svx_scan* s = jobs[fa].scan;
        const uint32_t before = m->h_ctr[C_BLOCKS_BEFORE];
        if (abort & kAbortKey) {
            // like the capacity path: the frames before the failing one are complete
            // (reported and numbered); the failing frame is numbered (the reference
            // numbers a frame before it can throw) and leaves no block behind: its
            // partially inserted blocks (possibly beyond the mapped, zero-filled pool)
            // are dropped and their dirty flags cleared
            for (int i = 0; i < fa; ++i) commit(i);
            m->tsdf_frames++;
            const uint64_t hi = std::min<uint64_t>(m->h_ctr[C_BLOCKS], m->cfg.max_blocks);
            if (hi > before) SVX_CUDA(cudaMemsetAsync(m->dirty + before, 0, hi - before, m->stream));
            m->n_blocks = before;
            rebuild_hash(m);
            reset_frame_state(m);
            throw Error(SVX_INVALID_ARGUMENT,
                        "block coordinate outside the device key range [-2^20, 2^20)");
        }
        if (abort & (kAbortCapacity | kAbortHash)) {
            for (int i = 0; i < fa; ++i) commit(i);
            m->tsdf_frames++;
            m->n_blocks = before;
            capacity_path(m, fps[fa], s, before);
        }
        int stage = kStageReport;
        const uint32_t par = fps[fa].parity;
        if (abort & (kAbortRecords | kAbortVoxList)) {
            // grow the buffer and re-run the band kernel of this frame with a fresh
            // stamp, after clearing what its first run left: this frame's mask
            // words (so every voxel is listed again), fallback counts, counters
            ensure_blocks(m, uint64_t(m->h_ctr[C_BLOCKS]) + head);
            if (abort & kAbortRecords) {
                m->rec_cap = std::max<uint32_t>(m->h_ctr[C_RECORDS] + (m->h_ctr[C_RECORDS] >> 1),
                                                m->rec_cap * 2);
                m->records.alloc(2ull * m->rec_cap);
                m->bucket.alloc(2ull * m->rec_cap);
                fps[fa].rec_cap = m->rec_cap;
            }
            if (abort & kAbortVoxList) {
                m->vox_cap = uint32_t(std::min<uint64_t>(uint64_t(m->h_ctr[C_VOXLIST]) * 2, 0xFFFFFFF0ull));
                m->vlist.alloc(m->vox_cap);
                fps[fa].vox_cap = m->vox_cap;
            }
            k_reset_fb<<<256, kThreads, 0, m->stream>>>(m->touched + uint64_t(par) * m->cap, m->fbcnt,
                                                        m->vmask, par, m->d_ctr);
            count_launch();
            // blocks created by the first run are found again (not created): zero them all here
            launch_zero_blocks(m, before, uint64_t(m->h_ctr[C_BLOCKS]) - before);
            fps[fa].frame_serial = ++m->frame_serial;
            for (int c : {C_RECORDS, C_TOUCHED, C_VOXLIST}) put_ctr(m, c, 0);
            stage = kStageBand;
        } else if (abort & kAbortPool) {
            // the band ran to completion; blocks beyond the mapped pool were not
            // zero-filled: map more, zero all of the frame's new blocks, fold
            ensure_blocks(m, uint64_t(m->h_ctr[C_BLOCKS]) + head);
            launch_zero_blocks(m, before, uint64_t(m->h_ctr[C_BLOCKS]) - before);
            stage = kStageFold;
        } else if (abort & kAbortBigBucket) {
            big_buckets(m);
            put_ctr(m, C_DONE, 0);
            stage = kStageReport;
        }
        put_ctr(m, C_ABORT, 0);
        put_ctr(m, C_MAPPED, uint32_t(m->mapped_blocks));
        f0 = fa;
        stage0 = stage;
        m->prof_acc.host_resume_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
    }
    for (int i = 0; i < n; ++i) commit(i);
    m->n_blocks = m->h_ctr[C_BLOCKS];
}

}  // namespace svx
