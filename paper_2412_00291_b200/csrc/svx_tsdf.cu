// K3-K5: TsdfIntegrator::integrate_frame on the device (tsdf_integrator.cpp:97-258),
// for GROUPS of up to kMaxG consecutive frames per launch sequence.
//
// What the reference does per frame, and what is independent across frames:
//   * phase 1 (.cpp:112-139) casts the band of every valid pixel: pure geometry of the
//     frame's images and pose, so every frame of a group runs its band in ONE launch;
//   * which voxels a frame updates, their own pixel (.cpp:232) and whether a visiting
//     ray's pixel is measurable (.cpp:172-181) are geometry too;
//   * only the VALUES depend on the voxel's state: the non-projective distance reads the
//     voxel's pre-update gradient (.cpp:190-196), and the fold reads W and D (.cpp:239-247).
// So a group is integrated as: project all frames; band DDA of all frames (visit masks per
// frame); then ONE thread per distinct visited voxel applies the group's frames to it in
// frame order, with the voxel in registers - exactly the sequence of the reference's
// consecutive integrate_frame calls for that voxel.
//
// Kernels per group (one stream, programmatic dependent launch, no host synchronisation):
//   k_band       CTA = (frame g, 32 x 8 pixel tile), thread = pixel: pixel cache (ray, range,
//                world normal; the measurement inputs of .cpp:173-186, once per pixel),
//                amortised band DDA (tsdf_integrator.hpp:93-135) into a shared-memory table
//                of the tile's blocks and 512-bit voxel masks; per visit the own-pixel test
//                of the voxel (FP32 with an exact-decision margin): a voxel whose own pixel
//                has no return is measured by every visiting ray in the reference
//                (.cpp:232-238), so such a visit becomes a fallback record (block, voxel,
//                frame, pixel). Epilogue: one hash find-or-insert per distinct block (new
//                block -> next pool index, zero-filled by the tile), the group's touched
//                list, the frame's visit-mask row (RED.OR) and the union row (ATOM.OR: the
//                words a tile sets first become the group's word list).
//   (sort)       the group's fallback records, radix-sorted on their (block, voxel,
//                frame, pixel) bits (cub::DeviceRadixSort over the record buffer; O(records)
//                however many rays visit a voxel).
//   k_fb_runs    one descriptor per (voxel, frame) run of the sorted records: per frame
//                the reference's ascending (v, u) visit order (.cpp:141-146,215-216).
//   k_fold       one launch per frame g of the group: thread per fallback descriptor of
//                frame g (its records in pixel order), then the frame's visited-voxel list,
//                32 per warp (own pixel, measurement, accumulate-then-merge fold, Eq. 4-5);
//                each voxel then holds frames 0..g. The last frame's launch marks dirty
//                blocks, counts per-frame touched / new blocks, clears the masks, and its
//                last CTA writes the frames' reports.
// Any abort (pool growth, buffer growth, capacity, key range) stops the batch; the host
// rolls the aborted group back (its blocks, hash entries and masks) and retries it
// (CapacityError and key-range errors: frame by frame, reproducing the reference's
// per-frame behaviour).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <math_constants.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <memory>
#include <vector>

#include "svx_map.hpp"

namespace svx {

// Constants shared by every frame of a group (same model, same integrator config).
struct GroupConsts {
    Model m;
    double tau, max_range, alpha_eps, nu, inv_nu;
    double inv_2tau;      // 1 / (2 tau), rounded: the weight's quotient estimate
    double ca_hi, ca_lo;  // cos(alpha_eps) +- 1e-12: margins of the alpha < eps branch
    float min_clamp;
    // band_all_own(): half voxel diagonal, safe min range, min sin(polar) over the
    // vertical field of view, pixel pitches
    float delta, min_range_safe, sin_min, dphi_f, dtheta_f;
    int nonproj, drop_unreliable, has_normals;
    int32_t shard_rank, shard_world;
    // exchange mode (multi-GPU data plane): this rank casts the rays of its
    // share of the tiles and sends the visits of blocks other ranks own to them
    int exchange;
    uint32_t xcap;  // send-list entries per destination rank
    uint32_t serial;    // group serial (touched stamps)
    uint32_t G, P, VW;  // frames, pixels per frame, valid-bit words per frame
    uint32_t tiles;     // band tiles per frame
    uint32_t max_blocks, rec_cap, vox_cap;
    uint32_t pbits;  // pixel bits of a fallback record (make_record)
};

// Per-frame pose data.
struct FramePose {
    Pose pose, w2s;
    d3 origin;
    float col[3][3];  // nu * (R^T e_m): sensor-frame step of +1 voxel along world axis m
    float pad;
};
static_assert(sizeof(FramePose) % 8 == 0, "FramePose layout");

struct GroupParams {
    GroupConsts c;
    FramePose f[kMaxG];
};

// Device images of the group's frames (frame g at slot g of the scan).
struct ScanSlots {
    const float* depth;
    const float* normals;
    const uint8_t* valid;
    const double* dirs;
    const uint8_t* rowdist;
    const uint32_t* validbits;
    uint8_t* cache;  // PixCache[slots][P]
};

struct PixCache {
    double ray[3];
    double range;
    float n[3];
    uint32_t flags;  // bit0: measurable, bit1: has normal
};
static_assert(sizeof(PixCache) == 48, "PixCache layout");

struct Term {  // one (pixel, voxel) measurement
    float wg, w, nx, ny, nz;
    uint32_t flags;  // bit0: measured, bit1: has normal
};

namespace {

constexpr int kThreads = 256;

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

__device__ inline const PixCache* cache_of(const ScanSlots& sc, const GroupConsts& c, uint32_t g) {
    return reinterpret_cast<const PixCache*>(sc.cache) + uint64_t(g) * c.P;
}

// Position of the r-th (0-based) set bit of x (r < popc(x)).
__device__ inline uint32_t select_bit(uint32_t x, uint32_t r) {
    uint32_t pos = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t low = x & ((1u << s) - 1u);
        const uint32_t n = __popc(low);
        if (r >= n) {
            r -= n;
            x >>= s;
            pos += uint32_t(s);
        } else {
            x = low;
        }
    }
    return pos;
}

// Own pixel of a voxel centre: project_point(world_to_sensor * c) (tsdf_integrator.cpp:232);
// pc is world_to_sensor * c in FP64 (reference formula).
__device__ inline uint32_t own_pixel(const Model& m, d3 pc) {
    const uint32_t q = pixel_fast(float(pc.x), float(pc.y), float(pc.z), m, m.r2_lo, m.r2_hi);
    return q == kNeedFp64 ? pixel_fp64(pc, m) : q;
}

// Row distance (columns, azimuth wraps) from each pixel to the nearest pixel of its row
// without a return, capped at kRmax + 1; plus the valid bits. For images the caller
// uploaded (the projection builds both itself).
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

// Chebyshev distance from pixel p to the nearest pixel without a return or to the
// top/bottom image edge, capped at kRmax + 1: every pixel closer than that holds a return.
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

// True when no voxel visited by the band of this ray can have its own pixel without a
// return: the voxel centre lies within delta = sqrt(3)/2 nu of the ray, so its direction is
// within angle a <= 1.1 delta / d_min of the pixel-centre direction, i.e. within k pixels;
// every pixel within k of p holds a return.
__device__ inline bool band_all_own(const GroupConsts& c, const uint8_t* __restrict__ hd,
                                    uint32_t p, float r) {
    const float dmin = r - float(c.tau) - c.delta;
    if (!(dmin > c.min_range_safe)) return false;
    const float x = c.delta / dmin;
    if (x > 0.3f) return false;
    const float a = 1.1f * x;  // asin(x) <= 1.1 x for x <= 0.3
    const float s = c.sin_min - a;
    if (s < 0.1f || a > s * (1.f / 3.f)) return false;
    // azimuth offset <= 2 asin(sin(a/2) / s) <= 1.05 a / s for a / s <= 1/3
    const int ku = int(floorf(1.05f * a / (s * c.dphi_f) + 0.5f)) + 1;
    const int kv = int(floorf(a / c.dtheta_f + 0.5f)) + 1;
    const int k = max(ku, kv);
    if (k > kRmax) return false;
    return valid_radius(hd, c.m.W, c.m.H, p) > k;
}

struct Accum {
    double wd, w, wx, wy, wz;
};

// nonprojective_distance (tsdf_integrator.cpp:39-46)
__device__ inline double nonprojective_distance(double psi, double theta, double alpha, double eps) {
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

// Gamma(d) of the non-projective distance from the clamped cosines ct = cos(theta) and
// ca = cos(alpha). The reference evaluates theta = acos(ct), alpha = acos(ca) and then
// cos/sin of both with libm (tsdf_integrator.cpp:39-46,195-196). Fast path without
// transcendentals: cos(acos(x)) = x and sin(acos(x)) = sqrt((1-x)(1+x)) up to
// |err| <= 2e-15 (1-ulp libm acos/cos/sin: pi * 2^-52 + 2^-52), an absolute bound E on the
// resulting d, and the f32 value the reference stores, float(clamp(d, +-tau)), accepted
// only when all of [d - E, d + E] rounds to it. The branch alpha < eps is decided on ca
// against cos(eps) with a 1e-12 margin (acos is strictly decreasing). Otherwise (ca near
// cos(eps), sin(alpha) < 1e-6, or an interval straddling a float boundary: ~1e-4 of the
// voxels) the reference formula is evaluated with CUDA's FP64 acos/sincos.
//
// ct and ca may carry an input error: the fast path forms them from g * rsqrt(|g|^2) instead
// of the reference's g / sqrt(|g|^2) (measure_term), within kDot of the reference's values.
// That error enters the bound additively (cosines) and through sqrt(1 - x^2), whose change
// is at most |x'^2 - x^2| / sqrt(1 - x'^2) <= 2.1 kDot / sqrt(1 - x'^2).
// Returns false when undecided; the caller then evaluates the reference formula from the
// reference's own ct, ca (gamma_reference).
constexpr double kDot = 3e-15;
__device__ __forceinline__ bool gamma_fast(const GroupConsts& c, double psi, double ct, double ca, float& out) {
    constexpr double kAbs = 2e-15 + kDot, kRel = 4e-15;  // kRel: libm + our rsqrt-based roots
    double d, e;
    if (ca > c.ca_hi) {  // alpha < eps: |cos theta| * psi
        d = fabs(ct) * psi;
        e = fabs(psi) * (kAbs + kRel * fabs(ct)) + 1e-15 * fabs(d);
    } else if (ca < c.ca_lo) {
        const double tt = (1.0 - ct) * (1.0 + ct), ss = (1.0 - ca) * (1.0 + ca);
        if (!(tt > 1e-14 && ss > 1e-12)) return false;  // sin theta < 1e-7 or sin alpha < 1e-6
        const double rt = rsqrt_est(tt), inv_sa = rsqrt_est(ss);  // (<= 3 ulp each)
        const double st = tt * rt, sa = ss * inv_sa;
        const double a = ca - 1.0;
        const double t1 = fabs(a * st * inv_sa), t2 = fabs(ct * psi);
        const double mag = t1 + t2;
        d = psi >= 0.0 ? mag : -mag;
        const double da = kAbs + kRel * fabs(a);
        const double dst = kAbs + kRel * st + 2.1 * kDot * rt;
        const double dsa = kAbs + kRel * sa + 2.1 * kDot * inv_sa;
        e = 1.01 * ((fabs(a) * dst + st * da + t1 * dsa) * inv_sa + fabs(psi) * (kAbs + kRel * fabs(ct))) +
            4e-15 * mag;
    } else {
        return false;
    }
    // float(clamp(x, +-tau)) is monotonic in x: [d - e, d + e] decides it when both ends agree
    const double lo = d - e, hi = d + e;
    if (lo > -c.tau && hi < c.tau) {
        const float flo = float(lo), fhi = float(hi);
        if (__float_as_uint(flo) != __float_as_uint(fhi)) return false;
        out = flo;
        return true;
    }
    const float flo = truncate_f(lo, c.tau), fhi = truncate_f(hi, c.tau);
    if (!(flo == fhi && __float_as_uint(flo) == __float_as_uint(fhi))) return false;
    out = flo;
    return true;
}

// The reference's own evaluation (the undecided cases).
__device__ inline float gamma_reference(const GroupConsts& c, double psi, d3 ray, d3 g, const float nw[3]) {
    const double gz = dot3(g, g);
    if (gz > 0.0) g = div3(g, sqrt(gz));
    double ct = dot3(neg3(ray), g);
    ct = ct < -1.0 ? -1.0 : (1.0 < ct ? 1.0 : ct);
    double ca = dot3(g, mk(nw[0], nw[1], nw[2]));
    ca = ca < -1.0 ? -1.0 : (1.0 < ca ? 1.0 : ca);
    return truncate_f(nonprojective_distance(psi, acos(ct), acos(ca), c.alpha_eps), c.tau);
}

// measure lambda (tsdf_integrator.cpp:172-205) for pixel p of a frame, from its pixel
// cache: the contribution (w * Gamma(d), w, w * n) as the reference forms it, in f32.
// vox is the voxel's state before this frame (the pre-update gradient).
__device__ inline Term measure_term(const GroupConsts& c, d3 origin, const PixCache* __restrict__ cache,
                                    uint32_t p, d3 center, const svx_tsdf_voxel& vox) {
    Term t{0.f, 0.f, 0.f, 0.f, 0.f, 0u};
    const PixCache& pc = cache[p];
    const uint32_t flags = pc.flags;
    if (!(flags & 1u)) return t;
    const bool have_normal = flags & 2u;
    const d3 ray = mk(pc.ray[0], pc.ray[1], pc.ray[2]);
    const double psi = pc.range - dot3(sub3(center, origin), ray);
    if (fabs(psi) > c.tau) return t;
    const float nw[3] = {pc.n[0], pc.n[1], pc.n[2]};
    float gamma;
    if (c.nonproj && have_normal) {
        float g[3] = {nw[0], nw[1], nw[2]};
        const float gsq =
            (vox.gradient[0] * vox.gradient[0] + vox.gradient[1] * vox.gradient[1]) + vox.gradient[2] * vox.gradient[2];
        if (vox.weight > 0.f && gsq > 1e-12f) {
            g[0] = vox.gradient[0];
            g[1] = vox.gradient[1];
            g[2] = vox.gradient[2];
        }
        // g.normalized() (g / sqrt(|g|^2)) as g * rsqrt(|g|^2): each component within 3 ulp,
        // so ct and ca within kDot of the reference's (|ray| = 1, |nw| = 1 + O(1e-7))
        const d3 g0 = mk(g[0], g[1], g[2]);
        const double gz = dot3(g0, g0);
        const d3 gd = gz > 0.0 ? scale3(rsqrt(gz), g0) : g0;
        double ct = dot3(neg3(ray), gd);
        ct = ct < -1.0 ? -1.0 : (1.0 < ct ? 1.0 : ct);
        double ca = dot3(gd, mk(nw[0], nw[1], nw[2]));
        ca = ca < -1.0 ? -1.0 : (1.0 < ca ? 1.0 : ca);
        if (!gamma_fast(c, psi, ct, ca, gamma)) gamma = gamma_reference(c, psi, ray, g0, nw);
    } else {
        gamma = truncate_f(psi, c.tau);
    }
    // observation_weight (tsdf_integrator.cpp:48-51): float(clamp((psi + tau) / 2 tau)),
    // from the quotient estimate when that decides the float, else the exact division
    const double lo = double(c.min_clamp);
    float w_obs;
    {
        const double q = (psi + c.tau) * c.inv_2tau, dq = fabs(q) * kQuotTol;
        const double q0 = q - dq, q1 = q + dq;
        const float f0 = float(q0 < lo ? lo : (1.0 < q0 ? 1.0 : q0));
        const float f1 = float(q1 < lo ? lo : (1.0 < q1 ? 1.0 : q1));
        if (__float_as_uint(f0) == __float_as_uint(f1)) {
            w_obs = f0;
        } else {
            double wr = (psi + c.tau) / (2.0 * c.tau);
            wr = wr < lo ? lo : (1.0 < wr ? 1.0 : wr);
            w_obs = float(wr);
        }
    }
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
// (the f32 quotients through f32_div / the rsqrt estimate: the same floats, fewer FP64
// divisions and square roots)
__device__ inline void fold(svx_tsdf_voxel& vox, const Accum& acc) {
    const double w_old = double(vox.weight);
    vox.distance = f32_div(w_old * double(vox.distance) + acc.wd, w_old + acc.w);
    vox.weight = float(w_old + acc.w);
    const d3 bl = mk(w_old * double(vox.gradient[0]) + acc.wx, w_old * double(vox.gradient[1]) + acc.wy,
                     w_old * double(vox.gradient[2]) + acc.wz);
    const double s2 = dot3(bl, bl);
    // norm > 1e-12 decided on s2 away from 1e-24; float(bl_i / norm) from bl_i * rsqrt(s2)
    // (within ~3 ulp of bl_i / fl(sqrt(s2))) when that decides the float
    bool upd;
    if (s2 > 1.0000001e-24) upd = true;
    else if (s2 < 0.9999999e-24) upd = false;
    else upd = sqrt(s2) > 1e-12;
    if (!upd) return;
    const double r = s2 < 1e300 ? rsqrt(s2) : 0.0;
    const double b[3] = {bl.x, bl.y, bl.z};
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double q = b[i] * r, d = fabs(q) * kQuotTol;
        const float f0 = float(q - d), f1 = float(q + d);
        if (r > 0.0 && __float_as_uint(f0) == __float_as_uint(f1)) {
            vox.gradient[i] = f0;
        } else {
            if (nrm == 0.0) nrm = sqrt(s2);
            vox.gradient[i] = float(b[i] / nrm);
        }
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

// Fallback visit record: (pool index, voxel, frame of the group, pixel), packed so that the
// unsigned order is (block, voxel, frame, pixel): pixel in the low pb bits (pb = bits of the
// scan's pixel count), frame in the next 4, voxel in the next 9, pool index above. The
// group's records are sorted on those bits (k_fb_runs).
__device__ inline unsigned long long make_record(uint32_t idx, int lin, uint32_t g, uint32_t p, uint32_t pb) {
    return (((static_cast<unsigned long long>(idx) << 9 | static_cast<unsigned long long>(lin)) << 4 |
             static_cast<unsigned long long>(g)) << pb) | p;
}
__device__ inline uint32_t rec_pixel(unsigned long long r, uint32_t pb) { return uint32_t(r & ((1ull << pb) - 1)); }

// Applies frame g to the voxel at vp (tsdf_integrator.cpp:224-248): the own pixel of the
// voxel centre if it holds a return (.cpp:232-233), else every visiting ray of the frame
// in ascending pixel order (.cpp:235-236), given as `recs` (its fallback records, sorted
// by pixel). Without records (kRec = false), a voxel whose own pixel has no return returns
// kFallback and is left alone: a fallback descriptor (k_fb_runs) applies it. Returns 1 when
// the voxel was updated.
constexpr uint32_t kFallback = 0xFFFFFFFFu;

// The own-pixel measurement and fold of one voxel through the generic code (each quotient
// decided separately, exact divisions where undecided): the rare voxels fold_own_fast
// cannot decide.
__device__ __noinline__ uint32_t fold_own_exact(const GroupConsts& c, d3 origin, const PixCache* __restrict__ cache,
                                                uint32_t own, d3 center, svx_tsdf_voxel* vp) {
    svx_tsdf_voxel vox = load_voxel(vp);
    const Term t = measure_term(c, origin, cache, own, center, vox);
    if (!(t.flags & 1u)) return 0;
    Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
    accumulate(acc, t);
    fold(vox, acc);
    store_voxel(vp, vox);
    return 1;
}

// Own-pixel measurement + fold (one term: tsdf_integrator.cpp:172-205,232-247) as ONE
// branch-free decision chain: every f32 result (Gamma, weight, D, gradient) comes from an
// estimate with an error bound, and the chain reports whether all of them were decided.
// Only an undecided voxel takes the generic path (fold_own_exact), so the common case pays
// one reconvergence point instead of one per quotient.
__device__ __forceinline__ uint32_t fold_own_fast(const GroupConsts& c, d3 origin, const PixCache* __restrict__ cache,
                                                  uint32_t own, d3 center, svx_tsdf_voxel* vp, svx_tsdf_voxel vox) {
    const PixCache& pc = cache[own];
    const uint32_t flags = pc.flags;
    if (!(flags & 1u)) return 0;
    const bool have_normal = flags & 2u;
    const d3 ray = mk(pc.ray[0], pc.ray[1], pc.ray[2]);
    const double psi = pc.range - dot3(sub3(center, origin), ray);
    if (fabs(psi) > c.tau) return 0;
    const float nw0 = pc.n[0], nw1 = pc.n[1], nw2 = pc.n[2];
    bool ok = true;
    float gamma;
    if (c.nonproj && have_normal) {
        const float gsq =
            (vox.gradient[0] * vox.gradient[0] + vox.gradient[1] * vox.gradient[1]) + vox.gradient[2] * vox.gradient[2];
        const bool use_g = vox.weight > 0.f && gsq > 1e-12f;
        const d3 g0 = mk(use_g ? vox.gradient[0] : nw0, use_g ? vox.gradient[1] : nw1, use_g ? vox.gradient[2] : nw2);
        const double gz = dot3(g0, g0);
        const d3 gd = gz > 1e-300 ? scale3(rsqrt_est(gz), g0) : (gz > 0.0 ? scale3(rsqrt(gz), g0) : g0);  // within kDot
        double ct = dot3(neg3(ray), gd);
        ct = fmin(fmax(ct, -1.0), 1.0);
        double ca = dot3(gd, mk(nw0, nw1, nw2));
        ca = fmin(fmax(ca, -1.0), 1.0);
        ok = gamma_fast(c, psi, ct, ca, gamma);
    } else {
        gamma = truncate_f(psi, c.tau);
    }
    // observation_weight: float(clamp((psi + tau) / 2 tau, min_clamp, 1))
    float w_obs;
    {
        const double lo = double(c.min_clamp);
        const double q = (psi + c.tau) * c.inv_2tau, dq = fabs(q) * kQuotTol;
        bool wok;
        if (q + dq < lo) {
            w_obs = c.min_clamp;
            wok = true;
        } else if (q - dq > 1.0) {
            w_obs = 1.f;
            wok = true;
        } else {
            wok = q - dq > lo && q + dq < 1.0 && f32_of_est(q, w_obs);
        }
        ok = ok && wok;
    }
    // the term and the accumulate-then-merge fold, in the reference's operation order
    const double wd = 0.0 + double(w_obs * gamma), w = 0.0 + double(w_obs);
    const double wx = have_normal ? 0.0 + double(w_obs * nw0) : 0.0;
    const double wy = have_normal ? 0.0 + double(w_obs * nw1) : 0.0;
    const double wz = have_normal ? 0.0 + double(w_obs * nw2) : 0.0;
    const double w_old = double(vox.weight);
    svx_tsdf_voxel out;
    {
        const double num = w_old * double(vox.distance) + wd, den = w_old + w;
        ok = ok && den > 1e-300 && den < 1e300 && f32_of_est(num * rcp_est(den), out.distance);
        out.weight = float(den);
    }
    const double bx = w_old * double(vox.gradient[0]) + wx, by = w_old * double(vox.gradient[1]) + wy,
                 bz = w_old * double(vox.gradient[2]) + wz;
    const double s2 = (bx * bx + by * by) + bz * bz;
    // norm > 1e-12 decided on s2 away from 1e-24 (else undecided); float(b_i / norm) from
    // b_i * rsqrt(s2) when that decides the float
    const bool upd = s2 > 1.0000001e-24;
    ok = ok && (upd || s2 < 0.9999999e-24) && s2 < 1e300;
    if (upd) {
        const double r = rsqrt_est(s2);
        const bool g0 = f32_of_est(bx * r, out.gradient[0]);
        const bool g1 = f32_of_est(by * r, out.gradient[1]);
        const bool g2 = f32_of_est(bz * r, out.gradient[2]);
        ok = ok && g0 && g1 && g2;
    } else {
        out.gradient[0] = vox.gradient[0];
        out.gradient[1] = vox.gradient[1];
        out.gradient[2] = vox.gradient[2];
    }
    if (!ok) return fold_own_exact(c, origin, cache, own, center, vp);
    store_voxel(vp, out);
    return 1;
}

template <bool kRec>
__device__ __forceinline__ uint32_t fold_one(const GroupConsts& c, const FramePose& f, uint32_t g, svx_tsdf_voxel* vp, d3 center,
                             const ScanSlots& sc, const unsigned long long* __restrict__ recs, uint32_t nrec) {
    const PixCache* cache = cache_of(sc, c, g);
    Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
    bool measured = false;
    svx_tsdf_voxel vox = load_voxel(vp);  // in flight while the own pixel is computed
    if constexpr (!kRec) {
        const uint32_t own = own_pixel(c.m, xform(f.w2s, center));
        if (own == kInvalid || !pixel_has_return(sc.validbits + uint64_t(g) * c.VW, own)) return kFallback;
        return fold_own_fast(c, f.origin, cache, own, center, vp, vox);
    } else {
        for (uint32_t j = 0; j < nrec; ++j) {
            const Term t = measure_term(c, f.origin, cache, rec_pixel(recs[j], c.pbits), center, vox);
            if (t.flags & 1u) {
                accumulate(acc, t);
                measured = true;
            }
        }
    }
    if (!measured) return 0;
    fold(vox, acc);
    store_voxel(vp, vox);
    return 1;
}

// A fallback voxel with many visiting rays in frame g: the lanes of one warp measure its
// records in parallel (32 at a time), lane 0 then takes the terms by shuffle in record
// (= ascending pixel) order and sums them as the reference does (tsdf_integrator.cpp:
// 235-236): the serial part per record is the accumulation, not the measurement. Returns 1
// on lane 0 when the voxel was updated.
#ifndef SVX_WARP_RECS
#define SVX_WARP_RECS 1
#endif
// descriptors with more records than this take a warp (A/B: 1 beats 3 and 8 at N = 1 and
// removes most of the fold's per-frame floor at 8 emulated ranks)
constexpr uint32_t kWarpRecs = SVX_WARP_RECS;
#ifndef SVX_FB_SERIAL_SMEM
#define SVX_FB_SERIAL_SMEM 1
#endif
__device__ __forceinline__ uint32_t fold_records_warp(const GroupConsts& c, const FramePose& f, uint32_t g,
                                                      svx_tsdf_voxel* vp, d3 center, const ScanSlots& sc,
                                                      const unsigned long long* __restrict__ recs, uint32_t nrec,
                                                      int lane) {
    const PixCache* cache = cache_of(sc, c, g);
    svx_tsdf_voxel vox = load_voxel(vp);
    Accum acc{0.0, 0.0, 0.0, 0.0, 0.0};
    bool measured = false;
#if SVX_FB_SERIAL_SMEM
    // the lanes' terms through shared memory; lane 0 sums them in record order (the serial
    // part is then the FP64 adds alone: a term not measured adds +0.0, the sums' identity,
    // as they never hold -0.0)
    __shared__ float4 s_ta[kThreads / 32][32];
    __shared__ float2 s_tb[kThreads / 32][32];
    const int wq = threadIdx.x >> 5;
    unsigned any = 0;
    for (uint32_t j0 = 0; j0 < nrec; j0 += 32u) {  // (warp-uniform)
        Term t{0.f, 0.f, 0.f, 0.f, 0.f, 0u};
        if (j0 + uint32_t(lane) < nrec)
            t = measure_term(c, f.origin, cache, rec_pixel(recs[j0 + lane], c.pbits), center, vox);
        s_ta[wq][lane] = make_float4(t.wg, t.w, t.nx, t.ny);
        s_tb[wq][lane] = make_float2(t.nz, __uint_as_float(t.flags));
        any |= __ballot_sync(0xFFFFFFFFu, (t.flags & 1u) != 0u);
        __syncwarp();
        if (lane == 0) {
            const uint32_t n = min(32u, nrec - j0);
#pragma unroll 4
            for (uint32_t k = 0; k < n; ++k) {
                const float4 a = s_ta[wq][k];
                const float2 b = s_tb[wq][k];
                const uint32_t fl = __float_as_uint(b.y);
                const bool m1 = (fl & 1u) != 0u, m2 = (fl & 3u) == 3u;
                acc.wd += m1 ? double(a.x) : 0.0;
                acc.w += m1 ? double(a.y) : 0.0;
                acc.wx += m2 ? double(a.z) : 0.0;
                acc.wy += m2 ? double(a.w) : 0.0;
                acc.wz += m2 ? double(b.x) : 0.0;
            }
        }
        __syncwarp();
    }
    if (!any || lane != 0) return 0;
    fold(vox, acc);
    store_voxel(vp, vox);
    return 1;
#else
    for (uint32_t j0 = 0; j0 < nrec; j0 += 32u) {  // (warp-uniform)
        Term t{0.f, 0.f, 0.f, 0.f, 0.f, 0u};
        if (j0 + uint32_t(lane) < nrec)
            t = measure_term(c, f.origin, cache, rec_pixel(recs[j0 + lane], c.pbits), center, vox);
        const uint32_t n = min(32u, nrec - j0);
        for (uint32_t k = 0; k < n; ++k) {
            Term tk;
            tk.wg = __shfl_sync(0xFFFFFFFFu, t.wg, int(k));
            tk.w = __shfl_sync(0xFFFFFFFFu, t.w, int(k));
            tk.nx = __shfl_sync(0xFFFFFFFFu, t.nx, int(k));
            tk.ny = __shfl_sync(0xFFFFFFFFu, t.ny, int(k));
            tk.nz = __shfl_sync(0xFFFFFFFFu, t.nz, int(k));
            tk.flags = __shfl_sync(0xFFFFFFFFu, t.flags, int(k));
            if (tk.flags & 1u) {  // (every lane keeps the same sums; lane 0 stores)
                accumulate(acc, tk);
                measured = true;
            }
        }
    }
    if (!measured) return 0;
    fold(vox, acc);
    if (lane != 0) return 0;
    store_voxel(vp, vox);
    return 1;
#endif
}

// Hash find-or-insert of a block key; a new block takes the next pool index.
struct SlotRef {
    uint32_t slot, idx;
    bool inserted;
};

// Pool index of an existing slot. A slot inserted concurrently by another CTA gets its
// index right after the key (find_or_insert): wait for it.
__device__ inline uint32_t block_index(HashView h, uint32_t slot) {
    uint32_t idx = __ldcg(&h.vals[slot]);
    while (idx == kInvalid) {
        __nanosleep(64);
        idx = *reinterpret_cast<volatile uint32_t*>(&h.vals[slot]);
    }
    return idx;
}

// Returns slot kInvalid when the block cannot be used by this group (hash full, capacity,
// pool not mapped); the matching abort bit is raised and the group is rolled back.
__device__ inline SlotRef find_or_insert(const GroupConsts& c, HashView h, uint64_t* __restrict__ block_keys,
                                         uint32_t* __restrict__ ctr, uint64_t key) {
    SlotRef r{kInvalid, kInvalid, false};
    int ins = 0;
    const uint32_t slot = hash_insert(h, key, &ins);
    if (slot == kInvalid) {
        atomicOr(&ctr[C_ABORT], kAbortHash | kAbortCapacity);
        return r;
    }
    uint32_t idx;
    if (ins) {
        idx = atomicAdd(&ctr[C_BLOCKS], 1u);
        if (idx < c.max_blocks) block_keys[idx] = key;
        __threadfence();
        atomicExch(&h.vals[slot], idx);
    } else {
        idx = block_index(h, slot);
    }
    if (idx >= c.max_blocks) {
        atomicOr(&ctr[C_ABORT], kAbortCapacity);
        return r;
    }
    if (idx >= __ldcg(&ctr[C_MAPPED])) {  // pool / mask memory not mapped yet: map, retry
        atomicOr(&ctr[C_ABORT], kAbortPool);
        return r;
    }
    r.slot = slot;
    r.idx = idx;
    r.inserted = ins != 0;
    return r;
}

__device__ inline void zero_block(svx_tsdf_voxel* __restrict__ pool, uint32_t idx, int lane, int lanes) {
    float4* z = reinterpret_cast<float4*>(pool + uint64_t(idx) * kBlockVoxels);
    for (int i = lane; i < kBlockVoxels * 5 / 4; i += lanes) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Send metadata per destination rank: [0] entries, [1 + g] voxel bits of frame g (a bound
// on the receiver's new voxel-list entries of frame g).
constexpr int kXMeta = 1 + kMaxG;
constexpr int kMaxXWorld = 16;  // ranks supported by exchange mode

// ---- exchange mode: visits of blocks another rank owns go to that rank as 16-byte
// entries (x, y = packed block key; z bit 31 = fallback record; word entry: z = g << 4 | w,
// w = the voxel bits of mask word w in frame g; record entry: z = g << 9 | voxel,
// w = pixel). The owner applies them with k_ingest exactly as its own band would have.
__device__ inline void send_remote(const GroupConsts& c, uint4* __restrict__ xsend, uint32_t* __restrict__ xcnt,
                                   uint32_t* __restrict__ ctr, uint64_t key, uint32_t z, uint32_t w) {
    const int32_t dest = owner_of(key, c.shard_world);
    uint32_t* meta = xcnt + dest * kXMeta;
    const uint32_t pos = atomicAdd(&meta[0], 1u);
    if (!(z & 0x80000000u)) atomicAdd(&meta[1 + (z >> 4)], uint32_t(__popc(w)));  // voxel bits per frame
    if (pos < c.xcap)
        xsend[uint64_t(dest) * c.xcap + pos] = make_uint4(uint32_t(key), uint32_t(key >> 32), z, w);
    else
        atomicOr(&ctr[C_ABORT], kAbortXchg);
}
__device__ inline bool is_remote(const GroupConsts& c, uint64_t key) {
    return c.exchange && owner_of(key, c.shard_world) != c.shard_rank;
}

// Per-visit work on global state (no tile staging): the path a visit takes when its tile's
// shared tables are full. Same effect as the staged path.
__device__ void visit_global(const GroupConsts& c, uint32_t g, HashView h, uint64_t* __restrict__ block_keys,
                             uint32_t* __restrict__ stamp, uint32_t* __restrict__ touched,
                             uint32_t* __restrict__ fm, unsigned long long* __restrict__ rec, svx_tsdf_voxel* __restrict__ pool,
                             uint32_t* __restrict__ vlist, uint32_t* __restrict__ fctr,
                             uint4* __restrict__ xsend, uint32_t* __restrict__ xcnt,
                             uint32_t* __restrict__ ctr, uint64_t key, int lin, bool fb, uint32_t p) {
    if (is_remote(c, key)) {
        send_remote(c, xsend, xcnt, ctr, key, (g << 4) | uint32_t(lin >> 5), 1u << (lin & 31));
        if (fb) send_remote(c, xsend, xcnt, ctr, key, 0x80000000u | (g << 9) | uint32_t(lin), p);
        return;
    }
    const SlotRef r = find_or_insert(c, h, block_keys, ctr, key);
    if (r.slot == kInvalid) return;
    if (atomicExch(&stamp[r.slot], c.serial) != c.serial) touched[atomicAdd(&ctr[C_TOUCHED], 1u)] = r.slot;
    if (r.inserted) zero_block(pool, r.idx, 0, 1);
    uint32_t* bm = fm + uint64_t(r.idx) * kMaskWords;
    atomicOr(&bm[kHdrRow * 16], 1u << g);
    const uint32_t bit = 1u << (lin & 31);
    if (!(atomicOr(&bm[g * 16 + (lin >> 5)], bit) & bit)) {  // the frame's first visit of the voxel
        const uint32_t pos = atomicAdd(&fctr[g * kFC + FC_VOX], 1u);
        if (pos < c.vox_cap) vlist[uint64_t(g) * c.vox_cap + pos] = (r.idx << 9) | uint32_t(lin);
        else atomicOr(&ctr[C_ABORT], kAbortVox);
    }
    if (!fb) return;
    const uint32_t pos = atomicAdd(&ctr[C_RECORDS], 1u);
    if (pos < c.rec_cap) rec[pos] = make_record(r.idx, lin, g, p, c.pbits);
    else atomicOr(&ctr[C_ABORT], kAbortRecords);
}

// CTA = one 32 x 8 pixel tile of frame g. The tile's rays run their DDA into shared memory:
// a local table of the distinct blocks they visit, per-block voxel masks (smem atomics) and
// the staged fallback visits. Global work is then one hash find-or-insert per distinct block
// (in parallel across threads) and two atomics per non-empty mask word, instead of global
// round trips per visit.
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
k_band(const __grid_constant__ GroupParams gp, const ScanSlots sc, HashView h,
       uint64_t* __restrict__ block_keys, uint32_t* __restrict__ stamp, uint32_t* __restrict__ touched,
       uint32_t* __restrict__ fm, unsigned long long* __restrict__ rec,
       svx_tsdf_voxel* __restrict__ pool, uint32_t* __restrict__ vlist,
       uint32_t* __restrict__ fctr, uint4* __restrict__ xsend, uint32_t* __restrict__ xcnt,
       uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (cta_aborted(ctr)) return;  // the group is rolled back and retried: stop early
    const GroupConsts& c = gp.c;
    __shared__ FramePose s_f;
    __shared__ unsigned long long lkey[kLocalKeys];
    __shared__ uint32_t lslot[kLocalKeys];
    __shared__ uint32_t lidx[kLocalKeys];
    __shared__ uint32_t lmask[kLocalKeys][16];
    __shared__ uint32_t lfb[kTileFb];
    __shared__ uint32_t lnew[kLocalKeys];  // pool indices of blocks this tile created
    __shared__ uint8_t s_occ[kLocalKeys];
    __shared__ uint32_t nfb, nnew, nocc;
    const int tid = threadIdx.x;
    const uint32_t g = blockIdx.x / c.tiles;
    const uint32_t tile = blockIdx.x - g * c.tiles;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&gp.f[g]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&s_f);
        for (int i = tid; i < int(sizeof(FramePose) / 4); i += kTileU * kTileV) dst[i] = src[i];
    }
    lkey[tid] = kEmptyKey;
#pragma unroll
    for (int w = 0; w < 16; ++w) lmask[tid][w] = 0u;
    if (tid == 0) nfb = nnew = nocc = 0;
    __syncthreads();

    const uint64_t pg = uint64_t(g) * c.P;
    const float* depth = sc.depth + pg;
    const uint8_t* hd = sc.rowdist + pg;
    const uint32_t* validbits = sc.validbits + uint64_t(g) * c.VW;
    PixCache* cache = reinterpret_cast<PixCache*>(sc.cache) + pg;
    const int tiles_u = (c.m.W + kTileU - 1) / kTileU;
    const int tu = int(tile) % tiles_u, tv = int(tile) / tiles_u;
    const int u = tu * kTileU + (tid % kTileU);
    const int v = tv * kTileV + (tid / kTileU);
    const uint32_t tile_p0 = uint32_t(tv * kTileV) * uint32_t(c.m.W) + uint32_t(tu * kTileU);
    const bool has_pix = u < c.m.W && v < c.m.H;
    const uint32_t p = has_pix ? uint32_t(v) * uint32_t(c.m.W) + uint32_t(u) : 0u;
    const float r = has_pix ? depth[p] : 0.f;
    const bool in_range = has_pix && !(r == 0.f || double(r) > c.max_range);
    const bool have_normal = has_pix && c.has_normals && sc.valid[pg + p];
    // pixel cache (measure lambda inputs, tsdf_integrator.cpp:173-186)
    d3 q = mk(0, 0, 0), ray = mk(0, 0, 0);
    if (has_pix) {
        PixCache pc{};
        if (in_range) {
            q = xform(s_f.pose, scale3(double(r), dir_at(sc.dirs, p)));
            const d3 dq = sub3(q, s_f.origin);
            const double range = sqrt(dot3(dq, dq));
            ray = div3(dq, range);
            pc.ray[0] = ray.x;
            pc.ray[1] = ray.y;
            pc.ray[2] = ray.z;
            pc.range = range;
            if (have_normal) {
                const float* nn = sc.normals + 3 * (pg + p);
                const d3 n = matvec(s_f.pose.R, mk(nn[0], nn[1], nn[2]));
                pc.n[0] = float(n.x);
                pc.n[1] = float(n.y);
                pc.n[2] = float(n.z);
            }
            pc.flags = ((have_normal || !c.drop_unreliable) ? 1u : 0u) | (have_normal ? 2u : 0u);
        }
        cache[p] = pc;
    }
    // band ray (tsdf_integrator.cpp:123-131); in exchange mode only the rays of this rank's
    // tiles (round robin over the group's tiles); every rank still writes the whole pixel
    // cache, which the folds of its own blocks read
    const bool my_tile = !c.exchange || int(blockIdx.x % uint32_t(c.shard_world)) == c.shard_rank;
    if (!my_tile) return;  // (CTA-uniform) another rank casts this tile's rays
    const bool cast = in_range && !(c.drop_unreliable && c.has_normals && !sc.valid[pg + p]);
    if (cast) {
        warp_agg_inc(&fctr[g * kFC + FC_RAYS]);
        const d3 tr = scale3(c.tau, ray);  // (q - o).normalized() == (q - o) / range
        const d3 a = sub3(q, tr), b = add3(q, tr);
        uint64_t cur_key = kEmptyKey;
        int cur_li = -1;
        bool cur_own = true;
        int pend_word = -1;
        uint32_t pend_bits = 0;
        int32_t x0 = 0, y0 = 0, z0 = 0;
        float p0x = 0.f, p0y = 0.f, p0z = 0.f;
        bool first = true;
        const bool all_own = band_all_own(c, hd, p, r);
        int32_t cbx = INT32_MIN, cby = 0, cbz = 0;  // block of the previous visit
        traverse_segment<true>(a, b, c.nu, c.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
            const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
            if (bx != cbx || by != cby || bz != cbz) {  // block change: key, range, local slot
                cbx = bx;
                cby = by;
                cbz = bz;
                cur_li = -1;
                if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) {
                    atomicOr(&ctr[C_ABORT], kAbortKey);  // (the group is rolled back)
                    cur_own = false;
                    return;
                }
                const uint64_t key = pack_key(bx, by, bz);
                cur_key = key;
                // key sharding without exchange: this rank's blocks only (its band is redundant);
                // with exchange: every block is staged, the epilogue routes the remote ones
                cur_own = c.exchange || !(c.shard_world > 1 && owner_of(key, c.shard_world) != c.shard_rank);
                if (cur_own) {  // local table insert (open addressing in smem)
                    uint32_t s = hash_slot(key, 8);
                    for (int probe = 0; probe < kLocalKeys; ++probe) {
                        // plain load first: most blocks are already in the table (neighbour rays)
                        unsigned long long old = lkey[s];
                        if (old == kEmptyKey) old = atomicCAS(&lkey[s], kEmptyKey, key);
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
                    const d3 pc0 = xform(s_f.w2s, voxel_center(x, y, z, c.nu));
                    p0x = float(pc0.x);
                    p0y = float(pc0.y);
                    p0z = float(pc0.z);
                    x0 = x;
                    y0 = y;
                    z0 = z;
                    first = false;
                }
                const float kx = float(x - x0), ky = float(y - y0), kz = float(z - z0);
                const float px = p0x + kx * s_f.col[0][0] + ky * s_f.col[1][0] + kz * s_f.col[2][0];
                const float py = p0y + kx * s_f.col[0][1] + ky * s_f.col[1][1] + kz * s_f.col[2][1];
                const float pz = p0z + kx * s_f.col[0][2] + ky * s_f.col[1][2] + kz * s_f.col[2][2];
                uint32_t own = pixel_fast(px, py, pz, c.m, c.m.r2_lo, c.m.r2_hi);
                if (own == kNeedFp64) own = pixel_fp64(xform(s_f.w2s, voxel_center(x, y, z, c.nu)), c.m);
                fb = own == kInvalid || !pixel_has_return(validbits, own);
            }
            if (cur_li < 0) {  // local table full: straight to global state
                visit_global(c, g, h, block_keys, stamp, touched, fm, rec, pool, vlist, fctr, xsend, xcnt, ctr, cur_key,
                             lin, fb, p);
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
                    visit_global(c, g, h, block_keys, stamp, touched, fm, rec, pool, vlist, fctr, xsend,
                                 xcnt, ctr, cur_key, lin, true, p);
            }
        });
        if (pend_word >= 0) atomicOr(&lmask[0][0] + pend_word, pend_bits);
    }
    __syncthreads();
    // one global hash operation per distinct block of the tile; first touches of the
    // group are appended to the touched list with one atomic per tile
    constexpr int kW = kTileU * kTileV / 32;
    __shared__ uint32_t s_w[2 * kW];
    uint32_t slot = kInvalid, idx = kInvalid;
    bool first_touch = false;
    if (lkey[tid] != kEmptyKey && !is_remote(c, lkey[tid])) {
        const SlotRef sr = find_or_insert(c, h, block_keys, ctr, lkey[tid]);
        if (sr.slot != kInvalid) {
            slot = sr.slot;
            idx = sr.idx;
            first_touch = atomicExch(&stamp[slot], c.serial) != c.serial;
            atomicOr(&fm[uint64_t(idx) * kMaskWords + kHdrRow * 16], 1u << g);
            if (sr.inserted) lnew[atomicAdd(&nnew, 1u)] = idx;
        }
    }
    lslot[tid] = slot;
    lidx[tid] = idx;
    // occupied local slots (the epilogue's loops run over their 16 mask words only)
    if (lkey[tid] != kEmptyKey) s_occ[atomicAdd(&nocc, 1u)] = uint8_t(tid);
    const uint32_t tpos = cta_append<kW>(first_touch, &ctr[C_TOUCHED], s_w);  // (barriers)
    if (first_touch) touched[tpos] = slot;
    // zero-fill the blocks this tile created (read from the fold on)
    for (uint32_t j = 0; j < nnew; ++j) zero_block(pool, lnew[j], tid, kTileU * kTileV);
    const uint32_t nf = min(nfb, uint32_t(kTileFb));
    const uint32_t nwords = nocc * 16u;
    // exchange mode: the tile's entries for other ranks are counted per destination in
    // shared memory and reserved with one global atomic per (tile, destination)
    __shared__ uint32_t s_xn[kMaxXWorld], s_xb[kMaxXWorld], s_xbase[kMaxXWorld];
    __shared__ uint8_t lown[kLocalKeys];
    if (c.exchange) {
        if (tid < kMaxXWorld) s_xn[tid] = s_xb[tid] = 0u;
        lown[tid] = (lkey[tid] != kEmptyKey) ? uint8_t(owner_of(lkey[tid], c.shard_world)) : uint8_t(255);
        __syncthreads();
        for (uint32_t i = tid; i < nf; i += kTileU * kTileV) {
            const uint32_t li = lfb[i] >> 24;
            if (lown[li] != c.shard_rank) atomicAdd(&s_xn[lown[li]], 1u);
        }
        for (uint32_t i = tid; i < nwords; i += kTileU * kTileV) {
            const int li = s_occ[i >> 4];
            const uint32_t bits = lmask[li][i & 15];
            if (bits && lown[li] != c.shard_rank) {
                atomicAdd(&s_xn[lown[li]], 1u);
                atomicAdd(&s_xb[lown[li]], uint32_t(__popc(bits)));
            }
        }
        __syncthreads();
        if (tid < c.shard_world) {
            uint32_t* meta = xcnt + tid * kXMeta;
            s_xbase[tid] = s_xn[tid] ? atomicAdd(&meta[0], s_xn[tid]) : 0u;
            if (s_xb[tid]) atomicAdd(&meta[1 + g], s_xb[tid]);
            if (s_xn[tid] && s_xbase[tid] + s_xn[tid] > c.xcap) atomicOr(&ctr[C_ABORT], kAbortXchg);
            s_xn[tid] = 0u;  // now the write cursor
        }
        __syncthreads();
    }
    auto xput = [&](uint32_t li, uint32_t z, uint32_t w) {
        const uint32_t d = lown[li];
        const uint32_t pos = s_xbase[d] + atomicAdd(&s_xn[d], 1u);
        if (pos < c.xcap)
            xsend[uint64_t(d) * c.xcap + pos] = make_uint4(uint32_t(lkey[li]), uint32_t(lkey[li] >> 32), z, w);
    };
    // staged fallback visits -> records (block, voxel, frame, pixel)
    uint32_t nrec = 0;
    for (uint32_t i = tid; i < nf; i += kTileU * kTileV) nrec += lidx[lfb[i] >> 24] != kInvalid ? 1u : 0u;
    uint32_t rpos = cta_reserve<kW>(nrec, &ctr[C_RECORDS], s_w);
    if (nrec && rpos + nrec > c.rec_cap) atomicOr(&ctr[C_ABORT], kAbortRecords);
    for (uint32_t i = tid; i < nf; i += kTileU * kTileV) {
        const uint32_t e = lfb[i], li = e >> 24;
        const uint32_t bi = lidx[li];
        const uint32_t t = e & 255u;
        const uint32_t px = tile_p0 + (t / kTileU) * uint32_t(c.m.W) + (t % kTileU);
        if (bi == kInvalid) {
            if (c.exchange && lown[li] != c.shard_rank) xput(li, 0x80000000u | (g << 9) | ((e >> 15) & 511u), px);
            continue;
        }
        if (rpos < c.rec_cap) rec[rpos] = make_record(bi, int((e >> 15) & 511u), g, px, c.pbits);
        ++rpos;
    }
    // voxel masks -> the frame's row of each block; the bits a tile sets first (the atomic
    // returns them clear) are those voxels' single entries in the frame's voxel list
    uint32_t nv = 0;
    for (uint32_t i = tid; i < nwords; i += kTileU * kTileV) {
        const int li = s_occ[i >> 4], w = i & 15;
        uint32_t bits = lmask[li][w];
        if (bits && lidx[li] != kInvalid) {
            bits &= ~atomicOr(&fm[uint64_t(lidx[li]) * kMaskWords + g * 16 + w], bits);
        } else {
            if (bits && c.exchange && lown[li] != c.shard_rank) xput(uint32_t(li), (g << 4) | uint32_t(w), bits);
            bits = 0u;
        }
        lmask[li][w] = bits;
        nv += __popc(bits);
    }
    uint32_t pos = cta_reserve<kW>(nv, &fctr[g * kFC + FC_VOX], s_w);
    if (nv && pos + nv > c.vox_cap) atomicOr(&ctr[C_ABORT], kAbortVox);
    // the list entries, written warp-cooperatively: per 32 words (one per lane), entry j of
    // the warp goes to the lane whose bit range holds j (binary search over the inclusive
    // popcount scan) and takes that lane's (j - excl)-th set bit; each lane's entries land
    // at its own running position, as a per-lane loop over its bits would place them
    uint32_t* vl = vlist + uint64_t(g) * c.vox_cap;
    const int lane = tid & 31;
    for (uint32_t base = uint32_t(tid & ~31); base < nwords; base += kTileU * kTileV) {  // warp-uniform
        const uint32_t i = base + uint32_t(lane);
        uint32_t bits = 0u, hi = 0u;
        if (i < nwords) {
            const int li = s_occ[i >> 4], w = int(i & 15u);
            bits = lmask[li][w];
            hi = (lidx[li] << 9) | (uint32_t(w) * 32u);
        }
        const uint32_t n = uint32_t(__popc(bits));
        uint32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t start = pos - (incl - n);  // this lane's entry k goes to start + excl + k
        pos += n;
        for (uint32_t jb = 0; jb < total; jb += 32u) {
            const uint32_t j = jb + uint32_t(lane);
            int l = 0;
#pragma unroll
            for (int s = 16; s; s >>= 1)
                if (__shfl_sync(0xFFFFFFFFu, incl, l + s - 1) <= j) l += s;
            const uint32_t bl = __shfl_sync(0xFFFFFFFFu, bits, l);
            const uint32_t hl = __shfl_sync(0xFFFFFFFFu, hi, l);
            const uint32_t sl = __shfl_sync(0xFFFFFFFFu, start, l);
            const uint32_t el = __shfl_sync(0xFFFFFFFFu, incl, l) - uint32_t(__popc(bl));
            if (j < total) {
                const uint32_t at = sl + j;
                if (at < c.vox_cap) vl[at] = hl | select_bit(bl, j - el);
            }
        }
    }
}

// End of the run of keys equal to `run` (on their bits above pb) that starts at pos in the
// sorted a[0..n): galloping then binary search, O(log run) loads (a voxel thousands of rays
// cross in one frame is one long run).
__device__ inline uint32_t run_end(const unsigned long long* __restrict__ a, uint32_t pos, uint32_t n,
                                   unsigned long long run, uint32_t pb) {
    uint32_t lo = pos + 1, step = 1;  // a[lo - 1] is in the run
    uint32_t hi = lo;
    while (hi < n && (a[hi] >> pb) == run) {
        lo = hi + 1;
        hi = (n - hi > step) ? hi + step : n;
        step *= 2;
    }
    // a[lo - 1] in the run; a[hi] (hi < n) past it, or hi = n
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if ((a[mid] >> pb) == run) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// The group's fallback records, sorted by (block, voxel, frame, pixel) (a device radix sort
// over the record bits precedes this kernel: O(records) whatever the number of rays per
// voxel), cut into (voxel, frame) runs: one descriptor per run (pool index, voxel | frame
// << 16, first record, count) - per frame the reference's ascending (v, u) visit order
// after its chunk-order merge + stable_sort (tsdf_integrator.cpp:141-146,215-216). The
// unsorted input is reset to the sort's padding key for the next group.
__global__ void __launch_bounds__(kThreads)
k_fb_runs(const unsigned long long* __restrict__ sorted, unsigned long long* __restrict__ rec, uint32_t rec_cap,
          uint32_t pb, uint4* __restrict__ fbdesc, uint32_t* __restrict__ fctr, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t n = min(ctr[C_RECORDS], rec_cap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        rec[i] = ~0ull;
        const unsigned long long k = sorted[i];
        const unsigned long long run = k >> pb;  // (block, voxel, frame)
        if (i > 0 && (sorted[i - 1] >> pb) == run) continue;
        const uint32_t j = run_end(sorted, i, n, run, pb);
        const uint32_t g = uint32_t(run) & 15u, lin = uint32_t(run >> 4) & 511u, idx = uint32_t(run >> 13);
        // frame g's list (its fold reads only its own descriptors)
        fbdesc[uint64_t(g) * rec_cap + atomicAdd(&fctr[g * kFC + FC_FBV], 1u)] = make_uint4(idx, lin | (g << 16), i, j - i);
    }
}

// ---- ordering of the fallback records: counted per block, bucketed per block, and each
// bucket sorted by one CTA (k_fb_sort): four PDL-chained kernels, one pass over the records
// each. (The global radix sort over the record buffer, CUB + k_fb_runs, is kept as an
// alternative: SVX_FB_GLOBAL=1.)
constexpr int kFbSortItems = 8;
#ifndef SVX_FB_GLOBAL_BUCKET
#define SVX_FB_GLOBAL_BUCKET 6144
#endif
constexpr uint32_t kFbGlobalBucket = SVX_FB_GLOBAL_BUCKET;  // a larger bucket: the next batch sorts globally
constexpr uint32_t kFbSortMax = kThreads * kFbSortItems;  // records per block one CTA sorts

__global__ void __launch_bounds__(kThreads)
k_fb_count(const unsigned long long* __restrict__ rec, uint32_t rec_cap, uint32_t pb, uint32_t* __restrict__ fbcnt,
           uint32_t* __restrict__ fbblocks, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t n = min(ctr[C_RECORDS], rec_cap);
    const int lane = threadIdx.x & 31;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t idx = uint32_t(rec[i] >> (pb + 13));
        // one atomic per distinct block among the warp's lanes (a tile's records of a block
        // are adjacent; a block many rays cross would serialise per-record atomics)
        const unsigned grp = __match_any_sync(__activemask(), idx);
        if (lane == __ffs(grp) - 1 && atomicAdd(&fbcnt[idx], uint32_t(__popc(grp))) == 0u)
            fbblocks[atomicAdd(&ctr[C_FB_BLOCKS], 1u)] = idx;
    }
}

__global__ void __launch_bounds__(kThreads)
k_fb_alloc(const uint32_t* __restrict__ fbcnt, const uint32_t* __restrict__ fbblocks, uint32_t* __restrict__ fbstart,
           uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t nb = ctr[C_FB_BLOCKS];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
        const uint32_t idx = fbblocks[t], cnt = fbcnt[idx];
        fbstart[idx] = atomicAdd(&ctr[C_BUCKET_TOP], cnt);
        if (cnt > kFbSortMax) atomicMax(&ctr[C_FB_MAXB], cnt);
    }
}

__global__ void __launch_bounds__(kThreads)
k_fb_bucket(unsigned long long* __restrict__ rec, uint32_t rec_cap, uint32_t pb, const uint32_t* __restrict__ fbstart,
            uint32_t* __restrict__ fbfill, unsigned long long* __restrict__ bucket, uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t n = min(ctr[C_RECORDS], rec_cap);
    const int lane = threadIdx.x & 31;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long r = rec[i];
        rec[i] = ~0ull;  // the record buffer holds the padding key outside a group's entries
        const uint32_t idx = uint32_t(r >> (pb + 13));
        const unsigned grp = __match_any_sync(__activemask(), idx);
        const int leader = __ffs(grp) - 1;
        uint32_t base = 0;
        if (lane == leader) base = fbstart[idx] + atomicAdd(&fbfill[idx], uint32_t(__popc(grp)));
        base = __shfl_sync(grp, base, leader);
        bucket[base + uint32_t(__popc(grp & ((1u << lane) - 1u)))] = r;
    }
}

// Sorts n keys src[0..n) into dst[0..n) with the whole CTA (n arbitrary): sorted tiles of
// kFbSortMax keys (cub::BlockRadixSort in shared memory), then pairwise merges of sorted runs
// through the two buffers (each key's rank in the other run by binary search: the keys are
// unique). Every thread of the CTA calls it with the same arguments.
template <typename SortT>
__device__ void cta_sort_range(typename SortT::TempStorage& tmp, unsigned long long* __restrict__ src,
                               unsigned long long* __restrict__ dst, uint32_t n, int end_bit) {
    for (uint32_t t0 = 0; t0 < n; t0 += kFbSortMax) {
        unsigned long long k[kFbSortItems];
#pragma unroll
        for (int j = 0; j < kFbSortItems; ++j) {
            const uint32_t pos = t0 + threadIdx.x * kFbSortItems + j;  // blocked arrangement
            k[j] = pos < n ? src[pos] : ~0ull;  // padding sorts last (the sort is stable)
        }
        SortT(tmp).Sort(k, 0, end_bit);
#pragma unroll
        for (int j = 0; j < kFbSortItems; ++j) {
            const uint32_t pos = t0 + threadIdx.x * kFbSortItems + j;
            if (pos < n) dst[pos] = k[j];
        }
        __syncthreads();  // tmp reused; the tile visible to the CTA
    }
    unsigned long long* a = dst;
    unsigned long long* b = src;
    for (uint32_t w = kFbSortMax; w < n; w *= 2) {  // runs of w in a -> runs of 2w in b
        for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
            const uint32_t p0 = (i / (2 * w)) * (2 * w);
            const uint32_t a1 = min(p0 + w, n), b1 = min(p0 + 2 * w, n);
            const unsigned long long key = a[i];
            uint32_t lo = i < a1 ? a1 : p0, hi = i < a1 ? b1 : a1;
            const uint32_t base = lo;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (a[mid] < key) lo = mid + 1;
                else hi = mid;
            }
            b[p0 + (i < a1 ? i - p0 : i - a1) + (lo - base)] = key;
        }
        __syncthreads();
        unsigned long long* x = a;
        a = b;
        b = x;
    }
    if (a != dst) {
        for (uint32_t i = threadIdx.x; i < n; i += kThreads) dst[i] = a[i];
        __syncthreads();
    }
}

// CTA per block with records: its bucket sorted by (voxel, frame, pixel), then one
// descriptor per (voxel, frame) run - per frame the reference's ascending (v, u) visit order
// (.cpp:141-146,215-216) - into the frame's list. A bucket of up to 256 records is ordered by
// a rank count per record, one of up to kFbSortMax in shared memory; a larger one (a block many rays cross) is first counting-sorted
// by voxel, then each voxel's records are ordered: up to 64 by a rank count per record, more
// by cta_sort_range (the wall case: thousands of rays through one voxel).
__global__ void __launch_bounds__(kThreads)
k_fb_sort(const uint32_t* __restrict__ fbblocks, uint32_t* __restrict__ fbcnt, const uint32_t* __restrict__ fbstart,
          uint32_t* __restrict__ fbfill, unsigned long long* __restrict__ bucket, unsigned long long* __restrict__ scratch,
          uint32_t pb, uint32_t rec_cap, uint4* __restrict__ fbdesc, uint32_t* __restrict__ fctr,
          uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (cta_aborted(ctr)) return;
    using Sort = cub::BlockRadixSort<unsigned long long, kThreads, kFbSortItems>;
    using Scan = cub::BlockScan<uint32_t, kThreads>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ uint32_t seg_start[kBlockVoxels], seg_cnt[kBlockVoxels], cursor[kBlockVoxels];
    const uint32_t nb = ctr[C_FB_BLOCKS];
    const int end_bit = int(pb) + 13;
    for (uint32_t t = blockIdx.x; t < nb; t += gridDim.x) {
        const uint32_t idx = fbblocks[t];
        const uint32_t cnt = fbcnt[idx], start = fbstart[idx];
        unsigned long long* bk = bucket + start;
        unsigned long long* sc = scratch + start;
        if (cnt <= kThreads) {  // most buckets: a rank count per record (keys are unique)
            unsigned long long k = 0;
            uint32_t r = 0;
            if (threadIdx.x < cnt) {
                k = bk[threadIdx.x];
                for (uint32_t j = 0; j < cnt; ++j) r += bk[j] < k ? 1u : 0u;
            }
            __syncthreads();
            if (threadIdx.x < cnt) bk[r] = k;
            __syncthreads();
        } else if (cnt <= kFbSortMax) {
            cta_sort_range<Sort>(tmp.sort, bk, bk, cnt, end_bit);
        } else {
            for (int v = threadIdx.x; v < kBlockVoxels; v += kThreads) seg_cnt[v] = 0u;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) atomicAdd(&seg_cnt[(bk[i] >> (pb + 4)) & 511u], 1u);
            __syncthreads();
            {
                constexpr int kPer = kBlockVoxels / kThreads;
                uint32_t cc[kPer];
#pragma unroll
                for (int j = 0; j < kPer; ++j) cc[j] = seg_cnt[threadIdx.x * kPer + j];
                Scan(tmp.scan).ExclusiveSum(cc, cc);
#pragma unroll
                for (int j = 0; j < kPer; ++j) seg_start[threadIdx.x * kPer + j] = cursor[threadIdx.x * kPer + j] = cc[j];
            }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
                const unsigned long long k = bk[i];
                sc[atomicAdd(&cursor[(k >> (pb + 4)) & 511u], 1u)] = k;
            }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {  // small voxel segments
                const unsigned long long k = sc[i];
                const uint32_t v = uint32_t(k >> (pb + 4)) & 511u;
                const uint32_t b0 = seg_start[v], e0 = b0 + seg_cnt[v];
                if (e0 - b0 > 64u) continue;
                uint32_t r = 0;
                for (uint32_t j = b0; j < e0; ++j) r += sc[j] < k ? 1u : 0u;
                bk[b0 + r] = k;
            }
            __syncthreads();
            for (int v = 0; v < kBlockVoxels; ++v)  // large voxel segments (CTA-uniform loop)
                if (seg_cnt[v] > 64u) cta_sort_range<Sort>(tmp.sort, sc + seg_start[v], bk + seg_start[v], seg_cnt[v], end_bit);
            __syncthreads();
        }
        for (uint32_t pos = threadIdx.x; pos < cnt; pos += kThreads) {
            const unsigned long long run = bk[pos] >> pb;  // (block, voxel, frame)
            if (pos > 0 && (bk[pos - 1] >> pb) == run) continue;
            const uint32_t e = run_end(bk, pos, cnt, run, pb);
            const uint32_t g = uint32_t(run) & 15u, lin = uint32_t(run >> 4) & 511u;
            fbdesc[uint64_t(g) * rec_cap + atomicAdd(&fctr[g * kFC + FC_FBV], 1u)] =
                make_uint4(idx, lin | (g << 16), start + pos, e - pos);
        }
        if (threadIdx.x == 0) fbcnt[idx] = fbfill[idx] = 0u;  // clean for the next group
        __syncthreads();
    }
}

// Frame g of the group: one thread per listed visited voxel of the frame (grid-stride, one
// wave of CTAs), then the group's fallback descriptors of frame g; each applies frame g to
// its voxel, whose state then holds frames 0..g, as after the reference's g + 1
// consecutive integrate_frame calls. The last frame's launch ends the group: dirty flags,
// per-frame touched / new block counts and the mask rows over the touched list; its last
// CTA writes the frames' reports.
#ifndef SVX_FOLD_MINB
#define SVX_FOLD_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, SVX_FOLD_MINB)
k_fold(const __grid_constant__ GroupConsts c, const __grid_constant__ FramePose f, const uint32_t g, const ScanSlots sc,
       const uint32_t* __restrict__ vals, const uint64_t* __restrict__ block_keys, svx_tsdf_voxel* __restrict__ pool,
       uint32_t* __restrict__ fm, const uint32_t* __restrict__ vlist, const uint4* __restrict__ fbdesc,
       const unsigned long long* __restrict__ bucket, const uint32_t* __restrict__ touched,
       uint8_t* __restrict__ dirty, uint32_t* __restrict__ fctr, FrameOut* __restrict__ outs,
       uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (cta_aborted(ctr)) return;
    __shared__ uint32_t s_touch[kMaxG], s_new[kMaxG];
    __shared__ bool last;
    const int lane = threadIdx.x & 31;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    uint32_t* fc = fctr + g * kFC;
    const uint32_t nv = min(fc[FC_VOX], c.vox_cap);
    const uint32_t* vl = vlist + uint64_t(g) * c.vox_cap;
    uint32_t n_upd = 0;
    // fallback descriptors first (a record chain starts early instead of in the tail): those
    // with many records one per warp, the rest one per thread
    const uint32_t nfv = min(fc[FC_FBV], c.rec_cap);
    const uint4* fd = fbdesc + uint64_t(g) * c.rec_cap;
    for (uint32_t i = gtid >> 5; i < nfv; i += stride >> 5) {  // (warp-uniform)
        const uint4 d = fd[i];
        if (d.w <= kWarpRecs) continue;
        const int lin = int(d.y & 511u);
        n_upd += fold_records_warp(c, f, g, pool + uint64_t(d.x) * kBlockVoxels + lin,
                                   center_of(block_keys[d.x], lin, c.nu), sc, bucket + d.z, d.w, lane);
    }
    for (uint32_t i = gtid; i < nfv; i += stride) {
        const uint4 d = fd[i];
        if (d.w > kWarpRecs) continue;
        const int lin = int(d.y & 511u);
        n_upd += fold_one<true>(c, f, g, pool + uint64_t(d.x) * kBlockVoxels + lin,
                                center_of(block_keys[d.x], lin, c.nu), sc, bucket + d.z, d.w);
    }
    // the visited voxels, 32 per warp: each warp's first chunk is its own (no atomic), the
    // rest come from a queue (threads that took a long fallback chain take fewer of them;
    // the queue atomics are spread over the kernel instead of all arriving at its start)
    const uint32_t nwarps = gridDim.x * (blockDim.x / 32u);
    uint32_t base = (blockIdx.x * (blockDim.x / 32u) + (threadIdx.x >> 5)) * 32u;
    while (base < nv) {
        const uint32_t i = base + uint32_t(lane);
        if (i < nv) {
            const uint32_t e = vl[i];
            const uint32_t idx = e >> 9;
            const int lin = int(e & 511u);
            const uint32_t u = fold_one<false>(c, f, g, pool + uint64_t(idx) * kBlockVoxels + lin,
                                               center_of(block_keys[idx], lin, c.nu), sc, nullptr, 0);
            n_upd += u == 1u ? 1u : 0u;  // kFallback: a fallback descriptor applies it
        }
        if (lane == 0) base = nwarps * 32u + atomicAdd(&fc[FC_VQ], 32u);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
    }
    for (int o = 16; o; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
    if (lane == 0 && n_upd) atomicAdd(&fc[FC_UPD], n_upd);
    if (g + 1 < c.G) return;  // (no barrier: warps leave as soon as their voxels are done)
    if (threadIdx.x < kMaxG) s_touch[threadIdx.x] = s_new[threadIdx.x] = 0u;
    __syncthreads();
    // group end: dirty blocks (tsdf_integrator.cpp:160-168 pushes every visited block),
    // per-frame touched blocks and new blocks (a block new to the map is new in the first
    // frame of the group that visits it)
    const uint32_t nt = ctr[C_TOUCHED];
    const uint32_t before = ctr[C_BLOCKS_BEFORE];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const uint32_t idx = vals[touched[t]];
        dirty[idx] = 1;
        uint32_t* bm = fm + uint64_t(idx) * kMaskWords;
        const uint32_t ft = bm[kHdrRow * 16];
        bm[kHdrRow * 16] = 0u;
        for (uint32_t u = ft; u; u &= u - 1) {  // the rows of the frames that touched the block
            const int gg = __ffs(u) - 1;
            uint4* row = reinterpret_cast<uint4*>(bm + gg * 16);
            row[0] = row[1] = row[2] = row[3] = make_uint4(0u, 0u, 0u, 0u);
            atomicAdd(&s_touch[gg], 1u);
        }
        if (idx >= before && ft) atomicAdd(&s_new[__ffs(ft) - 1], 1u);
    }
    __syncthreads();
    if (threadIdx.x < c.G) {
        const uint32_t gg = threadIdx.x;
        if (s_touch[gg]) atomicAdd(&fctr[gg * kFC + FC_TOUCH], s_touch[gg]);
        if (s_new[gg]) atomicAdd(&fctr[gg * kFC + FC_NEW], s_new[gg]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&ctr[C_DONE], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < c.G) {
        uint32_t* f = fctr + threadIdx.x * kFC;
        FrameOut o;
        o.updated = __ldcg(&f[FC_UPD]);
        o.new_blocks = __ldcg(&f[FC_NEW]);
        o.touched = __ldcg(&f[FC_TOUCH]);
        o.records = ctr[C_RECORDS];
        o.rays = __ldcg(&f[FC_RAYS]);
        o.dropped = __ldcg(&f[FC_DROPPED]);
        o.fb_voxels = __ldcg(&f[FC_FBV]);
        o.ok = 1;
        outs[threadIdx.x] = o;
        for (int k = 0; k < kFC; ++k) f[k] = 0u;
    }
    if (threadIdx.x == 0) {
        ctr[C_DONE] = 0;
        ctr[C_TOUCHED] = ctr[C_RECORDS] = ctr[C_FB_VOXELS] = ctr[C_FB_BLOCKS] = ctr[C_BUCKET_TOP] = 0;
        ctr[C_BLOCKS_BEFORE] = ctr[C_BLOCKS];
    }
}

// Exchange mode, owner side, phase 1: the visit entries other ranks sent (send_remote),
// applied as this rank's band applies its own visits: block find-or-insert (new blocks
// zero-filled), the group's touched list, the block's frame header, the frame's mask row
// (the bits set first are the voxels' single entries in the frame's voxel list: their
// positions are reserved here and written by phase 2, after the host has grown the lists
// if needed) and the fallback records.
__global__ void __launch_bounds__(kThreads)
k_ingest(const GroupConsts c, const uint4* __restrict__ recv, uint32_t n, HashView h,
         uint64_t* __restrict__ block_keys, uint32_t* __restrict__ stamp, uint32_t* __restrict__ touched,
         uint32_t* __restrict__ fm, unsigned long long* __restrict__ rec,
         svx_tsdf_voxel* __restrict__ pool, uint4* __restrict__ xaux, uint32_t* __restrict__ fctr,
         uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint4 e = recv[i];
        xaux[i] = make_uint4(0u, 0u, 0u, 0u);
        const uint64_t key = uint64_t(e.x) | (uint64_t(e.y) << 32);
        const SlotRef r = find_or_insert(c, h, block_keys, ctr, key);
        if (r.slot == kInvalid) continue;
        if (atomicExch(&stamp[r.slot], c.serial) != c.serial) touched[atomicAdd(&ctr[C_TOUCHED], 1u)] = r.slot;
        if (r.inserted) zero_block(pool, r.idx, 0, 1);
        uint32_t* bm = fm + uint64_t(r.idx) * kMaskWords;
        if (e.z & 0x80000000u) {  // fallback record
            const uint32_t g = (e.z >> 9) & 15u;
            atomicOr(&bm[kHdrRow * 16], 1u << g);
            const uint32_t pos = atomicAdd(&ctr[C_RECORDS], 1u);
            if (pos < c.rec_cap) rec[pos] = make_record(r.idx, int(e.z & 511u), g, e.w, c.pbits);
            else atomicOr(&ctr[C_ABORT], kAbortRecords);
        } else {
            const uint32_t g = (e.z >> 4) & 15u, w = e.z & 15u;
            atomicOr(&bm[kHdrRow * 16], 1u << g);
            const uint32_t nb = e.w & ~atomicOr(&bm[g * 16 + w], e.w);
            if (nb) xaux[i] = make_uint4(atomicAdd(&fctr[g * kFC + FC_VOX], uint32_t(__popc(nb))), nb, r.idx,
                                         (g << 4) | w);
        }
    }
}

// Exchange mode, owner side, phase 2: the reserved voxel-list entries.
__global__ void __launch_bounds__(kThreads)
k_ingest_list(const GroupConsts c, const uint4* __restrict__ xaux, uint32_t n, uint32_t* __restrict__ vlist,
              const uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint4 a = xaux[i];
        if (!a.y) continue;
        const uint32_t g = a.w >> 4, w = a.w & 15u;
        uint32_t* vl = vlist + uint64_t(g) * c.vox_cap;
        uint32_t pos = a.x;
        for (uint32_t bits = a.y; bits; bits &= bits - 1, ++pos)
            vl[pos] = (a.z << 9) | (w * 32u + uint32_t(__ffs(bits) - 1));
    }
}

// Exchange mode, sender side: the per-destination send lists packed back to back in
// destination order (blockIdx.y = destination).
__global__ void k_xpack(const uint4* __restrict__ xsend, uint32_t xcap, const uint32_t* __restrict__ xmeta,
                        uint4* __restrict__ out) {
    pdl_wait();  // the band's lists and counts are complete
    pdl_trigger();
    const uint32_t d = blockIdx.y;
    uint64_t off = 0;
    for (uint32_t k = 0; k < d; ++k) off += min(xmeta[k * kXMeta], xcap);
    const uint32_t n = min(xmeta[d * kXMeta], xcap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[off + i] = xsend[uint64_t(d) * xcap + i];
}

// Capacity path: every visited block key of frame slot 0 (duplicates allowed).
__global__ void __launch_bounds__(kThreads)
k_collect_keys(const __grid_constant__ GroupParams gp, const ScanSlots sc, unsigned long long* __restrict__ out,
               uint32_t cap, uint32_t* __restrict__ ctr) {
    const GroupConsts& c = gp.c;
    const FramePose& f = gp.f[0];
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(c.m.W) * uint32_t(c.m.H)) return;
    const float r = sc.depth[p];
    if (r == 0.f || double(r) > c.max_range) return;
    if (c.drop_unreliable && c.has_normals && !sc.valid[p]) return;
    const d3 q = xform(f.pose, scale3(double(r), dir_at(sc.dirs, p)));
    const d3 dq = sub3(q, f.origin);
    const d3 ray = div3(dq, sqrt(dot3(dq, dq)));
    const d3 tr = scale3(c.tau, ray);
    uint64_t cur_key = kEmptyKey;
    traverse_segment(sub3(q, tr), add3(q, tr), c.nu, c.inv_nu, [&](int32_t x, int32_t y, int32_t z) {
        const int32_t bx = block_coord(x), by = block_coord(y), bz = block_coord(z);
        if (!key_in_range(bx) || !key_in_range(by) || !key_in_range(bz)) return;
        const uint64_t key = pack_key(bx, by, bz);
        if (key == cur_key) return;
        cur_key = key;
        if (c.shard_world > 1 && owner_of(key, c.shard_world) != c.shard_rank) return;
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

GroupConsts make_consts(svx_map* m, svx_scan* s, const svx_integrator_cfg& cfg, uint32_t G, bool has_normals) {
    GroupConsts c{};
    c.m = s->dm;
    const double nu = double(m->cfg.voxel_size);
    c.tau = cfg.truncation > 0.f ? double(cfg.truncation) : double(m->cfg.truncation);
    c.inv_2tau = 1.0 / (2.0 * c.tau);
    c.max_range = cfg.max_range;
    c.alpha_eps = cfg.alpha_epsilon;
    if (!(cfg.alpha_epsilon > 0.0)) {  // alpha < eps never holds
        c.ca_hi = c.ca_lo = 2.0;
    } else if (cfg.alpha_epsilon > kPi) {  // always holds (alpha <= pi)
        c.ca_hi = c.ca_lo = -2.0;
    } else {
        c.ca_hi = std::cos(cfg.alpha_epsilon) + 1e-12;
        c.ca_lo = std::cos(cfg.alpha_epsilon) - 1e-12;
    }
    c.min_clamp = cfg.min_weight_clamp;
    c.nonproj = cfg.mode == SVX_NON_PROJECTIVE;
    c.drop_unreliable = cfg.drop_unreliable != 0;
    c.has_normals = has_normals;
    c.nu = nu;
    c.inv_nu = 1.0 / nu;
    c.delta = float(0.8660254037844386 * nu * (1.0 + 1e-6)) + 1e-6f;
    c.min_range_safe = float(s->model.min_range * (1.0 + 1e-4)) + 1e-4f;
    {
        const double t0 = s->model.theta0, t1 = s->model.theta0 + s->model.height_px * s->model.delta_theta;
        // polar range inside (0, pi): sin is smallest at an end of the range
        c.sin_min = (t0 > 0.0 && t1 < kPi) ? float(std::min(std::sin(t0), std::sin(t1)) - 1e-6) : 0.f;
    }
    c.dphi_f = float(s->model.delta_phi * (1.0 - 1e-6));
    c.dtheta_f = float(s->model.delta_theta * (1.0 - 1e-6));
    c.shard_rank = m->shard_rank;
    c.shard_world = m->shard_world;
    c.exchange = 0;
    c.xcap = m->xcap;
    c.serial = ++m->frame_serial;
    c.G = G;
    c.P = uint32_t(s->P);
    c.VW = uint32_t(s->VW);
    c.tiles = uint32_t(((s->dm.W + kTileU - 1) / kTileU) * ((s->dm.H + kTileV - 1) / kTileV));
    c.max_blocks = m->cfg.max_blocks;
    c.rec_cap = m->rec_cap;
    c.vox_cap = m->vox_cap;
    c.pbits = 1;
    while ((1ull << c.pbits) < s->P) ++c.pbits;
    return c;
}

FramePose make_pose(svx_map* m, const Pose& pose) {
    FramePose f{};
    f.pose = pose;
    f.w2s = inverse_pose(pose);
    f.origin = mk(pose.t[0], pose.t[1], pose.t[2]);
    const double nu = double(m->cfg.voxel_size);
    for (int a = 0; a < 3; ++a)      // world axis
        for (int i = 0; i < 3; ++i)  // sensor component: (R^T)_{i a} = R_{a i}
            f.col[a][i] = float(nu * pose.R[3 * a + i]);
    return f;
}

ScanSlots scan_slots(svx_scan* s) {
    return ScanSlots{s->depth.p, s->normals.p, s->valid.p, s->dirs.p, s->rowdist.p, s->validbits.p, s->pixcache.p};
}

// k_fold's grid: one wave of resident CTAs.
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

void launch_fold_kernels(svx_map* m, svx_scan* s, const GroupParams& gp, FrameOut* outs, LabelHook* labels,
                         int first);

// Enqueues the TSDF kernels of one group (the frames' images are in the scan's slots).
void launch_group_kernels(svx_map* m, svx_scan* s, const GroupParams& gp, FrameOut* outs, LabelHook* labels = nullptr,
                          int first = 0) {
    const GroupConsts& c = gp.c;
    HashView hv = hash_view(m);
    const ScanSlots sc = scan_slots(s);
    uint32_t* fm = mask_base(m);
    {
        ProfMark pm(m, SVX_K_RAYCAST);
        launch_pdl(k_band, c.G * c.tiles, kTileU * kTileV, m->stream, gp, sc, hv, m->block_keys, m->stamp,
                   m->touched, fm, m->records.p, tsdf_base(m), m->vlist.p, m->fctr, m->xsend.p,
                   m->xcnt.p, m->d_ctr);
        count_launch();
    }
    if (c.exchange) return;  // the rest runs after the exchange (run_group_xend)
    launch_fold_kernels(m, s, gp, outs, labels, first);
}

// The group's kernels after the band (and, in exchange mode, after the ingest); with
// `labels`, frame g's label images (frame first + g of the batch) follow its fold.
void launch_fold_kernels(svx_map* m, svx_scan* s, const GroupParams& gp, FrameOut* outs, LabelHook* labels,
                         int first) {
    const GroupConsts& c = gp.c;
    HashView hv = hash_view(m);
    const ScanSlots sc = scan_slots(s);
    const unsigned pg = persistent_grid(m->device);
    uint32_t* fm = mask_base(m);
    {
        ProfMark pm(m, SVX_K_FALLBACK);
      if (!m->fb_global) {  // per-block ordering (the default)
        const unsigned eg = pg / 2;
        launch_pdl(k_fb_count, eg, kThreads, m->stream, static_cast<const unsigned long long*>(m->records.p),
                   c.rec_cap, c.pbits, m->fbcnt, m->fbblocks, m->d_ctr);
        launch_pdl(k_fb_alloc, 64u, kThreads, m->stream, static_cast<const uint32_t*>(m->fbcnt),
                   static_cast<const uint32_t*>(m->fbblocks), m->fbstart, m->d_ctr);
        launch_pdl(k_fb_bucket, eg, kThreads, m->stream, m->records.p, c.rec_cap, c.pbits,
                   static_cast<const uint32_t*>(m->fbstart), m->fbfill, m->bucket.p, m->d_ctr);
        launch_pdl(k_fb_sort, pg / 4, kThreads, m->stream, static_cast<const uint32_t*>(m->fbblocks), m->fbcnt,
                   static_cast<const uint32_t*>(m->fbstart), m->fbfill, m->bucket.p, m->bucket2.p, c.pbits,
                   c.rec_cap, m->fbdesc.p, m->fctr, m->d_ctr);
        count_launch(4);
      } else {
        // the group's records sorted on their (block, voxel, frame, pixel) bits: the whole
        // buffer (the unused tail holds the padding key ~0, which sorts last)
        int end_bit = int(c.pbits) + 13, ib = 1;
        while ((1ull << ib) < m->cfg.max_blocks) ++ib;
        end_bit += ib;
        size_t bytes = 0;
        SVX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, m->records.p, m->bucket.p, int(c.rec_cap), 0, end_bit,
                                                m->stream));
        if (bytes > m->fb_tmp.n) m->fb_tmp.alloc(bytes);  // (set_rec_cap sized it for any bit range)
        SVX_CUDA(cub::DeviceRadixSort::SortKeys(m->fb_tmp.p, bytes, m->records.p, m->bucket.p, int(c.rec_cap), 0,
                                                end_bit, m->stream));
        launch_pdl(k_fb_runs, pg, kThreads, m->stream, m->bucket.p, m->records.p, c.rec_cap, c.pbits, m->fbdesc.p,
                   m->fctr, m->d_ctr);
        count_launch(1);
      }
    }
    // one profiling mark spans the group's folds when nothing runs between them (marks
    // between PDL launches cost their overlap), else one per fold
    std::unique_ptr<ProfMark> all_folds;
    if (!labels) all_folds = std::make_unique<ProfMark>(m, SVX_K_FOLD, c.G);
    for (uint32_t g = 0; g < c.G; ++g) {
        {
            std::unique_ptr<ProfMark> pm;
            if (labels) pm = std::make_unique<ProfMark>(m, SVX_K_FOLD);
            launch_pdl(k_fold, fold_grid(m->device), kThreads, m->stream, c, gp.f[g], g, sc, m->vals, m->block_keys,
                       tsdf_base(m), fm, m->vlist.p, m->fbdesc.p, m->bucket.p, m->touched, m->dirty, m->fctr, outs,
                       m->d_ctr);
            count_launch();
        }
        if (labels) {  // frame first + g's label images, after its fold, before the next
            const int f = first + int(g);
            if (labels->img_off[f + 1] > labels->img_off[f])
                labels_enqueue(m, *labels->lb, labels->img_off[f], labels->img_off[f + 1], g);
        }
    }
    all_folds.reset();
    SVX_CUDA(cudaGetLastError());
}

// CapacityError path (tsdf_integrator.cpp:160-168 + voxel_store.cpp:18-20) for the single
// frame in slot 0: blocks are allocated in sorted key order until max_blocks is reached;
// every block before the failing one is marked dirty; no voxel is updated.
[[noreturn]] void capacity_path(svx_map* m, svx_scan* s, const GroupParams& gp, uint32_t before) {
    uint32_t cap = uint32_t(std::min<uint64_t>(uint64_t(s->P) * 64, 1u << 30));
    for (;;) {
        m->records_alt.alloc(cap);
        SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_RECORDS, 0, 4, m->stream));
        k_collect_keys<<<grid_for(s->P), kThreads, 0, m->stream>>>(gp, scan_slots(s), m->records_alt.p, cap,
                                                                   m->d_ctr);
        count_launch();
        sync_counters(m);
        if (m->h_ctr[C_RECORDS] <= cap) break;
        cap = m->h_ctr[C_RECORDS];
    }
    const uint32_t n = m->h_ctr[C_RECORDS];
    std::vector<unsigned long long> keys(n);
    SVX_CUDA(cudaMemcpy(keys.data(), m->records_alt.p, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
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
        SVX_CUDA(cudaMemcpy(m->block_keys + before, alloc_new.data(), sizeof(unsigned long long) * alloc_new.size(),
                            cudaMemcpyHostToDevice));
    m->n_blocks = total;
    rebuild_hash(m);
    launch_zero_blocks(m, before, alloc_new.size());
    reset_frame_state(m);
    if (!dirty_keys.empty()) {
        m->records_alt.alloc(dirty_keys.size());
        SVX_CUDA(cudaMemcpy(m->records_alt.p, dirty_keys.data(), sizeof(unsigned long long) * dirty_keys.size(),
                            cudaMemcpyHostToDevice));
        k_mark_dirty<<<grid_for(dirty_keys.size()), kThreads, 0, m->stream>>>(
            reinterpret_cast<const uint64_t*>(m->records_alt.p), uint32_t(dirty_keys.size()), hash_view(m),
            m->dirty);
        count_launch();
    }
    SVX_CUDA(cudaStreamSynchronize(m->stream));
    throw Error(SVX_CAPACITY, "block budget exhausted (max_blocks = " + std::to_string(m->cfg.max_blocks) + ")");
}

}  // namespace

unsigned persistent_grid(int device) {
    static int sms[64] = {0};
    if (!sms[device]) cudaDeviceGetAttribute(&sms[device], cudaDevAttrMultiProcessorCount, device);
    return unsigned(sms[device] * 8);  // 8 CTAs x 8 warps per SM
}

// Fallback record buffers for `cap` records per group: the records (all ~0, the sort's
// padding key, outside a group's entries), their sorted copy and the run descriptors.
void set_rec_cap(svx_map* m, uint32_t cap) {
    const uint64_t had = m->records.n;
    m->records.alloc(cap);
    if (m->records.n != had)  // (re)allocated: contents undefined
        SVX_CUDA(cudaMemsetAsync(m->records.p, 0xFF, 8ull * m->records.n, m->stream));
    m->bucket.alloc(cap);
    m->bucket2.alloc(cap);  // merge scratch of big buckets (k_fb_sort)
    m->fbdesc.alloc(uint64_t(cap) * kMaxG);  // [frame of the group][cap]
    m->rec_cap = cap;
    size_t bytes = 0;  // the radix sort's scratch for every bit range (allocated here, not per group)
    SVX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, m->records.p, m->bucket.p, int(cap), 0, 64, m->stream));
    m->fb_tmp.alloc(bytes);
}

// Clears the group scratch (masks of the mapped blocks, fallback state, counters) after a
// host-side intervention, and re-arms the device block counters.
void reset_frame_state(svx_map* m) {
    if (m->mapped_blocks)
        SVX_CUDA(cudaMemsetAsync(mask_base(m), 0, 4ull * kMaskWords * m->mapped_blocks, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->records.p, 0xFF, 8ull * m->records.n, m->stream));  // the sort's padding
    SVX_CUDA(cudaMemsetAsync(m->fbcnt, 0, 4ull * m->cfg.max_blocks, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fbfill, 0, 4ull * m->cfg.max_blocks, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->fctr, 0, sizeof(uint32_t) * kMaxG * kFC, m->stream));
    for (int c : {C_TOUCHED, C_RECORDS, C_FB_VOXELS, C_FB_BLOCKS, C_BUCKET_TOP, C_ABORT, C_DONE})
        m->h_ctr[c] = 0;
    m->h_ctr[C_BLOCKS] = m->h_ctr[C_BLOCKS_BEFORE] = uint32_t(m->n_blocks);
    m->h_ctr[C_MAPPED] = uint32_t(m->mapped_blocks);
    SVX_CUDA(cudaMemcpyAsync(m->d_ctr, m->h_ctr, sizeof(uint32_t) * kNumCounters, cudaMemcpyHostToDevice,
                             m->stream));
    SVX_CUDA(cudaStreamSynchronize(m->stream));
}

namespace {

// Undoes an aborted group: its new blocks (and their hash entries, dirty flags), the visit
// masks and the rest of the group scratch (reset_frame_state); the scans' pixel keys are
// reset (later groups of the batch did not run). The frames before it are complete.
void rollback_group(svx_map* m, svx_scan* s, uint32_t before) {
    const uint64_t hi = std::min<uint64_t>(m->h_ctr[C_BLOCKS], m->cfg.max_blocks);
    if (hi > before) SVX_CUDA(cudaMemsetAsync(m->dirty + before, 0, hi - before, m->stream));
    m->n_blocks = before;
    rebuild_hash(m);
    if (s->slots) {
        SVX_CUDA(cudaMemsetAsync(s->pixkey.p, 0xFF, 16ull * s->P * s->slots, m->stream));
        for (int g = 0; g < kMaxG; ++g) s->parity[g] = 0;
    }
    reset_frame_state(m);
}

// Frames per group: up to kMaxG, with at most ~4M pixels of frame slots.
int group_cap(const svx_scan* s) {
    static const int knob = [] {  // experiment knob: SVX_GROUP=<frames per group>
        const char* e = std::getenv("SVX_GROUP");
        return e ? std::max(1, std::min(kMaxG, std::atoi(e))) : kMaxG;
    }();
    const uint64_t by_mem = std::max<uint64_t>(1, (uint64_t(1) << 22) / uint64_t(std::max(1, s->P)));
    return int(std::min<uint64_t>(uint64_t(knob), by_mem));
}

}  // namespace

namespace {
// The report of a completed frame (its FrameOut is final); numbers the frame.
void commit_frame(svx_map* m, svx_scan* s, const FrameOut& o, svx_frame_report& rep) {
    rep.frame = m->tsdf_frames++;
    rep.updated_voxels = o.updated;
    rep.new_blocks = o.new_blocks;
    m->new_ema = m->new_ema == 0.0 ? double(o.new_blocks) : 0.9 * m->new_ema + 0.1 * double(o.new_blocks);
    s->dropped = o.dropped;
    m->prof_acc.frames += 1;
    m->prof_acc.rays += o.rays;
    m->prof_acc.touched_blocks += o.touched;
    m->prof_acc.new_blocks += o.new_blocks;
    m->prof_acc.updated_voxels += o.updated;
    m->prof_acc.fallback_voxels += o.fb_voxels;
}

// DevBuf growth that keeps the first `keep` elements.
template <typename T>
void grow_keep(DevBuf<T>& b, size_t count, size_t keep, cudaStream_t stream) {
    if (count <= b.n) return;
    DevBuf<T> nb;
    nb.alloc(count);
    if (keep) SVX_CUDA(cudaMemcpyAsync(nb.p, b.p, sizeof(T) * keep, cudaMemcpyDeviceToDevice, stream));
    SVX_CUDA(cudaStreamSynchronize(stream));
    b.release();
    b = nb;
}
}  // namespace

namespace {
// Fallback ordering of the next batch: one CTA per block unless the per-block path just saw
// a bucket of more than kFbGlobalBucket records (a long single-CTA tail), then the global
// radix sort for kFbGlobalBatches batches before the per-block path is probed again (the
// global path does not measure bucket sizes).
constexpr int kFbGlobalBatches = 8;
void pick_fb_ordering(svx_map* m) {
    if (m->fb_env) return;
    if (m->fb_global) {
        if (--m->fb_global_left <= 0) m->fb_global = false;
        return;
    }
    if (m->h_ctr[C_FB_MAXB] > kFbGlobalBucket) {
        m->fb_global = true;
        m->fb_global_left = kFbGlobalBatches;
    }
    if (m->h_ctr[C_FB_MAXB]) {
        m->h_ctr[C_FB_MAXB] = 0;
        SVX_CUDA(cudaMemcpyAsync(m->d_ctr + C_FB_MAXB, &m->h_ctr[C_FB_MAXB], 4, cudaMemcpyHostToDevice, m->stream));
    }
}
}  // namespace

#ifndef SVX_INGEST_FIRST
#define SVX_INGEST_FIRST 4
#endif
constexpr int kIngestFirstGroup = SVX_INGEST_FIRST;

void run_frames(svx_map* m, const FrameJob* jobs, int n, const svx_integrator_cfg& cfg, svx_frame_report* reps,
                LabelHook* labels) {
    if (!(cfg.alpha_epsilon > 0.0)) throw Error(SVX_INVALID_ARGUMENT, "alpha_epsilon must be > 0");
    if (n <= 0) return;
    svx_scan* s = jobs[0].scan;
    for (int i = 0; i < n; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
        if (jobs[i].scan != s) throw Error(SVX_INVALID_ARGUMENT, "a batch integrates the frames of one scan model");
        if (!jobs[i].project && n != 1) throw Error(SVX_INVALID_ARGUMENT, "image frames are integrated one at a time");
        if (!jobs[i].project && !s->has_normals && cfg.mode == SVX_NON_PROJECTIVE)
            throw Error(SVX_INVALID_ARGUMENT, "non-projective mode needs a normal image");
    }
    if (uint64_t(s->P) >= (1ull << 28)) throw Error(SVX_INVALID_ARGUMENT, "scan image too large (>= 2^28 pixels)");
    const bool project = jobs[0].project;
    const bool ingest = jobs[0].host_ingest;
    const int gcap = project ? group_cap(s) : 1;
    const int gmax = std::min(gcap, n);
    uint64_t nmax = 1, most = 1;
    for (int i = 0; i < n; ++i) {
        nmax = std::max<uint64_t>(nmax, jobs[i].n);
        most = std::max<uint64_t>(most, jobs[i].n * uint64_t(jobs[i].stride));
    }
    ensure_scan_slots(s, gmax, project ? nmax : 0);
    m->outs.alloc(size_t(n));
    SVX_CUDA(cudaMemsetAsync(m->outs.p, 0, sizeof(FrameOut) * size_t(n), m->stream));
    if (m->h_outs_n < size_t(n)) {
        if (m->h_outs) cudaFreeHost(m->h_outs);
        SVX_CUDA(cudaMallocHost(&m->h_outs, sizeof(FrameOut) * n));
        m->h_outs_n = size_t(n);
    }
    // per-frame visited-voxel lists (~5 per pixel at cfg2, more in dense scenes): 12 per
    // pixel, grown on overflow (a growth costs a rollback and retry of the group)
    const uint64_t want_vox = std::min<uint64_t>(12ull * uint64_t(s->P) + 4096, 0x7FFFFFFFull);
    if (m->vox_cap < want_vox) m->vox_cap = uint32_t(want_vox);
    m->vlist.alloc(uint64_t(m->vox_cap) * uint64_t(gmax));
    // pool headroom for the batch (an exhausted headroom costs one rollback + retry; over-
    // mapping costs physical memory and cuMemCreate time, so size it from the recent rate)
    const uint64_t head =
        m->test_pool_head ? m->test_pool_head : std::max<uint64_t>(32768, uint64_t(2.0 * m->new_ema * n));
    ensure_blocks(m, m->n_blocks + head, 4 * head);
    // host ingest ring: group k's points are copied to staging slot k % R on the copy stream
    // while group k - 1 integrates
    constexpr int R = svx_map::kIngestSlots;
    if (ingest) {
        if (!m->copy_stream) {
            SVX_CUDA(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
            for (int r = 0; r < R; ++r) {
                SVX_CUDA(cudaEventCreateWithFlags(&m->ingest_ready[r], cudaEventDisableTiming));
                SVX_CUDA(cudaEventCreateWithFlags(&m->ingest_used[r], cudaEventDisableTiming));
            }
        }
        for (int r = 0; r < R; ++r) {
            m->ingest[r].alloc(most * uint64_t(gmax));
            SVX_CUDA(cudaEventRecord(m->ingest_used[r], m->stream));
        }
    }
    auto commit = [&](int i) { commit_frame(m, s, m->h_outs[i], reps[i]); };
    int f0 = 0;
    int single_lo = 0, single_hi = 0;  // frames run one per group (after a capacity / key abort)
    for (;;) {
        const auto te0 = std::chrono::steady_clock::now();
        std::vector<int> starts;
        GroupParams gp{};
        int k = 0;
        for (int a = f0; a < n; ++k) {
            // host ingest: the batch's first group is short (its H2D copy is the only one not
            // hidden behind a previous group's kernels)
            const int gfirst = (ingest && a == 0 && k == 0) ? std::min(gcap, kIngestFirstGroup) : gcap;
            const int G = (a >= single_lo && a < single_hi) ? 1 : std::min(gfirst, n - a);
            starts.push_back(a);
            gp.c = make_consts(m, s, cfg, uint32_t(G), project ? true : s->has_normals);
            for (int g = 0; g < G; ++g) gp.f[g] = make_pose(m, jobs[a + g].pose);
            if (project) {
                const void* pts[kMaxG];
                uint64_t cnt[kMaxG];
                Pose poses[kMaxG];
                const int r = k % R;
                if (ingest) {  // stage the group's points (pinned host -> device) on the copy stream
                    SVX_CUDA(cudaStreamWaitEvent(m->copy_stream, m->ingest_used[r], 0));
                    uint64_t off = 0;
                    for (int g = 0; g < G; ++g) {
                        const FrameJob& j = jobs[a + g];
                        if (j.n)
                            SVX_CUDA(cudaMemcpyAsync(m->ingest[r].p + off, j.pts, 4ull * j.n * j.stride,
                                                     cudaMemcpyHostToDevice, m->copy_stream));
                        pts[g] = m->ingest[r].p + off;
                        off += j.n * uint64_t(j.stride);
                    }
                    SVX_CUDA(cudaEventRecord(m->ingest_ready[r], m->copy_stream));
                    SVX_CUDA(cudaStreamWaitEvent(m->stream, m->ingest_ready[r], 0));
                } else {
                    for (int g = 0; g < G; ++g) pts[g] = jobs[a + g].pts;
                }
                for (int g = 0; g < G; ++g) {
                    cnt[g] = jobs[a + g].n;
                    poses[g] = jobs[a + g].pose;
                }
                launch_project_group(s, pts, cnt, G, jobs[a].stride, false, poses);
                if (ingest) SVX_CUDA(cudaEventRecord(m->ingest_used[r], m->stream));
            } else if (!s->rowdist_fresh) {  // images the caller uploaded into slot 0
                launch_pdl(k_row_dist, grid_for(s->P), kThreads, m->stream, s->depth.p, s->dm.W, s->dm.H,
                           s->rowdist.p, s->validbits.p, m->d_ctr);
                count_launch();
                s->rowdist_fresh = true;
            }
            launch_group_kernels(m, s, gp, m->outs.p + a, labels, a);
            a += G;
        }
        if (m->prof)
            m->prof_acc.host_enqueue_ms +=
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
        SVX_CUDA(cudaMemcpyAsync(m->h_outs, m->outs.p, sizeof(FrameOut) * n, cudaMemcpyDeviceToHost, m->stream));
        sync_counters(m);
        if (ingest) SVX_CUDA(cudaStreamSynchronize(m->copy_stream));
        const uint32_t abort = m->h_ctr[C_ABORT];
        if (!abort) break;
        const auto tr0 = std::chrono::steady_clock::now();
        for (int b = 0; b < 8; ++b) m->prof_acc.aborts[b] += (abort >> b) & 1u;
        // the first group whose frames have no report is the one that aborted
        int ga = 0;
        while (ga + 1 < int(starts.size()) && m->h_outs[starts[ga + 1] - 1].ok) ++ga;
        const int fa = starts[ga];
        const int fb = ga + 1 < int(starts.size()) ? starts[ga + 1] : n;
        for (int i = f0; i < fa; ++i) commit(i);
        const uint32_t before = m->h_ctr[C_BLOCKS_BEFORE];
        const uint32_t blocks_seen = m->h_ctr[C_BLOCKS], recs_seen = m->h_ctr[C_RECORDS];
        rollback_group(m, s, before);
        f0 = fa;
        if (abort & (kAbortCapacity | kAbortHash | kAbortKey)) {
            if (fb - fa > 1) {  // find the failing frame: the group again, one frame at a time
                single_lo = fa;
                single_hi = fb;
            } else if (abort & kAbortKey) {
                // the failing frame is numbered (the reference numbers a frame before it can
                // throw) and leaves no block behind (rolled back above)
                m->tsdf_frames++;
                throw Error(SVX_INVALID_ARGUMENT, "block coordinate outside the device key range [-2^20, 2^20)");
            } else {
                // the failing frame's images are in slot 0 (a group of one; its projection ran)
                m->tsdf_frames++;
                GroupParams g1{};
                g1.c = make_consts(m, s, cfg, 1, project ? true : s->has_normals);
                g1.f[0] = make_pose(m, jobs[fa].pose);
                capacity_path(m, s, g1, before);
            }
        }
        if (abort & kAbortPool) ensure_blocks(m, uint64_t(m->n_blocks) + 2 * head + (blocks_seen - before));
        if (abort & kAbortRecords) {
            set_rec_cap(m, std::max<uint32_t>(recs_seen + (recs_seen >> 1), m->rec_cap * 2));
        }
        if (abort & kAbortVox) {
            m->vox_cap = uint32_t(std::min<uint64_t>(uint64_t(m->vox_cap) * 2, 0x7FFFFFFFull));
            m->vlist.alloc(uint64_t(m->vox_cap) * uint64_t(gmax));
        }
        SVX_CUDA(cudaMemsetAsync(m->outs.p, 0, sizeof(FrameOut) * size_t(n), m->stream));
        m->prof_acc.host_resume_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
    }
    for (int i = f0; i < n; ++i) commit(i);
    m->n_blocks = m->h_ctr[C_BLOCKS];
    // fallback ordering for the next batch: one CTA per block is fastest unless some block
    // holds very many records (thousands of rays through a few voxels: a long single-CTA
    // tail), then the global radix sort over the record buffer
    pick_fb_ordering(m);
    // the record capacity follows use: the per-group sort covers all of it, so after a batch
    // whose largest group used less than half of it, it shrinks to 1.5x that group (+ slack);
    // a larger group later costs one rollback and retry with a grown buffer
    uint32_t hwm = 0;
    for (int i = 0; i < n; ++i) hwm = std::max(hwm, m->h_outs[i].records);
    const uint64_t want = (uint64_t(hwm) + hwm / 2 + 8192 + 4095) & ~uint64_t(4095);
    if (!m->test_rec_cap && 2 * uint64_t(hwm) < m->rec_cap && want < m->rec_cap) m->rec_cap = uint32_t(want);
}

namespace {
struct XState {  // a frame group between run_group_xbegin and run_group_xend
    GroupParams gp;
    svx_scan* s;
};
void free_xstate(void* p) { delete static_cast<XState*>(p); }
}  // namespace

void run_group_xbegin(svx_map* m, const FrameJob* jobs, int G, const svx_integrator_cfg& cfg,
                      uint64_t* send_meta, const void** d_send) {
    if (!(cfg.alpha_epsilon > 0.0)) throw Error(SVX_INVALID_ARGUMENT, "alpha_epsilon must be > 0");
    if (m->shard_world < 2 || m->shard_world > kMaxXWorld)
        throw Error(SVX_INVALID_ARGUMENT, "exchange mode needs a key-sharded map with 2..16 ranks");
    if (m->xstate) throw Error(SVX_INVALID_ARGUMENT, "xbegin: the previous group was not finished (xend)");
    if (G < 1 || G > kMaxG) throw Error(SVX_INVALID_ARGUMENT, "xbegin: 1..16 frames per group");
    svx_scan* s = jobs[0].scan;
    for (int i = 0; i < G; ++i)
        if (jobs[i].scan != s || !jobs[i].project)
            throw Error(SVX_INVALID_ARGUMENT, "xbegin: point clouds of one scan model");
    if (G > group_cap(s)) throw Error(SVX_INVALID_ARGUMENT, "xbegin: group too large for this scan size");
    const int world = m->shard_world;
    uint64_t nmax = 1;
    for (int i = 0; i < G; ++i) nmax = std::max<uint64_t>(nmax, jobs[i].n);
    ensure_scan_slots(s, G, nmax);
    m->outs.alloc(size_t(G));
    SVX_CUDA(cudaMemsetAsync(m->outs.p, 0, sizeof(FrameOut) * size_t(G), m->stream));
    if (m->h_outs_n < size_t(G)) {
        if (m->h_outs) cudaFreeHost(m->h_outs);
        SVX_CUDA(cudaMallocHost(&m->h_outs, sizeof(FrameOut) * G));
        m->h_outs_n = size_t(G);
    }
    const uint64_t want_vox = std::min<uint64_t>(8ull * uint64_t(s->P) + 4096, 0x7FFFFFFFull);
    if (m->vox_cap < want_vox) m->vox_cap = uint32_t(want_vox);
    m->vlist.alloc(uint64_t(m->vox_cap) * uint64_t(G));
    const uint64_t head = m->test_pool_head ? m->test_pool_head : std::max<uint64_t>(32768, uint64_t(2.0 * m->new_ema * G));
    ensure_blocks(m, m->n_blocks + head, 4 * head);
    if (!m->xcap) m->xcap = uint32_t(std::max<uint64_t>(1u << 16, 2ull * uint64_t(s->P) * uint64_t(G) / uint64_t(world)));
    m->xcnt.alloc(size_t(world) * kXMeta);
    m->xsend.alloc(uint64_t(world) * m->xcap);
    m->xpack.alloc(uint64_t(world) * m->xcap);
    if (!m->h_xmeta) SVX_CUDA(cudaMallocHost(&m->h_xmeta, 4ull * kMaxXWorld * kXMeta));
    uint32_t* meta = m->h_xmeta;  // pinned: the copy below stays asynchronous (one sync per group)
    auto xs = std::make_unique<XState>();
    xs->s = s;
    for (;;) {
        SVX_CUDA(cudaMemsetAsync(m->xcnt.p, 0, 4ull * world * kXMeta, m->stream));
        GroupParams& gp = xs->gp;
        gp.c = make_consts(m, s, cfg, uint32_t(G), true);
        gp.c.exchange = 1;
        gp.c.xcap = m->xcap;
        const void* pts[kMaxG];
        uint64_t n[kMaxG];
        Pose poses[kMaxG];
        for (int g = 0; g < G; ++g) {
            gp.f[g] = make_pose(m, jobs[g].pose);
            pts[g] = jobs[g].pts;
            n[g] = jobs[g].n;
            poses[g] = jobs[g].pose;
        }
        launch_project_group(s, pts, n, G, jobs[0].stride, false, poses);
        launch_group_kernels(m, s, gp, m->outs.p);  // exchange mode: the band only
        launch_pdl(k_xpack, dim3(64, unsigned(world)), kThreads, m->stream, static_cast<const uint4*>(m->xsend.p),
                   m->xcap, static_cast<const uint32_t*>(m->xcnt.p), m->xpack.p);
        count_launch();
        SVX_CUDA(cudaMemcpyAsync(meta, m->xcnt.p, 4ull * world * kXMeta, cudaMemcpyDeviceToHost, m->stream));
        SVX_CUDA(cudaMemcpyAsync(m->h_fctr, m->fctr, 4ull * kMaxG * kFC, cudaMemcpyDeviceToHost, m->stream));
        sync_counters(m);
        const uint32_t abort = m->h_ctr[C_ABORT];
        if (!abort) break;
        for (int b = 0; b < 8; ++b) m->prof_acc.aborts[b] += (abort >> b) & 1u;
        const uint32_t before = m->h_ctr[C_BLOCKS_BEFORE], blocks_seen = m->h_ctr[C_BLOCKS],
                       recs_seen = m->h_ctr[C_RECORDS];
        rollback_group(m, s, before);
        if (abort & kAbortKey)
            throw Error(SVX_INVALID_ARGUMENT, "block coordinate outside the device key range [-2^20, 2^20)");
        if (abort & (kAbortCapacity | kAbortHash))
            throw Error(SVX_CAPACITY, "block budget of this shard exhausted (max_blocks = " +
                                          std::to_string(m->cfg.max_blocks) + ")");
        if (abort & kAbortPool) ensure_blocks(m, uint64_t(m->n_blocks) + 2 * head + (blocks_seen - before));
        if (abort & kAbortRecords) {
            set_rec_cap(m, std::max<uint32_t>(recs_seen + (recs_seen >> 1), m->rec_cap * 2));
        }
        if (abort & kAbortVox) {
            m->vox_cap = uint32_t(std::min<uint64_t>(uint64_t(m->vox_cap) * 2, 0x7FFFFFFFull));
            m->vlist.alloc(uint64_t(m->vox_cap) * uint64_t(G));
        }
        if (abort & kAbortXchg) {
            uint32_t most = 0;
            for (int d = 0; d < world; ++d) most = std::max(most, meta[size_t(d) * kXMeta]);
            m->xcap = std::max<uint32_t>(m->xcap * 2, most + most / 2);
            m->xsend.alloc(uint64_t(world) * m->xcap);
            m->xpack.alloc(uint64_t(world) * m->xcap);
        }
        SVX_CUDA(cudaMemsetAsync(m->outs.p, 0, sizeof(FrameOut) * size_t(G), m->stream));
    }
    // (the lists were packed destination-major on the device by k_xpack)
    for (size_t i = 0; i < size_t(world) * kXMeta; ++i) send_meta[i] = meta[i];
    *d_send = m->xpack.p;
    m->xstate = xs.release();
    m->xstate_free = free_xstate;
}

void run_group_xend(svx_map* m, const void* d_recv, const uint64_t* recv_meta, svx_frame_report* reps) {
    XState* xs = static_cast<XState*>(m->xstate);
    if (!xs) throw Error(SVX_INVALID_ARGUMENT, "xend without xbegin");
    std::unique_ptr<XState> hold(xs);
    m->xstate = nullptr;
    GroupParams& gp = xs->gp;
    svx_scan* s = xs->s;
    const int G = int(gp.c.G);
    for (int i = 0; i < G; ++i) {
        reps[i].frame = -1;
        reps[i].updated_voxels = reps[i].new_blocks = 0;
    }
    const int world = m->shard_world;
    uint64_t n_recv = 0;
    uint64_t add[kMaxG] = {};  // bound on the received new voxels per frame
    for (int r = 0; r < world; ++r) {
        n_recv += recv_meta[size_t(r) * kXMeta];
        for (int g = 0; g < G; ++g) add[g] += recv_meta[size_t(r) * kXMeta + 1 + g];
    }
    if (n_recv >= (1ull << 31)) throw Error(SVX_INVALID_ARGUMENT, "xend: too many entries");
    // room for the received entries: each may add one block and one record
    ensure_blocks(m, uint64_t(m->h_ctr[C_BLOCKS]) + n_recv + 1);
    const uint64_t recs = m->h_ctr[C_RECORDS];
    if (recs + n_recv > m->rec_cap) {
        const uint32_t cap = uint32_t(std::min<uint64_t>((recs + n_recv) * 3 / 2 + 1024, 0xFFFFFFF0ull));
        grow_keep(m->records, cap, recs, m->stream);
        // the new tail holds the sort's padding key
        SVX_CUDA(cudaMemsetAsync(m->records.p + recs, 0xFF, 8ull * (m->records.n - recs), m->stream));
        set_rec_cap(m, cap);
    }
    gp.c.rec_cap = m->rec_cap;
    // the voxel lists: this rank's entries (xbegin) + at most the received voxel bits per
    // frame; grown here (keeping each frame's entries) before the ingest reserves positions
    uint64_t most = 0;
    for (int g = 0; g < G; ++g) most = std::max<uint64_t>(most, uint64_t(m->h_fctr[g * kFC + FC_VOX]) + add[g]);
    if (most > m->vox_cap) {
        const uint32_t ncap = uint32_t(std::min<uint64_t>(most * 5 / 4 + 1024, 0x7FFFFFFFull));
        DevBuf<uint32_t> nb;
        nb.alloc(uint64_t(ncap) * G);
        for (int g = 0; g < G; ++g) {
            const uint32_t keep = std::min(m->h_fctr[g * kFC + FC_VOX], m->vox_cap);
            if (keep)
                SVX_CUDA(cudaMemcpyAsync(nb.p + uint64_t(g) * ncap, m->vlist.p + uint64_t(g) * m->vox_cap, 4ull * keep,
                                         cudaMemcpyDeviceToDevice, m->stream));
        }
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        m->vlist.release();
        m->vlist = nb;
        m->vox_cap = ncap;
    }
    gp.c.vox_cap = m->vox_cap;
    const unsigned grid = persistent_grid(m->device);
    if (n_recv) {
        m->xaux.alloc(n_recv);
        launch_pdl(k_ingest, grid, kThreads, m->stream, gp.c, static_cast<const uint4*>(d_recv), uint32_t(n_recv),
                   hash_view(m), m->block_keys, m->stamp, m->touched, mask_base(m), m->records.p,
                   tsdf_base(m), m->xaux.p, m->fctr, m->d_ctr);
        count_launch();
        launch_pdl(k_ingest_list, grid, kThreads, m->stream, gp.c, static_cast<const uint4*>(m->xaux.p),
                   uint32_t(n_recv), m->vlist.p, m->d_ctr);
        count_launch();
    }
    launch_fold_kernels(m, s, gp, m->outs.p, nullptr, 0);
    SVX_CUDA(cudaMemcpyAsync(m->h_outs, m->outs.p, sizeof(FrameOut) * G, cudaMemcpyDeviceToHost, m->stream));
    sync_counters(m);
    if (m->h_ctr[C_ABORT]) throw Error(SVX_CUDA, "xend: fold aborted");
    for (int i = 0; i < G; ++i) commit_frame(m, s, m->h_outs[i], reps[i]);
    m->n_blocks = m->h_ctr[C_BLOCKS];
    pick_fb_ordering(m);  // for the next group (as after a batch in run_frames)
}

}  // namespace svx
