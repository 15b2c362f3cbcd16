// Shared device-side definitions of the B200 semvox hot path.
//
// Arithmetic contract: this code is compiled with --fmad=false, so every
// double/float expression below rounds exactly like the reference's Release
// build (-O3, no -march => no FMA contraction). Reductions follow Eigen's order:
// 3-term dot products are (a0*b0 + a1*b1) + a2*b2; Isometry*p = t + R p;
// normalized() divides by sqrt(squaredNorm). Transcendentals on the integer
// decision paths (pixel of a point / of a voxel centre) run in FP32 with a
// proven error margin and fall back to FP64 near a pixel boundary.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "../../include/svx.h"

namespace svx {

constexpr int kBlockSide = 8;
constexpr int kBlockVoxels = 512;
// TSDF frames integrated together by one group of kernel launches (svx_tsdf.cu)
constexpr int kMaxG = 16;
// Per-block visit masks of a frame group (svx_tsdf.cu), 16 words (512 voxel bits) per row:
// row g = voxels visited by frame g, row kHdrRow word 0 = frames that touched the block
// (bit g). Cleared as the group is folded.
constexpr int kHdrRow = kMaxG;
constexpr int kMaskWords = (kHdrRow + 1) * 16;
enum FrameCounter : int {
    FC_UPD = 0,  // voxels updated
    FC_RAYS,     // band rays cast
    FC_DROPPED,  // points dropped by project_point
    FC_TIES,     // tie-list entries (projection)
    FC_TOUCH,    // blocks touched
    FC_NEW,      // blocks new to the map
    FC_FBV,      // voxels measured by their visiting rays (own pixel without a return)
    FC_VOX,      // visited voxels listed (the frame's fold work)
    FC_VQ,       // k_fold work queue position (visited voxels)
    kFC = 16
};
constexpr double kPi = 3.14159265358979323846;

// Packed block key: 21 bits per axis, biased by 2^20 so that unsigned order of
// the packed value equals the lexicographic (x, y, z) order of BlockCoord
// (types.hpp:59-68). Valid block coordinates: [-2^20, 2^20).
constexpr int kKeyBits = 21;
constexpr int32_t kKeyBias = 1 << 20;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint32_t kInvalid = 0xFFFFFFFFu;

__host__ __device__ inline bool key_in_range(int32_t b) {
    return b >= -kKeyBias && b < kKeyBias;
}
__host__ __device__ inline uint64_t pack_key(int32_t bx, int32_t by, int32_t bz) {
    return (uint64_t(uint32_t(bx + kKeyBias)) << (2 * kKeyBits)) |
           (uint64_t(uint32_t(by + kKeyBias)) << kKeyBits) | uint64_t(uint32_t(bz + kKeyBias));
}
__host__ __device__ inline void unpack_key(uint64_t k, int32_t& bx, int32_t& by, int32_t& bz) {
    const uint64_t m = (1ull << kKeyBits) - 1;
    bx = int32_t((k >> (2 * kKeyBits)) & m) - kKeyBias;
    by = int32_t((k >> kKeyBits) & m) - kKeyBias;
    bz = int32_t(k & m) - kKeyBias;
}
// Fibonacci hashing into a power-of-two table.
__host__ __device__ inline uint32_t hash_slot(uint64_t key, int log2cap) {
    return uint32_t((key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap));
}
// Shard owner of a block: a mixed hash, uniform over ranks.
__host__ __device__ inline int32_t owner_of(uint64_t key, int32_t world) {
    uint64_t h = key ^ (key >> 31);
    h *= 0xD6E8FEB86659FD93ull;
    h ^= h >> 32;
    return world <= 1 ? 0 : int32_t(h % uint64_t(world));
}

struct d3 {
    double x, y, z;
};

__host__ __device__ inline d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__host__ __device__ inline double dot3(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ inline d3 sub3(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ inline d3 add3(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ inline d3 scale3(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
__host__ __device__ inline d3 div3(d3 a, double s) { return d3{a.x / s, a.y / s, a.z / s}; }
__host__ __device__ inline d3 neg3(d3 a) { return d3{-a.x, -a.y, -a.z}; }

// Rigid transform, row-major R; inverse precomputed on the host exactly like
// Eigen's Isometry::inverse(): (R^T, (-R^T) t).
struct Pose {
    double R[9];
    double t[3];
};

__host__ __device__ inline d3 matvec(const double* R, d3 p) {
    return d3{(R[0] * p.x + R[1] * p.y) + R[2] * p.z, (R[3] * p.x + R[4] * p.y) + R[5] * p.z,
              (R[6] * p.x + R[7] * p.y) + R[8] * p.z};
}
// Isometry * p = t + (R p)   (Eigen transform_right_product_impl)
__host__ __device__ inline d3 xform(const Pose& T, d3 p) {
    const d3 rp = matvec(T.R, p);
    return d3{T.t[0] + rp.x, T.t[1] + rp.y, T.t[2] + rp.z};
}
__host__ __device__ inline Pose inverse_pose(const Pose& T) {
    Pose inv;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) inv.R[3 * i + j] = T.R[3 * j + i];
    double negRt[9];
    for (int k = 0; k < 9; ++k) negRt[k] = -inv.R[k];
    const d3 ti = matvec(negRt, d3{T.t[0], T.t[1], T.t[2]});
    inv.t[0] = ti.x;
    inv.t[1] = ti.y;
    inv.t[2] = ti.z;
    return inv;
}

// ProjectionModel plus derived constants for the FP32 fast path.
struct Model {
    int32_t W, H;
    double dphi, dtheta, theta0, min_range;
    float inv_dphi_f, inv_dtheta_f, theta0_f;
    float margin_u, margin_v;  // pixel-coordinate error bound of the FP32 path
    float r2_lo, r2_hi;        // (min_range (1 -+ 1e-5))^2: decidable range band
};

// atan2 on the FMA pipe: octant reduction + odd minimax polynomial of degree 15
// (coefficients fitted offline; max |error| 1.2e-7 rad measured in float32 over
// 1e7 points of [0, 1], plus <= 2 ulp from __fdividef and the octant fix-ups).
// Only used where an explicit error margin decides whether the result is final.
__device__ inline float fast_atan2f(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float a = mx > 0.f ? __fdividef(mn, mx) : 0.f;
    const float s = a * a;
    float r = -4.054556135e-03f;
    r = __fmaf_rn(r, s, 2.186293714e-02f);
    r = __fmaf_rn(r, s, -5.591233820e-02f);
    r = __fmaf_rn(r, s, 9.642202407e-02f);
    r = __fmaf_rn(r, s, -1.390863359e-01f);
    r = __fmaf_rn(r, s, 1.994656771e-01f);
    r = __fmaf_rn(r, s, -3.332986236e-01f);
    r = __fmaf_rn(r, s, 9.999993443e-01f);
    r = r * a;
    if (ay > ax) r = 1.57079637f - r;
    if (x < 0.f) r = 3.14159274f - r;
    return copysignf(r, y);
}

constexpr uint32_t kNeedFp64 = 0xFFFFFFFEu;
constexpr int kRowDistMax = 11;  // cap of the row-distance map (valid-radius skip)

// Pixel of a sensor-frame vector p given in FP32 with |error| <= ~2e-6 |p|.
// Returns the pixel index, kInvalid (no pixel), or kNeedFp64 when the FP32
// value is too close to a pixel boundary / the min-range threshold to decide.
__device__ inline uint32_t pixel_fast(float px, float py, float pz, const Model& m, float r2_lo,
                                      float r2_hi) {
    const float r2 = px * px + py * py + pz * pz;
    if (r2 < r2_lo) return kInvalid;  // range < min_range for sure
    if (!(r2 > r2_hi)) return kNeedFp64;
    // The azimuth error of an input with absolute error ~3e-7 |p| is ~3e-7 |p| / rxy:
    // the fixed margin_u budget only covers rxy >= 0.05 |p| (polar angle >= ~2.9 deg
    // from either pole); closer to the pole the FP64 reference formula decides.
    const float rxy2 = px * px + py * py;
    if (!(rxy2 >= 0.0025f * r2)) return kNeedFp64;
    const float rxy = sqrtf(rxy2);
    const float uf = (3.14159274f - fast_atan2f(py, px)) * m.inv_dphi_f;
    const float vf = (fast_atan2f(rxy, pz) - m.theta0_f) * m.inv_dtheta_f;
    const float fu = uf - floorf(uf), fv = vf - floorf(vf);
    if (!(fu > m.margin_u && fu < 1.f - m.margin_u && fv > m.margin_v && fv < 1.f - m.margin_v))
        return kNeedFp64;
    int ui = int(floorf(uf)) % m.W;
    if (ui < 0) ui += m.W;
    const int vi = int(floorf(vf));
    if (vi < 0 || vi >= m.H) return kInvalid;
    return uint32_t(vi) * uint32_t(m.W) + uint32_t(ui);
}

// project_point (scan_projection.cpp:21-37) evaluated exactly as the reference
// does (FP64 atan2/acos); the slow path behind pixel_fast().
__device__ inline uint32_t pixel_fp64(d3 p, const Model& m) {
    const double range = sqrt(dot3(p, p));
    if (!isfinite(range) || range < m.min_range) return kInvalid;
    const double az = atan2(p.y, p.x);
    int ui = int(floor((kPi - az) / m.dphi));
    ui %= m.W;
    if (ui < 0) ui += m.W;
    double c = p.z / range;
    c = c < -1.0 ? -1.0 : (1.0 < c ? 1.0 : c);
    const int vi = int(floor((acos(c) - m.theta0) / m.dtheta));
    if (vi < 0 || vi >= m.H) return kInvalid;
    return uint32_t(vi) * uint32_t(m.W) + uint32_t(ui);
}

// project_point for a sensor-frame point: FP32 decision with FP64 fallback.
__device__ inline uint32_t project_pixel(d3 p, const Model& m) {
    const uint32_t q = pixel_fast(float(p.x), float(p.y), float(p.z), m, m.r2_lo, m.r2_hi);
    return q == kNeedFp64 ? pixel_fp64(p, m) : q;
}

// world_to_voxel (types.hpp:168-173)
__device__ inline void world_to_voxel(d3 p, double inv, int32_t c[3]) {
    c[0] = int32_t(floor(p.x * inv + 0.5));
    c[1] = int32_t(floor(p.y * inv + 0.5));
    c[2] = int32_t(floor(p.z * inv + 0.5));
}

// block_of / local_index for kBlockSide = 8: floor_div == arithmetic shift,
// nonneg_mod == & 7 on two's complement (types.hpp:35-44, 81-89).
__host__ __device__ inline int32_t block_coord(int32_t c) { return c >> 3; }

// One axis of traverse_segment's set-up (tsdf_integrator.hpp:108-120).
__device__ inline void dda_axis(double d, double a, int32_t c, double nu, int32_t& step,
                                double& t_max, double& t_delta) {
    if (fabs(d) < 1e-15) {
        step = 0;
        t_max = CUDART_INF;
        t_delta = CUDART_INF;
    } else {
        step = d > 0 ? 1 : -1;
        const double boundary = nu * (double(c) + 0.5 * step);
        t_max = (boundary - a) / d;
        t_delta = nu / fabs(d);
    }
}

// traverse_segment (tsdf_integrator.hpp:93-135); visit(x, y, z) per cell.
// (shared by the TSDF band and the occupancy carving)
// kArrays: the per-axis state in 3-element arrays indexed by the chosen axis (local
// memory; measured ~1% faster in the register-limited TSDF band kernel), else scalars
// (the occupancy visit: 1.3x, no stack frame).
template <bool kArrays = false, typename Visit>
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
    if constexpr (kArrays) {
        const double dv[3] = {dir.x, dir.y, dir.z};
        const double av[3] = {a.x, a.y, a.z};
        int32_t step[3];
        double t_max[3], t_delta[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) dda_axis(dv[i], av[i], cur[i], nu, step[i], t_max[i], t_delta[i]);
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
    } else {
        // Per-axis DDA state in scalars (no dynamically indexed arrays: those live in local
        // memory); the axis choice and every update are the reference's, in its order.
        int32_t cx = cur[0], cy = cur[1], cz = cur[2];
        int32_t sx, sy, sz;
        double tx, ty, tz, dx, dy, dz;
        dda_axis(dir.x, a.x, cx, nu, sx, tx, dx);
        dda_axis(dir.y, a.y, cy, nu, sy, ty, dy);
        dda_axis(dir.z, a.z, cz, nu, sz, tz, dz);
        const uint64_t max_steps = uint64_t(3.0 * len / nu) + 8;
        for (uint64_t n = 0; n < max_steps; ++n) {
            visit(cx, cy, cz);
            if (cx == end[0] && cy == end[1] && cz == end[2]) return;
            // m = argmin with the reference's strict comparisons (ties keep the lower axis)
            int m = 0;
            double tm = tx;
            if (ty < tm) { m = 1; tm = ty; }
            if (tz < tm) { m = 2; tm = tz; }
            if (tm > len) return;
            if (m == 0) { cx += sx; tx += dx; }
            else if (m == 1) { cy += sy; ty += dy; }
            else { cz += sz; tz += dz; }
        }
    }
}

__host__ __device__ inline int local_linear(int32_t x, int32_t y, int32_t z) {
    return (x & 7) + 8 * (y & 7) + 64 * (z & 7);
}

// ---- exact f32 results from one-reciprocal estimates
// The reference stores float(x / y) (or float(clamp(x / y))) of a correctly rounded double
// quotient. An estimate q with |q - fl(x / y)| <= kQuotTol |q| decides that float whenever
// both ends of [q - kQuotTol |q|, q + kQuotTol |q|] round to the same float (rounding is
// monotonic); otherwise the exact division is used. The estimates below are within ~5 ulp
// (2^-52 relative each): kQuotTol = 4e-15 is ~18 ulp. Undecided cases need the exact
// double to lie within 4e-15 of a float rounding boundary (relative spacing 6e-8).
constexpr double kQuotTol = 4e-15;

// 1 / b for 1e-300 < b < 1e300: hardware estimate + two Newton steps (rel. error ~2^-52).
__device__ __forceinline__ double rcp_est(double b) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    double e = __fma_rn(-b, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-b, r, 1.0);
    return __fma_rn(r, e, r);
}

// 1 / sqrt(x) for 1e-300 < x < 1e300: hardware estimate + two Newton steps (rel. error
// within ~3 ulp; no special-case handling: callers guarantee the range).
__device__ __forceinline__ double rsqrt_est(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double r = __fma_rn(-(hx * y), y, 0.5);
    y = __fma_rn(y, r, y);
    r = __fma_rn(-(hx * y), y, 0.5);
    return __fma_rn(y, r, y);
}

// float(x / y) for y > 0.
__device__ __forceinline__ float f32_div(double x, double y) {
    if (y > 1e-300 && y < 1e300) {
        const double q = x * rcp_est(y), d = fabs(q) * kQuotTol;
        const float lo = float(q - d), hi = float(q + d);
        if (__float_as_uint(lo) == __float_as_uint(hi)) return lo;
    }
    return float(x / y);
}

// float(x) from an estimate q with |q - x| <= kQuotTol |q| (<= 36 ulps of q), decided with
// one conversion: x and q round to the same float unless a rounding midpoint between two
// floats lies within the error interval. Within q's binade those midpoints are exactly the
// doubles whose 29 low mantissa bits equal 2^28 (the midpoint below a power of two included),
// so q decides when its low bits are more than 64 ulps away from that pattern. Normal-range
// results only (2^-126 <= |q| < 2^127, tested on the biased exponent), and q = 0 (an exact
// zero numerator). Integer tests only: no FP64 compares.
__device__ __forceinline__ bool f32_of_est(double q, float& f) {
    const uint32_t hi = uint32_t(__double2hiint(q)), lo = uint32_t(__double2loint(q));
    const uint32_t e = (hi >> 20) & 0x7FFu;                 // 1023 + exponent
    const bool normal = e - 897u <= 1149u - 897u;           // 2^-126 <= |q| < 2^127
    const uint32_t dist = (lo & 0x1FFFFFFFu) - 0x10000000u;   // low bits - the midpoint pattern
    const bool far = dist + 64u > 128u;                     // |dist| > 64 (two's complement)
    f = float(q);
    return (normal && far) || ((hi & 0x7FFFFFFFu) | lo) == 0u;
}

// ----------------------------------------------------------------- hash
struct HashView {
    uint64_t* keys;  // kEmptyKey = free
    uint32_t* vals;  // pool index of the block in the slot
    int log2cap;
    uint32_t mask;
};

__device__ inline uint32_t hash_find(const HashView& h, uint64_t key) {
    uint32_t s = hash_slot(key, h.log2cap);
    for (uint32_t probe = 0; probe <= h.mask; ++probe) {
        const uint64_t k = __ldcg(&h.keys[s]);
        if (k == key) return s;
        if (k == kEmptyKey) return kInvalid;
        s = (s + 1) & h.mask;
    }
    return kInvalid;
}

// Returns the slot; *inserted = 1 when this thread claimed it.
__device__ inline uint32_t hash_insert(const HashView& h, uint64_t key, int* inserted) {
    uint32_t s = hash_slot(key, h.log2cap);
    *inserted = 0;
    for (uint32_t probe = 0; probe <= h.mask; ++probe) {
        uint64_t k = __ldcg(&h.keys[s]);
        if (k == key) return s;
        if (k == kEmptyKey) {
            const unsigned long long old =
                atomicCAS(reinterpret_cast<unsigned long long*>(&h.keys[s]), kEmptyKey, key);
            if (old == kEmptyKey) {
                *inserted = 1;
                return s;
            }
            if (old == key) return s;
        }
        s = (s + 1) & h.mask;
    }
    return kInvalid;
}

// ------------------------------------------------------------ counters
// Per-map device counters (one 64-byte line each group).
enum Counter : int {
    C_BLOCKS = 0,       // allocated blocks (pool high-water mark)
    C_SEM = 1,          // allocated semantic layers
    C_TOUCHED = 2,      // blocks touched by the current frame group
    C_RECORDS = 5,      // fallback visit records of the group
    C_FB_VOXELS = 6,    // (unused since the per-frame descriptor lists: FC_FBV counts them)
    C_CAND = 10,        // semantic candidate blocks
    C_ERR_CONF = 11,    // confidence outside [0, 1]
    C_SEM_UPDATED = 12,
    C_ABORT = 16,       // bitmask of abort reasons (kAbort*); every frame kernel no-ops while set
    C_BLOCKS_BEFORE = 17,  // C_BLOCKS at the start of the current frame group
    C_MAPPED = 18,      // blocks with pool + visit-mask memory mapped (host-written)
    C_DONE = 24,        // CTAs of k_fold finished (the last one writes the group's reports)
    C_FB_BLOCKS = 25,   // blocks holding fallback records this group (per-block ordering)
    C_BUCKET_TOP = 26,  // fallback bucket space handed out this group
    C_FB_MAXB = 27,     // largest fallback bucket of the batch (the host picks the ordering)
    kNumCounters = 32
};

// Any abort stops the rest of the batch; the host rolls the aborted frame group back
// (svx_tsdf.cu, rollback_group) and retries it.
enum AbortBits : uint32_t {
    kAbortPool = 1,      // pool mapping exhausted: map more, retry the group
    kAbortCapacity = 2,  // max_blocks exceeded: frame by frame, then the CapacityError path
    kAbortKey = 4,       // block coordinate outside the key range
    kAbortHash = 8,      // hash table full (implies capacity)
    kAbortRecords = 16,  // fallback record buffer too small: grow, retry
    kAbortXchg = 32,     // exchange send list too small (multi-GPU data plane): grow, retry
    kAbortVox = 64       // visited-voxel list too small: grow, retry
};

// Per-frame results written by k_frame_end (device), read back per batch.
struct FrameOut {
    uint32_t updated, new_blocks, touched, records, rays, dropped, fb_voxels, ok;
};

__device__ inline uint32_t warp_agg_add(uint32_t* ctr, uint32_t n) {
    // warp-aggregated atomicAdd; returns this lane's base offset
    const unsigned active = __activemask();
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    const int leader = __ffs(active) - 1;
    // exclusive prefix over the active lanes, in lane order
    uint32_t prefix = 0, total = 0;
    for (int l = 0; l < 32; ++l) {
        if (!((active >> l) & 1u)) continue;
        const uint32_t nl = __shfl_sync(active, n, l);
        if (l < lane) prefix += nl;
        total += nl;
    }
    if (lane == leader && total) base = atomicAdd(ctr, total);
    base = __shfl_sync(active, base, leader);
    return base + prefix;
}

// Single-item variant: one atomic per warp (count of active lanes with pred).
__device__ inline uint32_t warp_agg_inc(uint32_t* ctr) {
    const unsigned active = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(active) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(ctr, uint32_t(__popc(active)));
    base = __shfl_sync(active, base, leader);
    return base + __popc(active & ((1u << lane) - 1u));
}

// Programmatic dependent launch (PDL): frame kernels are launched so that the
// next one can be scheduled while the previous one drains. pdl_wait() blocks
// until the previous grid has completed and its writes are visible (a no-op for
// a normal launch); pdl_trigger() lets the next grid start launching once every
// CTA of this grid has passed it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Whether pixel p has a return (depth != 0): one bit per pixel, built with the
// depth image (k_finish_pixels / k_row_dist). 16 KB at 131k pixels, so the
// per-visit own-pixel tests hit L1 instead of reading depth[] from L2.
__device__ __forceinline__ bool pixel_has_return(const uint32_t* __restrict__ bits, uint32_t p) {
    return (__ldg(&bits[p >> 5]) >> (p & 31)) & 1u;
}

// CTA-uniform read of the abort word (bits in `mask`): kernels with barriers must
// not let their threads disagree about it (another CTA may set it meanwhile).
__device__ inline bool cta_aborted(const uint32_t* ctr, uint32_t mask = 0xFFFFFFFFu) {
    return __syncthreads_or(threadIdx.x == 0 ? int((ctr[C_ABORT] & mask) != 0) : 0) != 0;
}

// CTA-wide reservation of n entries per thread in a list whose length lives in
// *counter: one atomic per CTA (a single global counter serialises per-thread or
// per-warp atomics at L2). Returns this thread's first position. Every thread of
// the CTA must call it; s_w is shared scratch of 2 * kWarps words.
template <int kWarps>
__device__ inline uint32_t cta_reserve(uint32_t n, uint32_t* counter, uint32_t* s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < kWarps; ++i) {
            const uint32_t c = s_w[i];
            s_w[kWarps + i] = s;
            s += c;
        }
        const uint32_t b = s ? atomicAdd(counter, s) : 0u;
        for (int i = 0; i < kWarps; ++i) s_w[kWarps + i] += b;
    }
    __syncthreads();
    const uint32_t pos = s_w[kWarps + wid] + incl - n;
    __syncthreads();  // s_w may be reused after return
    return pos;
}

// cta_reserve of one entry for the threads with take set.
template <int kWarps>
__device__ inline uint32_t cta_append(bool take, uint32_t* counter, uint32_t* s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, take);
    const uint32_t rank = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) s_w[wid] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < kWarps; ++i) {
            const uint32_t c = s_w[i];
            s_w[kWarps + i] = s;
            s += c;
        }
        const uint32_t b = s ? atomicAdd(counter, s) : 0u;
        for (int i = 0; i < kWarps; ++i) s_w[kWarps + i] += b;
    }
    __syncthreads();
    const uint32_t pos = s_w[kWarps + wid] + rank;
    __syncthreads();  // s_w may be reused after return
    return pos;
}

}  // namespace svx
