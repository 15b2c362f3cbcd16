// K1/K2: project_cloud + compute_normal_image on the device.
//
// project_cloud (scan_projection.cpp:39-76) is a serial nearer-wins scatter with
// a lexicographic tie-break. Here it is order-independent by construction, in two
// kernels per scan:
//   k_project_points  one thread per point: pixel (FP32 polynomial atan2 with an
//                     error margin, FP64 reference formula near a boundary), then
//                     atomicMin of (f32 range bits << 32 | point index) on the pixel.
//                     When two equal ranges meet, both points are appended to a tie
//                     list and the pixel is flagged (every point with the pixel's
//                     final range ends up in the list).
//   k_finish_pixels   one thread per pixel: flagged pixels pick the lexicographically
//                     smallest (x, y, z) among their equal-range points (std::tie in
//                     the reference); depth, height = (pose * p).z of the winner, and
//                     the normal of compute_normal_image (scan_projection.cpp:86-109)
//                     from the three neighbour depths, with back_project directions
//                     from a host-libm table (bit-exact). It also resets the other half
//                     of the double-buffered pixel keys for the next scan.
#include <algorithm>

#include "svx_map.hpp"

namespace svx {

namespace {

constexpr int kThreads = 256;

__device__ inline bool lex_less(d3 a, d3 b) {
    if (a.x < b.x) return true;
    if (b.x < a.x) return false;
    if (a.y < b.y) return true;
    if (b.y < a.y) return false;
    return a.z < b.z;
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_project_points(const T* __restrict__ pts, uint64_t n, int stride, Model m,
                 unsigned long long* __restrict__ pixkey, uint8_t* __restrict__ tie,
                 unsigned long long* __restrict__ ties, uint32_t tie_cap,
                 uint32_t* __restrict__ ctr) {
    // The point loads and the pixel computation read only this frame's input (never
    // written by the frame kernels before it), so they run before the dependency wait
    // and overlap the previous frame's last kernels; every write comes after it.
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double x = 0.0, y = 0.0, z = 0.0, r = 0.0;
    uint32_t pix = kInvalid;
    if (i < n) {
        x = pts[i * stride];
        y = pts[i * stride + 1];
        z = pts[i * stride + 2];
        r = sqrt(dot3(mk(x, y, z), mk(x, y, z)));
        if (isfinite(r) && !(r < m.min_range)) {
            pix = pixel_fast(float(x), float(y), float(z), m, m.r2_lo, m.r2_hi);
            if (pix == kNeedFp64) pix = pixel_fp64(mk(x, y, z), m);
        }
    }
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    if (i >= n) return;
    if (pix == kInvalid) {
        warp_agg_inc(&ctr[C_DROPPED]);
        return;
    }
    const unsigned long long key =
        (static_cast<unsigned long long>(__float_as_uint(float(r))) << 32) | uint32_t(i);
    const unsigned long long old = atomicMin(&pixkey[pix], key);
    if (old != ~0ull && (old >> 32) == (key >> 32)) {
        tie[pix] = 1;
        const uint32_t pos = atomicAdd(&ctr[C_TIES], 2u);
        if (pos + 1 < tie_cap) {
            ties[pos] = (static_cast<unsigned long long>(pix) << 32) | uint32_t(old);
            ties[pos + 1] = (static_cast<unsigned long long>(pix) << 32) | uint32_t(i);
        }
    }
}

__device__ inline float key_depth(unsigned long long k) {
    return k == ~0ull ? 0.f : __uint_as_float(uint32_t(k >> 32));
}

__device__ inline d3 dir_at(const double* __restrict__ dirs, uint32_t p) {
    return mk(dirs[3 * p], dirs[3 * p + 1], dirs[3 * p + 2]);
}

// compute_normal_image body for one pixel (scan_projection.cpp:91-107).
__device__ inline bool normal_at(const double* __restrict__ dirs, int W, int u, int v, float d0,
                                 float d1, float d2, float out[3]) {
    if (d0 == 0.f || d1 == 0.f || d2 == 0.f) return false;
    const d3 p = scale3(double(d0), dir_at(dirs, uint32_t(v) * W + u));
    const d3 p1 = scale3(double(d1), dir_at(dirs, uint32_t(v - 1) * W + u));
    const d3 p2 = scale3(double(d2), dir_at(dirs, uint32_t(v) * W + u - 1));
    const d3 a = sub3(p1, p), b = sub3(p2, p);
    d3 cr = mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
    const double norm = sqrt(dot3(cr, cr));
    if (norm < 1e-8) return false;
    cr = div3(cr, norm);
    if (dot3(cr, neg3(p)) < 0.0) cr = neg3(cr);
    out[0] = float(cr.x);
    out[1] = float(cr.y);
    out[2] = float(cr.z);
    return true;
}

template <typename T>
__device__ inline d3 point_at(const T* __restrict__ pts, int stride, uint32_t i) {
    return mk(pts[uint64_t(i) * stride], pts[uint64_t(i) * stride + 1],
              pts[uint64_t(i) * stride + 2]);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_finish_pixels(const T* __restrict__ pts, int stride, const unsigned long long* __restrict__ pixkey,
                unsigned long long* __restrict__ next_pixkey, const double* __restrict__ dirs,
                Pose pose, int W, int H, int with_normals, float* __restrict__ depth,
                float* __restrict__ height, float* __restrict__ normals,
                uint8_t* __restrict__ valid, uint8_t* __restrict__ tie,
                const unsigned long long* __restrict__ ties, uint32_t tie_cap,
                uint8_t* __restrict__ rowdist, uint32_t* __restrict__ validbits,
                const uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool inside = p < uint32_t(W) * H;
    const unsigned long long k = inside ? pixkey[p] : ~0ull;
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, k != ~0ull);  // pixels with a return
    if ((threadIdx.x & 31) == 0 && inside) validbits[p >> 5] = bits;
    if (!inside) return;
    next_pixkey[p] = ~0ull;  // the other half is clean for the next projection
    const float d0 = key_depth(k);
    depth[p] = d0;
    {   // row distance to the nearest pixel without a return (k_row_dist, from the keys)
        const int u = int(p % W);
        const unsigned long long* row = pixkey + (p - u);
        int d = 0;
        for (; d <= kRowDistMax; ++d) {
            int a = u + d, b = u - d;
            a -= a >= W ? W : 0;
            b += b < 0 ? W : 0;
            if (row[a] == ~0ull || row[b] == ~0ull) break;
        }
        rowdist[p] = uint8_t(d);
    }
    float h = 0.f;
    if (k != ~0ull) {
        uint32_t win = uint32_t(k);
        if (tie[p]) {
            // lexicographic minimum among the points of this pixel with its range
            d3 best = point_at(pts, stride, win);
            const uint32_t nt = min(ctr[C_TIES], tie_cap);
            for (uint32_t t = 0; t < nt; ++t) {
                const unsigned long long e = ties[t];
                if (uint32_t(e >> 32) != p) continue;
                const uint32_t i = uint32_t(e);
                const d3 q = point_at(pts, stride, i);
                if (__float_as_uint(float(sqrt(dot3(q, q)))) != uint32_t(k >> 32)) continue;
                if (lex_less(q, best)) {
                    best = q;
                    win = i;
                }
            }
            tie[p] = 0;
        }
        h = float(xform(pose, point_at(pts, stride, win)).z);
    }
    height[p] = h;
    if (!with_normals) return;
    const int u = int(p % W), v = int(p / W);
    float n[3] = {0.f, 0.f, 0.f};
    bool ok = false;
    if (u >= 1 && v >= 1)
        ok = normal_at(dirs, W, u, v, d0, key_depth(pixkey[p - W]), key_depth(pixkey[p - 1]), n);
    normals[3 * p] = ok ? n[0] : 0.f;
    normals[3 * p + 1] = ok ? n[1] : 0.f;
    normals[3 * p + 2] = ok ? n[2] : 0.f;
    valid[p] = ok ? 1 : 0;
}

__global__ void k_normals(const float* __restrict__ depth, const double* __restrict__ dirs, int W,
                          int H, float* __restrict__ normals, uint8_t* __restrict__ valid) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(W) * H) return;
    const int u = int(p % W), v = int(p / W);
    float n[3] = {0.f, 0.f, 0.f};
    bool ok = false;
    if (u >= 1 && v >= 1) ok = normal_at(dirs, W, u, v, depth[p], depth[p - W], depth[p - 1], n);
    normals[3 * p] = ok ? n[0] : 0.f;
    normals[3 * p + 1] = ok ? n[1] : 0.f;
    normals[3 * p + 2] = ok ? n[2] : 0.f;
    valid[p] = ok ? 1 : 0;
}

inline unsigned grid_for(uint64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

}  // namespace

// Gated on the abort word and double-buffered (no memsets), so a batch of
// frames can be queued without host synchronisation.
template <typename T>
void launch_project_t(svx_scan* s, const T* d_pts, uint64_t n, int stride, const Pose& pose) {
    svx_map* m = s->map;
    const uint32_t P = uint32_t(s->P);
    unsigned long long* cur = s->pixkey.p + uint64_t(s->parity) * P;
    unsigned long long* nxt = s->pixkey.p + uint64_t(s->parity ^ 1) * P;
    const uint32_t tie_cap = uint32_t(std::min<uint64_t>(2 * n + 2, 0xFFFFFFF0ull));
    s->lexkey.alloc(tie_cap);  // tie list: (pixel << 32) | point index
    ProfMark pm(m, SVX_K_PROJECT);
    m->prof_acc.points += n;
    if (n) {
        launch_pdl(k_project_points<T>, grid_for(n), kThreads, m->stream, d_pts, n, stride, s->dm, cur,
                   s->tie.p, s->lexkey.p, tie_cap, m->d_ctr);
        count_launch();
    }
    launch_pdl(k_finish_pixels<T>, grid_for(P), kThreads, m->stream, d_pts, stride, cur, nxt, s->dirs.p,
               pose, s->dm.W, s->dm.H, 1, s->depth.p, s->height.p, s->normals.p, s->valid.p, s->tie.p,
               s->lexkey.p, tie_cap, s->rowdist.p, s->validbits.p, m->d_ctr);
    count_launch();
    SVX_CUDA(cudaGetLastError());
    s->rowdist_fresh = true;
    s->parity ^= 1;
    s->has_normals = true;
    s->n_points = n;
}

void launch_project(svx_scan* s, const float* d_pts, uint64_t n, int stride, const Pose& pose) {
    launch_project_t(s, d_pts, n, stride, pose);
}
void launch_project(svx_scan* s, const double* d_pts, uint64_t n, int stride, const Pose& pose) {
    launch_project_t(s, d_pts, n, stride, pose);
}

void launch_normals(svx_scan* s) {
    svx_map* m = s->map;
    ProfMark pm(m, SVX_K_PROJECT);
    k_normals<<<grid_for(uint64_t(s->P)), kThreads, 0, m->stream>>>(
        s->depth.p, s->dirs.p, s->dm.W, s->dm.H, s->normals.p, s->valid.p);
    count_launch(1);
    SVX_CUDA(cudaGetLastError());
    s->has_normals = true;
}

}  // namespace svx
