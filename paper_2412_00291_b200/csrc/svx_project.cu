// K1/K2: project_cloud + compute_normal_image on the device.
//
// project_cloud (scan_projection.cpp:39-76) is a serial nearer-wins scatter with
// a lexicographic tie-break. Here it is order-independent by construction:
//   k_project_points  one thread per point: pixel (FP32 fast path, FP64 near
//                     boundaries), then atomicMin of (f32 range bits << 32 | index)
//                     on the pixel. A pixel where two equal ranges met is flagged.
//   k_tie_*           only for flagged pixels (gated on a device counter): the
//                     lexicographically smallest (x, y, z) among equal-range points
//                     wins, exactly as std::tie in the reference.
//   k_finish_pixels   one thread per pixel: depth, height = (pose * p).z of the
//                     winner, and (optionally) the normal of compute_normal_image
//                     (scan_projection.cpp:86-109) from the three neighbour depths,
//                     with back_project directions from a host-libm table (bit-exact).
#include "svx_map.hpp"

namespace svx {

namespace {

constexpr int kThreads = 256;

__device__ inline unsigned long long ord_key(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 and +0.0 compare equal in std::tie
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_project_points(const float* __restrict__ pts, uint64_t n, int stride, Model m,
                                 unsigned long long* __restrict__ pixkey,
                                 uint8_t* __restrict__ tie, uint32_t* __restrict__ pix_of_pt,
                                 uint32_t* __restrict__ ctr) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const d3 p = mk(pts[i * stride], pts[i * stride + 1], pts[i * stride + 2]);
    int u, v;
    double r;
    if (!project_point(p, m, u, v, r)) {
        pix_of_pt[i] = kInvalid;
        warp_agg_inc(&ctr[C_DROPPED]);
        return;
    }
    const uint32_t pix = uint32_t(v) * uint32_t(m.W) + uint32_t(u);
    pix_of_pt[i] = pix;
    const float rf = float(r);
    const unsigned long long key =
        (static_cast<unsigned long long>(__float_as_uint(rf)) << 32) | static_cast<uint32_t>(i);
    const unsigned long long old = atomicMin(&pixkey[pix], key);
    if (old != ~0ull && (old >> 32) == (key >> 32)) {
        if (tie[pix] == 0) {
            tie[pix] = 1;
            atomicAdd(&ctr[C_TIES], 1u);
        }
    }
}

// Tie resolution, pass `axis` (0 = x, 1 = y, 2 = z): among points of a flagged
// pixel whose range equals the minimum and whose earlier coordinates equal the
// running lexicographic minimum, take the minimum of this coordinate.
__global__ void k_tie_axis(const float* __restrict__ pts, uint64_t n, int stride,
                           const uint32_t* __restrict__ pix_of_pt,
                           const unsigned long long* __restrict__ pixkey,
                           const uint8_t* __restrict__ tie, unsigned long long* __restrict__ lex,
                           uint32_t P, int axis, const uint32_t* __restrict__ ctr) {
    if (ctr[C_TIES] == 0) return;
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t pix = pix_of_pt[i];
    if (pix == kInvalid || !tie[pix]) return;
    const double c[3] = {pts[i * stride], pts[i * stride + 1], pts[i * stride + 2]};
    const float rf = float(sqrt(dot3(mk(c[0], c[1], c[2]), mk(c[0], c[1], c[2]))));
    if (__float_as_uint(rf) != uint32_t(pixkey[pix] >> 32)) return;
    for (int a = 0; a < axis; ++a)
        if (ord_key(c[a]) != lex[uint64_t(a) * P + pix]) return;
    atomicMin(&lex[uint64_t(axis) * P + pix], ord_key(c[axis]));
}

__global__ void k_tie_reset(const uint8_t* __restrict__ tie, unsigned long long* __restrict__ lex,
                            uint32_t P, const uint32_t* __restrict__ ctr) {
    if (ctr[C_TIES] == 0) return;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !tie[p]) return;
    lex[p] = lex[uint64_t(P) + p] = lex[2ull * P + p] = ~0ull;
}

__global__ void k_tie_winner(const float* __restrict__ pts, uint64_t n, int stride,
                             const uint32_t* __restrict__ pix_of_pt,
                             unsigned long long* __restrict__ pixkey,
                             const uint8_t* __restrict__ tie,
                             const unsigned long long* __restrict__ lex, uint32_t P,
                             const uint32_t* __restrict__ ctr) {
    if (ctr[C_TIES] == 0) return;
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t pix = pix_of_pt[i];
    if (pix == kInvalid || !tie[pix]) return;
    const double c[3] = {pts[i * stride], pts[i * stride + 1], pts[i * stride + 2]};
    const unsigned long long cur = pixkey[pix];
    const float rf = float(sqrt(dot3(mk(c[0], c[1], c[2]), mk(c[0], c[1], c[2]))));
    if (__float_as_uint(rf) != uint32_t(cur >> 32)) return;
    for (int a = 0; a < 3; ++a)
        if (ord_key(c[a]) != lex[uint64_t(a) * P + pix]) return;
    // all winners have identical coordinates: any of them gives the same height
    pixkey[pix] = (cur & 0xFFFFFFFF00000000ull) | static_cast<uint32_t>(i);
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

__global__ void k_finish_pixels(const float* __restrict__ pts, int stride,
                                const unsigned long long* __restrict__ pixkey,
                                const double* __restrict__ dirs, Pose pose, int W, int H,
                                int with_normals, float* __restrict__ depth,
                                float* __restrict__ height, float* __restrict__ normals,
                                uint8_t* __restrict__ valid, uint8_t* __restrict__ tie) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= uint32_t(W) * H) return;
    const unsigned long long k = pixkey[p];
    const float d0 = key_depth(k);
    depth[p] = d0;
    float h = 0.f;
    if (k != ~0ull) {
        const uint32_t i = uint32_t(k);
        const d3 q = mk(pts[uint64_t(i) * stride], pts[uint64_t(i) * stride + 1],
                        pts[uint64_t(i) * stride + 2]);
        h = float(xform(pose, q).z);
    }
    height[p] = h;
    tie[p] = 0;
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

void launch_project(svx_scan* s, const float* d_pts, uint64_t n, int stride, const Pose& pose) {
    svx_map* m = s->map;
    const uint32_t P = uint32_t(s->P);
    s->pixkey.alloc(P);
    s->lexkey.alloc(3ull * P);
    s->tie.alloc(P);
    DevBuf<uint32_t>& pix_of_pt = s->pix_of_pt;
    pix_of_pt.alloc(n ? n : 1);
    ProfMark pm(m, SVX_K_PROJECT);
    m->prof_acc.points += n;
    SVX_CUDA(cudaMemsetAsync(s->pixkey.p, 0xFF, sizeof(unsigned long long) * P, m->stream));
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_TIES, 0, sizeof(uint32_t), m->stream));
    SVX_CUDA(cudaMemsetAsync(m->d_ctr + C_DROPPED, 0, sizeof(uint32_t), m->stream));
    if (n) {
        k_project_points<<<grid_for(n), kThreads, 0, m->stream>>>(d_pts, n, stride, s->dm,
                                                                    s->pixkey.p, s->tie.p,
                                                                    pix_of_pt.p, m->d_ctr);
        k_tie_reset<<<grid_for(P), kThreads, 0, m->stream>>>(s->tie.p, s->lexkey.p, P, m->d_ctr);
        for (int axis = 0; axis < 3; ++axis)
            k_tie_axis<<<grid_for(n), kThreads, 0, m->stream>>>(d_pts, n, stride, pix_of_pt.p,
                                                                  s->pixkey.p, s->tie.p,
                                                                  s->lexkey.p, P, axis, m->d_ctr);
        k_tie_winner<<<grid_for(n), kThreads, 0, m->stream>>>(d_pts, n, stride, pix_of_pt.p,
                                                                s->pixkey.p, s->tie.p,
                                                                s->lexkey.p, P, m->d_ctr);
        count_launch(6);
    }
    k_finish_pixels<<<grid_for(P), kThreads, 0, m->stream>>>(
        d_pts, stride, s->pixkey.p, s->dirs.p, pose, s->dm.W, s->dm.H, 1, s->depth.p,
        s->height.p, s->normals.p, s->valid.p, s->tie.p);
    count_launch(1);
    SVX_CUDA(cudaGetLastError());
    s->has_normals = true;
    s->n_points = n;
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
