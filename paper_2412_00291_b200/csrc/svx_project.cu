// K1/K2: project_cloud + compute_normal_image on the device, for a GROUP of frames at
// once (frame g of the group -> scan slot g; svx_tsdf.cu integrates the group).
//
// project_cloud (scan_projection.cpp:39-76) is a serial nearer-wins scatter with a
// lexicographic tie-break. Here it is order-independent by construction, in two kernels
// per group:
//   k_project_points  one thread per point of any frame of the group: pixel (FP32
//                     polynomial atan2 with an error margin, FP64 reference formula near a
//                     boundary), then atomicMin of (f32 range bits << 32 | point index) on
//                     the frame's pixel. When two equal ranges meet, both points are
//                     appended to the frame's tie list and the pixel is flagged (every
//                     point with the pixel's final range ends up in the list).
//   k_finish_pixels   one thread per (frame, pixel): flagged pixels pick the
//                     lexicographically smallest (x, y, z) among their equal-range points
//                     (std::tie in the reference); depth, height = (pose * p).z of the
//                     winner, and the normal of compute_normal_image (scan_projection.cpp:
//                     86-109) from the three neighbour depths, with back_project directions
//                     from a host-libm table (bit-exact); the row-distance map and valid
//                     bits of the band kernel. It also resets the other half of the
//                     double-buffered pixel keys for the slot's next projection.
#include <algorithm>

#include "svx_map.hpp"

namespace svx {

namespace {

constexpr int kThreads = 256;

// A group's projection inputs and per-slot outputs (frame g of an image array at g * P).
struct ProjGroup {
    const void* pts[kMaxG];              // float or double, `stride` components per point
    uint64_t n[kMaxG];
    uint32_t cta0[kMaxG + 1];            // CTA prefix of k_project_points over the frames
    Pose pose[kMaxG];
    unsigned long long* cur[kMaxG];      // pixel keys the frame projects into
    unsigned long long* nxt[kMaxG];      // the slot's other half, cleared for its next use
    Model m;
    int stride, G;
    uint32_t P, VW, cpf;                 // pixels, valid-bit words, k_finish CTAs per frame
    uint64_t tie_cap;                    // tie-list entries per slot
    float* depth;
    float* height;
    float* normals;
    uint8_t* valid;
    uint8_t* tie;
    unsigned long long* ties;
    uint8_t* rowdist;
    uint32_t* validbits;
    const double* dirs;
};

__device__ inline bool lex_less(d3 a, d3 b) {
    if (a.x < b.x) return true;
    if (b.x < a.x) return false;
    if (a.y < b.y) return true;
    if (b.y < a.y) return false;
    return a.z < b.z;
}

template <typename T>
__device__ inline d3 point_at(const T* __restrict__ pts, int stride, uint32_t i) {
    return mk(pts[uint64_t(i) * stride], pts[uint64_t(i) * stride + 1], pts[uint64_t(i) * stride + 2]);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_project_points(const __grid_constant__ ProjGroup pg, uint32_t* __restrict__ fctr, uint32_t* __restrict__ ctr) {
    // The point loads and the pixel computation read only this group's input (never
    // written by the frame kernels before it), so they run before the dependency wait
    // and overlap the previous group's last kernels; every write comes after it.
    uint32_t g = 0;
    while (g + 1 < uint32_t(pg.G) && pg.cta0[g + 1] <= blockIdx.x) ++g;
    const uint64_t i = uint64_t(blockIdx.x - pg.cta0[g]) * blockDim.x + threadIdx.x;
    const uint64_t n = pg.n[g];
    const T* pts = static_cast<const T*>(pg.pts[g]);
    double r = 0.0;
    uint32_t pix = kInvalid;
    if (i < n) {
        const d3 p = point_at(pts, pg.stride, uint32_t(i));
        r = sqrt(dot3(p, p));
        if (isfinite(r) && !(r < pg.m.min_range)) {
            pix = pixel_fast(float(p.x), float(p.y), float(p.z), pg.m, pg.m.r2_lo, pg.m.r2_hi);
            if (pix == kNeedFp64) pix = pixel_fp64(p, pg.m);
        }
    }
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    if (i >= n) return;
    if (pix == kInvalid) {
        warp_agg_inc(&fctr[g * kFC + FC_DROPPED]);
        return;
    }
    const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(float(r))) << 32) | uint32_t(i);
    const unsigned long long old = atomicMin(&pg.cur[g][pix], key);
    if (old != ~0ull && (old >> 32) == (key >> 32)) {
        pg.tie[uint64_t(g) * pg.P + pix] = 1;
        const uint32_t pos = atomicAdd(&fctr[g * kFC + FC_TIES], 2u);
        unsigned long long* ties = pg.ties + uint64_t(g) * pg.tie_cap;
        if (pos + 1 < pg.tie_cap) {
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
__device__ inline bool normal_at(const double* __restrict__ dirs, int W, int u, int v, float d0, float d1, float d2,
                                 float out[3]) {
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
__global__ void __launch_bounds__(kThreads)
k_finish_pixels(const __grid_constant__ ProjGroup pg, const uint32_t* __restrict__ fctr,
                const uint32_t* __restrict__ ctr) {
    pdl_wait();
    pdl_trigger();
    if (ctr[C_ABORT]) return;
    const uint32_t g = blockIdx.x / pg.cpf;
    const uint32_t p = (blockIdx.x - g * pg.cpf) * blockDim.x + threadIdx.x;
    const int W = pg.m.W;
    const bool inside = p < pg.P;
    const unsigned long long* pixkey = pg.cur[g];
    const unsigned long long k = inside ? pixkey[p] : ~0ull;
    const uint64_t o = uint64_t(g) * pg.P;
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, k != ~0ull);  // pixels with a return
    if ((threadIdx.x & 31) == 0 && inside) pg.validbits[uint64_t(g) * pg.VW + (p >> 5)] = bits;
    // row distance to the nearest pixel without a return (band kernel's valid radius), capped
    // at kRowDistMax + 1, the row wrapping around (azimuth): when a row is whole 32-pixel
    // words, from the no-return bits of this word and its two neighbours in the row
    int rd = -1;
    if (W % 32 == 0) {
        const int lane = int(threadIdx.x & 31);
        const uint32_t wpr = uint32_t(W) / 32u, word = (p / 32u) % wpr, row0 = p - (p % uint32_t(W));
        const uint32_t wp = row0 + ((word + wpr - 1u) % wpr) * 32u + uint32_t(lane);
        const uint32_t wn = row0 + ((word + 1u) % wpr) * 32u + uint32_t(lane);
        const unsigned long long kp = inside ? pixkey[wp] : 0ull, kn = inside ? pixkey[wn] : 0ull;
        const uint32_t ip = ~__ballot_sync(0xFFFFFFFFu, kp != ~0ull), is = ~bits,
                       in = ~__ballot_sync(0xFFFFFFFFu, kn != ~0ull);
        const unsigned long long right = (uint64_t(is) >> lane) | (uint64_t(in) << (32 - lane));
        const unsigned long long left = ((uint64_t(is) << 32) | ip) & ((2ull << (32 + lane)) - 1ull);
        const int dr = right ? __ffsll(static_cast<long long>(right)) - 1 : 64;
        const int dl = left ? (32 + lane) - (63 - __clzll(static_cast<long long>(left))) : 64;
        rd = min(min(dr, dl), kRowDistMax + 1);
    }
    if (!inside) return;
    pg.nxt[g][p] = ~0ull;  // the other half is clean for the slot's next projection
    const float d0 = key_depth(k);
    pg.depth[o + p] = d0;
    if (rd >= 0) {
        pg.rowdist[o + p] = uint8_t(rd);
    } else {
        const int u = int(p % W);
        const unsigned long long* row = pixkey + (p - u);
        int d = 0;
        for (; d <= kRowDistMax; ++d) {
            int a = u + d, b = u - d;
            a -= a >= W ? W : 0;
            b += b < 0 ? W : 0;
            if (row[a] == ~0ull || row[b] == ~0ull) break;
        }
        pg.rowdist[o + p] = uint8_t(d);
    }
    float h = 0.f;
    if (k != ~0ull) {
        const T* pts = static_cast<const T*>(pg.pts[g]);
        uint32_t win = uint32_t(k);
        if (pg.tie[o + p]) {
            // lexicographic minimum among the points of this pixel with its range
            d3 best = point_at(pts, pg.stride, win);
            const unsigned long long* ties = pg.ties + uint64_t(g) * pg.tie_cap;
            const uint64_t nties = fctr[g * kFC + FC_TIES];
            const uint32_t nt = uint32_t(nties < pg.tie_cap ? nties : pg.tie_cap);
            for (uint32_t t = 0; t < nt; ++t) {
                const unsigned long long e = ties[t];
                if (uint32_t(e >> 32) != p) continue;
                const uint32_t i = uint32_t(e);
                const d3 q = point_at(pts, pg.stride, i);
                if (__float_as_uint(float(sqrt(dot3(q, q)))) != uint32_t(k >> 32)) continue;
                if (lex_less(q, best)) {
                    best = q;
                    win = i;
                }
            }
            pg.tie[o + p] = 0;
        }
        h = float(xform(pg.pose[g], point_at(pts, pg.stride, win)).z);
    }
    pg.height[o + p] = h;
    const int u = int(p % W), v = int(p / W);
    float nn[3] = {0.f, 0.f, 0.f};
    bool ok = false;
    if (u >= 1 && v >= 1) ok = normal_at(pg.dirs, W, u, v, d0, key_depth(pixkey[p - W]), key_depth(pixkey[p - 1]), nn);
    pg.normals[3 * (o + p)] = ok ? nn[0] : 0.f;
    pg.normals[3 * (o + p) + 1] = ok ? nn[1] : 0.f;
    pg.normals[3 * (o + p) + 2] = ok ? nn[2] : 0.f;
    pg.valid[o + p] = ok ? 1 : 0;
}

__global__ void k_normals(const float* __restrict__ depth, const double* __restrict__ dirs, int W, int H,
                          float* __restrict__ normals, uint8_t* __restrict__ valid) {
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

void ensure_scan_slots(svx_scan* s, int G, uint64_t max_points) {
    svx_map* m = s->map;
    const uint64_t P = uint64_t(s->P);
    const uint64_t tie_cap = std::min<uint64_t>(2 * max_points + 2, 0xFFFFFFF0ull);
    if (G > s->slots) {
        // (re)allocate every slot array; slots hold no state between batches except
        // slot 0's images, which a growth only happens ahead of a projection to overwrite
        SVX_CUDA(cudaStreamSynchronize(m->stream));
        const uint64_t GP = uint64_t(G) * P;
        s->depth.release();
        s->height.release();
        s->normals.release();
        s->valid.release();
        s->tie.release();
        s->pixkey.release();
        s->pixcache.release();
        s->rowdist.release();
        s->validbits.release();
        s->depth.alloc(GP);
        s->height.alloc(GP);
        s->normals.alloc(3 * GP);
        s->valid.alloc(GP);
        s->tie.alloc(GP);
        s->pixkey.alloc(2 * GP);
        s->pixcache.alloc(48 * GP);
        s->rowdist.alloc(GP);
        s->validbits.alloc(uint64_t(G) * s->VW);
        SVX_CUDA(cudaMemset(s->depth.p, 0, 4 * GP));
        SVX_CUDA(cudaMemset(s->height.p, 0, 4 * GP));
        SVX_CUDA(cudaMemset(s->normals.p, 0, 12 * GP));
        SVX_CUDA(cudaMemset(s->valid.p, 0, GP));
        SVX_CUDA(cudaMemset(s->tie.p, 0, GP));
        SVX_CUDA(cudaMemset(s->pixkey.p, 0xFF, 16 * GP));
        SVX_CUDA(cudaMemset(s->pixcache.p, 0, 48 * GP));
        SVX_CUDA(cudaMemset(s->rowdist.p, 0, GP));
        SVX_CUDA(cudaMemset(s->validbits.p, 0, 4ull * G * s->VW));
        for (int g = 0; g < kMaxG; ++g) s->parity[g] = 0;
        s->slots = G;
        s->rowdist_fresh = false;
    }
    s->tie_cap = std::max(tie_cap, s->tie_cap);
    if (uint64_t(s->slots) * s->tie_cap > s->lexkey.n) s->lexkey.alloc(uint64_t(s->slots) * s->tie_cap);
}

// Gated on the abort word and double-buffered per slot (no memsets), so the groups of a
// batch can be queued without host synchronisation.
void launch_project_group(svx_scan* s, const void* const* d_pts, const uint64_t* n, int G, int stride, bool fp64,
                          const Pose* poses) {
    svx_map* m = s->map;
    uint64_t nmax = 0;
    for (int g = 0; g < G; ++g) nmax = std::max(nmax, n[g]);
    ensure_scan_slots(s, G, nmax);
    ProjGroup pg{};
    const uint32_t P = uint32_t(s->P);
    pg.m = s->dm;
    pg.stride = stride;
    pg.G = G;
    pg.P = P;
    pg.VW = uint32_t(s->VW);
    pg.cpf = grid_for(P);
    pg.tie_cap = s->tie_cap;
    pg.depth = s->depth.p;
    pg.height = s->height.p;
    pg.normals = s->normals.p;
    pg.valid = s->valid.p;
    pg.tie = s->tie.p;
    pg.ties = s->lexkey.p;
    pg.rowdist = s->rowdist.p;
    pg.validbits = s->validbits.p;
    pg.dirs = s->dirs.p;
    uint32_t ctas = 0;
    for (int g = 0; g < G; ++g) {
        pg.pts[g] = d_pts[g];
        pg.n[g] = n[g];
        pg.cta0[g] = ctas;
        ctas += grid_for(n[g]);
        pg.pose[g] = poses[g];
        pg.cur[g] = s->pixkey.p + (2 * uint64_t(g) + uint64_t(s->parity[g])) * P;
        pg.nxt[g] = s->pixkey.p + (2 * uint64_t(g) + uint64_t(s->parity[g] ^ 1)) * P;
        s->parity[g] ^= 1;
        m->prof_acc.points += n[g];
    }
    pg.cta0[G] = ctas;
    ProfMark pm(m, SVX_K_PROJECT);
    if (ctas) {
        if (fp64) launch_pdl(k_project_points<double>, ctas, kThreads, m->stream, pg, m->fctr, m->d_ctr);
        else launch_pdl(k_project_points<float>, ctas, kThreads, m->stream, pg, m->fctr, m->d_ctr);
        count_launch();
    }
    if (fp64) launch_pdl(k_finish_pixels<double>, pg.cpf * G, kThreads, m->stream, pg, m->fctr, m->d_ctr);
    else launch_pdl(k_finish_pixels<float>, pg.cpf * G, kThreads, m->stream, pg, m->fctr, m->d_ctr);
    count_launch();
    SVX_CUDA(cudaGetLastError());
    s->rowdist_fresh = true;
    s->has_normals = true;
    s->last_slot = G - 1;
    s->n_points = n[G - 1];
}

void launch_project(svx_scan* s, const float* d_pts, uint64_t n, int stride, const Pose& pose) {
    const void* p = d_pts;
    launch_project_group(s, &p, &n, 1, stride, false, &pose);
}
void launch_project(svx_scan* s, const double* d_pts, uint64_t n, int stride, const Pose& pose) {
    const void* p = d_pts;
    launch_project_group(s, &p, &n, 1, stride, true, &pose);
}

void launch_normals(svx_scan* s) {
    svx_map* m = s->map;
    ProfMark pm(m, SVX_K_PROJECT);
    const uint64_t o = uint64_t(s->last_slot) * s->P;
    k_normals<<<grid_for(uint64_t(s->P)), kThreads, 0, m->stream>>>(s->depth.p + o, s->dirs.p, s->dm.W, s->dm.H,
                                                                      s->normals.p + 3 * o, s->valid.p + o);
    count_launch(1);
    SVX_CUDA(cudaGetLastError());
    s->has_normals = true;
}

}  // namespace svx
