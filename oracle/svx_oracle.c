/*
 * TEST INFRASTRUCTURE ONLY — see svx_oracle.h. A serial plain-C restatement of
 * the reference hot path. Compiled with -ffp-contract=off (no FMA), matching the
 * reference's Release flags. Vector helpers reproduce Eigen's evaluation order:
 * 3-term reductions are (a0*b0 + a1*b1) + a2*b2, Isometry*p = t + R p,
 * normalized() divides by sqrt(squaredNorm).
 */
#define _GNU_SOURCE
#include "svx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KB 8
#define KV 512
static const double kPi = 3.14159265358979323846;

static __thread char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* svxo_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- vectors */
typedef struct { double v[3]; } d3;
typedef struct { float v[3]; } f3;

static double dot3(d3 a, d3 b) { return (a.v[0] * b.v[0] + a.v[1] * b.v[1]) + a.v[2] * b.v[2]; }
static double norm3(d3 a) { return sqrt(dot3(a, a)); }
static d3 sub3(d3 a, d3 b) { d3 r = {{a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]}}; return r; }
static d3 add3(d3 a, d3 b) { d3 r = {{a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]}}; return r; }
static d3 scale3(double s, d3 a) { d3 r = {{s * a.v[0], s * a.v[1], s * a.v[2]}}; return r; }
static d3 div3(d3 a, double s) { d3 r = {{a.v[0] / s, a.v[1] / s, a.v[2] / s}}; return r; }
static d3 normalized3(d3 a) {
    const double z = dot3(a, a);
    return z > 0.0 ? div3(a, sqrt(z)) : a;
}
/* R p, row-major R, Eigen coefficient order */
static d3 matvec(const double* R, d3 p) {
    d3 r;
    for (int i = 0; i < 3; ++i)
        r.v[i] = (R[3 * i + 0] * p.v[0] + R[3 * i + 1] * p.v[1]) + R[3 * i + 2] * p.v[2];
    return r;
}
/* Isometry * p = t + (R p)  (Eigen transform_right_product_impl) */
static d3 xform(const svx_pose* T, d3 p) {
    const d3 rp = matvec(T->R, p);
    d3 r = {{T->t[0] + rp.v[0], T->t[1] + rp.v[1], T->t[2] + rp.v[2]}};
    return r;
}
/* Isometry::inverse(): (R^T, (-R^T) t) */
static svx_pose inverse_pose(const svx_pose* T) {
    svx_pose inv;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) inv.R[3 * i + j] = T->R[3 * j + i];
    double negRt[9];
    for (int k = 0; k < 9; ++k) negRt[k] = -inv.R[k];
    d3 t = {{T->t[0], T->t[1], T->t[2]}};
    const d3 ti = matvec(negRt, t);
    for (int i = 0; i < 3; ++i) inv.t[i] = ti.v[i];
    return inv;
}
static d3 origin_of(const svx_pose* T) { d3 o = {{T->t[0], T->t[1], T->t[2]}}; return o; }

/* ------------------------------------------------------------- keys (types.hpp) */
static int32_t floor_div(int32_t a, int32_t b) { /* types.hpp:35-39 */
    int32_t q = a / b, r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}
static int32_t nonneg_mod(int32_t a, int32_t b) { /* types.hpp:41-44 */
    int32_t r = a % b;
    return r < 0 ? r + b : r;
}
static void world_to_voxel(d3 p, float voxel_size, int32_t out[3]) { /* types.hpp:168-173 */
    const double inv = 1.0 / (double)voxel_size;
    for (int i = 0; i < 3; ++i) out[i] = (int32_t)floor(p.v[i] * inv + 0.5);
}
static d3 voxel_center(const int32_t v[3], float voxel_size) { /* types.hpp:175-178 */
    const double s = (double)voxel_size;
    d3 c = {{s * v[0], s * v[1], s * v[2]}};
    return c;
}

/* --------------------------------------------------------------- block store */
typedef struct {
    int32_t key[3];
    svx_tsdf_voxel tsdf[KV];
    float* sem; /* NULL until ensure_semantics */
} oblock;

struct svxo_map {
    svx_map_cfg cfg;
    oblock** blocks;
    uint64_t n, cap;
    int64_t* table; /* open addressing, -1 empty, value = index into blocks */
    uint64_t tcap;
    int tsdf_frames, sem_frames;
    int32_t* dirty[2];
    uint64_t ndirty[2], capdirty[2];
    /* last extract_mesh result (svxo_mesh_extract) */
    float *mesh_v, *mesh_n;
    uint8_t* mesh_l;
    uint32_t* mesh_f;
    uint64_t mesh_nv, mesh_nf;
};

static uint64_t hkey(const int32_t k[3]) {
    uint64_t h = (uint64_t)(uint32_t)k[0] * 0x9E3779B97F4A7C15ULL;
    h ^= (uint64_t)(uint32_t)k[1] * 0xC2B2AE3D27D4EB4FULL;
    h ^= (uint64_t)(uint32_t)k[2] * 0x165667B19E3779F9ULL;
    return h ^ (h >> 29);
}
static int64_t find_idx(const svxo_map* m, const int32_t k[3]) {
    uint64_t s = hkey(k) & (m->tcap - 1);
    for (;;) {
        const int64_t i = m->table[s];
        if (i < 0) return -1;
        const oblock* b = m->blocks[i];
        if (b->key[0] == k[0] && b->key[1] == k[1] && b->key[2] == k[2]) return i;
        s = (s + 1) & (m->tcap - 1);
    }
}
static void table_insert(svxo_map* m, int64_t idx) {
    uint64_t s = hkey(m->blocks[idx]->key) & (m->tcap - 1);
    while (m->table[s] >= 0) s = (s + 1) & (m->tcap - 1);
    m->table[s] = idx;
}
static void grow_table(svxo_map* m) {
    free(m->table);
    m->tcap *= 2;
    m->table = malloc(m->tcap * sizeof(int64_t));
    memset(m->table, 0xFF, m->tcap * sizeof(int64_t));
    for (uint64_t i = 0; i < m->n; ++i) table_insert(m, (int64_t)i);
}

svxo_map* svxo_map_create(const svx_map_cfg* cfg, int* status) {
    /* MapConfig::validate (types.hpp:103-111) */
    int st = 0;
    if (!(cfg->voxel_size > 0.f)) st = fail(1, "voxel_size must be > 0");
    else if (!(cfg->truncation > 0.f)) st = fail(1, "truncation must be > 0");
    else if (cfg->truncation < cfg->voxel_size) st = fail(1, "truncation must be >= voxel_size");
    else if (cfg->num_labels < 1 || cfg->num_labels > 64) st = fail(1, "num_labels must be in [1, 64]");
    else if (cfg->max_blocks == 0) st = fail(1, "max_blocks must be > 0");
    if (status) *status = st;
    if (st) return NULL;
    svxo_map* m = calloc(1, sizeof *m);
    m->cfg = *cfg;
    m->tcap = 1024;
    m->table = malloc(m->tcap * sizeof(int64_t));
    memset(m->table, 0xFF, m->tcap * sizeof(int64_t));
    return m;
}

void svxo_map_destroy(svxo_map* m) {
    if (!m) return;
    for (uint64_t i = 0; i < m->n; ++i) {
        free(m->blocks[i]->sem);
        free(m->blocks[i]);
    }
    free(m->blocks);
    free(m->table);
    free(m->dirty[0]);
    free(m->dirty[1]);
    free(m->mesh_v);
    free(m->mesh_n);
    free(m->mesh_l);
    free(m->mesh_f);
    free(m);
}

/* VoxelStore::get_or_allocate_block (voxel_store.cpp:9-23): -1 on capacity. */
static int64_t get_or_alloc(svxo_map* m, const int32_t k[3], int* was_new) {
    int64_t i = find_idx(m, k);
    if (was_new) *was_new = 0;
    if (i >= 0) return i;
    if (m->n >= m->cfg.max_blocks) return -1;
    if (m->n == m->cap) {
        m->cap = m->cap ? 2 * m->cap : 256;
        m->blocks = realloc(m->blocks, m->cap * sizeof(oblock*));
    }
    oblock* b = calloc(1, sizeof *b);
    memcpy(b->key, k, sizeof b->key);
    m->blocks[m->n] = b;
    i = (int64_t)m->n++;
    if (2 * m->n > m->tcap) grow_table(m);
    else table_insert(m, i);
    if (was_new) *was_new = 1;
    return i;
}

int svxo_get_or_allocate_block(svxo_map* m, const int32_t bxyz[3]) {
    return get_or_alloc(m, bxyz, NULL) < 0 ? fail(2, "block budget exhausted") : 0;
}
uint64_t svxo_block_count(const svxo_map* m) { return m->n; }

static void ensure_semantics(svxo_map* m, oblock* b) { /* voxel_store.hpp:26-30 */
    if (b->sem) return;
    const int K = m->cfg.num_labels;
    b->sem = malloc((size_t)KV * K * sizeof(float));
    const float u = 1.f / (float)K;
    for (int i = 0; i < KV * K; ++i) b->sem[i] = u;
}

int svxo_block_write(svxo_map* m, const int32_t bxyz[3], const svx_tsdf_voxel* tsdf,
                     const float* sem, int32_t has_sem) {
    const int64_t i = get_or_alloc(m, bxyz, NULL);
    if (i < 0) return fail(2, "block budget exhausted");
    oblock* b = m->blocks[i];
    if (tsdf) memcpy(b->tsdf, tsdf, sizeof b->tsdf);
    if (has_sem) {
        ensure_semantics(m, b);
        if (sem) memcpy(b->sem, sem, (size_t)KV * m->cfg.num_labels * sizeof(float));
    }
    return 0;
}

static int local_index(const int32_t v[3]) { /* types.hpp:86-89 */
    return nonneg_mod(v[0], KB) + KB * nonneg_mod(v[1], KB) + KB * KB * nonneg_mod(v[2], KB);
}
static void block_of(const int32_t v[3], int32_t b[3]) { /* types.hpp:81-83 */
    for (int i = 0; i < 3; ++i) b[i] = floor_div(v[i], KB);
}
static void voxel_at(const int32_t b[3], int linear, int32_t v[3]) { /* types.hpp:91-95 */
    v[0] = b[0] * KB + linear % KB;
    v[1] = b[1] * KB + (linear / KB) % KB;
    v[2] = b[2] * KB + linear / (KB * KB);
}

int svxo_lookup(const svxo_map* m, const int32_t v[3], svx_tsdf_voxel* out, float* probs) {
    int32_t b[3];
    block_of(v, b);
    const int64_t i = find_idx(m, b);
    if (i < 0) return 0;
    const oblock* blk = m->blocks[i];
    const int li = local_index(v);
    if (out) *out = blk->tsdf[li];
    if (probs) {
        const int K = m->cfg.num_labels;
        for (int k = 0; k < K; ++k)
            probs[k] = blk->sem ? blk->sem[(size_t)li * K + k] : 1.f / (float)K;
    }
    return 1;
}

uint64_t svxo_observed(const svxo_map* m) {
    uint64_t c = 0;
    for (uint64_t i = 0; i < m->n; ++i)
        for (int j = 0; j < KV; ++j) c += m->blocks[i]->tsdf[j].weight > 0.f;
    return c;
}

static int key_cmp(const int32_t* a, const int32_t* b) {
    for (int i = 0; i < 3; ++i)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
static int cmp_blockptr(const void* a, const void* b) {
    return key_cmp((*(oblock* const*)a)->key, (*(oblock* const*)b)->key);
}
static int cmp_key3(const void* a, const void* b) { return key_cmp(a, b); }

static void push_dirty(svxo_map* m, int which, const int32_t k[3]) {
    if (m->ndirty[which] == m->capdirty[which]) {
        m->capdirty[which] = m->capdirty[which] ? 2 * m->capdirty[which] : 1024;
        m->dirty[which] = realloc(m->dirty[which], m->capdirty[which] * 3 * sizeof(int32_t));
    }
    memcpy(m->dirty[which] + 3 * m->ndirty[which]++, k, 3 * sizeof(int32_t));
}

uint64_t svxo_take_dirty(svxo_map* m, int32_t which, int32_t* out, uint64_t cap) {
    int32_t* d = m->dirty[which];
    uint64_t n = m->ndirty[which];
    qsort(d, n, 3 * sizeof(int32_t), cmp_key3);
    uint64_t u = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (u == 0 || key_cmp(d + 3 * (u - 1), d + 3 * i) != 0) memmove(d + 3 * u++, d + 3 * i, 12);
    if (out) memcpy(out, d, (u < cap ? u : cap) * 12);
    m->ndirty[which] = 0;
    return u;
}

/* SVOX1 (voxel_store.cpp:101-130) */
uint64_t svxo_save_mem(svxo_map* m, uint8_t* buf, uint64_t cap) {
    const int K = m->cfg.num_labels;
    uint64_t size = 5 + 4 + 4 + 4 + 8;
    for (uint64_t i = 0; i < m->n; ++i)
        size += 12 + sizeof(svx_tsdf_voxel) * KV + 1 + (m->blocks[i]->sem ? (uint64_t)KV * K * 4 : 0);
    if (!buf) return size;
    if (cap < size) return 0;
    oblock** sorted = malloc((m->n ? m->n : 1) * sizeof(oblock*));
    memcpy(sorted, m->blocks, m->n * sizeof(oblock*));
    qsort(sorted, m->n, sizeof(oblock*), cmp_blockptr);
    uint8_t* p = buf;
#define PUT(x) do { memcpy(p, &(x), sizeof(x)); p += sizeof(x); } while (0)
    memcpy(p, "SVOX1", 5);
    p += 5;
    PUT(m->cfg.voxel_size);
    PUT(m->cfg.truncation);
    const uint32_t k32 = (uint32_t)K;
    PUT(k32);
    const uint64_t nb = m->n;
    PUT(nb);
    for (uint64_t i = 0; i < m->n; ++i) {
        const oblock* b = sorted[i];
        memcpy(p, b->key, 12);
        p += 12;
        memcpy(p, b->tsdf, sizeof b->tsdf);
        p += sizeof b->tsdf;
        const uint8_t hs = b->sem ? 1 : 0;
        PUT(hs);
        if (hs) {
            memcpy(p, b->sem, (size_t)KV * K * 4);
            p += (size_t)KV * K * 4;
        }
    }
#undef PUT
    free(sorted);
    return size;
}

/* -------------------------------------------------------- projection (a2-a5) */
/* project_point (scan_projection.cpp:21-37) */
static int project_point(d3 p, const svx_lidar_model* m, int* u, int* v, double* range) {
    *range = norm3(p);
    if (!isfinite(*range) || *range < m->min_range) return 0;
    const double az = atan2(p.v[1], p.v[0]);
    int ui = (int)floor((kPi - az) / m->delta_phi);
    ui %= m->width;
    if (ui < 0) ui += m->width;
    double c = p.v[2] / *range;
    c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    const double polar = acos(c);
    const int vi = (int)floor((polar - m->theta0) / m->delta_theta);
    if (vi < 0 || vi >= m->height_px) return 0;
    *u = ui;
    *v = vi;
    return 1;
}

/* back_project (scan_projection.cpp:78-84): depth * (sp cos az, sp sin az, cos polar) */
static d3 back_project(int u, int v, double depth, const svx_lidar_model* m) {
    const double az = kPi - (u + 0.5) * m->delta_phi;
    const double polar = m->theta0 + (v + 0.5) * m->delta_theta;
    const double sp = sin(polar);
    d3 dir = {{sp * cos(az), sp * sin(az), cos(polar)}};
    return scale3(depth, dir);
}

static int validate_model(const svx_lidar_model* m) { /* scan_projection.hpp:26-33 */
    if (m->width <= 0 || m->height_px <= 0) return fail(1, "projection model: empty image");
    if (fabs(m->width * m->delta_phi - 2.0 * kPi) > 1e-6)
        return fail(1, "projection model: width * delta_phi must equal 2*pi");
    if (!(m->delta_theta > 0.0)) return fail(1, "projection model: delta_theta must be > 0");
    return 0;
}
static int validate_pose(const svx_pose* T) { /* scan_projection.hpp:65-69 */
    double mx = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            /* (R^T R)_ij = (R0i R0j + R1i R1j) + R2i R2j */
            const double rr = (T->R[0 + i] * T->R[0 + j] + T->R[3 + i] * T->R[3 + j]) +
                              T->R[6 + i] * T->R[6 + j];
            const double e = fabs(rr - (i == j ? 1.0 : 0.0));
            if (e > mx) mx = e;
        }
    return mx > 1e-6 ? fail(1, "pose rotation is not orthonormal") : 0;
}

static int lex_less(d3 a, d3 b) {
    for (int i = 0; i < 3; ++i) {
        if (a.v[i] < b.v[i]) return 1;
        if (b.v[i] < a.v[i]) return 0;
    }
    return 0;
}

/* project_cloud (scan_projection.cpp:39-76) */
int svxo_project(const svx_lidar_model* model, const float* pts, uint64_t n, int32_t stride,
                 const svx_pose* pose, float* depth, float* height, uint64_t* dropped) {
    int st = validate_model(model);
    if (st) return st;
    if ((st = validate_pose(pose))) return st;
    const size_t P = (size_t)model->width * model->height_px;
    memset(depth, 0, P * sizeof(float));
    memset(height, 0, P * sizeof(float));
    d3* kept = calloc(P, sizeof(d3));
    uint64_t drop = 0;
    for (uint64_t k = 0; k < n; ++k) {
        d3 p = {{pts[k * stride], pts[k * stride + 1], pts[k * stride + 2]}};
        int u, v;
        double r;
        if (!project_point(p, model, &u, &v, &r)) {
            ++drop;
            continue;
        }
        const size_t i = (size_t)v * model->width + u;
        const float rf = (float)r;
        int take = depth[i] == 0.f || rf < depth[i];
        if (!take && rf == depth[i]) take = lex_less(p, kept[i]);
        if (take) {
            depth[i] = rf;
            height[i] = (float)xform(pose, p).v[2];
            kept[i] = p;
        }
    }
    free(kept);
    if (dropped) *dropped = drop;
    return 0;
}

static d3 cross3(d3 a, d3 b) {
    d3 r = {{a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
             a.v[0] * b.v[1] - a.v[1] * b.v[0]}};
    return r;
}

/* compute_normal_image (scan_projection.cpp:86-109) */
int svxo_normals(const svx_lidar_model* m, const float* depth, float* normals, uint8_t* valid) {
    const int W = m->width, H = m->height_px;
    memset(normals, 0, (size_t)W * H * 3 * sizeof(float));
    memset(valid, 0, (size_t)W * H);
    for (int v = 1; v < H; ++v)
        for (int u = 1; u < W; ++u) {
            const float d0 = depth[(size_t)v * W + u];
            const float d1 = depth[(size_t)(v - 1) * W + u];
            const float d2 = depth[(size_t)v * W + u - 1];
            if (d0 == 0.f || d1 == 0.f || d2 == 0.f) continue;
            const d3 p = back_project(u, v, d0, m);
            const d3 p1 = back_project(u, v - 1, d1, m);
            const d3 p2 = back_project(u - 1, v, d2, m);
            d3 cr = cross3(sub3(p1, p), sub3(p2, p));
            const double nrm = norm3(cr);
            if (nrm < 1e-8) continue;
            cr = div3(cr, nrm);
            const d3 mp = {{-p.v[0], -p.v[1], -p.v[2]}};
            if (dot3(cr, mp) < 0.0) cr = scale3(-1.0, cr);
            const size_t i = (size_t)v * W + u;
            for (int c = 0; c < 3; ++c) normals[3 * i + c] = (float)cr.v[c];
            valid[i] = 1;
        }
    return 0;
}

/* ------------------------------------------------------- TSDF (a9-a13) */
typedef struct {
    int32_t b[3];
    uint16_t linear;
    uint32_t pix;
} visit;

typedef struct {
    visit* v;
    size_t n, cap;
} visit_vec;

static void push_visit(visit_vec* vv, const int32_t vc[3], uint32_t pix) {
    if (vv->n == vv->cap) {
        vv->cap = vv->cap ? 2 * vv->cap : 1 << 16;
        vv->v = realloc(vv->v, vv->cap * sizeof(visit));
    }
    visit* r = &vv->v[vv->n++];
    block_of(vc, r->b);
    r->linear = (uint16_t)local_index(vc);
    r->pix = pix;
}

/* traverse_segment (tsdf_integrator.hpp:93-135) */
static void traverse_segment(d3 a, d3 b, float voxel_size, visit_vec* out, uint32_t pix) {
    const double nu = voxel_size;
    int32_t cur[3], end[3];
    world_to_voxel(a, voxel_size, cur);
    world_to_voxel(b, voxel_size, end);
    d3 dir = sub3(b, a);
    const double len = norm3(dir);
    if (len < 1e-12) {
        push_visit(out, cur, pix);
        return;
    }
    dir = div3(dir, len);
    int32_t step[3];
    double t_max[3], t_delta[3];
    for (int i = 0; i < 3; ++i) {
        if (fabs(dir.v[i]) < 1e-15) {
            step[i] = 0;
            t_max[i] = INFINITY;
            t_delta[i] = INFINITY;
        } else {
            step[i] = dir.v[i] > 0 ? 1 : -1;
            const double boundary = nu * (cur[i] + 0.5 * step[i]);
            t_max[i] = (boundary - a.v[i]) / dir.v[i];
            t_delta[i] = nu / fabs(dir.v[i]);
        }
    }
    const size_t max_steps = (size_t)(3.0 * len / nu) + 8;
    for (size_t n = 0; n < max_steps; ++n) {
        push_visit(out, cur, pix);
        if (cur[0] == end[0] && cur[1] == end[1] && cur[2] == end[2]) return;
        int m = 0;
        if (t_max[1] < t_max[m]) m = 1;
        if (t_max[2] < t_max[m]) m = 2;
        if (t_max[m] > len) return;
        cur[m] += step[m];
        t_max[m] += t_delta[m];
    }
}

static int cmp_visit(const void* pa, const void* pb) {
    const visit* a = pa;
    const visit* b = pb;
    const int c = key_cmp(a->b, b->b);
    if (c) return c;
    if (a->linear != b->linear) return a->linear < b->linear ? -1 : 1;
    if (a->pix != b->pix) return a->pix < b->pix ? -1 : 1;
    return 0;
}

/* nonprojective_distance (tsdf_integrator.cpp:39-46) */
static double nonprojective_distance(double psi, double theta, double alpha, double eps) {
    const double ct = cos(theta);
    if (alpha < eps) return fabs(ct) * psi;
    const double mag = fabs((cos(alpha) - 1.0) * sin(theta) / sin(alpha)) + fabs(ct * psi);
    return psi >= 0.0 ? mag : -mag;
}
/* observation_weight (tsdf_integrator.cpp:48-51) */
static float observation_weight(double psi, double tau, float min_clamp) {
    double w = (psi + tau) / (2.0 * tau);
    const double lo = (double)min_clamp;
    w = w < lo ? lo : (w > 1.0 ? 1.0 : w);
    return (float)w;
}
/* truncate_distance (tsdf_integrator.hpp:57-59) */
static float truncate_distance(double d, double tau) {
    /* std::min(d, tau) = tau < d ? tau : d; std::max(d, -tau) = d < -tau ? -tau : d */
    return (float)(d >= 0.0 ? (tau < d ? tau : d) : (d < -tau ? -tau : d));
}

typedef struct {
    double wd, w;
    d3 wn;
} accum;

typedef struct {
    const svx_lidar_model* model;
    const float* depth;
    const float* normals;
    const uint8_t* valid;
    const svx_pose* pose;
    const svx_integrator_cfg* cfg;
    double tau;
    d3 origin;
} frame_ctx;

/* measure lambda (tsdf_integrator.cpp:172-205) */
static int measure(const frame_ctx* f, int u, int v, d3 center, const svx_tsdf_voxel* vox,
                   accum* acc) {
    const size_t idx = (size_t)v * f->model->width + u;
    const float depth = f->depth[idx];
    if (depth == 0.f || depth > f->cfg->max_range) return 0;
    const int have_normal = f->normals && f->valid[idx];
    if (!have_normal && f->cfg->drop_unreliable) return 0;

    const d3 q = xform(f->pose, back_project(u, v, depth, f->model));
    const d3 qo = sub3(q, f->origin);
    const double range = norm3(qo);
    const d3 ray = div3(qo, range);
    const double psi = range - dot3(sub3(center, f->origin), ray);
    if (fabs(psi) > f->tau) return 0;

    float nw[3] = {0.f, 0.f, 0.f};
    if (have_normal) {
        d3 ns = {{f->normals[3 * idx], f->normals[3 * idx + 1], f->normals[3 * idx + 2]}};
        const d3 r = matvec(f->pose->R, ns);
        for (int c = 0; c < 3; ++c) nw[c] = (float)r.v[c];
    }
    double d = psi;
    if (f->cfg->mode == SVX_NON_PROJECTIVE && have_normal) {
        float g[3] = {nw[0], nw[1], nw[2]};
        const float gsq = (vox->gradient[0] * vox->gradient[0] + vox->gradient[1] * vox->gradient[1]) +
                          vox->gradient[2] * vox->gradient[2];
        if (vox->weight > 0.f && gsq > 1e-12f)
            for (int c = 0; c < 3; ++c) g[c] = vox->gradient[c];
        const d3 gd = normalized3((d3){{g[0], g[1], g[2]}});
        const d3 mray = {{-ray.v[0], -ray.v[1], -ray.v[2]}};
        double ct = dot3(mray, gd);
        ct = ct < -1.0 ? -1.0 : (ct > 1.0 ? 1.0 : ct);
        double ca = dot3(gd, (d3){{nw[0], nw[1], nw[2]}});
        ca = ca < -1.0 ? -1.0 : (ca > 1.0 ? 1.0 : ca);
        d = nonprojective_distance(psi, acos(ct), acos(ca), f->cfg->alpha_epsilon);
    }
    const float w_obs = observation_weight(psi, f->tau, f->cfg->min_weight_clamp);
    acc->wd += (double)(w_obs * truncate_distance(d, f->tau));
    acc->w += w_obs;
    if (have_normal)
        for (int c = 0; c < 3; ++c) acc->wn.v[c] += (double)(w_obs * nw[c]);
    return 1;
}

/* TsdfIntegrator::integrate_frame (tsdf_integrator.cpp:97-258) */
int svxo_integrate(svxo_map* m, const svx_lidar_model* model, const float* depth,
                   const float* normals, const uint8_t* valid, const svx_pose* pose,
                   const svx_integrator_cfg* cfg, svx_frame_report* rep) {
    if (!(cfg->alpha_epsilon > 0.0)) return fail(1, "alpha_epsilon must be > 0");
    rep->frame = m->tsdf_frames++;
    rep->updated_voxels = 0;
    rep->new_blocks = 0;
    rep->elapsed_ms = 0.0;
    if (cfg->mode == SVX_NON_PROJECTIVE && !normals)
        return fail(1, "non-projective mode needs a normal image");
    frame_ctx f = {model, depth, normals, valid, pose, cfg, 0.0, origin_of(pose)};
    f.tau = cfg->truncation > 0.f ? (double)cfg->truncation : (double)m->cfg.truncation;
    const svx_pose w2s = inverse_pose(pose);
    const int W = model->width, H = model->height_px;

    /* phase 1: ray-cast the band (tsdf_integrator.cpp:119-139) */
    visit_vec vv = {0};
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            const size_t idx = (size_t)v * W + u;
            const float r = depth[idx];
            if (r == 0.f || r > cfg->max_range) continue;
            if (cfg->drop_unreliable && normals && !valid[idx]) continue;
            const d3 q = xform(pose, back_project(u, v, r, model));
            const d3 ray = normalized3(sub3(q, f.origin));
            const d3 tr = scale3(f.tau, ray);
            traverse_segment(sub3(q, tr), add3(q, tr), m->cfg.voxel_size, &vv, (uint32_t)idx);
        }
    if (vv.n == 0) {
        free(vv.v);
        return 0;
    }
    /* merge + sort (tsdf_integrator.cpp:141-158,215-216): per-voxel visits end up
     * in ascending pixel order, i.e. (v, u) order */
    qsort(vv.v, vv.n, sizeof(visit), cmp_visit);

    /* allocation in sorted block order (tsdf_integrator.cpp:160-168) */
    size_t nb = 0;
    for (size_t i = 0; i < vv.n; ++i)
        if (i == 0 || key_cmp(vv.v[i - 1].b, vv.v[i].b) != 0) ++nb;
    int64_t* bidx = malloc(nb * sizeof(int64_t));
    size_t bi = 0;
    for (size_t i = 0; i < vv.n; ++i) {
        if (i != 0 && key_cmp(vv.v[i - 1].b, vv.v[i].b) == 0) continue;
        int was_new = 0;
        const int64_t id = get_or_alloc(m, vv.v[i].b, &was_new);
        if (id < 0) {
            free(bidx);
            free(vv.v);
            return fail(2, "block budget exhausted");
        }
        rep->new_blocks += (uint64_t)was_new;
        bidx[bi++] = id;
        push_dirty(m, 0, vv.v[i].b);
    }

    /* phase 2: own-pixel rule, accumulate, fold (tsdf_integrator.cpp:211-252) */
    bi = (size_t)-1;
    for (size_t k = 0; k < vv.n;) {
        if (k == 0 || key_cmp(vv.v[k - 1].b, vv.v[k].b) != 0) ++bi;
        oblock* blk = m->blocks[bidx[bi]];
        const uint16_t linear = vv.v[k].linear;
        size_t k_end = k;
        while (k_end < vv.n && vv.v[k_end].linear == linear && key_cmp(vv.v[k_end].b, vv.v[k].b) == 0)
            ++k_end;
        int32_t vc[3];
        voxel_at(blk->key, linear, vc);
        const d3 center = voxel_center(vc, m->cfg.voxel_size);
        svx_tsdf_voxel* vox = &blk->tsdf[linear];
        accum acc = {0.0, 0.0, {{0.0, 0.0, 0.0}}};
        int own_u, own_v;
        double own_r;
        int measured = 0;
        if (project_point(xform(&w2s, center), model, &own_u, &own_v, &own_r) &&
            depth[(size_t)own_v * W + own_u] != 0.f) {
            measured = measure(&f, own_u, own_v, center, vox, &acc);
        } else {
            for (size_t j = k; j < k_end; ++j)
                measured |= measure(&f, (int)(vv.v[j].pix % W), (int)(vv.v[j].pix / W), center,
                                    vox, &acc);
        }
        if (measured) {
            const double w_old = vox->weight;
            vox->distance = (float)((w_old * vox->distance + acc.wd) / (w_old + acc.w));
            vox->weight = (float)(w_old + acc.w);
            d3 bl;
            for (int c = 0; c < 3; ++c) bl.v[c] = w_old * (double)vox->gradient[c] + acc.wn.v[c];
            const double nrm = norm3(bl);
            if (nrm > 1e-12)
                for (int c = 0; c < 3; ++c) vox->gradient[c] = (float)(bl.v[c] / nrm);
            ++rep->updated_voxels;
        }
        k = k_end;
    }
    free(bidx);
    free(vv.v);
    return 0;
}

/* ------------------------------------------------------ semantics (a15-a17) */
/* label_to_likelihood (semantic_integrator.cpp:24-39) */
static int label_to_likelihood(int label, float conf, int K, float floor_v, float* like) {
    if (conf < 0.f || conf > 1.f) return fail(1, "confidence must be in [0, 1]");
    const float base = K > 1 ? (1.f - conf) / (float)(K - 1) : 1.f;
    for (int k = 0; k < K; ++k) like[k] = base;
    if (label >= 0 && label < K) like[label] = K > 1 ? conf : 1.f;
    float sum = 0.f;
    for (int k = 0; k < K; ++k) {
        like[k] = like[k] < floor_v ? floor_v : like[k]; /* std::max(v, floor) */
        sum += like[k];
    }
    for (int k = 0; k < K; ++k) like[k] /= sum;
    return 0;
}

/* occluded_along_ray (semantic_integrator.cpp:64-84) */
static int occluded_along_ray(const svxo_map* m, d3 o, d3 center, double voxel_depth) {
    const double step = m->cfg.voxel_size;
    const double stop = voxel_depth - 2.5 * m->cfg.voxel_size;
    if (stop <= 2.0 * step) return 0;
    const d3 ray = normalized3(sub3(center, o));
    float prev = 0.f;
    int prev_valid = 0;
    for (double t = 2.0 * step; t < stop; t += step) {
        int32_t vc[3], b[3];
        world_to_voxel(add3(o, scale3(t, ray)), m->cfg.voxel_size, vc);
        block_of(vc, b);
        const int64_t i = find_idx(m, b);
        const svx_tsdf_voxel* vox = i >= 0 ? &m->blocks[i]->tsdf[local_index(vc)] : NULL;
        if (!vox || !(vox->weight > 0.f)) {
            prev_valid = 0;
            continue;
        }
        if (prev_valid && prev > 0.f && vox->distance <= 0.f) return 1;
        prev = vox->distance;
        prev_valid = 1;
    }
    return 0;
}

/* SemanticIntegrator::integrate_labels (semantic_integrator.cpp:91-165) */
int svxo_integrate_labels(svxo_map* m, const svx_label_image* img, const svx_semantic_cfg* cfg,
                          svx_frame_report* rep) {
    rep->frame = m->sem_frames++;
    rep->updated_voxels = 0;
    rep->new_blocks = 0;
    rep->elapsed_ms = 0.0;
    const int K = m->cfg.num_labels;
    const int has_tensor = img->prob_tensor != NULL;
    const double occlusion_floor = -0.5 * m->cfg.truncation;
    const svx_pose w2c = inverse_pose(&img->pose);
    const d3 cam_o = origin_of(&img->pose);
    float* like = malloc((size_t)K * sizeof(float));
    int st = 0;
    for (uint64_t bi = 0; bi < m->n && !st; ++bi) {
        oblock* blk = m->blocks[bi];
        uint64_t n_upd = 0;
        for (int li = 0; li < KV && !st; ++li) {
            const svx_tsdf_voxel* vox = &blk->tsdf[li];
            if (!(vox->weight > 0.f)) continue;
            if (vox->distance < occlusion_floor) continue;
            int32_t vc[3];
            voxel_at(blk->key, li, vc);
            const d3 center = voxel_center(vc, m->cfg.voxel_size);
            const d3 pc = xform(&w2c, center);
            if (pc.v[2] <= 0.0 || pc.v[2] > img->max_depth) continue;
            const int u = (int)floor(img->fx * pc.v[0] / pc.v[2] + img->cx);
            const int v = (int)floor(img->fy * pc.v[1] / pc.v[2] + img->cy);
            if (u < 0 || u >= img->width || v < 0 || v >= img->height) continue;
            if (cfg->occlusion == SVX_OCCLUSION_RAYCAST &&
                occluded_along_ray(m, cam_o, center, norm3(sub3(center, cam_o))))
                continue;
            const size_t pix = (size_t)v * img->width + u;
            if (has_tensor) {
                const float* t = img->prob_tensor + pix * K;
                float sum = 0.f;
                for (int k = 0; k < K; ++k) {
                    like[k] = t[k] < cfg->likelihood_floor ? cfg->likelihood_floor : t[k];
                    sum += like[k];
                }
                for (int k = 0; k < K; ++k) like[k] /= sum;
            } else {
                const float conf = img->confidence ? img->confidence[pix] : cfg->default_confidence;
                st = label_to_likelihood(img->labels[pix], conf, K, cfg->likelihood_floor, like);
                if (st) break;
            }
            ensure_semantics(m, blk);
            float* probs = blk->sem + (size_t)li * K;
            if (cfg->use_bayes) { /* apply_likelihood (semantic_integrator.cpp:44-52) */
                double z = 0.0;
                for (int k = 0; k < K; ++k) {
                    probs[k] *= like[k];
                    z += probs[k];
                }
                const float inv = (float)(1.0 / z);
                for (int k = 0; k < K; ++k) probs[k] *= inv;
            } else { /* apply_latest_argmax (semantic_integrator.cpp:54-59) */
                int best = 0;
                for (int k = 1; k < K; ++k)
                    if (like[k] > like[best]) best = k;
                for (int k = 0; k < K; ++k) probs[k] = k == best ? 1.f : 0.f;
            }
            ++n_upd;
        }
        rep->updated_voxels += n_upd;
        if (n_upd) push_dirty(m, 1, blk->key);
    }
    free(like);
    return st;
}

/* ------------------------------------------------- known-answer-test exports */
int svxo_project_point(const double p[3], const svx_lidar_model* m, int* u, int* v, double* r) {
    d3 q = {{p[0], p[1], p[2]}};
    return project_point(q, m, u, v, r);
}
void svxo_back_project(int u, int v, double depth, const svx_lidar_model* m, double out[3]) {
    const d3 q = back_project(u, v, depth, m);
    out[0] = q.v[0];
    out[1] = q.v[1];
    out[2] = q.v[2];
}
double svxo_nonprojective_distance(double psi, double theta, double alpha, double eps) {
    return nonprojective_distance(psi, theta, alpha, eps);
}
float svxo_observation_weight(double psi, double tau, float min_clamp) {
    return observation_weight(psi, tau, min_clamp);
}
float svxo_truncate_distance(double d, double tau) { return truncate_distance(d, tau); }
void svxo_world_to_voxel(const double p[3], float voxel_size, int32_t out[3]) {
    d3 q = {{p[0], p[1], p[2]}};
    world_to_voxel(q, voxel_size, out);
}
/* traverse_segment: writes up to cap voxel coords (x,y,z); returns the count. */
uint64_t svxo_traverse(const double a[3], const double b[3], float voxel_size, int32_t* out,
                       uint64_t cap) {
    visit_vec vv = {0};
    d3 A = {{a[0], a[1], a[2]}}, B = {{b[0], b[1], b[2]}};
    traverse_segment(A, B, voxel_size, &vv, 0);
    for (size_t i = 0; i < vv.n && i < cap; ++i) {
        const visit* r = &vv.v[i];
        out[3 * i] = r->b[0] * KB + (r->linear % KB);
        out[3 * i + 1] = r->b[1] * KB + (r->linear / KB) % KB;
        out[3 * i + 2] = r->b[2] * KB + r->linear / (KB * KB);
    }
    const uint64_t n = vv.n;
    free(vv.v);
    return n;
}
/* label_to_likelihood; returns 0 or 1 (invalid confidence). */
int svxo_label_to_likelihood(int label, float conf, int K, float floor_v, float* like) {
    return label_to_likelihood(label, conf, K, floor_v, like);
}
/* apply_likelihood (Bayes step) in place. */
void svxo_bayes(float* probs, const float* like, int K) {
    double z = 0.0;
    for (int k = 0; k < K; ++k) {
        probs[k] *= like[k];
        z += probs[k];
    }
    const float inv = (float)(1.0 / z);
    for (int k = 0; k < K; ++k) probs[k] *= inv;
}

/* ===================================================================== mesh
 * extract_mesh (mesh.cpp:105-229): marching cubes per block in sorted block order,
 * cells in linear (z, y, x) order, a vertex per lattice edge keyed by (lower corner,
 * axis). The reference dedups edges per block and then stitches blocks in sorted
 * order through a global edge map (mesh.cpp:192-216); one global edge map visited in
 * the same order assigns the same first-appearance indices, so that is what this
 * restatement does. Case tables: the classic Lorensen-Cline/Bourke tabulation, read
 * from the product header (pinned against the reference's mc_tables.hpp by
 * tests/test_oracle.py). */
#include "../paper_2412_00291_b200/csrc/svx_mc_tables.h"

typedef struct { int32_t c[3]; int axis; } edge_key;
typedef struct { edge_key k; uint32_t idx; int used; } edge_slot;
typedef struct {
    const svx_tsdf_voxel* tsdf;
    const oblock* blk;
    int linear;
    int32_t coord[3];
} cell_corner;

static uint64_t edge_hash(const edge_key* k) {
    return hkey(k->c) * 31u + (uint64_t)k->axis;
}
static float nonzero_distance(float d) { /* mesh.cpp:44-48 */
    const float eps = 1e-5f;
    if (d > -eps && d < eps) return d < 0.f ? -eps : eps;
    return d;
}

typedef struct {
    float *v, *n;
    uint8_t* l;
    uint32_t* f;
    uint64_t nv, nf, capv, capf;
} mesh_buf;

/* make_edge_vertex (mesh.cpp:52-95) */
static void make_edge_vertex(const svxo_map* m, const cell_corner* lo, const cell_corner* hi,
                             int reserved, float* pos, float* nrm, uint8_t* label) {
    const float dl = nonzero_distance(lo->tsdf->distance);
    const float dh = nonzero_distance(hi->tsdf->distance);
    const float t = dl / (dl - dh);
    const d3 cld = voxel_center(lo->coord, m->cfg.voxel_size);
    const d3 chd = voxel_center(hi->coord, m->cfg.voxel_size);
    float n[3];
    for (int c = 0; c < 3; ++c) {
        const float cl = (float)cld.v[c], ch = (float)chd.v[c];
        pos[c] = cl + t * (ch - cl);
        n[c] = (1.f - t) * lo->tsdf->gradient[c] + t * hi->tsdf->gradient[c];
    }
    const float norm = sqrtf((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
    for (int c = 0; c < 3; ++c) nrm[c] = norm > 1e-8f ? n[c] / norm : (c == 2 ? 1.f : 0.f);
    *label = 255;
    if (lo->blk->sem && hi->blk->sem) {
        const int K = m->cfg.num_labels;
        const float* pl = lo->blk->sem + (size_t)lo->linear * K;
        const float* ph = hi->blk->sem + (size_t)hi->linear * K;
        const float prior = 1.f / (float)K;
        int lp = 1, hp = 1;
        for (int k = 0; k < K; ++k) {
            if (pl[k] != prior) lp = 0;
            if (ph[k] != prior) hp = 0;
        }
        if (lp || hp) return;
        int best = 0;
        float best_p = -1.f;
        for (int k = 0; k < K; ++k) {
            const float p = (1.f - t) * pl[k] + t * ph[k];
            if (p > best_p) {
                best_p = p;
                best = k;
            }
        }
        *label = best == reserved ? 255 : (uint8_t)best;
    }
}

int svxo_mesh_extract(svxo_map* m, float min_weight, int32_t reserved, const int32_t* bxyz,
                      uint64_t n, uint64_t* n_vertices, uint64_t* n_faces) {
    /* the mesh blocks, sorted unique (block_coords_sorted, or the cached set of an
     * IncrementalMesher, mesh.cpp:261-285); absent blocks are skipped */
    oblock** blocks = malloc((m->n + 1) * sizeof(oblock*));
    uint64_t nb = 0;
    if (!bxyz) {
        memcpy(blocks, m->blocks, m->n * sizeof(oblock*));
        nb = m->n;
    } else {
        int32_t* ks = malloc((n + 1) * 12);
        memcpy(ks, bxyz, n * 12);
        qsort(ks, n, 12, cmp_key3);
        for (uint64_t i = 0; i < n; ++i) {
            if (i && key_cmp(ks + 3 * i, ks + 3 * (i - 1)) == 0) continue;
            const int64_t bi = find_idx(m, ks + 3 * i);
            if (bi >= 0) blocks[nb++] = m->blocks[bi];
        }
        free(ks);
    }
    qsort(blocks, nb, sizeof(oblock*), cmp_blockptr);

    uint8_t tris[256][16];
    for (int c = 0; c < 256; ++c) {
        const char* t = kMcTris[c];
        int k = 0;
        for (; t[k]; ++k) tris[c][k] = (uint8_t)(t[k] <= '9' ? t[k] - '0' : t[k] - 'a' + 10);
        tris[c][k] = 0xFF;
    }
    uint64_t hcap = 1 << 16;
    edge_slot* h = calloc(hcap, sizeof(edge_slot));
    mesh_buf out = {0};
    for (uint64_t bi = 0; bi < nb; ++bi) {
        const oblock* blk = blocks[bi];
        const int32_t o[3] = {blk->key[0] * KB, blk->key[1] * KB, blk->key[2] * KB};
        /* corner cache of the 9x9x9 voxels the block's cells touch (mesh.cpp:119-133) */
        const oblock* cb[9][9][9];
        for (int z = 0; z < 9; ++z)
            for (int y = 0; y < 9; ++y)
                for (int x = 0; x < 9; ++x) {
                    if (x < 8 && y < 8 && z < 8) {
                        cb[z][y][x] = blk;
                        continue;
                    }
                    const int32_t v[3] = {o[0] + x, o[1] + y, o[2] + z};
                    const int32_t bk[3] = {floor_div(v[0], KB), floor_div(v[1], KB), floor_div(v[2], KB)};
                    const int64_t j = find_idx(m, bk);
                    cb[z][y][x] = j >= 0 ? m->blocks[j] : NULL;
                }
        for (int z = 0; z < KB; ++z)
            for (int y = 0; y < KB; ++y)
                for (int x = 0; x < KB; ++x) {
                    cell_corner corners[8];
                    int usable = 1, cube = 0;
                    for (int c = 0; c < 8 && usable; ++c) {
                        const int cx = x + kMcCorner[c][0], cy = y + kMcCorner[c][1],
                                  cz = z + kMcCorner[c][2];
                        const oblock* b = cb[cz][cy][cx];
                        const int32_t vc[3] = {o[0] + cx, o[1] + cy, o[2] + cz};
                        const int lin = nonneg_mod(vc[0], KB) + KB * nonneg_mod(vc[1], KB) +
                                        KB * KB * nonneg_mod(vc[2], KB);
                        if (!b || b->tsdf[lin].weight < min_weight) {
                            usable = 0;
                            break;
                        }
                        corners[c].tsdf = &b->tsdf[lin];
                        corners[c].blk = b;
                        corners[c].linear = lin;
                        memcpy(corners[c].coord, vc, 12);
                        if (b->tsdf[lin].distance < 0.f) cube |= 1 << c;
                    }
                    const uint16_t emask = mc_edge_mask(cube);
                    if (!usable || emask == 0) continue;
                    uint32_t eidx[12];
                    for (int e = 0; e < 12; ++e) {
                        if (!(emask >> e & 1)) continue;
                        const cell_corner* a = &corners[kMcEdge[e][0]];
                        const cell_corner* b = &corners[kMcEdge[e][1]];
                        if (key_cmp(b->coord, a->coord) < 0) {
                            const cell_corner* t = a;
                            a = b;
                            b = t;
                        }
                        edge_key key;
                        memcpy(key.c, a->coord, 12);
                        key.axis = b->coord[1] != a->coord[1] ? 1 : (b->coord[2] != a->coord[2] ? 2 : 0);
                        if (2 * (out.nv + 1) > hcap) { /* grow the edge map */
                            edge_slot* nh = calloc(2 * hcap, sizeof(edge_slot));
                            for (uint64_t q = 0; q < hcap; ++q) {
                                if (!h[q].used) continue;
                                uint64_t s2 = edge_hash(&h[q].k) & (2 * hcap - 1);
                                while (nh[s2].used) s2 = (s2 + 1) & (2 * hcap - 1);
                                nh[s2] = h[q];
                            }
                            free(h);
                            h = nh;
                            hcap *= 2;
                        }
                        uint64_t sl = edge_hash(&key) & (hcap - 1);
                        while (h[sl].used && !(h[sl].k.axis == key.axis && key_cmp(h[sl].k.c, key.c) == 0))
                            sl = (sl + 1) & (hcap - 1);
                        if (!h[sl].used) {
                            h[sl].used = 1;
                            h[sl].k = key;
                            h[sl].idx = (uint32_t)out.nv;
                            if (out.nv == out.capv) {
                                out.capv = out.capv ? 2 * out.capv : 4096;
                                out.v = realloc(out.v, out.capv * 12);
                                out.n = realloc(out.n, out.capv * 12);
                                out.l = realloc(out.l, out.capv);
                            }
                            make_edge_vertex(m, a, b, reserved, out.v + 3 * out.nv, out.n + 3 * out.nv,
                                             out.l + out.nv);
                            ++out.nv;
                        }
                        eidx[e] = h[sl].idx;
                    }
                    for (int i = 0; tris[cube][i] != 0xFF; i += 3) { /* mesh.cpp:179-189 */
                        const uint32_t i0 = eidx[tris[cube][i]], i1 = eidx[tris[cube][i + 1]],
                                       i2 = eidx[tris[cube][i + 2]];
                        if (i0 == i1 || i1 == i2 || i0 == i2) continue;
                        if (out.nf == out.capf) {
                            out.capf = out.capf ? 2 * out.capf : 4096;
                            out.f = realloc(out.f, out.capf * 12);
                        }
                        out.f[3 * out.nf] = i0;
                        out.f[3 * out.nf + 1] = i2;
                        out.f[3 * out.nf + 2] = i1;
                        ++out.nf;
                    }
                }
    }
    free(h);
    free(blocks);
    free(m->mesh_v);
    free(m->mesh_n);
    free(m->mesh_l);
    free(m->mesh_f);
    m->mesh_v = out.v;
    m->mesh_n = out.n;
    m->mesh_l = out.l;
    m->mesh_f = out.f;
    m->mesh_nv = out.nv;
    m->mesh_nf = out.nf;
    *n_vertices = out.nv;
    *n_faces = out.nf;
    return 0;
}

void svxo_mesh_read(const svxo_map* m, float* vertices, float* normals, uint8_t* labels,
                    uint32_t* faces) {
    if (vertices && m->mesh_nv) memcpy(vertices, m->mesh_v, 12 * m->mesh_nv);
    if (normals && m->mesh_nv) memcpy(normals, m->mesh_n, 12 * m->mesh_nv);
    if (labels && m->mesh_nv) memcpy(labels, m->mesh_l, m->mesh_nv);
    if (faces && m->mesh_nf) memcpy(faces, m->mesh_f, 12 * m->mesh_nf);
}

/* ================================================================ occupancy
 * The occupancy extension of include/svx.h ("occupancy extension"), restated
 * serially. PARITY UNPINNED: the reference has no carving / log-odds / histogram
 * code (SPEC.md:255 declines carving), so this restates the project's own contract;
 * only the DDA it uses (traverse_segment above, tsdf_integrator.hpp:93-135) and the
 * key arithmetic are the reference's. */
typedef struct {
    int32_t key[3];
    uint32_t tag[KV];
    float L[KV];
    uint32_t hits[KV], misses[KV];
    uint32_t* hist; /* KV*K, NULL until a labelled hit */
    uint32_t touched_serial;
} oocc_block;

struct svxo_occ {
    svx_occ_cfg cfg;
    oocc_block** blocks;
    uint64_t n, cap;
    int64_t* table;
    uint64_t tcap;
    uint32_t serial;
    int32_t frames;
};

static int64_t occ_find(const svxo_occ* m, const int32_t k[3]) {
    uint64_t s = hkey(k) & (m->tcap - 1);
    for (;;) {
        const int64_t i = m->table[s];
        if (i < 0) return -1;
        if (key_cmp(m->blocks[i]->key, k) == 0) return i;
        s = (s + 1) & (m->tcap - 1);
    }
}
static void occ_table_insert(svxo_occ* m, int64_t idx) {
    uint64_t s = hkey(m->blocks[idx]->key) & (m->tcap - 1);
    while (m->table[s] >= 0) s = (s + 1) & (m->tcap - 1);
    m->table[s] = idx;
}
static int64_t occ_alloc(svxo_occ* m, const int32_t k[3]) {
    int64_t i = occ_find(m, k);
    if (i >= 0) return i;
    if (m->n == m->cap) {
        m->cap = m->cap ? 2 * m->cap : 256;
        m->blocks = realloc(m->blocks, m->cap * sizeof(oocc_block*));
    }
    oocc_block* b = calloc(1, sizeof *b);
    memcpy(b->key, k, 12);
    m->blocks[m->n] = b;
    i = (int64_t)m->n++;
    if (2 * m->n > m->tcap) {
        free(m->table);
        m->tcap *= 2;
        m->table = malloc(m->tcap * sizeof(int64_t));
        memset(m->table, 0xFF, m->tcap * sizeof(int64_t));
        for (uint64_t j = 0; j < m->n; ++j) occ_table_insert(m, (int64_t)j);
    } else {
        occ_table_insert(m, i);
    }
    return i;
}

svxo_occ* svxo_occ_create(const svx_occ_cfg* cfg) {
    svxo_occ* m = calloc(1, sizeof *m);
    m->cfg = *cfg;
    m->tcap = 1024;
    m->table = malloc(m->tcap * sizeof(int64_t));
    memset(m->table, 0xFF, m->tcap * sizeof(int64_t));
    return m;
}

void svxo_occ_destroy(svxo_occ* m) {
    if (!m) return;
    for (uint64_t i = 0; i < m->n; ++i) {
        free(m->blocks[i]->hist);
        free(m->blocks[i]);
    }
    free(m->blocks);
    free(m->table);
    free(m);
}

typedef struct {
    int32_t v[3];
    int kind;        /* 3 hit, 1 miss */
    uint32_t label;  /* >= K: none */
    uint32_t q;
} occ_visit;

typedef struct {
    occ_visit* v;
    size_t n, cap;
} occ_vec;

static void occ_push(occ_vec* o, const int32_t v[3], int kind, uint32_t label, uint32_t q) {
    if (o->n == o->cap) {
        o->cap = o->cap ? 2 * o->cap : 1 << 16;
        o->v = realloc(o->v, o->cap * sizeof(occ_visit));
    }
    occ_visit* r = &o->v[o->n++];
    memcpy(r->v, v, 12);
    r->kind = kind;
    r->label = label;
    r->q = q;
}

static uint32_t occ_q8(const float* conf, uint64_t i) {
    if (!conf) return 255u;
    const float c = conf[i];
    if (!isfinite(c)) return 0u;
    const float cc = c < 0.f ? 0.f : (c > 1.f ? 1.f : c);
    return (uint32_t)(cc * 255.f + 0.5f);
}

int svxo_occ_integrate(svxo_occ* m, const float* pts, const uint16_t* labels, const float* conf,
                       uint64_t n, int32_t stride, const svx_pose* pose, svx_occ_report* rep) {
    const svx_occ_cfg* c = &m->cfg;
    const int K = c->num_labels;
    occ_vec vis = {0};
    visit_vec ray = {0};
    uint64_t rays = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const float* q = pts + i * (uint64_t)stride;
        if (!(isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2]))) continue;
        const d3 ps = {{q[0], q[1], q[2]}};
        const double r = sqrt(dot3(ps, ps));
        if (r < c->min_range) continue;
        ++rays;
        const d3 pw = xform(pose, ps);
        const d3 o = origin_of(pose);
        const int hit = r <= c->max_range;
        const d3 end = hit ? pw : add3(o, scale3(c->max_range / r, sub3(pw, o)));
        int32_t ev[3];
        world_to_voxel(end, c->voxel_size, ev);
        const uint32_t lab = labels ? labels[i] : 0xFFFFFFFFu;
        if (c->carve) {
            ray.n = 0;
            traverse_segment(o, end, c->voxel_size, &ray, 0);
            for (size_t k = 0; k < ray.n; ++k) {
                const visit* t = &ray.v[k];
                const int32_t vc[3] = {t->b[0] * KB + (t->linear % KB), t->b[1] * KB + (t->linear / KB) % KB,
                                       t->b[2] * KB + t->linear / (KB * KB)};
                if (hit && vc[0] == ev[0] && vc[1] == ev[1] && vc[2] == ev[2]) continue;
                occ_push(&vis, vc, 1, 0xFFFFFFFFu, 0);
            }
        }
        if (hit) occ_push(&vis, ev, 3, lab, occ_q8(conf, i));
    }
    free(ray.v);
    /* capacity: the scan is rejected unchanged if its new blocks do not fit */
    uint64_t scap = 1024;
    while (scap < 4 * vis.n) scap *= 2;
    int32_t* seen = malloc(scap * 12);
    uint8_t* used = calloc(scap, 1);
    uint64_t fresh = 0;
    for (size_t k = 0; k < vis.n; ++k) {
        int32_t b[3];
        block_of(vis.v[k].v, b);
        for (int a = 0; a < 3; ++a)
            if (b[a] < -(1 << 20) || b[a] >= (1 << 20)) {
                free(seen), free(used), free(vis.v);
                return fail(1, "voxel outside the device key range [-2^23, 2^23)");
            }
        if (occ_find(m, b) >= 0) continue;
        uint64_t s = hkey(b) & (scap - 1);
        while (used[s] && key_cmp(seen + 3 * s, b) != 0) s = (s + 1) & (scap - 1);
        if (!used[s]) {
            used[s] = 1;
            memcpy(seen + 3 * s, b, 12);
            ++fresh;
        }
    }
    free(seen);
    free(used);
    if (m->n + fresh > c->max_blocks) {
        free(vis.v);
        return fail(2, "occupancy map: max_blocks reached");
    }
    const uint64_t old_n = m->n;
    m->serial += 1;
    const uint32_t S = m->serial;
    oocc_block** touched = malloc((m->n + fresh + 1) * sizeof(oocc_block*));
    uint64_t nt = 0;
    for (size_t k = 0; k < vis.n; ++k) {
        const occ_visit* t = &vis.v[k];
        int32_t b[3];
        block_of(t->v, b);
        const int64_t bi = occ_alloc(m, b); /* may grow m->blocks */
        oocc_block* blk = m->blocks[bi];
        if (blk->touched_serial != S) {
            blk->touched_serial = S;
            touched[nt++] = blk;
        }
        const int li = local_index(t->v);
        const uint32_t want = 4u * S + (uint32_t)t->kind;
        if (blk->tag[li] < want) blk->tag[li] = want;
        if (t->kind == 3 && t->label < (uint32_t)K) {
            if (!blk->hist) blk->hist = calloc((size_t)KV * K, sizeof(uint32_t));
            blk->hist[(size_t)li * K + t->label] += t->q;
        }
    }
    free(vis.v);
    uint64_t nh = 0, nm = 0;
    for (uint64_t k = 0; k < nt; ++k) {
        oocc_block* blk = touched[k];
        for (int v = 0; v < KV; ++v) {
            if (blk->tag[v] >> 2 != S) continue;
            if ((blk->tag[v] & 3u) == 3u) {
                const float t = blk->L[v] + c->l_hit;
                blk->L[v] = t > c->l_max ? c->l_max : t;
                blk->hits[v] += 1;
                ++nh;
            } else {
                const float t = blk->L[v] + c->l_miss;
                blk->L[v] = t < c->l_min ? c->l_min : t;
                blk->misses[v] += 1;
                ++nm;
            }
        }
    }
    free(touched);
    if (rep) {
        rep->frame = m->frames;
        rep->points = n;
        rep->rays = rays;
        rep->hit_voxels = nh;
        rep->miss_voxels = nm;
        rep->new_blocks = m->n - old_n;
        rep->elapsed_ms = 0.0;
    }
    m->frames += 1;
    return 0;
}

static int cmp_occptr(const void* a, const void* b) {
    return key_cmp((*(oocc_block* const*)a)->key, (*(oocc_block* const*)b)->key);
}

/* SOCC1 export (include/svx.h svx_occ_save_mem) */
#define PUT(x) do { memcpy(p, &(x), sizeof(x)); p += sizeof(x); } while (0)
/* Pinhole back-projection through the pixel centre (svx.h "pinhole depth images"; the
 * pixel convention of the reference's label projection, semantic_integrator.cpp:117-121),
 * FP64 in the contract's order, NaN for a dropped pixel. */
int svxo_occ_integrate_depth(svxo_occ* m, const float* depth, const uint16_t* labels,
                             const float* conf, const svx_pinhole* cam, const svx_pose* pose,
                             svx_occ_report* rep) {
    const uint64_t n = (uint64_t)cam->width * (uint64_t)cam->height;
    float* pts = malloc(sizeof(float) * 3 * (n ? n : 1));
    if (!pts) return 1;
    for (uint64_t i = 0; i < n; ++i) {
        const float z = depth[i];
        float x = NAN, y = NAN, zz = NAN;
        if (isfinite(z) && z > 0.f && (double)z <= cam->max_depth) {
            const uint32_t u = (uint32_t)(i % (uint64_t)cam->width), v = (uint32_t)(i / (uint64_t)cam->width);
            const double zd = (double)z;
            x = (float)(((double)u + 0.5 - cam->cx) * zd / cam->fx);
            y = (float)(((double)v + 0.5 - cam->cy) * zd / cam->fy);
            zz = z;
        }
        pts[3 * i] = x;
        pts[3 * i + 1] = y;
        pts[3 * i + 2] = zz;
    }
    const int st = svxo_occ_integrate(m, pts, labels, conf, n, 3, pose, rep);
    free(pts);
    return st;
}

uint64_t svxo_occ_save_mem(svxo_occ* m, uint8_t* buf, uint64_t cap) {
    const int K = m->cfg.num_labels;
    uint64_t size = 5 + 4 + 4 + 16 + 8;
    for (uint64_t i = 0; i < m->n; ++i)
        size += 12 + 3 * 4 * KV + 1 + (m->blocks[i]->hist ? (uint64_t)KV * K * 4 : 0);
    if (!buf) return size;
    if (cap < size) return 0;
    oocc_block** sorted = malloc((m->n + 1) * sizeof(oocc_block*));
    memcpy(sorted, m->blocks, m->n * sizeof(oocc_block*));
    qsort(sorted, m->n, sizeof(oocc_block*), cmp_occptr);
    uint8_t* p = buf;
    memcpy(p, "SOCC1", 5);
    p += 5;
    PUT(m->cfg.voxel_size);
    const uint32_t k32 = (uint32_t)K;
    PUT(k32);
    PUT(m->cfg.l_hit);
    PUT(m->cfg.l_miss);
    PUT(m->cfg.l_min);
    PUT(m->cfg.l_max);
    const uint64_t nb = m->n;
    PUT(nb);
    for (uint64_t i = 0; i < m->n; ++i) {
        const oocc_block* b = sorted[i];
        memcpy(p, b->key, 12);
        p += 12;
        memcpy(p, b->L, 4 * KV);
        p += 4 * KV;
        memcpy(p, b->hits, 4 * KV);
        p += 4 * KV;
        memcpy(p, b->misses, 4 * KV);
        p += 4 * KV;
        *p++ = b->hist != NULL;
        if (b->hist) {
            memcpy(p, b->hist, (size_t)KV * K * 4);
            p += (size_t)KV * K * 4;
        }
    }
    free(sorted);
    return size;
}
#undef PUT
