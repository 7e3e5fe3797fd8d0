/*
 * cdr_oracle.c — plain-C restatement of the reference's differentiable-render
 * hot path, used ONLY as the test oracle (tests/, __graft_entry__.smoke(),
 * bench.py cpu_baseline). It is never linked into, or called by, libcdr.so.
 *
 * Parity pin: tests/test_oracle_vs_ref.py checks every function below against
 * the reference library compiled from its own unmodified sources
 * (oracle/refbuild -> oracle/_ref), bit-exact where the reference is
 * deterministic single-threaded, and tests/golden/ holds fixtures generated
 * from that build (tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference is
 * compiled the same way, and the CUDA path disables contraction too).
 * Citations are relative to /root/reference/proj.
 */
#include "cdr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y, z; } d3;
typedef struct { double x, y; } d2;

static char g_err[256];
const char* orc_last_error(void) { return g_err; }

/* ---- vec.hpp:10-183 ---------------------------------------------------- */
static inline d3 v3(double x, double y, double z) { d3 r = {x, y, z}; return r; }
static inline d3 ld3(const double* p) { return v3(p[0], p[1], p[2]); }
static inline d3 add3(d3 a, d3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline d3 sub3(d3 a, d3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline d3 mul3(d3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
static inline d3 div3(d3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }
static inline d3 had3(d3 a, d3 b) { return v3(a.x * b.x, a.y * b.y, a.z * b.z); }
static inline double dot3(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline d3 cross3(d3 a, d3 b) {
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double len3(d3 a) { return sqrt(dot3(a, a)); }
static inline d3 norm3(d3 a) { return div3(a, len3(a)); }
static inline double comp3(d3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static inline d2 v2(double x, double y) { d2 r = {x, y}; return r; }

typedef struct { double m[9]; } m33;
/* Mat3::from_columns, det, inverse (vec.hpp:110-173) */
static m33 from_cols(d3 c0, d3 c1, d3 c2) {
    m33 r = {{c0.x, c1.x, c2.x, c0.y, c1.y, c2.y, c0.z, c1.z, c2.z}};
    return r;
}
static double det33(const m33* a) {
    const double* m = a->m;
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}
static m33 inv33(const m33* a) {
    const double* m = a->m;
    double inv = 1.0 / det33(a);
    m33 r = {{(m[4] * m[8] - m[5] * m[7]) * inv, (m[2] * m[7] - m[1] * m[8]) * inv,
              (m[1] * m[5] - m[2] * m[4]) * inv, (m[5] * m[6] - m[3] * m[8]) * inv,
              (m[0] * m[8] - m[2] * m[6]) * inv, (m[2] * m[3] - m[0] * m[5]) * inv,
              (m[3] * m[7] - m[4] * m[6]) * inv, (m[1] * m[6] - m[0] * m[7]) * inv,
              (m[0] * m[4] - m[1] * m[3]) * inv}};
    return r;
}
static d3 mv33(const m33* a, d3 v) {
    const double* m = a->m;
    return v3(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
              m[6] * v.x + m[7] * v.y + m[8] * v.z);
}
static d3 mtv33(const m33* a, d3 v) { /* Mat3::transpose_times */
    const double* m = a->m;
    return v3(m[0] * v.x + m[3] * v.y + m[6] * v.z, m[1] * v.x + m[4] * v.y + m[7] * v.z,
              m[2] * v.x + m[5] * v.y + m[8] * v.z);
}
static m33 skew33(d3 v) {
    m33 r = {{0, -v.z, v.y, v.z, 0, -v.x, -v.y, v.x, 0}};
    return r;
}
static m33 mm33(const m33* a, const m33* b) {
    m33 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += a->m[3 * i + k] * b->m[3 * k + j];
            r.m[3 * i + j] = s;
        }
    return r;
}
/* normalize_jacobian (vec.hpp:179-183) */
static m33 normalize_jacobian(d3 v) {
    double len = len3(v);
    d3 n = div3(v, len);
    double o[9] = {n.x * n.x, n.x * n.y, n.x * n.z, n.y * n.x, n.y * n.y,
                   n.y * n.z, n.z * n.x, n.z * n.y, n.z * n.z};
    double id[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    m33 r;
    double s = 1.0 / len;
    for (int i = 0; i < 9; ++i) r.m[i] = (id[i] - o[i]) * s;
    return r;
}

/* ---- rng.hpp:9-36 ------------------------------------------------------ */
static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static inline uint64_t hash_combine(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}
static inline uint64_t next_u64(uint64_t* s) { *s = splitmix64(*s); return *s; }
static inline double next_double(uint64_t* s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }

void orc_rng(uint64_t seed, int32_t nk, const uint64_t* keys, int32_t n, uint64_t* out) {
    uint64_t h = seed;
    for (int i = 0; i < nk; ++i) h = hash_combine(h, keys[i]);
    uint64_t st = splitmix64(h);
    for (int i = 0; i < n; ++i) out[i] = next_u64(&st);
}

/* ---- camera.cpp:25-59 -------------------------------------------------- */
static double tan_half_fov(const cdr_camera* c) { return tan(c->fov_deg * 3.14159265358979323846 / 360.0); }
static double aspect(const cdr_camera* c) { return (double)c->width / (double)c->height; }

static d3 primary_dir(const cdr_camera* c, d2 px) {
    const double th = tan_half_fov(c);
    double sx = (2.0 * px.x / c->width - 1.0) * th * aspect(c);
    double sy = (1.0 - 2.0 * px.y / c->height) * th;
    d3 f = ld3(c->forward), r = ld3(c->right), u = ld3(c->up);
    return norm3(add3(add3(f, mul3(r, sx)), mul3(u, sy)));
}
void orc_primary_ray(const cdr_camera* cam, double x, double y, double* dir) {
    d3 d = primary_dir(cam, v2(x, y));
    dir[0] = d.x; dir[1] = d.y; dir[2] = d.z;
}

static int project(const cdr_camera* c, d3 p, d2* q, double* depth) {
    d3 v = sub3(p, ld3(c->origin));
    double z = dot3(v, ld3(c->forward));
    if (depth) *depth = z;
    if (z <= 1e-12) return 0;
    const double th = tan_half_fov(c);
    double nx = dot3(v, ld3(c->right)) / (z * th * aspect(c));
    double ny = dot3(v, ld3(c->up)) / (z * th);
    *q = v2((nx + 1.0) * 0.5 * c->width, (1.0 - ny) * 0.5 * c->height);
    return 1;
}

static void projection_jacobian(const cdr_camera* c, d3 p, d3* dpx, d3* dpy) {
    d3 v = sub3(p, ld3(c->origin));
    d3 fw = ld3(c->forward);
    double z = dot3(v, fw);
    const double th = tan_half_fov(c);
    double r_dot = dot3(v, ld3(c->right)), u_dot = dot3(v, ld3(c->up));
    double cx = c->width / (2.0 * th * aspect(c));
    double cy = c->height / (2.0 * th);
    *dpx = mul3(sub3(mul3(ld3(c->right), 1.0 / z), mul3(fw, r_dot / (z * z))), cx);
    *dpy = mul3(sub3(mul3(ld3(c->up), 1.0 / z), mul3(fw, u_dot / (z * z))), -cy);
}

/* ---- render.cpp:10-22 -------------------------------------------------- */
static d2 pixel_sample_position(uint64_t seed, int view, int px, int py, int width, int sample,
                                int spp) {
    uint64_t st = splitmix64(hash_combine(
        hash_combine(hash_combine(seed, (uint64_t)view + 0x9e01),
                     (uint64_t)py * (uint64_t)width + (uint64_t)px),
        (uint64_t)sample));
    double u = next_double(&st), v = next_double(&st);
    int k = (int)lround(sqrt((double)spp));
    if (k * k == spp && k > 1) {
        u = ((sample % k) + u) / k;
        v = ((sample / k) + v) / k;
    }
    return v2(px + u, py + v);
}
void orc_pixel_sample_position(uint64_t seed, int32_t view, int32_t px, int32_t py,
                               int32_t width, int32_t sample, int32_t spp, double* out) {
    d2 p = pixel_sample_position(seed, view, px, py, width, sample, spp);
    out[0] = p.x; out[1] = p.y;
}

/* ---- bvh.cpp:11-26 ray_triangle ----------------------------------------- */
static int ray_triangle(d3 o, d3 d, d3 p0, d3 p1, d3 p2, double* t, double* b1, double* b2) {
    d3 e1 = sub3(p1, p0), e2 = sub3(p2, p0);
    d3 pvec = cross3(d, e2);
    double det = dot3(e1, pvec);
    if (fabs(det) < 1e-18) return 0;
    double inv_det = 1.0 / det;
    d3 tvec = sub3(o, p0);
    *b1 = dot3(tvec, pvec) * inv_det;
    if (*b1 < 0 || *b1 > 1) return 0;
    d3 qvec = cross3(tvec, e1);
    *b2 = dot3(d, qvec) * inv_det;
    if (*b2 < 0 || *b1 + *b2 > 1) return 0;
    *t = dot3(e2, qvec) * inv_det;
    return 1;
}

/* ---- texture.cpp:34-69 sample_texture ----------------------------------- */
typedef struct {
    d3 value, du, dv;
    int texel[4];
    double weight[4];
} texs;

static inline int wrapi(int i, int n) { i %= n; return i < 0 ? i + n : i; }
static d3 texel_rgb(const double* data, int ch, int idx) {
    const double* p = data + (size_t)idx * ch;
    return ch == 3 ? v3(p[0], p[1], p[2]) : v3(p[0], p[0], p[0]);
}
static texs sample_texture(const double* data, int w, int h, int ch, d2 uv) {
    texs s;
    double fu = uv.x - floor(uv.x);
    double fv = uv.y - floor(uv.y);
    double x = fu * w - 0.5;
    double y = fv * h - 0.5;
    int x0 = (int)floor(x), y0 = (int)floor(y);
    double tx = x - x0, ty = y - y0;
    int xs0 = wrapi(x0, w), xs1 = wrapi(x0 + 1, w), ys0 = wrapi(y0, h), ys1 = wrapi(y0 + 1, h);
    s.texel[0] = ys0 * w + xs0;
    s.texel[1] = ys0 * w + xs1;
    s.texel[2] = ys1 * w + xs0;
    s.texel[3] = ys1 * w + xs1;
    s.weight[0] = (1 - tx) * (1 - ty);
    s.weight[1] = tx * (1 - ty);
    s.weight[2] = (1 - tx) * ty;
    s.weight[3] = tx * ty;
    d3 v00 = texel_rgb(data, ch, s.texel[0]), v10 = texel_rgb(data, ch, s.texel[1]);
    d3 v01 = texel_rgb(data, ch, s.texel[2]), v11 = texel_rgb(data, ch, s.texel[3]);
    s.value = add3(add3(add3(mul3(v00, s.weight[0]), mul3(v10, s.weight[1])), mul3(v01, s.weight[2])),
                   mul3(v11, s.weight[3]));
    d3 dvx = add3(mul3(sub3(v10, v00), 1 - ty), mul3(sub3(v11, v01), ty));
    d3 dvy = add3(mul3(sub3(v01, v00), 1 - tx), mul3(sub3(v11, v10), tx));
    s.du = mul3(dvx, (double)w);
    s.dv = mul3(dvy, (double)h);
    return s;
}
void orc_sample_texture(const double* data, int32_t w, int32_t h, int32_t ch, double u,
                        double v, double* out, int32_t* texels) {
    texs s = sample_texture(data, w, h, ch, v2(u, v));
    double o[9] = {s.value.x, s.value.y, s.value.z, s.du.x, s.du.y, s.du.z, s.dv.x, s.dv.y, s.dv.z};
    memcpy(out, o, sizeof(o));
    for (int k = 0; k < 4; ++k) { out[9 + k] = s.weight[k]; texels[k] = s.texel[k]; }
}

/* ---- material.cpp:22-57 eval_brdf --------------------------------------- */
typedef struct {
    d3 value, d_roughness, d_mu;
    double d_diffuse, d_specular;
} brdf_t;

static brdf_t eval_brdf(d3 ad, d3 as, double alpha, double mu) {
    brdf_t e;
    memset(&e, 0, sizeof(e));
    if (mu <= 0) return e;
    const double kPi = 3.14159265358979323846;
    const double a2 = alpha * alpha;
    const double A = a2 * a2;
    const double B = mu * mu * (A - 1.0) + 1.0;
    const double k = (alpha + 1.0) * (alpha + 1.0) / 8.0;
    const double g = mu * (1.0 - k) + k;
    const double inv_B2g2 = 1.0 / (B * B * g * g);
    const double S = (A * mu / (4.0 * kPi)) * inv_B2g2;
    e.value = add3(mul3(ad, mu / kPi), mul3(as, S));
    e.d_diffuse = mu / kPi;
    e.d_specular = S;
    const double dA = 4.0 * a2 * alpha;
    const double dB_dalpha = mu * mu * dA;
    const double dk = (alpha + 1.0) / 4.0;
    const double dg_dalpha = dk * (1.0 - mu);
    const double dS_dalpha = S * (dA / A - 2.0 * dB_dalpha / B - 2.0 * dg_dalpha / g);
    e.d_roughness = mul3(as, dS_dalpha);
    const double dB_dmu = 2.0 * mu * (A - 1.0);
    const double dg_dmu = 1.0 - k;
    const double dS_dmu = (A / (4.0 * kPi)) * (1.0 - mu * (2.0 * dB_dmu / B + 2.0 * dg_dmu / g)) * inv_B2g2;
    e.d_mu = add3(mul3(ad, 1.0 / kPi), mul3(as, dS_dmu));
    return e;
}
void orc_eval_brdf(const double* ad, const double* as, double alpha, double mu, double* out) {
    brdf_t e = eval_brdf(ld3(ad), ld3(as), alpha, mu);
    double o[11] = {e.value.x, e.value.y, e.value.z, e.d_diffuse, e.d_specular,
                    e.d_roughness.x, e.d_roughness.y, e.d_roughness.z, e.d_mu.x, e.d_mu.y, e.d_mu.z};
    memcpy(out, o, sizeof(o));
}

/* ---- context: normals (mesh.cpp:65-95), normal Jacobians
 *      (diff_render.cpp:17-60), acceleration structure ------------------- */
typedef struct { double lo[3], hi[3]; int left, first, count; } onode;

struct orc_ctx {
    const orc_scene* s;
    double* normals; /* nv x 3 */
    double t_min;
    /* normal Jacobian CSR */
    int* nj_start;
    int* nj_w;
    m33* nj_m;
    /* BVH (oracle-private; any tree gives the same nearest-hit answer) */
    onode* nodes;
    int nnodes;
    int* order;
};

static d3 P(const orc_scene* s, int i) { return ld3(s->pos + 3 * (size_t)i); }
static d3 face_normal_un(const orc_scene* s, int f) {
    const int32_t* t = s->tris + 3 * (size_t)f;
    return cross3(sub3(P(s, t[1]), P(s, t[0])), sub3(P(s, t[2]), P(s, t[0])));
}

void orc_vertex_normals(const orc_scene* s, double* out) {
    d3* acc = (d3*)calloc((size_t)s->nv + 1, sizeof(d3));
    char* res = (char*)calloc((size_t)s->nv + 1, 1);
    for (int f = 0; f < s->nt; ++f) {
        d3 n = face_normal_un(s, f);
        for (int k = 0; k < 3; ++k) {
            int v = s->tris[3 * f + k];
            acc[v] = add3(acc[v], n);
        }
    }
    for (int v = 0; v < s->nv; ++v) {
        d3 n = v3(0, 0, 1);
        double len = len3(acc[v]);
        if (len >= 1e-12) { n = div3(acc[v], len); res[v] = 1; }
        out[3 * v] = n.x; out[3 * v + 1] = n.y; out[3 * v + 2] = n.z;
    }
    for (int f = 0; f < s->nt; ++f) {
        d3 n = face_normal_un(s, f);
        double len = len3(n);
        if (len < 1e-30) continue;
        for (int k = 0; k < 3; ++k) {
            int v = s->tris[3 * f + k];
            if (!res[v]) {
                d3 u = div3(n, len);
                out[3 * v] = u.x; out[3 * v + 1] = u.y; out[3 * v + 2] = u.z;
                res[v] = 1;
            }
        }
    }
    free(acc);
    free(res);
}

static void build_normal_jacobians(orc_ctx* c) {
    const orc_scene* s = c->s;
    int nv = s->nv;
    d3* acc = (d3*)calloc((size_t)nv + 1, sizeof(d3));
    int* cnt = (int*)calloc((size_t)nv + 1, sizeof(int));
    int* cap = (int*)calloc((size_t)nv + 1, sizeof(int));
    int** rw = (int**)calloc((size_t)nv + 1, sizeof(int*));
    m33** rm = (m33**)calloc((size_t)nv + 1, sizeof(m33*));
    for (int f = 0; f < s->nt; ++f) {
        d3 m = face_normal_un(s, f);
        for (int k = 0; k < 3; ++k) acc[s->tris[3 * f + k]] = add3(acc[s->tris[3 * f + k]], m);
    }
    for (int f = 0; f < s->nt; ++f) {
        const int32_t* t = s->tris + 3 * (size_t)f;
        d3 a = P(s, t[0]), b = P(s, t[1]), cc = P(s, t[2]);
        m33 dm[3] = {skew33(sub3(cc, b)), skew33(sub3(a, cc)), skew33(sub3(b, a))};
        for (int v = 0; v < 3; ++v)
            for (int q = 0; q < 3; ++q) {
                int row = t[v], w = t[q], found = 0;
                for (int e = 0; e < cnt[row]; ++e)
                    if (rw[row][e] == w) {
                        for (int i = 0; i < 9; ++i) rm[row][e].m[i] += dm[q].m[i];
                        found = 1;
                        break;
                    }
                if (!found) {
                    if (cnt[row] == cap[row]) {
                        cap[row] = cap[row] ? 2 * cap[row] : 8;
                        rw[row] = (int*)realloc(rw[row], sizeof(int) * cap[row]);
                        rm[row] = (m33*)realloc(rm[row], sizeof(m33) * cap[row]);
                    }
                    rw[row][cnt[row]] = w;
                    rm[row][cnt[row]] = dm[q];
                    cnt[row]++;
                }
            }
    }
    c->nj_start = (int*)calloc((size_t)nv + 1, sizeof(int));
    for (int v = 0; v < nv; ++v) c->nj_start[v + 1] = c->nj_start[v] + cnt[v];
    c->nj_w = (int*)malloc(sizeof(int) * ((size_t)c->nj_start[nv] + 1));
    c->nj_m = (m33*)malloc(sizeof(m33) * ((size_t)c->nj_start[nv] + 1));
    for (int v = 0; v < nv; ++v) {
        double len = len3(acc[v]);
        m33 jn;
        if (len >= 1e-12) jn = normalize_jacobian(acc[v]);
        else memset(&jn, 0, sizeof(jn));
        for (int e = 0; e < cnt[v]; ++e) {
            c->nj_w[c->nj_start[v] + e] = rw[v][e];
            c->nj_m[c->nj_start[v] + e] = mm33(&jn, &rm[v][e]);
        }
        free(rw[v]);
        free(rm[v]);
    }
    free(acc); free(cnt); free(cap); free(rw); free(rm);
}

/* Oracle BVH: median split on the longest centroid axis. Traversal prunes
 * with a padded box and never with a tie, so it returns exactly what the
 * brute-force scan of tests/support/test_scenes.hpp:20-39 returns. */
static const orc_scene* g_sort_scene;
static int g_sort_axis;
static double centroid_axis(const orc_scene* s, int f, int ax) {
    const int32_t* t = s->tris + 3 * (size_t)f;
    return s->pos[3 * t[0] + ax] + s->pos[3 * t[1] + ax] + s->pos[3 * t[2] + ax];
}
static int cmp_centroid(const void* a, const void* b) {
    int fa = *(const int*)a, fb = *(const int*)b;
    double ca = centroid_axis(g_sort_scene, fa, g_sort_axis), cb = centroid_axis(g_sort_scene, fb, g_sort_axis);
    if (ca < cb) return -1;
    if (ca > cb) return 1;
    return fa - fb;
}
static int build_node(orc_ctx* c, int first, int count) {
    const orc_scene* s = c->s;
    int id = c->nnodes++;
    onode* n = &c->nodes[id];
    double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
    for (int k = 0; k < 3; ++k) { n->lo[k] = 1e300; n->hi[k] = -1e300; }
    for (int i = first; i < first + count; ++i) {
        int f = c->order[i];
        for (int q = 0; q < 3; ++q) {
            const double* p = s->pos + 3 * (size_t)s->tris[3 * f + q];
            for (int k = 0; k < 3; ++k) {
                if (p[k] < n->lo[k]) n->lo[k] = p[k];
                if (p[k] > n->hi[k]) n->hi[k] = p[k];
            }
        }
        for (int k = 0; k < 3; ++k) {
            double cc = centroid_axis(s, f, k);
            if (cc < clo[k]) clo[k] = cc;
            if (cc > chi[k]) chi[k] = cc;
        }
    }
    n->left = -1;
    n->first = first;
    n->count = count;
    if (count <= 4) return id;
    int ax = 0;
    for (int k = 1; k < 3; ++k)
        if (chi[k] - clo[k] > chi[ax] - clo[ax]) ax = k;
    g_sort_scene = s;
    g_sort_axis = ax;
    qsort(c->order + first, (size_t)count, sizeof(int), cmp_centroid);
    int half = count / 2;
    int l = build_node(c, first, half);
    int r = build_node(c, first + half, count - half);
    n = &c->nodes[id];
    n->left = l;
    n->first = r; /* internal: right child index */
    n->count = 0;
    return id;
}

static int box_hit(const onode* n, d3 o, d3 d, double t_best, double pad) {
    double tmin = -1e300, tmax = 1e300;
    double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    for (int k = 0; k < 3; ++k) {
        double lo = n->lo[k] - pad, hi = n->hi[k] + pad;
        if (dd[k] == 0.0) {
            if (oo[k] < lo || oo[k] > hi) return 0;
            continue;
        }
        double t0 = (lo - oo[k]) / dd[k], t1 = (hi - oo[k]) / dd[k];
        if (t0 > t1) { double tt = t0; t0 = t1; t1 = tt; }
        if (t0 > tmin) tmin = t0;
        if (t1 < tmax) tmax = t1;
    }
    double slack = 1e-9 * (fabs(tmin) + fabs(tmax)) + pad;
    return tmax + slack >= tmin && tmin <= t_best + slack && tmax + slack >= 0;
}

static void consider(const orc_scene* s, int f, d3 o, d3 d, double t_min, double* bt, int* bf,
                     double* bb1, double* bb2) {
    const int32_t* t = s->tris + 3 * (size_t)f;
    double tt, b1, b2;
    if (ray_triangle(o, d, P(s, t[0]), P(s, t[1]), P(s, t[2]), &tt, &b1, &b2) && tt > t_min &&
        (tt < *bt || (tt == *bt && f < *bf))) {
        *bt = tt; *bf = f; *bb1 = b1; *bb2 = b2;
    }
}

static int trace(const orc_ctx* c, d3 o, d3 d, double t_min, double* t, double* b1, double* b2) {
    double bt = 1e300, bb1 = 0, bb2 = 0;
    int bf = -1;
    if (c->nnodes == 0) return -1;
    int stack[256], sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const onode* n = &c->nodes[stack[--sp]];
        if (!box_hit(n, o, d, bt, c->t_min * 1e-3)) continue;
        if (n->left < 0) {
            for (int i = n->first; i < n->first + n->count; ++i)
                consider(c->s, c->order[i], o, d, t_min, &bt, &bf, &bb1, &bb2);
        } else {
            stack[sp++] = n->first;
            stack[sp++] = n->left;
        }
    }
    *t = bt; *b1 = bb1; *b2 = bb2;
    return bf;
}

orc_ctx* orc_ctx_new(const orc_scene* s) {
    orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
    c->s = s;
    c->normals = (double*)malloc(sizeof(double) * 3 * ((size_t)s->nv + 1));
    orc_vertex_normals(s, c->normals);
    /* default_t_min_ = 1e-4 * bbox_diagonal (bvh.cpp:92, mesh.cpp:15-25) */
    if (s->nt > 0) {
        d3 lo = v3(1e300, 1e300, 1e300), hi = v3(-1e300, -1e300, -1e300);
        for (int i = 0; i < s->nv; ++i) {
            d3 p = P(s, i);
            lo = v3(fmin(lo.x, p.x), fmin(lo.y, p.y), fmin(lo.z, p.z));
            hi = v3(fmax(hi.x, p.x), fmax(hi.y, p.y), fmax(hi.z, p.z));
        }
        c->t_min = 1e-4 * len3(sub3(hi, lo));
    } else {
        c->t_min = 1e-8;
    }
    build_normal_jacobians(c);
    if (s->nt > 0) {
        c->nodes = (onode*)malloc(sizeof(onode) * 2 * (size_t)s->nt);
        c->order = (int*)malloc(sizeof(int) * (size_t)s->nt);
        for (int i = 0; i < s->nt; ++i) c->order[i] = i;
        build_node(c, 0, s->nt);
    }
    return c;
}

void orc_ctx_free(orc_ctx* c) {
    if (!c) return;
    free(c->normals); free(c->nj_start); free(c->nj_w); free(c->nj_m);
    free(c->nodes); free(c->order);
    free(c);
}
double orc_t_min(const orc_ctx* c) { return c->t_min; }

static int view_id(const orc_scene* s, int slot) { return s->view_ids ? s->view_ids[slot] : slot; }

int orc_intersect(const orc_ctx* c, int32_t n, const double* orig, const double* dir,
                  double t_min, int32_t* tri, double* t, double* b1, double* b2) {
    if (t_min < 0) t_min = c->t_min;
    for (int i = 0; i < n; ++i) tri[i] = trace(c, ld3(orig + 3 * i), ld3(dir + 3 * i), t_min, t + i, b1 + i, b2 + i);
    return 0;
}
int orc_intersect_brute(const orc_ctx* c, int32_t n, const double* orig, const double* dir,
                        double t_min, int32_t* tri, double* t, double* b1, double* b2) {
    if (t_min < 0) t_min = c->t_min;
    for (int i = 0; i < n; ++i) {
        double bt = 1e300, bb1 = 0, bb2 = 0;
        int bf = -1;
        for (int f = 0; f < c->s->nt; ++f)
            consider(c->s, f, ld3(orig + 3 * i), ld3(dir + 3 * i), t_min, &bt, &bf, &bb1, &bb2);
        tri[i] = bf; t[i] = bt; b1[i] = bb1; b2[i] = bb2;
    }
    return 0;
}

/* ---- render.cpp:24-33 radiance_at (+ make_hit_record bvh.cpp:28-51) ---- */
typedef struct {
    int tri;
    double t, b0, b1, b2;
    d2 uv;
    d3 normal;
} hitrec;

static d2 uv_of(const orc_scene* s, int v) { return s->uv ? v2(s->uv[2 * v], s->uv[2 * v + 1]) : v2(0, 0); }

static int radiance(const orc_ctx* c, int slot, d2 x, d3* out, hitrec* hr, int flat_normal) {
    const orc_scene* s = c->s;
    const cdr_camera* cam = &s->cams[slot];
    d3 o = ld3(cam->origin), d = primary_dir(cam, x);
    double t, b1, b2;
    int f = trace(c, o, d, c->t_min, &t, &b1, &b2);
    if (f < 0) { *out = ld3(s->background); return 0; }
    hitrec h;
    h.tri = f; h.t = t; h.b1 = b1; h.b2 = b2; h.b0 = 1.0 - b1 - b2;
    const int32_t* tv = s->tris + 3 * (size_t)f;
    h.uv = v2(0, 0);
    if (s->uv) {
        d2 a = uv_of(s, tv[0]), b = uv_of(s, tv[1]), cc = uv_of(s, tv[2]);
        h.uv = v2(a.x * h.b0 + b.x * b1 + cc.x * b2, a.y * h.b0 + b.y * b1 + cc.y * b2);
    }
    if (!flat_normal) {
        d3 n = add3(add3(mul3(ld3(c->normals + 3 * tv[0]), h.b0), mul3(ld3(c->normals + 3 * tv[1]), b1)),
                    mul3(ld3(c->normals + 3 * tv[2]), b2));
        double len = len3(n);
        h.normal = len > 1e-14 ? div3(n, len) : norm3(face_normal_un(s, f));
    } else {
        h.normal = norm3(face_normal_un(s, f));
    }
    if (hr) *hr = h;
    double mu = dot3(h.normal, v3(-d.x, -d.y, -d.z));
    texs sd = sample_texture(s->diffuse, s->tw, s->th, 3, h.uv);
    texs ss = sample_texture(s->specular, s->tw, s->th, 3, h.uv);
    texs sr = sample_texture(s->roughness, s->tw, s->th, 1, h.uv);
    brdf_t e = eval_brdf(sd.value, ss.value, sr.value.x, mu);
    *out = div3(had3(ld3(s->light), e.value), t * t);
    return 1;
}

int orc_radiance_at(const orc_ctx* c, int32_t view, int32_t n, const double* xy, double* rgb,
                    int32_t* tri) {
    for (int i = 0; i < n; ++i) {
        d3 r;
        hitrec h;
        int hit = radiance(c, view, v2(xy[2 * i], xy[2 * i + 1]), &r, &h, 0);
        rgb[3 * i] = r.x; rgb[3 * i + 1] = r.y; rgb[3 * i + 2] = r.z;
        if (tri) tri[i] = hit ? h.tri : -1;
    }
    return 0;
}

/* ---- render.cpp:35-64 render --------------------------------------------- */
int orc_render(const orc_ctx* c, int32_t view, int32_t spp_in, uint64_t seed, double* rgb,
               double* mask, int32_t* hit) {
    const orc_scene* s = c->s;
    const cdr_camera* cam = &s->cams[view];
    const int spp = spp_in < 1 ? 1 : spp_in;
    const int gid = view_id(s, view);
    for (int y = 0; y < cam->height; ++y)
        for (int x = 0; x < cam->width; ++x) {
            d3 sum = v3(0, 0, 0);
            int hits = 0;
            size_t pix = (size_t)y * cam->width + x;
            for (int q = 0; q < spp; ++q) {
                d2 pos = pixel_sample_position(seed, gid, x, y, cam->width, q, spp);
                d3 r;
                hitrec h;
                int ok = radiance(c, view, pos, &r, &h, 0);
                sum = add3(sum, r);
                if (hit) hit[pix * spp + q] = ok ? h.tri : -1;
                if (ok) ++hits;
            }
            d3 m = div3(sum, (double)spp);
            rgb[3 * pix] = m.x; rgb[3 * pix + 1] = m.y; rgb[3 * pix + 2] = m.z;
            if (mask) mask[pix] = (double)hits / (double)spp;
        }
    return 0;
}

/* ---- render.cpp:66-73 tone map; losses.cpp:15-49 view_rendering_loss ---- */
static double tone(double v, double gamma) {
    double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return pow(c, 1.0 / gamma);
}
static double tone_d(double v, double gamma) {
    if (v <= 0.0 || v >= 1.0) return 0.0;
    return pow(v, 1.0 / gamma - 1.0) / gamma;
}
static double sgn(double v) { return (double)((v > 0) - (v < 0)); }

int orc_view_loss(int32_t w, int32_t h, const double* r, const double* t, const double* tm,
                  double lambda, double gamma, int32_t use_mask, double* value, double* adj) {
    size_t n = (size_t)w * h;
    memset(adj, 0, sizeof(double) * 3 * n);
    *value = 0;
    if (lambda == 0) return 0;
    const int masked = use_mask && tm;
    double n_valid = 0;
    if (masked) {
        for (size_t i = 0; i < n; ++i) n_valid += tm[i];
        if (n_valid <= 0) return 0;
    } else {
        n_valid = (double)w * h;
    }
    const double scale = lambda / n_valid;
    double sum = 0;
    for (size_t i = 0; i < n; ++i) {
        double m = masked ? tm[i] : 1.0;
        if (m == 0) continue;
        for (int c = 0; c < 3; ++c) {
            double d = tone(r[3 * i + c], gamma) - tone(t[3 * i + c], gamma);
            sum += m * fabs(d);
            adj[3 * i + c] = scale * m * sgn(d) * tone_d(r[3 * i + c], gamma);
        }
    }
    *value = scale * sum;
    return 0;
}

/* ---- diff_render.cpp:62-201 interior_pass -------------------------------- */
static void addp(double* g, const cdr_layout* L, int v, d3 x) {
    g[L->positions + 3 * (int64_t)v] += x.x;
    g[L->positions + 3 * (int64_t)v + 1] += x.y;
    g[L->positions + 3 * (int64_t)v + 2] += x.z;
}

int orc_interior(const orc_ctx* c, int32_t view, const double* adjoint, int32_t spp_in,
                 uint64_t seed, const int32_t* hitc, const cdr_layout* Lay, double* g) {
    const orc_scene* s = c->s;
    const cdr_camera* cam = &s->cams[view];
    const int spp = spp_in < 1 ? 1 : spp_in;
    const int gid = view_id(s, view);
    const d3 L = ld3(s->light);
    const double Lc[3] = {L.x, L.y, L.z};
    for (int y = 0; y < cam->height; ++y)
        for (int x = 0; x < cam->width; ++x) {
            size_t pix = (size_t)y * cam->width + x;
            d3 adj = ld3(adjoint + 3 * pix);
            if (adj.x == 0 && adj.y == 0 && adj.z == 0) continue;
            d3 a3 = div3(adj, (double)spp);
            const double a[3] = {a3.x, a3.y, a3.z};
            for (int q = 0; q < spp; ++q) {
                int tri = hitc[pix * spp + q];
                if (tri < 0) continue;
                d2 pos = pixel_sample_position(seed, gid, x, y, cam->width, q, spp);
                d3 o = ld3(cam->origin), dir = primary_dir(cam, pos);
                const int32_t* tv = s->tris + 3 * (size_t)tri;
                d3 p0 = P(s, tv[0]), p1 = P(s, tv[1]), p2 = P(s, tv[2]);
                double t, b1, b2;
                if (!ray_triangle(o, dir, p0, p1, p2, &t, &b1, &b2)) continue;
                double b0 = 1.0 - b1 - b2;
                d2 uv0 = uv_of(s, tv[0]), uv1 = uv_of(s, tv[1]), uv2 = uv_of(s, tv[2]);
                d2 uv = v2(uv0.x * b0 + uv1.x * b1 + uv2.x * b2, uv0.y * b0 + uv1.y * b1 + uv2.y * b2);
                d3 N0 = ld3(c->normals + 3 * tv[0]), N1 = ld3(c->normals + 3 * tv[1]), N2 = ld3(c->normals + 3 * tv[2]);
                d3 nt = add3(add3(mul3(N0, b0), mul3(N1, b1)), mul3(N2, b2));
                double n_len = len3(nt);
                if (n_len < 1e-14) continue;
                d3 n_hat = div3(nt, n_len);
                d3 v_hat = v3(-dir.x, -dir.y, -dir.z);
                double mu = dot3(n_hat, v_hat);
                texs sd = sample_texture(s->diffuse, s->tw, s->th, 3, uv);
                texs ss = sample_texture(s->specular, s->tw, s->th, 3, uv);
                texs sr = sample_texture(s->roughness, s->tw, s->th, 1, uv);
                brdf_t br = eval_brdf(sd.value, ss.value, sr.value.x, mu);
                double inv_r2 = 1.0 / (t * t);
                for (int k = 0; k < 4; ++k) {
                    double wd = sd.weight[k] * br.d_diffuse * inv_r2;
                    double ws = ss.weight[k] * br.d_specular * inv_r2;
                    for (int cc = 0; cc < 3; ++cc) {
                        if (wd != 0) g[Lay->diffuse + 3 * (int64_t)sd.texel[k] + cc] += a[cc] * Lc[cc] * wd;
                        if (ws != 0) g[Lay->specular + 3 * (int64_t)ss.texel[k] + cc] += a[cc] * Lc[cc] * ws;
                    }
                    double wr = 0;
                    for (int cc = 0; cc < 3; ++cc) wr += a[cc] * Lc[cc] * comp3(br.d_roughness, cc) * inv_r2;
                    if (wr != 0) g[Lay->roughness + sr.texel[k]] += wr * sr.weight[k];
                }
                if (Lay->light >= 0)
                    for (int cc = 0; cc < 3; ++cc) g[Lay->light + cc] += a[cc] * comp3(br.value, cc) * inv_r2;
                if (mu <= 0) continue;
                m33 M = from_cols(dir, sub3(p0, p1), sub3(p0, p2));
                double det = det33(&M);
                if (fabs(det) < 1e-18) continue;
                m33 Mi = inv33(&M);
                d3 r0 = v3(Mi.m[0], Mi.m[1], Mi.m[2]), r1 = v3(Mi.m[3], Mi.m[4], Mi.m[5]), r2 = v3(Mi.m[6], Mi.m[7], Mi.m[8]);
                double cs = 0, cu = 0, cv = 0, cm = 0;
                for (int cc = 0; cc < 3; ++cc) {
                    double w = a[cc] * Lc[cc] * inv_r2;
                    cs += a[cc] * Lc[cc] * (-2.0 * comp3(br.value, cc) / (t * t * t));
                    double gu = br.d_diffuse * comp3(sd.du, cc) + br.d_specular * comp3(ss.du, cc) +
                                comp3(br.d_roughness, cc) * sr.du.x;
                    double gv = br.d_diffuse * comp3(sd.dv, cc) + br.d_specular * comp3(ss.dv, cc) +
                                comp3(br.d_roughness, cc) * sr.dv.x;
                    cu += w * gu;
                    cv += w * gv;
                    cm += w * comp3(br.d_mu, cc);
                }
                if (!isfinite(cs + cu + cv + cm)) {
                    snprintf(g_err, sizeof(g_err), "non-finite interior gradient at pixel (%d,%d)", x, y);
                    return CDR_ERR_NONFINITE;
                }
                m33 Jn = normalize_jacobian(nt);
                d3 h = mv33(&Jn, v_hat);
                double k1 = cu * (uv1.x - uv0.x) + cv * (uv1.y - uv0.y) + cm * (dot3(h, N1) - dot3(h, N0));
                double k2 = cu * (uv2.x - uv0.x) + cv * (uv2.y - uv0.y) + cm * (dot3(h, N2) - dot3(h, N0));
                d3 gc = add3(add3(mul3(r0, cs), mul3(r1, k1)), mul3(r2, k2));
                const double bc[3] = {b0, b1, b2};
                for (int j = 0; j < 3; ++j) addp(g, Lay, tv[j], mul3(gc, bc[j]));
                for (int j = 0; j < 3; ++j) {
                    double w = cm * bc[j];
                    if (w == 0) continue;
                    int vtx = tv[j];
                    for (int e = c->nj_start[vtx]; e < c->nj_start[vtx + 1]; ++e)
                        addp(g, Lay, c->nj_w[e], mul3(mtv33(&c->nj_m[e], h), w));
                }
            }
        }
    return 0;
}

/* ---- silhouette.cpp:14-106 ----------------------------------------------- */
static int clip_to_rect(d2 q0, d2 q1, double w, double h, double* s0, double* s1) {
    *s0 = 0;
    *s1 = 1;
    d2 d = v2(q1.x - q0.x, q1.y - q0.y);
    const double p[4] = {-d.x, d.x, -d.y, d.y};
    const double q[4] = {q0.x - 0.0, w - q0.x, q0.y - 0.0, h - q0.y};
    for (int i = 0; i < 4; ++i) {
        if (fabs(p[i]) < 1e-300) {
            if (q[i] < 0) return 0;
            continue;
        }
        double r = q[i] / p[i];
        if (p[i] < 0) {
            if (r > *s1) return 0;
            if (r > *s0) *s0 = r;
        } else {
            if (r < *s0) return 0;
            if (r < *s1) *s1 = r;
        }
    }
    return *s1 > *s0;
}
static int sign_of(double v) { return (v > 0) - (v < 0); }

int orc_silhouettes(const orc_ctx* c, int32_t view, cdr_segment* out, int32_t cap,
                    int32_t* count, double* total) {
    const orc_scene* s = c->s;
    const cdr_camera* cam = &s->cams[view];
    const double znear = 1e-6;
    d3 org = ld3(cam->origin), fw = ld3(cam->forward);
    int n = 0;
    double tot = 0;
    for (int i = 0; i < s->ne; ++i) {
        const int32_t* e = s->edges + 4 * (size_t)i;
        d3 a = P(s, e[0]), b = P(s, e[1]);
        if (e[3] >= 0) {
            d3 mid = mul3(add3(a, b), 0.5);
            d3 dd = sub3(mid, org);
            double sa = dot3(face_normal_un(s, e[2]), dd);
            double sb = dot3(face_normal_un(s, e[3]), dd);
            if (sign_of(sa) == sign_of(sb)) continue;
        }
        double za = dot3(sub3(a, org), fw), zb = dot3(sub3(b, org), fw);
        if (za <= znear && zb <= znear) continue;
        double t0 = 0, t1 = 1;
        if (za <= znear) t0 = (znear - za) / (zb - za);
        if (zb <= znear) t1 = (znear - za) / (zb - za);
        d3 pa = add3(a, mul3(sub3(b, a), t0)), pb = add3(a, mul3(sub3(b, a), t1));
        double z0, z1;
        d2 qa, qb;
        if (!project(cam, pa, &qa, &z0) || !project(cam, pb, &qb, &z1)) continue;
        double s0, s1;
        if (!clip_to_rect(qa, qb, cam->width, cam->height, &s0, &s1)) continue;
        cdr_segment g;
        g.v0 = e[0];
        g.v1 = e[1];
        g.p0[0] = a.x; g.p0[1] = a.y; g.p0[2] = a.z;
        g.p1[0] = b.x; g.p1[1] = b.y; g.p1[2] = b.z;
        g.q0[0] = qa.x + (qb.x - qa.x) * s0;
        g.q0[1] = qa.y + (qb.y - qa.y) * s0;
        g.q1[0] = qa.x + (qb.x - qa.x) * s1;
        g.q1[1] = qa.y + (qb.y - qa.y) * s1;
        double lx = g.q1[0] - g.q0[0], ly = g.q1[1] - g.q0[1];
        g.length_px = sqrt(lx * lx + ly * ly);
        if (g.length_px <= 0) continue;
        double u0 = ((1 - s0) / z0 * t0 + s0 / z1 * t1) / ((1 - s0) / z0 + s0 / z1);
        double u1 = ((1 - s1) / z0 * t0 + s1 / z1 * t1) / ((1 - s1) / z0 + s1 / z1);
        g.z0 = dot3(sub3(add3(a, mul3(sub3(b, a), u0)), org), fw);
        g.z1 = dot3(sub3(add3(a, mul3(sub3(b, a), u1)), org), fw);
        g.t0 = u0;
        g.t1 = u1;
        if (n < cap) out[n] = g;
        ++n;
        tot += g.length_px;
    }
    *count = n;
    *total = tot;
    return 0;
}

/* ---- diff_render.cpp:203-283 boundary_pass ------------------------------ */
/* boundary_pass with a caller's SilhouetteSet (diff_render.cpp:203-283 takes
 * the set as an argument); nseg segments, total = its total_length. */
int orc_boundary_segs(const orc_ctx* c, int32_t view, const double* adjoint, const cdr_segment* segs_in,
                      int32_t nseg, double tot, int32_t samples, uint64_t seed, int32_t probe,
                      const cdr_layout* Lay, double* g, int32_t* degenerate);

int orc_boundary(const orc_ctx* c, int32_t view, const double* adjoint, int32_t samples,
                 uint64_t seed, int32_t probe, const cdr_layout* Lay, double* g,
                 int32_t* degenerate) {
    int nseg = 0;
    double tot = 0;
    *degenerate = 0;
    orc_silhouettes(c, view, NULL, 0, &nseg, &tot);
    if (nseg == 0 || tot <= 0 || samples <= 0) return 0;
    cdr_segment* segs = (cdr_segment*)malloc(sizeof(cdr_segment) * (size_t)nseg);
    orc_silhouettes(c, view, segs, nseg, &nseg, &tot);
    int rc = orc_boundary_segs(c, view, adjoint, segs, nseg, tot, samples, seed, probe, Lay, g, degenerate);
    free(segs);
    return rc;
}

int orc_boundary_segs(const orc_ctx* c, int32_t view, const double* adjoint, const cdr_segment* segs_in,
                      int32_t nseg, double tot, int32_t samples, uint64_t seed, int32_t probe,
                      const cdr_layout* Lay, double* g, int32_t* degenerate) {
    const orc_scene* s = c->s;
    const cdr_camera* cam = &s->cams[view];
    const int gid = view_id(s, view);
    *degenerate = 0;
    if (nseg <= 0 || tot <= 0 || samples <= 0) return 0; /* diff_render.cpp:210-211 */
    cdr_segment* segs = (cdr_segment*)malloc(sizeof(cdr_segment) * (size_t)nseg);
    memcpy(segs, segs_in, sizeof(cdr_segment) * (size_t)nseg);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)nseg);
    double acc = 0;
    int usable = 0;
    for (int i = 0; i < nseg; ++i) {
        double len = segs[i].length_px;
        if (len < 1e-12) { ++*degenerate; len = 0; }
        else ++usable;
        acc += len;
        cdf[i] = acc;
    }
    if (usable == 0 || acc <= 0) { free(segs); free(cdf); return 0; }
    const double total_len = acc;
    int rc = 0;
    for (int64_t i = 0; i < samples; ++i) {
        uint64_t st = splitmix64(hash_combine(hash_combine(seed, (uint64_t)gid + 0xb0d1), (uint64_t)i));
        double pick = next_double(&st) * total_len;
        int lo = 0, hi = nseg; /* std::lower_bound */
        while (lo < hi) {
            int mid = lo + (hi - lo) / 2;
            if (cdf[mid] < pick) lo = mid + 1;
            else hi = mid;
        }
        int si = lo < nseg - 1 ? lo : nseg - 1;
        const cdr_segment* sg = &segs[si];
        if (sg->length_px < 1e-12) continue;
        double sp = next_double(&st);
        d2 xq = v2(sg->q0[0] + (sg->q1[0] - sg->q0[0]) * sp, sg->q0[1] + (sg->q1[1] - sg->q0[1]) * sp);
        int px = (int)floor(xq.x), py = (int)floor(xq.y);
        px = px < 0 ? 0 : (px > cam->width - 1 ? cam->width - 1 : px);
        py = py < 0 ? 0 : (py > cam->height - 1 ? cam->height - 1 : py);
        d3 adj = ld3(adjoint + 3 * ((size_t)py * cam->width + px));
        if (adj.x == 0 && adj.y == 0 && adj.z == 0) continue;
        d2 tg = v2((sg->q1[0] - sg->q0[0]) / sg->length_px, (sg->q1[1] - sg->q0[1]) / sg->length_px);
        d2 n2 = v2(-tg.y, tg.x);
        d2 xm = v2(xq.x - n2.x * 0.5, xq.y - n2.y * 0.5), xp = v2(xq.x + n2.x * 0.5, xq.y + n2.y * 0.5);
        d3 delta;
        if (probe == CDR_PROBE_RADIANCE) {
            d3 lo3, hi3;
            radiance(c, view, xm, &lo3, NULL, 0);
            radiance(c, view, xp, &hi3, NULL, 0);
            delta = sub3(lo3, hi3);
        } else {
            double t, b1, b2;
            d3 o = ld3(cam->origin);
            double cm = trace(c, o, primary_dir(cam, xm), c->t_min, &t, &b1, &b2) >= 0 ? 1.0 : 0.0;
            double cp = trace(c, o, primary_dir(cam, xp), c->t_min, &t, &b1, &b2) >= 0 ? 1.0 : 0.0;
            delta = v3(cm - cp, cm - cp, cm - cp);
        }
        double weighted = dot3(adj, delta);
        if (weighted == 0) continue;
        if (!isfinite(weighted)) {
            snprintf(g_err, sizeof(g_err), "non-finite boundary gradient at segment %d", si);
            rc = CDR_ERR_NONFINITE;
            break;
        }
        double w0 = (1.0 - sp) / sg->z0, w1 = sp / sg->z1;
        double t3 = (w0 * sg->t0 + w1 * sg->t1) / (w0 + w1);
        d3 p0 = ld3(sg->p0), p1 = ld3(sg->p1);
        d3 point = add3(p0, mul3(sub3(p1, p0), t3));
        d3 jx, jy;
        projection_jacobian(cam, point, &jx, &jy);
        d3 nj = add3(mul3(jx, n2.x), mul3(jy, n2.y));
        double scale = weighted * total_len / (double)samples;
        addp(g, Lay, sg->v0, mul3(nj, scale * (1.0 - t3)));
        addp(g, Lay, sg->v1, mul3(nj, scale * t3));
    }
    free(segs);
    free(cdf);
    return rc;
}

/* ---- laplacian.cpp:11-55 + losses.cpp:66-78 ------------------------------ */
static double cot_at(d3 apex, d3 a, d3 b) {
    d3 u = sub3(a, apex), v = sub3(b, apex);
    double cos_part = dot3(u, v);
    double sin_part = len3(cross3(u, v));
    if (sin_part < 1e-300) return INFINITY;
    return cos_part / sin_part;
}

/* CSC with rows sorted inside each column, entries V + 2E (no duplicates:
 * edges are unique and the diagonal is separate). */
int orc_laplacian(const orc_scene* s, int32_t mode, double lambda, double* value, double* grad,
                  int32_t* outer, int32_t* inner, double* vals) {
    int n = s->nv, ne = s->ne;
    double* w = (double*)malloc(sizeof(double) * ((size_t)ne + 1));
    double* diag = (double*)calloc((size_t)n + 1, sizeof(double));
    for (int i = 0; i < ne; ++i) {
        const int32_t* e = s->edges + 4 * (size_t)i;
        double wi = 1.0;
        if (mode == CDR_LAPLACIAN_COTANGENT) {
            wi = 0.0;
            for (int q = 0; q < 2; ++q) {
                int f = e[2 + q];
                if (f < 0) continue;
                const int32_t* t = s->tris + 3 * (size_t)f;
                int opp = t[0];
                for (int k = 0; k < 3; ++k)
                    if (t[k] != e[0] && t[k] != e[1]) opp = t[k];
                double cc = cot_at(P(s, opp), P(s, e[0]), P(s, e[1]));
                if (!isfinite(cc)) cc = 1e4;
                wi += 0.5 * cc;
            }
            wi = wi < 0.0 ? 0.0 : (wi > 1e4 ? 1e4 : wi);
        }
        w[i] = wi;
        diag[e[0]] -= wi;
        diag[e[1]] -= wi;
    }
    /* column counts: each column j holds its off-diagonal neighbours + diag */
    int32_t* cnt = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    for (int i = 0; i < ne; ++i) { cnt[s->edges[4 * i]]++; cnt[s->edges[4 * i + 1]]++; }
    int32_t* oc = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    oc[0] = 0;
    for (int j = 0; j < n; ++j) oc[j + 1] = oc[j] + cnt[j] + 1;
    int64_t nnz = oc[n];
    int32_t* ic = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nnz + 1));
    double* vc = (double*)malloc(sizeof(double) * ((size_t)nnz + 1));
    int32_t* fill = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    for (int j = 0; j < n; ++j) { ic[oc[j]] = j; vc[oc[j]] = diag[j]; fill[j] = 1; }
    for (int i = 0; i < ne; ++i) {
        int a = s->edges[4 * i], b = s->edges[4 * i + 1];
        ic[oc[b] + fill[b]] = a; vc[oc[b] + fill[b]++] = w[i];  /* (a, b) */
        ic[oc[a] + fill[a]] = b; vc[oc[a] + fill[a]++] = w[i];  /* (b, a) */
    }
    for (int j = 0; j < n; ++j) { /* insertion sort rows within the column */
        for (int k = oc[j] + 1; k < oc[j + 1]; ++k) {
            int32_t r = ic[k];
            double v = vc[k];
            int q = k - 1;
            while (q >= oc[j] && ic[q] > r) { ic[q + 1] = ic[q]; vc[q + 1] = vc[q]; --q; }
            ic[q + 1] = r;
            vc[q + 1] = v;
        }
    }
    if (outer) memcpy(outer, oc, sizeof(int32_t) * ((size_t)n + 1));
    if (inner) memcpy(inner, ic, sizeof(int32_t) * (size_t)nnz);
    if (vals) memcpy(vals, vc, sizeof(double) * (size_t)nnz);
    if (value) *value = 0;
    if (grad) memset(grad, 0, sizeof(double) * 3 * (size_t)n);
    if (lambda != 0) {
        /* LV = L * V (column by column, outer order), value = lambda ||LV||^2,
         * G = 2 lambda L^T (LV) */
        double* lv = (double*)calloc(3 * (size_t)n + 1, sizeof(double));
        for (int cc = 0; cc < 3; ++cc)
            for (int j = 0; j < n; ++j) {
                double xj = s->pos[3 * (size_t)j + cc];
                for (int k = oc[j]; k < oc[j + 1]; ++k) lv[(size_t)cc * n + ic[k]] += vc[k] * xj;
            }
        double sq = 0;
        for (size_t i = 0; i < 3 * (size_t)n; ++i) sq += lv[i] * lv[i];
        if (value) *value = lambda * sq;
        if (grad)
            for (int cc = 0; cc < 3; ++cc)
                for (int j = 0; j < n; ++j) {
                    double acc = 0;
                    for (int k = oc[j]; k < oc[j + 1]; ++k) acc += vc[k] * lv[(size_t)cc * n + ic[k]];
                    grad[3 * (size_t)j + cc] = (2.0 * lambda) * (0.0 + acc);
                }
        free(lv);
    }
    free(w); free(diag); free(cnt); free(oc); free(ic); free(vc); free(fill);
    return 0;
}

/* ---- losses.cpp:244-297 total_loss, hot subset (rendering + Laplacian) --- */
int orc_loss_grad(const orc_ctx* c, const double* targets_rgb, const double* targets_mask,
                  const cdr_settings* st, double lambda_rend, double lambda_lap,
                  int32_t lap_mode, int32_t use_mask, const cdr_layout* Lay,
                  double* loss_out, double* grad, double* rendered) {
    const orc_scene* s = c->s;
    size_t off = 0, moff = 0;
    loss_out[0] = 0;
    loss_out[1] = 0;
    const int spp = st->spp < 1 ? 1 : st->spp;
    for (int k = 0; k < s->nviews; ++k) {
        const cdr_camera* cam = &s->cams[k];
        size_t np = (size_t)cam->width * cam->height;
        double* rgb = (double*)malloc(sizeof(double) * 3 * np);
        double* adj = (double*)malloc(sizeof(double) * 3 * np);
        int32_t* hit = (int32_t*)malloc(sizeof(int32_t) * np * spp);
        orc_render(c, k, spp, st->seed, rgb, NULL, hit);
        double v;
        orc_view_loss(cam->width, cam->height, rgb, targets_rgb + off,
                      targets_mask ? targets_mask + moff : NULL, lambda_rend, st->gamma, use_mask, &v, adj);
        loss_out[0] += v;
        int rc = orc_interior(c, k, adj, spp, st->seed, hit, Lay, grad);
        if (rc == 0 && st->boundary_term) {
            int m = st->boundary_samples > 0 ? st->boundary_samples : cam->width * cam->height;
            int32_t deg;
            rc = orc_boundary(c, k, adj, m, st->seed, CDR_PROBE_RADIANCE, Lay, grad, &deg);
        }
        if (rendered) memcpy(rendered + off, rgb, sizeof(double) * 3 * np);
        free(rgb); free(adj); free(hit);
        if (rc) return rc;
        off += 3 * np;
        moff += np;
    }
    double* lg = (double*)malloc(sizeof(double) * (3 * (size_t)s->nv + 1));
    double lv = 0;
    orc_laplacian(s, lap_mode, lambda_lap, &lv, lg, NULL, NULL, NULL);
    loss_out[1] = lv;
    for (int v = 0; v < s->nv; ++v)
        for (int cc = 0; cc < 3; ++cc) {
            /* lap.grad[v] + nrm.grad[v] + edg.grad[v] with the out-of-scope
             * regularisers at weight 0 (losses.cpp:276-277) */
            double x = lg[3 * (size_t)v + cc] + 0.0 + 0.0;
            grad[Lay->positions + 3 * (int64_t)v + cc] += x;
        }
    free(lg);
    return 0;
}

/* ---- mesh / material regularisers (losses.cpp:80-238), SURVEY §8(f) row 1.
 * w[6] = normal, edge, spec, roug, sigma1, sigma2; values[4] = the four terms.
 * Gradients are WRITTEN (zeroed first): grad_pos nv x 3, grad_d / grad_s
 * tw*th*3, grad_r tw*th; any may be NULL. Sequential, in the reference order. */
static double sgnd(double v) { return (double)((v > 0) - (v < 0)); } /* losses.cpp:12 */

static d3 face_normal_unnorm(const orc_scene* s, int f) { /* mesh.hpp:30-33 */
    const int32_t* t = s->tris + 3 * (size_t)f;
    d3 a = ld3(s->pos + 3 * (size_t)t[0]);
    return cross3(sub3(ld3(s->pos + 3 * (size_t)t[1]), a), sub3(ld3(s->pos + 3 * (size_t)t[2]), a));
}

int orc_regularisers(const orc_scene* s, const double* w, double* values, double* grad_pos, double* grad_d,
                     double* grad_s, double* grad_r) {
    const int nv = s->nv, ne = s->ne, tw = s->tw, th = s->th, nt = tw * th;
    double* gn = (double*)calloc(3 * (size_t)nv + 1, sizeof(double));
    double* ge = (double*)calloc(3 * (size_t)nv + 1, sizeof(double));
    for (int i = 0; i < 4; ++i) values[i] = 0;
    /* normal_consistency_loss (losses.cpp:80-115) */
    if (w[0] != 0)
        for (int i = 0; i < ne; ++i) {
            const int32_t* e = s->edges + 4 * (size_t)i;
            if (e[3] < 0) continue;
            d3 m0 = face_normal_unnorm(s, e[2]), m1 = face_normal_unnorm(s, e[3]);
            double l0 = len3(m0), l1 = len3(m1);
            if (l0 < 1e-14 || l1 < 1e-14) continue;
            d3 n0 = div3(m0, l0), n1 = div3(m1, l1);
            double r = 1.0 - dot3(n0, n1);
            values[0] += w[0] * r * r;
            m33 j0 = normalize_jacobian(m0), j1 = normalize_jacobian(m1);
            d3 h0 = mv33(&j0, n1), h1 = mv33(&j1, n0);
            double wt = -2.0 * w[0] * r;
            for (int which = 0; which < 2; ++which) {
                const int32_t* t = s->tris + 3 * (size_t)(which == 0 ? e[2] : e[3]);
                d3 h = which == 0 ? h0 : h1;
                d3 a = ld3(s->pos + 3 * (size_t)t[0]), b = ld3(s->pos + 3 * (size_t)t[1]),
                   c = ld3(s->pos + 3 * (size_t)t[2]);
                m33 da = skew33(sub3(c, b)), db = skew33(sub3(a, c)), dc = skew33(sub3(b, a));
                d3 ga = mul3(mtv33(&da, h), wt), gb = mul3(mtv33(&db, h), wt), gc = mul3(mtv33(&dc, h), wt);
                double* q;
                q = gn + 3 * (size_t)t[0]; q[0] += ga.x; q[1] += ga.y; q[2] += ga.z;
                q = gn + 3 * (size_t)t[1]; q[0] += gb.x; q[1] += gb.y; q[2] += gb.z;
                q = gn + 3 * (size_t)t[2]; q[0] += gc.x; q[1] += gc.y; q[2] += gc.z;
            }
        }
    /* edge_length_loss (losses.cpp:117-134) */
    if (w[1] != 0 && ne > 0) {
        double sum_sq = 0;
        for (int i = 0; i < ne; ++i) {
            d3 d = sub3(ld3(s->pos + 3 * (size_t)s->edges[4 * i]), ld3(s->pos + 3 * (size_t)s->edges[4 * i + 1]));
            sum_sq += dot3(d, d);
        }
        if (sum_sq > 0) {
            double root = sqrt(sum_sq);
            values[1] = w[1] * root;
            double wt = w[1] / root;
            for (int i = 0; i < ne; ++i) {
                int a = s->edges[4 * i], b = s->edges[4 * i + 1];
                d3 d = mul3(sub3(ld3(s->pos + 3 * (size_t)a), ld3(s->pos + 3 * (size_t)b)), wt);
                ge[3 * (size_t)a] += d.x; ge[3 * (size_t)a + 1] += d.y; ge[3 * (size_t)a + 2] += d.z;
                ge[3 * (size_t)b] -= d.x; ge[3 * (size_t)b + 1] -= d.y; ge[3 * (size_t)b + 2] -= d.z;
            }
        }
    }
    if (grad_pos)
        for (size_t i = 0; i < 3 * (size_t)nv; ++i) grad_pos[i] = gn[i] + ge[i]; /* nrm + edg, losses.cpp:276 */
    free(gn);
    free(ge);
    /* specular_correlation_loss (losses.cpp:136-213) */
    double* gs = (double*)calloc(3 * (size_t)nt + 1, sizeof(double));
    double* gd = (double*)calloc(3 * (size_t)nt + 1, sizeof(double));
    if (w[2] != 0 && nt > 0) {
        const double lw[3] = {0.2126, 0.7152, 0.0722};
        const double i1 = 1.0 / (2.0 * w[4] * w[4]), i2 = 1.0 / (2.0 * w[5] * w[5]);
        double* lum = (double*)malloc(sizeof(double) * (size_t)nt);
        for (int i = 0; i < nt; ++i) lum[i] = dot3(ld3(s->diffuse + 3 * (size_t)i), v3(lw[0], lw[1], lw[2]));
        for (int p = 0; p < nt; ++p) {
            int px = p % tw, py = p / tw, cnt = 0, qs[49];
            double mus[49], mu_sum = 0;
            d3 avg = v3(0, 0, 0);
            for (int dy = -3; dy <= 3; ++dy) {
                int qy = py + dy;
                if (qy < 0 || qy >= th) continue;
                for (int dx = -3; dx <= 3; ++dx) {
                    int qx = px + dx;
                    if (qx < 0 || qx >= tw) continue;
                    int q = qy * tw + qx;
                    double dl = lum[p] - lum[q];
                    double mu = exp(-(dx * dx + dy * dy) * i1 - dl * dl * i2);
                    mus[cnt] = mu;
                    qs[cnt++] = q;
                    mu_sum += mu;
                    avg = add3(avg, mul3(ld3(s->specular + 3 * (size_t)q), mu));
                }
            }
            avg = div3(avg, mu_sum);
            d3 ctr = ld3(s->specular + 3 * (size_t)p);
            double sg[3];
            for (int c = 0; c < 3; ++c) {
                double d = comp3(ctr, c) - comp3(avg, c);
                values[2] += w[2] * fabs(d);
                sg[c] = sgnd(d);
            }
            for (int c = 0; c < 3; ++c) gs[3 * (size_t)p + c] += w[2] * sg[c];
            for (int k = 0; k < cnt; ++k) {
                int q = qs[k];
                double mu = mus[k], dtm = 0;
                for (int c = 0; c < 3; ++c) gs[3 * (size_t)q + c] -= w[2] * sg[c] * mu / mu_sum;
                d3 asq = ld3(s->specular + 3 * (size_t)q);
                for (int c = 0; c < 3; ++c) dtm += -w[2] * sg[c] * (comp3(asq, c) - comp3(avg, c)) / mu_sum;
                double dl = lum[p] - lum[q];
                double dp_ = mu * (-2.0 * dl * i2), dq = -dp_;
                for (int c = 0; c < 3; ++c) {
                    gd[3 * (size_t)p + c] += dtm * dp_ * lw[c];
                    gd[3 * (size_t)q + c] += dtm * dq * lw[c];
                }
            }
        }
        free(lum);
    }
    if (grad_s) memcpy(grad_s, gs, sizeof(double) * 3 * (size_t)nt);
    if (grad_d) memcpy(grad_d, gd, sizeof(double) * 3 * (size_t)nt);
    free(gs);
    free(gd);
    /* roughness_tv_loss (losses.cpp:215-238) */
    double* gr = (double*)calloc((size_t)nt + 1, sizeof(double));
    if (w[3] != 0)
        for (int y = 0; y < th; ++y)
            for (int x = 0; x < tw; ++x) {
                int i = y * tw + x;
                double v = s->roughness[i];
                if (x + 1 < tw) {
                    double d = s->roughness[i + 1] - v, sv = w[3] * sgnd(d);
                    values[3] += w[3] * fabs(d);
                    gr[i + 1] += sv;
                    gr[i] -= sv;
                }
                if (y + 1 < th) {
                    double d = s->roughness[i + tw] - v, sv = w[3] * sgnd(d);
                    values[3] += w[3] * fabs(d);
                    gr[i + tw] += sv;
                    gr[i] -= sv;
                }
            }
    if (grad_r) memcpy(grad_r, gr, sizeof(double) * (size_t)nt);
    free(gr);
    return 0;
}

/* ---- self_intersects (mesh.cpp:137-214), SURVEY §8(f) row 2. Brute force
 * over all pairs f < g with an exact fp64 AABB prefilter (a pair whose boxes
 * are disjoint cannot pass the separating-axis test), pairs in (f, g) order.
 * pairs (cap x 2) and n_pairs may be NULL. */
static int sat_separated(d3 axis, const d3* ta, const d3* tb, double tol) { /* mesh.cpp:147-157 */
    double l2 = dot3(axis, axis);
    if (l2 < 1e-24) return 0;
    double alo = dot3(axis, ta[0]), ahi = alo, blo = dot3(axis, tb[0]), bhi = blo;
    for (int i = 1; i < 3; ++i) {
        double da = dot3(axis, ta[i]), db = dot3(axis, tb[i]);
        alo = da < alo ? da : alo;
        ahi = ahi < da ? da : ahi;
        blo = db < blo ? db : blo;
        bhi = bhi < db ? db : bhi;
    }
    double g0 = blo - ahi, g1 = alo - bhi, gap = g0 < g1 ? g1 : g0;
    return gap > -tol * sqrt(l2);
}

int orc_triangles_intersect(const double* a0, const double* a1, const double* a2, const double* b0,
                            const double* b1, const double* b2, double tol) { /* mesh.cpp:160-182 */
    d3 ta[3] = {ld3(a0), ld3(a1), ld3(a2)}, tb[3] = {ld3(b0), ld3(b1), ld3(b2)};
    d3 ea[3] = {sub3(ta[1], ta[0]), sub3(ta[2], ta[1]), sub3(ta[0], ta[2])};
    d3 eb[3] = {sub3(tb[1], tb[0]), sub3(tb[2], tb[1]), sub3(tb[0], tb[2])};
    if (sat_separated(cross3(ea[0], ea[1]), ta, tb, tol)) return 0;
    if (sat_separated(cross3(eb[0], eb[1]), ta, tb, tol)) return 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (sat_separated(cross3(ea[i], eb[j]), ta, tb, tol)) return 0;
    return 1;
}

int orc_self_intersects(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, int32_t* result,
                        int32_t* pairs, int64_t cap, int64_t* n_pairs) {
    (void)nv;
    int64_t n = 0;
    double* box = (double*)malloc(sizeof(double) * 6 * ((size_t)nt + 1));
    for (int f = 0; f < nt; ++f)
        for (int k = 0; k < 3; ++k) {
            double a = pos[3 * (size_t)tris[3 * f] + k], b = pos[3 * (size_t)tris[3 * f + 1] + k],
                   c = pos[3 * (size_t)tris[3 * f + 2] + k];
            box[6 * (size_t)f + k] = fmin(a, fmin(b, c));
            box[6 * (size_t)f + 3 + k] = fmax(a, fmax(b, c));
        }
    const int want = pairs != NULL || n_pairs != NULL;
    for (int f = 0; f < nt && (want || n == 0); ++f) {
        const int32_t* t = tris + 3 * (size_t)f;
        for (int g = f + 1; g < nt; ++g) {
            const int32_t* u = tris + 3 * (size_t)g;
            const double *bf = box + 6 * (size_t)f, *bg = box + 6 * (size_t)g;
            if (bf[0] > bg[3] || bf[3] < bg[0] || bf[1] > bg[4] || bf[4] < bg[1] || bf[2] > bg[5] || bf[5] < bg[2])
                continue;
            int share = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) share |= t[i] == u[j];
            if (share) continue;
            if (orc_triangles_intersect(pos + 3 * (size_t)t[0], pos + 3 * (size_t)t[1], pos + 3 * (size_t)t[2],
                                        pos + 3 * (size_t)u[0], pos + 3 * (size_t)u[1], pos + 3 * (size_t)u[2],
                                        1e-10)) {
                if (pairs && n < cap) {
                    pairs[2 * n] = f;
                    pairs[2 * n + 1] = g;
                }
                ++n;
                if (!want) break;
            }
        }
    }
    free(box);
    *result = n > 0;
    if (n_pairs) *n_pairs = n;
    return 0;
}

/* ---- adam_step (adam.cpp:9-54) and robust_evolve (evolve.cpp:19-53), SURVEY
 * §8(f) row 3. cfg = beta1, beta2, epsilon, lr_positions, lr_textures,
 * lr_light. m, v, *step updated in place; params_out = params with texture /
 * light segments stepped and clamped; disp_out = V x 3 position deltas.
 * Returns CDR_ERR_NONFINITE (nothing updated) on a non-finite gradient. */
int orc_adam_step(const double* cfg, const cdr_layout* L, int64_t nv, int64_t n_tex, int64_t* step, double* m,
                  double* v, const double* params, const double* grad, double* params_out, double* disp_out) {
    for (int64_t i = 0; i < L->total; ++i)
        if (!isfinite(grad[i])) return CDR_ERR_NONFINITE;
    *step += 1;
    const double c1 = 1.0 - pow(cfg[0], (double)*step), c2 = 1.0 - pow(cfg[1], (double)*step);
    memcpy(params_out, params, sizeof(double) * (size_t)L->total);
    for (int64_t i = 0; i < L->total; ++i) {
        double lr = cfg[4], lo = 0.0, hi = 1.0;
        int pos = 0;
        if (i >= L->positions && i < L->positions + 3 * nv) { lr = cfg[3]; pos = 1; }
        else if (i >= L->roughness && i < L->roughness + n_tex) lo = 0.01; /* kAlphaMin */
        else if (L->light >= 0 && i >= L->light && i < L->light + 3) { lr = cfg[5]; hi = 1e30; }
        double g = grad[i];
        m[i] = cfg[0] * m[i] + (1.0 - cfg[0]) * g;
        v[i] = cfg[1] * v[i] + (1.0 - cfg[1]) * g * g;
        double mh = m[i] / c1, vh = v[i] / c2;
        double delta = -lr * mh / (sqrt(vh) + cfg[2]);
        if (pos) disp_out[i - L->positions] = delta;
        else {
            double x = params_out[i] + delta;
            params_out[i] = x < lo ? lo : (hi < x ? hi : x);
        }
    }
    return 0;
}

static double min_area(const double* pos, const int32_t* tris, int32_t nt) { /* evolve.cpp:11-15 */
    double best = 1e300;
    for (int f = 0; f < nt; ++f) {
        d3 a = ld3(pos + 3 * (size_t)tris[3 * f]);
        double ar = 0.5 * len3(cross3(sub3(ld3(pos + 3 * (size_t)tris[3 * f + 1]), a),
                                      sub3(ld3(pos + 3 * (size_t)tris[3 * f + 2]), a)));
        best = ar < best ? ar : best;
    }
    return best;
}

int orc_robust_evolve(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* disp,
                      double* pos_out, double* scale_out) {
    int32_t r = 0;
    orc_self_intersects(pos, nv, tris, nt, &r, NULL, 0, NULL);
    if (r) return CDR_ERR_SELF_INTERSECTING;
    memcpy(pos_out, pos, sizeof(double) * 3 * (size_t)nv);
    *scale_out = 0.0;
    int any = 0;
    for (int64_t i = 0; i < 3 * (int64_t)nv; ++i) any |= disp[i] != 0;
    if (!any) { *scale_out = 1.0; return 0; }
    double* cand = (double*)malloc(sizeof(double) * 3 * ((size_t)nv + 1));
    double s = 1.0;
    for (int attempt = 0; attempt <= 8; ++attempt, s *= 0.5) {
        for (int64_t i = 0; i < 3 * (int64_t)nv; ++i) cand[i] = pos[i] + disp[i] * s;
        if (min_area(cand, tris, nt) <= 1e-12) continue;
        orc_self_intersects(cand, nv, tris, nt, &r, NULL, 0, NULL);
        if (!r) {
            memcpy(pos_out, cand, sizeof(double) * 3 * (size_t)nv);
            *scale_out = s;
            break;
        }
    }
    free(cand);
    return 0;
}

/* ---- Bvh::closest_point (bvh.cpp:267-329) by brute force, SURVEY §8(f) row 4.
 * Ties go to the lowest triangle index. Outputs nullable. */
static d3 closest_on_tri(d3 p, d3 a, d3 b, d3 c) { /* mesh.cpp:96-126 */
    d3 ab = sub3(b, a), ac = sub3(c, a), ap = sub3(p, a);
    double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
    if (d1 <= 0 && d2 <= 0) return a;
    d3 bp = sub3(p, b);
    double d3_ = dot3(ab, bp), d4 = dot3(ac, bp);
    if (d3_ >= 0 && d4 <= d3_) return b;
    double vc = d1 * d4 - d3_ * d2;
    if (vc <= 0 && d1 >= 0 && d3_ <= 0) return add3(a, mul3(ab, d1 / (d1 - d3_)));
    d3 cp = sub3(p, c);
    double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    if (d6 >= 0 && d5 <= d6) return c;
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) return add3(a, mul3(ac, d2 / (d2 - d6)));
    double va = d3_ * d6 - d5 * d4;
    if (va <= 0 && (d4 - d3_) >= 0 && (d5 - d6) >= 0)
        return add3(b, mul3(sub3(c, b), (d4 - d3_) / ((d4 - d3_) + (d5 - d6))));
    double denom = 1.0 / (va + vb + vc);
    double v = vb * denom, w = vc * denom;
    return add3(add3(a, mul3(ab, v)), mul3(ac, w));
}

static double clamp01d(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }

int orc_closest_points(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* q, int32_t nq,
                       int32_t* tri_out, double* point_out, double* dist_out, double* bary_out) {
    (void)nv;
    for (int i = 0; i < nq; ++i) {
        d3 p = ld3(q + 3 * (size_t)i), bp = v3(0, 0, 0);
        double best = 1e300;
        int bt = -1;
        for (int f = 0; f < nt; ++f) {
            const int32_t* t = tris + 3 * (size_t)f;
            d3 cp = closest_on_tri(p, ld3(pos + 3 * (size_t)t[0]), ld3(pos + 3 * (size_t)t[1]),
                                   ld3(pos + 3 * (size_t)t[2]));
            double d = len3(sub3(p, cp));
            if (d < best) { best = d; bt = f; bp = cp; }
        }
        double b0 = 0, b1 = 0, b2 = 0;
        if (bt >= 0) { /* bvh.cpp:312-326 */
            const int32_t* t = tris + 3 * (size_t)bt;
            d3 a = ld3(pos + 3 * (size_t)t[0]);
            d3 v0 = sub3(ld3(pos + 3 * (size_t)t[1]), a), v1 = sub3(ld3(pos + 3 * (size_t)t[2]), a), v2 = sub3(bp, a);
            double d00 = dot3(v0, v0), d01 = dot3(v0, v1), d11 = dot3(v1, v1), d20 = dot3(v2, v0), d21 = dot3(v2, v1);
            double den = d00 * d11 - d01 * d01;
            if (fabs(den) > 1e-30) {
                b1 = clamp01d((d11 * d20 - d01 * d21) / den);
                b2 = clamp01d((d00 * d21 - d01 * d20) / den);
            }
            b0 = clamp01d(1.0 - b1 - b2);
        }
        if (tri_out) tri_out[i] = bt;
        if (dist_out) dist_out[i] = best;
        if (point_out) { point_out[3 * i] = bp.x; point_out[3 * i + 1] = bp.y; point_out[3 * i + 2] = bp.z; }
        if (bary_out) { bary_out[3 * i] = b0; bary_out[3 * i + 1] = b1; bary_out[3 * i + 2] = b2; }
    }
    return 0;
}

/* build_adjacency (mesh.cpp:27-63): edges sorted by (min, max); faces in
 * ascending face order; f1 = -1 on boundary; -1 return = non-manifold. */
typedef struct { int64_t key; int f; } ekey;
static int cmp_ekey(const void* a, const void* b) {
    const ekey* x = (const ekey*)a;
    const ekey* y = (const ekey*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->f - y->f;
}
int orc_adjacency(int32_t nv, int32_t nt, const int32_t* tris, int32_t* edges_out, int32_t* ne) {
    ekey* ks = (ekey*)malloc(sizeof(ekey) * 3 * ((size_t)nt + 1));
    for (int f = 0; f < nt; ++f)
        for (int k = 0; k < 3; ++k) {
            int a = tris[3 * f + k], b = tris[3 * f + (k + 1) % 3];
            int lo = a < b ? a : b, hi = a < b ? b : a;
            ks[3 * f + k].key = (int64_t)lo * nv + hi;
            ks[3 * f + k].f = f;
        }
    qsort(ks, 3 * (size_t)nt, sizeof(ekey), cmp_ekey);
    int n = 0;
    for (size_t i = 0; i < 3 * (size_t)nt;) {
        size_t j = i;
        while (j < 3 * (size_t)nt && ks[j].key == ks[i].key) ++j;
        if (j - i > 2) { free(ks); return -1; }
        if (edges_out) {
            edges_out[4 * n] = (int32_t)(ks[i].key / nv);
            edges_out[4 * n + 1] = (int32_t)(ks[i].key % nv);
            edges_out[4 * n + 2] = ks[i].f;
            edges_out[4 * n + 3] = j - i > 1 ? ks[i + 1].f : -1;
        }
        ++n;
        i = j;
    }
    *ne = n;
    free(ks);
    return 0;
}

/* ---- exported primitives for the known-answer tests ------------------------ */
double orc_tone_map(double v, double gamma) { return tone(v, gamma); }
double orc_tone_map_derivative(double v, double gamma) { return tone_d(v, gamma); }
int orc_project(const cdr_camera* cam, const double* p, double* q, double* depth) {
    d2 r;
    int ok = project(cam, ld3(p), &r, depth);
    if (ok) { q[0] = r.x; q[1] = r.y; }
    return ok;
}
void orc_projection_jacobian(const cdr_camera* cam, const double* p, double* out) {
    d3 a, b;
    projection_jacobian(cam, ld3(p), &a, &b);
    out[0] = a.x; out[1] = a.y; out[2] = a.z;
    out[3] = b.x; out[4] = b.y; out[5] = b.z;
}
int orc_ray_triangle(const double* o, const double* d, const double* p0, const double* p1,
                     const double* p2, double* tbb) {
    return ray_triangle(ld3(o), ld3(d), ld3(p0), ld3(p1), ld3(p2), &tbb[0], &tbb[1], &tbb[2]);
}
