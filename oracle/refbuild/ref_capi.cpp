// oracle/_ref driver: a flat extern "C" surface over the UNMODIFIED reference
// library compiled from /root/reference/proj/src (see oracle/refbuild/Makefile).
//
// TEST INFRASTRUCTURE ONLY. It is loaded by tests/ (to pin the C restatement
// in oracle/cdr_oracle.c and the CUDA path) and by bench.py's reference /
// cpu_baseline leg. It never participates in the product path.
//
// Every ref_* call forwards to the reference function named beside it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "cdr.h"
#include "collodiff/bvh.hpp"
#include "collodiff/camera.hpp"
#include "collodiff/diff_render.hpp"
#include "collodiff/errors.hpp"
#include "collodiff/laplacian.hpp"
#include "collodiff/losses.hpp"
#include "collodiff/material.hpp"
#include "collodiff/mesh.hpp"
#include "collodiff/optimize.hpp"
#include "collodiff/params.hpp"
#include "collodiff/render.hpp"
#include "collodiff/rng.hpp"
#include "collodiff/scene.hpp"
#include "collodiff/silhouette.hpp"
#include "collodiff/texture.hpp"

using namespace collodiff;

namespace {

thread_local std::string g_err;

struct RefScene {
    Scene scene;
    std::unique_ptr<GradContext> ctx;  // lazily built per positions version
    GradContext& grad_ctx() {
        if (!ctx) ctx = std::make_unique<GradContext>(scene);
        return *ctx;
    }
};

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const SizeMismatch*>(&e)) return CDR_ERR_SIZE_MISMATCH;
    if (dynamic_cast<const NonFiniteGradient*>(&e)) return CDR_ERR_NONFINITE;
    if (dynamic_cast<const InputSelfIntersecting*>(&e)) return CDR_ERR_SELF_INTERSECTING;
    if (dynamic_cast<const ProjectionTooFar*>(&e)) return CDR_ERR_PROJECTION_TOO_FAR;
    return CDR_ERR_ERROR;
}

#define GUARD(...)                           \
    try {                                    \
        __VA_ARGS__;                         \
        return CDR_OK;                       \
    } catch (const std::exception& e) {      \
        return fail(e);                      \
    }

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }

Texture make_tex(const double* data, int w, int h, int ch) {
    Texture t;
    t.width = w;
    t.height = h;
    t.channels = ch;
    t.data.assign(data, data + size_t(w) * h * ch);
    return t;
}

Camera make_cam(const cdr_camera& c) {
    Camera cam;
    cam.origin = v3(c.origin);
    cam.right = v3(c.right);
    cam.up = v3(c.up);
    cam.forward = v3(c.forward);
    cam.fov_deg = c.fov_deg;
    cam.width = c.width;
    cam.height = c.height;
    return cam;
}

void to_cam(const Camera& cam, cdr_camera* c) {
    const Vec3* vs[4] = {&cam.origin, &cam.right, &cam.up, &cam.forward};
    double* outs[4] = {c->origin, c->right, c->up, c->forward};
    for (int i = 0; i < 4; ++i) {
        outs[i][0] = vs[i]->x;
        outs[i][1] = vs[i]->y;
        outs[i][2] = vs[i]->z;
    }
    c->fov_deg = cam.fov_deg;
    c->width = cam.width;
    c->height = cam.height;
}

RenderSettings make_settings(int spp, uint64_t seed, int threads) {
    RenderSettings s;
    s.spp = spp;
    s.seed = seed;
    s.threads = threads;
    return s;
}

Image image_from(const double* rgb, const double* mask, int w, int h) {
    Image img(w, h, mask != nullptr);
    for (size_t i = 0; i < size_t(w) * h; ++i) {
        img.pixels[i] = v3(rgb + 3 * i);
        if (mask) img.mask[i] = mask[i];
    }
    return img;
}

void image_to(const Image& img, double* rgb, double* mask) {
    for (size_t i = 0; i < img.pixels.size(); ++i) {
        if (rgb) {
            rgb[3 * i] = img.pixels[i].x;
            rgb[3 * i + 1] = img.pixels[i].y;
            rgb[3 * i + 2] = img.pixels[i].z;
        }
        if (mask && img.has_mask()) mask[i] = img.mask[i];
    }
}

std::shared_ptr<const ParamLayout> layout_for(const Scene& s, int optimize_light) {
    return ParamLayout::for_scene(s, optimize_light != 0);
}

void copy_mesh(const Mesh& m, double* pos, double* uv, int32_t* tris) {
    for (int i = 0; i < m.vertex_count(); ++i) {
        if (pos) {
            pos[3 * i] = m.positions[i].x;
            pos[3 * i + 1] = m.positions[i].y;
            pos[3 * i + 2] = m.positions[i].z;
        }
        if (uv && m.uvs.size() == m.positions.size()) {
            uv[2 * i] = m.uvs[i].x;
            uv[2 * i + 1] = m.uvs[i].y;
        }
    }
    if (tris)
        for (int f = 0; f < m.triangle_count(); ++f)
            for (int k = 0; k < 3; ++k) tris[3 * f + k] = m.triangles[f][k];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Scene aggregate (scene.hpp:17-23) from flat arrays; build_adjacency
// (mesh.cpp:27-63) runs so silhouettes / Laplacian have the reference's edges.
int ref_scene_new(const double* pos, int32_t nv, const int32_t* tris, int32_t nt,
                  const double* uv, const double* diffuse, const double* specular,
                  const double* roughness, int32_t tw, int32_t th, const double* light,
                  const double* background, const cdr_camera* cams, int32_t nviews,
                  void** out) {
    GUARD({
        auto rs = std::make_unique<RefScene>();
        Mesh& m = rs->scene.mesh;
        m.positions.resize(nv);
        for (int i = 0; i < nv; ++i) m.positions[i] = v3(pos + 3 * i);
        if (uv) {
            m.uvs.resize(nv);
            for (int i = 0; i < nv; ++i) m.uvs[i] = Vec2(uv[2 * i], uv[2 * i + 1]);
        }
        m.triangles.resize(nt);
        for (int f = 0; f < nt; ++f) m.triangles[f] = {tris[3 * f], tris[3 * f + 1], tris[3 * f + 2]};
        build_adjacency(m);
        rs->scene.maps.diffuse = make_tex(diffuse, tw, th, 3);
        rs->scene.maps.specular = make_tex(specular, tw, th, 3);
        rs->scene.maps.roughness = make_tex(roughness, tw, th, 1);
        rs->scene.light.intensity = v3(light);
        rs->scene.background = v3(background);
        for (int k = 0; k < nviews; ++k) rs->scene.views.push_back(make_cam(cams[k]));
        *out = rs.release();
    })
}

void ref_scene_free(void* s) { delete static_cast<RefScene*>(s); }

int ref_set_positions(void* s, const double* pos) {
    auto* rs = static_cast<RefScene*>(s);
    for (int i = 0; i < rs->scene.mesh.vertex_count(); ++i) rs->scene.mesh.positions[i] = v3(pos + 3 * i);
    rs->ctx.reset();
    return CDR_OK;
}

int32_t ref_edge_count(void* s) { return int32_t(static_cast<RefScene*>(s)->scene.mesh.edges.size()); }

int ref_edges(void* s, int32_t* out) {
    const auto& es = static_cast<RefScene*>(s)->scene.mesh.edges;
    for (size_t i = 0; i < es.size(); ++i) {
        out[4 * i] = es[i].v0;
        out[4 * i + 1] = es[i].v1;
        out[4 * i + 2] = es[i].f0;
        out[4 * i + 3] = es[i].f1;
    }
    return CDR_OK;
}

// vertex_normals (mesh.cpp:65-95)
int ref_vertex_normals(void* s, double* out) {
    GUARD({
        auto n = vertex_normals(static_cast<RefScene*>(s)->scene.mesh);
        for (size_t i = 0; i < n.size(); ++i) {
            out[3 * i] = n[i].x;
            out[3 * i + 1] = n[i].y;
            out[3 * i + 2] = n[i].z;
        }
    })
}

// Bvh::default_t_min (bvh.cpp:92)
double ref_default_t_min(void* s) {
    return static_cast<RefScene*>(s)->grad_ctx().geom.bvh.default_t_min();
}

// Bvh::intersect (bvh.cpp:210-265) on n rays (o, d) with the scene's shading
// normals; t_min < 0 -> default.
int ref_intersect(void* s, int32_t n, const double* orig, const double* dir, double t_min,
                  int32_t* tri, double* t, double* b1, double* b2) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        auto& g = rs->grad_ctx().geom;
        for (int i = 0; i < n; ++i) {
            auto h = g.bvh.intersect(rs->scene.mesh, v3(orig + 3 * i), v3(dir + 3 * i), &g.normals, t_min);
            tri[i] = h ? h->tri : -1;
            t[i] = h ? h->t : 0;
            b1[i] = h ? h->b1 : 0;
            b2[i] = h ? h->b2 : 0;
        }
    })
}

// ray_triangle (bvh.cpp:11-26)
int ref_ray_triangle(const double* o, const double* d, const double* p0, const double* p1,
                     const double* p2, double* tbb) {
    double t = 0, b1 = 0, b2 = 0;
    bool hit = ray_triangle(v3(o), v3(d), v3(p0), v3(p1), v3(p2), t, b1, b2);
    tbb[0] = t;
    tbb[1] = b1;
    tbb[2] = b2;
    return hit ? 1 : 0;
}

// pixel_sample_position (render.cpp:10-22)
void ref_pixel_sample_position(uint64_t seed, int32_t view, int32_t px, int32_t py, int32_t width,
                               int32_t sample, int32_t spp, double* out) {
    Vec2 p = pixel_sample_position(seed, view, px, py, width, sample, spp);
    out[0] = p.x;
    out[1] = p.y;
}

// Rng stream (rng.hpp:20-36): n draws of next_u64 for a key tuple of length nk
void ref_rng(uint64_t seed, int32_t nk, const uint64_t* keys, int32_t n, uint64_t* out) {
    auto gen = [&](auto rng) {
        for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
    };
    if (nk == 0) gen(Rng(seed));
    else if (nk == 1) gen(Rng(seed, keys[0]));
    else if (nk == 2) gen(Rng(seed, keys[0], keys[1]));
    else gen(Rng(seed, keys[0], keys[1], keys[2]));
}

// primary_ray (camera.cpp:29-34)
void ref_primary_ray(const cdr_camera* c, double x, double y, double* dir_out) {
    Ray r = primary_ray(make_cam(*c), Vec2(x, y));
    dir_out[0] = r.dir.x;
    dir_out[1] = r.dir.y;
    dir_out[2] = r.dir.z;
}

// project (camera.cpp:36-45): returns 0 when behind the camera
int ref_project(const cdr_camera* c, const double* p, double* q, double* depth) {
    auto r = project(make_cam(*c), v3(p), depth);
    if (!r) return 0;
    q[0] = r->x;
    q[1] = r->y;
    return 1;
}

// projection_jacobian (camera.cpp:47-59): out = d_px (3), d_py (3)
void ref_projection_jacobian(const cdr_camera* c, const double* p, double* out) {
    auto j = projection_jacobian(make_cam(*c), v3(p));
    out[0] = j.d_px.x; out[1] = j.d_px.y; out[2] = j.d_px.z;
    out[3] = j.d_py.x; out[4] = j.d_py.y; out[5] = j.d_py.z;
}

// sample_views_on_sphere (camera.cpp:61-77)
int ref_sample_views_on_sphere(int32_t count, double radius, uint64_t seed, double fov,
                               int32_t w, int32_t h, cdr_camera* out) {
    GUARD({
        auto cams = sample_views_on_sphere(count, radius, seed, fov, w, h);
        for (int i = 0; i < count; ++i) to_cam(cams[i], out + i);
    })
}

// eval_brdf (material.cpp:22-57): out = value3, d_diffuse, d_specular, d_rough3, d_mu3
void ref_eval_brdf(const double* ad, const double* as, double alpha, double mu, double* out) {
    BrdfEval e = eval_brdf(v3(ad), v3(as), alpha, mu);
    out[0] = e.value.x; out[1] = e.value.y; out[2] = e.value.z;
    out[3] = e.d_diffuse;
    out[4] = e.d_specular;
    out[5] = e.d_roughness.x; out[6] = e.d_roughness.y; out[7] = e.d_roughness.z;
    out[8] = e.d_mu.x; out[9] = e.d_mu.y; out[10] = e.d_mu.z;
}

// sample_texture (texture.cpp:34-69). out = value3, du3, dv3, weights4; texels4
void ref_sample_texture(const double* data, int32_t w, int32_t h, int32_t ch, double u, double v,
                        double* out, int32_t* texels) {
    Texture t = make_tex(data, w, h, ch);
    TexSample s = sample_texture(t, Vec2(u, v));
    out[0] = s.value.x; out[1] = s.value.y; out[2] = s.value.z;
    out[3] = s.du.x; out[4] = s.du.y; out[5] = s.du.z;
    out[6] = s.dv.x; out[7] = s.dv.y; out[8] = s.dv.z;
    for (int k = 0; k < 4; ++k) {
        out[9 + k] = s.weight[k];
        texels[k] = s.texel[k];
    }
}

// tone_map_scalar / tone_map_derivative (render.cpp:66-73)
double ref_tone_map(double v, double gamma) { return tone_map_scalar(v, gamma); }
double ref_tone_map_derivative(double v, double gamma) { return tone_map_derivative(v, gamma); }

// radiance_at (render.cpp:24-33)
int ref_radiance_at(void* s, int32_t view, int32_t n, const double* xy, double* rgb, int32_t* tri) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        auto& g = rs->grad_ctx().geom;
        for (int i = 0; i < n; ++i) {
            std::optional<HitRecord> hit;
            Vec3 r = radiance_at(rs->scene, g, view, Vec2(xy[2 * i], xy[2 * i + 1]), &hit);
            rgb[3 * i] = r.x;
            rgb[3 * i + 1] = r.y;
            rgb[3 * i + 2] = r.z;
            if (tri) tri[i] = hit ? hit->tri : -1;
        }
    })
}

// render (render.cpp:35-64)
int ref_render(void* s, int32_t view, int32_t spp, uint64_t seed, int32_t threads, double* rgb,
               double* mask, int32_t* hit) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        std::vector<int> cache;
        Image img = render(rs->scene, rs->grad_ctx().geom, view, make_settings(spp, seed, threads),
                           hit ? &cache : nullptr);
        image_to(img, rgb, mask);
        if (hit) std::memcpy(hit, cache.data(), cache.size() * sizeof(int));
    })
}

// view_rendering_loss (losses.cpp:15-49)
int ref_view_loss(int32_t w, int32_t h, const double* rendered, const double* target,
                  const double* target_mask, double lambda, double gamma, int32_t use_mask,
                  double* value, double* adjoint) {
    GUARD({
        Image r = image_from(rendered, nullptr, w, h);
        Image t = image_from(target, target_mask, w, h);
        ViewLossResult vl = view_rendering_loss(r, t, lambda, gamma, use_mask != 0);
        *value = vl.value;
        image_to(vl.adjoint, adjoint, nullptr);
    })
}

// interior_pass (diff_render.cpp:62-201); grad is the layout-sized buffer (+=)
int ref_interior(void* s, int32_t view, const double* adjoint, int32_t spp, uint64_t seed,
                 int32_t threads, const int32_t* hit, int64_t hit_len, int32_t optimize_light,
                 double* grad) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        const Camera& cam = rs->scene.views[view];
        Image adj = image_from(adjoint, nullptr, cam.width, cam.height);
        std::vector<int> cache(hit, hit + hit_len);
        GradVector g(layout_for(rs->scene, optimize_light));
        std::memcpy(g.values.data(), grad, g.values.size() * sizeof(double));
        interior_pass(rs->scene, rs->grad_ctx(), view, adj, make_settings(spp, seed, threads), cache, g);
        std::memcpy(grad, g.values.data(), g.values.size() * sizeof(double));
    })
}

// extract_silhouettes (silhouette.cpp:55-106)
int ref_silhouettes(void* s, int32_t view, cdr_segment* out, int32_t cap, int32_t* count,
                    double* total) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        SilhouetteSet set = extract_silhouettes(rs->scene.mesh, rs->scene.views[view]);
        *count = int32_t(set.segments.size());
        *total = set.total_length;
        for (int i = 0; i < std::min<int>(cap, *count); ++i) {
            const auto& g = set.segments[i];
            cdr_segment& o = out[i];
            o.v0 = g.v0;
            o.v1 = g.v1;
            o.p0[0] = g.p0.x; o.p0[1] = g.p0.y; o.p0[2] = g.p0.z;
            o.p1[0] = g.p1.x; o.p1[1] = g.p1.y; o.p1[2] = g.p1.z;
            o.t0 = g.t0;
            o.t1 = g.t1;
            o.q0[0] = g.q0.x; o.q0[1] = g.q0.y;
            o.q1[0] = g.q1.x; o.q1[1] = g.q1.y;
            o.z0 = g.z0;
            o.z1 = g.z1;
            o.length_px = g.length_px;
        }
    })
}

// boundary_pass (diff_render.cpp:203-283) with the reference's own silhouettes
int ref_boundary(void* s, int32_t view, const double* adjoint, int32_t samples, uint64_t seed,
                 int32_t probe, int32_t optimize_light, double* grad, int32_t* degenerate) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        const Camera& cam = rs->scene.views[view];
        Image adj = image_from(adjoint, nullptr, cam.width, cam.height);
        SilhouetteSet set = extract_silhouettes(rs->scene.mesh, cam);
        GradVector g(layout_for(rs->scene, optimize_light));
        std::memcpy(g.values.data(), grad, g.values.size() * sizeof(double));
        BoundaryStats st = boundary_pass(rs->scene, rs->grad_ctx(), view, adj, set, samples, seed, g,
                                         probe ? BoundaryProbe::Coverage : BoundaryProbe::Radiance);
        if (degenerate) *degenerate = st.degenerate_skipped;
        std::memcpy(grad, g.values.data(), g.values.size() * sizeof(double));
    })
}

// cotangent_laplacian (laplacian.cpp:21-55) as CSC + laplacian_loss (losses.cpp:66-78)
int ref_laplacian(void* s, int32_t mode, double lambda, double* value, double* grad,
                  int32_t* outer, int32_t* inner, double* vals, int64_t* nnz) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        auto L = cotangent_laplacian(rs->scene.mesh,
                                     mode ? LaplacianMode::Uniform : LaplacianMode::Cotangent);
        if (nnz) *nnz = L.nonZeros();
        if (outer) std::memcpy(outer, L.outer().data(), L.outer().size() * sizeof(int));
        if (inner) std::memcpy(inner, L.inner().data(), L.inner().size() * sizeof(int));
        if (vals) std::memcpy(vals, L.values().data(), L.values().size() * sizeof(double));
        MeshLossResult r = laplacian_loss(rs->scene.mesh, L, lambda);
        if (value) *value = r.value;
        if (grad)
            for (size_t i = 0; i < r.grad.size(); ++i) {
                grad[3 * i] = r.grad[i].x;
                grad[3 * i + 1] = r.grad[i].y;
                grad[3 * i + 2] = r.grad[i].z;
            }
    })
}

// The four mesh/material regularisers (losses.cpp:80-238) with explicit
// sigmas. w = normal, edge, spec, roug, sigma1, sigma2. Gradients written
// (positions: nrm + edg as total_loss sums them, losses.cpp:276).
int ref_regularisers(void* s, const double* w, double* values, double* grad_pos, double* grad_d,
                     double* grad_s, double* grad_r) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        const Scene& sc = rs->scene;
        MeshLossResult nrm = normal_consistency_loss(sc.mesh, w[0]);
        MeshLossResult edg = edge_length_loss(sc.mesh, w[1]);
        LossWeights lw;
        lw.spec = w[2];
        lw.sigma1 = w[4];
        lw.sigma2 = w[5];
        SpecularLossResult spec = specular_correlation_loss(sc.maps, lw);
        RoughnessLossResult roug = roughness_tv_loss(sc.maps, w[3]);
        values[0] = nrm.value;
        values[1] = edg.value;
        values[2] = spec.value;
        values[3] = roug.value;
        if (grad_pos)
            for (size_t v = 0; v < nrm.grad.size(); ++v) {
                Vec3 g = nrm.grad[v] + edg.grad[v];
                grad_pos[3 * v] = g.x;
                grad_pos[3 * v + 1] = g.y;
                grad_pos[3 * v + 2] = g.z;
            }
        if (grad_d) std::memcpy(grad_d, spec.grad_diffuse.data.data(), spec.grad_diffuse.data.size() * sizeof(double));
        if (grad_s)
            std::memcpy(grad_s, spec.grad_specular.data.data(), spec.grad_specular.data.size() * sizeof(double));
        if (grad_r) std::memcpy(grad_r, roug.grad.data.data(), roug.grad.data.size() * sizeof(double));
    })
}

// self_intersects (mesh.cpp:184-214) with pairs, sorted by (f, g) for
// comparison (the reference's order follows its BVH traversal), and
// triangles_intersect (mesh.cpp:160-182).
int ref_self_intersects(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, int32_t* result,
                        int32_t* pairs, int64_t cap, int64_t* n_pairs) {
    GUARD({
        Mesh m;
        m.positions.resize(nv);
        for (int i = 0; i < nv; ++i) m.positions[i] = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        m.triangles.resize(nt);
        for (int f = 0; f < nt; ++f) m.triangles[f] = {tris[3 * f], tris[3 * f + 1], tris[3 * f + 2]};
        std::vector<std::pair<int, int>> pr;
        const bool want = pairs || n_pairs;
        *result = self_intersects(m, want ? &pr : nullptr) ? 1 : 0;
        std::sort(pr.begin(), pr.end());
        for (int64_t i = 0; i < std::min<int64_t>(cap, int64_t(pr.size())); ++i) {
            pairs[2 * i] = pr[size_t(i)].first;
            pairs[2 * i + 1] = pr[size_t(i)].second;
        }
        if (n_pairs) *n_pairs = int64_t(pr.size());
    })
}

int ref_triangles_intersect(const double* a0, const double* a1, const double* a2, const double* b0,
                            const double* b1, const double* b2, double tol) {
    auto v = [](const double* p) { return Vec3(p[0], p[1], p[2]); };
    return triangles_intersect(v(a0), v(a1), v(a2), v(b0), v(b1), v(b2), tol) ? 1 : 0;
}

// adam_step (adam.cpp:9-54) on a layout of nv vertices and tw x th maps
// (ParamLayout::for_scene). cfg = beta1, beta2, epsilon, lr_positions,
// lr_textures, lr_light; m, v, step updated in place.
int ref_adam_step(const double* cfg, int32_t nv, int32_t tw, int32_t th, int32_t light, int64_t* step, double* m,
                  double* v, const double* params, const double* grad, double* params_out, double* disp_out) {
    GUARD({
        Scene sc;
        sc.mesh.positions.assign(nv, Vec3());
        sc.maps.diffuse = Texture::constant(tw, th, 3, Vec3());
        sc.maps.specular = Texture::constant(tw, th, 3, Vec3());
        sc.maps.roughness = Texture::constant(tw, th, 1, Vec3());
        auto layout = ParamLayout::for_scene(sc, light != 0);
        AdamConfig c;
        c.beta1 = cfg[0];
        c.beta2 = cfg[1];
        c.epsilon = cfg[2];
        c.lr_positions = cfg[3];
        c.lr_textures = cfg[4];
        c.lr_light = cfg[5];
        AdamState st(layout, c);
        const size_t n = layout->total;
        st.m.assign(m, m + n);
        st.v.assign(v, v + n);
        st.step = *step;
        ParamVector pv;
        pv.layout = layout;
        pv.values.assign(params, params + n);
        GradVector gv(layout);
        gv.values.assign(grad, grad + n);
        AdamStepResult out = adam_step(st, pv, gv);
        std::memcpy(m, st.m.data(), n * sizeof(double));
        std::memcpy(v, st.v.data(), n * sizeof(double));
        *step = st.step;
        std::memcpy(params_out, out.params.values.data(), n * sizeof(double));
        for (size_t i = 0; i < out.displacement.size(); ++i) {
            disp_out[3 * i] = out.displacement[i].x;
            disp_out[3 * i + 1] = out.displacement[i].y;
            disp_out[3 * i + 2] = out.displacement[i].z;
        }
    })
}

// robust_evolve (evolve.cpp:19-53)
int ref_robust_evolve(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* disp,
                      double* pos_out, double* scale_out) {
    GUARD({
        Mesh m;
        m.positions.resize(nv);
        for (int i = 0; i < nv; ++i) m.positions[i] = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        m.triangles.resize(nt);
        for (int f = 0; f < nt; ++f) m.triangles[f] = {tris[3 * f], tris[3 * f + 1], tris[3 * f + 2]};
        std::vector<Vec3> d(nv);
        for (int i = 0; i < nv; ++i) d[i] = Vec3(disp[3 * i], disp[3 * i + 1], disp[3 * i + 2]);
        Mesh out = robust_evolve(m, d, scale_out);
        for (int i = 0; i < nv; ++i) {
            pos_out[3 * i] = out.positions[i].x;
            pos_out[3 * i + 1] = out.positions[i].y;
            pos_out[3 * i + 2] = out.positions[i].z;
        }
    })
}

// Bvh::closest_point (bvh.cpp:267-329) for nq queries
int ref_closest_points(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* q, int32_t nq,
                       int32_t* tri_out, double* point_out, double* dist_out, double* bary_out) {
    GUARD({
        Mesh m;
        m.positions.resize(nv);
        for (int i = 0; i < nv; ++i) m.positions[i] = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        m.triangles.resize(nt);
        for (int f = 0; f < nt; ++f) m.triangles[f] = {tris[3 * f], tris[3 * f + 1], tris[3 * f + 2]};
        Bvh bvh(m);
        for (int i = 0; i < nq; ++i) {
            ClosestPoint cp = bvh.closest_point(m, Vec3(q[3 * i], q[3 * i + 1], q[3 * i + 2]));
            tri_out[i] = cp.tri;
            dist_out[i] = cp.distance;
            point_out[3 * i] = cp.point.x;
            point_out[3 * i + 1] = cp.point.y;
            point_out[3 * i + 2] = cp.point.z;
            bary_out[3 * i] = cp.b0;
            bary_out[3 * i + 1] = cp.b1;
            bary_out[3 * i + 2] = cp.b2;
        }
    })
}

// point_to_mesh_distance (mesh.cpp:127-133) and uv_transfer (remesh.cpp:281-294)
int ref_point_to_mesh(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* q, int32_t nq,
                      double* out) {
    GUARD({
        Mesh m;
        m.positions.resize(nv);
        for (int i = 0; i < nv; ++i) m.positions[i] = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        m.triangles.resize(nt);
        for (int f = 0; f < nt; ++f) m.triangles[f] = {tris[3 * f], tris[3 * f + 1], tris[3 * f + 2]};
        std::vector<Vec3> pts(nq);
        for (int i = 0; i < nq; ++i) pts[i] = Vec3(q[3 * i], q[3 * i + 1], q[3 * i + 2]);
        *out = point_to_mesh_distance(pts, m);
    })
}

int ref_uv_transfer(const double* opos, int32_t onv, const int32_t* otris, int32_t ont, const double* ouv,
                    const double* npos, int32_t nnv, double max_distance, double* uv_out) {
    GUARD({
        Mesh o, n;
        o.positions.resize(onv);
        o.uvs.resize(onv);
        for (int i = 0; i < onv; ++i) {
            o.positions[i] = Vec3(opos[3 * i], opos[3 * i + 1], opos[3 * i + 2]);
            o.uvs[i] = Vec2(ouv[2 * i], ouv[2 * i + 1]);
        }
        o.triangles.resize(ont);
        for (int f = 0; f < ont; ++f) o.triangles[f] = {otris[3 * f], otris[3 * f + 1], otris[3 * f + 2]};
        n.positions.resize(nnv);
        for (int i = 0; i < nnv; ++i) n.positions[i] = Vec3(npos[3 * i], npos[3 * i + 1], npos[3 * i + 2]);
        uv_transfer(o, n, max_distance);
        for (int i = 0; i < nnv; ++i) {
            uv_out[2 * i] = n.uvs[i].x;
            uv_out[2 * i + 1] = n.uvs[i].y;
        }
    })
}

// total_loss (losses.cpp:244-297). weights[0..5] = rend, lap, normal, edge,
// spec, roug (sigma1/2 stay default). breakdown[0..6] = total, rend, lap,
// normal, edge, spec, roug. grad is written (fresh GradVector, losses.cpp:250).
int ref_total_loss(void* s, const double* targets_rgb, const double* targets_mask, int32_t spp,
                   uint64_t seed, int32_t threads, int32_t boundary_term, int32_t boundary_samples,
                   double gamma, const double* weights, int32_t use_masks, int32_t lap_mode,
                   int32_t optimize_light, double* grad, double* breakdown, double* rendered) {
    GUARD({
        auto* rs = static_cast<RefScene*>(s);
        std::vector<Image> targets;
        size_t off = 0, moff = 0;
        for (const auto& cam : rs->scene.views) {
            targets.push_back(image_from(targets_rgb + off, targets_mask ? targets_mask + moff : nullptr,
                                         cam.width, cam.height));
            off += size_t(cam.width) * cam.height * 3;
            moff += size_t(cam.width) * cam.height;
        }
        LossWeights w;
        w.rend = weights[0];
        w.lap = weights[1];
        w.normal = weights[2];
        w.edge = weights[3];
        w.spec = weights[4];
        w.roug = weights[5];
        LossOptions opt;
        opt.render = make_settings(spp, seed, threads);
        opt.render.gamma = gamma;
        opt.render.boundary_term = boundary_term != 0;
        opt.render.boundary_samples = boundary_samples;
        opt.use_target_masks = use_masks != 0;
        opt.laplacian_mode = lap_mode ? LaplacianMode::Uniform : LaplacianMode::Cotangent;
        TotalLossResult r = total_loss(rs->scene, targets, w, opt, layout_for(rs->scene, optimize_light));
        std::memcpy(grad, r.grad.values.data(), r.grad.values.size() * sizeof(double));
        const LossBreakdown& b = r.breakdown;
        double bd[7] = {b.total, b.rend, b.lap, b.normal, b.edge, b.spec, b.roug};
        std::memcpy(breakdown, bd, sizeof(bd));
        if (rendered) {
            size_t o = 0;
            for (const auto& img : r.rendered) {
                image_to(img, rendered + o, nullptr);
                o += img.pixels.size() * 3;
            }
        }
    })
}

// Procedural meshes (mesh.cpp:270-330). kind 0: make_icosphere(param, radius),
// kind 1: make_blob(param, seed, amplitude). Query sizes with pos == nullptr.
int ref_make_mesh(int32_t kind, int32_t subdiv, double radius_or_amp, uint64_t seed, int32_t* nv,
                  int32_t* nt, double* pos, double* uv, int32_t* tris) {
    GUARD({
        Mesh m = kind == 0 ? make_icosphere(subdiv, radius_or_amp)
                           : make_blob(subdiv, seed, radius_or_amp);
        *nv = m.vertex_count();
        *nt = m.triangle_count();
        if (pos) copy_mesh(m, pos, uv, tris);
    })
}

}  // extern "C"
