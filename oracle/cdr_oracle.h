/*
 * cdr_oracle.h — CPU restatement of the reference hot path (test oracle).
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER. The product (libcdr.so) never
 * links or calls it.
 *
 * Parity pin: every function is checked against the reference compiled from
 * its own sources (oracle/_ref, tests/test_oracle_vs_ref.py) and against the
 * golden fixtures in tests/golden/ generated from it.
 */
#ifndef CDR_ORACLE_H
#define CDR_ORACLE_H

#include <stdint.h>

#include "../include/cdr.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_scene {
    int32_t nv, nt, ne;
    const double* pos;     /* nv x 3 */
    const int32_t* tris;   /* nt x 3 */
    const double* uv;      /* nv x 2 or NULL */
    const int32_t* edges;  /* ne x 4 (v0, v1, f0, f1), build_adjacency order */
    int32_t tw, th;
    const double* diffuse;   /* tw*th*3 */
    const double* specular;  /* tw*th*3 */
    const double* roughness; /* tw*th */
    double light[3];
    double background[3];
    int32_t nviews;
    const cdr_camera* cams;
    const int32_t* view_ids; /* global ids for RNG keys, NULL = slot index */
} orc_scene;

typedef struct orc_ctx orc_ctx;

/* GradContext equivalent (diff_render.hpp:25-31): normals + BVH + t_min. */
orc_ctx* orc_ctx_new(const orc_scene* s);
void orc_ctx_free(orc_ctx* c);
double orc_t_min(const orc_ctx* c);
const char* orc_last_error(void);

void orc_vertex_normals(const orc_scene* s, double* out);
int orc_adjacency(int32_t nv, int32_t nt, const int32_t* tris, int32_t* edges_out, int32_t* ne);
int orc_intersect(const orc_ctx* c, int32_t n, const double* orig, const double* dir,
                  double t_min, int32_t* tri, double* t, double* b1, double* b2);
int orc_intersect_brute(const orc_ctx* c, int32_t n, const double* orig, const double* dir,
                        double t_min, int32_t* tri, double* t, double* b1, double* b2);
void orc_pixel_sample_position(uint64_t seed, int32_t view, int32_t px, int32_t py,
                               int32_t width, int32_t sample, int32_t spp, double* out);
void orc_rng(uint64_t seed, int32_t nk, const uint64_t* keys, int32_t n, uint64_t* out);
void orc_primary_ray(const cdr_camera* cam, double x, double y, double* dir);
void orc_eval_brdf(const double* ad, const double* as, double alpha, double mu, double* out);
void orc_sample_texture(const double* data, int32_t w, int32_t h, int32_t ch, double u,
                        double v, double* out, int32_t* texels);
int orc_radiance_at(const orc_ctx* c, int32_t view, int32_t n, const double* xy, double* rgb,
                    int32_t* tri);
int orc_render(const orc_ctx* c, int32_t view, int32_t spp, uint64_t seed, double* rgb,
               double* mask, int32_t* hit);
int orc_view_loss(int32_t w, int32_t h, const double* rendered, const double* target,
                  const double* target_mask, double lambda, double gamma, int32_t use_mask,
                  double* value, double* adjoint);
int orc_interior(const orc_ctx* c, int32_t view, const double* adjoint, int32_t spp,
                 uint64_t seed, const int32_t* hit, const cdr_layout* layout, double* grad);
int orc_silhouettes(const orc_ctx* c, int32_t view, cdr_segment* out, int32_t cap,
                    int32_t* count, double* total);
int orc_boundary(const orc_ctx* c, int32_t view, const double* adjoint, int32_t samples,
                 uint64_t seed, int32_t probe, const cdr_layout* layout, double* grad,
                 int32_t* degenerate);
int orc_boundary_segs(const orc_ctx* c, int32_t view, const double* adjoint, const cdr_segment* segs,
                      int32_t nseg, double total_length, int32_t samples, uint64_t seed, int32_t probe,
                      const cdr_layout* layout, double* grad, int32_t* degenerate);
int orc_laplacian(const orc_scene* s, int32_t mode, double lambda, double* value, double* grad,
                  int32_t* outer, int32_t* inner, double* vals);
/* normal_consistency / edge_length / specular_correlation / roughness_tv
 * (losses.cpp:80-238). w = normal, edge, spec, roug, sigma1, sigma2; values[4];
 * gradients written (any may be NULL). */
int orc_regularisers(const orc_scene* s, const double* w, double* values, double* grad_pos, double* grad_d,
                     double* grad_s, double* grad_r);
/* self_intersects / triangles_intersect (mesh.cpp:137-214): brute force, pairs
 * sorted by (f, g); pairs / n_pairs may be NULL. */
int orc_triangles_intersect(const double* a0, const double* a1, const double* a2, const double* b0,
                            const double* b1, const double* b2, double tol);
int orc_self_intersects(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, int32_t* result,
                        int32_t* pairs, int64_t cap, int64_t* n_pairs);
/* adam_step (adam.cpp:9-54) and robust_evolve (evolve.cpp:19-53). */
int orc_adam_step(const double* cfg, const cdr_layout* L, int64_t nv, int64_t n_tex, int64_t* step, double* m,
                  double* v, const double* params, const double* grad, double* params_out, double* disp_out);
int orc_robust_evolve(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* disp,
                      double* pos_out, double* scale_out);
/* Bvh::closest_point (bvh.cpp:267-329), brute force, ties to the lowest index. */
int orc_closest_points(const double* pos, int32_t nv, const int32_t* tris, int32_t nt, const double* q, int32_t nq,
                       int32_t* tri_out, double* point_out, double* dist_out, double* bary_out);
double orc_tone_map(double v, double gamma);
double orc_tone_map_derivative(double v, double gamma);
int orc_project(const cdr_camera* cam, const double* p, double* q, double* depth);
void orc_projection_jacobian(const cdr_camera* cam, const double* p, double* out);
int orc_ray_triangle(const double* o, const double* d, const double* p0, const double* p1,
                     const double* p2, double* tbb);
int orc_loss_grad(const orc_ctx* c, const double* targets_rgb, const double* targets_mask,
                  const cdr_settings* st, double lambda_rend, double lambda_lap,
                  int32_t lap_mode, int32_t use_mask, const cdr_layout* layout,
                  double* loss_out, double* grad, double* rendered);

#ifdef __cplusplus
}
#endif
#endif
