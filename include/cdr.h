/*
 * cdr.h — C-ABI of the B200 collocated differentiable renderer (the hot path of
 * arXiv 2103.15208 as implemented by the reference library "collodiff").
 *
 * Plain C types only: pointers, sizes, PODs. Every function returns an int
 * status (CDR_OK = 0); the message of the last failure on a context is
 * available from cdr_last_error(). Status codes map 1:1 onto the reference's
 * exception hierarchy (errors.hpp:8-46):
 *   CDR_ERR_SIZE_MISMATCH  -> collodiff::SizeMismatch       (errors.hpp:24-26)
 *   CDR_ERR_NONFINITE      -> collodiff::NonFiniteGradient  (errors.hpp:28-30)
 *   CDR_ERR_ERROR          -> collodiff::Error              (errors.hpp:8-10)
 *   CDR_ERR_SELF_INTERSECTING  -> collodiff::InputSelfIntersecting (errors.hpp:32-34)
 *   CDR_ERR_PROJECTION_TOO_FAR -> collodiff::ProjectionTooFar      (errors.hpp:40-42)
 *   CDR_ERR_CUDA / _NO_DEVICE / _INVALID_ARG -> collodiff::Error
 *
 * Each entry point names the reference interface it replaces (file:line is
 * relative to /root/reference/proj). The reference is a C++ static library with
 * no FFI of its own; its drop-in binding is the C++ shim described in
 * INTEGRATION.md, which defines the reference symbols on top of these calls.
 *
 * Conventions
 *   - All arithmetic is IEEE fp64 (as the reference); RNG keys are u64.
 *   - Arrays are row-major and AoS: positions V x 3, uvs V x 2, triangles T x 3,
 *     edges E x 4 (v0, v1, f0, f1) in the reference's build_adjacency order
 *     (mesh.cpp:27-63: sorted by (v0, v1), v0 < v1, f1 = -1 on boundary edges).
 *   - Images are W x H x 3 (pixel (x, y) at (y * W + x) * 3), masks W x H,
 *     hit caches W x H x spp pixel-major (render.cpp:44-57).
 *   - Gradients are accumulated (+=) into a caller buffer in ParamLayout order
 *     (params.cpp:30-43); offsets are given by cdr_layout, -1 = segment absent.
 *   - Textures are row-major, top-left origin, channels interleaved
 *     (texture.hpp:11-28). All three maps must share one resolution.
 *   - "view" arguments are slots into the array given to cdr_set_views; RNG
 *     streams use the slot's global view id (render.cpp:12, diff_render.cpp:232),
 *     so results do not depend on how views are sharded across GPUs.
 */
#ifndef CDR_H
#define CDR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDR_ABI_VERSION 2  /* 2: cdr_stats.shaded_samples appended */

enum {
    CDR_OK = 0,
    CDR_ERR_SIZE_MISMATCH = 1,
    CDR_ERR_NONFINITE = 2,
    CDR_ERR_ERROR = 3,
    CDR_ERR_CUDA = 4,
    CDR_ERR_INVALID_ARG = 5,
    CDR_ERR_NO_DEVICE = 6,
    CDR_ERR_SELF_INTERSECTING = 7, /* -> collodiff::InputSelfIntersecting (errors.hpp) */
    CDR_ERR_PROJECTION_TOO_FAR = 8 /* -> collodiff::ProjectionTooFar (errors.hpp) */
};

enum { CDR_PROBE_RADIANCE = 0, CDR_PROBE_COVERAGE = 1 };  /* diff_render.hpp:38 */
enum { CDR_LAPLACIAN_COTANGENT = 0, CDR_LAPLACIAN_UNIFORM = 1 }; /* laplacian.hpp:10 */

typedef struct cdr_ctx cdr_ctx;

/* Pinhole camera (camera.hpp:12-23). tan(fov/2) and the aspect ratio are
 * evaluated on the host exactly as Camera::tan_half_fov (camera.cpp:25-27). */
typedef struct cdr_camera {
    double origin[3];
    double right[3];
    double up[3];
    double forward[3];
    double fov_deg;
    int32_t width;
    int32_t height;
} cdr_camera;

/* cdr_settings.flags */
#define CDR_FLAG_GRAD_OVERWRITE 1 /* cdr_loss_grad / cdr_total_loss: grad_inout receives =
                                     (the fresh GradVector total_loss returns,
                                     losses.cpp:250) instead of +=, and is not read */

/* RenderSettings (render.hpp:27-35); `threads` has no meaning on the GPU. */
typedef struct cdr_settings {
    int32_t spp;
    int32_t boundary_term;    /* 0/1 */
    int32_t boundary_samples; /* 0 -> W*H (diff_render.cpp:300-301) */
    int32_t flags;            /* CDR_FLAG_* */
    uint64_t seed;
    double gamma;
} cdr_settings;

/* ParamLayout segment offsets (params.hpp:25-33, params.cpp:30-43). */
typedef struct cdr_layout {
    int64_t positions; /* 3V */
    int64_t diffuse;   /* 3 * texels */
    int64_t specular;  /* 3 * texels */
    int64_t roughness; /* texels */
    int64_t light;     /* 3, or -1 */
    int64_t total;
} cdr_layout;

/* SilhouetteSegment (silhouette.hpp:14-21), 128 bytes. */
typedef struct cdr_segment {
    int32_t v0, v1;
    double p0[3], p1[3];
    double t0, t1;
    double q0[2], q1[2];
    double z0, z1;
    double length_px;
} cdr_segment;

/* Work counters of the last call (the unit counts of the byte model in
 * DESIGN.md) and the device time of its stages, in milliseconds. */
typedef struct cdr_stats {
    int64_t pixels;
    int64_t samples;
    int64_t hit_samples;
    int64_t adjoint_samples;   /* hit samples whose pixel adjoint is non-zero */
    int64_t boundary_samples;  /* edge samples drawn */
    int64_t boundary_active;   /* edge samples that traced their two probes */
    int64_t segments;
    int32_t degenerate_skipped;
    int32_t nonfinite;         /* 1 if a NonFiniteGradient was raised */
    double ms_prepare;         /* normals + LBVH + t_min */
    double ms_render;          /* trace + fused shade/loss/interior kernels */
    double ms_silhouette;
    double ms_boundary;
    double ms_finalize;        /* normal chain + position gather + Laplacian */
    double ms_total;
    int64_t kernel_launches;   /* kernels this library launched in the call */
    double ms_trace;           /* primary-visibility kernels (part of ms_render) */
    int64_t beam_fallback_tiles; /* pixel tiles traced per ray (candidate-list overflow) */
    int64_t shaded_samples;    /* samples through the full shading kernel; the rest lie in
                                  beam tiles with no candidate triangle (background, no hit read) */
} cdr_stats;

int cdr_abi_version(void);
/* How the library was built: CDR_BUILD_CHECKED = device-side bounds checks on
 * (the test build that stands in for compute-sanitizer). */
#define CDR_BUILD_CHECKED 1
int cdr_build_flags(void);
int cdr_device_count(int* count);

int cdr_create(int device, cdr_ctx** out);
void cdr_destroy(cdr_ctx* ctx);
const char* cdr_last_error(const cdr_ctx* ctx);
/* cudaStream_t the context launches on (for CUDA-event timing by the caller). */
int cdr_get_stream(cdr_ctx* ctx, void** stream);

/* Mesh + adjacency (mesh.hpp:14-39). edges may be NULL (then built here with
 * build_adjacency's ordering, mesh.cpp:27-63). Replaces the per-pass setup of
 * SceneContext / GradContext (render.hpp:44-50, diff_render.hpp:25-31). */
int cdr_set_mesh(cdr_ctx* ctx, const double* positions, int32_t n_vertices,
                 const int32_t* triangles, int32_t n_triangles, const double* uvs,
                 const int32_t* edges, int32_t n_edges);
/* New positions, same topology (the optimiser's per-iteration apply()). */
int cdr_update_positions(cdr_ctx* ctx, const double* positions);
int cdr_get_edges(cdr_ctx* ctx, int32_t* edges_out /* E x 4 */, int32_t* n_edges);

/* MaterialMaps (material.hpp:22-26). */
int cdr_set_textures(cdr_ctx* ctx, const double* diffuse, const double* specular,
                     const double* roughness, int32_t width, int32_t height);
/* The next cdr_loss_grad / cdr_total_loss's parameters, read during that
 * call: positions (3V, NULL = unchanged) and the three maps (all or none,
 * as cdr_set_textures). The call uploads the maps on a copy stream beside
 * its visibility pass, and with CDR_FLAG_GRAD_OVERWRITE on one rank it
 * downloads the map/light gradient and the rendered images beside its
 * boundary pass. Same results as cdr_update_positions + cdr_set_textures
 * just before the call; the buffers must stay valid and unchanged until it
 * returns (pinned buffers overlap; pageable ones are copied at its start).
 * Any other entry point applies staged parameters first, synchronously.
 * Replaces the per-iteration `apply` + `total_loss(mesh, material, ...)`
 * hand-off of the reference optimiser (coarse_to_fine.cpp:157-158,
 * losses.hpp:94-96). */
int cdr_stage_params(cdr_ctx* ctx, const double* positions, const double* diffuse, const double* specular,
                     const double* roughness, int32_t width, int32_t height);
/* CollocatedLight::intensity, Scene::background (scene.hpp:13-23). */
int cdr_set_light(cdr_ctx* ctx, const double intensity[3], const double background[3]);
/* Scene::views (scene.hpp:21). global_ids may be NULL (= 0..n-1). */
int cdr_set_views(cdr_ctx* ctx, const cdr_camera* cameras, const int32_t* global_ids,
                  int32_t n_views);
/* Target image of a view slot (W x H x 3) and optional mask (W x H). */
int cdr_set_target(cdr_ctx* ctx, int32_t view, const double* rgb, const double* mask);
/* The same from fp32 data (PFM targets, texture.cpp:119-155, hold fp32): half
 * the upload, widened exactly on the device; identical to cdr_set_target on
 * the doubles the reference's load_pfm would produce. */
int cdr_set_target_f32(cdr_ctx* ctx, int32_t view, const float* rgb, const float* mask);

/* vertex_normals (mesh.cpp:65-95). */
int cdr_vertex_normals(cdr_ctx* ctx, double* normals_out /* V x 3 */);

/* render (render.hpp:67-68, render.cpp:35-64). hit_cache may be NULL. */
int cdr_render(cdr_ctx* ctx, int32_t view, const cdr_settings* settings, double* rgb_out,
               double* mask_out, int32_t* hit_cache_out);

/* radiance_at (render.hpp:61-62, render.cpp:24-33) for n continuous pixel
 * positions xy (n x 2); tri_out (nullable) receives the hit triangle or -1. */
int cdr_radiance_at(cdr_ctx* ctx, int32_t view, int32_t n, const double* xy, double* rgb_out,
                    int32_t* tri_out);

/* The radiance probes of boundary_pass (diff_render.cpp:246-252: radiance_at
 * at x - n/2 and x + n/2) as the fused loss call traces them: through the
 * per-pixel candidate lists the LAST cdr_render / cdr_loss_grad /
 * cdr_total_loss built for `view`, points taken in pairs (xy[2i], xy[2i+1])
 * exactly like one edge sample's two probes. Same outputs as cdr_radiance_at;
 * a test hook proving the list path bit-exact against per-ray traversal.
 * CDR_ERR_INVALID_ARG when the last call built no lists for the view. */
int cdr_probe_points(cdr_ctx* ctx, int32_t view, int32_t n, const double* xy, double* rgb_out,
                     int32_t* tri_out);

/* view_rendering_loss (losses.hpp:37-38, losses.cpp:15-49). target_mask may be
 * NULL. adjoint_out is W x H x 3. */
int cdr_view_loss(cdr_ctx* ctx, int32_t width, int32_t height, const double* rendered,
                  const double* target, const double* target_mask, double lambda_rend,
                  double gamma, int32_t use_target_mask, double* value_out,
                  double* adjoint_out);

/* interior_pass (diff_render.hpp:48-50, diff_render.cpp:62-201); += into grad. */
int cdr_interior_pass(cdr_ctx* ctx, int32_t view, const double* adjoint,
                      const cdr_settings* settings, const int32_t* hit_cache,
                      int64_t hit_cache_len, const cdr_layout* layout, double* grad_inout);

/* extract_silhouettes (silhouette.hpp:36, silhouette.cpp:55-106). Writes at most
 * `capacity` segments; *count receives the full count. */
int cdr_extract_silhouettes(cdr_ctx* ctx, int32_t view, cdr_segment* segments_out,
                            int32_t capacity, int32_t* count, double* total_length);

/* boundary_pass (diff_render.hpp:56-59, diff_render.cpp:203-283); += into grad.
 * segments may be NULL to use this context's own extract_silhouettes. */
int cdr_boundary_pass(cdr_ctx* ctx, int32_t view, const double* adjoint,
                      const cdr_segment* segments, int32_t n_segments, int32_t samples,
                      uint64_t seed, int32_t probe, const cdr_layout* layout,
                      double* grad_inout, int32_t* degenerate_skipped);

/* Hot subset of total_loss (losses.hpp:94-96, losses.cpp:244-297): for each
 * listed view slot render -> view_rendering_loss -> interior_pass ->
 * extract_silhouettes -> boundary_pass, then the Laplacian term
 * (laplacian.cpp:21-55, losses.cpp:66-78) with lambda_lap (0 disables it).
 * loss_out[0] = rendering term, loss_out[1] = Laplacian term.
 * grad_inout (nullable): += of the gradient in `layout` order; when NULL the
 * gradient stays on the device (cdr_get_grad / cdr_grad_device_ptr).
 * rendered_rgb / rendered_mask (nullable): n_views images, in call order.
 * When a communicator is attached (cdr_comm_init), the device gradient and
 * loss terms are summed across ranks before being returned. */
int cdr_loss_grad(cdr_ctx* ctx, const int32_t* views, int32_t n_views,
                  const cdr_settings* settings, double lambda_rend, double lambda_lap,
                  int32_t laplacian_mode, int32_t use_target_mask, const cdr_layout* layout,
                  double* loss_out, double* grad_inout, double* rendered_rgb,
                  double* rendered_mask, cdr_stats* stats);
/* LossWeights (losses.hpp:14-23) of the four mesh / material regularisers.
 * The reference defaults are normal 0.01, edge 1, spec 0.01, roug 0.001,
 * sigma1 2, sigma2 0.1. */
typedef struct cdr_reg_weights {
    double normal, edge, spec, roug, sigma1, sigma2;
} cdr_reg_weights;

/* total_loss (losses.hpp:94-96, losses.cpp:244-297): cdr_loss_grad plus
 * normal_consistency_loss, edge_length_loss, specular_correlation_loss and
 * roughness_tv_loss (losses.cpp:80-238) on the context's mesh and maps. Under
 * a communicator the mesh/material terms are computed once (rank 0) and summed
 * with the view shards. breakdown_out[7] = total, rend, lap, normal, edge,
 * spec, roug (LossBreakdown, losses.hpp:25-28). Other arguments as cdr_loss_grad. */
int cdr_total_loss(cdr_ctx* ctx, const int32_t* views, int32_t n_views, const cdr_settings* settings,
                   double lambda_rend, double lambda_lap, const cdr_reg_weights* reg, int32_t laplacian_mode,
                   int32_t use_target_mask, const cdr_layout* layout, double* breakdown_out,
                   double* grad_inout, double* rendered_rgb, double* rendered_mask, cdr_stats* stats);

/* The four regularisers alone. values_out[4] = normal, edge, spec, roug.
 * grad_inout (ParamLayout order) receives +=; with NULL the gradients are
 * added to the device gradient (cdr_grad_device_ptr) instead. */
int cdr_regularisers(cdr_ctx* ctx, const cdr_reg_weights* reg, const cdr_layout* layout,
                     double* values_out, double* grad_inout);

int cdr_get_grad(cdr_ctx* ctx, double* grad_out, int64_t n);
/* Replace the device gradient (n values, ParamLayout order): e.g. a gradient
 * assembled elsewhere, for cdr_adam_step. */
int cdr_set_grad(cdr_ctx* ctx, const double* grad, int64_t n);
int cdr_grad_device_ptr(cdr_ctx* ctx, void** ptr, int64_t* n);

/* cotangent_laplacian (laplacian.hpp:14-15) as CSC (Eigen's default storage):
 * outer V+1, inner/values nnz = V + 2E. Any output pointer may be NULL. */
int cdr_laplacian_matrix(cdr_ctx* ctx, int32_t mode, int32_t* outer, int32_t* inner,
                         double* values, int64_t* nnz);
/* laplacian_loss (losses.hpp:53-54, losses.cpp:66-78) on the matrix of `mode`;
 * grad_positions_inout (V x 3, nullable) receives +=. */
int cdr_laplacian_loss(cdr_ctx* ctx, int32_t mode, double lambda, double* value_out,
                       double* grad_positions_inout);

/* The LBVH's sorted leaf keys (Morton code << 32 | face index, ascending; the
 * leaf order of the hierarchy that replaces Bvh::build, bvh.cpp:90-208) for
 * the current positions: n = number of triangles. A test hook for the radix
 * sort. */
int cdr_lbvh_keys(cdr_ctx* ctx, uint64_t* keys_out, int32_t n);

/* Image and mask of `view` from the last cdr_render / cdr_loss_grad /
 * cdr_total_loss that rendered it (the rendered outputs of total_loss,
 * losses.cpp:259), read straight into the caller's W x H x 3 and W x H
 * buffers (either may be NULL). */
int cdr_get_rendered(cdr_ctx* ctx, int32_t view, double* rgb_out, double* mask_out);

/* Page-locked host memory (cudaHostAlloc) for the caller's per-iteration
 * buffers: the loss calls overlap their downloads into such buffers with the
 * boundary pass, and cdr_stage_params' uploads with the visibility pass.
 * (new; the drop-in shim stages total_loss's rendered images in one.) */
int cdr_host_alloc(size_t bytes, void** out);
void cdr_host_free(void* p);

/* self_intersects (mesh.hpp:67, mesh.cpp:184-214) on an arbitrary mesh (it
 * need not be the context's render mesh, nor manifold): result = 1 iff two
 * triangles sharing no vertex overlap (triangles_intersect, tol 1e-10). With
 * pairs (cap x 2, nullable) and/or n_pairs (nullable) every offending pair
 * (f < g) is found; pairs receives the first `cap` of them sorted by (f, g)
 * and n_pairs their count. Without either, the search stops at the first. */
int cdr_self_intersects(cdr_ctx* ctx, const double* positions, int32_t n_vertices,
                        const int32_t* triangles, int32_t n_triangles, int32_t* result,
                        int32_t* pairs, int64_t cap, int64_t* n_pairs);

/* Bvh::closest_point (bvh.hpp:44, bvh.cpp:267-329) of nq query points (nq x 3)
 * on an arbitrary mesh: triangle (-1 if the mesh is empty), closest point
 * (nq x 3), distance, barycentrics b0 b1 b2 (nq x 3); every output nullable.
 * The distance is the reference's; on an exact tie between triangles the
 * lowest index is returned (the reference: first met by its SAH traversal).
 * Used for uv_transfer (remesh.cpp:281-294) and point_to_mesh_distance. */
int cdr_closest_points(cdr_ctx* ctx, const double* positions, int32_t n_vertices,
                       const int32_t* triangles, int32_t n_triangles, const double* queries,
                       int32_t n_queries, int32_t* tri_out, double* point_out, double* dist_out,
                       double* bary_out);

/* ---- resident optimiser --------------------------------
 * AdamConfig (optimize.hpp:13-18). */
typedef struct cdr_adam_config {
    double beta1, beta2, epsilon, lr_positions, lr_textures, lr_light;
} cdr_adam_config;

/* AdamState(layout, config) (optimize.hpp:20-28) on the device: m = v = 0, step 0. */
int cdr_adam_init(cdr_ctx* ctx, const cdr_adam_config* config, const cdr_layout* layout);
/* adam_step (adam.cpp:9-54) + apply (params.cpp:103-134) on the resident
 * parameters, with the device gradient of the last cdr_loss_grad /
 * cdr_total_loss. Texture and light segments are updated and clamped in place
 * (the next pass renders them); the position segment is not applied: its
 * displacement stays on the device for cdr_evolve and is copied to
 * displacement_out (V x 3, nullable). CDR_ERR_NONFINITE (nothing updated) if a
 * gradient value is not finite. */
int cdr_adam_step(cdr_ctx* ctx, double* displacement_out, int64_t* step_out);
/* Moments and step for checkpoints / coarse-to-fine carries (layout order). */
int cdr_adam_get_state(cdr_ctx* ctx, double* m_out, double* v_out, int64_t* step_out);
int cdr_adam_set_state(cdr_ctx* ctx, const double* m, const double* v, int64_t step);
/* robust_evolve (evolve.cpp:19-53) on the device: positions += s * d for the
 * largest s in {1, 1/2, ..., 2^-8} that keeps every triangle area > 1e-12 and
 * the mesh free of self-intersections, else unchanged (s = 0). d = displacement
 * (V x 3) or, when NULL, the one of the last cdr_adam_step. scale_out and
 * positions_out (V x 3) are nullable. CDR_ERR_SELF_INTERSECTING if the current
 * mesh already self-intersects (evolve.cpp:23). */
int cdr_evolve(cdr_ctx* ctx, const double* displacement, double* scale_out, double* positions_out);
/* pack (params.cpp:70-100): the resident positions, maps and light in
 * ParamLayout order. */
int cdr_get_params(cdr_ctx* ctx, const cdr_layout* layout, double* params_out);

/* Multi-GPU view sharding: one context per GPU/rank, gradient all-reduce over
 * NCCL (loaded at run time). id is an ncclUniqueId (128 bytes). */
int cdr_nccl_unique_id(char id_out[128]);
int cdr_comm_init(cdr_ctx* ctx, const char id[128], int32_t n_ranks, int32_t rank);
/* One process driving n GPUs (the drop-in shim, CDR_DEVICES): one context per
 * device, all joined by ncclCommInitAll; context i becomes rank i. Each
 * context's cdr_loss_grad / cdr_total_loss must then be called concurrently
 * (one host thread per context), as for ranks in separate processes. */
int cdr_comm_init_all(cdr_ctx** ctxs, int32_t n);
/* Ranks and own rank as the attached NCCL communicator reports them
 * (ncclCommCount / ncclCommUserRank); 1 and 0 without one. */
int cdr_comm_info(cdr_ctx* ctx, int32_t* n_ranks, int32_t* rank);
/* View shard of a group summed by the caller instead of NCCL (several
 * contexts on one device, e.g. testing the sharding on one GPU): only rank 0
 * adds the once-per-iteration terms (Laplacian, regularisers), as under a
 * communicator. Not allowed on a context with a communicator. */
int cdr_set_rank(cdr_ctx* ctx, int32_t rank, int32_t n_ranks);

#ifdef __cplusplus
}
#endif

#endif /* CDR_H */
