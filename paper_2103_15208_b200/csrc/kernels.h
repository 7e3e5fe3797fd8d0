// kernels.h — host launch wrappers of the sm_100a kernels (one per stage).
#pragma once

#include <stdexcept>
#include <string>

#include "context.h"
#include "shade.cuh"

namespace cdr {

inline ShadeScene shade_scene(const cdr_ctx* c) {
    ShadeScene sc{};
    sc.nodes = c->nodes.p;
    sc.recs = c->recs.p;
    sc.n_tris = c->T;
    sc.pos = c->pos.p;
    sc.tris = c->tris.p;
    sc.uv = c->has_uv ? c->uv.p : nullptr;
    sc.normals = c->normals.p;
    sc.fnormal = c->fnormal.p;
    sc.tex = c->tex.p;
    sc.tex64 = c->tex64.p;
    sc.tw = c->tw;
    sc.th = c->th;
    for (int i = 0; i < 3; ++i) {
        sc.L[i] = c->light[i];
        sc.bg[i] = c->background[i];
    }
    return sc;
}

// prepare.cu — per-iteration geometry: face normals, vertex normals
// (mesh.cpp:65-95), bbox + t_min (bvh.cpp:92), LBVH (Morton -> radix sort ->
// Karras hierarchy -> bottom-up fp32 refit).
void launch_prepare(cdr_ctx* c, double cam_abs_max);
void launch_bvh(cdr_ctx* c, double cam_abs_max);
void free_render_statics(cdr_ctx* c);    // render.cu per-context buffers
void free_boundary_statics(cdr_ctx* c);  // boundary.cu per-context buffers  // bbox + t_min + LBVH (no normals)
// self_intersects (mesh.cpp:184-214) on the context's mesh and LBVH: returns
// the number of intersecting pairs (early exit after the first when pairs ==
// nullptr); pairs (f < g) written up to cap, in no particular order.
long long launch_self_intersect(cdr_ctx* c, int2* pairs, long long cap);
void launch_widen(cdr_ctx* c, const float* in, int64_t n, double* out);  // fp32 -> fp64 (exact)
// closest.cu: Bvh::closest_point for nq queries on c's mesh + LBVH (device outputs)
void launch_closest(cdr_ctx* c, const double* queries, int nq, int32_t* tri, double* point, double* dist,
                    double* bary);
// optimize.cu: resident adam_step / robust_evolve building blocks
bool any_nonfinite(cdr_ctx* c, const double* g, int64_t n);
bool any_nonzero(cdr_ctx* c, const double* d, int64_t n);
void launch_adam(cdr_ctx* c, const double* grad, double corr1, double corr2);
double min_triangle_area(cdr_ctx* c, const double* pos);  // over c's triangles, positions `pos`
void launch_candidate(cdr_ctx* c, const double* pos, const double* disp, double s, double* out);

// render.cu — fused per-sample kernel. Modes:
//   kTrace     primary-ray generation + LBVH traversal + shading (render.cpp:35-64)
//   kLoss      per-pixel tone-mapped L1 + adjoint (losses.cpp:15-49)
//   kInterior  interior adjoint scatter (diff_render.cpp:62-201)
struct RenderArgs {
    int spp;
    int k;  // lround(sqrt(spp))
    uint64_t seed;
    double gamma;
    double loss_scale;  // lambda / n_valid (per call, all views share W*H here)
    int use_mask;
    int write_hits;
    int64_t lay_diffuse, lay_specular, lay_roughness, lay_light;  // -1 = absent
    cudaEvent_t wait_before_shade = nullptr;  // joined after the visibility pass, before the shading
    // page-locked destinations of the call's images and masks (views in call
    // order): a queue-mode call shades view group by view group and downloads
    // each group's images on the copy stream while the next group shades
    // (sets c->images_downloaded)
    double* img_rgb_host = nullptr;
    double* img_mask_host = nullptr;
};
void launch_render(cdr_ctx* c, const int* view_slots, int n_views, const RenderArgs& a,
                   bool trace, bool loss, bool interior, const double* loss_scales,
                   cudaEvent_t after_trace = nullptr);
// normal / edge / specular / roughness regularisers (regularisers.cu):
// values_dev[0..3] written, gradients += into grad (ParamLayout order) if given
void launch_regularisers(cdr_ctx* c, const cdr_reg_weights& w, const cdr_layout& lay, double* grad,
                         double* values_dev);
// Σ over the view chunks of the last timed launch_render: lists + trace time (ms)
float render_trace_ms(cdr_ctx* c);

// boundary.cu — extract_silhouettes (silhouette.cpp:55-106), the CDF of
// boundary_pass (diff_render.cpp:213-228) and its edge samples (:230-278).
// view list of the next silhouette/CDF/boundary launches; samples[i] = M per view
// min_stride: per-view capacity of the segment arrays when a caller supplies
// more segments than the mesh has edges (cdr_boundary_pass)
void set_view_calls(cdr_ctx* c, const int* view_slots, const int* samples, int n_views, int min_stride = 0);
void launch_silhouettes(cdr_ctx* c, int n_views);
void launch_cdf(cdr_ctx* c, int n_views);
// use_beam: probes may use the candidate lists the preceding render call built
// for the same view list (cdr_loss_grad); otherwise per-ray traversal
void launch_boundary(cdr_ctx* c, int n_views, int max_samples, uint64_t seed, int probe,
                     int64_t lay_pos, bool use_beam = false);
// The same in two stages for the fused loss call: the edge samples' RNG picks,
// CDF searches and binning need only the segments and the CDF, so they run on
// the side stream beside the render; the probes and deposits follow the
// render (they need its adjoint and candidate lists).
void launch_boundary_sampling(cdr_ctx* c, int n_views, int max_samples, uint64_t seed);
void launch_boundary_probes(cdr_ctx* c, int n_views, int max_samples, uint64_t seed, int probe, int64_t lay_pos,
                            bool use_beam);
// The boundary probes' visibility on its own (cdr_probe_points): n points of
// the view at index vi of the last render call, traced in pairs through that
// call's candidate lists exactly as k_boundary traces x -/+ n/2 (rgb nullable).
void launch_probe_points(cdr_ctx* c, int vi, int n, const double* xy, double* rgb, int32_t* tri);

// finalize.cu — position gradient assembly: per-corner interior sums, the
// one-ring normal chain (diff_render.cpp:174-184) restated as q_v x d_{f,w},
// and the Laplacian (laplacian.cpp:21-55, losses.cpp:66-78) as CSR SpMVs.
void launch_finalize_positions(cdr_ctx* c, int64_t lay_pos);
void launch_laplacian(cdr_ctx* c, int mode, double lambda, double* grad_pos /* nullable */);

// generic loss kernel over device images (cdr_view_loss)
// Φ(target) for all target pixels (losses.cpp:38 evaluates it per pixel)
void launch_tone_targets(cdr_ctx* c, double gamma);
// y += x over n doubles
void launch_axpy(cdr_ctx* c, double* y, const double* x, int64_t n);
// add the texel-major accumulators into the gradient's texture segments
void launch_texel_flush(cdr_ctx* c, int64_t lay_d, int64_t lay_s, int64_t lay_r);
// radiance_at for n pixel positions of one view (device buffers)
void launch_radiance_points(cdr_ctx* c, int slot, int n, const double* xy, double* rgb, int32_t* tri);
// pack diffuse/specular/roughness (fp64, device) into 32-byte fp32 texel records
void launch_pack_textures(cdr_ctx* c, const double* d, const double* s, const double* r, int n);
void tex64_resolve(cdr_ctx* c);  // the texel record choice of the last packed maps (host)

void launch_view_loss(cdr_ctx* c, int W, int H, const double* rendered, const double* target,
                      const double* tmask, double scale, double gamma, int masked, double* adj,
                      double* sum);

}  // namespace cdr

#define CDR_CUDA_CHECK(x)                                                              \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw cdr::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));     \
    } while (0)

namespace cdr {
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
}  // namespace cdr
