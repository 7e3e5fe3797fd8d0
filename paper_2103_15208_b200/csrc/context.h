// context.h — host-side state of one cdr_ctx (one GPU).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/cdr.h"
#include "beam.cuh"
#include "bvh.cuh"
#include "common.cuh"

namespace cdr {

struct SceneInfo {        // device-resident, rewritten by prepare()
    double lo[3], hi[3];  // vertex bounding box (Mesh::bbox_min/max, mesh.cpp:15-25)
    double t_min;         // Bvh::default_t_min_ (bvh.cpp:92)
    double pad;           // absolute box padding for the fp32 traversal
};

// Device buffer with grow-only capacity. Owns its allocation: freed on
// destruction (cdr_destroy deletes the context with its device current), so a
// destroyed context returns all of its device memory. Move-only.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void ensure(size_t count) {
        if (count <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (cudaMalloc(&p, sizeof(T) * (count ? count : 1)) != cudaSuccess) throw std::bad_alloc();
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct ViewData {
    DevCamera cam;
    bool has_target = false;
    bool has_target_mask = false;
    double target_mask_sum = 0;  // Σ target mask in pixel order (losses.cpp:26)
    size_t pix_off = 0;          // offset (pixels) of this view in the image arena
};

struct ErrorInfo {  // device-side NonFiniteGradient report
    int flag;
    int x, y;
    int segment;
};

struct Counters {  // device-side work counters (cdr_stats)
    unsigned long long hit_samples;
    unsigned long long adjoint_samples;
    unsigned long long boundary_active;
    unsigned long long beam_fallback_tiles;  // tiles traced per ray (list overflow)
    unsigned long long shaded_samples;       // samples through k_render's full path (not an empty beam tile)
    double loss_sum[1];
};

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace cdr

struct cdr_ctx {
    int device = 0;
    cudaStream_t side = nullptr;  // silhouettes + CDF and the regularisers run here, beside the render
    cudaEvent_t ev_fork = nullptr, ev_sil = nullptr, ev_reg = nullptr;
    cudaStream_t bg = nullptr;  // k_background of a queue-mode render, beside k_trace / k_render
    cudaEvent_t ev_bg = nullptr;
    // cdr_stage_params: host parameters read by the next loss call (maps
    // uploaded on `copy` beside the visibility pass; gradient pieces and
    // images downloaded on `copy` beside the boundary pass)
    struct Staged {
        const double* pos = nullptr;
        const double *d = nullptr, *s = nullptr, *r = nullptr;
        int w = 0, h = 0;
    } staged;
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_copy = nullptr, ev_maps = nullptr;
    cudaEvent_t img_ev[16] = {};  // per shading group (launch_render)
    cdr::DBuf<int> queue_starts;           // per call: first tile-queue entry
    int* queue_starts_host = nullptr;      // pinned copy of it
    int queue_starts_cap = 0;
    bool images_downloaded = false;        // the last launch_render downloaded its images itself
    cdr_ctx* geo = nullptr;  // geometry-only context of cdr_self_intersects / cdr_evolve (lazy)
    // Per-context scratch (device memory of this context's GPU): used inside one
    // synchronous entry point at a time, never across calls.
    cdr::DBuf<double> scr_d[5];
    cdr::DBuf<int32_t> scr_i;
    cdr::DBuf<float> scr_f;
    cdr::DBuf<int> scr_flag;
    cdr::DBuf<unsigned long long> scr_u64;
    void* render_statics = nullptr;    // render.cu (freed by free_render_statics)
    void* boundary_statics = nullptr;  // boundary.cu (freed by free_boundary_statics)
    uint64_t topo_version = 0;  // bumped by cdr_set_mesh; geo->topo_version = the copy it holds
    // resident optimiser (optimize.cu): AdamState (optimize.hpp:20-28) on the device
    bool adam_ready = false;
    cdr_adam_config adam_cfg{};
    cdr_layout adam_lay{};
    int64_t adam_step = 0;
    cdr::DBuf<double> adam_m, adam_v, adam_disp, adam_light;
    cdr::DBuf<int2> si_pairs;
    cudaStream_t stream = nullptr;
    std::string err;

    // mesh (topology fixed between set_mesh calls)
    int V = 0, T = 0, E = 0;
    bool has_uv = false;
    std::vector<int32_t> h_tris, h_edges;
    cdr::DBuf<double> pos, uv, normals, accum, fnormal;
    cdr::DBuf<int32_t> tris;
    cdr::DBuf<int4> edges;
    cdr::DBuf<int32_t> vf_start, vf_list;   // vertex -> (face*3+corner), ascending face
    cdr::DBuf<int32_t> lap_rowptr, lap_col;  // CSR pattern of the Laplacian (symmetric)
    cdr::DBuf<int2> lap_edge_slot;           // per edge: slot of (v0,v1) and (v1,v0)
    cdr::DBuf<int32_t> lap_diag_slot;
    cdr::DBuf<double> lap_val, lap_lv, lap_grad, lap_partial;
    bool geometry_dirty = true;

    // per-iteration acceleration data
    cdr::DBuf<cdr::SceneInfo> info;
    cdr::DBuf<double> bbox_partial;
    cdr::DBuf<unsigned long long> keys, keys_alt;
    cdr::DBuf<unsigned char> sort_tmp;
    cdr::DBuf<int32_t> parent_internal, parent_leaf, refit_flag;
    cdr::DBuf<float> node_box;  // internal node boxes (6 floats) for the refit
    cdr::DBuf<cdr::BNode> nodes;
    cdr::DBuf<cdr::TriRec> recs;
    // beam traversal (beam.cuh): per-tile headers and the candidate pool
    cdr::DBuf<cdr::TileHdr> beam_hdr;
    cdr::DBuf<cdr::BeamCand> beam_pool;
    cdr::DBuf<int> beam_used;
    cdr::DBuf<unsigned char> beam_pix_list, beam_pix_cnt;
    cdr::DBuf<int> beam_tile_base;
    cdr::DBuf<int2> beam_big_queue;  // tiles rebuilt with the big candidate cap
    cdr::DBuf<int> beam_top;         // k_top_walk: per tile block, the shared top frontier
    cdr::DBuf<int2> beam_blk_queue;  // k_top_walk: the non-empty tile blocks (the list builder's queue)
    cdr::DBuf<int> beam_blk_count;
    cdr::DBuf<int> beam_big_count;   // [0] big queue, [1] split queue
    cdr::DBuf<int4> beam_split_queue;  // split work items (levels 0 and 1)
    cdr::DBuf<int2> beam_split_hdr;    // groups of 4 quadrant lists
    cdr::DBuf<unsigned char> beam_big_pix_list, beam_big_pix_cnt;      // per view index of the last render call
    cdr::DBuf<int2> tile_queue;         // non-empty tiles (call, tile) of a queue-mode loss call
    cdr::DBuf<int> tile_queue_count;
    int* tile_queue_host = nullptr;     // pinned: its length, read back during k_trace
    cudaEvent_t tile_queue_ev = nullptr;
    double queue_frac_last = 1.0;       // non-empty tile fraction of the last queue-mode call
    cdr::BeamView beam_view{};          // lists of the last render call (valid flag)
    std::vector<int> beam_slots;        // view slots of that call, in call order (beam_view's view index)
    int* beam_used_host = nullptr;   // pinned; previous call's pool use
    int beam_used_last = 0;
    double t_min_host = 1e-8;

    // materials, light
    int tw = 0, th = 0;
    cdr::DBuf<cdr::Texel> tex;      // fp32 texel records (maps on the fp32 grid)
    cdr::DBuf<cdr::Texel64> tex64;  // fp64 texel records (any maps)
    cdr::DBuf<int> tex_flag;        // k_pack_textures: 1 = some value off the fp32 grid
    int* tex_flag_host = nullptr;   // pinned copy of it
    cudaEvent_t ev_texflag = nullptr;
    bool tex_flag_pending = false;  // the copy is in flight: tex64_resolve reads it
    bool tex64_on = false;          // shading kernels read tex64
    cdr::DBuf<double> map_d, map_s, map_r;  // fp64 maps, resident (the regularisers read them)
    cdr::DBuf<double> reg_part, reg_lum, reg_stats, reg_vals, reg_grad;
    double light[3] = {1, 1, 1};
    double background[3] = {0, 0, 0};

    // views and per-view device images (arena indexed by ViewData::pix_off)
    std::vector<cdr::ViewData> views;
    cdr::DBuf<cdr::DevCamera> d_cams;
    size_t total_pixels = 0;
    cdr::DBuf<double> target, target_mask, img, mask, adj;
    cdr::DBuf<double> target_tone;   // Φ(target) for target_tone_gamma
    double target_tone_gamma = -1;   // < 0: stale
    cdr::DBuf<int32_t> hit;  // hit caches (per view W*H*spp), arena sized on demand
    size_t hit_stride_spp = 0;

    // silhouettes (per view slot capacity E)
    cdr::DBuf<unsigned char> sil_flag;
    cdr::DBuf<int32_t> sil_block_count, sil_block_off, sil_count;
    int seg_stride = 1;  // per-view stride of segs/cdf/cdf_guide/bin arrays (set_view_calls)
    cdr::DBuf<cdr_segment> segs;
    cdr::DBuf<double> cdf, total_len;
    cdr::DBuf<int32_t> cdf_guide;  // per view: lower_bound guide over the CDF (k_cdf)
    cdr::DBuf<int32_t> degenerate;
    // boundary samples binned by segment
    cdr::DBuf<int32_t> b_seg_count, b_seg_off, b_n_active, b_key, b_slot, b_sorted_si;
    cdr::DBuf<double> b_s, b_sorted_s;

    // gradient + accumulators
    int64_t grad_n = 0;
    cdr::DBuf<double> grad;
    cdr::DBuf<double> grad_tmp;    // staging of the caller's += buffer
    cdr::DBuf<double> corner_acc;  // T x 3 corners x (g[3], h[3])
    cdr::DBuf<cdr::TexAcc> tex_acc;  // texel-major interior texel gradients
    cdr::DBuf<double> qvec;        // V x 3: Jn_v * H_v
    cdr::DBuf<double> loss_acc;    // per view: Σ m |d|
    cdr::DBuf<cdr::ErrorInfo> errinfo;
    cdr::DBuf<cdr::Counters> counters;

    // timing and launch accounting (cdr_stats::kernel_launches)
    std::vector<cudaEvent_t> ev;
    std::vector<cudaEvent_t> chunk_ev;  // per view chunk of a timed render: start, after trace
    int chunk_ev_used = 0;
    int64_t launches = 0;

    // multi-GPU
    void* nccl_comm = nullptr;
    int n_ranks = 1, rank = 0;
};
