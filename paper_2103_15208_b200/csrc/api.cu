// api.cu — the C-ABI of include/cdr.h over the sm_100a kernels.
//
// Host-side work here is bookkeeping only (validation, topology tables built
// once per set_mesh, uploads/downloads); every per-sample, per-edge and
// per-vertex computation of the hot path runs in the kernels of prepare.cu,
// render.cu, boundary.cu and finalize.cu. There is no CPU fallback: without a
// CUDA device every call fails with CDR_ERR_NO_DEVICE / CDR_ERR_CUDA.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: stage ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <new>
#include <optional>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

using namespace cdr;

namespace {

struct SizeMismatchErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ApiErr : std::runtime_error {
    int code;
    ApiErr(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int handle(cdr_ctx* c, const std::function<void()>& fn, bool staged_consumer = false);

#define API_BEGIN(ctx)                                            \
    if (!(ctx)) return CDR_ERR_INVALID_ARG;                       \
    return handle((ctx), [&]() {
#define API_END \
    });
// the loss entry points consume cdr_stage_params' parameters themselves
#define API_BEGIN_STAGED(ctx)                                     \
    if (!(ctx)) return CDR_ERR_INVALID_ARG;                       \
    return handle((ctx), [&]() {
#define API_END_STAGED \
    }, true);

void apply_staged_sync(cdr_ctx* c);
int handle_error(cdr_ctx* c);

int handle(cdr_ctx* c, const std::function<void()>& fn, bool staged_consumer) {
    try {
        if (cudaSetDevice(c->device) != cudaSuccess) throw ApiErr(CDR_ERR_NO_DEVICE, "cudaSetDevice failed");
        if (!staged_consumer) apply_staged_sync(c);  // as cdr_update_positions + cdr_set_textures now
        fn();
        c->err.clear();
        return CDR_OK;
    } catch (...) {
        // no copy may still read a caller's buffer once the call has returned
        if (c->copy) cudaStreamSynchronize(c->copy);
        c->staged = cdr_ctx::Staged{};
        return handle_error(c);
    }
}

int handle_error(cdr_ctx* c) {
    try {
        throw;
    } catch (const SizeMismatchErr& e) {
        c->err = e.what();
        return CDR_ERR_SIZE_MISMATCH;
    } catch (const ApiErr& e) {
        c->err = e.what();
        return e.code;
    } catch (const CudaError& e) {
        c->err = e.what();
        return CDR_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        c->err = "out of device or host memory";
        return CDR_ERR_CUDA;
    } catch (const std::exception& e) {
        c->err = e.what();
        return CDR_ERR_ERROR;
    } catch (...) {
        c->err = "unknown error";
        return CDR_ERR_ERROR;
    }
}

template <typename T>
void h2d(DBuf<T>& b, const T* src, size_t n, cudaStream_t s) {
    b.ensure(std::max<size_t>(1, n));
    if (n) CDR_CUDA_CHECK(cudaMemcpyAsync(b.p, src, sizeof(T) * n, cudaMemcpyHostToDevice, s));
}

void sync(cdr_ctx* c) { CDR_CUDA_CHECK(cudaStreamSynchronize(c->stream)); }

double cam_abs_max(const cdr_ctx* c) {
    double m = 0;
    for (const auto& v : c->views)
        for (int k = 0; k < 3; ++k) m = std::max(m, std::fabs(v.cam.o[k]));
    return m;
}

void ensure_prepared(cdr_ctx* c, bool force = false) {
    if (!force && !c->geometry_dirty) return;
    launch_prepare(c, cam_abs_max(c));
    c->geometry_dirty = false;
}

void check_view(const cdr_ctx* c, int view) {
    if (view < 0 || view >= int(c->views.size()))
        throw ApiErr(CDR_ERR_INVALID_ARG, "view slot " + std::to_string(view) + " out of range");
}

void check_ready(const cdr_ctx* c) {
    if (c->T > 0 && c->tw <= 0) throw ApiErr(CDR_ERR_INVALID_ARG, "textures not set");
}

int spp_of(const cdr_settings* s) { return std::max(1, s->spp); }

void check_spp(int spp) {
    if (spp > 256)
        throw ApiErr(CDR_ERR_INVALID_ARG, "spp > 256 is not supported by the fused kernel");
}

RenderArgs render_args(const cdr_ctx* c, const cdr_settings* s, const cdr_layout* lay) {
    RenderArgs a{};
    a.spp = spp_of(s);
    a.k = int(std::lround(std::sqrt(double(a.spp))));  // render.cpp:15
    a.seed = s->seed;
    a.gamma = s->gamma;
    a.write_hits = 1;
    if (lay) {
        a.lay_diffuse = lay->diffuse;
        a.lay_specular = lay->specular;
        a.lay_roughness = lay->roughness;
        a.lay_light = lay->light;
    } else {
        a.lay_diffuse = a.lay_specular = a.lay_roughness = a.lay_light = -1;
    }
    (void)c;
    return a;
}

void check_layout(const cdr_ctx* c, const cdr_layout* lay, int tw = -1, int th = -1) {
    if (!lay) throw ApiErr(CDR_ERR_INVALID_ARG, "layout is null");
    int64_t n = tw >= 0 ? int64_t(tw) * th : int64_t(c->tw) * c->th;
    auto seg = [&](int64_t off, int64_t size, const char* name) {
        if (off < 0 || off + size > lay->total)
            throw SizeMismatchErr(std::string("gradient layout segment ") + name + " out of range");
    };
    seg(lay->positions, 3 * int64_t(c->V), "positions");
    seg(lay->diffuse, 3 * n, "diffuse");
    seg(lay->specular, 3 * n, "specular");
    seg(lay->roughness, n, "roughness");
    if (lay->light >= 0) seg(lay->light, 3, "light");
}

void zero_grad(cdr_ctx* c, int64_t total) {
    c->grad.ensure(std::max<int64_t>(1, total));
    c->grad_n = total;
    CDR_CUDA_CHECK(cudaMemsetAsync(c->grad.p, 0, sizeof(double) * std::max<int64_t>(1, total), c->stream));
    c->corner_acc.ensure(std::max<size_t>(1, size_t(c->T) * 18));
    CDR_CUDA_CHECK(cudaMemsetAsync(c->corner_acc.p, 0, sizeof(double) * std::max<size_t>(1, size_t(c->T) * 18),
                                   c->stream));
    const size_t nt = std::max<size_t>(1, size_t(c->tw) * c->th);
    c->tex_acc.ensure(nt);
    CDR_CUDA_CHECK(cudaMemsetAsync(c->tex_acc.p, 0, sizeof(TexAcc) * nt, c->stream));
}

void reset_flags(cdr_ctx* c) {
    CDR_CUDA_CHECK(cudaMemsetAsync(c->errinfo.p, 0, sizeof(ErrorInfo), c->stream));
    CDR_CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, sizeof(Counters), c->stream));
}

void raise_device_error(cdr_ctx* c) {
    ErrorInfo e;
    CDR_CUDA_CHECK(cudaMemcpy(&e, c->errinfo.p, sizeof(e), cudaMemcpyDeviceToHost));
    if (e.flag == 1)
        throw ApiErr(CDR_ERR_NONFINITE, "non-finite interior gradient at pixel (" + std::to_string(e.x) + "," +
                                            std::to_string(e.y) + ")");
    if (e.flag == 2)
        throw ApiErr(CDR_ERR_NONFINITE, "non-finite boundary gradient at segment " + std::to_string(e.segment));
}

// += of a device gradient slice into the caller's host buffer, done on the
// device: upload the caller's values, add, download in place (two copies at
// full speed when the caller's buffer is pinned; no host-side loop).
void add_grad_to_host(cdr_ctx* c, double* host, int64_t off, int64_t n) {
    if (!host || n <= 0) return;
    c->grad_tmp.ensure(size_t(n));
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->grad_tmp.p, host + off, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    launch_axpy(c, c->grad_tmp.p, c->grad.p + off, n);  // grad_tmp += grad
    CDR_CUDA_CHECK(cudaMemcpyAsync(host + off, c->grad_tmp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
}

void ensure_hit_arena(cdr_ctx* c, int spp) {
    c->hit.ensure(std::max<size_t>(1, c->total_pixels * size_t(spp)));
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    int (*commInitRank)(void**, int, const void* /* by value 128B */, int) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*commCount)(void*, int*) = nullptr;
    int (*commUserRank)(void*, int*) = nullptr;
    int (*commInitAll)(void**, int, const int*) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    const char* (*getErrorString)(int) = nullptr;
    bool ok = false;
};

struct NcclUid {
    char internal[128];
};

NcclApi load_nccl() {
    NcclApi api;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
    }
    if (!api.h) return api;
    api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<int (*)(void**, int, const void*, int)>(dlsym(api.h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(api.h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclCommDestroy"));
    api.getErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(api.h, "ncclGetErrorString"));
    api.commCount = reinterpret_cast<int (*)(void*, int*)>(dlsym(api.h, "ncclCommCount"));
    api.commUserRank = reinterpret_cast<int (*)(void*, int*)>(dlsym(api.h, "ncclCommUserRank"));
    api.commInitAll = reinterpret_cast<int (*)(void**, int, const int*)>(dlsym(api.h, "ncclCommInitAll"));
    api.groupStart = reinterpret_cast<int (*)()>(dlsym(api.h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<int (*)()>(dlsym(api.h, "ncclGroupEnd"));
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy;
    return api;
}

NcclApi& nccl() {
    static NcclApi api = load_nccl();  // loaded once, thread-safe (C++11 static init)
    return api;
}

using CommInitByValue = int (*)(void**, int, NcclUid, int);

void nccl_check(int r, const char* what) {
    if (r != 0) {
        const char* m = nccl().getErrorString ? nccl().getErrorString(r) : "?";
        throw ApiErr(CDR_ERR_ERROR, std::string(what) + ": " + m);
    }
}

constexpr int kNcclFloat64 = 8, kNcclSum = 0;

// Enqueues the maps' upload and the texel packing on c->stream (no sync).
void set_textures_impl(cdr_ctx* c, const double* diffuse, const double* specular, const double* roughness,
                              int32_t w, int32_t h) {
    if (w <= 0 || h <= 0 || !diffuse || !specular || !roughness)
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad texture arguments");
    size_t n = size_t(w) * h;
    c->tw = w;
    c->th = h;
    c->tex.ensure(n);
    // fp64 maps stay resident (regularisers); shading reads fp32 texel records
    h2d(c->map_d, diffuse, 3 * n, c->stream);
    h2d(c->map_s, specular, 3 * n, c->stream);
    h2d(c->map_r, roughness, n, c->stream);
    launch_pack_textures(c, c->map_d.p, c->map_s.p, c->map_r.p, int(n));
}

// Staged parameters applied now, as cdr_update_positions + cdr_set_textures
// would have (any entry point other than the loss calls).
void apply_staged_sync(cdr_ctx* c) {
    if (!c->staged.pos && !c->staged.d) return;
    const cdr_ctx::Staged sp = std::exchange(c->staged, cdr_ctx::Staged{});
    if (sp.pos && c->V > 0) {
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->pos.p, sp.pos, sizeof(double) * 3 * size_t(c->V), cudaMemcpyHostToDevice,
                                       c->stream));
        c->geometry_dirty = true;
    }
    if (sp.d) set_textures_impl(c, sp.d, sp.s, sp.r, sp.w, sp.h);
    sync(c);
}
}  // namespace

extern "C" {

int cdr_abi_version(void) { return CDR_ABI_VERSION; }

int cdr_build_flags(void) {
#ifdef CDR_CHECKED
    return CDR_BUILD_CHECKED;
#else
    return 0;
#endif
}

int cdr_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = e == cudaSuccess ? n : 0;
    return e == cudaSuccess ? CDR_OK : CDR_ERR_NO_DEVICE;
}

int cdr_create(int device, cdr_ctx** out) {
    if (!out) return CDR_ERR_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return CDR_ERR_NO_DEVICE;
    if (device < 0 || device >= n) return CDR_ERR_INVALID_ARG;
    auto c = std::make_unique<cdr_ctx>();
    c->device = device;
    try {
        CDR_CUDA_CHECK(cudaSetDevice(device));
        CDR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CDR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CDR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->bg, cudaStreamNonBlocking));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_bg, cudaEventDisableTiming));
        CDR_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_maps, cudaEventDisableTiming));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_sil, cudaEventDisableTiming));
        CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_reg, cudaEventDisableTiming));
        c->errinfo.ensure(1);
        c->counters.ensure(1);
        c->info.ensure(1);
        c->ev.resize(8);
        for (auto& e : c->ev) CDR_CUDA_CHECK(cudaEventCreate(&e));
    } catch (...) {
        return CDR_ERR_CUDA;
    }
    *out = c.release();
    return CDR_OK;
}

void cdr_destroy(cdr_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->geo) cdr_destroy(c->geo);
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    if (c->bg) cudaStreamSynchronize(c->bg);
    if (c->copy) cudaStreamSynchronize(c->copy);
    free_render_statics(c);
    free_boundary_statics(c);
    if (c->nccl_comm && nccl().ok) nccl().commDestroy(c->nccl_comm);
    for (auto& e : c->ev) cudaEventDestroy(e);
    for (auto& e : c->chunk_ev) cudaEventDestroy(e);
    if (c->beam_used_host) cudaFreeHost(c->beam_used_host);
    if (c->tile_queue_host) cudaFreeHost(c->tile_queue_host);
    if (c->tex_flag_host) cudaFreeHost(c->tex_flag_host);
    if (c->queue_starts_host) cudaFreeHost(c->queue_starts_host);
    for (auto& e : c->img_ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_texflag) cudaEventDestroy(c->ev_texflag);
    if (c->tile_queue_ev) cudaEventDestroy(c->tile_queue_ev);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_sil) cudaEventDestroy(c->ev_sil);
    if (c->ev_reg) cudaEventDestroy(c->ev_reg);
    if (c->ev_bg) cudaEventDestroy(c->ev_bg);
    if (c->ev_copy) cudaEventDestroy(c->ev_copy);
    if (c->ev_maps) cudaEventDestroy(c->ev_maps);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->bg) cudaStreamDestroy(c->bg);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;  // every DBuf member frees its device allocation (context.h)
}

const char* cdr_last_error(const cdr_ctx* c) { return c ? c->err.c_str() : "null context"; }

int cdr_get_stream(cdr_ctx* c, void** stream) {
    if (!c || !stream) return CDR_ERR_INVALID_ARG;
    *stream = reinterpret_cast<void*>(c->stream);
    return CDR_OK;
}

int cdr_set_mesh(cdr_ctx* c, const double* positions, int32_t nv, const int32_t* triangles, int32_t nt,
                 const double* uvs, const int32_t* edges, int32_t ne) {
    API_BEGIN(c)
    if (nv < 0 || nt < 0 || (nv > 0 && !positions) || (nt > 0 && !triangles))
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad mesh arguments");
    // Everything is built and validated in locals first; the context changes
    // only after every check has passed, so a rejected mesh leaves the
    // previous one fully usable.
    // build_adjacency validation (mesh.cpp:27-38)
    for (int f = 0; f < nt; ++f) {
        const int32_t* t = triangles + 3 * f;
        for (int k = 0; k < 3; ++k)
            if (t[k] < 0 || t[k] >= nv)
                throw ApiErr(CDR_ERR_ERROR, "triangle " + std::to_string(f) + " references vertex " +
                                                std::to_string(t[k]) + " out of range");
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2])
            throw ApiErr(CDR_ERR_ERROR, "triangle " + std::to_string(f) + " repeats a vertex");
    }
    // edges: caller's (reference order) or rebuilt with build_adjacency's order
    std::vector<int32_t> h_edges;
    if (edges) {
        if (ne < 0) throw ApiErr(CDR_ERR_INVALID_ARG, "negative edge count");
        h_edges.assign(edges, edges + 4 * size_t(ne));
    } else {
        std::vector<std::pair<int64_t, int>> keys;
        keys.reserve(3 * size_t(nt));
        for (int f = 0; f < nt; ++f)
            for (int k = 0; k < 3; ++k) {
                int a = triangles[3 * f + k], b = triangles[3 * f + (k + 1) % 3];
                keys.push_back({int64_t(std::min(a, b)) * nv + std::max(a, b), f});
            }
        std::sort(keys.begin(), keys.end());
        for (size_t i = 0; i < keys.size();) {
            size_t j = i;
            while (j < keys.size() && keys[j].first == keys[i].first) ++j;
            int64_t key = keys[i].first;
            if (j - i > 2)
                throw ApiErr(CDR_ERR_ERROR, "non-manifold edge (" + std::to_string(key / nv) + "," +
                                                std::to_string(key % nv) + ") with " + std::to_string(j - i) +
                                                " incident faces");
            h_edges.push_back(int32_t(key / nv));
            h_edges.push_back(int32_t(key % nv));
            h_edges.push_back(keys[i].second);
            h_edges.push_back(j - i > 1 ? keys[i + 1].second : -1);
            i = j;
        }
    }
    const int ecount = int(h_edges.size() / 4);
    for (int e = 0; e < ecount; ++e) {  // k_sil_flag reads face normals through f0/f1
        const int32_t a = h_edges[4 * e], b = h_edges[4 * e + 1], f0 = h_edges[4 * e + 2], f1 = h_edges[4 * e + 3];
        if (a < 0 || a >= nv || b < 0 || b >= nv)
            throw ApiErr(CDR_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": vertex out of range");
        if (f0 < 0 || f0 >= nt || f1 < -1 || f1 >= nt)
            throw ApiErr(CDR_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": face out of range");
    }
    // vertex -> (face*3+corner), ascending face (the reference's face-loop order)
    std::vector<int32_t> vstart(size_t(nv) + 1, 0), vlist(3 * size_t(nt));
    for (int f = 0; f < nt; ++f)
        for (int k = 0; k < 3; ++k) vstart[triangles[3 * f + k] + 1]++;
    for (int v = 0; v < nv; ++v) vstart[v + 1] += vstart[v];
    {
        std::vector<int32_t> fill(vstart.begin(), vstart.end() - 1);
        for (int f = 0; f < nt; ++f)
            for (int k = 0; k < 3; ++k) vlist[fill[triangles[3 * f + k]]++] = 3 * f + k;
    }
    // Laplacian CSR pattern: row i = sorted {neighbours} ∪ {i}
    std::vector<std::vector<int32_t>> nb(nv);
    for (int e = 0; e < ecount; ++e) {
        int a = h_edges[4 * e], b = h_edges[4 * e + 1];
        nb[a].push_back(b);
        nb[b].push_back(a);
    }
    std::vector<int32_t> rowptr(size_t(nv) + 1, 0), col, dslot(nv);
    col.reserve(size_t(nv) + 2 * size_t(ecount));
    for (int i = 0; i < nv; ++i) {
        nb[i].push_back(i);
        std::sort(nb[i].begin(), nb[i].end());
        for (int32_t j : nb[i]) {
            if (j == i) dslot[i] = int32_t(col.size());
            col.push_back(j);
        }
        rowptr[i + 1] = int32_t(col.size());
    }
    std::vector<int2> eslot(ecount);
    for (int e = 0; e < ecount; ++e) {
        int a = h_edges[4 * e], b = h_edges[4 * e + 1];
        auto find = [&](int row, int cc) {
            auto it = std::lower_bound(col.begin() + rowptr[row], col.begin() + rowptr[row + 1], cc);
            return int32_t(it - col.begin());
        };
        eslot[e] = make_int2(find(a, b), find(b, a));
    }
    // commit: host state, then the device copies (a failed upload leaves an
    // empty mesh rather than a mix of old buffers and new sizes)
    c->V = nv;
    c->T = nt;
    c->E = ecount;
    c->h_tris.assign(triangles, triangles + 3 * size_t(nt));
    c->h_edges.swap(h_edges);
    ++c->topo_version;
    c->adam_ready = false;  // a new vertex set: the optimiser state no longer matches
    c->geometry_dirty = true;
    c->beam_view.valid = false;
    try {
        cudaStream_t s = c->stream;
        h2d(c->pos, positions, 3 * size_t(nv), s);
        c->has_uv = uvs != nullptr;
        if (uvs) h2d(c->uv, uvs, 2 * size_t(nv), s);
        h2d(c->tris, triangles, 3 * size_t(nt), s);
        h2d(c->edges, reinterpret_cast<const int4*>(c->h_edges.data()), size_t(c->E), s);
        h2d(c->vf_start, vstart.data(), vstart.size(), s);
        h2d(c->vf_list, vlist.data(), vlist.size(), s);
        h2d(c->lap_rowptr, rowptr.data(), rowptr.size(), s);
        h2d(c->lap_col, col.data(), col.size(), s);
        h2d(c->lap_diag_slot, dslot.data(), dslot.size(), s);
        h2d(c->lap_edge_slot, eslot.data(), eslot.size(), s);
        c->lap_val.ensure(std::max<size_t>(1, col.size()));
        c->normals.ensure(3 * size_t(std::max(1, nv)));
        c->accum.ensure(3 * size_t(std::max(1, nv)));
        c->fnormal.ensure(3 * size_t(std::max(1, nt)));
        sync(c);
    } catch (...) {
        c->V = c->T = c->E = 0;
        c->h_tris.clear();
        c->h_edges.clear();
        throw;
    }
    API_END
}

int cdr_update_positions(cdr_ctx* c, const double* positions) {
    API_BEGIN(c)
    if (!positions && c->V > 0) throw ApiErr(CDR_ERR_INVALID_ARG, "positions is null");
    if (c->V > 0)
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->pos.p, positions, sizeof(double) * 3 * size_t(c->V),
                                       cudaMemcpyHostToDevice, c->stream));
    c->geometry_dirty = true;
    sync(c);  // a pinned buffer is read asynchronously: done before the caller can reuse it
    API_END
}

int cdr_get_edges(cdr_ctx* c, int32_t* out, int32_t* n) {
    API_BEGIN(c)
    if (n) *n = c->E;
    if (out) std::memcpy(out, c->h_edges.data(), sizeof(int32_t) * c->h_edges.size());
    API_END
}

int cdr_set_textures(cdr_ctx* c, const double* diffuse, const double* specular, const double* roughness,
                     int32_t w, int32_t h) {
    API_BEGIN(c)
    set_textures_impl(c, diffuse, specular, roughness, w, h);
    sync(c);
    API_END
}


int cdr_stage_params(cdr_ctx* c, const double* positions, const double* diffuse, const double* specular,
                     const double* roughness, int32_t w, int32_t h) {
    API_BEGIN(c)  // (applies anything staged before)
    const bool maps = diffuse || specular || roughness;
    if (maps && (!diffuse || !specular || !roughness || w <= 0 || h <= 0))
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad texture arguments");
    c->staged.pos = positions;
    if (maps) {
        c->staged.d = diffuse;
        c->staged.s = specular;
        c->staged.r = roughness;
        c->staged.w = w;
        c->staged.h = h;
    }
    API_END
}

int cdr_set_light(cdr_ctx* c, const double intensity[3], const double background[3]) {
    API_BEGIN(c)
    for (int i = 0; i < 3; ++i) {
        if (intensity) c->light[i] = intensity[i];
        if (background) c->background[i] = background[i];
    }
    API_END
}

int cdr_set_views(cdr_ctx* c, const cdr_camera* cams, const int32_t* gids, int32_t n) {
    API_BEGIN(c)
    if (n < 0 || (n > 0 && !cams)) throw ApiErr(CDR_ERR_INVALID_ARG, "bad views");
    c->views.assign(n, ViewData{});
    size_t off = 0;
    std::vector<DevCamera> dc(n);
    for (int i = 0; i < n; ++i) {
        const cdr_camera& k = cams[i];
        if (k.width <= 0 || k.height <= 0) throw ApiErr(CDR_ERR_INVALID_ARG, "bad view size");
        DevCamera& d = dc[i];
        std::memset(&d, 0, sizeof(d));
        for (int j = 0; j < 3; ++j) {
            d.o[j] = k.origin[j];
            d.r[j] = k.right[j];
            d.u[j] = k.up[j];
            d.f[j] = k.forward[j];
        }
        d.th = std::tan(k.fov_deg * 3.14159265358979323846 / 360.0);  // camera.cpp:25-27
        d.aspect = double(k.width) / double(k.height);                 // camera.hpp:22
        d.inv_w = (k.width & (k.width - 1)) == 0 ? 1.0 / k.width : 0.0;  // exact powers of two
        d.inv_h = (k.height & (k.height - 1)) == 0 ? 1.0 / k.height : 0.0;
        d.W = k.width;
        d.H = k.height;
        d.gid = gids ? gids[i] : i;
        c->views[i].cam = d;
        c->views[i].pix_off = off;
        off += size_t(k.width) * k.height;
    }
    c->total_pixels = off;
    c->target_tone_gamma = -1;
    h2d(c->d_cams, dc.data(), dc.size(), c->stream);
    size_t np = std::max<size_t>(1, off);
    c->img.ensure(3 * np);
    c->mask.ensure(np);
    c->adj.ensure(3 * np);
    c->target.ensure(3 * np);
    c->target_mask.ensure(np);
    c->loss_acc.ensure(std::max(1, n));
    sync(c);
    API_END
}

int cdr_set_target(cdr_ctx* c, int32_t view, const double* rgb, const double* mask) {
    API_BEGIN(c)
    check_view(c, view);
    if (!rgb) throw ApiErr(CDR_ERR_INVALID_ARG, "target rgb is null");
    ViewData& v = c->views[view];
    size_t np = size_t(v.cam.W) * v.cam.H;
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->target.p + 3 * v.pix_off, rgb, sizeof(double) * 3 * np,
                                   cudaMemcpyHostToDevice, c->stream));
    v.has_target = true;
    c->target_tone_gamma = -1;  // Φ(target) must be recomputed
    v.has_target_mask = mask != nullptr;
    v.target_mask_sum = 0;
    if (mask) {
        for (size_t i = 0; i < np; ++i) v.target_mask_sum += mask[i];  // losses.cpp:26 order
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->target_mask.p + v.pix_off, mask, sizeof(double) * np,
                                       cudaMemcpyHostToDevice, c->stream));
    }
    sync(c);
    API_END
}

int cdr_set_target_f32(cdr_ctx* c, int32_t view, const float* rgb, const float* mask) {
    API_BEGIN(c)
    check_view(c, view);
    if (!rgb) throw ApiErr(CDR_ERR_INVALID_ARG, "target rgb is null");
    ViewData& v = c->views[view];
    const size_t np = size_t(v.cam.W) * v.cam.H;
    DBuf<float>& stage = c->scr_f;
    h2d(stage, rgb, 3 * np, c->stream);
    launch_widen(c, stage.p, int64_t(3 * np), c->target.p + 3 * v.pix_off);
    v.has_target = true;
    c->target_tone_gamma = -1;
    v.has_target_mask = mask != nullptr;
    v.target_mask_sum = 0;
    if (mask) {
        sync(c);  // the staging buffer is reused
        for (size_t i = 0; i < np; ++i) v.target_mask_sum += double(mask[i]);  // losses.cpp:26 order
        h2d(stage, mask, np, c->stream);
        launch_widen(c, stage.p, int64_t(np), c->target_mask.p + v.pix_off);
    }
    sync(c);
    API_END
}

int cdr_vertex_normals(cdr_ctx* c, double* out) {
    API_BEGIN(c)
    ensure_prepared(c);
    if (c->V > 0 && out)
        CDR_CUDA_CHECK(cudaMemcpyAsync(out, c->normals.p, sizeof(double) * 3 * c->V, cudaMemcpyDeviceToHost,
                                       c->stream));
    sync(c);
    API_END
}

int cdr_render(cdr_ctx* c, int32_t view, const cdr_settings* st, double* rgb, double* mask, int32_t* hit) {
    API_BEGIN(c)
    check_view(c, view);
    check_ready(c);
    if (!st) throw ApiErr(CDR_ERR_INVALID_ARG, "settings is null");
    int spp = spp_of(st);
    check_spp(spp);
    ensure_prepared(c);
    ensure_hit_arena(c, spp);
    reset_flags(c);
    RenderArgs a = render_args(c, st, nullptr);
    a.write_hits = hit != nullptr;
    int slot = view;
    launch_render(c, &slot, 1, a, true, false, false, nullptr);
    const ViewData& v = c->views[view];
    size_t np = size_t(v.cam.W) * v.cam.H;
    if (rgb)
        CDR_CUDA_CHECK(cudaMemcpyAsync(rgb, c->img.p + 3 * v.pix_off, sizeof(double) * 3 * np,
                                       cudaMemcpyDeviceToHost, c->stream));
    if (mask)
        CDR_CUDA_CHECK(cudaMemcpyAsync(mask, c->mask.p + v.pix_off, sizeof(double) * np, cudaMemcpyDeviceToHost,
                                       c->stream));
    if (hit)
        CDR_CUDA_CHECK(cudaMemcpyAsync(hit, c->hit.p + v.pix_off * spp, sizeof(int32_t) * np * spp,
                                       cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

int cdr_radiance_at(cdr_ctx* c, int32_t view, int32_t n, const double* xy, double* rgb, int32_t* tri) {
    API_BEGIN(c)
    check_view(c, view);
    check_ready(c);
    if (n <= 0) return;
    ensure_prepared(c);
    DBuf<double>&dxy = c->scr_d[0], &drgb = c->scr_d[1];
    DBuf<int32_t>& dtri = c->scr_i;
    h2d(dxy, xy, 2 * size_t(n), c->stream);
    drgb.ensure(3 * size_t(n));
    dtri.ensure(n);
    launch_radiance_points(c, view, n, dxy.p, drgb.p, dtri.p);
    CDR_CUDA_CHECK(cudaMemcpyAsync(rgb, drgb.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (tri) CDR_CUDA_CHECK(cudaMemcpyAsync(tri, dtri.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

int cdr_probe_points(cdr_ctx* c, int32_t view, int32_t n, const double* xy, double* rgb, int32_t* tri) {
    API_BEGIN(c)
    check_view(c, view);
    check_ready(c);
    if (n < 0 || (n > 0 && !xy)) throw ApiErr(CDR_ERR_INVALID_ARG, "bad probe points");
    if (n == 0) return;
    const auto it = std::find(c->beam_slots.begin(), c->beam_slots.end(), view);
    if (!c->beam_view.valid || it == c->beam_slots.end())
        throw ApiErr(CDR_ERR_INVALID_ARG, "the last render call built no candidate lists for this view");
    DBuf<double>&dxy = c->scr_d[0], &drgb = c->scr_d[1];
    DBuf<int32_t>& dtri = c->scr_i;
    h2d(dxy, xy, 2 * size_t(n), c->stream);
    drgb.ensure(3 * size_t(n));
    dtri.ensure(n);
    launch_probe_points(c, int(it - c->beam_slots.begin()), n, dxy.p, drgb.p, dtri.p);
    if (rgb) CDR_CUDA_CHECK(cudaMemcpyAsync(rgb, drgb.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    if (tri) CDR_CUDA_CHECK(cudaMemcpyAsync(tri, dtri.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

int cdr_view_loss(cdr_ctx* c, int32_t w, int32_t h, const double* rendered, const double* target,
                  const double* tmask, double lambda, double gamma, int32_t use_mask, double* value,
                  double* adjoint) {
    API_BEGIN(c)
    if (w <= 0 || h <= 0 || !rendered || !target || !adjoint)
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad view_loss arguments");
    size_t np = size_t(w) * h;
    if (value) *value = 0;
    std::memset(adjoint, 0, sizeof(double) * 3 * np);
    if (lambda == 0) return;  // losses.cpp:21
    const bool masked = use_mask && tmask;
    double n_valid = 0;
    if (masked) {
        for (size_t i = 0; i < np; ++i) n_valid += tmask[i];
        if (n_valid <= 0) return;
    } else {
        n_valid = double(w) * h;
    }
    const double scale = lambda / n_valid;
    DBuf<double>&dr = c->scr_d[0], &dt = c->scr_d[1], &dm = c->scr_d[2], &da = c->scr_d[3], &ds = c->scr_d[4];
    h2d(dr, rendered, 3 * np, c->stream);
    h2d(dt, target, 3 * np, c->stream);
    if (masked) h2d(dm, tmask, np, c->stream);
    da.ensure(3 * np);
    ds.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(ds.p, 0, sizeof(double), c->stream));
    launch_view_loss(c, w, h, dr.p, dt.p, masked ? dm.p : nullptr, scale, gamma, masked ? 1 : 0, da.p, ds.p);
    double sum = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(adjoint, da.p, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaMemcpyAsync(&sum, ds.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (value) *value = scale * sum;
    API_END
}

int cdr_interior_pass(cdr_ctx* c, int32_t view, const double* adjoint, const cdr_settings* st,
                      const int32_t* hit_cache, int64_t hit_len, const cdr_layout* lay, double* grad) {
    API_BEGIN(c)
    check_view(c, view);
    check_ready(c);
    check_layout(c, lay);
    if (!st || !adjoint || !grad) throw ApiErr(CDR_ERR_INVALID_ARG, "null argument");
    const ViewData& v = c->views[view];
    const int spp = spp_of(st);
    check_spp(spp);
    size_t np = size_t(v.cam.W) * v.cam.H;
    if (!hit_cache || hit_len != int64_t(np) * spp)  // diff_render.cpp:69-70
        throw SizeMismatchErr("hit cache does not match view and spp");
    ensure_prepared(c);
    ensure_hit_arena(c, spp);
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->adj.p + 3 * v.pix_off, adjoint, sizeof(double) * 3 * np,
                                   cudaMemcpyHostToDevice, c->stream));
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->hit.p + v.pix_off * spp, hit_cache, sizeof(int32_t) * np * spp,
                                   cudaMemcpyHostToDevice, c->stream));
    zero_grad(c, lay->total);
    reset_flags(c);
    RenderArgs a = render_args(c, st, lay);
    int slot = view;
    launch_render(c, &slot, 1, a, false, false, true, nullptr);
    launch_texel_flush(c, lay->diffuse, lay->specular, lay->roughness);
    launch_finalize_positions(c, lay->positions);
    sync(c);
    raise_device_error(c);
    add_grad_to_host(c, grad, 0, lay->total);
    API_END
}

int cdr_extract_silhouettes(cdr_ctx* c, int32_t view, cdr_segment* out, int32_t cap, int32_t* count,
                            double* total) {
    API_BEGIN(c)
    check_view(c, view);
    ensure_prepared(c);
    int slot = view;
    set_view_calls(c, &slot, nullptr, 1);
    launch_silhouettes(c, 1);
    launch_cdf(c, 1);
    int32_t n = 0;
    double tot[3] = {0, 0, 0};
    CDR_CUDA_CHECK(cudaMemcpyAsync(&n, c->sil_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaMemcpyAsync(tot, c->total_len.p, sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (count) *count = n;
    if (total) *total = tot[2];
    if (out && cap > 0 && n > 0)
        CDR_CUDA_CHECK(cudaMemcpy(out, c->segs.p, sizeof(cdr_segment) * std::min(cap, n), cudaMemcpyDeviceToHost));
    API_END
}

int cdr_boundary_pass(cdr_ctx* c, int32_t view, const double* adjoint, const cdr_segment* segments,
                      int32_t nseg, int32_t samples, uint64_t seed, int32_t probe, const cdr_layout* lay,
                      double* grad, int32_t* degenerate) {
    API_BEGIN(c)
    check_view(c, view);
    check_ready(c);
    check_layout(c, lay);
    if (!adjoint || !grad) throw ApiErr(CDR_ERR_INVALID_ARG, "null argument");
    if (degenerate) *degenerate = 0;
    if (samples <= 0) return;  // diff_render.cpp:210-211
    const ViewData& v = c->views[view];
    size_t np = size_t(v.cam.W) * v.cam.H;
    ensure_prepared(c);
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->adj.p + 3 * v.pix_off, adjoint, sizeof(double) * 3 * np,
                                   cudaMemcpyHostToDevice, c->stream));
    int slot = view;
    int m = samples;
    if (segments) {
        if (nseg < 0) throw ApiErr(CDR_ERR_INVALID_ARG, "negative segment count");
        for (int32_t i = 0; i < nseg; ++i)  // the deposits index the position gradient by v0/v1
            if (segments[i].v0 < 0 || segments[i].v0 >= c->V || segments[i].v1 < 0 || segments[i].v1 >= c->V)
                throw ApiErr(CDR_ERR_INVALID_ARG, "silhouette segment " + std::to_string(i) +
                                                      " references a vertex out of range (stale set?)");
        // a caller-provided set may hold more segments than the mesh has
        // edges: every per-view array (segments, CDF, guide, bins) is sized
        // and strided by max(E, nseg)
        set_view_calls(c, &slot, &m, 1, nseg);
        if (nseg > 0)
            CDR_CUDA_CHECK(cudaMemcpyAsync(c->segs.p, segments, sizeof(cdr_segment) * nseg, cudaMemcpyHostToDevice,
                                           c->stream));
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->sil_count.p, &nseg, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
        sync(c);
    } else {
        set_view_calls(c, &slot, &m, 1);
        launch_silhouettes(c, 1);
    }
    launch_cdf(c, 1);
    zero_grad(c, lay->total);
    reset_flags(c);
    launch_boundary(c, 1, m, seed, probe, lay->positions);
    sync(c);
    raise_device_error(c);
    if (degenerate)
        CDR_CUDA_CHECK(cudaMemcpy(degenerate, c->degenerate.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    add_grad_to_host(c, grad, lay->positions, 3 * int64_t(c->V));
    API_END
}

// NVTX range of one pipeline stage (host launch time; ncu --nvtx filters on it).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Scope in which the context's launchers target its side stream.
struct OnSideStream {
    cdr_ctx* c;
    explicit OnSideStream(cdr_ctx* ctx) : c(ctx) { std::swap(c->stream, c->side); }
    ~OnSideStream() { std::swap(c->stream, c->side); }
};
struct OnCopyStream {
    cdr_ctx* c;
    explicit OnCopyStream(cdr_ctx* ctx) : c(ctx) { std::swap(c->stream, c->copy); }
    ~OnCopyStream() { std::swap(c->stream, c->copy); }
};

// Page-locked host memory (cudaHostAlloc / cudaHostRegister): a copy into it
// on the copy stream runs asynchronously. Pageable destinations are copied
// at the end of the call as before (a pageable device-to-host copy blocks the
// host, which would hold back the launches behind it).
static bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// [off, off + n) pieces of a gradient layout
struct Span {
    int64_t off, n;
};
// The map and light segments of `lay` (final once the render and the texel
// flush are done, while the boundary pass still adds to the positions) when
// all segments are pairwise disjoint; empty otherwise.
static std::vector<Span> early_spans(const cdr_ctx* c, const cdr_layout* lay) {
    const int64_t nt = int64_t(c->tw) * c->th;
    std::vector<Span> all{{lay->positions, 3 * int64_t(c->V)}, {lay->diffuse, 3 * nt}, {lay->specular, 3 * nt},
                          {lay->roughness, nt}};
    if (lay->light >= 0) all.push_back({lay->light, 3});
    std::vector<Span> sorted = all;
    std::sort(sorted.begin(), sorted.end(), [](const Span& a, const Span& b) { return a.off < b.off; });
    for (size_t i = 1; i < sorted.size(); ++i)
        if (sorted[i - 1].off + sorted[i - 1].n > sorted[i].off) return {};
    return std::vector<Span>(all.begin() + 1, all.end());
}
// [0, total) minus the (disjoint) spans
static std::vector<Span> complement(std::vector<Span> sp, int64_t total) {
    std::sort(sp.begin(), sp.end(), [](const Span& a, const Span& b) { return a.off < b.off; });
    std::vector<Span> out;
    int64_t at = 0;
    for (const Span& x : sp) {
        if (x.off > at) out.push_back({at, x.off - at});
        at = std::max(at, x.off + x.n);
    }
    if (total > at) out.push_back({at, total - at});
    return out;
}

// The fused total_loss pipeline (losses.cpp:244-297). terms[6] = rend, lap,
// normal, edge, spec, roug; reg == nullptr leaves the last four at 0.
static void loss_grad_impl(cdr_ctx* c, const int32_t* views, int32_t n, const cdr_settings* st, double lambda_rend,
                    double lambda_lap, const cdr_reg_weights* reg, int32_t lap_mode, int32_t use_mask,
                    const cdr_layout* lay, double* terms_out, double* grad, double* rendered_rgb,
                    double* rendered_mask, cdr_stats* stats) {
    if (!st || n < 0 || (n > 0 && !views)) throw ApiErr(CDR_ERR_INVALID_ARG, "bad arguments");
    // parameters staged by cdr_stage_params: uploaded below, after every check
    const cdr_ctx::Staged sp = std::exchange(c->staged, cdr_ctx::Staged{});
    if (sp.d) check_layout(c, lay, sp.w, sp.h);
    else check_layout(c, lay);
    check_ready(c);
    const int spp = spp_of(st);
    check_spp(spp);
    std::vector<int> slots(views, views + n);
    std::vector<double> scales(n);
    std::vector<int> samples(n);
    int max_samples = 0;
    for (int i = 0; i < n; ++i) {
        check_view(c, slots[i]);
        const ViewData& v = c->views[slots[i]];
        if (!v.has_target) throw SizeMismatchErr("target count does not match views");  // losses.cpp:247
        const bool masked = use_mask && v.has_target_mask;
        double n_valid = masked ? v.target_mask_sum : double(v.cam.W) * v.cam.H;
        scales[i] = (lambda_rend == 0 || n_valid <= 0) ? 0.0 : lambda_rend / n_valid;
        samples[i] = st->boundary_samples > 0 ? st->boundary_samples : v.cam.W * v.cam.H;
        max_samples = std::max(max_samples, samples[i]);
    }
    NvtxRange whole("cdr.total_loss");
    cudaStream_t s = c->stream;
    auto& ev = c->ev;
    c->launches = 0;
    if (sp.pos && c->V > 0) {  // needed first (normals, LBVH): on the main stream
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->pos.p, sp.pos, sizeof(double) * 3 * size_t(c->V), cudaMemcpyHostToDevice, s));
        c->geometry_dirty = true;
    }
    // staged maps: upload + texel packing on the copy stream, beside the
    // LBVH, silhouettes and visibility; joined before the regularisers and
    // the shading (pinned buffers overlap; pageable ones block here)
    const bool maps_pending = sp.d != nullptr;
    if (maps_pending) {
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_copy, s));
        CDR_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->ev_copy, 0));
        {
            OnCopyStream cs(c);
            set_textures_impl(c, sp.d, sp.s, sp.r, sp.w, sp.h);
        }
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_maps, c->copy));
    }
    std::optional<NvtxRange> stage(std::in_place, "cdr.prepare (normals, LBVH)");
    CDR_CUDA_CHECK(cudaEventRecord(ev[0], s));
    zero_grad(c, lay->total);  // fresh GradVector (losses.cpp:250)
    reset_flags(c);
    ensure_hit_arena(c, spp);
    CDR_CUDA_CHECK(cudaMemsetAsync(c->loss_acc.p, 0, sizeof(double) * c->views.size(), s));
    ensure_prepared(c, /*force=*/true);  // GradContext is rebuilt per total_loss (losses.cpp:251)
    if (c->target_tone_gamma != st->gamma) {
        launch_tone_targets(c, st->gamma);
        c->target_tone_gamma = st->gamma;
    }
    CDR_CUDA_CHECK(cudaEventRecord(ev[1], s));
    stage.emplace("cdr.silhouettes+cdf+regularisers (side stream)");
    // Side stream: silhouettes + CDF (they need only the prepared geometry) and
    // the regularisers (mesh + maps, into their own gradient buffer) run
    // beside the render; the main stream joins them where their results are used.
    const bool lap_here = c->rank == 0;  // computed once across ranks
    const bool reg_here = lap_here && reg;
    CDR_CUDA_CHECK(cudaEventRecord(c->ev_fork, s));
    CDR_CUDA_CHECK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    c->reg_vals.ensure(4);
    {
        OnSideStream side(c);
        if (st->boundary_term) {
            set_view_calls(c, slots.data(), samples.data(), n);
            launch_silhouettes(c, n);
            launch_cdf(c, n);
            launch_boundary_sampling(c, n, max_samples, st->seed);  // beside the render as well
        }
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_sil, c->stream));
        CDR_CUDA_CHECK(cudaMemsetAsync(c->reg_vals.p, 0, sizeof(double) * 4, c->stream));
        if (reg_here) {
            if (maps_pending) CDR_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_maps, 0));
            c->reg_grad.ensure(std::max<int64_t>(1, lay->total));
            CDR_CUDA_CHECK(cudaMemsetAsync(c->reg_grad.p, 0, sizeof(double) * std::max<int64_t>(1, lay->total),
                                           c->stream));
            launch_regularisers(c, *reg, *lay, c->reg_grad.p, c->reg_vals.p);
        }
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_reg, c->stream));
    }
    RenderArgs a = render_args(c, st, lay);
    a.use_mask = use_mask;
    // page-locked image destinations: downloaded on the copy stream, group by
    // group during the shading when the call runs in queue mode, else after it
    const bool out_images = (rendered_rgb || rendered_mask) && (!rendered_rgb || is_pinned(rendered_rgb)) &&
                            (!rendered_mask || is_pinned(rendered_mask));
    if (out_images) {
        a.img_rgb_host = rendered_rgb;
        a.img_mask_host = rendered_mask;
    }
    stage.emplace("cdr.render (lists, trace, shade+loss+interior)");
    if (maps_pending) {  // the list builders and k_trace read no texel: join just before the shading
        a.wait_before_shade = c->ev_maps;
    }
    launch_render(c, slots.data(), n, a, true, true, true, scales.data(), ev[7]);
    CDR_CUDA_CHECK(cudaEventRecord(ev[2], s));
    // Downloads that need only the render run on the copy stream beside the
    // boundary pass: the K images, then (one rank, overwrite) the map and
    // light segments of the gradient once the texel flush has written them.
    if (out_images && !c->images_downloaded) {
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_copy, s));
        CDR_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->ev_copy, 0));
        size_t ro = 0, mo = 0;
        for (int i = 0; i < n; ++i) {
            const ViewData& v = c->views[slots[i]];
            size_t np = size_t(v.cam.W) * v.cam.H;
            if (rendered_rgb)
                CDR_CUDA_CHECK(cudaMemcpyAsync(rendered_rgb + ro, c->img.p + 3 * v.pix_off, sizeof(double) * 3 * np,
                                               cudaMemcpyDeviceToHost, c->copy));
            if (rendered_mask)
                CDR_CUDA_CHECK(cudaMemcpyAsync(rendered_mask + mo, c->mask.p + v.pix_off, sizeof(double) * np,
                                               cudaMemcpyDeviceToHost, c->copy));
            ro += 3 * np;
            mo += np;
        }
    }
    launch_texel_flush(c, lay->diffuse, lay->specular, lay->roughness);  // independent of the boundary pass
    const std::vector<Span> early =
        (grad && (st->flags & CDR_FLAG_GRAD_OVERWRITE) && !c->nccl_comm && is_pinned(grad)) ? early_spans(c, lay)
                                                                                             : std::vector<Span>{};
    if (!early.empty()) {
        CDR_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_reg, 0));  // the regularisers' map gradient
        if (reg_here)
            for (const Span& x : early) launch_axpy(c, c->grad.p + x.off, c->reg_grad.p + x.off, x.n);
        CDR_CUDA_CHECK(cudaEventRecord(c->ev_copy, s));
        CDR_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->ev_copy, 0));
        for (const Span& x : early)
            if (x.n > 0)
                CDR_CUDA_CHECK(cudaMemcpyAsync(grad + x.off, c->grad.p + x.off, sizeof(double) * x.n,
                                               cudaMemcpyDeviceToHost, c->copy));
    }
    CDR_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_sil, 0));  // segments + CDF for the boundary pass
    CDR_CUDA_CHECK(cudaEventRecord(ev[3], s));
    stage.emplace("cdr.boundary");
    if (st->boundary_term)  // the render above built candidate lists for exactly these views
        launch_boundary_probes(c, n, max_samples, st->seed, CDR_PROBE_RADIANCE, lay->positions, /*use_beam=*/true);
    CDR_CUDA_CHECK(cudaEventRecord(ev[4], s));
    stage.emplace("cdr.finalize (texel flush, normal chain, Laplacian)");
    launch_finalize_positions(c, lay->positions);
    if (lap_here) launch_laplacian(c, lap_mode, lambda_lap, c->grad.p + lay->positions);
    CDR_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_reg, 0));  // the regularisers' gradient and values
    const std::vector<Span> late = early.empty() ? std::vector<Span>{{0, lay->total}} : complement(early, lay->total);
    if (reg_here)  // grad += reg_grad (the early segments got theirs above)
        for (const Span& x : late) launch_axpy(c, c->grad.p + x.off, c->reg_grad.p + x.off, x.n);
    CDR_CUDA_CHECK(cudaEventRecord(ev[5], s));
    stage.emplace("cdr.allreduce + download");
    if (c->nccl_comm)
        nccl_check(nccl().allReduce(c->grad.p, c->grad.p, size_t(lay->total), kNcclFloat64, kNcclSum, c->nccl_comm, s),
                   "ncclAllReduce(grad)");
    CDR_CUDA_CHECK(cudaEventRecord(ev[6], s));
    std::vector<double> lacc(c->views.size());
    double lap_sq = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(lacc.data(), c->loss_acc.p, sizeof(double) * lacc.size(), cudaMemcpyDeviceToHost, s));
    if (lap_here)  // ranks > 0 never run the Laplacian (its buffers may not exist)
        CDR_CUDA_CHECK(cudaMemcpyAsync(&lap_sq, c->lap_partial.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    double regv[4] = {0, 0, 0, 0};
    CDR_CUDA_CHECK(cudaMemcpyAsync(regv, c->reg_vals.p, sizeof(regv), cudaMemcpyDeviceToHost, s));
    if (grad && (st->flags & CDR_FLAG_GRAD_OVERWRITE)) {
        for (const Span& x : late)
            if (x.n > 0)
                CDR_CUDA_CHECK(cudaMemcpyAsync(grad + x.off, c->grad.p + x.off, sizeof(double) * x.n,
                                               cudaMemcpyDeviceToHost, s));
    } else if (grad) {
        add_grad_to_host(c, grad, 0, lay->total);
    }
    if (!out_images) {  // pageable (or no) image buffers: at the end, on the main stream
        size_t ro = 0, mo = 0;
        for (int i = 0; i < n; ++i) {
            const ViewData& v = c->views[slots[i]];
            size_t np = size_t(v.cam.W) * v.cam.H;
            if (rendered_rgb)
                CDR_CUDA_CHECK(cudaMemcpyAsync(rendered_rgb + ro, c->img.p + 3 * v.pix_off, sizeof(double) * 3 * np,
                                               cudaMemcpyDeviceToHost, s));
            if (rendered_mask)
                CDR_CUDA_CHECK(cudaMemcpyAsync(rendered_mask + mo, c->mask.p + v.pix_off, sizeof(double) * np,
                                               cudaMemcpyDeviceToHost, s));
            ro += 3 * np;
            mo += np;
        }
    }
    sync(c);
    CDR_CUDA_CHECK(cudaStreamSynchronize(c->copy));
    raise_device_error(c);
    // rendering term in view order, each view scale * Σ m|d| (losses.cpp:44-47, :257)
    double terms[6] = {0.0, lap_here ? lambda_lap * lap_sq : 0.0, regv[0], regv[1], regv[2], regv[3]};
    for (int i = 0; i < n; ++i) terms[0] += scales[i] * lacc[slots[i]];
    if (c->nccl_comm) {  // sum the loss terms of all view shards
        DBuf<double>& dterm = c->scr_d[0];
        dterm.ensure(6);
        CDR_CUDA_CHECK(cudaMemcpyAsync(dterm.p, terms, sizeof(terms), cudaMemcpyHostToDevice, s));
        nccl_check(nccl().allReduce(dterm.p, dterm.p, 6, kNcclFloat64, kNcclSum, c->nccl_comm, s),
                   "ncclAllReduce(loss)");
        CDR_CUDA_CHECK(cudaMemcpyAsync(terms, dterm.p, sizeof(terms), cudaMemcpyDeviceToHost, s));
        sync(c);
    }
    if (terms_out)
        for (int i = 0; i < 6; ++i) terms_out[i] = terms[i];
    if (stats) {
        Counters k;
        CDR_CUDA_CHECK(cudaMemcpy(&k, c->counters.p, sizeof(k), cudaMemcpyDeviceToHost));
        std::memset(stats, 0, sizeof(*stats));
        for (int i = 0; i < n; ++i) {
            const ViewData& v = c->views[slots[i]];
            stats->pixels += int64_t(v.cam.W) * v.cam.H;
            stats->samples += int64_t(v.cam.W) * v.cam.H * spp;
            if (st->boundary_term) stats->boundary_samples += samples[i];
        }
        stats->hit_samples = int64_t(k.hit_samples);
        stats->adjoint_samples = int64_t(k.adjoint_samples);
        stats->boundary_active = int64_t(k.boundary_active);
        stats->beam_fallback_tiles = int64_t(k.beam_fallback_tiles);
        stats->shaded_samples = int64_t(k.shaded_samples);
        if (st->boundary_term) {
            std::vector<int32_t> cnt(n), deg(n);
            CDR_CUDA_CHECK(cudaMemcpy(cnt.data(), c->sil_count.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
            CDR_CUDA_CHECK(cudaMemcpy(deg.data(), c->degenerate.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
            for (int i = 0; i < n; ++i) {
                stats->segments += cnt[i];
                stats->degenerate_skipped += deg[i];
            }
        }
        float ms[7];
        for (int i = 0; i < 6; ++i) CDR_CUDA_CHECK(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
        stats->ms_prepare = ms[0];
        stats->ms_render = ms[1];
        stats->ms_trace = render_trace_ms(c);
        stats->ms_silhouette = ms[2];
        stats->ms_boundary = ms[3];
        stats->ms_finalize = ms[4];
        float tot;
        CDR_CUDA_CHECK(cudaEventElapsedTime(&tot, ev[0], ev[6]));
        stats->ms_total = tot;
        stats->kernel_launches = c->launches;
    }
}



int cdr_loss_grad(cdr_ctx* c, const int32_t* views, int32_t n, const cdr_settings* st, double lambda_rend,
                  double lambda_lap, int32_t lap_mode, int32_t use_mask, const cdr_layout* lay, double* loss_out,
                  double* grad, double* rendered_rgb, double* rendered_mask, cdr_stats* stats) {
    API_BEGIN_STAGED(c)
    double terms[6];
    loss_grad_impl(c, views, n, st, lambda_rend, lambda_lap, nullptr, lap_mode, use_mask, lay, terms, grad,
                   rendered_rgb, rendered_mask, stats);
    if (loss_out) {
        loss_out[0] = terms[0];
        loss_out[1] = terms[1];
    }
    API_END_STAGED
}

int cdr_total_loss(cdr_ctx* c, const int32_t* views, int32_t n, const cdr_settings* st, double lambda_rend,
                   double lambda_lap, const cdr_reg_weights* reg, int32_t lap_mode, int32_t use_mask,
                   const cdr_layout* lay, double* breakdown, double* grad, double* rendered_rgb,
                   double* rendered_mask, cdr_stats* stats) {
    API_BEGIN_STAGED(c)
    if (!reg) throw ApiErr(CDR_ERR_INVALID_ARG, "reg weights are required");
    double t[6];
    loss_grad_impl(c, views, n, st, lambda_rend, lambda_lap, reg, lap_mode, use_mask, lay, t, grad, rendered_rgb,
                   rendered_mask, stats);
    if (breakdown) {  // LossBreakdown, total in the reference's order (losses.cpp:294-295)
        breakdown[0] = t[0] + t[1] + t[2] + t[3] + t[4] + t[5];
        for (int i = 0; i < 6; ++i) breakdown[1 + i] = t[i];
    }
    API_END_STAGED
}

int cdr_regularisers(cdr_ctx* c, const cdr_reg_weights* reg, const cdr_layout* lay, double* values,
                     double* grad) {
    API_BEGIN(c)
    if (!reg) throw ApiErr(CDR_ERR_INVALID_ARG, "reg weights are required");
    check_layout(c, lay);
    check_ready(c);
    c->reg_vals.ensure(4);
    double* gdev = nullptr;
    if (grad) {  // private zeroed gradient, then += into the caller's buffer
        c->reg_grad.ensure(std::max<int64_t>(1, lay->total));
        CDR_CUDA_CHECK(cudaMemsetAsync(c->reg_grad.p, 0, sizeof(double) * std::max<int64_t>(1, lay->total),
                                       c->stream));
        gdev = c->reg_grad.p;
    } else {
        if (c->grad_n != lay->total) zero_grad(c, lay->total);
        gdev = c->grad.p;
    }
    launch_regularisers(c, *reg, *lay, gdev, c->reg_vals.p);
    double v[4];
    CDR_CUDA_CHECK(cudaMemcpyAsync(v, c->reg_vals.p, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (values)
        for (int i = 0; i < 4; ++i) values[i] = v[i];
    if (grad) {
        std::vector<double> g(size_t(lay->total));
        CDR_CUDA_CHECK(cudaMemcpy(g.data(), gdev, sizeof(double) * g.size(), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < g.size(); ++i) grad[i] += g[i];
    }
    API_END
}

int cdr_get_grad(cdr_ctx* c, double* out, int64_t n) {
    API_BEGIN(c)
    if (n > c->grad_n) throw SizeMismatchErr("gradient buffer smaller than requested");
    if (n > 0) CDR_CUDA_CHECK(cudaMemcpyAsync(out, c->grad.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

int cdr_set_grad(cdr_ctx* c, const double* g, int64_t n) {
    API_BEGIN(c)
    if (n < 0 || (n > 0 && !g)) throw ApiErr(CDR_ERR_INVALID_ARG, "bad gradient");
    c->grad.ensure(std::max<int64_t>(1, n));
    c->grad_n = n;
    if (n > 0) CDR_CUDA_CHECK(cudaMemcpyAsync(c->grad.p, g, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    sync(c);
    API_END
}

int cdr_grad_device_ptr(cdr_ctx* c, void** ptr, int64_t* n) {
    if (!c || !ptr) return CDR_ERR_INVALID_ARG;
    *ptr = c->grad.p;
    if (n) *n = c->grad_n;
    return CDR_OK;
}

int cdr_laplacian_matrix(cdr_ctx* c, int32_t mode, int32_t* outer, int32_t* inner, double* values, int64_t* nnz) {
    API_BEGIN(c)
    int64_t z = int64_t(c->V) + 2 * int64_t(c->E);
    if (nnz) *nnz = z;
    if (!outer && !inner && !values) return;
    launch_laplacian(c, mode, 0.0, nullptr);
    // L is symmetric, so its CSR (row-sorted) equals Eigen's CSC layout
    if (outer) CDR_CUDA_CHECK(cudaMemcpyAsync(outer, c->lap_rowptr.p, sizeof(int32_t) * (size_t(c->V) + 1),
                                              cudaMemcpyDeviceToHost, c->stream));
    if (inner && z) CDR_CUDA_CHECK(cudaMemcpyAsync(inner, c->lap_col.p, sizeof(int32_t) * z, cudaMemcpyDeviceToHost,
                                                   c->stream));
    if (values && z) CDR_CUDA_CHECK(cudaMemcpyAsync(values, c->lap_val.p, sizeof(double) * z, cudaMemcpyDeviceToHost,
                                                    c->stream));
    sync(c);
    API_END
}

int cdr_laplacian_loss(cdr_ctx* c, int32_t mode, double lambda, double* value, double* grad) {
    API_BEGIN(c)
    if (value) *value = 0;
    if (lambda == 0 || c->V == 0) return;  // losses.cpp:69
    c->lap_grad.ensure(size_t(3) * c->V);
    CDR_CUDA_CHECK(cudaMemsetAsync(c->lap_grad.p, 0, sizeof(double) * 3 * c->V, c->stream));
    launch_laplacian(c, mode, lambda, c->lap_grad.p);
    double sq = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(&sq, c->lap_partial.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    std::vector<double> g(size_t(3) * c->V);
    CDR_CUDA_CHECK(cudaMemcpyAsync(g.data(), c->lap_grad.p, sizeof(double) * g.size(), cudaMemcpyDeviceToHost,
                                   c->stream));
    sync(c);
    if (value) *value = lambda * sq;
    if (grad)
        for (size_t i = 0; i < g.size(); ++i) grad[i] += g[i];
    API_END
}

int cdr_lbvh_keys(cdr_ctx* c, uint64_t* keys_out, int32_t n) {
    API_BEGIN(c)
    if (n != c->T) throw SizeMismatchErr("key buffer must hold one key per triangle");
    ensure_prepared(c);
    if (n > 0)
        CDR_CUDA_CHECK(cudaMemcpyAsync(keys_out, c->keys.p, sizeof(uint64_t) * size_t(n), cudaMemcpyDeviceToHost,
                                       c->stream));
    sync(c);
    API_END
}

int cdr_get_rendered(cdr_ctx* c, int32_t view, double* rgb, double* mask) {
    API_BEGIN(c)
    check_view(c, view);
    const ViewData& v = c->views[view];
    const size_t np = size_t(v.cam.W) * v.cam.H;
    if (c->img.n < v.pix_off + np) throw ApiErr(CDR_ERR_INVALID_ARG, "view has not been rendered");
    if (rgb)
        CDR_CUDA_CHECK(cudaMemcpyAsync(rgb, c->img.p + 3 * v.pix_off, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost,
                                       c->stream));
    if (mask)
        CDR_CUDA_CHECK(cudaMemcpyAsync(mask, c->mask.p + v.pix_off, sizeof(double) * np, cudaMemcpyDeviceToHost,
                                       c->stream));
    sync(c);
    API_END
}

int cdr_host_alloc(size_t bytes, void** out) {
    if (!out) return CDR_ERR_INVALID_ARG;
    *out = nullptr;
    if (cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return CDR_ERR_CUDA;
    }
    return CDR_OK;
}

void cdr_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

namespace {
// The geometry-only context (lazy): an arbitrary mesh for the query entry
// points, its LBVH built; the render mesh stays untouched. The topology is
// cached across calls (robust_evolve / uv_transfer pass one topology often).
cdr_ctx* load_geometry(cdr_ctx* c, const double* positions, int32_t nv, const int32_t* triangles, int32_t nt) {
    for (int64_t i = 0; i < 3 * int64_t(nt); ++i)
        if (triangles[i] < 0 || triangles[i] >= nv)
            throw ApiErr(CDR_ERR_INVALID_ARG, "triangle references a vertex out of range");
    if (!c->geo) {
        const int rc = cdr_create(c->device, &c->geo);
        if (rc != CDR_OK) throw ApiErr(rc, "cannot create the geometry context");
    }
    cdr_ctx* g = c->geo;
    cudaStream_t s = g->stream;
    if (g->T != nt || g->V != nv || g->h_tris.size() != 3 * size_t(nt) ||
        std::memcmp(g->h_tris.data(), triangles, sizeof(int32_t) * 3 * size_t(nt)) != 0) {
        g->V = nv;
        g->T = nt;
        g->h_tris.assign(triangles, triangles + 3 * size_t(nt));
        h2d(g->tris, triangles, 3 * size_t(nt), s);
        g->topo_version = ~0ull;  // not a copy of c's topology (sync_topology re-copies)
    }
    h2d(g->pos, positions, 3 * size_t(nv), s);
    launch_bvh(g, 0.0);
    return g;
}
}  // namespace

int cdr_closest_points(cdr_ctx* c, const double* positions, int32_t nv, const int32_t* triangles, int32_t nt,
                       const double* queries, int32_t nq, int32_t* tri_out, double* point_out, double* dist_out,
                       double* bary_out) {
    API_BEGIN(c)
    if (nv < 0 || nt < 0 || nq < 0 || (nv > 0 && !positions) || (nt > 0 && !triangles) || (nq > 0 && !queries))
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad closest_points arguments");
    if (nq == 0) return;
    if (nt == 0) {  // bvh.cpp:270: no nodes -> tri -1, distance 1e300
        for (int i = 0; i < nq; ++i) {
            if (tri_out) tri_out[i] = -1;
            if (dist_out) dist_out[i] = 1e300;
            for (int k = 0; k < 3; ++k) {
                if (point_out) point_out[3 * i + k] = 0;
                if (bary_out) bary_out[3 * i + k] = 0;
            }
        }
        return;
    }
    cdr_ctx* g = load_geometry(c, positions, nv, triangles, nt);
    DBuf<double>&q = g->scr_d[0], &pt = g->scr_d[1], &di = g->scr_d[2], &ba = g->scr_d[3];
    DBuf<int32_t>& tr = g->scr_i;
    h2d(q, queries, 3 * size_t(nq), g->stream);
    tr.ensure(nq);
    pt.ensure(3 * size_t(nq));
    di.ensure(nq);
    ba.ensure(3 * size_t(nq));
    launch_closest(g, q.p, nq, tr.p, pt.p, di.p, ba.p);
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        if (dst) CDR_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g->stream));
    };
    d2h(tri_out, tr.p, sizeof(int32_t) * nq);
    d2h(point_out, pt.p, sizeof(double) * 3 * nq);
    d2h(dist_out, di.p, sizeof(double) * nq);
    d2h(bary_out, ba.p, sizeof(double) * 3 * nq);
    CDR_CUDA_CHECK(cudaStreamSynchronize(g->stream));
    API_END
}

int cdr_self_intersects(cdr_ctx* c, const double* positions, int32_t nv, const int32_t* triangles, int32_t nt,
                        int32_t* result, int32_t* pairs, int64_t cap, int64_t* n_pairs) {
    API_BEGIN(c)
    if (nv < 0 || nt < 0 || (nv > 0 && !positions) || (nt > 0 && !triangles) || !result || cap < 0 ||
        (cap > 0 && !pairs))
        throw ApiErr(CDR_ERR_INVALID_ARG, "bad self_intersects arguments");
    for (int64_t i = 0; i < 3 * int64_t(nt); ++i)
        if (triangles[i] < 0 || triangles[i] >= nv)
            throw ApiErr(CDR_ERR_INVALID_ARG, "triangle references a vertex out of range");
    *result = 0;
    if (n_pairs) *n_pairs = 0;
    if (nt < 2) return;  // mesh.cpp:186
    cdr_ctx* g = load_geometry(c, positions, nv, triangles, nt);
    const bool want = pairs != nullptr || n_pairs != nullptr;
    long long n = 0;
    if (!want) {
        n = launch_self_intersect(g, nullptr, 0);
    } else {
        size_t capd = std::max<size_t>(4096, c->si_pairs.n);
        while (true) {
            c->si_pairs.ensure(capd);
            n = launch_self_intersect(g, c->si_pairs.p, (long long)c->si_pairs.n);
            if (n <= (long long)c->si_pairs.n) break;
            capd = size_t(n);  // rerun with room for every pair
        }
        std::vector<int2> h(static_cast<size_t>(n));
        if (n > 0)
            CDR_CUDA_CHECK(cudaMemcpy(h.data(), c->si_pairs.p, sizeof(int2) * size_t(n), cudaMemcpyDeviceToHost));
        std::sort(h.begin(), h.end(), [](int2 a, int2 b) { return a.x != b.x ? a.x < b.x : a.y < b.y; });
        for (int64_t i = 0; i < std::min<int64_t>(cap, n); ++i) {
            pairs[2 * i] = h[size_t(i)].x;
            pairs[2 * i + 1] = h[size_t(i)].y;
        }
        if (n_pairs) *n_pairs = n;
    }
    *result = n > 0 ? 1 : 0;
    API_END
}

// ---- resident optimiser (optimize.cu) --------------------------------------
namespace {
cdr_ctx* geometry_ctx(cdr_ctx* c) {
    if (!c->geo) {
        const int rc = cdr_create(c->device, &c->geo);
        if (rc != CDR_OK) throw ApiErr(rc, "cannot create the geometry context");
    }
    return c->geo;
}

// geo <- c's topology (device copy), tracked by version
void sync_topology(cdr_ctx* c, cdr_ctx* g) {
    if (g->topo_version == c->topo_version && g->T == c->T && g->V == c->V && g->h_tris.size() == c->h_tris.size())
        return;
    g->V = c->V;
    g->T = c->T;
    g->h_tris = c->h_tris;
    g->tris.ensure(std::max<size_t>(1, 3 * size_t(c->T)));
    CDR_CUDA_CHECK(cudaMemcpyAsync(g->tris.p, c->tris.p, sizeof(int32_t) * 3 * size_t(c->T), cudaMemcpyDeviceToDevice,
                                   g->stream));
    g->pos.ensure(std::max<size_t>(1, 3 * size_t(c->V)));
    g->topo_version = c->topo_version;
}

// self_intersects of g's mesh (positions already in g->pos)
bool geo_self_intersects(cdr_ctx* g) {
    launch_bvh(g, 0.0);
    return launch_self_intersect(g, nullptr, 0) > 0;
}
}  // namespace

int cdr_adam_init(cdr_ctx* c, const cdr_adam_config* cfg, const cdr_layout* lay) {
    API_BEGIN(c)
    if (!cfg) throw ApiErr(CDR_ERR_INVALID_ARG, "config is required");
    check_layout(c, lay);
    c->adam_cfg = *cfg;
    c->adam_lay = *lay;
    c->adam_step = 0;
    const size_t n = std::max<int64_t>(1, lay->total);
    c->adam_m.ensure(n);
    c->adam_v.ensure(n);
    CDR_CUDA_CHECK(cudaMemsetAsync(c->adam_m.p, 0, sizeof(double) * n, c->stream));
    CDR_CUDA_CHECK(cudaMemsetAsync(c->adam_v.p, 0, sizeof(double) * n, c->stream));
    c->adam_disp.ensure(std::max<size_t>(1, 3 * size_t(c->V)));
    CDR_CUDA_CHECK(cudaMemsetAsync(c->adam_disp.p, 0, sizeof(double) * std::max<size_t>(1, 3 * size_t(c->V)),
                                   c->stream));
    c->adam_light.ensure(3);
    c->adam_ready = true;
    sync(c);
    API_END
}

int cdr_adam_step(cdr_ctx* c, double* disp_out, int64_t* step_out) {
    API_BEGIN(c)
    if (!c->adam_ready) throw ApiErr(CDR_ERR_INVALID_ARG, "cdr_adam_init first (or again after cdr_set_mesh)");
    const cdr_layout& L = c->adam_lay;
    if (c->grad_n != L.total) throw SizeMismatchErr("adam state/params/grad layout mismatch");  // adam.cpp:10-11
    if (any_nonfinite(c, c->grad.p, L.total))
        throw ApiErr(CDR_ERR_NONFINITE, "non-finite gradient entering adam");  // adam.cpp:12-13
    c->adam_step += 1;
    const double corr1 = 1.0 - std::pow(c->adam_cfg.beta1, double(c->adam_step));
    const double corr2 = 1.0 - std::pow(c->adam_cfg.beta2, double(c->adam_step));
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->adam_light.p, c->light, sizeof(double) * 3, cudaMemcpyHostToDevice, c->stream));
    launch_adam(c, c->grad.p, corr1, corr2);
    if (L.light >= 0)
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->light, c->adam_light.p, sizeof(double) * 3, cudaMemcpyDeviceToHost,
                                       c->stream));
    if (c->tw > 0) launch_pack_textures(c, c->map_d.p, c->map_s.p, c->map_r.p, c->tw * c->th);
    if (disp_out)
        CDR_CUDA_CHECK(cudaMemcpyAsync(disp_out, c->adam_disp.p, sizeof(double) * 3 * size_t(c->V),
                                       cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (step_out) *step_out = c->adam_step;
    API_END
}

int cdr_adam_get_state(cdr_ctx* c, double* m, double* v, int64_t* step) {
    API_BEGIN(c)
    if (!c->adam_ready) throw ApiErr(CDR_ERR_INVALID_ARG, "no optimiser state");
    const size_t n = size_t(c->adam_lay.total);
    if (m) CDR_CUDA_CHECK(cudaMemcpyAsync(m, c->adam_m.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    if (v) CDR_CUDA_CHECK(cudaMemcpyAsync(v, c->adam_v.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (step) *step = c->adam_step;
    API_END
}

int cdr_adam_set_state(cdr_ctx* c, const double* m, const double* v, int64_t step) {
    API_BEGIN(c)
    if (!c->adam_ready) throw ApiErr(CDR_ERR_INVALID_ARG, "cdr_adam_init first");
    const size_t n = size_t(c->adam_lay.total);
    if (m) CDR_CUDA_CHECK(cudaMemcpyAsync(c->adam_m.p, m, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    if (v) CDR_CUDA_CHECK(cudaMemcpyAsync(c->adam_v.p, v, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    c->adam_step = step;
    sync(c);
    API_END
}

int cdr_evolve(cdr_ctx* c, const double* disp_host, double* scale_out, double* positions_out) {
    API_BEGIN(c)
    if (scale_out) *scale_out = 0.0;
    cdr_ctx* g = geometry_ctx(c);
    sync(c);
    sync_topology(c, g);
    const int64_t n = 3 * int64_t(c->V);
    const double* disp = c->adam_disp.p;
    if (disp_host) {
        c->grad_tmp.ensure(std::max<int64_t>(1, n));
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->grad_tmp.p, disp_host, sizeof(double) * n, cudaMemcpyHostToDevice, g->stream));
        disp = c->grad_tmp.p;
    } else if (!c->adam_ready) {
        throw ApiErr(CDR_ERR_INVALID_ARG, "no displacement: pass one or run cdr_adam_step");
    }
    // evolve.cpp:23: the input must be intersection-free
    CDR_CUDA_CHECK(cudaMemcpyAsync(g->pos.p, c->pos.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, g->stream));
    if (geo_self_intersects(g)) throw ApiErr(CDR_ERR_SELF_INTERSECTING, "input mesh self-intersects");
    double applied = 0.0;
    if (!any_nonzero(g, disp, n)) {
        applied = 1.0;  // evolve.cpp:26-35
    } else {
        double s = 1.0;
        for (int attempt = 0; attempt <= 8; ++attempt, s *= 0.5) {  // evolve.cpp:39-48
            launch_candidate(g, c->pos.p, disp, s, g->pos.p);
            if (min_triangle_area(g, g->pos.p) <= 1e-12) continue;
            if (!geo_self_intersects(g)) {
                CDR_CUDA_CHECK(cudaMemcpyAsync(c->pos.p, g->pos.p, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                               g->stream));
                CDR_CUDA_CHECK(cudaStreamSynchronize(g->stream));
                c->geometry_dirty = true;
                applied = s;
                break;
            }
        }
    }
    CDR_CUDA_CHECK(cudaStreamSynchronize(g->stream));
    if (positions_out)
        CDR_CUDA_CHECK(cudaMemcpy(positions_out, c->pos.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (scale_out) *scale_out = applied;
    API_END
}

int cdr_get_params(cdr_ctx* c, const cdr_layout* lay, double* out) {
    API_BEGIN(c)
    check_layout(c, lay);
    if (!out) throw ApiErr(CDR_ERR_INVALID_ARG, "params_out is required");
    const size_t nt = size_t(c->tw) * c->th;
    auto d2h = [&](int64_t off, const double* src, size_t n) {
        if (off >= 0 && n)
            CDR_CUDA_CHECK(cudaMemcpyAsync(out + off, src, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    };
    d2h(lay->positions, c->pos.p, 3 * size_t(c->V));
    d2h(lay->diffuse, c->map_d.p, 3 * nt);
    d2h(lay->specular, c->map_s.p, 3 * nt);
    d2h(lay->roughness, c->map_r.p, nt);
    sync(c);
    if (lay->light >= 0)
        for (int i = 0; i < 3; ++i) out[lay->light + i] = c->light[i];
    API_END
}

int cdr_nccl_unique_id(char id_out[128]) {
    NcclApi& api = nccl();
    if (!api.ok) return CDR_ERR_ERROR;
    return api.getUniqueId(id_out) == 0 ? CDR_OK : CDR_ERR_ERROR;
}

int cdr_comm_init(cdr_ctx* c, const char id[128], int32_t n_ranks, int32_t rank) {
    API_BEGIN(c)
    NcclApi& api = nccl();
    if (!api.ok) throw ApiErr(CDR_ERR_ERROR, "NCCL (libnccl.so.2) not loadable");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) throw ApiErr(CDR_ERR_INVALID_ARG, "bad rank");
    NcclUid uid;
    std::memcpy(uid.internal, id, 128);
    void* comm = nullptr;
    auto init = reinterpret_cast<CommInitByValue>(api.commInitRank);
    nccl_check(init(&comm, n_ranks, uid, rank), "ncclCommInitRank");
    c->nccl_comm = comm;
    c->n_ranks = n_ranks;
    c->rank = rank;
    API_END
}

int cdr_comm_info(cdr_ctx* c, int32_t* n_ranks, int32_t* rank) {
    API_BEGIN(c)
    int n = 1, r = 0;
    if (c->nccl_comm) {
        NcclApi& api = nccl();
        if (!api.commCount || !api.commUserRank) throw ApiErr(CDR_ERR_ERROR, "ncclCommCount not available");
        nccl_check(api.commCount(c->nccl_comm, &n), "ncclCommCount");
        nccl_check(api.commUserRank(c->nccl_comm, &r), "ncclCommUserRank");
    }
    if (n_ranks) *n_ranks = n;
    if (rank) *rank = r;
    API_END
}

int cdr_comm_init_all(cdr_ctx** ctxs, int32_t n) {
    if (!ctxs || n < 1) return CDR_ERR_INVALID_ARG;
    for (int i = 0; i < n; ++i)
        if (!ctxs[i]) return CDR_ERR_INVALID_ARG;
    return handle(ctxs[0], [&]() {
        NcclApi& api = nccl();
        if (!api.ok || !api.commInitAll) throw ApiErr(CDR_ERR_ERROR, "NCCL (libnccl.so.2) not loadable");
        std::vector<int> devs(n);
        for (int i = 0; i < n; ++i) {
            devs[i] = ctxs[i]->device;
            for (int j = 0; j < i; ++j)
                if (devs[j] == devs[i])
                    throw ApiErr(CDR_ERR_INVALID_ARG, "one NCCL rank per device: contexts share device " +
                                                          std::to_string(devs[i]));
        }
        std::vector<void*> comms(n, nullptr);
        nccl_check(api.commInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
        for (int i = 0; i < n; ++i) {
            ctxs[i]->nccl_comm = comms[i];
            ctxs[i]->n_ranks = n;
            ctxs[i]->rank = i;
        }
    });
}

int cdr_set_rank(cdr_ctx* c, int32_t rank, int32_t n_ranks) {
    API_BEGIN(c)
    if (c->nccl_comm) throw ApiErr(CDR_ERR_INVALID_ARG, "the context has a communicator: its rank is NCCL's");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) throw ApiErr(CDR_ERR_INVALID_ARG, "bad rank");
    c->rank = rank;
    c->n_ranks = n_ranks;
    API_END
}

}  // extern "C"
