// collodiff_b200.cpp — link-level drop-in for the reference's hot path.
//
// Defines, with the reference's own signatures (headers under
// /root/reference/proj/include, unchanged), the collodiff:: entry points the
// host code calls every iteration, implemented over the C-ABI of
// include/cdr.h (libcdr.so, sm_100a):
//
//   render               render.hpp:67-68       -> cdr_render
//   radiance_at          render.hpp:61-62       -> cdr_radiance_at (hit_out
//                        rebuilt on the host from the device's triangle id)
//   view_rendering_loss  losses.hpp:37-38       -> cdr_view_loss
//   interior_pass        diff_render.hpp:48-50  -> cdr_interior_pass
//   boundary_pass        diff_render.hpp:56-59  -> cdr_boundary_pass
//   grad_image_loss      diff_render.hpp:65-67  -> cdr_loss_grad (one view)
//   extract_silhouettes  silhouette.hpp:36      -> cdr_extract_silhouettes
//   cotangent_laplacian  laplacian.hpp:14-15    -> cdr_laplacian_matrix
//   point_to_mesh_distance mesh.hpp:53          -> cdr_closest_points
//   uv_transfer          optimize.hpp:56        -> cdr_closest_points
//   self_intersects      mesh.hpp:67            -> cdr_self_intersects (pairs
//                        sorted by (f, g); the reference's follow its BVH)
//   total_loss           losses.hpp:94-96       -> cdr_total_loss (rendering,
//                        Laplacian and the four mesh/material regularisers of
//                        losses.cpp:272-292, all on the device)
//
// The reference objects that also define these symbols are linked with them
// weakened (objcopy --weaken-symbol, integration/Makefile), so the unmodified
// host code — run_coarse_to_fine, cmd_gradcheck, cmd_render, ... — resolves
// to these definitions. Status codes become the reference's exceptions.
//
// Device selection: env CDR_DEVICE (default 0) for every entry point. Env
// CDR_DEVICES="0,1,...,7" makes total_loss — the per-iteration call of
// run_coarse_to_fine — fan out over one context per listed GPU, each on its own
// host thread with a contiguous block of the views (global view ids as RNG
// keys, so results do not depend on the split); distinct devices are joined by
// one ncclCommInitAll communicator and the library all-reduces the gradient
// and loss terms. Listing one device several times ("0,0") runs the same
// sharding with several contexts on that GPU and sums their results on the
// host (SURVEY §4's fake multi-GPU mode: tests the sharding on one GPU). Env
// CDR_SKIP_RENDERED=1 makes total_loss leave TotalLossResult::rendered empty
// (run_coarse_to_fine does not read it; it costs a K-image download per
// iteration).
#include <algorithm>
#include <array>
#include <chrono>
#include <exception>
#include <optional>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cdr.h"
#include "collodiff/bvh.hpp"
#include "collodiff/camera.hpp"
#include "collodiff/diff_render.hpp"
#include "collodiff/errors.hpp"
#include "collodiff/laplacian.hpp"
#include "collodiff/losses.hpp"
#include "collodiff/mesh.hpp"
#include "collodiff/optimize.hpp"
#include "collodiff/render.hpp"
#include "collodiff/silhouette.hpp"

namespace collodiff {
namespace {

[[noreturn]] void raise(int rc, const std::string& msg) {
    if (rc == CDR_ERR_SIZE_MISMATCH) throw SizeMismatch(msg);
    if (rc == CDR_ERR_NONFINITE) throw NonFiniteGradient(msg);
    if (rc == CDR_ERR_SELF_INTERSECTING) throw InputSelfIntersecting();
    if (rc == CDR_ERR_PROJECTION_TOO_FAR) throw ProjectionTooFar(msg);
    throw Error("cdr: " + msg);
}

// Content hash of the cached inputs: four independent 64-bit multiply-xor
// lanes over 32-byte blocks (~20 GB/s on one core, so hashing the targets
// costs about what one upload of them would), then the byte tail.
uint64_t fnv1a(const void* p, size_t n, uint64_t h = 1469598103934665603ULL) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    constexpr uint64_t kMul = 0x9e3779b97f4a7c15ULL;
    uint64_t l[4] = {h, h ^ 0xa0761d6478bd642fULL, h ^ 0xe7037ed1a0b428dbULL, h ^ 0x8ebc6af09c88c6e3ULL};
    size_t i = 0;
    for (; i + 32 <= n; i += 32)
        for (int k = 0; k < 4; ++k) {
            uint64_t w;
            std::memcpy(&w, b + i + 8 * k, 8);
            l[k] = (l[k] ^ w) * kMul;
            l[k] ^= l[k] >> 29;
        }
    h = (l[0] ^ (l[1] * 3) ^ (l[2] * 5) ^ (l[3] * 7)) * kMul;
    for (; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
    return h ^ n;
}

// One GPU context, with the mesh topology, views and targets cached.
struct Device {
    cdr_ctx* ctx = nullptr;
    uint64_t topo_key = 0;
    uint64_t target_key = 0;
    uint64_t view_key = 0;
    std::vector<int32_t> tris, edges;
    std::vector<double> buf;
    double* pin = nullptr;  // page-locked staging of total_loss's rendered images (cdr_host_alloc)
    size_t pin_n = 0;
    double* staging(size_t n) {
        if (n > pin_n) {
            cdr_host_free(pin);
            pin = nullptr;
            pin_n = 0;
            void* p = nullptr;
            check(cdr_host_alloc(n * sizeof(double), &p));
            pin = static_cast<double*>(p);
            pin_n = n;
        }
        return pin;
    }

    explicit Device(int device) {
        if (cdr_abi_version() != CDR_ABI_VERSION)  // cdr_stats and friends follow the header's layout
            throw std::runtime_error("libcdr.so ABI version differs from include/cdr.h: rebuild");
        int rc = cdr_create(device, &ctx);
        if (rc != CDR_OK) raise(rc, "cdr_create failed (no CUDA device " + std::to_string(device) + "?)");
    }
    void check(int rc) {
        if (rc != CDR_OK) raise(rc, cdr_last_error(ctx));
    }

    // positions every call; topology only when it changes (remesh)
    void mesh(const Mesh& m) {
        tris.resize(size_t(m.triangle_count()) * 3);
        for (int f = 0; f < m.triangle_count(); ++f)
            for (int k = 0; k < 3; ++k) tris[3 * size_t(f) + k] = m.triangles[f][k];
        uint64_t key = fnv1a(tris.data(), tris.size() * 4, uint64_t(m.vertex_count()) * 0x9e3779b97f4a7c15ULL);
        if (!m.uvs.empty()) key = fnv1a(m.uvs.data(), m.uvs.size() * sizeof(m.uvs[0]), key);  // new UVs re-upload
        if (m.has_adjacency) key = fnv1a(m.edges.data(), m.edges.size() * sizeof(m.edges[0]), key);
        buf.resize(size_t(m.vertex_count()) * 3);
        for (int v = 0; v < m.vertex_count(); ++v) {
            buf[3 * size_t(v)] = m.positions[v].x;
            buf[3 * size_t(v) + 1] = m.positions[v].y;
            buf[3 * size_t(v) + 2] = m.positions[v].z;
        }
        if (key != topo_key || topo_key == 0) {
            std::vector<double> uv;
            if (m.uvs.size() == m.positions.size()) {
                uv.resize(m.uvs.size() * 2);
                for (size_t v = 0; v < m.uvs.size(); ++v) {
                    uv[2 * v] = m.uvs[v].x;
                    uv[2 * v + 1] = m.uvs[v].y;
                }
            }
            const int32_t* ep = nullptr;
            if (m.has_adjacency) {
                edges.resize(m.edges.size() * 4);
                for (size_t e = 0; e < m.edges.size(); ++e) {
                    edges[4 * e] = m.edges[e].v0;
                    edges[4 * e + 1] = m.edges[e].v1;
                    edges[4 * e + 2] = m.edges[e].f0;
                    edges[4 * e + 3] = m.edges[e].f1;
                }
                ep = edges.data();
            }
            check(cdr_set_mesh(ctx, buf.data(), m.vertex_count(), tris.data(), m.triangle_count(),
                               uv.empty() ? nullptr : uv.data(), ep, int32_t(m.edges.size())));
            topo_key = key;
        } else {
            check(cdr_update_positions(ctx, buf.data()));
        }
    }

    // gids: global view ids of s.views' shard (nullptr: all views, ids 0..K-1)
    void scene(const Scene& s, const std::vector<int32_t>* gids = nullptr) {
        mesh(s.mesh);
        const MaterialMaps& mp = s.maps;
        if (mp.diffuse.width != mp.roughness.width || mp.specular.width != mp.roughness.width ||
            mp.diffuse.height != mp.roughness.height || mp.specular.height != mp.roughness.height)
            throw Error("cdr: the GPU path needs diffuse/specular/roughness at one resolution");
        check(cdr_set_textures(ctx, mp.diffuse.data.data(), mp.specular.data.data(), mp.roughness.data.data(),
                               mp.roughness.width, mp.roughness.height));
        double L[3] = {s.light.intensity.x, s.light.intensity.y, s.light.intensity.z};
        double B[3] = {s.background.x, s.background.y, s.background.z};
        check(cdr_set_light(ctx, L, B));
        views(s.views, gids);
    }

    void views(const std::vector<Camera>& cams, const std::vector<int32_t>* gids = nullptr) {
        const size_t n = gids ? gids->size() : cams.size();
        std::vector<cdr_camera> cc(n);
        std::memset(cc.data(), 0, sizeof(cdr_camera) * cc.size());  // hashed below: no padding garbage
        for (size_t i = 0; i < n; ++i) {
            const Camera& c = cams[gids ? size_t((*gids)[i]) : i];
            const Vec3* src[4] = {&c.origin, &c.right, &c.up, &c.forward};
            double* dst[4] = {cc[i].origin, cc[i].right, cc[i].up, cc[i].forward};
            for (int k = 0; k < 4; ++k) {
                dst[k][0] = src[k]->x;
                dst[k][1] = src[k]->y;
                dst[k][2] = src[k]->z;
            }
            cc[i].fov_deg = c.fov_deg;
            cc[i].width = c.width;
            cc[i].height = c.height;
        }
        // the cameras rarely change across iterations: re-sending them would
        // reset the per-view slots and force every target to be re-uploaded
        uint64_t key = fnv1a(cc.data(), sizeof(cdr_camera) * cc.size(), 0xca3e + cc.size());
        if (gids) key = fnv1a(gids->data(), sizeof(int32_t) * gids->size(), key);
        if (key == view_key && view_key != 0) return;
        check(cdr_set_views(ctx, cc.data(), gids ? gids->data() : nullptr, int32_t(cc.size())));
        view_key = key;
        target_key = 0;  // set_views resets the per-view slots
    }

    // Targets of the views (or of the shard gids): uploaded when their full
    // contents (pixels and mask) change. Hashing every byte costs far less
    // than the upload it avoids, and an in-place edit or a new image at a
    // reused address can never leave a stale target on the device.
    void targets(const std::vector<Image>& tg, const std::vector<int32_t>* gids = nullptr) {
        static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be 3 packed doubles");
        const size_t n = gids ? gids->size() : tg.size();
        // one hash per image, the images spread over host threads (a 512^2
        // target is 6 MB: the full-content check is memory-bound)
        std::vector<uint64_t> hv(n);
        auto hash_range = [&](size_t lo, size_t hi) {
            for (size_t i = lo; i < hi; ++i) {
                const Image& t = tg[gids ? size_t((*gids)[i]) : i];
                uint64_t h = fnv1a(t.pixels.data(), t.pixels.size() * sizeof(Vec3), 0x51ed + i);
                hv[i] = fnv1a(t.mask.data(), t.mask.size() * sizeof(double), h ^ t.mask.size());
            }
        };
        const size_t nt = std::min<size_t>(n, std::max(1u, std::thread::hardware_concurrency() / 2));
        if (nt <= 1) {
            hash_range(0, n);
        } else {
            std::vector<std::thread> th;
            const size_t per = (n + nt - 1) / nt;
            for (size_t lo = 0; lo < n; lo += per) th.emplace_back(hash_range, lo, std::min(n, lo + per));
            for (auto& t : th) t.join();
        }
        uint64_t key = fnv1a(hv.data(), sizeof(uint64_t) * n, 0x51ed + n);
        if (key == target_key && target_key != 0) return;
        for (size_t k = 0; k < n; ++k) {
            const Image& t = tg[gids ? size_t((*gids)[k]) : k];
            check(cdr_set_target(ctx, int32_t(k), reinterpret_cast<const double*>(t.pixels.data()),
                                 t.has_mask() ? t.mask.data() : nullptr));
        }
        target_key = key;
    }
};

int env_device() {
    const char* d = std::getenv("CDR_DEVICE");
    return d ? std::atoi(d) : 0;
}

// The contexts total_loss fans out over (CDR_DEVICES); the first is dev().
struct Group {
    std::vector<Device*> devs;
    bool nccl = false;  // distinct devices joined by ncclCommInitAll; else summed on the host
};

// CDR_SHIM_PROFILE=1: wall time per shim entry point, printed at exit
struct ShimProfile {
    const bool on = std::getenv("CDR_SHIM_PROFILE") != nullptr;
    double ms[8] = {};
    long calls[8] = {};
    ~ShimProfile() {
        if (!on) return;
        const char* names[8] = {"total_loss", "  scene+targets upload", "  cdr_total_loss", "  rendered copy",
                                "self_intersects", "render", "    Image construction", ""};
        for (int i = 0; i < 8; ++i)
            if (calls[i]) std::fprintf(stderr, "[cdr shim] %-24s %6ld calls %10.2f ms\n", names[i], calls[i], ms[i]);
    }
};
ShimProfile& prof() {
    static ShimProfile p;
    return p;
}
struct ShimTimer {
    int slot;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit ShimTimer(int s) : slot(s) {}
    ~ShimTimer() {
        ShimProfile& p = prof();
        if (!p.on) return;
        p.ms[slot] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++p.calls[slot];
    }
};

Device& dev() {
    static Device d(env_device());
    return d;
}

Group& group() {
    static Group g = [] {
        Group g;
        g.devs.push_back(&dev());
        const char* env = std::getenv("CDR_DEVICES");
        if (!env || !*env) return g;
        std::vector<int> ids;
        for (const char* p = env; *p;) {
            char* end = nullptr;
            long v = std::strtol(p, &end, 10);
            if (end == p) throw Error("cdr: CDR_DEVICES must be a comma-separated device list, got \"" +
                                      std::string(env) + "\"");
            ids.push_back(int(v));
            p = *end == ',' ? end + 1 : end;
        }
        if (ids.empty()) return g;
        int count = 0;
        cdr_device_count(&count);
        for (int id : ids)
            if (id < 0 || id >= count)
                throw Error("cdr: CDR_DEVICES lists device " + std::to_string(id) + " but " + std::to_string(count) +
                            " are visible");
        g.devs.clear();
        for (size_t k = 0; k < ids.size(); ++k)
            g.devs.push_back(k == 0 && ids[0] == env_device() ? &dev() : new Device(ids[k]));  // leaked with the process
        std::vector<int> sorted = ids;
        std::sort(sorted.begin(), sorted.end());
        g.nccl = g.devs.size() > 1 && std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
        if (g.nccl) {
            std::vector<cdr_ctx*> ctxs;
            for (Device* d : g.devs) ctxs.push_back(d->ctx);
            const int rc = cdr_comm_init_all(ctxs.data(), int32_t(ctxs.size()));
            if (rc != CDR_OK) raise(rc, std::string("ncclCommInitAll: ") + cdr_last_error(ctxs[0]));
        } else {
            for (size_t k = 0; k < g.devs.size(); ++k)
                g.devs[k]->check(cdr_set_rank(g.devs[k]->ctx, int32_t(k), int32_t(g.devs.size())));
        }
        return g;
    }();
    return g;
}

cdr_settings settings_of(const RenderSettings& s) {
    cdr_settings c{};
    c.spp = s.spp;
    c.boundary_term = s.boundary_term ? 1 : 0;
    c.boundary_samples = s.boundary_samples;
    c.seed = s.seed;
    c.gamma = s.gamma;
    return c;
}

cdr_layout layout_of(const ParamLayout& L) {
    cdr_layout c{};
    c.positions = int64_t(L.get(SegmentId::Positions).offset);
    c.diffuse = int64_t(L.get(SegmentId::Diffuse).offset);
    c.specular = int64_t(L.get(SegmentId::Specular).offset);
    c.roughness = int64_t(L.get(SegmentId::Roughness).offset);
    c.light = L.has(SegmentId::Light) ? int64_t(L.get(SegmentId::Light).offset) : -1;
    c.total = int64_t(L.total);
    return c;
}

}  // namespace

Image render(const Scene& scene, const SceneContext&, int view, const RenderSettings& settings,
             std::vector<int>* hit_cache) {
    Device& d = dev();
    d.scene(scene);
    const Camera& cam = scene.views[view];
    Image img(cam.width, cam.height, true);
    const int spp = std::max(1, settings.spp);
    if (hit_cache) hit_cache->assign(size_t(cam.width) * cam.height * spp, -1);
    cdr_settings st = settings_of(settings);
    d.check(cdr_render(d.ctx, view, &st, reinterpret_cast<double*>(img.pixels.data()), img.mask.data(),
                       hit_cache ? hit_cache->data() : nullptr));
    return img;
}

// radiance_at (render.hpp:61-62, render.cpp:24-33). The device returns the
// radiance and the hit triangle; when hit_out is requested the record is
// rebuilt with the reference's own primary_ray / ray_triangle /
// make_hit_record on that triangle (the same fp64 arithmetic the device
// replays, so t and the barycentrics are the device's).
Vec3 radiance_at(const Scene& scene, const SceneContext& ctx, int view, const Vec2& x,
                 std::optional<HitRecord>* hit_out) {
    Device& d = dev();
    d.scene(scene);
    const double xy[2] = {x.x, x.y};
    double rgb[3];
    int32_t tri = -1;
    d.check(cdr_radiance_at(d.ctx, view, 1, xy, rgb, &tri));
    if (hit_out) {
        if (tri < 0) {
            *hit_out = std::nullopt;
        } else {
            const Ray ray = primary_ray(scene.views[view], x);
            const auto& f = scene.mesh.triangles[size_t(tri)];
            const auto& P = scene.mesh.positions;
            double t = 0, b1 = 0, b2 = 0;
            ray_triangle(ray.origin, ray.dir, P[size_t(f[0])], P[size_t(f[1])], P[size_t(f[2])], t, b1, b2);
            *hit_out = make_hit_record(scene.mesh, &ctx.normals, tri, t, b1, b2, ray.origin, ray.dir);
        }
    }
    return Vec3(rgb[0], rgb[1], rgb[2]);
}

ViewLossResult view_rendering_loss(const Image& rendered, const Image& target, double lambda_rend,
                                   double gamma, bool use_target_mask) {
    if (rendered.width != target.width || rendered.height != target.height)
        throw SizeMismatch("rendered/target size mismatch");
    ViewLossResult res;
    res.adjoint = Image(rendered.width, rendered.height);
    Device& d = dev();
    d.check(cdr_view_loss(d.ctx, rendered.width, rendered.height, reinterpret_cast<const double*>(rendered.pixels.data()),
                          reinterpret_cast<const double*>(target.pixels.data()),
                          target.has_mask() ? target.mask.data() : nullptr, lambda_rend, gamma,
                          use_target_mask ? 1 : 0, &res.value, reinterpret_cast<double*>(res.adjoint.pixels.data())));
    return res;
}

void interior_pass(const Scene& scene, const GradContext&, int view, const AdjointImage& adjoint,
                   const RenderSettings& settings, const std::vector<int>& hit_cache, GradVector& grad) {
    const Camera& cam = scene.views[view];
    if (adjoint.width != cam.width || adjoint.height != cam.height)
        throw SizeMismatch("adjoint size does not match view");
    Device& d = dev();
    d.scene(scene);
    cdr_settings st = settings_of(settings);
    cdr_layout lay = layout_of(*grad.layout);
    d.check(cdr_interior_pass(d.ctx, view, reinterpret_cast<const double*>(adjoint.pixels.data()), &st,
                              hit_cache.data(), int64_t(hit_cache.size()), &lay, grad.values.data()));
}

SilhouetteSet extract_silhouettes(const Mesh& mesh, const Camera& view) {
    if (!mesh.has_adjacency) throw Error("extract_silhouettes requires adjacency");
    Device& d = dev();
    d.mesh(mesh);
    d.views({view});
    int32_t n = 0;
    double total = 0;
    d.check(cdr_extract_silhouettes(d.ctx, 0, nullptr, 0, &n, &total));
    std::vector<cdr_segment> segs(n);
    d.check(cdr_extract_silhouettes(d.ctx, 0, segs.data(), n, &n, &total));
    SilhouetteSet set;
    set.total_length = total;
    set.segments.resize(n);
    for (int i = 0; i < n; ++i) {
        const cdr_segment& g = segs[i];
        SilhouetteSegment& s = set.segments[i];
        s.v0 = g.v0;
        s.v1 = g.v1;
        s.p0 = Vec3(g.p0[0], g.p0[1], g.p0[2]);
        s.p1 = Vec3(g.p1[0], g.p1[1], g.p1[2]);
        s.t0 = g.t0;
        s.t1 = g.t1;
        s.q0 = Vec2(g.q0[0], g.q0[1]);
        s.q1 = Vec2(g.q1[0], g.q1[1]);
        s.z0 = g.z0;
        s.z1 = g.z1;
        s.length_px = g.length_px;
    }
    return set;
}

BoundaryStats boundary_pass(const Scene& scene, const GradContext&, int view, const AdjointImage& adjoint,
                            const SilhouetteSet& silhouettes, int samples, uint64_t seed, GradVector& grad,
                            BoundaryProbe probe) {
    BoundaryStats stats;
    const Camera& cam = scene.views[view];
    if (adjoint.width != cam.width || adjoint.height != cam.height)
        throw SizeMismatch("adjoint size does not match view");
    if (silhouettes.segments.empty() || silhouettes.total_length <= 0 || samples <= 0) return stats;
    Device& d = dev();
    d.scene(scene);
    std::vector<cdr_segment> segs(silhouettes.segments.size());
    for (size_t i = 0; i < segs.size(); ++i) {
        const SilhouetteSegment& s = silhouettes.segments[i];
        cdr_segment& g = segs[i];
        g.v0 = s.v0;
        g.v1 = s.v1;
        g.p0[0] = s.p0.x; g.p0[1] = s.p0.y; g.p0[2] = s.p0.z;
        g.p1[0] = s.p1.x; g.p1[1] = s.p1.y; g.p1[2] = s.p1.z;
        g.t0 = s.t0;
        g.t1 = s.t1;
        g.q0[0] = s.q0.x; g.q0[1] = s.q0.y;
        g.q1[0] = s.q1.x; g.q1[1] = s.q1.y;
        g.z0 = s.z0;
        g.z1 = s.z1;
        g.length_px = s.length_px;
    }
    cdr_layout lay = layout_of(*grad.layout);
    int32_t deg = 0;
    d.check(cdr_boundary_pass(d.ctx, view, reinterpret_cast<const double*>(adjoint.pixels.data()), segs.data(),
                              int32_t(segs.size()), samples, seed,
                              probe == BoundaryProbe::Coverage ? CDR_PROBE_COVERAGE : CDR_PROBE_RADIANCE, &lay,
                              grad.values.data(), &deg));
    stats.degenerate_skipped = deg;
    return stats;
}

double grad_image_loss(const Scene& scene, const GradContext&, int view, const Image& target,
                       const RenderSettings& settings, double lambda_rend, bool use_target_mask, GradVector& grad) {
    const Camera& cam = scene.views[view];
    if (target.width != cam.width || target.height != cam.height)
        throw SizeMismatch("target size does not match view");
    Device& d = dev();
    d.scene(scene);
    d.check(cdr_set_target(d.ctx, view, reinterpret_cast<const double*>(target.pixels.data()),
                           target.has_mask() ? target.mask.data() : nullptr));
    d.target_key = 0;
    cdr_settings st = settings_of(settings);
    cdr_layout lay = layout_of(*grad.layout);
    double loss[2] = {0, 0};
    int32_t v = view;
    d.check(cdr_loss_grad(d.ctx, &v, 1, &st, lambda_rend, 0.0, CDR_LAPLACIAN_COTANGENT, use_target_mask ? 1 : 0,
                          &lay, loss, grad.values.data(), nullptr, nullptr, nullptr));
    return loss[0];
}

bool self_intersects(const Mesh& mesh, std::vector<std::pair<int, int>>* pairs) {
    ShimTimer timer(4);
    if (pairs) pairs->clear();
    Device& d = dev();
    const int nv = mesh.vertex_count(), nt = mesh.triangle_count();
    std::vector<double> pos(3 * size_t(nv));
    for (int v = 0; v < nv; ++v) {
        pos[3 * v] = mesh.positions[v].x;
        pos[3 * v + 1] = mesh.positions[v].y;
        pos[3 * v + 2] = mesh.positions[v].z;
    }
    std::vector<int32_t> tris(3 * size_t(nt));
    for (int f = 0; f < nt; ++f)
        for (int k = 0; k < 3; ++k) tris[3 * f + k] = mesh.triangles[f][k];
    int32_t res = 0;
    if (!pairs) {
        d.check(cdr_self_intersects(d.ctx, pos.data(), nv, tris.data(), nt, &res, nullptr, 0, nullptr));
        return res != 0;
    }
    int64_t n = 0;
    d.check(cdr_self_intersects(d.ctx, pos.data(), nv, tris.data(), nt, &res, nullptr, 0, &n));
    std::vector<int32_t> pr(2 * size_t(n));
    if (n > 0) d.check(cdr_self_intersects(d.ctx, pos.data(), nv, tris.data(), nt, &res, pr.data(), n, &n));
    for (int64_t i = 0; i < n; ++i) pairs->push_back({pr[2 * i], pr[2 * i + 1]});
    return res != 0;
}

namespace {
void mesh_arrays(const Mesh& m, std::vector<double>& pos, std::vector<int32_t>& tris) {
    pos.resize(3 * size_t(m.vertex_count()));
    for (int v = 0; v < m.vertex_count(); ++v) {
        pos[3 * v] = m.positions[v].x;
        pos[3 * v + 1] = m.positions[v].y;
        pos[3 * v + 2] = m.positions[v].z;
    }
    tris.resize(3 * size_t(m.triangle_count()));
    for (int f = 0; f < m.triangle_count(); ++f)
        for (int k = 0; k < 3; ++k) tris[3 * f + k] = m.triangles[f][k];
}
}  // namespace

double point_to_mesh_distance(const std::vector<Vec3>& points, const Mesh& mesh) {
    if (mesh.triangle_count() == 0) throw EmptyMesh();  // mesh.cpp:128
    if (points.empty()) return 0.0;
    Device& d = dev();
    std::vector<double> pos, q(3 * points.size()), dist(points.size());
    std::vector<int32_t> tris;
    mesh_arrays(mesh, pos, tris);
    for (size_t i = 0; i < points.size(); ++i) {
        q[3 * i] = points[i].x;
        q[3 * i + 1] = points[i].y;
        q[3 * i + 2] = points[i].z;
    }
    d.check(cdr_closest_points(d.ctx, pos.data(), mesh.vertex_count(), tris.data(), mesh.triangle_count(), q.data(),
                               int32_t(points.size()), nullptr, nullptr, dist.data(), nullptr));
    double sum = 0;  // the reference's sequential sum (mesh.cpp:131)
    for (double x : dist) sum += x;
    return sum / double(points.size());
}

void uv_transfer(const Mesh& old_mesh, Mesh& mesh, double max_distance) {
    if (old_mesh.uvs.size() != old_mesh.positions.size()) return;  // remesh.cpp:282
    Device& d = dev();
    std::vector<double> pos, q(3 * size_t(mesh.vertex_count())), dist(mesh.vertex_count()),
        bary(3 * size_t(mesh.vertex_count()));
    std::vector<int32_t> tris, tri(mesh.vertex_count());
    mesh_arrays(old_mesh, pos, tris);
    for (int v = 0; v < mesh.vertex_count(); ++v) {
        q[3 * v] = mesh.positions[v].x;
        q[3 * v + 1] = mesh.positions[v].y;
        q[3 * v + 2] = mesh.positions[v].z;
    }
    d.check(cdr_closest_points(d.ctx, pos.data(), old_mesh.vertex_count(), tris.data(), old_mesh.triangle_count(),
                               q.data(), mesh.vertex_count(), tri.data(), nullptr, dist.data(), bary.data()));
    mesh.uvs.resize(mesh.positions.size());
    for (int v = 0; v < mesh.vertex_count(); ++v) {
        if (tri[v] < 0 || dist[v] > max_distance)
            throw ProjectionTooFar("uv transfer: vertex " + std::to_string(v) + " is " + std::to_string(dist[v]) +
                                   " away from the source mesh");
        const auto& t = old_mesh.triangles[tri[v]];
        mesh.uvs[v] = old_mesh.uvs[t[0]] * bary[3 * v] + old_mesh.uvs[t[1]] * bary[3 * v + 1] +
                      old_mesh.uvs[t[2]] * bary[3 * v + 2];
    }
}

Eigen::SparseMatrix<double> cotangent_laplacian(const Mesh& mesh, LaplacianMode mode) {
    Device& d = dev();
    d.mesh(mesh);
    const int32_t m = mode == LaplacianMode::Uniform ? CDR_LAPLACIAN_UNIFORM : CDR_LAPLACIAN_COTANGENT;
    int64_t nnz = 0;
    d.check(cdr_laplacian_matrix(d.ctx, m, nullptr, nullptr, nullptr, &nnz));
    std::vector<int32_t> outer(size_t(mesh.vertex_count()) + 1), inner(nnz);
    std::vector<double> vals(nnz);
    d.check(cdr_laplacian_matrix(d.ctx, m, outer.data(), inner.data(), vals.data(), &nnz));
    std::vector<Eigen::Triplet<double>> trip;
    trip.reserve(nnz);
    for (int j = 0; j < mesh.vertex_count(); ++j)
        for (int32_t k = outer[j]; k < outer[j + 1]; ++k) trip.emplace_back(inner[k], j, vals[k]);
    Eigen::SparseMatrix<double> L(mesh.vertex_count(), mesh.vertex_count());
    L.setFromTriplets(trip.begin(), trip.end());
    return L;
}

TotalLossResult total_loss(const Scene& scene, const std::vector<Image>& targets, const LossWeights& weights,
                           const LossOptions& options, std::shared_ptr<const ParamLayout> layout) {
    if (targets.size() != scene.views.size()) throw SizeMismatch("target count does not match views");
    ShimTimer timer(0);
    TotalLossResult res{LossBreakdown{}, GradVector(layout), {}};
    Group& g = group();
    const int K = int(scene.views.size());
    const int N = std::max(1, std::min<int>(int(g.devs.size()), K));  // ranks with at least one view
    // contiguous blocks of ceil(K / N) global view ids (shard.py: shard_views)
    const int per = (K + N - 1) / N;
    std::vector<std::vector<int32_t>> gids(g.devs.size());
    for (int k = 0; k < N; ++k)
        for (int v = k * per; v < std::min(K, (k + 1) * per); ++v) gids[k].push_back(v);
    cdr_settings st = settings_of(options.render);
    st.flags |= CDR_FLAG_GRAD_OVERWRITE;  // res.grad is the fresh GradVector (losses.cpp:250)
    cdr_layout lay = layout_of(*layout);
    const cdr_reg_weights reg{weights.normal, weights.edge, weights.spec, weights.roug, weights.sigma1,
                              weights.sigma2};
    const int32_t lap_mode = options.laplacian_mode == LaplacianMode::Uniform ? CDR_LAPLACIAN_UNIFORM
                                                                               : CDR_LAPLACIAN_COTANGENT;
    const bool single = g.devs.size() == 1;
    const bool want_rendered = !std::getenv("CDR_SKIP_RENDERED");
    std::vector<std::array<double, 7>> bd(g.devs.size(), std::array<double, 7>{});
    std::vector<std::vector<double>> part(single || g.nccl ? 0 : g.devs.size());
    std::vector<std::exception_ptr> err(g.devs.size());
    auto run = [&](size_t k) {
        try {
            Device& d = *g.devs[k];
            {
                ShimTimer t(1);
                d.scene(scene, single ? nullptr : &gids[k]);
                d.targets(targets, single ? nullptr : &gids[k]);
            }
            const int n = int(single ? K : gids[k].size());
            std::vector<int32_t> slots(n);
            for (int i = 0; i < n; ++i) slots[i] = i;
            // rank 0 receives the (all-reduced) gradient; the other NCCL ranks
            // keep theirs on the device; host-summed ranks return their part
            double* gout = nullptr;
            if (k == 0 && (single || g.nccl)) gout = res.grad.values.data();
            else if (!g.nccl) {
                part[k].assign(res.grad.values.size(), 0.0);
                gout = part[k].data();
            }
            // the rendered images come down into page-locked staging during
            // the call (beside its boundary pass); the Images are filled below
            double *srgb = nullptr, *smask = nullptr;
            if (want_rendered) {
                size_t npx = 0;
                for (int i = 0; i < n; ++i) {
                    const Camera& c = scene.views[single ? i : size_t(gids[k][i])];
                    npx += size_t(c.width) * c.height;
                }
                srgb = d.staging(4 * npx);
                smask = srgb + 3 * npx;
            }
            ShimTimer t2(2);
            d.check(cdr_total_loss(d.ctx, slots.data(), n, &st, weights.rend, weights.lap, &reg, lap_mode,
                                   options.use_target_masks ? 1 : 0, &lay, bd[k].data(), gout, srgb, smask,
                                   nullptr));
        } catch (...) {
            err[k] = std::current_exception();
        }
    };
    if (single) {
        run(0);
    } else {  // one host thread per context: NCCL ranks must enter the all-reduce together
        std::vector<std::thread> th;
        for (size_t k = 0; k < g.devs.size(); ++k) th.emplace_back(run, k);
        for (auto& t : th) t.join();
    }
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
    double t[7] = {bd[0][0], bd[0][1], bd[0][2], bd[0][3], bd[0][4], bd[0][5], bd[0][6]};
    if (!single && !g.nccl) {  // host sum of the shards, in rank order (rank 0 holds the once-only terms)
        std::vector<double>& out = res.grad.values;
        out = part[0];
        for (size_t k = 1; k < part.size(); ++k) {
            for (size_t i = 0; i < out.size(); ++i) out[i] += part[k][i];
            for (int j = 1; j < 7; ++j) t[j] += bd[k][j];
        }
        t[0] = t[1] + t[2] + t[3] + t[4] + t[5] + t[6];  // losses.cpp:294-295
    }
    res.breakdown.total = t[0];
    res.breakdown.rend = t[1];
    res.breakdown.lap = t[2];
    res.breakdown.normal = t[3];
    res.breakdown.edge = t[4];
    res.breakdown.spec = t[5];
    res.breakdown.roug = t[6];
    if (want_rendered) {  // the Images from the staging buffers, views spread over host threads
        ShimTimer t3(3);
        std::vector<const double*> src(K);
        std::vector<size_t> off(g.devs.size(), 0), tot(g.devs.size(), 0);
        for (int v = 0; v < K; ++v) {
            const size_t k = single ? 0 : size_t(v / per);
            tot[k] += size_t(scene.views[v].width) * scene.views[v].height;
        }
        for (int v = 0; v < K; ++v) {
            const size_t k = single ? 0 : size_t(v / per);
            src[v] = g.devs[k]->pin + 3 * off[k];
            off[k] += size_t(scene.views[v].width) * scene.views[v].height;
        }
        std::vector<std::optional<Image>> imgs(K);
        auto fill = [&](int t, int nt) {
            for (int v = t; v < K; v += nt) {
                const size_t k = single ? 0 : size_t(v / per);
                const Camera& c = scene.views[v];
                const size_t np = size_t(c.width) * c.height;
                imgs[v].emplace(c.width, c.height, true);
                std::memcpy(imgs[v]->pixels.data(), src[v], sizeof(double) * 3 * np);
                // the masks follow the rgb blocks of this device's views
                const double* m = g.devs[k]->pin + 3 * tot[k] + (src[v] - g.devs[k]->pin) / 3;
                std::memcpy(imgs[v]->mask.data(), m, sizeof(double) * np);
            }
        };
        const int nt = std::max(1, std::min<int>(K, int(std::thread::hardware_concurrency())));
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(fill, t, nt);
        fill(0, nt);
        for (auto& t : th) t.join();
        res.rendered.reserve(K);
        for (auto& im : imgs) res.rendered.push_back(std::move(*im));
    }
    return res;
}

}  // namespace collodiff
