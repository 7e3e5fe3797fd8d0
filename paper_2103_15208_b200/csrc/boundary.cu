// boundary.cu — the silhouette-edge boundary term.
//
//   k_sil_flag / k_sil_scan / k_sil_write : extract_silhouettes
//       (silhouette.cpp:55-106) for all views of the call at once, with an
//       order-preserving compaction so segments keep the reference's edge order
//       (mesh.edges order, mesh.cpp:40-61). All predicate and clipping math is
//       the reference's, unfused, so the segment set is bit-identical.
//   k_cdf  : the running fp64 length sum (diff_render.cpp:213-228), sequential
//       per view so the CDF — and therefore every sample's segment pick — is
//       bit-identical too.
//   k_boundary : one thread per edge sample (diff_render.cpp:230-278): RNG pick,
//       lower_bound, adjoint lookup, two radiance probes, n.dx'/dp deposit to
//       the two edge vertices (warp-aggregated by segment).
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kBlock = 256;

struct SilCall {
    int slot;
    int samples;  // M of boundary_pass for this view
};

__device__ __forceinline__ int sign_of(double v) { return (v > 0) - (v < 0); }

// Liang-Barsky clip of q0 + s (q1 - q0) to [0,w] x [0,h] (silhouette.cpp:14-35)
__device__ __forceinline__ bool clip_to_rect(D2 q0, D2 q1, double w, double h, double& s0,
                                             double& s1) {
    s0 = 0;
    s1 = 1;
    D2 d{q1.x - q0.x, q1.y - q0.y};
    const double pp[4] = {-d.x, d.x, -d.y, d.y};
    const double qq[4] = {q0.x - 0.0, w - q0.x, q0.y - 0.0, h - q0.y};
    for (int i = 0; i < 4; ++i) {
        if (fabs(pp[i]) < 1e-300) {
            if (qq[i] < 0) return false;
            continue;
        }
        double r = qq[i] / pp[i];
        if (pp[i] < 0) {
            if (r > s1) return false;
            if (r > s0) s0 = r;
        } else {
            if (r < s0) return false;
            if (r < s1) s1 = r;
        }
    }
    return s1 > s0;
}

// is_silhouette_edge + near clip + project + rect clip (silhouette.cpp:39-104)
__device__ __forceinline__ bool make_segment(const double* __restrict__ pos,
                                             const double* __restrict__ fn, int4 e,
                                             const DevCamera& cam, cdr_segment* out) {
    D3 a = ld3(pos + 3 * e.x), b = ld3(pos + 3 * e.y);
    D3 org{cam.o[0], cam.o[1], cam.o[2]}, fw{cam.f[0], cam.f[1], cam.f[2]};
    if (e.w >= 0) {
        D3 mid = (a + b) * 0.5;
        D3 d = mid - org;
        double sa = dot(ld3(fn + 3 * e.z), d);
        double sb = dot(ld3(fn + 3 * e.w), d);
        if (sign_of(sa) == sign_of(sb)) return false;
    }
    const double znear = 1e-6;
    double za = dot(a - org, fw), zb = dot(b - org, fw);
    if (za <= znear && zb <= znear) return false;
    double t0 = 0, t1 = 1;
    if (za <= znear) t0 = (znear - za) / (zb - za);
    if (zb <= znear) t1 = (znear - za) / (zb - za);
    D3 pa = a + (b - a) * t0;
    D3 pb = a + (b - a) * t1;
    double z0, z1;
    D2 qa, qb;
    if (!project(cam, pa, &qa, &z0)) return false;
    if (!project(cam, pb, &qb, &z1)) return false;
    double s0, s1;
    if (!clip_to_rect(qa, qb, double(cam.W), double(cam.H), s0, s1)) return false;
    D2 q0{qa.x + (qb.x - qa.x) * s0, qa.y + (qb.y - qa.y) * s0};
    D2 q1{qa.x + (qb.x - qa.x) * s1, qa.y + (qb.y - qa.y) * s1};
    double lx = q1.x - q0.x, ly = q1.y - q0.y;
    double len = sqrt(lx * lx + ly * ly);
    if (len <= 0) return false;
    if (out) {
        double u0 = ((1 - s0) / z0 * t0 + s0 / z1 * t1) / ((1 - s0) / z0 + s0 / z1);
        double u1 = ((1 - s1) / z0 * t0 + s1 / z1 * t1) / ((1 - s1) / z0 + s1 / z1);
        cdr_segment g;
        g.v0 = e.x;
        g.v1 = e.y;
        g.p0[0] = a.x; g.p0[1] = a.y; g.p0[2] = a.z;
        g.p1[0] = b.x; g.p1[1] = b.y; g.p1[2] = b.z;
        g.q0[0] = q0.x; g.q0[1] = q0.y;
        g.q1[0] = q1.x; g.q1[1] = q1.y;
        g.length_px = len;
        g.z0 = dot((a + (b - a) * u0) - org, fw);
        g.z1 = dot((a + (b - a) * u1) - org, fw);
        g.t0 = u0;
        g.t1 = u1;
        *out = g;
    }
    return true;
}

__global__ void k_sil_flag(const double* __restrict__ pos, const double* __restrict__ fn,
                           const int4* __restrict__ edges, int E, const DevCamera* __restrict__ cams,
                           const SilCall* __restrict__ calls, unsigned char* __restrict__ flags,
                           int32_t* __restrict__ block_count, int nb) {
    const int vi = blockIdx.y;
    const DevCamera& cam = cams[calls[vi].slot];
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool f = false;
    if (i < E) f = make_segment(pos, fn, edges[i], cam, nullptr);
    if (i < E) flags[size_t(vi) * E + i] = f;
    int cnt = __syncthreads_count(f);
    if (threadIdx.x == 0) block_count[size_t(vi) * nb + blockIdx.x] = cnt;
}

// exclusive scan of the per-block counts of one view (one CTA per view)
__global__ void k_sil_scan(const int32_t* __restrict__ block_count, int nb,
                           int32_t* __restrict__ block_off, int32_t* __restrict__ count) {
    const int vi = blockIdx.x;
    __shared__ int32_t s[1024];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        int i = base + threadIdx.x;
        int v = i < nb ? block_count[size_t(vi) * nb + i] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < nb) block_off[size_t(vi) * nb + i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) count[vi] = carry;
}

__global__ void k_sil_write(const double* __restrict__ pos, const double* __restrict__ fn,
                            const int4* __restrict__ edges, int E, const DevCamera* __restrict__ cams,
                            const SilCall* __restrict__ calls, const unsigned char* __restrict__ flags,
                            const int32_t* __restrict__ block_off, int nb,
                            cdr_segment* __restrict__ segs) {
    const int vi = blockIdx.y;
    const DevCamera& cam = cams[calls[vi].slot];
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool f = i < E && flags[size_t(vi) * E + i];
    unsigned bal = __ballot_sync(0xffffffffu, f);
    __shared__ int warp_tot[kBlock / 32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int off = block_off[size_t(vi) * nb + blockIdx.x];
    for (int k = 0; k < w; ++k) off += warp_tot[k];
    off += __popc(bal & ((1u << lane) - 1u));
    if (f) make_segment(pos, fn, edges[i], cam, &segs[size_t(vi) * E + off]);
}

// Running CDF in segment order, one thread per view (diff_render.cpp:213-228).
// info[vi] = {total_len (acc), extract_total, usable, degenerate}
__global__ void k_cdf(const cdr_segment* __restrict__ segs, const int32_t* __restrict__ count, int E,
                      int n_views, double* __restrict__ cdf, double* __restrict__ totals,
                      int32_t* __restrict__ degenerate) {
    int vi = blockIdx.x * blockDim.x + threadIdx.x;
    if (vi >= n_views) return;
    int n = count[vi];
    double acc = 0, ext = 0;
    int usable = 0, deg = 0;
    for (int i = 0; i < n; ++i) {
        double len = segs[size_t(vi) * E + i].length_px;
        ext += len;  // SilhouetteSet::total_length (silhouette.cpp:103)
        if (len < 1e-12) {
            ++deg;
            len = 0;
        } else {
            ++usable;
        }
        acc += len;
        cdf[size_t(vi) * E + i] = acc;
    }
    totals[3 * vi] = acc;
    totals[3 * vi + 1] = (n == 0 || ext <= 0 || usable == 0 || acc <= 0) ? 0.0 : 1.0;
    totals[3 * vi + 2] = ext;
    degenerate[vi] = (n == 0 || ext <= 0) ? 0 : deg;
}

struct BParams {
    ShadeScene sc;
    const SceneInfo* info;
    const DevCamera* cams;
    const SilCall* calls;
    const size_t* pix_off;
    const cdr_segment* segs;
    const double* cdf;
    const double* totals;
    const int32_t* count;
    int E;
    uint64_t seed;
    int probe;
    const double* adj;
    double* grad;
    int64_t lay_pos;
    ErrorInfo* err;
    Counters* counters;
};

__global__ void __launch_bounds__(kBlock) k_boundary(BParams p) {
    const int vi = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const DevCamera& cam = p.cams[p.calls[vi].slot];
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int nseg = p.count[vi];
    const int samples = p.calls[vi].samples;
    const bool enabled = p.totals[3 * vi + 1] != 0.0;
    const double total_len = p.totals[3 * vi];
    bool act = enabled && i < samples;
    int si = 0;
    double s = 0;
    D2 xq{0, 0}, n2{0, 0};
    D3 adj{0, 0, 0};
    const cdr_segment* sg = nullptr;
    if (act) {
        Rng rng = rng2(p.seed, uint64_t(cam.gid) + 0xb0d1, uint64_t(i));
        double pick = rng.next_double() * total_len;
        const double* cdf = p.cdf + size_t(vi) * p.E;
        int lo = 0, hi = nseg;  // std::lower_bound
        while (lo < hi) {
            int mid = lo + ((hi - lo) >> 1);
            if (cdf[mid] < pick) lo = mid + 1;
            else hi = mid;
        }
        si = lo < nseg - 1 ? lo : nseg - 1;
        sg = p.segs + size_t(vi) * p.E + si;
        if (sg->length_px < 1e-12) act = false;
        if (act) {
            s = rng.next_double();
            xq = D2{sg->q0[0] + (sg->q1[0] - sg->q0[0]) * s, sg->q0[1] + (sg->q1[1] - sg->q0[1]) * s};
            int px = int(floor(xq.x)), py = int(floor(xq.y));
            px = px < 0 ? 0 : (px > cam.W - 1 ? cam.W - 1 : px);
            py = py < 0 ? 0 : (py > cam.H - 1 ? cam.H - 1 : py);
            adj = ld3(p.adj + 3 * (p.pix_off[p.calls[vi].slot] + size_t(py) * cam.W + px));
            if (adj.x == 0 && adj.y == 0 && adj.z == 0) act = false;
        }
    }
    double weighted = 0;
    if (act) {
        D2 tg{(sg->q1[0] - sg->q0[0]) / sg->length_px, (sg->q1[1] - sg->q0[1]) / sg->length_px};
        n2 = D2{-tg.y, tg.x};
        D2 xm{xq.x - n2.x * 0.5, xq.y - n2.y * 0.5}, xp{xq.x + n2.x * 0.5, xq.y + n2.y * 0.5};
        const double t_min = p.info->t_min;
        D3 delta;
        if (p.probe == CDR_PROBE_RADIANCE) {
            D3 lo3 = radiance_at(p.sc, cam, xm, t_min, nullptr);
            D3 hi3 = radiance_at(p.sc, cam, xp, t_min, nullptr);
            delta = lo3 - hi3;
        } else {
            D3 org{cam.o[0], cam.o[1], cam.o[2]};
            double cm = trace(p.sc.nodes, p.sc.recs, p.sc.n_tris, org, primary_dir(cam, xm), t_min).tri >= 0 ? 1.0 : 0.0;
            double cp = trace(p.sc.nodes, p.sc.recs, p.sc.n_tris, org, primary_dir(cam, xp), t_min).tri >= 0 ? 1.0 : 0.0;
            delta = D3{cm - cp, cm - cp, cm - cp};
        }
        weighted = dot(adj, delta);
        if (weighted == 0) act = false;
        else if (!isfinite(weighted)) {
            if (atomicCAS(&p.err->flag, 0, 2) == 0) p.err->segment = si;
            act = false;
        }
    }
    {
        int na = __syncthreads_count(act);
        if (threadIdx.x == 0 && na) atomicAdd(&p.counters->boundary_active, (unsigned long long)na);
    }
    double v[6] = {0, 0, 0, 0, 0, 0};
    if (act) {
        double w0 = (1.0 - s) / sg->z0, w1 = s / sg->z1;
        double t3 = (w0 * sg->t0 + w1 * sg->t1) / (w0 + w1);  // segment_param_2d_to_3d
        D3 p0{sg->p0[0], sg->p0[1], sg->p0[2]}, p1{sg->p1[0], sg->p1[1], sg->p1[2]};
        D3 point = p0 + (p1 - p0) * t3;
        D3 jx, jy;
        projection_jacobian(cam, point, &jx, &jy);
        D3 nj = jx * n2.x + jy * n2.y;
        double scale = weighted * total_len / double(samples);
        D3 g0 = nj * (scale * (1.0 - t3)), g1 = nj * (scale * t3);
        v[0] = g0.x; v[1] = g0.y; v[2] = g0.z;
        v[3] = g1.x; v[4] = g1.y; v[5] = g1.z;
    }
    const int key = act ? si : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    reduce_peers<6>(0xffffffffu, peers, v);
    if (act && (__ffs(peers) - 1) == lane) {
        double* g = p.grad + p.lay_pos;
        for (int c = 0; c < 3; ++c) {
            if (v[c] != 0) atomicAdd(g + 3 * int64_t(sg->v0) + c, v[c]);
            if (v[3 + c] != 0) atomicAdd(g + 3 * int64_t(sg->v1) + c, v[3 + c]);
        }
    }
}

struct BStatics {
    DBuf<SilCall> calls;
    DBuf<size_t> pix_off;
    int n_calls = 0;
};

BStatics& bstatics(cdr_ctx* c) {
    static thread_local std::vector<std::pair<cdr_ctx*, BStatics*>> reg;
    for (auto& e : reg)
        if (e.first == c) return *e.second;
    reg.push_back({c, new BStatics()});
    return *reg.back().second;
}

}  // namespace

void set_view_calls(cdr_ctx* c, const int* view_slots, const int* samples, int n_views) {
    BStatics& st = bstatics(c);
    std::vector<SilCall> calls(n_views);
    for (int i = 0; i < n_views; ++i) calls[i] = SilCall{view_slots[i], samples ? samples[i] : 0};
    st.calls.ensure(std::max(1, n_views));
    st.n_calls = n_views;
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.calls.p, calls.data(), sizeof(SilCall) * n_views,
                                   cudaMemcpyHostToDevice, c->stream));
    const int E = std::max(1, c->E);
    c->segs.ensure(size_t(std::max(1, n_views)) * E);
    c->cdf.ensure(size_t(std::max(1, n_views)) * E);
    c->sil_count.ensure(std::max(1, n_views));
    c->total_len.ensure(size_t(3) * std::max(1, n_views));
    c->degenerate.ensure(std::max(1, n_views));
}

void launch_silhouettes(cdr_ctx* c, int n_views) {
    if (n_views <= 0) return;
    BStatics& st = bstatics(c);
    const int E = std::max(1, c->E);
    const int nb = (E + kBlock - 1) / kBlock;
    c->sil_flag.ensure(size_t(n_views) * E);
    c->sil_block_count.ensure(size_t(n_views) * nb);
    c->sil_block_off.ensure(size_t(n_views) * nb);
    if (c->E == 0) {
        CDR_CUDA_CHECK(cudaMemsetAsync(c->sil_count.p, 0, sizeof(int32_t) * n_views, c->stream));
        return;
    }
    dim3 grid(nb, n_views);
    k_sil_flag<<<grid, kBlock, 0, c->stream>>>(c->pos.p, c->fnormal.p, c->edges.p, c->E, c->d_cams.p,
                                               st.calls.p, c->sil_flag.p, c->sil_block_count.p, nb);
    k_sil_scan<<<n_views, 1024, 0, c->stream>>>(c->sil_block_count.p, nb, c->sil_block_off.p,
                                                c->sil_count.p);
    k_sil_write<<<grid, kBlock, 0, c->stream>>>(c->pos.p, c->fnormal.p, c->edges.p, c->E, c->d_cams.p,
                                                st.calls.p, c->sil_flag.p, c->sil_block_off.p, nb,
                                                c->segs.p);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_cdf(cdr_ctx* c, int n_views) {
    if (n_views <= 0) return;
    k_cdf<<<(n_views + 31) / 32, 32, 0, c->stream>>>(c->segs.p, c->sil_count.p, std::max(1, c->E),
                                                     n_views, c->cdf.p, c->total_len.p, c->degenerate.p);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_boundary(cdr_ctx* c, int n_views, int samples, uint64_t seed, int probe,
                     int64_t lay_pos) {
    if (n_views <= 0 || samples <= 0) return;
    BStatics& st = bstatics(c);
    size_t nslots = c->views.size();
    std::vector<size_t> offs(nslots);
    for (size_t i = 0; i < nslots; ++i) offs[i] = c->views[i].pix_off;
    st.pix_off.ensure(nslots);
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.pix_off.p, offs.data(), sizeof(size_t) * nslots,
                                   cudaMemcpyHostToDevice, c->stream));
    BParams p{};
    p.sc = shade_scene(c);
    p.info = c->info.p;
    p.cams = c->d_cams.p;
    p.calls = st.calls.p;
    p.pix_off = st.pix_off.p;
    p.segs = c->segs.p;
    p.cdf = c->cdf.p;
    p.totals = c->total_len.p;
    p.count = c->sil_count.p;
    p.E = std::max(1, c->E);
    p.seed = seed;
    p.probe = probe;
    p.adj = c->adj.p;
    p.grad = c->grad.p;
    p.lay_pos = lay_pos;
    p.err = c->errinfo.p;
    p.counters = c->counters.p;
    dim3 grid((samples + kBlock - 1) / kBlock, n_views);
    k_boundary<<<grid, kBlock, 0, c->stream>>>(p);
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr
