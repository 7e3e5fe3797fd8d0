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
                            const int32_t* __restrict__ block_off, int nb, int stride,
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
    if (f) make_segment(pos, fn, edges[i], cam, &segs[size_t(vi) * stride + off]);
}

// Running CDF in segment order (diff_render.cpp:213-228), one warp per view:
// the lanes load 32 segment lengths at once, then every lane steps through the
// same sequence of 32 additions (shuffled in segment order) and keeps the
// prefix at its own position, so each value is the reference's sequential
// sum, bit for bit, without a load latency per segment.
// totals[3 vi] = {total_len (acc), usable, extract_total}
__global__ void __launch_bounds__(32) k_cdf(const cdr_segment* __restrict__ segs, const int32_t* __restrict__ count,
                                            int E, int n_views, double* __restrict__ cdf,
                                            double* __restrict__ totals, int32_t* __restrict__ degenerate,
                                            int32_t* __restrict__ guide) {
    const int vi = blockIdx.x, lane = threadIdx.x;
    if (vi >= n_views) return;
    const int n = count[vi];
    double acc = 0, ext = 0;
    int usable = 0, deg = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const double raw = i < n ? segs[size_t(vi) * E + i].length_px : 0.0;
        const bool dg = i < n && raw < 1e-12;
        const double len = dg ? 0.0 : raw;
        deg += __popc(__ballot_sync(0xffffffffu, dg));
        usable += __popc(__ballot_sync(0xffffffffu, i < n && !dg));
        const int m = min(32, n - base);
        double mine = 0;
        for (int k = 0; k < m; ++k) {
            ext += __shfl_sync(0xffffffffu, raw, k);  // SilhouetteSet::total_length (silhouette.cpp:103)
            acc += __shfl_sync(0xffffffffu, len, k);
            if (k == lane) mine = acc;
        }
        if (i < n) cdf[size_t(vi) * E + i] = mine;
    }
    // Guide table for the samples' lower_bound: guide[k] = lower_bound(cdf,
    // acc * k / n) for k = 0..n (n buckets). A pick in bucket g (rounding can
    // misplace it by one) has its lower_bound in [guide[g-1], guide[g+2]], so
    // the search there returns the full search's index (boundary_setup).
    __syncwarp();  // the lanes' cdf stores are visible to the whole warp
    const double* cv = cdf + size_t(vi) * E;
    int32_t* gd = guide + size_t(vi) * (E + 1);
    for (int k = lane; k <= n && n > 0; k += 32) {
        const double bnd = acc * double(k) / double(n);
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = lo + ((hi - lo) >> 1);
            if (cv[mid] < bnd) lo = mid + 1;
            else hi = mid;
        }
        gd[k] = lo;
    }
    if (lane == 0) {
        totals[3 * vi] = acc;
        totals[3 * vi + 1] = (n == 0 || ext <= 0 || usable == 0 || acc <= 0) ? 0.0 : 1.0;
        totals[3 * vi + 2] = ext;
        degenerate[vi] = (n == 0 || ext <= 0) ? 0 : deg;
    }
}

struct BParams {
    ShadeScene sc;
    BeamView beam;  // candidate lists of the render call (beam.cuh)
    const SceneInfo* info;
    const DevCamera* cams;
    const SilCall* calls;
    const size_t* pix_off;
    const cdr_segment* segs;
    const double* cdf;
    const int32_t* guide;  // n_views x (E + 1): k_cdf's lower_bound guide
    const double* totals;
    const int32_t* count;
    int E;
    int m_stride;  // per-view stride of the sample arrays (max M)
    uint64_t seed;
    int probe;
    int sample_adj;  // k_bsample drops zero-adjoint samples (else k_boundary does, before its probes)
    const double* adj;
    double* grad;
    int64_t lay_pos;
    ErrorInfo* err;
    Counters* counters;
    int32_t* seg_count;  // n_views x E : active samples per segment
    int32_t* seg_off;    // n_views x E : exclusive scan of seg_count
    int32_t* n_active;   // n_views
    int32_t* key;        // n_views x m_stride : segment of sample i (-1 inactive)
    int32_t* slot;       // n_views x m_stride : rank inside its segment
    double* s_param;     // n_views x m_stride : s of sample i (pass 1)
    int32_t* sorted_si;  // n_views x m_stride : segment of the j-th grouped sample
    double* sorted_s;    // n_views x m_stride : its s
};

// Steps of diff_render.cpp:232-244 for sample i: RNG pick, lower_bound,
// position on the segment, pixel adjoint; false when the sample is skipped.
struct BSample {
    int si;
    double s;
    D2 xq;
    D3 adj;
    const cdr_segment* sg;
};

__device__ __forceinline__ bool boundary_setup(const BParams& p, int vi, int64_t i, BSample& b) {
    const DevCamera& cam = p.cams[p.calls[vi].slot];
    const int nseg = p.count[vi];
    if (p.totals[3 * vi + 1] == 0.0 || i >= p.calls[vi].samples) return false;
    const double total_len = p.totals[3 * vi];
    Rng rng = rng2(p.seed, uint64_t(cam.gid) + 0xb0d1, uint64_t(i));
    double pick = rng.next_double() * total_len;
    const double* cdf = p.cdf + size_t(vi) * p.E;
    int lo = 0, hi = nseg;  // std::lower_bound, narrowed by the guide to a range holding its answer
    {
        int g = int(pick * double(nseg) / total_len);
        g = g < 0 ? 0 : (g > nseg - 1 ? nseg - 1 : g);
        const int32_t* gd = p.guide + size_t(vi) * (p.E + 1);
        lo = gd[g > 0 ? g - 1 : 0];
        hi = gd[g + 2 <= nseg ? g + 2 : nseg];
    }
    while (lo < hi) {
        int mid = lo + ((hi - lo) >> 1);
        if (cdf[mid] < pick) lo = mid + 1;
        else hi = mid;
    }
    b.si = lo < nseg - 1 ? lo : nseg - 1;
    CDR_DCHECK(b.si >= 0 && b.si < nseg && nseg <= p.E);
    b.sg = p.segs + size_t(vi) * p.E + b.si;
    if (b.sg->length_px < 1e-12) return false;
    b.s = rng.next_double();
    const cdr_segment* sg = b.sg;
    if (!p.sample_adj) return true;  // the adjoint is not known yet: k_boundary checks it
    b.xq = D2{sg->q0[0] + (sg->q1[0] - sg->q0[0]) * b.s, sg->q0[1] + (sg->q1[1] - sg->q0[1]) * b.s};
    int px = int(floor(b.xq.x)), py = int(floor(b.xq.y));
    px = px < 0 ? 0 : (px > cam.W - 1 ? cam.W - 1 : px);
    py = py < 0 ? 0 : (py > cam.H - 1 ? cam.H - 1 : py);
    b.adj = ld3(p.adj + 3 * (p.pix_off[p.calls[vi].slot] + size_t(py) * cam.W + px));
    return !(b.adj.x == 0 && b.adj.y == 0 && b.adj.z == 0);
}

// Samples are binned by (segment, position along it): kSBins buckets of s per
// segment, so a warp of the probe kernel traces nearly identical rays.
#ifndef CDR_SBINS
#define CDR_SBINS 32
#endif
constexpr int kSBins = CDR_SBINS;

// pass 1: classify every sample, count active samples per (segment, s bucket)
__global__ void __launch_bounds__(kBlock) k_bsample(BParams p) {
    const int vi = blockIdx.y;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    BSample b;
    bool act = i < p.m_stride && boundary_setup(p, vi, i, b);
    const int bin = act ? b.si * kSBins + min(kSBins - 1, int(b.s * kSBins)) : 0;
    const int key = act ? bin : -1 - int(threadIdx.x & 31);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (act && lane == leader) base = atomicAdd(&p.seg_count[size_t(vi) * p.E * kSBins + bin], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (i < p.m_stride) {
        size_t o = size_t(vi) * p.m_stride + i;
        p.key[o] = act ? bin : -1;
        p.slot[o] = base + __popc(peers & ((1u << lane) - 1u));
        if (act) p.s_param[o] = b.s;
    }
}

// pass 2 (one CTA per view): exclusive scan of the per-bin counts. Chunks of
// 4,096 bins: four consecutive bins per thread, a warp-shuffle scan of the
// thread sums, one more over the 32 warp totals (two barriers per chunk).
__global__ void __launch_bounds__(1024) k_bscan(int32_t* __restrict__ count, const int32_t* __restrict__ nseg, int E,
                                                int32_t* __restrict__ off, int32_t* __restrict__ n_active) {
    const int vi = blockIdx.x;
    const int n = nseg[vi] * kSBins;
    const size_t vb = size_t(vi) * size_t(E) * kSBins;  // per-view stride of the bin arrays
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __shared__ int32_t wsum[32];
    int carry = 0;
    for (int base = 0; base < n; base += 4 * 1024) {
        const int i0 = base + 4 * int(threadIdx.x);
        int v[4];
        int tsum = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k;
            v[k] = i < n ? count[vb + i] : 0;
            if (i < n) count[vb + i] = 0;  // counters are left zeroed for the next call
            tsum += v[k];
        }
        int x = tsum;  // inclusive scan of the thread sums within the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int t = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        int e = carry + (w > 0 ? wsum[w - 1] : 0) + x - tsum;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k;
            if (i < n) off[vb + i] = e;
            e += v[k];
        }
        carry += wsum[31];
        __syncthreads();  // wsum is rewritten by the next chunk
    }
    if (threadIdx.x == 0) n_active[vi] = carry;
}

// pass 3: each sample's segment and position, grouped by (segment, position bucket)
__global__ void k_bscatter(BParams p) {
    const int vi = blockIdx.y;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.m_stride) return;
    size_t o = size_t(vi) * p.m_stride + i;
    int k = p.key[o];
    if (k < 0) return;
    size_t d = size_t(vi) * p.m_stride + p.seg_off[size_t(vi) * p.E * kSBins + k] + p.slot[o];
    p.sorted_si[d] = k / kSBins;
    p.sorted_s[d] = p.s_param[o];
}

// pass 4: the two radiance probes and the vertex deposit, in segment order so a
// warp traces neighbouring rays along one silhouette edge (diff_render.cpp:246-277)
#ifndef CDR_BOUNDARY_MIN_BLOCKS
#define CDR_BOUNDARY_MIN_BLOCKS 5  // 5 x 256-thread CTAs / SM, 48 regs: cfg4 boundary 17.41 -> 16.54 ms vs 4 (3, 6, 7 slower)
#endif
#ifndef CDR_BND_BLOCK
#define CDR_BND_BLOCK 256  // 4 x 256-thread CTAs per SM: boundary cfg2 4.05 -> 3.90 ms vs 128, cfg4 35.6 -> 35.2
#endif
constexpr int kBndBlock = CDR_BND_BLOCK;  // a CTA waits for its slowest warp, yet 256 measured best (64 / 128 / 512 slower)

// One warp-wide step: sample j (< n_act: active) of view vi, lanes holding
// consecutive grouped samples. Returns the warp's count of samples with a
// non-zero contribution (uniform across the warp).
template <bool kT64>
__device__ __forceinline__ int boundary_samples(const BParams& p, int vi, const DevCamera& cam, int64_t j, bool act,
                                                int lane) {
    // the RNG pick and lower_bound were done in pass 1: read the grouped result
    BSample b;
    if (act) {
        const size_t o = size_t(vi) * p.m_stride + j;
        b.si = p.sorted_si[o];
        b.s = p.sorted_s[o];
        CDR_DCHECK(b.si >= 0 && b.si < p.count[vi]);
        b.sg = p.segs + size_t(vi) * p.E + b.si;
        const cdr_segment* sg = b.sg;
        b.xq = D2{sg->q0[0] + (sg->q1[0] - sg->q0[0]) * b.s, sg->q0[1] + (sg->q1[1] - sg->q0[1]) * b.s};
        int px = int(floor(b.xq.x)), py = int(floor(b.xq.y));
        px = px < 0 ? 0 : (px > cam.W - 1 ? cam.W - 1 : px);
        py = py < 0 ? 0 : (py > cam.H - 1 ? cam.H - 1 : py);
        b.adj = ld3(p.adj + 3 * (p.pix_off[p.calls[vi].slot] + size_t(py) * cam.W + px));
        if (b.adj.x == 0 && b.adj.y == 0 && b.adj.z == 0) act = false;  // diff_render.cpp:243-244: no probes
    }
    const int samples = p.calls[vi].samples;
    const double total_len = p.totals[3 * vi];
    double weighted = 0;
    D2 n2{0, 0};
    if (act) {
        const cdr_segment* sg = b.sg;
        // the two quotients with one reciprocal (common.cuh operator/(D3, double): bit-identical)
        const D3 tq = D3{sg->q1[0] - sg->q0[0], sg->q1[1] - sg->q0[1], 1.0} / sg->length_px;
        D2 tg{tq.x, tq.y};
        n2 = D2{-tg.y, tg.x};
        D2 xm{b.xq.x - n2.x * 0.5, b.xq.y - n2.y * 0.5}, xp{b.xq.x + n2.x * 0.5, b.xq.y + n2.y * 0.5};
        const double t_min = p.info->t_min;
        D3 delta;
        if (p.probe == CDR_PROBE_RADIANCE) {
            // radiance_at (render.cpp:24-33) through the pixels' candidate lists
            const D3 dm = primary_dir(cam, xm), dp = primary_dir(cam, xp);
#ifdef CDR_PROBES_SEQUENTIAL
            const Hit hm = trace_point(p.beam, vi, cam, p.sc.nodes, p.sc.recs, p.sc.n_tris, xm, dm, t_min);
            const Hit hp = trace_point(p.beam, vi, cam, p.sc.nodes, p.sc.recs, p.sc.n_tris, xp, dp, t_min);
#else
            Hit hm, hp;
            trace_points2(p.beam, vi, cam, p.sc.nodes, p.sc.recs, p.sc.n_tris, xm, dm, xp, dp, t_min, hm, hp);
#endif
            const D3 bg{p.sc.bg[0], p.sc.bg[1], p.sc.bg[2]};
            // (one shade_hit call in a loop over the two probes: smaller code, slower at cfg4)
            D3 lo3 = hm.tri >= 0 ? shade_hit<kT64>(p.sc, hm, dm) : bg;
            D3 hi3 = hp.tri >= 0 ? shade_hit<kT64>(p.sc, hp, dp) : bg;
            delta = lo3 - hi3;
        } else {
            D3 org{cam.o[0], cam.o[1], cam.o[2]};
            double cm = trace_out_of_line(p.sc.nodes, p.sc.recs, p.sc.n_tris, org, primary_dir(cam, xm), t_min).tri >= 0
                            ? 1.0 : 0.0;
            double cp = trace_out_of_line(p.sc.nodes, p.sc.recs, p.sc.n_tris, org, primary_dir(cam, xp), t_min).tri >= 0
                            ? 1.0 : 0.0;
            delta = D3{cm - cp, cm - cp, cm - cp};
        }
        weighted = dot(b.adj, delta);
        if (weighted == 0) act = false;
        else if (!isfinite(weighted)) {
            if (atomicCAS(&p.err->flag, 0, 2) == 0) p.err->segment = b.si;
            act = false;
        }
    }
    const int na = __popc(__ballot_sync(0xffffffffu, act));
    double v[6] = {0, 0, 0, 0, 0, 0};
    if (act) {
        const cdr_segment* sg = b.sg;
        double w0 = (1.0 - b.s) / sg->z0, w1 = b.s / sg->z1;
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
    const int key = act ? b.si : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    reduce_peers<6>(0xffffffffu, peers, v);
    if (act && (__ffs(peers) - 1) == lane) {
        double* g = p.grad + p.lay_pos;
        for (int c = 0; c < 3; ++c) {
            if (v[c] != 0) atomicAdd(g + 3 * int64_t(b.sg->v0) + c, v[c]);
            if (v[3 + c] != 0) atomicAdd(g + 3 * int64_t(b.sg->v1) + c, v[3 + c]);
        }
    }
    return na;
}

template <bool kT64>
__global__ void __launch_bounds__(kBndBlock, CDR_BOUNDARY_MIN_BLOCKS * 256 / kBndBlock) k_boundary(BParams p) {
    const int vi = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const DevCamera cam = p.cams[p.calls[vi].slot];
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int n_act = p.n_active[vi];
    if (int64_t(blockIdx.x) * blockDim.x >= n_act) return;  // whole CTA idle (uniform)
    const int na = boundary_samples<kT64>(p, vi, cam, j, j < n_act, lane);
    if (lane == 0 && na) atomicAdd(&p.counters->boundary_active, (unsigned long long)na);
}

// cdr_probe_points: point pairs (2i, 2i+1) through trace_points2, the odd last
// point through trace_point, then shade_hit / background as the probes do.
template <bool kT64>
__global__ void k_probe_points(ShadeScene sc, const SceneInfo* __restrict__ info, DevCamera cam, BeamView bv,
                               int vi, int n, const double* __restrict__ xy, double* __restrict__ rgb,
                               int32_t* __restrict__ tri) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = 2 * i, b = 2 * i + 1;
    if (a >= n) return;
    const double t_min = info->t_min;
    const D2 xa{xy[2 * a], xy[2 * a + 1]};
    const D3 da = primary_dir(cam, xa);
    Hit ha, hb;
    D3 db{0, 0, 0};
    if (b < n) {
        const D2 xb{xy[2 * b], xy[2 * b + 1]};
        db = primary_dir(cam, xb);
        trace_points2(bv, vi, cam, sc.nodes, sc.recs, sc.n_tris, xa, da, xb, db, t_min, ha, hb);
    } else {
        ha = trace_point(bv, vi, cam, sc.nodes, sc.recs, sc.n_tris, xa, da, t_min);
    }
    const D3 bg{sc.bg[0], sc.bg[1], sc.bg[2]};
    for (int k = 0; k < 2; ++k) {
        const int j = k == 0 ? a : b;
        if (j >= n) break;
        const Hit& h = k == 0 ? ha : hb;
        if (tri) tri[j] = h.tri;
        if (rgb) {
            const D3 r = h.tri >= 0 ? shade_hit<kT64>(sc, h, k == 0 ? da : db) : bg;
            rgb[3 * j] = r.x;
            rgb[3 * j + 1] = r.y;
            rgb[3 * j + 2] = r.z;
        }
    }
}

struct BStatics {
    DBuf<SilCall> calls;
    DBuf<size_t> pix_off;
    int n_calls = 0;
};

BStatics& bstatics(cdr_ctx* c) {  // owned by the context (free_boundary_statics)
    if (!c->boundary_statics) c->boundary_statics = new BStatics();
    return *static_cast<BStatics*>(c->boundary_statics);
}

}  // namespace

void free_boundary_statics(cdr_ctx* c) {
    auto* st = static_cast<BStatics*>(c->boundary_statics);
    if (!st) return;
    st->calls.release();
    st->pix_off.release();
    delete st;
    c->boundary_statics = nullptr;
}

void set_view_calls(cdr_ctx* c, const int* view_slots, const int* samples, int n_views, int min_stride) {
    BStatics& st = bstatics(c);
    std::vector<SilCall> calls(n_views);
    for (int i = 0; i < n_views; ++i) calls[i] = SilCall{view_slots[i], samples ? samples[i] : 0};
    st.calls.ensure(std::max(1, n_views));
    st.n_calls = n_views;
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.calls.p, calls.data(), sizeof(SilCall) * n_views,
                                   cudaMemcpyHostToDevice, c->stream));
    // per-view stride of the segment/CDF/bin arrays: E, or more for a
    // caller-supplied silhouette set (cdr_boundary_pass) larger than E
    const int E = std::max(std::max(1, c->E), min_stride);
    c->seg_stride = E;
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
    { ++c->launches; k_sil_flag<<<grid, kBlock, 0, c->stream>>>(c->pos.p, c->fnormal.p, c->edges.p, c->E, c->d_cams.p,
                                               st.calls.p, c->sil_flag.p, c->sil_block_count.p, nb); }
    { ++c->launches; k_sil_scan<<<n_views, 1024, 0, c->stream>>>(c->sil_block_count.p, nb, c->sil_block_off.p,
                                                c->sil_count.p); }
    { ++c->launches; k_sil_write<<<grid, kBlock, 0, c->stream>>>(c->pos.p, c->fnormal.p, c->edges.p, c->E, c->d_cams.p,
                                                st.calls.p, c->sil_flag.p, c->sil_block_off.p, nb,
                                                c->seg_stride, c->segs.p); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_cdf(cdr_ctx* c, int n_views) {
    if (n_views <= 0) return;
    c->cdf_guide.ensure(size_t(n_views) * (size_t(c->seg_stride) + 1));
    { ++c->launches; k_cdf<<<n_views, 32, 0, c->stream>>>(c->segs.p, c->sil_count.p, c->seg_stride,
                                                     n_views, c->cdf.p, c->total_len.p, c->degenerate.p,
                                                     c->cdf_guide.p); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

static BParams boundary_params(cdr_ctx* c, int n_views, int samples, uint64_t seed, int probe, int64_t lay_pos,
                               bool use_beam) {
    BStatics& st = bstatics(c);
    const int E = c->seg_stride;  // set_view_calls
    const size_t nm = size_t(n_views) * samples;
    const size_t nbins = size_t(n_views) * E * kSBins;
    if (c->b_seg_count.n < nbins) {  // zeroed once; k_bscan re-zeroes what it consumed
        c->b_seg_count.ensure(nbins);
        CDR_CUDA_CHECK(cudaMemsetAsync(c->b_seg_count.p, 0, sizeof(int32_t) * nbins, c->stream));
    }
    c->b_seg_off.ensure(nbins);
    c->b_n_active.ensure(n_views);
    c->b_key.ensure(nm);
    c->b_slot.ensure(nm);
    c->b_s.ensure(nm);
    c->b_sorted_si.ensure(nm);
    c->b_sorted_s.ensure(nm);
    BParams p{};
    p.sc = shade_scene(c);
    p.info = c->info.p;
    p.cams = c->d_cams.p;
    p.calls = st.calls.p;
    p.pix_off = st.pix_off.p;
    p.segs = c->segs.p;
    p.cdf = c->cdf.p;
    p.guide = c->cdf_guide.p;
    p.totals = c->total_len.p;
    p.count = c->sil_count.p;
    p.E = E;
    p.m_stride = samples;
    p.seed = seed;
    p.probe = probe;
    p.adj = c->adj.p;
    p.grad = c->grad.p;
    p.lay_pos = lay_pos;
    p.err = c->errinfo.p;
    p.counters = c->counters.p;
    p.seg_count = c->b_seg_count.p;
    p.seg_off = c->b_seg_off.p;
    p.n_active = c->b_n_active.p;
    p.key = c->b_key.p;
    p.slot = c->b_slot.p;
    p.beam = c->beam_view;
    p.beam.valid = c->beam_view.valid && use_beam;
    p.s_param = c->b_s.p;
    p.sorted_si = c->b_sorted_si.p;
    p.sorted_s = c->b_sorted_s.p;
    return p;
}

static void upload_pix_off(cdr_ctx* c) {
    BStatics& st = bstatics(c);
    const size_t nslots = c->views.size();
    std::vector<size_t> offs(nslots);
    for (size_t i = 0; i < nslots; ++i) offs[i] = c->views[i].pix_off;
    st.pix_off.ensure(std::max<size_t>(1, nslots));
    // pageable source: the copy is staged before cudaMemcpyAsync returns
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.pix_off.p, offs.data(), sizeof(size_t) * nslots, cudaMemcpyHostToDevice,
                                   c->stream));
}

void launch_boundary_sampling(cdr_ctx* c, int n_views, int samples, uint64_t seed) {
    if (n_views <= 0 || samples <= 0) return;
    BParams p = boundary_params(c, n_views, samples, seed, CDR_PROBE_RADIANCE, 0, false);
    p.sample_adj = 0;
    dim3 grid((samples + kBlock - 1) / kBlock, n_views);
    { ++c->launches; k_bsample<<<grid, kBlock, 0, c->stream>>>(p); }
    { ++c->launches; k_bscan<<<n_views, 1024, 0, c->stream>>>(p.seg_count, p.count, p.E, p.seg_off, p.n_active); }
    { ++c->launches; k_bscatter<<<grid, kBlock, 0, c->stream>>>(p); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

static void launch_k_boundary(cdr_ctx* c, dim3 bgrid, const BParams& p) {
    tex64_resolve(c);
    ++c->launches;
    if (c->tex64_on) k_boundary<true><<<bgrid, kBndBlock, 0, c->stream>>>(p);
    else k_boundary<false><<<bgrid, kBndBlock, 0, c->stream>>>(p);
}

void launch_boundary_probes(cdr_ctx* c, int n_views, int samples, uint64_t seed, int probe, int64_t lay_pos,
                            bool use_beam) {
    if (n_views <= 0 || samples <= 0) return;
    upload_pix_off(c);
    BParams p = boundary_params(c, n_views, samples, seed, probe, lay_pos, use_beam);
    dim3 bgrid((samples + kBndBlock - 1) / kBndBlock, n_views);
    launch_k_boundary(c, bgrid, p);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_boundary(cdr_ctx* c, int n_views, int samples, uint64_t seed, int probe,
                     int64_t lay_pos, bool use_beam) {
    if (n_views <= 0 || samples <= 0) return;
    upload_pix_off(c);
    BParams p = boundary_params(c, n_views, samples, seed, probe, lay_pos, use_beam);
    p.sample_adj = 1;  // the adjoint is on the device: sampling drops zero-adjoint samples itself
    dim3 grid((samples + kBlock - 1) / kBlock, n_views);
    { ++c->launches; k_bsample<<<grid, kBlock, 0, c->stream>>>(p); }
    { ++c->launches; k_bscan<<<n_views, 1024, 0, c->stream>>>(p.seg_count, p.count, p.E, p.seg_off, p.n_active); }
    { ++c->launches; k_bscatter<<<grid, kBlock, 0, c->stream>>>(p); }
    dim3 bgrid((samples + kBndBlock - 1) / kBndBlock, n_views);
    launch_k_boundary(c, bgrid, p);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_probe_points(cdr_ctx* c, int vi, int n, const double* xy, double* rgb, int32_t* tri) {
    if (n <= 0) return;
    const int pairs = (n + 1) / 2;
    const DevCamera cam = c->views[c->beam_slots[vi]].cam;
    tex64_resolve(c);
    ++c->launches;
    if (c->tex64_on)
        k_probe_points<true><<<(pairs + 127) / 128, 128, 0, c->stream>>>(shade_scene(c), c->info.p, cam, c->beam_view,
                                                                         vi, n, xy, rgb, tri);
    else
        k_probe_points<false><<<(pairs + 127) / 128, 128, 0, c->stream>>>(shade_scene(c), c->info.p, cam,
                                                                          c->beam_view, vi, n, xy, rgb, tri);
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr

#ifdef CDR_TRACE_STATS
// debug builds: traversal counters of the boundary probes (this translation unit)
extern "C" int cdr_debug_trace_stats_boundary(unsigned long long out[4]) {
    cudaMemcpyFromSymbol(out, cdr::g_trace_stats, sizeof(unsigned long long) * 4);
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(cdr::g_trace_stats, z, sizeof(z));
    return 0;
}

extern "C" int cdr_debug_probe_stats(unsigned long long out[8]) {
    cudaMemcpyFromSymbol(out, cdr::g_probe_stats, sizeof(unsigned long long) * 8);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(cdr::g_probe_stats, z, sizeof(z));
    return 0;
}
#endif
