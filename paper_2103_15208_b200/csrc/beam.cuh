// beam.cuh — tile-frustum ("beam") traversal of the LBVH for primary rays.
//
// All primary rays of a pixel tile leave the camera origin through one small
// pixel rectangle, so their BVH paths nearly coincide. Instead of every sample
// traversing the tree (13 node visits and a stack per ray), ONE frustum
// traversal per tile collects the candidate triangles: every leaf whose padded
// box is not entirely outside one of the tile frustum's five planes. A sample
// then scans the tile's candidates in order of a lower bound on their hit
// distance, rejects most with an fp32 screen-space edge test, runs the exact
// fp64 Moller-Trumbore (bvh.cuh leaf_test) on the rest, and stops as soon as
// the next candidate's bound exceeds its best hit.
//
// Exactness: a triangle any ray of the tile can hit intersects
// the tile frustum, so its box survives the conservative plane tests and it is
// a candidate; the 2D test only rejects sample points farther than 0.01 px
// outside the projected triangle (fp32 error is ~1e-5 px), and triangles whose
// projection is unreliable (a vertex near or behind the camera plane, edge-on)
// always go to the exact test; the distance bound is a lower bound on t
// (rays are unit length), compared strictly, so ties to a lower triangle index
// are never cut off. The answer is the brute-force oracle's, as for trace().
// Tiles with more than kBeamCap candidates fall back to per-ray traversal.
#pragma once

#include <cuda_fp16.h>

#include "bvh.cuh"

namespace cdr {

#ifndef CDR_BEAM_CAP
#define CDR_BEAM_CAP 128
#endif
#ifndef CDR_FRONT_CAP
#define CDR_FRONT_CAP 256
#endif
constexpr int kBeamCap = CDR_BEAM_CAP;    // candidates per tile; more -> per-ray traversal
#ifndef CDR_PIX_CAP
#define CDR_PIX_CAP 64
#endif
#ifndef CDR_BIG_PIX_CAP
#define CDR_BIG_PIX_CAP 128
#endif
constexpr int kPixCap = CDR_PIX_CAP;         // candidates per pixel list; more -> scan the tile list
constexpr int kBigPixCap = CDR_BIG_PIX_CAP;  // the same for big tiles (over kBeamCap candidates)
static_assert(kPixCap < 255 && kBigPixCap < 255, "255 marks an overflowed pixel list");
static_assert(kPixCap % 4 == 0 && kBigPixCap % 4 == 0, "lists are read four entries per 32-bit load");
constexpr int kFrontCap = CDR_FRONT_CAP;  // builder frontier per tile; more -> per-ray traversal

// Candidate record, 32 B = one sector (the list scans are L1-bandwidth bound:
// 48-B records measured the boundary probes at 72 % L1 throughput): the
// distance bound, the leaf index with the "always run the exact test" flag in
// bit 31, and three edge functions E_i = A_i x + B_i y + C_i in pixels
// relative to the tile origin, normalised by the edge length (|A|, |B| <= 1),
// E_i >= 0 for all i -> possible hit. A and B are stored as fp16; C (fp32,
// rounded up) carries the 0.01 px margin plus the fp16 rounding error of A and
// B over the tile (|dA| TW + |dB| TH), so the test stays conservative.
struct __align__(16) BeamCand {
    float4 a;  // dmin, leaf | flag << 31, half2 (A0, B0), half2 (A1, B1)
    float4 b;  // half2 (A2, B2), C0, C1, C2
};

__device__ __forceinline__ float2 cand_ab(float f) {
    const unsigned u = __float_as_uint(f);
    return make_float2(__half2float(__ushort_as_half((unsigned short)(u & 0xffffu))),
                       __half2float(__ushort_as_half((unsigned short)(u >> 16))));
}
__device__ __forceinline__ bool cand_always(const float4& a) { return __float_as_int(a.y) < 0; }
__device__ __forceinline__ int cand_leaf(const float4& a) { return __float_as_int(a.y) & 0x7fffffff; }
// edge coefficients A[3], B[3], C[3] of a record
__device__ __forceinline__ void cand_edges(const float4& a, const float4& b, float A[3], float B[3], float C[3]) {
    const float2 e0 = cand_ab(a.z), e1 = cand_ab(a.w), e2 = cand_ab(b.x);
    A[0] = e0.x; B[0] = e0.y; C[0] = b.y;
    A[1] = e1.x; B[1] = e1.y; C[1] = b.z;
    A[2] = e2.x; B[2] = e2.y; C[2] = b.w;
}
// the 2D test at tile-relative point (x, y)
__device__ __forceinline__ bool cand_covers(const float4& a, const float4& b, float x, float y) {
    if (cand_always(a)) return true;
    const float2 e0 = cand_ab(a.z), e1 = cand_ab(a.w), e2 = cand_ab(b.x);
    return e0.x * x + e0.y * y + b.y >= 0.0f && e1.x * x + e1.y * y + b.z >= 0.0f && e2.x * x + e2.y * y + b.w >= 0.0f;
}

struct TileHdr {
    int off;  // first candidate in the pool; split tiles: index of their 4 quadrant lists
    int cnt;  // candidates, or -1: overflow (per-ray traversal), -2: split into quadrants
    int big;  // index of the tile's kBigPixCap pixel lists, -1: the kPixCap ones
    int pad;
};

// A tile whose big-pass list overflows (> 255 candidates: silhouette-dense
// tiles of thin geometry) is split into its four pixel quadrants, each with
// its own candidate list (off, cnt; cnt -1: that quadrant traverses per ray,
// -2: split once more into its own quadrants, off = their group). The pixel
// lists of every level stay in the tile's big slot (pixel q's list indexes
// its own list's candidates), and the edge functions stay relative to the
// tile origin, so a consumer only swaps the (off, cnt) it scans.
// (first candidate, count) of the list pixel q of tile header h scans.
__device__ __forceinline__ int2 pixel_tile_list(const TileHdr& h, const int2* __restrict__ split, int q, int TW,
                                                int TH) {
    if (h.cnt != -2) return make_int2(h.off, h.cnt);
    const int qx = q % TW, qy = q / TW;
    int rx = 0, ry = 0, rw = TW, rh = TH, g = h.off;
    while (true) {  // descend the quadrant splits (k_tile_lists_split): at most two levels
        const int hw = rw / 2, hh = rh / 2;
        const bool bx = qx - rx >= hw, by = qy - ry >= hh;
        const int2 e = split[4 * g + (by ? 2 : 0) + (bx ? 1 : 0)];
        if (e.y != -2) return e;
        g = e.x;
        if (bx) {
            rx += hw;
            rw -= hw;
        } else {
            rw = hw;
        }
        if (by) {
            ry += hh;
            rh -= hh;
        } else {
            rh = hh;
        }
    }
}

struct FrustumPlanes {
    float n[5][3];  // inward normals through the camera origin
};

// Inward plane normals of the frustum through pixel rectangle [x0,x1]x[y0,y1]
// (camera.cpp:29-34: pixel x <-> (q.r)/(q.f) = (2x/W - 1) th aspect, y <-> (q.u)/(q.f) = (1 - 2y/H) th).
__device__ __forceinline__ FrustumPlanes tile_frustum(const DevCamera& c, double x0, double x1, double y0,
                                                      double y1) {
    // culling planes only: one reciprocal per axis (its rounding is far below
    // the callers' 0.01 px margins and box_outside's slack)
    const double kx = 2.0 / c.W, ky = 2.0 / c.H;
    const double s0 = (x0 * kx - 1.0) * c.th * c.aspect, s1 = (x1 * kx - 1.0) * c.th * c.aspect;
    const double v0 = (1.0 - y0 * ky) * c.th, v1 = (1.0 - y1 * ky) * c.th;
    FrustumPlanes fp;
    for (int k = 0; k < 3; ++k) {
        fp.n[0][k] = float(c.r[k] - s0 * c.f[k]);  // x >= x0
        fp.n[1][k] = float(s1 * c.f[k] - c.r[k]);  // x <= x1
        fp.n[2][k] = float(v0 * c.f[k] - c.u[k]);  // y >= y0
        fp.n[3][k] = float(c.u[k] - v1 * c.f[k]);  // y <= y1
        fp.n[4][k] = float(c.f[k]);                // in front of the camera
    }
    return fp;
}

// Conservative: true only if the box is certainly outside one plane.
__device__ __forceinline__ bool box_outside(const FrustumPlanes& fp, const float o[3], float lx, float ly,
                                            float lz, float hx, float hy, float hz) {
    const float cx = 0.5f * (lx + hx) - o[0], cy = 0.5f * (ly + hy) - o[1], cz = 0.5f * (lz + hz) - o[2];
    const float ex = 0.5f * (hx - lx), ey = 0.5f * (hy - ly), ez = 0.5f * (hz - lz);
    const float mag = fabsf(cx) + fabsf(cy) + fabsf(cz) + ex + ey + ez;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const float* n = fp.n[k];
        const float d = n[0] * cx + n[1] * cy + n[2] * cz;
        const float r = fabsf(n[0]) * ex + fabsf(n[1]) * ey + fabsf(n[2]) * ez;
        const float slack = 1e-5f * (fabsf(n[0]) + fabsf(n[1]) + fabsf(n[2])) * mag;
        if (d + r < -slack) return true;
    }
    return false;
}

// Conservative overlap of a candidate's (margined) projected triangle with the
// pixel rectangle [x0,x0+1]x[y0,y0+1] (tile-relative): false only if one edge
// function is negative on all four corners.
__device__ __forceinline__ bool cand_overlaps_pixel(const BeamCand& c, float x0, float y0) {
    if (cand_always(c.a)) return true;
    const float x1 = x0 + 1.0f, y1 = y0 + 1.0f;
    float A[3], B[3], C[3];
    cand_edges(c.a, c.b, A, B, C);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = A[i] * (A[i] > 0 ? x1 : x0) + B[i] * (B[i] > 0 ? y1 : y0) + C[i];
        if (m < 0.0f) return false;
    }
    return true;
}

// cand_overlaps_pixel for every pixel of a tile of P <= 32 pixels, TW wide:
// bit q set when pixel (q % TW, q / TW) may be covered. Same arithmetic per
// pixel as cand_overlaps_pixel, so the same decisions.
__device__ __forceinline__ unsigned cand_pixel_mask(const BeamCand& c, int TW, int P) {
    const unsigned all = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
    if (cand_always(c.a)) return all;
    float A[3], B[3], C[3];
    cand_edges(c.a, c.b, A, B, C);
    unsigned m = 0;
    int qx = 0, qy = 0;
    for (int q = 0; q < P; ++q) {
        const float x0 = float(qx), y0 = float(qy), x1 = x0 + 1.0f, y1 = y0 + 1.0f;
        bool in = true;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const float v = A[i] * (A[i] > 0 ? x1 : x0) + B[i] * (B[i] > 0 ? y1 : y0) + C[i];
            in = in && !(v < 0.0f);
        }
        m |= unsigned(in) << q;
        if (++qx == TW) {
            qx = 0;
            ++qy;
        }
    }
    return m;
}

// Nearest hit of one sample ray using its tile's candidate list (smem or
// global). Same result as trace(): exact fp64 test, strict t_min < t, ties to
// the lowest triangle index.
__device__ __forceinline__ Hit trace_beam(const BeamCand* __restrict__ cand, int n, const TriRec* __restrict__ recs,
                                          D3 o, D3 d, double t_min, float px, float py) {
    Hit best{-1, 1e300, 0.0, 0.0};
    for (int k = 0; k < n; ++k) {
        // the whole 32-B record in one round trip (the edge functions are
        // needed unless the bound stops the scan)
        const float4 ra = cand[k].a, rb = cand[k].b;
        if (double(ra.x) > best.t) break;  // every remaining candidate is farther
        CDR_STAT(3, 1);
        if (cand_covers(ra, rb, px, py)) leaf_test(recs, cand_leaf(ra), o, d, t_min, best);
    }
    return best;
}

// Same scan over an index list (a pixel's candidates, in distance order).
__device__ __forceinline__ Hit trace_beam_list(const BeamCand* __restrict__ cand, const unsigned char* __restrict__ idx,
                                               int n, const TriRec* __restrict__ recs, D3 o, D3 d, double t_min,
                                               float px, float py) {
    Hit best{-1, 1e300, 0.0, 0.0};
    unsigned iw = 0;  // four list entries per load (lists are 4-byte aligned, kPix % 4 == 0)
    for (int j = 0; j < n; ++j) {
        if ((j & 3) == 0) iw = __ldg(reinterpret_cast<const unsigned*>(idx + j));
        const int k = int((iw >> (8 * (j & 3))) & 0xffu);
        CDR_DCHECK(k < 255);
        const float4 ra = cand[k].a, rb = cand[k].b;
        if (double(ra.x) > best.t) break;
        CDR_STAT(3, 1);
        if (cand_covers(ra, rb, px, py)) leaf_test(recs, cand_leaf(ra), o, d, t_min, best);
    }
    return best;
}

// Per-call view of the beam lists for consumers other than k_trace (the
// boundary probes): tile geometry of the render call and its per-view bases.
struct BeamView {
    const TileHdr* hdr;
    const BeamCand* pool;
    const unsigned char* pix_list;
    const unsigned char* pix_cnt;
    const unsigned char* big_pix_list;
    const unsigned char* big_pix_cnt;
    const int* tile_base;  // per view index of the call
    const int2* split;     // quadrant lists of split tiles (4 per split tile)
    int TW, TH, P;
    int valid;
};

// Nearest hit for a ray through continuous pixel point x of view vi, using
// the candidate list of the pixel containing x; per-ray traversal when x is
// outside the image, the tile overflowed, or no lists exist for this call.
__device__ __forceinline__ Hit trace_point(const BeamView& bv, int vi, const DevCamera& cam, const BNode* nodes,
                                           const TriRec* recs, int n_tris, D2 x, D3 d, double t_min) {
    const D3 o{cam.o[0], cam.o[1], cam.o[2]};
    if (bv.valid) {
        const double fx = floor(x.x), fy = floor(x.y);
        if (fx >= 0 && fy >= 0 && fx < cam.W && fy < cam.H) {
            const int px = int(fx), py = int(fy);
            const int tiles_x = (cam.W + bv.TW - 1) / bv.TW;
            const int tx = px / bv.TW, ty = py / bv.TH;
            const size_t tile = size_t(bv.tile_base[vi]) + ty * tiles_x + tx;
            const TileHdr h = bv.hdr[tile];
            const int q = (py - ty * bv.TH) * bv.TW + (px - tx * bv.TW);
            const int2 tl = pixel_tile_list(h, bv.split, q, bv.TW, bv.TH);
            if (tl.y >= 0) {
                const size_t li = h.big >= 0 ? size_t(h.big) * bv.P + q : tile * bv.P + q;
                const int cnt = h.big >= 0 ? bv.big_pix_cnt[li] : bv.pix_cnt[li];
                const unsigned char* lst = h.big >= 0 ? bv.big_pix_list + li * kBigPixCap : bv.pix_list + li * kPixCap;
                const float lx = float(x.x - tx * bv.TW), ly = float(x.y - ty * bv.TH);
                if (cnt == 0) return Hit{-1, 1e300, 0.0, 0.0};
                if (cnt == 255) return trace_beam(bv.pool + tl.x, tl.y, recs, o, d, t_min, lx, ly);
                return trace_beam_list(bv.pool + tl.x, lst, cnt, recs, o, d, t_min, lx, ly);
            }
        }
    }
    return trace(nodes, recs, n_tris, o, d, t_min);
}

// Two probes at once (the boundary pass traces x - n/2 and x + n/2 of every
// edge sample): the same scans as trace_point, stepped in one loop so each
// thread keeps two independent candidate -> triangle load chains in flight.
// Per-ray traversal (off-image points, overflowing tiles) runs afterwards.
#ifdef CDR_TRACE_STATS
// debug build only: [0] per-ray (off-image / no lists), [1] per-ray (overflow
// tile), [2] small-tile pixel list, [3] big-tile pixel list, [4] whole small
// tile scanned, [5] whole big tile scanned, [6] scan steps, [7] empty list
static __device__ unsigned long long g_probe_stats[8];
#define CDR_PSTAT(i, v) atomicAdd(&g_probe_stats[i], (unsigned long long)(v))
#else
#define CDR_PSTAT(i, v)
#endif

// The scan keeps only the best hit's triangle, t and leaf; its barycentrics
// are recomputed once at the end by the same ray_triangle (identical values),
// which keeps two doubles per probe out of the scan's register set.
struct ProbeScan {
    const BeamCand* cand;
    const unsigned char* lst;  // nullptr: scan the whole tile list
    unsigned iw;               // the current 4-entry word of lst
    int n, j;
    float lx, ly;
    int mode;  // 0 done, 1 scanning, 2 per-ray traversal
    int tri, leaf;
    double t;
};

__device__ __forceinline__ void probe_leaf_test(const TriRec* __restrict__ recs, int leaf, D3 o, D3 d, double t_min,
                                                ProbeScan& s) {
    const TriRec* p = recs + leaf;
    const double2 a = __ldg(&p->a), b = __ldg(&p->b), c = __ldg(&p->c), dd = __ldg(&p->d);
    const double e = __ldg(&p->e);
    const int tri = __ldg(&p->tri);
    double t, b1, b2;
    if (ray_triangle(o, d, D3{a.x, a.y, b.x}, D3{b.y, c.x, c.y}, D3{dd.x, dd.y, e}, t, b1, b2) && t > t_min &&
        (t < s.t || (t == s.t && tri < s.tri))) {
        s.t = t;
        s.tri = tri;
        s.leaf = leaf;
    }
}

// the Hit of a finished scan (barycentrics of its triangle, as leaf_test had them)
__device__ __forceinline__ Hit probe_hit(const TriRec* __restrict__ recs, D3 o, D3 d, const ProbeScan& s) {
    Hit h{-1, 1e300, 0.0, 0.0};
    if (s.tri < 0) return h;
    const TriRec* p = recs + s.leaf;
    const double2 a = __ldg(&p->a), b = __ldg(&p->b), c = __ldg(&p->c), dd = __ldg(&p->d);
    const double e = __ldg(&p->e);
    double t, b1, b2;
    ray_triangle(o, d, D3{a.x, a.y, b.x}, D3{b.y, c.x, c.y}, D3{dd.x, dd.y, e}, t, b1, b2);
    h.tri = s.tri;
    h.t = t;
    h.b1 = b1;
    h.b2 = b2;
    return h;
}

__device__ __forceinline__ void probe_setup(const BeamView& bv, int vi, const DevCamera& cam, D2 x, ProbeScan& s) {
    s.tri = -1;
    s.leaf = 0;
    s.t = 1e300;
    s.mode = 2;
    s.j = 0;
    if (!bv.valid) {
        CDR_PSTAT(0, 1);
        return;
    }
    const double fx = floor(x.x), fy = floor(x.y);
    if (!(fx >= 0 && fy >= 0 && fx < cam.W && fy < cam.H)) {
        CDR_PSTAT(0, 1);
        return;
    }
    const int px = int(fx), py = int(fy);
    const int tiles_x = (cam.W + bv.TW - 1) / bv.TW;
    const int tx = px / bv.TW, ty = py / bv.TH;
    const size_t tile = size_t(bv.tile_base[vi]) + ty * tiles_x + tx;
    const TileHdr h = bv.hdr[tile];
    const int q = (py - ty * bv.TH) * bv.TW + (px - tx * bv.TW);
    const int2 tl = pixel_tile_list(h, bv.split, q, bv.TW, bv.TH);
    if (tl.y < 0) {
        CDR_PSTAT(1, 1);
        return;
    }
    const size_t li = h.big >= 0 ? size_t(h.big) * bv.P + q : tile * bv.P + q;
    const int cnt = h.big >= 0 ? bv.big_pix_cnt[li] : bv.pix_cnt[li];
    s.cand = bv.pool + tl.x;
    s.lx = float(x.x - tx * bv.TW);
    s.ly = float(x.y - ty * bv.TH);
    if (cnt == 255) {
        s.lst = nullptr;
        s.n = tl.y;
    } else {
        s.lst = h.big >= 0 ? bv.big_pix_list + li * kBigPixCap : bv.pix_list + li * kPixCap;
        s.n = cnt;
    }
    s.mode = s.n > 0 ? 1 : 0;
    CDR_PSTAT(s.n == 0 ? 7 : (cnt == 255 ? (h.big >= 0 ? 5 : 4) : (h.big >= 0 ? 3 : 2)), 1);
}

// one candidate of trace_beam / trace_beam_list
__device__ __forceinline__ void probe_step(ProbeScan& s, const TriRec* __restrict__ recs, D3 o, D3 d, double t_min) {
    if (s.j >= s.n) {
        s.mode = 0;
        return;
    }
    int k = s.j;
    if (s.lst) {  // four list entries per load: no dependent byte load on most steps
        if ((s.j & 3) == 0) s.iw = __ldg(reinterpret_cast<const unsigned*>(s.lst + s.j));
        k = int((s.iw >> (8 * (s.j & 3))) & 0xffu);
    }
    ++s.j;
    CDR_PSTAT(6, 1);
    const float4 ra = s.cand[k].a, rb = s.cand[k].b;
    if (double(ra.x) > s.t) {  // every remaining candidate is farther
        s.mode = 0;
        return;
    }
    if (cand_covers(ra, rb, s.lx, s.ly)) probe_leaf_test(recs, cand_leaf(ra), o, d, t_min, s);
}

// Per-ray traversal for the rare probe without a usable list (off-image
// points, lists that overflowed every pass): out of line, so its stack and
// registers do not weigh on the list scans around it.
static __device__ __noinline__ Hit trace_out_of_line(const BNode* nodes, const TriRec* recs, int n_tris, D3 o, D3 d,
                                              double t_min) {
    return trace(nodes, recs, n_tris, o, d, t_min);
}

__device__ __forceinline__ void trace_points2(const BeamView& bv, int vi, const DevCamera& cam, const BNode* nodes,
                                              const TriRec* recs, int n_tris, D2 xa, D3 da, D2 xb, D3 db,
                                              double t_min, Hit& ha, Hit& hb) {
    const D3 o{cam.o[0], cam.o[1], cam.o[2]};
    ProbeScan a, b;
    probe_setup(bv, vi, cam, xa, a);
    probe_setup(bv, vi, cam, xb, b);
    while (a.mode == 1 || b.mode == 1) {
        if (a.mode == 1) probe_step(a, recs, o, da, t_min);
        if (b.mode == 1) probe_step(b, recs, o, db, t_min);
    }
    ha = a.mode == 2 ? trace_out_of_line(nodes, recs, n_tris, o, da, t_min) : probe_hit(recs, o, da, a);
    hb = b.mode == 2 ? trace_out_of_line(nodes, recs, n_tris, o, db, t_min) : probe_hit(recs, o, db, b);
}

}  // namespace cdr
