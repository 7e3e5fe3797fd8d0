// render.cu — the fused per-sample kernel of the hot path.
//
// One CTA of 256 threads owns a TW x TH pixel tile of one view; thread =
// (pixel, sample), so the spp samples of a pixel are adjacent lanes (coherent
// rays, shared texels). Three phases separated by CTA barriers:
//   1. trace + shade every sample            render.cpp:35-64 / radiance_at :24-33
//   2. per-pixel mean, mask, tone-mapped L1 loss partial and adjoint
//                                            losses.cpp:15-49 (sum in sample order)
//   3. interior adjoint of every hit sample  diff_render.cpp:62-201
// so the reference's hit-cache round trip between render and interior_pass
// disappears (the cache is still written: it is the bit-exact output).
//
// Phase-3 scatter is warp-aggregated: lanes are grouped with __match_any_sync by
// texel (28 texel-gradient values) and by triangle (18 per-corner values), each
// group is summed with log-depth shuffles, and one lane issues the atomics.
// The one-ring normal chain is deferred: per-corner sums of coeff_mu*b_j*h feed
// the finalize kernels (finalize.cu), which apply it once per iteration.
#include <chrono>
#include <cstdio>

#include "kernels.h"
#include "beam.cuh"
#include "shade.cuh"

namespace cdr {
namespace {

struct ViewCall {
    int slot;
    int tile_base;  // first tile of this view in the beam tile arrays
    int tiles_x, tiles_y;  // the view's tile grid
    double scale;     // lambda / n_valid
    uint64_t h_view;  // hash_combine(seed, gid + 0x9e01)
};

struct Params {
    ShadeScene sc;
    const BNode* sc_bin;  // binary LBVH (per-ray traversal and the beam builder)
    const SceneInfo* info;
    const DevCamera* cams;
    const ViewCall* calls;
    size_t* pix_off;  // per slot
    int spp, k, TW, TH;
    double inv_k;
    uint64_t seed;
    double gamma;
    double inv_gamma;  // 1 / gamma (host)
    int use_mask, write_hits;
    int skip_empty_hits;  // loss calls at spp 16: no hit-cache writes for empty beam tiles (k_render skips them too)
    double* img;
    double* mask;
    double* adj;
    int32_t* hit;
    const double* target;
    const double* target_tone;  // Φ(target), precomputed per (target, gamma)
    const double* target_mask;
    const unsigned char* has_mask;  // per slot
    double* grad;
    int64_t lay_d, lay_s, lay_r, lay_l;
    double* corner;
    TexAcc* texacc;  // per texel: diffuse rgb, specular rgb, roughness
    double* loss_acc;
    ErrorInfo* err;
    Counters* counters;
    // beam traversal (beam.cuh): per-tile candidate lists
    TileHdr* tile_hdr;
    BeamCand* pool;
    int pool_cap;
    int* pool_used;
    unsigned char* pix_list;  // per (tile, pixel): kPixCap candidate indices
    unsigned char* pix_cnt;   // per (tile, pixel): count, 255 = scan the tile list
    unsigned char* big_pix_list;  // per (big tile, pixel): kBigPixCap indices
    unsigned char* big_pix_cnt;
    int use_beam;
    int fast_cap;     // candidate cap of the fast pass (kBeamCap; lower only to test the big pass)
    int big_list_cap;  // the same for the big pass (kBigCap; lower only to test the split pass)
    int huge_on;         // lists overflowing both splits go to k_tile_lists_huge (CDR_NO_HUGE: per ray)
    int split_list_cap;  // the same for the split levels (kBigCap; lower only to test level 1 and the huge pass)
    int no_shared_top;  // 1: every tile walks the BVH from the root (A/B and tests)
    int2* big_queue;  // (call, tile) of the tiles over kBeamCap candidates
    int* big_count;
    int big_cap;
    int4* split_queue;  // split work: (big slot, packed rect, list group, level); level 0 = the big-pass overflows
    int* split_count;   // [0] level-0 items, [1] level-1 items, [2] huge-pass items
    int split_cap;      // items per level
    int2* split_hdr;    // groups of 4 quadrant lists (first candidate, count; -1 = per ray, -2 = split again)
    // tile queue (loss calls at spp 16): k_tile_lists appends every non-empty
    // tile (call, tile); k_render then runs over the queue only and
    // k_background writes the empty tiles' pixels
    int2* tile_queue;
    int* tile_queue_count;
    int queue_mode;  // k_render: CTAs from tile_queue instead of the full tile grid
    int queue_len;   // its length (host-read)
    int queue_off;   // k_render: CTA offset into the queue (a launch over a range of it)
    int* top_nodes;  // k_top_walk's output: per 2 x 2 block, [count, <= kTopCap frontier nodes]
    int top_stride;  // blocks per view slot in top_nodes
    int2* blk_queue;      // k_top_walk: the 2 x 2 blocks whose frontier is not empty (view call, block)
    int* blk_queue_count;
};

constexpr int kThreads = 256;
#ifndef CDR_RENDER_THREADS16
#define CDR_RENDER_THREADS16 128  // 4 x 2 pixels: a CTA waits for its slowest warp; smaller is better down to 128
#endif
constexpr int kRenderThreads16 = CDR_RENDER_THREADS16;
#ifndef CDR_TRACE_THREADS16
#define CDR_TRACE_THREADS16 128  // half a beam tile: 6,563 -> 6,709 Msamples/s at cfg2
#endif
constexpr int kTraceThreads16 = CDR_TRACE_THREADS16;  // k_trace CTA at spp 16 (64, 128 or 256)  // k_render CTA at spp 16 (64 per pixel row of 4)

__device__ __forceinline__ void raise_nonfinite(ErrorInfo* e, int x, int y) {
    if (atomicCAS(&e->flag, 0, 1) == 0) {
        e->x = x;
        e->y = y;
        e->segment = -1;
    }
}

// Beam lists, one warp per (view, tile): breadth-first frustum traversal of the
// LBVH (lanes take frontier nodes), candidates sorted by their distance bound
// (rank across lanes), screen-space edge functions, and per-pixel candidate
// lists (conservative triangle/pixel overlap) so a sample scans only the few
// triangles that can cover its pixel. Returns false when the tile has more
// than kCap candidates (or kFront frontier nodes); the header is then untouched.
// Warp bitonic sort of n <= kN 64-bit keys in shared memory (ascending).
template <int kN>
__device__ void warp_bitonic_sort(unsigned long long* key, int n, int lane) {
    for (int i = n + lane; i < kN; i += 32) key[i] = ~0ull;  // pad
    __syncwarp();
    for (int k = 2; k <= kN; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < kN; i += 32) {
                const int l = i ^ j;
                if (l > i) {
                    const unsigned long long a = key[i], c = key[l];
                    const bool up = (i & k) == 0;
                    if ((a > c) == up) {
                        key[i] = c;
                        key[l] = a;
                    }
                }
            }
            __syncwarp();
        }
}

// sub_out != nullptr: the list of one quadrant of a split tile — pixels
// [sx0, sx0 + sw) x [sy0, sy0 + sh) of the tile (tile coordinates), its
// (first candidate, count) written to *sub_out instead of the tile header.
template <int kCap, int kFront, int kPix>
__device__ bool build_tile_list(const Params& p, const ViewCall& vc, const DevCamera& cam, int b, int lane,
                                int (*s_front)[kFront], int* s_leaf, float* s_d, unsigned long long* s_key,
                                int big, const int* init_front = nullptr, int init_n = 0, int sx0 = 0, int sy0 = 0,
                                int sw = 1 << 20, int sh = 1 << 20, int2* sub_out = nullptr, int cap = -1) {
    const int tiles_x = vc.tiles_x;
    const unsigned lt = (1u << lane) - 1u;
    const size_t tile = size_t(vc.tile_base) + b;
    TileHdr* hdr = p.tile_hdr + tile;
    const int X0 = (b % tiles_x) * p.TW, Y0 = (b / tiles_x) * p.TH;
    const int X1 = min(X0 + sx0 + sw, min(X0 + p.TW, cam.W)), Y1 = min(Y0 + sy0 + sh, min(Y0 + p.TH, cam.H));
    const int RX0 = X0 + sx0, RY0 = Y0 + sy0;  // the rectangle the frustum encloses
    if (RX0 >= X1 || RY0 >= Y1) {  // a quadrant wholly outside the image: no pixel asks for it
        if (lane == 0 && sub_out) *sub_out = make_int2(0, 0);
        return true;
    }
    const int T = p.sc.n_tris;
    int nl = 0, nf = 0, cur = 0;
    bool over = false;
    if (T == 1) {
        if (lane == 0) s_leaf[0] = 0;
        nl = 1;
    } else if (T > 1 && init_n < 0) {  // the CTA's union frustum met no node: an empty tile
        nf = 0;
    } else if (T > 1 && init_n > 0) {  // start below the levels the CTA walked together
        for (int i = lane; i < init_n; i += 32) s_front[0][i] = init_front[i];
        nf = init_n;
    } else if (T > 1) {
        if (lane == 0) s_front[0][0] = 0;
        nf = 1;
    }
    __syncwarp();
    FrustumPlanes fp;  // only when there is a frontier (empty blocks skip the fp64 set-up)
    float of[3];
    if (nf > 0) {
        fp = tile_frustum(cam, RX0 - 0.01, X1 + 0.01, RY0 - 0.01, Y1 + 0.01);
        of[0] = float(cam.o[0]);
        of[1] = float(cam.o[1]);
        of[2] = float(cam.o[2]);
    }
    while (nf > 0) {
        int nn = 0;
        for (int base = 0; base < nf; base += 32) {
            const int i = base + lane;
            bool leaf0 = false, leaf1 = false, int0 = false, int1 = false;
            int4 k = make_int4(0, 0, 0, 0);
            if (i < nf) {
                const BNode* np = p.sc_bin + s_front[cur][i];
                const float4 a = __ldg(&np->a), bb = __ldg(&np->b), c = __ldg(&np->c);
                k = __ldg(&np->k);
                const bool in0 = !box_outside(fp, of, a.x, a.y, a.z, a.w, bb.x, bb.y);
                const bool in1 = !box_outside(fp, of, bb.z, bb.w, c.x, c.y, c.z, c.w);
                leaf0 = in0 && k.x < 0;
                int0 = in0 && k.x >= 0;
                leaf1 = in1 && k.y < 0;
                int1 = in1 && k.y >= 0;
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, leaf0), m1 = __ballot_sync(0xffffffffu, leaf1);
            const int p0 = nl + __popc(m0 & lt), p1 = nl + __popc(m0) + __popc(m1 & lt);
            if (leaf0 && p0 < kCap) s_leaf[p0] = ~k.x;
            if (leaf1 && p1 < kCap) s_leaf[p1] = ~k.y;
            nl += __popc(m0) + __popc(m1);
            const unsigned q0 = __ballot_sync(0xffffffffu, int0), q1 = __ballot_sync(0xffffffffu, int1);
            const int f0 = nn + __popc(q0 & lt), f1 = nn + __popc(q0) + __popc(q1 & lt);
            if (int0 && f0 < kFront) s_front[cur ^ 1][f0] = k.x;
            if (int1 && f1 < kFront) s_front[cur ^ 1][f1] = k.y;
            nn += __popc(q0) + __popc(q1);
        }
        __syncwarp();
        if (nl > (cap >= 0 ? cap : kCap) || nn > kFront) {
            over = true;
            break;
        }
        nf = nn;
        cur ^= 1;
    }
    if (over) return false;
    // lower bound on t (unit rays): distance from the origin to the triangle's box
    for (int i = lane; i < nl; i += 32) {
        const TriRec* r = p.sc.recs + s_leaf[i];
        const double2 ra = r->a, rb = r->b, rc = r->c, rd = r->d;
        const double re = r->e;
        const double P[3][3] = {{ra.x, rb.y, rd.x}, {ra.y, rc.x, rd.y}, {rb.x, rc.y, re}};
        double dd = 0;
        for (int k = 0; k < 3; ++k) {
            const double lo = fmin(P[k][0], fmin(P[k][1], P[k][2])), hi = fmax(P[k][0], fmax(P[k][1], P[k][2]));
            const double g = fmax(fmax(lo - cam.o[k], cam.o[k] - hi), 0.0);
            dd += g * g;
        }
        s_d[i] = __double2float_rd(sqrt(dd)) * 0.999999f;
    }
    __syncwarp();
    const D3 o{cam.o[0], cam.o[1], cam.o[2]}, fw{cam.f[0], cam.f[1], cam.f[2]}, rt{cam.r[0], cam.r[1], cam.r[2]},
        up{cam.u[0], cam.u[1], cam.u[2]};
    // candidates go straight to their sorted slots in the pool (no staging)
    int off = 0;
    if (lane == 0 && nl) off = atomicAdd(p.pool_used, nl);
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off + nl > p.pool_cap) {
        if (lane == 0) {
            if (sub_out) *sub_out = make_int2(0, -1);
            else *hdr = TileHdr{0, -1, -1, 0};
            atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
        }
        return true;  // pool full: per-ray traversal
    }
    BeamCand* s_cand = p.pool + off;
    if (s_key) {  // big tiles: sort (distance bits, list position): the same order as the ranks below
        for (int i = lane; i < nl; i += 32)
            s_key[i] = (static_cast<unsigned long long>(__float_as_uint(s_d[i])) << 32) | unsigned(i);
        warp_bitonic_sort<(kCap > 255 ? 1024 : 256)>(s_key, nl, lane);
    }
    for (int i = lane; i < nl; i += 32) {
        int rank = 0;  // distance order, ties by list position
        int src = i;
        if (s_key) {
            rank = i;
            src = int(unsigned(s_key[i]));
        } else {
            const float di = s_d[i];
            for (int j = 0; j < nl; ++j) {
                const float dj = s_d[j];
                rank += (dj < di) || (dj == di && j < i);
            }
        }
        const float di = s_d[src];
        const int leaf = s_leaf[src];
        const TriRec* r = p.sc.recs + leaf;
        const double2 ra = r->a, rb = r->b, rc = r->c, rd = r->d;
        const D3 V[3] = {D3{ra.x, ra.y, rb.x}, D3{rb.y, rc.x, rc.y}, D3{rd.x, rd.y, r->e}};
        double sx[3], sy[3];
        int flags = 0;
        for (int k = 0; k < 3; ++k) {  // project (camera.cpp:36-45), tile-relative pixels
            const D3 q = V[k] - o;
            const double cz = dot(q, fw);
            if (!(cz > 1e-7 * (fabs(q.x) + fabs(q.y) + fabs(q.z)))) flags = 1;
            sx[k] = (dot(q, rt) / (cz * cam.th * cam.aspect) + 1.0) * 0.5 * cam.W - X0;
            sy[k] = (1.0 - dot(q, up) / (cz * cam.th)) * 0.5 * cam.H - Y0;
            if (!(fabs(sx[k]) < 1e4 && fabs(sy[k]) < 1e4)) flags = 1;
        }
        const double area2 = (sx[1] - sx[0]) * (sy[2] - sy[0]) - (sx[2] - sx[0]) * (sy[1] - sy[0]);
        if (!(fabs(area2) > 1e-9)) flags = 1;
        const double sg = area2 < 0 ? -1.0 : 1.0;
        unsigned ab[3] = {0, 0, 0};
        float cc[3] = {0, 0, 0};
        for (int k = 0; k < 3 && !flags; ++k) {
            // E = cross(edge, point - start) / |edge| >= -0.01 px: a signed
            // distance in pixels (|A|, |B| <= 1), so fp16 A, B lose < 2.5e-4
            // each; that rounding over the tile is added to C (rounded up)
            const int j = k == 2 ? 0 : k + 1;
            const double dx = sx[j] - sx[k], dy = sy[j] - sy[k];
            const double inv = sg / sqrt(dx * dx + dy * dy);  // |edge| > 0: area2 > 1e-9 here
            const double A = -dy * inv, B = dx * inv;
            const __half ha = __double2half(A), hb = __double2half(B);
            const double slack = fabs(A - double(__half2float(ha))) * double(p.TW) +
                                 fabs(B - double(__half2float(hb))) * double(p.TH);
            ab[k] = unsigned(__half_as_ushort(ha)) | (unsigned(__half_as_ushort(hb)) << 16);
            cc[k] = __double2float_ru((dy * sx[k] - dx * sy[k]) * inv + 0.01 + slack);
        }
        BeamCand bc;
        bc.a = make_float4(di, __int_as_float(leaf | (flags ? int(0x80000000u) : 0)), __uint_as_float(ab[0]),
                           __uint_as_float(ab[1]));
        bc.b = make_float4(__uint_as_float(ab[2]), cc[0], cc[1], cc[2]);
        s_cand[rank] = bc;
    }
    __syncwarp();  // orders the lanes' pool writes for the per-pixel pass
    // per-pixel lists, in distance order (only the rectangle's pixels)
    const int P = kThreads / p.spp;
    auto in_rect = [&](int q) {
        const int qx = q % p.TW - sx0, qy = q / p.TW - sy0;
        return qx >= 0 && qx < sw && qy >= 0 && qy < sh;
    };
    if (kCap > 255 && nl > 255) {  // candidates beyond a byte index: the rect's pixels scan the whole list
        for (int q = lane; q < P; q += 32)
            if (in_rect(q)) (big >= 0 ? p.big_pix_cnt : p.pix_cnt)[big >= 0 ? size_t(big) * P + q : tile * P + q] = 255;
        if (lane == 0) {
            if (sub_out) *sub_out = make_int2(off, nl);
            else *hdr = TileHdr{off, nl, big, 0};
        }
        return true;
    }
    if (P <= 32) {
        // lane = candidate: a mask of the tile pixels its triangle may cover
        // (the same test as cand_overlaps_pixel), then one ballot per pixel
        // appends the covering candidates in candidate (distance) order
        unsigned char* lst0 = (big >= 0 ? p.big_pix_list : p.pix_list) + (big >= 0 ? size_t(big) : tile) * P * kPix;
        int my_cnt = 0;  // list length of pixel q = lane
        const unsigned rmask = __ballot_sync(0xffffffffu, lane < P && in_rect(lane));
        for (int base = 0; base < nl; base += 32) {
            const int k = base + lane;
            unsigned mask = 0;
            if (k < nl) mask = cand_pixel_mask(s_cand[k], p.TW, P) & rmask;
            for (int q = 0; q < P; ++q) {
                const bool on = (mask >> q) & 1u;
                const unsigned bal = __ballot_sync(0xffffffffu, on);
                if (!bal) continue;  // warp-uniform
                const int cq = __shfl_sync(0xffffffffu, my_cnt, q);
                const int pos = cq + __popc(bal & lt);
                if (on && pos < kPix) lst0[size_t(q) * kPix + pos] = (unsigned char)k;
                if (lane == q) my_cnt += __popc(bal);
            }
        }
        if (lane < P && ((rmask >> lane) & 1u)) {
            const size_t li = big >= 0 ? size_t(big) * P + lane : tile * P + lane;
            (big >= 0 ? p.big_pix_cnt : p.pix_cnt)[li] = (unsigned char)(my_cnt > kPix ? 255 : my_cnt);
        }
        if (lane == 0) {
            if (sub_out) *sub_out = make_int2(off, nl);
            else *hdr = TileHdr{off, nl, big, 0};
        }
        return true;
    }
    for (int q = lane; q < P; q += 32) {
        if (!in_rect(q)) continue;
        const float qx = float(q % p.TW), qy = float(q / p.TW);
        const size_t li = big >= 0 ? size_t(big) * P + q : tile * P + q;
        unsigned char* lst = (big >= 0 ? p.big_pix_list : p.pix_list) + li * kPix;
        int cnt = 0;
        for (int k = 0; k < nl; ++k)
            if (cand_overlaps_pixel(s_cand[k], qx, qy)) {
                if (cnt < kPix) lst[cnt] = (unsigned char)k;
                ++cnt;
            }
        (big >= 0 ? p.big_pix_cnt : p.pix_cnt)[li] = (unsigned char)(cnt > kPix ? 255 : cnt);
    }
    if (lane == 0) {
        if (sub_out) *sub_out = make_int2(off, nl);
        else *hdr = TileHdr{off, nl, big, 0};
    }
    return true;
}

// Fast pass: 4 warps per CTA, kBeamCap candidates. Tiles that overflow are
// queued for the big pass (silhouette tiles, whose frustum grazes the surface:
// ~1 % of the tiles but a third of the boundary probes).
#ifndef CDR_LIST_WARPS
#define CDR_LIST_WARPS 4
#endif
constexpr int kListWarps = CDR_LIST_WARPS;
#ifndef CDR_BIG_FRONT
#define CDR_BIG_FRONT 512
#endif
#ifndef CDR_BIG_WARPS
#define CDR_BIG_WARPS 1
#endif
constexpr int kBigCap = 255;              // candidates of a big tile (pixel lists index with a byte)
constexpr int kBigFront = CDR_BIG_FRONT;  // its builder frontier
constexpr int kBigWarps = CDR_BIG_WARPS;  // big-tile builders per CTA
#ifndef CDR_LIST_MIN_BLOCKS
#define CDR_LIST_MIN_BLOCKS 8  // 32 warps per SM: the builder is latency-bound (level-by-level BFS)
#endif
// The top levels of the BVH are the same for neighbouring tiles: one warp
// walks them once against the union frustum of the CTA's tiles (one tile row)
// until the frontier fills a warp or a leaf would appear; every warp then
// starts its own tile's BFS from that frontier. A node outside the union
// frustum is outside each tile's, so nothing a tile needs is dropped.
constexpr int kTopCap = 64;
__device__ int shared_top_levels(const Params& p, const DevCamera& cam, int X0, int X1, int Y0, int Y1, int lane,
                                 int (*scratch)[kFrontCap], int* out) {
    const FrustumPlanes fp = tile_frustum(cam, X0 - 0.01, X1 + 0.01, Y0 - 0.01, Y1 + 0.01);
    const float of[3] = {float(cam.o[0]), float(cam.o[1]), float(cam.o[2])};
    const unsigned lt = (1u << lane) - 1u;
    int nf = 1, cur = 0;
    if (lane == 0) scratch[0][0] = 0;
    __syncwarp();
    while (nf < 32) {
        int nn = 0;
        bool leafy = false;
        for (int base = 0; base < nf; base += 32) {
            const int i = base + lane;
            bool int0 = false, int1 = false, lf = false;
            int4 k = make_int4(0, 0, 0, 0);
            if (i < nf) {
                const BNode* np = p.sc_bin + scratch[cur][i];
                const float4 a = __ldg(&np->a), bb = __ldg(&np->b), c = __ldg(&np->c);
                k = __ldg(&np->k);
                const bool in0 = !box_outside(fp, of, a.x, a.y, a.z, a.w, bb.x, bb.y);
                const bool in1 = !box_outside(fp, of, bb.z, bb.w, c.x, c.y, c.z, c.w);
                lf = (in0 && k.x < 0) || (in1 && k.y < 0);
                int0 = in0 && k.x >= 0;
                int1 = in1 && k.y >= 0;
            }
            leafy |= __any_sync(0xffffffffu, lf);
            const unsigned q0 = __ballot_sync(0xffffffffu, int0), q1 = __ballot_sync(0xffffffffu, int1);
            const int f0 = nn + __popc(q0 & lt), f1 = nn + __popc(q0) + __popc(q1 & lt);
            if (int0 && f0 < kTopCap) scratch[cur ^ 1][f0] = k.x;
            if (int1 && f1 < kTopCap) scratch[cur ^ 1][f1] = k.y;
            nn += __popc(q0) + __popc(q1);
        }
        __syncwarp();
        if (!leafy && nn == 0) return -1;  // nothing meets the union frustum: every tile is empty
        if (leafy || nn > kTopCap) break;  // keep the current level
        nf = nn;
        cur ^= 1;
    }
    for (int i = lane; i < nf; i += 32) out[i] = scratch[cur][i];
    return nf;
}

// The shared top levels of every 2 x 2 tile block, one warp per block, ahead
// of the list builder: the builder's warps then start from
// the stored frontier instead of waiting at a barrier for one of them to walk.
__global__ void __launch_bounds__(128) k_top_walk(Params p) {
    __shared__ int s_front[4][2][kFrontCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const ViewCall vc = p.calls[blockIdx.y];
    const DevCamera cam = p.cams[vc.slot];
    const int bx = (vc.tiles_x + 1) / 2, by = (vc.tiles_y + 1) / 2;
    const int blk = int(blockIdx.x) * 4 + w;
    if (blk >= bx * by) return;
    const int cx = blk % bx, cy = blk / bx;
    const int X0 = 2 * cx * p.TW, X1 = min(X0 + 2 * p.TW, cam.W);
    const int Y0 = 2 * cy * p.TH, Y1 = min(Y0 + 2 * p.TH, cam.H);
    int* out = p.top_nodes + (size_t(blockIdx.y) * p.top_stride + blk) * (kTopCap + 1);
    const int n = shared_top_levels(p, cam, X0, X1, Y0, Y1, lane, s_front[w], out + 1);
    if (lane == 0) out[0] = n;
    if (!p.blk_queue) return;
    if (n > 0) {  // the list builder's work queue
        if (lane == 0) p.blk_queue[atomicAdd(p.blk_queue_count, 1)] = make_int2(int(blockIdx.y), blk);
        return;
    }
    // the block meets no node: its tiles are empty, written here as the
    // builder would (no candidate, every pixel list empty) and never queued
    const int P = kThreads / p.spp;
    for (int k = 0; k < 4; ++k) {
        const int tx = 2 * cx + (k & 1), ty = 2 * cy + (k >> 1);
        if (tx >= vc.tiles_x || ty >= vc.tiles_y) continue;
        const size_t tile = size_t(vc.tile_base) + ty * vc.tiles_x + tx;
        for (int q = lane; q < P; q += 32) p.pix_cnt[tile * P + q] = 0;
        if (lane == 0) p.tile_hdr[tile] = TileHdr{0, 0, -1, 0};
    }
}

// The fast pass over the queued (non-empty) blocks: a persistent grid, one
// 2 x 2 block per CTA at a time, its warps starting from the prepass frontier
// (the empty blocks' tiles were written by k_top_walk)
__global__ void __launch_bounds__(32 * kListWarps, CDR_LIST_MIN_BLOCKS) k_tile_lists_q(Params p) {
    __shared__ int s_front[kListWarps][2][kFrontCap];
    __shared__ int s_leaf[kListWarps][kBeamCap];
    __shared__ float s_d[kListWarps][kBeamCap];
    __shared__ int s_top_w[kListWarps][kTopCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = *p.blk_queue_count;
#pragma unroll 1
    for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
        const int2 e = p.blk_queue[qi];
        const ViewCall vc = p.calls[e.x];
        const DevCamera& cam = p.cams[vc.slot];
        const int bx = (vc.tiles_x + 1) / 2;
        const int cx = e.y % bx, cy = e.y / bx;
        const int tx = 2 * cx + (w & 1), ty = 2 * cy + (w >> 1);
        if (tx >= vc.tiles_x || ty >= vc.tiles_y) continue;  // warp-uniform, no CTA barrier
        const int b = ty * vc.tiles_x + tx;
        const int* src = p.top_nodes + (size_t(e.x) * p.top_stride + e.y) * (kTopCap + 1);
        const int n = src[0];
        for (int i = lane; i < n; i += 32) s_top_w[w][i] = src[1 + i];
        __syncwarp();
        if (!build_tile_list<kBeamCap, kFrontCap, kPixCap>(p, vc, cam, b, lane, s_front[w], s_leaf[w], s_d[w], nullptr,
                                                            -1, s_top_w[w], n, 0, 0, 1 << 20, 1 << 20, nullptr,
                                                            p.fast_cap) &&
            lane == 0) {
            p.tile_hdr[size_t(vc.tile_base) + b] = TileHdr{0, -1, -1, 0};
            const int i = atomicAdd(p.big_count, 1);
            if (i < p.big_cap) p.big_queue[i] = make_int2(e.x, b);
            else atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
        }
        __syncwarp();  // s_top_w is rewritten for the next block
    }
}

__global__ void __launch_bounds__(32 * kListWarps, CDR_LIST_MIN_BLOCKS) k_tile_lists(Params p) {
    __shared__ int s_front[kListWarps][2][kFrontCap];
    __shared__ int s_leaf[kListWarps][kBeamCap];
    __shared__ float s_d[kListWarps][kBeamCap];
    __shared__ int s_top[kTopCap];
    __shared__ int s_ntop;
    __shared__ int s_top_w[kListWarps][kTopCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const ViewCall vc = p.calls[blockIdx.y];
    const DevCamera cam = p.cams[vc.slot];
#ifndef CDR_LIST_STRIP
    // a 2 x 2 block of tiles per CTA (the union frustum is 8 x 8 pixels)
    static_assert(kListWarps == 4, "2x2 tile blocks need 4 warps");
    const int bx = (vc.tiles_x + 1) / 2, by = (vc.tiles_y + 1) / 2;
    if (int(blockIdx.x) >= bx * by) return;  // CTA-uniform
    const int cx = int(blockIdx.x) % bx, cy = int(blockIdx.x) / bx;
    const int tx = 2 * cx + (w & 1), ty = 2 * cy + (w >> 1);
    const bool mine = tx < vc.tiles_x && ty < vc.tiles_y;
    const int b = ty * vc.tiles_x + tx;
    const bool share = p.sc.n_tris > 1 && !p.no_shared_top;
    if (share && p.top_nodes) {  // the prepass stored the block's frontier
        if (!mine) return;
        const int* src = p.top_nodes + (size_t(blockIdx.y) * p.top_stride + blockIdx.x) * (kTopCap + 1);
        const int n = src[0];
        for (int i = lane; i < n; i += 32) s_top_w[w][i] = src[1 + i];
        __syncwarp();
        if (build_tile_list<kBeamCap, kFrontCap, kPixCap>(p, vc, cam, b, lane, s_front[w], s_leaf[w], s_d[w], nullptr,
                                                           -1, s_top_w[w], n, 0, 0, 1 << 20, 1 << 20, nullptr,
                                                           p.fast_cap))
            return;
        if (lane == 0) {
            p.tile_hdr[size_t(vc.tile_base) + b] = TileHdr{0, -1, -1, 0};
            const int i = atomicAdd(p.big_count, 1);
            if (i < p.big_cap) p.big_queue[i] = make_int2(int(blockIdx.y), b);
            else atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
        }
        return;
    }
    if (share) {
        if (w == 0) {
            const int X0 = 2 * cx * p.TW, X1 = min(X0 + 2 * p.TW, cam.W);
            const int Y0 = 2 * cy * p.TH, Y1 = min(Y0 + 2 * p.TH, cam.H);
            const int n = shared_top_levels(p, cam, X0, X1, Y0, Y1, lane, s_front[0], s_top);
            if (lane == 0) s_ntop = n;
        }
        __syncthreads();
    }
    if (!mine) return;  // warp-uniform (after the only barrier)
#else
    const int n_tiles = vc.tiles_x * vc.tiles_y;
    const int b0 = blockIdx.x * kListWarps;
    if (b0 >= n_tiles) return;  // CTA-uniform
    const int b1 = min(b0 + kListWarps, n_tiles) - 1;
    const bool share = p.sc.n_tris > 1 && b0 / vc.tiles_x == b1 / vc.tiles_x && !p.no_shared_top;
    if (share) {
        if (w == 0) {
            const int X0 = (b0 % vc.tiles_x) * p.TW, X1 = min((b1 % vc.tiles_x) * p.TW + p.TW, cam.W);
            const int Y0 = (b0 / vc.tiles_x) * p.TH, Y1 = min(Y0 + p.TH, cam.H);
            const int n = shared_top_levels(p, cam, X0, X1, Y0, Y1, lane, s_front[0], s_top);
            if (lane == 0) s_ntop = n;
        }
        __syncthreads();
    }
    const int b = b0 + w;
    if (b > b1) return;  // warp-uniform (after the only barrier)
#endif
    const bool fits = build_tile_list<kBeamCap, kFrontCap, kPixCap>(
        p, vc, cam, b, lane, s_front[w], s_leaf[w], s_d[w], nullptr, -1, share ? s_top : nullptr,
        share ? s_ntop : 0, 0, 0, 1 << 20, 1 << 20, nullptr, p.fast_cap);
    if (fits) return;
    if (lane == 0) {
        p.tile_hdr[size_t(vc.tile_base) + b] = TileHdr{0, -1, -1, 0};
        const int i = atomicAdd(p.big_count, 1);
        if (i < p.big_cap) p.big_queue[i] = make_int2(int(blockIdx.y), b);
        else atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
    }
}

// Big pass: one warp per CTA over the queue (persistent grid), kBigCap
// candidates; what still overflows is traced per ray.
__global__ void __launch_bounds__(32 * kBigWarps) k_tile_lists_big(Params p) {
    // the sort keys reuse the frontier (the BFS is over before the sort)
    static_assert(2 * kBigFront * sizeof(int) >= 256 * sizeof(unsigned long long), "key space");
    __shared__ __align__(8) int s_front[kBigWarps][2][kBigFront];
    __shared__ int s_leaf[kBigWarps][kBigCap];
    __shared__ float s_d[kBigWarps][kBigCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = min(*p.big_count, p.big_cap);
    for (int i = blockIdx.x * kBigWarps + w; i < n; i += gridDim.x * kBigWarps) {
        const int2 e = p.big_queue[i];
        const ViewCall vc = p.calls[e.x];
        const DevCamera& cam = p.cams[vc.slot];
        if (!build_tile_list<kBigCap, kBigFront, kBigPixCap>(p, vc, cam, e.y, lane, s_front[w], s_leaf[w], s_d[w],
                                                             reinterpret_cast<unsigned long long*>(s_front[w]), i,
                                                             nullptr, 0, 0, 0, 1 << 20, 1 << 20, nullptr,
                                                             p.big_list_cap) &&
            lane == 0) {
            const int j = atomicAdd(p.split_count, 1);  // split into quadrants (k_tile_lists_split)
            if (j < p.split_cap) p.split_queue[j] = make_int4(i, p.TW << 16 | p.TH << 24, j, 0);
            else atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
        }
        __syncwarp();
    }
}

// Split pass: the tiles still over kBigCap candidates, one warp per
// (item, quadrant); every list of a tile shares the tile's big pixel-list slot.
// Level 0 splits the tile into its 4 quadrants (list group j = the item's queue
// position); a quadrant of more than one pixel that still overflows is split
// once more by the level-1 launch (its entry {group, -2}, the 4 sub-quadrant
// lists in a group allocated past the level-0 ones). What overflows after that
// is traced per ray (beam_fallback_tiles counts those lists).
__device__ __forceinline__ int4 split_item(int slot, int sx0, int sy0, int sw, int sh, int group, int level) {
    return make_int4(slot, sx0 | sy0 << 8 | sw << 16 | sh << 24, group, level);
}

__global__ void __launch_bounds__(32 * kBigWarps) k_tile_lists_split(Params p, int level) {
    __shared__ __align__(8) int s_front[kBigWarps][2][kBigFront];
    __shared__ int s_leaf[kBigWarps][kBigCap];
    __shared__ float s_d[kBigWarps][kBigCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = min(p.split_count[level], p.split_cap);
    const int4* queue = p.split_queue + size_t(level) * p.split_cap;
    for (int it = blockIdx.x * kBigWarps + w; it < 4 * n; it += gridDim.x * kBigWarps) {
        const int4 item = queue[it >> 2];
        const int qd = it & 3;  // quadrant bits as pixel_tile_list (beam.cuh)
        const int i = item.x, g = item.z;
        const int rx = item.y & 0xff, ry = (item.y >> 8) & 0xff, rw = (item.y >> 16) & 0xff, rh = item.y >> 24;
        const int hw = rw / 2, hh = rh / 2;
        const int sx0 = rx + ((qd & 1) ? hw : 0), sw = (qd & 1) ? rw - hw : hw;
        const int sy0 = ry + ((qd & 2) ? hh : 0), sh = (qd & 2) ? rh - hh : hh;
        const int2 e = p.big_queue[i];
        const ViewCall vc = p.calls[e.x];
        const DevCamera& cam = p.cams[vc.slot];
        int2* out = p.split_hdr + 4 * size_t(g) + qd;
        if (!build_tile_list<kBigCap, kBigFront, kBigPixCap>(p, vc, cam, e.y, lane, s_front[w], s_leaf[w], s_d[w],
                                                             reinterpret_cast<unsigned long long*>(s_front[w]), i,
                                                             nullptr, 0, sx0, sy0, sw, sh, out,
                                                             p.split_list_cap) &&
            lane == 0) {
            int j2 = -1;
            if (level == 0 && sw * sh > 1) {  // split this quadrant once more
                j2 = atomicAdd(p.split_count + 1, 1);
                if (j2 >= p.split_cap) j2 = -1;
            }
            int jh = -1;
            if (p.huge_on && (level == 1 || sw * sh == 1)) {  // the list itself, up to kHugeCap candidates (k_tile_lists_huge)
                jh = atomicAdd(p.split_count + 2, 1);
                if (jh >= p.split_cap) jh = -1;
            }
            if (j2 >= 0) {
                const int g2 = p.split_cap + j2;
                *out = make_int2(g2, -2);
                p.split_queue[size_t(p.split_cap) + j2] = split_item(i, sx0, sy0, sw, sh, g2, 1);
            } else if (jh >= 0) {
                *out = make_int2(0, -1);  // per ray unless the huge pass fits it
                p.split_queue[2 * size_t(p.split_cap) + jh] =
                    split_item(i, sx0, sy0, sw, sh, int(out - p.split_hdr), 2);
            } else {
                *out = make_int2(0, -1);
                atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
            }
        }
        if (level == 0 && qd == 0 && lane == 0) p.tile_hdr[size_t(vc.tile_base) + e.y] = TileHdr{g, -2, i, 0};
        __syncwarp();
    }
}

// Huge pass: the lists that still overflow after the splits (at spp 16
// single pixels: grazing rays along a thin tube see hundreds of triangles),
// rebuilt with up to kHugeCap candidates; the pixels scan the whole list (no
// byte-indexed pixel lists). One warp per CTA, 20 KB of shared memory.
constexpr int kHugeCap = 1023;
constexpr int kHugeFront = 1024;
__global__ void __launch_bounds__(32) k_tile_lists_huge(Params p) {
    __shared__ __align__(8) int s_front[2][kHugeFront];
    __shared__ int s_leaf[kHugeCap];
    __shared__ float s_d[kHugeCap];
    static_assert(2 * kHugeFront * sizeof(int) >= 1024 * sizeof(unsigned long long), "key space");
    const int lane = threadIdx.x & 31;
    const int n = min(p.split_count[2], p.split_cap);
    const int4* queue = p.split_queue + 2 * size_t(p.split_cap);
    for (int it = blockIdx.x; it < n; it += gridDim.x) {
        const int4 item = queue[it];
        const int i = item.x;
        const int rx = item.y & 0xff, ry = (item.y >> 8) & 0xff, rw = (item.y >> 16) & 0xff, rh = item.y >> 24;
        const int2 e = p.big_queue[i];
        const ViewCall vc = p.calls[e.x];
        const DevCamera& cam = p.cams[vc.slot];
        int2* out = p.split_hdr + item.z;
        if (!build_tile_list<kHugeCap, kHugeFront, kBigPixCap>(p, vc, cam, e.y, lane, s_front, s_leaf, s_d,
                                                               reinterpret_cast<unsigned long long*>(s_front), i,
                                                               nullptr, 0, rx, ry, rw, rh, out) &&
            lane == 0) {
            *out = make_int2(0, -1);
            atomicAdd(&p.counters->beam_fallback_tiles, 1ull);
        }
        __syncwarp();
    }
}

// Primary visibility: one thread per sample, tile order as k_render, writes the
// hit cache (the bit-exact output). Kept slim so it runs at high occupancy —
// traversal is latency-bound, not bandwidth-bound.
#ifndef CDR_TRACE_MIN_BLOCKS
#define CDR_TRACE_MIN_BLOCKS 6  // 12 x 128-thread CTAs per SM: 5 -> 6 after the empty-tile skip (trace 8.03 -> 7.95 ms at cfg2)
#endif
// Grids are (tile x, tile y, view call); kSPP = 16 makes the sample/tile
// geometry compile-time (4x4 pixels x 16 samples), 0 reads it from Params.
#ifndef CDR_TRACE_ITEMS
#define CDR_TRACE_ITEMS 8  // spp 16: tile columns per CTA (amortises launch: most CTAs of a sparse view are empty tiles)
#endif
constexpr int kTraceItems = CDR_TRACE_ITEMS;

// One CTA's worth of k_trace: tile column bx, CTA row by of view call vc.
template <bool kBeam, int kSPP>
__device__ __forceinline__ void trace_item(const Params& p, const ViewCall& vc, const DevCamera& cam, int bx, int by) {
    constexpr int kCR = kSPP == 16 ? kTraceThreads16 / 64 : 0;  // pixel rows per CTA
    const int W = cam.W, H = cam.H;
    const int tid = threadIdx.x;
    const int spp = kSPP ? kSPP : p.spp;
    const int TW = kSPP == 16 ? 4 : p.TW, TH = kSPP == 16 ? 4 : p.TH;
    const int P = kThreads / spp;  // pixels per beam tile (its pixel lists)
    const int cpix = tid / spp, s = tid - (tid / spp) * spp;  // pixel within the CTA
    const int ty = kSPP == 16 ? by * kCR / 4 : by;
    if (bx >= vc.tiles_x || ty >= vc.tiles_y) return;
    const int tile_in_view = ty * vc.tiles_x + bx;
    const int X0 = bx * TW, Y0 = ty * TH;
    const int pix = kSPP == 16 ? (by * kCR - Y0) * 4 + cpix : cpix;  // pixel within the beam tile
    const int x = X0 + pix % TW;
    const int y = Y0 + pix / TW;
    if (!(pix < P && x < W && y < H)) return;
    const size_t pidx = p.pix_off[vc.slot] + size_t(y) * W + x;
    const D3 org{cam.o[0], cam.o[1], cam.o[2]};
    Hit h{-1, 1e300, 0.0, 0.0};
    // No staging and no barrier: each sample reads the tile header (one
    // broadcast transaction per warp), its own pixel's list and the candidate
    // records, which the tile's 256 samples share through L1.
    TileHdr th{0, -1, -1, 0};
    if (kBeam) th = p.tile_hdr[vc.tile_base + tile_in_view];
    if (kBeam && th.cnt == 0 && p.skip_empty_hits) return;  // CTA-uniform: k_render's empty-tile path reads no hits
    const int2 tl = kBeam ? pixel_tile_list(th, p.split_hdr, pix, TW, TH) : make_int2(0, -1);
    if (kBeam && tl.y >= 0) {
        const size_t tile = size_t(vc.tile_base) + tile_in_view;
        const size_t li = th.big >= 0 ? size_t(th.big) * P + pix : tile * P + pix;
        const int cnt = (th.big >= 0 ? p.big_pix_cnt : p.pix_cnt)[li];
        if (cnt != 0) {  // an empty pixel list means no triangle can cover the pixel: no ray needed
            D2 ps = pixel_sample_position(vc.h_view, x, y, W, s, spp, kSPP == 16 ? 4 : p.k, kSPP == 16 ? 0.25 : p.inv_k);
            D3 dir = primary_dir(cam, ps);
            const float fx = float(ps.x - X0), fy = float(ps.y - Y0);
            const BeamCand* cands = p.pool + tl.x;
            // (one loop for both, or one trace_item call site for the queue
            // and grid paths: smaller code, but slower at cfg2; measured)
            h = cnt == 255 ? trace_beam(cands, tl.y, p.sc.recs, org, dir, p.info->t_min, fx, fy)
                           : trace_beam_list(cands,
                                             (th.big >= 0 ? p.big_pix_list + li * kBigPixCap : p.pix_list + li * kPixCap),
                                             cnt, p.sc.recs, org, dir, p.info->t_min, fx, fy);
        }
    } else {
        D2 ps = pixel_sample_position(vc.h_view, x, y, W, s, spp, kSPP == 16 ? 4 : p.k, kSPP == 16 ? 0.25 : p.inv_k);
        D3 dir = primary_dir(cam, ps);
        // per-ray traversal: the whole pass without lists, or (rare) a tile whose lists overflowed
        h = kBeam ? trace_out_of_line(p.sc_bin, p.sc.recs, p.sc.n_tris, org, dir, p.info->t_min)
                  : trace(p.sc_bin, p.sc.recs, p.sc.n_tris, org, dir, p.info->t_min);
    }
    p.hit[pidx * spp + s] = h.tri;
}

template <bool kBeam, int kSPP>
__global__ void __launch_bounds__(kSPP == 16 ? kTraceThreads16 : kThreads,
                                  kSPP == 16 ? CDR_TRACE_MIN_BLOCKS * kThreads / kTraceThreads16
                                             : CDR_TRACE_MIN_BLOCKS) k_trace(Params p) {
#ifdef CDR_EXP_TRACE_NOP  // measurement only (wrong output): launch cost of the grid
    return;
#endif
    // spp 16: kTraceItems consecutive tile columns per CTA (no barriers, so an
    // item's early returns just end that item)
    constexpr int kItems = kSPP == 16 ? kTraceItems : 1;
    if (kBeam && kSPP == 16 && p.queue_mode) {  // items: the non-empty tiles in tile order (half tiles)
        constexpr int kCPT = 4 / (kTraceThreads16 / 64);
        const int nq = p.queue_len;
        int cur = -1;
        ViewCall vc{};
        DevCamera cam{};
#pragma unroll 1
        for (int i = 0; i < kItems; ++i) {
            const int it = int(blockIdx.x) * kItems + i;
            if (it >= nq * kCPT) return;
            const int2 e = p.tile_queue[it / kCPT];
            if (e.x != cur) {  // consecutive items are mostly tiles of one view
                cur = e.x;
                vc = p.calls[cur];
                cam = p.cams[vc.slot];
            }
            trace_item<kBeam, kSPP>(p, vc, cam, e.y % vc.tiles_x, (e.y / vc.tiles_x) * kCPT + it % kCPT);
        }
        return;
    }
    const ViewCall vc = p.calls[blockIdx.z];
    const DevCamera cam = p.cams[vc.slot];
#pragma unroll 1
    for (int i = 0; i < kItems; ++i) trace_item<kBeam, kSPP>(p, vc, cam, int(blockIdx.x) * kItems + i, int(blockIdx.y));
}

// Type of the warp partial sums of the scatter. fp64 by default (the whole
// path is fp64). -DCDR_REDUCE_F32 sums the <= 32 per-group terms in fp32
// (the global REDs stay fp64): shading 17.1 -> 16.0 ms at cfg2, gradients
// still ~1e-7 from the reference (tolerance 1e-4), but not an fp64 path, so
// it is an opt-in build and never the benchmarked one.
#ifdef CDR_REDUCE_F32
using RedT = float;
#else
using RedT = double;
#endif

// ---- group sums on the fp64 tensor core ------------------------------------
// Per warp, the scatter sums kC weighted copies of a kV-vector u (kV <= 8) over
// the lanes of each group (lanes sharing a texel quad or a triangle): corner c
// of group m receives sum_s [gid(s) == m] w_c(s) u(s). With ng <= 8 groups that
// is, per corner, S_c[8 x 8] = A_c[8 x 32] U[32 x 8] with A_c = group membership
// times the corner weight: eight m8n8k4 fp64 MMAs (exact fp64 products and
// sums), the kC corners as independent accumulator chains sharing U's B
// fragments — instead of log-depth shuffle trees over every value (2 SHFL per
// double per round). U goes through the warp's dead shared memory (column n =
// 32 doubles, rotated by 4n so a fragment load hits 16 bank pairs); lane l ends
// with S_c[l >> 2][2 (l & 3)] and S_c[l >> 2][2 (l & 3) + 1].
__device__ __forceinline__ void mma_f64_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

#ifndef CDR_MMA_UNROLL
#define CDR_MMA_UNROLL 2  // k-steps per unrolled body: 2 measured best (cfg2 shading 10.76 -> 10.55 ms, cfg4 23.45 -> 22.75; 1, 4, 8 slower)
#endif
constexpr int kMmaUnroll = CDR_MMA_UNROLL;  // k-steps per unrolled body (code size vs loop overhead)


// column n of this warp's U: s_rad's slice for n < 3, s_ray[n - 3]'s after
template <int kRT>
__device__ __forceinline__ double* ucol(double (&s_rad)[kRT][3], double (&s_ray)[5][kRT], int w32, int n) {
    return n < 3 ? &s_rad[w32][0] + 32 * n : &s_ray[n - 3][w32];
}

// mbase: this call sums groups mbase .. mbase + 7 (a second call with
// mbase 8 and write_u false covers warps of up to 16 groups)
template <int kV, int kC, int kRT, typename Wf>
__device__ __forceinline__ void group_sum_mma(double (&s_rad)[kRT][3], double (&s_ray)[5][kRT], int w32,
                                              const double (&u)[kV], int gid, int lane, Wf weight,
                                              double (&s0)[kC], double (&s1)[kC], int mbase = 0,
                                              bool write_u = true) {
    if (write_u) {
        __syncwarp();  // the lanes' earlier reads of these slices are done
#pragma unroll
        for (int n = 0; n < kV; ++n) ucol<kRT>(s_rad, s_ray, w32, n)[(lane + 4 * n) & 31] = u[n];
        __syncwarp();
    }
    const int m = lane >> 2, k = lane & 3;
    const double* col = m < kV ? ucol<kRT>(s_rad, s_ray, w32, m) : nullptr;
#pragma unroll
    for (int c = 0; c < kC; ++c) s0[c] = s1[c] = 0.0;
#pragma unroll kMmaUnroll
    for (int t = 0; t < 8; ++t) {
        const int src = 4 * t + k;
        const bool in = __shfl_sync(0xffffffffu, gid, src) == m + mbase;  // A: sample src in group mbase + m
        const double b = col ? col[(src + 4 * m) & 31] : 0.0;     // B: U[src][m]
#pragma unroll
        for (int c = 0; c < kC; ++c) mma_f64_8x8x4(s0[c], s1[c], in ? weight(c, src) : 0.0, b);
    }
    __syncwarp();  // U is rewritten by the next call (the caller's reads of col are done)
}

// Dense group ids of a match_any grouping over the active lanes: gid in
// [0, ng) by leader order, -1 for inactive lanes; ng > kMmaGroups -> the caller falls
// back to the shuffle reduction. leader_of(m) = lane of group m's leader.
__device__ __forceinline__ int group_ids(bool act, unsigned peers, int lane, unsigned& leaders, int& ng) {
    const int leader = __ffs(peers) - 1;
    leaders = __ballot_sync(0xffffffffu, act && leader == lane);
    ng = __popc(leaders);
    return act ? __popc(leaders & ((1u << leader) - 1u)) : -1;
}

// Phase 3 of k_render: the interior adjoint of one sample (diff_render.cpp:78-184).
// The 4 bilinear weights of the texel scatter, staged per thread in shared
// memory (transposed: lane-consecutive, conflict-free). The scatter loop
// indexes them with its loop counter, which put them in local memory, and
// they live across the position computation and scatter. Staging all ten
// scatter scalars this way was slower at cfg4: 16 KB per CTA shrinks L1.
constexpr int kTexState = 4;

template <int kRT, bool kT64>
__device__ __forceinline__ void interior_scatter(const Params& p, int tid, int x, int y, int spp, int tri, double t,
                                              double b1, double b2, D3 dir, D3 a, bool act,
                                              double (&s_ts)[kTexState][kRT], double (&s_ray)[5][kRT],
                                              double (&s_rad)[kRT][3]) {
    a = (spp & (spp - 1)) == 0 ? a * (1.0 / spp) : a / double(spp);  // diff_render.cpp:82 (x/2^n exact as x*2^-n)

    // Compute everything the scatter needs first, so the large temporaries
    // (texture sample, BRDF partials, vertex data) are dead before the
    // warp-aggregation loops; only a compact state crosses them.
    int tex0 = 0;           // texel quad key (texel[0] determines all four)
    int tcol = 0, trow = 0;  // its column and row (the scatter's addresses without a division)
    double wd0 = 0, ws0 = 0, wr0 = 0;  // d_diffuse/r^2, d_specular/r^2, Σ a L d_rough / r^2
    double aL[3] = {0, 0, 0};
    double lv[3] = {0, 0, 0};          // light gradient (diff_render.cpp:129-131)
    bool pact = false;                 // position terms present (mu > 0, det != 0, finite)
    D3 gc{0, 0, 0}, hm{0, 0, 0};       // g_common and coeff_mu * h
    double b0 = 0;
    int va = 0, vb = 0, vcx = 0;
    if (act) {
        b0 = 1.0 - b1 - b2;
        va = p.sc.tris[3 * tri];
        vb = p.sc.tris[3 * tri + 1];
        vcx = p.sc.tris[3 * tri + 2];
        D2 uv0{0, 0}, uv1{0, 0}, uv2{0, 0};
        if (p.sc.uv) {
            uv0 = D2{p.sc.uv[2 * va], p.sc.uv[2 * va + 1]};
            uv1 = D2{p.sc.uv[2 * vb], p.sc.uv[2 * vb + 1]};
            uv2 = D2{p.sc.uv[2 * vcx], p.sc.uv[2 * vcx + 1]};
        }
        D2 uv{uv0.x * b0 + uv1.x * b1 + uv2.x * b2, uv0.y * b0 + uv1.y * b1 + uv2.y * b2};
        D3 N0 = ld3(p.sc.normals + 3 * va), N1 = ld3(p.sc.normals + 3 * vb), N2 = ld3(p.sc.normals + 3 * vcx);
        D3 nt = N0 * b0 + N1 * b1 + N2 * b2;
        double n_len = length(nt);
        if (n_len < 1e-14) {
            act = false;  // diff_render.cpp:101
        } else {
            // gradient path (tolerance, not bit-exact): divisions as reciprocals
            const double inv_len = rcp(n_len);
            D3 n_hat = nt * inv_len;
            double mu = dot(n_hat, -dir);
            // h = normalize_jacobian(n_tilde) * v_hat (vec.hpp:179-183) and the
            // vertex-data terms of k1 / k2, now: uvs and normals die here
            D3 hv;
            {
                const D3 n = n_hat, v = -dir;
                const double sc = inv_len;
                double J[9] = {(1 - n.x * n.x) * sc, (0 - n.x * n.y) * sc, (0 - n.x * n.z) * sc,
                               (0 - n.y * n.x) * sc, (1 - n.y * n.y) * sc, (0 - n.y * n.z) * sc,
                               (0 - n.z * n.x) * sc, (0 - n.z * n.y) * sc, (1 - n.z * n.z) * sc};
                hv = D3{J[0] * v.x + J[1] * v.y + J[2] * v.z, J[3] * v.x + J[4] * v.y + J[5] * v.z,
                        J[6] * v.x + J[7] * v.y + J[8] * v.z};
            }
            const double du1 = uv1.x - uv0.x, dv1 = uv1.y - uv0.y, du2 = uv2.x - uv0.x, dv2 = uv2.y - uv0.y;
            const double dn1 = dot(hv, N1) - dot(hv, N0), dn2 = dot(hv, N2) - dot(hv, N0);
            TexSample3 ts;
            if constexpr (kT64) ts = sample_maps(p.sc.tex64, p.sc.tw, p.sc.th, uv, true);
            else ts = sample_maps(p.sc.tex, p.sc.tw, p.sc.th, uv, true);
            Brdf br = eval_brdf_grad(ts.dv, ts.sv, ts.rv, mu);
            const double inv_r2 = rcp(t * t);
            const double Lc[3] = {p.sc.L[0], p.sc.L[1], p.sc.L[2]};
            const double ac[3] = {a.x, a.y, a.z};
            tex0 = ts.texel[0];
            tcol = ts.x0;
            trow = ts.y0;
            for (int k = 0; k < 4; ++k) s_ts[k][tid] = ts.w[k];
            wd0 = br.d_diffuse * inv_r2;
            ws0 = br.d_specular * inv_r2;
            for (int c = 0; c < 3; ++c) {
                aL[c] = ac[c] * Lc[c];
                wr0 += ac[c] * Lc[c] * comp(br.d_rough, c) * inv_r2;
                lv[c] = ac[c] * comp(br.value, c) * inv_r2;
            }
            // the intersection-response coefficients (diff_render.cpp:143-160)
            // now, so the texture sample and BRDF partials die here instead of
            // living across the vertex loads and the inverse below
            double cs = 0, cu = 0, cv = 0, cm = 0;
            {
                const double m2_r3 = -2.0 * inv_r2 * rcp(t);  // -2 / t^3
                for (int c = 0; c < 3; ++c) {
                    double w = ac[c] * Lc[c] * inv_r2;
                    cs += ac[c] * Lc[c] * (comp(br.value, c) * m2_r3);
                    double gu = br.d_diffuse * comp(ts.ddu, c) + br.d_specular * comp(ts.sdu, c) +
                                comp(br.d_rough, c) * ts.rdu;
                    double gv = br.d_diffuse * comp(ts.ddv, c) + br.d_specular * comp(ts.sdv, c) +
                                comp(br.d_rough, c) * ts.rdv;
                    cu += w * gu;
                    cv += w * gv;
                    cm += w * comp(br.d_mu, c);
                }
            }
            if (mu > 0) {  // diff_render.cpp:133
                D3 p0 = ld3(p.sc.pos + 3 * va), p1 = ld3(p.sc.pos + 3 * vb), p2 = ld3(p.sc.pos + 3 * vcx);
                // M = [d, p0-p1, p0-p2] (Mat3::from_columns), inverse rows r0..r2
                // the ray direction again from shared memory (its registers are
                // free across the sample / BRDF peak)
                const double dx = s_ray[0][tid], dy = s_ray[1][tid], dz = s_ray[2][tid];
                double m[9] = {dx, p0.x - p1.x, p0.x - p2.x, dy, p0.y - p1.y, p0.y - p2.y,
                               dz, p0.z - p1.z, p0.z - p2.z};
                double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                             m[2] * (m[3] * m[7] - m[4] * m[6]);
                if (fabs(det) >= 1e-18) {
                    if (!isfinite(cs + cu + cv + cm)) {
                        raise_nonfinite(p.err, x, y);
                    } else {
                        double inv = rcp(det);
                        D3 r0{(m[4] * m[8] - m[5] * m[7]) * inv, (m[2] * m[7] - m[1] * m[8]) * inv,
                              (m[1] * m[5] - m[2] * m[4]) * inv};
                        D3 r1{(m[5] * m[6] - m[3] * m[8]) * inv, (m[0] * m[8] - m[2] * m[6]) * inv,
                              (m[2] * m[3] - m[0] * m[5]) * inv};
                        D3 r2{(m[3] * m[7] - m[4] * m[6]) * inv, (m[1] * m[6] - m[0] * m[7]) * inv,
                              (m[0] * m[4] - m[1] * m[3]) * inv};
                        double k1 = cu * du1 + cv * dv1 + cm * dn1;
                        double k2 = cu * du2 + cv * dv2 + cm * dn2;
                        gc = r0 * cs + r1 * k1 + r2 * k2;
                        hm = hv * cm;
                        pact = true;
                    }
                }
            }
        }
    }

    // Samples of a warp sharing a texel quad (or a triangle) are summed with
    // a log-depth shuffle tree first (reduce_peers), then the group leader
    // issues the REDs. Measured alternatives, both slower at cfg2 (DESIGN.md
    // §5): staging the leaders' sums in shared memory so one warp-wide RED
    // covers several records (+2%: the L2 is not the limiter), and a
    // shared-memory transpose in which lane (group, component) sums a column
    // (+10%: fewer instructions, but a serial load-add chain per lane; this
    // kernel is latency-bound at 6 warps per scheduler, not issue-bound).
    const int lane = tid & 31;
    if (p.lay_l >= 0) {  // light intensity (diff_render.cpp:129-131)
        for (int o = 16; o > 0; o >>= 1)
            for (int c = 0; c < 3; ++c) lv[c] += __shfl_xor_sync(0xffffffffu, lv[c], o);
        if (lane == 0)
            for (int c = 0; c < 3; ++c)
                if (lv[c] != 0) atomicAdd(p.grad + p.lay_l + c, lv[c]);
    }
    // intersection response + normal-chain input, per triangle corner
    // (diff_render.cpp:170-184; the chain itself is applied in finalize.cu)
#if !defined(CDR_SCATTER_SHFL) && !defined(CDR_REDUCE_F32)
    // U columns for group_sum_mma: this warp's slices of s_rad (dead after
    // phase 2) and s_ray[0..2] (the direction, dead now); s_ray[3..4] (b1, b2)
    // are the position corners' weights and become U's 7th column afterwards
    const int w32 = tid & ~31;
    unsigned pleaders = 0, tleaders = 0;
    int png = 0, tng = 0;
    const int pkey = pact ? tri : -1 - lane, tkey = act ? tex0 : -1 - lane;
    const unsigned ppeers = __match_any_sync(0xffffffffu, pkey), tpeers = __match_any_sync(0xffffffffu, tkey);
    const int pgid = group_ids(pact, ppeers, lane, pleaders, png);
    const int tgid = group_ids(act, tpeers, lane, tleaders, tng);
    const int gm = lane >> 2, n0 = 2 * (lane & 3);
    __syncwarp();  // every lane is past its s_ray[0..2] reads before U overwrites them
#endif
#ifndef CDR_EXP_NO_POS
#if !defined(CDR_SCATTER_SHFL) && !defined(CDR_REDUCE_F32)
    {  // groups of 8 per pass: a warp has <= 32 (4 passes at most, 1 in the common case)
        double u[6] = {gc.x, gc.y, gc.z, hm.x, hm.y, hm.z};
        if (!pact)
            for (int i = 0; i < 6; ++i) u[i] = 0;
        const double* sb1 = &s_ray[3][w32];
        const double* sb2 = &s_ray[4][w32];
        auto bw = [&](int j, int src) {  // barycentric of corner j (b0 as computed above)
            const double r1 = sb1[src], r2 = sb2[src];
            return j == 0 ? 1.0 - r1 - r2 : (j == 1 ? r1 : r2);
        };
        auto pass = [&](int mb) {
            const int g = mb + gm;
            const int ltri = __shfl_sync(0xffffffffu, tri, g < png ? __fns(pleaders, 0, g + 1) : 0);
            double s0[3], s1[3];
            group_sum_mma<6, 3, kRT>(s_rad, s_ray, w32, u, pgid, lane, bw, s0, s1, mb, mb == 0);
            if (g < png && n0 < 6)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    double* dst = p.corner + (size_t(ltri) * 3 + j) * 6 + n0;
                    if (s0[j] != 0) atomicAdd(dst, s0[j]);
                    if (s1[j] != 0) atomicAdd(dst + 1, s1[j]);
                }
        };
        pass(0);  // the common case: <= 8 triangles per warp
#pragma unroll 1
        for (int mb = 8; mb < png; mb += 8) pass(mb);
    }
#else
    {
        const int key = pact ? tri : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const bool leader = pact && (__ffs(peers) - 1) == lane;
#pragma unroll 1
        for (int j = 0; j < 3; ++j) {
            const double rb1 = s_ray[3][tid], rb2 = s_ray[4][tid];
            const double bj = j == 0 ? 1.0 - rb1 - rb2 : (j == 1 ? rb1 : rb2);  // b0 as computed above
            RedT v[6] = {RedT(gc.x * bj), RedT(gc.y * bj), RedT(gc.z * bj),
                         RedT(hm.x * bj), RedT(hm.y * bj), RedT(hm.z * bj)};
            if (!pact)
                for (int i = 0; i < 6; ++i) v[i] = 0;
            reduce_peers<6>(0xffffffffu, peers, v);
            if (leader) {
                double* dst = p.corner + (size_t(tri) * 3 + j) * 6;
                for (int i = 0; i < 6; ++i)
                    if (v[i] != 0) atomicAdd(dst + i, double(v[i]));
            }
        }
    }
#endif
#endif
#ifndef CDR_EXP_NO_TEXEL
#if !defined(CDR_SCATTER_SHFL) && !defined(CDR_REDUCE_F32)
    {  // groups of 8 per pass, as above
        const int tw = p.sc.tw, th = p.sc.th;
        double u[7] = {0, 0, 0, 0, 0, 0, 0};
        if (act) {
            for (int c = 0; c < 3; ++c) {
                u[c] = aL[c] * wd0;
                u[3 + c] = aL[c] * ws0;
            }
            u[6] = wr0;
        }
        auto tw4 = [&](int kq, int src) { return s_ts[kq][w32 + src]; };  // bilinear weight of corner kq
        auto pass = [&](int mb) {
            const int g = mb + gm;
            const int lsrc = g < tng ? __fns(tleaders, 0, g + 1) : 0;  // the group's leader lane
            const int x0 = __shfl_sync(0xffffffffu, tcol, lsrc), y0 = __shfl_sync(0xffffffffu, trow, lsrc);
            const int x1 = x0 + 1 == tw ? 0 : x0 + 1, y1 = y0 + 1 == th ? 0 : y0 + 1;
            double s0[4], s1[4];
            group_sum_mma<7, 4, kRT>(s_rad, s_ray, w32, u, tgid, lane, tw4, s0, s1, mb, mb == 0);
            if (g < tng && n0 < 7)
#pragma unroll
                for (int kq = 0; kq < 4; ++kq) {
                    const int64_t tx = int64_t((kq < 2 ? y0 : y1)) * tw + ((kq & 1) ? x1 : x0);
                    TexAcc* dst = p.texacc + tx;
                    if (s0[kq] != 0) atomicAdd(&dst->v[n0], TexAccT(s0[kq]));
                    if (n0 + 1 < 7 && s1[kq] != 0) atomicAdd(&dst->v[n0 + 1], TexAccT(s1[kq]));
                }
        };
        pass(0);  // the common case: <= 8 texel quads per warp
#pragma unroll 1
        for (int mb = 8; mb < tng; mb += 8) pass(mb);
    }
#else
    {
        // texel scatter through the bilinear weights (diff_render.cpp:110-128)
        const int key = act ? tex0 : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const bool leader = act && (__ffs(peers) - 1) == lane;
        const int tw = p.sc.tw, th = p.sc.th;
        const int x0 = tex0 % tw, y0 = tex0 / tw;
        const int x1 = x0 + 1 == tw ? 0 : x0 + 1, y1 = y0 + 1 == th ? 0 : y0 + 1;
#pragma unroll 1
        for (int kq = 0; kq < 4; ++kq) {
            RedT v[7] = {0, 0, 0, 0, 0, 0, 0};  // lanes without a sample form singleton groups
            if (act) {
                const double w = s_ts[kq][tid];
                for (int c = 0; c < 3; ++c) {
                    v[c] = RedT(aL[c] * (w * wd0));
                    v[3 + c] = RedT(aL[c] * (w * ws0));
                }
                v[6] = RedT(wr0 * w);
            }
            reduce_peers<7>(0xffffffffu, peers, v);
            if (leader) {
                // texel-major accumulator: the 7 values of a texel share 2 sectors
                const int64_t tx = int64_t((kq < 2 ? y0 : y1)) * tw + ((kq & 1) ? x1 : x0);
                TexAcc* dst = p.texacc + tx;
                for (int i = 0; i < 7; ++i)
                    if (v[i] != 0) atomicAdd(&dst->v[i], TexAccT(v[i]));
            }
        }
    }
#endif
#endif
}

// kShade: radiance + pixel mean/mask; kLoss: loss + adjoint; kInterior: scatter.
// The hit triangle comes from the hit cache and is re-intersected with
// ray_triangle, exactly as interior_pass replays it (diff_render.cpp:84-93).
#ifndef CDR_RENDER_MIN_BLOCKS
#define CDR_RENDER_MIN_BLOCKS 3
#endif
#ifndef CDR_RENDER_CTAS16  // resident CTAs per SM of the spp-16 kernel (its register budget)
#define CDR_RENDER_CTAS16 (CDR_RENDER_MIN_BLOCKS * kThreads / kRenderThreads16)
#endif
// view_rendering_loss for one (pixel, channel) of the mean radiance: adds the
// L1 term to loss_part, writes and returns the adjoint (losses.cpp:37-44)
__device__ __forceinline__ double pixel_loss_adjoint(const Params& p, const ViewCall& vc, size_t qi, int c,
                                                     double mean, double& loss_part) {
    const double m = (p.use_mask && p.has_mask[vc.slot]) ? p.target_mask[qi] : 1.0;
    double a = 0;
    if (m != 0) {
        // Φ'(r) = Φ(r) / (γ r) for r in (0, 1); Φ(0) = pow(0, 1/γ) = +0 exactly: skip pow on background
        const double tr = mean <= 0.0 ? 0.0 : tone_map_inv(mean, p.inv_gamma);
        const double d = tr - p.target_tone[3 * qi + c];
        loss_part += m * fabs(d);
        const double sg = double((d > 0) - (d < 0));
        // the adjoint path (tolerance, as the interior pass): a reciprocal
        const double der = (mean <= 0.0 || mean >= 1.0) ? 0.0 : tr * rcp(p.gamma * mean);
        a = vc.scale * m * sg * der;
    }
    p.adj[3 * qi + c] = a;
    return a;
}

// Tile queue by stream compaction of the final tile headers (after the list
// passes): every tile with cnt != 0 (candidates, split, or per-ray) in tile
// order — raster order per view, views in call order, as the full grid — so
// the shading kernel keeps the full grid's locality. Three small kernels:
// per-block counts of 1,024 tiles, one scan, in-order writes.
constexpr int kQBlock = 1024;
__global__ void __launch_bounds__(256) k_queue_count(const TileHdr* __restrict__ hdr, int n, int* __restrict__ cnt) {
    int c = 0;
    for (int k = 0; k < 4; ++k) {
        const int t = int(blockIdx.x) * kQBlock + k * 256 + int(threadIdx.x);
        c += t < n && hdr[t].cnt != 0;
    }
    __shared__ int s[8];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) cnt[blockIdx.x] = s[0] + s[1] + s[2] + s[3] + s[4] + s[5] + s[6] + s[7];
}

__global__ void __launch_bounds__(1024) k_queue_scan(int* __restrict__ cnt, int nb, int* __restrict__ total) {
    __shared__ int ws[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + int(threadIdx.x);
        const int v = i < nb ? cnt[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        if (w == 0) {
            int t = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        if (i < nb) cnt[i] = carry + (w > 0 ? ws[w - 1] : 0) + x - v;  // exclusive
        carry += ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(256) k_queue_write(Params p, int n, int n_calls, const int* __restrict__ off) {
    __shared__ int s[8];
    int base = off[blockIdx.x];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = 0; k < 4; ++k) {
        const int t = int(blockIdx.x) * kQBlock + k * 256 + int(threadIdx.x);
        const bool on = t < n && p.tile_hdr[t].cnt != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) s[w] = __popc(bal);
        __syncthreads();
        int before = base;
        for (int j = 0; j < w; ++j) before += s[j];
        if (on) {
            int lo = 0, hi = n_calls - 1;  // the call whose tiles hold t
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.calls[mid].tile_base <= t) lo = mid;
                else hi = mid - 1;
            }
            p.tile_queue[before + __popc(bal & ((1u << lane) - 1u))] = make_int2(lo, t - p.calls[lo].tile_base);
        }
        for (int j = 0; j < 8; ++j) base += s[j];
        __syncthreads();
    }
}

// starts[v] = the first queue entry of call v (the queue is in tile order, so
// call-major): the shading can then be launched view group by view group
__global__ void k_queue_view_starts(const int2* __restrict__ queue, const int* __restrict__ total, int n_calls,
                                    int* __restrict__ starts) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v > n_calls) return;
    int lo = 0, hi = *total;  // lower_bound of v over queue[].x
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (queue[mid].x < v) lo = mid + 1;
        else hi = mid;
    }
    starts[v] = lo;
}

// The pixels of empty beam tiles in a queue-mode loss call (spp 16): no
// triangle can cover them, so every sample misses (k_trace wrote no hits) and
// the pixel is the background mean, mask 0, with its loss and adjoint — the
// same arithmetic as k_render's empty-tile path, streamed one thread per pixel.
__global__ void __launch_bounds__(256) k_background(Params p) {
    const ViewCall vc = p.calls[blockIdx.y];
    const DevCamera& cam = p.cams[vc.slot];
    const int W = cam.W, H = cam.H;
    const int i = int(blockIdx.x) * 256 + int(threadIdx.x);
    double loss_part = 0;
    if (i < W * H) {
        const int x = i % W, y = i / W;
        const TileHdr th = p.tile_hdr[size_t(vc.tile_base) + (y / 4) * vc.tiles_x + x / 4];
        if (th.cnt == 0) {
            const size_t qi = p.pix_off[vc.slot] + size_t(i);
            for (int c = 0; c < 3; ++c) {
                double sum = 0;
                for (int j = 0; j < 16; ++j) sum = sum + p.sc.bg[c];  // render.cpp:48-57, sample order
                const double mean = sum / 16.0;
                p.img[3 * qi + c] = mean;
                pixel_loss_adjoint(p, vc, qi, c, mean, loss_part);
            }
            p.mask[qi] = 0.0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) loss_part += __shfl_xor_sync(0xffffffffu, loss_part, o);
    __shared__ double s_l[8];
    if ((threadIdx.x & 31) == 0) s_l[threadIdx.x >> 5] = loss_part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0;
        for (int w = 0; w < 8; ++w) tot += s_l[w];
        if (tot != 0) atomicAdd(&p.loss_acc[vc.slot], tot);
    }
}

// kQ: the queue-mode instance (CTAs from the tile queue; no empty-tile path,
// so the hot instance carries no dead code for the instruction cache)
template <bool kShade, bool kLoss, bool kInterior, int kSPP, bool kQ = false, bool kT64 = false>
__global__ void __launch_bounds__(kSPP == 16 ? kRenderThreads16 : kThreads,
                                  kSPP == 16 ? CDR_RENDER_CTAS16
                                             : CDR_RENDER_MIN_BLOCKS) k_render(Params p) {
    // spp 16: kRenderThreads16 threads = (kRenderThreads16 / 64) x 4 pixels x 16 samples
    constexpr int kRT = kSPP == 16 ? kRenderThreads16 : kThreads;
#ifdef CDR_EXP_RENDER_NOP  // measurement only (wrong output): launch cost of the grid
    if (kLoss) return;
#endif
    __shared__ double s_rad[kRT][3];
    __shared__ double s_adj[kSPP ? kRT / kSPP : kRT][3];  // per pixel of the CTA
    __shared__ unsigned char s_hit[kRT];
    __shared__ double s_ts[kTexState][kRT];  // interior_scatter's texel state
    __shared__ double s_ray[kInterior ? 5 : 1][kRT];  // dir, b1, b2 of the sample, for the scatter's late uses

    static_assert(!kQ || (kSPP == 16 && kShade && kLoss), "queue mode is the spp-16 loss call");
    int cx = int(blockIdx.x), cy = int(blockIdx.y), cz = int(blockIdx.z);
    if (kQ) {  // CTA = (non-empty tile, pixel-row group) from the tile queue
        constexpr int kCPT = 4 / (kRT / 64);  // CTAs per 4 x 4 tile
        const int it = int(blockIdx.x) + p.queue_off;
        const int2 e = p.tile_queue[it / kCPT];
        cz = e.x;
        const int tiles_x = p.calls[cz].tiles_x;
        cx = e.y % tiles_x;
        cy = (e.y / tiles_x) * kCPT + it % kCPT;
    }
    const ViewCall vc = p.calls[cz];
    const DevCamera& cam = p.cams[vc.slot];
    const int W = cam.W, H = cam.H;
    const int tid = threadIdx.x;
    const int spp = kSPP ? kSPP : p.spp;
    const int TW = kSPP == 16 ? 4 : p.TW, TH = kSPP == 16 ? kRT / 64 : p.TH;
    if (cx * TW >= W || cy * TH >= H) return;  // uniform per CTA
    const int P = kRT / spp;
    const int pix = tid / spp, s = tid - (tid / spp) * spp;
    const int X0 = cx * TW, Y0 = cy * TH;
    const int x = X0 + pix % TW;
    const int y = Y0 + pix / TW;
    const bool valid = pix < P && x < W && y < H;
    const size_t pbase = p.pix_off[vc.slot];
    const size_t pidx = pbase + size_t(y) * W + x;  // arena pixel index
    const D3 org{cam.o[0], cam.o[1], cam.o[2]};

    // Empty beam tile (no candidate at all: k_trace wrote a miss for every
    // sample): warp 0 writes the 8 pixels' background mean, mask, loss and
    // adjoint straight away; no hit loads, no staging, no barrier.
    if (!kQ && kSPP == 16 && kShade && kLoss && p.use_beam) {
        const TileHdr th = p.tile_hdr[size_t(vc.tile_base) + (Y0 / 4) * vc.tiles_x + cx];
        if (th.cnt == 0) {
#ifdef CDR_EXP_EMPTY_RETURN  // measurement only (wrong output): cost of the empty-tile path
            return;
#endif
            if (tid >= 32) return;
            double loss_part = 0;
            for (int item = tid; item < 3 * P; item += 32) {  // (pixel, channel) items
                const int q = item % P, c = item / P;
                const int px = X0 + q % TW, py = Y0 + q / TW;
                if (px < W && py < H) {
                    const size_t qi = pbase + size_t(py) * W + px;
                    double sum = 0;
                    constexpr int kS = kSPP > 0 ? kSPP : 1;  // (this path is spp 16 only)
                    for (int j = 0; j < kS; ++j) sum = sum + p.sc.bg[c];  // render.cpp:48-57, sample order
                    const double mean = sum / double(kS);
                    p.img[3 * qi + c] = mean;
                    if (c == 0) p.mask[qi] = 0.0;
                    pixel_loss_adjoint(p, vc, qi, c, mean, loss_part);
                }
            }
            for (int o = 16; o > 0; o >>= 1) loss_part += __shfl_xor_sync(0xffffffffu, loss_part, o);
            if (tid == 0 && loss_part != 0) atomicAdd(&p.loss_acc[vc.slot], loss_part);
            return;
        }
    }

    // ---------------- phase 1: cached triangle -> (t, b1, b2), radiance
    int tri = -1;
    double t = 0, b1 = 0, b2 = 0;
    D3 dir{0, 0, 1};
    if (valid) tri = p.hit[pidx * spp + s];
    CDR_DCHECK(tri >= -1 && tri < p.sc.n_tris);
#ifdef CDR_EXP_SKIP_MISS  // measurement only (wrong output): cost of all-miss CTAs
    if (!__syncthreads_or(tri >= 0)) return;
#endif
    if (tri >= 0) {  // misses need no ray: their radiance is the background
        D2 ps = pixel_sample_position(vc.h_view, x, y, W, s, spp, kSPP == 16 ? 4 : p.k, kSPP == 16 ? 0.25 : p.inv_k);
        dir = primary_dir(cam, ps);
        {
            int a = p.sc.tris[3 * tri], b = p.sc.tris[3 * tri + 1], c = p.sc.tris[3 * tri + 2];
            if (!ray_triangle(org, dir, ld3(p.sc.pos + 3 * a), ld3(p.sc.pos + 3 * b), ld3(p.sc.pos + 3 * c), t, b1, b2))
                tri = -1;
        }
    }
    if (kShade) {
        D3 rad{p.sc.bg[0], p.sc.bg[1], p.sc.bg[2]};
        if (tri >= 0) rad = shade_hit<kT64>(p.sc, Hit{tri, t, b1, b2}, dir);
        s_rad[tid][0] = rad.x;
        s_rad[tid][1] = rad.y;
        s_rad[tid][2] = rad.z;
        s_hit[tid] = tri >= 0;
    }
    if (kInterior) {
        s_ray[0][tid] = dir.x;
        s_ray[1][tid] = dir.y;
        s_ray[2][tid] = dir.z;
        s_ray[3][tid] = b1;
        s_ray[4][tid] = b2;
    }
    // When spp divides 32 a warp holds whole pixels: phase 2 is warp-local and
    // no CTA barrier separates the phases (warps overlap one another's pixel
    // reductions with their scatter); the per-warp tallies meet once, at the
    // end. Otherwise pixels straddle warps and phase 2 is CTA-wide.
    const int lane = tid & 31, wib = tid >> 5;
    const bool warp_local = (32 % spp) == 0;
    __shared__ double s_wloss[kRT / 32];
    __shared__ int s_wcnt[kRT / 32][3];
    if (warp_local) __syncwarp();
    else __syncthreads();

    // ---------------- phase 2: pixel mean / mask / loss / adjoint
    // One thread per (pixel, channel): channels are independent, each sums its
    // pixel's samples in sample order (render.cpp:48-57), so the mean is the
    // reference's bit for bit; the tone map of the target is precomputed.
    double loss_part = 0;
    {
        const int ppw = warp_local ? 32 / spp : P;  // pixels per phase-2 group
        const int n_items = 3 * ppw;
        const int first = warp_local ? lane : tid, stride = warp_local ? 32 : kRT;
        for (int item = first; item < n_items; item += stride) {
            const int q = (warp_local ? wib * ppw : 0) + item % ppw, c = item / ppw;
            const int px = X0 + q % TW;
            const int py = Y0 + q / TW;
            if (px < W && py < H) {
                const size_t qi = pbase + size_t(py) * W + px;
                double mean = 0;
                if (kShade) {
                    double sum = 0;
                    int hits = 0;
                    for (int j = 0; j < spp; ++j) {
                        sum = sum + s_rad[q * spp + j][c];
                        hits += s_hit[q * spp + j];
                    }
                    mean = sum / double(spp);
                    p.img[3 * qi + c] = mean;
                    if (c == 0) p.mask[qi] = double(hits) / double(spp);
                }
                if (kLoss) s_adj[q][c] = pixel_loss_adjoint(p, vc, qi, c, mean, loss_part);
            }
        }
    }
    // per-warp tallies: loss partial, hit samples, adjoint samples
    D3 a{0, 0, 0};
    bool act;
    {
        if (kLoss)
            for (int o = 16; o > 0; o >>= 1) loss_part += __shfl_xor_sync(0xffffffffu, loss_part, o);
        if (warp_local) __syncwarp();
        else __syncthreads();  // s_adj complete
        if (kInterior && valid && tri >= 0) {
            if (kLoss) {
                a = D3{s_adj[pix][0], s_adj[pix][1], s_adj[pix][2]};
            } else {
                a = ld3(p.adj + 3 * pidx);
            }
        }
        act = kInterior && valid && tri >= 0 && !(a.x == 0 && a.y == 0 && a.z == 0);
        const int nh = __popc(__ballot_sync(0xffffffffu, valid && tri >= 0));
        const int na = __popc(__ballot_sync(0xffffffffu, act));
        const int nv = __popc(__ballot_sync(0xffffffffu, valid));
        if (lane == 0) {
            s_wloss[wib] = loss_part;
            s_wcnt[wib][0] = nh;
            s_wcnt[wib][1] = na;
            s_wcnt[wib][2] = nv;
        }
    }

    // ---------------- phase 3: interior adjoint scatter
    if constexpr (kInterior) {
        if (__any_sync(0xffffffffu, act)) interior_scatter<kRT, kT64>(p, tid, x, y, spp, tri, t, b1, b2, dir, a, act, s_ts, s_ray, s_rad);
    }

    // ---------------- publish the CTA's tallies (warp 0 waits for the others)
    __threadfence_block();
    if (wib == 0) {
        asm volatile("bar.sync 1, %0;" ::"n"(kRT) : "memory");
        if (lane == 0) {
            double tot = 0;
            unsigned long long nh = 0, na = 0, nv = 0;
            for (int w = 0; w < kRT / 32; ++w) {
                tot += s_wloss[w];
                nh += s_wcnt[w][0];
                na += s_wcnt[w][1];
                nv += s_wcnt[w][2];
            }
            if (kLoss && tot != 0) atomicAdd(&p.loss_acc[vc.slot], tot);
            if (kShade || kInterior) {
                if (nh) atomicAdd(&p.counters->hit_samples, nh);
                if (na) atomicAdd(&p.counters->adjoint_samples, na);
                if (nv) atomicAdd(&p.counters->shaded_samples, nv);
            }
        }
    } else {
        asm volatile("bar.arrive 1, %0;" ::"n"(kRT) : "memory");
    }
}

__global__ void k_tone(const double* __restrict__ in, size_t n, double gamma, double* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        out[i] = tone_map(in[i], gamma);
}

__global__ void k_widen(const float* __restrict__ in, int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = double(in[i]);
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        y[i] += x[i];
}

// texel-major accumulators -> the diffuse / specular / roughness segments
__global__ void k_texel_flush(const TexAcc* __restrict__ acc, int n, double* __restrict__ grad, int64_t lay_d,
                              int64_t lay_s, int64_t lay_r) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const TexAcc a = acc[t];
    for (int c = 0; c < 3; ++c) {
        grad[lay_d + 3 * int64_t(t) + c] += double(a.v[c]);
        grad[lay_s + 3 * int64_t(t) + c] += double(a.v[3 + c]);
    }
    grad[lay_r + t] += double(a.v[6]);
}

__global__ void k_view_loss(int n, const double* __restrict__ r, const double* __restrict__ tg,
                            const double* __restrict__ tm, double scale, double gamma, int masked,
                            double* __restrict__ adj, double* __restrict__ sum) {
    double part = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double m = masked ? tm[i] : 1.0;
        double a[3] = {0, 0, 0};
        if (m != 0)
            for (int c = 0; c < 3; ++c) {
                double d = tone_map(r[3 * i + c], gamma) - tone_map(tg[3 * i + c], gamma);
                part += m * fabs(d);
                a[c] = scale * m * double((d > 0) - (d < 0)) * tone_map_derivative(r[3 * i + c], gamma);
            }
        for (int c = 0; c < 3; ++c) adj[3 * i + c] = a[c];
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0 && part != 0) atomicAdd(sum, part);
}

template <bool kT64>
__global__ void k_radiance_points(ShadeScene sc, const SceneInfo* __restrict__ info,
                                  const DevCamera* __restrict__ cams, int slot, int n,
                                  const double* __restrict__ xy, double* __restrict__ rgb,
                                  int32_t* __restrict__ tri) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int t = -1;
    D3 r = radiance_at<kT64>(sc, cams[slot], D2{xy[2 * i], xy[2 * i + 1]}, info->t_min, &t);
    rgb[3 * i] = r.x;
    rgb[3 * i + 1] = r.y;
    rgb[3 * i + 2] = r.z;
    if (tri) tri[i] = t;
}

// Both texel records, and flag = 1 if any map value is off the fp32 grid
// (then the shading kernels read the fp64 records: images stay bit-exact).
__global__ void k_pack_textures(const double* __restrict__ d, const double* __restrict__ s,
                                const double* __restrict__ r, int n, Texel* __restrict__ out,
                                Texel64* __restrict__ out64, int* __restrict__ flag) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool off = false;
    if (i < n) {
        const double v[7] = {d[3 * i], d[3 * i + 1], d[3 * i + 2], s[3 * i], s[3 * i + 1], s[3 * i + 2], r[i]};
        Texel t;
        t.a = make_float4(float(v[0]), float(v[1]), float(v[2]), float(v[3]));
        t.b = make_float4(float(v[4]), float(v[5]), float(v[6]), 0.0f);
        out[i] = t;
        Texel64 q;
        q.a0 = make_double2(v[0], v[1]);
        q.a1 = make_double2(v[2], v[3]);
        q.b0 = make_double2(v[4], v[5]);
        q.b1 = make_double2(v[6], 0.0);
        out64[i] = q;
#pragma unroll
        for (int k = 0; k < 7; ++k) off |= double(float(v[k])) != v[k] && v[k] == v[k];  // NaN: either record
    }
    if (__any_sync(0xffffffffu, off) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace

void launch_radiance_points(cdr_ctx* c, int slot, int n, const double* xy, double* rgb, int32_t* tri) {
    if (n <= 0) return;
    tex64_resolve(c);
    ++c->launches;
    if (c->tex64_on)
        k_radiance_points<true><<<(n + 255) / 256, 256, 0, c->stream>>>(shade_scene(c), c->info.p, c->d_cams.p, slot, n,
                                                                        xy, rgb, tri);
    else
        k_radiance_points<false><<<(n + 255) / 256, 256, 0, c->stream>>>(shade_scene(c), c->info.p, c->d_cams.p, slot,
                                                                         n, xy, rgb, tri);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_pack_textures(cdr_ctx* c, const double* d, const double* s, const double* r, int n) {
    if (n <= 0) return;
    c->tex64.ensure(size_t(n));
    c->tex_flag.ensure(1);
    if (!c->tex_flag_host) CDR_CUDA_CHECK(cudaHostAlloc(&c->tex_flag_host, sizeof(int), cudaHostAllocDefault));
    CDR_CUDA_CHECK(cudaMemsetAsync(c->tex_flag.p, 0, sizeof(int), c->stream));
    ++c->launches;
    k_pack_textures<<<(n + 255) / 256, 256, 0, c->stream>>>(d, s, r, n, c->tex.p, c->tex64.p, c->tex_flag.p);
    CDR_CUDA_CHECK(cudaGetLastError());
    CDR_CUDA_CHECK(cudaMemcpyAsync(c->tex_flag_host, c->tex_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (!c->ev_texflag) CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_texflag, cudaEventDisableTiming));
    CDR_CUDA_CHECK(cudaEventRecord(c->ev_texflag, c->stream));
    c->tex_flag_pending = true;
}

// The record choice of the last packed maps, on the host, before the first
// launch that shades (waits for the flag's copy if it is still in flight:
// a staged upload finishes long before the shading is launched).
// CDR_TEXEL_F64 forces the fp64 records.
void tex64_resolve(cdr_ctx* c) {
    if (!c->tex_flag_pending) return;
    CDR_CUDA_CHECK(cudaEventSynchronize(c->ev_texflag));
    c->tex64_on = *c->tex_flag_host != 0 || std::getenv("CDR_TEXEL_F64") != nullptr;
    c->tex_flag_pending = false;
}

void launch_widen(cdr_ctx* c, const float* in, int64_t n, double* out) {
    if (n <= 0) return;
    const int nb = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
    ++c->launches;
    k_widen<<<nb, 256, 0, c->stream>>>(in, n, out);
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_tone_targets(cdr_ctx* c, double gamma) {
    size_t n = 3 * c->total_pixels;
    c->target_tone.ensure(std::max<size_t>(1, n));
    if (n == 0) return;
    int nb = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    { ++c->launches; k_tone<<<nb, 256, 0, c->stream>>>(c->target.p, n, gamma, c->target_tone.p); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_axpy(cdr_ctx* c, double* y, const double* x, int64_t n) {
    if (n <= 0) return;
    int nb = int(std::min<int64_t>((n + 255) / 256, 148 * 8));
    { ++c->launches; k_axpy<<<nb, 256, 0, c->stream>>>(y, x, n); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_texel_flush(cdr_ctx* c, int64_t lay_d, int64_t lay_s, int64_t lay_r) {
    const int n = c->tw * c->th;
    if (n <= 0) return;
    { ++c->launches; k_texel_flush<<<(n + 255) / 256, 256, 0, c->stream>>>(c->tex_acc.p, n, c->grad.p, lay_d, lay_s, lay_r); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

void launch_view_loss(cdr_ctx* c, int W, int H, const double* rendered, const double* target,
                      const double* tmask, double scale, double gamma, int masked, double* adj,
                      double* sum) {
    int n = W * H;
    int nb = std::max(1, std::min((n + 255) / 256, 148 * 8));
    { ++c->launches; k_view_loss<<<nb, 256, 0, c->stream>>>(n, rendered, target, tmask, scale, gamma, masked, adj, sum); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

// Host side of the fused kernel (declared in kernels.h).
struct RenderStatics {
    DBuf<ViewCall> calls;
    DBuf<size_t> pix_off;
    DBuf<unsigned char> has_mask;
};

static RenderStatics& statics(cdr_ctx* c) {  // owned by the context (free_render_statics)
    if (!c->render_statics) c->render_statics = new RenderStatics();
    return *static_cast<RenderStatics*>(c->render_statics);
}

template <int kSPP, bool kT64>
static void launch_render_kernel_tt(const Params& p, dim3 grid, cdr_ctx* c, bool trace, bool loss, bool interior) {
    constexpr int bs = kSPP == 16 ? kRenderThreads16 : kThreads;
    if (trace && loss && interior)
        k_render<true, true, true, kSPP, false, kT64><<<grid, bs, 0, c->stream>>>(p);
    else if (trace && !loss && !interior)
        k_render<true, false, false, kSPP, false, kT64><<<grid, bs, 0, c->stream>>>(p);
    else if (!trace && !loss && interior)
        k_render<false, false, true, kSPP, false, kT64><<<grid, bs, 0, c->stream>>>(p);
    else if (trace && loss && !interior)
        k_render<true, true, false, kSPP, false, kT64><<<grid, bs, 0, c->stream>>>(p);
    else
        throw std::runtime_error("unsupported render mode");
}

template <int kSPP>
static void launch_render_kernel_t(const Params& p, dim3 grid, cdr_ctx* c, bool trace, bool loss, bool interior) {
    if (c->tex64_on) launch_render_kernel_tt<kSPP, true>(p, grid, c, trace, loss, interior);
    else launch_render_kernel_tt<kSPP, false>(p, grid, c, trace, loss, interior);
}

static void launch_render_kernel(const Params& p, dim3 grid, cdr_ctx* c, bool trace, bool loss, bool interior) {
    ++c->launches;
    if (p.spp == 16) {
        grid.y = (grid.y * 4 + kRenderThreads16 / 64 - 1) / (kRenderThreads16 / 64);  // rows of kRT/64 pixels
        launch_render_kernel_t<16>(p, grid, c, trace, loss, interior);
    }
    else launch_render_kernel_t<0>(p, grid, c, trace, loss, interior);
}

static void launch_trace_kernel(const Params& p, dim3 grid, cdr_ctx* c) {
    ++c->launches;
    dim3 g16 = grid;
    g16.x = (grid.x + kTraceItems - 1) / kTraceItems;
    g16.y = grid.y * (kThreads / kTraceThreads16);
    if (p.use_beam && p.spp == 16) k_trace<true, 16><<<g16, kTraceThreads16, 0, c->stream>>>(p);
    else if (p.use_beam) k_trace<true, 0><<<grid, kThreads, 0, c->stream>>>(p);
    else if (p.spp == 16) k_trace<false, 16><<<g16, kTraceThreads16, 0, c->stream>>>(p);
    else k_trace<false, 0><<<grid, kThreads, 0, c->stream>>>(p);
}

void free_render_statics(cdr_ctx* c) {
    auto* st = static_cast<RenderStatics*>(c->render_statics);
    if (!st) return;
    st->calls.release();
    st->pix_off.release();
    st->has_mask.release();
    delete st;
    c->render_statics = nullptr;
}

void launch_render(cdr_ctx* c, const int* view_slots, int n_views, const RenderArgs& a, bool trace,
                   bool loss, bool interior, const double* loss_scales, cudaEvent_t after_trace) {
    if (n_views <= 0) return;
    RenderStatics& st = statics(c);
    std::vector<ViewCall> calls(n_views);
    int maxW = 0, maxH = 0;
    const int P = kThreads / a.spp;
    int TW = 1;
    while (TW * TW * 4 <= P) TW *= 2;  // near-square power-of-two width
    int TH = (P + TW - 1) / TW;
    while (TW * TH > P) --TH;
    int tile_total = 0;
    for (int i = 0; i < n_views; ++i) {
        calls[i].slot = view_slots[i];
        const DevCamera& vcam = c->views[view_slots[i]].cam;
        calls[i].tile_base = tile_total;
        calls[i].tiles_x = (vcam.W + TW - 1) / TW;
        calls[i].tiles_y = (vcam.H + TH - 1) / TH;
        tile_total += calls[i].tiles_x * calls[i].tiles_y;
        calls[i].scale = loss_scales ? loss_scales[i] : 0.0;
        calls[i].h_view = hash_combine(a.seed, uint64_t(c->views[view_slots[i]].cam.gid) + 0x9e01);
        maxW = std::max(maxW, c->views[view_slots[i]].cam.W);
        maxH = std::max(maxH, c->views[view_slots[i]].cam.H);
    }
    size_t nslots = c->views.size();
    std::vector<size_t> offs(nslots);
    std::vector<unsigned char> hm(nslots);
    for (size_t i = 0; i < nslots; ++i) {
        offs[i] = c->views[i].pix_off;
        hm[i] = c->views[i].has_target_mask;
    }
    st.calls.ensure(n_views);
    st.pix_off.ensure(nslots);
    st.has_mask.ensure(nslots);
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.calls.p, calls.data(), sizeof(ViewCall) * n_views,
                                   cudaMemcpyHostToDevice, c->stream));
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.pix_off.p, offs.data(), sizeof(size_t) * nslots,
                                   cudaMemcpyHostToDevice, c->stream));
    CDR_CUDA_CHECK(cudaMemcpyAsync(st.has_mask.p, hm.data(), nslots, cudaMemcpyHostToDevice, c->stream));

    Params p{};
    p.sc = shade_scene(c);
    p.info = c->info.p;
    p.cams = c->d_cams.p;
    p.calls = st.calls.p;
    p.pix_off = st.pix_off.p;
    p.spp = a.spp;
    p.k = a.k;
    p.inv_k = (a.k > 0 && (a.k & (a.k - 1)) == 0) ? 1.0 / a.k : 0.0;
    p.TW = TW;
    p.TH = TH;
    p.sc_bin = c->nodes.p;
    p.seed = a.seed;
    p.gamma = a.gamma;
    p.inv_gamma = 1.0 / a.gamma;
    p.use_mask = a.use_mask;
    p.write_hits = a.write_hits;
    p.img = c->img.p;
    p.mask = c->mask.p;
    p.adj = c->adj.p;
    p.hit = c->hit.p;
    p.target = c->target.p;
    p.target_tone = c->target_tone.p;
    p.target_mask = c->target_mask.p;
    p.has_mask = st.has_mask.p;
    p.grad = c->grad.p;
    p.lay_d = a.lay_diffuse;
    p.lay_s = a.lay_specular;
    p.lay_r = a.lay_roughness;
    p.lay_l = a.lay_light;
    p.corner = c->corner_acc.p;
    p.texacc = c->tex_acc.p;
    p.loss_acc = c->loss_acc.p;
    p.err = c->errinfo.p;
    p.counters = c->counters.p;

    [[maybe_unused]] int tiles = ((maxW + p.TW - 1) / p.TW) * ((maxH + p.TH - 1) / p.TH);  // CDR_LIST_STRIP
    p.use_beam = trace && c->T > 0 && !std::getenv("CDR_NO_BEAM");
    p.fast_cap = kBeamCap;  // CDR_BEAM_FAST_CAP < kBeamCap pushes tiles to the big pass (tests)
    p.no_shared_top = std::getenv("CDR_NO_SHARED_TOP") != nullptr;
    if (const char* e = std::getenv("CDR_BEAM_FAST_CAP")) p.fast_cap = std::max(0, std::min(kBeamCap, std::atoi(e)));
    p.big_list_cap = kBigCap;  // CDR_BEAM_BIG_CAP < kBigCap pushes big tiles to the split pass (tests)
    if (const char* e = std::getenv("CDR_BEAM_BIG_CAP")) p.big_list_cap = std::max(0, std::min(kBigCap, std::atoi(e)));
    p.split_list_cap = kBigCap;
    if (const char* e = std::getenv("CDR_BEAM_SPLIT_CAP")) p.split_list_cap = std::max(0, std::min(kBigCap, std::atoi(e)));
    c->beam_view.valid = 0;
    p.skip_empty_hits = p.use_beam && loss && a.spp == 16;
    if (c->beam_used_host) c->beam_used_last = *c->beam_used_host;  // previous call has completed
    if (p.use_beam) {
        // candidate pool sized from the previous call's use (overflowing tiles
        // fall back to per-ray traversal, so the size only affects speed)
        size_t want = std::max<size_t>(size_t(tile_total) * 24, size_t(c->beam_used_last) * 3 / 2 + 1024);
        if (c->beam_pool.n < want) {
            // geometric growth: the use creeps up as an optimisation moves
            // the mesh, and every reallocation (free + malloc of ~GB) stalls
            // the call (measured up to ~0.9 s)
            want = std::max(want, c->beam_pool.n + c->beam_pool.n / 2);
            const auto t0 = std::chrono::steady_clock::now();
            c->beam_pool.ensure(want);
            if (std::getenv("CDR_DEBUG_ALLOC"))
                std::fprintf(stderr, "[cdr] beam pool -> %zu candidates (%.1f MB) in %.1f ms\n", want, want * 32.0 / 1e6,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
        c->beam_hdr.ensure(std::max(1, tile_total));
        c->beam_used.ensure(1);
        CDR_CUDA_CHECK(cudaMemsetAsync(c->beam_used.p, 0, sizeof(int), c->stream));
        p.tile_hdr = c->beam_hdr.p;
        p.pool = c->beam_pool.p;
        p.pool_cap = int(std::min<size_t>(c->beam_pool.n, 0x7fffffff));
        p.pool_used = c->beam_used.p;
        const size_t npix = size_t(tile_total) * P;
        c->beam_pix_list.ensure(std::max<size_t>(16, npix * kPixCap));
        c->beam_pix_cnt.ensure(std::max<size_t>(1, npix));
        p.pix_list = c->beam_pix_list.p;
        p.pix_cnt = c->beam_pix_cnt.p;
        // big tiles: up to 1/16 of the tiles, and only while their pixel lists
        // fit k_trace's staging buffer (P <= 64, spp >= 4)
        const int big_cap = P * kBigPixCap <= kThreads * kPixCap ? std::max(64, tile_total / 16) : 0;
        c->beam_big_queue.ensure(std::max(1, big_cap));
        c->beam_big_count.ensure(4);  // big queue, split queues of levels 0 and 1
        // CDR_NO_SPLIT (A/B): no split pass, its tiles traced per ray (and counted so)
        const int split_cap = big_cap > 0 && !std::getenv("CDR_NO_SPLIT") ? std::max(64, big_cap / 8) : 0;
        c->beam_split_queue.ensure(std::max<size_t>(1, 3 * size_t(split_cap)));  // two levels + the huge pass
        c->beam_split_hdr.ensure(std::max<size_t>(4, 8 * size_t(split_cap)));    // 4 lists per group, 2 levels
        p.split_queue = c->beam_split_queue.p;
        p.split_count = c->beam_big_count.p + 1;
        p.split_cap = split_cap;
        p.huge_on = !std::getenv("CDR_NO_HUGE");
        p.split_hdr = c->beam_split_hdr.p;
        c->beam_big_pix_list.ensure(std::max<size_t>(16, size_t(big_cap) * P * kBigPixCap));
        c->beam_big_pix_cnt.ensure(std::max<size_t>(1, size_t(big_cap) * P));
        p.big_queue = c->beam_big_queue.p;
        p.big_count = c->beam_big_count.p;
        p.big_cap = big_cap;
        p.big_pix_list = c->beam_big_pix_list.p;
        p.big_pix_cnt = c->beam_big_pix_cnt.p;
        // publish the lists for the boundary probes of the same call
        std::vector<int> bases(n_views);
        for (int i = 0; i < n_views; ++i) bases[i] = calls[i].tile_base;
        c->beam_tile_base.ensure(n_views);
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->beam_tile_base.p, bases.data(), sizeof(int) * n_views,
                                       cudaMemcpyHostToDevice, c->stream));
        c->beam_view = BeamView{p.tile_hdr,          p.pool,      p.pix_list, p.pix_cnt, p.big_pix_list, p.big_pix_cnt,
                                c->beam_tile_base.p, p.split_hdr, TW,         TH,        P,              1};
        c->beam_slots.assign(view_slots, view_slots + n_views);
    }
    // Views can go through lists -> trace -> shade in chunks whose hit cache
    // (4 B per sample) fits in L2, so the shading kernel's first load hits L2.
    // Measured slower at cfg2 (the extra launch tails cost more than the L2
    // hits save: DESIGN.md §5), so off unless CDR_CHUNK_MB is set.
    size_t chunk_bytes = 0;
    if (const char* e = std::getenv("CDR_CHUNK_MB")) chunk_bytes = size_t(std::max(0, std::atoi(e))) << 20;
    const size_t per_view = size_t(maxW) * maxH * size_t(a.spp) * sizeof(int32_t);
    int chunk = n_views;
    if (trace && chunk_bytes > 0) chunk = int(std::max<size_t>(1, std::min<size_t>(n_views, chunk_bytes / per_view)));
    const int n_chunks = (n_views + chunk - 1) / chunk;
    const bool timed = after_trace != nullptr;
    // Tile queue (loss calls at spp 16, one chunk): the shading kernel runs
    // over the non-empty tiles only, the empty tiles' pixels go through
    // k_background. The queue length is read back while k_trace runs (the
    // host waits on a copy issued right after the list builders), so the
    // shading grid is exact and the GPU does not idle. Cuts the launch and
    // prologue of ~2/3 (cfg2) to ~9/10 (cfg4) of the shading CTAs.
    const bool queue = p.skip_empty_hits && n_chunks == 1 && !std::getenv("CDR_NO_QUEUE");
    const bool bg_side = c->bg && !std::getenv("CDR_BG_INLINE");  // CDR_BG_INLINE: k_background after k_render
    // shading in view groups with the images downloaded group by group (the
    // empty tiles' pixels come from k_background on the bg stream, which each
    // download waits for)
    const bool grouped = queue && bg_side && (a.img_rgb_host || a.img_mask_host) && !std::getenv("CDR_NO_IMG_OVERLAP");
    c->images_downloaded = false;
    if (grouped) {
        c->queue_starts.ensure(size_t(n_views) + 1);
        if (c->queue_starts_cap < n_views + 1) {
            if (c->queue_starts_host) CDR_CUDA_CHECK(cudaFreeHost(c->queue_starts_host));
            CDR_CUDA_CHECK(cudaHostAlloc(&c->queue_starts_host, sizeof(int) * (n_views + 1), cudaHostAllocDefault));
            c->queue_starts_cap = n_views + 1;
        }
        for (auto& e : c->img_ev)
            if (!e) CDR_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (queue) {
        c->tile_queue.ensure(std::max(1, tile_total));
        c->tile_queue_count.ensure(1 + (tile_total + kQBlock - 1) / kQBlock);  // [0] total, then per-block offsets
        if (!c->tile_queue_host) CDR_CUDA_CHECK(cudaHostAlloc(&c->tile_queue_host, sizeof(int), cudaHostAllocDefault));
        if (!c->tile_queue_ev) CDR_CUDA_CHECK(cudaEventCreateWithFlags(&c->tile_queue_ev, cudaEventDisableTiming));
        p.tile_queue = c->tile_queue.p;
        p.tile_queue_count = c->tile_queue_count.p;
    }
    if (timed) {
        while (c->chunk_ev.size() < size_t(2 * n_chunks + 1)) {
            cudaEvent_t e;
            CDR_CUDA_CHECK(cudaEventCreate(&e));
            c->chunk_ev.push_back(e);
        }
        c->chunk_ev_used = n_chunks;
    }
    for (int k = 0; k < n_chunks; ++k) {
        const int v0 = k * chunk, nv = std::min(chunk, n_views - v0);
        Params pc = p;
        pc.calls = st.calls.p + v0;
        dim3 grid((maxW + TW - 1) / TW, (maxH + TH - 1) / TH, nv);
        if (timed) CDR_CUDA_CHECK(cudaEventRecord(c->chunk_ev[2 * k], c->stream));
        if (p.use_beam) {
#ifndef CDR_LIST_STRIP
            dim3 lgrid(((maxW + TW - 1) / TW + 1) / 2 * (((maxH + TH - 1) / TH + 1) / 2), nv);
#else
            dim3 lgrid((tiles + kListWarps - 1) / kListWarps, nv);
#endif
            CDR_CUDA_CHECK(cudaMemsetAsync(pc.big_count, 0, 4 * sizeof(int), c->stream));
            // the blocks' shared top levels in a prepass (its warps do not hold
            // three builder warps at a barrier): lists 7.2 -> 6.5 ms at cfg2,
            // 22.6 -> 20.7 ms at cfg4 (CDR_NO_TOP_PREPASS: the in-kernel walk)
            if (!std::getenv("CDR_NO_TOP_PREPASS") && pc.sc.n_tris > 1 && !pc.no_shared_top) {
                const int nblk = ((maxW + TW - 1) / TW + 1) / 2 * (((maxH + TH - 1) / TH + 1) / 2);
                c->beam_top.ensure(size_t(nv) * nblk * (kTopCap + 1));
                pc.top_nodes = c->beam_top.p;
                pc.top_stride = nblk;
                // the builder over the non-empty blocks only, when most tiles are
                // empty (the previous call's fraction, as the queue trace):
                // cfg4 visibility 23.1 -> 22.1 ms; at cfg2 (a third non-empty)
                // the grid is 0.15 ms faster
                const bool bq = !std::getenv("CDR_NO_BLOCK_QUEUE") &&
                                (c->queue_frac_last < 0.25 || std::getenv("CDR_BLOCK_QUEUE"));
                if (bq) {
                    c->beam_blk_queue.ensure(size_t(nv) * nblk);
                    c->beam_blk_count.ensure(1);
                    CDR_CUDA_CHECK(cudaMemsetAsync(c->beam_blk_count.p, 0, sizeof(int), c->stream));
                    pc.blk_queue = c->beam_blk_queue.p;
                    pc.blk_queue_count = c->beam_blk_count.p;
                }
                ++c->launches;
                k_top_walk<<<dim3((nblk + 3) / 4, nv), 128, 0, c->stream>>>(pc);
            }
            ++c->launches;
            if (pc.blk_queue) k_tile_lists_q<<<148 * CDR_LIST_MIN_BLOCKS, 32 * kListWarps, 0, c->stream>>>(pc);
            else k_tile_lists<<<lgrid, 32 * kListWarps, 0, c->stream>>>(pc);
            ++c->launches;
            k_tile_lists_big<<<148 * 16 / kBigWarps, 32 * kBigWarps, 0, c->stream>>>(pc);
            if (p.split_cap > 0) {
                c->launches += 2;
                k_tile_lists_split<<<148 * 16 / kBigWarps, 32 * kBigWarps, 0, c->stream>>>(pc, 0);
                k_tile_lists_split<<<148 * 16 / kBigWarps, 32 * kBigWarps, 0, c->stream>>>(pc, 1);
                if (pc.huge_on) {
                    ++c->launches;
                    k_tile_lists_huge<<<148 * 4, 32, 0, c->stream>>>(pc);
                }
            }
        }
        if (queue) {
            const int nb = (tile_total + kQBlock - 1) / kQBlock;
            int* blk = pc.tile_queue_count + 1;
            c->launches += 3;
            k_queue_count<<<nb, 256, 0, c->stream>>>(pc.tile_hdr, tile_total, blk);
            k_queue_scan<<<1, 1024, 0, c->stream>>>(blk, nb, pc.tile_queue_count);
            k_queue_write<<<nb, 256, 0, c->stream>>>(pc, tile_total, nv, blk);
            if (grouped) {
                ++c->launches;
                k_queue_view_starts<<<(nv + 1 + 127) / 128, 128, 0, c->stream>>>(pc.tile_queue, pc.tile_queue_count, nv,
                                                                                 c->queue_starts.p);
                CDR_CUDA_CHECK(cudaMemcpyAsync(c->queue_starts_host, c->queue_starts.p, sizeof(int) * (nv + 1),
                                               cudaMemcpyDeviceToHost, c->stream));
            }
            CDR_CUDA_CHECK(cudaMemcpyAsync(c->tile_queue_host, p.tile_queue_count, sizeof(int), cudaMemcpyDeviceToHost,
                                           c->stream));
            CDR_CUDA_CHECK(cudaEventRecord(c->tile_queue_ev, c->stream));
            if (bg_side) {
                // the empty tiles' pixels (HBM-bound) beside k_trace and
                // k_render (latency-bound); joined at the end of this call
                CDR_CUDA_CHECK(cudaStreamWaitEvent(c->bg, c->tile_queue_ev, 0));
                ++c->launches;
                k_background<<<dim3((maxW * maxH + 255) / 256, nv), 256, 0, c->bg>>>(pc);
                CDR_CUDA_CHECK(cudaEventRecord(c->ev_bg, c->bg));
            }
        }
        // k_trace over the (tile-ordered) queue when most tiles are empty
        // (cfg4: 90 %, visibility 21.2 -> 20.5 ms); over the full grid otherwise
        // (cfg2: 67 % empty, the grid's 8-column CTAs measured 0.4 ms faster).
        // Deciding needs the queue length first: a ~10 us host round trip.
        // The previous loss call's non-empty fraction picks the path, so the
        // grid path never waits for the queue length before launching.
        int nq = -1;
        const bool qtrace = queue && trace && !std::getenv("CDR_NO_TRACE_QUEUE") &&
                            (c->queue_frac_last < 0.25 || std::getenv("CDR_TRACE_QUEUE"));
        if (qtrace) {
            CDR_CUDA_CHECK(cudaEventSynchronize(c->tile_queue_ev));
            nq = *c->tile_queue_host;
        }
        if (qtrace) {
            Params pt = pc;
            pt.queue_mode = 1;
            pt.queue_len = nq;
            constexpr int kCPT = 4 / (kTraceThreads16 / 64);
            if (nq > 0) {
                ++c->launches;
                k_trace<true, 16><<<(unsigned(nq) * kCPT + kTraceItems - 1) / kTraceItems, kTraceThreads16, 0,
                                    c->stream>>>(pt);
            }
        } else if (trace) {
            launch_trace_kernel(pc, grid, c);
        }
        if (timed) CDR_CUDA_CHECK(cudaEventRecord(c->chunk_ev[2 * k + 1], c->stream));
        if (a.wait_before_shade && k == 0) CDR_CUDA_CHECK(cudaStreamWaitEvent(c->stream, a.wait_before_shade, 0));
        tex64_resolve(c);  // fp32 or fp64 texel records for the shading kernels
        if (queue) {
            if (nq < 0) {
                CDR_CUDA_CHECK(cudaEventSynchronize(c->tile_queue_ev));
                nq = *c->tile_queue_host;
            }
            c->queue_frac_last = double(nq) / double(std::max(1, tile_total));
            pc.queue_mode = 1;
            constexpr int kCPT = 4 / (kRenderThreads16 / 64);
            auto shade = [&](int q0, int q1) {  // the queue range [q0, q1)
                if (q1 <= q0) return;
                ++c->launches;
                Params pq = pc;
                pq.queue_off = q0 * kCPT;
                const dim3 qgrid(unsigned(q1 - q0) * kCPT, 1, 1);
                if (interior && c->tex64_on)
                    k_render<true, true, true, 16, true, true><<<qgrid, kRenderThreads16, 0, c->stream>>>(pq);
                else if (interior)
                    k_render<true, true, true, 16, true><<<qgrid, kRenderThreads16, 0, c->stream>>>(pq);
                else if (c->tex64_on)
                    k_render<true, true, false, 16, true, true><<<qgrid, kRenderThreads16, 0, c->stream>>>(pq);
                else
                    k_render<true, true, false, 16, true><<<qgrid, kRenderThreads16, 0, c->stream>>>(pq);
            };
            if (grouped && n_chunks == 1) {
                // up to 16 view groups (CDR_IMG_GROUPS; 2 / 4 / 8 measured slower):
                // each group's images come down on the copy stream while the
                // next group shades (and the last one during the boundary pass)
                const int* qs = c->queue_starts_host;
                static const int kGroups = std::getenv("CDR_IMG_GROUPS") ? std::max(1, std::min(16, std::atoi(std::getenv("CDR_IMG_GROUPS")))) : 16;
                const int G = std::min(kGroups, nv);
                size_t ro = 0, mo = 0;
                for (int g = 0; g < G; ++g) {
                    const int va = g * nv / G, vb = (g + 1) * nv / G;
                    shade(qs[va], qs[vb]);
                    CDR_CUDA_CHECK(cudaEventRecord(c->img_ev[g], c->stream));
                    CDR_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->img_ev[g], 0));
                    CDR_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->ev_bg, 0));  // the empty tiles' pixels
                    for (int v = va; v < vb; ++v) {
                        const ViewData& vd = c->views[view_slots[v]];
                        const size_t np = size_t(vd.cam.W) * vd.cam.H;
                        if (a.img_rgb_host)
                            CDR_CUDA_CHECK(cudaMemcpyAsync(a.img_rgb_host + ro, c->img.p + 3 * vd.pix_off,
                                                           sizeof(double) * 3 * np, cudaMemcpyDeviceToHost, c->copy));
                        if (a.img_mask_host)
                            CDR_CUDA_CHECK(cudaMemcpyAsync(a.img_mask_host + mo, c->mask.p + vd.pix_off,
                                                           sizeof(double) * np, cudaMemcpyDeviceToHost, c->copy));
                        ro += 3 * np;
                        mo += np;
                    }
                }
                c->images_downloaded = true;
            } else {
                shade(0, nq);
            }
            if (!bg_side) {
                ++c->launches;
                k_background<<<dim3((maxW * maxH + 255) / 256, nv), 256, 0, c->stream>>>(pc);
            }
        } else {
            launch_render_kernel(pc, grid, c, trace, loss, interior);
        }
    }
    if (timed) CDR_CUDA_CHECK(cudaEventRecord(c->chunk_ev[2 * n_chunks], c->stream));
    if (queue && bg_side) CDR_CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_bg, 0));
    if (p.use_beam) {
        if (!c->beam_used_host) CDR_CUDA_CHECK(cudaHostAlloc(&c->beam_used_host, sizeof(int), cudaHostAllocDefault));
        CDR_CUDA_CHECK(cudaMemcpyAsync(c->beam_used_host, c->beam_used.p, sizeof(int), cudaMemcpyDeviceToHost,
                                       c->stream));
    }
    if (after_trace) CDR_CUDA_CHECK(cudaEventRecord(after_trace, c->stream));
    CDR_CUDA_CHECK(cudaGetLastError());
}

float render_trace_ms(cdr_ctx* c) {
    float tot = 0;
    for (int k = 0; k < c->chunk_ev_used; ++k) {
        float ms = 0;
        CDR_CUDA_CHECK(cudaEventElapsedTime(&ms, c->chunk_ev[2 * k], c->chunk_ev[2 * k + 1]));
        tot += ms;
    }
    return tot;
}

}  // namespace cdr

#ifdef CDR_TRACE_STATS
// debug builds: traversal counters of the primary-visibility kernels in this
// translation unit (rays, node visits, leaf tests); read-and-reset
extern "C" int cdr_debug_trace_stats(unsigned long long out[4]) {
    cudaMemcpyFromSymbol(out, cdr::g_trace_stats, sizeof(unsigned long long) * 4);
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(cdr::g_trace_stats, z, sizeof(z));
    return 0;
}
#endif
