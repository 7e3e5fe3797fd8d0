// bvh.cuh — LBVH node layout and nearest-hit traversal (replaces Bvh::intersect,
// bvh.cpp:210-265).
//
// Layout: internal node i of the Karras hierarchy stores BOTH
// children's boxes (fp32, rounded outward and padded) and their indices in one
// 64-byte record, so one node visit is four 16-byte loads and tests two boxes.
// Children < 0 are leaves (~leaf). Leaf l holds triangle tri_rec[l] — its
// three fp64 vertices (80-byte record, five 16-byte loads) in Morton order.
//
// Exactness: boxes only prune, and they are conservative (outward rounding +
// padding >> fp32 ray error), so the nearest hit is decided solely by the fp64
// Moller-Trumbore test with strict t_min < t and ties to the lowest triangle
// index — the answer of the brute-force oracle (tests/support/test_scenes.hpp:
// 20-39), independent of tree shape.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace cdr {

struct __align__(16) BNode {
    float4 a;  // lo0.x lo0.y lo0.z hi0.x
    float4 b;  // hi0.y hi0.z lo1.x lo1.y
    float4 c;  // lo1.z hi1.x hi1.y hi1.z
    int4 k;    // child0 child1 - -
};

struct __align__(16) TriRec {
    double2 a;  // p0.x p0.y
    double2 b;  // p0.z p1.x
    double2 c;  // p1.y p1.z
    double2 d;  // p2.x p2.y
    double e;   // p2.z
    int tri;
    int pad;
};

#ifdef CDR_TRACE_STATS
// debug build only: [0] rays, [1] node visits, [2] leaf (triangle) tests
static __device__ unsigned long long g_trace_stats[4];  // per translation unit
#define CDR_STAT(i, v) atomicAdd(&g_trace_stats[i], (unsigned long long)(v))
#else
#define CDR_STAT(i, v)
#endif

struct Hit {
    int tri;
    double t, b1, b2;
};

struct FRay {
    float ox, oy, oz;   // o * inv (negated in the fma)
    float ix, iy, iz;   // 1 / d
};

__device__ __forceinline__ float safe_inv(double d) {
    float f = float(d);
    if (fabsf(f) < 1e-20f) f = copysignf(1e-20f, f);
    return 1.0f / f;
}

__device__ __forceinline__ FRay make_fray(D3 o, D3 d) {
    FRay r;
    r.ix = safe_inv(d.x);
    r.iy = safe_inv(d.y);
    r.iz = safe_inv(d.z);
    r.ox = float(o.x) * r.ix;
    r.oy = float(o.y) * r.iy;
    r.oz = float(o.z) * r.iz;
    return r;
}

// Slab test; returns entry distance in tn. Pure pruning: never decides a hit.
__device__ __forceinline__ bool box_test(const FRay& r, float lx, float ly, float lz, float hx,
                                         float hy, float hz, float tbest, float& tn) {
    float x0 = __fmaf_rn(lx, r.ix, -r.ox), x1 = __fmaf_rn(hx, r.ix, -r.ox);
    float y0 = __fmaf_rn(ly, r.iy, -r.oy), y1 = __fmaf_rn(hy, r.iy, -r.oy);
    float z0 = __fmaf_rn(lz, r.iz, -r.oz), z1 = __fmaf_rn(hz, r.iz, -r.oz);
    float tmin = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.0f));
    float tmax = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), tbest));
    tn = tmin;
    return tmin <= tmax;
}

__device__ __forceinline__ void leaf_test(const TriRec* __restrict__ recs, int leaf, D3 o, D3 d,
                                          double t_min, Hit& best) {
    const TriRec* p = recs + leaf;
    double2 a = __ldg(&p->a), b = __ldg(&p->b), c = __ldg(&p->c), dd = __ldg(&p->d);
    double e = __ldg(&p->e);
    int tri = __ldg(&p->tri);
    CDR_STAT(2, 1);
    double t, b1, b2;
    if (ray_triangle(o, d, D3{a.x, a.y, b.x}, D3{b.y, c.x, c.y}, D3{dd.x, dd.y, e}, t, b1, b2) &&
        t > t_min && (t < best.t || (t == best.t && tri < best.tri))) {
        best.t = t;
        best.tri = tri;
        best.b1 = b1;
        best.b2 = b2;
    }
}

__device__ __forceinline__ float tbest_f(double t) {
    // rounded up and relaxed: pruning must never discard a tie or a closer hit
    return t >= 1e30 ? FLT_MAX : __double2float_ru(t) * 1.00001f + 1e-6f;
}

// Nearest hit with t > t_min; best.tri = -1 on a miss.
__device__ __forceinline__ Hit trace(const BNode* __restrict__ nodes,
                                     const TriRec* __restrict__ recs, int n_tris, D3 o, D3 d,
                                     double t_min) {
    Hit best{-1, 1e300, 0.0, 0.0};
    if (n_tris <= 0) return best;
    if (n_tris == 1) {
        leaf_test(recs, 0, o, d, t_min, best);
        return best;
    }
    FRay r = make_fray(o, d);
    CDR_STAT(0, 1);
    int stack[64];
    int sp = 0;
    int node = 0;
    float tb = FLT_MAX;
    while (true) {
        const BNode* np = nodes + node;
        CDR_STAT(1, 1);
        float4 a = __ldg(&np->a), b = __ldg(&np->b), c = __ldg(&np->c);
        int4 k = __ldg(&np->k);
        float t0, t1;
        bool h0 = box_test(r, a.x, a.y, a.z, a.w, b.x, b.y, tb, t0);
        bool h1 = box_test(r, b.z, b.w, c.x, c.y, c.z, c.w, tb, t1);
        if (h0 && k.x < 0) {
            leaf_test(recs, ~k.x, o, d, t_min, best);
            tb = tbest_f(best.t);
            h0 = false;
        }
        if (h1 && k.y < 0) {
            leaf_test(recs, ~k.y, o, d, t_min, best);
            tb = tbest_f(best.t);
            h1 = false;
        }
        if (h0 && h1) {
            int nearc = t0 <= t1 ? k.x : k.y;
            int farc = t0 <= t1 ? k.y : k.x;
            // Depth bound: a Karras node splits its key range at a strictly lower
            // bit than its parent, and keys have 62 bits (30 Morton + 32 index),
            // so a root-to-leaf path holds <= 62 internal nodes and the stack
            // (one entry per internal node on the path) never exceeds 62 < 64.
            // An overflow would mean a corrupt hierarchy: fail loudly.
            if (sp >= 64) __trap();
            stack[sp++] = farc;
            node = nearc;
        } else if (h0) {
            node = k.x;
        } else if (h1) {
            node = k.y;
        } else {
            if (sp == 0) break;
            node = stack[--sp];
        }
    }
    return best;
}

}  // namespace cdr
