// closest.cu — Bvh::closest_point (bvh.cpp:267-329) on the LBVH: SURVEY §8(f)
// row 4 (uv_transfer after a remesh, remesh.cpp:281-294; the point-to-mesh
// metric, mesh.cpp:127-133).
//
// One thread per query point: depth-first, nearer child first, pruned by the
// squared distance to a child's box; leaves run the reference's
// closest_point_on_triangle (mesh.cpp:96-126, restated in fp64, -fmad=false),
// then the barycentrics are recovered exactly as bvh.cpp:312-326.
//
// The distance is the reference's (exact per triangle, the minimum is
// unique); the boxes are conservative fp32, so pruning uses a relative
// margin and never discards a triangle at the best distance. On an exact tie
// (e.g. a query nearest a vertex shared by several triangles) the lowest
// triangle index wins, where the reference keeps the first its SAH traversal
// meets: the point and distance agree, the triangle may differ.
#include "bvh.cuh"
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kCpBlock = 128;

// closest_point_on_triangle (mesh.cpp:96-126), Ericson 5.1.5
__device__ D3 closest_on_triangle(D3 p, D3 a, D3 b, D3 c) {
    const D3 ab = b - a, ac = c - a, ap = p - a;
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0 && d2 <= 0) return a;
    const D3 bp = p - b;
    const double d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0 && d4 <= d3) return b;
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        const double v = d1 / (d1 - d3);
        return a + ab * v;
    }
    const D3 cp = p - c;
    const double d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0 && d5 <= d6) return c;
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        const double w = d2 / (d2 - d6);
        return a + ac * w;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return b + (c - b) * w;
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    return a + ab * v + ac * w;
}

__device__ __forceinline__ double box_dist_sq(D3 q, float lx, float ly, float lz, float hx, float hy, float hz) {
    const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz}, p[3] = {q.x, q.y, q.z};
    double d = 0;
    for (int k = 0; k < 3; ++k) {
        if (p[k] < lo[k]) d += (lo[k] - p[k]) * (lo[k] - p[k]);
        else if (p[k] > hi[k]) d += (p[k] - hi[k]) * (p[k] - hi[k]);
    }
    return d;
}

__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }  // std::clamp

__global__ void __launch_bounds__(kCpBlock) k_closest(const BNode* __restrict__ nodes, const TriRec* __restrict__ recs,
                                                      const double* __restrict__ pos, const int32_t* __restrict__ tris,
                                                      int T, const double* __restrict__ queries, int nq,
                                                      int32_t* __restrict__ tri_out, double* __restrict__ point_out,
                                                      double* __restrict__ dist_out, double* __restrict__ bary_out) {
    const int qi = blockIdx.x * kCpBlock + threadIdx.x;
    if (qi >= nq) return;
    const D3 q = ld3(queries + 3 * size_t(qi));
    int best_tri = -1;
    double best = 1e300;
    D3 best_pt{0, 0, 0};
    auto leaf = [&](int l) {
        const int f = __ldg(&recs[l].tri);
        const D3 a = ld3(pos + 3 * tris[3 * f]), b = ld3(pos + 3 * tris[3 * f + 1]), c = ld3(pos + 3 * tris[3 * f + 2]);
        const D3 cp = closest_on_triangle(q, a, b, c);
        const double d = length(q - cp);
        if (d < best || (d == best && f < best_tri)) {
            best = d;
            best_tri = f;
            best_pt = cp;
        }
    };
    // prune only boxes certainly farther than the best (fp32 boxes, fp64 sums)
    auto far = [&](double dsq) { return dsq * (1.0 - 1e-9) > best * best; };
    if (T == 1) {
        leaf(0);
    } else if (T > 1) {
        int stack[64];
        double sd[64];
        int sp = 0;
        stack[sp] = 0;
        sd[sp++] = 0.0;
        while (sp > 0) {
            --sp;
            if (far(sd[sp])) continue;
            const BNode* np = nodes + stack[sp];
            const float4 A = __ldg(&np->a), B = __ldg(&np->b), Cc = __ldg(&np->c);
            const int4 k = __ldg(&np->k);
            const double d0 = box_dist_sq(q, A.x, A.y, A.z, A.w, B.x, B.y);
            const double d1 = box_dist_sq(q, B.z, B.w, Cc.x, Cc.y, Cc.z, Cc.w);
            // leaves at once; inner children pushed farther first
            int ch[2] = {k.x, k.y};
            double dd[2] = {d0, d1};
            if (d1 < d0) {
                ch[0] = k.y;
                ch[1] = k.x;
                dd[0] = d1;
                dd[1] = d0;
            }
            for (int j = 1; j >= 0; --j) {
                if (far(dd[j])) continue;
                if (ch[j] < 0) {
                    leaf(~ch[j]);
                } else {
                    // <= one entry per level of the path plus the sibling just
                    // pushed: <= 63 by the LBVH depth bound (bvh.cuh trace)
                    if (sp >= 64) __trap();
                    stack[sp] = ch[j];
                    sd[sp++] = dd[j];
                }
            }
        }
    }
    double b0 = 0, b1 = 0, b2 = 0;
    if (best_tri >= 0) {  // bvh.cpp:312-326
        const int f = best_tri;
        const D3 a = ld3(pos + 3 * tris[3 * f]), b = ld3(pos + 3 * tris[3 * f + 1]), c = ld3(pos + 3 * tris[3 * f + 2]);
        const D3 v0 = b - a, v1 = c - a, v2 = best_pt - a;
        const double d00 = dot(v0, v0), d01 = dot(v0, v1), d11 = dot(v1, v1);
        const double d20 = dot(v2, v0), d21 = dot(v2, v1);
        const double denom = d00 * d11 - d01 * d01;
        if (fabs(denom) > 1e-30) {
            b1 = clamp01((d11 * d20 - d01 * d21) / denom);
            b2 = clamp01((d00 * d21 - d01 * d20) / denom);
        }
        b0 = clamp01(1.0 - b1 - b2);
    }
    if (tri_out) tri_out[qi] = best_tri;
    if (dist_out) dist_out[qi] = best;
    if (point_out) {
        point_out[3 * size_t(qi)] = best_pt.x;
        point_out[3 * size_t(qi) + 1] = best_pt.y;
        point_out[3 * size_t(qi) + 2] = best_pt.z;
    }
    if (bary_out) {
        bary_out[3 * size_t(qi)] = b0;
        bary_out[3 * size_t(qi) + 1] = b1;
        bary_out[3 * size_t(qi) + 2] = b2;
    }
}

}  // namespace

void launch_closest(cdr_ctx* c, const double* queries, int nq, int32_t* tri, double* point, double* dist,
                    double* bary) {
    if (nq <= 0) return;
    ++c->launches;
    k_closest<<<(nq + kCpBlock - 1) / kCpBlock, kCpBlock, 0, c->stream>>>(c->nodes.p, c->recs.p, c->pos.p, c->tris.p,
                                                                          c->T, queries, nq, tri, point, dist, bary);
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr
