// selfint.cu — self_intersects (mesh.cpp:184-214) on the LBVH: SURVEY §8(f)
// row 2. robust_evolve calls it on the input mesh and on every trial
// displacement (evolve.cpp:23, :43), verify_safety once more
// (coarse_to_fine.cpp:173); on the host it is a serial BVH pass per call.
//
// One thread per triangle f: the triangle's exact fp64 AABB, rounded outward
// to fp32, is tested against the LBVH's conservative fp32 node boxes; every
// overlapping leaf g > f that shares no vertex with f goes through the
// reference's separating-axis test (triangles_intersect, mesh.cpp:160-182),
// restated in fp64 with the same operation order (-fmad=false).
//
// Same answer as the reference: the SAT test only ever separates MORE than
// the exact test (tol = 1e-10 treats near-touching as disjoint, degenerate
// axes carry no information), so a reported pair truly intersects and its
// exact AABBs overlap; the reference's candidate set (SAH leaves,
// bvh.cpp:331-348) and this one (fp32 outward-rounded boxes) both contain
// every such pair. The set of pairs is identical; only the order in which
// they are found differs (the API returns them sorted by (f, g)).
#include "bvh.cuh"
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kSiBlock = 128;

// separated_on_axis (mesh.cpp:147-157)
__device__ __forceinline__ bool separated_on_axis(D3 axis, const D3* ta, const D3* tb, double tol) {
    const double l2 = dot(axis, axis);  // length_squared
    if (l2 < 1e-24) return false;       // degenerate axis carries no information
    double alo = dot(axis, ta[0]), ahi = alo, blo = dot(axis, tb[0]), bhi = blo;
    for (int i = 1; i < 3; ++i) {  // project_onto_axis (mesh.cpp:137-145): std::min / std::max
        const double da = dot(axis, ta[i]), db = dot(axis, tb[i]);
        alo = da < alo ? da : alo;
        ahi = ahi < da ? da : ahi;
        blo = db < blo ? db : blo;
        bhi = bhi < db ? db : bhi;
    }
    const double g0 = blo - ahi, g1 = alo - bhi;
    const double gap = g0 < g1 ? g1 : g0;  // std::max(g0, g1)
    return gap > -tol * sqrt(l2);
}

// triangles_intersect (mesh.cpp:160-182), tol = 1e-10 (mesh.hpp:61-63)
__device__ bool triangles_intersect(const D3* ta, const D3* tb) {
    constexpr double tol = 1e-10;
    const D3 ea[3] = {ta[1] - ta[0], ta[2] - ta[1], ta[0] - ta[2]};
    const D3 eb[3] = {tb[1] - tb[0], tb[2] - tb[1], tb[0] - tb[2]};
    if (separated_on_axis(cross(ea[0], ea[1]), ta, tb, tol)) return false;
    if (separated_on_axis(cross(eb[0], eb[1]), ta, tb, tol)) return false;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (separated_on_axis(cross(ea[i], eb[j]), ta, tb, tol)) return false;
    return true;
}

__device__ __forceinline__ bool box_overlap(float lx, float ly, float lz, float hx, float hy, float hz,
                                            const float* lo, const float* hi) {
    return lx <= hi[0] && hx >= lo[0] && ly <= hi[1] && hy >= lo[1] && lz <= hi[2] && hz >= lo[2];
}

__global__ void __launch_bounds__(kSiBlock) k_self_intersect(const BNode* __restrict__ nodes,
                                                             const TriRec* __restrict__ recs,
                                                             const double* __restrict__ pos,
                                                             const int32_t* __restrict__ tris, int T,
                                                             int2* __restrict__ pairs, long long cap,
                                                             unsigned long long* __restrict__ count) {
    const int f = blockIdx.x * kSiBlock + threadIdx.x;
    if (f >= T) return;
    if (!pairs && *reinterpret_cast<volatile unsigned long long*>(count)) return;  // answer known
    const int t0 = tris[3 * f], t1 = tris[3 * f + 1], t2 = tris[3 * f + 2];
    const D3 ta[3] = {ld3(pos + 3 * t0), ld3(pos + 3 * t1), ld3(pos + 3 * t2)};
    float lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        const double a = comp(ta[0], k), b = comp(ta[1], k), c = comp(ta[2], k);
        lo[k] = __double2float_rd(fmin(a, fmin(b, c)));
        hi[k] = __double2float_ru(fmax(a, fmax(b, c)));
    }
    int stack[64];
    int sp = 0;
    int node = 0;
    auto visit_leaf = [&](int leaf) -> bool {  // false: stop (answer found, no pair list)
        const int g = __ldg(&recs[leaf].tri);
        if (g <= f) return true;
        const int s0 = tris[3 * g], s1 = tris[3 * g + 1], s2 = tris[3 * g + 2];
        if (t0 == s0 || t0 == s1 || t0 == s2 || t1 == s0 || t1 == s1 || t1 == s2 || t2 == s0 || t2 == s1 ||
            t2 == s2)
            return true;  // adjacent: shares a vertex
        const D3 tb[3] = {ld3(pos + 3 * s0), ld3(pos + 3 * s1), ld3(pos + 3 * s2)};
        if (!triangles_intersect(ta, tb)) return true;
        const unsigned long long i = atomicAdd(count, 1ull);
        if (!pairs) return false;
        if (i < (unsigned long long)cap) pairs[i] = make_int2(f, g);
        return true;
    };
    if (T == 1) return;
    while (true) {
        const BNode* np = nodes + node;
        const float4 a = __ldg(&np->a), b = __ldg(&np->b), c = __ldg(&np->c);
        const int4 k = __ldg(&np->k);
        bool h0 = box_overlap(a.x, a.y, a.z, a.w, b.x, b.y, lo, hi);
        bool h1 = box_overlap(b.z, b.w, c.x, c.y, c.z, c.w, lo, hi);
        if (h0 && k.x < 0) {
            if (!visit_leaf(~k.x)) return;
            h0 = false;
        }
        if (h1 && k.y < 0) {
            if (!visit_leaf(~k.y)) return;
            h1 = false;
        }
        if (h0 && h1) {
            if (sp >= 64) __trap();  // LBVH depth bound (bvh.cuh trace): never taken
            stack[sp++] = k.y;
            node = k.x;
        } else if (h0) {
            node = k.x;
        } else if (h1) {
            node = k.y;
        } else {
            if (sp == 0) break;
            node = stack[--sp];
        }
    }
}

}  // namespace

long long launch_self_intersect(cdr_ctx* c, int2* pairs, long long cap) {
    if (c->T < 2) return 0;
    DBuf<unsigned long long>& cnt = c->scr_u64;
    cnt.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), c->stream));
    ++c->launches;
    k_self_intersect<<<(c->T + kSiBlock - 1) / kSiBlock, kSiBlock, 0, c->stream>>>(c->nodes.p, c->recs.p, c->pos.p,
                                                                                  c->tris.p, c->T, pairs, cap, cnt.p);
    CDR_CUDA_CHECK(cudaGetLastError());
    unsigned long long n = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(&n, cnt.p, sizeof(n), cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return (long long)n;
}

}  // namespace cdr
