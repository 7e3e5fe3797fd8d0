// shade.cuh — radiance of a primary-ray hit: make_hit_record (bvh.cpp:28-51)
// + eval_collocated (material.cpp:59-66) + I_e * f_r / t^2 (render.cpp:24-33).
#pragma once

#include "bvh.cuh"

namespace cdr {

struct ShadeScene {
    const BNode* nodes;
    const TriRec* recs;
    int n_tris;
    const double* pos;
    const int32_t* tris;
    const double* uv;  // nullptr: uvs absent -> uv = (0, 0)
    const double* normals;
    const double* fnormal;
    const Texel* tex;      // fp32 records (maps on the fp32 grid)
    const Texel64* tex64;  // fp64 records (any maps); kernels pick one at compile time (kT64)
    int tw, th;
    double L[3], bg[3];
};

// the degenerate-normal fallback of shade_hit, out of line (cold)
static __device__ __noinline__ D3 unit_face_normal(const double* fnormal, int tri) {
    return normalize(ld3(fnormal + 3 * tri));
}

template <bool kT64>
__device__ __forceinline__ D3 shade_hit(const ShadeScene& sc, const Hit& h, D3 dir) {
    const double b1 = h.b1, b2 = h.b2;
    const double b0 = 1.0 - b1 - b2;
    const int va = sc.tris[3 * h.tri], vb = sc.tris[3 * h.tri + 1], vc = sc.tris[3 * h.tri + 2];
    D2 uv{0, 0};
    if (sc.uv) {
        D2 u0{sc.uv[2 * va], sc.uv[2 * va + 1]}, u1{sc.uv[2 * vb], sc.uv[2 * vb + 1]},
            u2{sc.uv[2 * vc], sc.uv[2 * vc + 1]};
        uv = D2{u0.x * b0 + u1.x * b1 + u2.x * b2, u0.y * b0 + u1.y * b1 + u2.y * b2};
    }
    D3 n = ld3(sc.normals + 3 * va) * b0 + ld3(sc.normals + 3 * vb) * b1 + ld3(sc.normals + 3 * vc) * b2;
    double len = length(n);
    n = len > 1e-14 ? n / len : unit_face_normal(sc.fnormal, h.tri);
    double mu = dot(n, -dir);
    TexSample3 ts;
    if constexpr (kT64) ts = sample_maps(sc.tex64, sc.tw, sc.th, uv, false);
    else ts = sample_maps(sc.tex, sc.tw, sc.th, uv, false);
    Brdf br = eval_brdf(ts.dv, ts.sv, ts.rv, mu, false);
    return hadamard(D3{sc.L[0], sc.L[1], sc.L[2]}, br.value) / (h.t * h.t);
}

// radiance_at for a continuous pixel position (render.cpp:24-33)
template <bool kT64>
__device__ __forceinline__ D3 radiance_at(const ShadeScene& sc, const DevCamera& cam, D2 x,
                                          double t_min, int* tri_out) {
    D3 dir = primary_dir(cam, x);
    Hit h = trace(sc.nodes, sc.recs, sc.n_tris, D3{cam.o[0], cam.o[1], cam.o[2]}, dir, t_min);
    if (tri_out) *tri_out = h.tri;
    if (h.tri < 0) return D3{sc.bg[0], sc.bg[1], sc.bg[2]};
    return shade_hit<kT64>(sc, h, dir);
}

}  // namespace cdr
