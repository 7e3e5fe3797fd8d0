// regularisers.cu — the mesh and material regularisers of total_loss
// (losses.cpp:80-238, summed at :272-292) on the device: SURVEY §8(f) row 1.
//
//   normal_consistency_loss  (losses.cpp:80-115)  one thread per edge, fp64 RED
//                                                  into the position gradient
//   edge_length_loss         (losses.cpp:117-134)  Σ|e|² reduction, then per edge
//   specular_correlation_loss(losses.cpp:136-213)  two gather passes, no atomics
//   roughness_tv_loss        (losses.cpp:215-238)  one gather pass, no atomics
//
// The texture terms are restated as gathers: a texel's gradient is the sum of
// the contributions the reference scatters to it, added in the reference's own
// order (ascending source texel, and inside the source the window order), so
// every texture-gradient element has a single writer and a fixed summation
// order. Values reduce through per-block partials in a fixed grid, so every
// result is deterministic run to run. Exact reproduction is limited by exp()
// (CUDA's and glibc's may differ in the last bit) and, for the two position
// terms, by the order of the fp64 REDs: tolerance 1e-12 relative on values,
// bit-exact texture gradients of the TV term.
#include <algorithm>

#include "common.cuh"
#include "context.h"
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kRegBlock = 256;
constexpr int kRegGrid = 148 * 4;  // fixed: partial sums reduce in a fixed order
__constant__ double kLumW[3] = {0.2126, 0.7152, 0.0722};  // losses.cpp:149

__device__ __forceinline__ double sgn(double v) { return double((v > 0) - (v < 0)); }  // losses.cpp:12

// Block sum of one value per thread into part[blockIdx.x] (fixed tree order).
__device__ __forceinline__ void block_partial(double v, double* part) {
    __shared__ double s[kRegBlock / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < kRegBlock / 32; ++w) t += s[w];
        part[blockIdx.x] = t;
    }
}

// Σ of the kRegGrid partials of each term (one warp per term, fixed order).
__global__ void k_reg_finish(const double* __restrict__ part, int n_terms, double* __restrict__ out) {
    const int term = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (term >= n_terms) return;
    double v = 0;
    for (int i = lane; i < kRegGrid; i += 32) v += part[term * kRegGrid + i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[term] = v;
}

__device__ __forceinline__ D3 face_normal_unnormalized(const double* pos, const int32_t* tris, int f) {
    // mesh.hpp:30-33
    const int a = tris[3 * f], b = tris[3 * f + 1], c = tris[3 * f + 2];
    const D3 pa = ld3(pos + 3 * a);
    return cross(ld3(pos + 3 * b) - pa, ld3(pos + 3 * c) - pa);
}

// normalize_jacobian(m) * v (vec.hpp:179-183): ((I - n n^T) * (1/|m|)) v, row by row
__device__ __forceinline__ D3 normalize_jacobian_times(D3 m, D3 v) {
    const double len = length(m);
    const D3 n = m / len;
    const double s = 1.0 / len;
    const double nn[3] = {n.x, n.y, n.z};
    double J[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) J[3 * i + j] = ((i == j ? 1.0 : 0.0) - nn[i] * nn[j]) * s;
    return D3{J[0] * v.x + J[1] * v.y + J[2] * v.z, J[3] * v.x + J[4] * v.y + J[5] * v.z,
              J[6] * v.x + J[7] * v.y + J[8] * v.z};
}

// Mat3::skew(v).transpose_times(h) (vec.hpp:104-109, :153-157), terms as written
__device__ __forceinline__ D3 skew_t_times(D3 v, D3 h) {
    return D3{0.0 * h.x + v.z * h.y + -v.y * h.z, -v.z * h.x + 0.0 * h.y + v.x * h.z,
              v.y * h.x + -v.x * h.y + 0.0 * h.z};
}

__device__ __forceinline__ void red3(double* g, D3 v) {
    atomicAdd(g, v.x);
    atomicAdd(g + 1, v.y);
    atomicAdd(g + 2, v.z);
}

// normal_consistency_loss (losses.cpp:80-115): per interior edge, r = 1 - n0.n1,
// value λ r², gradient -2 λ r (skew^T h) to the 6 corners of the two faces.
__global__ void __launch_bounds__(kRegBlock) k_normal_consistency(const int4* __restrict__ edges, int E,
                                                                   const double* __restrict__ pos,
                                                                   const int32_t* __restrict__ tris, double lambda,
                                                                   double* __restrict__ grad_pos,
                                                                   double* __restrict__ part) {
    double val = 0;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < E; i += kRegGrid * kRegBlock) {
        const int4 e = edges[i];
        if (e.w < 0) continue;
        const D3 m0 = face_normal_unnormalized(pos, tris, e.z), m1 = face_normal_unnormalized(pos, tris, e.w);
        const double l0 = length(m0), l1 = length(m1);
        if (l0 < 1e-14 || l1 < 1e-14) continue;  // degenerate face skipped
        const D3 n0 = m0 / l0, n1 = m1 / l1;
        const double r = 1.0 - dot(n0, n1);
        val += lambda * r * r;
        if (!grad_pos) continue;
        const D3 h0 = normalize_jacobian_times(m0, n1), h1 = normalize_jacobian_times(m1, n0);
        const double w = -2.0 * lambda * r;
        for (int which = 0; which < 2; ++which) {
            const int f = which == 0 ? e.z : e.w;
            const D3 h = which == 0 ? h0 : h1;
            const int ta = tris[3 * f], tb = tris[3 * f + 1], tc = tris[3 * f + 2];
            const D3 a = ld3(pos + 3 * ta), b = ld3(pos + 3 * tb), c = ld3(pos + 3 * tc);
            red3(grad_pos + 3 * ta, skew_t_times(c - b, h) * w);
            red3(grad_pos + 3 * tb, skew_t_times(a - c, h) * w);
            red3(grad_pos + 3 * tc, skew_t_times(b - a, h) * w);
        }
    }
    block_partial(val, part);
}

// edge_length_loss (losses.cpp:117-134), pass 1: Σ |p_v0 - p_v1|²
__global__ void __launch_bounds__(kRegBlock) k_edge_sumsq(const int4* __restrict__ edges, int E,
                                                           const double* __restrict__ pos, double* __restrict__ part) {
    double s = 0;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < E; i += kRegGrid * kRegBlock) {
        const int4 e = edges[i];
        const D3 d = ld3(pos + 3 * e.x) - ld3(pos + 3 * e.y);
        s += dot(d, d);
    }
    block_partial(s, part);
}

// pass 2: value λ sqrt(Σ) and gradient ±d λ/sqrt(Σ) (sum_sq <= 0: no gradient)
__global__ void __launch_bounds__(kRegBlock) k_edge_grad(const int4* __restrict__ edges, int E,
                                                          const double* __restrict__ pos, double lambda,
                                                          const double* __restrict__ sum_sq, double* __restrict__ value,
                                                          double* __restrict__ grad_pos) {
    const double ss = *sum_sq;
    if (ss <= 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *value = 0;
        return;
    }
    const double root = sqrt(ss);
    if (blockIdx.x == 0 && threadIdx.x == 0) *value = lambda * root;
    if (!grad_pos) return;
    const double w = lambda / root;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < E; i += kRegGrid * kRegBlock) {
        const int4 e = edges[i];
        const D3 d = ld3(pos + 3 * e.x) - ld3(pos + 3 * e.y);
        red3(grad_pos + 3 * e.x, d * w);
        red3(grad_pos + 3 * e.y, -(d * w));
    }
}

// ---- specular_correlation_loss (losses.cpp:136-213) -------------------------
struct SpecParams {
    const double* ad;  // diffuse  tw*th*3
    const double* as;  // specular tw*th*3
    double* lum;       // tw*th
    double* stats;     // tw*th*8: mu_sum, avg[3], sign[3], -
    int w, h;
    double spec, inv_2s1, inv_2s2;
};

__global__ void k_luminance(SpecParams p) {
    const int n = p.w * p.h;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < n; i += gridDim.x * kRegBlock)
        p.lum[i] = dot(ld3(p.ad + 3 * size_t(i)), D3{kLumW[0], kLumW[1], kLumW[2]});  // losses.cpp:152
}

__device__ __forceinline__ double bilateral_mu(int dx, int dy, double dl, double inv_2s1, double inv_2s2) {
    return exp(-(dx * dx + dy * dy) * inv_2s1 - dl * dl * inv_2s2);  // losses.cpp:168
}

// pass 1 (losses.cpp:154-190): per texel p the window weights' sum, the
// weighted specular average and the sign of (center - average); value partials.
__global__ void __launch_bounds__(kRegBlock) k_spec_stats(SpecParams p, double* __restrict__ part) {
    const int n = p.w * p.h;
    double val = 0;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < n; i += kRegGrid * kRegBlock) {
        const int px = i % p.w, py = i / p.w;
        const double lp = p.lum[i];
        double mu_sum = 0;
        D3 avg{0, 0, 0};
        for (int dy = -3; dy <= 3; ++dy) {
            const int qy = py + dy;
            if (qy < 0 || qy >= p.h) continue;
            for (int dx = -3; dx <= 3; ++dx) {
                const int qx = px + dx;
                if (qx < 0 || qx >= p.w) continue;
                const int q = qy * p.w + qx;
                const double mu = bilateral_mu(dx, dy, lp - p.lum[q], p.inv_2s1, p.inv_2s2);
                mu_sum += mu;
                avg = avg + ld3(p.as + 3 * size_t(q)) * mu;
            }
        }
        avg = avg / mu_sum;
        const D3 center = ld3(p.as + 3 * size_t(i));
        double* st = p.stats + 8 * size_t(i);
        st[0] = mu_sum;
        st[1] = avg.x;
        st[2] = avg.y;
        st[3] = avg.z;
        for (int c = 0; c < 3; ++c) {
            const double d = comp(center, c) - comp(avg, c);
            val += p.spec * fabs(d);
            st[4 + c] = sgn(d);
        }
    }
    block_partial(val, part);
}

// d_to_mu(p, q) of losses.cpp:197-200 from p's stats and the specular at q
__device__ __forceinline__ double d_to_mu(const double* st_p, D3 as_q, double spec) {
    double s = 0;
    s += -spec * st_p[4] * (as_q.x - st_p[1]) / st_p[0];
    s += -spec * st_p[5] * (as_q.y - st_p[2]) / st_p[0];
    s += -spec * st_p[6] * (as_q.z - st_p[3]) / st_p[0];
    return s;
}

// pass 2: gather of the gradients the reference scatters (losses.cpp:191-210).
// For texel x, in the reference's order of updates to x:
//   specular: sources p ascending; at p = x the center term precedes the
//             window terms; each source p contributes -spec sign_p mu_px / mu_sum_p;
//   diffuse:  sources p < x contribute as q (dmu/dl_q terms); at p = x the
//             whole window of x in order (dmu/dl_p terms, with the q = x term
//             of the same step right after its p term); then p > x as q.
__global__ void __launch_bounds__(kRegBlock) k_spec_grad(SpecParams p, double* __restrict__ grad_d,
                                                          double* __restrict__ grad_s) {
    const int n = p.w * p.h;
    for (int x = blockIdx.x * kRegBlock + threadIdx.x; x < n; x += gridDim.x * kRegBlock) {
        const int px = x % p.w, py = x / p.w;
        const double lx = p.lum[x];
        const double* st_x = p.stats + 8 * size_t(x);
        const D3 as_x = ld3(p.as + 3 * size_t(x));
        double gs[3] = {0, 0, 0}, gd[3] = {0, 0, 0};
        for (int dy = -3; dy <= 3; ++dy) {
            const int yy = py + dy;
            if (yy < 0 || yy >= p.h) continue;
            for (int dx = -3; dx <= 3; ++dx) {
                const int xx = px + dx;
                if (xx < 0 || xx >= p.w) continue;
                const int y = yy * p.w + xx;  // source texel (p of the reference)
                const double* st_y = p.stats + 8 * size_t(y);
                if (y == x) {
                    for (int c = 0; c < 3; ++c) gs[c] += p.spec * st_x[4 + c];  // center term
                    // x's own window, in order: dmu/dl_p terms to x, and the q = x term
                    for (int ey = -3; ey <= 3; ++ey) {
                        const int qy = py + ey;
                        if (qy < 0 || qy >= p.h) continue;
                        for (int ex = -3; ex <= 3; ++ex) {
                            const int qx = px + ex;
                            if (qx < 0 || qx >= p.w) continue;
                            const int q = qy * p.w + qx;
                            const double dl = lx - p.lum[q];
                            const double mu = bilateral_mu(ex, ey, dl, p.inv_2s1, p.inv_2s2);
                            const double dtm = d_to_mu(st_x, ld3(p.as + 3 * size_t(q)), p.spec);
                            const double dmu_dlp = mu * (-2.0 * dl * p.inv_2s2);
                            for (int c = 0; c < 3; ++c) gd[c] += dtm * dmu_dlp * kLumW[c];
                            if (q == x) {
                                const double dmu_dlq = -dmu_dlp;
                                for (int c = 0; c < 3; ++c) gd[c] += dtm * dmu_dlq * kLumW[c];
                            }
                        }
                    }
                }
                // x inside y's window: y's window term to x (x plays q)
                const double dl = p.lum[y] - lx;
                const double mu = bilateral_mu(-dx, -dy, dl, p.inv_2s1, p.inv_2s2);
                for (int c = 0; c < 3; ++c) gs[c] -= p.spec * st_y[4 + c] * mu / st_y[0];
                if (y != x) {
                    const double dtm = d_to_mu(st_y, as_x, p.spec);
                    const double dmu_dlq = -(mu * (-2.0 * dl * p.inv_2s2));
                    for (int c = 0; c < 3; ++c) gd[c] += dtm * dmu_dlq * kLumW[c];
                }
            }
        }
        for (int c = 0; c < 3; ++c) {
            if (grad_s) grad_s[3 * size_t(x) + c] += gs[c];
            if (grad_d) grad_d[3 * size_t(x) + c] += gd[c];
        }
    }
}

// roughness_tv_loss (losses.cpp:215-238): value partials and the gathered
// gradient of texel (x, y) in the reference's update order:
// +s_v(x, y-1), +s_h(x-1, y), -s_h(x, y), -s_v(x, y).
__global__ void __launch_bounds__(kRegBlock) k_roughness_tv(const double* __restrict__ r, int w, int h, double lambda,
                                                             double* __restrict__ grad_r, double* __restrict__ part) {
    const int n = w * h;
    double val = 0;
    for (int i = blockIdx.x * kRegBlock + threadIdx.x; i < n; i += kRegGrid * kRegBlock) {
        const int x = i % w, y = i / w;
        const double v = r[i];
        double g = 0;
        if (y > 0) g += lambda * sgn(v - r[i - w]);
        if (x > 0) g += lambda * sgn(v - r[i - 1]);
        if (x + 1 < w) {
            const double d = r[i + 1] - v;
            val += lambda * fabs(d);
            g -= lambda * sgn(d);
        }
        if (y + 1 < h) {
            const double d = r[i + w] - v;
            val += lambda * fabs(d);
            g -= lambda * sgn(d);
        }
        if (grad_r) grad_r[i] += g;
    }
    block_partial(val, part);
}

}  // namespace

// values_dev[0..3] = normal, edge, spec, roug; gradients += into grad (ParamLayout
// order, device) when grad != nullptr. Every term is skipped at weight 0.
void launch_regularisers(cdr_ctx* c, const cdr_reg_weights& w, const cdr_layout& lay, double* grad,
                         double* values_dev) {
    c->reg_part.ensure(size_t(4) * kRegGrid + 8);
    double* part = c->reg_part.p;
    CDR_CUDA_CHECK(cudaMemsetAsync(part, 0, sizeof(double) * (4 * kRegGrid + 8), c->stream));
    double* gpos = grad ? grad + lay.positions : nullptr;
    if (w.normal != 0 && c->E > 0) {
        ++c->launches;
        k_normal_consistency<<<kRegGrid, kRegBlock, 0, c->stream>>>(c->edges.p, c->E, c->pos.p, c->tris.p, w.normal,
                                                                   gpos, part);
    }
    if (w.edge != 0 && c->E > 0) {
        ++c->launches;
        k_edge_sumsq<<<kRegGrid, kRegBlock, 0, c->stream>>>(c->edges.p, c->E, c->pos.p, part + kRegGrid);
        double* ss = part + 4 * kRegGrid;  // scratch scalar
        ++c->launches;
        k_reg_finish<<<1, 32, 0, c->stream>>>(part + kRegGrid, 1, ss);
        ++c->launches;
        k_edge_grad<<<kRegGrid, kRegBlock, 0, c->stream>>>(c->edges.p, c->E, c->pos.p, w.edge, ss, ss + 1, gpos);
    }
    const int n = c->tw * c->th;
    if (w.spec != 0 && n > 0) {
        c->reg_lum.ensure(n);
        c->reg_stats.ensure(size_t(8) * n);
        SpecParams sp{c->map_d.p, c->map_s.p, c->reg_lum.p, c->reg_stats.p, c->tw, c->th, w.spec,
                      1.0 / (2.0 * w.sigma1 * w.sigma1), 1.0 / (2.0 * w.sigma2 * w.sigma2)};
        const int nb = std::min(kRegGrid * 4, (n + kRegBlock - 1) / kRegBlock);
        ++c->launches;
        k_luminance<<<nb, kRegBlock, 0, c->stream>>>(sp);
        ++c->launches;
        k_spec_stats<<<kRegGrid, kRegBlock, 0, c->stream>>>(sp, part + 2 * kRegGrid);
        if (grad) {
            ++c->launches;
            k_spec_grad<<<nb, kRegBlock, 0, c->stream>>>(sp, grad + lay.diffuse, grad + lay.specular);
        }
    }
    if (w.roug != 0 && n > 0) {
        ++c->launches;
        k_roughness_tv<<<kRegGrid, kRegBlock, 0, c->stream>>>(c->map_r.p, c->tw, c->th, w.roug,
                                                             grad ? grad + lay.roughness : nullptr,
                                                             part + 3 * kRegGrid);
    }
    // values: normal, (edge from k_edge_grad), spec, roug
    ++c->launches;
    k_reg_finish<<<1, 128, 0, c->stream>>>(part, 4, values_dev);
    if (w.edge != 0 && c->E > 0)
        CDR_CUDA_CHECK(cudaMemcpyAsync(values_dev + 1, part + 4 * kRegGrid + 1, sizeof(double),
                                       cudaMemcpyDeviceToDevice, c->stream));
    else
        CDR_CUDA_CHECK(cudaMemsetAsync(values_dev + 1, 0, sizeof(double), c->stream));
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr
