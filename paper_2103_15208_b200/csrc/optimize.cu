// optimize.cu — the optimiser step on resident parameters: SURVEY §8(f) row 3.
//
//   adam_step (adam.cpp:9-54) + apply (params.cpp:103-134): one element-wise
//     kernel over the ParamLayout; the gradient is the device gradient of the
//     last loss pass, the moments stay on the device, texture and light
//     segments are updated and clamped in place (the maps the next pass
//     renders), the position segment becomes a device displacement.
//   robust_evolve (evolve.cpp:19-53): candidates pos + s * displacement for
//     s = 1, 1/2, ..., 2^-8, rejected on a triangle area <= 1e-12 (min over
//     faces, mesh.hpp:34) or a self-intersection (selfint.cu).
//
// Bit-exact with the reference: same fp64 operation order (-fmad=false), the
// bias corrections 1 - beta^step are evaluated on the host with the same pow.
#include <algorithm>
#include <cstring>

#include "kernels.h"

namespace cdr {
namespace {

constexpr int kOptBlock = 256;
constexpr double kAlphaMin = 0.01;  // material.hpp:10

__global__ void k_nonfinite(const double* __restrict__ g, int64_t n, int* __restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(kOptBlock) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kOptBlock)
        if (!isfinite(g[i])) *flag = 1;
}

struct AdamArgs {
    const double* grad;
    double* m;
    double* v;
    int64_t n;
    cdr_layout lay;
    int64_t n_pos;  // 3V
    int64_t n_tex;  // texels
    double beta1, beta2, eps, lr_pos, lr_tex, lr_light, corr1, corr2;
    double* disp;   // V x 3
    double* map_d;  // 3 n_tex
    double* map_s;  // 3 n_tex
    double* map_r;  // n_tex
    double* light;  // 3
};

// adam.cpp:36-51 for element i of the layout
__global__ void k_adam(AdamArgs a) {
    for (int64_t i = blockIdx.x * int64_t(kOptBlock) + threadIdx.x; i < a.n; i += int64_t(gridDim.x) * kOptBlock) {
        const cdr_layout& L = a.lay;
        double lr = a.lr_tex, lo = 0.0, hi = 1.0;
        double* param = nullptr;
        if (i >= L.positions && i < L.positions + a.n_pos) {
            lr = a.lr_pos;
        } else if (i >= L.diffuse && i < L.diffuse + 3 * a.n_tex) {
            param = a.map_d + (i - L.diffuse);
        } else if (i >= L.specular && i < L.specular + 3 * a.n_tex) {
            param = a.map_s + (i - L.specular);
        } else if (i >= L.roughness && i < L.roughness + a.n_tex) {
            param = a.map_r + (i - L.roughness);
            lo = kAlphaMin;
        } else if (L.light >= 0 && i >= L.light && i < L.light + 3) {
            param = a.light + (i - L.light);
            lr = a.lr_light;
            hi = 1e30;  // intensity only floored at 0
        } else {
            continue;
        }
        const double g = a.grad[i];
        const double m = a.beta1 * a.m[i] + (1.0 - a.beta1) * g;
        const double v = a.beta2 * a.v[i] + (1.0 - a.beta2) * g * g;
        a.m[i] = m;
        a.v[i] = v;
        const double m_hat = m / a.corr1, v_hat = v / a.corr2;
        const double delta = -lr * m_hat / (sqrt(v_hat) + a.eps);
        if (!param) {
            a.disp[i - L.positions] = delta;
        } else {
            const double x = *param + delta;
            *param = x < lo ? lo : (hi < x ? hi : x);  // std::clamp
        }
    }
}

// min over faces of Mesh::face_area (mesh.hpp:34) as a non-negative double's
// bit pattern (its integer order is the numeric order)
__global__ void k_min_area(const double* __restrict__ pos, const int32_t* __restrict__ tris, int T,
                           unsigned long long* __restrict__ out) {
    unsigned long long best = ~0ull;
    for (int f = blockIdx.x * kOptBlock + threadIdx.x; f < T; f += gridDim.x * kOptBlock) {
        const D3 a = ld3(pos + 3 * tris[3 * f]);
        const double area = 0.5 * length(cross(ld3(pos + 3 * tris[3 * f + 1]) - a, ld3(pos + 3 * tris[3 * f + 2]) - a));
        const unsigned long long b = (unsigned long long)__double_as_longlong(area);
        best = b < best ? b : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x < best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(out, best);
}

// candidate = mesh.positions[v] + displacement[v] * s (evolve.cpp:40-41)
__global__ void k_candidate(const double* __restrict__ pos, const double* __restrict__ disp, double s, int64_t n,
                            double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(kOptBlock) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kOptBlock)
        out[i] = pos[i] + disp[i] * s;
}

__global__ void k_any_nonzero(const double* __restrict__ d, int64_t n, int* __restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(kOptBlock) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kOptBlock)
        if (d[i] != 0) *flag = 1;
}

int grid_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + kOptBlock - 1) / kOptBlock, 148 * 8))); }

}  // namespace

bool any_nonfinite(cdr_ctx* c, const double* g, int64_t n) {
    DBuf<int>& flag = c->scr_flag;
    flag.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
    ++c->launches;
    k_nonfinite<<<grid_for(n), kOptBlock, 0, c->stream>>>(g, n, flag.p);
    int h = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return h != 0;
}

void launch_adam(cdr_ctx* c, const double* grad, double corr1, double corr2) {
    AdamArgs a{};
    a.grad = grad;
    a.m = c->adam_m.p;
    a.v = c->adam_v.p;
    a.n = c->adam_lay.total;
    a.lay = c->adam_lay;
    a.n_pos = 3 * int64_t(c->V);
    a.n_tex = int64_t(c->tw) * c->th;
    a.beta1 = c->adam_cfg.beta1;
    a.beta2 = c->adam_cfg.beta2;
    a.eps = c->adam_cfg.epsilon;
    a.lr_pos = c->adam_cfg.lr_positions;
    a.lr_tex = c->adam_cfg.lr_textures;
    a.lr_light = c->adam_cfg.lr_light;
    a.corr1 = corr1;
    a.corr2 = corr2;
    a.disp = c->adam_disp.p;
    a.map_d = c->map_d.p;
    a.map_s = c->map_s.p;
    a.map_r = c->map_r.p;
    a.light = c->adam_light.p;
    ++c->launches;
    k_adam<<<grid_for(a.n), kOptBlock, 0, c->stream>>>(a);
    CDR_CUDA_CHECK(cudaGetLastError());
}

double min_triangle_area(cdr_ctx* c, const double* pos) {
    DBuf<unsigned long long>& out = c->scr_u64;
    out.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(out.p, 0xff, sizeof(unsigned long long), c->stream));
    if (c->T > 0) {
        ++c->launches;
        k_min_area<<<grid_for(c->T), kOptBlock, 0, c->stream>>>(pos, c->tris.p, c->T, out.p);
    }
    unsigned long long h = ~0ull;
    CDR_CUDA_CHECK(cudaMemcpyAsync(&h, out.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (h == ~0ull) return 1e300;  // evolve.cpp:12: best = 1e300 with no faces
    double d;
    std::memcpy(&d, &h, sizeof(d));
    return d;
}

void launch_candidate(cdr_ctx* c, const double* pos, const double* disp, double s, double* out) {
    const int64_t n = 3 * int64_t(c->V);
    ++c->launches;
    k_candidate<<<grid_for(n), kOptBlock, 0, c->stream>>>(pos, disp, s, n, out);
    CDR_CUDA_CHECK(cudaGetLastError());
}

bool any_nonzero(cdr_ctx* c, const double* d, int64_t n) {
    DBuf<int>& flag = c->scr_flag;
    flag.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
    ++c->launches;
    k_any_nonzero<<<grid_for(n), kOptBlock, 0, c->stream>>>(d, n, flag.p);
    int h = 0;
    CDR_CUDA_CHECK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CDR_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return h != 0;
}

}  // namespace cdr
