// finalize.cu — assembly of the position gradient once per iteration.
//
// 1. k_corner_gather: per vertex, sum the per-(triangle, corner) interior
//    accumulators written by the fused kernel: G_v = Σ b_j g_common (the direct
//    intersection response, diff_render.cpp:170-172) and H_v = Σ coeff_mu b_j h
//    (the input of the one-ring chain, :174-184); q_v = Jn(accum_v) H_v with
//    Jn = normalize_jacobian of the unnormalised normal sum (diff_render.cpp:53-54).
// 2. k_normal_chain: the reference deposits J(v,w)^T h for every w in the one
//    ring of v, with J(v,w) = Jn_v Σ_{f∋v,w} skew(d_{f,w}). Since skew(d)^T q =
//    q x d, that is grad[w] += Σ_{f∋w} (Σ_{v∈f} q_v) x d_{f,w}, with
//    d = (c-b, a-c, b-a) for corners (a, b, c) (diff_render.cpp:40-45).
//    Same sum in real arithmetic, no 9-double Jacobian per one-ring entry.
// 3. Laplacian (laplacian.cpp:21-55, losses.cpp:66-78): cotangent weights per
//    edge into a fixed CSR pattern; diagonal = -(row sum) in edge order; LV and
//    L^T(LV) as CSR SpMVs in the reference's (Eigen column) summation order.
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kBlock = 256;

__global__ void k_corner_gather(const double* __restrict__ corner, const int32_t* __restrict__ vf_start,
                                const int32_t* __restrict__ vf_list, const double* __restrict__ accum,
                                int V, double* __restrict__ grad_pos, double* __restrict__ q) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    D3 G{0, 0, 0}, Hs{0, 0, 0};
    for (int i = vf_start[v]; i < vf_start[v + 1]; ++i) {
        const double* c = corner + size_t(vf_list[i]) * 6;
        G = G + D3{c[0], c[1], c[2]};
        Hs = Hs + D3{c[3], c[4], c[5]};
    }
    grad_pos[3 * v] += G.x;
    grad_pos[3 * v + 1] += G.y;
    grad_pos[3 * v + 2] += G.z;
    D3 a = ld3(accum + 3 * v);
    double len = length(a);
    D3 out{0, 0, 0};
    if (len >= 1e-12) {
        D3 n = a / len;
        double s = 1.0 / len;
        // (I - n n^T) / len is symmetric: Jn^T H = Jn H
        out = (Hs - n * dot(n, Hs)) * s;
    }
    q[3 * v] = out.x;
    q[3 * v + 1] = out.y;
    q[3 * v + 2] = out.z;
}

__global__ void k_normal_chain(const double* __restrict__ pos, const int32_t* __restrict__ tris,
                               const int32_t* __restrict__ vf_start, const int32_t* __restrict__ vf_list,
                               const double* __restrict__ q, int V, double* __restrict__ grad_pos) {
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= V) return;
    D3 acc{0, 0, 0};
    for (int i = vf_start[w]; i < vf_start[w + 1]; ++i) {
        int f = vf_list[i] / 3, corner = vf_list[i] - 3 * f;
        int ia = tris[3 * f], ib = tris[3 * f + 1], ic = tris[3 * f + 2];
        D3 Q = ld3(q + 3 * ia) + ld3(q + 3 * ib) + ld3(q + 3 * ic);
        D3 a = ld3(pos + 3 * ia), b = ld3(pos + 3 * ib), c = ld3(pos + 3 * ic);
        D3 d = corner == 0 ? c - b : (corner == 1 ? a - c : b - a);
        acc = acc + cross(Q, d);
    }
    grad_pos[3 * w] += acc.x;
    grad_pos[3 * w + 1] += acc.y;
    grad_pos[3 * w + 2] += acc.z;
}

// cot_at (laplacian.cpp:11-19)
__device__ __forceinline__ double cot_at(D3 apex, D3 a, D3 b) {
    D3 u = a - apex, v = b - apex;
    double cos_part = dot(u, v);
    double sin_part = length(cross(u, v));
    if (sin_part < 1e-300) return __longlong_as_double(0x7ff0000000000000ULL);
    return cos_part / sin_part;
}

__global__ void k_lap_weights(const double* __restrict__ pos, const int32_t* __restrict__ tris,
                              const int4* __restrict__ edges, const int2* __restrict__ slots, int E,
                              int mode, double* __restrict__ val) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int4 ed = edges[e];
    double w = 1.0;
    if (mode == CDR_LAPLACIAN_COTANGENT) {
        w = 0.0;
        int fs[2] = {ed.z, ed.w};
        for (int k = 0; k < 2; ++k) {
            int f = fs[k];
            if (f < 0) continue;
            int opp = tris[3 * f];
            for (int j = 0; j < 3; ++j) {
                int t = tris[3 * f + j];
                if (t != ed.x && t != ed.y) opp = t;
            }
            double c = cot_at(ld3(pos + 3 * opp), ld3(pos + 3 * ed.x), ld3(pos + 3 * ed.y));
            if (!isfinite(c)) c = 1e4;
            w += 0.5 * c;
        }
        w = w < 0.0 ? 0.0 : (w > 1e4 ? 1e4 : w);
    }
    int2 s = slots[e];
    val[s.x] = w;
    val[s.y] = w;
}

// diag = -Σ w over the row in ascending column order == the reference's edge
// order for that vertex (edges sorted by (v0, v1)), so the value is identical.
__global__ void k_lap_diag(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const int32_t* __restrict__ diag_slot, int V, double* __restrict__ val) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    double d = 0.0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k)
        if (col[k] != i) d -= val[k];
    val[diag_slot[i]] = d;
}

// LV = L V, component-major (Eigen MatrixX3d column order); partial ||LV||^2
__global__ void k_lap_lv(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                         const double* __restrict__ val, const double* __restrict__ pos, int V,
                         double* __restrict__ lv, double* __restrict__ sq) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double part = 0;
    if (i < V) {
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += val[k] * pos[3 * col[k] + c];
            lv[size_t(c) * V + i] = acc;
            part += acc * acc;
        }
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0 && part != 0) atomicAdd(sq, part);
}

// G = 2 lambda L^T (LV) (L symmetric: column j of L == row j), += into grad
__global__ void k_lap_grad(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ lv, int V,
                           double two_lambda, double* __restrict__ grad_pos) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = rowptr[j]; k < rowptr[j + 1]; ++k) acc += val[k] * lv[size_t(c) * V + col[k]];
        grad_pos[3 * j + c] += two_lambda * (0.0 + acc);
    }
}

inline int blocks(long n) { return int((n + kBlock - 1) / kBlock); }

}  // namespace

void launch_finalize_positions(cdr_ctx* c, int64_t lay_pos) {
    if (c->V == 0) return;
    c->qvec.ensure(size_t(3) * c->V);
    double* gp = c->grad.p + lay_pos;
    { ++c->launches; k_corner_gather<<<blocks(c->V), kBlock, 0, c->stream>>>(c->corner_acc.p, c->vf_start.p, c->vf_list.p,
                                                            c->accum.p, c->V, gp, c->qvec.p); }
    { ++c->launches; k_normal_chain<<<blocks(c->V), kBlock, 0, c->stream>>>(c->pos.p, c->tris.p, c->vf_start.p,
                                                           c->vf_list.p, c->qvec.p, c->V, gp); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

// Fills lap_val for `mode`; if lambda != 0 also writes ||LV||^2 into
// lap_partial[0] and adds the gradient into grad_pos (V x 3) when given.
void launch_laplacian(cdr_ctx* c, int mode, double lambda, double* grad_pos) {
    const int V = c->V;
    c->lap_partial.ensure(1);
    CDR_CUDA_CHECK(cudaMemsetAsync(c->lap_partial.p, 0, sizeof(double), c->stream));
    if (V == 0) return;
    if (c->E > 0)
        { ++c->launches; k_lap_weights<<<blocks(c->E), kBlock, 0, c->stream>>>(c->pos.p, c->tris.p, c->edges.p,
                                                              c->lap_edge_slot.p, c->E, mode, c->lap_val.p); }
    { ++c->launches; k_lap_diag<<<blocks(V), kBlock, 0, c->stream>>>(c->lap_rowptr.p, c->lap_col.p, c->lap_diag_slot.p, V,
                                                    c->lap_val.p); }
    if (lambda != 0) {
        c->lap_lv.ensure(size_t(3) * V);
        { ++c->launches; k_lap_lv<<<blocks(V), kBlock, 0, c->stream>>>(c->lap_rowptr.p, c->lap_col.p, c->lap_val.p, c->pos.p,
                                                      V, c->lap_lv.p, c->lap_partial.p); }
        if (grad_pos)
            { ++c->launches; k_lap_grad<<<blocks(V), kBlock, 0, c->stream>>>(c->lap_rowptr.p, c->lap_col.p, c->lap_val.p,
                                                            c->lap_lv.p, V, 2.0 * lambda, grad_pos); }
    }
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr
