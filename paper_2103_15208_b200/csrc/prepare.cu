// prepare.cu — per-iteration geometry (the GradContext constructor,
// diff_render.hpp:29-30 / render.hpp:48-49): face normals, area-weighted vertex
// normals (mesh.cpp:65-95), bounding box + default t_min (bvh.cpp:92), and the
// LBVH: Morton codes -> radix sort -> Karras hierarchy -> bottom-up refit.
// Replaces the host SAH build (bvh.cpp:90-208) that the reference runs on every
// total_loss call.
#include "kernels.h"

namespace cdr {
namespace {

constexpr int kBlock = 256;

__global__ void k_face_normals(const double* __restrict__ pos, const int32_t* __restrict__ tris,
                               int T, double* __restrict__ fn) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= T) return;
    int a = tris[3 * f], b = tris[3 * f + 1], c = tris[3 * f + 2];
    D3 p0 = ld3(pos + 3 * a), p1 = ld3(pos + 3 * b), p2 = ld3(pos + 3 * c);
    D3 n = cross(p1 - p0, p2 - p0);  // Mesh::face_normal_unnormalized (mesh.hpp:30-33)
    fn[3 * f] = n.x;
    fn[3 * f + 1] = n.y;
    fn[3 * f + 2] = n.z;
}

// Gather over incident faces in ascending face order: the same summation order
// as the reference's face loop, so normals are bit-identical.
__global__ void k_vertex_normals(const double* __restrict__ fn, const int32_t* __restrict__ vf_start,
                                 const int32_t* __restrict__ vf_list, int V,
                                 double* __restrict__ normals, double* __restrict__ accum) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    D3 acc{0, 0, 0};
    int s = vf_start[v], e = vf_start[v + 1];
    for (int i = s; i < e; ++i) acc = acc + ld3(fn + 3 * (vf_list[i] / 3));
    D3 n{0, 0, 1};
    double len = length(acc);
    if (len >= 1e-12) {
        n = acc / len;
    } else {
        for (int i = s; i < e; ++i) {  // degenerate sum: first incident face normal
            D3 m = ld3(fn + 3 * (vf_list[i] / 3));
            double l = length(m);
            if (l < 1e-30) continue;
            n = m / l;
            break;
        }
    }
    normals[3 * v] = n.x;
    normals[3 * v + 1] = n.y;
    normals[3 * v + 2] = n.z;
    accum[3 * v] = acc.x;
    accum[3 * v + 1] = acc.y;
    accum[3 * v + 2] = acc.z;
}

__global__ void k_bbox_partial(const double* __restrict__ pos, int V, double* __restrict__ part) {
    __shared__ double s[6][kBlock];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            double x = pos[3 * v + k];
            lo[k] = fmin(lo[k], x);
            hi[k] = fmax(hi[k], x);
        }
    for (int k = 0; k < 3; ++k) {
        s[k][threadIdx.x] = lo[k];
        s[3 + k][threadIdx.x] = hi[k];
    }
    __syncthreads();
    for (int st = kBlock / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st)
            for (int k = 0; k < 3; ++k) {
                s[k][threadIdx.x] = fmin(s[k][threadIdx.x], s[k][threadIdx.x + st]);
                s[3 + k][threadIdx.x] = fmax(s[3 + k][threadIdx.x], s[3 + k][threadIdx.x + st]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) part[6 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

// min / max are exact in any order: one CTA folds the per-block partials
__global__ void __launch_bounds__(kBlock) k_bbox_final(const double* __restrict__ part, int nb, int T,
                                                      double cam_abs_max, SceneInfo* __restrict__ info) {
    __shared__ double s[6][kBlock];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int b = threadIdx.x; b < nb; b += kBlock)
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], part[6 * b + k]);
            hi[k] = fmax(hi[k], part[6 * b + 3 + k]);
        }
    for (int k = 0; k < 3; ++k) {
        s[k][threadIdx.x] = lo[k];
        s[3 + k][threadIdx.x] = hi[k];
    }
    __syncthreads();
    for (int st = kBlock / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st)
            for (int k = 0; k < 3; ++k) {
                s[k][threadIdx.x] = fmin(s[k][threadIdx.x], s[k][threadIdx.x + st]);
                s[3 + k][threadIdx.x] = fmax(s[3 + k][threadIdx.x], s[3 + k][threadIdx.x + st]);
            }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    for (int k = 0; k < 3; ++k) {
        lo[k] = s[k][0];
        hi[k] = s[3 + k][0];
    }
    SceneInfo si;
    double mag = cam_abs_max;
    for (int k = 0; k < 3; ++k) {
        si.lo[k] = lo[k];
        si.hi[k] = hi[k];
        if (T > 0) mag = fmax(mag, fmax(fabs(lo[k]), fabs(hi[k])));
    }
    D3 d{hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    double diag = T > 0 ? length(d) : 0.0;
    si.t_min = T > 0 ? 1e-4 * diag : 1e-8;
    // fp32 ray error is ~1e-7 x |coordinates|; pad boxes far beyond it
    si.pad = 1e-5 * diag + 4e-6 * mag + 1e-30;
    *info = si;
}

__device__ __forceinline__ unsigned expand_bits10(unsigned v) {
    v = (v * 0x00010001u) & 0xFF0000FFu;
    v = (v * 0x00000101u) & 0x0F00F00Fu;
    v = (v * 0x00000011u) & 0xC30C30C3u;
    v = (v * 0x00000005u) & 0x49249249u;
    return v;
}

__global__ void k_morton(const double* __restrict__ pos, const int32_t* __restrict__ tris, int T,
                         const SceneInfo* __restrict__ info, unsigned long long* __restrict__ keys) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= T) return;
    SceneInfo si = *info;
    unsigned q[3];
    for (int k = 0; k < 3; ++k) {
        double a = pos[3 * tris[3 * f] + k], b = pos[3 * tris[3 * f + 1] + k],
               c = pos[3 * tris[3 * f + 2] + k];
        double cen = 0.5 * (fmin(a, fmin(b, c)) + fmax(a, fmax(b, c)));
        double ext = si.hi[k] - si.lo[k];
        double u = ext > 0 ? (cen - si.lo[k]) / ext : 0.5;
        int qi = int(u * 1024.0);
        q[k] = unsigned(min(max(qi, 0), 1023));
    }
    unsigned m = (expand_bits10(q[0]) << 2) | (expand_bits10(q[1]) << 1) | expand_bits10(q[2]);
    keys[f] = (static_cast<unsigned long long>(m) << 32) | unsigned(f);
}

__device__ __forceinline__ int delta(const unsigned long long* __restrict__ keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    return __clzll(keys[i] ^ keys[j]);
}

// Karras 2012, "Maximizing parallelism in the construction of BVHs": internal
// node i covers a key range whose split is the highest differing bit.
__global__ void k_hierarchy(const unsigned long long* __restrict__ keys, int n,
                            BNode* __restrict__ nodes, int32_t* __restrict__ parent_internal,
                            int32_t* __restrict__ parent_leaf) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int s = 0;
    for (int div = 2;; div <<= 1) {
        int t = (l + div - 1) / div;
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
        if (t <= 1) break;
    }
    int gamma = i + s * d + min(d, 0);
    int left, right;
    if (min(i, j) == gamma) {
        left = ~gamma;
        parent_leaf[gamma] = i;
    } else {
        left = gamma;
        parent_internal[gamma] = i;
    }
    if (max(i, j) == gamma + 1) {
        right = ~(gamma + 1);
        parent_leaf[gamma + 1] = i;
    } else {
        right = gamma + 1;
        parent_internal[gamma + 1] = i;
    }
    nodes[i].k = make_int4(left, right, 0, 0);
    if (i == 0) parent_internal[0] = -1;
}

__device__ __forceinline__ void write_child_box(BNode* node, int side, const float b[6]) {
    float* f = reinterpret_cast<float*>(node);
    int o = side * 6;
    for (int k = 0; k < 6; ++k) __stcg(f + o + k, b[k]);
}

// One thread per leaf walks to the root; the second arrival at a node merges
// its two child boxes (flags reset before launch).
__global__ void k_refit(const unsigned long long* __restrict__ keys, const double* __restrict__ pos,
                        const int32_t* __restrict__ tris, int n, const SceneInfo* __restrict__ info,
                        const int32_t* __restrict__ parent_internal,
                        const int32_t* __restrict__ parent_leaf, int32_t* __restrict__ flags,
                        BNode* __restrict__ nodes, TriRec* __restrict__ recs) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n) return;
    int f = int(keys[l] & 0xffffffffull);
    int v0 = tris[3 * f], v1 = tris[3 * f + 1], v2 = tris[3 * f + 2];
    D3 p0 = ld3(pos + 3 * v0), p1 = ld3(pos + 3 * v1), p2 = ld3(pos + 3 * v2);
    TriRec r;
    r.a = make_double2(p0.x, p0.y);
    r.b = make_double2(p0.z, p1.x);
    r.c = make_double2(p1.y, p1.z);
    r.d = make_double2(p2.x, p2.y);
    r.e = p2.z;
    r.tri = f;
    r.pad = 0;
    recs[l] = r;
    if (n == 1) return;
    double pad = info->pad;
    float box[6];
    box[0] = __double2float_rd(fmin(p0.x, fmin(p1.x, p2.x)) - pad);
    box[1] = __double2float_rd(fmin(p0.y, fmin(p1.y, p2.y)) - pad);
    box[2] = __double2float_rd(fmin(p0.z, fmin(p1.z, p2.z)) - pad);
    box[3] = __double2float_ru(fmax(p0.x, fmax(p1.x, p2.x)) + pad);
    box[4] = __double2float_ru(fmax(p0.y, fmax(p1.y, p2.y)) + pad);
    box[5] = __double2float_ru(fmax(p0.z, fmax(p1.z, p2.z)) + pad);
    int code = ~l;
    int p = parent_leaf[l];
    while (p >= 0) {
        int side = (__ldcg(&nodes[p].k.x) == code) ? 0 : 1;
        write_child_box(&nodes[p], side, box);
        __threadfence();
        if (atomicAdd(&flags[p], 1) == 0) return;  // sibling not done yet
        __threadfence();
        const float* fb = reinterpret_cast<const float*>(&nodes[p]);
        float o[12];
        for (int k = 0; k < 12; ++k) o[k] = __ldcg(fb + k);
        for (int k = 0; k < 3; ++k) {
            box[k] = fminf(o[k], o[6 + k]);
            box[3 + k] = fmaxf(o[3 + k], o[9 + k]);
        }
        code = p;
        p = parent_internal[p];
    }
}

// ---------------------------------------------------------------------------
// Radix sort of the LBVH keys (Morton << 32 | face index), hand-written.
//
// The keys are created in face order, so a STABLE sort on the 30 Morton bits
// alone yields exactly the order of a full 62-bit sort (ties by face index):
// four 8-bit LSD passes (bits 32-39, 40-47, 48-55, 56-61) instead of eight.
// One histogram kernel counts all four digits in a single read of the keys;
// each pass is then ONE "onesweep" kernel (Merrill & Garland, decoupled
// look-back): a CTA takes the next 4,096-key tile (dynamic tile id, so every
// tile it looks back on is already running), ranks its keys stably per digit
// with __match_any_sync warp multi-split, publishes its per-digit counts, sums
// the predecessors' counts by look-back, stages the tile sorted by digit in
// shared memory and writes each digit's run contiguously.
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortPasses = 4;
constexpr unsigned kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1;

__device__ __forceinline__ int sort_digit(unsigned long long k, int pass) {
    return int((k >> (32 + 8 * pass)) & 0xffu);
}

// all four digit histograms (hist[pass][256]) in one read; also clears the
// look-back status words and the per-pass tile counters of the sort
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const unsigned long long* __restrict__ keys, int n,
                                                           unsigned* __restrict__ hist, unsigned* __restrict__ status,
                                                           int n_status, unsigned* __restrict__ tile_ctr) {
    __shared__ unsigned h[kSortPasses][256];
    for (int i = threadIdx.x; i < kSortPasses * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const unsigned long long k = keys[i];
#pragma unroll
        for (int p = 0; p < kSortPasses; ++p) atomicAdd(&h[p][sort_digit(k, p)], 1u);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_status; i += stride) status[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x < kSortPasses) tile_ctr[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < kSortPasses * 256; i += blockDim.x)
        if ((&h[0][0])[i]) atomicAdd(hist + i, (&h[0][0])[i]);
}

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const unsigned long long* __restrict__ in,
                                                           unsigned long long* __restrict__ out, int n, int pass,
                                                           const unsigned* __restrict__ hist,
                                                           unsigned* __restrict__ status, unsigned* __restrict__ tile_ctr) {
    __shared__ unsigned long long stage[kSortTile];
    __shared__ unsigned whist[kSortWarps][257];  // per warp and digit; 256 = past the end of the keys
    __shared__ unsigned digit_base[256];         // global position of the tile's first key of each digit
    __shared__ unsigned tile_excl[257];          // tile-local exclusive scan over digits
    __shared__ int s_tile;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = int(atomicAdd(tile_ctr + pass, 1u));
    for (int i = tid; i < kSortWarps * 257; i += kSortThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    const int tile = s_tile;
    const size_t base = size_t(tile) * kSortTile + size_t(w) * 32 * kSortItems;
    // warp-striped items: item j of lane l is key base + j*32 + l (index order = (warp, j, lane))
    unsigned long long k[kSortItems];
    int rank[kSortItems], dg[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const size_t i = base + size_t(j) * 32 + lane;
        k[j] = i < size_t(n) ? in[i] : ~0ull;
        dg[j] = i < size_t(n) ? sort_digit(k[j], pass) : 256;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const unsigned peers = __match_any_sync(0xffffffffu, dg[j]);
        const int leader = __ffs(peers) - 1;
        unsigned b = 0;
        if (lane == leader) {
            b = whist[w][dg[j]];
            whist[w][dg[j]] = b + __popc(peers);
        }
        b = __shfl_sync(0xffffffffu, b, leader);
        rank[j] = int(b) + __popc(peers & ((1u << lane) - 1u));
        __syncwarp();
    }
    __syncthreads();
    // per digit: counts of the tile, and each warp's exclusive prefix inside it
    unsigned cnt = 0;
    for (int d = tid; d < 257; d += kSortThreads) {
        unsigned run = 0;
        for (int ww = 0; ww < kSortWarps; ++ww) {
            const unsigned c = whist[ww][d];
            whist[ww][d] = run;
            run += c;
        }
        if (d < 256) cnt = run;
    }
    // publish this tile's aggregate per digit (thread d = digit d)
    unsigned* st = status + (size_t(pass) * gridDim.x + tile) * 256;
    __stcg(st + tid, (tile == 0 ? kFlagPrefix : kFlagAgg) | cnt);
    // exclusive scans over the 256 digits, both at once: the tile's counts
    // (tile-local run starts) and the global histogram (run starts in `out`)
    __shared__ unsigned wsum[2][kSortWarps];
    unsigned a = cnt, g = hist[pass * 256 + tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned ta = __shfl_up_sync(0xffffffffu, a, o), tg = __shfl_up_sync(0xffffffffu, g, o);
        if (lane >= o) {
            a += ta;
            g += tg;
        }
    }
    if (lane == 31) {
        wsum[0][w] = a;
        wsum[1][w] = g;
    }
    __syncthreads();
    unsigned pa = 0, pg = 0;
    for (int ww = 0; ww < w; ++ww) {
        pa += wsum[0][ww];
        pg += wsum[1][ww];
    }
    tile_excl[tid] = pa + a - cnt;
    if (tid == 255) tile_excl[256] = pa + a;  // the past-the-end keys stage after every valid one
    unsigned excl = pg + g - hist[pass * 256 + tid];
    // + the counts of all earlier tiles (decoupled look-back)
    if (tile > 0) {
        unsigned prev = 0;
        for (int t = tile - 1; t >= 0; --t) {
            const volatile unsigned* sp = status + (size_t(pass) * gridDim.x + t) * 256 + tid;
            unsigned x;
            do {
                x = *sp;
            } while ((x & ~kValMask) == 0u);
            prev += x & kValMask;
            if (x & kFlagPrefix) break;
        }
        __stcg(st + tid, kFlagPrefix | (prev + cnt));
        excl += prev;
    }
    digit_base[tid] = excl;
    __syncthreads();
    // stage the tile sorted by digit (stable), then write each digit's run
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        CDR_DCHECK(tile_excl[dg[j]] + whist[w][dg[j]] + rank[j] < unsigned(kSortTile));
        stage[tile_excl[dg[j]] + whist[w][dg[j]] + rank[j]] = k[j];
    }
    __syncthreads();
    const int valid = int(min(size_t(kSortTile), size_t(n) - size_t(tile) * kSortTile));
    for (int i = tid; i < valid; i += kSortThreads) {
        const unsigned long long x = stage[i];
        const int d = sort_digit(x, pass);
        CDR_DCHECK(digit_base[d] + (unsigned(i) - tile_excl[d]) < unsigned(n));
        out[digit_base[d] + (unsigned(i) - tile_excl[d])] = x;
    }
}

inline int blocks(long n, int b = kBlock) { return int((n + b - 1) / b); }

}  // namespace

void launch_prepare(cdr_ctx* c, double cam_abs_max) {
    cudaStream_t s = c->stream;
    const int V = c->V, T = c->T;
    if (T > 0) { ++c->launches; k_face_normals<<<blocks(T), kBlock, 0, s>>>(c->pos.p, c->tris.p, T, c->fnormal.p); }
    if (V > 0)
        { ++c->launches; k_vertex_normals<<<blocks(V), kBlock, 0, s>>>(c->fnormal.p, c->vf_start.p, c->vf_list.p, V,
                                                      c->normals.p, c->accum.p); }
    launch_bvh(c, cam_abs_max);
}

// Bounding box + t_min + LBVH only (no normals): also the build of the
// geometry-only context behind cdr_self_intersects.
void launch_bvh(cdr_ctx* c, double cam_abs_max) {
    cudaStream_t s = c->stream;
    const int V = c->V, T = c->T;
    c->info.ensure(1);
    int nb = std::max(1, std::min(blocks(V), 1184));
    c->bbox_partial.ensure(size_t(nb) * 6);
    { ++c->launches; k_bbox_partial<<<nb, kBlock, 0, s>>>(c->pos.p, V, c->bbox_partial.p); }
    { ++c->launches; k_bbox_final<<<1, kBlock, 0, s>>>(c->bbox_partial.p, nb, T, cam_abs_max, c->info.p); }
    if (T == 0) return;

    c->keys.ensure(T);
    c->keys_alt.ensure(T);
    c->recs.ensure(T);
    c->nodes.ensure(std::max(1, T - 1));
    c->parent_internal.ensure(std::max(1, T - 1));
    c->parent_leaf.ensure(T);
    c->refit_flag.ensure(std::max(1, T - 1));
    { ++c->launches; k_morton<<<blocks(T), kBlock, 0, s>>>(c->pos.p, c->tris.p, T, c->info.p, c->keys.p); }
    // radix sort (above): keys -> keys_alt -> keys -> keys_alt -> keys
    const int tiles = (T + kSortTile - 1) / kSortTile;
    const int n_status = kSortPasses * tiles * 256;
    c->sort_tmp.ensure(sizeof(unsigned) * (size_t(kSortPasses) * 256 + kSortPasses + size_t(n_status)));
    unsigned* hist = reinterpret_cast<unsigned*>(c->sort_tmp.p);
    unsigned* tile_ctr = hist + kSortPasses * 256;
    unsigned* status = tile_ctr + kSortPasses;
    CDR_CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(unsigned) * kSortPasses * 256, s));
    { ++c->launches; k_sort_hist<<<std::max(1, std::min(blocks(T, kSortThreads), 148)), kSortThreads, 0, s>>>(
          c->keys.p, T, hist, status, n_status, tile_ctr); }
    unsigned long long* buf[2] = {c->keys.p, c->keys_alt.p};
    for (int pass = 0; pass < kSortPasses; ++pass) {
        ++c->launches;
        k_sort_pass<<<tiles, kSortThreads, 0, s>>>(buf[pass & 1], buf[(pass + 1) & 1], T, pass, hist, status,
                                                   tile_ctr);
    }
    if (T > 1) {
        { ++c->launches; k_hierarchy<<<blocks(T - 1), kBlock, 0, s>>>(c->keys.p, T, c->nodes.p,
                                                     c->parent_internal.p, c->parent_leaf.p); }
        CDR_CUDA_CHECK(cudaMemsetAsync(c->refit_flag.p, 0, sizeof(int32_t) * (T - 1), s));
    }
    { ++c->launches; k_refit<<<blocks(T), kBlock, 0, s>>>(c->keys.p, c->pos.p, c->tris.p, T, c->info.p,
                                         c->parent_internal.p, c->parent_leaf.p, c->refit_flag.p,
                                         c->nodes.p, c->recs.p); }
    CDR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace cdr
