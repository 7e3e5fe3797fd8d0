// Bit-exactness of the shared-reciprocal fp64 division (common.cuh,
// operator/(D3, double)) and of div_pi (x / pi) against the compiler's `/`: random numerators and
// divisors over and around its fast-path range [2^-500, 2^501) (outside it the
// operator takes the plain divisions), plus exact and near-1 quotients.
// Built and run by tests/test_division_exact.py.
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "../../paper_2103_15208_b200/csrc/common.cuh"

using cdr::D3;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ double rnd(uint64_t h, int emin, int emax) {
    const uint64_t m = h & 0xfffffffffffffULL;
    const int e = emin + int((h >> 52) % uint64_t(emax - emin + 1));
    const uint64_t sign = (h >> 63) << 63;
    return __longlong_as_double((long long)(sign | (uint64_t(e + 1023) << 52) | m));
}
__global__ void k(uint64_t seed, long long n, int emin, int emax, unsigned long long* bad, double* ex) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix(seed ^ (4 * i)), h2 = mix(seed ^ (4 * i + 1)), h3 = mix(seed ^ (4 * i + 2)),
                       h4 = mix(seed ^ (4 * i + 3));
        double b = rnd(h4, emin, emax);
        D3 a{rnd(h1, emin, emax), rnd(h2, emin, emax), rnd(h3, emin, emax)};
        if ((h1 & 0xff) == 0) a.x = b * double(int(h2 & 0xff) + 1);          // exact quotients
        if ((h1 & 0xff) == 1) b = 1.0 + double(h2 & 0xffff) * 0x1p-52;       // near-1 divisors
        if ((h1 & 0xff) == 2) a.y = 0.0;                                      // a zero numerator
        const D3 q = a / b;
        const double r[4] = {a.x / b, a.y / b, a.z / b, a.x / cdr::kPiD};
        const double g[4] = {q.x, q.y, q.z, cdr::div_pi(a.x)};
        for (int c = 0; c < 4; ++c)
            if (__double_as_longlong(g[c]) != __double_as_longlong(r[c]) && !(r[c] != r[c] && g[c] != g[c])) {
                if (atomicAdd(bad, 1ull) == 0) {
                    ex[0] = c == 0 || c == 3 ? a.x : (c == 1 ? a.y : a.z);
                    ex[1] = c == 3 ? cdr::kPiD : b;
                    ex[2] = g[c];
                    ex[3] = r[c];
                }
            }
    }
}
int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : (1ll << 30);
    unsigned long long* bad;
    double* ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 32);
    const int ranges[][2] = {{-500, 500}, {-30, 30}, {-2, 2}, {-520, -480}, {480, 520}, {-1022, 1023}};
    unsigned long long total = 0;
    for (int t = 0; t < 6; ++t) {
        *bad = 0;
        k<<<148 * 16, 256>>>(0x1234567ull + t, n, ranges[t][0], ranges[t][1], bad, ex);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("CUDA error\n");
            return 2;
        }
        printf("range [2^%d, 2^%d]: %lld x 4 quotients, %llu differ", ranges[t][0], ranges[t][1], n, *bad);
        if (*bad) printf(" (e.g. %a / %a = %a, '/' gives %a)", ex[0], ex[1], ex[2], ex[3]);
        printf("\n");
        total += *bad;
    }
    printf(total ? "FAIL\n" : "OK\n");
    return total ? 1 : 0;
}
