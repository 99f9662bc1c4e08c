// Branch-free float64 division / square root (the fast paths of CUDA's IEEE
// sequences without the slow-path branch) vs the IEEE operators, bitwise.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_08528_b200/csrc/dg_fastmath.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}
__device__ __forceinline__ double rnd(uint64_t k, double lo_exp, double hi_exp) {
    const uint64_t h = mix(k);
    const double u = (h >> 11) * (1.0 / 9007199254740992.0);
    const double e = lo_exp + (hi_exp - lo_exp) * ((mix(h) >> 11) * (1.0 / 9007199254740992.0));
    const double v = exp2(e) * (1.0 + u);
    return (h & 1) ? -v : v;
}

__global__ void check(unsigned long long* bad_div, unsigned long long* bad_sqrt, long long n, int range) {
    const double lo = range == 0 ? -40.0 : -1000.0, hi = range == 0 ? 40.0 : 1000.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = rnd(2 * i, lo, hi), b = rnd(2 * i + 1, lo, hi);
        if (dg::ddiv(a, b) != a / b) atomicAdd(bad_div, 1ULL);
        const double s = fabs(a);
        if (dg::dsqrt(s) != sqrt(s)) atomicAdd(bad_sqrt, 1ULL);
        // exact zeros and integers
        const double z = double(i % 1000);
        if (dg::ddiv(z, b) != z / b) atomicAdd(bad_div, 1ULL);
        if (dg::dsqrt(z) != sqrt(z)) atomicAdd(bad_sqrt, 1ULL);
    }
}

template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = dg::ddiv(x, b) + 1.0;
        if (OP == 1) x = dg::dsqrt(x) + 1.0;
    }
    cyc[0] = clock64() - t0;
    out[0] = x;
}

int main() {
    unsigned long long *bd, *bs;
    cudaMalloc(&bd, 8); cudaMalloc(&bs, 8);
    for (int range = 0; range < 2; ++range) {
        cudaMemset(bd, 0, 8); cudaMemset(bs, 0, 8);
        const long long n = 1LL << 28;
        check<<<148 * 8, 256>>>(bd, bs, n, range);
        cudaDeviceSynchronize();
        unsigned long long hd, hs;
        cudaMemcpy(&hd, bd, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hs, bs, 8, cudaMemcpyDeviceToHost);
        printf("range 2^[%s]: %lld pairs: ddiv mismatches %llu, dsqrt mismatches %llu\n",
               range == 0 ? "-40,40" : "-1000,1000", 2 * n, hd, hs);
    }
    double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 8);
    long long h;
    lat<0><<<1, 1>>>(d, c, 1.0, 1.7, 4096); lat<0><<<1, 1>>>(d, c, 1.0, 1.7, 4096); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("ddiv+dadd  %.1f cycles/iter\n", h / 4096.0);
    lat<1><<<1, 1>>>(d, c, 2.0, 0.0, 4096); lat<1><<<1, 1>>>(d, c, 2.0, 0.0, 4096); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dsqrt+dadd %.1f cycles/iter\n", h / 4096.0);
    return 0;
}
