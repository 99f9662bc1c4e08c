// Odd/even symmetry of CUDA's float64 sincos and atan2 (bitwise), plus the
// composite wrap used by the neighbour rows: atan2(sin(-d), cos(-d)) == -atan2(sin d, cos d).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}
__global__ void check(unsigned long long* bad, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h = mix(i);
        double d = ((h >> 11) * (1.0 / 9007199254740992.0)) * 20.0 - 10.0;   // |yaw difference| <= 10 rad
        if (i % 7 == 0) d = double(int64_t(h % 2000) - 1000) * 0.0078125;   // dyadic values
        double s1, c1, s2, c2;
        sincos(d, &s1, &c1);
        sincos(-d, &s2, &c2);
        if (s2 != -s1 || c2 != c1) atomicAdd(bad, 1ULL);
        const double w1 = atan2(s1, c1), w2 = atan2(s2, c2);
        if (w2 != -w1) atomicAdd(bad + 1, 1ULL);
    }
}
int main() {
    unsigned long long* b; cudaMalloc(&b, 16); cudaMemset(b, 0, 16);
    const long long n = 1LL << 30;
    check<<<148 * 8, 256>>>(b, n);
    unsigned long long h[2]; cudaMemcpy(h, b, 16, cudaMemcpyDeviceToHost);
    printf("%lld samples: sincos symmetry violations %llu, wrap antisymmetry violations %llu\n", n, h[0], h[1]);
    return 0;
}
