// Dependent-chain latency of float64 operations on this GPU (one thread).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = x * b + 1e-9;                  // DFMA (contracted)
        if (OP == 1) x = __dadd_rn(x, b);               // DADD
        if (OP == 2) x = __dmul_rn(x, b);               // DMUL
        if (OP == 3) x = x / b + 1.0;                   // DDIV (+add)
        if (OP == 4) x = sqrt(x) + 1.0;                 // DSQRT (+add)
        if (OP == 5) { double s, c; sincos(x, &s, &c); x = s + c + b; }
        if (OP == 6) x = atan2(x, b) + 1.0;
        if (OP == 7) x = exp(-x * x) + b;
        if (OP == 8) { float f = (float)x; x = (double)(f * 1.0001f); }
    }
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}

int main() {
    double* d; long long* c;
    cudaMalloc(&d, 8); cudaMalloc(&c, 8);
    const char* names[] = {"dfma", "dadd", "dmul", "ddiv+dadd", "dsqrt+dadd", "sincos+2add", "atan2+add", "exp(-x2)+add", "f2f roundtrip+fmul"};
    const int n = 4096;
    for (int op = 0; op < 9; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 1>>>(d, c, 1.0, 0.999, n); break;
                case 1: chain<1><<<1, 1>>>(d, c, 1.0, 1e-9, n); break;
                case 2: chain<2><<<1, 1>>>(d, c, 1.0, 0.9999999, n); break;
                case 3: chain<3><<<1, 1>>>(d, c, 1.0, 1.7, n); break;
                case 4: chain<4><<<1, 1>>>(d, c, 2.0, 0.0, n); break;
                case 5: chain<5><<<1, 1>>>(d, c, 0.3, 0.001, n); break;
                case 6: chain<6><<<1, 1>>>(d, c, 0.3, 1.1, n); break;
                case 7: chain<7><<<1, 1>>>(d, c, 0.3, 0.2, n); break;
                case 8: chain<8><<<1, 1>>>(d, c, 0.3, 0.2, n); break;
            }
            cudaDeviceSynchronize();
        }
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-20s %7.1f cycles/iter\n", names[op], double(h) / n);
    }
    return 0;
}
