// tcgen05.ld throughput (TMEM -> registers) on one SM: 4 warps (one per TMEM
// lane quarter) each load 16 consecutive fp32 columns per instruction, sweeping
// 256 columns, repeated; reports bytes per cycle per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2605_08528_b200/csrc tmem_ld.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "dg_umma.cuh"

template <int WARPS_PER_QUARTER>
__global__ void tmem_ld_bench(long long* cyc, float* sink, int reps) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) umma::tmem_alloc(&slot, 256);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = slot;
    const uint32_t lane_base = uint32_t(32 * (warp & 3)) << 16;
    const int c0 = 64 * (warp >> 2);               // extra warps of a quarter take other columns
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 64; c += 16) {
            float v[16];
            umma::tmem_ld16(tmem + lane_base + ((c0 + c) & 255), v);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += v[i];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    sink[threadIdx.x] = acc;
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 256);
}

int main() {
    long long* cyc; float* sink;
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 4096);
    const int reps = 2000;
    for (int wq = 1; wq <= 4; wq *= 2) {
        const int threads = 128 * wq;
        for (int k = 0; k < 2; ++k) {
            if (wq == 1) tmem_ld_bench<1><<<1, threads>>>(cyc, sink, reps);
            else if (wq == 2) tmem_ld_bench<2><<<1, threads>>>(cyc, sink, reps);
            else tmem_ld_bench<4><<<1, threads>>>(cyc, sink, reps);
            cudaDeviceSynchronize();
        }
        long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double bytes = double(reps) * 64 * 4 * threads;   // 64 fp32 columns per thread per rep
        printf("warps %2d: %.1f bytes/cycle/SM (%.0f cycles)\n", threads / 32, bytes / h, double(h));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
