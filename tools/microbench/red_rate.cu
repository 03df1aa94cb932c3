// Microbenchmark: L2 fp64 reduction (red.global.add.f64) throughput on B200 for the access
// patterns of the opposite-spin scatter: (a) target-sorted (a warp's 32 lanes hit 32 consecutive
// doubles), (b) scattered inside one 103 KB sigma row per CTA (lanes hit random doubles of the
// row), as a direct-from-accumulator scatter would issue them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rate red_rate.cu && ./red_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// each CTA owns a row of `row` doubles; every thread issues `per` reductions
__global__ void k_red(double* y, int64_t row, int per, int mode) {
    double* r = y + (int64_t)blockIdx.x * row;
    uint32_t s = 2654435761u * (threadIdx.x + 1) + 97u * blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < per; ++i) {
        int64_t idx;
        if (mode == 0) {  // sorted: warp-contiguous 32-double runs, runs spread over the row
            s = s * 1664525u + 1013904223u;
            const int64_t base = ((int64_t)(__shfl_sync(0xffffffffu, s, 0) % (uint32_t)(row / 32))) * 32;
            idx = base + lane;
        } else {  // scattered: independent random doubles of the row
            s = s * 1664525u + 1013904223u;
            idx = s % (uint32_t)row;
        }
        red_add(r + idx, 1.0 + w * 1e-9);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t row = 12896;  // c4 padded beta row
    const int ctas = nsm * 8, threads = 256, per = 512;
    double* y;
    cudaMalloc(&y, (size_t)ctas * row * 8);
    cudaMemset(y, 0, (size_t)ctas * row * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        k_red<<<ctas, threads>>>(y, row, per / 8, mode);
        cudaEventRecord(e0);
        k_red<<<ctas, threads>>>(y, row, per, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = (double)ctas * threads * per;
        printf("%s: %.3e reductions/s (%.1f GB/s of fp64 payload)\n", mode ? "scattered" : "sorted", n / (ms * 1e-3),
               n * 8 / (ms * 1e-3) / 1e9);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
    return 0;
}
