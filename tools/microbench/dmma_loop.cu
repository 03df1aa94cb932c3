// Microbenchmark: the sigma_ab inner loop shape (A in registers, B double-buffered from smem,
// NBT n8 blocks) without the scatter, to find the attainable DMMA rate for this instruction mix.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
template <int KS, int NBT, bool SYNC>
__global__ void __launch_bounds__(256, 1) k(double* out, int tiles) {
    constexpr int DS = NBT * 8 + 4;
    __shared__ double D[KS * 4 * DS];
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int i = tid; i < KS * 4 * DS; i += blockDim.x) D[i] = 1.0 + i * 1e-9;
    double a0[KS], a1[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) { a0[j] = 1e-3 * (j + w); a1[j] = 2e-3 * (j + g); }
    __syncthreads();
    double tot = 0;
    for (int it = 0; it < tiles; ++it) {
        double acc[NBT][4] = {};
        double b[2][NBT];
#pragma unroll
        for (int nb = 0; nb < NBT; ++nb) b[0][nb] = D[t * DS + g + nb * 8];
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int cur = j & 1;
            if (j + 1 < KS) {
#pragma unroll
                for (int nb = 0; nb < NBT; ++nb) b[cur ^ 1][nb] = D[(4 * (j + 1) + t) * DS + g + nb * 8];
            }
#pragma unroll
            for (int nb = 0; nb < NBT; ++nb) dmma16(acc[nb], a0[j], a1[j], b[cur][nb]);
        }
#pragma unroll
        for (int nb = 0; nb < NBT; ++nb) tot += acc[nb][0] + acc[nb][1] + acc[nb][2] + acc[nb][3];
        if (SYNC) __syncthreads();
    }
    out[blockIdx.x * blockDim.x + tid] = tot;
}
template <int KS, int NBT, bool SYNC>
void run(int warps, double* out, int nsm) {
    int tiles = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<KS, NBT, SYNC><<<nsm, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    k<KS, NBT, SYNC><<<nsm, warps * 32>>>(out, tiles);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 4 * KS * NBT * (double)tiles * warps * nsm;
    printf("KS=%d NBT=%d sync=%d warps=%d: %.2f TFLOP/s\n", KS, NBT, (int)SYNC, warps, fl / ms / 1e9);
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 1 << 24);
    for (int w : {4, 7, 8}) { run<13, 4, false>(w, out, nsm); run<13, 4, true>(w, out, nsm); }
    for (int w : {8}) { run<17, 4, false>(w, out, nsm); run<17, 2, false>(w, out, nsm); run<17, 4, true>(w, out, nsm); run<17, 2, true>(w, out, nsm); }
    run<17, 4, false>(12, out, nsm);
    return 0;
}
