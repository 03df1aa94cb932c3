// Microbenchmark: what the per-tile hand-offs of K6 cost the FP64 tensor pipe.
// The K6 loop shape (KS k-steps, NBT n8 blocks, A in registers, B fragments from shared memory,
// accumulators staged to a shared G tile in the epilogue) under four synchronisation regimes:
//   0  free-running warps (no barrier)                   -> the ceiling for this instruction mix
//   1  one block-wide barrier per tile (lockstep)        -> today's K6: DREADY + EMPTY rendezvous
//   2  two block-wide barriers per tile
//   3  barrier per PAIR of warps sharing nothing (skewed halves: warps 0-3 and 4-7 on separate
//      named barriers, the second half started half a tile late)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_sync dmma_sync.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
template <int KS, int NBT, int MODE, int JUNK = 0>
__global__ void __launch_bounds__(256, 1) k(double* out, int tiles) {
    constexpr int DS = NBT * 8 + 4, GS = NBT * 8 + 8;
    extern __shared__ double sm[];
    double* D = sm;                       // [2][KS*4][DS]
    double* G = sm + 2 * KS * 4 * DS;     // [2][128][GS]
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int i = tid; i < 2 * KS * 4 * DS; i += blockDim.x) D[i] = 1.0 + i * 1e-9;
    double a0[KS], a1[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) { a0[j] = 1e-3 * (j + w); a1[j] = 2e-3 * (j + g); }
    __syncthreads();
    const int r0 = 16 * w + g;
    int junk = tid;
    const int half = w >> 2;
    if (MODE == 3 && half == 1) {  // start the second half late: ~half a tile of DMMA time
        long long t0 = clock64();
        while (clock64() - t0 < 16 * KS * NBT * 2) {}
    }
    for (int it = 0; it < tiles; ++it) {
        const double* Dt = D + (it & 1) * KS * 4 * DS;
        double* Gt = G + (it & 1) * 128 * GS;
        if (MODE == 1 || MODE == 2) bar_sync(1, 256);
        if (MODE == 2) bar_sync(2, 256);
        if (MODE == 3) bar_sync(1 + half, 128);
        double acc[NBT][4] = {};
        double b[2][NBT];
#pragma unroll
        for (int nb = 0; nb < NBT; ++nb) b[0][nb] = Dt[t * DS + g + nb * 8];
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int cur = j & 1;
            if (j + 1 < KS) {
#pragma unroll
                for (int nb = 0; nb < NBT; ++nb) b[cur ^ 1][nb] = Dt[(4 * (j + 1) + t) * DS + g + nb * 8];
            }
#pragma unroll
            for (int nb = 0; nb < NBT; ++nb) dmma16(acc[nb], a0[j], a1[j], b[cur][nb]);
            // JUNK dependent integer selects per k-step: do the non-DMMA instructions of a DMMA warp
            // hide behind the other warp's DMMAs, or do they add to the tile time?
#pragma unroll
            for (int q = 0; q < JUNK; ++q)
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(junk) : "r"(it + q));
        }
#pragma unroll
        for (int nb = 0; nb < NBT; ++nb) {
            const int col = nb * 8 + 2 * t;
            *reinterpret_cast<double2*>(Gt + r0 * GS + col) = make_double2(acc[nb][0], acc[nb][1]);
            *reinterpret_cast<double2*>(Gt + (r0 + 8) * GS + col) = make_double2(acc[nb][2], acc[nb][3]);
        }
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + tid] = G[tid] + junk;
}
template <int KS, int NBT, int MODE, int JUNK = 0>
void run(double* out, int nsm) {
    const int tiles = 4000;
    const size_t smem = (2 * KS * 4 * (NBT * 8 + 4) + 2 * 128 * (NBT * 8 + 8)) * 8;
    cudaFuncSetAttribute(k<KS, NBT, MODE, JUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<KS, NBT, MODE, JUNK><<<nsm, 256, smem>>>(out, 10);
    cudaEventRecord(e0);
    k<KS, NBT, MODE, JUNK><<<nsm, 256, smem>>>(out, tiles);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 4 * KS * NBT * (double)tiles * 8 * nsm;
    printf("KS=%d NBT=%d mode=%d junk=%d: %.2f TFLOP/s  (%s)\n", KS, NBT, MODE, JUNK, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 1 << 24);
    run<16, 4, 0>(out, nsm); run<16, 4, 1>(out, nsm); run<16, 4, 2>(out, nsm); run<16, 4, 3>(out, nsm);
    run<16, 8, 0>(out, nsm); run<16, 8, 1>(out, nsm); run<16, 8, 3>(out, nsm);
    run<12, 4, 0>(out, nsm); run<12, 4, 1>(out, nsm);
    run<16, 4, 0, 4>(out, nsm); run<16, 4, 0, 8>(out, nsm); run<16, 4, 0, 16>(out, nsm); run<16, 4, 0, 32>(out, nsm);
    run<16, 4, 1, 8>(out, nsm); run<16, 4, 1, 16>(out, nsm);
    return 0;
}
