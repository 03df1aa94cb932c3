// selftest.cu — verifies on the device the DMMA fragment layouts assumed by sigma_ab.cu and
// sigma_ss.cu (common.cuh), against a host product. Returns 0 when both shapes match exactly.
#include <cmath>
#include <vector>
#include <nccl.h>

#include "comm.hpp"
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {
__global__ void k_mma_probe(const double* A, const double* B, double* C16, double* C8) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double c[4] = {0, 0, 0, 0};
    dmma_16x8x4(c, A[g * 4 + t], A[(g + 8) * 4 + t], B[t * 8 + g]);
    C16[g * 8 + 2 * t] = c[0];
    C16[g * 8 + 2 * t + 1] = c[1];
    C16[(g + 8) * 8 + 2 * t] = c[2];
    C16[(g + 8) * 8 + 2 * t + 1] = c[3];
    double e[2] = {0, 0};
    dmma_8x8x4(e, A[g * 4 + t], B[t * 8 + g]);
    C8[g * 8 + 2 * t] = e[0];
    C8[g * 8 + 2 * t + 1] = e[1];
}
}  // namespace

int run_mma_selftest() {
    std::vector<double> A(64), B(32), C16(128), C8(64);
    for (int i = 0; i < 64; ++i) A[i] = (double)((i * 7) % 13) - 6.0;
    for (int i = 0; i < 32; ++i) B[i] = (double)((i * 5) % 11) - 5.0;
    double *dA, *dB, *dC16, *dC8;
    SBG_CUDA(cudaMalloc(&dA, 64 * 8));
    SBG_CUDA(cudaMalloc(&dB, 32 * 8));
    SBG_CUDA(cudaMalloc(&dC16, 128 * 8));
    SBG_CUDA(cudaMalloc(&dC8, 64 * 8));
    SBG_CUDA(cudaMemcpy(dA, A.data(), 64 * 8, cudaMemcpyHostToDevice));
    SBG_CUDA(cudaMemcpy(dB, B.data(), 32 * 8, cudaMemcpyHostToDevice));
    k_mma_probe<<<1, 32>>>(dA, dB, dC16, dC8);
    SBG_LAUNCH_CHECK();
    SBG_CUDA(cudaMemcpy(C16.data(), dC16, 128 * 8, cudaMemcpyDeviceToHost));
    SBG_CUDA(cudaMemcpy(C8.data(), dC8, 64 * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC16);
    cudaFree(dC8);
    int bad = 0;
    for (int i = 0; i < 16; ++i)
        for (int j = 0; j < 8; ++j) {
            double s = 0;
            for (int k = 0; k < 4; ++k) s += A[i * 4 + k] * B[k * 8 + j];
            if (C16[i * 8 + j] != s) ++bad;
            if (i < 8 && C8[i * 8 + j] != s) ++bad;
        }
    return bad;
}

// The production collectives (NcclComm, comm.hpp) on a one-rank NCCL communicator: all-gather into
// a larger buffer, in-place all-reduce, and a grouped send/recv to self, on the caller's current device. Multi-rank NCCL needs one
// GPU per rank; this pins the link against libnccl and the call sequence on the box that has one.
// Returns the number of wrong entries.
int run_nccl_selftest() {
    // RAII: buffers and the stream are released even when an NCCL call throws
    struct DevBuf {
        double* p = nullptr;
        explicit DevBuf(size_t n) { SBG_CUDA(cudaMalloc(&p, n * 8)); }
        ~DevBuf() { cudaFree(p); }
    };
    struct Stream {
        cudaStream_t s = nullptr;
        Stream() { SBG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
        ~Stream() {
            if (s) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        }
    };
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw DeviceError("ncclGetUniqueId failed");
    const size_t n = 4099;
    std::vector<double> h(n), out(n);
    for (size_t i = 0; i < n; ++i) h[i] = 0.5 * (double)i - 17.25;
    Stream st;
    DevBuf a(n), b(n), c(n);
    auto comm = make_nccl_comm(1, 0, &id);
    SBG_CUDA(cudaMemcpy(a.p, h.data(), n * 8, cudaMemcpyHostToDevice));
    SBG_CUDA(cudaMemset(b.p, 0, n * 8));
    SBG_CUDA(cudaMemset(c.p, 0, n * 8));
    int bad = 0;
    comm->all_gather(a.p, b.p, n, st.s);
    comm->all_reduce_sum(b.p, n, st.s);
    comm->exchange({CommBlock{b.p, n, 0}}, {CommBlock{c.p, n, 0}}, st.s);
    SBG_CUDA(cudaStreamSynchronize(st.s));
    SBG_CUDA(cudaMemcpy(out.data(), c.p, n * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) bad += out[i] != h[i];
    return bad;
}

}  // namespace sbg
