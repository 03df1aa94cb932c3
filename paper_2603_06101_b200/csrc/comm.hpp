// comm.hpp — the three collectives the sharded path needs, behind one interface:
//   all_gather      x blocks -> full x before a sigma build (the only data-path collective of the
//                   opposite-spin and beta-beta terms)
//   all_reduce_sum  the small dot buffers, so every rank takes identical scalar branches
//   exchange        the alpha-alpha term's block exchange (grouped point-to-point)
// Production: NCCL over NVLink/NVSwitch, one process per GPU. Testing aid: LocalGroup runs the ranks
// as threads of one process (any device assignment, one device included) with host barriers and
// device copies, so the sharded data flow executes on real kernels without several GPUs. Its
// kernels never wait on one another: every collective synchronizes on the host first.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <memory>
#include <mutex>
#include <vector>

namespace sbg {

struct CommBlock {
    double* ptr;
    size_t count;
    int peer;
};

struct Comm {
    virtual ~Comm() = default;
    // recv[r * count .. (r+1) * count) = rank r's send; send may alias recv + rank * count
    virtual void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
    virtual void all_reduce_sum(double* buf, size_t count, cudaStream_t s) = 0;
    // point-to-point blocks, at most one per peer and direction; counts must match pairwise
    virtual void exchange(const std::vector<CommBlock>& sends, const std::vector<CommBlock>& recvs,
                          cudaStream_t s) = 0;
};

std::unique_ptr<Comm> make_nccl_comm(int world, int rank, const void* nccl_unique_id);

// in-process rank group (testing aid)
struct LocalGroup {
    explicit LocalGroup(int w) : world(w), ptr(w, nullptr), sends(w) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<const double*> ptr;
    std::vector<std::vector<CommBlock>> sends;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

std::unique_ptr<Comm> make_local_comm(LocalGroup* group, int rank);

}  // namespace sbg
