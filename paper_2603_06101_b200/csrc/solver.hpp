// solver.hpp — device-resident SBCI1 driver: the reference's solve_n_states_sbci1 /
// solve_state_sbci1 / sbci1_step_impl (sbci1.hpp:45-579) with every length-n_det vector in HBM
// and every vector pass fused (vec.cu); host code only runs the reference's scalar logic on
// all-reduced dot products, so every rank takes identical branches.
#pragma once

#include <functional>
#include <optional>
#include <vector>

#include "context.hpp"
#include "host_math.hpp"

namespace sbg {

struct TraceRec {
    int state = 0, t = 0;
    double energy = 0, dE = 0, res_norm = 0, x_norm = 0, kinetic = 0;
    uint64_t matvecs = 0;
    int restart_reason = -1;
    double b = 0, c = 0;
};

struct StateResult {
    int state = 0;
    double energy = 0.0;
    int iterations = 0, restarts = 0;
    double final_residual = 0.0;
    DBuf vector;  // unit norm, padded local layout
};

struct MultiStateResult {
    std::vector<StateResult> pairs;  // sorted by energy
    uint64_t matvecs = 0;
    long total_iterations = 0;
    int total_restarts = 0, hx_refreshes = 0, peak_vectors = 0;
    double wall_time_s = 0.0;
};

MultiStateResult solve_n_states_sbci1(Context& ctx, int n, const SolverConfig& cfg,
                                      const std::function<void(const TraceRec&)>& trace);

}  // namespace sbg
