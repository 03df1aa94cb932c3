// solver.hpp — device-resident SBCI1 driver: the reference's solve_n_states_sbci1 /
// solve_state_sbci1 / sbci1_step_impl (sbci1.hpp:45-579) with every length-n_det vector in HBM
// and every vector pass fused (vec.cu); host code only runs the reference's scalar logic on
// all-reduced dot products, so every rank takes identical branches.
#pragma once

#include <functional>
#include <limits>
#include <optional>
#include <vector>

#include "context.hpp"
#include "host_math.hpp"

namespace sbg {

// TraceRecord (trace.hpp:22-44); fields a method does not produce stay NaN
struct TraceRec {
    static constexpr double absent = std::numeric_limits<double>::quiet_NaN();
    int method = 1;         // 1 sbci1, 2 sbci2, 3 davidson
    int state = 0, t = 0;
    int pair_partner = -1;  // alpha+1 for sbci2 rows
    double energy = absent, dE = absent, res_norm = absent, x_norm = absent, kinetic = absent;
    uint64_t matvecs = 0;
    int restart_reason = -1;
    double b = absent, c = absent;
    double b_ab = absent, b_ba = absent, b_bb = absent, c_ab = absent, c_ba = absent, c_bb = absent;
    double a_ab = absent, a_ba = absent;
    double energy_partner = absent, x_norm_partner = absent, res_norm_partner = absent;
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

constexpr int detail_max_roots = 9;  // deflation sets of up to 8 states (precondition pass)

MultiStateResult solve_n_states_sbci1(Context& ctx, int n, const SolverConfig& cfg,
                                      const std::function<void(const TraceRec&)>& trace);
// davidson_solve(op, nroots, cfg) (davidson.hpp:53-244): block Davidson cross-check
// max_space: DavidsonConfig::max_space (davidson.hpp:19-38), 0 = 12 * nroots
MultiStateResult davidson_solve(Context& ctx, int nroots, const SolverConfig& cfg,
                                const std::function<void(const TraceRec&)>& trace, int max_space = 0);
// solve_n_states_sbci2 (sbci2.hpp:527-623): pair-sequential lowest-n driver
MultiStateResult solve_n_states_sbci2(Context& ctx, int n, const SolverConfig& cfg,
                                      const std::function<void(const TraceRec&)>& trace);

}  // namespace sbg
