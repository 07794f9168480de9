// Host-side warm-start generator: the balanced-degree annealed topology the
// reference's solve()/solve_het() use when no warm start is passed
// (proj/src/anneal.cpp:189-273, AnnealConfig at proj/include/topoopt/anneal.hpp:12-20).
// It sets the ADMM start point, not the iteration (out of
// scope for kernels), and must reproduce the reference's edge set for a seed.
#pragma once

#include <cstdint>
#include <vector>

namespace tpb {

struct AnnealParams {
    double t0 = 1.0;
    double cooling = 0.995;
    int steps = 200;
    int moves_per_temp = 0;  // 0: n moves per temperature step
    uint64_t seed = 0;
};

// Connected graph realising `degrees`, tuned toward small mean path length;
// returned as ascending packed edge indices. Throws tpb::Error(kInfeasible)
// when no connected realisation exists, kInvalidArgument on bad input.
std::vector<int> anneal_degree_packed(const std::vector<int>& degrees, const AnnealParams& p);

// Same result as (i, j) pairs, lexicographic.
std::vector<std::pair<int, int>> anneal_degree_edges(const std::vector<int>& degrees,
                                                     const AnnealParams& p);

// Capacity rows (rows -> edge columns CSR, upper-bound capacities, allowed
// mask) of an inequality system.
struct CapRows {
    int nrows = 0;
    std::vector<int> row_ptr, cols, caps, allowed;
};

// anneal_topology on a capacity-bound system (proj/src/anneal.cpp:275-407),
// host; lexicographic (i, j) pairs. Throws kInfeasible / kInvalidArgument.
std::vector<std::pair<int, int>> anneal_capacity_edges(int n, const CapRows& sys, int r,
                                                       const AnnealParams& p);

}  // namespace tpb
