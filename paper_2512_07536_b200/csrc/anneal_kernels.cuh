// Device warm-start annealer (proj/src/anneal.cpp:189-241): simulated
// annealing over double edge swaps minimising the mean shortest-path length,
// with the reference's random stream reproduced on the device so the result
// is the reference's edge set for the same seed.
#pragma once

#include <utility>
#include <vector>

#include "common.cuh"

namespace tpb {

struct AnnealParams;

// Capacity veto of anneal_capacity_topology (proj/src/anneal.cpp:357-385):
// packed columns -> rows CSR, per-row capacities and the loads of the
// starting edge set, per-column allowed mask.
struct CapVeto {
    std::vector<int> allowed, cr_ptr, cr, caps, load;
};

// Anneal the connected edge list `es` (n nodes) in place on the current
// device, vetoing swaps that break `veto` when given; returns false when no
// device is usable (caller falls back to the host annealer). Throws
// tpb::Error on CUDA failures.
bool anneal_device(int n, std::vector<std::pair<int, int>>& es, const AnnealParams& p,
                   const CapVeto* veto = nullptr);

// First k outputs of the device mt19937_64 for `seed` (tests against the
// host std::mt19937_64).
void device_mt19937_64(uint64_t seed, int k, uint64_t* out);

}  // namespace tpb
