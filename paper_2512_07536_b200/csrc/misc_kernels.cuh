#pragma once

#include "admm_kernels.cuh"

namespace tpb {

// Feasible start, part 1 (per solve, one CTA): degrees of the warm topology,
// g0 = 1/(dmax+1) on its edges, lap(i,i) by sequential accumulation.
// node_out[b*4n + 3n + i] = lap(i,i); fs_scal[b*2] = g0.
void launch_feasible_a(const Dev& d, const int* warm_list, const int* warm_count, int warm_cap,
                       double* fs_scal, cudaStream_t st);
// Part 2 (tiles): lambda0 = max(1e-3, 1 - acf), S, T, y, lambda, het z/nu.
void launch_feasible_b(const Dev& d, const XConst& c, const double* slem_out, const double* fs_scal,
                       cudaStream_t st);

// Alg. 1 (proj/src/bandwidth.cpp:28-89), one warp per problem.
// status[p]: 0 ok, 1 invalid argument, 2 infeasible.
void launch_allocate(const double* b, const int* caps, int n, const int* r, int P, double* b_unit,
                     int* e, int* status, cudaStream_t st);

// Extraction (proj/src/admm.cpp:299-335): on the already-thinned support in
// `list` (ascending), node sums in the reference's accumulation order, the
// uniform down-scaling, and outputs; scaled weights also written packed to
// `packed_out` (zeroed beforehand) for the final SLEM.
void launch_extract(int n, long long m, const double* g, long long stride, const int* list,
                    const int* count, int list_cap, int* out_i, int* out_j, double* out_w,
                    double* packed_out, double* worst_out, int* cidx_scratch, int B,
                    cudaStream_t st);

// t = (g > floor) ? g : 0 (support of extract_topology)
void launch_floor_mask(const double* g, long long stride, long long m, double floor, double* t,
                       int B, cudaStream_t st);

}  // namespace tpb
