#pragma once

#include "common.cuh"

namespace tpb {

struct SelectArgs {
    double* base;        // per-solve vector to select on (in place)
    const double* gbase; // het: clamped weights to compact for the SLEM
    long long stride;    // elements between solves
    long long m;
    const int* r;        // per-solve budget
    int binary;          // 0: thin weights (keep values), 1: binary z
    int* list;           // per-solve ascending list of kept nonzero edges
    int* list_count;
    int list_cap;
    const int* done;     // ictl (done flag at [b*8+1]) or null
};

void launch_topr(const SelectArgs& a, int B, cudaStream_t st);
void launch_compact(const double* g, long long stride, long long m, int* list, int* count, int cap,
                    int B, cudaStream_t st);

// Once-per-device opt-in for > 48 KB dynamic shared memory.
template <typename K>
inline void ensure_smem(K kernel, int bytes) {
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    (void)dev;
}

}  // namespace tpb
