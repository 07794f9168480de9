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
    double* list_w;      // weights aligned with the list (per solve at b*list_cap), or null
    int* it_snap;        // per solve: iteration counter ictl[b*8] at selection, -1 if done (or null)
    const int* done;     // ictl (done flag at [b*8+1], iteration counter at [b*8]) or null
    int topr_cache = 0;  // grid top-r: values per CTA kept in shared memory (set by launch_topr_grid)
};

void launch_topr(const SelectArgs& a, int B, cudaStream_t st);
// keep_top_r of one large solve (B = 1, hom) over a cooperative grid:
// gh >= kTopRGridHist ints, zero before the first launch (each launch leaves
// it zero), cnt >= 2 x topr_grid_ctas(m) ints (scratch).
constexpr int kTopRGridHist = 6 * 2048;
int topr_grid_ctas(long long m);
void launch_topr_grid(const SelectArgs& a, int* gh, int* cnt, cudaStream_t st);

// project_binary_z_capped (proj/src/admm_het.cpp:125-154): ones taken in the
// order (v desc, index asc) while every capacity row through the column has
// room and the column is allowed, until r are taken. One CTA per solve:
// bitonic sort of (key, index) in the per-solve scratch, then the greedy scan.
struct CappedArgs {
    double* base;           // per-solve z values (in place), base + b*stride
    long long stride;
    long long m;
    const int* r;           // per-solve edge total
    const int* colr_ptr;    // column -> capacity rows (CSR, m+1)
    const int* colr;
    const int* caps;        // per row
    int nrows;
    const int* allowed;     // per column
    unsigned long long* keys;  // scratch B x pad
    int* idx;                  // scratch B x pad
    int* load;                 // scratch B x nrows
    int pad;                   // power of two >= m
    const int* done;           // ictl or null
};
void launch_capped_z(const CappedArgs& a, int B, cudaStream_t st);
// ascending nonzero entries of g (+ aligned weights / iteration snapshot as in SelectArgs)
void launch_compact(const double* g, long long stride, long long m, int* list, int* count, int cap,
                    int B, cudaStream_t st, double* list_w = nullptr, int* it_snap = nullptr,
                    const int* done = nullptr);

// Once-per-device opt-in for > 48 KB dynamic shared memory.
template <typename K>
inline void ensure_smem(K kernel, int bytes) {
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    (void)dev;
}

}  // namespace tpb
