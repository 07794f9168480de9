// Deterministic per-node incidence of an ascending edge list (one CTA).
#pragma once

#include "common.cuh"

namespace tpb {

// Builds, for the ascending packed edge list `list[0..ne)`:
//   ei/ej/ew   endpoints and weights g[list[e]] (aligned: g[e])
//   rowptr     edges e with ei[e] == v are rowptr[v]..rowptr[v+1] (ascending e)
//   colptr/cidx edges with ej[e] == v, cidx[colptr[v]..colptr[v+1]) ascending e
// so "column part then row part" visits a node's incident edges in ascending
// edge index — the accumulation order of the reference's loops over pairs.
// rowptr/colptr/cur live in shared memory (n+1, n+1, n ints).
__device__ inline void build_csr(int n, int ne, const int* list, const double* g, bool aligned, int* ei,
                                 int* ej, double* ew, int* rowptr, int* colptr, int* cur, int* cidx,
                                 int* iscr) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int e = tid; e < ne; e += nthr) {
        int i, j;
        edge_pair(n, list[e], i, j);
        ei[e] = i;
        ej[e] = j;
        ew[e] = aligned ? g[e] : g[list[e]];
    }
    for (int v = tid; v < n; v += nthr) {
        rowptr[v] = 0;
        colptr[v] = 0;
    }
    __syncthreads();
    for (int e = tid; e < ne; e += nthr) {
        atomicAdd(&rowptr[ei[e]], 1);
        atomicAdd(&colptr[ej[e]], 1);
    }
    __syncthreads();
    int run_r = 0, run_c = 0;
    for (int base = 0; base < n; base += nthr) {
        const int v = base + tid;
        const int cr = v < n ? rowptr[v] : 0, cc = v < n ? colptr[v] : 0;
        int tr, tc;
        const int er = block_exclusive_scan(cr, iscr, &tr);
        const int ec = block_exclusive_scan(cc, iscr, &tc);
        if (v < n) {
            rowptr[v] = run_r + er;
            colptr[v] = run_c + ec;
            cur[v] = run_c + ec;
        }
        run_r += tr;
        run_c += tc;
        __syncthreads();
    }
    if (tid == 0) {
        rowptr[n] = run_r;
        colptr[n] = run_c;
    }
    __syncthreads();
    // stable counting sort by second endpoint: warps take turns in order
    const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
    for (int base = 0; base < ne; base += nthr) {
        const int e = base + tid;
        const int key = e < ne ? ej[e] : -1 - lane;  // unique dummy keys
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int rank = __popc(peers & ((1u << lane) - 1));
        const int leader = __ffs(peers) - 1;
        for (int ww = 0; ww < nw; ++ww) {
            if (wid == ww) {
                int basepos = 0;
                if (e < ne && lane == leader) {
                    basepos = cur[key];
                    cur[key] = basepos + __popc(peers);
                }
                basepos = __shfl_sync(0xffffffffu, basepos, leader);
                if (e < ne) cidx[basepos + rank] = e;
            }
            __syncthreads();
        }
    }
    __syncthreads();
}

}  // namespace tpb
