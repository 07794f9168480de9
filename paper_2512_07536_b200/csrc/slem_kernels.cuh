#pragma once

#include "common.cuh"

namespace tpb {

// SLEM (second-largest eigenvalue modulus) of W = I - L(g) for the weights g
// of the listed edges; spectral_report semantics (proj/src/topology.cpp:125-144).
struct SlemArgs {
    int n;
    long long m;
    const double* g;       // packed weights, per solve at g + b*stride
    long long stride;
    const int* list;       // ascending nonzero edge indices, per solve at list + b*list_cap
    const int* count;
    int list_cap;
    // scratch (global, per solve)
    int* e_i;              // list_cap
    int* e_j;
    double* e_w;
    int* col_idx;          // list_cap
    double* basis;         // kmax x n per solve in global memory, or null: shared memory
    int kmax;              // Krylov dimension per cycle (<= n-1); >= n-1: exact mode
    int max_restarts;      // explicit restarts from the extreme Ritz vectors
    int min_steps;         // restarted mode: matvecs before the first residual test
    int check_every;       // plain (trace) Lanczos: residual tests every this many steps of a cycle (0: 16)
    double noise;          // warm start: weight of the fixed random component
    double tol;            // residual tolerance relative to the spectral scale
    // optional warm start: ritz[b*2n ..] = previous (v_min, v_max); ritz_ok[b]
    double* ritz;
    int* ritz_ok;
    // outputs: out[b*8 + {0:acf, 1:lambda2, 2:lambda_n, 3:connected, 4:steps, 5:converged}]
    double* out;
    // trace mode: acf -> tr_acf[b*max_iter + it], it = it_snap[b] (the
    // iteration recorded by the select kernel; < 0 skips the solve) or, without
    // it_snap, ictl[b*8] (skipped when ictl[b*8+1] marks the solve done)
    double* tr_acf;
    const int* ictl;
    const int* it_snap;
    const double* gw;      // weights aligned with the list (gw + b*list_cap), or null: g[list[e]]
    int max_iter;
    int plain;             // trace mode: plain Lanczos (no reorthogonalisation), basis write-only
    int* nbr;              // plain mode, dense supports: node-major incidence scratch (2 list_cap per solve)
    double* nwt;
    int smem_nm;           // plain mode: entries of a node-major incidence kept in shared memory (set by launch_slem)
    int cluster;           // plain mode: CTAs per solve (a thread-block cluster; 0/1: one CTA)
};

// n <= kSmallDense: dense Householder tridiagonalisation in shared memory
// (exact, no iteration); larger n: Lanczos (exact or restarted, see SlemArgs).
constexpr int kSmallDense = 128;
void launch_slem(const SlemArgs& a, int B, cudaStream_t st);
// Krylov dimension of a one-off plain-Lanczos report at n > kFinalExactDim:
// up to kOneOffKrylov steps in one cycle (no restart in the usual case: a
// restart from two Ritz vectors discards the recurrence), capped so the
// trace kernel's shared memory fits.
constexpr int kOneOffKrylov = 1024;
// CTAs of the thread-block cluster that runs a one-off report of one solve
// (slem_trace_kernel: node slices per CTA, q exchanged through DSMEM)
constexpr int kOneOffCluster = 8;
int slem_oneoff_kmax(int n);
// dynamic shared memory of launch_slem (basis_in_smem: a.basis == null)
size_t slem_smem_bytes(int n, int kmax, bool basis_in_smem);

// Dense symmetric W (row-major n x n), full spectrum Lanczos with full
// reorthogonalisation; out[0..4) = {acf, lambda2, lambda_n, connected}.
// deflate=1 when W 1 = 1 (gossip matrix): the Krylov space is built on 1-perp.
void launch_slem_dense(const double* w, int n, double* basis, double* out, int deflate, cudaStream_t st);

}  // namespace tpb
