// Kernel interfaces of the ADMM iteration (projection prep, closed-form
// x-step passes, dual update, residual, bookkeeping). See DESIGN.md §3.
#pragma once

#include "common.cuh"

namespace tpb {

// Scalars of the closed-form x-step. All derived on the host
// in FP64 from rho, alpha, n and the KKT shift delta = 1e-8.
struct XConst {
    double rho, inv_rho, alpha, alpha_over_n, delta, s;  // s = 1/(1+delta)
    // homogeneous: g = f(K) h, f(k) = 1/(a + b k), K = D^T D
    double f0, c1, c2, lam_den;                           // lam_den = 1 + 2 n s
    // heterogeneous (node-level): 2x2 block G(k) of [[a1+b1 k, -s], [-s, a2]]^-1
    double g11_0, g12_0, g22_0;                           // G(0)
    double c1_11, c2_11, c1_12, c2_12, c1_22, c2_22;      // (G(q)-G(0))/q at q=n-2, 2n-2
    double g12_p, g22_p, g12_1, g22_1;                    // G12/G22 at n-2 and 2n-2
    double mu_den_p, mu_den_1;                            // (n-2)G22(n-2)+delta, (2n-2)G22(2n-2)+delta
    // matrix-free CG on H_gg = cg_a I + cg_b D^T D
    double cg_a, cg_b;
};

XConst make_xconst(int n, double alpha, double rho);

// Per-batch device views (every array has a leading batch dimension).
struct Dev {
    Layout lo;
    int B = 1;       // solves in lockstep
    int cap = 0;             // capacity-bound het system: no degree rows (q = 0)
    int het = 0;
    int nb = 0;      // 32-wide node blocks
    int ntile = 0;   // nb (nb+1) / 2 upper block pairs
    int ld = 0;      // padded projection dimension
    long long nx = 0;
    // state
    double *X, *Y, *D, *bestY, *bestScore;
    // projection
    double* A;         // B x 2 x ld x ld  (S, T inputs, symmetrized)
    double* frob_part; // B x 2 x ntile
    double* inv_scale; // B x 2   (1 / min(||A||_F, ||A||_inf))
    double* row_part;  // B x 2 x nb x n: |A| row sums of row r over column block C at [C][r]
    // x-step scratch
    double* h;         // B x m
    double* PU;        // B x nb x n  (row partials of h)
    double* PZ;        // B x nb x n  (het: row partials of h_z')
    double* PG;        // B x nb x n  (row partials of g)
    double* node;      // B x 4 x n   (hom: t; het: t_g, t_z, mu_d)
    double* tile_aux;  // B x ntile x 2  per-tile totals of the node partials of h (h_z')
    double* blk;       // B x nb x 4  diagonal tiles: tr r_S, tr r_T, sum deg over the block
    double* res_node;  // B x n       residual terms of the diagonal entries
    double* blk_inf;   // B x 2 x nb  max |A| row sum per node block (prep)
    int* cnt;          // B x cnt_stride self-resetting arrival counters (Cnt)
    int cnt_stride = 0;  // 2 nb + 2: per-block counters of pass B / prep, then per-solve
    double* res_part;  // B x ntile
    double* scal;      // B x 8 : [lambda, res, best_res, ...]
    int* ictl;         // B x 8 : [iter, done, best_iter, improved, active]
    const int* r;      // B     edge budgets
    const double* deg; // B x n (het degree targets as doubles)
    // traces (B x max_iter): residual, lambda, acf
    double *tr_res, *tr_lam, *tr_acf;
    int max_iter;
    double epsilon;
    int track_best;
    int upd_duals;   // 0: x-step only (substep API), no dual update / bookkeeping
    int bookkeep = 1;  // 0: no iteration counter / trace / stop flags (phase benchmarks)
    // matrix-free CG x-step (hom; linear_solver = 1). r lives in h (in place).
    int cg = 0;        // 1: g from CG on H_gg g = h instead of the closed form
    int cg_max = 0;    // CG iterations launched per x-step
    double cg_tol2 = 0.0;  // stop when |r|^2 <= cg_tol2 |h|^2
    int cg_grid = 1;   // launch grid: > 0 global-memory kernel, < 0 register kernel (-items)
    double* cg_x;      // B x m  solution
    double* cg_p;      // B x m  search direction
    double* cg_pq;     // B x ntile      partials of p.Hp
    double* cg_rr;     // B x 2 x ntile  partials of |r|^2: [h (pass A), r_k+1]
    double* cg_nr;     // B x nb x n     node partials of D r
    double* cg_u;      // B x 2 x n      D p (parity)
};

enum Ctl { kIter = 0, kDone = 1, kBestIter = 2, kImproved = 3 };
enum Scal { kLambda = 0, kRes = 1, kBestRes = 2 };
// arrival counter sets: block counters at [set * nb, set * nb + nb), the
// solve counter at 2 nb + set
enum Cnt { kCntB = 0, kCntP = 1 };

// v = X + D/rho; symmetrized S/T into A (ld-padded), clamps of g, lambda, y,
// nu; z-scores into Y_z. Frobenius and row-sum partials per tile; the last
// tile of the solve writes 1 / min(||A||_F, ||A||_inf) per matrix.
void launch_prep(const Dev& d, const XConst& c, cudaStream_t st);
// x-step pass A: h (packed), node partials of h (h_z') and their per-tile
// totals; diagonal tiles add the block's traces of r_S, r_T and degree sum.
void launch_xstep_a(const Dev& d, const XConst& c, cudaStream_t st);
// Matrix-free CG on H_gg g = h (hom) in one persistent cooperative launch:
// iteration k = direction pass (p, Hp inline, p.Hp partials) + update pass
// (x, r, |r|^2 and D r partials), per-solve scalars from fixed-order partial
// sums on the device, grid barriers between phases; the loop stops when
// every solve has reached |r| <= linear_tol |h| (or cg_max iterations).
void launch_xstep_cg(const Dev& d, const XConst& c, cudaStream_t st);
// Launch grid of the CG x-step for d's device and batch (Dev::cg_grid).
int cg_launch_grid(const Dev& d);
// Statistics of the last CG solve: ictl[b*8+5] = iterations,
// scal[b*8+3] = |r| / |h|.
enum CgStat { kCgIters = 5, kCgRes = 3, kCgFail = 6 };  // kCgFail: ictl, relative residual > 1e-8
// x-step pass B: node-space solve for its two node blocks (from pass A's
// partials), g (z, nu), S/T, dual update, residual partials; the last tile
// of each node block writes the block's diagonal entries and y, the last
// block of a solve lambda, the residual, trace row and best/done flags.
void launch_xstep_b(const Dev& d, const XConst& c, cudaStream_t st);
// best_y <- Y (and best_score) where the last iteration improved.
void launch_best_copy(const Dev& d, const XConst& c, cudaStream_t st);

}  // namespace tpb
