/*
 * topoopt_b200 — C ABI of the B200-native ADMM topology solver.
 *
 * Drop-in boundary for the hot path of the reference library `topoopt`
 * (arXiv 2512.07536, /root/reference/proj). The reference exposes a C++ API
 * (no FFI); every entry point below replaces one reference function, cited as
 * file:line under proj/. The reference-compatible C++ API
 * (include/topoopt/ headers, namespace topoopt) is a thin host layer over these.
 *
 * Conventions
 *  - plain pointers and sizes, caller-owned HOST buffers; device memory is
 *    owned by the library (or by a tp_solver handle);
 *  - every function returns a status code mirroring the reference exception
 *    taxonomy (proj/include/topoopt/errors.hpp): TP_OK, or one of TP_ERR_*;
 *    tp_last_error_message() holds the reference's message text;
 *  - edges are (i, j) int32 pairs with i < j, lexicographically sorted
 *    (Topology invariants, proj/include/topoopt/topology.hpp:16-28); packed
 *    edge vectors follow edge_index (proj/src/topology.cpp:78-84);
 *  - state vectors use the reference block layout (proj/src/admm.cpp:24-44):
 *    [g (m) | lambda | S (n*n, column-major) | y (n) | T (n*n) | z (m) | nu (m)];
 *  - all arithmetic is FP64 on the GPU (sm_100a); there is no CPU fallback:
 *    without a CUDA device every call returns TP_ERR_CUDA.
 *  - thread safety: one tp_solver per host thread; stateless calls are safe.
 */
#ifndef TOPOOPT_B200_H
#define TOPOOPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_OK 0
#define TP_ERR_INVALID_ARGUMENT 1  /* std::invalid_argument */
#define TP_ERR_INFEASIBLE 2        /* InfeasibleError */
#define TP_ERR_LINEAR_SOLVE 3      /* LinearSolveError */
#define TP_ERR_DEGENERATE 4        /* DegenerateSolutionError */
#define TP_ERR_PIVOT 5             /* PivotError (never raised: no factorisation) */
#define TP_ERR_INTERNAL 6
#define TP_ERR_CUDA 7

/* SolverConfig (proj/include/topoopt/admm.hpp:15-25) plus device options. */
typedef struct tp_config {
    double rho;            /* 1.0 */
    double epsilon;        /* 1e-6: stop when sum (x-y)^2 <= epsilon */
    int32_t max_iter;      /* 20000 */
    double alpha;          /* 2.0 */
    double weight_floor;   /* 1e-6 */
    uint64_t seed;         /* 0: warm-start annealer seed */
    double linear_tol;     /* 1e-10 (accepted; the x-step is solved exactly) */
    int32_t trace_stride;  /* 1: acf_iterate every iteration, as the reference */
    int32_t chunk;         /* 0: auto; iterations per CUDA graph launch */
    int32_t linear_solver; /* 0: closed-form x-step (default); 1: matrix-free CG on
                              the edge-incidence operator to linear_tol (hom only) */
    int32_t cg_max_iter;   /* 8: CG iterations per x-step (early exit) */
} tp_config;

/* Solution scalars (proj/include/topoopt/admm.hpp:38-53). */
typedef struct tp_result {
    int32_t iterations;
    int32_t converged;
    int32_t connected;
    int32_t repaired;
    int32_t n_edges;
    int32_t best_iter;
    double residual;
    double lambda_tilde;
    double acf;
    double lambda2;
    double lambda_n;
} tp_result;

void tp_config_default(tp_config* cfg);
/* SolverConfig::validate (proj/src/admm.cpp:186-195). */
int tp_config_validate(const tp_config* cfg);
const char* tp_last_error_message(void);
int tp_version(void);
int tp_set_device(int device);
/* tp_solve keeps, per host thread, the last homogeneous solver plan (device
 * buffers + captured iteration graphs) for the next call with the same n, r,
 * configuration, device and TPB_* environment; every call resets the whole
 * state, so results equal a fresh solver's bit for bit. This frees it. */
int tp_release_plans(void);

/* ---------------------------------------------------------------- solves */

/* topoopt::solve (proj/src/admm.cpp:356-428). warm_edges may be NULL
 * (n_warm < 0): the balanced-degree annealed start default_warm_start
 * (proj/src/admm.cpp:337-354) is generated on the host. Outputs: result,
 * up to r edges (2 ints each) and weights, trace rows (iterations x 3:
 * residual, lambda_tilde, acf_iterate) when trace != NULL (capacity
 * max_iter rows), the note string. */
int tp_solve(int32_t n, int32_t r, const tp_config* cfg, const int32_t* warm_edges, int32_t n_warm,
             tp_result* out, int32_t* edges, double* weights, double* trace, char* note,
             int32_t note_cap);

/* topoopt::solve_het on node_level_constraints(n, degrees)
 * (proj/src/admm_het.cpp:231-369, proj/src/bandwidth.cpp:116-146). */
int tp_solve_het_node(int32_t n, const int32_t* degrees, const tp_config* cfg,
                      const int32_t* warm_edges, int32_t n_warm, tp_result* out, int32_t* edges,
                      double* weights, double* trace, char* note, int32_t note_cap);

/* Warm starts (host): anneal_degree_topology (proj/src/anneal.cpp:245-273) and
 * default_warm_start (proj/src/admm.cpp:337-354); edges capacity sum(degrees)/2
 * resp. r pairs. */
int tp_anneal_degree(int32_t n, const int32_t* degrees, double t0, double cooling, int32_t steps,
                     int32_t moves_per_temp, uint64_t seed, int32_t* edges, int32_t* n_edges);
int tp_default_warm_start(int32_t n, int32_t r, uint64_t seed, int32_t* edges, int32_t* n_edges);
/* The annealing loop runs on the device when one is present (the reference's
 * random stream reproduced there; TPB_HOST_ANNEAL=1 forces the host loop).
 * First k outputs of the device std::mt19937_64 for `seed` (tests). */
int tp_device_mt19937_64(uint64_t seed, int32_t k, uint64_t* out);

/* ------------------------------------------------ batched solver handle */
/* Independent solves of one n in lockstep (edge-budget sweeps, bandwidth
 * scenarios, restarts). r[batch] (hom) or degrees[batch*n] (node-level het). */
typedef struct tp_solver tp_solver;
int tp_solver_create(int32_t n, int32_t batch, const int32_t* r, const int32_t* degrees,
                     const tp_config* cfg, tp_solver** out);
int tp_solver_destroy(tp_solver* s);
int tp_solver_set_warm(tp_solver* s, int32_t b, const int32_t* edges, int32_t n_edges);
int tp_solver_start(tp_solver* s);                  /* feasible start (admm.cpp:143-173) */
int tp_solver_iterate(tp_solver* s, int32_t k);     /* enqueue k ADMM iterations, async */
int tp_solver_sync(tp_solver* s, int32_t* all_done);
int tp_solver_run(tp_solver* s);                    /* iterate until every solve stops */
int tp_solver_finish(tp_solver* s);                 /* extraction + spectral report */
int tp_solver_result(tp_solver* s, int32_t b, tp_result* out, int32_t* edges, double* weights,
                     double* trace, char* note, int32_t note_cap);
void* tp_solver_stream(tp_solver* s);               /* cudaStream_t of the main stream */
/* {n, m, nx, neq, off_s, off_y, off_t, lambda_ix, off_z, off_nu, batch, het} */
int tp_solver_dims(tp_solver* s, int32_t* dims);
/* Device pointers of the state (X, Y, D), each batch*nx doubles. */
int tp_solver_state(tp_solver* s, double** x, double** y, double** d);
/* Host copies of the state X, Y, D of every solve (batch x nx each; NULL skips). */
int tp_solver_download(tp_solver* s, double* x, double* y, double* d);

/* Instrumentation: enqueue `reps` repetitions of one iteration phase on the
 * solver stream (0 cone projection, 1 x-step, 2 top-r, 3 trace SLEM, 4 prep)
 * so callers can time it with events; the state is left undefined. */
int tp_solver_bench_phase(tp_solver* s, int32_t phase, int32_t reps, int32_t* launches_per_rep);
int tp_solver_launches_per_iteration(tp_solver* s, int32_t* out);

/* ------------------------------------------- sharded single large instance */
/* one instance too large for one GPU's projection row-shards its
 * cone-projection GEMMs over G ranks (one process per GPU): rank k computes
 * the tiles of its n/G rows of every sign-iteration product, then an
 * in-place NCCL all-gather over NVLink completes the iterate on every rank.
 * Everything else is replicated; results are bitwise the single-GPU ones.
 * The reference has no multi-GPU path (its solve is single-threaded,
 * proj/src/admm.cpp:356-428); these calls extend the handle API.
 * Requires n > 64 and (n rounded up to 128)/128 divisible by G. */
#define TP_COMM_ID_BYTES 128
typedef struct tp_comm tp_comm;
int tp_comm_unique_id(uint8_t* id);                 /* rank 0; broadcast the bytes */
int tp_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, tp_comm** out);
int tp_comm_destroy(tp_comm* c);
int tp_solver_set_comm(tp_solver* s, tp_comm* c);   /* before tp_solver_start; NULL: unsharded */
/* this rank's lower-tile indices of an ld x ld iterate (host helper) */
int tp_shard_tiles(int32_t ld, int32_t nranks, int32_t rank, int32_t* tiles, int32_t* count);
/* CG x-step statistics of solve b's last iteration (linear_solver = 1):
 * iterations and |r| / |h|. */
int tp_solver_cg_stats(tp_solver* s, int32_t b, int32_t* iters, double* rel_res);

/* One Ozaki-scheme GEMM on the int8 tensor cores (tcgen05 kind::i8) over nmat
 * symmetric ld x ld host matrices (ld % 128 == 0): C = alpha A.B + beta E
 * (E = A if use_e), operands split into 7 digit planes with exponents ea, eb;
 * optional digit planes of C (exponent ec, nmat x 7 x ld x ld int8; 128 <= ld <= 16384). reps > 0
 * re-runs the GEMM and returns the event-timed ms per launch. */
int tp_oz_gemm(int32_t ld, int32_t nmat, const double* a, int32_t ea, const double* b, int32_t eb,
               int32_t use_e, double alpha, double beta, double* c, int8_t* cd, int32_t ec,
               int32_t reps, double* ms);

/* ---------------------------------------------------------------- capacity systems */
/* Capacity-bound (inequality) systems (proj/include/topoopt/bandwidth.hpp:41-51,
 * equality = false; intra_server_constraints / bcube_constraints): nrows rows
 * given as CSR over the n(n-1)/2 edge columns (row_ptr[nrows+1], cols),
 * upper-bound capacities caps[nrows], allowed[n(n-1)/2] mask.
 * solve_het with an explicit edge total r (proj/src/admm_het.cpp:231-369);
 * warm_edges null / n_warm < 0: anneal_topology on the system (host). */
int tp_solve_het_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                          const int32_t* caps, const int32_t* allowed, int32_t r, const tp_config* cfg,
                          const int32_t* warm_edges, int32_t n_warm, tp_result* out, int32_t* edges,
                          double* weights, double* trace, char* note, int32_t note_cap);
/* anneal_capacity_topology (proj/src/anneal.cpp:275-391), host. */
int tp_anneal_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols, const int32_t* caps,
                       const int32_t* allowed, int32_t r, double t0, double cooling, int32_t steps,
                       int32_t moves_per_temp, uint64_t seed, int32_t* edges, int32_t* n_edges);
/* project_binary_z_capped (proj/src/admm_het.cpp:125-154), v and z of n(n-1)/2. */
/* project_Y_het (proj/src/admm_het.cpp:156-171) for a capacity-bound system:
 * clamps, cones, z by project_binary_z_capped with edge total r, nu clamp. */
int tp_project_Y_het_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                              const int32_t* caps, const int32_t* allowed, int32_t r, double alpha, double rho,
                              const double* x, const double* d, double* y);
int tp_project_binary_z_capped(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                               const int32_t* caps, const int32_t* allowed, const double* v, int32_t r,
                               double* z);

/* ---------------------------------------------------------------- evaluation */
/* Consensus simulation (proj/src/consensus.cpp:29-67): errors[0..iters] of
 * x <- W x from the reference's seeded normal start, W dense row-major n x n
 * (validate_gossip rules: TP_ERR_INVALID_ARGUMENT). */
int tp_consensus_simulate(int32_t n, const double* w, int32_t dim, int32_t iters, uint64_t seed,
                          double* errors);

/* ---------------------------------------------------------------- substeps */
/* project_Y (proj/src/admm.cpp:268-277); x, d, y of length nx. */
int tp_project_Y(int32_t n, int32_t r, double alpha, double rho, const double* x, const double* d,
                 double* y);
/* project_Y_het (proj/src/admm_het.cpp:156-171), node-level system. */
int tp_project_Y_het_node(int32_t n, const int32_t* degrees, double alpha, double rho,
                          const double* x, const double* d, double* y);
/* update_X (proj/src/admm.cpp:279-293): kkt_out = [x (nx) ; mu (neq)], the
 * exact solution of the delta-regularised KKT system the reference solves
 * with BiCGSTAB. */
int tp_update_X(int32_t n, int32_t r, double alpha, double rho, const double* y, const double* d,
                double* kkt_out);
/* update_X with the paper's CG linear substep (proj/src/admm.cpp:279-293,
 * linear_tol as in the reference's update_X signature): matrix-free CG on
 * the g block of the reduced KKT system, H_gg = (1+4s) I + 3s D^T D, to
 * |r| <= linear_tol |h|. Same kkt_out layout; cg_iters / cg_rel_res report
 * the solve (either may be NULL). Fails with TP_ERR_LINEAR_SOLVE when the
 * relative residual is above 1e-8 after cg_max_iter iterations, as the
 * reference's BiCGSTAB guard (admm.cpp:287). */
int tp_update_X_cg(int32_t n, int32_t r, double alpha, double rho, const double* y, const double* d,
                   double linear_tol, int32_t cg_max_iter, double* kkt_out, int32_t* cg_iters,
                   double* cg_rel_res);
int tp_update_X_het_node(int32_t n, const int32_t* degrees, double alpha, double rho,
                         const double* y, const double* d, double* kkt_out);
/* update_duals (proj/src/admm.cpp:295-297): d += rho (x - y). */
int tp_update_duals(int64_t nx, double rho, const double* x, const double* y, double* d);
/* project_binary_z (proj/src/admm_het.cpp:116-123). */
int tp_project_binary_z(const double* v, int64_t m, int32_t r, double* z);
/* extract_topology (proj/src/admm.cpp:299-335); edges/weights capacity r. */
int tp_extract_topology(int32_t n, int32_t r, const double* g, double weight_floor,
                        int32_t* edges, double* weights, int32_t* n_edges);
/* allocate_edge_capacity (proj/src/bandwidth.cpp:28-89); caps may be NULL. */
int tp_allocate(const double* b, const int32_t* caps, int32_t n, int32_t r, double* b_unit,
                int32_t* e);
/* P independent allocations of n nodes (b: P*n, caps: P*n or NULL, r: P);
 * status[p] = TP_OK / TP_ERR_INVALID_ARGUMENT / TP_ERR_INFEASIBLE. */
int tp_allocate_batch(const double* b, const int32_t* caps, int32_t n, const int32_t* r, int32_t P,
                      double* b_unit, int32_t* e, int32_t* status);
/* spectral_report (proj/src/topology.cpp:125-144) of a dense row-major W;
 * out = {acf, lambda2, lambda_n, connected}. */
int tp_spectral_report(int32_t n, const double* w, double* out4);
/* spectral_report(gossip_matrix(t)) for a topology given as edges/weights. */
int tp_spectral_edges(int32_t n, const int32_t* edges, const double* weights, int32_t k,
                      double* out4);
/* project_psd / project_nsd (proj/src/eig.cpp:174-176), row-major n x n. */
/* sym_eig (proj/src/eig.cpp:149-172) on the device: one-sided Jacobi on the
 * shifted matrix (eig_kernels.cu). values ascending; vectors row-major, column k
 * the eigenvector of values[k]. */
int tp_sym_eig(int32_t n, const double* a, double* values, double* vectors);
int tp_project_psd(int32_t n, const double* a, double* out);
int tp_project_nsd(int32_t n, const double* a, double* out);

#ifdef __cplusplus
}
#endif

#endif /* TOPOOPT_B200_H */
