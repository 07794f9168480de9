// Device-resident batched ADMM solver (one or many independent solves of the
// same n in lockstep). Host orchestration of the kernels; no CPU fallback.
#pragma once

#include <vector>

#include "admm_kernels.cuh"
#include "cone_kernels.cuh"
#include "misc_kernels.cuh"
#include "ozaki_kernels.cuh"
#include "select_kernels.cuh"
#include "slem_kernels.cuh"

namespace tpb {

struct Config {
    double rho = 1.0;
    double epsilon = 1e-6;
    int max_iter = 20000;
    double alpha = 2.0;
    double weight_floor = 1e-6;
    double linear_tol = 1e-10;  // accepted for API parity; the x-step is exact
    int trace_stride = 1;       // acf_iterate every k-th iteration (reference: 1)
    double slem_tol = 1e-6;     // trace Lanczos residual tolerance (eigenvalue error <= tol^2/gap)
    int chunk = 0;              // iterations per CUDA graph (0: auto)
    int linear_solver = 0;      // x-step: 0 closed form, 1 matrix-free CG (hom; tol = linear_tol)
    int cg_max_iter = 8;        // CG iterations launched per x-step (early exit on convergence)
};

void validate(const Config& c);

// Capacity-bound (inequality) het system (proj/include/topoopt/bandwidth.hpp:
// 41-51 with equality = false): rows over edge columns with upper-bound
// capacities and an allowed mask; no selection rows in the KKT (q = 0), the
// binary projection is project_binary_z_capped.
struct CapSystem {
    int nrows = 0;
    std::vector<int> row_ptr, cols, caps;  // rows -> edge columns (CSR)
    std::vector<int> allowed;              // per edge column
};
void phase_mark(const char* what);

// One-off spectral reports (feasible start, final topology): complete Krylov
// space up to this dimension, restarted Lanczos with this basis beyond.
constexpr int kFinalExactDim = 256;
// single homogeneous solves with at least this many candidate edges select
// top-r over the whole GPU (select_kernels.cu::topr_grid_kernel)
constexpr long long kTopRGridMin = 65536;

struct SolveResult {
    int iterations = 0;
    bool converged = false;
    bool connected = false;
    bool repaired = false;
    int best_iter = 0;
    double residual = 0.0;
    double lambda_tilde = 0.0;
    double acf = 1.0, lambda2 = 1.0, lambda_n = 0.0;
    std::vector<int> ei, ej;
    std::vector<double> w;
    std::vector<double> tr_res, tr_lam, tr_acf;
    std::string note;
};

class Solver {
   public:
    // r: per-solve edge budget (hom) ; degrees: B x n targets (het node-level).
    Solver(int n, int B, bool het, const std::vector<int>& r, const std::vector<int>& degrees,
           const Config& cfg, const CapSystem* cap = nullptr);
    ~Solver();
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;

    int n() const { return lo_.n; }
    int batch() const { return B_; }
    const Layout& layout() const { return lo_; }
    cudaStream_t stream() const { return s0_; }
    Dev& dev() { return d_; }
    const XConst& xconst() const { return c_; }

    // warm topology of solve b: ascending packed edge indices
    void set_warm(int b, const std::vector<int>& packed);
    void start();                    // feasible start of every solve
    void iterate_async(int k);       // enqueue k iterations (graphs)
    bool all_done();                 // sync + read flags
    void run_to_completion();        // chunks until every solve stops
    void finish();                   // extraction + final SLEM (hom) / het epilogue
    SolveResult result(int b) const;

    // single-step entry points for the substep API
    void upload(const double* X, const double* Y, const double* D);  // host, each B*nx or null
    void download(double* X, double* Y, double* D);
    void project_only();             // Y <- project_Y(X, D)
    void xstep_only(bool update_duals);  // X <- update_X(Y, D) [, D += rho (X - Y)]
    const double* node_dev() const { return d_.node; }
    // Enqueue `reps` repetitions of one phase of the iteration on the main
    // stream (for live per-kernel timing): 0 projection (cone GEMMs),
    // 1 x-step, 2 top-r selection, 3 trace SLEM, 4 prep, 5 x-step pass A,
    // 6 x-step pass B. Returns the number
    // of kernel launches per repetition.
    // 7: pass A + the CG solve of one x-step (linear_solver = 1).
    int bench_phase(int phase, int reps);
    // CG statistics of the last x-step of solve b: iterations, |r|/|h|
    void cg_stats(int b, int* iters, double* rel_res);
    int launches_per_iteration() const;
    // Row-shard the cone projections of this (replicated) solver over an NCCL
    // communicator of nranks ranks (OzShard, ozaki_kernels.cuh). Every rank
    // runs the same solves; results are bitwise the single-GPU ones.
    void set_shard(void* nccl_comm, int nranks, int rank);
    bool sharded() const { return shard_.nranks > 1; }
    bool eager() const;  // iterations launched without graphs (sharded)

   private:
    void alloc();
    void enqueue_iteration(bool with_slem, int parity);
    void enqueue_xstep(const Dev& d);  // pass A, node, [CG], pass B
    void enqueue_projection();
    void enqueue_select(cudaStream_t st, int parity = 0);
    void enqueue_slem_trace(cudaStream_t st, int parity = 0);
    void join_slem(cudaStream_t st);  // st waits for the last enqueued trace SLEM
    void build_graphs();
    void epilogue_hom();
    void epilogue_het();
    void final_slem(const double* packed, const int* list, const int* count, double* out);

    Layout lo_;
    int B_;
    bool het_;
    Config cfg_;
    XConst c_;
    SignSchedule sch_;
    Dev d_{};
    bool small_;
    int ld_;
    int list_cap_;
    int chunk_;
    std::vector<int> r_host_;
    std::vector<std::vector<int>> warm_;
    // device buffers
    std::vector<void*> allocs_;
    int* d_r_ = nullptr;
    int* topr_gh_ = nullptr;   // grid top-r scratch (single large hom solve)
    int* topr_cnt_ = nullptr;
    double* d_deg_ = nullptr;
    bool ozaki_ = false;        // cone GEMMs on the int8 tensor cores (else FP64 DMMA)
    bool cap_ = false;          // capacity-bound het system
    CapSystem capsys_;
    int cap_pad_ = 0;
    int *cap_colr_ptr_ = nullptr, *cap_colr_ = nullptr, *cap_caps_ = nullptr, *cap_allowed_ = nullptr;
    unsigned long long* cap_keys_ = nullptr;
    int *cap_idx_ = nullptr, *cap_load_ = nullptr;
    OzWork oz_;
    OzShard shard_;
    std::vector<void*> shard_mem_;        // cudaMalloc'd buffers of the sharded mode
    int8_t* pool_planes_[4] = {};         // the solver's own digit buffers (unsharded)
    void release_shard();
    void check_shard();
    int *list_ = nullptr, *list_count_ = nullptr;
    // Per-iteration selection output for the trace SLEM in kSets buffer sets
    // (iteration k uses set k % kSets; set 0 aliases list_/list_count_). The
    // trace SLEMs run on kLanes streams (iteration k on lane k % kLanes, each
    // lane warm-starting from its own previous report's Ritz vectors), so two
    // reports can be in flight beside the projections; the select of
    // iteration k + kSets waits for the SLEM of iteration k
    static constexpr int kSets = 4, kLanes = 2;
    int* tlist_[kSets] = {};
    int* tcount_[kSets] = {};
    double* tlw_[kSets] = {};
    int* tsnap_[kSets] = {};
    cudaEvent_t ev_slem_p_[kSets] = {};
    bool slem_pending_[kSets] = {};
    bool slem_any_[kLanes] = {};
    int slem_last_[kLanes] = {};
    // per-lane SLEM scratch (lane 0 also serves extraction and the one-offs)
    int *e_i_[kLanes] = {}, *e_j_[kLanes] = {}, *col_idx_[kLanes] = {};
    double* e_w_[kLanes] = {};
    double* basis_[kLanes] = {};     // trace Lanczos basis (B x kmax x n)
    int trace_kmax_ = 0;
    int kfin_ = 1;  // Krylov dimension of the one-off reports
    double* ritz_[kLanes] = {};      // B x 2n extreme Ritz vectors (warm start)
    int* ritz_ok_[kLanes] = {};
    int* slem_nbr_[kLanes] = {};     // het trace SLEM: node-major incidence scratch
    double* slem_nwt_[kLanes] = {};
    double* basis_final_ = nullptr;  // final report
    double* slem_out_ = nullptr;     // B x 8
    double* tmp_m_ = nullptr;        // B x m
    double* tmp_m2_ = nullptr;       // B x m
    double* worst_ = nullptr;        // B
    double* fs_scal_ = nullptr;      // B x 2
    int* h_ctl_ = nullptr;           // pinned B x 8
    // streams / graphs
    cudaStream_t s0_ = nullptr, s1_ = nullptr, s2_[kLanes] = {};
    cudaEvent_t ev_fork_ = nullptr, ev_sel_ = nullptr, ev_slem_ = nullptr;
    cudaGraphExec_t g_chunk_ = nullptr, g_one_[kSets] = {};
    int it_enqueued_ = 0;
    // results
    std::vector<SolveResult> res_;
};

}  // namespace tpb
