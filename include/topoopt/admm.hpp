// Homogeneous ADMM solver (proj/include/topoopt/admm.hpp:15-101): same names,
// signatures, value semantics and exceptions; solve() and the substeps run on
// the GPU behind the C ABI (include/topoopt_b200.h).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "topoopt/dense.hpp"
#include "topoopt/solvers.hpp"
#include "topoopt/sparse.hpp"
#include "topoopt/topology.hpp"

namespace topoopt {

struct SolverConfig {
    double rho = 1.0;
    double epsilon = 1e-6;       // threshold on the combined squared residual
    int max_iter = 20000;
    double alpha = 2.0;          // rank-one shift making the gap constraint an LMI
    double weight_floor = 1e-6;  // extraction drops weights at or below this
    std::uint64_t seed = 0;
    double linear_tol = 1e-10;   // relative inner-solver tolerance (CG x-step)
    // device extension: 0 exact closed-form x-step, 1 the paper's matrix-free
    // CG linear substep to linear_tol (homogeneous solves)
    int linear_solver = 0;
    void validate() const;
};

// {"rho", "epsilon", "max_iter", "alpha", "weight_floor", "seed",
//  "linear_tol"}: any subset; unknown keys and non-objects are rejected.
SolverConfig solver_config_from_json(const std::string& text);

struct TraceRow {
    int iter = 0;
    double residual = 0.0;
    double lambda_tilde = 0.0;
    double acf_iterate = 1.0;
};

struct Solution {
    Topology topology;
    Matrix w;
    double lambda_tilde = 0.0;
    double acf_value = 1.0;
    bool converged = false;
    bool connected = false;
    bool repaired = false;
    double residual = 0.0;
    int iterations = 0;
    double wall_time_ms = 0.0;
    std::string note;
    std::vector<TraceRow> trace;
    std::string trace_csv() const;  // "iter,residual,lambda_tilde,acf_iterate"
};

// The saddle-point matrix [[I, A^T], [A, -1e-8 I]] of a problem, assembled on
// the host on first use (the GPU solver is matrix-free and never needs it):
// rows()/cols() are known without assembly; every other member assembles the
// CSC matrix once (thread-safe) and forwards to it.
class KktMatrix {
   public:
    KktMatrix() = default;
    KktMatrix(int dim, std::function<SparseMatrix()> build);
    int rows() const { return dim_; }
    int cols() const { return dim_; }
    const SparseMatrix& matrix() const;
    operator const SparseMatrix&() const { return matrix(); }
    int nnz() const { return matrix().nnz(); }
    const std::vector<int>& col_ptr() const { return matrix().col_ptr(); }
    const std::vector<int>& row_idx() const { return matrix().row_idx(); }
    const std::vector<double>& values() const { return matrix().values(); }
    void multiply(const Vec& x, Vec& y) const { matrix().multiply(x, y); }
    Vec multiply(const Vec& x) const { return matrix().multiply(x); }
    Matrix to_dense() const { return matrix().to_dense(); }
    void save(std::ostream& out) const { matrix().save(out); }

   private:
    struct State;
    int dim_ = 0;
    std::shared_ptr<State> st_;
};

// ILU(0) factors of a KktMatrix, computed on first use.
class KktIlu {
   public:
    KktIlu() = default;
    explicit KktIlu(KktMatrix kkt);
    const IluFactors& factors() const;
    operator const IluFactors&() const { return factors(); }
    void apply(const Vec& r, Vec& z) const { factors().apply(r, z); }

   private:
    struct State;
    std::shared_ptr<State> st_;
};

// Block layout and equality data of the homogeneous problem (admm.hpp:59-69).
struct ProblemData {
    int n = 0, m = 0, r = 0;
    double alpha = 2.0, rho = 1.0;
    int nx = 0;   // m+1 + n^2 + n + n^2
    int neq = 0;  // 2 n^2 + n
    int off_s = 0, off_y = 0, off_t = 0, lambda_ix = 0;
    std::vector<Edge> pairs;
    Vec beq;
    KktMatrix kkt;
    KktIlu ilu;
};

ProblemData assemble(int n, int r, double alpha, double rho);
Vec project_Y(const ProblemData& pd, const Vec& x_state, const Vec& duals);
// Exact solve of the same delta-regularised KKT system on the GPU; kkt_warm
// (length nx + neq) receives [x; mu]. linear_tol is accepted for signature
// parity (the closed form is exact).
Vec update_X(const ProblemData& pd, const Vec& y_state, const Vec& duals, Vec& kkt_warm,
             double linear_tol);
// The paper's matrix-free CG x-step (LinearSolveError above 1e-8 relative).
Vec update_X_cg(const ProblemData& pd, const Vec& y_state, const Vec& duals, Vec& kkt_warm,
                double linear_tol, int* cg_iters = nullptr);
void update_duals(const ProblemData& pd, const Vec& x_state, const Vec& y_state, Vec& duals);

struct Extraction {
    Topology topology;
    Matrix w;
};
Extraction extract_topology(int n, int r, const Vec& g, double weight_floor);
Topology default_warm_start(int n, int r, std::uint64_t seed);
Solution solve(int n, int r, const SolverConfig& cfg,
               const std::optional<Topology>& warm_start = std::nullopt);

}  // namespace topoopt
