// Reference-compatible C++ API of the B200 topology solver (namespace topoopt).
//
// A caller of the reference library (proj/include/topoopt/*.hpp) recompiles
// against these headers and links libtopoopt_b200.so instead of libtopoopt:
// the hot-path entry points keep their names, argument meaning, value
// semantics and exception types, and forward to the C ABI
// (include/topoopt_b200.h), which runs on the GPU (sm_100a, FP64).
//
// Scope: the ADMM solvers solve / solve_het (node-level systems),
// their substeps, Alg. 1 allocation, the spectral report and cone
// projections, plus the value types they exchange. ProblemData carries the
// block layout and beq but no assembled KKT/ILU: the device x-step is
// matrix-free.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace topoopt {

// ------------------------------------------------------------------ errors
// proj/include/topoopt/errors.hpp:9-27
struct InfeasibleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct PivotError : std::runtime_error {
    int index;
    PivotError(const std::string& m, int i) : std::runtime_error(m), index(i) {}
};
struct LinearSolveError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DegenerateSolutionError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ dense
using Vec = std::vector<double>;

// Row-major dense matrix (proj/include/topoopt/dense.hpp:12-33).
class Matrix {
   public:
    Matrix() = default;
    Matrix(int rows, int cols, double fill = 0.0)
        : r_(rows), c_(cols), v_(static_cast<size_t>(rows) * cols, fill) {}
    static Matrix identity(int n);
    int rows() const { return r_; }
    int cols() const { return c_; }
    double& operator()(int i, int j) { return v_[static_cast<size_t>(i) * c_ + j]; }
    double operator()(int i, int j) const { return v_[static_cast<size_t>(i) * c_ + j]; }
    const std::vector<double>& data() const { return v_; }
    std::vector<double>& data() { return v_; }

   private:
    int r_ = 0, c_ = 0;
    std::vector<double> v_;
};

Matrix matmul(const Matrix& a, const Matrix& b);
Matrix transpose(const Matrix& a);
double max_abs_diff(const Matrix& a, const Matrix& b);
double frobenius_norm(const Matrix& a);
bool is_symmetric(const Matrix& a, double tol);
Matrix symmetrize(const Matrix& a);
double dot(const Vec& a, const Vec& b);
double norm2(const Vec& a);
void axpy(double alpha, const Vec& x, Vec& y);

// ------------------------------------------------------------------ topology
using Edge = std::pair<int, int>;

struct Topology {  // proj/include/topoopt/topology.hpp:16-28
    int n = 0;
    std::vector<Edge> edges;
    std::vector<double> weights;
    void normalize_and_validate();
    void validate() const;
    std::vector<int> degrees() const;
    bool has_uniform_weights(double tol = 0.0) const;
};

std::vector<Edge> enumerate_edges(int n);
int edge_index(int n, int i, int j);
Matrix laplacian(const Topology& t);
Matrix gossip_matrix(const Topology& t);

struct SpectralReport {
    double acf = 1.0;
    double lambda2 = 1.0;
    double lambda_n = 0.0;
    bool connected = false;
};
SpectralReport spectral_report(const Matrix& w);  // GPU Lanczos
double acf(const Matrix& w);
void validate_gossip(const Matrix& w);

// On-disk formats (proj/include/topoopt/topology.hpp:78-85): JSON in
// nlohmann's dump(2) layout, CSV with %.17g.
std::string g17(double value);
std::string topology_to_json(const Topology& t);
Topology topology_from_json(const std::string& text);
std::string matrix_to_csv(const Matrix& m);
std::string matrix_to_triplet_csv(const Matrix& m, double drop_below = 0.0);

enum class BenchmarkKind { ring, grid2d, torus2d, exponential };
BenchmarkKind benchmark_kind_from_string(const std::string& name);
Topology generate_benchmark(BenchmarkKind kind, int n);

// ------------------------------------------------------------------ consensus
// proj/include/topoopt/consensus.hpp:11-54
inline constexpr int kDefaultSimDim = 128;
struct ConsensusTrace {
    std::vector<double> errors;  // length iters + 1; errors[0] is the start
    double t_iter_ms = 0.0;
    std::string label;
    std::uint64_t seed = 0;
    std::string to_csv() const;  // "iter,time_ms,error"
};
ConsensusTrace simulate(const Matrix& w, int dim, int iters, std::uint64_t seed);  // GPU
double convergence_time(const ConsensusTrace& trace, double threshold, double t_iter);
struct CompareEntry {
    std::string label;
    Matrix w;
    double t_iter_ms = 0.0;
};
struct CompareReport {
    std::vector<ConsensusTrace> traces;
    std::vector<double> convergence_ms;
    std::string to_csv() const;  // "time_ms,label,error"
};
CompareReport compare(const std::vector<CompareEntry>& entries, int dim, int iters, double threshold,
                      std::uint64_t seed, int threads = 1);

// ------------------------------------------------------------------ eig
Matrix project_nsd(const Matrix& s);  // GPU sign iteration
Matrix project_psd(const Matrix& s);

// ------------------------------------------------------------------ bandwidth
struct BandwidthProfile {
    std::vector<double> bandwidths;
    std::vector<int> edge_caps;  // empty: n-1 for all
};
struct Allocation {
    double b_unit = 0.0;
    std::vector<int> edges_per_node;
};
Allocation allocate_edge_capacity(const BandwidthProfile& profile, int r);  // GPU Alg. 1

struct CapacityRow {
    std::string label;
    std::vector<int> edge_cols;
    int capacity = 0;
};
struct CapacitySystem {
    int n = 0;
    int num_edges = 0;
    bool equality = false;
    std::vector<CapacityRow> rows;
    std::vector<char> allowed;
    std::vector<int> loads(const std::vector<char>& selected) const;
    int implied_edge_total() const;
};
CapacitySystem node_level_constraints(int n, const std::vector<int>& degrees);

// proj/include/topoopt/bandwidth.hpp:57-110: capacity-bound (inequality) systems
struct ServerLink {
    std::string name;
    double bandwidth = 0.0;
    int capacity = 0;
};
struct ServerTree {
    int n_devices = 0;
    std::vector<ServerLink> links;
    std::vector<std::vector<int>> routes;  // per device pair column: links it uses
    void validate() const;
};
ServerTree tiered8_tree(double leaf_bw, double group_bw, double root_bw);
CapacitySystem intra_server_constraints(const ServerTree& tree);
struct BCubeSpec {
    int p = 2, k = 1;
    std::vector<double> layer_bandwidths;
    int n_servers() const;
};
CapacitySystem bcube_constraints(const BCubeSpec& spec);

// ------------------------------------------------------------------ anneal
struct AnnealConfig {  // proj/include/topoopt/anneal.hpp:12-20
    double t0 = 1.0;
    double cooling = 0.995;
    int steps = 200;
    int moves_per_temp = 0;
    std::uint64_t seed = 0;
    void validate() const;
};
Topology anneal_degree_topology(const std::vector<int>& degrees, const AnnealConfig& cfg);
Topology anneal_topology(const CapacitySystem& sys, std::optional<int> r, const AnnealConfig& cfg);

// ------------------------------------------------------------------ admm
struct SolverConfig {  // proj/include/topoopt/admm.hpp:15-25
    double rho = 1.0;
    double epsilon = 1e-6;
    int max_iter = 20000;
    double alpha = 2.0;
    double weight_floor = 1e-6;
    std::uint64_t seed = 0;
    double linear_tol = 1e-10;
    // device extension: 0 closed-form x-step, 1 the paper's matrix-free CG
    // linear substep to linear_tol (homogeneous solves)
    int linear_solver = 0;
    void validate() const;
};

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
    std::string trace_csv() const;
};

// Layout and equality right-hand side of the homogeneous problem.
struct ProblemData {
    int n = 0, m = 0, r = 0;
    double alpha = 2.0, rho = 1.0;
    int nx = 0, neq = 0;
    int off_s = 0, off_y = 0, off_t = 0, lambda_ix = 0;
    std::vector<Edge> pairs;
    Vec beq;
};

ProblemData assemble(int n, int r, double alpha, double rho);
Vec project_Y(const ProblemData& pd, const Vec& x_state, const Vec& duals);
// kkt_warm (length nx + neq) receives the exact KKT solution [x; mu].
Vec update_X(const ProblemData& pd, const Vec& y_state, const Vec& duals, Vec& kkt_warm,
             double linear_tol);
// The same x-step with the CG linear substep (matrix-free over the edge
// incidence); throws LinearSolveError above 1e-8 relative residual.
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

// ------------------------------------------------------------------ admm_het
struct ProblemDataHet {
    int n = 0, m = 0, r = 0;
    double alpha = 2.0, rho = 1.0;
    int nx = 0, neq = 0;
    int off_s = 0, off_y = 0, off_t = 0, off_z = 0, off_nu = 0, lambda_ix = 0;
    int q = 0;
    std::vector<Edge> pairs;
    CapacitySystem sys;
    Vec beq;
};

// Node-level equality systems (degree rows) and capacity-bound systems
// (intra-server trees, BCube; capped binary projection) run on the GPU.
ProblemDataHet assemble_het(const CapacitySystem& sys, std::optional<int> r, double alpha,
                            double rho);
Vec project_binary_z(const Vec& v, int r);
Vec project_Y_het(const ProblemDataHet& pd, const Vec& x_state, const Vec& duals);
Solution solve_het(const CapacitySystem& sys, std::optional<int> r, const SolverConfig& cfg,
                   const std::optional<Topology>& warm_start = std::nullopt);

struct UtilizationRow {
    std::string label;
    int capacity = 0;
    int used = 0;
};
std::vector<UtilizationRow> utilization(const CapacitySystem& sys, const Topology& t);
std::string utilization_csv(const std::vector<UtilizationRow>& rows);

}  // namespace topoopt
