// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exposes
// the reference's own public API (proj/include/topoopt/*.hpp) with plain
// pointers so Python tests, the golden-fixture generator and bench.py's CPU
// baseline can call the reference itself. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.
//
// Status codes mirror the exception taxonomy (proj/include/topoopt/errors.hpp):
// 0 ok, 1 invalid_argument, 2 InfeasibleError, 3 LinearSolveError,
// 4 DegenerateSolutionError, 5 PivotError, 6 other.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include "admm_shared.hpp"  // proj/src: detail::feasible_start / kkt_rhs / acf_of_g
#include "topoopt/admm.hpp"
#include "topoopt/admm_het.hpp"
#include "topoopt/anneal.hpp"
#include "topoopt/consensus.hpp"
#include "topoopt/bandwidth.hpp"
#include "topoopt/eig.hpp"
#include "topoopt/errors.hpp"
#include "topoopt/solvers.hpp"
#include "topoopt/topology.hpp"

using namespace topoopt;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return 2;
    } catch (const LinearSolveError& e) {
        g_err = e.what();
        return 3;
    } catch (const DegenerateSolutionError& e) {
        g_err = e.what();
        return 4;
    } catch (const PivotError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

SolverConfig make_cfg(const double* c) {
    // c = {rho, epsilon, max_iter, alpha, weight_floor, seed, linear_tol}
    SolverConfig cfg;
    cfg.rho = c[0];
    cfg.epsilon = c[1];
    cfg.max_iter = static_cast<int>(c[2]);
    cfg.alpha = c[3];
    cfg.weight_floor = c[4];
    cfg.seed = static_cast<std::uint64_t>(c[5]);
    cfg.linear_tol = c[6];
    return cfg;
}

Topology make_topo(int n, const int* edges, const double* weights, int ne) {
    Topology t;
    t.n = n;
    for (int k = 0; k < ne; ++k) {
        t.edges.push_back({edges[2 * k], edges[2 * k + 1]});
        t.weights.push_back(weights ? weights[k] : 0.1);
    }
    t.normalize_and_validate();
    return t;
}

Matrix from_flat(int n, const double* a) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m(i, j) = a[static_cast<size_t>(i) * n + j];
    return m;
}

void to_flat(const Matrix& m, double* out) {
    for (int i = 0; i < m.rows(); ++i)
        for (int j = 0; j < m.cols(); ++j) out[static_cast<size_t>(i) * m.cols() + j] = m(i, j);
}

struct SolOut {
    Solution sol;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- solutions
// Solutions are returned as opaque handles; accessors copy fields out.
void* ref_solve(int n, int r, const double* cfg, const int* warm_edges, int n_warm,
                int has_warm, int* status) {
    auto* out = new SolOut;
    *status = guarded([&] {
        std::optional<Topology> warm;
        if (has_warm) warm = make_topo(n, warm_edges, nullptr, n_warm);
        out->sol = solve(n, r, make_cfg(cfg), warm);
    });
    if (*status != 0) {
        delete out;
        return nullptr;
    }
    return out;
}

// Node-level heterogeneous solve: CapacitySystem from the degree list
// (node_level_constraints, proj/src/bandwidth.cpp:116-146).
void* ref_solve_het_node(int n, const int* degrees, const double* cfg, const int* warm_edges,
                         int n_warm, int has_warm, int* status) {
    auto* out = new SolOut;
    *status = guarded([&] {
        std::vector<int> deg(degrees, degrees + n);
        CapacitySystem sys = node_level_constraints(n, deg);
        std::optional<Topology> warm;
        if (has_warm) warm = make_topo(n, warm_edges, nullptr, n_warm);
        out->sol = solve_het(sys, std::nullopt, make_cfg(cfg), warm);
    });
    if (*status != 0) {
        delete out;
        return nullptr;
    }
    return out;
}

// ---------------------------------------------------------------- capacity systems
// kind 0: intra_server_constraints(tiered8_tree(a, b, c)); kind 1:
// bcube_constraints({p = a, k = b}); drop_last removes the last row (the
// relaxation of proj/tests/test_admm_het.cpp:214-229).
static CapacitySystem make_capacity_system(int kind, double a, double b, double c, int drop_last) {
    CapacitySystem sys = kind == 0 ? intra_server_constraints(tiered8_tree(a, b, c))
                                   : bcube_constraints({static_cast<int>(a), static_cast<int>(b), {}});
    if (drop_last) sys.rows.pop_back();
    return sys;
}

// sizes: {n, num_edges, rows, total row entries}
int ref_capacity_system_sizes(int kind, double a, double b, double c, int drop_last, int* sizes) {
    return guarded([&] {
        CapacitySystem sys = make_capacity_system(kind, a, b, c, drop_last);
        int nnz = 0;
        for (const auto& row : sys.rows) nnz += static_cast<int>(row.edge_cols.size());
        sizes[0] = sys.n;
        sizes[1] = sys.num_edges;
        sizes[2] = static_cast<int>(sys.rows.size());
        sizes[3] = nnz;
    });
}

int ref_capacity_system(int kind, double a, double b, double c, int drop_last, int* row_ptr, int* cols,
                        int* caps, int* allowed) {
    return guarded([&] {
        CapacitySystem sys = make_capacity_system(kind, a, b, c, drop_last);
        int k = 0;
        row_ptr[0] = 0;
        for (size_t r = 0; r < sys.rows.size(); ++r) {
            for (int col : sys.rows[r].edge_cols) cols[k++] = col;
            row_ptr[r + 1] = k;
            caps[r] = sys.rows[r].capacity;
        }
        for (int l = 0; l < sys.num_edges; ++l) allowed[l] = sys.allowed[l];
    });
}

int ref_project_binary_z_capped(int kind, double a, double b, double c, int drop_last, const double* v,
                                int r, double* z) {
    return guarded([&] {
        CapacitySystem sys = make_capacity_system(kind, a, b, c, drop_last);
        const Vec out = project_binary_z_capped(Vec(v, v + sys.num_edges), r, sys);
        std::copy(out.begin(), out.end(), z);
    });
}

int ref_anneal_capacity(int kind, double a, double b, double c, int drop_last, int r, int steps,
                        int moves_per_temp, uint64_t seed, int* edges, int* n_edges) {
    return guarded([&] {
        CapacitySystem sys = make_capacity_system(kind, a, b, c, drop_last);
        AnnealConfig ac;
        ac.steps = steps;
        ac.moves_per_temp = moves_per_temp;
        ac.seed = seed;
        Topology t = anneal_topology(sys, r, ac);
        *n_edges = static_cast<int>(t.edges.size());
        for (size_t k = 0; k < t.edges.size(); ++k) {
            edges[2 * k] = t.edges[k].first;
            edges[2 * k + 1] = t.edges[k].second;
        }
    });
}

void* ref_solve_het_capacity(int kind, double a, double b, double c, int drop_last, int r, const double* cfg,
                             const int* warm_edges, int n_warm, int has_warm, int* status) {
    auto* out = new SolOut;
    *status = guarded([&] {
        CapacitySystem sys = make_capacity_system(kind, a, b, c, drop_last);
        std::optional<Topology> warm;
        if (has_warm) warm = make_topo(sys.n, warm_edges, nullptr, n_warm);
        out->sol = solve_het(sys, r, make_cfg(cfg), warm);
    });
    if (*status != 0) {
        delete out;
        return nullptr;
    }
    return out;
}

// ---------------------------------------------------------------- text formats
// (proj/src/topology.cpp:283-324, admm.cpp:223-236): the string is copied into
// buf (cap bytes); returns its full length
static int copy_out(const std::string& text, char* buf, int cap) {
    const int k = std::min<int>(cap - 1, static_cast<int>(text.size()));
    if (cap > 0) {
        std::memcpy(buf, text.data(), k);
        buf[k] = 0;
    }
    return static_cast<int>(text.size());
}

int ref_topology_to_json(int n, const int* edges, const double* weights, int ne, char* buf, int cap) {
    int len = 0;
    const int st = guarded([&] { len = copy_out(topology_to_json(make_topo(n, edges, weights, ne)), buf, cap); });
    return st != 0 ? -1 : len;
}

// The `topoopt optimize` artefacts the CLI builds itself
// (proj/tools/topoopt.cpp:244-246, 285-296): allocation.json and
// solution.json, nlohmann objects dumped with indent 2 (restated here, test
// infrastructure: the CLI is not built).
int ref_allocation_json(double b_unit, const int* e, int n, char* buf, int cap) {
    int len = 0;
    const int st = guarded([&] {
        nlohmann::json aj;
        aj["b_unit"] = b_unit;
        aj["e"] = std::vector<int>(e, e + n);
        len = copy_out(aj.dump(2) + "\n", buf, cap);
    });
    return st != 0 ? -1 : len;
}

int ref_solution_json(const char* mode, double acf, double lambda_tilde, int converged, int connected,
                      int repaired, int iterations, double residual, int n_edges, const char* note, char* buf,
                      int cap) {
    int len = 0;
    const int st = guarded([&] {
        nlohmann::json sj;
        sj["mode"] = std::string(mode);
        sj["acf"] = acf;
        sj["lambda_tilde"] = lambda_tilde;
        sj["converged"] = converged != 0;
        sj["connected"] = connected != 0;
        sj["repaired"] = repaired != 0;
        sj["iterations"] = iterations;
        sj["residual"] = residual;
        sj["edges"] = (size_t)n_edges;
        sj["note"] = std::string(note);
        len = copy_out(sj.dump(2) + "\n", buf, cap);
    });
    return st != 0 ? -1 : len;
}

int ref_matrix_to_csv(int n, const double* w, char* buf, int cap) {
    int len = 0;
    const int st = guarded([&] { len = copy_out(matrix_to_csv(from_flat(n, w)), buf, cap); });
    return st != 0 ? -1 : len;
}

int ref_solution_trace_csv(void* h, char* buf, int cap) {
    return copy_out(static_cast<SolOut*>(h)->sol.trace_csv(), buf, cap);
}

void ref_solution_free(void* h) { delete static_cast<SolOut*>(h); }

// scalars: {acf, lambda_tilde, residual, wall_ms, converged, connected, repaired,
//           iterations, n_edges, trace_len}
void ref_solution_scalars(void* h, double* s) {
    const auto& sol = static_cast<SolOut*>(h)->sol;
    s[0] = sol.acf_value;
    s[1] = sol.lambda_tilde;
    s[2] = sol.residual;
    s[3] = sol.wall_time_ms;
    s[4] = sol.converged;
    s[5] = sol.connected;
    s[6] = sol.repaired;
    s[7] = sol.iterations;
    s[8] = static_cast<double>(sol.topology.edges.size());
    s[9] = static_cast<double>(sol.trace.size());
}

void ref_solution_edges(void* h, int* edges, double* weights) {
    const auto& t = static_cast<SolOut*>(h)->sol.topology;
    for (size_t k = 0; k < t.edges.size(); ++k) {
        edges[2 * k] = t.edges[k].first;
        edges[2 * k + 1] = t.edges[k].second;
        weights[k] = t.weights[k];
    }
}

void ref_solution_w(void* h, double* w) { to_flat(static_cast<SolOut*>(h)->sol.w, w); }

// trace rows: iter, residual, lambda_tilde, acf_iterate
void ref_solution_trace(void* h, double* rows) {
    const auto& tr = static_cast<SolOut*>(h)->sol.trace;
    for (size_t k = 0; k < tr.size(); ++k) {
        rows[4 * k] = tr[k].iter;
        rows[4 * k + 1] = tr[k].residual;
        rows[4 * k + 2] = tr[k].lambda_tilde;
        rows[4 * k + 3] = tr[k].acf_iterate;
    }
}

int ref_solution_note(void* h, char* buf, int cap) {
    const auto& note = static_cast<SolOut*>(h)->sol.note;
    const int len = static_cast<int>(note.size());
    if (cap > 0) {
        std::memcpy(buf, note.data(), std::min(len, cap - 1));
        buf[std::min(len, cap - 1)] = 0;
    }
    return len;
}

// ---------------------------------------------------------------- allocation
int ref_allocate(const double* b, const int* caps, int n, int r, double* b_unit, int* e) {
    return guarded([&] {
        BandwidthProfile p;
        p.bandwidths.assign(b, b + n);
        if (caps) p.edge_caps.assign(caps, caps + n);
        Allocation a = allocate_edge_capacity(p, r);
        *b_unit = a.b_unit;
        std::copy(a.edges_per_node.begin(), a.edges_per_node.end(), e);
    });
}

// ---------------------------------------------------------------- warm starts
int ref_default_warm_start(int n, int r, std::uint64_t seed, int* edges, int* n_edges) {
    return guarded([&] {
        Topology t = default_warm_start(n, r, seed);
        *n_edges = static_cast<int>(t.edges.size());
        for (size_t k = 0; k < t.edges.size(); ++k) {
            edges[2 * k] = t.edges[k].first;
            edges[2 * k + 1] = t.edges[k].second;
        }
    });
}

int ref_anneal_degree(int n, const int* degrees, double t0, double cooling, int steps,
                      int moves_per_temp, std::uint64_t seed, int* edges, int* n_edges) {
    return guarded([&] {
        AnnealConfig ac;
        ac.t0 = t0;
        ac.cooling = cooling;
        ac.steps = steps;
        ac.moves_per_temp = moves_per_temp;
        ac.seed = seed;
        Topology t = anneal_degree_topology(std::vector<int>(degrees, degrees + n), ac);
        *n_edges = static_cast<int>(t.edges.size());
        for (size_t k = 0; k < t.edges.size(); ++k) {
            edges[2 * k] = t.edges[k].first;
            edges[2 * k + 1] = t.edges[k].second;
        }
    });
}

int ref_generate_benchmark(const char* kind, int n, int* edges, double* weights, int* n_edges) {
    return guarded([&] {
        Topology t = generate_benchmark(benchmark_kind_from_string(kind), n);
        *n_edges = static_cast<int>(t.edges.size());
        for (size_t k = 0; k < t.edges.size(); ++k) {
            edges[2 * k] = t.edges[k].first;
            edges[2 * k + 1] = t.edges[k].second;
            weights[k] = t.weights[k];
        }
    });
}

// ---------------------------------------------------------------- consensus
// simulate (proj/src/consensus.cpp:29-67): errors[0..iters]
int ref_simulate(int n, const double* w, int dim, int iters, uint64_t seed, double* errors) {
    return guarded([&] {
        ConsensusTrace t = simulate(from_flat(n, w), dim, iters, seed);
        for (size_t k = 0; k < t.errors.size(); ++k) errors[k] = t.errors[k];
    });
}

// ---------------------------------------------------------------- spectra
int ref_spectral_report(int n, const double* w, double* out4) {
    return guarded([&] {
        SpectralReport rep = spectral_report(from_flat(n, w));
        out4[0] = rep.acf;
        out4[1] = rep.lambda2;
        out4[2] = rep.lambda_n;
        out4[3] = rep.connected ? 1.0 : 0.0;
    });
}

int ref_sym_eig(int n, const double* a, double* values, double* vectors) {
    return guarded([&] {
        EigDecomposition eg = sym_eig(from_flat(n, a));
        std::copy(eg.values.begin(), eg.values.end(), values);
        if (vectors) to_flat(eg.vectors, vectors);
    });
}

int ref_project_psd(int n, const double* a, double* out) {
    return guarded([&] { to_flat(project_psd(from_flat(n, a)), out); });
}

int ref_project_nsd(int n, const double* a, double* out) {
    return guarded([&] { to_flat(project_nsd(from_flat(n, a)), out); });
}

// ---------------------------------------------------------------- substeps
struct RefProblem {
    ProblemData pd;
    std::optional<ProblemDataHet> het;
};

void* ref_problem_create(int n, int r, double alpha, double rho, int* status) {
    auto* p = new RefProblem;
    *status = guarded([&] { p->pd = assemble(n, r, alpha, rho); });
    if (*status) {
        delete p;
        return nullptr;
    }
    return p;
}

void* ref_problem_het_node_create(int n, const int* degrees, double alpha, double rho,
                                  int* status) {
    auto* p = new RefProblem;
    *status = guarded([&] {
        CapacitySystem sys = node_level_constraints(n, std::vector<int>(degrees, degrees + n));
        p->het = assemble_het(sys, std::nullopt, alpha, rho);
    });
    if (*status) {
        delete p;
        return nullptr;
    }
    return p;
}

void ref_problem_free(void* h) { delete static_cast<RefProblem*>(h); }

// {n, m, r, nx, neq, off_s, off_y, off_t, lambda_ix, off_z, off_nu, q}
void ref_problem_dims(void* h, int* d) {
    auto* p = static_cast<RefProblem*>(h);
    if (p->het) {
        const auto& q = *p->het;
        int v[12] = {q.n, q.m, q.r, q.nx, q.neq, q.off_s, q.off_y, q.off_t, q.lambda_ix,
                     q.off_z, q.off_nu, q.q};
        std::copy(v, v + 12, d);
    } else {
        const auto& q = p->pd;
        int v[12] = {q.n, q.m, q.r, q.nx, q.neq, q.off_s, q.off_y, q.off_t, q.lambda_ix,
                     -1, -1, 0};
        std::copy(v, v + 12, d);
    }
}

void ref_problem_beq(void* h, double* beq) {
    auto* p = static_cast<RefProblem*>(h);
    const Vec& b = p->het ? p->het->beq : p->pd.beq;
    std::copy(b.begin(), b.end(), beq);
}

int ref_project_Y(void* h, const double* x, const double* d, double* y) {
    auto* p = static_cast<RefProblem*>(h);
    return guarded([&] {
        const int nx = p->het ? p->het->nx : p->pd.nx;
        Vec xs(x, x + nx), ds(d, d + nx);
        Vec out = p->het ? project_Y_het(*p->het, xs, ds) : project_Y(p->pd, xs, ds);
        std::copy(out.begin(), out.end(), y);
    });
}

// x-step through the reference KKT (BiCGSTAB + ILU(0)). kkt_warm has length
// nx + neq (in/out). chunk > 0 restarts BiCGSTAB every `chunk` iterations
// (needed at n=1024 where the un-restarted solve stagnates).
int ref_update_X(void* h, const double* y, const double* d, double* kkt_warm, double tol,
                 int chunk, double* x_out, int* inner_iters) {
    auto* p = static_cast<RefProblem*>(h);
    return guarded([&] {
        const bool het = p->het.has_value();
        const int nx = het ? p->het->nx : p->pd.nx;
        const int neq = het ? p->het->neq : p->pd.neq;
        const SparseMatrix& kkt = het ? p->het->kkt : p->pd.kkt;
        const IluFactors& ilu = het ? p->het->ilu : p->pd.ilu;
        const Vec& beq = het ? p->het->beq : p->pd.beq;
        const double rho = het ? p->het->rho : p->pd.rho;
        const int n = het ? p->het->n : p->pd.n;
        Vec ys(y, y + nx), ds(d, d + nx), warm(kkt_warm, kkt_warm + nx + neq);
        detail::Layout lo = het ? detail::het_layout(n, p->het->q) : detail::hom_layout(n);
        int total = 0;
        if (chunk <= 0 && !het) {
            Vec xo = update_X(p->pd, ys, ds, warm, tol);
            std::copy(xo.begin(), xo.end(), x_out);
        } else {
            const Vec rhs = detail::kkt_rhs(lo, ys, ds, beq, rho);
            for (int round = 0; round < 100000; ++round) {
                SolveReport rep = bicgstab(kkt, rhs, warm, &ilu, tol, chunk > 0 ? chunk : -1);
                total += rep.iterations;
                if (rep.converged) break;
                if (chunk <= 0) {
                    const double scale = std::max(norm2(rhs), 1e-30);
                    if (rep.residual > 1e-8 * scale)
                        throw LinearSolveError("saddle-point solve stalled");
                    break;
                }
            }
            std::copy(warm.begin(), warm.begin() + nx, x_out);
        }
        std::copy(warm.begin(), warm.end(), kkt_warm);
        if (inner_iters) *inner_iters = total;
    });
}

// Feasible start (proj/src/admm.cpp:143-173 and, for het, admm_het.cpp:247-250).
int ref_feasible_start(void* h, const int* warm_edges, int n_warm, double* x) {
    auto* p = static_cast<RefProblem*>(h);
    return guarded([&] {
        const bool het = p->het.has_value();
        const int n = het ? p->het->n : p->pd.n;
        const double alpha = het ? p->het->alpha : p->pd.alpha;
        Topology warm = make_topo(n, warm_edges, nullptr, n_warm);
        detail::Layout lo = het ? detail::het_layout(n, p->het->q) : detail::hom_layout(n);
        Vec xs = detail::feasible_start(lo, warm, alpha);
        if (het) {
            for (const auto& [i, j] : warm.edges) xs[p->het->off_z + edge_index(n, i, j)] = 1.0;
            for (int l = 0; l < p->het->m; ++l)
                xs[p->het->off_nu + l] = std::max(0.0, xs[p->het->off_z + l] - xs[l]);
        }
        std::copy(xs.begin(), xs.end(), x);
    });
}

double ref_acf_of_g(int n, const double* g) {
    const auto pairs = enumerate_edges(n);
    return detail::acf_of_g(n, pairs, g);
}

int ref_extract_topology(int n, int r, const double* g, double floor, int* edges,
                         double* weights, int* n_edges) {
    return guarded([&] {
        const int m = n * (n - 1) / 2;
        Extraction ex = extract_topology(n, r, Vec(g, g + m), floor);
        *n_edges = static_cast<int>(ex.topology.edges.size());
        for (size_t k = 0; k < ex.topology.edges.size(); ++k) {
            edges[2 * k] = ex.topology.edges[k].first;
            edges[2 * k + 1] = ex.topology.edges[k].second;
            weights[k] = ex.topology.weights[k];
        }
    });
}

int ref_project_binary_z(const double* v, int m, int r, double* z) {
    return guarded([&] {
        Vec out = project_binary_z(Vec(v, v + m), r);
        std::copy(out.begin(), out.end(), z);
    });
}

// ---------------------------------------------------------------- CPU baseline
// One homogeneous ADMM iteration of the reference at (n, r), decomposed into
// its four substeps (proj/src/admm.cpp:386-396): project_nsd(S),
// project_psd(T) [= project_Y], the x-step (kkt_rhs + restarted BiCGSTAB),
// and the trace SLEM acf_of_g. Each substep is timed on its own thread
// concurrently so the wall time is ~max instead of the sum; the returned
// per-substep seconds add up to the single-core iteration time.
// times = {t_nsd, t_psd, t_xstep, t_acf, t_setup, bicg_iters}
int ref_iteration_sample(int n, int r, const int* warm_edges, int n_warm, double rho,
                         int chunk, double* times) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto sec = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double>(b - a).count();
        };
        const auto t0 = clk::now();
        ProblemData pd = assemble(n, r, 2.0, rho);
        const auto lo = detail::hom_layout(n);
        Topology warm = make_topo(n, warm_edges, nullptr, n_warm);
        Vec x = detail::feasible_start(lo, warm, 2.0);
        Vec dual(pd.nx, 0.0);
        const auto t1 = clk::now();
        times[4] = sec(t0, t1);
        // Inputs of the cone projections, as project_Y forms them.
        Matrix s(n, n), t(n, n);
        for (int c = 0; c < n; ++c)
            for (int rr = 0; rr < n; ++rr) {
                s(rr, c) = x[pd.off_s + c * n + rr];
                t(rr, c) = x[pd.off_t + c * n + rr];
            }
        // x-step input: the feasible start moved off the constraint set (as the
        // cone projection does), so BiCGSTAB works as in a real iteration
        Vec y = x;
        for (size_t k = 0; k < y.size(); ++k) y[k] += 1e-3 * std::sin(0.7 * (double)k);
        Vec warm_kkt(pd.nx + pd.neq, 0.0);
        std::copy(x.begin(), x.end(), warm_kkt.begin());
        double tn = 0, tp = 0, tx = 0, ta = 0;
        int iters = 0;
        std::thread th1([&] {
            auto a = clk::now();
            Matrix o = project_nsd(s);
            tn = sec(a, clk::now());
        });
        std::thread th2([&] {
            auto a = clk::now();
            Matrix o = project_psd(t);
            tp = sec(a, clk::now());
        });
        std::thread th3([&] {
            auto a = clk::now();
            const Vec rhs = detail::kkt_rhs(lo, y, dual, pd.beq, pd.rho);
            for (int round = 0; round < 100000; ++round) {
                SolveReport rep = bicgstab(pd.kkt, rhs, warm_kkt, &pd.ilu, 1e-10, chunk);
                iters += rep.iterations;
                if (rep.converged) break;
            }
            tx = sec(a, clk::now());
        });
        std::thread th4([&] {
            auto a = clk::now();
            volatile double v = detail::acf_of_g(n, pd.pairs, x.data());
            (void)v;
            ta = sec(a, clk::now());
        });
        th1.join();
        th2.join();
        th3.join();
        th4.join();
        times[0] = tn;
        times[1] = tp;
        times[2] = tx;
        times[3] = ta;
        times[5] = iters;
    });
}

// The reference's homogeneous ADMM loop (proj/src/admm.cpp:360-401) run
// sequentially on the calling thread for `iters` iterations, with the one
// sanctioned change: the x-step solves its KKT system with the
// reference's own kkt_rhs + ILU(0) BiCGSTAB restarted every `chunk`
// iterations (update_X's un-restarted BiCGSTAB stagnates at n = 1024,
// SURVEY §6). Every other call is the reference's: assemble,
// feasible_start, project_Y, update_duals, the residual, acf_of_g, the
// best-iterate copy. out = {setup_s, iter_1_s, ..., iter_k_s, residual_k,
// bicgstab_iterations_total}.
int ref_admm_run(int n, int r, const int* warm_edges, int n_warm, double rho, int iters, int chunk,
                 double* out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto sec = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double>(b - a).count();
        };
        const auto t0 = clk::now();
        ProblemData pd = assemble(n, r, 2.0, rho);
        const auto lo = detail::hom_layout(n);
        Topology warm = make_topo(n, warm_edges, nullptr, n_warm);
        Vec x_state = detail::feasible_start(lo, warm, 2.0);
        Vec y_state = x_state;
        Vec duals(pd.nx, 0.0);
        Vec kkt_warm(pd.nx + pd.neq, 0.0);
        std::copy(x_state.begin(), x_state.end(), kkt_warm.begin());
        double best_res = std::numeric_limits<double>::infinity();
        Vec best_y = y_state;
        out[0] = sec(t0, clk::now());
        double res = 0.0;
        long long bicg = 0;
        for (int it = 1; it <= iters; ++it) {
            const auto a = clk::now();
            y_state = project_Y(pd, x_state, duals);
            const Vec rhs = detail::kkt_rhs(lo, y_state, duals, pd.beq, pd.rho);
            for (int round = 0; round < 100000; ++round) {
                SolveReport rep = bicgstab(pd.kkt, rhs, kkt_warm, &pd.ilu, 1e-10, chunk);
                bicg += rep.iterations;
                if (rep.converged) break;
            }
            x_state.assign(kkt_warm.begin(), kkt_warm.begin() + pd.nx);
            update_duals(pd, x_state, y_state, duals);
            res = 0.0;
            for (int k = 0; k < pd.nx; ++k) {
                const double d = x_state[k] - y_state[k];
                res += d * d;
            }
            volatile double acf = detail::acf_of_g(n, pd.pairs, y_state.data());
            (void)acf;
            if (res < best_res) {
                best_res = res;
                best_y = y_state;
            }
            out[it] = sec(a, clk::now());
        }
        out[iters + 1] = res;
        out[iters + 2] = (double)bicg;
    });
}

// The reference's node-level heterogeneous ADMM loop (proj/src/admm_het.cpp:
// 235-297) sequential on the calling thread, the x-step's BiCGSTAB restarted
// every `chunk` iterations (as ref_admm_run). out as ref_admm_run.
int ref_admm_het_run(int n, const int* degrees, const int* warm_edges, int n_warm, double rho, int iters,
                     int chunk, double* out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto sec = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double>(b - a).count();
        };
        const auto t0 = clk::now();
        CapacitySystem sys = node_level_constraints(n, std::vector<int>(degrees, degrees + n));
        ProblemDataHet pd = assemble_het(sys, std::nullopt, 2.0, rho);
        const auto lo = detail::het_layout(pd.n, pd.q);
        const int m = pd.m;
        Topology warm = make_topo(n, warm_edges, nullptr, n_warm);
        Vec x_state = detail::feasible_start(lo, warm, 2.0);
        for (const auto& [i, j] : warm.edges) x_state[pd.off_z + edge_index(n, i, j)] = 1.0;
        for (int l = 0; l < m; ++l) x_state[pd.off_nu + l] = std::max(0.0, x_state[pd.off_z + l] - x_state[l]);
        Vec y_state = x_state;
        Vec duals(pd.nx, 0.0);
        Vec kkt_warm(pd.nx + pd.neq, 0.0);
        std::copy(x_state.begin(), x_state.end(), kkt_warm.begin());
        double best_res = std::numeric_limits<double>::infinity();
        Vec best_y = y_state, best_score(m, 0.0);
        out[0] = sec(t0, clk::now());
        double res = 0.0;
        long long bicg = 0;
        for (int it = 1; it <= iters; ++it) {
            const auto a = clk::now();
            y_state = project_Y_het(pd, x_state, duals);
            const Vec rhs = detail::kkt_rhs(lo, y_state, duals, pd.beq, pd.rho);
            for (int round = 0; round < 100000; ++round) {
                SolveReport rep = bicgstab(pd.kkt, rhs, kkt_warm, &pd.ilu, 1e-10, chunk);
                bicg += rep.iterations;
                if (rep.converged) break;
            }
            x_state.assign(kkt_warm.begin(), kkt_warm.begin() + pd.nx);
            for (int k = 0; k < pd.nx; ++k) duals[k] += pd.rho * (x_state[k] - y_state[k]);
            res = 0.0;
            for (int k = 0; k < pd.nx; ++k) {
                const double d = x_state[k] - y_state[k];
                res += d * d;
            }
            volatile double acf = detail::acf_of_g(n, pd.pairs, y_state.data());
            (void)acf;
            if (res < best_res) {
                best_res = res;
                best_y = y_state;
                for (int l = 0; l < m; ++l) best_score[l] = x_state[pd.off_z + l] + duals[pd.off_z + l] / pd.rho;
            }
            out[it] = sec(a, clk::now());
        }
        out[iters + 1] = res;
        out[iters + 2] = (double)bicg;
    });
}


// The same loop as ref_admm_het_run, recording the trace row of every
// iteration (residual, lambda of the projected iterate, acf_of_g) for a
// lockstep golden at n = 256 (tests/golden/make_config5.py): the reference's
// solve_het loop (proj/src/admm_het.cpp:266-301) with BiCGSTAB restarted in
// chunks until it meets its 1e-10 tolerance.
int ref_admm_het_trace(int n, const int* degrees, const int* warm_edges, int n_warm, double rho, int iters,
                       int chunk, double* trace) {
    return guarded([&] {
        CapacitySystem sys = node_level_constraints(n, std::vector<int>(degrees, degrees + n));
        ProblemDataHet pd = assemble_het(sys, std::nullopt, 2.0, rho);
        const auto lo = detail::het_layout(pd.n, pd.q);
        const int m = pd.m;
        Topology warm = make_topo(n, warm_edges, nullptr, n_warm);
        Vec x_state = detail::feasible_start(lo, warm, 2.0);
        for (const auto& [i, j] : warm.edges) x_state[pd.off_z + edge_index(n, i, j)] = 1.0;
        for (int l = 0; l < m; ++l) x_state[pd.off_nu + l] = std::max(0.0, x_state[pd.off_z + l] - x_state[l]);
        Vec y_state = x_state;
        Vec duals(pd.nx, 0.0);
        Vec kkt_warm(pd.nx + pd.neq, 0.0);
        std::copy(x_state.begin(), x_state.end(), kkt_warm.begin());
        for (int it = 1; it <= iters; ++it) {
            y_state = project_Y_het(pd, x_state, duals);
            const Vec rhs = detail::kkt_rhs(lo, y_state, duals, pd.beq, pd.rho);
            for (int round = 0; round < 100000; ++round) {
                SolveReport rep = bicgstab(pd.kkt, rhs, kkt_warm, &pd.ilu, 1e-10, chunk);
                if (rep.converged) break;
            }
            x_state.assign(kkt_warm.begin(), kkt_warm.begin() + pd.nx);
            for (int k = 0; k < pd.nx; ++k) duals[k] += pd.rho * (x_state[k] - y_state[k]);
            double res = 0.0;
            for (int k = 0; k < pd.nx; ++k) {
                const double d = x_state[k] - y_state[k];
                res += d * d;
            }
            trace[3 * (it - 1)] = res;
            trace[3 * (it - 1) + 1] = y_state[lo.lambda_ix];
            trace[3 * (it - 1) + 2] = detail::acf_of_g(n, pd.pairs, y_state.data());
        }
    });
}

}  // extern "C"
