// C ABI (include/topoopt_b200.h): host entry points over the device solver.
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/topoopt_b200.h"
#include "host_anneal.hpp"
#include "anneal_kernels.cuh"
#include "solver.cuh"

#include "nccl_shim.hpp"

using namespace tpb;

namespace {


template <typename F>
int guarded(F&& f) {
    try {
        f();
        return TP_OK;
    } catch (const Error& e) {
        last_error_ref() = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        last_error_ref() = std::string("out of memory: ") + e.what();
        return TP_ERR_INTERNAL;
    } catch (const std::exception& e) {
        last_error_ref() = e.what();
        return TP_ERR_INTERNAL;
    }
}

Config to_cfg(const tp_config* c) {
    Config k;
    if (c) {
        k.rho = c->rho;
        k.epsilon = c->epsilon;
        k.max_iter = c->max_iter;
        k.alpha = c->alpha;
        k.weight_floor = c->weight_floor;
        k.linear_tol = c->linear_tol;
        k.trace_stride = c->trace_stride;
        k.chunk = c->chunk;
        k.linear_solver = c->linear_solver;
        k.cg_max_iter = c->cg_max_iter;
    }
    return k;
}

void require_device() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Error(kCuda, "no CUDA device: the B200 solver has no CPU fallback");
}

// Topology::normalize_and_validate (proj/src/topology.cpp:19-51) on an edge
// list, returned as ascending packed indices.
std::vector<int> packed_edges(int n, const int32_t* edges, int k) {
    if (k > 0 && !edges) throw Error(kInvalidArgument, "topology: null edge list with a positive edge count");
    std::vector<long long> idx(k);
    for (int e = 0; e < k; ++e) {
        const int i = edges[2 * e], j = edges[2 * e + 1];
        if (i < 0 || j < 0 || i >= n || j >= n)
            throw Error(kInvalidArgument, "topology: edge endpoint out of range");
        if (i >= j) throw Error(kInvalidArgument, "topology: edge endpoints must satisfy i < j");
        idx[e] = edge_idx(n, i, j);
    }
    std::sort(idx.begin(), idx.end());
    for (int e = 1; e < k; ++e)
        if (idx[e] == idx[e - 1])
            throw Error(kInvalidArgument, "topology: edges must be sorted without duplicates");
    return std::vector<int>(idx.begin(), idx.end());
}

void fill_result(const SolveResult& R, tp_result* out, int32_t* edges, double* weights,
                 double* trace, char* note, int note_cap) {
    if (out) {
        out->iterations = R.iterations;
        out->converged = R.converged;
        out->connected = R.connected;
        out->repaired = R.repaired;
        out->n_edges = (int32_t)R.w.size();
        out->best_iter = R.best_iter;
        out->residual = R.residual;
        out->lambda_tilde = R.lambda_tilde;
        out->acf = R.acf;
        out->lambda2 = R.lambda2;
        out->lambda_n = R.lambda_n;
    }
    if (edges)
        for (size_t k = 0; k < R.w.size(); ++k) {
            edges[2 * k] = R.ei[k];
            edges[2 * k + 1] = R.ej[k];
        }
    if (weights) std::copy(R.w.begin(), R.w.end(), weights);
    if (trace)
        for (int k = 0; k < R.iterations; ++k) {
            trace[3 * k] = R.tr_res[k];
            trace[3 * k + 1] = R.tr_lam[k];
            trace[3 * k + 2] = R.tr_acf[k];
        }
    if (note && note_cap > 0) {
        const size_t len = std::min<size_t>(R.note.size(), note_cap - 1);
        std::memcpy(note, R.note.data(), len);
        note[len] = 0;
    }
}

// default warm start through the host annealer + device Alg. 1
std::vector<int> default_warm(int n, int r, uint64_t seed);

}  // namespace

namespace tpb {
std::string& last_error_ref() {
    thread_local std::string msg;
    return msg;
}
}  // namespace tpb

struct tp_solver {
    std::unique_ptr<Solver> s;
};

extern "C" {

void tp_config_default(tp_config* c) {
    c->rho = 1.0;
    c->epsilon = 1e-6;
    c->max_iter = 20000;
    c->alpha = 2.0;
    c->weight_floor = 1e-6;
    c->seed = 0;
    c->linear_tol = 1e-10;
    c->trace_stride = 1;
    c->chunk = 0;
    c->linear_solver = 0;
    c->cg_max_iter = 8;
}

int tp_config_validate(const tp_config* c) {
    return guarded([&] { validate(to_cfg(c)); });
}

const char* tp_last_error_message(void) { return last_error_ref().c_str(); }
int tp_version(void) { return 1; }

int tp_set_device(int device) {
    return guarded([&] { TPB_CUDA(cudaSetDevice(device)); });
}

int tp_solver_create(int32_t n, int32_t batch, const int32_t* r, const int32_t* degrees,
                     const tp_config* cfg, tp_solver** out) {
    return guarded([&] {
        require_device();
        std::vector<int> rv, dg;
        if (r) rv.assign(r, r + batch);
        if (degrees) dg.assign(degrees, degrees + (size_t)batch * n);
        auto h = std::make_unique<tp_solver>();
        h->s = std::make_unique<Solver>(n, batch, degrees != nullptr, rv, dg, to_cfg(cfg));
        *out = h.release();
    });
}

int tp_solver_destroy(tp_solver* s) {
    return guarded([&] { delete s; });
}

int tp_solver_set_warm(tp_solver* s, int32_t b, const int32_t* edges, int32_t k) {
    return guarded([&] { s->s->set_warm(b, packed_edges(s->s->n(), edges, k)); });
}

int tp_solver_start(tp_solver* s) {
    return guarded([&] { s->s->start(); });
}

int tp_solver_iterate(tp_solver* s, int32_t k) {
    return guarded([&] { s->s->iterate_async(k); });
}

int tp_solver_sync(tp_solver* s, int32_t* all_done) {
    return guarded([&] {
        const bool d = s->s->all_done();
        if (all_done) *all_done = d ? 1 : 0;
    });
}

int tp_solver_run(tp_solver* s) {
    return guarded([&] { s->s->run_to_completion(); });
}

int tp_solver_finish(tp_solver* s) {
    return guarded([&] { s->s->finish(); });
}

int tp_solver_result(tp_solver* s, int32_t b, tp_result* out, int32_t* edges, double* weights,
                     double* trace, char* note, int32_t note_cap) {
    return guarded([&] { fill_result(s->s->result(b), out, edges, weights, trace, note, note_cap); });
}

void* tp_solver_stream(tp_solver* s) { return (void*)s->s->stream(); }

// ---------------------------------------------------------------- sharded single instance
struct tp_comm {
    ncclComm_t c = nullptr;
    int nranks = 1, rank = 0;
};

int tp_comm_unique_id(uint8_t* id) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == TP_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        TPB_NCCL(nccl().get_unique_id(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

int tp_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, tp_comm** out) {
    return guarded([&] {
        require_device();
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(kInvalidArgument, "tp_comm_create: bad rank");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto c = std::make_unique<tp_comm>();
        TPB_NCCL(nccl().comm_init_rank(&c->c, nranks, u, rank));
        c->nranks = nranks;
        c->rank = rank;
        *out = c.release();
    });
}

int tp_comm_destroy(tp_comm* c) {
    return guarded([&] {
        if (!c) return;
        if (c->c) nccl().comm_destroy(c->c);
        delete c;
    });
}

int tp_solver_set_comm(tp_solver* s, tp_comm* c) {
    return guarded([&] {
        if (c) s->s->set_shard(c->c, c->nranks, c->rank);
        else s->s->set_shard(nullptr, 1, 0);
    });
}

int tp_shard_tiles(int32_t ld, int32_t nranks, int32_t rank, int32_t* tiles, int32_t* count) {
    return guarded([&] {
        const std::vector<int> t = oz_shard_tiles(ld, nranks, rank);
        if (tiles) std::copy(t.begin(), t.end(), tiles);
        *count = (int32_t)t.size();
    });
}

int tp_solver_dims(tp_solver* s, int32_t* d) {
    return guarded([&] {
        const Layout& lo = s->s->layout();
        const int32_t v[12] = {lo.n, lo.m, lo.nx, lo.neq, lo.off_s, lo.off_y, lo.off_t,
                               lo.lambda_ix, lo.off_z, lo.off_nu, s->s->batch(), lo.off_z >= 0};
        std::copy(v, v + 12, d);
    });
}

int tp_solver_state(tp_solver* s, double** x, double** y, double** d) {
    return guarded([&] {
        Dev& dv = s->s->dev();
        if (x) *x = dv.X;
        if (y) *y = dv.Y;
        if (d) *d = dv.D;
    });
}

int tp_solver_download(tp_solver* s, double* x, double* y, double* d) {
    return guarded([&] { s->s->download(x, y, d); });
}

int tp_solver_bench_phase(tp_solver* s, int32_t phase, int32_t reps, int32_t* launches_per_rep) {
    return guarded([&] {
        const int per = s->s->bench_phase(phase, reps);
        if (launches_per_rep) *launches_per_rep = per;
    });
}

int tp_solver_launches_per_iteration(tp_solver* s, int32_t* out) {
    return guarded([&] { *out = s->s->launches_per_iteration(); });
}

int tp_solver_cg_stats(tp_solver* s, int32_t b, int32_t* iters, double* rel_res) {
    return guarded([&] {
        int it = 0;
        double rr = 0.0;
        s->s->cg_stats(b, &it, &rr);
        if (iters) *iters = it;
        if (rel_res) *rel_res = rr;
    });
}

namespace {
// Plan cache of tp_solve: a small process-wide pool of idle homogeneous
// solvers (device buffers, digit planes, TMA maps, captured iteration graphs).
// A call checks out a plan of its shape (device, n, r, config) exclusively
// and returns it afterwards, so concurrent callers never share a solver, and
// at most kPlanCap idle plans are retained (least recently used evicted).
// Solver::start() resets every piece of iteration state, so a reused solver
// returns bitwise what a fresh one does (tested). tp_release_plans() frees
// the pool. The pool itself is never destroyed at exit (no CUDA calls after
// the runtime may have shut down).
struct HomPlan {
    int dev = -1, n = 0, r = 0;
    Config c;
    std::unique_ptr<Solver> s;
};
constexpr size_t kPlanCap = 2;
std::mutex g_plan_mu;
std::vector<std::unique_ptr<HomPlan>>& plan_pool() {
    static auto* pool = new std::vector<std::unique_ptr<HomPlan>>();
    return *pool;
}

bool same_cfg(const Config& a, const Config& b) {
    return a.rho == b.rho && a.epsilon == b.epsilon && a.max_iter == b.max_iter && a.alpha == b.alpha &&
           a.weight_floor == b.weight_floor && a.linear_tol == b.linear_tol &&
           a.trace_stride == b.trace_stride && a.slem_tol == b.slem_tol && a.chunk == b.chunk &&
           a.linear_solver == b.linear_solver && a.cg_max_iter == b.cg_max_iter;
}

std::unique_ptr<HomPlan> take_plan(int n, int r, const Config& c) {
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto& pool = plan_pool();
        for (auto it = pool.end(); it != pool.begin();) {
            --it;
            HomPlan& p = **it;
            if (p.dev == dev && p.n == n && p.r == r && same_cfg(p.c, c)) {
                std::unique_ptr<HomPlan> out = std::move(*it);
                pool.erase(it);
                return out;
            }
        }
    }
    auto p = std::make_unique<HomPlan>();
    p->dev = dev;
    p->n = n;
    p->r = r;
    p->c = c;
    p->s = std::make_unique<Solver>(n, 1, false, std::vector<int>{r}, std::vector<int>{}, c);
    return p;
}

void give_plan(std::unique_ptr<HomPlan> p) {
    std::unique_ptr<HomPlan> evicted;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto& pool = plan_pool();
        pool.push_back(std::move(p));
        if (pool.size() > kPlanCap) {
            evicted = std::move(pool.front());
            pool.erase(pool.begin());
        }
    }
    if (evicted) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(evicted->dev);
        evicted.reset();
        cudaSetDevice(cur);
    }
}

void release_plans() {
    std::vector<std::unique_ptr<HomPlan>> all;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        all.swap(plan_pool());
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& p : all) {
        cudaSetDevice(p->dev);
        p.reset();
    }
    cudaSetDevice(cur);
}
}  // namespace

int tp_release_plans(void) {
    return guarded([&] { release_plans(); });
}

int tp_solve(int32_t n, int32_t r, const tp_config* cfg, const int32_t* warm_edges, int32_t n_warm,
             tp_result* out, int32_t* edges, double* weights, double* trace, char* note,
             int32_t note_cap) {
    return guarded([&] {
        require_device();
        const Config c = to_cfg(cfg);
        validate(c);
        std::vector<int> warm;
        if (n_warm >= 0) warm = packed_edges(n, warm_edges, n_warm);
        else warm = default_warm(n, r, cfg ? cfg->seed : 0);
        std::unique_ptr<HomPlan> plan = take_plan(n, r, c);
        Solver& s = *plan->s;
        s.set_warm(0, warm);  // a failed solve drops its plan (may be unusable)
        s.start();
        s.run_to_completion();
        s.finish();
        const SolveResult R = s.result(0);
        give_plan(std::move(plan));
        if (R.w.empty()) throw Error(kDegenerate, "every edge weight is at or below the floor");
        fill_result(R, out, edges, weights, trace, note, note_cap);
    });
}

int tp_solve_het_node(int32_t n, const int32_t* degrees, const tp_config* cfg,
                      const int32_t* warm_edges, int32_t n_warm, tp_result* out, int32_t* edges,
                      double* weights, double* trace, char* note, int32_t note_cap) {
    return guarded([&] {
        require_device();
        const Config c = to_cfg(cfg);
        validate(c);
        std::vector<int> dg(degrees, degrees + n);
        Solver s(n, 1, true, {}, dg, c);
        std::vector<int> warm;
        if (n_warm >= 0) {
            warm = packed_edges(n, warm_edges, n_warm);
        } else {
            // anneal_topology -> anneal_degree_topology (proj/src/anneal.cpp:393-407)
            AnnealParams ap;
            ap.seed = cfg ? cfg->seed : 0;
            warm = anneal_degree_packed(dg, ap);
        }
        s.set_warm(0, warm);
        s.start();
        s.run_to_completion();
        s.finish();
        fill_result(s.result(0), out, edges, weights, trace, note, note_cap);
    });
}

int tp_anneal_degree(int32_t n, const int32_t* degrees, double t0, double cooling, int32_t steps,
                     int32_t moves_per_temp, uint64_t seed, int32_t* edges, int32_t* n_edges) {
    return guarded([&] {
        AnnealParams ap;
        ap.t0 = t0;
        ap.cooling = cooling;
        ap.steps = steps;
        ap.moves_per_temp = moves_per_temp;
        ap.seed = seed;
        const auto es = anneal_degree_edges(std::vector<int>(degrees, degrees + n), ap);
        for (size_t k = 0; k < es.size(); ++k) {
            edges[2 * k] = es[k].first;
            edges[2 * k + 1] = es[k].second;
        }
        *n_edges = (int32_t)es.size();
    });
}

int tp_device_mt19937_64(uint64_t seed, int32_t k, uint64_t* out) {
    return guarded([&] {
        if (k < 0) throw Error(kInvalidArgument, "negative count");
        device_mt19937_64(seed, k, out);
    });
}

int tp_default_warm_start(int32_t n, int32_t r, uint64_t seed, int32_t* edges, int32_t* n_edges) {
    return guarded([&] {
        if (n < 2) throw Error(kInvalidArgument, "enumerate_edges: need at least two nodes");
        const auto packed = default_warm(n, r, seed);
        for (size_t k = 0; k < packed.size(); ++k) {
            // invert the packed index on the host
            long long l = packed[k];
            int i = 0;
            while (edge_base(n, i + 1) <= l && i < n - 2) ++i;
            edges[2 * k] = i;
            edges[2 * k + 1] = (int)(l - edge_base(n, i)) + i + 1;
        }
        *n_edges = (int32_t)packed.size();
    });
}

}  // extern "C"

namespace {

std::vector<int> default_warm(int n, int r, uint64_t seed) {
    // proj/src/admm.cpp:337-354: Alg. 1 with unit bandwidths, then the
    // balanced-degree anneal; r < n-1 falls back to a chain of r edges.
    std::vector<double> b(n, 1.0);
    std::vector<int32_t> e(n);
    double bu = 0.0;
    const int st = tp_allocate(b.data(), nullptr, n, r, &bu, e.data());
    if (st == TP_OK) {
        try {
            AnnealParams ap;
            ap.seed = seed;
            return anneal_degree_packed(std::vector<int>(e.begin(), e.end()), ap);
        } catch (const Error& err) {
            if (err.status != kInfeasible) throw;
        }
    } else if (st != TP_ERR_INFEASIBLE) {
        throw Error(st, last_error_ref());
    }
    std::vector<int> chain;
    for (int i = 0; i < r; ++i) chain.push_back((int)edge_idx(n, i, i + 1));
    return chain;
}

}  // namespace

namespace {

// capacity rows from the C ABI arrays, checked as check_system does
// (proj/src/admm_het.cpp:20-31)
CapSystem cap_system(int n, int nrows, const int32_t* row_ptr, const int32_t* cols, const int32_t* caps,
                     const int32_t* allowed) {
    if (n < 2) throw Error(kInvalidArgument, "capacity system: need at least 2 nodes");
    if (nrows < 0 || !row_ptr || !allowed || (nrows > 0 && (!cols || !caps)))
        throw Error(kInvalidArgument, "capacity system: malformed rows");
    const int m = n * (n - 1) / 2;
    CapSystem s;
    s.nrows = nrows;
    s.row_ptr.assign(row_ptr, row_ptr + nrows + 1);
    if (s.row_ptr[0] != 0) throw Error(kInvalidArgument, "capacity system: malformed rows");
    for (int r = 0; r < nrows; ++r)
        if (s.row_ptr[r + 1] < s.row_ptr[r]) throw Error(kInvalidArgument, "capacity system: malformed rows");
    s.cols.assign(cols ? cols : row_ptr, (cols ? cols : row_ptr) + s.row_ptr[nrows]);
    for (int r = 0; r < nrows; ++r)
        for (int q = s.row_ptr[r]; q < s.row_ptr[r + 1]; ++q)
            if (s.cols[q] < 0 || s.cols[q] >= m)
                throw Error(kInvalidArgument, "capacity system: row " + std::to_string(r) +
                                                  " references a column outside [0, |E|)");
    s.caps.assign(caps ? caps : row_ptr, (caps ? caps : row_ptr) + nrows);
    s.allowed.assign(allowed, allowed + m);
    return s;
}

CapRows cap_rows(const CapSystem& s) {
    CapRows r;
    r.nrows = s.nrows;
    r.row_ptr = s.row_ptr;
    r.cols = s.cols;
    r.caps = s.caps;
    r.allowed = s.allowed;
    return r;
}

}  // namespace

extern "C" {

int tp_solve_het_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                          const int32_t* caps, const int32_t* allowed, int32_t r, const tp_config* cfg,
                          const int32_t* warm_edges, int32_t n_warm, tp_result* out, int32_t* edges,
                          double* weights, double* trace, char* note, int32_t note_cap) {
    return guarded([&] {
        require_device();
        const Config c = to_cfg(cfg);
        validate(c);
        const CapSystem sys = cap_system(n, nrows, row_ptr, cols, caps, allowed);
        const int m = n * (n - 1) / 2;
        if (r < 1 || r > m) throw Error(kInvalidArgument, "assemble_het: edge total outside [1, |E|]");
        std::vector<int> warm;
        if (n_warm >= 0) {
            warm = packed_edges(n, warm_edges, n_warm);
        } else {
            // anneal_topology -> anneal_capacity_topology (proj/src/anneal.cpp:393-407)
            AnnealParams ap;
            ap.seed = cfg ? cfg->seed : 0;
            for (const auto& e : anneal_capacity_edges(n, cap_rows(sys), r, ap))
                warm.push_back((int)edge_idx(n, e.first, e.second));
        }
        Solver s(n, 1, true, {r}, {}, c, &sys);
        s.set_warm(0, warm);
        s.start();
        s.run_to_completion();
        s.finish();
        fill_result(s.result(0), out, edges, weights, trace, note, note_cap);
    });
}

int tp_project_Y_het_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                              const int32_t* caps, const int32_t* allowed, int32_t r, double alpha, double rho,
                              const double* x, const double* d, double* y) {
    return guarded([&] {
        require_device();
        const CapSystem sys = cap_system(n, nrows, row_ptr, cols, caps, allowed);
        Config c;
        c.alpha = alpha;
        c.rho = rho;
        c.max_iter = 1;
        Solver s(n, 1, true, {r}, {}, c, &sys);
        s.upload(x, nullptr, d);
        s.project_only();
        s.download(nullptr, y, nullptr);
    });
}

int tp_anneal_capacity(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols, const int32_t* caps,
                       const int32_t* allowed, int32_t r, double t0, double cooling, int32_t steps,
                       int32_t moves_per_temp, uint64_t seed, int32_t* edges, int32_t* n_edges) {
    return guarded([&] {
        const CapSystem sys = cap_system(n, nrows, row_ptr, cols, caps, allowed);
        AnnealParams ap;
        ap.t0 = t0;
        ap.cooling = cooling;
        ap.steps = steps;
        ap.moves_per_temp = moves_per_temp;
        ap.seed = seed;
        const auto es = anneal_capacity_edges(n, cap_rows(sys), r, ap);
        for (size_t k = 0; k < es.size(); ++k) {
            edges[2 * k] = es[k].first;
            edges[2 * k + 1] = es[k].second;
        }
        *n_edges = (int32_t)es.size();
    });
}

}  // extern "C"
