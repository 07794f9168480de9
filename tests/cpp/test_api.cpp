// Drop-in check: reference-style C++ code compiled against include/topoopt/
// and linked with libtopoopt_b200.so (the checks mirror proj/tests/test_admm.cpp,
// test_admm_het.cpp, test_bandwidth.cpp and acceptance gate 2). Exit code =
// number of failed checks.
#include <cmath>
#include <cstdio>
#include <optional>
#include <string>

#include "topoopt/admm.hpp"
#include "topoopt/consensus.hpp"
#include "topoopt/admm_het.hpp"
#include "topoopt/bandwidth.hpp"
#include "topoopt/eig.hpp"
#include "topoopt/errors.hpp"
#include "topoopt/topology.hpp"

using namespace topoopt;

static int failures = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        if (!(cond)) {                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
            ++failures;                                                         \
        }                                                                       \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                             \
    do {                                                                        \
        bool caught = false;                                                    \
        try {                                                                   \
            (void)(expr);                                                       \
        } catch (const type&) {                                                 \
            caught = true;                                                      \
        } catch (...) {                                                         \
        }                                                                       \
        if (!caught) {                                                          \
            std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, \
                        #expr, #type);                                          \
            ++failures;                                                         \
        }                                                                       \
    } while (0)

static bool near(double a, double b, double tol) { return std::abs(a - b) <= tol; }

int main() {
    // layout (test_admm.cpp:15-34)
    ProblemData p16 = assemble(16, 32, 2.0, 1.0);
    CHECK(p16.m == 120 && p16.nx == 649 && p16.neq == 528);
    CHECK_THROWS_AS(assemble(4, 0, 2.0, 1.0), std::invalid_argument);

    // cardinality thinning with ties (test_admm.cpp:79-99)
    ProblemData tie = assemble(3, 2, 2.0, 1.0);
    Vec xt(tie.nx, 0.0), dt(tie.nx, 0.0);
    xt[0] = xt[1] = xt[2] = 0.4;
    Vec yt = project_Y(tie, xt, dt);
    CHECK(yt[0] == 0.4 && yt[1] == 0.4 && yt[2] == 0.0);

    // x-step satisfies the KKT equality rows to the shift (test_admm.cpp:121-137)
    ProblemData pd = assemble(4, 4, 2.0, 1.0);
    Vec y(pd.nx), du(pd.nx, 0.0);
    for (int k = 0; k < pd.nx; ++k) y[k] = std::sin(0.37 * k);
    Vec warm;
    Vec x = update_X(pd, y, du, warm, 1e-12);
    CHECK((int)warm.size() == pd.nx + pd.neq);
    // row block 2: diag L(g) + y_slack = 1 (up to the 1e-8 regularisation)
    for (int i = 0; i < pd.n; ++i) {
        double deg = 0.0;
        for (int l = 0; l < pd.m; ++l)
            if (pd.pairs[l].first == i || pd.pairs[l].second == i) deg += x[l];
        CHECK(near(deg + x[pd.off_y + i] - 1e-8 * warm[pd.nx + 2 * 16 + i], 1.0, 1e-6));
    }

    // dual ascent (test_admm.cpp:139-144)
    ProblemData pdd = assemble(3, 2, 2.0, 2.5);
    Vec xo(pdd.nx, 1.0), yo(pdd.nx, 0.25), dd(pdd.nx, 0.5);
    update_duals(pdd, xo, yo, dd);
    CHECK(near(dd[5], 0.5 + 2.5 * 0.75, 1e-15));

    // acceptance gate 2: n=16, r=32 design (acceptance.cpp:83-96)
    SolverConfig cfg;
    cfg.rho = 10.0;
    cfg.epsilon = 1e-8;
    cfg.max_iter = 40000;
    Solution sol = solve(16, 32, cfg);
    CHECK(sol.converged && sol.connected);
    CHECK(sol.iterations == 556);
    CHECK(sol.acf_value <= 0.57);
    CHECK(near(sol.acf_value, 0.52512880769628756, 1e-6));
    CHECK(sol.topology.edges.size() == 32);
    CHECK(max_abs_diff(sol.w, gossip_matrix(sol.topology)) < 1e-12);
    CHECK(near(acf(sol.w), sol.acf_value, 1e-10));
    CHECK(sol.trace_csv().rfind("iter,residual,lambda_tilde,acf_iterate\n", 0) == 0);

    // warm start steering (test_admm.cpp:231-247)
    Topology star;
    star.n = 5;
    for (int leaf = 1; leaf < 5; ++leaf) {
        star.edges.push_back({0, leaf});
        star.weights.push_back(0.25);
    }
    cfg.max_iter = 10000;
    Solution s5 = solve(5, 4, cfg, star);
    CHECK(s5.connected && near(s5.acf_value, 0.75, 0.01));

    // two-tier allocation goldens (test_bandwidth.cpp:38-52)
    BandwidthProfile prof;
    prof.bandwidths.assign(8, 9.76);
    prof.bandwidths.insert(prof.bandwidths.end(), 8, 3.25);
    Allocation a32 = allocate_edge_capacity(prof, 32);
    CHECK(near(a32.b_unit, 1.625, 1e-15) && a32.edges_per_node[0] == 6 && a32.edges_per_node[15] == 2);

    // node-level heterogeneous solve: exact degrees (acceptance gate 6)
    CapacitySystem sys = node_level_constraints(16, a32.edges_per_node);
    SolverConfig hc;
    hc.rho = 10.0;
    hc.epsilon = 1e-8;
    hc.max_iter = 3000;
    Solution hs = solve_het(sys, std::nullopt, hc);
    CHECK(hs.connected && hs.topology.degrees() == a32.edges_per_node);

    // cones and spectra
    Matrix m(3, 3, 0.0);
    m(0, 0) = 2.0;
    m(1, 1) = -3.0;
    m(2, 2) = 0.5;
    Matrix mp = project_psd(m), mn = project_nsd(m);
    CHECK(near(mp(0, 0), 2.0, 1e-12) && near(mp(1, 1), 0.0, 1e-12) && near(mn(1, 1), -3.0, 1e-12));
    Topology ex = generate_benchmark(BenchmarkKind::exponential, 256);
    CHECK(near(acf(gossip_matrix(ex)), 7.0 / 9.0, 1e-12));

    // capacity-bound systems (proj/tests/test_admm_het.cpp:171-202)
    CapacitySystem tree = intra_server_constraints(tiered8_tree(4.88, 4.88, 9.76));
    CHECK(!tree.equality && tree.rows.size() == 7 && tree.rows[6].capacity == 16);
    SolverConfig tight;
    tight.rho = 10.0;
    tight.epsilon = 1e-8;
    tight.max_iter = 3000;
    Solution ts = solve_het(tree, 12, tight);
    CHECK(ts.connected && ts.topology.edges.size() <= 12);
    const auto util = utilization(tree, ts.topology);
    for (size_t k = 0; k < util.size(); ++k) CHECK(util[k].used <= util[k].capacity);
    CHECK(utilization_csv(util).rfind("resource,capacity,used\n", 0) == 0);
    CapacitySystem cube = bcube_constraints({2, 2, {}});
    Topology cycle;
    cycle.n = 4;
    cycle.edges = {{0, 1}, {0, 2}, {1, 3}, {2, 3}};
    cycle.weights.assign(4, 1.0 / 3.0);
    Solution cs = solve_het(cube, 5, tight, cycle);
    CHECK(cs.topology.edges.size() == 4);
    CHECK(cs.note.find("capacity limits stopped selection at 4 of 5") != std::string::npos);
    CHECK_THROWS_AS(solve_het(cube, std::nullopt, tight), std::invalid_argument);

    // consensus evaluation (proj/src/consensus.cpp)
    ConsensusTrace tr = simulate(gossip_matrix(ex), 8, 50, 3);
    CHECK(tr.errors.size() == 51 && tr.errors[50] < tr.errors[0]);
    CHECK(convergence_time(tr, tr.errors[10], 2.0) <= 20.0);
    CompareReport rep = compare({{"exp", gossip_matrix(ex), 1.0}}, 4, 20, 1e-3, 0);
    CHECK(rep.traces.size() == 1 && rep.to_csv().rfind("time_ms,label,error\n", 0) == 0);

    // on-disk formats (proj/src/topology.cpp:283-324)
    Topology small;
    small.n = 4;
    small.edges = {{2, 3}, {0, 1}, {0, 3}};
    small.weights = {0.30000000000000004, 1e-05, 0.5};
    const std::string js = topology_to_json(small);
    CHECK(js.find("\"weights\": [\n    1e-05,\n    0.5,\n    0.30000000000000004\n  ]") != std::string::npos);
    Topology back = topology_from_json(js);
    CHECK(back.n == 4 && back.edges.size() == 3 && back.edges[0] == Edge(0, 1) && back.weights[2] == 0.30000000000000004);
    CHECK(matrix_to_csv(gossip_matrix(back)).rfind("0.49999000000000005,1.0000000000000001e-05,0,0.5\n", 0) == 0);
    CHECK_THROWS_AS(topology_from_json("{\"n\": 4}"), std::invalid_argument);

    // errors
    CHECK_THROWS_AS(extract_topology(3, 2, Vec{0.0, 0.0, 0.0}, 1e-6), DegenerateSolutionError);
    CHECK_THROWS_AS(node_level_constraints(3, {1, 1, 1}), InfeasibleError);
    SolverConfig bad;
    bad.epsilon = 0.0;
    CHECK_THROWS_AS(bad.validate(), std::invalid_argument);

    std::printf("cpp api: %d failure(s)\n", failures);
    return failures;
}
