// Reference-compatible C++ API (include/topoopt/topoopt_b200.hpp) over the C
// ABI (include/topoopt_b200.h). Host value types and formatting live here; the
// numerical work of every hot-path call runs on the GPU behind the ABI.
#include "topoopt/topoopt_b200.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cctype>
#include <numeric>
#include <limits>
#include <map>
#include <set>

#include "topoopt_b200.h"
#include "json_lite.hpp"

#include <deque>
#include <functional>
#include <variant>

namespace topoopt {

namespace detail {
SparseMatrix build_kkt(int n, int q, bool het, const std::vector<std::vector<int>>& degree_rows);
}

namespace {

// ABI status -> the reference's exception taxonomy
void raise(int status) {
    if (status == TP_OK) return;
    const std::string msg = tp_last_error_message();
    switch (status) {
        case TP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TP_ERR_INFEASIBLE: throw InfeasibleError(msg);
        case TP_ERR_LINEAR_SOLVE: throw LinearSolveError(msg);
        case TP_ERR_DEGENERATE: throw DegenerateSolutionError(msg);
        case TP_ERR_PIVOT: throw PivotError(msg, -1);
        default: throw std::runtime_error(msg);
    }
}

tp_config to_c(const SolverConfig& c) {
    tp_config k;
    tp_config_default(&k);
    k.rho = c.rho;
    k.epsilon = c.epsilon;
    k.max_iter = c.max_iter;
    k.alpha = c.alpha;
    k.weight_floor = c.weight_floor;
    k.seed = c.seed;
    k.linear_tol = c.linear_tol;
    k.linear_solver = c.linear_solver;
    return k;
}

std::vector<int32_t> flat_edges(const Topology& t) {
    std::vector<int32_t> e;
    e.reserve(2 * t.edges.size());
    for (const auto& p : t.edges) {
        e.push_back(p.first);
        e.push_back(p.second);
    }
    return e;
}

Topology from_flat(int n, const int32_t* e, const double* w, int k) {
    Topology t;
    t.n = n;
    for (int i = 0; i < k; ++i) {
        t.edges.push_back({e[2 * i], e[2 * i + 1]});
        t.weights.push_back(w ? w[i] : 0.0);
    }
    return t;
}

Solution collect(int n, const tp_result& res, const std::vector<int32_t>& edges,
                 const std::vector<double>& weights, const std::vector<double>& trace,
                 const char* note) {
    Solution sol;
    sol.topology = from_flat(n, edges.data(), weights.data(), res.n_edges);
    sol.topology.validate();
    sol.w = gossip_matrix(sol.topology);
    sol.lambda_tilde = res.lambda_tilde;
    sol.acf_value = res.acf;
    sol.converged = res.converged != 0;
    sol.connected = res.connected != 0;
    sol.repaired = res.repaired != 0;
    sol.residual = res.residual;
    sol.iterations = res.iterations;
    sol.note = note;
    sol.trace.resize(res.iterations);
    for (int k = 0; k < res.iterations; ++k)
        sol.trace[k] = {k + 1, trace[3 * k], trace[3 * k + 1], trace[3 * k + 2]};
    return sol;
}

// node-level system: equality rows, row i = pairs incident to node i
bool node_level_degrees(const CapacitySystem& sys, std::vector<int32_t>& degrees) {
    if (!sys.equality || (int)sys.rows.size() != sys.n) return false;
    const auto pairs = enumerate_edges(sys.n);
    for (int i = 0; i < sys.n; ++i) {
        std::vector<int> want;
        for (int c = 0; c < (int)pairs.size(); ++c)
            if (pairs[c].first == i || pairs[c].second == i) want.push_back(c);
        std::vector<int> have = sys.rows[i].edge_cols;
        std::sort(have.begin(), have.end());
        if (have != want) return false;
    }
    for (char a : sys.allowed)
        if (!a) return false;
    degrees.resize(sys.n);
    for (int i = 0; i < sys.n; ++i) degrees[i] = sys.rows[i].capacity;
    return true;
}

}  // namespace

// ------------------------------------------------------------------ dense
Matrix Matrix::identity(int n) {
    Matrix m(n, n, 0.0);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: shape mismatch");
    Matrix c(a.rows(), b.cols(), 0.0);
    for (int i = 0; i < a.rows(); ++i)
        for (int k = 0; k < a.cols(); ++k) {
            const double x = a(i, k);
            for (int j = 0; j < b.cols(); ++j) c(i, j) += x * b(k, j);
        }
    return c;
}

Matrix transpose(const Matrix& a) {
    Matrix t(a.cols(), a.rows());
    for (int i = 0; i < a.rows(); ++i)
        for (int j = 0; j < a.cols(); ++j) t(j, i) = a(i, j);
    return t;
}

double max_abs_diff(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw std::invalid_argument("max_abs_diff: shape mismatch");
    double m = 0.0;
    for (size_t k = 0; k < a.data().size(); ++k) m = std::max(m, std::abs(a.data()[k] - b.data()[k]));
    return m;
}

double frobenius_norm(const Matrix& a) {
    double s = 0.0;
    for (double v : a.data()) s += v * v;
    return std::sqrt(s);
}

bool is_symmetric(const Matrix& a, double tol) {
    if (a.rows() != a.cols()) return false;
    for (int i = 0; i < a.rows(); ++i)
        for (int j = i + 1; j < a.cols(); ++j)
            if (std::abs(a(i, j) - a(j, i)) > tol) return false;
    return true;
}

Matrix symmetrize(const Matrix& a) {
    Matrix s(a.rows(), a.cols());
    for (int i = 0; i < a.rows(); ++i)
        for (int j = 0; j < a.cols(); ++j) s(i, j) = 0.5 * (a(i, j) + a(j, i));
    return s;
}

double dot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t k = 0; k < a.size(); ++k) s += a[k] * b[k];
    return s;
}

double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }

void axpy(double alpha, const Vec& x, Vec& y) {
    for (size_t k = 0; k < x.size(); ++k) y[k] += alpha * x[k];
}

// ------------------------------------------------------------------ topology
void Topology::validate() const {
    if (n < 1) throw std::invalid_argument("topology: n must be positive");
    if (weights.size() != edges.size())
        throw std::invalid_argument("topology: weights length differs from edge count");
    for (size_t k = 0; k < edges.size(); ++k) {
        const int i = edges[k].first, j = edges[k].second;
        if (i < 0 || j < 0 || i >= n || j >= n)
            throw std::invalid_argument("topology: edge endpoint out of range");
        if (i >= j) throw std::invalid_argument("topology: edge endpoints must satisfy i < j");
        if (k > 0 && !(edges[k - 1] < edges[k]))
            throw std::invalid_argument("topology: edges must be sorted without duplicates");
        if (!(weights[k] >= 0.0)) throw std::invalid_argument("topology: negative or NaN weight");
    }
}

void Topology::normalize_and_validate() {
    if (weights.size() != edges.size())
        throw std::invalid_argument("topology: weights length differs from edge count");
    std::vector<size_t> ord(edges.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return edges[a] < edges[b]; });
    std::vector<Edge> e2;
    std::vector<double> w2;
    for (size_t k : ord) {
        e2.push_back(edges[k]);
        w2.push_back(weights[k]);
    }
    edges.swap(e2);
    weights.swap(w2);
    validate();
}

std::vector<int> Topology::degrees() const {
    std::vector<int> d(n, 0);
    for (const auto& e : edges) {
        ++d[e.first];
        ++d[e.second];
    }
    return d;
}

bool Topology::has_uniform_weights(double tol) const {
    for (double w : weights)
        if (std::abs(w - weights.front()) > tol) return false;
    return true;
}

std::vector<Edge> enumerate_edges(int n) {
    if (n < 2) throw std::invalid_argument("enumerate_edges: need at least two nodes");
    std::vector<Edge> out;
    out.reserve(static_cast<size_t>(n) * (n - 1) / 2);
    for (int i = 0; i + 1 < n; ++i)
        for (int j = i + 1; j < n; ++j) out.push_back({i, j});
    return out;
}

int edge_index(int n, int i, int j) {
    if (i == j) throw std::invalid_argument("edge_index: self loop");
    if (i > j) std::swap(i, j);
    if (i < 0 || j >= n) throw std::invalid_argument("edge_index: endpoint out of range");
    return i * n - i * (i + 1) / 2 + (j - i - 1);
}

Matrix incidence_matrix(const Topology& t) {
    // proj/include/topoopt/topology.hpp:36-38: column per edge, +1 at the
    // lower endpoint, -1 at the higher one
    t.validate();
    Matrix a(t.n, (int)t.edges.size());
    for (size_t c = 0; c < t.edges.size(); ++c) {
        a(t.edges[c].first, (int)c) = 1.0;
        a(t.edges[c].second, (int)c) = -1.0;
    }
    return a;
}

double aspl(const Topology& t) {
    // mean hop distance over unordered pairs (BFS from every node);
    // +infinity when disconnected (proj/include/topoopt/topology.hpp:60-62)
    t.validate();
    const int n = t.n;
    if (n < 2) return 0.0;
    std::vector<std::vector<int>> adj(n);
    for (const auto& [i, j] : t.edges) {
        adj[i].push_back(j);
        adj[j].push_back(i);
    }
    long long total = 0;
    std::vector<int> dist(n);
    std::deque<int> q;
    for (int s0 = 0; s0 < n; ++s0) {
        std::fill(dist.begin(), dist.end(), -1);
        dist[s0] = 0;
        q.assign(1, s0);
        int seen = 1;
        while (!q.empty()) {
            const int u = q.front();
            q.pop_front();
            for (int v : adj[u])
                if (dist[v] < 0) {
                    dist[v] = dist[u] + 1;
                    total += dist[v];
                    ++seen;
                    q.push_back(v);
                }
        }
        if (seen < n) return std::numeric_limits<double>::infinity();
    }
    return (double)total / ((double)n * (n - 1));  // each pair counted twice
}

Matrix laplacian(const Topology& t) {
    t.validate();
    Matrix l(t.n, t.n, 0.0);
    for (size_t k = 0; k < t.edges.size(); ++k) {
        const int i = t.edges[k].first, j = t.edges[k].second;
        const double w = t.weights[k];
        l(i, i) += w;
        l(j, j) += w;
        l(i, j) -= w;
        l(j, i) -= w;
    }
    return l;
}

Matrix gossip_matrix(const Topology& t) {
    Matrix l = laplacian(t);
    for (int i = 0; i < t.n; ++i)
        if (l(i, i) > 1.0 + 1e-12)
            throw std::invalid_argument("gossip_matrix: weighted degree " + std::to_string(l(i, i)) +
                                        " at node " + std::to_string(i) + " exceeds 1");
    Matrix w = Matrix::identity(t.n);
    for (size_t k = 0; k < w.data().size(); ++k) w.data()[k] -= l.data()[k];
    return w;
}

SpectralReport spectral_report(const Matrix& w) {
    if (w.rows() != w.cols()) throw std::invalid_argument("spectral_report: matrix not square");
    double out[4];
    raise(tp_spectral_report(w.rows(), w.data().data(), out));
    return SpectralReport{out[0], out[1], out[2], out[3] != 0.0};
}

double acf(const Matrix& w) { return spectral_report(w).acf; }

void validate_gossip(const Matrix& w) {
    const int n = w.rows();
    if (n < 1 || w.cols() != n) throw std::invalid_argument("gossip matrix must be square");
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) {
            if (std::abs(w(i, j) - w(j, i)) > 1e-8)
                throw std::invalid_argument("gossip matrix asymmetric beyond 1e-8");
            if (w(i, j) < -1e-8) throw std::invalid_argument("gossip matrix has an entry below -1e-8");
            s += w(i, j);
        }
        if (std::abs(s - 1.0) > 1e-8)
            throw std::invalid_argument("gossip matrix row " + std::to_string(i) + " does not sum to 1");
    }
}

BenchmarkKind benchmark_kind_from_string(const std::string& name) {
    if (name == "ring") return BenchmarkKind::ring;
    if (name == "grid2d") return BenchmarkKind::grid2d;
    if (name == "torus2d") return BenchmarkKind::torus2d;
    if (name == "exponential") return BenchmarkKind::exponential;
    throw std::invalid_argument("unknown benchmark kind: " + name);
}

Topology generate_benchmark(BenchmarkKind kind, int n) {
    // baselines of proj/src/topology.cpp:227-281 (uniform 1/(d_max+1), or
    // 1/(2 (hops+1)) for the exponential graph)
    if (n < 2) throw std::invalid_argument("generate_benchmark: need at least two nodes");
    std::set<Edge> es;
    auto add = [&](int a, int b) {
        if (a != b) es.insert({std::min(a, b), std::max(a, b)});
    };
    double weight = 0.0;
    if (kind == BenchmarkKind::ring) {
        if (n < 3) throw std::invalid_argument("generate_benchmark: ring needs n >= 3");
        for (int i = 0; i < n; ++i) add(i, (i + 1) % n);
        weight = 1.0 / 3.0;
    } else if (kind == BenchmarkKind::exponential) {
        int hops = 0;
        for (int h = 1; h <= n - 1; h *= 2, ++hops)
            for (int i = 0; i < n; ++i) add(i, (i + h) % n);
        weight = 1.0 / (2.0 * (hops + 1));
    } else {
        const int s = (int)std::lround(std::sqrt((double)n));
        if (s * s != n || s < 2)
            throw std::invalid_argument("generate_benchmark: grid/torus needs a perfect square n >= 4");
        const bool torus = kind == BenchmarkKind::torus2d;
        for (int r = 0; r < s; ++r)
            for (int c = 0; c < s; ++c) {
                const int u = r * s + c;
                if (torus) {
                    add(u, r * s + (c + 1) % s);
                    add(u, ((r + 1) % s) * s + c);
                } else {
                    if (c + 1 < s) add(u, u + 1);
                    if (r + 1 < s) add(u, u + s);
                }
            }
        weight = 1.0 / ((s >= 3 ? 4 : 2) + 1);
    }
    Topology t;
    t.n = n;
    t.edges.assign(es.begin(), es.end());
    t.weights.assign(t.edges.size(), weight);
    t.normalize_and_validate();
    return t;
}

// ------------------------------------------------------------------ formats
std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

namespace {
// nlohmann::json's double layout: shortest round-trip digits, fixed notation
// for decimal exponents in (-5, 15], d.ddde+XX otherwise, ".0" on integers
std::string json_number(double v) {
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*e", p - 1, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string t(buf), sign;
    if (t[0] == '-') {
        sign = "-";
        t = t.substr(1);
    }
    const size_t epos = t.find('e');
    const int e10 = std::atoi(t.c_str() + epos + 1);
    std::string digits;
    for (size_t i = 0; i < epos; ++i)
        if (t[i] != '.') digits += t[i];
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = (int)digits.size(), n = e10 + 1;
    std::string body;
    if (k <= n && n <= 15) {
        body = digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        body = digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        body = "0." + std::string(-n, '0') + digits;
    } else {
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e10 < 0 ? '-' : '+', std::abs(e10));
        body = digits.substr(0, 1) + (k > 1 ? "." + digits.substr(1) : "") + eb;
    }
    return sign + body;
}

// minimal JSON reader for the topology schema
struct JsonReader {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    }
    [[noreturn]] void fail() const { throw std::invalid_argument("topology json: malformed document"); }
    void expect(char c) {
        ws();
        if (i >= s.size() || s[i] != c) fail();
        ++i;
    }
    bool peek(char c) {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\' && i + 1 < s.size()) ++i;
            out += s[i++];
        }
        if (i >= s.size()) fail();
        ++i;
        return out;
    }
    std::string token() {
        ws();
        const size_t b = i;
        while (i < s.size() && (std::isalnum((unsigned char)s[i]) || s[i] == '-' || s[i] == '+' || s[i] == '.')) ++i;
        if (b == i) fail();
        return s.substr(b, i - b);
    }
    bool is_int(const std::string& t) const { return t.find_first_of(".eE") == std::string::npos; }
};
}  // namespace

std::string topology_to_json(const Topology& t) {
    // proj/src/topology.cpp:283-290
    Topology c = t;
    c.normalize_and_validate();
    std::string out = "{\n  \"edges\": ";
    if (c.edges.empty()) {
        out += "[]";
    } else {
        out += "[\n";
        for (size_t k = 0; k < c.edges.size(); ++k)
            out += "    [\n      " + std::to_string(c.edges[k].first) + ",\n      " +
                   std::to_string(c.edges[k].second) + "\n    ]" + (k + 1 < c.edges.size() ? ",\n" : "\n");
        out += "  ]";
    }
    out += ",\n  \"n\": " + std::to_string(c.n) + ",\n  \"weights\": ";
    if (c.weights.empty()) {
        out += "[]";
    } else {
        out += "[\n";
        for (size_t k = 0; k < c.weights.size(); ++k)
            out += "    " + json_number(c.weights[k]) + (k + 1 < c.weights.size() ? ",\n" : "\n");
        out += "  ]";
    }
    return out + "\n}\n";
}

Topology topology_from_json(const std::string& text) {
    // proj/src/topology.cpp:292-310
    JsonReader r{text};
    Topology t;
    bool has_n = false, has_e = false, has_w = false;
    r.expect('{');
    while (!r.peek('}')) {
        const std::string key = r.str();
        r.expect(':');
        if (key == "n") {
            const std::string tok = r.token();
            if (!r.is_int(tok)) throw std::invalid_argument("topology json: missing integer field 'n'");
            t.n = std::stoi(tok);
            has_n = true;
        } else if (key == "edges" || key == "weights") {
            if (!r.peek('[')) throw std::invalid_argument("topology json: missing array field '" + key + "'");
            r.expect('[');
            while (!r.peek(']')) {
                if (key == "edges") {
                    if (!r.peek('[')) throw std::invalid_argument("topology json: each edge must be a pair");
                    r.expect('[');
                    const int a = std::stoi(r.token());
                    r.expect(',');
                    const int b = std::stoi(r.token());
                    if (!r.peek(']')) throw std::invalid_argument("topology json: each edge must be a pair");
                    r.expect(']');
                    t.edges.push_back({a, b});
                } else {
                    t.weights.push_back(std::strtod(r.token().c_str(), nullptr));
                }
                if (r.peek(',')) r.expect(',');
            }
            r.expect(']');
            (key == "edges" ? has_e : has_w) = true;
        } else {
            // skip a scalar value of an unknown key
            if (r.peek('"')) r.str();
            else r.token();
        }
        if (r.peek(',')) r.expect(',');
    }
    r.expect('}');
    if (!has_n) throw std::invalid_argument("topology json: missing integer field 'n'");
    if (!has_e) throw std::invalid_argument("topology json: missing array field 'edges'");
    if (!has_w) throw std::invalid_argument("topology json: missing array field 'weights'");
    t.normalize_and_validate();
    return t;
}

std::string matrix_to_csv(const Matrix& m) {
    // proj/src/topology.cpp:312-324
    std::string out;
    for (int i = 0; i < m.rows(); ++i) {
        for (int j = 0; j < m.cols(); ++j) {
            out += g17(m(i, j));
            if (j + 1 < m.cols()) out += ',';
        }
        out += '\n';
    }
    return out;
}

std::string matrix_to_triplet_csv(const Matrix& m, double drop_below) {
    std::string out = "i,j,value\n";
    for (int i = 0; i < m.rows(); ++i)
        for (int j = 0; j < m.cols(); ++j) {
            if (std::abs(m(i, j)) <= drop_below) continue;
            out += std::to_string(i) + "," + std::to_string(j) + "," + g17(m(i, j)) + "\n";
        }
    return out;
}

// ------------------------------------------------------------------ consensus

std::string ConsensusTrace::to_csv() const {
    std::string out = "iter,time_ms,error\n";
    for (size_t k = 0; k < errors.size(); ++k)
        out += std::to_string(k) + "," + g17(static_cast<double>(k) * t_iter_ms) + "," + g17(errors[k]) + "\n";
    return out;
}

ConsensusTrace simulate(const Matrix& w, int dim, int iters, std::uint64_t seed) {
    if (w.rows() != w.cols()) throw std::invalid_argument("gossip matrix must be square");
    ConsensusTrace t;
    t.seed = seed;
    t.errors.assign(iters >= 0 ? iters + 1 : 1, 0.0);
    raise(tp_consensus_simulate(w.rows(), w.data().data(), dim, iters, seed, t.errors.data()));
    return t;
}

double convergence_time(const ConsensusTrace& trace, double threshold, double t_iter) {
    // proj/src/consensus.cpp:69-75
    if (!(threshold > 0.0)) throw std::invalid_argument("convergence_time: threshold <= 0");
    if (!(t_iter > 0.0)) throw std::invalid_argument("convergence_time: t_iter <= 0");
    for (size_t k = 0; k < trace.errors.size(); ++k)
        if (trace.errors[k] <= threshold) return static_cast<double>(k) * t_iter;
    return std::numeric_limits<double>::infinity();
}

std::string CompareReport::to_csv() const {
    std::string out = "time_ms,label,error\n";
    for (const auto& trace : traces)
        for (size_t k = 0; k < trace.errors.size(); ++k)
            out += g17(static_cast<double>(k) * trace.t_iter_ms) + "," + trace.label + "," + g17(trace.errors[k]) +
                   "\n";
    return out;
}

CompareReport compare(const std::vector<CompareEntry>& entries, int dim, int iters, double threshold,
                      std::uint64_t seed, int /*threads: the simulations run on the device in turn*/) {
    // proj/src/consensus.cpp:91-120: every entry with the same seed and dim
    CompareReport report;
    for (const auto& e : entries) {
        ConsensusTrace t = simulate(e.w, dim, iters, seed);
        t.label = e.label;
        t.t_iter_ms = e.t_iter_ms;
        report.convergence_ms.push_back(convergence_time(t, threshold, e.t_iter_ms));
        report.traces.push_back(std::move(t));
    }
    return report;
}

// ------------------------------------------------------------------ eig
static Matrix cone(const Matrix& s, bool psd) {
    if (s.rows() != s.cols()) throw std::invalid_argument("sym_eig: matrix not square");
    Matrix out(s.rows(), s.cols());
    raise(psd ? tp_project_psd(s.rows(), s.data().data(), out.data().data())
              : tp_project_nsd(s.rows(), s.data().data(), out.data().data()));
    return out;
}
Matrix project_nsd(const Matrix& s) { return cone(s, false); }

EigDecomposition sym_eig(const Matrix& s) {
    if (s.rows() != s.cols()) throw std::invalid_argument("sym_eig: matrix not square");
    const int n = s.rows();
    EigDecomposition d;
    d.values.assign(n, 0.0);
    d.vectors = Matrix(n, n);
    if (n == 0) return d;
    raise(tp_sym_eig(n, s.data().data(), d.values.data(), d.vectors.data().data()));
    return d;
}
Matrix project_psd(const Matrix& s) { return cone(s, true); }

// ------------------------------------------------------------------ bandwidth
Allocation allocate_edge_capacity(const BandwidthProfile& p, int r) {
    const int n = (int)p.bandwidths.size();
    if (!p.edge_caps.empty() && (int)p.edge_caps.size() != n)
        throw std::invalid_argument("allocate_edge_capacity: edge_caps size mismatch");
    Allocation a;
    a.edges_per_node.assign(std::max(n, 1), 0);
    std::vector<int32_t> e(std::max(n, 1));
    std::vector<int32_t> caps(p.edge_caps.begin(), p.edge_caps.end());
    raise(tp_allocate(p.bandwidths.data(), caps.empty() ? nullptr : caps.data(), n, r, &a.b_unit,
                      e.data()));
    a.edges_per_node.assign(e.begin(), e.begin() + n);
    return a;
}

std::vector<int> CapacitySystem::loads(const std::vector<char>& selected) const {
    if ((int)selected.size() != num_edges)
        throw std::invalid_argument("CapacitySystem::loads: selection size mismatch");
    std::vector<int> out(rows.size(), 0);
    for (size_t k = 0; k < rows.size(); ++k)
        for (int c : rows[k].edge_cols) out[k] += selected[c] ? 1 : 0;
    return out;
}

int CapacitySystem::implied_edge_total() const {
    long long s = 0;
    for (const auto& row : rows) s += row.capacity;
    if (s % 2) throw std::invalid_argument("CapacitySystem: capacity sum is odd, no edge total");
    return (int)(s / 2);
}

SparseMatrix CapacitySystem::row_matrix() const {
    std::vector<Triplet> t;
    for (size_t k = 0; k < rows.size(); ++k)
        for (int c : rows[k].edge_cols) t.push_back({(int)k, c, 1.0});
    return SparseMatrix::from_triplets((int)rows.size(), num_edges, t);
}

CapacitySystem node_level_constraints(int n, const std::vector<int>& degrees) {
    if (n < 2) throw std::invalid_argument("node_level_constraints: need at least 2 nodes");
    if ((int)degrees.size() != n)
        throw std::invalid_argument("node_level_constraints: degree list size mismatch");
    long long sum = 0;
    for (int i = 0; i < n; ++i) {
        if (degrees[i] < 0 || degrees[i] > n - 1)
            throw std::invalid_argument("node_level_constraints: degree of node " + std::to_string(i) +
                                        " outside [0, n-1]");
        sum += degrees[i];
    }
    if (sum % 2) throw InfeasibleError("degree sum " + std::to_string(sum) + " is odd");
    CapacitySystem sys;
    sys.n = n;
    sys.num_edges = n * (n - 1) / 2;
    sys.equality = true;
    sys.allowed.assign(sys.num_edges, 1);
    sys.rows.resize(n);
    int col = 0;
    for (int i = 0; i < n; ++i) {
        sys.rows[i].label = "node" + std::to_string(i);
        sys.rows[i].capacity = degrees[i];
    }
    for (int i = 0; i + 1 < n; ++i)
        for (int j = i + 1; j < n; ++j, ++col) {
            sys.rows[i].edge_cols.push_back(col);
            sys.rows[j].edge_cols.push_back(col);
        }
    for (auto& row : sys.rows) std::sort(row.edge_cols.begin(), row.edge_cols.end());
    return sys;
}

// ------------------------------------------------------------------ anneal
void AnnealConfig::validate() const {
    if (!(t0 > 0.0)) throw std::invalid_argument("AnnealConfig: t0 must be positive");
    if (!(cooling > 0.0 && cooling < 1.0))
        throw std::invalid_argument("AnnealConfig: cooling must lie in (0, 1)");
    if (steps < 1) throw std::invalid_argument("AnnealConfig: steps must be >= 1");
    if (moves_per_temp < 0) throw std::invalid_argument("AnnealConfig: moves_per_temp must be >= 0");
}

Topology anneal_degree_topology(const std::vector<int>& degrees, const AnnealConfig& cfg) {
    cfg.validate();
    const int n = (int)degrees.size();
    long long sum = 0;
    for (int d : degrees) sum += d;
    std::vector<int32_t> e(2 * std::max<long long>(sum / 2, 1));
    int32_t k = 0;
    std::vector<int32_t> deg(degrees.begin(), degrees.end());
    raise(tp_anneal_degree(n, deg.data(), cfg.t0, cfg.cooling, cfg.steps, cfg.moves_per_temp, cfg.seed,
                           e.data(), &k));
    Topology t = from_flat(n, e.data(), nullptr, k);
    int dmax = 0;
    for (int d : t.degrees()) dmax = std::max(dmax, d);
    t.weights.assign(k, 1.0 / (dmax + 1));
    t.validate();
    return t;
}

namespace {
struct FlatRows {
    std::vector<int32_t> row_ptr{0}, cols, caps, allowed;
};
FlatRows flat_rows(const CapacitySystem& sys) {
    FlatRows f;
    for (const auto& row : sys.rows) {
        for (int c : row.edge_cols) f.cols.push_back(c);
        f.row_ptr.push_back((int32_t)f.cols.size());
        f.caps.push_back(row.capacity);
    }
    f.allowed.assign(sys.allowed.begin(), sys.allowed.end());
    if ((int)f.allowed.size() != sys.num_edges)
        throw std::invalid_argument("capacity system: allowed mask size differs from |E|");
    if (f.cols.empty()) f.cols.push_back(0);
    if (f.caps.empty()) f.caps.push_back(0);
    return f;
}
}  // namespace

Topology anneal_topology(const CapacitySystem& sys, std::optional<int> r, const AnnealConfig& cfg) {
    // proj/src/anneal.cpp:393-407
    if (sys.equality) {
        std::vector<int32_t> deg;
        if (!node_level_degrees(sys, deg))
            throw std::invalid_argument("anneal_topology: equality system is not node-level");
        if (r && *r != sys.implied_edge_total())
            throw std::invalid_argument("anneal_topology: r conflicts with the degree sum");
        return anneal_degree_topology(std::vector<int>(deg.begin(), deg.end()), cfg);
    }
    if (!r) throw std::invalid_argument("anneal_topology: capacity mode needs an explicit r");
    return anneal_capacity_topology(sys, *r, cfg);
}

Topology anneal_capacity_topology(const CapacitySystem& sys, int r, const AnnealConfig& cfg) {
    // proj/src/anneal.cpp:275-391
    cfg.validate();
    const FlatRows f = flat_rows(sys);
    std::vector<int32_t> e(2 * (size_t)std::max(r, 1));
    int32_t k = 0;
    raise(tp_anneal_capacity(sys.n, (int32_t)sys.rows.size(), f.row_ptr.data(), f.cols.data(), f.caps.data(),
                             f.allowed.data(), r, cfg.t0, cfg.cooling, cfg.steps, cfg.moves_per_temp, cfg.seed,
                             e.data(), &k));
    Topology t;
    t.n = sys.n;
    int dmax = 0;
    std::vector<int> deg(sys.n, 0);
    for (int q = 0; q < k; ++q) {
        t.edges.push_back({e[2 * q], e[2 * q + 1]});
        dmax = std::max({dmax, ++deg[e[2 * q]], ++deg[e[2 * q + 1]]});
    }
    t.weights.assign(t.edges.size(), 1.0 / (dmax + 1));  // finish (proj/src/anneal.cpp:172-185)
    return t;
}

// ------------------------------------------------------------------ capacity systems
void ServerTree::validate() const {
    // proj/src/bandwidth.cpp:148-170
    if (n_devices < 2) throw std::invalid_argument("ServerTree: need at least 2 devices");
    const int m = n_devices * (n_devices - 1) / 2;
    if ((int)routes.size() != m) throw std::invalid_argument("ServerTree: expected one route per device pair");
    for (const auto& link : links) {
        if (link.name.empty()) throw std::invalid_argument("ServerTree: unnamed link");
        if (!(link.bandwidth > 0.0))
            throw std::invalid_argument("ServerTree: link " + link.name + " needs positive bandwidth");
        if (link.capacity < 0) throw std::invalid_argument("ServerTree: link " + link.name + " has negative capacity");
    }
    for (int col = 0; col < m; ++col) {
        if (routes[col].empty())
            throw std::invalid_argument("ServerTree: pair column " + std::to_string(col) + " routes over no link");
        for (int lix : routes[col])
            if (lix < 0 || lix >= (int)links.size())
                throw std::invalid_argument("ServerTree: route references unknown link");
    }
}

ServerTree tiered8_tree(double leaf_bw, double group_bw, double root_bw) {
    ServerTree tree;
    tree.n_devices = 8;
    for (int l = 0; l < 4; ++l) tree.links.push_back({"leaf" + std::to_string(l), leaf_bw, 1});
    tree.links.push_back({"group0", group_bw, 4});
    tree.links.push_back({"group1", group_bw, 4});
    tree.links.push_back({"root", root_bw, 16});
    for (int i = 0; i + 1 < 8; ++i)
        for (int j = i + 1; j < 8; ++j)
            tree.routes.push_back({i / 2 == j / 2 ? i / 2 : (i / 4 == j / 4 ? 4 + i / 4 : 6)});
    tree.validate();
    return tree;
}

CapacitySystem intra_server_constraints(const ServerTree& tree) {
    tree.validate();
    CapacitySystem sys;
    sys.n = tree.n_devices;
    sys.num_edges = sys.n * (sys.n - 1) / 2;
    sys.equality = false;
    sys.allowed.assign(sys.num_edges, 1);
    sys.rows.resize(tree.links.size());
    for (size_t l = 0; l < tree.links.size(); ++l) {
        sys.rows[l].label = tree.links[l].name;
        sys.rows[l].capacity = tree.links[l].capacity;
    }
    for (int col = 0; col < sys.num_edges; ++col)
        for (int lix : tree.routes[col]) sys.rows[lix].edge_cols.push_back(col);
    return sys;
}

int BCubeSpec::n_servers() const {
    if (p < 2 || k < 1) throw std::invalid_argument("BCubeSpec: need p >= 2 and k >= 1");
    long long n = 1;
    for (int i = 0; i < k; ++i) {
        n *= p;
        if (n > 4096) throw std::invalid_argument("BCubeSpec: p^k exceeds 4096 servers");
    }
    return (int)n;
}

CapacitySystem bcube_constraints(const BCubeSpec& spec) {
    const int n = spec.n_servers();
    if (!spec.layer_bandwidths.empty() && (int)spec.layer_bandwidths.size() != spec.k)
        throw std::invalid_argument("BCubeSpec: expected one bandwidth per layer");
    CapacitySystem sys;
    sys.n = n;
    sys.num_edges = n * (n - 1) / 2;
    sys.equality = false;
    sys.allowed.assign(sys.num_edges, 0);
    sys.rows.resize((size_t)spec.k * n);
    for (int layer = 0; layer < spec.k; ++layer)
        for (int u = 0; u < n; ++u) {
            auto& row = sys.rows[(size_t)layer * n + u];
            row.label = "layer" + std::to_string(layer) + "/server" + std::to_string(u);
            row.capacity = spec.p - 1;
        }
    int col = 0;
    for (int u = 0; u + 1 < n; ++u)
        for (int v = u + 1; v < n; ++v, ++col) {
            int diff_layer = -1, diffs = 0, du = u, dv = v;
            for (int layer = 0; layer < spec.k; ++layer) {
                if (du % spec.p != dv % spec.p) {
                    ++diffs;
                    diff_layer = layer;
                }
                du /= spec.p;
                dv /= spec.p;
            }
            if (diffs != 1) continue;
            sys.allowed[col] = 1;
            sys.rows[(size_t)diff_layer * n + u].edge_cols.push_back(col);
            sys.rows[(size_t)diff_layer * n + v].edge_cols.push_back(col);
        }
    return sys;
}

// ------------------------------------------------------------------ time model
// The reference's evaluation-side wall-clock model (proj/include/topoopt/
// bandwidth.hpp:85-128): per-edge bandwidth when every node / link splits its
// capacity over the edges mapped to it, the iteration/epoch times built on the
// bottleneck, and the scenario JSON. Outside the solver's hot path.
namespace {

std::vector<double> node_split(const Topology& t, const std::vector<double>& node_bw) {
    const auto deg = t.degrees();
    std::vector<double> out;
    out.reserve(t.edges.size());
    for (const auto& [i, j] : t.edges) out.push_back(std::min(node_bw[i] / deg[i], node_bw[j] / deg[j]));
    return out;
}

std::vector<double> resource_split(const Topology& t, const CapacitySystem& sys, const std::vector<double>& row_bw) {
    std::vector<char> sel(sys.num_edges, 0);
    for (const auto& [i, j] : t.edges) {
        const int c = edge_index(sys.n, i, j);
        if (!sys.allowed[c])
            throw std::invalid_argument("edge {" + std::to_string(i) + "," + std::to_string(j) +
                                        "} is not carried by any resource");
        sel[c] = 1;
    }
    const auto load = sys.loads(sel);
    std::vector<double> best(sys.num_edges, std::numeric_limits<double>::infinity());
    for (size_t k = 0; k < sys.rows.size(); ++k) {
        if (load[k] == 0) continue;
        const double share = row_bw[k] / load[k];
        for (int c : sys.rows[k].edge_cols) best[c] = std::min(best[c], share);
    }
    std::vector<double> out;
    out.reserve(t.edges.size());
    for (const auto& [i, j] : t.edges) out.push_back(best[edge_index(sys.n, i, j)]);
    return out;
}

struct EdgeBandwidth {
    const Topology& t;
    std::vector<double> operator()(const HomogeneousScenario& h) const {
        if (!(h.bandwidth > 0.0)) throw std::invalid_argument("homogeneous bandwidth must be positive");
        return node_split(t, std::vector<double>(t.n, h.bandwidth));
    }
    std::vector<double> operator()(const NodeScenario& ns) const {
        if ((int)ns.bandwidths.size() != t.n) throw std::invalid_argument("node bandwidth list size mismatch");
        for (double b : ns.bandwidths)
            if (!(b > 0.0)) throw std::invalid_argument("node bandwidths must be positive");
        return node_split(t, ns.bandwidths);
    }
    std::vector<double> operator()(const IntraScenario& is) const {
        const CapacitySystem sys = intra_server_constraints(is.tree);
        if (t.n != sys.n) throw std::invalid_argument("topology size mismatch with server");
        std::vector<double> bw;
        for (const auto& link : is.tree.links) bw.push_back(link.bandwidth);
        return resource_split(t, sys, bw);
    }
    std::vector<double> operator()(const BCubeScenario& bs) const {
        const CapacitySystem sys = bcube_constraints(bs.spec);
        if (t.n != sys.n) throw std::invalid_argument("topology size mismatch with bcube");
        std::vector<double> bw(sys.rows.size());
        for (int layer = 0; layer < bs.spec.k; ++layer) {
            const double b = bs.spec.layer_bandwidths.empty() ? kDefaultBandwidth : bs.spec.layer_bandwidths[layer];
            if (!(b > 0.0)) throw std::invalid_argument("layer bandwidths must be positive");
            std::fill(bw.begin() + (size_t)layer * sys.n, bw.begin() + (size_t)(layer + 1) * sys.n, b);
        }
        return resource_split(t, sys, bw);
    }
    std::vector<double> operator()(const FixedScenario&) const {
        throw std::invalid_argument("fixed-time scenario carries no bandwidth model");
    }
};

ServerTree tree_from_json(const json_lite::Value& j) {
    if (j.contains("preset")) {
        const std::string& preset = j.at("preset").as_string("preset");
        if (preset != "tiered8") throw std::invalid_argument("unknown server preset: " + preset);
        auto num = [&](const char* k, double dflt) { return j.contains(k) ? j.at(k).as_double(k) : dflt; };
        return tiered8_tree(num("leaf_bandwidth", kDefaultBandwidth / 2.0), num("group_bandwidth", kDefaultBandwidth / 2.0),
                            num("root_bandwidth", kDefaultBandwidth));
    }
    if (!j.contains("devices") || !j.contains("links") || !j.contains("routes"))
        throw std::invalid_argument("server tree config needs devices, links, routes");
    ServerTree tree;
    tree.n_devices = (int)j.at("devices").as_int("devices");
    std::map<std::string, int> index;
    for (const auto& lj : j.at("links").items) {
        ServerLink link{lj.at("name").as_string("name"), lj.at("bandwidth").as_double("bandwidth"),
                        (int)lj.at("capacity").as_int("capacity")};
        if (!index.emplace(link.name, (int)tree.links.size()).second)
            throw std::invalid_argument("duplicate link name: " + link.name);
        tree.links.push_back(link);
    }
    tree.routes.assign(tree.n_devices * (tree.n_devices - 1) / 2, {});
    for (const auto& rj : j.at("routes").items) {
        const auto& pair = rj.at("pair");
        if (!pair.is_array() || pair.items.size() != 2) throw std::invalid_argument("route pair must be [i, j]");
        const int col = edge_index(tree.n_devices, (int)pair.items[0].as_int("pair"), (int)pair.items[1].as_int("pair"));
        if (!tree.routes[col].empty()) throw std::invalid_argument("duplicate route for one device pair");
        for (const auto& name : rj.at("links").items) {
            auto it = index.find(name.as_string("link"));
            if (it == index.end()) throw std::invalid_argument("route references unknown link: " + name.text);
            tree.routes[col].push_back(it->second);
        }
    }
    tree.validate();
    return tree;
}

}  // namespace

std::vector<double> edge_bandwidths(const Topology& t, const Scenario& s) {
    t.validate();
    return std::visit(EdgeBandwidth{t}, s);
}

double min_edge_bandwidth(const Topology& t, const Scenario& s) {
    if (t.edges.empty()) throw std::invalid_argument("min_edge_bandwidth: topology has no edges");
    const auto bw = edge_bandwidths(t, s);
    return *std::min_element(bw.begin(), bw.end());
}

double iter_time(double b_avail, double b_min, double t_comm) {
    if (!(b_avail > 0.0) || !(b_min > 0.0) || !(t_comm > 0.0))
        throw std::invalid_argument("iter_time: arguments must be positive");
    return (b_avail / b_min) * t_comm;
}

double epoch_time(double b_avail, double b_min, double t_comm, double t_comp, int c_iter) {
    if (t_comp < 0.0) throw std::invalid_argument("epoch_time: negative compute time");
    if (c_iter < 1) throw std::invalid_argument("epoch_time: need at least one step per epoch");
    return (iter_time(b_avail, b_min, t_comm) + t_comp) * c_iter;
}

double iter_time(const TimeModel& m, double b_min) { return iter_time(m.b_avail, b_min, m.t_comm); }
double epoch_time(const TimeModel& m, double b_min) {
    return epoch_time(m.b_avail, b_min, m.t_comm, m.t_comp, m.c_iter);
}

Scenario scenario_from_json(const std::string& text) {
    const json_lite::Value j = json_lite::parse(text);
    if (!j.is_object() || !j.contains("mode")) throw std::invalid_argument("scenario config needs a mode");
    const std::string& mode = j.at("mode").as_string("mode");
    if (mode == "homogeneous")
        return HomogeneousScenario{j.contains("bandwidth") ? j.at("bandwidth").as_double("bandwidth") : kDefaultBandwidth};
    if (mode == "node") {
        if (!j.contains("bandwidths")) throw std::invalid_argument("node scenario needs bandwidths");
        return NodeScenario{j.at("bandwidths").as_doubles("bandwidths")};
    }
    if (mode == "intra") {
        if (!j.contains("tree")) throw std::invalid_argument("intra scenario needs a tree");
        return IntraScenario{tree_from_json(j.at("tree"))};
    }
    if (mode == "bcube") {
        BCubeSpec spec;
        spec.p = j.contains("p") ? (int)j.at("p").as_int("p") : 0;
        spec.k = j.contains("k") ? (int)j.at("k").as_int("k") : 0;
        if (j.contains("layer_bandwidths")) spec.layer_bandwidths = j.at("layer_bandwidths").as_doubles("layer_bandwidths");
        spec.n_servers();  // validates p, k
        return BCubeScenario{spec};
    }
    if (mode == "fixed") {
        if (!j.contains("t_iter_ms")) throw std::invalid_argument("fixed scenario needs t_iter_ms");
        FixedScenario f{j.at("t_iter_ms").as_double("t_iter_ms")};
        if (!(f.t_iter_ms > 0.0)) throw std::invalid_argument("t_iter_ms must be positive");
        return f;
    }
    throw std::invalid_argument("unknown scenario mode: " + mode);
}

std::vector<UtilizationRow> utilization(const CapacitySystem& sys, const Topology& t) {
    // proj/src/admm_het.cpp:371-392 (edges need not be sorted)
    if (t.n != sys.n) throw std::invalid_argument("utilization: node count mismatch");
    std::vector<char> sel(sys.num_edges, 0);
    for (const auto& [i, j] : t.edges) sel[edge_index(t.n, i, j)] = 1;
    const auto used = sys.loads(sel);
    std::vector<UtilizationRow> out;
    for (size_t k = 0; k < sys.rows.size(); ++k) out.push_back({sys.rows[k].label, sys.rows[k].capacity, used[k]});
    return out;
}

std::string utilization_csv(const std::vector<UtilizationRow>& rows) {
    std::string out = "resource,capacity,used\n";
    for (const auto& r : rows) out += r.label + "," + std::to_string(r.capacity) + "," + std::to_string(r.used) + "\n";
    return out;
}

// ------------------------------------------------------------------ admm
void SolverConfig::validate() const {
    const tp_config c = to_c(*this);
    raise(tp_config_validate(&c));
}

SolverConfig solver_config_from_json(const std::string& text) {
    // proj/src/admm.cpp:197-221: any subset of the fields, unknown keys and
    // non-objects rejected, then validate()
    const json_lite::Value j = json_lite::parse(text);
    if (!j.is_object()) throw std::invalid_argument("solver config must be a JSON object");
    SolverConfig cfg;
    for (const auto& [key, v] : j.members) {
        if (key == "rho") cfg.rho = v.as_double("rho");
        else if (key == "epsilon") cfg.epsilon = v.as_double("epsilon");
        else if (key == "max_iter") cfg.max_iter = (int)v.as_int("max_iter");
        else if (key == "alpha") cfg.alpha = v.as_double("alpha");
        else if (key == "weight_floor") cfg.weight_floor = v.as_double("weight_floor");
        else if (key == "seed") cfg.seed = v.as_u64("seed");
        else if (key == "linear_tol") cfg.linear_tol = v.as_double("linear_tol");
        else throw std::invalid_argument("solver config: unknown field " + key);
    }
    cfg.validate();
    return cfg;
}

std::string Solution::trace_csv() const {
    std::string out = "iter,residual,lambda_tilde,acf_iterate\n";
    char buf[128];
    for (const auto& row : trace) {
        std::snprintf(buf, sizeof buf, "%d,%.17g,%.17g,%.17g\n", row.iter, row.residual,
                      row.lambda_tilde, row.acf_iterate);
        out += buf;
    }
    return out;
}

ProblemData assemble(int n, int r, double alpha, double rho) {
    if (n < 2) throw std::invalid_argument("assemble: need at least 2 nodes");
    const int m = n * (n - 1) / 2;
    if (r < 1 || r > m) throw std::invalid_argument("assemble: r outside [1, n(n-1)/2]");
    if (!(alpha > 0.0)) throw std::invalid_argument("assemble: alpha must be positive");
    if (!(rho > 0.0)) throw std::invalid_argument("assemble: rho must be positive");
    ProblemData pd;
    pd.n = n;
    pd.m = m;
    pd.r = r;
    pd.alpha = alpha;
    pd.rho = rho;
    pd.lambda_ix = m;
    pd.off_s = m + 1;
    pd.off_y = pd.off_s + n * n;
    pd.off_t = pd.off_y + n;
    pd.nx = pd.off_t + n * n;
    pd.neq = 2 * n * n + n;
    pd.pairs = enumerate_edges(n);
    pd.beq.assign(n * n, -alpha / n);
    for (int c = 0; c < n; ++c)
        for (int rr = 0; rr < n; ++rr) pd.beq.push_back(rr == c ? 2.0 : 0.0);
    pd.beq.insert(pd.beq.end(), n, 1.0);
    pd.kkt = KktMatrix(pd.nx + pd.neq, [n] { return detail::build_kkt(n, 0, false, {}); });
    pd.ilu = KktIlu(pd.kkt);
    return pd;
}

Vec project_Y(const ProblemData& pd, const Vec& x, const Vec& d) {
    if ((int)x.size() != pd.nx || (int)d.size() != pd.nx)
        throw std::invalid_argument("project_Y: state length differs from nx");
    Vec y(pd.nx);
    raise(tp_project_Y(pd.n, pd.r, pd.alpha, pd.rho, x.data(), d.data(), y.data()));
    return y;
}

Vec update_X(const ProblemData& pd, const Vec& y, const Vec& d, Vec& kkt_warm, double) {
    if ((int)y.size() != pd.nx || (int)d.size() != pd.nx)
        throw std::invalid_argument("update_X: state length differs from nx");
    kkt_warm.resize(pd.nx + pd.neq);
    raise(tp_update_X(pd.n, pd.r, pd.alpha, pd.rho, y.data(), d.data(), kkt_warm.data()));
    return Vec(kkt_warm.begin(), kkt_warm.begin() + pd.nx);
}

Vec update_X_cg(const ProblemData& pd, const Vec& y, const Vec& d, Vec& kkt_warm, double linear_tol,
                int* cg_iters) {
    if ((int)y.size() != pd.nx || (int)d.size() != pd.nx)
        throw std::invalid_argument("update_X: state length differs from nx");
    kkt_warm.resize(pd.nx + pd.neq);
    int32_t it = 0;
    raise(tp_update_X_cg(pd.n, pd.r, pd.alpha, pd.rho, y.data(), d.data(), linear_tol, 8, kkt_warm.data(),
                         &it, nullptr));
    if (cg_iters) *cg_iters = it;
    return Vec(kkt_warm.begin(), kkt_warm.begin() + pd.nx);
}

void update_duals(const ProblemData& pd, const Vec& x, const Vec& y, Vec& d) {
    raise(tp_update_duals(pd.nx, pd.rho, x.data(), y.data(), d.data()));
}

Extraction extract_topology(int n, int r, const Vec& g, double weight_floor) {
    if (n < 2) throw std::invalid_argument("enumerate_edges: need at least two nodes");
    const int m = n * (n - 1) / 2;
    if ((int)g.size() < m) throw std::invalid_argument("extract_topology: weight vector shorter than |E|");
    const int cap = std::max(1, std::min(r, m));
    std::vector<int32_t> e(2 * cap);
    std::vector<double> w(cap);
    int32_t k = 0;
    raise(tp_extract_topology(n, r, g.data(), weight_floor, e.data(), w.data(), &k));
    Extraction ex;
    ex.topology = from_flat(n, e.data(), w.data(), k);
    ex.topology.validate();
    ex.w = gossip_matrix(ex.topology);
    return ex;
}

Topology default_warm_start(int n, int r, std::uint64_t seed) {
    std::vector<int32_t> e(2 * std::max(r, 1));
    int32_t k = 0;
    raise(tp_default_warm_start(n, r, seed, e.data(), &k));
    Topology t = from_flat(n, e.data(), nullptr, k);
    if (k > 0) {
        int dmax = 0;
        for (int d : t.degrees()) dmax = std::max(dmax, d);
        // annealed starts carry 1/(d_max+1); the chain fallback carries 1/3
        const bool chain = k == r && k < n - 1;
        t.weights.assign(k, chain ? 1.0 / 3.0 : 1.0 / (dmax + 1));
    }
    t.validate();
    return t;
}

Solution solve(int n, int r, const SolverConfig& cfg, const std::optional<Topology>& warm) {
    const auto t0 = std::chrono::steady_clock::now();
    cfg.validate();
    const tp_config c = to_c(cfg);
    tp_result res{};
    const int cap = std::max(1, r);
    std::vector<int32_t> edges(2 * cap);
    std::vector<double> weights(cap), trace(3 * (size_t)cfg.max_iter);
    char note[512] = {0};
    if (warm) {
        warm->validate();
        if (warm->n != n) throw std::invalid_argument("solve: warm start node count mismatch");
        const auto we = flat_edges(*warm);
        raise(tp_solve(n, r, &c, we.data(), (int32_t)warm->edges.size(), &res, edges.data(),
                       weights.data(), trace.data(), note, sizeof note));
    } else {
        raise(tp_solve(n, r, &c, nullptr, -1, &res, edges.data(), weights.data(), trace.data(), note,
                       sizeof note));
    }
    Solution sol = collect(n, res, edges, weights, trace, note);
    sol.wall_time_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

// ------------------------------------------------------------------ admm_het
ProblemDataHet assemble_het(const CapacitySystem& sys, std::optional<int> r, double alpha, double rho) {
    // proj/src/admm_het.cpp:20-114: node-level (equality) systems carry their
    // degree rows in the KKT and imply r; capacity-bound systems need r in
    // [1, |E|] and keep their rows out of the equality block (q = 0)
    if (sys.n < 2) throw std::invalid_argument("assemble_het: need at least 2 nodes");
    if (sys.num_edges != sys.n * (sys.n - 1) / 2 || (int)sys.allowed.size() != sys.num_edges)
        throw std::invalid_argument("assemble_het: capacity system columns differ from the pair set");
    for (const auto& row : sys.rows)
        for (int c : row.edge_cols)
            if (c < 0 || c >= sys.num_edges)
                throw std::invalid_argument("assemble_het: a row references a column outside [0, |E|)");
    if (!(alpha > 0.0)) throw std::invalid_argument("assemble_het: alpha must be positive");
    if (!(rho > 0.0)) throw std::invalid_argument("assemble_het: rho must be positive");
    int total = 0, q = 0;
    std::vector<std::vector<int>> degree_rows;
    if (sys.equality) {
        const int implied = sys.implied_edge_total();
        if (r && *r != implied) throw std::invalid_argument("edge total conflicts with the degree rows");
        total = implied;
        q = (int)sys.rows.size();
        for (const auto& row : sys.rows) degree_rows.push_back(row.edge_cols);
    } else {
        if (!r) throw std::invalid_argument("capacity-bound system needs an explicit edge total");
        total = *r;
    }
    const int m = sys.num_edges;
    if (total < 1 || total > m) throw std::invalid_argument("assemble_het: edge total outside [1, |E|]");
    const ProblemData base = assemble(sys.n, total, alpha, rho);
    ProblemDataHet pd;
    pd.n = base.n;
    pd.m = base.m;
    pd.r = total;
    pd.alpha = alpha;
    pd.rho = rho;
    pd.q = q;
    pd.lambda_ix = base.lambda_ix;
    pd.off_s = base.off_s;
    pd.off_y = base.off_y;
    pd.off_t = base.off_t;
    pd.off_z = base.nx;
    pd.off_nu = base.nx + m;
    pd.nx = base.nx + 2 * m;
    pd.neq = base.neq + q + m;
    pd.pairs = base.pairs;
    pd.sys = sys;
    pd.beq = base.beq;
    for (int k = 0; k < q; ++k) pd.beq.push_back((double)sys.rows[k].capacity);
    pd.beq.insert(pd.beq.end(), m, 0.0);
    const int n = sys.n;
    pd.kkt = KktMatrix(pd.nx + pd.neq, [n, q, degree_rows] { return detail::build_kkt(n, q, true, degree_rows); });
    pd.ilu = KktIlu(pd.kkt);
    return pd;
}

Vec project_binary_z(const Vec& v, int r) {
    Vec z(v.size());
    raise(tp_project_binary_z(v.data(), (int64_t)v.size(), r, z.data()));
    return z;
}

Vec project_binary_z_capped(const Vec& v, int r, const CapacitySystem& sys) {
    // proj/src/admm_het.cpp:125-154 on the device (select_kernels.cu::capped_z_kernel)
    if ((int)v.size() != sys.num_edges)
        throw std::invalid_argument("project_binary_z_capped: score length differs from |E|");
    const FlatRows f = flat_rows(sys);
    Vec z(v.size());
    raise(tp_project_binary_z_capped(sys.n, (int32_t)sys.rows.size(), f.row_ptr.data(), f.cols.data(),
                                     f.caps.data(), f.allowed.data(), v.data(), r, z.data()));
    return z;
}

Vec project_Y_het(const ProblemDataHet& pd, const Vec& x, const Vec& d) {
    if ((int)x.size() != pd.nx || (int)d.size() != pd.nx)
        throw std::invalid_argument("project_Y_het: state length differs from nx");
    Vec y(pd.nx);
    std::vector<int32_t> deg;
    if (pd.sys.equality && node_level_degrees(pd.sys, deg)) {
        raise(tp_project_Y_het_node(pd.n, deg.data(), pd.alpha, pd.rho, x.data(), d.data(), y.data()));
        return y;
    }
    if (pd.sys.equality)
        throw std::invalid_argument("project_Y_het: equality systems must be one degree row per node");
    const FlatRows f = flat_rows(pd.sys);
    raise(tp_project_Y_het_capacity(pd.n, (int32_t)pd.sys.rows.size(), f.row_ptr.data(), f.cols.data(),
                                    f.caps.data(), f.allowed.data(), pd.r, pd.alpha, pd.rho, x.data(), d.data(),
                                    y.data()));
    return y;
}

Solution solve_het(const CapacitySystem& sys, std::optional<int> r, const SolverConfig& cfg,
                   const std::optional<Topology>& warm) {
    const auto t0 = std::chrono::steady_clock::now();
    cfg.validate();
    if (!sys.equality) {
        // capacity-bound rows (proj/src/admm_het.cpp:37-48: explicit edge total)
        if (!r) throw std::invalid_argument("capacity-bound system needs an explicit edge total");
        const FlatRows f = flat_rows(sys);
        const tp_config c = to_c(cfg);
        tp_result res{};
        const int m = sys.n * (sys.n - 1) / 2;
        std::vector<int32_t> edges(2 * std::max(m, 1));
        std::vector<double> weights(std::max(m, 1)), trace(3 * (size_t)cfg.max_iter);
        char note[512] = {0};
        std::vector<int32_t> we;
        if (warm) {
            warm->validate();
            if (warm->n != sys.n) throw std::invalid_argument("solve_het: warm start node count mismatch");
            we = flat_edges(*warm);
        }
        raise(tp_solve_het_capacity(sys.n, (int32_t)sys.rows.size(), f.row_ptr.data(), f.cols.data(), f.caps.data(),
                                    f.allowed.data(), *r, &c, warm ? we.data() : nullptr,
                                    warm ? (int32_t)warm->edges.size() : -1, &res, edges.data(), weights.data(),
                                    trace.data(), note, sizeof note));
        Solution sol = collect(sys.n, res, edges, weights, trace, note);
        sol.wall_time_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return sol;
    }
    std::vector<int32_t> deg;
    if (!node_level_degrees(sys, deg))
        throw std::invalid_argument("assemble_het: equality system must be one row per node");
    long long total = 0;
    for (int d : deg) total += d;
    if (total % 2 == 0 && r && *r != total / 2)
        throw std::invalid_argument("edge total conflicts with the degree rows");
    const tp_config c = to_c(cfg);
    tp_result res{};
    const int m = sys.n * (sys.n - 1) / 2;
    std::vector<int32_t> edges(2 * std::max(m, 1));
    std::vector<double> weights(std::max(m, 1)), trace(3 * (size_t)cfg.max_iter);
    char note[512] = {0};
    if (warm) {
        warm->validate();
        if (warm->n != sys.n) throw std::invalid_argument("solve_het: warm start node count mismatch");
        const auto we = flat_edges(*warm);
        raise(tp_solve_het_node(sys.n, deg.data(), &c, we.data(), (int32_t)warm->edges.size(), &res,
                                edges.data(), weights.data(), trace.data(), note, sizeof note));
    } else {
        raise(tp_solve_het_node(sys.n, deg.data(), &c, nullptr, -1, &res, edges.data(), weights.data(),
                                trace.data(), note, sizeof note));
    }
    Solution sol = collect(sys.n, res, edges, weights, trace, note);
    sol.wall_time_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

}  // namespace topoopt
