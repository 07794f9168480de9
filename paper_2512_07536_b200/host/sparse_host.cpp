// The reference's L1 sparse utilities for API completeness
// (proj/include/topoopt/sparse.hpp, solvers.hpp): a CSC container, ILU(0)
// and preconditioned BiCGSTAB, plus the lazily assembled KKT matrix of
// ProblemData / ProblemDataHet (proj/src/admm.cpp:46-94, admm_het.cpp:58-114).
// None of this is on the solver's path: the GPU x-step is matrix-free
// (DESIGN.md §3.3). Textbook algorithms, host C++.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <istream>
#include <mutex>
#include <numeric>
#include <ostream>
#include <sstream>

#include "topoopt/topoopt_b200.hpp"

namespace topoopt {

// ------------------------------------------------------------------ CSC
SparseMatrix SparseMatrix::from_triplets(int rows, int cols, const std::vector<Triplet>& entries) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("SparseMatrix: negative dimensions");
    for (const Triplet& t : entries)
        if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols)
            throw std::invalid_argument("SparseMatrix: triplet index out of range");
    // bucket by column, then sort each column by row and merge duplicates
    std::vector<int> count(cols + 1, 0);
    for (const Triplet& t : entries) ++count[t.col + 1];
    for (int c = 0; c < cols; ++c) count[c + 1] += count[c];
    std::vector<std::pair<int, double>> bucket(entries.size());
    std::vector<int> fill(count.begin(), count.end() - 1);
    for (const Triplet& t : entries) bucket[fill[t.col]++] = {t.row, t.value};
    SparseMatrix a;
    a.rows_ = rows;
    a.cols_ = cols;
    a.col_ptr_.assign(cols + 1, 0);
    a.row_idx_.reserve(entries.size());
    a.val_.reserve(entries.size());
    for (int c = 0; c < cols; ++c) {
        auto b = bucket.begin() + count[c], e = bucket.begin() + count[c + 1];
        std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
        for (auto it = b; it != e; ++it) {
            if (!a.row_idx_.empty() && (int)a.row_idx_.size() > a.col_ptr_[c] && a.row_idx_.back() == it->first)
                a.val_.back() += it->second;  // duplicate: sum (explicit zeros stay)
            else {
                a.row_idx_.push_back(it->first);
                a.val_.push_back(it->second);
            }
        }
        a.col_ptr_[c + 1] = (int)a.row_idx_.size();
    }
    return a;
}

void SparseMatrix::multiply(const Vec& x, Vec& y) const {
    if ((int)x.size() != cols_) throw std::invalid_argument("SparseMatrix::multiply: size mismatch");
    y.assign(rows_, 0.0);
    for (int c = 0; c < cols_; ++c) {
        const double xc = x[c];
        for (int k = col_ptr_[c]; k < col_ptr_[c + 1]; ++k) y[row_idx_[k]] += val_[k] * xc;
    }
}

Vec SparseMatrix::multiply(const Vec& x) const {
    Vec y;
    multiply(x, y);
    return y;
}

Matrix SparseMatrix::to_dense() const {
    Matrix d(rows_, cols_);
    for (int c = 0; c < cols_; ++c)
        for (int k = col_ptr_[c]; k < col_ptr_[c + 1]; ++k) d(row_idx_[k], c) += val_[k];
    return d;
}

void SparseMatrix::save(std::ostream& out) const {
    out << rows_ << ' ' << cols_ << ' ' << nnz() << '\n';
    for (int c = 0; c < cols_; ++c)
        for (int k = col_ptr_[c]; k < col_ptr_[c + 1]; ++k)
            out << row_idx_[k] << ' ' << c << ' ' << g17(val_[k]) << '\n';
}

SparseMatrix SparseMatrix::load(std::istream& in) {
    int rows = 0, cols = 0, nnz = 0;
    if (!(in >> rows >> cols >> nnz) || nnz < 0)
        throw std::invalid_argument("SparseMatrix::load: malformed header");
    std::vector<Triplet> t(nnz);
    for (Triplet& e : t) {
        std::string v;
        if (!(in >> e.row >> e.col >> v)) throw std::invalid_argument("SparseMatrix::load: truncated entries");
        e.value = std::strtod(v.c_str(), nullptr);
    }
    return from_triplets(rows, cols, t);
}

// ------------------------------------------------------------------ ILU(0)
IluFactors ilu0(const SparseMatrix& a) {
    if (a.rows() != a.cols()) throw std::invalid_argument("ilu0: matrix must be square");
    const int n = a.rows();
    IluFactors f;
    f.n = n;
    // CSR view with sorted column indices
    f.row_ptr.assign(n + 1, 0);
    for (int r : a.row_idx()) ++f.row_ptr[r + 1];
    for (int i = 0; i < n; ++i) f.row_ptr[i + 1] += f.row_ptr[i];
    f.col_idx.resize(a.nnz());
    f.val.resize(a.nnz());
    std::vector<int> fill(f.row_ptr.begin(), f.row_ptr.end() - 1);
    for (int c = 0; c < n; ++c)
        for (int k = a.col_ptr()[c]; k < a.col_ptr()[c + 1]; ++k) {
            const int p = fill[a.row_idx()[k]]++;
            f.col_idx[p] = c;  // columns arrive in increasing order
            f.val[p] = a.values()[k];
        }
    f.diag_pos.assign(n, -1);
    for (int i = 0; i < n; ++i)
        for (int p = f.row_ptr[i]; p < f.row_ptr[i + 1]; ++p)
            if (f.col_idx[p] == i) f.diag_pos[i] = p;
    // IKJ elimination restricted to the pattern
    std::vector<int> where(n, -1);
    for (int i = 0; i < n; ++i) {
        if (f.diag_pos[i] < 0) throw PivotError("ilu0: structurally zero pivot in row " + std::to_string(i), i);
        for (int p = f.row_ptr[i]; p < f.row_ptr[i + 1]; ++p) where[f.col_idx[p]] = p;
        for (int p = f.row_ptr[i]; p < f.row_ptr[i + 1] && f.col_idx[p] < i; ++p) {
            const int k = f.col_idx[p];
            const double piv = f.val[f.diag_pos[k]];
            const double l = f.val[p] / piv;
            f.val[p] = l;
            for (int q = f.diag_pos[k] + 1; q < f.row_ptr[k + 1]; ++q) {
                const int w = where[f.col_idx[q]];
                if (w >= 0) f.val[w] -= l * f.val[q];
            }
        }
        for (int p = f.row_ptr[i]; p < f.row_ptr[i + 1]; ++p) where[f.col_idx[p]] = -1;
        const double d = f.val[f.diag_pos[i]];
        if (!(std::abs(d) > 1e-300) || !std::isfinite(d))
            throw PivotError("ilu0: zero pivot in row " + std::to_string(i), i);
    }
    return f;
}

void IluFactors::apply(const Vec& r, Vec& z) const {
    if ((int)r.size() != n) throw std::invalid_argument("IluFactors::apply: size mismatch");
    z = r;
    for (int i = 0; i < n; ++i)  // unit lower
        for (int p = row_ptr[i]; p < diag_pos[i]; ++p) z[i] -= val[p] * z[col_idx[p]];
    for (int i = n - 1; i >= 0; --i) {  // upper
        for (int p = diag_pos[i] + 1; p < row_ptr[i + 1]; ++p) z[i] -= val[p] * z[col_idx[p]];
        z[i] /= val[diag_pos[i]];
    }
}

// ------------------------------------------------------------------ BiCGSTAB
SolveReport bicgstab(const SparseMatrix& a, const Vec& b, Vec& x, const IluFactors* precond, double tol,
                     int max_iter) {
    const int n = a.rows();
    if (a.cols() != n || (int)b.size() != n) throw std::invalid_argument("bicgstab: dimension mismatch");
    if (max_iter < 0) max_iter = 10 * n;
    if ((int)x.size() != n) x.assign(n, 0.0);
    SolveReport rep;
    const double bnorm = norm2(b);
    if (bnorm == 0.0) {
        x.assign(n, 0.0);
        rep.converged = true;
        return rep;
    }
    const double target = tol * bnorm;
    auto prec = [&](const Vec& in, Vec& out) {
        if (precond) precond->apply(in, out);
        else out = in;
    };
    auto true_residual = [&](Vec& r) {
        a.multiply(x, r);
        for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
        return norm2(r);
    };
    Vec r(n), rhat, p(n, 0.0), v(n, 0.0), ph(n), s(n), sh(n), t(n);
    double res = true_residual(r);
    if (res <= target) {
        rep.converged = true;
        rep.residual = res;
        return rep;
    }
    int restarts = 0;
    auto reset = [&] {
        rhat = r;
        std::fill(p.begin(), p.end(), 0.0);
        std::fill(v.begin(), v.end(), 0.0);
    };
    reset();
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    while (rep.iterations < max_iter) {
        const double rho_new = dot(rhat, r);
        if (rho_new == 0.0 || !std::isfinite(rho_new) || omega == 0.0) {
            if (restarts++ >= 1) {
                rep.note = "BiCGSTAB breakdown after a restart";
                break;
            }
            res = true_residual(r);
            reset();
            rho = alpha = omega = 1.0;
            continue;
        }
        ++rep.iterations;
        const double beta = (rho_new / rho) * (alpha / omega);
        rho = rho_new;
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        prec(p, ph);
        a.multiply(ph, v);
        const double rv = dot(rhat, v);
        if (rv == 0.0 || !std::isfinite(rv)) {
            omega = 0.0;  // breakdown: restart on the next pass
            continue;
        }
        alpha = rho / rv;
        for (int i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
        if (norm2(s) <= target) {
            axpy(alpha, ph, x);
            res = true_residual(r);
            if (res <= target) {
                rep.converged = true;
                break;
            }
            reset();  // recursive residual drifted: continue from the true one
            rho = alpha = omega = 1.0;
            continue;
        }
        prec(s, sh);
        a.multiply(sh, t);
        const double tt = dot(t, t);
        omega = tt > 0.0 ? dot(t, s) / tt : 0.0;
        for (int i = 0; i < n; ++i) x[i] += alpha * ph[i] + omega * sh[i];
        for (int i = 0; i < n; ++i) r[i] = s[i] - omega * t[i];
        if (norm2(r) <= target) {
            res = true_residual(r);
            if (res <= target) {
                rep.converged = true;
                break;
            }
            reset();
            rho = alpha = omega = 1.0;
        }
    }
    rep.residual = true_residual(r);
    if (!rep.converged && rep.note.empty()) rep.note = "BiCGSTAB reached max_iter";
    return rep;
}

// ------------------------------------------------------------------ KKT
struct KktMatrix::State {
    std::once_flag once;
    std::function<SparseMatrix()> build;
    SparseMatrix m;
};

KktMatrix::KktMatrix(int dim, std::function<SparseMatrix()> build) : dim_(dim), st_(std::make_shared<State>()) {
    st_->build = std::move(build);
}

const SparseMatrix& KktMatrix::matrix() const {
    if (!st_) throw std::invalid_argument("KktMatrix: empty (no problem assembled)");
    std::call_once(st_->once, [this] {
        st_->m = st_->build();
        st_->build = nullptr;
    });
    return st_->m;
}

struct KktIlu::State {
    std::once_flag once;
    KktMatrix kkt;
    IluFactors f;
};

KktIlu::KktIlu(KktMatrix kkt) : st_(std::make_shared<State>()) { st_->kkt = std::move(kkt); }

const IluFactors& KktIlu::factors() const {
    if (!st_) throw std::invalid_argument("KktIlu: empty (no problem assembled)");
    std::call_once(st_->once, [this] { st_->f = ilu0(st_->kkt.matrix()); });
    return st_->f;
}

namespace detail {

// Equality rows A x = beq of the homogeneous blocks (rows [B- | B+ | D]):
//   L(g) - lam I + S = -alpha/n J,   L(g) + lam I + T = 2 I,   diag L(g) + y = 1
// with S, T column-major (row c n + r <-> entry (r, c)), plus for het systems
// q degree rows over z and m coupling rows g - z + nu = 0. Returns the
// triplets of [[I, A^T], [A, -1e-8 I]] (proj/src/admm.cpp:46-94,
// proj/src/admm_het.cpp:58-114; kKktShift, admm_shared.hpp:16).
SparseMatrix build_kkt(int n, int q, bool het, const std::vector<std::vector<int>>& degree_rows) {
    const int m = n * (n - 1) / 2, n2 = n * n;
    const int lambda_ix = m, off_s = m + 1, off_y = off_s + n2, off_t = off_y + n;
    const int nx_hom = off_t + n2, off_z = nx_hom, off_nu = off_z + m;
    const int nx = het ? nx_hom + 2 * m : nx_hom;
    const int neq = 2 * n2 + n + (het ? q + m : 0);
    std::vector<Triplet> A;  // (row, col, value) of the equality block
    A.reserve((size_t)m * 10 + 2 * n2 + 4 * n);
    int l = 0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j, ++l) {
            for (int blk = 0; blk < 2; ++blk) {
                const int ro = blk * n2;
                A.push_back({ro + i * n + i, l, 1.0});
                A.push_back({ro + j * n + j, l, 1.0});
                A.push_back({ro + j * n + i, l, -1.0});
                A.push_back({ro + i * n + j, l, -1.0});
            }
            A.push_back({2 * n2 + i, l, 1.0});
            A.push_back({2 * n2 + j, l, 1.0});
        }
    for (int i = 0; i < n; ++i) {
        A.push_back({i * n + i, lambda_ix, -1.0});
        A.push_back({n2 + i * n + i, lambda_ix, 1.0});
    }
    for (int k = 0; k < n2; ++k) {
        A.push_back({k, off_s + k, 1.0});
        A.push_back({n2 + k, off_t + k, 1.0});
    }
    for (int i = 0; i < n; ++i) A.push_back({2 * n2 + i, off_y + i, 1.0});
    if (het) {
        const int hom_rows = 2 * n2 + n;
        for (int rr = 0; rr < q; ++rr)
            for (int col : degree_rows[rr]) A.push_back({hom_rows + rr, off_z + col, 1.0});
        for (int e = 0; e < m; ++e) {
            const int row = hom_rows + q + e;
            A.push_back({row, e, 1.0});
            A.push_back({row, off_z + e, -1.0});
            A.push_back({row, off_nu + e, 1.0});
        }
    }
    std::vector<Triplet> K;
    K.reserve(2 * A.size() + nx + neq);
    for (int k = 0; k < nx; ++k) K.push_back({k, k, 1.0});
    for (const Triplet& t : A) {
        K.push_back({nx + t.row, t.col, t.value});  // A
        K.push_back({t.col, nx + t.row, t.value});  // A^T
    }
    for (int k = 0; k < neq; ++k) K.push_back({nx + k, nx + k, -1e-8});
    return SparseMatrix::from_triplets(nx + neq, nx + neq, K);
}

}  // namespace detail
}  // namespace topoopt
