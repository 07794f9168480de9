// C ABI substep entry points: each reference substep run once on the device
// with caller-owned host buffers (used by the parity tests and by callers that
// drive their own loop, e.g. proj/tests/test_admm.cpp's substep checks).
#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/topoopt_b200.h"
#include "eig_kernels.cuh"
#include "ozaki_kernels.cuh"
#include "solver.cuh"

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
    } catch (const std::exception& e) {
        last_error_ref() = e.what();
        return TP_ERR_INTERNAL;
    }
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DBuf(size_t count) : n(count) {
        TPB_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf&) = delete;
    void up(const T* h, size_t count) {
        h2d(p, h, count * sizeof(T));
    }
    void down(T* h, size_t count) const {
        TPB_CUDA(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost));
    }
    void zero() { TPB_CUDA(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T))); }
};

void require_device() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw Error(kCuda, "no CUDA device: the B200 solver has no CPU fallback");
}

Config sub_cfg(double alpha, double rho) {
    Config c;
    c.alpha = alpha;
    c.rho = rho;
    c.max_iter = 1;
    if (!(alpha > 0.0)) throw Error(kInvalidArgument, "assemble: alpha must be positive");
    if (!(rho > 0.0)) throw Error(kInvalidArgument, "assemble: rho must be positive");
    return c;
}

// mu = [r_S - S ; r_T - T ; r_y - y ; mu_d ; r_nu - nu] (the KKT multipliers)
__global__ void kkt_mu_kernel(Layout lo, const double* X, const double* Y, const double* D,
                              const double* node, double rho, double* mu) {
    const long long n2 = (long long)lo.n * lo.n;
    const long long st = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < lo.neq; k += st) {
        long long src;
        if (k < n2) src = lo.off_s + k;
        else if (k < 2 * n2) src = lo.off_t + (k - n2);
        else if (k < 2 * n2 + lo.n) src = lo.off_y + (k - 2 * n2);
        else if (k < 2 * n2 + lo.n + lo.q) {
            mu[k] = node[2 * lo.n + (k - 2 * n2 - lo.n)];
            continue;
        } else src = lo.off_nu + (k - 2 * n2 - lo.n - lo.q);
        mu[k] = (Y[src] - D[src] / rho) - X[src];
    }
}

__global__ void duals_kernel(long long nx, double rho, const double* x, const double* y, double* d) {
    const long long st = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nx; k += st)
        d[k] += rho * (x[k] - y[k]);
}

// A (ld-padded, slot w of a pair) = (a + a^T)/2 ; scale = 1/||A||_F
__global__ void sym_pad_kernel(const double* a, int n, int ld, int w, double* A) {
    const long long nn = (long long)n * n;
    const long long st = (long long)gridDim.x * blockDim.x;
    double* dst = A + (long long)w * ld * ld;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nn; p += st) {
        const int r = (int)(p / n), c = (int)(p % n);
        dst[(long long)r * ld + c] = 0.5 * (a[(long long)r * n + c] + a[(long long)c * n + r]);
    }
}

// 1 / min(||A||_F, ||A||_inf) of matrix w (as the solver's prep tail)
__global__ void frob_kernel(const double* A, int ld, int w, double* scale) {
    __shared__ double scratch[32];
    const double* src = A + (long long)w * ld * ld;
    double s = 0.0, inf = 0.0;
    for (long long p = threadIdx.x; p < (long long)ld * ld; p += blockDim.x) s += src[p] * src[p];
    for (int r = threadIdx.x; r < ld; r += blockDim.x) {
        double rs = 0.0;
        for (int c = 0; c < ld; ++c) rs += fabs(src[(long long)r * ld + c]);
        inf = fmax(inf, rs);
    }
    s = block_sum(s, scratch);
    inf = block_max(inf, scratch);
    if (threadIdx.x == 0) {
        scale[0] = 0.0;
        scale[1] = 0.0;
        const double c = fmin(sqrt(s), inf);
        scale[w] = c > 0.0 ? 1.0 / c : 0.0;
    }
}

// dense W checks: max |W - W^T|, max |row sum - 1|
__global__ void dense_check_kernel(const double* W, int n, double* out2) {
    __shared__ double scratch[32];
    double asym = 0.0, dev = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double rs = 0.0;
        for (int c = 0; c < n; ++c) {
            asym = fmax(asym, fabs(W[(long long)r * n + c] - W[(long long)c * n + r]));
            rs += W[(long long)r * n + c];
        }
        dev = fmax(dev, fabs(rs - 1.0));
    }
    asym = block_max(asym, scratch);
    dev = block_max(dev, scratch);
    if (threadIdx.x == 0) {
        out2[0] = asym;
        out2[1] = dev;
    }
}

__global__ void sym_copy_kernel(const double* W, int n, double* S) {
    const long long nn = (long long)n * n;
    const long long st = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nn; p += st) {
        const int r = (int)(p / n), c = (int)(p % n);
        S[p] = 0.5 * (W[p] + W[(long long)c * n + r]);  // sym_eig symmetrizes (eig.cpp:157)
    }
}

void cone_dense(int n, const double* a, double* out, bool psd) {
    require_device();
    if (n < 1) throw Error(kInvalidArgument, "project: empty matrix");
    init_attrs();
    const bool small = n <= 64;
    const int ld = small ? ((n + 7) & ~7) : ((n + 127) / 128) * 128;
    if (!small) check_oz_ld(ld);
    const long long ld2 = (long long)ld * ld;
    const int w = psd ? 1 : 0;  // slot 0 -> NSD, slot 1 -> PSD
    DBuf<double> da((size_t)n * n), A(2 * ld2), C(2 * (size_t)n * n), scale(2);
    da.up(a, (size_t)n * n);
    A.zero();
    C.zero();
    const int blocks = (int)std::min<long long>(((long long)n * n + 255) / 256, 1024);
    sym_pad_kernel<<<blocks, 256>>>(da.p, n, ld, w, A.p);
    TPB_CHECK_LAUNCH();
    if (small) {
        launch_cone_small(A.p, ld2, ld, n, C.p, 0, (long long)n * n, nullptr, 2, SignSchedule{}, 0);
    } else {
        frob_kernel<<<1, 1024>>>(A.p, ld, w, scale.p);
        TPB_CHECK_LAUNCH();
        OzWork oz_w;
        std::vector<std::unique_ptr<DBuf<int8_t>>> bufs;
        for (int q = 0; q < 4; ++q) {
            bufs.emplace_back(new DBuf<int8_t>((size_t)2 * kOzSlices * ld2));
            bufs.back()->zero();
            oz_w.d[q] = bufs.back()->p;
            make_oz_maps(oz_w.d[q], ld, 2, &oz_w.maps[q]);
        }
        enqueue_cone_ozaki(A.p, oz_w, ld, n, scale.p, C.p, 0, (long long)n * n, nullptr, 2, ozaki_schedule(), 0);
    }
    TPB_CUDA(cudaDeviceSynchronize());
    // column-major output of a symmetric matrix == row-major
    TPB_CUDA(cudaMemcpy(out, C.p + (size_t)w * n * n, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost));
}

void slem_edges(int n, const std::vector<int>& packed, const std::vector<double>& wts, double* out4) {
    const long long m = (long long)n * (n - 1) / 2;
    const int k = (int)packed.size();
    init_attrs();
    const bool exact = n - 1 <= kFinalExactDim;
    const int kfin = exact ? std::max(1, n - 1) : slem_oneoff_kmax(n);
    DBuf<double> g(m), out(8), basis((size_t)kfin * n), ew(std::max(1, k));
    DBuf<int> list(std::max(1, k)), count(1), ei(std::max(1, k)), ej(std::max(1, k)), ci(std::max(1, k));
    g.zero();
    std::vector<double> packedw(m, 0.0);
    for (int e = 0; e < k; ++e) packedw[packed[e]] = wts[e];
    g.up(packedw.data(), m);
    if (k) list.up(packed.data(), k);
    count.up(&k, 1);
    SlemArgs a{};
    a.n = n;
    a.m = m;
    a.g = g.p;
    a.stride = m;
    a.list = list.p;
    a.count = count.p;
    a.list_cap = std::max(1, k);
    a.e_i = ei.p;
    a.e_j = ej.p;
    a.e_w = ew.p;
    a.col_idx = ci.p;
    a.basis = basis.p;
    a.kmax = kfin;
    a.plain = exact ? 0 : 1;  // as the solver's one-off reports (Solver::final_slem)
    a.cluster = kOneOffCluster;
    a.max_restarts = 200;
    // first residual check: the plain recurrence at n ~ 1000 needs ~380
    // steps to 1e-10, so a check at 128 is wasted (a check at k costs ~k us)
    a.min_steps = std::min(std::max(64, n / 4), 256);
    a.check_every = 128;
    a.tol = 1e-10;
    a.out = out.p;
    launch_slem(a, 1, 0);
    TPB_CUDA(cudaDeviceSynchronize());
    double o[8];
    out.down(o, 8);
    std::copy(o, o + 4, out4);
}

}  // namespace

extern "C" {

int tp_project_Y(int32_t n, int32_t r, double alpha, double rho, const double* x, const double* d,
                 double* y) {
    return guarded([&] {
        require_device();
        Solver s(n, 1, false, {r}, {}, sub_cfg(alpha, rho));
        s.upload(x, nullptr, d);
        s.project_only();
        s.download(nullptr, y, nullptr);
    });
}

int tp_sym_eig(int32_t n, const double* a, double* values, double* vectors) {
    return guarded([&] {
        require_device();
        sym_eig_device(n, a, values, vectors);
    });
}

int tp_project_Y_het_node(int32_t n, const int32_t* degrees, double alpha, double rho,
                          const double* x, const double* d, double* y) {
    return guarded([&] {
        require_device();
        Solver s(n, 1, true, {}, std::vector<int>(degrees, degrees + n), sub_cfg(alpha, rho));
        s.upload(x, nullptr, d);
        s.project_only();
        s.download(nullptr, y, nullptr);
    });
}

static void update_x_common(Solver& s, double rho, const double* y, const double* d, double* kkt_out) {
    s.upload(nullptr, y, d);
    s.xstep_only(false);
    const Layout& lo = s.layout();
    DBuf<double> mu(lo.neq);
    Dev& dv = s.dev();
    kkt_mu_kernel<<<256, 256, 0, s.stream()>>>(lo, dv.X, dv.Y, dv.D, dv.node, rho, mu.p);
    TPB_CHECK_LAUNCH();
    TPB_CUDA(cudaStreamSynchronize(s.stream()));
    s.download(kkt_out, nullptr, nullptr);
    mu.down(kkt_out + lo.nx, lo.neq);
}

int tp_update_X(int32_t n, int32_t r, double alpha, double rho, const double* y, const double* d,
                double* kkt_out) {
    return guarded([&] {
        require_device();
        Solver s(n, 1, false, {r}, {}, sub_cfg(alpha, rho));
        update_x_common(s, rho, y, d, kkt_out);
    });
}

int tp_update_X_cg(int32_t n, int32_t r, double alpha, double rho, const double* y, const double* d,
                   double linear_tol, int32_t cg_max_iter, double* kkt_out, int32_t* cg_iters,
                   double* cg_rel_res) {
    return guarded([&] {
        require_device();
        Config c = sub_cfg(alpha, rho);
        c.linear_solver = 1;
        c.linear_tol = linear_tol;
        c.cg_max_iter = cg_max_iter;
        validate(c);
        Solver s(n, 1, false, {r}, {}, c);
        update_x_common(s, rho, y, d, kkt_out);
        int it = 0;
        double rr = 0.0;
        s.cg_stats(0, &it, &rr);
        if (cg_iters) *cg_iters = it;
        if (cg_rel_res) *cg_rel_res = rr;
        // the reference's guard after BiCGSTAB (proj/src/admm.cpp:287)
        if (!(rr <= 1e-8))
            throw Error(kLinearSolve, "update_X: CG relative residual " + std::to_string(rr) +
                                          " after " + std::to_string(it) + " iterations");
    });
}

int tp_update_X_het_node(int32_t n, const int32_t* degrees, double alpha, double rho,
                         const double* y, const double* d, double* kkt_out) {
    return guarded([&] {
        require_device();
        Solver s(n, 1, true, {}, std::vector<int>(degrees, degrees + n), sub_cfg(alpha, rho));
        update_x_common(s, rho, y, d, kkt_out);
    });
}

int tp_update_duals(int64_t nx, double rho, const double* x, const double* y, double* d) {
    return guarded([&] {
        require_device();
        DBuf<double> dx(nx), dy(nx), dd(nx);
        dx.up(x, nx);
        dy.up(y, nx);
        dd.up(d, nx);
        duals_kernel<<<(int)std::min<long long>((nx + 255) / 256, 4096), 256>>>(nx, rho, dx.p, dy.p, dd.p);
        TPB_CHECK_LAUNCH();
        dd.down(d, nx);
    });
}

int tp_project_binary_z(const double* v, int64_t m, int32_t r, double* z) {
    return guarded([&] {
        require_device();
        if (r < 0 || r > m) throw Error(kInvalidArgument, "project_binary_z: r outside [0, |E|]");
        init_attrs();
        DBuf<double> dv(m);
        DBuf<int> dr(1);
        dv.up(v, m);
        dr.up(&r, 1);
        SelectArgs a{};
        a.base = dv.p;
        a.stride = m;
        a.m = m;
        a.r = dr.p;
        a.binary = 1;
        launch_topr(a, 1, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        dv.down(z, m);
    });
}

int tp_extract_topology(int32_t n, int32_t r, const double* g, double weight_floor,
                        int32_t* edges, double* weights, int32_t* n_edges) {
    return guarded([&] {
        require_device();
        if (n < 2) throw Error(kInvalidArgument, "enumerate_edges: need at least two nodes");
        if (r < 1) throw Error(kInvalidArgument, "extract_topology: r must be >= 1");
        init_attrs();
        const long long m = (long long)n * (n - 1) / 2;
        const int cap = (int)std::min<long long>(r, m);
        DBuf<double> dg(m), t(m), packed(m), ew(cap), worst(1);
        DBuf<int> dr(1), list(cap), count(1), ei(cap), ej(cap), ci(cap);
        dg.up(g, m);
        dr.up(&r, 1);
        launch_floor_mask(dg.p, m, m, weight_floor, t.p, 1, 0);
        SelectArgs a{};
        a.base = t.p;
        a.stride = m;
        a.m = m;
        a.r = dr.p;
        a.binary = 0;
        a.list = list.p;
        a.list_count = count.p;
        a.list_cap = cap;
        launch_topr(a, 1, 0);
        packed.zero();
        launch_extract(n, m, t.p, m, list.p, count.p, cap, ei.p, ej.p, ew.p, packed.p, worst.p, ci.p, 1, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        int k = 0;
        count.down(&k, 1);
        if (k == 0) throw Error(kDegenerate, "every edge weight is at or below the floor");
        std::vector<int> hi(k), hj(k);
        ei.down(hi.data(), k);
        ej.down(hj.data(), k);
        ew.down(weights, k);
        for (int e = 0; e < k; ++e) {
            edges[2 * e] = hi[e];
            edges[2 * e + 1] = hj[e];
        }
        *n_edges = k;
    });
}

int tp_allocate_batch(const double* b, const int32_t* caps, int32_t n, const int32_t* r, int32_t P,
                      double* b_unit, int32_t* e, int32_t* status) {
    return guarded([&] {
        require_device();
        if (P < 1) throw Error(kInvalidArgument, "allocate: no problems");
        if (n < 2) {
            for (int p = 0; p < P; ++p) status[p] = TP_ERR_INVALID_ARGUMENT;
            return;
        }
        DBuf<double> db((size_t)P * n), bu(P);
        DBuf<int> dc(caps ? (size_t)P * n : 1), dr(P), de((size_t)P * n), ds(P);
        db.up(b, (size_t)P * n);
        if (caps) dc.up(caps, (size_t)P * n);
        dr.up(r, P);
        launch_allocate(db.p, caps ? dc.p : nullptr, n, dr.p, P, bu.p, de.p, ds.p, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        bu.down(b_unit, P);
        de.down(e, (size_t)P * n);
        ds.down(status, P);
    });
}

int tp_allocate(const double* b, const int32_t* caps, int32_t n, int32_t r, double* b_unit,
                int32_t* e) {
    int32_t st = 0;
    const int rc = tp_allocate_batch(b, caps, n, &r, 1, b_unit, e, &st);
    if (rc != TP_OK) return rc;
    if (st == TP_ERR_INVALID_ARGUMENT) last_error_ref() = "allocate_edge_capacity: invalid argument";
    if (st == TP_ERR_INFEASIBLE) last_error_ref() = "allocate_edge_capacity: edge budget infeasible";
    return st;
}

int tp_spectral_report(int32_t n, const double* w, double* out4) {
    return guarded([&] {
        require_device();
        if (n < 1) throw Error(kInvalidArgument, "spectral_report: matrix not square");
        init_attrs();
        DBuf<double> dw((size_t)n * n), sw((size_t)n * n), chk(2), basis((size_t)n * n), out(4);
        dw.up(w, (size_t)n * n);
        dense_check_kernel<<<1, 256>>>(dw.p, n, chk.p);
        TPB_CHECK_LAUNCH();
        double c2[2];
        chk.down(c2, 2);
        if (c2[0] > 1e-8) throw Error(kInvalidArgument, "spectral_report: matrix asymmetric beyond 1e-8");
        sym_copy_kernel<<<256, 256>>>(dw.p, n, sw.p);
        TPB_CHECK_LAUNCH();
        const int deflate = (n > 1 && c2[1] <= 1e-12 * n) ? 1 : 0;
        launch_slem_dense(sw.p, n, basis.p, out.p, deflate, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        out.down(out4, 4);
    });
}

int tp_spectral_edges(int32_t n, const int32_t* edges, const double* weights, int32_t k,
                      double* out4) {
    return guarded([&] {
        require_device();
        if (n < 2) throw Error(kInvalidArgument, "spectral: need at least two nodes");
        std::vector<std::pair<long long, double>> es(k);
        for (int e = 0; e < k; ++e) {
            const int i = edges[2 * e], j = edges[2 * e + 1];
            if (i < 0 || j < 0 || i >= n || j >= n || i >= j)
                throw Error(kInvalidArgument, "topology: invalid edge");
            if (!(weights[e] >= 0.0)) throw Error(kInvalidArgument, "topology: negative or NaN weight");
            es[e] = {edge_idx(n, i, j), weights[e]};
        }
        std::sort(es.begin(), es.end());
        std::vector<int> packed;
        std::vector<double> wts;
        for (auto& p : es)
            if (p.second != 0.0) {
                packed.push_back((int)p.first);
                wts.push_back(p.second);
            }
        slem_edges(n, packed, wts, out4);
    });
}

int tp_project_psd(int32_t n, const double* a, double* out) {
    return guarded([&] { cone_dense(n, a, out, true); });
}

int tp_project_nsd(int32_t n, const double* a, double* out) {
    return guarded([&] { cone_dense(n, a, out, false); });
}

// One Ozaki-scheme GEMM (ozaki_kernels.cuh) on nmat symmetric ld x ld
// matrices (host, ld % 128 == 0): digit planes of A and B (exponents eA, eB)
// are made on the device, then C = alpha A.B + beta E (E = A if use_e) with
// FP64 output C and, if cd != null, the digit planes of C (exponent eC).
// Repeats the GEMM `reps` times (event-timed, ms per launch in *ms).
int tp_oz_gemm(int32_t ld, int32_t nmat, const double* a, int32_t ea, const double* b, int32_t eb,
               int32_t use_e, double alpha, double beta, double* c, int8_t* cd, int32_t ec,
               int32_t reps, double* ms) {
    return guarded([&] {
        require_device();
        init_attrs();
        check_oz_ld(ld);
        if (nmat <= 0) throw Error(kInvalidArgument, "tp_oz_gemm: nmat must be positive");
        const size_t sz = (size_t)nmat * ld * ld;
        DBuf<double> A(sz), B(sz), C(sz);
        DBuf<int8_t> Ad(sz * kOzSlices), Bd(sz * kOzSlices), Cd(sz * kOzSlices);
        A.up(a, sz);
        B.up(b, sz);
        C.zero();
        Cd.zero();
        launch_oz_split(A.p, (long long)ld * ld, ld, nmat, nullptr, ea, Ad.p, nullptr, 0);
        launch_oz_split(B.p, (long long)ld * ld, ld, nmat, nullptr, eb, Bd.p, nullptr, 0);
        OzMaps ma, mb;
        make_oz_maps(Ad.p, ld, nmat, &ma);
        make_oz_maps(Bd.p, ld, nmat, &mb);
        OzGemm g{};
        g.ma = &ma;
        g.mb = &mb;
        g.eA = ea;
        g.eB = eb;
        g.ld = ld;
        g.nmat = nmat;
        g.alpha_c = alpha;
        g.beta_c = beta;
        g.E = use_e ? A.p : nullptr;
        g.C = C.p;
        g.c_stride_b = 2LL * ld * ld;
        g.c_stride_w = (long long)ld * ld;
        g.ldc = ld;
        g.nvalid = ld;
        g.Cd = cd ? Cd.p : nullptr;
        g.eC = ec;
        launch_oz_gemm(g, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        C.down(c, sz);
        if (cd) Cd.down(cd, sz * kOzSlices);
        // timed repetitions: with a digit output requested, digits only (the
        // cone iteration's intermediate products); else the FP64 output
        if (cd) g.C = nullptr;
        if (reps > 0) {
            cudaEvent_t e0, e1;
            TPB_CUDA(cudaEventCreate(&e0));
            TPB_CUDA(cudaEventCreate(&e1));
            TPB_CUDA(cudaEventRecord(e0, 0));
            for (int k = 0; k < reps; ++k) launch_oz_gemm(g, 0);
            TPB_CUDA(cudaEventRecord(e1, 0));
            TPB_CUDA(cudaEventSynchronize(e1));
            float t = 0.f;
            TPB_CUDA(cudaEventElapsedTime(&t, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            if (ms) *ms = t / reps;
        }
    });
}

// project_binary_z_capped (proj/src/admm_het.cpp:125-154) on the device.
int tp_project_binary_z_capped(int32_t n, int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                               const int32_t* caps, const int32_t* allowed, const double* v, int32_t r,
                               double* z) {
    return guarded([&] {
        require_device();
        if (n < 2) throw Error(kInvalidArgument, "capacity system: need at least 2 nodes");
        const int m = n * (n - 1) / 2;
        if (r < 0 || r > m) throw Error(kInvalidArgument, "project_binary_z_capped: r outside [0, |E|]");
        const int nnz = row_ptr[nrows];
        for (int q = 0; q < nnz; ++q)
            if (cols[q] < 0 || cols[q] >= m)
                throw Error(kInvalidArgument, "capacity system: a row references a column outside [0, |E|)");
        std::vector<int> cnt(m + 1, 0), colr(std::max(nnz, 1));
        for (int q = 0; q < nnz; ++q) ++cnt[cols[q] + 1];
        for (int l = 0; l < m; ++l) cnt[l + 1] += cnt[l];
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int rr = 0; rr < nrows; ++rr)
            for (int q = row_ptr[rr]; q < row_ptr[rr + 1]; ++q) colr[pos[cols[q]]++] = rr;
        int pad = 1;
        while (pad < m) pad <<= 1;
        DBuf<double> dv(m);
        DBuf<int> dcp(m + 1), dcr(colr.size()), dcaps(std::max(nrows, 1)), dal(m), dr(1), didx(pad),
            dload(std::max(nrows, 1));
        DBuf<unsigned long long> dkeys(pad);
        dv.up(v, m);
        dcp.up(cnt.data(), m + 1);
        dcr.up(colr.data(), colr.size());
        if (nrows > 0) dcaps.up(caps, nrows);
        dal.up(allowed, m);
        dr.up(&r, 1);
        CappedArgs a{};
        a.base = dv.p;
        a.stride = m;
        a.m = m;
        a.r = dr.p;
        a.colr_ptr = dcp.p;
        a.colr = dcr.p;
        a.caps = dcaps.p;
        a.nrows = nrows;
        a.allowed = dal.p;
        a.keys = dkeys.p;
        a.idx = didx.p;
        a.load = dload.p;
        a.pad = pad;
        a.done = nullptr;
        launch_capped_z(a, 1, 0);
        TPB_CUDA(cudaDeviceSynchronize());
        dv.down(z, m);
    });
}
}  // extern "C"
