// SLEM of the gossip matrix W = I - L(g) by Lanczos on the Laplacian, one CTA
// per solve. Replaces the dense Householder + QL eigendecomposition that the
// reference runs every ADMM iteration for the trace column acf_iterate
// (acf_of_g, proj/src/admm.cpp:136-141 -> spectral_report,
// proj/src/topology.cpp:125-144) and once for the final report.
//
//  * L has <= r nonzero edges; the 1-vector is its known null vector, so the
//    Krylov space is built on 1-perp (explicit mean deflation every step).
//    lambda2(W) = 1 - mu_min(L|1perp), lambda_n(W) = 1 - mu_max(L).
//  * SpMV is a deterministic gather: per node, incident edges in ascending
//    edge index (column part from a stable counting sort, then row part).
//  * Full reorthogonalisation (CGS2 against the stored basis) when a basis
//    buffer is given; otherwise plain three-term Lanczos (extreme Ritz values
//    stay correct; ghosts only duplicate converged values).
//  * Extreme Ritz values by warp multisection on Sturm counts; convergence by
//    the residual bound beta_k |s_k| from inverse iteration on T_k.
#include "slem_kernels.cuh"
#include "csr.cuh"

namespace tpb {

namespace {

constexpr int kThreads = 512;
constexpr int kMaxK = 2048;  // smem alpha/beta capacity

// Sturm count: number of eigenvalues of the k x k tridiagonal (al, be) < x.
__device__ int sturm_count(const double* al, const double* be, int k, double x) {
    int cnt = 0;
    double d = 1.0;
    const double pivmin = 1e-300;
    for (int i = 0; i < k; ++i) {
        const double b2 = i > 0 ? be[i - 1] * be[i - 1] : 0.0;
        d = (al[i] - x) - (i > 0 ? b2 / d : 0.0);
        if (fabs(d) < pivmin) d = -pivmin;
        if (d < 0.0) ++cnt;
    }
    return cnt;
}

// idx-th smallest eigenvalue (0-based) of T_k by warp multisection.
__device__ double tri_eig(const double* al, const double* be, int k, int idx, double lo, double hi) {
    const int lane = threadIdx.x & 31;
    for (int round = 0; round < 40; ++round) {
        const double x = lo + (hi - lo) * (lane + 1) / 33.0;
        const int c = sturm_count(al, be, k, x);
        // first lane whose count exceeds idx bounds the eigenvalue from above
        const unsigned mask = __ballot_sync(0xffffffffu, c > idx);
        const int first = mask ? __ffs(mask) - 1 : 32;
        const double nlo = first == 0 ? lo : lo + (hi - lo) * first / 33.0;
        const double nhi = first == 32 ? hi : lo + (hi - lo) * (first + 1) / 33.0;
        lo = nlo;
        hi = nhi;
        if (hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300) break;
    }
    return 0.5 * (lo + hi);
}

// |last component| of the unit eigenvector of T_k for eigenvalue theta, by two
// steps of inverse iteration (Thomas algorithm on T - theta I). Single thread.
__device__ double ritz_last(const double* al, const double* be, int k, double theta, double* wk) {
    // wk: 3k doubles (c', d', x)
    double* cp = wk;
    double* dp = wk + k;
    double* x = wk + 2 * k;
    const double shift = theta + 1e-14 * fmax(1.0, fabs(theta));
    for (int i = 0; i < k; ++i) x[i] = 1.0;
    for (int it = 0; it < 2; ++it) {
        // solve (T - shift) y = x
        double denom = al[0] - shift;
        if (fabs(denom) < 1e-300) denom = 1e-300;
        cp[0] = k > 1 ? be[0] / denom : 0.0;
        dp[0] = x[0] / denom;
        for (int i = 1; i < k; ++i) {
            double dn = (al[i] - shift) - be[i - 1] * cp[i - 1];
            if (fabs(dn) < 1e-300) dn = 1e-300;
            cp[i] = i < k - 1 ? be[i] / dn : 0.0;
            dp[i] = (x[i] - be[i - 1] * dp[i - 1]) / dn;
        }
        x[k - 1] = dp[k - 1];
        for (int i = k - 2; i >= 0; --i) x[i] = dp[i] - cp[i] * x[i + 1];
        double nrm = 0.0;
        for (int i = 0; i < k; ++i) nrm += x[i] * x[i];
        nrm = sqrt(nrm);
        if (!(nrm > 0.0) || !isfinite(nrm)) return 1.0;
        for (int i = 0; i < k; ++i) x[i] /= nrm;
    }
    return fabs(x[k - 1]);
}

__device__ inline double hash_unit(int i) {
    unsigned x = 2166136261u ^ (unsigned)i * 16777619u;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    return (double)(x & 0xffffff) / 16777216.0 - 0.5;
}

}  // namespace

__global__ void __launch_bounds__(kThreads) slem_kernel(SlemArgs a) {
    const int b = blockIdx.x;
    if (a.ictl && a.ictl[b * 8 + 1]) return;  // solve already finished
    const int n = a.n;
    const int tid = threadIdx.x;
    const int ne = min(a.count[b], a.list_cap);
    const int* list = a.list + (long long)b * a.list_cap;
    const double* g = a.g + (long long)b * a.stride;
    int* ei = a.e_i + (long long)b * a.list_cap;
    int* ej = a.e_j + (long long)b * a.list_cap;
    double* ew = a.e_w + (long long)b * a.list_cap;
    int* cidx = a.col_idx + (long long)b * a.list_cap;
    double* basis = a.basis ? a.basis + (long long)b * a.kmax * n : nullptr;

    extern __shared__ double sh[];
    double* q = sh;            // n
    double* qp = sh + n;       // n
    double* w = sh + 2 * n;    // n
    double* al = sh + 3 * n;   // kMaxK
    double* be = al + kMaxK;   // kMaxK
    double* wk = be + kMaxK;   // 4*kMaxK
    int* rowptr = (int*)(wk + 4 * kMaxK);  // n+1
    int* colptr = rowptr + (n + 1);        // n+1
    int* cur = colptr + (n + 1);           // n
    __shared__ double scratch[32];
    __shared__ int iscr[32];
    __shared__ int s_stop, s_k;
    __shared__ double s_res[2];

    // ---- deterministic incidence of the support
    build_csr(n, ne, list, g, ei, ej, ew, rowptr, colptr, cur, cidx, iscr);

    // ---- Lanczos on L restricted to 1-perp
    const int dim = n - 1;
    int kmax = min(a.kmax, min(dim, kMaxK));
    if (kmax < 1) kmax = 1;
    {
        double s = 0.0;
        for (int v = tid; v < n; v += kThreads) {
            q[v] = hash_unit(v);
            qp[v] = 0.0;
            s += q[v];
        }
        s = block_sum(s, scratch);
        const double mean = s / n;
        double nn = 0.0;
        for (int v = tid; v < n; v += kThreads) {
            q[v] -= mean;
            nn += q[v] * q[v];
        }
        nn = block_sum(nn, scratch);
        const double inv = 1.0 / sqrt(nn);
        for (int v = tid; v < n; v += kThreads) q[v] *= inv;
    }
    if (tid == 0) {
        s_stop = 0;
        s_k = 0;
    }
    __syncthreads();
    double beta_prev = 0.0;
    double th_min = 0.0, th_max = 0.0;
    int k = 0;
    for (k = 0; k < kmax; ++k) {
        if (basis)
            for (int v = tid; v < n; v += kThreads) basis[(long long)k * n + v] = q[v];
        // w = L q - beta_prev q_prev
        for (int v = tid; v < n; v += kThreads) {
            const double qv = q[v];
            double acc = 0.0;
            for (int p = colptr[v]; p < colptr[v + 1]; ++p) {
                const int e = cidx[p];
                acc += ew[e] * (qv - q[ei[e]]);
            }
            for (int e = rowptr[v]; e < rowptr[v + 1]; ++e) acc += ew[e] * (qv - q[ej[e]]);
            w[v] = acc - beta_prev * qp[v];
        }
        __syncthreads();
        double dot = 0.0;
        for (int v = tid; v < n; v += kThreads) dot += w[v] * q[v];
        const double alpha = block_sum(dot, scratch);
        for (int v = tid; v < n; v += kThreads) w[v] -= alpha * q[v];
        __syncthreads();
        if (basis) {
            // CGS2 against q_0..q_k: dots by warps, update by nodes
            const int lane = tid & 31, wid = tid >> 5;
            for (int pass = 0; pass < 2; ++pass) {
                for (int j = wid; j <= k; j += kThreads / 32) {
                    double c = 0.0;
                    for (int v = lane; v < n; v += 32) c += basis[(long long)j * n + v] * w[v];
                    c = warp_sum(c);
                    if (lane == 0) wk[j] = c;
                }
                __syncthreads();
                for (int v = tid; v < n; v += kThreads) {
                    double acc = w[v];
                    for (int j = 0; j <= k; ++j) acc -= wk[j] * basis[(long long)j * n + v];
                    w[v] = acc;
                }
                __syncthreads();
            }
        }
        // deflate the 1-vector last, so reorthogonalisation round-off is not
        // amplified by 1/beta into the null direction
        double s = 0.0;
        for (int v = tid; v < n; v += kThreads) s += w[v];
        s = block_sum(s, scratch);
        const double mean = s / n;
        for (int v = tid; v < n; v += kThreads) w[v] -= mean;
        double nn = 0.0;
        for (int v = tid; v < n; v += kThreads) nn += w[v] * w[v];
        nn = block_sum(nn, scratch);
        const double beta = sqrt(nn);
        if (tid == 0) {
            al[k] = alpha;
            be[k] = beta;
        }
        __syncthreads();
        const int kk = k + 1;
        const double scale = fmax(fabs(alpha), 1e-300);
        bool breakdown = !(beta > 1e-13 * fmax(scale, fabs(th_max)));
        const bool check = breakdown || kk == kmax || (kk % 8 == 0);
        if (check) {
            if (tid < 32) {
                // Gershgorin bounds
                double lo = 1e300, hi = -1e300;
                for (int i = 0; i < kk; ++i) {
                    const double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i < kk - 1 ? fabs(be[i]) : 0.0);
                    lo = fmin(lo, al[i] - r);
                    hi = fmax(hi, al[i] + r);
                }
                lo -= 1e-12 * fmax(1.0, fabs(lo));
                hi += 1e-12 * fmax(1.0, fabs(hi));
                const double tmin = tri_eig(al, be, kk, 0, lo, hi);
                const double tmax = tri_eig(al, be, kk, kk - 1, lo, hi);
                if (tid == 0) {
                    double r1 = 0.0, r2 = 0.0;
                    if (!breakdown && kk < dim) {
                        r1 = beta * ritz_last(al, be, kk, tmin, wk + kMaxK / 2);
                        r2 = beta * ritz_last(al, be, kk, tmax, wk + kMaxK / 2);
                    }
                    const double sc = fmax(fabs(tmax), 1e-300);
                    s_res[0] = tmin;
                    s_res[1] = tmax;
                    if (breakdown || kk >= dim || (r1 <= a.tol * sc && r2 <= a.tol * sc)) s_stop = 1;
                    s_k = kk;
                }
            }
            __syncthreads();
            th_min = s_res[0];
            th_max = s_res[1];
            if (s_stop) break;
        }
        // advance
        const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
        for (int v = tid; v < n; v += kThreads) {
            qp[v] = q[v];
            q[v] = w[v] * inv;
        }
        beta_prev = beta;
        __syncthreads();
    }
    if (tid == 0) {
        const double l2 = 1.0 - th_min, ln = 1.0 - th_max;
        const double acf = fmax(fabs(l2), fabs(ln));
        if (a.tr_acf) {
            const int it = a.ictl[b * 8];
            a.tr_acf[(long long)b * a.max_iter + it] = acf;
        }
        if (a.out) {
            double* o = a.out + b * 8;
            o[0] = n == 1 ? 0.0 : acf;
            o[1] = l2;
            o[2] = ln;
            o[3] = (l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
            o[4] = s_k;
            o[5] = s_stop;
        }
    }
}

void launch_slem(const SlemArgs& a, int B, cudaStream_t st) {
    const int n = a.n;
    const size_t smem = (3 * (size_t)n + 6 * kMaxK) * sizeof(double) + (3 * (size_t)n + 2) * sizeof(int);
    slem_kernel<<<B, kThreads, smem, st>>>(a);
    TPB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- dense
// Full-spectrum Lanczos with CGS2 reorthogonalisation to k = n (exact up to
// rounding), then lambda2 = second largest and lambda_n = smallest Ritz value.
__global__ void __launch_bounds__(kThreads) slem_dense_kernel(const double* W, int n, double* basis,
                                                             double* out, int deflate) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    extern __shared__ double sh[];
    double* q = sh;
    double* w = sh + n;
    double* al = sh + 2 * n;
    double* be = al + kMaxK;
    double* cf = be + kMaxK;
    __shared__ double scratch[32];
    __shared__ int s_stop;
    double s = 0.0;
    for (int v = tid; v < n; v += kThreads) {
        q[v] = hash_unit(v) + (deflate ? 0.0 : 1.0);
        s += q[v];
    }
    s = block_sum(s, scratch);
    double nn0 = 0.0;
    for (int v = tid; v < n; v += kThreads) {
        if (deflate) q[v] -= s / n;
        nn0 += q[v] * q[v];
    }
    nn0 = block_sum(nn0, scratch);
    for (int v = tid; v < n; v += kThreads) q[v] /= sqrt(nn0);
    if (tid == 0) s_stop = 0;
    __syncthreads();
    const int kmax = min(deflate ? n - 1 : n, kMaxK);
    int kk = 0;
    for (int k = 0; k < kmax; ++k) {
        for (int v = tid; v < n; v += kThreads) basis[(long long)k * n + v] = q[v];
        // w = W q (row-major; one warp per row)
        for (int r = wid; r < n; r += kThreads / 32) {
            double acc = 0.0;
            for (int c = lane; c < n; c += 32) acc += W[(long long)r * n + c] * q[c];
            acc = warp_sum(acc);
            if (lane == 0) w[r] = acc;
        }
        __syncthreads();
        double dot = 0.0;
        for (int v = tid; v < n; v += kThreads) dot += w[v] * q[v];
        const double alpha = block_sum(dot, scratch);
        for (int pass = 0; pass < 2; ++pass) {
            for (int j = wid; j <= k; j += kThreads / 32) {
                double c = 0.0;
                for (int v = lane; v < n; v += 32) c += basis[(long long)j * n + v] * w[v];
                c = warp_sum(c);
                if (lane == 0) cf[j] = c;
            }
            __syncthreads();
            for (int v = tid; v < n; v += kThreads) {
                double acc = w[v];
                for (int j = 0; j <= k; ++j) acc -= cf[j] * basis[(long long)j * n + v];
                w[v] = acc;
            }
            __syncthreads();
        }
        if (deflate) {  // last, see slem_kernel
            double sm = 0.0;
            for (int v = tid; v < n; v += kThreads) sm += w[v];
            sm = block_sum(sm, scratch);
            for (int v = tid; v < n; v += kThreads) w[v] -= sm / n;
            __syncthreads();
        }
        double nn = 0.0;
        for (int v = tid; v < n; v += kThreads) nn += w[v] * w[v];
        nn = block_sum(nn, scratch);
        const double beta = sqrt(nn);
        if (tid == 0) {
            al[k] = alpha;
            be[k] = beta;
            if (!(beta > 1e-13 * fmax(fabs(alpha), 1e-300))) s_stop = 1;
        }
        __syncthreads();
        kk = k + 1;
        if (s_stop) break;
        for (int v = tid; v < n; v += kThreads) q[v] = w[v] / beta;
        __syncthreads();
    }
    if (tid < 32) {
        double lo = 1e300, hi = -1e300;
        for (int i = 0; i < kk; ++i) {
            const double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i < kk - 1 ? fabs(be[i]) : 0.0);
            lo = fmin(lo, al[i] - r);
            hi = fmax(hi, al[i] + r);
        }
        lo -= 1e-12 * fmax(1.0, fabs(lo));
        hi += 1e-12 * fmax(1.0, fabs(hi));
        const double lmin = tri_eig(al, be, kk, 0, lo, hi);
        double l2;
        if (deflate) {
            // spectrum = {1 (eigenvector 1)} U spectrum on 1-perp
            const double top = tri_eig(al, be, kk, kk - 1, lo, hi);
            const double sec = kk >= 2 ? tri_eig(al, be, kk, kk - 2, lo, hi) : -1e300;
            l2 = top <= 1.0 ? top : fmax(1.0, sec);
        } else {
            l2 = kk >= 2 ? tri_eig(al, be, kk, kk - 2, lo, hi) : lmin;
        }
        const double lminall = deflate ? fmin(lmin, 1.0) : lmin;
        if (tid == 0) {
            out[0] = n == 1 ? 0.0 : fmax(fabs(l2), fabs(lminall));
            out[1] = n == 1 ? 0.0 : l2;
            out[2] = lminall;
            out[3] = (n == 1 || l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
        }
    }
}

void launch_slem_dense(const double* w, int n, double* basis, double* out, int deflate, cudaStream_t st) {
    const size_t smem = (2 * (size_t)n + 3 * kMaxK) * sizeof(double);
    slem_dense_kernel<<<1, kThreads, smem, st>>>(w, n, basis, out, deflate);
    TPB_CHECK_LAUNCH();
}

void init_attrs_slem() {
    set_max_dyn_smem(slem_kernel);
    set_max_dyn_smem(slem_dense_kernel);
}

}  // namespace tpb
