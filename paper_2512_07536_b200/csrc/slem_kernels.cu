// SLEM of the gossip matrix W = I - L(g) by Lanczos on the Laplacian, one CTA
// per solve. Replaces the dense Householder + QL eigendecomposition that the
// reference runs every ADMM iteration for the trace column acf_iterate
// (acf_of_g, proj/src/admm.cpp:136-141 -> spectral_report,
// proj/src/topology.cpp:125-144) and once for the final report.
//
//  * L has <= r nonzero edges; the 1-vector is its known null vector, so the
//    Krylov space is built on 1-perp. lambda2(W) = 1 - mu_min(L|1perp),
//    lambda_n(W) = 1 - mu_max(L).
//  * SpMV is a deterministic gather: per node, incident edges in ascending
//    edge index (column part from a stable counting sort, then row part).
//  * Full reorthogonalisation (CGS2 against the stored basis); the 1-vector is
//    deflated last so round-off is not amplified by 1/beta.
//  * Explicit restarts from the two extreme Ritz vectors, and a warm start
//    from the previous ADMM iteration's Ritz vectors (the support moves
//    slowly), keep the trace evaluation at a few dozen matvecs.
//  * Extreme Ritz values by warp multisection on Sturm counts; convergence by
//    the residual bound beta_k |s_k| (s from inverse iteration on T_k).
#include "slem_kernels.cuh"

#include <cooperative_groups.h>
#include "csr.cuh"

namespace tpb {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 512;

// number of eigenvalues of the k x k tridiagonal (al, be) below x: sign
// changes of the Sturm sequence p_i = det(T_i - x I),
//   p_i = (al_i - x) p_{i-1} - be_{i-1}^2 p_{i-2},
// division-free (two FMAs per step; the LDL^T form has a dependent FP64
// division per step), rescaled by exact powers of two. A zero p_i counts as
// a change (the LDL^T convention d_i -> -0).
__device__ int sturm_count(const double* al, const double* be, int k, double x) {
    int cnt = 0;
    double pm = 1.0, p = 1.0;  // p_{i-2}, p_{i-1}
    bool prev_neg = false;     // sign of p_{i-1} (p_0 = 1 > 0), zero -> opposite of its predecessor
    for (int i = 0; i < k; ++i) {
        const double b2 = i > 0 ? be[i - 1] * be[i - 1] : 0.0;
        const double pn = fma(al[i] - x, p, -b2 * pm);
        // sign and zero tests on the bits (integer pipe; the FP64 pipe keeps
        // only the recurrence): pn < 0 <=> sign set and nonzero (no NaN here)
        const long long pb = __double_as_longlong(pn);
        const bool zero = (pb & 0x7fffffffffffffffLL) == 0;
        const bool neg = zero ? !prev_neg : pb < 0;
        cnt += neg != prev_neg;
        prev_neg = neg;
        pm = p;
        p = pn;
        // rescale every 8 steps (|p| grows by < 2^5 per step with the spectra
        // bounded by Gershgorin here, far inside the 2^400 margin): keeps the
        // dependent chain per step at two FMAs
        if ((i & 7) == 7) {
            const double mx = fmax(fabs(p), fabs(pm));
            if (mx > 0x1p400) {
                p *= 0x1p-400;
                pm *= 0x1p-400;
            } else if (mx < 0x1p-400 && mx > 0.0) {
                p *= 0x1p400;
                pm *= 0x1p400;
            }
        }
    }
    return cnt;
}

// idx-th smallest eigenvalue (0-based) of T_k by warp multisection (one warp).
__device__ double tri_eig(const double* al, const double* be, int k, int idx, double lo, double hi) {
    const int lane = threadIdx.x & 31;
    for (int round = 0; round < 40; ++round) {
        const double x = lo + (hi - lo) * (lane + 1) / 33.0;
        const int c = sturm_count(al, be, k, x);
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

__device__ void gershgorin(const double* al, const double* be, int k, double& lo, double& hi) {
    lo = 1e300;
    hi = -1e300;
    for (int i = 0; i < k; ++i) {
        const double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i < k - 1 ? fabs(be[i]) : 0.0);
        lo = fmin(lo, al[i] - r);
        hi = fmax(hi, al[i] + r);
    }
    lo -= 1e-12 * fmax(1.0, fabs(lo));
    hi += 1e-12 * fmax(1.0, fabs(hi));
}

// Unit eigenvector s of T_k for eigenvalue theta (two inverse iterations,
// Thomas algorithm, one reciprocal per row); returns |s_{k-1}|. Single
// thread; work: 2k doubles.
__device__ double tri_vec(const double* al, const double* be, int k, double theta, double* work,
                          double* s) {
    double* cp = work;
    double* dp = work + k;
    const double shift = theta + 1e-14 * fmax(1.0, fabs(theta));
    for (int i = 0; i < k; ++i) s[i] = 1.0;
    for (int it = 0; it < 2; ++it) {
        double den = al[0] - shift;
        if (fabs(den) < 1e-300) den = 1e-300;
        double inv = 1.0 / den;
        cp[0] = k > 1 ? be[0] * inv : 0.0;
        dp[0] = s[0] * inv;
        for (int i = 1; i < k; ++i) {
            double dn = fma(-be[i - 1], cp[i - 1], al[i] - shift);
            if (fabs(dn) < 1e-300) dn = 1e-300;
            inv = 1.0 / dn;
            cp[i] = i < k - 1 ? be[i] * inv : 0.0;
            dp[i] = fma(-be[i - 1], dp[i - 1], s[i]) * inv;
        }
        s[k - 1] = dp[k - 1];
        double nrm = s[k - 1] * s[k - 1];
        for (int i = k - 2; i >= 0; --i) {
            s[i] = fma(-cp[i], s[i + 1], dp[i]);
            nrm = fma(s[i], s[i], nrm);
        }
        nrm = sqrt(nrm);
        if (!(nrm > 0.0) || !isfinite(nrm)) {
            for (int i = 0; i < k; ++i) s[i] = (i == k - 1) ? 1.0 : 0.0;
            return 1.0;
        }
        const double rn = 1.0 / nrm;
        for (int i = 0; i < k; ++i) s[i] *= rn;
    }
    return fabs(s[k - 1]);
}

__device__ inline double hash_unit(int i) {
    unsigned x = 2166136261u ^ (unsigned)i * 16777619u;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    return (double)(x & 0xffffff) / 16777216.0 - 0.5;
}

// q <- (q - mean q) / ||q - mean q||
__device__ void deflate_normalize(double* q, int n, double* scratch) {
    double s = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) s += q[v];
    s = block_sum(s, scratch);
    const double mean = s / n;
    double nn = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        q[v] -= mean;
        nn += q[v] * q[v];
    }
    nn = block_sum(nn, scratch);
    const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) q[v] *= inv;
    __syncthreads();
}

// convergence checks at k = 4, 8, 12, 16, 24, 32, 48, 64, 96, ...
__device__ inline bool check_step(int kk) {
    if (kk <= 16) return (kk & 3) == 0;
    int p = 16;
    while (p < kk) {
        if (p + p / 2 == kk) return true;
        p <<= 1;
    }
    return p == kk;
}

}  // namespace

__device__ inline void block_sum2(double& a, double& b, double* scratch) {
    // deterministic fused reduction of two values (scratch: 64 doubles)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if (lane == 0) {
        scratch[wid] = a;
        scratch[32 + wid] = b;
    }
    __syncthreads();
    double x = 0.0, y = 0.0;
    for (int k = 0; k < nw; ++k) {
        x += scratch[k];
        y += scratch[32 + k];
    }
    a = x;
    b = y;
}

// One-barrier reductions for the Lanczos step (block_sum's trees: warp
// sums, then every warp reduces the warp partials), with the leading and
// trailing barriers dropped. The caller alternates scratch buffers so that a
// buffer is rewritten only after a barrier that follows its last read.
__device__ inline double allreduce1(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    return warp_sum(lane < nw ? scratch[lane] : 0.0);
}

__device__ inline void allreduce2(double& a, double& b, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
        scratch[wid] = a;
        scratch[32 + wid] = b;
    }
    __syncthreads();
    a = warp_sum(lane < nw ? scratch[lane] : 0.0);
    b = warp_sum(lane < nw ? scratch[32 + lane] : 0.0);
}

// w <- w - sum_{j<=k} (Q_j . w) Q_j, twice (CGS2); cf[j] receives the first
// pass coefficients (cf[k] = alpha when q_k is the current Lanczos vector).
__device__ inline void cgs2(const double* Q, int n, int ldq, int k, double* w, double* cf,
                            double* cf2, bool q_in_smem) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    for (int pass = 0; pass < 2; ++pass) {
        double* c_out = pass == 0 ? cf : cf2;
        if (q_in_smem && k < (int)blockDim.x) {
            // one thread per basis vector: no shuffles on the critical path
            if (tid <= k) {
                const double* qj = Q + (long long)tid * ldq;
                double c0 = 0.0, c1 = 0.0;
                int v = 0;
                for (; v + 1 < n; v += 2) {
                    c0 += qj[v] * w[v];
                    c1 += qj[v + 1] * w[v + 1];
                }
                if (v < n) c0 += qj[v] * w[v];
                c_out[tid] = c0 + c1;
            }
        } else {
            for (int j = wid; j <= k; j += nw) {
                double c = 0.0;
                for (int v = lane; v < n; v += 32) c += Q[(long long)j * ldq + v] * w[v];
                c = warp_sum(c);
                if (lane == 0) c_out[j] = c;
            }
        }
        __syncthreads();
        for (int v = tid; v < n; v += blockDim.x) {
            double acc = w[v];
            for (int j = 0; j <= k; ++j) acc -= c_out[j] * Q[(long long)j * ldq + v];
            w[v] = acc;
        }
        __syncthreads();
    }
}

#ifdef OZ_STAMPS
// instrumentation build only (make STAMPS=1): per-kernel {calls, steps} of the
// Lanczos SLEM kernels, slot 0 trace reports, slot 1 one-off reports
// slots 8..13: clocks of the check parts (Gershgorin, multisection, inverse
// iteration) in warp 0 / lane 0, trace (8..10) and one-off (11..13); 14, 15:
// number of checks (trace, one-off)
__device__ unsigned long long g_slem_stats[16];
extern "C" int tp_slem_stats(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_slem_stats, sizeof(g_slem_stats)) != cudaSuccess) return 7;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_slem_stats, z, sizeof(z));
    }
    return 0;
}
#define SLEM_STAT(oneoff, steps)                                   \
    do {                                                           \
        atomicAdd(&g_slem_stats[(oneoff) ? 2 : 0], 1ull);          \
        atomicAdd(&g_slem_stats[(oneoff) ? 3 : 1], (unsigned long long)(steps)); \
    } while (0)
#define SLEM_CLK(slot, t0) \
    if (threadIdx.x == 0) atomicAdd(&g_slem_stats[slot], (unsigned long long)(clock64() - (t0)))
#else
#define SLEM_STAT(oneoff, steps) ((void)0)
#define SLEM_CLK(slot, t0) ((void)0)
#endif

// Trace mode: the iteration a report belongs to, or -1 when the solve is done.
__device__ inline int slem_iter(const SlemArgs& a, int b) {
    if (a.it_snap) return a.it_snap[b];
    if (a.ictl) return a.ictl[b * 8 + 1] ? -1 : a.ictl[b * 8];
    return 0;
}

__global__ void __launch_bounds__(kThreads) slem_kernel(SlemArgs a) {
    const int b = blockIdx.x;
    const int it_rec = slem_iter(a, b);
    if (it_rec < 0) return;  // solve already finished
    const int n = a.n;
    const int tid = threadIdx.x, nthr = blockDim.x, wid = tid >> 5;
    const int ne = min(a.count[b], a.list_cap);
    const int* list = a.list + (long long)b * a.list_cap;
    const double* g = a.gw ? a.gw + (long long)b * a.list_cap : a.g + (long long)b * a.stride;
    int* ei = a.e_i + (long long)b * a.list_cap;
    int* ej = a.e_j + (long long)b * a.list_cap;
    double* ew = a.e_w + (long long)b * a.list_cap;
    int* cidx = a.col_idx + (long long)b * a.list_cap;
    const int dim = n - 1;
    const int kmax = max(1, min(a.kmax, dim));

    extern __shared__ double sh[];
    double* q = sh;                   // n
    double* w = q + n;                // n
    double* al = w + n;               // kmax
    double* be = al + kmax;           // kmax
    double* smin = be + kmax;         // kmax
    double* smax = smin + kmax;       // kmax
    double* cf = smax + kmax;         // kmax
    double* cf2 = cf + kmax;          // kmax
    double* wk = cf2 + kmax;          // 2 kmax
    int* rowptr = (int*)(wk + 2 * kmax);  // n+1
    int* colptr = rowptr + (n + 1);       // n+1
    int* cur = colptr + (n + 1);          // n
    // Krylov basis: shared memory when it fits (a.basis == null), else global
    // (odd row stride in shared memory: conflict-free per-vector dot products)
    const int ldq = a.basis ? n : (n | 1);
    double* Q = a.basis ? a.basis + (long long)b * a.kmax * n
                        : (double*)(((uintptr_t)(cur + n) + 15) & ~(uintptr_t)15);
    __shared__ double scratch[64];
    __shared__ int iscr[32];
    __shared__ int s_flag;  // bit0 stop, bit1 converged
    __shared__ double s_th[2];

    build_csr(n, ne, list, g, a.gw != nullptr, ei, ej, ew, rowptr, colptr, cur, cidx, iscr);

    // Exact mode (Krylov dimension covers 1-perp): run to completion, no early
    // stop, so the extreme Ritz values are eigenvalues up to rounding.
    // Restarted mode: random start, or a warm start from the previous extreme
    // Ritz vectors plus a small fixed random component, and at least
    // a.min_steps matvecs before the residual test.
    const bool exact = kmax >= dim;
    const bool warm = !exact && a.ritz && a.ritz_ok && a.ritz_ok[b];
    double* rz = a.ritz ? a.ritz + (long long)b * 2 * n : nullptr;
    if (warm) {
        for (int v = tid; v < n; v += nthr) w[v] = hash_unit(v);
        __syncthreads();
        deflate_normalize(w, n, scratch);
        for (int v = tid; v < n; v += nthr) q[v] = rz[v] + rz[n + v];
        __syncthreads();
        deflate_normalize(q, n, scratch);
        for (int v = tid; v < n; v += nthr) q[v] += a.noise * w[v];
    } else {
        for (int v = tid; v < n; v += nthr) q[v] = hash_unit(v);
    }
    __syncthreads();
    deflate_normalize(q, n, scratch);

    double th_min = 0.0, th_max = 0.0;
    int steps = 0, converged = 0, kk = 0;
    for (int cycle = 0; cycle <= a.max_restarts; ++cycle) {
        if (tid == 0) s_flag = 0;
        __syncthreads();
        for (int k = 0; k < kmax; ++k) {
            for (int v = tid; v < n; v += nthr) Q[(long long)k * ldq + v] = q[v];
            // w = L q (gather, ascending edge order)
            for (int v = tid; v < n; v += nthr) {
                const double qv = q[v];
                double acc = 0.0;
                for (int p = colptr[v]; p < colptr[v + 1]; ++p) {
                    const int e = cidx[p];
                    acc += ew[e] * (qv - q[ei[e]]);
                }
                for (int e = rowptr[v]; e < rowptr[v + 1]; ++e) acc += ew[e] * (qv - q[ej[e]]);
                w[v] = acc;
            }
            __syncthreads();
            cgs2(Q, n, ldq, k, w, cf, cf2, a.basis == nullptr);
            const double alpha = cf[k] + cf2[k];
            // deflate the 1-vector last; ||w - mean||^2 = sum w^2 - n mean^2
            double s = 0.0, s2 = 0.0;
            for (int v = tid; v < n; v += nthr) {
                s += w[v];
                s2 += w[v] * w[v];
            }
            block_sum2(s, s2, scratch);
            const double mean = s / n;
            const double beta = sqrt(fmax(s2 - n * mean * mean, 0.0));
            if (tid == 0) {
                al[k] = alpha;
                be[k] = beta;
            }
            kk = k + 1;
            ++steps;
            const bool breakdown = !(beta > 1e-13 * fmax(fabs(alpha), fabs(th_max)) + 1e-300);
            if (breakdown && kk < dim && kk < kmax) {
                // invariant subspace found early: continue with a fresh direction
                // orthogonal to the basis (T decouples, beta_k = 0)
                for (int v = tid; v < n; v += nthr) w[v] = hash_unit(v * 7 + 13 * kk + 1);
                __syncthreads();
                cgs2(Q, n, ldq, k, w, cf, cf2, a.basis == nullptr);
                if (tid == 0) be[k] = 0.0;
                for (int v = tid; v < n; v += nthr) q[v] = w[v];
                __syncthreads();
                deflate_normalize(q, n, scratch);
                continue;
            }
            const bool want_check =
                exact ? (kk >= dim || breakdown)
                      : (breakdown || kk == kmax || (steps >= a.min_steps && check_step(kk)));
            if (want_check) {
                __syncthreads();
                if (wid == 0) {
                    double lo, hi;
                    gershgorin(al, be, kk, lo, hi);
                    const double tmin = tri_eig(al, be, kk, 0, lo, hi);
                    const double tmax = tri_eig(al, be, kk, kk - 1, lo, hi);
                    if (tid == 0) {
                        const double r1 = beta * tri_vec(al, be, kk, tmin, wk, smin);
                        const double r2 = beta * tri_vec(al, be, kk, tmax, wk, smax);
                        const double sc = fmax(fabs(tmax), 1e-300);
                        const bool conv = kk >= dim || (!exact && (breakdown || (r1 <= a.tol * sc &&
                                                                                   r2 <= a.tol * sc)));
                        s_th[0] = tmin;
                        s_th[1] = tmax;
                        s_flag = (conv || kk == kmax) ? (1 | (conv ? 2 : 0)) : 0;
                    }
                }
                __syncthreads();
                th_min = s_th[0];
                th_max = s_th[1];
                if (s_flag & 1) {
                    converged = (s_flag >> 1) & 1;
                    break;
                }
            }
            const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
            for (int v = tid; v < n; v += nthr) q[v] = (w[v] - mean) * inv;
            __syncthreads();
        }
        // Ritz vectors y = Q s of both extremes (restart vector / next warm start)
        if (rz || !converged) {
            for (int v = tid; v < n; v += nthr) {
                double y1 = 0.0, y2 = 0.0;
                for (int j = 0; j < kk; ++j) {
                    const double qj = Q[(long long)j * ldq + v];
                    y1 += smin[j] * qj;
                    y2 += smax[j] * qj;
                }
                w[v] = y1;
                q[v] = y2;
            }
            __syncthreads();
            if (rz) {
                for (int v = tid; v < n; v += nthr) {
                    rz[v] = w[v];
                    rz[n + v] = q[v];
                }
            }
            for (int v = tid; v < n; v += nthr) q[v] += w[v];
            __syncthreads();
            deflate_normalize(q, n, scratch);
        }
        if (converged) break;
    }
    if (tid == 0) {
        if (a.ritz_ok) a.ritz_ok[b] = 1;
        const double l2 = 1.0 - th_min, ln = 1.0 - th_max;
        const double acf = fmax(fabs(l2), fabs(ln));
        if (a.tr_acf) a.tr_acf[(long long)b * a.max_iter + it_rec] = acf;
        SLEM_STAT(a.out != nullptr, steps);
        if (a.out) {
            double* o = a.out + b * 8;
            o[0] = acf;
            o[1] = l2;
            o[2] = ln;
            o[3] = (l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
            o[4] = steps;
            o[5] = converged;
        }
    }
}

size_t slem_smem_bytes(int n, int kmax, bool basis_in_smem) {
    kmax = std::max(1, std::min(kmax, n - 1));
    size_t bytes = (2 * (size_t)n + 8 * (size_t)kmax) * sizeof(double) + (3 * (size_t)n + 2) * sizeof(int);
    if (basis_in_smem) bytes = ((bytes + 15) & ~(size_t)15) + (size_t)kmax * (n | 1) * sizeof(double);
    return bytes;
}

// ---------------------------------------------------------------- small n
// n <= kSmallDense: dense W = I - L(g) in shared memory, Householder
// tridiagonalisation in FP64, then the two eigenvalues spectral_report reads
// (values[n-2], values[0]) by Sturm multisection. Exact up to rounding like
// the reference's Householder + QL (eig.cpp:18-129), without iterating.
__global__ void __launch_bounds__(256) slem_small_kernel(SlemArgs a) {
    const int b = blockIdx.x;
    const int it_rec = slem_iter(a, b);
    if (it_rec < 0) return;
    const int n = a.n, ld = n + 1;
    const int tid = threadIdx.x, nthr = blockDim.x, wid = tid >> 5;
    const int ne = min(a.count[b], a.list_cap);
    const int* list = a.list + (long long)b * a.list_cap;
    const double* g = a.gw ? a.gw + (long long)b * a.list_cap : a.g + (long long)b * a.stride;
    extern __shared__ double sh[];
    double* A = sh;              // n x ld
    double* v = A + n * ld;      // n
    double* p = v + n;           // n
    double* d = p + n;           // n
    double* e = d + n;           // n
    __shared__ double red1[32], red2[32];  // one-barrier reductions, alternating
    __shared__ int s_it;
    if (tid == 0) s_it = it_rec;
    // W: off-diagonals +g, diagonal 1 - (sum of incident g, ascending edges)
    for (int k = tid; k < n * ld; k += nthr) A[k] = 0.0;
    __syncthreads();
    for (int t = tid; t < ne; t += nthr) {
        int i, j;
        edge_pair(n, list[t], i, j);
        const double w = a.gw ? g[t] : g[list[t]];
        A[i * ld + j] = w;
        A[j * ld + i] = w;
    }
    __syncthreads();
    for (int i = tid; i < n; i += nthr) {
        double s = 0.0;
        for (int j = 0; j < n; ++j)
            if (j != i) s += A[i * ld + j];
        A[i * ld + i] = 1.0 - s;
    }
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const int m0 = k + 1, len = n - m0;
        double nn = 0.0;
        for (int i = m0 + tid; i < n; i += nthr) nn += A[i * ld + k] * A[i * ld + k];
        nn = allreduce1(nn, red1);
        const double a0 = A[m0 * ld + k];
        if (nn == 0.0) {
            if (tid == 0) {
                d[k] = A[k * ld + k];
                e[k] = 0.0;
            }
            __syncthreads();
            continue;
        }
        const double s = sqrt(nn);
        const double sg = a0 >= 0.0 ? 1.0 : -1.0;
        const double beta = 1.0 / (s * (s + fabs(a0)));
        for (int i = m0 + tid; i < n; i += nthr) v[i] = A[i * ld + k] + (i == m0 ? sg * s : 0.0);
        __syncthreads();
        // p = beta A[m0:, m0:] v: four lanes per row (interleaved columns,
        // then two xor shuffles; fixed order)
        for (int i0 = m0; i0 < n; i0 += nthr / 4) {
            const int i = i0 + (tid >> 2), part = tid & 3;
            double acc = 0.0;
            if (i < n)
                for (int j = m0 + part; j < n; j += 4) acc += A[i * ld + j] * v[j];
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (part == 0 && i < n) p[i] = beta * acc;
        }
        __syncthreads();
        double pv = 0.0;
        for (int i = m0 + tid; i < n; i += nthr) pv += p[i] * v[i];
        pv = allreduce1(pv, red2);
        const double K = 0.5 * beta * pv;
        for (int i = m0 + tid; i < n; i += nthr) p[i] -= K * v[i];  // w
        __syncthreads();
        for (int idx = tid; idx < len * len; idx += nthr) {
            const int i = m0 + idx / len, j = m0 + idx % len;
            A[i * ld + j] -= v[i] * p[j] + p[i] * v[j];
        }
        if (tid == 0) {
            d[k] = A[k * ld + k];
            e[k] = -sg * s;
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) * ld + n - 2];
            e[n - 2] = A[(n - 1) * ld + n - 2];
        }
        d[n - 1] = A[(n - 1) * ld + n - 1];
    }
    __syncthreads();
    if (wid == 0) {
        double lo, hi;
        gershgorin(d, e, n, lo, hi);
        const double ln = tri_eig(d, e, n, 0, lo, hi);
        const double l2 = n >= 2 ? tri_eig(d, e, n, n - 2, lo, hi) : ln;
        if (tid == 0) {
            const double acf = n == 1 ? 0.0 : fmax(fabs(l2), fabs(ln));
            if (a.tr_acf) a.tr_acf[(long long)b * a.max_iter + s_it] = acf;
            if (a.out) {
                double* o = a.out + b * 8;
                o[0] = acf;
                o[1] = l2;
                o[2] = ln;
                o[3] = (l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
                o[4] = n;
                o[5] = 1.0;
            }
        }
    }
}

// ---------------------------------------------------------------- trace
// Trace SLEM (acf_iterate every ADMM iteration): plain three-term Lanczos
// without reorthogonalisation, the 1-vector deflated every step. Loss of
// orthogonality only adds ghost copies of converged extremes; the extreme
// Ritz values and the residual bound beta_k |s_k| stay valid (Paige), so the
// per-step cost is one SpMV and two block reductions instead of CGS2 against
// the stored basis (which streams kmax x n doubles per step). The basis rows
// are written (not read) each step for the Ritz vectors that warm-start the
// next iteration. Every Ritz value lies in [mu_min, mu_max], so the extremes
// are tracked across restarts.
constexpr int kTraceThreads = 1024;

__global__ void __launch_bounds__(kTraceThreads) slem_trace_kernel(SlemArgs a) {
    // a cluster of C CTAs per solve (one-off reports of one large solve) or
    // one CTA (C = 1): CTA `rank` owns nodes [v_lo, v_hi) of every
    // node-indexed pass; q is kept whole in every CTA, and each step's new
    // slice is pushed to the others through distributed shared memory
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int b = blockIdx.x / C;
    const int it_rec = slem_iter(a, b);
    if (it_rec < 0) return;  // solve already finished (uniform over the cluster)
    const int n = a.n;
    const int tid = threadIdx.x, nthr = blockDim.x, wid = tid >> 5;
    const int per = (n + C - 1) / C, v_lo = min(n, rank * per), v_hi = min(n, v_lo + per);
    const int ne = min(a.count[b], a.list_cap);
    const int* list = a.list + (long long)b * a.list_cap;
    const double* g = a.gw ? a.gw + (long long)b * a.list_cap : a.g + (long long)b * a.stride;
    int* ei = a.e_i + (long long)b * a.list_cap;
    int* ej = a.e_j + (long long)b * a.list_cap;
    double* ew = a.e_w + (long long)b * a.list_cap;
    int* cidx = a.col_idx + (long long)b * a.list_cap;
    const int dim = n - 1;
    const int kcap = max(2, min(a.kmax, dim));

    extern __shared__ double sh[];
    double* q = sh;                   // n
    double* qp = q + n;               // n
    double* w = qp + n;               // n
    double* al = w + n;               // kcap
    double* be = al + kcap;           // kcap
    double* smin = be + kcap;         // kcap
    double* smax = smin + kcap;       // kcap
    double* wk = smax + kcap;         // 4 kcap (two inverse-iteration work arrays)
    int* rowptr = (int*)(wk + 4 * kcap);  // n+1
    int* colptr = rowptr + (n + 1);       // n+1
    int* cur = colptr + (n + 1);          // n
    double* Q = a.basis + (long long)b * a.kmax * n;
    __shared__ double scratch[64];
    __shared__ double red1[32], red2[64];  // Lanczos step reductions (alternating with each other)
    __shared__ int iscr[32];
    __shared__ int s_flag;  // bit0 stop, bit1 converged
    __shared__ double s_th[2];
    __shared__ double s_res[2];
    __shared__ double xch[2][16][2];  // cluster partials (two alternating buffers)
    auto csync = [&] {
        if (C > 1)
            cl.sync();
        else
            __syncthreads();
    };
    // cluster-wide sum of a CTA value pair (CTA partials in rank order)
    auto cluster_sum2 = [&](double& x, double& y, int buf) {
        if (C == 1) return;
        if (tid == 0)
            for (int r = 0; r < C; ++r) {
                double* dst = cl.map_shared_rank(&xch[buf][rank][0], r);
                dst[0] = x;
                dst[1] = y;
            }
        cl.sync();
        double sx = 0.0, sy = 0.0;
        for (int r = 0; r < C; ++r) {
            sx += xch[buf][r][0];
            sy += xch[buf][r][1];
        }
        x = sx;
        y = sy;
    };

    // the incidence: built once (CTA 0 writes the global edge arrays), the
    // cluster's other CTAs take rowptr / colptr from CTA 0's shared memory
    if (rank == 0) build_csr(n, ne, list, g, a.gw != nullptr, ei, ej, ew, rowptr, colptr, cur, cidx, iscr);
    if (C > 1) {
        cl.sync();
        if (rank != 0) {
            const int* r0 = cl.map_shared_rank(rowptr, 0);
            for (int v = tid; v < 2 * (n + 1); v += nthr) rowptr[v] = r0[v];  // rowptr, colptr adjacent
        }
        cl.sync();
    }
    // dense supports (het trace: every positive g): node-major incidence
    // (column part then row part, i.e. ascending edge order) for a warp-per-
    // node SpMV with coalesced loads
    // Sparse supports whose node-major incidence fits the shared memory the
    // launch reserved (a.smem_nm entries) keep it there: the matvec then
    // reads no global memory (thread per node, same ascending edge order).
    const bool dense = a.nbr && 2 * ne >= 32 * n;
    const bool snm = !dense && 2 * ne <= a.smem_nm;
    int* nptr = cur;  // n+1 ints: reuses the counting-sort cursor
    double* snwt = reinterpret_cast<double*>(((uintptr_t)(cur + n + 1) + 15) & ~(uintptr_t)15);
    int* snbr = reinterpret_cast<int*>(snwt + a.smem_nm);
    int* nbr = snm ? snbr : (a.nbr ? a.nbr + (long long)b * 2 * a.list_cap : nullptr);
    double* nwt = snm ? snwt : (a.nwt ? a.nwt + (long long)b * 2 * a.list_cap : nullptr);
    if (dense || snm) {
        __syncthreads();
        if (tid == 0) nptr[0] = 0;
        for (int v = tid; v < n; v += nthr)
            nptr[v + 1] = (colptr[v + 1] - colptr[v]) + (rowptr[v + 1] - rowptr[v]);
        __syncthreads();
        if (tid == 0)
            for (int v = 0; v < n; ++v) nptr[v + 1] += nptr[v];
        __syncthreads();
        for (int v = tid; v < n; v += nthr) {
            int o = nptr[v];
            for (int p = colptr[v]; p < colptr[v + 1]; ++p, ++o) {
                const int e = cidx[p];
                nbr[o] = ei[e];
                nwt[o] = ew[e];
            }
            for (int e = rowptr[v]; e < rowptr[v + 1]; ++e, ++o) {
                nbr[o] = ej[e];
                nwt[o] = ew[e];
            }
        }
        __syncthreads();
    }

#ifdef OZ_STAMPS
    const long long tk0 = clock64();
#endif
    const bool warm = a.ritz && a.ritz_ok && a.ritz_ok[b];
    double* rz = a.ritz ? a.ritz + (long long)b * 2 * n : nullptr;
    for (int v = tid; v < n; v += nthr) q[v] = warm ? rz[v] + rz[n + v] : hash_unit(v);
    __syncthreads();
    deflate_normalize(q, n, scratch);

    double th_min = 1e300, th_max = -1e300;
    int steps = 0, converged = 0, kk = 0;
    for (int cycle = 0; cycle <= a.max_restarts; ++cycle) {
        if (tid == 0) s_flag = 0;
        for (int v = v_lo + tid; v < v_hi; v += nthr) qp[v] = 0.0;
        double beta_prev = 0.0;
        double c_min = 0.0, c_max = 0.0;
        bool broke = false;
        // residual tests: the first after min_steps (rounded up to a multiple
        // of check_every), then where the residual's decay rate since the
        // previous test predicts convergence (at least 8, at most
        // check_every steps ahead); identical in every thread
        const int every = a.check_every > 0 ? a.check_every : 16;
        int next_check = ((max(a.min_steps - steps, 1) + every - 1) / every) * every;
        int prev_k = 0;
        double prev_r = 0.0;
        __syncthreads();
        for (int k = 0; k < kcap; ++k) {
            // w = L q - beta_{k-1} q_{k-1} (gather, ascending edge order); alpha = q.w
            double pa = 0.0;
            if (dense) {
                // warp per node over the node-major incidence (coalesced), fixed
                // lane/tree order: deterministic
                // The first 8 entries of each lane are loaded before any is
                // used (same summation order): the L2 latency of the
                // incidence overlaps instead of serialising per entry.
                const int lane = tid & 31, nw = nthr >> 5;
                constexpr int NB = 8;
                for (int v = v_lo + wid; v < v_hi; v += nw) {
                    const double qv = q[v];
                    const int p0 = nptr[v] + lane, p1 = nptr[v + 1];
                    double wb[NB];
                    int jb[NB];
#pragma unroll
                    for (int u = 0; u < NB; ++u) {
                        const int p = p0 + 32 * u;
                        wb[u] = p < p1 ? nwt[p] : 0.0;  // written above in this kernel: no __ldg
                        jb[u] = p < p1 ? nbr[p] : v;
                    }
                    double acc = 0.0;
#pragma unroll
                    for (int u = 0; u < NB; ++u)
                        if (p0 + 32 * u < p1) acc += wb[u] * (qv - q[jb[u]]);
                    for (int p = p0 + 32 * NB; p < p1; p += 32) acc += nwt[p] * (qv - q[nbr[p]]);
                    acc = warp_sum(acc);
                    if (lane == 0) {
                        Q[(long long)k * n + v] = qv;
                        acc -= beta_prev * qp[v];
                        w[v] = acc;
                        pa += qv * acc;
                    }
                }
            } else if (snm) {
                // eight lanes per node over its incidence (consecutive
                // entries: no shared-memory bank conflicts; a thread per
                // node strode the node-major arrays by the degree), fixed
                // lane/tree order: deterministic
                constexpr int SG = 8;
                const int sub = tid / SG, sl = tid % SG, nsub = nthr / SG;
                for (int v0 = v_lo; v0 < v_hi; v0 += nsub) {
                    const int v = v0 + sub;
                    double acc = 0.0, qv = 0.0;
                    if (v < v_hi) {
                        qv = q[v];
                        for (int p = nptr[v] + sl; p < nptr[v + 1]; p += SG) acc += nwt[p] * (qv - q[nbr[p]]);
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                    if (sl == 0 && v < v_hi) {
                        Q[(long long)k * n + v] = qv;
                        acc -= beta_prev * qp[v];
                        w[v] = acc;
                        pa += qv * acc;
                    }
                }
            } else {
                // the same eight-lane split and entry order as the shared-
                // memory incidence above (column part, then row part), so a
                // batch gives the single solve's values bit for bit
                constexpr int SG = 8;
                const int sub = tid / SG, sl = tid % SG, nsub = nthr / SG;
                for (int v0 = v_lo; v0 < v_hi; v0 += nsub) {
                    const int v = v0 + sub;
                    double acc = 0.0, qv = 0.0;
                    if (v < v_hi) {
                        qv = q[v];
                        const int c0 = colptr[v], nc = colptr[v + 1] - c0, r0 = rowptr[v];
                        const int deg = nc + rowptr[v + 1] - r0;
                        for (int t = sl; t < deg; t += SG) {
                            if (t < nc) {
                                const int e = cidx[c0 + t];
                                acc += ew[e] * (qv - q[ei[e]]);
                            } else {
                                const int e = r0 + t - nc;
                                acc += ew[e] * (qv - q[ej[e]]);
                            }
                        }
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                    if (sl == 0 && v < v_hi) {
                        Q[(long long)k * n + v] = qv;
                        acc -= beta_prev * qp[v];
                        w[v] = acc;
                        pa += qv * acc;
                    }
                }
            }
            // this CTA's slice of w goes to the other CTAs before the alpha
            // reduction, whose cluster barrier orders it: ONE cluster barrier
            // per step. Receive buffers alternate with the step parity (w on
            // even steps, the foreign part of qp, unused otherwise, on odd
            // ones), so a CTA one step ahead never overwrites entries another
            // CTA still reads.
            double* wsrc = (C > 1 && (k & 1)) ? qp : w;
            double alpha = allreduce1(pa, red1);  // its CTA barrier: the slice is complete
            if (C > 1)
                for (int v = v_lo + tid; v < v_hi; v += nthr) {
                    const double wv = w[v];
                    for (int r = 0; r < C; ++r)
                        if (r != rank) *cl.map_shared_rank(wsrc + v, r) = wv;
                }
            {
                double dummy = 0.0;
                cluster_sum2(alpha, dummy, k & 1);
            }
            // every CTA now holds the whole w: x = w - alpha q over all nodes
            // (kept implicit), its sums in block order, identical in every CTA
            auto w_at = [&](int v) { return (v >= v_lo && v < v_hi) ? w[v] : wsrc[v]; };
            double s = 0.0, s2 = 0.0;
            for (int v = tid; v < n; v += nthr) {
                const double x = w_at(v) - alpha * q[v];
                s += x;
                s2 += x * x;
            }
            allreduce2(s, s2, red2);
            const double mean = s / n;
            const double beta = sqrt(fmax(s2 - n * mean * mean, 0.0));
            if (tid == 0) {
                al[k] = alpha;
                be[k] = beta;
            }
            kk = k + 1;
            ++steps;
            const bool breakdown = !(beta > 1e-13 * fmax(fabs(alpha), fabs(c_max)) + 1e-300);
            // residual tests (two Sturm multisections + two inverse iterations
            // on T_k, ~100 us at k = 256) only every check_every steps: a
            // matvec costs ~1 us, a test up to 100x more
            const bool want_check = breakdown || kk == kcap || kk >= next_check;
#ifdef OZ_STAMPS
            const long long tck = clock64();
#endif
            if (want_check) {
                __syncthreads();
                // warp 0: smallest Ritz pair, warp 1: largest, concurrently
                if (wid < 2) {
                    double lo, hi;
#ifdef OZ_STAMPS
                    const long long c0 = clock64();
#endif
                    gershgorin(al, be, kk, lo, hi);
#ifdef OZ_STAMPS
                    const long long c1 = clock64();
#endif
                    const double t = tri_eig(al, be, kk, wid == 0 ? 0 : kk - 1, lo, hi);
#ifdef OZ_STAMPS
                    const long long c2 = clock64();
#endif
                    if ((tid & 31) == 0) {
                        s_th[wid] = t;
                        s_res[wid] = beta * tri_vec(al, be, kk, t, wk + 2 * kcap * wid, wid == 0 ? smin : smax);
                    }
#ifdef OZ_STAMPS
                    if (tid == 0 && rank == 0) {
                        const int o = a.out ? 11 : 8;
                        atomicAdd(&g_slem_stats[o], (unsigned long long)(c1 - c0));
                        atomicAdd(&g_slem_stats[o + 1], (unsigned long long)(c2 - c1));
                        atomicAdd(&g_slem_stats[o + 2], (unsigned long long)(clock64() - c2));
                        atomicAdd(&g_slem_stats[a.out ? 15 : 14], 1ull);  // checks
                    }
#endif
                }
                __syncthreads();
                if (tid == 0) {
                    const double sc = fmax(fabs(s_th[1]), 1e-300);
                    const bool conv = !breakdown && s_res[0] <= a.tol * sc && s_res[1] <= a.tol * sc;
                    s_flag = (conv || breakdown || kk == kcap) ? (1 | (conv ? 2 : 0) | (breakdown ? 4 : 0)) : 0;
                }
                __syncthreads();
                c_min = s_th[0];
                c_max = s_th[1];
                {
                    const double r = fmax(s_res[0], s_res[1]) / fmax(fabs(s_th[1]), 1e-300);
                    int ahead = every;
                    if (prev_k > 0 && r < prev_r && r > 0.0) {
                        const double rate = log(r / prev_r) / (kk - prev_k);  // < 0
                        const double need = log(a.tol / r) / rate;
                        ahead = (int)fmin((double)every, fmax(8.0, ceil(1.1 * need)));
                    }
                    prev_k = kk;
                    prev_r = r;
                    next_check = kk + ahead;
                }
                SLEM_CLK(a.out ? 5 : 4, tck);
                if (s_flag & 1) {
                    converged = (s_flag >> 1) & 1;
                    broke = (s_flag >> 2) & 1;
                    break;
                }
            }
            const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
            for (int v = tid; v < n; v += nthr) {
                const double qo = q[v];
                if (v >= v_lo && v < v_hi) qp[v] = qo;  // q_{k-1} of this CTA's nodes
                q[v] = (w_at(v) - alpha * qo - mean) * inv;
            }
            beta_prev = beta;
            __syncthreads();
        }
        th_min = fmin(th_min, c_min);
        th_max = fmax(th_max, c_max);
        // Ritz vectors y = Q s of both extremes (restart vector / next warm
        // start), this CTA's nodes
        for (int v = v_lo + tid; v < v_hi; v += nthr) {
            double y1 = 0.0, y2 = 0.0;
            for (int j = 0; j < kk; ++j) {
                const double qj = Q[(long long)j * n + v];
                y1 += smin[j] * qj;
                y2 += smax[j] * qj;
            }
            w[v] = y1;
            q[v] = y2;
        }
        __syncthreads();
        if (rz && !broke) {
            for (int v = v_lo + tid; v < v_hi; v += nthr) {
                rz[v] = w[v];
                rz[n + v] = q[v];
            }
        }
        if (converged) break;
        // restart from the Ritz pair (a fresh random direction after a
        // breakdown); the whole vector in every CTA of the cluster
        for (int v = v_lo + tid; v < v_hi; v += nthr) {
            const double qn = broke ? hash_unit(v * 7 + 13 * cycle + 1) : q[v] + w[v];
            q[v] = qn;
            for (int r = 0; r < C; ++r)
                if (r != rank) *cl.map_shared_rank(q + v, r) = qn;
        }
        csync();
        deflate_normalize(q, n, scratch);
    }
    if (tid == 0 && rank == 0) {
        if (a.ritz_ok) a.ritz_ok[b] = 1;
        const double l2 = 1.0 - th_min, ln = 1.0 - th_max;
        const double acf = fmax(fabs(l2), fabs(ln));
        if (a.tr_acf) a.tr_acf[(long long)b * a.max_iter + it_rec] = acf;
        SLEM_CLK(a.out ? 7 : 6, tk0);
        SLEM_STAT(a.out != nullptr, steps);
        if (a.out) {
            double* o = a.out + b * 8;
            o[0] = acf;
            o[1] = l2;
            o[2] = ln;
            o[3] = (l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
            o[4] = steps;
            o[5] = converged;
        }
    }
}

size_t slem_trace_smem_bytes(int n, int kmax) {
    const int kcap = std::max(2, std::min(kmax, n - 1));
    return (3 * (size_t)n + 8 * (size_t)kcap) * sizeof(double) + (3 * (size_t)n + 3) * sizeof(int);
}

int slem_oneoff_kmax(int n) {
    int dev = 0, optin = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int k = std::max(2, std::min(n - 1, kOneOffKrylov));
    while (k > 64 && slem_trace_smem_bytes(n, k) + 2048 > (size_t)optin) k -= 64;
    return k;
}

void launch_slem(const SlemArgs& a, int B, cudaStream_t st) {
    const int n = a.n;
    if (n <= kSmallDense) {
        const size_t smem = ((size_t)n * (n + 1) + 4 * (size_t)n) * sizeof(double);
        slem_small_kernel<<<B, 256, smem, st>>>(a);
        TPB_CHECK_LAUNCH();
        return;
    }
    if (a.plain) {
        // (batched het solves keep n-sized CTAs: several fit an SM between the
        // concurrent GEMM waves, measured faster for the config-5 sweep than
        // one 1024-thread CTA per SM)
        const int threads = std::min(kTraceThreads, std::max(128, ((n + 31) / 32) * 32));
        // single solves: the node-major incidence of up to list_cap edges in
        // shared memory when it fits (batches keep the small CTAs)
        size_t smem = slem_trace_smem_bytes(n, a.kmax);
        SlemArgs b = a;
        b.smem_nm = 0;
        const size_t nm = 2 * (size_t)a.list_cap;
        static int optin = 0;
        if (!optin) {
            int dev = 0;
            TPB_CUDA(cudaGetDevice(&dev));
            TPB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        }
        const size_t extra = 16 + nm * (sizeof(double) + sizeof(int));
        if (B == 1 && smem + extra + 2048 <= (size_t)optin) {
            b.smem_nm = (int)nm;
            smem += extra;
        }
        const int C = std::max(1, std::min(a.cluster, 8));
        if (C == 1) {
            slem_trace_kernel<<<B, threads, smem, st>>>(b);
            TPB_CHECK_LAUNCH();
            return;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(B * C);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        TPB_CUDA(cudaLaunchKernelEx(&cfg, slem_trace_kernel, b));
        return;
    }
    const size_t smem = slem_smem_bytes(n, a.kmax, a.basis == nullptr);
    // one thread per node up to 512; small graphs use fewer warps (cheaper barriers)
    const int threads = std::min(kThreads, std::max(128, ((n + 31) / 32) * 32));
    slem_kernel<<<B, threads, smem, st>>>(a);
    TPB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- dense
// Full-spectrum Lanczos with CGS2 reorthogonalisation to k = n (exact up to
// rounding), then lambda2 = second largest and lambda_n = smallest Ritz value.
__global__ void __launch_bounds__(kThreads) slem_dense_kernel(const double* W, int n, double* basis,
                                                             double* out, int deflate) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int kmax = deflate ? max(1, n - 1) : n;
    extern __shared__ double sh[];
    double* q = sh;
    double* w = q + n;
    double* al = w + n;
    double* be = al + kmax;
    double* cf = be + kmax;
    __shared__ double scratch[32];
    __shared__ int s_stop;
    for (int v = tid; v < n; v += kThreads) q[v] = hash_unit(v) + (deflate ? 0.0 : 1.0);
    __syncthreads();
    if (deflate) {
        deflate_normalize(q, n, scratch);
    } else {
        double nn = 0.0;
        for (int v = tid; v < n; v += kThreads) nn += q[v] * q[v];
        nn = block_sum(nn, scratch);
        for (int v = tid; v < n; v += kThreads) q[v] /= sqrt(nn);
        __syncthreads();
    }
    if (tid == 0) s_stop = 0;
    __syncthreads();
    int kk = 0;
    for (int k = 0; k < kmax; ++k) {
        for (int v = tid; v < n; v += kThreads) basis[(long long)k * n + v] = q[v];
        for (int r = wid; r < n; r += kThreads / 32) {  // w = W q, one warp per row
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
        if (deflate) {  // last, so reorthogonalisation round-off is not amplified
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
    if (wid == 0) {
        double lo, hi;
        gershgorin(al, be, kk, lo, hi);
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
        if (lane == 0) {
            out[0] = n == 1 ? 0.0 : fmax(fabs(l2), fabs(lminall));
            out[1] = n == 1 ? 0.0 : l2;
            out[2] = lminall;
            out[3] = (n == 1 || l2 < 1.0 - 1e-8) ? 1.0 : 0.0;
        }
    }
}

void launch_slem_dense(const double* w, int n, double* basis, double* out, int deflate, cudaStream_t st) {
    const int kmax = deflate ? std::max(1, n - 1) : n;
    const size_t smem = (2 * (size_t)n + 3 * (size_t)kmax) * sizeof(double);
    slem_dense_kernel<<<1, kThreads, smem, st>>>(w, n, basis, out, deflate);
    TPB_CHECK_LAUNCH();
}

void init_attrs_slem() {
    set_max_dyn_smem(slem_kernel);
    set_max_dyn_smem(slem_trace_kernel);
    set_max_dyn_smem(slem_dense_kernel);
    set_max_dyn_smem(slem_small_kernel);
}

}  // namespace tpb
