// Consensus simulation (proj/src/consensus.cpp:29-67, §8f row 2): the error
// trace of x <- W x from i.i.d. normal starts, recentred every step. The
// start state comes from the reference's own random stream (std::mt19937_64 +
// Box-Muller with the cached spare, proj/include/topoopt/rng.hpp:31-47) on
// the host; the iterations run on the device with the reference's
// arithmetic order — W's nonzeros of a row in ascending column order, plain
// multiply then add from 0.0 (the reference's i-k-j matmul skipping zeros),
// the per-coordinate mean as a sequential sum over rows — so the state
// evolves bit for bit. Only the Frobenius norm of each step is a
// deterministic tree reduction instead of the reference's sequential sum.
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "../../include/topoopt_b200.h"
#include "common.cuh"

namespace tpb {

namespace {

constexpr int kThreads = 1024;

// One CTA iterates the whole trace (n x dim state, L2-resident).
__global__ void __launch_bounds__(kThreads) consensus_kernel(int n, int dim, int iters, const int* rowptr,
                                                             const int* col, const double* val, double* s,
                                                             double* t, double* errors) {
    extern __shared__ double mean[];  // dim
    __shared__ double scratch[32];
    const long long total = (long long)n * dim;
    for (int it = 0; it < iters; ++it) {
        for (long long idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int i = (int)(idx / dim), d = (int)(idx % dim);
            double acc = 0.0;
            for (int p = rowptr[i]; p < rowptr[i + 1]; ++p)
                acc = __dadd_rn(acc, __dmul_rn(val[p], s[(long long)col[p] * dim + d]));
            t[idx] = acc;
        }
        __syncthreads();
        for (int d = threadIdx.x; d < dim; d += blockDim.x) {
            double m = 0.0;
            for (int i = 0; i < n; ++i) m = __dadd_rn(m, t[(long long)i * dim + d]);
            mean[d] = __ddiv_rn(m, (double)n);
        }
        __syncthreads();
        double ss = 0.0;
        for (long long idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const double v = __dadd_rn(t[idx], -mean[idx % dim]);
            t[idx] = v;
            ss += v * v;
        }
        ss = block_sum(ss, scratch);
        if (threadIdx.x == 0) errors[it + 1] = sqrt(ss);
        double* tmp = s;
        s = t;
        t = tmp;
        __syncthreads();
    }
}

// The reference's Rng::normal() stream (host; identical libm calls).
struct HostRng {
    std::mt19937_64 eng;
    double spare = 0.0;
    bool have = false;
    explicit HostRng(uint64_t seed) : eng(seed) {}
    double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have) {
            have = false;
            return spare;
        }
        double u1;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        const double u2 = uniform();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 6.283185307179586476925286766559 * u2;
        spare = radius * std::sin(angle);
        have = true;
        return radius * std::cos(angle);
    }
};

void validate_gossip(int n, const double* w) {
    // proj/src/topology.cpp:148-164
    if (n < 1) throw Error(kInvalidArgument, "gossip matrix must be square");
    for (int i = 0; i < n; ++i) {
        double row_sum = 0.0;
        for (int j = 0; j < n; ++j) {
            const double a = w[(long long)i * n + j], b = w[(long long)j * n + i];
            if (std::abs(a - b) > 1e-8) throw Error(kInvalidArgument, "gossip matrix asymmetric beyond 1e-8");
            if (a < -1e-8) throw Error(kInvalidArgument, "gossip matrix has an entry below -1e-8");
            row_sum += a;
        }
        if (std::abs(row_sum - 1.0) > 1e-8)
            throw Error(kInvalidArgument, "gossip matrix row " + std::to_string(i) + " does not sum to 1");
    }
}

template <typename T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { TPB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Dev() { cudaFree(p); }
    void up(const T* h, size_t n) { h2d(p, h, n * sizeof(T)); }
};

}  // namespace

void consensus_simulate(int n, const double* w, int dim, int iters, uint64_t seed, double* errors) {
    validate_gossip(n, w);
    if (dim < 1) throw Error(kInvalidArgument, "simulate: dim must be >= 1");
    if (iters < 0) throw Error(kInvalidArgument, "simulate: iters must be >= 0");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw Error(kCuda, "no CUDA device: the B200 solver has no CPU fallback");
    // start state exactly as the reference: row-major normals, recentred
    HostRng rng(seed);
    const size_t total = (size_t)n * dim;
    std::vector<double> s(total);
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < dim; ++d) s[(size_t)i * dim + d] = rng.normal();
    for (int d = 0; d < dim; ++d) {
        double mean = 0.0;
        for (int i = 0; i < n; ++i) mean += s[(size_t)i * dim + d];
        mean /= n;
        for (int i = 0; i < n; ++i) s[(size_t)i * dim + d] -= mean;
    }
    double f = 0.0;
    for (double v : s) f += v * v;
    errors[0] = std::sqrt(f);
    if (iters == 0) return;
    // W's nonzeros per row, ascending columns (the matmul's k order)
    std::vector<int> rowptr(n + 1, 0), col;
    std::vector<double> val;
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < n; ++k) {
            const double a = w[(long long)i * n + k];
            if (a == 0.0) continue;
            col.push_back(k);
            val.push_back(a);
        }
        rowptr[i + 1] = (int)col.size();
    }
    Dev<int> d_row(n + 1), d_col(col.size());
    Dev<double> d_val(val.size()), d_s(total), d_t(total), d_err(iters + 1);
    d_row.up(rowptr.data(), n + 1);
    d_col.up(col.data(), col.size());
    d_val.up(val.data(), val.size());
    d_s.up(s.data(), total);
    consensus_kernel<<<1, kThreads, (size_t)dim * sizeof(double)>>>(n, dim, iters, d_row.p, d_col.p, d_val.p,
                                                                     d_s.p, d_t.p, d_err.p);
    TPB_CHECK_LAUNCH();
    TPB_CUDA(cudaMemcpy(errors + 1, d_err.p + 1, (size_t)iters * sizeof(double), cudaMemcpyDeviceToHost));
}

}  // namespace tpb

extern "C" int tp_consensus_simulate(int32_t n, const double* w, int32_t dim, int32_t iters, uint64_t seed,
                                     double* errors) {
    try {
        if (!w || !errors) throw tpb::Error(tpb::kInvalidArgument, "simulate: null buffer");
        tpb::consensus_simulate(n, w, dim, iters, seed, errors);
        return TP_OK;
    } catch (const tpb::Error& e) {
        tpb::last_error_ref() = e.what();
        return e.status;
    } catch (const std::exception& e) {
        tpb::last_error_ref() = e.what();
        return TP_ERR_INTERNAL;
    }
}
