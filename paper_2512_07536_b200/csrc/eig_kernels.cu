// Symmetric eigendecomposition on the GPU for the API's sym_eig
// (proj/include/topoopt/eig.hpp:17-22; the reference uses Householder + QL,
// proj/src/eig.cpp:18-129). The solver's own cone projections do not need
// eigenvectors (tcgen05 sign iteration, ozaki_kernels.cu); this serves
// callers of the reference API.
//
// One-sided (Hestenes) Jacobi on B = sym(A) + sigma I, sigma >= the spectral
// radius (min of the Frobenius and infinity norms), so B is PSD and its
// singular vectors are its eigenvectors: column pairs (p, q) of U = B V are
// rotated until orthogonal (round-robin ordering, n/2 independent pairs per
// step, one CTA per pair, grid-wide barrier between steps), then
// lambda_i = |u_i| - sigma with eigenvector v_i. Every reduction has a fixed
// order, so results are reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "eig_kernels.cuh"

namespace cg = cooperative_groups;

namespace tpb {

namespace {

constexpr int kThreads = 256;

// position k of the circle method (n2 even): index 0 fixed, the others rotate
__device__ __forceinline__ int rr_member(int pos, int step, int n2) {
    if (pos == 0) return 0;
    return 1 + (pos - 1 + step) % (n2 - 1);
}

}  // namespace

// U, V: column-major n x n (column c at c * n). One sweep = n2 - 1 steps.
__global__ void __launch_bounds__(kThreads) jacobi_sweep_kernel(double* U, double* V, int n, int n2, double tol,
                                                                int* rotations) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double scratch[4][32];
    const int npairs = n2 / 2;
    for (int step = 0; step < n2 - 1; ++step) {
        for (int k = blockIdx.x; k < npairs; k += gridDim.x) {
            int p = rr_member(k, step, n2), q = rr_member(n2 - 1 - k, step, n2);
            if (p > q) {
                const int t = p;
                p = q;
                q = t;
            }
            if (q >= n) continue;  // padding index of odd n
            double* up = U + (long long)p * n;
            double* uq = U + (long long)q * n;
            double a = 0.0, b = 0.0, g = 0.0;
            for (int i = threadIdx.x; i < n; i += kThreads) {
                const double x = up[i], y = uq[i];
                a += x * x;
                b += y * y;
                g += x * y;
            }
            double sums[4] = {a, b, g, 0.0};
            block_sum4(sums, scratch);
            a = sums[0];
            b = sums[1];
            g = sums[2];
            if (!(std::fabs(g) > tol * std::sqrt(a * b)) || g == 0.0) continue;
            const double zeta = (b - a) / (2.0 * g);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
            double* vp = V + (long long)p * n;
            double* vq = V + (long long)q * n;
            for (int i = threadIdx.x; i < n; i += kThreads) {
                const double x = up[i], y = uq[i];
                up[i] = c * x - s * y;
                uq[i] = s * x + c * y;
                const double vx = vp[i], vy = vq[i];
                vp[i] = c * vx - s * vy;
                vq[i] = s * vx + c * vy;
            }
            if (threadIdx.x == 0) atomicAdd(rotations, 1);
        }
        grid.sync();
    }
}

// |u_i| per column (fixed-order block reduction)
__global__ void __launch_bounds__(kThreads) column_norms_kernel(const double* U, int n, double* out) {
    __shared__ double scratch[32];
    const int c = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += kThreads) s += U[(long long)c * n + i] * U[(long long)c * n + i];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) out[c] = std::sqrt(s);
}

void sym_eig_device(int n, const double* a, double* values, double* vectors) {
    if (n < 1) throw Error(kInvalidArgument, "sym_eig: empty matrix");
    // symmetrize (proj/src/eig.cpp:157) and shift on the host: O(n^2)
    std::vector<double> B((size_t)n * n), Vh((size_t)n * n, 0.0);
    double fro = 0.0, inf = 0.0;
    for (int i = 0; i < n; ++i) {
        double row = 0.0;
        for (int j = 0; j < n; ++j) {
            const double v = 0.5 * (a[(size_t)i * n + j] + a[(size_t)j * n + i]);
            B[(size_t)j * n + i] = v;  // column-major (symmetric anyway)
            fro += v * v;
            row += std::fabs(v);
        }
        inf = std::max(inf, row);
    }
    const double sigma = std::min(std::sqrt(fro), inf);
    for (int i = 0; i < n; ++i) {
        B[(size_t)i * n + i] += sigma;
        Vh[(size_t)i * n + i] = 1.0;
    }
    double *dU = nullptr, *dV = nullptr, *dN = nullptr;
    int* dRot = nullptr;
    const size_t bytes = (size_t)n * n * sizeof(double);
    TPB_CUDA(cudaMalloc(&dU, bytes));
    TPB_CUDA(cudaMalloc(&dV, bytes));
    TPB_CUDA(cudaMalloc(&dN, (size_t)n * sizeof(double)));
    TPB_CUDA(cudaMalloc(&dRot, sizeof(int)));
    struct Free {
        void* p[4];
        ~Free() {
            for (void* q : p) cudaFree(q);
        }
    } guard{{dU, dV, dN, dRot}};
    h2d(dU, B.data(), bytes);
    h2d(dV, Vh.data(), bytes);
    const int n2 = n + (n & 1);
    if (n2 >= 2) {
        int dev = 0, sms = 0, per_sm = 0;
        TPB_CUDA(cudaGetDevice(&dev));
        TPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_sweep_kernel, kThreads, 0));
        const int grid = std::max(1, std::min(n2 / 2, sms * std::max(per_sm, 1)));
        double tol = std::max(1e-15, 2.2e-16 * std::sqrt((double)n));
        for (int sweep = 0; sweep < 80; ++sweep) {
            TPB_CUDA(cudaMemset(dRot, 0, sizeof(int)));
            void* args[] = {&dU, &dV, (void*)&n, (void*)&n2, &tol, &dRot};
            TPB_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_sweep_kernel, dim3(grid), dim3(kThreads), args, 0,
                                                 0));
            int rot = 0;
            TPB_CUDA(cudaMemcpy(&rot, dRot, sizeof(int), cudaMemcpyDeviceToHost));
            if (rot == 0) break;
        }
    }
    column_norms_kernel<<<n, kThreads>>>(dU, n, dN);
    TPB_CHECK_LAUNCH();
    std::vector<double> norms(n);
    TPB_CUDA(cudaMemcpy(norms.data(), dN, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
    TPB_CUDA(cudaMemcpy(Vh.data(), dV, bytes, cudaMemcpyDeviceToHost));
    // ascending eigenvalues (stable on ties), vectors row-major: vectors[i n + k] = v_k[i]
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> lam(n);
    for (int k = 0; k < n; ++k) lam[k] = norms[k] - sigma;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return lam[x] < lam[y]; });
    for (int k = 0; k < n; ++k) {
        values[k] = lam[order[k]];
        for (int i = 0; i < n; ++i) vectors[(size_t)i * n + k] = Vh[(size_t)order[k] * n + i];
    }
}

}  // namespace tpb
