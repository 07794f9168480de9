// PSD / NSD cone projections of small slack blocks (n <= 64) on the FP64
// tensor pipe (DMMA, mma.sync.m8n8k4.f64): one CTA per matrix keeps the whole
// sign iteration (cone_kernels.cuh) in shared memory. Replaces the
// reference's per-iteration eigen-clamps project_nsd(S) / project_psd(T)
// (proj/src/admm.cpp:96-112 -> clamp_spectrum, proj/src/eig.cpp:131-176).
// Larger blocks take the tiled tcgen05 path (ozaki_kernels.cu). Every product
// is of commuting symmetric matrices, so only lower 8x8 fragments are
// computed and mirrored (exact symmetry, as the reference's symmetrize()).
#include "cone_kernels.cuh"

#include <algorithm>
#include <cstdlib>

namespace tpb {

namespace {

__device__ inline void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

}  // namespace

int sm_count() {
    static int cached[64] = {};
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) dev = 63;
    if (!cached[dev]) TPB_CUDA(cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev));
    return cached[dev];
}

// ---------------------------------------------------------------- small n
// One CTA per matrix; all iterates in shared memory (npad <= 64).
namespace {
constexpr int ST = 512;  // 16 warps
}

__global__ void __launch_bounds__(ST) cone_small_kernel(const double* Ag, long long mstride, int ld, int n,
                                                       double* Cg, long long c_stride_b,
                                                       long long c_stride_w, const int* ictl,
                                                       SignSchedule sch) {
    const int mat = blockIdx.x;
    if (ictl && ictl[(mat >> 1) * 8 + 1]) return;
    const int np = (n + 7) & ~7;
    const int P = np + 4;  // padded stride
    extern __shared__ __align__(16) double sm[];
    double* A = sm;
    double* X = A + np * P;
    double* Y = X + np * P;
    double* Z = Y + np * P;
    double* T = Z + np * P;
    __shared__ double scratch[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* src = Ag + (long long)mat * mstride;
    double fro = 0.0;
    for (int idx = tid; idx < np * np; idx += ST) {
        const int r = idx / np, c = idx % np;
        const double v = (r < n && c < n) ? src[(long long)r * ld + c] : 0.0;
        A[r * P + c] = v;
        fro += v * v;
    }
    fro = block_sum(fro, scratch);
    const double s = fro > 0.0 ? 1.0 / sqrt(fro) : 0.0;
    const int nf = np / 8;
    const int nfr = nf * (nf + 1) / 2;  // lower 8x8 fragments

    // dst = alpha * (a . b) + beta * e ; lower frags computed, mirrored
    auto gemm = [&](const double* a, const double* b, const double* e, double* dst, double alpha,
                    double beta) {
        for (int f = warp; f < nfr; f += ST / 32) {
            int fi = (int)((sqrt(8.0 * f + 1.0) - 1.0) * 0.5);
            while ((fi + 1) * (fi + 2) / 2 <= f) ++fi;
            while (fi * (fi + 1) / 2 > f) --fi;
            const int fj = f - fi * (fi + 1) / 2;
            // four independent accumulator pairs over k (the DMMA chain is
            // latency-bound), added pairwise at the end
            const double* ar = a + (fi * 8 + (lane >> 2)) * P + (lane & 3);
            const double* br = b + (fj * 8 + (lane >> 2)) * P + (lane & 3);
            double e0[4] = {0.0, 0.0, 0.0, 0.0}, e1[4] = {0.0, 0.0, 0.0, 0.0};
            int k = 0;
            for (; k + 16 <= np; k += 16) {
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma(e0[q], e1[q], ar[k + 4 * q], br[k + 4 * q]);
            }
            if (k < np) {  // np % 16 == 8: two more k steps
                dmma(e0[0], e1[0], ar[k], br[k]);
                dmma(e0[1], e1[1], ar[k + 4], br[k + 4]);
            }
            const double d0 = (e0[0] + e0[1]) + (e0[2] + e0[3]);
            const double d1 = (e1[0] + e1[1]) + (e1[2] + e1[3]);
            const int r = fi * 8 + (lane >> 2);
            const int c = fj * 8 + (lane & 3) * 2;
            double v0 = alpha * d0, v1 = alpha * d1;
            if (e) {
                v0 += beta * e[r * P + c];
                v1 += beta * e[r * P + c + 1];
            }
            if (fi == fj) {
                // keep lower entries (c <= r) and mirror them
                if (c <= r) {
                    dst[r * P + c] = v0;
                    dst[c * P + r] = v0;
                }
                if (c + 1 <= r) {
                    dst[r * P + c + 1] = v1;
                    dst[(c + 1) * P + r] = v1;
                }
            } else {
                dst[r * P + c] = v0;
                dst[c * P + r] = v0;
                dst[r * P + c + 1] = v1;
                dst[(c + 1) * P + r] = v1;
            }
        }
        __syncthreads();
    };

    // first quintic step from X0 = s A (scale folded into the coefficients)
    const double* Xc = A;
    double xs = s;  // pending scale of Xc
    double* bufs[4] = {X, Y, Z, T};
    auto free3 = [&](double*& f0, double*& f1, double*& f2) {
        double* fr[4];
        int k = 0;
        for (int q = 0; q < 4; ++q)
            if (bufs[q] != Xc) fr[k++] = bufs[q];
        f0 = fr[0];
        f1 = fr[1];
        f2 = fr[2];
    };
    for (int it = 0; it < sch.k1; ++it) {
        double *Yb, *Zb, *Xn;
        free3(Yb, Zb, Xn);
        gemm(Xc, Xc, nullptr, Yb, xs * xs, 0.0);
        gemm(Yb, Yb, Yb, Zb, sch.qc, sch.qb);
        gemm(Xc, Zb, Xc, Xn, xs, sch.qa * xs);
        xs = 1.0;
        Xc = Xn;
    }
    for (int it = 0; it < sch.k2; ++it) {
        double *Yb, *Xn, *unused;
        free3(Yb, Xn, unused);
        gemm(Xc, Xc, nullptr, Yb, xs * xs, 0.0);
        gemm(Xc, Yb, Xc, Xn, -0.5 * xs, 1.5 * xs);
        xs = 1.0;
        Xc = Xn;
    }
    // P = 0.5 A -/+ 0.5 A X
    double *out, *u1, *u2;
    free3(out, u1, u2);
    const double sg = (mat & 1) == 0 ? -0.5 : 0.5;  // S -> NSD, T -> PSD
    gemm(A, Xc, A, out, sg * xs, 0.5);
    double* C = Cg + (long long)(mat >> 1) * c_stride_b + (long long)(mat & 1) * c_stride_w;
    for (int idx = tid; idx < n * n; idx += ST) {
        const int r = idx / n, c = idx % n;
        C[(long long)c * n + r] = out[r * P + c];
    }
}

void launch_cone_small(const double* A, long long mstride, int ld, int n, double* C,
                       long long c_stride_b, long long c_stride_w, const int* ictl, int nmat,
                       const SignSchedule& sch, cudaStream_t st) {
    const int np = (n + 7) & ~7;
    const int smem = 5 * np * (np + 4) * sizeof(double);
    cone_small_kernel<<<nmat, ST, smem, st>>>(A, mstride, ld, n, C, c_stride_b, c_stride_w, ictl, sch);
    TPB_CHECK_LAUNCH();
}

void init_attrs_cone() {
    set_max_dyn_smem(cone_small_kernel);
}

}  // namespace tpb
