#pragma once

#include "common.cuh"

namespace tpb {

// Polynomial sign iteration for the PSD/NSD cone projections.
//   X0 = A / ||A||_F
//   K1 quintic steps  X <- a X + b X^3 + c X^5      (inflate small |mu|)
//   K2 Newton-Schulz  X <- 1.5 X - 0.5 X^3          (converge to sign)
//   P_psd(A) = (A + A X)/2,  P_nsd(A) = (A - A X)/2
// k1 = 22: worst relative error 6e-14 of ||A||_F on 16-decade clustered
// spectra (tools/proto/sign_schedule.py); 24 gives 6e-15 at +6 GEMMs.
struct SignSchedule {
    int k1 = 22, k2 = 6;
    double qa = 3.4445, qb = -4.7750, qc = 2.0315;
    int gemms() const { return 3 * k1 + 2 * k2 + 1; }
};

// Schedule of the tiled Ozaki path: the inflation quintic with the largest
// guaranteed growth on [0, 0.55] that keeps [0.55, 1.3] invariant (an LP over
// the coefficients, tools/proto/sign_schedule.py), 20 steps + 6 Newton-Schulz
// = 73 products instead of 79. Scalar-map error max_mu mu |1 - s(mu)| / 2 =
// 4.4e-14 of ||A||_F (1.8e-14 for the default above). Digit bounds: |X| <=
// 1.3, |U| <= 1.26, |Z'| <= 3.73, |V| <= 1.5 (exponents unchanged).
// TPB_SIGN_SCHEDULE=default selects the default above.
SignSchedule ozaki_schedule();

// One symmetric GEMM step over a batch of matrices (blockIdx.y = matrix):
//   C = alpha * (A . B) + beta * E,   alpha = alpha_c * s^pa, beta = beta_c * s^pb
// with s = scale[mat]; A, B, E symmetric ld x ld (row-major, zero padded),
// C symmetric: lower 64x64 tiles computed, mirrored on store.
struct GemmArgs {
    const double* A;
    const double* B;
    const double* E;
    long long mstride;      // elements between matrices for A, B, E
    double* C;
    long long c_stride_b;   // C base of matrix (b, w) = C + b*c_stride_b + w*c_stride_w
    long long c_stride_w;
    int ldc;
    int nvalid;             // rows/cols of C to store (n for the state, ld for work)
    int ld;
    double alpha_c, beta_c;
    int pa, pb;
    const double* scale;    // per matrix (1/||A||_F)
    const int* ictl;        // done flags per solve (matrix/2), or null
    double sign_b;          // +1 psd-style / -1: multiplies alpha for odd matrices (w = 1)
    int sign_mode;          // 1: alpha *= (w == 0 ? -1 : +1)  (S -> NSD, T -> PSD)
    // stream-K workspace for single-pair launches (null: tiled kernel only)
    double* sk_ws;          // stream_k_ctas(ld) x 64 x 64 doubles
    int* sk_flags;          // 2 x tiles ints, zero-initialised
};

void launch_sym_gemm(const GemmArgs& g, int nmat, cudaStream_t st);
int sm_count();  // multiprocessors of the current device (cached)
// CTAs of the stream-K decomposition for one (S, T) pair of order ld (0: not used)
int stream_k_ctas(int ld);
// tile/pipeline variants of the DMMA GEMM (for tuning; 0 = production)
int sym_gemm_variants();
void set_sym_gemm_variant(int v);
int get_sym_gemm_variant();

// Fused small-n projection: one CTA per matrix, whole iteration in shared
// memory (npad <= 64). A at A + mat*mstride (ld-padded, symmetric); output to
// C + b*c_stride_b + w*c_stride_w (column-major n x n). S (w=0) -> NSD,
// T (w=1) -> PSD.
void launch_cone_small(const double* A, long long mstride, int ld, int n, double* C,
                       long long c_stride_b, long long c_stride_w, const int* ictl, int nmat,
                       const SignSchedule& sch, cudaStream_t st);

// Host driver for the tiled path: enqueue the full schedule on `st`.
// bufs: 3 work buffers (each nmat * ld * ld).
void enqueue_cone_tiled(const double* A, double* w0, double* w1, double* w2, int ld, int n,
                        const double* scale, double* C, long long c_stride_b,
                        long long c_stride_w, const int* ictl, int nmat, const SignSchedule& sch,
                        cudaStream_t st, double* sk_ws = nullptr, int* sk_flags = nullptr);

}  // namespace tpb
