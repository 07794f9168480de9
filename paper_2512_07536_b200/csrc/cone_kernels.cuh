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
// the coefficients, tools/proto/sign_schedule.py), 18 steps + 6 Newton-Schulz
// = 67 products. X0 = A / c with c = min(||A||_F, ||A||_inf) (both bound the
// spectral radius; prep_kernel tail): scalar-map error
// max_mu mu |1 - s(mu)| / 2 = 6.1e-13 of c <= 6.1e-13 ||A||_F (the slack
// blocks have c ~ ||A||_F / 5 at n = 1024, so ~1e-13 of ||A||_F there).
// Digit bounds: |X| <= 1.3, |U| <= 1.26, |Z'| <= 3.73, |V| <= 1.5.
SignSchedule ozaki_schedule();

int sm_count();  // multiprocessors of the current device (cached)

// Fused small-n projection: one CTA per matrix, whole iteration in shared
// memory (npad <= 64). A at A + mat*mstride (ld-padded, symmetric); output to
// C + b*c_stride_b + w*c_stride_w (column-major n x n). S (w=0) -> NSD,
// T (w=1) -> PSD.
void launch_cone_small(const double* A, long long mstride, int ld, int n, double* C,
                       long long c_stride_b, long long c_stride_w, const int* ictl, int nmat,
                       const SignSchedule& sch, cudaStream_t st);

}  // namespace tpb
