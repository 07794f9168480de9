// FP64 products of symmetric matrices on the int8 tensor cores (tcgen05
// kind::i8): Ozaki scheme I with fixed power-of-two operand scales.
//
//   M = 2^e sum_{s=1..KS} 2^{-7s} M_s,   M_s int8 "digit planes" in [-127, 127]
//   A.B ~= 2^{eA+eB} sum_{d=2..KS+1} 2^{-7d} G_d,   G_d = sum_{s+t=d} A_s . B_t
//
// KS = 7 digits (49 bits) and the KS(KS+1)/2 = 28 products with s + t <= KS+1:
// the dropped products and the operand truncation are both ~2^-49 of
// |A||B| per entry, the size of an FP64 GEMM's own accumulated rounding
// (K u ~ 1e-13 worst case at K = 1024). Every A_s . B_t is exact (int32
// accumulation in TMEM: |G_d| <= KS * K * 127^2 < 2^31 needs K <= 19020, so
// ld <= kOzMaxLd = 16384 is enforced); only the FP64 epilogue rounds. The
// scales are static bounds from the sign iteration, so a
// producer GEMM writes its consumer's digit planes in its own epilogue.
// Accuracy study: tools/proto/ozaki.py.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace tpb {

constexpr int kOzSlices = 7;     // digits per operand (49 bits)
constexpr int kOzBM = 128;       // tile rows (UMMA M)
constexpr int kOzBN = 64;        // tile columns
constexpr int kOzMaxLd = 16384;  // int32 accumulator bound (see above)
constexpr int kOzMaxRanks = 8;   // GPUs of one NVLink/NVSwitch domain sharing a projection

// Throws kInvalidArgument unless ld is a multiple of 128 in [128, kOzMaxLd].
void check_oz_ld(int ld);

// TMA maps of one digit-plane buffer: loads in the A role (64-byte k block x
// 128 rows) and in the B role (64-byte k block x 64 rows).
struct OzMaps {
    CUtensorMap a, b;
};
void make_oz_maps(const int8_t* planes, int ld, int nmat, OzMaps* out);

struct OzGemm {
    const OzMaps* ma;        // operand A planes (row block i0)
    const OzMaps* mb;        // operand B planes (row block j0 of B = column block of B^T)
    int eA, eB;
    int ld, nmat;
    double alpha_c, beta_c;  // C = alpha (A.B) + beta E, alpha = alpha_c s^pa, beta = beta_c s^pb
    int pa, pb;
    const double* scale;     // per matrix s, or null (s = 1)
    int sign_mode;           // alpha *= -1 for even matrices (S -> NSD)
    double dshift;           // added to the diagonal after alpha/beta
    const double* E;         // FP64 symmetric, mat stride ld*ld, or null
    double* C;               // FP64 out, or null
    long long c_stride_b, c_stride_w;
    int ldc, nvalid;
    int8_t* Cd;              // digit planes out ([mat][slice][ld][ld]), or null
    int eC;
    const int* ictl;         // done flags per solve (matrix / 2), or null
    int no_pdl;              // launch without programmatic dependent launch
    const int* tiles;        // row-sharded products: this rank's lower-tile indices, or null (all)
    int ntiles;              // entries of tiles
    int mstep;               // matrices of this launch: blockIdx.y * mstep + moff (mstep 0 -> 1)
    int moff;
    int rc;                  // plane layout: rows per chunk (0 -> ld; see OzShard)
    // sharded product over nranks GPUs (nranks > 1): the epilogue stores every
    // digit-plane tile into all ranks' output buffers over NVLink, and the
    // launch waits for / publishes per-rank product counters (OzShard)
    int nranks, rank;
    int8_t* peer_cd[kOzMaxRanks];                 // rank r's output digit buffer (slot rank: Cd)
    unsigned long long* flags;                    // local [kOzMaxRanks]: products completed by rank r
    unsigned long long* peer_flags[kOzMaxRanks];  // rank r's flag array
    int* done;                                    // local arrival counter of the launch's CTAs
    int* err;                                     // wait timeout (results invalid)
    unsigned long long epoch;                     // products every rank completed before this one
};

void launch_oz_gemm(const OzGemm& g, cudaStream_t st);
int oz_gemm_tiles(int ld);

// Digit-plane buffers of the cone projection: [0..2] hold the rotating
// iterates, [3] holds X0 = A / ||A||_F.
struct OzWork {
    int8_t* d[4] = {nullptr, nullptr, nullptr, nullptr};
    OzMaps maps[4];
};

// Sharded projection of one large instance over G ranks of one NVLink /
// NVSwitch domain. The lower tiles of every product are dealt
// round-robin to the ranks; each rank's GEMM epilogue stores its tiles'
// digit planes (direct and mirrored rows) into every rank's copy of the
// output buffer through peer pointers (CUDA IPC), so the all-gather is fused
// into the product: NVLink traffic overlaps the remaining tiles' math. Per
// product each rank's last CTA publishes its product counter into every
// peer's flag array (system-scope release), and the next product's CTAs wait
// until every peer has published (acquire) before reading operands; the same
// kernel computes every tile, so the iterate is bitwise the single-GPU one.
// NCCL is used once, to exchange the IPC handles.
struct OzShard {
    int rank = 0, nranks = 1;
    void* comm = nullptr;     // ncclComm_t (setup only)
    int* tiles = nullptr;     // device: this rank's tile indices
    int ntiles = 0;
    int8_t* peer_d[4][kOzMaxRanks] = {};          // every rank's digit buffer q
    unsigned long long* flags = nullptr;          // local flag array (peers write their slots)
    unsigned long long* peer_flags[kOzMaxRanks] = {};
    int* done = nullptr;
    int* err = nullptr;
    unsigned long long epoch = 0;                 // products launched so far (same on every rank)
};
// Host tile list of `rank`: the lower tiles t with t % nranks == rank.
std::vector<int> oz_shard_tiles(int ld, int nranks, int rank);

struct SignSchedule;
// The cone projections of nmat symmetric ld x ld inputs A (S at even, T at
// odd matrices): the sign iteration of cone_kernels.cuh with every product
// on the int8 tensor cores; P_nsd / P_psd written to C.
void enqueue_cone_ozaki(const double* A, const OzWork& oz, int ld, int n, const double* scale, double* C,
                        long long c_stride_b, long long c_stride_w, const int* ictl, int nmat,
                        const SignSchedule& sch, cudaStream_t st, OzShard* shard = nullptr);

// Digit planes of s * A (s = scale[mat] or 1) with exponent e (layout rc as in OzGemm).
void launch_oz_split(const double* A, long long mstride, int ld, int nmat, const double* scale,
                     int e, int8_t* planes, const int* ictl, cudaStream_t st, int rc = 0);

}  // namespace tpb
