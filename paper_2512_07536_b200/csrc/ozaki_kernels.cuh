// FP64 products of symmetric matrices on the int8 tensor cores (tcgen05
// kind::i8): Ozaki scheme I with fixed power-of-two operand scales.
//
//   M = 2^e sum_{s=1..KS} 2^{-7s} M_s,   M_s int8 "digit planes" in [-127, 127]
//   A.B ~= 2^{eA+eB} sum_{d=2..KS+1} 2^{-7d} G_d,   G_d = sum_{s+t=d} A_s . B_t
//
// Every A_s . B_t is exact (int32 accumulation in TMEM, |G_d| < 2^31 for
// K <= 16384); only the FP64 epilogue rounds. The scales are static bounds
// from the sign iteration (|X| <= 1.21, |Y| <= 1.45,
// |Z| <= 2.81 in spectral norm, hence entrywise), so a producer GEMM writes
// its consumer's digit planes in its own epilogue. Accuracy study:
// tools/proto/ozaki.py.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace tpb {

constexpr int kOzSlices = 8;   // digits per operand (56 bits)
constexpr int kOzBM = 128;     // tile rows (UMMA M)
constexpr int kOzBN = 64;      // tile cols of the one-CTA-per-SM variant (a 128 x 32 variant runs
                               // two CTAs per SM for multi-wave grids; ozaki_kernels.cu)

// Digit planes of nmat symmetric ld x ld matrices: [mat][slice][ld][ld] int8.
struct OzPlanes {
    int8_t* d = nullptr;
    int e = 0;  // matrix = 2^e sum_s 2^{-7s} plane_s
};

// TMA maps of one plane buffer for both tile variants: loads in the A role
// (k block x 128 rows) and the B role (k block x BN rows), epilogue stores.
struct OzMaps {
    CUtensorMap a, b, st;     // 128 x 64 tiles (64-byte k blocks, 64 x 64 store boxes)
    CUtensorMap a2, b2, st2;  // 128 x 32 tiles (32-byte k blocks, 32 x 32 store boxes)
    CUtensorMap bp;           // persistent 128 x 32 tiles: B boxes of 32 rows x 64 bytes
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
    const OzMaps* mc;        // TMA maps of Cd (stores use the 64-row box)
    int eC;
    const int* ictl;         // done flags per solve (matrix / 2), or null
    long long* dbg_t;        // instrumentation: 4 globaltimer stamps per CTA, or null
    int dbg_mode;            // instrumentation: bit 0 skips the MMAs, bit 1 the TMA loads
    int no_pdl;              // launch without programmatic dependent launch
    int dstore;              // digit planes by direct 16-byte global stores (else TMA stores)
    const int* tiles;        // row-sharded products: this rank's lower-tile indices, or null (all)
    int ntiles;              // entries of tiles
    int mstep;               // matrices of this launch: blockIdx.y * mstep + moff (mstep 0 -> 1)
    int moff;
    int rc;                  // plane layout: rows per chunk (0 -> ld; see OzShard)
};

void launch_oz_gemm(const OzGemm& g, cudaStream_t st);
// Tiled cone projections use this kernel unless TPB_CONE=dmma (FP64 DMMA).
bool cone_uses_ozaki();
int oz_gemm_tiles(int ld);

// Digit-plane buffers of the cone projection: [0..2] pair with the three FP64
// work buffers, [3] holds X0 = A / ||A||_F.
struct OzWork {
    int8_t* d[4] = {nullptr, nullptr, nullptr, nullptr};
    OzMaps maps[4];
};

// Row-sharded projection of one large instance over G ranks:
// rank k owns the 128-row blocks [k NB/G, (k+1) NB/G) of every iterate. Its
// tiles are the lower tiles of those row blocks plus the lower tiles whose
// mirror lands in them, so its rows are complete after its GEMM; an
// in-place NCCL all-gather of the row blocks of every digit plane then gives
// every rank the whole iterate. The same kernel computes every tile, so the
// result is bitwise the single-GPU one. (The final FP64 product is
// replicated.)
// Sharded runs store each matrix's planes row-chunk-major,
// [mat][chunk][slice][rc rows][ld] with rc = ld / G (rc = ld is the plain
// [mat][slice][ld][ld] layout), so a rank's rows of all eight planes are one
// contiguous block: one all-gather per matrix. Tiles never straddle chunks.
// The S (even matrices) and T (odd) chains of the sign iteration are
// independent, so each product runs as two launches and one chain's
// all-gather (comm stream) overlaps the other chain's GEMM.
struct OzShard {
    int rank = 0, nranks = 1;
    void* comm = nullptr;    // ncclComm_t
    int* tiles = nullptr;    // device: this rank's tile indices
    int ntiles = 0;
    cudaStream_t cs = nullptr;                    // all-gathers
    cudaEvent_t gemm_done[2] = {nullptr, nullptr};  // per chain
    cudaEvent_t ag_done[2] = {nullptr, nullptr};
};
// Host tile list of `rank` for an ld x ld iterate (ld % 128 == 0, ld/128 % nranks == 0).
std::vector<int> oz_shard_tiles(int ld, int nranks, int rank);

struct SignSchedule;
// Ozaki-scheme counterpart of enqueue_cone_tiled (cone_kernels.cuh): the
// same sign iteration, every product on the int8 tensor cores.
void enqueue_cone_ozaki(const double* A, double* w0, double* w1, double* w2, const OzWork& oz, int ld,
                        int n, const double* scale, double* C, long long c_stride_b, long long c_stride_w,
                        const int* ictl, int nmat, const SignSchedule& sch, cudaStream_t st,
                        const OzShard* shard = nullptr);

// Digit planes of s * A (s = scale[mat] or 1) with exponent e (layout rc as in OzGemm).
void launch_oz_split(const double* A, long long mstride, int ld, int nmat, const double* scale,
                     int e, int8_t* planes, const int* ictl, cudaStream_t st, int rc = 0);

}  // namespace tpb
