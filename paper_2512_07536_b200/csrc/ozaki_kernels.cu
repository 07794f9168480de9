// Ozaki-scheme FP64 GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM, operands staged by TMA). See
// ozaki_kernels.cuh for the arithmetic and DESIGN.md §3.2 for its place in
// the cone projection (replacing the reference's eigen-clamps,
// proj/src/eig.cpp:131-176).
//
// One CTA per 128 x 64 lower-triangular output tile of one matrix:
//   warp 0      TMA producer (one lane): per 64-byte k block, the KS digit
//               planes of the A rows and of the B rows -> one pipeline stage
//   warp 1      TMEM owner + MMA issuer (one lane): for every pair (s, t) with
//               s + t <= KS + 1, D[s+t] += A_s . B_t: per A plane one MMA over
//               the contiguous B planes (M=128, N <= 256, K=32 steps)
//   warps 2-9   epilogue: TMEM -> FP64 (smallest group first), alpha/beta/E,
//               FP64 and digit-plane stores, mirrored across the diagonal
// The KS accumulator groups (KS x 64 int32 columns) fill TMEM's 512 columns.
#include "ozaki_kernels.cuh"

#include "cone_kernels.cuh"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace tpb {

namespace {

constexpr int KS = kOzSlices, BM = kOzBM, BN = kOzBN, BK = kOzBK;
constexpr int STAGES = 2;
constexpr int A_PLANE = BM * BK, B_PLANE = BN * BK;              // bytes
constexpr int STAGE_BYTES = KS * (A_PLANE + B_PLANE);            // 96 KB
constexpr int CP = BM + 1;       // epilogue FP64 staging pitch (doubles)
constexpr int DP = BN / 4 + 1;   // epilogue digit-word staging pitch (words)
constexpr int CS_BYTES = BN * CP * 8;
constexpr int DW_BYTES = KS * BM * DP * 4;
constexpr int TB_BYTES = KS * BN * BM;
constexpr int EPI_BYTES = CS_BYTES + DW_BYTES + TB_BYTES;
constexpr int SMEM_BYTES = (STAGES * STAGE_BYTES > EPI_BYTES ? STAGES * STAGE_BYTES : EPI_BYTES) + 1024;
constexpr int EPI_WARPS = 8, EPI_THREADS = 32 * EPI_WARPS;
constexpr int THREADS = 64 + EPI_THREADS;  // producer warp, MMA warp, epilogue warps
constexpr int HN = BN / 2;                  // tile columns per epilogue thread
static_assert(KS * BN <= 512, "accumulator groups exceed TMEM");
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// 32 lanes x 16 consecutive 32-bit columns (one row segment per thread)
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major operand tile in SWIZZLE_64B layout (64-byte rows, 8-row atoms of
// 512 B): start address, SBO = 512 B, version 1, layout type 4.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 128, N = nn
__host__ __device__ constexpr uint32_t idesc_n(int nn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double spow(double s, int p) {
    return p == 0 ? 1.0 : (p == 1 ? s : (p == 2 ? s * s : (p == -1 ? 1.0 / s : 1.0)));
}

// Truncated base-128 digits of v * 2^-e (|v| 2^-e < 1): byte `lane4` of each
// of the KS plane words.
__device__ __forceinline__ void put_digits(double v, double inv2e, int lane4, uint32_t (&w)[KS]) {
    const long long q = __double2ll_rz(v * inv2e * 0x1p56);
    unsigned long long a = q < 0 ? (unsigned long long)(-q) : (unsigned long long)q;
    a = a > 0xFFFFFFFFFFFFFFull ? 0xFFFFFFFFFFFFFFull : a;  // saturate (bounds are static)
    const uint32_t hi = (uint32_t)(a >> 28), lo = (uint32_t)(a & 0xFFFFFFF);
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        const uint32_t h = s < 4 ? hi : lo;
        int dg = (int)((h >> (21 - 7 * (s & 3))) & 127u);
        if (q < 0) dg = -dg;
        w[s] |= ((uint32_t)dg & 0xFFu) << (8 * lane4);
    }
}
// lower tiles of a (ld/BM) x (ld/BN) grid: row block I holds col blocks
// J < ceil((I+1) BM / BN)
__host__ __device__ inline int tiles_before(int I) {
    constexpr int R = BM / BN;  // 2
    return R * I * (I + 1) / 2;
}
__device__ inline void oz_tile(int t, int& I, int& J) {
    int b = 0;
    while (tiles_before(b + 1) <= t) ++b;
    I = b;
    J = t - tiles_before(b);
}

}  // namespace

__global__ void __launch_bounds__(THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   OzGemm g) {
    const int mat = blockIdx.y;
    if (g.ictl && g.ictl[(mat >> 1) * 8 + 1]) return;
    const long long t_start = g.dbg_t ? gtimer() : 0;
    int I, J;
    oz_tile(blockIdx.x, I, J);
    const int i0 = I * BM, j0 = J * BN;
    const int ld = g.ld;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[2 * STAGES + 1];
    __shared__ uint32_t tmem_slot;
    const uint32_t sbase = (su32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - su32(smem_raw));
    auto full_bar = [&](int s) { return su32(&bars[s]); };
    auto empty_bar = [&](int s) { return su32(&bars[STAGES + s]); };
    const uint32_t tfull_bar = su32(&bars[2 * STAGES]);
    auto a_tile = [&](int st, int s) { return sbase + st * STAGE_BYTES + s * A_PLANE; };
    auto b_tile = [&](int st, int s) { return sbase + st * STAGE_BYTES + KS * A_PLANE + s * B_PLANE; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(tfull_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         su32(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const int KB = ld / BK;
    const long long plane_rows = (long long)mat * KS * ld;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int st = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(empty_bar(st), ph ^ 1);
                if (g.dbg_mode & 2) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full_bar(st)) : "memory");
                    continue;
                }
                mbar_expect_tx(full_bar(st), STAGE_BYTES);
#pragma unroll 1
                for (int s = 0; s < KS; ++s) {
                    tma_load_2d(a_tile(st, s), &mapA, full_bar(st), kb * BK,
                                (int)(plane_rows + (long long)s * ld + i0));
                    tma_load_2d(b_tile(st, s), &mapB, full_bar(st), kb * BK,
                                (int)(plane_rows + (long long)s * ld + j0));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int st = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(full_bar(st), ph);
                tc_fence_after();
                if (g.dbg_mode & 1) {
                    tc_commit(empty_bar(st));
                    continue;
                }
#pragma unroll
                for (int kk = 0; kk < BK / 32; ++kk) {
                    // A_s . [B_t0 | ... | B_t1] in one MMA: the B planes are
                    // contiguous rows in smem and the groups d = s + t are
                    // contiguous 64-column blocks in TMEM.
#pragma unroll
                    for (int s = 1; s <= KS; ++s) {
                        const uint64_t ad = sw64_desc(a_tile(st, s - 1) + kk * 32);
#pragma unroll
                        for (int t0 = 1; t0 <= KS + 1 - s; t0 += 4) {
                            const int t1 = t0 + 3 < KS + 1 - s ? t0 + 3 : KS + 1 - s;
                            const int nn = BN * (t1 - t0 + 1);
                            const uint64_t bd = sw64_desc(b_tile(st, t0 - 1) + kk * 32);
                            const uint32_t acc = (kb | kk) != 0 || s != 1;
                            mma_i8(tmem + (uint32_t)((s + t0 - 2) * BN), ad, bd, idesc_n(nn), acc);
                        }
                    }
                }
                tc_commit(empty_bar(st));
            }
            tc_commit(tfull_bar);
        }
    } else {
        // ---------------- epilogue: warps 2..9; thread <-> (tile row = TMEM
        // lane of its warp's quarter, one half of the tile's columns)
        const int q = warp & 3;                 // TMEM lane quarter this warp may access
        const int h = (warp - 2) >> 2;          // column half
        const int r = q * 32 + lane;            // tile row
        const int c0 = h * HN;                  // first tile column of this thread
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
        const long long t_setup = g.dbg_t ? gtimer() : 0;
        mbar_wait(tfull_bar, 0);
        tc_fence_after();
        const long long t_full = g.dbg_t ? gtimer() : 0;
        double acc[HN];
#pragma unroll
        for (int j = 0; j < HN; ++j) acc[j] = 0.0;
#pragma unroll
        for (int d = KS + 1; d >= 2; --d) {  // smallest contributions first
            const double sc = ldexp(1.0, -7 * d);
            uint32_t v[HN];
#pragma unroll
            for (int c = 0; c < HN / 16; ++c)
                tmem_ld16(taddr + (uint32_t)((d - 2) * BN + c * 16), *reinterpret_cast<uint32_t(*)[16]>(v + c * 16));
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < HN; ++j) acc[j] = fma((double)(int)v[j], sc, acc[j]);
        }
        const double s = g.scale ? g.scale[mat] : 1.0;
        double alpha = g.alpha_c * spow(s, g.pa) * ldexp(1.0, g.eA + g.eB);
        const double beta = g.beta_c * spow(s, g.pb);
        if (g.sign_mode && (mat & 1) == 0) alpha = -alpha;
        const double* E = g.E ? g.E + (long long)mat * ld * ld : nullptr;
        const int i = i0 + r;
#pragma unroll
        for (int j = 0; j < HN; ++j) {
            double v = alpha * acc[j];
            if (E) v = fma(beta, __ldg(E + (long long)(j0 + c0 + j) * ld + i), v);  // E symmetric
            acc[j] = v;
        }
        // Stores. Every element (a, b) of C is written by exactly one tile:
        // the lower tile holding (max, min) writes (a >= b) directly and
        // (a > b) mirrored, so runs are deterministic.
        const int nv = g.nvalid;
        double* C = g.C ? g.C + (long long)(mat >> 1) * g.c_stride_b + (long long)(mat & 1) * g.c_stride_w
                        : nullptr;
        int8_t* Cd = g.Cd ? g.Cd + (long long)mat * KS * ld * ld : nullptr;
        const long long ld2 = (long long)ld * ld;
        double* Cs = reinterpret_cast<double*>(sgen);                      // [BN][CP] FP64
        uint32_t* Dw = reinterpret_cast<uint32_t*>(sgen + CS_BYTES);       // [KS][BM][DP] words
        uint8_t* Tb = sgen + CS_BYTES + DW_BYTES;                          // [KS][BN][BM] bytes
        if (C) {
            // mirrored part straight from registers: lanes hold consecutive columns
#pragma unroll
            for (int j = 0; j < HN; ++j) {
                const int jj = j0 + c0 + j;
                if (i > jj && i < nv && jj < nv) C[(long long)jj * g.ldc + i] = acc[j];
            }
#pragma unroll
            for (int j = 0; j < HN; ++j) Cs[(c0 + j) * CP + r] = acc[j];
        }
        if (Cd) {
            const double inv2e = ldexp(1.0, -g.eC);
#pragma unroll
            for (int jw = 0; jw < HN / 4; ++jw) {
                uint32_t w[KS];
#pragma unroll
                for (int s2 = 0; s2 < KS; ++s2) w[s2] = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) put_digits(acc[4 * jw + k], inv2e, k, w);
#pragma unroll
                for (int s2 = 0; s2 < KS; ++s2) {
                    Dw[(s2 * BM + r) * DP + c0 / 4 + jw] = w[s2];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        Tb[(s2 * BN + c0 + 4 * jw + k) * BM + r] = (uint8_t)(w[s2] >> (8 * k));
                }
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        const int et = threadIdx.x - 64;        // 0 .. EPI_THREADS-1
        const int ew = et >> 5;                 // epilogue warp 0..7
        if (C) {
            // direct part (row ii, columns j0..j0+BN) from the staged tile
            for (int rr = ew; rr < BM; rr += EPI_WARPS) {
                const int ii = i0 + rr;
#pragma unroll
                for (int j = lane; j < BN; j += 32) {
                    const int jj = j0 + j;
                    if (ii >= jj && ii < nv && jj < nv) C[(long long)ii * g.ldc + jj] = Cs[j * CP + rr];
                }
            }
        }
        if (Cd) {
            // direct digit rows: BN bytes = BN/4 words, BN/4 threads per row
            constexpr int WPR = BN / 4;
            for (int row = et / WPR; row < KS * BM; row += EPI_THREADS / WPR) {
                const int s2 = row / BM, rr = row % BM, w = et % WPR;
                const int ii = i0 + rr, jj0 = j0 + 4 * w;
                const uint32_t word = Dw[(s2 * BM + rr) * DP + w];
                int8_t* dst = Cd + s2 * ld2 + (long long)ii * ld + jj0;
                if (jj0 + 3 <= ii) {
                    *reinterpret_cast<uint32_t*>(dst) = word;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (jj0 + k <= ii) dst[k] = (int8_t)(word >> (8 * k));
                }
            }
            // mirrored digit rows (row j0 + j, columns i0..i0+BM): one warp per row
            for (int row = ew; row < KS * BN; row += EPI_WARPS) {
                const int s2 = row / BN, j = row % BN;
                const int jj = j0 + j, ic = i0 + 4 * lane;
                if (ic + 3 <= jj) continue;
                const uint32_t word = reinterpret_cast<const uint32_t*>(Tb + (s2 * BN + j) * BM)[lane];
                int8_t* dst = Cd + s2 * ld2 + (long long)jj * ld + ic;
                if (ic > jj) {
                    *reinterpret_cast<uint32_t*>(dst) = word;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (ic + k > jj) dst[k] = (int8_t)(word >> (8 * k));
                }
            }
        }
        if (g.dbg_t) asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");  // warp-uniform
        if (g.dbg_t && et == 0) {
            long long* o = g.dbg_t + 4LL * (blockIdx.y * gridDim.x + blockIdx.x);
            o[0] = t_start;
            o[1] = t_setup;
            o[2] = t_full;
            o[3] = gtimer();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// Digit planes of s A, 4 consecutive row elements per thread.
__global__ void oz_split_kernel(const double* A, long long mstride, int ld, const double* scale,
                                int e, int8_t* planes, const int* ictl) {
    const int mat = blockIdx.y;
    if (ictl && ictl[(mat >> 1) * 8 + 1]) return;
    const long long n4 = (long long)ld * ld / 4;
    const double s = (scale ? scale[mat] : 1.0) * ldexp(1.0, -e);
    const double* a = A + (long long)mat * mstride;
    int8_t* out = planes + (long long)mat * KS * ld * ld;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n4;
         idx += (long long)gridDim.x * blockDim.x) {
        const double4 v = *reinterpret_cast<const double4*>(a + idx * 4);
        uint32_t w[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) w[k] = 0;
        put_digits(v.x, s, 0, w);
        put_digits(v.y, s, 1, w);
        put_digits(v.z, s, 2, w);
        put_digits(v.w, s, 3, w);
#pragma unroll
        for (int k = 0; k < KS; ++k)
            reinterpret_cast<uint32_t*>(out + (long long)k * ld * ld)[idx] = w[k];
    }
}

// ------------------------------------------------------------------ host
namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                 CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                 CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        TPB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw Error(kCuda, "cuTensorMapEncodeTiled is not available from the driver");
        fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

void encode(CUtensorMap* m, const int8_t* base, int ld, long long rows, int box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld};
    const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

}  // namespace

void make_oz_maps(const int8_t* planes, int ld, int nmat, OzMaps* out) {
    if (ld % BM != 0) throw Error(kInvalidArgument, "ozaki GEMM needs ld % 128 == 0");
    const long long rows = (long long)nmat * KS * ld;
    encode(&out->a, planes, ld, rows, BM);
    encode(&out->b, planes, ld, rows, BN);
}

int oz_gemm_tiles(int ld) { return tiles_before(ld / BM); }

void init_attrs_ozaki() {
    TPB_CUDA(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
}

void launch_oz_gemm(const OzGemm& g, cudaStream_t st) {
    const dim3 grid(oz_gemm_tiles(g.ld), g.nmat);
    oz_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(g.ma->a, g.mb->b, g);
    TPB_CHECK_LAUNCH();
}

void launch_oz_split(const double* A, long long mstride, int ld, int nmat, const double* scale, int e,
                     int8_t* planes, const int* ictl, cudaStream_t st) {
    const long long n4 = (long long)ld * ld / 4;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 1024);
    oz_split_kernel<<<dim3(blocks, nmat), 256, 0, st>>>(A, mstride, ld, scale, e, planes, ictl);
    TPB_CHECK_LAUNCH();
}

// Static spectral bounds of the sign-iteration operands as
// digit-plane exponents: |X| <= 1.21, |Y| <= 1.45 -> 2^1; |Z| <= 2.81 -> 2^2;
// X0 = A / ||A||_F has |X0| <= 1 -> 2^1 (strict bound needed).
namespace {
constexpr int kEX = 1, kEY = 1, kEZ = 2, kEX0 = 1;
}

void enqueue_cone_ozaki(const double* A, double* w0, double* w1, double* w2, const OzWork& oz, int ld,
                        int n, const double* scale, double* C, long long c_stride_b, long long c_stride_w,
                        const int* ictl, int nmat, const SignSchedule& sch, cudaStream_t st) {
    const long long ms = (long long)ld * ld;
    launch_oz_split(A, ms, ld, nmat, scale, kEX0, oz.d[3], ictl, st);
    OzGemm g{};
    g.ld = ld;
    g.nmat = nmat;
    g.scale = scale;
    g.ictl = ictl;
    g.ldc = ld;
    g.nvalid = ld;
    g.c_stride_b = 2 * ms;
    g.c_stride_w = ms;
    double* fb[3] = {w0, w1, w2};
    // one product: operands are digit buffers (index 0..3), outputs FP64
    // buffer / digit buffer index (-1: none)
    auto step = [&](int ia, int ea, int ib, int eb, double al, int pa, const double* e, double be, int pb,
                    int oc, int od, int ec) {
        g.ma = &oz.maps[ia];
        g.mb = &oz.maps[ib];
        g.eA = ea;
        g.eB = eb;
        g.alpha_c = al;
        g.pa = pa;
        g.E = e;
        g.beta_c = be;
        g.pb = pb;
        g.C = oc >= 0 ? fb[oc] : nullptr;
        g.Cd = od >= 0 ? oz.d[od] : nullptr;
        g.eC = ec;
        launch_oz_gemm(g, st);
    };
    int x = -1;  // FP64/digit buffer holding X (-1: X0 = s A, FP64 A, digits in [3])
    auto free_pair = [&](int& f0, int& f1) {
        int k = 0, fr[3];
        for (int q = 0; q < 3; ++q)
            if (q != x) fr[k++] = q;
        f0 = fr[0];
        f1 = fr[1];
    };
    for (int it = 0; it < sch.k1; ++it) {
        int y, z;
        free_pair(y, z);
        const int xd = x < 0 ? 3 : x;
        const double* xe = x < 0 ? A : fb[x];
        const int xpb = x < 0 ? 1 : 0;
        step(xd, kEX, xd, kEX, 1.0, 0, nullptr, 0.0, 0, y, y, kEY);                // Y = X^2
        step(y, kEY, y, kEY, sch.qc, 0, fb[y], sch.qb, 0, -1, z, kEZ);             // Z = c Y^2 + b Y
        step(xd, kEX, z, kEZ, 1.0, 0, xe, sch.qa, xpb, y, y, kEX);                // X' = X Z + a X
        x = y;
    }
    for (int it = 0; it < sch.k2; ++it) {
        int y, xn;
        free_pair(y, xn);
        const int xd = x < 0 ? 3 : x;
        const double* xe = x < 0 ? A : fb[x];
        const int xpb = x < 0 ? 1 : 0;
        step(xd, kEX, xd, kEX, 1.0, 0, nullptr, 0.0, 0, -1, y, kEY);               // Y = X^2
        step(xd, kEX, y, kEY, -0.5, 0, xe, 1.5, xpb, xn, xn, kEX);                // X' = 1.5 X - 0.5 X Y
        x = xn;
    }
    // P = 0.5 A -/+ 0.5 A X = 0.5 A -/+ (0.5 / s) X0 X into the state blocks
    g.ldc = n;
    g.nvalid = n;
    g.c_stride_b = c_stride_b;
    g.c_stride_w = c_stride_w;
    g.sign_mode = 1;
    g.ma = &oz.maps[3];
    g.mb = &oz.maps[x < 0 ? 3 : x];
    g.eA = kEX0;
    g.eB = kEX;
    g.alpha_c = 0.5;
    g.pa = -1;
    g.E = A;
    g.beta_c = 0.5;
    g.pb = 0;
    g.C = C;
    g.Cd = nullptr;
    launch_oz_gemm(g, st);
}

}  // namespace tpb
