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

#include "nccl_shim.hpp"

#include "cone_kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace tpb {

#ifndef OZ_EPI_WARPS
#define OZ_EPI_WARPS 16
#endif

namespace {

constexpr int KS = kOzSlices, BM = kOzBM;

// Tile configuration: BN output columns (one accumulator group = BN TMEM
// columns, KS groups), BK k-bytes per pipeline stage. <64, 64>: one CTA per
// SM, 512 TMEM columns; <32, 32>: 256 TMEM columns and 98 KB of shared
// memory, so two CTAs share an SM and one's epilogue overlaps the other's
// main loop (batched small-n products, where the epilogue dominates).
template <int BN_, int BK_, int EW_>
struct Tile {
    static constexpr int BN = BN_, BK = BK_;
    // producer warp, MMA warp, EW epilogue warps (EW / 4 per TMEM lane quarter)
    static constexpr int EPI_WARPS = EW_, EPI_THREADS = 32 * EW_, THREADS = 64 + 32 * EW_;
    static constexpr int R = BM / BN;          // tiles per 128-row diagonal block
    static constexpr int STAGES = 2;
    static constexpr int A_PLANE = BM * BK, B_PLANE = BN * BK;  // bytes
    static constexpr int STAGE_BYTES = KS * (A_PLANE + B_PLANE);
    static constexpr int CP = BM + 1;          // epilogue FP64 staging pitch (doubles)
    static constexpr int CS_BYTES = (BN * CP * 8 + 1023) / 1024 * 1024;
    static constexpr int BB = BN;              // TMA store box: BB rows x BB bytes
    static constexpr int BOX_BYTES = BB * BB;
    static constexpr int NBOX = BM / BB;       // boxes per plane and orientation
    static constexpr int DIG_BYTES = 2 * KS * NBOX * BOX_BYTES;
    static constexpr int EPI_BYTES = CS_BYTES + DIG_BYTES;
    static constexpr int SMEM_BYTES =
        (STAGES * STAGE_BYTES > EPI_BYTES ? STAGES * STAGE_BYTES : EPI_BYTES) + 1024;
    static constexpr int HN = BN / (EW_ / 4);  // tile columns per epilogue thread
    static constexpr int TMEM_COLS = KS * BN <= 256 ? 256 : 512;
    static constexpr int TCHUNK = 256 / BN;    // B planes per MMA (N <= 256)
    static constexpr int MIN_BLOCKS = 2 * (SMEM_BYTES + 1024) <= 228 * 1024 ? 2 : 1;
    static_assert(KS * BN <= 512, "accumulator groups exceed TMEM");
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
    static_assert(BK == 32 || BK == 64, "k block is one or two MMA k-steps");
    static_assert(HN % 16 == 0, "TMEM loads of 16 columns");
};
using TileL = Tile<64, 64, OZ_EPI_WARPS>;
using TileS = Tile<32, 32, 8>;

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
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major operand tile, BK-byte rows in the matching swizzle (8-row atoms of
// 8 BK bytes): start address, SBO = 8 BK, version 1, layout type 4 (64B) /
// 6 (32B).
template <int BK>
__device__ __forceinline__ uint64_t op_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((8 * BK) >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)(BK == 64 ? 4 : 6) << 61);
}

// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 128, N = nn
__host__ __device__ constexpr uint32_t idesc_n(int nn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// Exact int32 -> FP64 without the quarter-rate conversion pipe: the bits
// 0x43300000:(x ^ 2^31) are the double 2^52 + 2^31 + x; one DADD removes the
// offset (exact). Same value as (double)(int)x.
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
    return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
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
// Magnitude digits of 4 values as 8 plane words (byte k of word s = digit
// s+1 of value k), negated bytewise for negative values: |v| 2^-e < 1.
__device__ __forceinline__ uint32_t neg4(uint32_t w) {  // bytewise -b for b in [0, 127]
    return ((~w & 0x7F7F7F7Fu) + 0x01010101u) ^ 0x80808080u;
}
__device__ __forceinline__ uint32_t spread7(uint32_t a) {  // 28-bit a -> [a&127, a>>7&127, ...]
    return (a & 0x7Fu) | ((a << 1) & 0x7F00u) | ((a << 2) & 0x7F0000u) | ((a << 3) & 0x7F000000u);
}
__device__ __forceinline__ void digits4(const double (&v)[4], double s28, uint32_t (&w)[KS]) {
    // |v| 2^-e = hi 2^-28 + lo 2^-56 with hi = rint(|v| 2^(28-e)) in [0, 2^28)
    // and |lo| <= 2^27 (its own sign), both taken from the low mantissa bits
    // after adding 1.5 2^52 (no conversion instructions); digit bytes are
    // 7-bit groups of hi and |lo|, negated bytewise where needed.
    constexpr double kM = 6755399441055744.0;  // 1.5 * 2^52
    uint32_t ph[4], pl[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double a = fabs(v[k]) * s28;
        const double th = a + kM;
        uint32_t hi = (uint32_t)__double2loint(th);
        const double rem = a - (th - kM);
        const int lo = __double2loint(fma(rem, 268435456.0, kM));
        hi = hi > 0xFFFFFFFu ? 0xFFFFFFFu : hi;  // saturate (outside the static bounds)
        uint32_t xh = spread7(hi), xl = spread7((uint32_t)(lo < 0 ? -lo : lo));
        const bool neg = v[k] < 0.0;
        if (neg) xh = neg4(xh);
        if (neg != (lo < 0)) xl = neg4(xl);
        ph[k] = xh;  // bytes: digit 4, 3, 2, 1
        pl[k] = xl;  // bytes: digit 8, 7, 6, 5
    }
    // 4x4 byte transposes: word s collects digit s+1 of the four values
    const uint32_t a = __byte_perm(ph[0], ph[1], 0x7362), b = __byte_perm(ph[2], ph[3], 0x7362);
    const uint32_t c = __byte_perm(ph[0], ph[1], 0x5140), d = __byte_perm(ph[2], ph[3], 0x5140);
    w[0] = __byte_perm(a, b, 0x7632);
    w[1] = __byte_perm(a, b, 0x5410);
    w[2] = __byte_perm(c, d, 0x7632);
    w[3] = __byte_perm(c, d, 0x5410);
    const uint32_t e = __byte_perm(pl[0], pl[1], 0x7362), f = __byte_perm(pl[2], pl[3], 0x7362);
    const uint32_t g = __byte_perm(pl[0], pl[1], 0x5140), h = __byte_perm(pl[2], pl[3], 0x5140);
    w[4] = __byte_perm(e, f, 0x7632);
    w[5] = __byte_perm(e, f, 0x5410);
    w[6] = __byte_perm(g, h, 0x7632);
    w[7] = __byte_perm(g, h, 0x5410);
}

// Row slot of the FP64 staging tile: conflict-free both for 32 consecutive
// rows (TMEM drain) and for rows 4 rb + q, rb = 0..31 (4 x 4 digit blocks).
__device__ __forceinline__ int csr(int r) { return r ^ ((r >> 4) & 3); }

// 4 x 4 byte transpose: rows r[q] (byte c = column c) -> columns o[c] (byte q = row q)
__device__ __forceinline__ void transpose4x4(const uint32_t (&r)[4], uint32_t (&o)[4]) {
    const uint32_t t0 = __byte_perm(r[0], r[1], 0x5140), t1 = __byte_perm(r[0], r[1], 0x7362);
    const uint32_t t2 = __byte_perm(r[2], r[3], 0x5140), t3 = __byte_perm(r[2], r[3], 0x7362);
    o[0] = __byte_perm(t0, t2, 0x5410);
    o[1] = __byte_perm(t0, t2, 0x7632);
    o[2] = __byte_perm(t1, t3, 0x5410);
    o[3] = __byte_perm(t1, t3, 0x7632);
}

// 16-byte chunk address inside a BB x BB-byte box in the SWIZZLE_{BB}B layout
template <int BB>
__device__ __forceinline__ uint32_t box_off(int row, int chunk) {
    const int x = BB == 64 ? ((row >> 1) & 3) : ((row >> 2) & 1);
    return (uint32_t)(row * BB + ((chunk ^ x) << 4));
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}

// lower tiles of a (ld/BM) x (ld/BN) grid: row block I holds col blocks
// J < (I+1) R, R = BM / BN
__host__ __device__ inline int tiles_before(int R, int I) { return R * I * (I + 1) / 2; }
__device__ inline void oz_tile(int R, int t, int& I, int& J) {
    int b = 0;
    while (tiles_before(R, b + 1) <= t) ++b;
    I = b;
    J = t - tiles_before(R, b);
}

}  // namespace

template <typename TL>
__global__ void __launch_bounds__(TL::THREADS, TL::MIN_BLOCKS)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, OzGemm g) {
    constexpr int BN = TL::BN, BK = TL::BK, STAGES = TL::STAGES, R = TL::R, HN = TL::HN, CP = TL::CP;
    constexpr int EPI_WARPS = TL::EPI_WARPS, EPI_THREADS = TL::EPI_THREADS;
    constexpr int BB = TL::BB, NBOX = TL::NBOX;
    constexpr int A_PLANE = TL::A_PLANE, B_PLANE = TL::B_PLANE, STAGE_BYTES = TL::STAGE_BYTES;
    constexpr int TMEM_COLS = TL::TMEM_COLS;
    const int mat = g.mstep ? blockIdx.y * g.mstep + g.moff : blockIdx.y;
    if (g.ictl && g.ictl[(mat >> 1) * 8 + 1]) return;
    const long long t_start = g.dbg_t ? gtimer() : 0;
    int I, J;
    oz_tile(R, g.tiles ? g.tiles[blockIdx.x] : blockIdx.x, I, J);
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // Programmatic dependent launch: everything above overlaps the previous
    // GEMM's tail; its digit planes (our operands) and its reads of the
    // buffer we overwrite are complete after this wait. Our own dependents
    // may then be scheduled as SMs free up.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const int KB = ld / BK;
    const int rc = g.rc ? g.rc : ld;  // plane layout (OzShard)
    // plane row of (slice 0, row i): slice s adds s * rc
    auto prow = [&](int i) { return (long long)mat * KS * ld + (long long)(i / rc) * KS * rc + i % rc; };
    const long long a_row0 = prow(i0), b_row0 = prow(j0);

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
                    tma_load_2d(a_tile(st, s), &mapA, full_bar(st), kb * BK, (int)(a_row0 + (long long)s * rc));
                    tma_load_2d(b_tile(st, s), &mapB, full_bar(st), kb * BK, (int)(b_row0 + (long long)s * rc));
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
                    // contiguous BN-column blocks in TMEM.
#pragma unroll
                    for (int s = 1; s <= KS; ++s) {
                        const uint64_t ad = op_desc<BK>(a_tile(st, s - 1) + kk * 32);
#pragma unroll
                        for (int t0 = 1; t0 <= KS + 1 - s; t0 += TL::TCHUNK) {
                            const int t1 = t0 + TL::TCHUNK - 1 < KS + 1 - s ? t0 + TL::TCHUNK - 1 : KS + 1 - s;
                            const int nn = BN * (t1 - t0 + 1);
                            const uint64_t bd = op_desc<BK>(b_tile(st, t0 - 1) + kk * 32);
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
        const int h = (warp - 2) >> 2;          // column slice
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
        static_assert(KS % 2 == 0, "groups are drained in pairs");
#pragma unroll
        for (int d = KS + 1; d >= 2; d -= 2) {  // smallest contributions first, two groups per wait
            uint32_t v[2][HN];
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                for (int c = 0; c < HN / 16; ++c)
                    tmem_ld16(taddr + (uint32_t)((d - q2 - 2) * BN + c * 16),
                              *reinterpret_cast<uint32_t(*)[16]>(&v[q2][c * 16]));
            tmem_wait_ld();
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2) {
                const double sc = ldexp(1.0, -7 * (d - q2));
#pragma unroll
                for (int j = 0; j < HN; ++j) acc[j] = fma(i32_to_f64(v[q2][j]), sc, acc[j]);
            }
        }
        const long long t_acc = g.dbg_t ? gtimer() : 0;
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
            if (i == j0 + c0 + j) v += g.dshift;
            acc[j] = v;
        }
        // Stores. Ownership keeps C exactly symmetric and every element
        // written once (deterministic): off-diagonal tiles (J < R I) write
        // themselves and their mirror; in the diagonal 128-row block the tile
        // t = J - R I owns rows BN t.. (its BN x BN diagonal sub-block
        // symmetrised) and mirrors rows BN (t+1).. into the tiles to its right.
        const int tdiag = J - R * I;
        const int dr0 = tdiag < 0 ? 0 : BN * tdiag;          // first directly owned tile row
        const int mr0 = tdiag < 0 ? 0 : BN * (tdiag + 1);    // first mirrored tile row
        const int nv = g.nvalid;
        double* C = g.C ? g.C + (long long)(mat >> 1) * g.c_stride_b + (long long)(mat & 1) * g.c_stride_w
                        : nullptr;
        double* Cs = reinterpret_cast<double*>(sgen);  // [BN][CP]: Cs[c][csr(r)] = tile (r, c)
#pragma unroll
        for (int j = 0; j < HN; ++j) Cs[(c0 + j) * CP + csr(r)] = acc[j];
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        const int et = threadIdx.x - 64;        // 0 .. EPI_THREADS-1
        const int ew = et >> 5;                 // epilogue warp 0..7
        const long long t_stage = g.dbg_t ? gtimer() : 0;
        if (tdiag >= 0) {
            // symmetrise the diagonal BN x BN sub-block (tile rows dr0.., all columns)
            for (int idx = et; idx < BN * BN; idx += EPI_THREADS) {
                const int u = idx / BN, v = idx % BN;  // sub-block row, column
                if (u < v) Cs[v * CP + csr(dr0 + u)] = Cs[u * CP + csr(dr0 + v)];
            }
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        }
        if (C) {
            for (int rr = dr0 + ew; rr < BM; rr += EPI_WARPS) {
                const int ii = i0 + rr;
#pragma unroll
                for (int j = lane; j < BN; j += 32) {
                    const int jj = j0 + j;
                    if (ii < nv && jj < nv) C[(long long)ii * g.ldc + jj] = Cs[j * CP + csr(rr)];
                }
            }
            for (int j = ew; j < BN; j += EPI_WARPS) {
                const int jj = j0 + j;
                for (int rr = mr0 + lane; rr < BM; rr += 32) {
                    const int ii = i0 + rr;
                    if (ii < nv && jj < nv) C[(long long)jj * g.ldc + ii] = Cs[j * CP + csr(rr)];
                }
            }
        }
        const long long t_cst = g.dbg_t ? gtimer() : 0;
        if (g.Cd && g.dstore) {
            // Each thread splits one 4 x 4 block (rows 4 rb.., columns 4 cb..)
            // into digits once. Mirror rows: a 4 x 4 byte transpose per plane
            // and 4-byte stores, 32 lanes = 128 contiguous bytes of a plane
            // row. Direct rows: words staged in shared memory (XOR-swizzled),
            // then 16-byte stores, four lanes per 64-byte row segment.
            constexpr int NCB = BN / 4;              // column blocks
            const double s28 = ldexp(1.0, 28 - g.eC);
            const long long pstride = (long long)rc * ld;  // next slice of the same row
            uint32_t* Dg = reinterpret_cast<uint32_t*>(sgen + TL::CS_BYTES);  // [KS][BM][NCB]
            uint32_t sink = 0;
            const bool nost = (g.dbg_mode & 4) != 0;  // instrumentation: split without the stores
            for (int blk = et; blk < 32 * NCB; blk += EPI_THREADS) {
                const int rb = blk & 31, cb = blk >> 5;
                const int r0 = 4 * rb;
                if (r0 < dr0 && r0 < mr0) continue;
                uint32_t w[4][KS];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    double v4[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) v4[c] = Cs[(4 * cb + c) * CP + csr(r0 + q)];
#pragma unroll
                    for (int s2 = 0; s2 < KS; ++s2) w[q][s2] = 0u;
                    digits4(v4, s28, w[q]);
                }
                if (r0 >= dr0) {
                    const int sw = cb ^ (rb & (NCB - 1));
#pragma unroll
                    for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
                        for (int q = 0; q < 4; ++q) Dg[(s2 * BM + r0 + q) * NCB + sw] = w[q][s2];
                }
                if (r0 >= mr0) {
                    // plane-0 address of mirror row j0 + 4 cb, bytes i0 + r0..
                    int8_t* mp = g.Cd + prow(j0 + 4 * cb) * ld + i0 + r0;
#pragma unroll
                    for (int s2 = 0; s2 < KS; ++s2, mp += pstride) {
                        const uint32_t rows[4] = {w[0][s2], w[1][s2], w[2][s2], w[3][s2]};
                        uint32_t cols[4];
                        transpose4x4(rows, cols);
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            if (nost) { sink ^= cols[c]; continue; }
                            *reinterpret_cast<uint32_t*>(mp + c * ld) = cols[c];
                        }
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
            constexpr int NC4 = BN / 16;             // 16-byte chunks per row segment
            static_assert(EPI_THREADS % NC4 == 0, "read-back mapping");
            for (int rr = dr0 + et / NC4; rr < BM; rr += EPI_THREADS / NC4) {
                const int c4 = et % NC4;
                const int f = (rr >> 2) & (NCB - 1);
                const int k0 = (4 * c4) ^ f, k1 = (4 * c4 + 1) ^ f, k2 = (4 * c4 + 2) ^ f, k3 = (4 * c4 + 3) ^ f;
                const uint32_t* src = Dg + rr * NCB;
                int8_t* dp = g.Cd + prow(i0 + rr) * ld + j0 + 16 * c4;
#pragma unroll
                for (int s2 = 0; s2 < KS; ++s2, src += BM * NCB, dp += pstride) {
                    const uint4 v = make_uint4(src[k0], src[k1], src[k2], src[k3]);
                    if (nost) { sink ^= v.x ^ v.y ^ v.z ^ v.w; continue; }
                    *reinterpret_cast<uint4*>(dp) = v;
                }
            }
            if (nost && sink == 0x9E3779B9u) g.Cd[0] = 1;  // keep the split live
        } else if (g.Cd) {
            // digit planes staged in the TMA-store layout: direct boxes
            // [s][h] (tile rows BB h.., the BN columns) and mirror boxes [s][h]
            // (the BN tile columns as rows, tile rows BB h.. as bytes)
            uint8_t* dig = sgen + TL::CS_BYTES;
            const uint32_t dig_s = su32(dig);
            const double s28 = ldexp(1.0, 28 - g.eC);
            for (int it = et; it < BM * (BN / 16); it += EPI_THREADS) {  // direct items
                const int rr = it % BM, cc = it / BM;               // tile row, 16-column chunk
                if (rr < dr0) continue;
                uint32_t w[4][KS];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    double v4[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) v4[k] = Cs[(16 * cc + 4 * q4 + k) * CP + csr(rr)];
                    digits4(v4, s28, w[q4]);
                }
                const int h2 = rr / BB, rb = rr % BB;
#pragma unroll
                for (int s2 = 0; s2 < KS; ++s2) {
                    uint8_t* box = dig + (s2 * NBOX + h2) * TL::BOX_BYTES;
                    *reinterpret_cast<uint4*>(box + box_off<BB>(rb, cc)) =
                        make_uint4(w[0][s2], w[1][s2], w[2][s2], w[3][s2]);
                }
            }
            for (int it = et; it < BN * (BM / 16); it += EPI_THREADS) {  // mirror items
                const int j = it % BN, rc = it / BN;                  // tile column, 16-row chunk
                if (16 * rc < mr0) continue;
                uint32_t w[4][KS];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    double v4[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) v4[k] = Cs[j * CP + csr(16 * rc + 4 * q4 + k)];
                    digits4(v4, s28, w[q4]);
                }
                const int h2 = (16 * rc) / BB, cb = ((16 * rc) % BB) / 16;
#pragma unroll
                for (int s2 = 0; s2 < KS; ++s2) {
                    uint8_t* box = dig + (KS * NBOX + s2 * NBOX + h2) * TL::BOX_BYTES;
                    *reinterpret_cast<uint4*>(box + box_off<BB>(j, cb)) =
                        make_uint4(w[0][s2], w[1][s2], w[2][s2], w[3][s2]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
            if (et == 0) {
                const int base_row = mat * KS * ld;
                for (int s2 = 0; s2 < KS; ++s2) {
                    for (int h2 = dr0 / BB; h2 < NBOX; ++h2)
                        tma_store_2d(&mapC, dig_s + (s2 * NBOX + h2) * TL::BOX_BYTES, j0,
                                     base_row + s2 * ld + i0 + BB * h2);
                    for (int h2 = mr0 / BB; h2 < NBOX; ++h2)
                        tma_store_2d(&mapC, dig_s + (KS * NBOX + s2 * NBOX + h2) * TL::BOX_BYTES, i0 + BB * h2,
                                     base_row + s2 * ld + j0);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        }
        if (g.dbg_t) asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");  // warp-uniform
        if (g.dbg_t && et == 0) {
            long long* o = g.dbg_t + 8LL * (blockIdx.y * gridDim.x + blockIdx.x);
            o[0] = t_start;
            o[1] = t_setup;
            o[2] = t_full;
            o[3] = gtimer();
            o[4] = t_acc;
            o[5] = t_stage;
            o[6] = t_cst;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS)
                     : "memory");
    }
}


// ---------------------------------------------------------------------------
// Persistent variant (default): one CTA per SM walks 128 x 32 lower tiles of
// all matrices; TMEM holds two accumulator sets (2 x 8 groups x 32 columns),
// so the MMAs of the next tile run while the epilogue warps split and store
// the previous one. Per-element arithmetic is that of oz_gemm_kernel (same
// group order and FP64 operations): the outputs are bitwise identical.
namespace {
struct PT {
    static constexpr int BN = 32, BK = 64, STAGES = 2, R = BM / BN;
    // 8 epilogue warps: 320 threads x 96 registers leave room on the SM for a
    // concurrent trace-SLEM CTA (256 threads x 64 registers, 22 KB)
    static constexpr int EPI_WARPS = 8, EPI_THREADS = 32 * EPI_WARPS, THREADS = 64 + EPI_THREADS;
    static constexpr int HN = BN / (EPI_WARPS / 4);  // 16 columns per epilogue thread
    static constexpr int A_PLANE = BM * BK, B_PLANE = BN * BK;
    static constexpr int STAGE_BYTES = KS * (A_PLANE + B_PLANE);
    static constexpr int CP = BM + 1;
    static constexpr int CS_OFF = STAGES * STAGE_BYTES;            // FP64 staging [BN][CP]
    // digit words [KS][BM][BN/4] reuse the FP64 staging area once every
    // thread holds its 4 x 4 block in registers: 194 KB per CTA leaves room
    // on the SM for the trace-SLEM CTAs of the concurrent stream
    static constexpr int DG_OFF = CS_OFF;
    static_assert(KS * BM * (BN / 4) * 4 <= BN * CP * 8, "digit staging fits the FP64 staging");
    static constexpr int SMEM_BYTES = CS_OFF + BN * CP * 8 + 1024;
    static constexpr int ACC_COLS = KS * BN;                        // one accumulator set
    static_assert(2 * ACC_COLS <= 512, "two accumulator sets in TMEM");
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};
}  // namespace

// <= 152 registers: 320 x 152 + a trace-SLEM CTA (256 x 64) fit one SM's 64 K
__global__ void __maxnreg__(152)
    oz_gemm_pkernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    OzGemm g, int tiles_per_mat) {
    constexpr int BN = PT::BN, BK = PT::BK, STAGES = PT::STAGES, R = PT::R, HN = PT::HN, CP = PT::CP;
    constexpr int EPI_THREADS = PT::EPI_THREADS, EPI_WARPS = PT::EPI_WARPS;
    constexpr int A_PLANE = PT::A_PLANE, B_PLANE = PT::B_PLANE, STAGE_BYTES = PT::STAGE_BYTES;
    const int ld = g.ld;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nitems = tiles_per_mat * g.nmat;

    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[2 * STAGES + 4];
    __shared__ uint32_t tmem_slot;
    const uint32_t sbase = (su32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - su32(smem_raw));
    auto full_bar = [&](int s) { return su32(&bars[s]); };
    auto empty_bar = [&](int s) { return su32(&bars[STAGES + s]); };
    auto tfull_bar = [&](int b) { return su32(&bars[2 * STAGES + b]); };
    auto tempty_bar = [&](int b) { return su32(&bars[2 * STAGES + 2 + b]); };
    auto a_tile = [&](int st, int s) { return sbase + st * STAGE_BYTES + s * A_PLANE; };
    auto b_tile = [&](int st, int s) { return sbase + st * STAGE_BYTES + KS * A_PLANE + s * B_PLANE; };
    auto skip = [&](int mat) { return g.ictl && g.ictl[(mat >> 1) * 8 + 1]; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const int KB = ld / BK;

    if (warp == 0) {
        if (lane == 0) {
            int c = 0;
            for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
                const int mat = w / tiles_per_mat;
                if (skip(mat)) continue;
                int I, J;
                oz_tile(R, w - mat * tiles_per_mat, I, J);
                const long long plane_rows = (long long)mat * KS * ld;
                for (int kb = 0; kb < KB; ++kb, ++c) {
                    const int st = c % STAGES;
                    mbar_wait(empty_bar(st), ((c / STAGES) & 1) ^ 1);
                    mbar_expect_tx(full_bar(st), STAGE_BYTES);
#pragma unroll 1
                    for (int s = 0; s < KS; ++s) {
                        tma_load_2d(a_tile(st, s), &mapA, full_bar(st), kb * BK,
                                    (int)(plane_rows + (long long)s * ld + I * BM));
                        tma_load_2d(b_tile(st, s), &mapB, full_bar(st), kb * BK,
                                    (int)(plane_rows + (long long)s * ld + J * BN));
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int c = 0, tc = 0;
            for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
                if (skip(w / tiles_per_mat)) continue;
                const int buf = tc & 1, use = tc >> 1;
                mbar_wait(tempty_bar(buf), (use & 1) ^ 1);  // epilogue drained this set
                tc_fence_after();
                const uint32_t dbase = tmem + (uint32_t)(buf * PT::ACC_COLS);
                for (int kb = 0; kb < KB; ++kb, ++c) {
                    const int st = c % STAGES;
                    mbar_wait(full_bar(st), (c / STAGES) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk) {
#pragma unroll
                        for (int s = 1; s <= KS; ++s) {
                            // A_s . [B_1 | ... | B_{KS+1-s}] in one MMA (N = 32 (KS+1-s))
                            const uint64_t ad = op_desc<BK>(a_tile(st, s - 1) + kk * 32);
                            const uint64_t bd = op_desc<BK>(b_tile(st, 0) + kk * 32);
                            const uint32_t acc = (kb | kk) != 0 || s != 1;
                            mma_i8(dbase + (uint32_t)((s - 1) * BN), ad, bd, idesc_n(BN * (KS + 1 - s)), acc);
                        }
                    }
                    tc_commit(empty_bar(st));
                }
                tc_commit(tfull_bar(buf));
                ++tc;
            }
        }
    } else {
        const int q = warp & 3;                 // TMEM lane quarter of this warp
        const int h = (warp - 2) >> 2;          // column slice
        const int r = q * 32 + lane;            // tile row
        const int c0 = h * HN;
        const int et = threadIdx.x - 64;
        double* Cs = reinterpret_cast<double*>(sgen + PT::CS_OFF);
        uint32_t* Dg = reinterpret_cast<uint32_t*>(sgen + PT::DG_OFF);
        constexpr int NCB = BN / 4, NC4 = BN / 16;
        int tc = 0;
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            const int mat = w / tiles_per_mat;
            if (skip(mat)) continue;
            int I, J;
            oz_tile(R, w - mat * tiles_per_mat, I, J);
            const int i0 = I * BM, j0 = J * BN;
            const int buf = tc & 1, use = tc >> 1;
            ++tc;
            mbar_wait(tfull_bar(buf), use & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * PT::ACC_COLS + c0);
            double acc[HN];
#pragma unroll
            for (int j = 0; j < HN; ++j) acc[j] = 0.0;
            // group d = s + t sits at columns (d - 2) BN; smallest contributions first
#pragma unroll
            for (int d = KS + 1; d >= 2; d -= 2) {
                uint32_t v[2][HN];
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    if constexpr (HN == 8) {
                        tmem_ld8(taddr + (uint32_t)((d - q2 - 2) * BN), *reinterpret_cast<uint32_t(*)[8]>(v[q2]));
                    } else {
#pragma unroll
                        for (int c = 0; c < HN / 16; ++c)
                            tmem_ld16(taddr + (uint32_t)((d - q2 - 2) * BN + c * 16),
                                      *reinterpret_cast<uint32_t(*)[16]>(&v[q2][c * 16]));
                    }
                }
                tmem_wait_ld();
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    const double sc = ldexp(1.0, -7 * (d - q2));
#pragma unroll
                    for (int j = 0; j < HN; ++j) acc[j] = fma(i32_to_f64(v[q2][j]), sc, acc[j]);
                }
            }
            // this accumulator set is free for the tile after next
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar(buf)) : "memory");
            const double s = g.scale ? g.scale[mat] : 1.0;
            double alpha = g.alpha_c * spow(s, g.pa) * ldexp(1.0, g.eA + g.eB);
            const double beta = g.beta_c * spow(s, g.pb);
            if (g.sign_mode && (mat & 1) == 0) alpha = -alpha;
            const double* E = g.E ? g.E + (long long)mat * ld * ld : nullptr;
            const int i = i0 + r;
#pragma unroll
            for (int j = 0; j < HN; ++j) {
                double v = alpha * acc[j];
                if (E) v = fma(beta, __ldg(E + (long long)(j0 + c0 + j) * ld + i), v);
                if (i == j0 + c0 + j) v += g.dshift;
                acc[j] = v;
            }
            const int tdiag = J - R * I;
            const int dr0 = tdiag < 0 ? 0 : BN * tdiag;
            const int mr0 = tdiag < 0 ? 0 : BN * (tdiag + 1);
            // the previous tile's readers of Cs / Dg are done
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
#pragma unroll
            for (int j = 0; j < HN; ++j) Cs[(c0 + j) * CP + csr(r)] = acc[j];
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
            if (tdiag >= 0) {
                for (int idx = et; idx < BN * BN; idx += EPI_THREADS) {
                    const int u = idx / BN, v = idx % BN;
                    if (u < v) Cs[v * CP + csr(dr0 + u)] = Cs[u * CP + csr(dr0 + v)];
                }
                asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
            }
            if (g.C) {
                double* C = g.C + (long long)(mat >> 1) * g.c_stride_b + (long long)(mat & 1) * g.c_stride_w;
                const int nv = g.nvalid, ew = et >> 5;
                for (int rr = dr0 + ew; rr < BM; rr += EPI_WARPS) {
                    const int ii = i0 + rr, jj = j0 + lane;
                    if (lane < BN && ii < nv && jj < nv) C[(long long)ii * g.ldc + jj] = Cs[lane * CP + csr(rr)];
                }
                for (int j = ew; j < BN; j += EPI_WARPS) {
                    const int jj = j0 + j;
                    for (int rr = mr0 + lane; rr < BM; rr += 32) {
                        const int ii = i0 + rr;
                        if (ii < nv && jj < nv) C[(long long)jj * g.ldc + ii] = Cs[j * CP + csr(rr)];
                    }
                }
            }
            if (g.Cd) {
                const double s28 = ldexp(1.0, 28 - g.eC);
                int8_t* base = g.Cd + (long long)mat * KS * ld * ld;
                const long long pstride = (long long)ld * ld;
                static_assert(32 * NCB <= EPI_THREADS, "one 4 x 4 block per thread");
                const int rb = et & 31, cb = et >> 5;
                const int r0 = 4 * rb;
                const bool active = et < 32 * NCB && (r0 >= dr0 || r0 >= mr0);
                double bv[4][4];
                if (active) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
                        for (int c = 0; c < 4; ++c) bv[qq][c] = Cs[(4 * cb + c) * CP + csr(r0 + qq)];
                }
                // every block is in registers: Dg may now overwrite Cs
                asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
                if (active) {
                    uint32_t wd[4][KS];
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) digits4(bv[qq], s28, wd[qq]);
                    if (r0 >= dr0) {
                        const int sw = cb ^ (rb & (NCB - 1));
#pragma unroll
                        for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
                            for (int qq = 0; qq < 4; ++qq) Dg[(s2 * BM + r0 + qq) * NCB + sw] = wd[qq][s2];
                    }
                    if (r0 >= mr0) {
                        int8_t* mp = base + (long long)(j0 + 4 * cb) * ld + i0 + r0;
#pragma unroll
                        for (int s2 = 0; s2 < KS; ++s2, mp += pstride) {
                            const uint32_t rows[4] = {wd[0][s2], wd[1][s2], wd[2][s2], wd[3][s2]};
                            uint32_t cols[4];
                            transpose4x4(rows, cols);
#pragma unroll
                            for (int c = 0; c < 4; ++c) *reinterpret_cast<uint32_t*>(mp + c * ld) = cols[c];
                        }
                    }
                }
                asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
                for (int rr = dr0 + et / NC4; rr < BM; rr += EPI_THREADS / NC4) {
                    const int c4 = et % NC4;
                    const int f = (rr >> 2) & (NCB - 1);
                    const int k0 = (4 * c4) ^ f, k1 = (4 * c4 + 1) ^ f, k2 = (4 * c4 + 2) ^ f, k3 = (4 * c4 + 3) ^ f;
                    const uint32_t* src = Dg + rr * NCB;
                    int8_t* dp = base + (long long)(i0 + rr) * ld + j0 + 16 * c4;
#pragma unroll
                    for (int s2 = 0; s2 < KS; ++s2, src += BM * NCB, dp += pstride)
                        *reinterpret_cast<uint4*>(dp) = make_uint4(src[k0], src[k1], src[k2], src[k3]);
                }
            }
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
                                int e, int8_t* planes, const int* ictl, int rc) {
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
        const long long e0 = idx * 4;
        const int i = (int)(e0 / ld), c = (int)(e0 - (long long)i * ld);
        int8_t* o = out + ((long long)(i / rc) * KS * rc + i % rc) * ld + c;  // slice 0 (OzShard layout)
#pragma unroll
        for (int k = 0; k < KS; ++k) *reinterpret_cast<uint32_t*>(o + (long long)k * rc * ld) = w[k];
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

void encode(CUtensorMap* m, const int8_t* base, int ld, long long rows, int box_cols, int box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

}  // namespace

void make_oz_maps(const int8_t* planes, int ld, int nmat, OzMaps* out) {
    if (ld % BM != 0) throw Error(kInvalidArgument, "ozaki GEMM needs ld % 128 == 0");
    const long long rows = (long long)nmat * KS * ld;
    encode(&out->a, planes, ld, rows, TileL::BK, BM);
    encode(&out->b, planes, ld, rows, TileL::BK, TileL::BN);
    encode(&out->st, planes, ld, rows, TileL::BB, TileL::BB);
    encode(&out->a2, planes, ld, rows, TileS::BK, BM);
    encode(&out->b2, planes, ld, rows, TileS::BK, TileS::BN);
    encode(&out->st2, planes, ld, rows, TileS::BB, TileS::BB);
    encode(&out->bp, planes, ld, rows, 64, 32);
}

int oz_gemm_tiles(int ld) { return tiles_before(TileL::R, ld / BM); }

namespace {
// 128 x 32 tiles (two CTAs per SM) only on request (TPB_OZ_TILE=32): measured
// slower than 128 x 64 tiles even on multi-wave batched grids (n=256 x 384
// matrices: 24.5 vs 22.1 ms per projection) — the narrower MMAs' extra
// shared-memory traffic outweighs the epilogue overlap.
bool use_small_tiles(int, int) {
    static const bool on = [] {
        const char* e = std::getenv("TPB_OZ_TILE");
        return e && std::atoi(e) == 32;
    }();
    return on;
}
}  // namespace

bool cone_uses_ozaki() {
    const char* c = std::getenv("TPB_CONE");
    return !(c && std::strcmp(c, "dmma") == 0);
}

void init_attrs_ozaki() {
    TPB_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<TileL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  TileL::SMEM_BYTES));
    TPB_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<TileS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  TileS::SMEM_BYTES));
    TPB_CUDA(cudaFuncSetAttribute(oz_gemm_pkernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  PT::SMEM_BYTES));
}

namespace {
// Persistent 128 x 32 tiles with double-buffered TMEM (opt-in,
// TPB_OZ_PERSIST=1: ld <= 512, 2: always). Isolated digits-only products at
// ld <= 512 run faster (us: ld=256 x2 15.9 -> 11.0, x384 258.9 -> 226.5;
// ld=512 x2 21.5 -> 15.3, x64 202.6 -> 185.9), but the config-5 sweep is
// not: the resident grid keeps the concurrent trace-SLEM CTAs off the SMs
// and the denser tensor load meets the power cap (7.5 vs 8.3 solves/s, 26.3
// vs 25.5 ms per lockstep iteration of 192 het solves). At ld >= 1024 the
// half-width tiles' second read of the A planes costs more than the overlap
// saves (40.5 vs 35.0 us at n=1024).
bool use_persistent(int ld, int) {
    static const int mode = [] {
        const char* e = std::getenv("TPB_OZ_PERSIST");
        return e ? std::atoi(e) : 0;
    }();
    if (mode == 0) return false;
    if (mode == 2) return true;
    return ld <= 512;
}
}  // namespace

// Digit-plane output path: direct 16-byte global stores (default; the
// writes stream out during the split, -1 us per GEMM at n=1024) or, with
// TPB_OZ_DSTORE=0, TMA bulk stores of swizzled boxes staged in shared memory.
int dstore_mode() {
    static const int m = [] {
        const char* e = std::getenv("TPB_OZ_DSTORE");
        return e ? std::atoi(e) : 1;
    }();
    return m;
}

void launch_oz_gemm(const OzGemm& g0, cudaStream_t st) {
    OzGemm g = g0;
    g.dstore = dstore_mode();
    if (g.rc && g.rc != g.ld) g.dstore = 1;  // chunked planes: direct stores only
    if (g.Cd && !g.mc) throw Error(kInvalidArgument, "ozaki GEMM: digit output needs its TMA map");
    if (use_persistent(g.ld, g.nmat) && g.dstore && !g.dbg_t && !g.dbg_mode && !g.tiles && g.mstep <= 1 &&
        (!g.rc || g.rc == g.ld)) {
        const int tpm = tiles_before(PT::R, g.ld / BM);
        cudaLaunchConfig_t cfg{};
        // TPB_OZ_PGRID: SMs left free for concurrent streams (trace SLEM)
        static const int spare = [] {
            const char* e = std::getenv("TPB_OZ_PGRID");
            return e ? std::max(0, std::atoi(e)) : 0;
        }();
        cfg.gridDim = dim3(std::min(tpm * g.nmat, std::max(1, sm_count() - spare)));
        cfg.blockDim = dim3(PT::THREADS);
        cfg.dynamicSmemBytes = PT::SMEM_BYTES;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = g.no_pdl ? 0 : 1;
        TPB_CUDA(cudaLaunchKernelEx(&cfg, oz_gemm_pkernel, g.ma->a, g.mb->bp, g, tpm));
        return;
    }
    const bool small = use_small_tiles(g.ld, g.nmat) && !g.tiles;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g.tiles ? g.ntiles : small ? tiles_before(TileS::R, g.ld / BM) : oz_gemm_tiles(g.ld),
                       g.mstep > 1 ? (g.nmat - g.moff + g.mstep - 1) / g.mstep : g.nmat);
    cfg.blockDim = dim3(small ? TileS::THREADS : TileL::THREADS);
    cfg.dynamicSmemBytes = small ? TileS::SMEM_BYTES : TileL::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g.no_pdl ? 0 : 1;
    const OzMaps* mc = g.mc ? g.mc : g.mb;
    if (small)
        TPB_CUDA(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<TileS>, g.ma->a2, g.mb->b2, mc->st2, g));
    else
        TPB_CUDA(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<TileL>, g.ma->a, g.mb->b, mc->st, g));
}

void launch_oz_split(const double* A, long long mstride, int ld, int nmat, const double* scale, int e,
                     int8_t* planes, const int* ictl, cudaStream_t st, int rc) {
    const long long n4 = (long long)ld * ld / 4;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 1024);
    oz_split_kernel<<<dim3(blocks, nmat), 256, 0, st>>>(A, mstride, ld, scale, e, planes, ictl, rc ? rc : ld);
    TPB_CHECK_LAUNCH();
}

// The sign iteration rewritten so that every product but the last is a plain
// (scaled) product of two digit-plane operands plus a diagonal shift, with
// digit planes as its only output (no FP64 intermediates, no E reads):
//   inflation  X' = X (a + b X^2 + c X^4) = X Z',  Z' = c U^2 + gamma I,
//              U = X^2 + beta I,  beta = b / 2c,  gamma = a - b^2 / 4c
//   Newton-Schulz  X' = X V,  V = 1.5 I - 0.5 X^2
//   final      P = 0.5 A -/+ 0.5 A X = 0.5 A -/+ (0.5 / s) X0 X   (FP64 out)
// Static spectral bounds give the digit exponents: |X| <=
// 1.21, |U| <= 1.18, |V| <= 1.5 -> 2^1; |Z'| <= 3.45 -> 2^2; |X0| <= 1 -> 2^1.
namespace {
constexpr int kEX = 1, kEU = 1, kEZ = 2, kEV = 1, kEX0 = 1;
}

SignSchedule ozaki_schedule() {
    SignSchedule s;
    const char* e = std::getenv("TPB_SIGN_SCHEDULE");
    if (e && std::strcmp(e, "default") == 0) return s;
    s.k1 = 20;
    s.k2 = 6;
    s.qa = 3.73052;
    s.qb = -5.13486;
    s.qc = 2.0372;
    return s;
}

std::vector<int> oz_shard_tiles(int ld, int nranks, int rank) {
    const int NB = ld / BM, R = TileL::R;
    if (ld % BM || nranks < 1 || NB % nranks || rank < 0 || rank >= nranks)
        throw Error(kInvalidArgument, "sharded projection: ld/128 must be a multiple of the rank count");
    const int per = NB / nranks;
    std::vector<int> t;
    for (int I = rank * per; I < (rank + 1) * per; ++I) {
        for (int J = 0; J < R * (I + 1); ++J) t.push_back(tiles_before(R, I) + J);  // rows of block I
        for (int I2 = I + 1; I2 < NB; ++I2)                                         // mirrors into it
            for (int J = R * I; J < R * (I + 1); ++J) t.push_back(tiles_before(R, I2) + J);
    }
    // a tile below the diagonal inside the rank's rows serves both lists
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    return t;
}

namespace {
// in-place all-gather of the row blocks of every plane of the matrices
// moff, moff + 2, ... (one NCCL group)
void shard_allgather(const OzShard& sh, int8_t* planes, int ld, int nmat, int moff, cudaStream_t st) {
    // row-chunk-major planes: the rank's rows of all KS planes are one block
    const size_t count = (size_t)KS * (ld / sh.nranks) * ld;
    ncclComm_t comm = static_cast<ncclComm_t>(sh.comm);
    TPB_NCCL(nccl().group_start());
    for (int mat = moff; mat < nmat; mat += 2) {
        int8_t* base = planes + (size_t)mat * KS * ld * ld;
        TPB_NCCL(nccl().all_gather(base + (size_t)sh.rank * count, base, count, ncclInt8, comm, st));
    }
    TPB_NCCL(nccl().group_end());
}
}  // namespace

void enqueue_cone_ozaki(const double* A, double* /*w0*/, double* /*w1*/, double* /*w2*/, const OzWork& oz,
                        int ld, int n, const double* scale, double* C, long long c_stride_b,
                        long long c_stride_w, const int* ictl, int nmat, const SignSchedule& sch,
                        cudaStream_t st, const OzShard* shard) {
    const bool sharded = shard && shard->nranks > 1;
    const int rc = sharded ? ld / shard->nranks : 0;
    bool ag_pending[2] = {false, false};
    const long long ms = (long long)ld * ld;
    launch_oz_split(A, ms, ld, nmat, scale, kEX0, oz.d[3], ictl, st, rc);
    const double beta = sch.qb / (2.0 * sch.qc);
    const double gamma = sch.qa - sch.qb * sch.qb / (4.0 * sch.qc);
    OzGemm g{};
    g.ld = ld;
    g.nmat = nmat;
    g.scale = scale;
    g.ictl = ictl;
    g.rc = rc;
    // one product of digit buffers ia, ib into digit buffer od
    auto step = [&](int ia, int ea, int ib, int eb, double al, double shift, int od, int ec) {
        g.ma = &oz.maps[ia];
        g.mb = &oz.maps[ib];
        g.eA = ea;
        g.eB = eb;
        g.alpha_c = al;
        g.dshift = shift;
        g.Cd = oz.d[od];
        g.mc = &oz.maps[od];
        g.eC = ec;
        if (!sharded) {
            launch_oz_gemm(g, st);
            return;
        }
        // chain par's product waits for its operands' all-gather only; its
        // own all-gather then overlaps the other chain's GEMM
        g.tiles = shard->tiles;
        g.ntiles = shard->ntiles;
        g.no_pdl = 1;
        g.mstep = 2;
        for (int par = 0; par < 2; ++par) {
            if (ag_pending[par]) TPB_CUDA(cudaStreamWaitEvent(st, shard->ag_done[par], 0));
            g.moff = par;
            launch_oz_gemm(g, st);
            TPB_CUDA(cudaEventRecord(shard->gemm_done[par], st));
            TPB_CUDA(cudaStreamWaitEvent(shard->cs, shard->gemm_done[par], 0));
            shard_allgather(*shard, oz.d[od], ld, nmat, par, shard->cs);
            TPB_CUDA(cudaEventRecord(shard->ag_done[par], shard->cs));
            ag_pending[par] = true;
        }
    };
    int x = 3;  // digit buffer holding X (3: X0)
    auto others = [&](int& f0, int& f1) {
        int k = 0, fr[3];
        for (int q = 0; q < 3; ++q)
            if (q != x) fr[k++] = q;
        f0 = fr[0];
        f1 = fr[1];
    };
    for (int it = 0; it < sch.k1; ++it) {
        int u, z;
        others(u, z);
        step(x, kEX, x, kEX, 1.0, beta, u, kEU);      // U = X^2 + beta I
        step(u, kEU, u, kEU, sch.qc, gamma, z, kEZ);  // Z' = c U^2 + gamma I
        step(x, kEX, z, kEZ, 1.0, 0.0, u, kEX);       // X' = X Z'
        x = u;
    }
    for (int it = 0; it < sch.k2; ++it) {
        int v, xn;
        others(v, xn);
        step(x, kEX, x, kEX, -0.5, 1.5, v, kEV);      // V = 1.5 I - 0.5 X^2
        step(x, kEX, v, kEV, 1.0, 0.0, xn, kEX);      // X' = X V
        x = xn;
    }
    // P into the state blocks (column-major n x n == row-major by symmetry)
    g.ma = &oz.maps[3];
    g.mb = &oz.maps[x];
    g.eA = kEX0;
    g.eB = kEX;
    g.alpha_c = 0.5;
    g.pa = -1;
    g.dshift = 0.0;
    g.E = A;
    g.beta_c = 0.5;
    g.pb = 0;
    g.sign_mode = 1;
    g.C = C;
    g.c_stride_b = c_stride_b;
    g.c_stride_w = c_stride_w;
    g.ldc = n;
    g.nvalid = n;
    g.Cd = nullptr;
    g.mc = nullptr;
    g.tiles = nullptr;  // the FP64 product is replicated
    g.ntiles = 0;
    g.mstep = 0;
    g.moff = 0;
    g.no_pdl = 0;
    for (int par = 0; par < 2; ++par)
        if (ag_pending[par]) TPB_CUDA(cudaStreamWaitEvent(st, shard->ag_done[par], 0));
    launch_oz_gemm(g, st);
}

}  // namespace tpb
