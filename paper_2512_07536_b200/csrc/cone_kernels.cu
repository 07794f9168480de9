// PSD / NSD cone projections of the n x n slack blocks on the FP64 tensor
// pipe (DMMA, mma.sync.m8n8k4.f64). Replaces the reference's per-iteration
// eigen-clamps project_nsd(S) / project_psd(T) (proj/src/admm.cpp:96-112 ->
// clamp_spectrum, proj/src/eig.cpp:131-176: Householder tridiagonalisation +
// implicit QL + rank-1 rebuild, O(n^3) scalar code).
//
// tcgen05 has no FP64 kind; B200's FP64 tensor path is DMMA,
// measured at ~37 TFLOP/s (tools/microbench/fp64_peak.cu). The projection is
// a polynomial sign iteration (cone_kernels.cuh) whose every product is of
// commuting symmetric matrices, so only lower-triangular 64x64 tiles are
// computed (half the flops) and mirrored on store (exact symmetry, as the
// reference's symmetrize() gives).
#include "cone_kernels.cuh"

#include <algorithm>
#include <cstdlib>

namespace tpb {

namespace {

constexpr int BM = 64;        // tile edge

__device__ inline void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ inline void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ inline void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ inline void lower_tile(int t, int& bi, int& bj) {
    // t enumerates (bi >= bj): t = bi (bi+1)/2 + bj
    int b = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    while (b * (b + 1) / 2 > t) --b;
    bi = b;
    bj = t - b * (b + 1) / 2;
}

__device__ inline double powi(double s, int p) { return p == 0 ? 1.0 : (p == 1 ? s : s * s); }

}  // namespace

// 64x64 lower tile per CTA; WM x WN warps, each an (64/WM) x (64/WN) block of
// 8x8 DMMA fragments; BK-deep k stages, STG-stage cp.async pipeline.
template <int BK, int STG, int WM, int WN>
__global__ void __launch_bounds__(WM* WN * 32) sym_gemm_kernel(GemmArgs g) {
    constexpr int GT = WM * WN * 32;
    constexpr int PAD = BK + 4;  // smem row stride (doubles): conflict-free fragments
    constexpr int MI = 64 / WM / 8, NI = 64 / WN / 8;
    const int mat = blockIdx.y;
    if (g.ictl && g.ictl[(mat >> 1) * 8 + 1]) return;
    int bi, bj;
    lower_tile(blockIdx.x, bi, bj);
    const int i0 = bi * BM, j0 = bj * BM;
    const int ld = g.ld;
    const double* A = g.A + (long long)mat * g.mstride;
    const double* B = g.B + (long long)mat * g.mstride;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                       // STG x BM x PAD
    double* Bs = smem + STG * BM * PAD;      // STG x BM x PAD
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = (warp / WN) * (64 / WM), wc = (warp % WN) * (64 / WN);

    auto load_stage = [&](int slot, int kt) {
        const int k0 = kt * BK;
        double* as = As + slot * BM * PAD;
        double* bs = Bs + slot * BM * PAD;
        // 64 rows x BK/2 chunks of 16 B per panel
#pragma unroll
        for (int c = tid; c < BM * (BK / 2); c += GT) {
            const int r = c / (BK / 2), q = (c % (BK / 2)) * 2;
            cp_async16(as + r * PAD + q, A + (long long)(i0 + r) * ld + k0 + q);
            cp_async16(bs + r * PAD + q, B + (long long)(j0 + r) * ld + k0 + q);
        }
    };

    double acc[MI][NI][2];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
        for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    const int KT = ld / BK;
#pragma unroll
    for (int s = 0; s < STG - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
        cp_wait<STG - 2>();
        __syncthreads();
        const int nk = kt + STG - 1;
        if (nk < KT) load_stage(nk % STG, nk);
        cp_commit();
        const double* as = As + (kt % STG) * BM * PAD;
        const double* bs = Bs + (kt % STG) * BM * PAD;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double af[MI], bf[NI];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
                af[mi] = as[(wr + mi * 8 + (lane >> 2)) * PAD + ks * 4 + (lane & 3)];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                bf[ni] = bs[(wc + ni * 8 + (lane >> 2)) * PAD + ks * 4 + (lane & 3)];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_wait<0>();
    __syncthreads();

    // epilogue: C = alpha acc + beta E, staged through smem for the mirror store
    const double s = g.scale ? g.scale[mat] : 1.0;
    double alpha = g.alpha_c * powi(s, g.pa);
    const double beta = g.beta_c * powi(s, g.pb);
    if (g.sign_mode && (mat & 1) == 0) alpha = -alpha;
    const double* E = g.E ? g.E + (long long)mat * g.mstride : nullptr;
    double* Cs = smem;  // BM x (BM + 1)
    constexpr int CP = BM + 1;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            const int r = wr + mi * 8 + (lane >> 2);
            const int c = wc + ni * 8 + (lane & 3) * 2;
            double v0 = alpha * acc[mi][ni][0], v1 = alpha * acc[mi][ni][1];
            if (E) {
                const double* e = E + (long long)(i0 + r) * ld + j0 + c;
                v0 += beta * e[0];
                v1 += beta * e[1];
            }
            Cs[r * CP + c] = v0;
            Cs[r * CP + c + 1] = v1;
        }
    __syncthreads();
    double* C = g.C + (long long)(mat >> 1) * g.c_stride_b + (long long)(mat & 1) * g.c_stride_w;
    const int nv = g.nvalid;
    for (int idx = tid; idx < BM * BM; idx += GT) {
        const int r = idx / BM, c = idx % BM;
        const int i = i0 + r, j = j0 + c;
        if (i < nv && j < nv) {
            // diagonal tiles: take the lower-triangle value for exact symmetry
            const double v = (bi == bj && c > r) ? Cs[c * CP + r] : Cs[r * CP + c];
            C[(long long)i * g.ldc + j] = v;
        }
    }
    if (bi != bj) {
        for (int idx = tid; idx < BM * BM; idx += GT) {
            const int r = idx / BM, c = idx % BM;  // write (j0 + r, i0 + c) = Cs[c][r]
            const int i = j0 + r, j = i0 + c;
            if (i < nv && j < nv) C[(long long)i * g.ldc + j] = Cs[c * CP + r];
        }
    }
}

// ---------------------------------------------------------------- stream-K
// For a single large instance the 2 x T lower tiles of one (S, T) pair do not
// fill the GPU evenly (n=1024: 272 tiles on 148 SMs x 2 slots -> 10% tail).
// Stream-K splits the pair's 2 T KT k-iterations evenly over G CTAs; a tile
// cut between CTAs is finished by the CTA owning its last k-iteration, which
// adds the earlier pieces (published to `ws`, counted in `flags`) in CTA
// order — deterministic for a given (n, G). Each CTA walks its range from the
// top, so its only partial piece is produced first and its only waiting piece
// comes last: waits never chain.
template <int BK, int STG, int WM, int WN>
__global__ void __launch_bounds__(WM* WN * 32) sym_gemm_sk_kernel(GemmArgs g, int G, double* ws,
                                                                  int* flags) {
    constexpr int GT = WM * WN * 32;
    constexpr int PAD = BK + 4;
    constexpr int MI = 64 / WM / 8, NI = 64 / WN / 8;
    constexpr int NACC = MI * NI * 2;
    const int pair = blockIdx.y, c = blockIdx.x;
    if (g.ictl && g.ictl[pair * 8 + 1]) return;
    const int ld = g.ld;
    const int nt = ld / BM, T = nt * (nt + 1) / 2, KT = ld / BK;
    const long long U = 2LL * T * KT;
    auto start_of = [&](long long cc) { return cc * U / G; };
    const long long u0 = start_of(c), u1 = start_of(c + 1);
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STG * BM * PAD;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = (warp / WN) * (64 / WM), wc = (warp % WN) * (64 / WN);
    __shared__ int s_go;

    long long u = u1;
    while (u > u0) {
        const int tg = (int)((u - 1) / KT);       // tile within the pair
        const long long ts = (long long)tg * KT;
        const int kb = (int)(max(u0, ts) - ts), ke = (int)(u - ts);
        const int mat = 2 * pair + tg / T;
        int bi, bj;
        lower_tile(tg % T, bi, bj);
        const int i0 = bi * BM, j0 = bj * BM;
        const double* A = g.A + (long long)mat * g.mstride;
        const double* B = g.B + (long long)mat * g.mstride;
        auto load_stage = [&](int slot, int kt) {
            const int k0 = kt * BK;
            double* as = As + slot * BM * PAD;
            double* bs = Bs + slot * BM * PAD;
#pragma unroll
            for (int q = tid; q < BM * (BK / 2); q += GT) {
                const int r = q / (BK / 2), o = (q % (BK / 2)) * 2;
                cp_async16(as + r * PAD + o, A + (long long)(i0 + r) * ld + k0 + o);
                cp_async16(bs + r * PAD + o, B + (long long)(j0 + r) * ld + k0 + o);
            }
        };
        double acc[MI][NI][2];
#pragma unroll
        for (int a = 0; a < MI; ++a)
#pragma unroll
            for (int bb = 0; bb < NI; ++bb) acc[a][bb][0] = acc[a][bb][1] = 0.0;
        __syncthreads();  // smem reuse across pieces
#pragma unroll
        for (int s = 0; s < STG - 1; ++s) {
            if (kb + s < ke) load_stage(s, kb + s);
            cp_commit();
        }
        for (int kt = kb; kt < ke; ++kt) {
            cp_wait<STG - 2>();
            __syncthreads();
            const int nk = kt + STG - 1;
            if (nk < ke) load_stage((nk - kb) % STG, nk);
            cp_commit();
            const double* as = As + ((kt - kb) % STG) * BM * PAD;
            const double* bs = Bs + ((kt - kb) % STG) * BM * PAD;
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                double af[MI], bf[NI];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
                    af[mi] = as[(wr + mi * 8 + (lane >> 2)) * PAD + ks * 4 + (lane & 3)];
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
                    bf[ni] = bs[(wc + ni * 8 + (lane >> 2)) * PAD + ks * 4 + (lane & 3)];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            }
        }
        cp_wait<0>();
        __syncthreads();
        int* flag = flags + (long long)pair * 2 * T + tg;
        if (ke < KT) {
            // partial piece: publish, then count it
            double* dst = ws + ((long long)pair * G + c) * (BM * BM) + (long long)tid * NACC;
#pragma unroll
            for (int a = 0; a < MI; ++a)
#pragma unroll
                for (int bb = 0; bb < NI; ++bb) {
                    dst[(a * NI + bb) * 2] = acc[a][bb][0];
                    dst[(a * NI + bb) * 2 + 1] = acc[a][bb][1];
                }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(flag, 1);
        } else {
            if (kb > 0) {
                // final piece: wait for the earlier pieces, add them in CTA order
                long long cf = c;
                while (cf > 0 && start_of(cf) > ts) --cf;
                const int expect = (int)(c - cf);
                if (tid == 0) {
                    while (atomicAdd(flag, 0) < expect) __nanosleep(64);
                    s_go = 1;
                }
                __syncthreads();
                __threadfence();
                for (long long q = cf; q < c; ++q) {
                    const double* src = ws + ((long long)pair * G + q) * (BM * BM) + (long long)tid * NACC;
#pragma unroll
                    for (int a = 0; a < MI; ++a)
#pragma unroll
                        for (int bb = 0; bb < NI; ++bb) {
                            acc[a][bb][0] += __ldcg(src + (a * NI + bb) * 2);
                            acc[a][bb][1] += __ldcg(src + (a * NI + bb) * 2 + 1);
                        }
                }
                __syncthreads();
                if (tid == 0) *flag = 0;  // ready for the next launch
            }
            // epilogue (as in sym_gemm_kernel)
            const double s = g.scale ? g.scale[mat] : 1.0;
            double alpha = g.alpha_c * powi(s, g.pa);
            const double beta = g.beta_c * powi(s, g.pb);
            if (g.sign_mode && (mat & 1) == 0) alpha = -alpha;
            const double* E = g.E ? g.E + (long long)mat * g.mstride : nullptr;
            double* Cs = smem;
            constexpr int CP = BM + 1;
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int r = wr + mi * 8 + (lane >> 2);
                    const int cc = wc + ni * 8 + (lane & 3) * 2;
                    double v0 = alpha * acc[mi][ni][0], v1 = alpha * acc[mi][ni][1];
                    if (E) {
                        const double* e = E + (long long)(i0 + r) * ld + j0 + cc;
                        v0 += beta * e[0];
                        v1 += beta * e[1];
                    }
                    Cs[r * CP + cc] = v0;
                    Cs[r * CP + cc + 1] = v1;
                }
            __syncthreads();
            double* C = g.C + (long long)(mat >> 1) * g.c_stride_b + (long long)(mat & 1) * g.c_stride_w;
            const int nv = g.nvalid;
            for (int idx = tid; idx < BM * BM; idx += GT) {
                const int r = idx / BM, cc = idx % BM;
                const int i = i0 + r, j = j0 + cc;
                if (i < nv && j < nv) {
                    const double v = (bi == bj && cc > r) ? Cs[cc * CP + r] : Cs[r * CP + cc];
                    C[(long long)i * g.ldc + j] = v;
                }
            }
            if (bi != bj) {
                for (int idx = tid; idx < BM * BM; idx += GT) {
                    const int r = idx / BM, cc = idx % BM;
                    const int i = j0 + r, j = i0 + cc;
                    if (i < nv && j < nv) C[(long long)i * g.ldc + j] = Cs[cc * CP + r];
                }
            }
        }
        u = ts + kb;
    }
}

namespace {

template <int BK, int STG, int WM, int WN>
void launch_variant(const GemmArgs& g, int nmat, cudaStream_t st) {
    const int nt = g.ld / BM;
    const int tiles = nt * (nt + 1) / 2;
    const int smem = 2 * STG * BM * (BK + 4) * sizeof(double);
    sym_gemm_kernel<BK, STG, WM, WN><<<dim3(tiles, nmat), WM * WN * 32, smem, st>>>(g);
    TPB_CHECK_LAUNCH();
}

int g_gemm_variant = 0;  // production default (profiles/)

}  // namespace

int sym_gemm_variants() { return 4; }
void set_sym_gemm_variant(int v) { g_gemm_variant = v; }
int get_sym_gemm_variant() { return g_gemm_variant; }

int sm_count() {
    static int cached[64] = {};
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) dev = 63;
    if (!cached[dev]) TPB_CUDA(cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev));
    return cached[dev];
}

int stream_k_ctas(int ld) {
    // Measured slower than the tiled kernel at n=1024 (95 vs 83 us per GEMM,
    // profiles/README.md): opt-in only (TPB_STREAM_K=1) until tuned.
    static const bool enabled = std::getenv("TPB_STREAM_K") != nullptr;
    if (!enabled) return 0;
    const int nt = ld / BM, T = nt * (nt + 1) / 2, KT = ld / 16;
    const long long U = 2LL * T * KT;
    // worthwhile when one pair's tiles leave SM slots idle; >= 16 k-tiles per CTA
    if (2 * T >= 4 * sm_count() || ld < 512) return 0;
    return (int)std::min<long long>(2LL * sm_count(), U / 16);
}

void launch_sym_gemm(const GemmArgs& g, int nmat, cudaStream_t st) {
    if (g.sk_ws && nmat == 2 && g_gemm_variant == 0) {
        const int G = stream_k_ctas(g.ld);
        if (G > 0) {
            const int smem = 2 * 3 * BM * (16 + 4) * sizeof(double);
            sym_gemm_sk_kernel<16, 3, 2, 2><<<dim3(G, 1), 128, smem, st>>>(g, G, g.sk_ws, g.sk_flags);
            TPB_CHECK_LAUNCH();
            return;
        }
    }
    switch (g_gemm_variant) {
        case 1: launch_variant<32, 3, 2, 2>(g, nmat, st); break;   // 4 warps, BK 32
        case 2: launch_variant<16, 3, 2, 4>(g, nmat, st); break;   // 8 warps (32x16), BK 16
        case 3: launch_variant<32, 3, 2, 4>(g, nmat, st); break;   // 8 warps, BK 32
        default: launch_variant<16, 3, 2, 2>(g, nmat, st); break;  // 4 warps (32x32), BK 16
    }
}

void enqueue_cone_tiled(const double* A, double* w0, double* w1, double* w2, int ld, int n,
                        const double* scale, double* C, long long c_stride_b,
                        long long c_stride_w, const int* ictl, int nmat, const SignSchedule& sch,
                        cudaStream_t st, double* sk_ws, int* sk_flags) {
    const long long ms = (long long)ld * ld;
    GemmArgs g{};
    g.sk_ws = sk_ws;
    g.sk_flags = sk_flags;
    g.mstride = ms;
    g.ld = ld;
    g.scale = scale;
    g.ictl = ictl;
    g.ldc = ld;
    g.nvalid = ld;
    g.c_stride_b = 2 * ms;
    g.c_stride_w = ms;
    auto step = [&](const double* a, const double* b, const double* e, double* c, double al,
                    double be, int pa, int pb) {
        g.A = a;
        g.B = b;
        g.E = e;
        g.C = c;
        g.alpha_c = al;
        g.beta_c = be;
        g.pa = pa;
        g.pb = pb;
        launch_sym_gemm(g, nmat, st);
    };
    // X lives in one work buffer (or is A before the first step); each step
    // takes the two buffers X does not occupy.
    const double* X = A;  // X0 = s A: the scale is folded into alpha/beta powers
    double* bufs[3] = {w0, w1, w2};
    auto free_pair = [&](double*& f0, double*& f1) {
        int k = 0;
        double* fr[3];
        for (int q = 0; q < 3; ++q)
            if (bufs[q] != X) fr[k++] = bufs[q];
        f0 = fr[0];
        f1 = fr[1];
    };
    int first = 1;
    for (int it = 0; it < sch.k1; ++it) {
        double *Y, *Z;
        free_pair(Y, Z);
        step(X, X, nullptr, Y, 1.0, 0.0, first ? 2 : 0, 0);             // Y = X^2
        step(Y, Y, Y, Z, sch.qc, sch.qb, 0, 0);                          // Z = c Y^2 + b Y
        step(X, Z, X, Y, 1.0, sch.qa, first ? 1 : 0, first ? 1 : 0);     // X' = X Z + a X (into Y)
        X = Y;
        first = 0;
    }
    for (int it = 0; it < sch.k2; ++it) {
        double *Y, *Xn;
        free_pair(Y, Xn);
        step(X, X, nullptr, Y, 1.0, 0.0, first ? 2 : 0, 0);              // Y = X^2
        step(X, Y, X, Xn, -0.5, 1.5, first ? 1 : 0, first ? 1 : 0);      // X' = 1.5 X - 0.5 X Y
        X = Xn;
        first = 0;
    }
    // P = 0.5 A -/+ 0.5 A X into the state (column-major n x n == row-major by symmetry)
    g.ldc = n;
    g.nvalid = n;
    g.c_stride_b = c_stride_b;
    g.c_stride_w = c_stride_w;
    g.sign_mode = 1;
    step(A, X, A, C, 0.5, 0.5, 0, 0);
}

// ---------------------------------------------------------------- small n
// One CTA per matrix; all iterates in shared memory (npad <= 64).
namespace {
constexpr int ST = 256;  // 8 warps
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
            double d0 = 0.0, d1 = 0.0;
            for (int k = 0; k < np; k += 4) {
                const double av = a[(fi * 8 + (lane >> 2)) * P + k + (lane & 3)];
                const double bv = b[(fj * 8 + (lane >> 2)) * P + k + (lane & 3)];
                dmma(d0, d1, av, bv);
            }
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
    set_max_dyn_smem(sym_gemm_kernel<16, 3, 2, 2>);
    set_max_dyn_smem(sym_gemm_sk_kernel<16, 3, 2, 2>);
    set_max_dyn_smem(sym_gemm_kernel<32, 3, 2, 2>);
    set_max_dyn_smem(sym_gemm_kernel<16, 3, 2, 4>);
    set_max_dyn_smem(sym_gemm_kernel<32, 3, 2, 4>);
    set_max_dyn_smem(cone_small_kernel);
}

}  // namespace tpb
