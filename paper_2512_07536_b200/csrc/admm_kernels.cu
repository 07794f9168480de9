// ADMM iteration kernels: projection prep, closed-form x-step, dual update,
// residual and bookkeeping. All HBM-bound; tiles of 32 x 32 node pairs so the
// column-major S/T blocks are read once per orientation with coalesced rows.
//
// Reference mapping (all in /root/reference/proj):
//   prep            <- project_Y / project_Y_het first half (src/admm.cpp:268-277,
//                      src/admm_het.cpp:156-171): v = x + d/rho, clamps.
//   xstep a/node/b/diag <- update_X: kkt_rhs + bicgstab on [[I,A^T],[A,-1e-8 I]]
//                      (src/admm.cpp:175-182, 279-293; src/admm_het.cpp:270-280),
//                      solved here in closed form.
//   diag (tail)     <- update_duals + residual + trace + best iterate + stop test
//                      (src/admm.cpp:388-405, src/admm_het.cpp:281-300).
#include "admm_kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>

namespace tpb {

namespace cg = cooperative_groups;

namespace {

constexpr int TB = 32;  // tile edge
constexpr int TY = 8;   // threads in y

__device__ inline void tile_of(int t, int& bi, int& bj) {
    int b = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    while (b * (b + 1) / 2 > t) --b;
    bj = b;
    bi = t - b * (b + 1) / 2;
}

__device__ inline bool solve_done(const Dev& d, int b) { return d.ictl[b * 8 + kDone] != 0; }

// 2-D block (TB x TY) deterministic sum; every thread receives the result.
__device__ inline double block_sum_2d(double v, double* scratch) {
    const int t = threadIdx.y * TB + threadIdx.x;
    const int lane = t & 31, wid = t >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < TB * TY / 32; ++w) s += scratch[w];
    __syncthreads();
    return s;
}

// fixed-order total of `cnt` partials (identical in every CTA)
__device__ inline double sum_tiles(const double* P, int cnt, double* scratch) {
    const int t = threadIdx.y * TB + threadIdx.x;
    constexpr int NT = TB * TY, NP = 4;
    double v = 0.0;
    if (cnt <= NP * NT) {
        // all loads in flight together, summed in the same k order
        double q[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) q[j] = t + j * NT < cnt ? P[t + j * NT] : 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j)
            if (t + j * NT < cnt) v += q[j];
    } else {
        for (int k = t; k < cnt; k += NT) v += P[k];
    }
    return block_sum_2d(v, scratch);
}

// fixed-order warp sum of `cnt` partials: lane sums k = lane, lane + 32, ...
// in k order (loads issued together), then the warp tree
__device__ inline double warp_sum_partials(const double* P, int cnt, int lane) {
    constexpr int NP = 17;  // ntile <= 544 (n <= 1056)
    double v = 0.0;
    if (cnt <= NP * 32) {
        double q[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) q[j] = lane + j * 32 < cnt ? P[lane + j * 32] : 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j)
            if (lane + j * 32 < cnt) v += q[j];
    } else {
        for (int k = lane; k < cnt; k += 32) v += P[k];
    }
    return warp_sum(v);
}

// Arrival of a finished tile at the node blocks it touches (bi and bj):
// after a CTA barrier thread 0 fences (release, cumulative over the CTA's
// stores) and adds one arrival per block.
// Returns the blocks whose last tile this CTA was (bit 0: bi, bit 1: bj);
// the completer resets the counter for the next launch.
__device__ inline int arrive_blocks(int* cnt, int nb, int bi, int bj, int* s_flag) {
    __syncthreads();  // the CTA's stores precede thread 0's release fence (cumulative)
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence();
        int fin = 0;
        if (atomicAdd(cnt + bi, 1) == nb - 1) {
            atomicExch(cnt + bi, 0);
            fin |= 1;
        }
        if (bi != bj && atomicAdd(cnt + bj, 1) == nb - 1) {
            atomicExch(cnt + bj, 0);
            fin |= 2;
        }
        *s_flag = fin;
    }
    __syncthreads();
    const int fin = *s_flag;
    if (fin) __threadfence();
    return fin;
}

// Arrival of a completed node block at the solve counter: true in the CTA
// that completed the solve's last block (all nb of them).
__device__ inline bool arrive_solve(int* cnt, int nb, int* s_flag) {
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence();
        const bool last = atomicAdd(cnt, 1) == nb - 1;
        if (last) atomicExch(cnt, 0);
        *s_flag = last ? 1 : 0;
    }
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

// Node sums over the nb tile partials P[q][k n + i] (K arrays) for the 32
// nodes of block `blk`: warp w sums k = w, w + TY, ... in k order (all
// loads of a batch in flight together), warp 0 adds the TY warp partials in
// warp order. Valid in warp 0 (0 for i >= n). `pre` runs between the loads
// and the barrier (warp 0 can issue its own independent loads there).
template <int K, class Pre>
__device__ inline void node_sum(const double* const (&P)[K], int nb, int n, int blk, double (*sm)[TY][TB + 1],
                                double (&out)[K], Pre pre) {
    const int tx = threadIdx.x, ty = threadIdx.y, i = blk * TB + tx;
    double v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = 0.0;
    if (i < n) {
        constexpr int NQ = 8 / K;
        int k = ty;
        for (; k + (NQ - 1) * TY < nb; k += NQ * TY) {
            double x[K][NQ];
#pragma unroll
            for (int q = 0; q < K; ++q)
#pragma unroll
                for (int u = 0; u < NQ; ++u) x[q][u] = __ldcg(P[q] + (long long)(k + u * TY) * n + i);
#pragma unroll
            for (int q = 0; q < K; ++q)
#pragma unroll
                for (int u = 0; u < NQ; ++u) v[q] += x[q][u];
        }
        for (; k < nb; k += TY)
#pragma unroll
            for (int q = 0; q < K; ++q) v[q] += __ldcg(P[q] + (long long)k * n + i);
    }
    pre();
#pragma unroll
    for (int q = 0; q < K; ++q) sm[q][ty][tx] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double s = 0.0;
        if (ty == 0) {
#pragma unroll
            for (int y = 0; y < TY; ++y) s += sm[q][y][tx];
        }
        out[q] = s;
    }
    __syncthreads();
}

// Fixed-order sums of two values over the CTA (warp trees, then warps in
// order); every thread receives them.
__device__ inline void block_sum2_2d(double& a, double& b, double (*scratch)[2]) {
    const int t = threadIdx.y * TB + threadIdx.x;
    const int lane = t & 31, wid = t >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if (lane == 0) {
        scratch[wid][0] = a;
        scratch[wid][1] = b;
    }
    __syncthreads();
    a = b = 0.0;
#pragma unroll
    for (int w = 0; w < TB * TY / 32; ++w) {
        a += scratch[w][0];
        b += scratch[w][1];
    }
    __syncthreads();
}

}  // namespace

XConst make_xconst(int n, double alpha, double rho) {
    XConst c{};
    const double delta = kKktShift;
    const double s = 1.0 / (1.0 + delta);
    c.rho = rho;
    c.inv_rho = 1.0 / rho;
    c.alpha = alpha;
    c.alpha_over_n = alpha / n;
    c.delta = delta;
    c.s = s;
    c.lam_den = 1.0 + 2.0 * n * s;
    // homogeneous H_gg = a I + b K, f(k) = 1/(a + b k)
    const double a = 1.0 + 4.0 * s, b = 3.0 * s;
    const double qp = n - 2.0, q1 = 2.0 * n - 2.0;
    c.f0 = 1.0 / a;
    c.c1 = -b / (a * (a + b * qp));
    c.c2 = -b / (a * (a + b * q1));
    // heterogeneous node-level
    const double a1 = 1.0 + 5.0 * s, b1 = 3.0 * s, a2 = 1.0 + s;
    auto det = [&](double k) { return (a1 + b1 * k) * a2 - s * s; };
    const double d0 = det(0), dp = det(qp), d1 = det(q1);
    c.g11_0 = a2 / d0;
    c.g12_0 = s / d0;
    c.g22_0 = a1 / d0;
    c.c1_11 = -b1 * a2 * a2 / (dp * d0);
    c.c2_11 = -b1 * a2 * a2 / (d1 * d0);
    c.c1_12 = -b1 * s * a2 / (dp * d0);
    c.c2_12 = -b1 * s * a2 / (d1 * d0);
    c.c1_22 = -b1 * s * s / (dp * d0);
    c.c2_22 = -b1 * s * s / (d1 * d0);
    c.g12_p = s / dp;
    c.g22_p = (a1 + b1 * qp) / dp;
    c.g12_1 = s / d1;
    c.g22_1 = (a1 + b1 * q1) / d1;
    c.mu_den_p = qp * c.g22_p + delta;
    c.mu_den_1 = q1 * c.g22_1 + delta;
    c.cg_a = a;
    c.cg_b = b;
    return c;
}

// ---------------------------------------------------------------- prep
#ifdef OZ_STAMPS
// instrumentation build only (make STAMPS=1): globaltimer stamps per CTA of
// the tile kernels (prep, passes A and B), 16 slots
__device__ long long* g_tile_stamps = nullptr;
__device__ __forceinline__ void tile_stamp(int slot) {
    if (!g_tile_stamps || threadIdx.x || threadIdx.y) return;
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tile_stamps[16LL * (blockIdx.y * gridDim.x + blockIdx.x) + slot] = t;
}
extern "C" int tp_tile_set_stamps(void* dev_ptr) {
    return cudaMemcpyToSymbol(g_tile_stamps, &dev_ptr, sizeof(void*)) == cudaSuccess ? 0 : 7;
}
#define TILE_STAMP(slot) tile_stamp(slot)
#else
#define TILE_STAMP(slot) do {} while (0)
#endif

// Block (bi <= bj) of node pairs. Writes A_S/A_T = sym(v) in both triangles of
// the ld-padded buffers, clamps the packed edge blocks for pairs in the tile,
// and the per-node blocks (lambda, y) from tile 0.
__global__ void __launch_bounds__(TB* TY, 4) prep_kernel(Dev d, XConst c) {
    // programmatic dependent of the best-iterate copy (the launch overlaps
    // its tail), which has read the improved flag: cleared here for every
    // solve, done or not
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int b = blockIdx.y;
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) d.ictl[b * 8 + kImproved] = 0;
    if (solve_done(d, b)) return;
    int bi, bj;
    tile_of(blockIdx.x, bi, bj);
    const Layout& lo = d.lo;
    const int n = lo.n;
    const double* X = d.X + (long long)b * d.nx;
    const double* D = d.D + (long long)b * d.nx;
    double* Y = d.Y + (long long)b * d.nx;
    const long long ld2 = (long long)d.ld * d.ld;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i0 = bi * TB, j0 = bj * TB;
    __shared__ double red[TB * TY / 32];
    double fro[2] = {0.0, 0.0};
    TILE_STAMP(0);

    for (int which = 0; which < 2; ++which) {
        const int off = which == 0 ? lo.off_s : lo.off_t;
        double* A = d.A + ((long long)b * 2 + which) * ld2;
        __shared__ double Vs[TB][TB + 1];  // Vs[jl][il] = v(i0+il, j0+jl)
        // both orientations' X and D loads are issued before any use (their
        // HBM latencies overlap): orientation 1 = entries (i, j) at j*n + i,
        // orientation 2 = entries (j, i) at i*n + j
        constexpr int NE = TB / TY;
        double x1[NE], d1[NE], x2[NE], d2[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int cc = ty + k * TY;
            const int i = i0 + tx, j = j0 + cc;
            if (i < n && j < n) {
                const long long p = off + (long long)j * n + i;
                x1[k] = X[p];
                d1[k] = D[p];
            }
            const int j2 = j0 + tx, i2 = i0 + cc;
            if (i2 < n && j2 < n) {
                const long long p = off + (long long)i2 * n + j2;
                x2[k] = X[p];
                d2[k] = D[p];
            }
        }
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int cc = ty + k * TY;
            const int i = i0 + tx, j = j0 + cc;
            Vs[cc][tx] = (i < n && j < n) ? x1[k] + d1[k] * c.inv_rho : 0.0;
        }
        __syncthreads();
        // orientation 2: symmetrize with (i, j)
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int cc = ty + k * TY;
            const int j = j0 + tx, i = i0 + cc;  // entry (row j, col i)
            if (i < n && j < n) {
                const double vji = x2[k] + d2[k] * c.inv_rho;
                const double vij = Vs[tx][cc];
                const double a = 0.5 * (vij + vji);  // symmetrize (proj/src/eig.cpp:157)
                // A is symmetric: entry (i, j) of the row-major buffer, lanes
                // along the row (coalesced)
                A[(long long)i * d.ld + j] = a;
                Vs[tx][cc] = a;  // hand (i, j) to the mirrored write below
                const double w = (bi == bj) ? (i == j ? 1.0 : (j > i ? 2.0 : 0.0)) : 2.0;
                fro[which] += w * a * a;
            }
        }
        __syncthreads();
        // |A| row-sum partials (for ||A||_inf): rows of block bi over the
        // columns of block bj and, off the diagonal, rows of bj over bi;
        // fixed-order sums (lanes: warp tree; rows: ascending)
        {
            double* rp = d.row_part + ((long long)b * 2 + which) * d.nb * n;
            for (int cc = ty; cc < TB; cc += TY) {  // row i0 + cc over columns j0 + tx
                const double v = warp_sum(fabs(Vs[tx][cc]));
                if (tx == 0 && i0 + cc < n) rp[(long long)bj * n + i0 + cc] = v;
            }
            if (bi != bj && ty == 0) {  // row j0 + tx over columns i0 + cc
                double v = 0.0;
                for (int cc = 0; cc < TB; ++cc) v += fabs(Vs[tx][cc]);
                if (j0 + tx < n) rp[(long long)bi * n + j0 + tx] = v;
            }
        }
        __syncthreads();
        if (bi != bj) {
            // the mirror (j, i), j in block bj: rows j0 + cc, lanes along them
            for (int cc = ty; cc < TB; cc += TY) {
                const int i = i0 + tx, j = j0 + cc;
                if (i < n && j < n) A[(long long)j * d.ld + i] = Vs[cc][tx];
            }
        }
        __syncthreads();
        TILE_STAMP(1 + which);
    }
    // packed edge blocks for pairs (i, j), i < j, i in block bi, j in block bj
    // (the g loads of the thread's rows in flight together)
    {
        constexpr int NE = TB / TY;
        double xg[NE], dg[NE];
        long long lg[NE];
        bool okg[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int i = i0 + ty + k * TY, j = j0 + tx;
            okg[k] = i < n && j < n && j > i;
            lg[k] = okg[k] ? edge_idx(n, i, j) : 0;
            if (okg[k]) {
                xg[k] = X[lg[k]];
                dg[k] = D[lg[k]];
            }
        }
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            if (!okg[k]) continue;
            const double vg = xg[k] + dg[k] * c.inv_rho;
            Y[lg[k]] = (0.0 < vg) ? vg : 0.0;  // std::max(0.0, v) (proj/src/admm.cpp:273)
        }
    }
    for (int il = ty; il < TB && d.het; il += TY) {
        const int i = i0 + il, j = j0 + tx;
        if (i >= n || j >= n || j <= i) continue;
        const long long l = edge_idx(n, i, j);
        {
            const long long lz = lo.off_z + l, lv = lo.off_nu + l;
            Y[lz] = X[lz] + D[lz] * c.inv_rho;  // z-score; binary projection follows
            const double vn = X[lv] + D[lv] * c.inv_rho;
            Y[lv] = (0.0 < vn) ? vn : 0.0;
        }
    }
    TILE_STAMP(3);
    if (blockIdx.x == 0) {
        const int t = ty * TB + tx;
        if (t == 0) {
            const double vl = X[lo.lambda_ix] + D[lo.lambda_ix] * c.inv_rho;
            Y[lo.lambda_ix] = (0.0 < vl) ? vl : 0.0;
        }
        for (int i = t; i < n; i += TB * TY) {
            const double vy = X[lo.off_y + i] + D[lo.off_y + i] * c.inv_rho;
            Y[lo.off_y + i] = (0.0 < vy) ? vy : 0.0;
        }
    }
    // deterministic per-tile Frobenius partials
    for (int which = 0; which < 2; ++which) {
        double* part = d.frob_part + ((long long)b * 2 + which) * d.ntile;
        // block sum over 2D block: flatten thread id
        double v = fro[which];
        const int lane = (ty * TB + tx) & 31, wid = (ty * TB + tx) >> 5;
        v = warp_sum(v);
        __syncthreads();
        if (lane == 0) red[wid] = v;
        __syncthreads();
        if (ty == 0 && tx == 0) {
            double s = 0.0;
            for (int w = 0; w < TB * TY / 32; ++w) s += red[w];
            part[blockIdx.x] = s;
        }
        __syncthreads();
    }
    // the last tile of a node block: max |A| row sum of the block's rows; the
    // last block of the solve: 1 / min(||A||_F, ||A||_inf) per matrix
    __shared__ int s_fin;
    __shared__ double sm8[2][TY][TB + 1];
    int* cnt = d.cnt + (long long)b * d.cnt_stride;
    TILE_STAMP(4);
    const int fin = arrive_blocks(cnt + kCntP * d.nb, d.nb, bi, bj, &s_fin);
    TILE_STAMP(5);
    if (!fin) return;
    bool last = false;
    for (int q = 0; q < 2; ++q) {
        if (!(fin >> q & 1)) continue;
        const int k = q == 0 ? bi : bj;
        const double* const rp[2] = {d.row_part + (long long)b * 2 * d.nb * n,
                                     d.row_part + ((long long)b * 2 + 1) * d.nb * n};
        double rs[2];
        node_sum<2>(rp, d.nb, n, k, sm8, rs, [] {});
        if (ty == 0) {
            const double m0 = warp_max(rs[0]), m1 = warp_max(rs[1]);
            if (tx == 0) {
                d.blk_inf[(long long)b * 2 * d.nb + k] = m0;
                d.blk_inf[((long long)b * 2 + 1) * d.nb + k] = m1;
            }
        }
        last |= arrive_solve(cnt + 2 * d.nb + kCntP, d.nb, &s_fin);
    }
    TILE_STAMP(6);
    if (!last) return;
    const int t = ty * TB + tx;
    double f0 = 0.0, f1 = 0.0, inf = 0.0;
    {
        const double* p0 = d.frob_part + (long long)b * 2 * d.ntile;
        for (int k = t; k < d.ntile; k += TB * TY) {
            f0 += __ldcg(p0 + k);
            f1 += __ldcg(p0 + d.ntile + k);
        }
        if (ty < 2) {
            const double* bm = d.blk_inf + ((long long)b * 2 + ty) * d.nb;
            for (int k = tx; k < d.nb; k += TB) inf = fmax(inf, __ldcg(bm + k));
            inf = warp_max(inf);
        }
    }
    block_sum2_2d(f0, f1, reinterpret_cast<double (*)[2]>(&sm8[0][0]));
    if (ty < 2 && tx == 0) {
        const double cc = fmin(sqrt(ty == 0 ? f0 : f1), inf);
        d.inv_scale[b * 2 + ty] = cc > 0.0 ? 1.0 / cc : 0.0;
    }
    TILE_STAMP(7);
}

// launch as a programmatic dependent of the previous kernel in the stream
// (the kernel calls griddepcontrol.wait before touching memory)
template <class K, class... Args>
void launch_dependent(K kernel, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TPB_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

void launch_prep(const Dev& d, const XConst& c, cudaStream_t st) {
    launch_dependent(prep_kernel, dim3(d.ntile, d.B), dim3(TB, TY), st, d, c);
}


// ---------------------------------------------------------------- x-step A
// h_g(i,j) = r_g + s (4 - R_ii - R_jj + R_ij + R_ji + v2_i + v2_j) [- s r_nu]
// with r = Y - (D + c)/rho, R = r_S + r_T, v2 = 1 - r_y.
__global__ void __launch_bounds__(TB* TY, 4) xstep_a_kernel(Dev d, XConst c) {
    // pass B (launched as a programmatic dependent) may be scheduled now; it
    // waits for this grid's completion before it touches memory
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int b = blockIdx.y;
    if (solve_done(d, b)) return;
    int bi, bj;
    tile_of(blockIdx.x, bi, bj);
    const Layout& lo = d.lo;
    const int n = lo.n;
    const double* Y = d.Y + (long long)b * d.nx;
    const double* D = d.D + (long long)b * d.nx;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i0 = bi * TB, j0 = bj * TB;
    __shared__ double Rs[TB][TB + 1];  // Rs[il][jl] = R(i,j) + R(j,i)
    __shared__ double Hs[TB][TB + 1];  // Hs[il][jl] = h(i,j) (valid for pairs)
    __shared__ double Zs[TB][TB + 1];  // het: h_z'(i,j)
    __shared__ double rd_i[TB], rd_j[TB], v2_i[TB], v2_j[TB];
    TILE_STAMP(8);

    auto rS = [&](long long p) { return Y[lo.off_s + p] - D[lo.off_s + p] * c.inv_rho; };
    auto rT = [&](long long p) { return Y[lo.off_t + p] - D[lo.off_t + p] * c.inv_rho; };
    constexpr int NE = TB / TY;
    // the NE entries a thread owns per orientation: all 4 NE loads are issued
    // before any use, so their HBM latencies overlap
    auto load_r = [&](const long long (&pos)[NE], const bool (&ok)[NE], double (&out)[NE]) {
        double ys[NE], ds[NE], yt[NE], dt[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            if (!ok[k]) continue;
            ys[k] = Y[lo.off_s + pos[k]];
            ds[k] = D[lo.off_s + pos[k]];
            yt[k] = Y[lo.off_t + pos[k]];
            dt[k] = D[lo.off_t + pos[k]];
        }
#pragma unroll
        for (int k = 0; k < NE; ++k)
            out[k] = ok[k] ? (ys[k] - ds[k] * c.inv_rho) + (yt[k] - dt[k] * c.inv_rho) : 0.0;
    };
    // diagonals and v2 of both node blocks: issued first, so their latency
    // overlaps the block loads instead of following them
    double dgi = 0.0, dgj = 0.0, v2vi = 0.0, v2vj = 0.0, rsi = 0.0, rti = 0.0;
    if (ty == 0) {
        const int i = i0 + tx, j = j0 + tx;
        if (i < n) {
            const long long p = (long long)i * n + i;
            rsi = rS(p);
            rti = rT(p);
            dgi = rsi + rti;
            v2vi = 1.0 - (Y[lo.off_y + i] - D[lo.off_y + i] * c.inv_rho);
        }
        if (j < n) {
            const long long p = (long long)j * n + j;
            dgj = rS(p) + rT(p);
            v2vj = 1.0 - (Y[lo.off_y + j] - D[lo.off_y + j] * c.inv_rho);
        }
    }
    // both orientations' loads are issued before any use: orientation 1
    // R(i, j) at j*n + i, orientation 2 R(j, i) at i*n + j
    long long pos1[NE], pos2[NE];
    bool ok1[NE], ok2[NE];
    double v1[NE], v2o[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const int a = i0 + tx, bcol = j0 + ty + k * TY;
        ok1[k] = a < n && bcol < n;
        pos1[k] = (long long)bcol * n + a;
        const int j = j0 + tx, i = i0 + ty + k * TY;
        ok2[k] = i < n && j < n;
        pos2[k] = (long long)i * n + j;
    }
    load_r(pos1, ok1, v1);
    load_r(pos2, ok2, v2o);
    // hom: the thread's edge loads (h over the tile's pairs, packed index
    // contiguous in j) are issued together with the block loads
    double rg_pre[NE];
    if (!d.het) {
        long long lp[NE];
        bool okp[NE];
        double yg[NE], dg[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int i = i0 + ty + k * TY, j = j0 + tx;
            okp[k] = i < n && j < n && j > i;
            lp[k] = okp[k] ? edge_idx(n, i, j) : 0;
            if (okp[k]) {
                yg[k] = Y[lp[k]];
                dg[k] = D[lp[k]];
            }
        }
#pragma unroll
        for (int k = 0; k < NE; ++k) rg_pre[k] = okp[k] ? yg[k] - dg[k] * c.inv_rho : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) Rs[tx][ty + k * TY] = v1[k];
    if (ty == 0) {
        rd_i[tx] = dgi;
        v2_i[tx] = v2vi;
        rd_j[tx] = dgj;
        v2_j[tx] = v2vj;
    }
    __syncthreads();
    // orientation 2 (loaded above)
#pragma unroll
    for (int k = 0; k < NE; ++k)
        if (ok2[k]) Rs[ty + k * TY][tx] += v2o[k];
    __syncthreads();
    for (int il = ty; il < TB; il += TY) {
        const int i = i0 + il, jl = tx, j = j0 + jl;
        double hv = 0.0, hz = 0.0;
        if (i < n && j < n && j > i) {
            const long long l = edge_idx(n, i, j);
            const double rg = d.het ? Y[l] - D[l] * c.inv_rho : rg_pre[(il - ty) / TY];
            hv = rg + c.s * (4.0 - rd_i[il] - rd_j[jl] + Rs[il][jl] + v2_i[il] + v2_j[jl]);
            if (d.het) {
                const long long lz = lo.off_z + l, lv = lo.off_nu + l;
                const double rnu = Y[lv] - D[lv] * c.inv_rho;
                const double rz = Y[lz] - D[lz] * c.inv_rho;
                hv -= c.s * rnu;
                hz = rz + c.s * rnu;
            }
            d.h[(long long)b * lo.m + l] = hv;
        }
        Hs[il][jl] = hv;
        if (d.het) Zs[il][jl] = hz;
    }
    __syncthreads();
    if (d.cg) {
        // |h|^2 partial of the tile: r_0 = h for the CG x-step
        __shared__ double red[TB * TY / 32];
        double hh = 0.0;
        for (int il = ty; il < TB; il += TY) hh += Hs[il][tx] * Hs[il][tx];
        hh = block_sum_2d(hh, red);
        if (ty == 0 && tx == 0) d.cg_rr[(long long)b * 2 * d.ntile + blockIdx.x] = hh;
    }
    // node partials: PU[bj][i] = row sums of the tile (rows of block bi),
    // PU[bi][j] = column sums (cols of block bj); on a diagonal tile h sits
    // in the upper triangle only (zeros elsewhere), so node i's sum there is
    // row i + column i. All warps reduce: warp ty owns rows ty + k*TY (warp
    // sum over the lanes), lane tx accumulates column tx over those rows.
    __shared__ double rowp[2][TB];
    __shared__ double colp[2][TY][TB + 1];
    {
        double cu = 0.0, cz = 0.0;
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int il = ty + k * TY;
            const double hv = Hs[il][tx];
            cu += hv;
            const double ru = warp_sum(hv);
            if (tx == 0) rowp[0][il] = ru;
            if (d.het) {
                const double hz = Zs[il][tx];
                cz += hz;
                const double rz = warp_sum(hz);
                if (tx == 0) rowp[1][il] = rz;
            }
        }
        colp[0][ty][tx] = cu;
        colp[1][ty][tx] = cz;
    }
    __syncthreads();
    const int t = ty * TB + tx;
    double* PU = d.PU + (long long)b * d.nb * n;
    double* PZ = d.PZ + (long long)b * d.nb * n;
    auto colsum = [&](int which, int l) {
        double s = 0.0;
#pragma unroll
        for (int y = 0; y < TY; ++y) s += colp[which][y][l];
        return s;
    };
    // node partials, and their tile totals (sum u = 2 sum h) for pass B's
    // node-space solve: warp 0 the rows, warp 1 the columns
    double pu = 0.0, pz = 0.0;
    if (t < TB) {
        const int il = t, i = i0 + il;
        if (i < n) {
            pu = rowp[0][il] + (bi == bj ? colsum(0, il) : 0.0);
            PU[(long long)bj * n + i] = pu;
            if (d.het) {
                pz = rowp[1][il] + (bi == bj ? colsum(1, il) : 0.0);
                PZ[(long long)bj * n + i] = pz;
            }
        }
    } else if (t < 2 * TB && bi != bj) {
        const int jl = t - TB, j = j0 + jl;
        if (j < n) {
            pu = colsum(0, jl);
            PU[(long long)bi * n + j] = pu;
            if (d.het) {
                pz = colsum(1, jl);
                PZ[(long long)bi * n + j] = pz;
            }
        }
    }
    __shared__ double s_tot[2][2];
    if (ty < 2) {
        const double a0 = warp_sum(pu), a1 = warp_sum(pz);
        if (tx == 0) {
            s_tot[ty][0] = a0;
            s_tot[ty][1] = a1;
        }
    }
    // diagonal tiles: tr r_S, tr r_T and the degree targets over the block
    double4 bk = make_double4(0.0, 0.0, 0.0, 0.0);
    if (bi == bj && ty == 0) {
        const int i = i0 + tx;
        const double dg = d.het && i < n ? d.deg[(long long)b * n + i] : 0.0;
        bk = make_double4(warp_sum(rsi), warp_sum(rti), warp_sum(dg), 0.0);
    }
    __syncthreads();
    if (t == 0) {
        double* ta = d.tile_aux + ((long long)b * d.ntile + blockIdx.x) * 2;
        ta[0] = s_tot[0][0] + s_tot[1][0];
        ta[1] = s_tot[0][1] + s_tot[1][1];
        if (bi == bj) reinterpret_cast<double4*>(d.blk)[(long long)b * d.nb + bi] = bk;
    }
    TILE_STAMP(9);
}

void launch_xstep_a(const Dev& d, const XConst& c, cudaStream_t st) {
    dim3 grid(d.ntile, d.B), block(TB, TY);
    xstep_a_kernel<<<grid, block, 0, st>>>(d, c);
    TPB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- CG x-step
// The paper's linear substep as matrix-free CG on the g block of the reduced
// KKT system: H_gg = (1 + 4s) I + 3s D^T D, applied as one
// node-sum scatter (u = D p, fixed-order tile partials) and one per-edge
// gather (u_i + u_j). On the complete candidate graph H_gg has three
// eigenvalues, so CG stops after three iterations at ~1e-15; the closed form
// (pass B's node-space prologue) is the default and this path is its
// operator-level cross-check and the general-graph formulation.

namespace {

// node partials of a tile's packed values Vs (pairs il < jl on diagonal tiles):
// 4 adjacent lanes per node sum interleaved quarters, then two shuffles
__device__ inline void tile_node_partials(const double (&Vs)[TB][TB + 1], int bi, int bj, int n, double* P) {
    const int t = threadIdx.y * TB + threadIdx.x;
    const int i0 = bi * TB, j0 = bj * TB;
    const int nl = t >> 2, part = t & 3;
    double s = 0.0;
    bool valid = false;
    if (nl < TB) {
        const int il = nl;
        valid = i0 + il < n;
#pragma unroll
        for (int q = 0; q < TB / 4; ++q) {
            const int jl = part + 4 * q;
            if (bi == bj) {
                if (jl != il) s += jl > il ? Vs[il][jl] : Vs[jl][il];
            } else {
                s += Vs[il][jl];
            }
        }
    } else if (bi != bj) {
        const int jl = nl - TB;
        valid = j0 + jl < n;
#pragma unroll
        for (int q = 0; q < TB / 4; ++q) s += Vs[part + 4 * q][jl];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (part == 0 && valid) {
        if (nl < TB)
            P[(long long)bj * n + i0 + nl] = s;
        else
            P[(long long)bi * n + j0 + nl - TB] = s;
    }
}

}  // namespace

// One persistent cooperative grid runs the whole CG solve: the CTAs stride
// over the (solve, tile) work items; per iteration a direction
// pass (beta, u = D p from node partials, p = r + beta p, p.Hp partials) and
// an update pass (alpha, x += alpha p, r -= alpha Hp, |r|^2 and D r
// partials), separated by grid-wide barriers. Every CTA derives the
// per-solve scalars itself from the fixed-order partials (a warp per solve),
// so the decisions are identical everywhere without extra barriers, and the
// result is bitwise reproducible. The loop ends when every solve has stopped.
__global__ void __launch_bounds__(TB* TY, 4) xstep_cg_kernel(Dev d, XConst c) {
    cg::grid_group grid = cg::this_grid();
    const Layout& lo = d.lo;
    const int n = lo.n;
    const int nitems = d.B * d.ntile;
    const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TB + tx;
    const int lane = t & 31, warp = t >> 5;
    constexpr int NR_ = TB / TY, NW = TB * TY / 32;
    __shared__ double scratch[NW];
    __shared__ double ui[TB], uj[TB];
    __shared__ double Rs[TB][TB + 1];
    __shared__ int s_any;
    extern __shared__ double dyn[];  // per solve: rr0, rr_k, beta | active flags
    double* s_rr0 = dyn;
    double* s_rrk = dyn + d.B;
    double* s_beta = dyn + 2 * d.B;
    int* s_act = reinterpret_cast<int*>(dyn + 3 * d.B);

    // fixed-order warp sum of one solve's tile partials
    auto wsum = [&](const double* P) { return warp_sum_partials(P, d.ntile, lane); };

    for (int k = 0; k <= d.cg_max; ++k) {
        // ---- per-solve scalars (every CTA; warp per solve)
        for (int b = warp; b < d.B; b += NW) {
            const double* RR = d.cg_rr + (long long)b * 2 * d.ntile;
            const bool was = k == 0 ? !solve_done(d, b) : s_act[b] != 0;
            double rr1 = 0.0;
            if (k == 0) {
                rr1 = wsum(RR);  // |h|^2 (pass A)
                if (lane == 0) s_rr0[b] = rr1;
            } else if (was) {
                rr1 = wsum(RR + d.ntile);  // |r_k|^2 (update pass k-1)
            }
            if (lane == 0) {
                bool act = was;
                if (was) {
                    const double rr0 = s_rr0[b];
                    const bool conv = k == 0 ? !(rr0 > 0.0) : rr1 <= d.cg_tol2 * rr0;
                    if (conv || k == d.cg_max) {
                        act = false;
                        if (blockIdx.x == 0) {
                            d.ictl[b * 8 + kCgIters] = k;
                            d.scal[b * 8 + kCgRes] = rr0 > 0.0 ? sqrt(rr1 / rr0) : 0.0;
                            // the reference's guard after its linear solve (admm.cpp:287):
                            // sticky, raised by the host after the chunk
                            if (rr0 > 0.0 && !(rr1 <= 1e-16 * rr0)) d.ictl[b * 8 + kCgFail] = 1;
                        }
                    }
                    s_beta[b] = k == 0 ? 0.0 : rr1 / s_rrk[b];
                    s_rrk[b] = rr1;
                }
                s_act[b] = act;
            }
        }
        __syncthreads();
        if (t == 0) {
            int any = 0;
            for (int b = 0; b < d.B && !any; ++b) any = s_act[b];
            s_any = any;
        }
        __syncthreads();
        if (!s_any) break;  // uniform: every CTA computed the same flags

        // ---- direction pass
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            const int b = w / d.ntile, tile = w - b * d.ntile;
            if (!s_act[b]) continue;
            const double beta = s_beta[b];
            int bi, bj;
            tile_of(tile, bi, bj);
            const int i0 = bi * TB, j0 = bj * TB;
            const double* NRp = k == 0 ? d.PU + (long long)b * d.nb * n : d.cg_nr + (long long)b * d.nb * n;
            const double* Uprev = d.cg_u + ((long long)b * 2 + ((k - 1) & 1)) * n;
            double* Ucur = d.cg_u + ((long long)b * 2 + (k & 1)) * n;
            {
                // u of the tile's 64 nodes: 4 threads per node (adjacent
                // lanes) sum interleaved quarters of the nb node partials
                const int nl = t >> 2, part = t & 3;
                const int node = nl < TB ? i0 + nl : j0 + nl - TB;
                double u = 0.0;
                if (node < n) {
                    int q = part;
                    for (; q + 12 < d.nb; q += 16) {
                        double v[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) v[j] = NRp[(long long)(q + 4 * j) * n + node];
#pragma unroll
                        for (int j = 0; j < 4; ++j) u += v[j];
                    }
                    for (; q < d.nb; q += 4) u += NRp[(long long)q * n + node];
                }
                u += __shfl_xor_sync(0xffffffffu, u, 1);
                u += __shfl_xor_sync(0xffffffffu, u, 2);
                if (part == 0 && node < n) {
                    if (k > 0) u += beta * Uprev[node];
                    if (bi == bj && nl < TB) Ucur[node] = u;  // one diagonal tile per node block
                }
                if (part == 0) {
                    if (nl < TB) ui[nl] = u; else uj[nl - TB] = u;
                }
            }
            __syncthreads();
            const double* R = d.h + (long long)b * lo.m;
            double* P = d.cg_p + (long long)b * lo.m;
            long long l[NR_];
            bool ok[NR_];
            double rv[NR_], pv[NR_];
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                const int i = i0 + ty + q * TY, j = j0 + tx;
                ok[q] = i < n && j < n && j > i;
                l[q] = ok[q] ? edge_idx(n, i, j) : 0;
                if (ok[q]) {
                    rv[q] = R[l[q]];
                    pv[q] = k == 0 ? 0.0 : P[l[q]];
                }
            }
            double pq = 0.0;
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                if (!ok[q]) continue;
                const double p = rv[q] + beta * pv[q];
                P[l[q]] = p;
                pq += p * (c.cg_a * p + c.cg_b * (ui[ty + q * TY] + uj[tx]));
            }
            pq = block_sum_2d(pq, scratch);  // (its barriers also retire ui/uj)
            if (t == 0) d.cg_pq[w] = pq;
        }
        grid.sync();

        // ---- update pass
        int alpha_b = -1;
        double alpha = 0.0;
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            const int b = w / d.ntile, tile = w - b * d.ntile;
            if (!s_act[b]) continue;
            if (b != alpha_b) {
                const double pq = sum_tiles(d.cg_pq + (long long)b * d.ntile, d.ntile, scratch);
                alpha = pq > 0.0 ? s_rrk[b] / pq : 0.0;
                alpha_b = b;
            }
            int bi, bj;
            tile_of(tile, bi, bj);
            const int i0 = bi * TB, j0 = bj * TB;
            const double* U = d.cg_u + ((long long)b * 2 + (k & 1)) * n;
            if (t < TB) ui[t] = i0 + t < n ? U[i0 + t] : 0.0;
            else if (t < 2 * TB) uj[t - TB] = j0 + t - TB < n ? U[j0 + t - TB] : 0.0;
            __syncthreads();
            double* R = d.h + (long long)b * lo.m;
            double* X = d.cg_x + (long long)b * lo.m;
            const double* P = d.cg_p + (long long)b * lo.m;
            long long l[NR_];
            bool ok[NR_];
            double rv[NR_], pv[NR_], xv[NR_];
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                const int i = i0 + ty + q * TY, j = j0 + tx;
                ok[q] = i < n && j < n && j > i;
                l[q] = ok[q] ? edge_idx(n, i, j) : 0;
                if (ok[q]) {
                    rv[q] = R[l[q]];
                    pv[q] = P[l[q]];
                    xv[q] = k == 0 ? 0.0 : X[l[q]];
                }
            }
            double rr = 0.0;
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                double r = 0.0;
                if (ok[q]) {
                    const double hp = c.cg_a * pv[q] + c.cg_b * (ui[ty + q * TY] + uj[tx]);
                    X[l[q]] = xv[q] + alpha * pv[q];
                    r = rv[q] - alpha * hp;
                    R[l[q]] = r;
                    rr += r * r;
                }
                Rs[ty + q * TY][tx] = r;
            }
            __syncthreads();
            tile_node_partials(Rs, bi, bj, n, d.cg_nr + (long long)b * d.nb * n);
            rr = block_sum_2d(rr, scratch);  // (its barriers also retire ui/uj/Rs)
            if (t == 0) d.cg_rr[((long long)b * 2 + 1) * d.ntile + tile] = rr;
        }
        grid.sync();
    }
}

// Register-resident variant: when every (solve, tile) item gets its own
// co-resident CTA, each thread keeps its edges' x, r and p in registers and
// the tile's node values u in shared memory for the whole solve; between the
// phases global memory carries only the per-tile and node partials. The
// tile's node partials are prefetched before the scalar sums, so a phase is
// one L2 round trip plus the grid barrier (instead of re-reading r, p, x and
// u). Same arithmetic and reduction order as xstep_cg_kernel: bitwise
// identical results (tested).
constexpr int kCgRegNb = 32;  // node blocks the per-thread prefetch covers (n <= 1024)

__global__ void __launch_bounds__(TB* TY, 4) xstep_cg_reg_kernel(Dev d, XConst c) {
    cg::grid_group grid = cg::this_grid();
    const Layout& lo = d.lo;
    const int n = lo.n;
    const int nitems = d.B * d.ntile;
    const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TB + tx;
    const int lane = t & 31, warp = t >> 5;
    constexpr int NR_ = TB / TY, NW = TB * TY / 32, NQ = (kCgRegNb + 3) / 4;
    __shared__ double scratch[NW];
    __shared__ double ui[TB], uj[TB];
    __shared__ double Rs[TB][TB + 1];
    __shared__ int s_any;
    extern __shared__ double dyn[];  // per solve: rr0, rr_k, beta | active flags
    double* s_rr0 = dyn;
    double* s_rrk = dyn + d.B;
    double* s_beta = dyn + 2 * d.B;
    int* s_act = reinterpret_cast<int*>(dyn + 3 * d.B);

    // this CTA's item (CTAs past the last item only take part in the barriers)
    const int w = blockIdx.x;
    const bool own = w < nitems;
    const int b = own ? w / d.ntile : 0, tile = own ? w - b * d.ntile : 0;
    int bi = 0, bj = 0;
    if (own) tile_of(tile, bi, bj);
    const int i0 = bi * TB, j0 = bj * TB;
    int l[NR_];  // packed edge index (m < 2^31 here)
    bool ok[NR_];
    double xv[NR_], rv[NR_], pv[NR_];
#pragma unroll
    for (int q = 0; q < NR_; ++q) {
        const int i = i0 + ty + q * TY, j = j0 + tx;
        ok[q] = own && i < n && j < n && j > i;
        l[q] = ok[q] ? (int)edge_idx(n, i, j) : 0;
        rv[q] = ok[q] ? d.h[(long long)b * lo.m + l[q]] : 0.0;  // r_0 = h (pass A)
        pv[q] = 0.0;
        xv[q] = 0.0;
    }
    // node of the u sums: 4 threads per node, as in xstep_cg_kernel
    const int nl = t >> 2, part = t & 3;
    const int node = nl < TB ? i0 + nl : j0 + nl - TB;
    const bool node_ok = own && node < n;
    double uprev = 0.0;  // the node's u of the previous direction (part 0)
    bool ran = false;

    auto wsum = [&](const double* P) { return warp_sum_partials(P, d.ntile, lane); };

    for (int k = 0; k <= d.cg_max; ++k) {
        // prefetch the tile's node partials of r_k (independent of the scalars)
        const double* NRp = k == 0 ? d.PU + (long long)b * d.nb * n : d.cg_nr + (long long)b * d.nb * n;
        double nv[NQ];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const int q = part + 4 * j;
            nv[j] = (node_ok && q < d.nb) ? NRp[(long long)q * n + node] : 0.0;
        }
        // ---- per-solve scalars (every CTA; warp per solve)
        for (int bb = warp; bb < d.B; bb += NW) {
            const double* RR = d.cg_rr + (long long)bb * 2 * d.ntile;
            const bool was = k == 0 ? !solve_done(d, bb) : s_act[bb] != 0;
            double rr1 = 0.0;
            if (k == 0) {
                rr1 = wsum(RR);
                if (lane == 0) s_rr0[bb] = rr1;
            } else if (was) {
                rr1 = wsum(RR + d.ntile);
            }
            if (lane == 0) {
                bool act = was;
                if (was) {
                    const double rr0 = s_rr0[bb];
                    const bool conv = k == 0 ? !(rr0 > 0.0) : rr1 <= d.cg_tol2 * rr0;
                    if (conv || k == d.cg_max) {
                        act = false;
                        if (blockIdx.x == 0) {
                            d.ictl[bb * 8 + kCgIters] = k;
                            d.scal[bb * 8 + kCgRes] = rr0 > 0.0 ? sqrt(rr1 / rr0) : 0.0;
                            // the reference's guard after its linear solve (admm.cpp:287):
                            // sticky, raised by the host after the chunk
                            if (rr0 > 0.0 && !(rr1 <= 1e-16 * rr0)) d.ictl[bb * 8 + kCgFail] = 1;
                        }
                    }
                    s_beta[bb] = k == 0 ? 0.0 : rr1 / s_rrk[bb];
                    s_rrk[bb] = rr1;
                }
                s_act[bb] = act;
            }
        }
        __syncthreads();
        if (t == 0) {
            int any = 0;
            for (int bb = 0; bb < d.B && !any; ++bb) any = s_act[bb];
            s_any = any;
        }
        __syncthreads();
        if (!s_any) break;  // uniform: every CTA computed the same flags
        const bool act = own && s_act[b];

        // ---- direction phase: u = D r_k + beta u_{k-1}, p = r + beta p
        if (act) {
            const double beta = s_beta[b];
            double u = 0.0;
#pragma unroll
            for (int j = 0; j < NQ; ++j)
                if (part + 4 * j < d.nb) u += nv[j];  // q order of xstep_cg_kernel
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            u += __shfl_xor_sync(0xffffffffu, u, 2);
            if (part == 0 && node_ok) {
                if (k > 0) u += beta * uprev;
                uprev = u;
            }
            if (part == 0) {
                if (nl < TB) ui[nl] = u; else uj[nl - TB] = u;
            }
            __syncthreads();
            double pq = 0.0;
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                if (!ok[q]) continue;
                const double p = rv[q] + beta * pv[q];
                pv[q] = p;
                pq += p * (c.cg_a * p + c.cg_b * (ui[ty + q * TY] + uj[tx]));
            }
            pq = block_sum_2d(pq, scratch);
            if (t == 0) d.cg_pq[w] = pq;
        }
        grid.sync();

        // ---- update phase: x += alpha p, r -= alpha Hp, |r|^2 and D r partials
        if (act) {
            ran = true;
            const double pq = sum_tiles(d.cg_pq + (long long)b * d.ntile, d.ntile, scratch);
            const double alpha = pq > 0.0 ? s_rrk[b] / pq : 0.0;
            double rr = 0.0;
#pragma unroll
            for (int q = 0; q < NR_; ++q) {
                double r = 0.0;
                if (ok[q]) {
                    const double hp = c.cg_a * pv[q] + c.cg_b * (ui[ty + q * TY] + uj[tx]);
                    xv[q] = xv[q] + alpha * pv[q];
                    r = rv[q] - alpha * hp;
                    rv[q] = r;
                    rr += r * r;
                }
                Rs[ty + q * TY][tx] = r;
            }
            __syncthreads();
            tile_node_partials(Rs, bi, bj, n, d.cg_nr + (long long)b * d.nb * n);
            rr = block_sum_2d(rr, scratch);
            if (t == 0) d.cg_rr[((long long)b * 2 + 1) * d.ntile + tile] = rr;
        }
        grid.sync();
    }
    // x for pass B; r back into h, where xstep_cg_kernel leaves it
    if (ran) {
#pragma unroll
        for (int q = 0; q < NR_; ++q) {
            if (!ok[q]) continue;
            d.cg_x[(long long)b * lo.m + l[q]] = xv[q];
            d.h[(long long)b * lo.m + l[q]] = rv[q];
        }
    }
}

size_t cg_dyn_smem(const Dev& d) { return (size_t)d.B * (3 * sizeof(double) + sizeof(int)); }

namespace {
int cg_capacity(const void* kernel, const Dev& d) {
    int dev = 0, sms = 0, per_sm = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, TB * TY, cg_dyn_smem(d)));
    return std::max(1, sms * per_sm);
}
}  // namespace

// Launch shape of the CG x-step for this solver's device and batch (set once
// per solver in Dev::cg_grid; 0 ... register-resident kernel, one CTA per
// (solve, tile) item, when every item fits one co-resident CTA).
int cg_launch_grid(const Dev& d) {
    if (d.nb <= kCgRegNb && (long long)d.B * d.ntile <= cg_capacity((const void*)xstep_cg_reg_kernel, d))
        return -d.B * d.ntile;  // negative: register kernel
    return std::max(1, std::min(cg_capacity((const void*)xstep_cg_kernel, d), d.B * d.ntile));
}

void launch_xstep_cg(const Dev& d, const XConst& c, cudaStream_t st) {
    const bool reg = d.cg_grid < 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(reg ? -d.cg_grid : d.cg_grid);
    cfg.blockDim = dim3(TB, TY);
    cfg.stream = st;
    cfg.dynamicSmemBytes = cg_dyn_smem(d);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (reg)
        TPB_CUDA(cudaLaunchKernelEx(&cfg, xstep_cg_reg_kernel, d, c));
    else
        TPB_CUDA(cudaLaunchKernelEx(&cfg, xstep_cg_kernel, d, c));
}

// ---------------------------------------------------------------- x-step B
// Node-space part of the closed form for node blocks bi and bj (DESIGN.md
// §3.3/§3.4), formed by every pass-B CTA from pass A's partials: the totals
// of u = D h (and u_z) from the per-tile sums, the traces and degree totals
// from the diagonal tiles (fixed order, identical in every CTA), u_i from
// the nb node partials (four k-strided groups, added in group order).
//   hom: t = c1 (u - ubar) + c2 ubar
//   het: rhs = G21(Q) u_g + G22(Q) u_z - e with Q = (n-2) I + J, whose mean
//        is g12(2n-2) ubar + g22(2n-2) zbar - mean(e), so mean(mu_d) =
//        mean(rhs) / mu_den_1 and u_z'' = u_z - Q mu_d in closed form.
// Leaves nv[q][0..2][lane] (het: t_g, t_z, mu_d of block q; hom: t, u = D h
// and the total of t) and, in thread 0, returns lambda. Ends with a CTA
// barrier.
__device__ double node_space(const Dev& d, const XConst& c, int b, int bi, int bj, double (*nv)[3][TB],
                             double (*sp)[2][4][TB], double (*scr)[2]) {
    const Layout& lo = d.lo;
    const int n = lo.n;
    const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TB + tx;
    // per-tile totals (thread-strided, then the CTA tree)
    double su = 0.0, sz = 0.0;
    const double* ta = d.tile_aux + (long long)b * d.ntile * 2;
    for (int k = t; k < d.ntile; k += TB * TY) {
        su += ta[2 * k];
        sz += ta[2 * k + 1];
    }
    // node partials of the two blocks: warp w takes block w & 1, partials
    // k = w >> 1, (w >> 1) + 4, ...
    const int q = ty & 1, g = ty >> 1;
    const int i = (q ? bj : bi) * TB + tx;
    double pu = 0.0, pz = 0.0;
    if (i < n) {
        const double* PU = d.PU + (long long)b * d.nb * n;
        const double* PZ = d.PZ + (long long)b * d.nb * n;
        for (int k = g; k < d.nb; k += 4) {
            pu += PU[(long long)k * n + i];
            if (d.het) pz += PZ[(long long)k * n + i];
        }
    }
    // traces and degree totals of the diagonal tiles (warps 0 and 1 alike)
    double trS = 0.0, trT = 0.0, sdeg = 0.0;
    if (ty < 2) {
        const double4* bk = reinterpret_cast<const double4*>(d.blk) + (long long)b * d.nb;
        for (int k = tx; k < d.nb; k += TB) {
            const double4 v = bk[k];
            trS += v.x;
            trT += v.y;
            sdeg += v.z;
        }
        trS = warp_sum(trS);
        trT = warp_sum(trT);
        sdeg = warp_sum(sdeg);
    }
    sp[q][0][g][tx] = pu;
    sp[q][1][g][tx] = pz;
    block_sum2_2d(su, sz, scr);  // barriers: sp is visible after
    double lam = 0.0;
    if (t == 0) {
        const double rl = d.Y[(long long)b * d.nx + lo.lambda_ix] - d.D[(long long)b * d.nx + lo.lambda_ix] * c.inv_rho +
                          c.inv_rho;  // +1/rho: c = -1 at lambda
        lam = (rl + c.s * (c.alpha + trS + 2.0 * n - trT)) / c.lam_den;
    }
    if (ty < 2) {
        const double ubar = su / n;
        double u = 0.0, uz = 0.0;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
            u += sp[ty][0][gg][tx];
            uz += sp[ty][1][gg][tx];
        }
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        const double pg = u - ubar;
        if (!d.het) {
            v0 = c.c1 * pg + c.c2 * ubar;
            v1 = u;               // (D h)_i and sum_k t_k = c2 n ubar: the closed-form
            v2 = c.c2 * su;       // node degrees of pass B's diagonal tiles
        } else {
            const double zbar = sz / n;
            double z2bar = zbar, uz2 = uz;
            if (!d.cap && i < n) {
                const double rbar = c.g12_1 * ubar + c.g22_1 * zbar - sdeg / n;
                const double mbar = rbar / c.mu_den_1, smu = n * mbar;
                const double rhs = c.g12_p * pg + c.g12_1 * ubar + c.g22_p * (uz - zbar) + c.g22_1 * zbar -
                                   d.deg[(long long)b * n + i];
                v2 = (rhs - rbar) / c.mu_den_p + mbar;
                uz2 = uz - (n - 2.0) * v2 - smu;
                z2bar = zbar - (n - 2.0) * mbar - smu;
            }
            const double pz = uz2 - z2bar;
            v0 = c.c1_11 * pg + c.c2_11 * ubar + c.c1_12 * pz + c.c2_12 * z2bar;
            v1 = c.c1_12 * pg + c.c2_12 * ubar + c.c1_22 * pz + c.c2_22 * z2bar;
        }
        if (i >= n) v0 = v1 = v2 = 0.0;
        nv[ty][0][tx] = v0;
        nv[ty][1][tx] = v1;
        nv[ty][2][tx] = v2;
        if (bi == bj && ty == 0 && i < n) {
            // the node-space vector itself (substep API: mu_d)
            double* node = d.node + (long long)b * 4 * n;
            node[i] = v0;
            if (d.het) {
                node[n + i] = v1;
                node[2 * n + i] = v2;
            }
        }
    }
    __syncthreads();
    return lam;
}

__global__ void __launch_bounds__(TB* TY, 4) xstep_b_kernel(Dev d, XConst c) {
    // programmatic dependent of pass A (or the CG kernel): the launch overlaps
    // their tail; everything below reads their results
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the best-iterate copy
    const int b = blockIdx.y;
    if (solve_done(d, b)) return;
    int bi, bj;
    tile_of(blockIdx.x, bi, bj);
    const Layout& lo = d.lo;
    const int n = lo.n;
    const double* Y = d.Y + (long long)b * d.nx;
    double* X = d.X + (long long)b * d.nx;
    double* D = d.D + (long long)b * d.nx;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i0 = bi * TB, j0 = bj * TB;
    __shared__ double Gs[TB][TB + 1];  // g(i, j) of the tile's pairs
    __shared__ double red[TB * TY / 32];
    __shared__ double nv[2][3][TB];    // node vectors of blocks bi (0) and bj (1)
    double res = 0.0;

    __shared__ double sp[2][2][4][TB];
    __shared__ double scr2[TB * TY / 32][2];
    __shared__ int s_fin;
    __shared__ double s_lam;
    // hom closed form: the node degrees are closed-form too (deg_i = f0 u_i +
    // (n - 2) t_i + sum_k t_k), so the diagonal tiles write the diagonal
    // entries and no block finisher is needed; the CG x-step and het keep it
    const bool closed = !d.het && !d.cg;
    TILE_STAMP(10);
    const double lam = node_space(d, c, b, bi, bj, nv, sp, scr2);  // thread 0
    if (tx == 0 && ty == 0) s_lam = lam;
    TILE_STAMP(11);

    // edge loads of the thread's rows (hom), batched
    constexpr int NR = TB / TY;
    long long l[NR];
    bool ok[NR];
    double hv[NR], yg[NR], dg[NR];
    if (!d.het) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int i = i0 + ty + k * TY, j = j0 + tx;
            ok[k] = i < n && j < n && j > i;
            l[k] = ok[k] ? edge_idx(n, i, j) : 0;
            if (ok[k]) {
                hv[k] = d.h[(long long)b * lo.m + l[k]];
                yg[k] = Y[l[k]];
                dg[k] = D[l[k]];
            }
        }
    }
    const int cg_it = d.cg ? d.ictl[b * 8 + kCgIters] : 0;
    if (!d.het) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int il = ty + k * TY;
            double g = 0.0;
            if (ok[k]) {
                // CG: zero iterations means h = 0 and g = 0
                g = d.cg ? (cg_it > 0 ? d.cg_x[(long long)b * lo.m + l[k]] : 0.0)
                         : c.f0 * hv[k] + nv[0][0][il] + nv[1][0][tx];
                const double e = g - yg[k];
                X[l[k]] = g;
                if (d.upd_duals) D[l[k]] = dg[k] + c.rho * e;
                res += e * e;
            }
            Gs[il][tx] = g;
        }
    }
    for (int il = ty; il < TB && d.het; il += TY) {
        const int i = i0 + il, jl = tx, j = j0 + jl;
        double g = 0.0;
        if (i < n && j < n && j > i) {
            const long long l = edge_idx(n, i, j);
            const double hv = d.h[(long long)b * lo.m + l];
            {
                const long long lz = lo.off_z + l, lv = lo.off_nu + l;
                const double rz = Y[lz] - D[lz] * c.inv_rho;
                const double rnu = Y[lv] - D[lv] * c.inv_rho;
                const double hz2 = rz + c.s * rnu - nv[0][2][il] - nv[1][2][jl];
                g = c.g11_0 * hv + c.g12_0 * hz2 + nv[0][0][il] + nv[1][0][jl];
                const double z = c.g12_0 * hv + c.g22_0 * hz2 + nv[0][1][il] + nv[1][1][jl];
                // nu = s (delta r_nu - (g - z))   (slack of g - z + nu = 0)
                const double nu = c.s * (c.delta * rnu - (g - z));
                const double dz = z - Y[lz], dnu = nu - Y[lv];
                X[lz] = z;
                X[lv] = nu;
                if (d.upd_duals) {
                    D[lz] += c.rho * dz;
                    D[lv] += c.rho * dnu;
                }
                res += dz * dz + dnu * dnu;
            }
            const double dgv = g - Y[l];
            X[l] = g;
            if (d.upd_duals) D[l] += c.rho * dgv;
            res += dgv * dgv;
        }
        Gs[il][jl] = g;
    }
    __syncthreads();
    if (closed && bi == bj && ty == 0 && i0 + tx < n) {
        // diagonal entries of the tile's nodes (see the tail below for the
        // formulas), deg_i in closed form
        const int i = i0 + tx;
        const long long p = (long long)i * n + i;
        const long long ps = lo.off_s + p, pt = lo.off_t + p, py = lo.off_y + i;
        const double ys = Y[ps], yt = Y[pt], yy = Y[py], ds = D[ps], dt = D[pt], dy = D[py];
        const double deg = c.f0 * nv[0][1][tx] + (n - 2.0) * nv[0][0][tx] + nv[0][2][tx];
        const double rs = ys - ds * c.inv_rho, rt = yt - dt * c.inv_rho, ry = yy - dy * c.inv_rho;
        const double xs = c.s * (c.delta * rs - c.alpha_over_n - deg + s_lam);
        const double xt = c.s * (c.delta * rt + 2.0 - deg - s_lam);
        const double xy = c.s * (c.delta * ry + 1.0 - deg);
        X[ps] = xs;
        X[pt] = xt;
        X[py] = xy;
        if (d.upd_duals) {
            D[ps] = ds + c.rho * (xs - ys);
            D[pt] = dt + c.rho * (xt - yt);
            D[py] = dy + c.rho * (xy - yy);
        }
        res += (xs - ys) * (xs - ys) + (xt - yt) * (xt - yt) + (xy - yy) * (xy - yy);
    }
    // off-diagonal S/T entries: L_ij = -g, so
    //   S_ij = s (delta r_S,ij - alpha/n + g),  T_ij = s (delta r_T,ij + g)
    // The TB/TY entries a thread owns per orientation are handled as one
    // batch: all loads first (independent, in flight together), then the
    // arithmetic and the stores (X/D may alias Y in the compiler's view).
    constexpr int NE = TB / TY;
    auto upd_batch = [&](const long long (&pos)[NE], const double (&gv)[NE], const bool (&okb)[NE]) {
        double ys[NE], yt[NE], ds[NE], dt[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            if (!okb[k]) continue;
            ys[k] = Y[lo.off_s + pos[k]];
            yt[k] = Y[lo.off_t + pos[k]];
            ds[k] = D[lo.off_s + pos[k]];
            dt[k] = D[lo.off_t + pos[k]];
        }
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            if (!okb[k]) continue;
            const double rs = ys[k] - ds[k] * c.inv_rho, rt = yt[k] - dt[k] * c.inv_rho;
            const double xs = c.s * (c.delta * rs - c.alpha_over_n + gv[k]);
            const double xt = c.s * (c.delta * rt + gv[k]);
            X[lo.off_s + pos[k]] = xs;
            X[lo.off_t + pos[k]] = xt;
            if (d.upd_duals) {
                D[lo.off_s + pos[k]] = ds[k] + c.rho * (xs - ys[k]);
                D[lo.off_t + pos[k]] = dt[k] + c.rho * (xt - yt[k]);
            }
            res += (xs - ys[k]) * (xs - ys[k]) + (xt - yt[k]) * (xt - yt[k]);
        }
    };
    {
        // orientation 1: entries (i, j), address j*n + i
        long long pos[NE];
        double gv[NE];
        bool okb[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int cc = ty + k * TY;
            const int i = i0 + tx, j = j0 + cc;
            okb[k] = i < n && j < n && i != j;
            pos[k] = (long long)j * n + i;
            // diagonal tiles hold each pair once: entry (i, j) with either order
            gv[k] = (bi == bj && i > j) ? Gs[cc][tx] : Gs[tx][cc];
        }
        upd_batch(pos, gv, okb);
    }
    if (bi != bj) {
        // orientation 2: entries (j, i), address i*n + j
        long long pos[NE];
        double gv[NE];
        bool okb[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int cc = ty + k * TY;
            const int j = j0 + tx, i = i0 + cc;
            okb[k] = i < n && j < n;
            pos[k] = (long long)i * n + j;
            gv[k] = Gs[cc][tx];
        }
        upd_batch(pos, gv, okb);
    }
    // node partials of g (deg = L_ii)
    const int t = ty * TB + tx;
    double* PG = d.PG + (long long)b * d.nb * n;
    if (closed) {
    } else if (t < TB) {
        const int il = t, i = i0 + il;
        if (i < n) {
            double s = 0.0;
            for (int jl = 0; jl < TB; ++jl) {
                if (bi == bj) {
                    if (jl == il) continue;
                    s += jl > il ? Gs[il][jl] : Gs[jl][il];
                } else {
                    s += Gs[il][jl];
                }
            }
            PG[(long long)bj * n + i] = s;
        }
    } else if (t < 2 * TB && bi != bj) {
        const int jl = t - TB, j = j0 + jl;
        if (j < n) {
            double s = 0.0;
            for (int il = 0; il < TB; ++il) s += Gs[il][jl];
            PG[(long long)bi * n + j] = s;
        }
    }
    // residual partial of this tile
    {
        const int lane = t & 31, wid = t >> 5;
        double v = warp_sum(res);
        __syncthreads();
        if (lane == 0) red[wid] = v;
        __syncthreads();
        if (t == 0) {
            double s = 0.0;
            for (int w = 0; w < TB * TY / 32; ++w) s += red[w];
            d.res_part[(long long)b * d.ntile + blockIdx.x] = s;
        }
    }

    // ---- tail (CG and het; the hom closed form wrote these in its diagonal
    // tiles and only needs the solve-level arrival): the last tile of a node
    // block writes the block's diagonal entries (deg_i = L_ii = node sums of g):
    //   S_ii = s (delta r_S,ii - alpha/n - deg_i + lambda)
    //   T_ii = s (delta r_T,ii + 2 - deg_i - lambda)
    //   y_i  = s (delta r_y,i + 1 - deg_i)
    // and the CTA completing the solve's last block adds the residual (the
    // reduction tree of a node_threads(n)-thread pass: node terms, then the
    // tile partials), the trace row, the best iterate and the stop flags.
    int* cnt = d.cnt + (long long)b * d.cnt_stride;
    double* rnode = d.res_node + (long long)b * n;
    bool last = false;
    TILE_STAMP(12);
    if (closed) {
        // every tile arrives at the solve counter; the last one finishes
        last = arrive_solve(cnt + 2 * d.nb + kCntB, d.ntile, &s_fin);
    } else {
    const int fin = arrive_blocks(cnt + kCntB * d.nb, d.nb, bi, bj, &s_fin);
    if (!fin) return;
    for (int q = 0; q < 2; ++q) {
        if (!(fin >> q & 1)) continue;
        const int k = q == 0 ? bi : bj;
        const int i = k * TB + tx;
        const long long p = (long long)i * n + i;
        const long long ps = lo.off_s + p, pt = lo.off_t + p, py = lo.off_y + i;
        double ys = 0.0, yt = 0.0, yy = 0.0, ds = 0.0, dt = 0.0, dy = 0.0;
        const double* const pg1[1] = {PG};
        double degv[1];
        node_sum<1>(pg1, d.nb, n, k, reinterpret_cast<double (*)[TY][TB + 1]>(&Gs[0][0]), degv, [&] {
            if (ty == 0 && i < n) {  // the diagonal entries' loads overlap the partial sums
                ys = Y[ps];
                yt = Y[pt];
                yy = Y[py];
                ds = D[ps];
                dt = D[pt];
                dy = D[py];
            }
        });
        const double deg = degv[0];
        if (ty == 0 && i < n) {
            const double rs = ys - ds * c.inv_rho, rt = yt - dt * c.inv_rho, ry = yy - dy * c.inv_rho;
            const double xs = c.s * (c.delta * rs - c.alpha_over_n - deg + s_lam);
            const double xt = c.s * (c.delta * rt + 2.0 - deg - s_lam);
            const double xy = c.s * (c.delta * ry + 1.0 - deg);
            X[ps] = xs;
            X[pt] = xt;
            X[py] = xy;
            if (d.upd_duals) {
                D[ps] = ds + c.rho * (xs - ys);
                D[pt] = dt + c.rho * (xt - yt);
                D[py] = dy + c.rho * (xy - yy);
            }
            rnode[i] = (xs - ys) * (xs - ys) + (xt - yt) * (xt - yt) + (xy - yy) * (xy - yy);
        }
        last |= arrive_solve(cnt + 2 * d.nb + kCntB, d.nb, &s_fin);
    }
    }
    TILE_STAMP(13);
    if (!last) return;
    int* ctl = d.ictl + b * 8;
    double yl = 0.0, dl = 0.0, best = 0.0;
    int it = 0;
    if (t == 0) {  // independent of the reduction: in flight alongside it
        yl = Y[lo.lambda_ix];
        dl = D[lo.lambda_ix];
        best = d.scal[b * 8 + kBestRes];
        it = ctl[kIter];
    }
    double rsum = 0.0, dummy = 0.0;
    {
        const double* rp = d.res_part + (long long)b * d.ntile;
        if (!closed)
            for (int k = t; k < n; k += TB * TY) rsum += __ldcg(rnode + k);
        for (int k = t; k < d.ntile; k += TB * TY) rsum += __ldcg(rp + k);
    }
    block_sum2_2d(rsum, dummy, scr2);
    if (t != 0) return;
    const double lamv = s_lam;
    d.scal[b * 8 + kLambda] = lamv;
    X[lo.lambda_ix] = lamv;
    TILE_STAMP(14);
    if (!d.upd_duals) return;
    D[lo.lambda_ix] = dl + c.rho * (lamv - yl);
    rsum += (lamv - yl) * (lamv - yl);
    if (!d.bookkeep) return;
    // it: 0-based index of this iteration
    d.tr_res[(long long)b * d.max_iter + it] = rsum;
    d.tr_lam[(long long)b * d.max_iter + it] = yl;
    d.scal[b * 8 + kRes] = rsum;
    ctl[kIter] = it + 1;
    if (d.track_best && rsum < best) {
        d.scal[b * 8 + kBestRes] = rsum;
        ctl[kBestIter] = it + 1;
        ctl[kImproved] = 1;
    }
    if (rsum <= d.epsilon) {
        ctl[kDone] = 1;
        ctl[4] = 1;  // converged
    } else if (it + 1 >= d.max_iter) {
        ctl[kDone] = 1;
    }
}

void launch_xstep_b(const Dev& d, const XConst& c, cudaStream_t st) {
    launch_dependent(xstep_b_kernel, dim3(d.ntile, d.B), dim3(TB, TY), st, d, c);
}

// ---------------------------------------------------------------- best copy
__global__ void best_copy_kernel(Dev d, XConst c) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // pass B set the flag
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next prep
    const int b = blockIdx.y;
    int* ctl = d.ictl + b * 8;
    if (!ctl[kImproved]) return;
    const double* Y = d.Y + (long long)b * d.nx;
    double* bY = d.bestY + (long long)b * d.nx;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < d.nx; k += stride)
        bY[k] = Y[k];
    if (d.het) {
        const Layout& lo = d.lo;
        const double* X = d.X + (long long)b * d.nx;
        const double* D = d.D + (long long)b * d.nx;
        double* sc = d.bestScore + (long long)b * lo.m;
        for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < lo.m; l += stride)
            sc[l] = X[lo.off_z + l] + D[lo.off_z + l] * c.inv_rho;  // proj/src/admm_het.cpp:293-294
    }
}

// (the improved flag is cleared by the next prep)
void launch_best_copy(const Dev& d, const XConst& c, cudaStream_t st) {
    const int blocks = (int)std::min<long long>((d.nx + 255) / 256, 512);
    launch_dependent(best_copy_kernel, dim3(blocks, d.B), dim3(256), st, d, c);
}

void init_attrs_admm() {}

}  // namespace tpb
