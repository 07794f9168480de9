// Once-per-solve kernels: feasible start, Alg. 1 allocation, extraction.
#include "misc_kernels.cuh"
#include "csr.cuh"

namespace tpb {

// ---------------------------------------------------------------- feasible start
// proj/src/admm.cpp:143-173: g0 = 1/(dmax+1) on the warm edges, lap(i,i)
// accumulated edge by edge (bitwise as the reference), lambda0 from the SLEM.
__global__ void feasible_a_kernel(Dev d, const int* warm_list, const int* warm_count, int warm_cap,
                                  double* fs_scal) {
    const int b = blockIdx.x;
    const int n = d.lo.n;
    const int nw = warm_count[b];
    const int* list = warm_list + (long long)b * warm_cap;
    double* X = d.X + (long long)b * d.nx;
    extern __shared__ int deg[];
    __shared__ double scratch[32];
    for (int v = threadIdx.x; v < n; v += blockDim.x) deg[v] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nw; e += blockDim.x) {
        int i, j;
        edge_pair(n, list[e], i, j);
        atomicAdd(&deg[i], 1);
        atomicAdd(&deg[j], 1);
    }
    __syncthreads();
    double dm = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) dm = fmax(dm, (double)deg[v]);
    dm = block_max(dm, scratch);
    const int dmax = nw > 0 ? (int)dm : 0;
    const double g0 = 1.0 / (dmax + 1);
    for (int e = threadIdx.x; e < nw; e += blockDim.x) X[list[e]] = g0;
    double* lapd = d.node + (long long)b * 4 * n + 3 * n;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        double acc = 0.0;  // lap(i,i) += g0 once per incident warm edge
        for (int k = 0; k < deg[v]; ++k) acc += g0;
        lapd[v] = acc;
    }
    if (threadIdx.x == 0) fs_scal[b * 2] = g0;
}

void launch_feasible_a(const Dev& d, const int* warm_list, const int* warm_count, int warm_cap,
                       double* fs_scal, cudaStream_t st) {
    feasible_a_kernel<<<d.B, 256, d.lo.n * sizeof(int), st>>>(d, warm_list, warm_count, warm_cap, fs_scal);
    TPB_CHECK_LAUNCH();
}

__global__ void feasible_b_kernel(Dev d, XConst c, const double* slem_out) {
    const int b = blockIdx.y;
    const Layout& lo = d.lo;
    const int n = lo.n;
    double* X = d.X + (long long)b * d.nx;
    const double* lapd = d.node + (long long)b * 4 * n + 3 * n;
    const double lambda0 = fmax(1e-3, 1.0 - slem_out[b * 8]);
    const long long nn = (long long)n * n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nn; p += stride) {
        const int col = (int)(p / n), row = (int)(p % n);  // column-major (r, c) at c*n + r
        double lrc;
        if (row == col) {
            lrc = lapd[row];
        } else {
            const int i = row < col ? row : col, j = row < col ? col : row;
            const double gg = X[edge_idx(n, i, j)];
            lrc = gg != 0.0 ? 0.0 - gg : 0.0;
        }
        const double diag = row == col ? 1.0 : 0.0;
        X[lo.off_s + p] = -(lrc + c.alpha_over_n - diag * lambda0);
        X[lo.off_t + p] = diag * (2.0 - lambda0) - lrc;
    }
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long i = tid; i < n; i += stride) X[lo.off_y + i] = 1.0 - lapd[i];
    if (tid == 0) X[lo.lambda_ix] = lambda0;
    if (d.het) {
        // proj/src/admm_het.cpp:248-250: z = 1 on warm edges, nu = max(0, z - g)
        for (long long l = tid; l < lo.m; l += stride) {
            const double g = X[l];
            const double z = g != 0.0 ? 1.0 : 0.0;
            X[lo.off_z + l] = z;
            X[lo.off_nu + l] = fmax(0.0, z - g);
        }
    }
}

void launch_feasible_b(const Dev& d, const XConst& c, const double* slem_out, const double* fs_scal,
                       cudaStream_t st) {
    (void)fs_scal;
    const int blocks = (int)std::min<long long>(((long long)d.lo.n * d.lo.n + 255) / 256, 1024);
    feasible_b_kernel<<<dim3(blocks, d.B), 256, 0, st>>>(d, c, slem_out);
    TPB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- Alg. 1
namespace {

// floor(x + 1e-9 (1 + |x|)) without contraction (proj/src/bandwidth.cpp:22-24)
__device__ inline long long guarded_floor(double x) {
    const double t = __dadd_rn(x, __dmul_rn(1e-9, __dadd_rn(1.0, fabs(x))));
    return (long long)floor(t);
}

__device__ inline double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace

__global__ void alloc_kernel(const double* b_all, const int* caps_all, int n, const int* r_all,
                             double* b_unit_out, int* e_out, int* status) {
    const int p = blockIdx.x, lane = threadIdx.x;
    const double* b = b_all + (long long)p * n;
    const int* caps = caps_all ? caps_all + (long long)p * n : nullptr;
    const long long r = r_all[p];
    extern __shared__ int sm[];
    int* e = sm;
    int* gr = sm + n;
    auto cap = [&](int i) { return caps ? caps[i] : n - 1; };
    // validation (proj/src/bandwidth.cpp:30-52)
    bool bad = n < 2;
    long long cap_sum = 0;
    for (int i = lane; i < n; i += 32) {
        if (!(b[i] > 0.0)) bad = true;
        const int ci = cap(i);
        if (ci < 0 || ci > n - 1) bad = true;
        cap_sum += ci;
    }
    bad = __any_sync(0xffffffffu, bad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cap_sum += __shfl_xor_sync(0xffffffffu, cap_sum, o);
    const long long max_edges = (long long)n * (n - 1) / 2;
    if (bad || r < 0 || r > max_edges) {
        if (lane == 0) status[p] = 1;
        return;
    }
    if (cap_sum < 2 * r) {
        if (lane == 0) status[p] = 2;
        return;
    }
    double bu = INFINITY;
    for (int i = lane; i < n; i += 32) bu = fmin(bu, b[i]);
    bu = warp_min_d(bu);
    auto recount = [&](double unit, int* out) {
        long long s = 0;
        for (int i = lane; i < n; i += 32) {
            const long long q = guarded_floor(__ddiv_rn(b[i], unit));
            const int v = (int)(q < cap(i) ? q : cap(i));
            out[i] = v;
            s += v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __syncwarp();
        return s;
    };
    long long sum = recount(bu, e);
    while (sum < 2 * r) {
        double nxt = 0.0;
        for (int i = lane; i < n; i += 32) nxt = fmax(nxt, __ddiv_rn(b[i], (double)(e[i] + 1)));
        nxt = warp_max(nxt);
        const long long s2 = recount(nxt, gr);
        bool same = true;
        for (int i = lane; i < n; i += 32) same = same && gr[i] == e[i];
        same = __all_sync(0xffffffffu, same);
        if (same) {
            if (lane == 0) status[p] = 2;
            return;
        }
        bu = nxt;
        for (int i = lane; i < n; i += 32) e[i] = gr[i];
        __syncwarp();
        sum = s2;
    }
    while (sum > 2 * r) {
        // largest count, ties to the highest index (proj/src/bandwidth.cpp:81-87)
        int best = -1, bidx = -1;
        for (int i = lane; i < n; i += 32)
            if (e[i] > best || (e[i] == best && i > bidx)) {
                best = e[i];
                bidx = i;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
            if (ob > best || (ob == best && oi > bidx)) {
                best = ob;
                bidx = oi;
            }
        }
        if (lane == 0) e[bidx] -= 1;
        __syncwarp();
        --sum;
    }
    for (int i = lane; i < n; i += 32) e_out[(long long)p * n + i] = e[i];
    if (lane == 0) {
        b_unit_out[p] = bu;
        status[p] = 0;
    }
}

void launch_allocate(const double* b, const int* caps, int n, const int* r, int P, double* b_unit,
                     int* e, int* status, cudaStream_t st) {
    alloc_kernel<<<P, 32, 2 * n * sizeof(int), st>>>(b, caps, n, r, b_unit, e, status);
    TPB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- extraction
__global__ void extract_kernel(int n, long long m, const double* gall, long long stride,
                               const int* list_all, const int* count, int list_cap, int* out_i,
                               int* out_j, double* out_w, double* packed_out, double* worst_out,
                               int* cidx_all) {
    const int b = blockIdx.x;
    const double* g = gall + (long long)b * stride;
    const int* list = list_all + (long long)b * list_cap;
    const int ne = min(count[b], list_cap);
    int* ei = out_i + (long long)b * list_cap;
    int* ej = out_j + (long long)b * list_cap;
    double* ew = out_w + (long long)b * list_cap;
    extern __shared__ int shi[];
    int* rowptr = shi;
    int* colptr = rowptr + n + 1;
    int* cur = colptr + n + 1;
    int* cidx = cidx_all + (long long)b * list_cap;
    __shared__ int iscr[32];
    __shared__ double scratch[32];
    build_csr(n, ne, list, g, false, ei, ej, ew, rowptr, colptr, cur, cidx, iscr);
    double worst = -INFINITY;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        double s = 0.0;  // ascending edge index: (u, v) u < v first, then (v, j)
        for (int p = colptr[v]; p < colptr[v + 1]; ++p) s += ew[cidx[p]];
        for (int e = rowptr[v]; e < rowptr[v + 1]; ++e) s += ew[e];
        worst = fmax(worst, s);
    }
    worst = block_max(worst, scratch);
    const double scale = worst > 1.0 ? 1.0 / worst : 1.0;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const double w = ew[e] * scale;
        ew[e] = w;
        packed_out[(long long)b * m + list[e]] = w;
    }
    if (threadIdx.x == 0) worst_out[b] = worst;
}

void launch_extract(int n, long long m, const double* g, long long stride, const int* list,
                    const int* count, int list_cap, int* out_i, int* out_j, double* out_w,
                    double* packed_out, double* worst_out, int* cidx_scratch, int B,
                    cudaStream_t st) {
    const size_t smem = (3 * (size_t)n + 2) * sizeof(int);
    extract_kernel<<<B, 512, smem, st>>>(n, m, g, stride, list, count, list_cap, out_i, out_j, out_w,
                                          packed_out, worst_out, cidx_scratch);
    TPB_CHECK_LAUNCH();
}

__global__ void floor_mask_kernel(const double* g, long long stride, long long m, double floor, double* t) {
    const int b = blockIdx.y;
    const long long st = (long long)gridDim.x * blockDim.x;
    for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < m; l += st) {
        const double v = g[(long long)b * stride + l];
        t[(long long)b * m + l] = v > floor ? v : 0.0;
    }
}

void launch_floor_mask(const double* g, long long stride, long long m, double floor, double* t,
                       int B, cudaStream_t st) {
    const int blocks = (int)std::min<long long>((m + 255) / 256, 1024);
    floor_mask_kernel<<<dim3(blocks, B), 256, 0, st>>>(g, stride, m, floor, t);
    TPB_CHECK_LAUNCH();
}

void init_attrs_misc() {
    set_max_dyn_smem(extract_kernel);
}

}  // namespace tpb
