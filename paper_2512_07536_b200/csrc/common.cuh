// Shared device helpers for the B200 ADMM topology solver.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace tpb {

// Error taxonomy of the C ABI; mirrors proj/include/topoopt/errors.hpp.
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kInfeasible = 2,
    kLinearSolve = 3,
    kDegenerate = 4,
    kPivot = 5,
    kInternal = 6,
    kCuda = 7,
};

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define TPB_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::tpb::Error(::tpb::kCuda, std::string("CUDA error ") +                \
                                                 cudaGetErrorString(e_) + " at " +       \
                                                 __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define TPB_CHECK_LAUNCH() TPB_CUDA(cudaGetLastError())

#define TPB_NCCL(call)                                                                   \
    do {                                                                                 \
        const int r_ = (int)(call);                                                      \
        if (r_ != 0)                                                                     \
            throw ::tpb::Error(::tpb::kCuda, std::string("NCCL error ") + std::to_string(r_) + \
                                                 " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

// Host -> device copy that has landed when it returns. cudaMemcpy from
// pageable memory may return before its DMA completes, and only the legacy
// stream is ordered after it -- the solver's non-blocking streams are not.
inline void h2d(void* dst, const void* src, size_t bytes) {
    TPB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    TPB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

// Thread-local message of the last failed C ABI call (capi.cu).
std::string& last_error_ref();

constexpr double kKktShift = 1e-8;  // proj/src/admm_shared.hpp:16
// Opt a kernel into the largest dynamic shared memory the device allows
// (opt-in limit minus the kernel's static shared memory).
template <typename K>
inline void set_max_dyn_smem(K kernel) {
    int dev = 0, optin = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    TPB_CUDA(cudaFuncGetAttributes(&fa, kernel));
    TPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - (int)fa.sharedSizeBytes));
}

// Per-file opt-in of the >48 KB dynamic shared memory kernels (call once per
// device before any launch or graph capture).
void init_attrs_select();
void init_attrs_slem();
void init_attrs_cone();
void init_attrs_admm();
void init_attrs_misc();
void init_attrs_ozaki();
inline void init_attrs() {
    init_attrs_select();
    init_attrs_slem();
    init_attrs_cone();
    init_attrs_admm();
    init_attrs_misc();
    init_attrs_ozaki();
}

// Flat state layout of one solve (proj/src/admm.cpp:24-44). g is the packed
// lexicographic edge vector (edge_index, proj/src/topology.cpp:78-84); S and T
// are column-major n x n blocks; z / nu exist only for the het solver.
struct Layout {
    int n = 0, m = 0;
    int lambda_ix = 0, off_s = 0, off_y = 0, off_t = 0;
    int off_z = -1, off_nu = -1;
    int nx = 0, neq = 0, q = 0;
};

inline Layout hom_layout(int n) {
    Layout lo;
    lo.n = n;
    lo.m = n * (n - 1) / 2;
    lo.lambda_ix = lo.m;
    lo.off_s = lo.m + 1;
    lo.off_y = lo.off_s + n * n;
    lo.off_t = lo.off_y + n;
    lo.nx = lo.off_t + n * n;
    lo.neq = 2 * n * n + n;
    return lo;
}

inline Layout het_layout(int n, int q) {
    Layout lo = hom_layout(n);
    lo.off_z = lo.nx;
    lo.off_nu = lo.off_z + lo.m;
    lo.nx = lo.off_nu + lo.m;
    lo.neq += q + lo.m;
    lo.q = q;
    return lo;
}

__host__ __device__ inline long long edge_base(int n, int i) {
    return (long long)i * n - (long long)i * (i + 1) / 2;
}

// Packed index of pair (i, j), i < j (proj/src/topology.cpp:78-84).
__host__ __device__ inline long long edge_idx(int n, int i, int j) {
    return edge_base(n, i) + (j - i - 1);
}

// Inverse of edge_idx: the pair (i, j) of packed index l.
__device__ inline void edge_pair(int n, long long l, int& i, int& j) {
    // i = largest i with edge_base(n, i) <= l
    double nn = (double)n - 0.5;
    double disc = nn * nn - 2.0 * (double)l;
    int ii = (int)floor(nn - sqrt(disc > 0 ? disc : 0.0));
    if (ii < 0) ii = 0;
    if (ii > n - 2) ii = n - 2;
    while (ii > 0 && edge_base(n, ii) > l) --ii;
    while (ii < n - 2 && edge_base(n, ii + 1) <= l) ++ii;
    i = ii;
    j = (int)(l - edge_base(n, ii)) + ii + 1;
}

// Deterministic block-wide sum (fixed shuffle tree + fixed smem order).
// All threads receive the result. `scratch` needs blockDim.x/32 doubles.
__device__ inline double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Four block sums with one pair of barriers; each value follows exactly the
// reduction tree of block_sum, so the results are bitwise the same.
__device__ inline void block_sum4(double (&v)[4], double (*scratch)[32]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) scratch[q][wid] = v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double t = lane < nw ? scratch[q][lane] : 0.0;
        v[q] = warp_sum(t);  // every warp reduces the same 32 values
    }
}

__device__ inline double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = lane < nw ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    t = scratch[0];
    __syncthreads();
    return t;
}

__device__ inline double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ inline double block_max(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = -INFINITY;
    if (wid == 0) {
        t = lane < nw ? scratch[lane] : -INFINITY;
        t = warp_max(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    t = scratch[0];
    __syncthreads();
    return t;
}

// Exclusive block scan of ints (any blockDim multiple of 32, <= 1024).
// Returns the exclusive prefix; *total receives the block total.
__device__ inline int block_exclusive_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < nw ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) scratch[lane] = s;  // inclusive per-warp totals
    }
    __syncthreads();
    const int warp_off = wid > 0 ? scratch[wid - 1] : 0;
    const int tot = scratch[nw - 1];
    __syncthreads();
    if (total) *total = tot;
    return warp_off + x - v;
}

// Monotone unsigned key of a double (value order == key order), with -0.0
// folded onto +0.0 so that the reference's `v[a] != v[b]` tie semantics hold.
__device__ inline unsigned long long order_key(double v) {
    v = v + 0.0;  // -0.0 -> +0.0
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

}  // namespace tpb
