// Exact top-r selection with the reference's tie rule, one CTA per solve.
//
//   keep_top_r        (proj/src/admm.cpp:114-121): zero all but the r largest
//                     clamped weights, ties to the lower index;
//   project_binary_z  (proj/src/admm_het.cpp:116-123): ones at the r largest
//                     z-scores, ties to the lower index.
//
// Radix select (8-bit digits, MSB first) over the order-preserving 64-bit key
// of each double finds the r-th largest key K*; candidates are compacted into
// shared memory once they fit. The final pass walks the array in index order
// with a block scan, so ties at K* go to the lowest indices exactly as the
// reference's std::sort comparator orders them, and it emits the ascending
// list of kept nonzero edges consumed by the SLEM kernel.
#include "select_kernels.cuh"

namespace tpb {

namespace {

constexpr int kThreads = 1024;
constexpr int kItems = 4;
constexpr int kCap = 8192;  // smem candidates (64 KB of keys)

__device__ inline unsigned long long key_of(double v, int binary) {
    if (binary) return order_key(v);
    // clamped weights are >= +0.0: the raw bit pattern is order-preserving
    return (unsigned long long)__double_as_longlong(v + 0.0);
}

}  // namespace

// mode 0: hom thinning of Y_g in place; mode 1: binary z in place (het) and
// compaction of the nonzero clamped Y_g.
__global__ void __launch_bounds__(kThreads) topr_kernel(SelectArgs a) {
    const int b = blockIdx.x;
    if (a.done && a.done[b * 8 + 1]) return;
    const long long m = a.m;
    double* v = a.base + (long long)b * a.stride;
    const long long r = a.r[b];
    __shared__ int hist[256];
    __shared__ int scan_scratch[32];
    __shared__ unsigned long long s_prefix, s_thresh;
    __shared__ int s_need, s_mode, s_ncand, s_fin;
    extern __shared__ unsigned long long cand[];  // kCap keys
    const int tid = threadIdx.x;

    // ------------------------------------------------------------ select
    int mode;  // 0: keep all; 1: keep key >= thresh; 2: key > thresh + ties
    if (r >= m) {
        mode = 0;
    } else if (r <= 0) {
        mode = 3;  // keep none
    } else {
        if (tid == 0) {
            s_prefix = 0;
            s_need = (int)r;
            s_fin = 0;
            s_ncand = -1;
        }
        __syncthreads();
        unsigned long long pmask = 0;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int k = tid; k < 256; k += kThreads) hist[k] = 0;
            __syncthreads();
            const unsigned long long prefix = s_prefix;
            if (s_ncand >= 0) {
                for (int k = tid; k < s_ncand; k += kThreads) {
                    const unsigned long long key = cand[k];
                    if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
                }
            } else {
                for (long long k = tid; k < m; k += kThreads) {
                    const unsigned long long key = key_of(v[k], a.binary);
                    if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
                }
            }
            __syncthreads();
            if (tid == 0) {
                int need = s_need, cum = 0, dg = 0;
                for (dg = 255; dg >= 0; --dg) {
                    if (cum + hist[dg] >= need) break;
                    cum += hist[dg];
                }
                need -= cum;
                s_need = need;
                s_prefix = prefix | ((unsigned long long)dg << shift);
                // whole bucket kept -> threshold on the bucket floor
                if (hist[dg] == need) s_fin = 1;
                s_mode = hist[dg];  // bucket population (for compaction test)
            }
            __syncthreads();
            pmask |= (255ull << shift);
            if (s_fin) break;
            // compact the surviving bucket into shared memory once it fits
            if (s_ncand < 0 && s_mode <= kCap && shift > 0) {
                if (tid == 0) s_ncand = 0;
                __syncthreads();
                const unsigned long long pf = s_prefix;
                for (long long k = tid; k < m; k += kThreads) {
                    const unsigned long long key = key_of(v[k], a.binary);
                    if ((key & pmask) == pf) cand[atomicAdd(&s_ncand, 1)] = key;
                }
                __syncthreads();
            }
        }
        __syncthreads();
        mode = s_fin ? 1 : 2;
        if (tid == 0) s_thresh = s_prefix;
        __syncthreads();
        // all remaining equal keys kept -> plain threshold
        if (mode == 2) {
            // count keys == thresh (bucket population at the last digit)
            if (s_mode == s_need) mode = 1;
        }
    }
    const unsigned long long thresh = (mode == 1 || mode == 2) ? s_thresh : 0ull;
    const int need_eq = (mode == 2) ? s_need : 0;

    // ------------------------------------------------------------ final pass
    int tie_run = 0, kept_run = 0;
    for (long long base = 0; base < m; base += (long long)kThreads * kItems) {
        bool keep[kItems];
        bool tie[kItems];
        double val[kItems];
        int nt = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const long long k = base + (long long)tid * kItems + q;
            tie[q] = false;
            keep[q] = false;
            val[q] = 0.0;
            if (k < m) {
                val[q] = v[k];
                const unsigned long long key = key_of(val[q], a.binary);
                if (mode == 0) keep[q] = true;
                else if (mode == 1) keep[q] = key >= thresh;
                else if (mode == 2) {
                    keep[q] = key > thresh;
                    tie[q] = key == thresh;
                    nt += tie[q];
                }
            }
        }
        if (mode == 2) {
            int tot;
            int ex = block_exclusive_scan(nt, scan_scratch, &tot);
            int rank = tie_run + ex;
#pragma unroll
            for (int q = 0; q < kItems; ++q)
                if (tie[q]) {
                    keep[q] = rank < need_eq;
                    ++rank;
                }
            tie_run += tot;
        }
        int nk = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const long long k = base + (long long)tid * kItems + q;
            if (k >= m) continue;
            if (a.binary) {
                v[k] = keep[q] ? 1.0 : 0.0;
            } else {
                if (!keep[q]) v[k] = 0.0;
                else nk += (val[q] != 0.0);
            }
        }
        if (!a.binary && a.list) {
            int tot;
            int pos = kept_run + block_exclusive_scan(nk, scan_scratch, &tot);
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const long long k = base + (long long)tid * kItems + q;
                if (k < m && keep[q] && val[q] != 0.0 && pos < a.list_cap)
                    a.list[(long long)b * a.list_cap + pos++] = (int)k;
            }
            kept_run += tot;
        }
    }
    if (!a.binary && a.list && tid == 0) a.list_count[b] = kept_run;

    // het: compact the nonzero clamped weights for the SLEM
    if (a.binary && a.list) {
        const double* g = a.gbase + (long long)b * a.stride;
        int run = 0;
        for (long long base = 0; base < m; base += (long long)kThreads * kItems) {
            int nk = 0;
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const long long k = base + (long long)tid * kItems + q;
                nk += (k < m && g[k] != 0.0);
            }
            int tot;
            int pos = run + block_exclusive_scan(nk, scan_scratch, &tot);
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const long long k = base + (long long)tid * kItems + q;
                if (k < m && g[k] != 0.0 && pos < a.list_cap)
                    a.list[(long long)b * a.list_cap + pos++] = (int)k;
            }
            run += tot;
        }
        if (tid == 0) a.list_count[b] = run;
    }
}

void launch_topr(const SelectArgs& a, int B, cudaStream_t st) {
    const int smem = kCap * sizeof(unsigned long long);
    topr_kernel<<<B, kThreads, smem, st>>>(a);
    TPB_CHECK_LAUNCH();
}

// Compaction of the nonzero entries of a packed vector into an ascending list
// (used when no selection runs, e.g. the SLEM of an arbitrary weight vector).
__global__ void __launch_bounds__(kThreads) compact_kernel(const double* g, long long stride, long long m,
                                                          int* list, int* count, int cap) {
    const int b = blockIdx.x;
    g += (long long)b * stride;
    __shared__ int scan_scratch[32];
    int run = 0;
    for (long long base = 0; base < m; base += (long long)kThreads * kItems) {
        int nk = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const long long k = base + (long long)threadIdx.x * kItems + q;
            nk += (k < m && g[k] != 0.0);
        }
        int tot;
        int pos = run + block_exclusive_scan(nk, scan_scratch, &tot);
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const long long k = base + (long long)threadIdx.x * kItems + q;
            if (k < m && g[k] != 0.0 && pos < cap) list[(long long)b * cap + pos++] = (int)k;
        }
        run += tot;
    }
    if (threadIdx.x == 0) count[b] = run;
}

void launch_compact(const double* g, long long stride, long long m, int* list, int* count, int cap,
                    int B, cudaStream_t st) {
    compact_kernel<<<B, kThreads, 0, st>>>(g, stride, m, list, count, cap);
    TPB_CHECK_LAUNCH();
}

void init_attrs_select() {
    set_max_dyn_smem(topr_kernel);
}


// ---------------------------------------------------------------- capped
__global__ void __launch_bounds__(1024) capped_z_kernel(CappedArgs a) {
    const int b = blockIdx.x;
    if (a.done && a.done[b * 8 + 1]) return;
    const long long m = a.m;
    const int pad = a.pad, tid = threadIdx.x, nt = blockDim.x;
    double* v = a.base + (long long)b * a.stride;
    unsigned long long* key = a.keys + (long long)b * pad;
    int* idx = a.idx + (long long)b * pad;
    int* load = a.load + (long long)b * a.nrows;
    // ascending (key, index) with key = ~order_key(v): v descending, ties to
    // the lower index (the reference's order_desc comparator)
    for (int k = tid; k < pad; k += nt) {
        key[k] = k < m ? ~order_key(v[k]) : ~0ULL;
        idx[k] = k;
    }
    for (int k = tid; k < a.nrows; k += nt) load[k] = 0;
    __syncthreads();
    for (int size = 2; size <= pad; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = tid; k < pad; k += nt) {
                const int p = k ^ stride;
                if (p <= k) continue;
                const bool up = (k & size) == 0;
                const unsigned long long ka = key[k], kb = key[p];
                const int ia = idx[k], ib = idx[p];
                const bool gt = ka > kb || (ka == kb && ia > ib);
                if (gt == up) {
                    key[k] = kb;
                    key[p] = ka;
                    idx[k] = ib;
                    idx[p] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (long long k = tid; k < m; k += nt) v[k] = 0.0;
    __syncthreads();
    if (tid == 0) {
        const int r = a.r[b];
        int taken = 0;
        for (int p = 0; p < pad && taken < r; ++p) {
            const int col = idx[p];
            if (col >= m || !a.allowed[col]) continue;
            bool fits = true;
            for (int q = a.colr_ptr[col]; q < a.colr_ptr[col + 1]; ++q)
                if (load[a.colr[q]] + 1 > a.caps[a.colr[q]]) {
                    fits = false;
                    break;
                }
            if (!fits) continue;
            v[col] = 1.0;
            for (int q = a.colr_ptr[col]; q < a.colr_ptr[col + 1]; ++q) ++load[a.colr[q]];
            ++taken;
        }
    }
}

void launch_capped_z(const CappedArgs& a, int B, cudaStream_t st) {
    capped_z_kernel<<<B, 1024, 0, st>>>(a);
    TPB_CHECK_LAUNCH();
}

}  // namespace tpb
