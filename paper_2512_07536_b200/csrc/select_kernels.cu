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

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

#include <algorithm>

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
    if (a.done && a.done[b * 8 + 1]) {
        if (a.it_snap && threadIdx.x == 0) a.it_snap[b] = -1;
        return;
    }
    if (a.it_snap && threadIdx.x == 0) a.it_snap[b] = a.done ? a.done[b * 8] : 0;
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
            // compact the surviving bucket into shared memory once it fits;
            // every thread reads the condition before thread 0 resets the
            // count (a thread reading the reset count would skip the block
            // and its barrier)
            const bool compact = s_ncand < 0 && s_mode <= kCap && shift > 0;
            __syncthreads();
            if (compact) {
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
                if (k < m && keep[q] && val[q] != 0.0 && pos < a.list_cap) {
                    if (a.list_w) a.list_w[(long long)b * a.list_cap + pos] = val[q];
                    a.list[(long long)b * a.list_cap + pos++] = (int)k;
                }
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
                if (k < m && g[k] != 0.0 && pos < a.list_cap) {
                    if (a.list_w) a.list_w[(long long)b * a.list_cap + pos] = g[k];
                    a.list[(long long)b * a.list_cap + pos++] = (int)k;
                }
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

// ---------------------------------------------------------------------------
// keep_top_r of ONE large solve across the whole GPU (hom thinning, B = 1):
// a cooperative grid of G CTAs, CTA g owning the contiguous index range g of
// the packed weights. Radix select MSB first with 11-bit digits (64-bit keys:
// 53, 42, 31, 20, 9, 0): per round every CTA histograms the keys of its
// range that match the prefix so far into shared memory and adds the bins
// into a global histogram with integer atomics (order-independent, so
// deterministic); after a grid barrier every CTA reads the same histogram and
// derives the same next digit. The final pass counts ties (== K*) and
// keys > K* per CTA; after one more barrier each CTA knows its exclusive
// prefix over lower CTAs, so ties go to the lowest indices exactly as the
// reference's comparator (v desc, index asc) orders them
// (proj/src/admm.cpp:114-121), and the ascending kept-edge list for the
// SLEM is written without a further pass. Small register and shared-memory
// footprint (256 threads x 32 registers) so its CTAs co-reside with the
// concurrent cone-projection GEMM CTAs (one per SM).
namespace {
constexpr int kGThreads = 256;
constexpr int kGBins = 2048;
constexpr int kGRounds = 6;
constexpr int kTopRCacheBytes = 32 * 1024;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGCand = 2048;  // compacted candidates after the first round (cached ranges)
__device__ __forceinline__ int g_shift(int round) { return round < 5 ? 53 - 11 * round : 0; }
__device__ __forceinline__ int g_bits(int round) { return round < 5 ? 11 : 9; }
}  // namespace

#ifdef OZ_STAMPS
// instrumentation build only (make STAMPS=1): globaltimer stamps per CTA
__device__ long long* g_topr_stamps = nullptr;
__device__ __forceinline__ void topr_stamp(int slot) {
    if (!g_topr_stamps || threadIdx.x) return;
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_topr_stamps[16LL * blockIdx.x + slot] = t;
}
extern "C" int tp_topr_set_stamps(void* dev_ptr) {
    return cudaMemcpyToSymbol(g_topr_stamps, &dev_ptr, sizeof(void*)) == cudaSuccess ? 0 : 7;
}
#define TOPR_STAMP(slot) topr_stamp(slot)
#else
#define TOPR_STAMP(slot) do {} while (0)
#endif

__global__ void __launch_bounds__(kGThreads, 8) topr_grid_kernel(SelectArgs a, int* gh, int* cnt) {
    cg::grid_group grid = cg::this_grid();
    if (a.done && a.done[1]) {  // uniform across the grid
        if (a.it_snap && blockIdx.x == 0 && threadIdx.x == 0) a.it_snap[0] = -1;
        return;
    }
    TOPR_STAMP(0);
    if (a.it_snap && blockIdx.x == 0 && threadIdx.x == 0) a.it_snap[0] = a.done ? a.done[0] : 0;
    const long long m = a.m;
    double* v = a.base;
    const long long r = a.r[0];
    const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
    const long long per = (m + G - 1) / G;
    const long long lo = (long long)g * per, hi = lo + per < m ? lo + per : m;
    __shared__ int sh[kGBins];
    __shared__ int scan_scratch[32];
    __shared__ int s_sel[4];  // digit, need after, bucket population, count above
    __shared__ unsigned short cand[kGCand];  // offsets into sv of the keys matching the prefix
    __shared__ int s_ncand;
    __shared__ int s_tw[kGWarps], s_kw[kGWarps];  // per-warp ties / kept nonzero (cached final passes)
    const int lane = tid & 31, wid = tid >> 5;
    // the CTA's range of values, read from HBM once and kept in shared
    // memory for every later pass when the launch reserved room for it
    extern __shared__ double sv[];
    const bool cached = a.topr_cache >= hi - lo;
    if (cached) {
        // all of a thread's loads in flight before the first store
        constexpr int NL = 8;
        for (long long k0 = lo + tid; k0 < hi; k0 += NL * kGThreads) {
            double t[NL];
#pragma unroll
            for (int u = 0; u < NL; ++u) {
                const long long k = k0 + (long long)u * kGThreads;
                t[u] = k < hi ? v[k] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NL; ++u) {
                const long long k = k0 + (long long)u * kGThreads;
                if (k < hi) sv[k - lo] = t[u];
            }
        }
    }
    auto val = [&](long long k) { return cached ? sv[k - lo] : v[k]; };
    TOPR_STAMP(1);

    // the global histograms are zero on entry (zeroed at allocation and by
    // the previous launch after its last barrier)
    int mode;  // 0 keep all, 1 key >= thresh, 2 key > thresh + first need ties, 3 keep none
    unsigned long long prefix = 0, pmask = 0;
    long long need = r;
    if (r >= m) {
        mode = 0;
    } else if (r <= 0) {
        mode = 3;
    } else {
        mode = 2;
        int ncand = -1;  // >= 0: the rounds scan only cand[0, ncand)
        for (int round = 0; round < kGRounds; ++round) {
            const int shift = g_shift(round), nb = 1 << g_bits(round);
            for (int k = tid; k < nb; k += kGThreads) sh[k] = 0;
            __syncthreads();
            if (ncand >= 0) {
                for (int c = tid; c < ncand; c += kGThreads) {
                    const unsigned long long key = (unsigned long long)__double_as_longlong(sv[cand[c]] + 0.0);
                    if ((key & pmask) == prefix) atomicAdd(&sh[(key >> shift) & (nb - 1)], 1);
                }
            } else {
                // warp-aggregated: the early rounds put most keys of a warp
                // in one bin (same exponent), so one atomic per distinct bin;
                // four keys per thread loaded before the first atomic
                constexpr int U = 4;
                for (long long base = lo; base < hi; base += U * kGThreads) {
                    unsigned bin[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const long long k = base + u * kGThreads + tid;
                        bin[u] = 0xffffffffu;
                        if (k < hi) {
                            const unsigned long long key = (unsigned long long)__double_as_longlong(val(k) + 0.0);
                            if ((key & pmask) == prefix) bin[u] = (unsigned)((key >> shift) & (nb - 1));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const unsigned peers = __match_any_sync(0xffffffffu, bin[u]);
                        if (bin[u] != 0xffffffffu && (__ffs(peers) - 1) == lane) atomicAdd(&sh[bin[u]], __popc(peers));
                    }
                }
            }
            __syncthreads();
            int* ghr = gh + round * kGBins;
            for (int k = tid; k < nb; k += kGThreads)
                if (sh[k]) atomicAdd(&ghr[k], sh[k]);
            TOPR_STAMP(2 + 2 * round);
            grid.sync();
            TOPR_STAMP(3 + 2 * round);
            // every CTA: bucket of the need-th largest key (suffix scan, 8 bins per thread)
            // (the bins stay in registers: all loads in flight at once, and
            // the selecting thread walks its copies, not L2)
            const int per_t = nb / kGThreads;  // 8 (or 2 in the last round)
            int hb[8];
            int own = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                hb[q] = q < per_t ? __ldcg(&ghr[nb - 1 - (tid * per_t + q)]) : 0;  // descending order
                own += hb[q];
            }
            int tot;
            const int before = block_exclusive_scan(own, scan_scratch, &tot);
            if (before < need && before + own >= need) {
                long long cum = before;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int bin = nb - 1 - (tid * per_t + q);
                    const int h = hb[q];
                    if (q < per_t && cum + h >= need) {
                        s_sel[0] = bin;
                        s_sel[1] = (int)(need - cum);
                        s_sel[2] = h;
                        break;
                    }
                    cum += h;
                }
            }
            if (tid == 0) s_ncand = 0;  // every read of the last compaction's count is behind us
            __syncthreads();
            prefix |= (unsigned long long)s_sel[0] << shift;
            pmask |= (unsigned long long)(nb - 1) << shift;
            need = s_sel[1];
            const bool fin = s_sel[2] == need;  // whole bucket kept
            __syncthreads();
            if (fin) {
                mode = 1;
                break;
            }
            if (cached && ncand < 0 && round + 1 < kGRounds) {
                // the keys still matching the prefix (a few per CTA once the
                // exponent is fixed), so later rounds skip the full range
                for (long long base = lo; base < hi; base += kGThreads) {
                    const long long k = base + tid;
                    const bool match = k < hi && (((unsigned long long)__double_as_longlong(sv[k - lo] + 0.0)) & pmask) == prefix;
                    const unsigned bal = __ballot_sync(0xffffffffu, match);
                    int off = 0;
                    if (lane == 0 && bal) off = atomicAdd(&s_ncand, __popc(bal));
                    off = __shfl_sync(0xffffffffu, off, 0) + __popc(bal & ((1u << lane) - 1u));
                    if (match && off < kGCand) cand[off] = (unsigned short)(k - lo);
                }
                __syncthreads();
                ncand = s_ncand <= kGCand ? s_ncand : -1;
            }
        }
    }
    const unsigned long long thresh = prefix;
    auto classify = [&](double x, bool& keep, bool& tie) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(x + 0.0);
        keep = mode == 0 || (mode == 1 && key >= thresh) || (mode == 2 && key > thresh);
        tie = mode == 2 && key == thresh;
    };
    // cached ranges: warp w owns the contiguous segment [s0, s1) of the CTA's
    // range, lane l its elements s0 + l + 32j (index order = (j, l)), so tie
    // ranks and list positions come from ballots and one per-warp prefix
    const long long segw = (hi - lo + kGThreads - 1) / kGThreads * 32;
    const long long s0 = lo + wid * segw < hi ? lo + wid * segw : hi, s1 = s0 + segw < hi ? s0 + segw : hi;
    // final pass 1: ties and kept-nonzero keys above the threshold, per CTA
    if (cached) {
        int tw = 0, kw = 0;
        for (long long base = s0; base < s1; base += 32) {
            const long long k = base + lane;
            bool keep = false, tie = false;
            double x = 0.0;
            if (k < s1) {
                x = sv[k - lo];
                classify(x, keep, tie);
            }
            tw += __popc(__ballot_sync(0xffffffffu, tie));
            kw += __popc(__ballot_sync(0xffffffffu, keep && x != 0.0));
        }
        if (lane == 0) {
            s_tw[wid] = tw;
            s_kw[wid] = kw;
        }
        __syncthreads();
        if (tid == 0) {
            int tt = 0, kt = 0;
            for (int w = 0; w < kGWarps; ++w) {
                tt += s_tw[w];
                kt += s_kw[w];
            }
            cnt[2 * g] = tt;
            cnt[2 * g + 1] = kt;
        }
    } else {
        int t_own = 0, k_own = 0;
        for (long long k = lo + tid; k < hi; k += kGThreads) {
            const double x = val(k);
            bool keep, tie;
            classify(x, keep, tie);
            t_own += tie;
            k_own += keep && x != 0.0;
        }
        int ttot, ktot;
        block_exclusive_scan(t_own, scan_scratch, &ttot);
        block_exclusive_scan(k_own, scan_scratch, &ktot);
        if (tid == 0) {
            cnt[2 * g] = ttot;
            cnt[2 * g + 1] = ktot;
        }
    }
    TOPR_STAMP(14);
    grid.sync();
    TOPR_STAMP(15);
    // every CTA is past its histogram reads: zero them for the next launch
    for (int k = g * kGThreads + tid; k < kGRounds * kGBins; k += G * kGThreads) gh[k] = 0;
    // exclusive prefixes over the lower CTAs (index order)
    long long tie_off = 0, list_off = 0;
    for (int q = tid; q < g; q += kGThreads) {
        tie_off += __ldcg(&cnt[2 * q]);
        list_off += __ldcg(&cnt[2 * q + 1]);
    }
    __shared__ long long red[2][kGThreads / 32];
    {
        long long a0 = tie_off, a1 = list_off;
        for (int o = 16; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        if ((tid & 31) == 0) {
            red[0][tid >> 5] = a0;
            red[1][tid >> 5] = a1;
        }
        __syncthreads();
        tie_off = list_off = 0;
        for (int w = 0; w < kGThreads / 32; ++w) {
            tie_off += red[0][w];
            list_off += red[1][w];
        }
    }
    // kept ties precede the list entries of later CTAs: add the ties kept by
    // lower CTAs (thresh > 0: ties are nonzero) to the list offset
    const long long need_eq = mode == 2 ? need : 0;
    const bool tie_nonzero = thresh != 0ull;
    {
        const long long kept_before = tie_off < need_eq ? tie_off : need_eq;
        if (tie_nonzero) list_off += kept_before;
    }
    if (cached) {
        // final pass 2: the warp's offsets from the per-warp counts, then
        // ballots per 32 elements; values already +0 are not rewritten
        long long tie_run = tie_off, pos_run = list_off;
        int tb_before = 0;
        for (int w = 0; w < wid; ++w) {
            tb_before += s_tw[w];
            pos_run += s_kw[w];
        }
        tie_run += tb_before;
        if (tie_nonzero) {
            const long long room = need_eq - tie_off > 0 ? need_eq - tie_off : 0;
            pos_run += room < tb_before ? room : tb_before;  // ties kept by lower warps
        }
        const unsigned lt = (1u << lane) - 1u;
        for (long long base = s0; base < s1; base += 32) {
            const long long k = base + lane;
            bool keep = false, tie = false;
            double x = 0.0;
            if (k < s1) {
                x = sv[k - lo];
                classify(x, keep, tie);
            }
            const unsigned tb = __ballot_sync(0xffffffffu, tie);
            if (tie) keep = tie_run + __popc(tb & lt) < need_eq;
            const bool nz = keep && x != 0.0;
            const unsigned kb = __ballot_sync(0xffffffffu, nz);
            if (k < s1 && !keep && __double_as_longlong(x) != 0) v[k] = 0.0;
            if (nz && a.list) {
                const long long pos = pos_run + __popc(kb & lt);
                if (pos < a.list_cap) {
                    a.list[pos] = (int)k;
                    if (a.list_w) a.list_w[pos] = x;
                }
            }
            tie_run += __popc(tb);
            pos_run += __popc(kb);
        }
        if (a.list && g == G - 1 && wid == kGWarps - 1 && lane == 0) a.list_count[0] = (int)pos_run;
        TOPR_STAMP(13);
        return;
    }
    // final pass 2: in index order, chunks of kGThreads with block scans
    long long tie_run = tie_off, pos_run = list_off;
    for (long long base = lo; base < hi; base += kGThreads) {
        const long long k = base + tid;
        double x = 0.0;
        bool keep = false, tie = false;
        if (k < hi) {
            x = val(k);
            const unsigned long long key = (unsigned long long)__double_as_longlong(x + 0.0);
            keep = mode == 0 || (mode == 1 && key >= thresh) || (mode == 2 && key > thresh);
            tie = mode == 2 && key == thresh;
        }
        int tt;
        const int tex = block_exclusive_scan(tie ? 1 : 0, scan_scratch, &tt);
        if (tie) keep = tie_run + tex < need_eq;
        tie_run += tt;
        const int nz = (keep && x != 0.0) ? 1 : 0;
        int kt;
        const int kex = block_exclusive_scan(nz, scan_scratch, &kt);
        if (k < hi) {
            if (!keep) v[k] = 0.0;
            if (nz && a.list && pos_run + kex < a.list_cap) {
                a.list[pos_run + kex] = (int)k;
                if (a.list_w) a.list_w[pos_run + kex] = x;
            }
        }
        pos_run += kt;
    }
    if (a.list && g == G - 1 && tid == 0) a.list_count[0] = (int)pos_run;
}

int topr_grid_ctas(long long m) {
    static int cap[64] = {};
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) dev = 63;
    if (!cap[dev]) {
        int sms = 0, per_sm = 0;
        TPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, topr_grid_kernel, kGThreads, 0));
        cap[dev] = std::max(1, sms * std::min(per_sm, 1));  // one CTA per SM
    }
    return (int)std::max<long long>(1, std::min<long long>(cap[dev], (m + 2047) / 2048));
}

void launch_topr_grid(const SelectArgs& a, int* gh, int* cnt, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    const int G = topr_grid_ctas(a.m);
    const long long per = (a.m + G - 1) / G;
    SelectArgs b = a;
    // the range cache fits beside a cone-GEMM CTA (173 KB) on the same SM
    b.topr_cache = per * (long long)sizeof(double) <= kTopRCacheBytes ? (int)per : 0;
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = b.topr_cache * sizeof(double);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TPB_CUDA(cudaLaunchKernelEx(&cfg, topr_grid_kernel, b, gh, cnt));
}

// Compaction of the nonzero entries of a packed vector into an ascending list
// (used when no selection runs, e.g. the SLEM of an arbitrary weight vector).
__global__ void __launch_bounds__(kThreads) compact_kernel(const double* g, long long stride, long long m,
                                                          int* list, int* count, int cap, double* list_w,
                                                          int* it_snap, const int* done) {
    const int b = blockIdx.x;
    if (done && done[b * 8 + 1]) {
        if (it_snap && threadIdx.x == 0) it_snap[b] = -1;
        return;
    }
    if (it_snap && threadIdx.x == 0) it_snap[b] = done ? done[b * 8] : 0;
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
            if (k < m && g[k] != 0.0 && pos < cap) {
                if (list_w) list_w[(long long)b * cap + pos] = g[k];
                list[(long long)b * cap + pos++] = (int)k;
            }
        }
        run += tot;
    }
    if (threadIdx.x == 0) count[b] = run;
}

void launch_compact(const double* g, long long stride, long long m, int* list, int* count, int cap,
                    int B, cudaStream_t st, double* list_w, int* it_snap, const int* done) {
    compact_kernel<<<B, kThreads, 0, st>>>(g, stride, m, list, count, cap, list_w, it_snap, done);
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
