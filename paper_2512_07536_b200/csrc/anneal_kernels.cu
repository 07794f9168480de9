// Device warm-start annealer: the reference's simulated annealing over double
// edge swaps (proj/src/anneal.cpp:189-241) with its random stream
// (std::mt19937_64 + the bounded()/unit() mappings of
// proj/include/topoopt/rng.hpp:12-53) reproduced on the device, so every
// draw, candidate and accept/reject decision is the reference's. The energy
// (mean shortest-path length) is an exact integer sum of hop distances: each
// candidate's all-pairs BFS runs in parallel over the sources on the
// device (bitset frontiers, one lane group per source, adjacency bitmatrix in
// shared memory), instead of n sequential BFS on the host.
//
// One cooperative grid; CTA 0 thread 0 is the "master" that owns the random
// stream and the (step, move) schedule. Per candidate: the master scans
// moves until a valid swap (skipped moves need no other thread), every CTA
// applies the swap to its own copy of the graph and sums hop distances over
// its share of the sources, the master reduces the partials in CTA order and
// decides, everyone keeps or reverts. Three grid barriers per candidate.
#include "anneal_kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "host_anneal.hpp"

namespace tpb {

namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;

// ---------------------------------------------------------------- mt19937_64
struct MT64 {
    uint64_t x[312];
    int i;
};

__host__ __device__ inline void mt_seed(MT64& s, uint64_t seed) {
    s.x[0] = seed;
    for (int k = 1; k < 312; ++k) s.x[k] = 6364136223846793005ULL * (s.x[k - 1] ^ (s.x[k - 1] >> 62)) + (uint64_t)k;
    s.i = 312;
}

__host__ __device__ inline uint64_t mt_next(MT64& s) {
    if (s.i >= 312) {
        constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (s.x[k] & kUpper) | (s.x[(k + 1) % 312] & kLower);
            s.x[k] = s.x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        s.i = 0;
    }
    uint64_t y = s.x[s.i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// proj/include/topoopt/rng.hpp: rejection-sampled bounded draw, 53-bit unit
__device__ inline uint64_t bounded(MT64& s, uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    for (;;) {
        const uint64_t x = mt_next(s);
        if (x < limit) return x % bound;
    }
}
__device__ inline double unit(MT64& s) { return (double)(mt_next(s) >> 11) * 0x1.0p-53; }

// ---------------------------------------------------------------- graph
__device__ inline int2 ordered2(int a, int b) { return a < b ? make_int2(a, b) : make_int2(b, a); }
__device__ inline bool has_edge(const uint32_t* adj, int W, int2 e) {
    return (adj[e.x * W + (e.y >> 5)] >> (e.y & 31)) & 1u;
}
__device__ inline void set_edge(uint32_t* adj, int W, int2 e, bool on) {
    const uint32_t bx = 1u << (e.y & 31), by = 1u << (e.x & 31);
    if (on) {
        adj[e.x * W + (e.y >> 5)] |= bx;
        adj[e.y * W + (e.x >> 5)] |= by;
    } else {
        adj[e.x * W + (e.y >> 5)] &= ~bx;
        adj[e.y * W + (e.x >> 5)] &= ~by;
    }
}

struct Args {
    int n, m, W, GS, G;
    const int2* es_in;
    int2* best;
    double t0, cooling;
    int steps, moves;
    uint64_t seed;
    unsigned long long* part;  // G partial distance totals
    int* bad;                  // G "some source did not reach every node" flags
    int* cmd;                  // master -> all: [0] kind, [1] i1, [2] i2, [3..6] n1, n2, [8] decision
    double* energy_out;
    // capacity veto (anneal_capacity_topology, proj/src/anneal.cpp:357-385);
    // allowed == nullptr: unconstrained. Only the master touches these.
    const int* allowed;  // per packed column
    const int* cr_ptr;   // column -> rows CSR
    const int* cr;
    const int* caps;     // per row
    int* load;           // per row, current edge count (master-owned)
};

// Row-load change of the swap (r1, r2) -> (a1, a2) at `row`.
__device__ inline int row_delta(const Args& a, const long long c[4], int row) {
    int d = 0;
    for (int k = 0; k < 4; ++k)
        for (int q = a.cr_ptr[c[k]]; q < a.cr_ptr[c[k] + 1]; ++q)
            if (a.cr[q] == row) d += k < 2 ? -1 : 1;
    return d;
}

// The reference's feasible(): both new columns allowed and every row the
// swap touches within capacity. Rows only losing load cannot overflow, so
// only the rows of the added columns are checked.
__device__ bool cap_feasible(const Args& a, const long long c[4]) {
    if (!a.allowed[c[2]] || !a.allowed[c[3]]) return false;
    for (int k = 2; k < 4; ++k)
        for (int q = a.cr_ptr[c[k]]; q < a.cr_ptr[c[k] + 1]; ++q) {
            const int row = a.cr[q];
            if (a.load[row] + row_delta(a, c, row) > a.caps[row]) return false;
        }
    return true;
}

__device__ void cap_apply(const Args& a, const long long c[4]) {
    for (int k = 0; k < 4; ++k)
        for (int q = a.cr_ptr[c[k]]; q < a.cr_ptr[c[k] + 1]; ++q) a.load[a.cr[q]] += k < 2 ? -1 : 1;
}

// Sum of hop distances from this CTA's sources (lane groups of GS lanes; a
// group's lane w < W holds word w of the frontier / visited bitsets).
__device__ void distance_part(const uint32_t* adj, const Args& a, unsigned long long* s_tot, int* s_bad) {
    const int n = a.n, W = a.W, GS = a.GS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = lane / GS, gs = lane % GS;
    const int per_warp = 32 / GS;
    const int per_cta = (int)(blockDim.x >> 5) * per_warp;
    const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << (gw * GS));
    unsigned long long tot = 0;
    int bad = 0;
    for (int s = blockIdx.x * per_cta + warp * per_warp + gw; s < n; s += a.G * per_cta) {
        uint32_t V = (gs == (s >> 5)) ? (1u << (s & 31)) : 0u;
        uint32_t F = V;
        int reached = 1;
        for (int level = 1;; ++level) {
            uint32_t next = 0;
            for (int w = 0; w < W; ++w) {
                uint32_t fw = __shfl_sync(gmask, F, w, GS);
                while (fw) {
                    const int v = w * 32 + __ffs(fw) - 1;
                    fw &= fw - 1;
                    if (gs < W) next |= adj[v * W + gs];
                }
            }
            const uint32_t nb = next & ~V;
            const int cnt = (int)__reduce_add_sync(gmask, (unsigned)__popc(nb));
            if (cnt == 0) break;
            V |= nb;
            F = nb;
            tot += (unsigned long long)level * (unsigned long long)cnt;
            reached += cnt;
        }
        if (reached < n) bad = 1;
    }
    if (gs == 0 && tot) atomicAdd(s_tot, tot);
    if (bad) atomicOr(s_bad, 1);
}

__global__ void __launch_bounds__(kThreads, 1) anneal_kernel(Args a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = a.n, m = a.m, W = a.W;
    const int tid = threadIdx.x;
    uint32_t* adj = reinterpret_cast<uint32_t*>(smem);
    int2* es = reinterpret_cast<int2*>(smem + ((size_t)n * W * 4 + 15) / 16 * 16);
    MT64* rng = reinterpret_cast<MT64*>(reinterpret_cast<unsigned char*>(es) + ((size_t)m * 8 + 15) / 16 * 16);
    __shared__ unsigned long long s_tot;
    __shared__ int s_bad;
    __shared__ int2 s_old[2];
    const bool master = blockIdx.x == 0 && tid == 0;
    volatile int* cmd = a.cmd;

    for (int k = tid; k < n * W; k += blockDim.x) adj[k] = 0;
    for (int e = tid; e < m; e += blockDim.x) es[e] = a.es_in[e];
    __syncthreads();
    for (int e = tid; e < m; e += blockDim.x) {
        const int2 p = es[e];
        atomicOr(&adj[p.x * W + (p.y >> 5)], 1u << (p.y & 31));
        atomicOr(&adj[p.y * W + (p.x >> 5)], 1u << (p.x & 31));
    }
    if (master) mt_seed(*rng, a.seed);
    __syncthreads();

    auto evaluate = [&]() {
        if (tid == 0) {
            s_tot = 0;
            s_bad = 0;
        }
        __syncthreads();
        distance_part(adj, a, &s_tot, &s_bad);
        __syncthreads();
        if (tid == 0) {
            a.part[blockIdx.x] = s_tot;
            a.bad[blockIdx.x] = s_bad;
        }
        grid.sync();
    };
    auto energy_of = [&]() {  // master only: partials in CTA order (exact integers)
        unsigned long long t = 0;
        int bad = 0;
        for (int c = 0; c < a.G; ++c) {
            t += __ldcg(a.part + c);
            bad |= __ldcg(a.bad + c);
        }
        return bad ? __longlong_as_double(0x7FF0000000000000LL)
                   : (double)t / ((double)n * (double)(n - 1));
    };

    evaluate();
    double energy = 0.0, best_e = 0.0, temp = a.t0;
    int step = 0, mv = 0;
    if (master) {
        energy = energy_of();
        best_e = energy;
    }
    if (blockIdx.x == 0)
        for (int e = tid; e < m; e += blockDim.x) a.best[e] = es[e];
    const uint64_t mm = (uint64_t)m;
    for (;;) {
        if (master) {
            int kind = 2;
            while (step < a.steps) {
                if (mv >= a.moves) {
                    mv = 0;
                    ++step;
                    temp *= a.cooling;
                    continue;
                }
                ++mv;
                const uint64_t i1 = bounded(*rng, mm);
                uint64_t i2 = bounded(*rng, mm - 1);
                if (i2 >= i1) ++i2;
                const int2 e1 = es[i1], e2 = es[i2];
                if (e1.x == e2.x || e1.x == e2.y || e1.y == e2.x || e1.y == e2.y) continue;
                const bool cross = bounded(*rng, 2) != 0;
                const int2 n1 = ordered2(e1.x, cross ? e2.y : e2.x);
                const int2 n2 = ordered2(e1.y, cross ? e2.x : e2.y);
                if (has_edge(adj, W, n1) || has_edge(adj, W, n2)) continue;
                if (a.allowed) {
                    const long long c[4] = {edge_idx(n, e1.x, e1.y), edge_idx(n, e2.x, e2.y),
                                            edge_idx(n, n1.x, n1.y), edge_idx(n, n2.x, n2.y)};
                    if (!cap_feasible(a, c)) continue;
                }
                kind = 1;
                cmd[1] = (int)i1;
                cmd[2] = (int)i2;
                cmd[3] = n1.x;
                cmd[4] = n1.y;
                cmd[5] = n2.x;
                cmd[6] = n2.y;
                break;
            }
            cmd[0] = kind;
            __threadfence();
        }
        grid.sync();
        if (cmd[0] == 2) break;
        const int i1 = cmd[1], i2 = cmd[2];
        const int2 n1 = make_int2(cmd[3], cmd[4]), n2 = make_int2(cmd[5], cmd[6]);
        if (tid == 0) {
            s_old[0] = es[i1];
            s_old[1] = es[i2];
            set_edge(adj, W, es[i1], false);
            set_edge(adj, W, es[i2], false);
            set_edge(adj, W, n1, true);
            set_edge(adj, W, n2, true);
            es[i1] = n1;
            es[i2] = n2;
        }
        __syncthreads();
        evaluate();
        if (master) {
            const double cand = energy_of();
            const double delta = cand - energy;
            bool take = delta <= 0.0;
            if (!take && isfinite(delta)) take = unit(*rng) < exp(-delta / temp);
            int improved = 0;
            if (take) {
                if (a.allowed) {
                    const int2 o1 = s_old[0], o2 = s_old[1];
                    const long long c[4] = {edge_idx(n, o1.x, o1.y), edge_idx(n, o2.x, o2.y),
                                            edge_idx(n, n1.x, n1.y), edge_idx(n, n2.x, n2.y)};
                    cap_apply(a, c);
                }
                energy = cand;
                if (energy < best_e) {
                    best_e = energy;
                    improved = 1;
                }
            }
            cmd[8] = (take ? 1 : 0) | (improved << 1);
            __threadfence();
        }
        grid.sync();
        const int dec = cmd[8];
        if (!(dec & 1) && tid == 0) {
            set_edge(adj, W, n1, false);
            set_edge(adj, W, n2, false);
            set_edge(adj, W, s_old[0], true);
            set_edge(adj, W, s_old[1], true);
            es[i1] = s_old[0];
            es[i2] = s_old[1];
        }
        __syncthreads();
        if ((dec & 2) && blockIdx.x == 0)
            for (int e = tid; e < m; e += blockDim.x) a.best[e] = es[e];
    }
    if (master) *a.energy_out = best_e;
}

__global__ void mt_kernel(uint64_t seed, int k, uint64_t* out) {
    MT64 s;
    mt_seed(s, seed);
    for (int i = 0; i < k; ++i) out[i] = mt_next(s);
}

template <typename T>
struct Buf {
    T* p = nullptr;
    explicit Buf(size_t n) { TPB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Buf() { cudaFree(p); }
};

}  // namespace

bool anneal_device(int n, std::vector<std::pair<int, int>>& es, const AnnealParams& p, const CapVeto* veto) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return false;
    }
    const int m = (int)es.size();
    if (m < 2 || n < 2) return true;  // nothing to anneal (proj/src/anneal.cpp:190)
    const int W = (n + 31) / 32;
    int GS = 1;
    while (GS < W) GS <<= 1;
    const size_t smem = ((size_t)n * W * 4 + 15) / 16 * 16 + ((size_t)m * 8 + 15) / 16 * 16 + sizeof(MT64);
    int dev = 0, optin = 0, sms = 0, coop = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    TPB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    TPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TPB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop || smem + 1024 > (size_t)optin) return false;
    TPB_CUDA(cudaFuncSetAttribute(anneal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    TPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, anneal_kernel, kThreads, smem));
    if (per_sm < 1) return false;
    const int per_cta = (kThreads / 32) * (32 / GS);
    const int G = std::max(1, std::min(sms, (n + per_cta - 1) / per_cta));

    std::vector<int2> h(m);
    for (int e = 0; e < m; ++e) h[e] = make_int2(es[e].first, es[e].second);
    Buf<int2> d_in(m), d_best(m);
    Buf<unsigned long long> d_part(G);
    Buf<int> d_bad(G), d_cmd(16);
    Buf<double> d_energy(1);
    h2d(d_in.p, h.data(), m * sizeof(int2));
    TPB_CUDA(cudaMemset(d_cmd.p, 0, 16 * sizeof(int)));
    Args a{};
    a.n = n;
    a.m = m;
    a.W = W;
    a.GS = GS;
    a.G = G;
    a.es_in = d_in.p;
    a.best = d_best.p;
    a.t0 = p.t0;
    a.cooling = p.cooling;
    a.steps = p.steps;
    a.moves = p.moves_per_temp > 0 ? p.moves_per_temp : n;
    a.seed = p.seed;
    a.part = d_part.p;
    a.bad = d_bad.p;
    a.cmd = d_cmd.p;
    a.energy_out = d_energy.p;
    const CapVeto empty{};
    const CapVeto& v = veto ? *veto : empty;
    Buf<int> d_allowed(v.allowed.size()), d_crp(v.cr_ptr.size()), d_cr(v.cr.size()), d_caps(v.caps.size()),
        d_load(v.load.size());
    if (veto) {
        h2d(d_allowed.p, v.allowed.data(), v.allowed.size() * sizeof(int));
        h2d(d_crp.p, v.cr_ptr.data(), v.cr_ptr.size() * sizeof(int));
        if (!v.cr.empty()) h2d(d_cr.p, v.cr.data(), v.cr.size() * sizeof(int));
        if (!v.caps.empty()) h2d(d_caps.p, v.caps.data(), v.caps.size() * sizeof(int));
        if (!v.load.empty()) h2d(d_load.p, v.load.data(), v.load.size() * sizeof(int));
        a.allowed = d_allowed.p;
        a.cr_ptr = d_crp.p;
        a.cr = d_cr.p;
        a.caps = d_caps.p;
        a.load = d_load.p;
    }
    void* args[] = {&a};
    TPB_CUDA(cudaLaunchCooperativeKernel((const void*)anneal_kernel, dim3(G), dim3(kThreads), args, smem, 0));
    TPB_CUDA(cudaDeviceSynchronize());
    TPB_CUDA(cudaMemcpy(h.data(), d_best.p, m * sizeof(int2), cudaMemcpyDeviceToHost));
    for (int e = 0; e < m; ++e) es[e] = {h[e].x, h[e].y};
    return true;
}

void device_mt19937_64(uint64_t seed, int k, uint64_t* out) {
    Buf<uint64_t> d(k);
    mt_kernel<<<1, 1>>>(seed, k, d.p);
    TPB_CHECK_LAUNCH();
    TPB_CUDA(cudaMemcpy(out, d.p, k * sizeof(uint64_t), cudaMemcpyDeviceToHost));
}

}  // namespace tpb
