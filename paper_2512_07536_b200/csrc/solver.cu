// Device-resident batched ADMM driver. Mirrors the control flow of
// topoopt::solve / topoopt::solve_het (proj/src/admm.cpp:356-428,
// proj/src/admm_het.cpp:231-369): feasible start, Y-X-D iterations with the
// residual stop test and best-iterate bookkeeping, then extraction and the
// final spectral report. Each iteration is one CUDA-graph segment with three
// streams: cone projections (s0) || top-r selection (s1) -> trace SLEM (s2).
#include "solver.cuh"

#include "nccl_shim.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>

namespace tpb {

void validate(const Config& c) {
    // proj/src/admm.cpp:186-195
    if (!(c.rho > 0.0)) throw Error(kInvalidArgument, "SolverConfig: rho must be positive");
    if (!(c.epsilon > 0.0)) throw Error(kInvalidArgument, "SolverConfig: epsilon must be positive");
    if (c.max_iter < 1) throw Error(kInvalidArgument, "SolverConfig: max_iter must be >= 1");
    if (!(c.alpha > 0.0)) throw Error(kInvalidArgument, "SolverConfig: alpha must be positive");
    if (c.weight_floor < 0.0) throw Error(kInvalidArgument, "SolverConfig: weight_floor must be >= 0");
    if (!(c.linear_tol > 0.0)) throw Error(kInvalidArgument, "SolverConfig: linear_tol must be positive");
    if (c.trace_stride < 1) throw Error(kInvalidArgument, "SolverConfig: trace_stride must be >= 1");
    if (c.linear_solver != 0 && c.linear_solver != 1)
        throw Error(kInvalidArgument, "SolverConfig: linear_solver must be 0 (closed form) or 1 (CG)");
    if (c.linear_solver == 1 && (c.cg_max_iter < 1 || c.cg_max_iter > 64))
        throw Error(kInvalidArgument, "SolverConfig: cg_max_iter must be in [1, 64]");
}

// Built with -DTPB_PHASE_TIMING: device-synchronised phase timings on stderr
// (setup overheads); compiled out otherwise.
void phase_mark(const char* what) {
#ifndef TPB_PHASE_TIMING
    (void)what;
    return;
#else
    static auto last = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tpb] %-24s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
#endif
}

namespace {

// Pinned host blocks for the control-word readback, recycled across solvers:
// cudaMallocHost page-locks memory and occasionally takes tens of
// milliseconds, which showed up in the end-to-end time of short solves.
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;

int* pinned_take(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.lower_bound(bytes);
        if (it != g_pin_free.end()) {
            void* p = it->second;
            g_pin_free.erase(it);
            return static_cast<int*>(p);
        }
    }
    void* p = nullptr;
    const size_t cap = std::max<size_t>(bytes, 4096);
    TPB_CUDA(cudaMallocHost(&p, cap));
    std::memset(p, 0, cap);
    return static_cast<int*>(p);
}

void pinned_give(int* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.emplace(std::max<size_t>(bytes, 4096), p);
}

// Stream-ordered allocation from the device's default memory pool, whose
// release threshold is raised to 1 GiB so that the blocks of recently freed
// solvers stay reserved (repeated tp_solve calls neither map nor unmap device
// memory) while the retention stays bounded for other CUDA users.
template <typename T>
T* dalloc(cudaStream_t st, std::vector<void*>& pool, size_t count) {
    static bool pool_ready[64] = {};
    int dev = 0;
    TPB_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !pool_ready[dev]) {
        cudaMemPool_t mp;
        TPB_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
        uint64_t thr = 1ull << 30;
        TPB_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
        pool_ready[dev] = true;
    }
    void* p = nullptr;
    if (count == 0) count = 1;
    TPB_CUDA(cudaMallocAsync(&p, count * sizeof(T), st));
    pool.push_back(p);
    return static_cast<T*>(p);
}

}  // namespace

Solver::Solver(int n, int B, bool het, const std::vector<int>& r, const std::vector<int>& degrees,
               const Config& cfg, const CapSystem* cap)
    : B_(B), het_(het || cap != nullptr), cfg_(cfg) {
    het = het_;
    phase_mark("(caller, before the solver)");
    validate(cfg);
    if (n < 2) throw Error(kInvalidArgument, "assemble: need at least 2 nodes");
    if (B < 1) throw Error(kInvalidArgument, "batch must be >= 1");
    lo_ = het ? het_layout(n, n) : hom_layout(n);
    const int m = lo_.m;
    r_host_.resize(B);
    if (cap) {
        // proj/src/admm_het.cpp:20-31, 37-48 (check_system, resolve_edge_total)
        cap_ = true;
        capsys_ = *cap;
        if ((int)capsys_.allowed.size() != m)
            throw Error(kInvalidArgument, "capacity system: allowed mask size differs from |E|");
        if ((int)capsys_.row_ptr.size() != capsys_.nrows + 1 || (int)capsys_.caps.size() != capsys_.nrows)
            throw Error(kInvalidArgument, "capacity system: malformed rows");
        for (int c : capsys_.cols)
            if (c < 0 || c >= m)
                throw Error(kInvalidArgument, "capacity system: a row references a column outside [0, |E|)");
        if ((int)r.size() != B) throw Error(kInvalidArgument, "capacity-bound system needs an explicit edge total");
        for (int b = 0; b < B; ++b) {
            if (r[b] < 1 || r[b] > m) throw Error(kInvalidArgument, "assemble_het: edge total outside [1, |E|]");
            r_host_[b] = r[b];
        }
    } else if (het) {
        if ((int)degrees.size() != B * n)
            throw Error(kInvalidArgument, "node_level_constraints: degree list size mismatch");
        for (int b = 0; b < B; ++b) {
            long long sum = 0;
            for (int i = 0; i < n; ++i) {
                const int dgi = degrees[(size_t)b * n + i];
                if (dgi < 0 || dgi > n - 1)
                    throw Error(kInvalidArgument, "node_level_constraints: degree of node " +
                                                      std::to_string(i) + " outside [0, n-1]");
                sum += dgi;
            }
            if (sum % 2) throw Error(kInfeasible, "degree sum " + std::to_string(sum) + " is odd");
            const int total = (int)(sum / 2);
            if (!r.empty() && r[b] >= 0 && r[b] != total)
                throw Error(kInvalidArgument, "edge total conflicts with the degree rows");
            if (total < 1 || total > m)
                throw Error(kInvalidArgument, "assemble_het: edge total outside [1, |E|]");
            r_host_[b] = total;
        }
    } else {
        if ((int)r.size() != B) throw Error(kInvalidArgument, "one edge budget per solve expected");
        for (int b = 0; b < B; ++b) {
            if (r[b] < 1 || r[b] > m) throw Error(kInvalidArgument, "assemble: r outside [1, n(n-1)/2]");
            r_host_[b] = r[b];
        }
    }
    if (cfg.linear_solver == 1 && het_)
        throw Error(kInvalidArgument,
                    "SolverConfig: the CG x-step covers the homogeneous system; the node-level "
                    "system (stiff 1e8 coupling) uses the closed form");
    c_ = make_xconst(n, cfg.alpha, cfg.rho);
    small_ = n <= 64;
    // Tiled projections (n > 64): int8 tensor-core (Ozaki) GEMMs, ld % 128 == 0.
    ozaki_ = !small_;
    if (ozaki_) sch_ = ozaki_schedule();
    ld_ = small_ ? ((n + 7) & ~7) : ((n + 127) / 128) * 128;
    if (ozaki_) check_oz_ld(ld_);
    list_cap_ = het ? m : *std::max_element(r_host_.begin(), r_host_.end());
    int chunk = cfg.chunk > 0 ? cfg.chunk : (n <= 64 ? 32 : (n <= 256 ? 16 : 8));
    // a multiple of the trace stride (the SLEM pattern repeats per chunk) and
    // a multiple of kSets (chunks start and end at selection set 0)
    int unit = cfg.trace_stride;
    while (unit % kSets) unit += cfg.trace_stride;
    chunk_ = ((chunk + unit - 1) / unit) * unit;
    init_attrs();
    phase_mark("solver init_attrs");
    TPB_CUDA(cudaStreamCreateWithFlags(&s0_, cudaStreamNonBlocking));
    TPB_CUDA(cudaStreamCreateWithFlags(&s1_, cudaStreamNonBlocking));
    for (auto& st : s2_) TPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    TPB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    TPB_CUDA(cudaEventCreateWithFlags(&ev_sel_, cudaEventDisableTiming));
    TPB_CUDA(cudaEventCreateWithFlags(&ev_slem_, cudaEventDisableTiming));
    for (auto& e : ev_slem_p_) TPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    phase_mark("solver streams");
    alloc();
    if (het && !cap_) {
        std::vector<double> dg(degrees.begin(), degrees.end());
        h2d(d_deg_, dg.data(), dg.size() * sizeof(double));
    }
    if (cap_) {
        // column -> rows CSR for the capped projection
        std::vector<int> cnt(m + 1, 0), colr(capsys_.cols.size());
        for (int c : capsys_.cols) ++cnt[c + 1];
        for (int l = 0; l < m; ++l) cnt[l + 1] += cnt[l];
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int rr = 0; rr < capsys_.nrows; ++rr)
            for (int q = capsys_.row_ptr[rr]; q < capsys_.row_ptr[rr + 1]; ++q) colr[pos[capsys_.cols[q]]++] = rr;
        h2d(cap_colr_ptr_, cnt.data(), cnt.size() * sizeof(int));
        if (!colr.empty())
            h2d(cap_colr_, colr.data(), colr.size() * sizeof(int));
        h2d(cap_caps_, capsys_.caps.data(), capsys_.nrows * sizeof(int));
        h2d(cap_allowed_, capsys_.allowed.data(), m * sizeof(int));
    }
    h2d(d_r_, r_host_.data(), B * sizeof(int));
    warm_.assign(B, {});
    res_.assign(B, {});
    phase_mark("solver alloc");
}

Solver::~Solver() {
    phase_mark("(before teardown)");
    if (g_chunk_) cudaGraphExecDestroy(g_chunk_);
    for (auto& g1 : g_one_)
        if (g1) cudaGraphExecDestroy(g1);
    phase_mark("graph destroy");
    // stream-ordered frees return the blocks to the device pool (no unmap)
    for (void* p : allocs_) cudaFreeAsync(p, s0_);
    cudaStreamSynchronize(s0_);
    phase_mark("free");
    if (h_ctl_) pinned_give(h_ctl_, (size_t)B_ * 8 * sizeof(int));
    release_shard();
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_sel_) cudaEventDestroy(ev_sel_);
    if (ev_slem_) cudaEventDestroy(ev_slem_);
    for (auto& e : ev_slem_p_)
        if (e) cudaEventDestroy(e);
    if (s0_) cudaStreamDestroy(s0_);
    if (s1_) cudaStreamDestroy(s1_);
    for (auto& st : s2_)
        if (st) cudaStreamDestroy(st);
}

void Solver::alloc() {
    const int n = lo_.n;
    const long long m = lo_.m, nx = lo_.nx;
    const int B = B_;
    d_.lo = lo_;
    d_.B = B;
    d_.het = het_ ? 1 : 0;
    d_.cap = cap_ ? 1 : 0;
    d_.nb = (n + 31) / 32;
    d_.ntile = d_.nb * (d_.nb + 1) / 2;
    d_.ld = ld_;
    d_.nx = nx;
    d_.max_iter = cfg_.max_iter;
    d_.epsilon = cfg_.epsilon;
    d_.track_best = 1;
    d_.upd_duals = 1;
    const long long ld2 = (long long)ld_ * ld_;
    d_.X = dalloc<double>(s0_, allocs_,B * nx);
    d_.Y = dalloc<double>(s0_, allocs_,B * nx);
    d_.D = dalloc<double>(s0_, allocs_,B * nx);
    d_.bestY = dalloc<double>(s0_, allocs_,B * nx);
    d_.bestScore = dalloc<double>(s0_, allocs_,het_ ? B * m : 1);
    d_.A = dalloc<double>(s0_, allocs_,(size_t)B * 2 * ld2);
    TPB_CUDA(cudaMemsetAsync(d_.A, 0, (size_t)B * 2 * ld2 * sizeof(double), s0_));
    d_.frob_part = dalloc<double>(s0_, allocs_,(size_t)B * 2 * d_.ntile);
    d_.inv_scale = dalloc<double>(s0_, allocs_,(size_t)B * 2);
    d_.row_part = dalloc<double>(s0_, allocs_, (size_t)B * 2 * d_.nb * n);
    d_.h = dalloc<double>(s0_, allocs_,B * m);
    if (cfg_.linear_solver == 1) {
        d_.cg = 1;
        d_.cg_max = cfg_.cg_max_iter;
        d_.cg_tol2 = cfg_.linear_tol * cfg_.linear_tol;
        d_.cg_x = dalloc<double>(s0_, allocs_, B * m);
        d_.cg_p = dalloc<double>(s0_, allocs_, B * m);
        d_.cg_pq = dalloc<double>(s0_, allocs_, (size_t)B * d_.ntile);
        d_.cg_rr = dalloc<double>(s0_, allocs_, (size_t)B * 2 * d_.ntile);
        d_.cg_nr = dalloc<double>(s0_, allocs_, (size_t)B * d_.nb * n);
        d_.cg_u = dalloc<double>(s0_, allocs_, (size_t)B * 2 * n);
        d_.cg_grid = cg_launch_grid(d_);
    }
    d_.PU = dalloc<double>(s0_, allocs_,(size_t)B * d_.nb * n);
    d_.PZ = dalloc<double>(s0_, allocs_,(size_t)B * d_.nb * n);
    d_.PG = dalloc<double>(s0_, allocs_,(size_t)B * d_.nb * n);
    d_.node = dalloc<double>(s0_, allocs_,(size_t)B * 4 * n);
    d_.tile_aux = dalloc<double>(s0_, allocs_, (size_t)B * d_.ntile * 2);
    d_.blk = dalloc<double>(s0_, allocs_, (size_t)B * d_.nb * 4);
    d_.res_node = dalloc<double>(s0_, allocs_, (size_t)B * n);
    d_.blk_inf = dalloc<double>(s0_, allocs_, (size_t)B * 2 * d_.nb);
    d_.cnt_stride = 2 * d_.nb + 2;
    d_.cnt = dalloc<int>(s0_, allocs_, (size_t)B * d_.cnt_stride);
    TPB_CUDA(cudaMemsetAsync(d_.cnt, 0, (size_t)B * d_.cnt_stride * sizeof(int), s0_));
    d_.res_part = dalloc<double>(s0_, allocs_,(size_t)B * d_.ntile);
    d_.scal = dalloc<double>(s0_, allocs_,(size_t)B * 8);
    d_.ictl = dalloc<int>(s0_, allocs_,(size_t)B * 8);
    d_r_ = dalloc<int>(s0_, allocs_,B);
    d_.r = d_r_;
    d_deg_ = dalloc<double>(s0_, allocs_,het_ ? (size_t)B * n : 1);
    d_.deg = d_deg_;
    d_.tr_res = dalloc<double>(s0_, allocs_,(size_t)B * cfg_.max_iter);
    d_.tr_lam = dalloc<double>(s0_, allocs_,(size_t)B * cfg_.max_iter);
    d_.tr_acf = dalloc<double>(s0_, allocs_,(size_t)B * cfg_.max_iter);
    phase_mark("alloc: state and scratch");
    if (ozaki_) {
        // digit planes of the cone-projection iterates
        for (int q = 0; q < 4; ++q) {
            oz_.d[q] = dalloc<int8_t>(s0_, allocs_, (size_t)B * 2 * kOzSlices * ld2);
            pool_planes_[q] = oz_.d[q];
            TPB_CUDA(cudaMemsetAsync(oz_.d[q], 0, (size_t)B * 2 * kOzSlices * ld2, s0_));
            make_oz_maps(oz_.d[q], ld_, 2 * B, &oz_.maps[q]);
        }
        phase_mark("alloc: digit planes + TMA maps");
    }
    if (cap_) {
        cap_pad_ = 1;
        while (cap_pad_ < m) cap_pad_ <<= 1;
        cap_colr_ptr_ = dalloc<int>(s0_, allocs_, (size_t)m + 1);
        cap_colr_ = dalloc<int>(s0_, allocs_, std::max<size_t>(capsys_.cols.size(), 1));
        cap_caps_ = dalloc<int>(s0_, allocs_, std::max(capsys_.nrows, 1));
        cap_allowed_ = dalloc<int>(s0_, allocs_, (size_t)m);
        cap_keys_ = dalloc<unsigned long long>(s0_, allocs_, (size_t)B * cap_pad_);
        cap_idx_ = dalloc<int>(s0_, allocs_, (size_t)B * cap_pad_);
        cap_load_ = dalloc<int>(s0_, allocs_, (size_t)B * std::max(capsys_.nrows, 1));
        TPB_CUDA(cudaStreamSynchronize(s0_));
    }
    if (het_ && n > kSmallDense) {
        // node-major incidence of dense het supports for the trace SLEM
        for (int L = 0; L < kLanes; ++L) {
            slem_nbr_[L] = dalloc<int>(s0_, allocs_, (size_t)B * 2 * list_cap_);
            slem_nwt_[L] = dalloc<double>(s0_, allocs_, (size_t)B * 2 * list_cap_);
        }
    }
    if (!het_ && !cap_ && B == 1 && m >= kTopRGridMin) {
        topr_gh_ = dalloc<int>(s0_, allocs_, kTopRGridHist);
        TPB_CUDA(cudaMemsetAsync(topr_gh_, 0, kTopRGridHist * sizeof(int), s0_));  // kept zero by each launch
        topr_cnt_ = dalloc<int>(s0_, allocs_, 2 * (size_t)topr_grid_ctas(m));
    }
    list_ = dalloc<int>(s0_, allocs_,(size_t)B * list_cap_);
    list_count_ = dalloc<int>(s0_, allocs_,B);
    tlist_[0] = list_;
    tcount_[0] = list_count_;
    for (int q = 0; q < kSets; ++q) {
        if (q > 0) {
            tlist_[q] = dalloc<int>(s0_, allocs_, (size_t)B * list_cap_);
            tcount_[q] = dalloc<int>(s0_, allocs_, B);
        }
        tlw_[q] = dalloc<double>(s0_, allocs_, (size_t)B * list_cap_);
        tsnap_[q] = dalloc<int>(s0_, allocs_, B);
    }
    for (int L = 0; L < kLanes; ++L) {
        e_i_[L] = dalloc<int>(s0_, allocs_, (size_t)B * list_cap_);
        e_j_[L] = dalloc<int>(s0_, allocs_, (size_t)B * list_cap_);
        col_idx_[L] = dalloc<int>(s0_, allocs_, (size_t)B * list_cap_);
        e_w_[L] = dalloc<double>(s0_, allocs_, (size_t)B * list_cap_);
    }
    // trace Lanczos: exact for n <= 97, else restarted and warm-started from
    // the previous Ritz vectors; basis in shared memory when it fits
    // Krylov basis in global memory: a shared-memory basis (~200 KB at n=256)
    // would pin one SLEM CTA per SM and starve the concurrent cone GEMMs.
    // plain trace Lanczos (slem_trace_kernel): longer recurrences, write-only basis
    trace_kmax_ = std::max(1, std::min(n - 1, n > kSmallDense ? 256 : 96));
    for (int L = 0; L < kLanes; ++L) {
        basis_[L] = dalloc<double>(s0_, allocs_, (size_t)B * trace_kmax_ * n);
        ritz_[L] = dalloc<double>(s0_, allocs_, (size_t)B * 2 * n);
        ritz_ok_[L] = dalloc<int>(s0_, allocs_, B);
    }
    // one-off reports: complete space up to kFinalExactDim, else one long
    // plain-Lanczos cycle
    kfin_ = n - 1 <= kFinalExactDim ? std::max(1, n - 1) : slem_oneoff_kmax(n);
    basis_final_ = dalloc<double>(s0_, allocs_, (size_t)B * kfin_ * n);
    slem_out_ = dalloc<double>(s0_, allocs_,(size_t)B * 8);
    tmp_m_ = dalloc<double>(s0_, allocs_,(size_t)B * m);
    tmp_m2_ = dalloc<double>(s0_, allocs_,(size_t)B * m);
    worst_ = dalloc<double>(s0_, allocs_,B);
    fs_scal_ = dalloc<double>(s0_, allocs_,(size_t)B * 2);
    h_ctl_ = pinned_take((size_t)B * 8 * sizeof(int));
    TPB_CUDA(cudaMemsetAsync(d_.ictl, 0, (size_t)B * 8 * sizeof(int), s0_));
    // allocations are ordered on s0_; later work also runs on s1_/s2_ and the
    // legacy stream, so complete them here
    TPB_CUDA(cudaStreamSynchronize(s0_));
}

void Solver::set_warm(int b, const std::vector<int>& packed) {
    if (b < 0 || b >= B_) throw Error(kInvalidArgument, "set_warm: solve index out of range");
    if ((int)packed.size() > r_host_[b])
        throw Error(kInvalidArgument, het_ ? "solve_het: warm start has more than r edges"
                                           : "solve: warm start has more than r edges");
    warm_[b] = packed;
}

void Solver::start() {
    const int B = B_;
    const long long nx = lo_.nx;
    TPB_CUDA(cudaMemsetAsync(d_.X, 0, B * nx * sizeof(double), s0_));
    TPB_CUDA(cudaMemsetAsync(d_.D, 0, B * nx * sizeof(double), s0_));
    TPB_CUDA(cudaMemsetAsync(d_.ictl, 0, (size_t)B * 8 * sizeof(int), s0_));
    for (auto* r : ritz_ok_) TPB_CUDA(cudaMemsetAsync(r, 0, (size_t)B * sizeof(int), s0_));
    if (het_) TPB_CUDA(cudaMemsetAsync(d_.bestScore, 0, (size_t)B * lo_.m * sizeof(double), s0_));
    {
        std::vector<double> sc((size_t)B * 8, 0.0);
        for (int b = 0; b < B; ++b) sc[(size_t)b * 8 + kBestRes] = std::numeric_limits<double>::infinity();
        TPB_CUDA(cudaMemcpyAsync(d_.scal, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice, s0_));
        std::vector<double> nanv((size_t)B * cfg_.max_iter, std::numeric_limits<double>::quiet_NaN());
        TPB_CUDA(cudaMemcpyAsync(d_.tr_acf, nanv.data(), nanv.size() * sizeof(double), cudaMemcpyHostToDevice, s0_));
        // warm lists
        std::vector<int> lists((size_t)B * list_cap_, 0), counts(B, 0);
        for (int b = 0; b < B; ++b) {
            counts[b] = (int)warm_[b].size();
            std::copy(warm_[b].begin(), warm_[b].end(), lists.begin() + (size_t)b * list_cap_);
        }
        TPB_CUDA(cudaMemcpyAsync(list_, lists.data(), lists.size() * sizeof(int), cudaMemcpyHostToDevice, s0_));
        TPB_CUDA(cudaMemcpyAsync(list_count_, counts.data(), B * sizeof(int), cudaMemcpyHostToDevice, s0_));
        launch_feasible_a(d_, list_, list_count_, list_cap_, fs_scal_, s0_);
        final_slem(d_.X, list_, list_count_, slem_out_);  // SLEM of the warm start, stride nx
        phase_mark("feasible start (pre-SLEM)");
        launch_feasible_b(d_, c_, slem_out_, fs_scal_, s0_);
        phase_mark("feasible SLEM + fill");
        TPB_CUDA(cudaStreamSynchronize(s0_));  // host vectors above go out of scope
    }
    TPB_CUDA(cudaMemcpyAsync(d_.Y, d_.X, B * nx * sizeof(double), cudaMemcpyDeviceToDevice, s0_));
    TPB_CUDA(cudaMemcpyAsync(d_.bestY, d_.X, B * nx * sizeof(double), cudaMemcpyDeviceToDevice, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
    if (!g_chunk_ && !eager()) build_graphs();
    phase_mark("graph capture");
    it_enqueued_ = 0;
}

void Solver::final_slem(const double* packed, const int* list, const int* count, double* out) {
    SlemArgs a{};
    a.n = lo_.n;
    a.m = lo_.m;
    a.g = packed;
    a.stride = packed == d_.X ? lo_.nx : lo_.m;
    a.list = list;
    a.count = count;
    a.list_cap = list_cap_;
    a.e_i = e_i_[0];
    a.e_j = e_j_[0];
    a.e_w = e_w_[0];
    a.col_idx = col_idx_[0];
    // exact (complete Krylov space, CGS2) up to n = 257; beyond, the plain
    // Lanczos recurrence of the trace kernel at residual tolerance 1e-10
    // (eigenvalue error <= 1e-20 / gap) in one cycle of up to kfin_ steps
    const int n = lo_.n;
    const bool exact = n - 1 <= kFinalExactDim;
    a.plain = exact ? 0 : 1;
    a.basis = basis_final_;
    a.kmax = kfin_;
    // the report's Lanczos spread over a cluster of CTAs per solve (node
    // slices, q shared through distributed shared memory); for every batch
    // size, so a batch reproduces the single solve bit for bit
    a.cluster = kOneOffCluster;
    // the final topology is the last trace iterate's neighbour: start from
    // the trace's extreme Ritz vectors (tolerance unchanged)
    if (a.plain) {
        a.ritz = ritz_[0];
        a.ritz_ok = ritz_ok_[0];
    }
    a.max_restarts = 200;
    // first residual check: the plain recurrence at n ~ 1000 needs ~380
    // steps to 1e-10, so a check at 128 is wasted (a check at k costs ~k us)
    a.min_steps = std::min(std::max(64, lo_.n / 4), 256);
    a.check_every = 128;
    a.tol = 1e-10;
    a.out = out;
    a.tr_acf = nullptr;
    a.ictl = nullptr;
    launch_slem(a, B_, s0_);
}

void Solver::enqueue_select(cudaStream_t st, int parity) {
    SelectArgs a{};
    a.stride = lo_.nx;
    a.m = lo_.m;
    a.r = d_r_;
    a.list = tlist_[parity];
    a.list_count = tcount_[parity];
    a.list_cap = list_cap_;
    a.list_w = tlw_[parity];
    a.it_snap = tsnap_[parity];
    a.done = d_.ictl;
    if (cap_) {
        // project_binary_z_capped on the z block, then the g support for the SLEM
        CappedArgs c{};
        c.base = d_.Y + lo_.off_z;
        c.stride = lo_.nx;
        c.m = lo_.m;
        c.r = d_r_;
        c.colr_ptr = cap_colr_ptr_;
        c.colr = cap_colr_;
        c.caps = cap_caps_;
        c.nrows = capsys_.nrows;
        c.allowed = cap_allowed_;
        c.keys = cap_keys_;
        c.idx = cap_idx_;
        c.load = cap_load_;
        c.pad = cap_pad_;
        c.done = d_.ictl;
        launch_capped_z(c, B_, st);
        launch_compact(d_.Y, lo_.nx, lo_.m, tlist_[parity], tcount_[parity], list_cap_, B_, st, tlw_[parity],
                       tsnap_[parity], d_.ictl);
        return;
    }
    if (het_) {
        a.base = d_.Y + lo_.off_z;
        a.gbase = d_.Y;
        a.binary = 1;
    } else {
        a.base = d_.Y;
        a.gbase = nullptr;
        a.binary = 0;
    }
    if (topr_gh_) {
        launch_topr_grid(a, topr_gh_, topr_cnt_, st);  // one large solve: the whole GPU
        return;
    }
    launch_topr(a, B_, st);
}

void Solver::enqueue_slem_trace(cudaStream_t st, int parity) {
    SlemArgs a{};
    a.n = lo_.n;
    a.m = lo_.m;
    a.g = d_.Y;
    a.gw = tlw_[parity];  // weights captured by the select kernel (Y moves on)
    a.it_snap = tsnap_[parity];
    a.stride = lo_.nx;
    a.list = tlist_[parity];
    a.count = tcount_[parity];
    a.list_cap = list_cap_;
    const int L = parity % kLanes;
    a.e_i = e_i_[L];
    a.e_j = e_j_[L];
    a.e_w = e_w_[L];
    a.col_idx = col_idx_[L];
    a.basis = basis_[L];
    a.kmax = trace_kmax_;
    a.max_restarts = 40;
    a.min_steps = 8;
    a.check_every = 24;
    a.noise = 0.0;
    a.ritz = ritz_[L];
    a.ritz_ok = ritz_ok_[L];
    a.tol = cfg_.slem_tol;
    a.out = nullptr;
    a.tr_acf = d_.tr_acf;
    a.ictl = d_.ictl;
    a.max_iter = cfg_.max_iter;
    a.plain = lo_.n > kSmallDense;
    a.nbr = slem_nbr_[L];
    a.nwt = slem_nwt_[L];
    launch_slem(a, B_, st);
}

void Solver::enqueue_projection() {
    const long long cb = lo_.nx, cw = lo_.off_t - lo_.off_s;
    if (small_) {
        launch_cone_small(d_.A, (long long)ld_ * ld_, ld_, lo_.n, d_.Y + lo_.off_s, cb, cw, d_.ictl,
                          2 * B_, sch_, s0_);
    } else {
        enqueue_cone_ozaki(d_.A, oz_, ld_, lo_.n, d_.inv_scale, d_.Y + lo_.off_s, cb, cw, d_.ictl, 2 * B_,
                           sch_, s0_, sharded() ? &shard_ : nullptr);
    }
}

void Solver::release_shard() {
    TPB_CUDA(cudaDeviceSynchronize());
    for (int r = 0; r < kOzMaxRanks; ++r) {
        if (r == shard_.rank) continue;
        for (int q = 0; q < 4; ++q)
            if (shard_.peer_d[q][r]) cudaIpcCloseMemHandle(shard_.peer_d[q][r]);
        if (shard_.peer_flags[r]) cudaIpcCloseMemHandle(shard_.peer_flags[r]);
    }
    for (void* p : shard_mem_) cudaFree(p);
    shard_mem_.clear();
    shard_ = OzShard{};
}

// Sharded projection over the ranks of `comm`: the digit
// buffers (plain cudaMalloc, IPC-exportable) and a flag array per rank are
// mapped into every rank through CUDA IPC handles exchanged with one NCCL
// all-gather; the GEMM epilogues then store each tile into every rank's
// buffer over NVLink (ozaki_kernels.cuh, OzShard).
void Solver::set_shard(void* comm, int nranks, int rank) {
    if (sharded() || !shard_mem_.empty()) {
        // back to the pool-allocated planes of alloc()
        for (int q = 0; q < 4; ++q) oz_.d[q] = pool_planes_[q];
        for (int q = 0; q < 4 && ozaki_; ++q) make_oz_maps(oz_.d[q], ld_, 2 * B_, &oz_.maps[q]);
        release_shard();
    }
    if (nranks > 1) {
        if (!ozaki_) throw Error(kInvalidArgument, "sharded projection: needs the tiled Ozaki path (n > 64)");
        if (B_ != 1) throw Error(kInvalidArgument, "sharded projection: one instance per solver");
        if (nranks > kOzMaxRanks) throw Error(kInvalidArgument, "sharded projection: at most 8 ranks");
        const std::vector<int> t = oz_shard_tiles(ld_, nranks, rank);
        TPB_CUDA(cudaStreamSynchronize(s0_));
        const size_t pbytes = (size_t)2 * kOzSlices * ld_ * ld_;
        auto raw = [&](size_t bytes) {
            void* p = nullptr;
            TPB_CUDA(cudaMalloc(&p, bytes));
            TPB_CUDA(cudaMemset(p, 0, bytes));
            shard_mem_.push_back(p);
            return p;
        };
        for (int q = 0; q < 4; ++q) {
            oz_.d[q] = static_cast<int8_t*>(raw(pbytes));
            make_oz_maps(oz_.d[q], ld_, 2, &oz_.maps[q]);
        }
        shard_.flags = static_cast<unsigned long long*>(raw(kOzMaxRanks * sizeof(unsigned long long)));
        shard_.done = static_cast<int*>(raw(sizeof(int)));
        shard_.err = static_cast<int*>(raw(sizeof(int)));
        int* dtiles = static_cast<int*>(raw(t.size() * sizeof(int)));
        h2d(dtiles, t.data(), t.size() * sizeof(int));
        // IPC handles of the 4 digit buffers and the flag array, all-gathered
        constexpr int NH = 5;
        std::vector<cudaIpcMemHandle_t> mine(NH), all((size_t)NH * nranks);
        for (int q = 0; q < 4; ++q) TPB_CUDA(cudaIpcGetMemHandle(&mine[q], oz_.d[q]));
        TPB_CUDA(cudaIpcGetMemHandle(&mine[4], shard_.flags));
        const size_t hb = NH * sizeof(cudaIpcMemHandle_t);
        void* dh = raw(hb * nranks);
        h2d(static_cast<char*>(dh) + hb * rank, mine.data(), hb);
        TPB_NCCL(nccl().all_gather(static_cast<char*>(dh) + hb * rank, dh, hb, ncclInt8,
                                   static_cast<ncclComm_t>(comm), s0_));
        TPB_CUDA(cudaStreamSynchronize(s0_));
        TPB_CUDA(cudaMemcpy(all.data(), dh, hb * nranks, cudaMemcpyDeviceToHost));
        shard_.rank = rank;
        shard_.nranks = nranks;
        shard_.comm = comm;
        shard_.tiles = dtiles;
        shard_.ntiles = (int)t.size();
        shard_.epoch = 0;
        for (int r = 0; r < nranks; ++r) {
            if (r == rank) {
                for (int q = 0; q < 4; ++q) shard_.peer_d[q][r] = oz_.d[q];
                shard_.peer_flags[r] = shard_.flags;
                continue;
            }
            for (int q = 0; q < 4; ++q) {
                void* p = nullptr;
                TPB_CUDA(cudaIpcOpenMemHandle(&p, all[(size_t)r * NH + q], cudaIpcMemLazyEnablePeerAccess));
                shard_.peer_d[q][r] = static_cast<int8_t*>(p);
            }
            void* f = nullptr;
            TPB_CUDA(cudaIpcOpenMemHandle(&f, all[(size_t)r * NH + 4], cudaIpcMemLazyEnablePeerAccess));
            shard_.peer_flags[r] = static_cast<unsigned long long*>(f);
        }
        // every rank's buffers exist and are zeroed before anyone stores
        TPB_NCCL(nccl().all_gather(static_cast<char*>(dh) + hb * rank, dh, hb, ncclInt8,
                                   static_cast<ncclComm_t>(comm), s0_));
        TPB_CUDA(cudaStreamSynchronize(s0_));
    }
    // graphs captured before hold the old projection
    if (g_chunk_) cudaGraphExecDestroy(g_chunk_);
    for (auto& g1 : g_one_) {
        if (g1) cudaGraphExecDestroy(g1);
        g1 = nullptr;
    }
    g_chunk_ = nullptr;
}

void Solver::check_shard() {
    if (!sharded()) return;
    int e = 0;
    TPB_CUDA(cudaMemcpy(&e, shard_.err, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) throw Error(kCuda, "sharded projection: a peer did not publish its product (timeout)");
}

// One ADMM iteration on three streams: prep on s0, then the
// selection (top-r / binary z) on s1 beside the cone projections on s0; the
// x-step joins the selection. The trace SLEM of this iteration runs on s2 from
// the selection's parity buffers and is joined by nobody in the iteration: it
// overlaps the next iteration, whose successor's selection (same parity)
// waits for it. Stream capture and eager chunks end with join_slem().
void Solver::enqueue_iteration(bool with_slem, int parity) {
    launch_prep(d_, c_, s0_);
    TPB_CUDA(cudaEventRecord(ev_fork_, s0_));
    TPB_CUDA(cudaStreamWaitEvent(s1_, ev_fork_, 0));
    if (slem_pending_[parity]) TPB_CUDA(cudaStreamWaitEvent(s1_, ev_slem_p_[parity], 0));
    enqueue_select(s1_, parity);
    TPB_CUDA(cudaEventRecord(ev_sel_, s1_));
    slem_pending_[parity] = false;
    if (with_slem) {
        const int L = parity % kLanes;
        TPB_CUDA(cudaStreamWaitEvent(s2_[L], ev_sel_, 0));
        enqueue_slem_trace(s2_[L], parity);
        TPB_CUDA(cudaEventRecord(ev_slem_p_[parity], s2_[L]));
        slem_pending_[parity] = true;
        slem_any_[L] = true;
        slem_last_[L] = parity;
    }
    enqueue_projection();
    TPB_CUDA(cudaStreamWaitEvent(s0_, ev_sel_, 0));
    enqueue_xstep(d_);
    launch_best_copy(d_, c_, s0_);
}

void Solver::join_slem(cudaStream_t st) {
    for (int L = 0; L < kLanes; ++L) {
        if (slem_any_[L]) TPB_CUDA(cudaStreamWaitEvent(st, ev_slem_p_[slem_last_[L]], 0));
        slem_any_[L] = false;
    }
    for (auto& p : slem_pending_) p = false;
}

void Solver::enqueue_xstep(const Dev& d) {
    launch_xstep_a(d, c_, s0_);
    if (d.cg) launch_xstep_cg(d, c_, s0_);
    launch_xstep_b(d, c_, s0_);
}

void Solver::cg_stats(int b, int* iters, double* rel_res) {
    if (b < 0 || b >= B_) throw Error(kInvalidArgument, "cg_stats: solve index out of range");
    int it = 0;
    double rr = 0.0;
    TPB_CUDA(cudaStreamSynchronize(s0_));
    if (d_.cg) {
        TPB_CUDA(cudaMemcpy(&it, d_.ictl + b * 8 + kCgIters, sizeof(int), cudaMemcpyDeviceToHost));
        TPB_CUDA(cudaMemcpy(&rr, d_.scal + b * 8 + kCgRes, sizeof(double), cudaMemcpyDeviceToHost));
    }
    *iters = it;
    *rel_res = rr;
}

void Solver::build_graphs() {
    // chunk_ is a multiple of kSets: a chunk starts and ends at set 0;
    // single-iteration graphs exist for every set
    auto capture = [&](int iters, int parity0, bool stride_aligned) {
        cudaGraph_t g;
        for (auto& p : slem_pending_) p = false;  // earlier graphs have completed
        for (auto& a : slem_any_) a = false;
        TPB_CUDA(cudaStreamBeginCapture(s0_, cudaStreamCaptureModeThreadLocal));
        for (int j = 0; j < iters; ++j) {
            const bool slem = stride_aligned ? (j % cfg_.trace_stride == 0) : (cfg_.trace_stride == 1);
            enqueue_iteration(slem, (parity0 + j) % kSets);
        }
        join_slem(s0_);
        TPB_CUDA(cudaStreamEndCapture(s0_, &g));
        cudaGraphExec_t ex;
        TPB_CUDA(cudaGraphInstantiate(&ex, g, 0));
        TPB_CUDA(cudaGraphDestroy(g));
        return ex;
    };
    g_chunk_ = capture(chunk_, 0, true);
    for (int q = 0; q < kSets; ++q) g_one_[q] = capture(1, q, false);
}

// Sharded solvers launch their iterations eagerly: the all-gathers' stream
// priority (SMs to the NCCL CTAs first) does not survive graph capture, and
// at the sizes that shard a launch is ~0.01 % of an iteration. Same
// iteration sequence as the graphs.
bool Solver::eager() const { return sharded(); }

void Solver::iterate_async(int k) {
    if (eager()) {
        while (k > 0) {
            const int run = (it_enqueued_ % kSets == 0 && k >= chunk_) ? chunk_ : 1;
            for (int j = 0; j < run; ++j) {
                const bool slem = run == chunk_ ? (j % cfg_.trace_stride == 0) : (cfg_.trace_stride == 1);
                enqueue_iteration(slem, (it_enqueued_ + j) % kSets);
            }
            join_slem(s0_);
            k -= run;
            it_enqueued_ += run;
        }
        return;
    }
    while (k > 0) {
        if (it_enqueued_ % kSets == 0 && k >= chunk_) {
            TPB_CUDA(cudaGraphLaunch(g_chunk_, s0_));
            k -= chunk_;
            it_enqueued_ += chunk_;
        } else {
            TPB_CUDA(cudaGraphLaunch(g_one_[it_enqueued_ % kSets], s0_));
            --k;
            ++it_enqueued_;
        }
    }
}

bool Solver::all_done() {
    TPB_CUDA(cudaMemcpyAsync(h_ctl_, d_.ictl, (size_t)B_ * 8 * sizeof(int), cudaMemcpyDeviceToHost, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
    check_shard();
    for (int b = 0; b < B_; ++b)
        if (d_.cg && h_ctl_[b * 8 + kCgFail])
            throw Error(kLinearSolve, "update_X: CG relative residual above 1e-8 (solve " + std::to_string(b) +
                                          "; raise cg_max_iter)");
    for (int b = 0; b < B_; ++b)
        if (!h_ctl_[b * 8 + kDone]) return false;
    return true;
}

void Solver::run_to_completion() {
    while (!all_done()) iterate_async(chunk_);
}

void Solver::finish() {
    TPB_CUDA(cudaStreamSynchronize(s0_));
    all_done();
    std::vector<double> scal((size_t)B_ * 8);
    TPB_CUDA(cudaMemcpy(scal.data(), d_.scal, scal.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int b = 0; b < B_; ++b) {
        SolveResult& R = res_[b];
        R = SolveResult{};
        R.iterations = h_ctl_[b * 8 + kIter];
        R.converged = h_ctl_[b * 8 + 4] != 0;
        R.best_iter = h_ctl_[b * 8 + kBestIter];
        R.residual = R.converged ? scal[(size_t)b * 8 + kRes] : scal[(size_t)b * 8 + kBestRes];
        if (!R.converged)
            R.note = "stopped at max_iter; best iterate from iteration " + std::to_string(R.best_iter);
        const int it = R.iterations;
        R.tr_res.resize(it);
        R.tr_lam.resize(it);
        R.tr_acf.resize(it);
        const size_t off = (size_t)b * cfg_.max_iter;
        TPB_CUDA(cudaMemcpy(R.tr_res.data(), d_.tr_res + off, it * sizeof(double), cudaMemcpyDeviceToHost));
        TPB_CUDA(cudaMemcpy(R.tr_lam.data(), d_.tr_lam + off, it * sizeof(double), cudaMemcpyDeviceToHost));
        TPB_CUDA(cudaMemcpy(R.tr_acf.data(), d_.tr_acf + off, it * sizeof(double), cudaMemcpyDeviceToHost));
        const double* pick = (R.converged ? d_.Y : d_.bestY) + (size_t)b * lo_.nx;
        TPB_CUDA(cudaMemcpy(&R.lambda_tilde, pick + lo_.lambda_ix, sizeof(double), cudaMemcpyDeviceToHost));
    }
    phase_mark("iterations");
    if (het_) epilogue_het();
    else epilogue_hom();
    phase_mark("extraction + final SLEM");
}

void Solver::epilogue_hom() {
    const long long m = lo_.m, nx = lo_.nx;
    for (int b = 0; b < B_; ++b) {
        const double* pick = (res_[b].converged ? d_.Y : d_.bestY) + (size_t)b * nx;
        TPB_CUDA(cudaMemcpyAsync(tmp_m_ + (size_t)b * m, pick, m * sizeof(double), cudaMemcpyDeviceToDevice, s0_));
    }
    launch_floor_mask(tmp_m_, m, m, cfg_.weight_floor, tmp_m2_, B_, s0_);
    SelectArgs a{};
    a.base = tmp_m2_;
    a.stride = m;
    a.m = m;
    a.r = d_r_;
    a.binary = 0;
    a.list = list_;
    a.list_count = list_count_;
    a.list_cap = list_cap_;
    a.done = nullptr;
    launch_topr(a, B_, s0_);
    TPB_CUDA(cudaMemsetAsync(tmp_m_, 0, (size_t)B_ * m * sizeof(double), s0_));
    launch_extract(lo_.n, m, tmp_m2_, m, list_, list_count_, list_cap_, e_i_[0], e_j_[0], e_w_[0], tmp_m_, worst_,
                   col_idx_[0], B_, s0_);
    std::vector<int> counts(B_);
    TPB_CUDA(cudaMemcpyAsync(counts.data(), list_count_, B_ * sizeof(int), cudaMemcpyDeviceToHost, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
    std::vector<int> ei((size_t)B_ * list_cap_), ej((size_t)B_ * list_cap_);
    std::vector<double> ew((size_t)B_ * list_cap_);
    TPB_CUDA(cudaMemcpy(ei.data(), e_i_[0], ei.size() * sizeof(int), cudaMemcpyDeviceToHost));
    TPB_CUDA(cudaMemcpy(ej.data(), e_j_[0], ej.size() * sizeof(int), cudaMemcpyDeviceToHost));
    TPB_CUDA(cudaMemcpy(ew.data(), e_w_[0], ew.size() * sizeof(double), cudaMemcpyDeviceToHost));
    final_slem(tmp_m_, list_, list_count_, slem_out_);
    std::vector<double> so((size_t)B_ * 8);
    TPB_CUDA(cudaMemcpyAsync(so.data(), slem_out_, so.size() * sizeof(double), cudaMemcpyDeviceToHost, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
    for (int b = 0; b < B_; ++b) {
        SolveResult& R = res_[b];
        const int k = std::min(counts[b], list_cap_);
        R.ei.assign(ei.begin() + (size_t)b * list_cap_, ei.begin() + (size_t)b * list_cap_ + k);
        R.ej.assign(ej.begin() + (size_t)b * list_cap_, ej.begin() + (size_t)b * list_cap_ + k);
        R.w.assign(ew.begin() + (size_t)b * list_cap_, ew.begin() + (size_t)b * list_cap_ + k);
        R.acf = so[(size_t)b * 8 + 0];
        R.lambda2 = so[(size_t)b * 8 + 1];
        R.lambda_n = so[(size_t)b * 8 + 2];
        R.connected = so[(size_t)b * 8 + 3] != 0.0;
    }
}

namespace {

// proj/src/admm_het.cpp:179-227 (sequential greedy; runs once per solve).
bool repair_selection(int n, const std::vector<int>& target, std::vector<char>& sel,
                      const std::vector<double>& w, const std::vector<double>& score, bool* changed) {
    const long long m = (long long)n * (n - 1) / 2;
    std::vector<int> pi(m), pj(m);
    {
        long long l = 0;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j, ++l) {
                pi[l] = i;
                pj[l] = j;
            }
    }
    std::vector<int> deg(n, 0);
    for (long long l = 0; l < m; ++l)
        if (sel[l]) {
            ++deg[pi[l]];
            ++deg[pj[l]];
        }
    *changed = false;
    for (;;) {
        int node = -1;
        for (int i = 0; i < n; ++i)
            if (deg[i] > target[i] && (node < 0 || deg[i] - target[i] > deg[node] - target[node])) node = i;
        if (node < 0) break;
        long long drop = -1;
        for (long long l = 0; l < m; ++l) {
            if (!sel[l] || (pi[l] != node && pj[l] != node)) continue;
            if (drop < 0 || w[l] < w[drop]) drop = l;
        }
        if (drop < 0) return false;
        sel[drop] = 0;
        --deg[pi[drop]];
        --deg[pj[drop]];
        *changed = true;
    }
    for (;;) {
        bool deficit = false;
        for (int i = 0; i < n; ++i) deficit = deficit || deg[i] < target[i];
        if (!deficit) break;
        long long add = -1;
        for (long long l = 0; l < m; ++l) {
            if (sel[l]) continue;
            if (deg[pi[l]] >= target[pi[l]] || deg[pj[l]] >= target[pj[l]]) continue;
            if (add < 0 || score[l] > score[add]) add = l;
        }
        if (add < 0) return false;
        sel[add] = 1;
        ++deg[pi[add]];
        ++deg[pj[add]];
        *changed = true;
    }
    return true;
}

}  // namespace

void Solver::epilogue_het() {
    const int n = lo_.n;
    const long long m = lo_.m, nx = lo_.nx;
    std::vector<double> degd((size_t)B_ * n);
    TPB_CUDA(cudaMemcpy(degd.data(), d_deg_, degd.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<int> lists((size_t)B_ * list_cap_, 0), counts(B_, 0);
    std::vector<double> packed((size_t)B_ * m, 0.0);
    for (int b = 0; b < B_; ++b) {
        SolveResult& R = res_[b];
        const double* pick = (R.converged ? d_.Y : d_.bestY) + (size_t)b * nx;
        std::vector<double> pg(m), pz(m), score(m);
        TPB_CUDA(cudaMemcpy(pg.data(), pick, m * sizeof(double), cudaMemcpyDeviceToHost));
        TPB_CUDA(cudaMemcpy(pz.data(), pick + lo_.off_z, m * sizeof(double), cudaMemcpyDeviceToHost));
        if (R.converged) {
            std::vector<double> xz(m), dz(m);
            TPB_CUDA(cudaMemcpy(xz.data(), d_.X + (size_t)b * nx + lo_.off_z, m * sizeof(double), cudaMemcpyDeviceToHost));
            TPB_CUDA(cudaMemcpy(dz.data(), d_.D + (size_t)b * nx + lo_.off_z, m * sizeof(double), cudaMemcpyDeviceToHost));
            for (long long l = 0; l < m; ++l) score[l] = xz[l] + dz[l] / cfg_.rho;
        } else {
            TPB_CUDA(cudaMemcpy(score.data(), d_.bestScore + (size_t)b * m, m * sizeof(double), cudaMemcpyDeviceToHost));
        }
        // proj/src/admm_het.cpp:315-358
        std::vector<char> sel(m);
        std::vector<double> w(m);
        for (long long l = 0; l < m; ++l) {
            sel[l] = pz[l] > 0.5 ? 1 : 0;
            w[l] = std::max(0.0, pg[l]);
        }
        std::vector<int> target(n);
        for (int i = 0; i < n; ++i) target[i] = (int)degd[(size_t)b * n + i];
        bool changed = false;
        if (!cap_ && !repair_selection(n, target, sel, w, score, &changed)) {
            if (!R.note.empty()) R.note += "; ";
            R.note += "degree repair incomplete";
        }
        if (changed) {
            R.repaired = true;
            if (R.note.find("degree repair incomplete") == std::string::npos) {
                if (!R.note.empty()) R.note += "; ";
                R.note += "degree rows restored by edge swap";
            }
        }
        int count = 0;
        for (long long l = 0; l < m; ++l) count += sel[l];
        if (count == 0) throw Error(kDegenerate, "no edge selected");
        if (count < r_host_[b]) {
            if (!R.note.empty()) R.note += "; ";
            R.note += "capacity limits stopped selection at " + std::to_string(count) + " of " +
                      std::to_string(r_host_[b]) + " edges";
        }
        std::vector<double> node_sum(n, 0.0);
        std::vector<int> pi, pj;
        std::vector<long long> ls;
        {
            long long l = 0;
            for (int i = 0; i < n; ++i)
                for (int j = i + 1; j < n; ++j, ++l)
                    if (sel[l]) {
                        node_sum[i] += w[l];
                        node_sum[j] += w[l];
                        pi.push_back(i);
                        pj.push_back(j);
                        ls.push_back(l);
                    }
        }
        const double worst = *std::max_element(node_sum.begin(), node_sum.end());
        const double scale = worst > 1.0 ? 1.0 / worst : 1.0;
        R.ei = pi;
        R.ej = pj;
        R.w.resize(ls.size());
        for (size_t k = 0; k < ls.size(); ++k) {
            R.w[k] = w[ls[k]] * scale;
            packed[(size_t)b * m + ls[k]] = R.w[k];
            if ((int)k < list_cap_) lists[(size_t)b * list_cap_ + k] = (int)ls[k];
        }
        counts[b] = (int)ls.size();
    }
    h2d(tmp_m_, packed.data(), packed.size() * sizeof(double));
    h2d(list_, lists.data(), lists.size() * sizeof(int));
    h2d(list_count_, counts.data(), counts.size() * sizeof(int));
    final_slem(tmp_m_, list_, list_count_, slem_out_);
    std::vector<double> so((size_t)B_ * 8);
    TPB_CUDA(cudaMemcpyAsync(so.data(), slem_out_, so.size() * sizeof(double), cudaMemcpyDeviceToHost, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
    for (int b = 0; b < B_; ++b) {
        SolveResult& R = res_[b];
        R.acf = so[(size_t)b * 8 + 0];
        R.lambda2 = so[(size_t)b * 8 + 1];
        R.lambda_n = so[(size_t)b * 8 + 2];
        R.connected = so[(size_t)b * 8 + 3] != 0.0;
    }
}

SolveResult Solver::result(int b) const { return res_.at(b); }

void Solver::upload(const double* X, const double* Y, const double* D) {
    const size_t bytes = (size_t)B_ * lo_.nx * sizeof(double);
    if (X) h2d(d_.X, X, bytes);
    if (Y) h2d(d_.Y, Y, bytes);
    if (D) h2d(d_.D, D, bytes);
}

void Solver::download(double* X, double* Y, double* D) {
    TPB_CUDA(cudaStreamSynchronize(s0_));
    const size_t bytes = (size_t)B_ * lo_.nx * sizeof(double);
    if (X) TPB_CUDA(cudaMemcpy(X, d_.X, bytes, cudaMemcpyDeviceToHost));
    if (Y) TPB_CUDA(cudaMemcpy(Y, d_.Y, bytes, cudaMemcpyDeviceToHost));
    if (D) TPB_CUDA(cudaMemcpy(D, d_.D, bytes, cudaMemcpyDeviceToHost));
}

void Solver::project_only() {
    TPB_CUDA(cudaMemsetAsync(d_.ictl, 0, (size_t)B_ * 8 * sizeof(int), s0_));
    launch_prep(d_, c_, s0_);
    enqueue_select(s0_);
    enqueue_projection();
    TPB_CUDA(cudaStreamSynchronize(s0_));
}

void Solver::xstep_only(bool update_duals) {
    TPB_CUDA(cudaMemsetAsync(d_.ictl, 0, (size_t)B_ * 8 * sizeof(int), s0_));
    Dev d = d_;
    d.upd_duals = update_duals ? 1 : 0;
    d.track_best = 0;
    enqueue_xstep(d);
    TPB_CUDA(cudaStreamSynchronize(s0_));
    // keep the CG statistics for cg_stats(); clear the iteration control words
    std::vector<int> keep(B_ * 8, 0);
    TPB_CUDA(cudaMemcpy(keep.data(), d_.ictl, keep.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int b = 0; b < B_; ++b)
        for (int w = 0; w < 8; ++w)
            if (w != kCgIters) keep[b * 8 + w] = 0;
    TPB_CUDA(cudaMemcpyAsync(d_.ictl, keep.data(), keep.size() * sizeof(int), cudaMemcpyHostToDevice, s0_));
    TPB_CUDA(cudaStreamSynchronize(s0_));
}

int Solver::launches_per_iteration() const {
    const int cone = small_ ? 1 : sch_.gemms();
    // prep, top-r, trace SLEM, the cone chain, x-step passes A and B, the
    // best-iterate copy (+ the CG solve)
    return 1 + 1 + 1 + cone + 2 + 1 + (d_.cg ? 1 : 0);
}

int Solver::bench_phase(int phase, int reps) {
    int per = 0;
    for (int k = 0; k < reps; ++k) {
        switch (phase) {
            case 0:
                enqueue_projection();
                per = small_ ? 1 : sch_.gemms();
                break;
            case 1: {
                // as in the iteration (dual update on), without the iteration
                // counter, trace row and stop flags
                Dev d = d_;
                d.track_best = 0;
                d.bookkeep = 0;
                enqueue_xstep(d);
                per = 2 + (d.cg ? 1 : 0);
                break;
            }
            case 7: {
                // pass A (fresh right-hand side h; CG keeps r in h) + the CG
                // solve: subtract phase 5 for the CG alone
                if (!d_.cg) throw Error(kInvalidArgument, "bench_phase 7: linear_solver is not CG");
                launch_xstep_a(d_, c_, s0_);
                launch_xstep_cg(d_, c_, s0_);
                per = 2;
                break;
            }
            case 5:
                launch_xstep_a(d_, c_, s0_);  // scatter/gather pass A alone
                per = 1;
                break;
            case 6: {
                Dev d = d_;                   // pass B alone (dual update on)
                d.track_best = 0;
                d.bookkeep = 0;
                launch_xstep_b(d, c_, s0_);
                per = 1;
                break;
            }
            case 2:
                enqueue_select(s0_);
                per = 1;
                break;
            case 3:
                enqueue_slem_trace(s0_);
                per = 1;
                break;
            case 4:
                launch_prep(d_, c_, s0_);
                per = 1;
                break;
            default:
                throw Error(kInvalidArgument, "bench_phase: unknown phase");
        }
    }
    return per;
}

}  // namespace tpb
