// tcgen05.mma kind::i8 issue/throughput microbenchmark (sm_100a).
// One CTA per SM, one thread issues R MMAs (M=128, N=NN, K=32, SS operands
// in SWIZZLE_64B smem) cycling over NACC accumulators and NOP distinct A/B
// tiles; reports cycles per MMA and int8 TOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imma imma_rate.cu && /tmp/imma
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw64_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int NN, int NACC, int NOP>
__global__ void __launch_bounds__(128, 1) bench(int R, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t base = (su32(sm) + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | (8u << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int it = 0; it < R; it += NACC * NOP) {
#pragma unroll
            for (int o = 0; o < NOP; ++o)
#pragma unroll
                for (int a = 0; a < NACC; ++a) {
                    const uint64_t ad = sw64_desc(base + o * 8192);
                    const uint64_t bd = sw64_desc(base + 65536 + o * 4096);
                    mma_i8(tmem + a * NN, ad, bd, idesc, it > 0);
                }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        uint32_t ok = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(su32(&bar)));
        } while (!ok);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int NN, int NACC, int NOP>
void run(int sms) {
    const int R = 4096;
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    auto k = bench<NN, NACC, NOP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<<<sms, 128, 100 * 1024>>>(R, d);
    k<<<sms, 128, 100 * 1024>>>(R, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, 100 * 1024>>>(R, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[256];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    const double ops = 2.0 * 128 * NN * 32 * (double)R * sms;
    printf("N=%3d acc=%d tiles=%d ctas=%3d: %6.1f cycles/MMA (floor %d)  %7.1f TOP/s  err=%s\n", NN, NACC, NOP, sms,
           avg / R, 128 * NN / 256, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<64, 1, 1>(1);
    run<64, 8, 1>(1);
    run<64, 8, 8>(1);
    run<64, 8, 8>(148);
    run<128, 4, 1>(1);
    run<128, 4, 4>(148);
    run<256, 2, 1>(1);
    run<256, 2, 2>(148);
    run<32, 8, 8>(148);
    return 0;
}
