// Read-bandwidth microbenchmark for the scan's data path (diagnostic, not product code):
// cp.async.bulk stages into a shared-memory ring (S slots x B bytes per block, one block
// per SM, stages dealt round-robin or in contiguous runs) versus a plain coalesced
// LDG.128 grid-stride loop.  Prints GB/s per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)),
                 "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
    } while (!done);
}

// S slots of B bytes; all threads consume (sum) each stage; thread 0 refills after a barrier
template <int S>
__global__ void __launch_bounds__(512, 1) tma_kernel(const uint4* __restrict__ src, uint64_t n_stages, uint32_t B,
                                                     int contiguous, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ __align__(8) uint64_t bar[S];
    if (threadIdx.x == 0)
        for (int i = 0; i < S; i++) mbar_init(&bar[i], 1);
    __syncthreads();
    const uint64_t per_block = (n_stages + gridDim.x - 1) / gridDim.x;
    auto stage_of = [&](uint64_t i) -> uint64_t {
        return contiguous ? blockIdx.x * per_block + i : blockIdx.x + i * gridDim.x;
    };
    const uint64_t my_n = contiguous ? (blockIdx.x * per_block < n_stages ? min(per_block, n_stages - blockIdx.x * per_block) : 0)
                                     : (n_stages > blockIdx.x ? (n_stages - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
    if (threadIdx.x == 0)
        for (int i = 0; i < S && i < (int)my_n; i++) {
            expect_tx(&bar[i], B);
            bulk(ring + (size_t)i * B, (const char*)src + stage_of(i) * B, B, &bar[i]);
        }
    unsigned long long acc = 0;
    for (uint64_t k = 0; k < my_n; k++) {
        const int s = (int)(k % S);
        wait(&bar[s], (uint32_t)((k / S) & 1));
        const uint4* p = reinterpret_cast<const uint4*>(ring + (size_t)s * B);
        for (uint32_t i = threadIdx.x; i < B / 16; i += blockDim.x) acc += p[i].x;
        __syncthreads();
        if (threadIdx.x == 0 && k + S < my_n) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            expect_tx(&bar[s], B);
            bulk(ring + (size_t)s * B, (const char*)src + stage_of(k + S) * B, B, &bar[s]);
        }
    }
    if (acc == 0x12345) atomicAdd(sink, acc);
}

__global__ void ldg_kernel(const uint4* __restrict__ src, uint64_t n16, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
        acc += __ldg(&src[i]).x;
    if (acc == 0x12345) atomicAdd(sink, acc);
}

int main() {
    const size_t bytes = 12ull << 30;  // 12 GiB, like the C2 scan
    uint4* d;
    unsigned long long* sink;
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(d, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 2; w++) launch();
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.1f GB/s  (%s)\n", name, 5.0 * bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run("ldg grid-stride 4x148x256", [&] { ldg_kernel<<<4 * sms, 256>>>(d, bytes / 16, sink); });
    run("ldg grid-stride 8x148x256", [&] { ldg_kernel<<<8 * sms, 256>>>(d, bytes / 16, sink); });
    for (int contiguous = 0; contiguous < 2; contiguous++) {
        char nm[96];
        {
            const uint32_t B = 32768;
            cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * B);
            snprintf(nm, sizeof nm, "tma 4 x 32KB %s", contiguous ? "contig" : "round-robin");
            run(nm, [&] { tma_kernel<4><<<sms, 512, 4 * B>>>(d, bytes / B, B, contiguous, sink); });
        }
        {
            const uint32_t B = 32768;
            cudaFuncSetAttribute(tma_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * B);
            snprintf(nm, sizeof nm, "tma 6 x 32KB %s", contiguous ? "contig" : "round-robin");
            run(nm, [&] { tma_kernel<6><<<sms, 512, 6 * B>>>(d, bytes / B, B, contiguous, sink); });
        }
        {
            const uint32_t B = 16384;
            cudaFuncSetAttribute(tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * B);
            snprintf(nm, sizeof nm, "tma 8 x 16KB %s", contiguous ? "contig" : "round-robin");
            run(nm, [&] { tma_kernel<8><<<sms, 512, 8 * B>>>(d, bytes / B, B, contiguous, sink); });
        }
        {
            const uint32_t B = 65536;
            cudaFuncSetAttribute(tma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * B);
            snprintf(nm, sizeof nm, "tma 3 x 64KB %s", contiguous ? "contig" : "round-robin");
            run(nm, [&] { tma_kernel<3><<<sms, 512, 3 * B>>>(d, bytes / B, B, contiguous, sink); });
        }
    }
    return 0;
}
