// Microbenchmark: HBM write throughput of 32 B records under the eval kernel's store
// pattern (each lane owns a contiguous row of `row` records) vs fully coalesced stores.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void st256(void* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__global__ void rows(uint64_t* out, uint64_t nrows, uint32_t row) {
    for (uint64_t H = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; H < nrows; H += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t* p = out + H * row * 4;
        for (uint32_t j = 0; j < row; j++) st256(p + 4 * j, H, j, H ^ j, 7);
    }
}
__global__ void coal(uint64_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        st256(out + 4 * i, i, 1, 2, 3);
}
int main() {
    const uint64_t n = 429981696ull; const uint32_t row = 144;
    uint64_t* d; cudaMalloc(&d, n * 32);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8, 16}) {
        for (int it = 0; it < 3; it++) {
            cudaEventRecord(a); rows<<<sms * occ, 128>>>(d, n / row, row); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it == 2) printf("rows(row=%u) grid=%d x128: %.3f ms  %.1f GB/s\n", row, sms * occ, ms, n * 32 / ms / 1e6);
        }
    }
    for (int it = 0; it < 3; it++) {
        cudaEventRecord(a); coal<<<sms * 8, 256>>>(d, n); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it == 2) printf("coalesced: %.3f ms  %.1f GB/s\n", ms, n * 32 / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
