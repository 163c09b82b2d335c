// Write-pattern check for the line kernel's store stream: grid-stride chunks vs each CTA
// walking its own contiguous region (the line kernel: 444 CTAs x 2 matrices, 22 KB per bulk
// store, one tile in flight per CTA).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/store_pattern tools/store_pattern.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_store(char* __restrict__ A, char* __restrict__ B, size_t bytes_each, int chunk, int contiguous,
                        int both) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < 2 * chunk / 8; i += blockDim.x) sm[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const size_t chunks = bytes_each / chunk;
    const size_t per = (chunks + gridDim.x - 1) / gridDim.x;
    for (size_t m = 0; m < per; ++m) {
        const size_t c = contiguous ? blockIdx.x * per + m : m * gridDim.x + blockIdx.x;
        if (c >= chunks) break;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(A + c * chunk), "r"(s),
                     "r"(chunk)
                     : "memory");
        if (both)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B + c * chunk),
                         "r"(s + chunk), "r"(chunk)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t each = (size_t)8 << 30;
    char *A, *B;
    cudaMalloc(&A, each);
    cudaMalloc(&B, each);
    cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int chunk_kb : {22, 44})
        for (int per_sm : {1, 3})
            for (int contiguous : {0, 1})
                for (int both : {0, 1}) {
                    const int chunk = chunk_kb * 1024 - (chunk_kb == 22 ? 1024 - 448 : 0);   // ~21.9 KB like 8x343x8
                    float best = 1e30f;
                    for (int r = 0; r < 4; ++r) {
                        cudaEventRecord(e0);
                        k_store<<<sms * per_sm, 64, 2 * chunk>>>(A, B, each, chunk, contiguous, both);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (r && ms < best) best = ms;
                    }
                    const double bytes = (double)(each / chunk) * chunk * (both ? 2 : 1);
                    printf("chunk %6d ctas/sm %d %-10s %-6s GB/s %.1f\n", chunk, per_sm,
                           contiguous ? "contig" : "strided", both ? "A+B" : "A", bytes / (best * 1e6));
                }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
