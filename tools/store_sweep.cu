// Bulk-store in-flight sweep: how many bytes must be in flight per SM (CTAs x depth x chunk)
// for cp.async.bulk shared->global stores to reach the write-only HBM peak.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/store_sweep tools/store_sweep.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_store_bulk(char* __restrict__ out, size_t chunks, int chunk, int depth) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < chunk / 8; i += blockDim.x) sm[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * chunk), "r"(s),
                     "r"(chunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (++inflight >= depth) {
            if (depth == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else if (depth == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)8 << 30;
    char* buf;
    cudaMalloc(&buf, bytes);
    cudaFuncSetAttribute(k_store_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int chunks_kb[] = {8, 16, 22, 32, 44, 64, 88};
    for (int ck : chunks_kb)
        for (int per : {1, 2, 3, 4})
            for (int depth : {1, 2, 4}) {
                const int chunk = ck * 1024;
                if ((size_t)per * chunk > 220 * 1024) continue;
                const size_t n = bytes / chunk;
                float best = 1e30f;
                for (int r = 0; r < 4; ++r) {
                    cudaEventRecord(a);
                    k_store_bulk<<<sms * per, 64, chunk>>>(buf, n, chunk, depth);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (r && ms < best) best = ms;
                }
                printf("chunk_kb %3d ctas_per_sm %d depth %d inflight_kb_per_sm %4d  GB/s %.1f\n", ck, per, depth,
                       ck * per * depth, n * (double)chunk / (best * 1e6));
            }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
