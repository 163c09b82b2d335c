// Write-pattern probe for the C5 store stream (round 2): bulk stores (cp.async.bulk from shared
// memory) of CH-byte tiles into two arrays (M and K), comparing
//   lines : CTA b owns "lines" b, b + G, ... of T tiles each and writes them in order (the line
//           kernel's pattern: G write fronts LB bytes apart),
//   tiles : CTA b writes tiles b, b + G, ... of the flattened (line, tile) order (G consecutive
//           tiles in flight: one compact write front),
//   oneshot: one CTA per tile.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/write_probe3 tools/write_probe3.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk(char* dst, uint32_t s, int bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst), "r"(s),
                 "r"(bytes), "l"(pol)
                 : "memory");
}

__device__ unsigned long long g_ticket;
// MODE 0: lines, 1: tiles (grid-stride over flattened tiles), 2: oneshot, 3: tiles with
// write-completion waits (wait_group, not .read), 4: tiles fetched from a global ticket counter
template <int MODE>
__global__ void k_pat(char* A, char* B, long long tiles_total, int T, int CH, int depth) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < CH / 8; i += blockDim.x) sm[i] = 1.0 + i * 1e-3 + blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t pol = pol_first();
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    auto one = [&](long long tile) {
        bulk(A + tile * CH, s, CH, pol);
        bulk(B + tile * CH, s, CH, pol);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (++inflight >= depth) {
            if (MODE == 3) asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
    };
    if (MODE == 0) {
        const long long lines = tiles_total / T;
        for (long long l = blockIdx.x; l < lines; l += gridDim.x)
            for (int t = 0; t < T; ++t) one(l * T + t);
    } else if (MODE == 1 || MODE == 3) {
        for (long long c = blockIdx.x; c < tiles_total; c += gridDim.x) one(c);
    } else if (MODE == 4) {
        for (;;) {
            const long long c = (long long)atomicAdd(&g_ticket, 1ull);
            if (c >= tiles_total) break;
            one(c);
        }
    } else if (MODE == 5) {                 // ticket per group of `depth`... per line of T tiles
        const long long lines = tiles_total / T;
        for (;;) {
            const long long l = (long long)atomicAdd(&g_ticket, 1ull);
            if (l >= lines) break;
            for (int t = 0; t < T; ++t) one(l * T + t);
        }
    } else {
        one(blockIdx.x);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float best_ms(F f, int reps = 7) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t each = (size_t)6 << 30;   // per array
    char *A, *B;
    if (cudaMalloc(&A, each) != cudaSuccess || cudaMalloc(&B, each) != cudaSuccess) return 1;
    const int CH = 32928, T = 22;
    const long long tiles = (long long)(each / CH) / T * T;
    const double bytes = 2.0 * tiles * CH;
    for (auto f : {&k_pat<0>, &k_pat<1>, &k_pat<2>, &k_pat<3>, &k_pat<4>, &k_pat<5>})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const unsigned long long zero = 0;
    for (int Tl : {22, 11, 4, 2}) {                    // tiles per ticket (a line = 22 tiles of 12 rows)
        const long long tl = tiles / Tl * Tl;
        for (int per : {2, 3}) {
            const int G = sms * per;
            float k = best_ms([&] {
                cudaMemcpyToSymbolAsync(g_ticket, &zero, sizeof(zero));
                k_pat<5><<<G, 32, CH>>>(A, B, tl, Tl, CH, 2);
            });
            printf("ticket per %2d consecutive tiles, %d CTAs/SM: %.0f GB/s\n", Tl, per, 2.0 * tl * CH / (k * 1e6));
        }
    }
    return 0;
}
