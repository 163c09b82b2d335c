// Write-only HBM ceiling probe: which store flavour writes fastest on this B200?
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/write_probe tools/write_probe.cu
// Prints GB/s (best of 5) for each variant over an 8 GiB buffer (and cudaMemsetAsync for reference).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int MODE>
__global__ void k_st(double* __restrict__ out, size_t n, double v) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint64_t pol = pol_first();
    if (MODE == 0) {   // st.global.v2.f64
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += stride)
            asm volatile("st.global.v2.f64 [%0], {%1, %1};" ::"l"(out + 2 * i), "d"(v) : "memory");
    } else if (MODE == 1) {   // st.global.v4.f64 (256-bit)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride)
            asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(out + 4 * i), "d"(v) : "memory");
    } else if (MODE == 2) {   // v2 + L1::no_allocate + L2 evict_first
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += stride)
            asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %1}, %2;" ::"l"(out + 2 * i),
                         "d"(v), "l"(pol)
                         : "memory");
    } else if (MODE == 3) {   // v4 + L2 evict_first
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride)
            asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1, %1, %1, %1}, %2;" ::"l"(out + 4 * i),
                         "d"(v), "l"(pol)
                         : "memory");
    } else if (MODE == 4) {   // st.global.cs.v2 (streaming)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += stride)
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %1};" ::"l"(out + 2 * i), "d"(v) : "memory");
    }
}

// cp.async.bulk smem -> global, chunk bytes per op, `depth` ops in flight per CTA, optional L2 hint
template <bool HINT>
__global__ void k_bulk(char* __restrict__ out, size_t chunks, int chunk, int depth) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < chunk / 8; i += blockDim.x) sm[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t pol = pol_first();
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
        if (HINT)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                             out + c * chunk),
                         "r"(s), "r"(chunk), "l"(pol)
                         : "memory");
        else
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

// the same, but CTA b writes its own contiguous range of chunks (b*per .. (b+1)*per-1), like the
// line kernel whose CTAs own whole lines, instead of a grid-stride front sweeping the buffer
__global__ void k_bulk_blocked(char* __restrict__ out, size_t chunks, int chunk) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < chunk / 8; i += blockDim.x) sm[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t pol = pol_first();
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const size_t per = (chunks + gridDim.x - 1) / gridDim.x;
    const size_t c0 = blockIdx.x * per, c1 = c0 + per < chunks ? c0 + per : chunks;
    for (size_t c = c0; c < c1; ++c) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(out + c * chunk),
                     "r"(s), "r"(chunk), "l"(pol)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)8 << 30, n = bytes / 8;
    double* buf;
    cudaMalloc(&buf, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto&& launch) {
        float best = 1e30f;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r && ms < best) best = ms;
        }
        return bytes / (best * 1e6);
    };
    printf("memset 0x00        GB/s %.1f\n", timeit([&] { cudaMemsetAsync(buf, 0, bytes); }));
    printf("memset 0x5a        GB/s %.1f\n", timeit([&] { cudaMemsetAsync(buf, 0x5a, bytes); }));
    for (double v : {0.0, 1.0, 1.2345678901234567}) {
        for (int bps : {4, 8})
            printf("st.v4 value %-20.17g blocks/SM %d GB/s %.1f\n", v, bps,
                   timeit([&] { k_st<1><<<sms * bps, 256>>>(buf, n, v); }));
    }
    const char* names[] = {"st.v2", "st.v4", "st.v2.noalloc.evfirst", "st.v4.noalloc.evfirst", "st.cs.v2"};
    for (int blocksPerSm : {4, 8, 16, 32})
        for (int threads : {256, 512}) {
            const int grid = sms * blocksPerSm;
            if (blocksPerSm * threads > 2048) continue;
            double r[5];
            r[0] = timeit([&] { k_st<0><<<grid, threads>>>(buf, n, 1.0); });
            r[1] = timeit([&] { k_st<1><<<grid, threads>>>(buf, n, 1.0); });
            r[2] = timeit([&] { k_st<2><<<grid, threads>>>(buf, n, 1.0); });
            r[3] = timeit([&] { k_st<3><<<grid, threads>>>(buf, n, 1.0); });
            r[4] = timeit([&] { k_st<4><<<grid, threads>>>(buf, n, 1.0); });
            for (int m = 0; m < 5; ++m) printf("%-22s blocks/SM %2d threads %3d GB/s %.1f\n", names[m], blocksPerSm, threads, r[m]);
        }
    cudaFuncSetAttribute(k_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ck : {16, 32, 44, 64})
        for (int per : {2, 3, 4})
            for (int depth : {2, 4}) {
                const int chunk = ck * 1024;
                if ((size_t)per * chunk > 200 * 1024) continue;
                const size_t nch = bytes / chunk;
                const double g0 = timeit([&] { k_bulk<false><<<sms * per, 64, chunk>>>((char*)buf, nch, chunk, depth); });
                const double g1 = timeit([&] { k_bulk<true><<<sms * per, 64, chunk>>>((char*)buf, nch, chunk, depth); });
                printf("bulk chunk_kb %2d ctas/SM %d depth %d  GB/s %.1f  (evict_first %.1f)\n", ck, per, depth, g0, g1);
            }
    // the line kernel's pattern: per tile one chunk into each of two regions (M, K), 2 or 3 CTAs/SM,
    // and large single chunks at 1 CTA/SM
    for (int ck : {22, 33, 44, 66, 96, 128, 192})
        for (int per : {1, 2, 3})
            for (int depth : {1, 2}) {
                const int chunk = ck * 1024;
                if ((size_t)per * chunk > 200 * 1024 || (per == 1 && ck < 66)) continue;
                const size_t nch = bytes / chunk;
                const double g1 = timeit([&] { k_bulk<true><<<sms * per, 64, chunk>>>((char*)buf, nch, chunk, depth); });
                printf("bulk-ef chunk_kb %3d ctas/SM %d depth %d  GB/s %.1f\n", ck, per, depth, g1);
            }
    cudaFuncSetAttribute(k_bulk_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ck : {22, 33, 44, 66})
        for (int per : {2, 3}) {
            const int chunk = ck * 1024;
            if ((size_t)per * chunk > 200 * 1024) continue;
            const size_t nch = bytes / chunk;
            const double g = timeit([&] { k_bulk_blocked<<<sms * per, 64, chunk>>>((char*)buf, nch, chunk); });
            printf("bulk-blocked chunk_kb %3d ctas/SM %d  GB/s %.1f\n", ck, per, g);
        }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
