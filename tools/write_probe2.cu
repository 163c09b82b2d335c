// Write-only HBM probe, round 2: one-shot grids (one small chunk per thread, the grid covers the
// buffer, like a library elementwise fill) vs grid-stride loops, constant vs position-dependent
// values.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/write_probe2 tools/write_probe2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

// one-shot: thread t writes VEC double2 at [t * VEC, t * VEC + VEC) (block-contiguous)
template <int VEC, bool VAR>
__global__ void k_oneshot(double2* __restrict__ out, size_t n2, double v) {
    const size_t base = ((size_t)blockIdx.x * blockDim.x) * VEC + threadIdx.x;
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
        const size_t i = base + (size_t)k * blockDim.x;
        if (i < n2) out[i] = VAR ? make_double2(v * (double)i, v + (double)i) : make_double2(v, v);
    }
}

template <bool VAR>
__global__ void k_stride(double2* __restrict__ out, size_t n2, double v) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
        out[i] = VAR ? make_double2(v * (double)i, v + (double)i) : make_double2(v, v);
}

template <class F>
float best_ms(F f, int reps = 10) {
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
    const size_t bytes = (size_t)12 << 30;
    char* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    const size_t n2 = bytes / 16;
    auto gbs = [&](float ms) { return bytes / (ms * 1e6); };
    printf("memset            %.0f GB/s\n", gbs(best_ms([&] { cudaMemsetAsync(buf, 0x3f, bytes); })));
    printf("oneshot v1 const  %.0f\n", gbs(best_ms([&] { k_oneshot<1, false><<<(n2 + 127) / 128, 128>>>((double2*)buf, n2, 1.0); })));
    printf("oneshot v2 const  %.0f\n", gbs(best_ms([&] { k_oneshot<2, false><<<(n2 + 255) / 256, 128>>>((double2*)buf, n2, 1.0); })));
    printf("oneshot v2 var    %.0f\n", gbs(best_ms([&] { k_oneshot<2, true><<<(n2 + 255) / 256, 128>>>((double2*)buf, n2, 1.0); })));
    printf("oneshot v4 var    %.0f\n", gbs(best_ms([&] { k_oneshot<4, true><<<(n2 + 511) / 512, 128>>>((double2*)buf, n2, 1.0); })));
    printf("oneshot v8 var    %.0f\n", gbs(best_ms([&] { k_oneshot<8, true><<<(n2 + 2047) / 2048, 256>>>((double2*)buf, n2, 1.0); })));
    for (int per : {4, 8, 16, 32})
        printf("stride x%-2d var    %.0f\n", per,
               gbs(best_ms([&] { k_stride<true><<<sms * per, 256>>>((double2*)buf, n2, 1.0); })));
    printf("stride x8 const   %.0f\n", gbs(best_ms([&] { k_stride<false><<<sms * 8, 256>>>((double2*)buf, n2, 1.0); })));
    return 0;
}
