// Peak microbenchmarks for the roofline denominators (SURVEY §8(d) "Peak microbenchmarks"):
//   (i)   write-only HBM: grid-stride 16-byte st.global and cp.async.bulk shared->global
//         store loops over an 8 GiB buffer, best of 10;
//   (ii)  copy (read + write bytes), the same definition as MEASURED_PEAKS.json hbm_gbs;
//   (iii) FP64: independent DFMA chains at full occupancy.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peaks tools/peaks.cu
// Prints one JSON line.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__global__ void k_store_v2(double2* __restrict__ out, size_t n2, double v) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
        out[i] = make_double2(v, v);
}

__global__ void k_copy_v2(const double2* __restrict__ in, double2* __restrict__ out, size_t n2) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) out[i] = in[i];
}

// each CTA fills CHUNK bytes of shared memory once, then issues bulk stores of it over its
// share of the buffer, keeping up to DEPTH groups in flight
template <int CHUNK>
__global__ void k_store_bulk(char* __restrict__ out, size_t chunks, double v) {
    extern __shared__ __align__(128) double sm[];
    for (int i = threadIdx.x; i < CHUNK / 8; i += blockDim.x) sm[i] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CHUNK), "r"(s),
                     "r"(CHUNK)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (++inflight >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;
}

template <class F>
float best_ms(F f, int reps = 10) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = (size_t)8 << 30;
    char *buf, *src;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&src, bytes / 2));
    const size_t n2 = bytes / 16;
    float st = best_ms([&] { k_store_v2<<<sms * 8, 256>>>((double2*)buf, n2, 1.0); });
    float cp = best_ms([&] { k_copy_v2<<<sms * 8, 256>>>((const double2*)src, (double2*)buf, n2 / 2); });
    constexpr int CH = 32768;
    CK(cudaFuncSetAttribute(k_store_bulk<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH));
    float bk = best_ms([&] { k_store_bulk<CH><<<sms * 4, 128, CH>>>(buf, bytes / CH, 1.0); });
    const int iters = 1 << 16;
    float fm = best_ms([&] { k_dfma<<<sms * 8, 256>>>((double*)buf, iters, 0.999999, 1e-7); }, 3);
    const double dfma_flops = 2.0 * 8 * iters * (double)sms * 8 * 256;
    printf("{\"sms\": %d, \"write_v2_gbs\": %.1f, \"write_bulk_gbs\": %.1f, \"copy_gbs\": %.1f, \"fp64_tflops\": %.2f, "
           "\"bytes\": %zu}\n",
           sms, bytes / (st * 1e6), bytes / (bk * 1e6), 2.0 * (bytes / 2) / (cp * 1e6), dfma_flops / (fm * 1e9), bytes);
    return 0;
}
