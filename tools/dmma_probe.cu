// DMMA (mma.sync m8n8k4 f64) latency and throughput vs parallelism on one B200 (sm_100a).
// How many independent DMMAs must be in flight per SM sub-partition to reach the FP64 tensor
// peak?  (The C3 interior kernel runs 16 warps per SM with 3-6 independent DMMA chains each.)
// Prints one JSON line: latency_cycles (one warp, one dependent chain) and, for W warps per SM
// and C independent accumulator chains per warp, the achieved TF/s.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/dmma_probe tools/dmma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int C>
__global__ void k_chains(double* out, long long* cyc, int iters, double a, double b) {
    double d0[C], d1[C];
#pragma unroll
    for (int j = 0; j < C; ++j) d0[j] = d1[j] = j * 1e-3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < C; ++j) dmma(d0[j], d1[j], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) s += d0[j] + d1[j];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

// C DMMA chains interleaved with X independent integer ops per lane (4 chains of IMADs):
// does the sub-partition issue other instructions while its DMMAs occupy the tensor pipe?
template <int C, int X>
__global__ void k_mixed(double* out, int* iout, int iters, double a, double b, int m) {
    double d0[C], d1[C];
    int q[4] = {(int)threadIdx.x, (int)threadIdx.x + 1, (int)threadIdx.x + 2, (int)threadIdx.x + 3};
#pragma unroll
    for (int j = 0; j < C; ++j) d0[j] = d1[j] = j * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < C; ++j) dmma(d0[j], d1[j], a, b);
#pragma unroll
        for (int x = 0; x < X; ++x) q[x & 3] = q[x & 3] * m + 7;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) s += d0[j] + d1[j];
    if (s == 12345.678) out[0] = s;
    if (q[0] + q[1] + q[2] + q[3] == 12345) iout[0] = 1;
}

template <int C, int X>
float mixed_ms(int sms, int warps_per_sm, int iters, double* out, int* iout) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_mixed<C, X><<<sms, 32 * warps_per_sm>>>(out, iout, iters, 0.999999, 1e-7, 3);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        k_mixed<C, X><<<sms, 32 * warps_per_sm>>>(out, iout, iters, 0.999999, 1e-7, 3);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    return best;
}

template <int C>
double tflops(int sms, int warps_per_sm, int iters, double* out, long long* cyc) {
    // one block of warps_per_sm warps per SM
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_chains<C><<<sms, 32 * warps_per_sm>>>(out, cyc, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        k_chains<C><<<sms, 32 * warps_per_sm>>>(out, cyc, iters, 0.999999, 1e-7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    const double fmas = (double)sms * warps_per_sm * iters * C * 256.0;
    return 2.0 * fmas / (best * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    long long* cyc;
    CK(cudaMalloc(&out, 8));
    CK(cudaMalloc(&cyc, 8));
    const int iters = 4096;
    // latency: one warp, one chain
    k_chains<1><<<1, 32>>>(out, cyc, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    long long c = 0;
    k_chains<1><<<1, 32>>>(out, cyc, iters, 0.999999, 1e-7);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("{\"latency_cycles\": %.1f", (double)c / iters);
    const int W[] = {4, 8, 16, 32};
    for (int w : W) {
        printf(", \"w%d_c1\": %.2f", w, tflops<1>(sms, w, iters, out, cyc));
        printf(", \"w%d_c2\": %.2f", w, tflops<2>(sms, w, iters, out, cyc));
        printf(", \"w%d_c3\": %.2f", w, tflops<3>(sms, w, iters, out, cyc));
        printf(", \"w%d_c4\": %.2f", w, tflops<4>(sms, w, iters, out, cyc));
        printf(", \"w%d_c6\": %.2f", w, tflops<6>(sms, w, iters, out, cyc));
    }
    // 16 warps / SM, 4 DMMA chains, with 0 / 16 / 32 / 64 integer ops per 4 DMMAs
    int* iout;
    CK(cudaMalloc(&iout, 4));
    const float m0 = mixed_ms<4, 0>(sms, 16, iters, out, iout);
    const float m16 = mixed_ms<4, 16>(sms, 16, iters, out, iout);
    const float m32 = mixed_ms<4, 32>(sms, 16, iters, out, iout);
    const float m64 = mixed_ms<4, 64>(sms, 16, iters, out, iout);
    const float i64 = mixed_ms<0 + 1, 64>(sms, 16, iters, out, iout);
    printf(", \"mix16w_4dmma_ms\": %.3f, \"plus16int_ms\": %.3f, \"plus32int_ms\": %.3f, \"plus64int_ms\": %.3f, "
           "\"1dmma_64int_ms\": %.3f", m0, m16, m32, m64, i64);
    printf("}\n");
    return 0;
}
