// FP64 pipe microbenchmark (B200, sm_100a): is DMMA (mma.sync m8n8k4 f64) a pipe of its own
// next to DFMA, and at what rate?  Prints one JSON line:
//   dfma_tflops        independent DFMA chains, full occupancy
//   dmma_tflops        independent DMMA chains (256 FMA per warp instruction), full occupancy
//   mixed_*            each warp interleaves R DFMA per lane with one DMMA; reports the time
//                      relative to the two kernels run separately (1.0 = fully overlapped)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/fp64_pipes tools/fp64_pipes.cu
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

// F DFMA chains of depth 1 per iteration, C independent DMMA accumulators per iteration
template <int F, int C>
__global__ void k_mix(double* out, int iters, double a, double b) {
    double x[F > 0 ? F : 1];
    double d0[C > 0 ? C : 1], d1[C > 0 ? C : 1];
#pragma unroll
    for (int j = 0; j < (F > 0 ? F : 1); ++j) x[j] = threadIdx.x * 1e-9 + j;
#pragma unroll
    for (int j = 0; j < (C > 0 ? C : 1); ++j) d0[j] = d1[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < F; ++j) x[j] = fma(x[j], a, b);
#pragma unroll
        for (int j = 0; j < C; ++j) dmma(d0[j], d1[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < (F > 0 ? F : 1); ++j) s += x[j];
#pragma unroll
    for (int j = 0; j < (C > 0 ? C : 1); ++j) s += d0[j] + d1[j];
    if (s == 12345.678) out[0] = s;
}

template <int F, int C>
double run(int blocks, int iters, double* out, float* ms_out) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_mix<F, C><<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        k_mix<F, C><<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    *ms_out = best;
    const double fmas = (double)blocks * 256 * iters * F + (double)blocks * 8 * iters * C * 256.0;
    return 2.0 * fmas / (best * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 8));
    const int blocks = sms * 8, iters = 4096;
    float t_f, t_c, t_m1, t_m2, t_m3;
    const double tf = run<8, 0>(blocks, iters, out, &t_f);
    const double tc = run<0, 4>(blocks, iters, out, &t_c);
    // mixed: 8 DFMA per lane (8 warp instr) + 4 DMMA per iteration -- same work as the two above
    const double tm = run<8, 4>(blocks, iters, out, &t_m1);
    const double tm2 = run<16, 4>(blocks, iters, out, &t_m2);
    const double tm3 = run<4, 4>(blocks, iters, out, &t_m3);
    printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f, "
           "\"mixed_8f4c_tflops\": %.2f, \"mixed_8f4c_ms\": %.3f, \"mixed_over_sum\": %.3f, "
           "\"mixed_16f4c_tflops\": %.2f, \"mixed_4f4c_tflops\": %.2f}\n",
           tf, tc, t_f, t_c, tm, t_m1, t_m1 / (t_f + t_c), tm2, tm3);
    return 0;
}
