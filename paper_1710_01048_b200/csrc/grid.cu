// Device generation of the seeded, smoothed lognormal vertex field used as the C5
// coefficient: white noise g0 from splitmix64 keys of the
// extended vertex (a,b,c) in [-4, n+4]^d, three separable "valid" binomial-8 passes,
// normalisation to unit variance, c = exp(sigma * g).  Each rank generates only its slab
// (plus the 4-plane filter margin) from global keys, so slabs agree with a global field.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace wgq {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double unit53(uint64_t z) { return (double)(z >> 11) * 0x1.0p-53; }

// key = ((c+4) ext_y + (b+4)) ext_x + (a+4), ext = n + 9 per direction (c.4 for equal counts)
__device__ __forceinline__ double white(uint64_t seed, int64_t nx, int64_t ny, int64_t a, int64_t b, int64_t c) {
    const uint64_t key = (uint64_t)(((c + 4) * (ny + 9) + (b + 4)) * (nx + 9) + (a + 4));
    const double u1 = unit53(mix64(seed ^ (2ull * key)));
    const double u2 = unit53(mix64(seed ^ (2ull * key + 1ull)));
    return sqrt(-2.0 * log(1.0 - u1)) * cospi(2.0 * u2);
}

__constant__ double kBinom[9] = {1.0 / 256, 8.0 / 256, 28.0 / 256, 56.0 / 256, 70.0 / 256,
                                 56.0 / 256, 28.0 / 256, 8.0 / 256, 1.0 / 256};

// pass 1: x-filtered white noise on [0,nx] x ext(b) x ext(c)
__global__ void k_pass_x(uint64_t seed, int64_t n, int64_t ny, int dim, int64_t c0, int64_t nb, int64_t nc, double* out) {
    const int64_t nv = n + 1;
    const int64_t total = nv * nb * nc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t % nv;
        const int64_t bi = (t / nv) % nb;
        const int64_t ci = t / (nv * nb);
        int64_t b, c;
        if (dim == 3) {
            b = bi - 4;
            c = c0 - 4 + ci;
        } else if (dim == 2) {
            b = c0 - 4 + bi;
            c = 0;
        } else {
            b = 0;
            c = 0;
        }
        double s = 0.0;
        for (int q = 0; q < 9; ++q) s += kBinom[q] * white(seed, n, ny, a - 4 + q, b, c);
        out[t] = s;
    }
}

// generic "valid" 9-tap pass along an axis of a [nc][nb][na] array: in has L+8 along the axis
__global__ void k_pass_axis(const double* in, double* out, int64_t na, int64_t nb, int64_t nc, int axis, int64_t in_na,
                            int64_t in_nb) {
    const int64_t total = na * nb * nc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t % na, b = (t / na) % nb, c = t / (na * nb);
        double s = 0.0;
        for (int q = 0; q < 9; ++q) {
            int64_t aa = a, bb = b, cc = c;
            if (axis == 1) bb += q;
            else cc += q;
            s += kBinom[q] * in[(cc * in_nb + bb) * in_na + aa];
        }
        out[t] = s;
    }
}

__global__ void k_finish(double* g, int64_t count, double scale) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
        g[t] = exp(scale * g[t]);
}

}  // namespace

int launch_generate_grid(const int64_t* ns, int dim, uint64_t seed, double sigma, int64_t plane0, int64_t planes,
                         double* grid, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = ns[0], ny = dim >= 2 ? ns[1] : ns[0];       // x count, key stride of y
    const int64_t nv = n + 1, nvy = ny + 1;
    const double norm = std::sqrt(std::pow(12870.0 / 65536.0, dim));   // std of the filtered noise
    const double scale = sigma / norm;
    const int threads = 256;
    auto blocks = [](int64_t total) { return (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64); };
    if (dim == 1) {
        k_pass_x<<<blocks(nv), threads, 0, st>>>(seed, n, ny, 1, 0, 1, 1, grid);
        k_finish<<<blocks(nv), threads, 0, st>>>(grid, nv, scale);
        return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
    }
    double *A = nullptr, *B = nullptr;
    if (dim == 2) {
        const int64_t nb = planes + 8;
        if (cudaMallocAsync((void**)&A, nv * nb * sizeof(double), st) != cudaSuccess) return WGQ_ECUDA;
        k_pass_x<<<blocks(nv * nb), threads, 0, st>>>(seed, n, ny, 2, plane0, nb, 1, A);
        k_pass_axis<<<blocks(nv * planes), threads, 0, st>>>(A, grid, nv, planes, 1, 1, nv, nb);
        k_finish<<<blocks(nv * planes), threads, 0, st>>>(grid, nv * planes, scale);
        cudaFreeAsync(A, st);
        return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
    }
    const int64_t nb = nvy + 8, nc = planes + 8;
    if (cudaMallocAsync((void**)&A, nv * nb * nc * sizeof(double), st) != cudaSuccess) return WGQ_ECUDA;
    if (cudaMallocAsync((void**)&B, nv * nvy * nc * sizeof(double), st) != cudaSuccess) {
        cudaFreeAsync(A, st);
        return WGQ_ECUDA;
    }
    k_pass_x<<<blocks(nv * nb * nc), threads, 0, st>>>(seed, n, ny, 3, plane0, nb, nc, A);
    k_pass_axis<<<blocks(nv * nvy * nc), threads, 0, st>>>(A, B, nv, nvy, nc, 1, nv, nb);
    k_pass_axis<<<blocks(nv * nvy * planes), threads, 0, st>>>(B, grid, nv, nvy, planes, 2, nv, nvy);
    k_finish<<<blocks(nv * nvy * planes), threads, 0, st>>>(grid, nv * nvy * planes, scale);
    cudaFreeAsync(A, st);
    cudaFreeAsync(B, st);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

}  // namespace wgq
