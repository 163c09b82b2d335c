// CSR structure (closed-form row pointers), full-coverage row moments and checksums.
// Not part of the timed hot path; used to build CSR outputs and to check results at
// sizes no host copy can hold.
#include <cuda_runtime.h>

#include "internal.h"

namespace wgq {
namespace {

// number of columns of 1D row r: a(r) = min(r+p, N-1) - max(r-p, 0) + 1
__device__ __host__ __forceinline__ int64_t cols_1d(int64_t r, int p, int64_t N) {
    int64_t hi = r + p < N - 1 ? r + p : N - 1;
    int64_t lo = r - p > 0 ? r - p : 0;
    return hi - lo + 1;
}

// A(r) = sum_{r' < r} a(r') in closed form (no scan):
//   r(2p+1) - [q p - q(q-1)/2]_{q = min(r,p)} - u(u+1)/2, u = max(0, r - N + p)
__device__ __host__ __forceinline__ int64_t prefix_1d(int64_t r, int p, int64_t N) {
    int64_t q = r < p ? r : p;
    int64_t u = r - N + p;
    u = u > 0 ? u : 0;
    return r * (2 * p + 1) - (q * p - q * (q - 1) / 2) - u * (u + 1) / 2;
}

// global number of nonzeros before row i (lexicographic, x fastest); per-direction sizes
__device__ __host__ __forceinline__ int64_t nnz_before(int64_t row, int p, const Dims& D) {
    const int dim = D.dim;
    int64_t idx[3] = {0, 0, 0};
    int64_t rem = row;
    for (int q = 0; q < dim - 1; ++q) {
        idx[q] = rem % D.N[q];
        rem /= D.N[q];
    }
    idx[dim - 1] = rem;                  // may equal N_d for row == rows (end of the matrix)
    int64_t width = 1;
    // rows are ordered by (i_d, ..., i_1): accumulate from the slowest direction
    int64_t acc = 0;
    for (int q = dim - 1; q >= 0; --q) {
        int64_t Sp = 1;
        for (int k = 0; k < q; ++k) Sp *= prefix_1d(D.N[k], p, D.N[k]);
        acc += width * prefix_1d(idx[q], p, D.N[q]) * Sp;
        width *= cols_1d(idx[q], p, D.N[q]);
    }
    return acc;
}

__global__ void k_row_ptr(int p, const Dims D, int64_t row_begin, int64_t rows, int64_t* row_ptr) {
    const int64_t base = nnz_before(row_begin, p, D);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= rows; t += (int64_t)gridDim.x * blockDim.x)
        row_ptr[t] = nnz_before(row_begin + t, p, D) - base;
}

__global__ void k_col_idx(int p, const Dims D, int64_t row_begin, int64_t rows, const int64_t* row_ptr,
                          int32_t* col_idx) {
    const int dim = D.dim;
    const int S = 2 * p + 1;
    int NS = 1;
    for (int q = 0; q < dim; ++q) NS *= S;
    const int64_t total = rows * NS;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t orow = t / NS;
        const int slot = (int)(t % NS);
        int64_t rem = row_begin + orow;
        int64_t pos = 0, stride = 1, col = 0, cstride = 1;
        bool ok = true;
        int s = slot;
        for (int q = 0; q < dim; ++q) {
            const int64_t N = D.N[q];
            const int64_t i = rem % N;
            rem /= N;
            const int o = s % S - p;
            s /= S;
            const int64_t lo = i - p < 0 ? -i : -p;
            const int64_t hi = i + p > N - 1 ? N - 1 - i : p;
            if (o < lo || o > hi) ok = false;
            pos += (o - lo) * stride;
            stride *= hi - lo + 1;
            col += (i + o) * cstride;
            cstride *= N;
        }
        if (ok) col_idx[row_ptr[orow] + pos] = (int32_t)col;
    }
}

__device__ __forceinline__ double knot_t(int64_t i, int p, int64_t n) {
    int64_t k = i - p;
    k = k < 0 ? 0 : (k > n ? n : k);
    return (double)k / (double)n;
}

__device__ __forceinline__ double greville(int64_t j, int p, int64_t n) {
    double s = 0.0;
    for (int q = 1; q <= p; ++q) s += knot_t(j + q, p, n);
    return s / p;
}

__global__ void k_row_moments(int p, const Dims D, int64_t row_begin, int64_t rows, const double* vals, int64_t ld,
                              double* out) {
    const int dim = D.dim;
    const int S = 2 * p + 1;
    int NS = 1;
    for (int q = 0; q < dim; ++q) NS *= S;
    for (int64_t orow = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; orow < rows;
         orow += (int64_t)gridDim.x * blockDim.x) {
        int64_t idx[3];
        D.decode(row_begin + orow, idx);
        double m[4] = {0.0, 0.0, 0.0, 0.0};
        for (int slot = 0; slot < NS; ++slot) {
            int s = slot;
            bool ok = true;
            double g[3];
            for (int q = 0; q < dim; ++q) {
                const int64_t j = idx[q] + (s % S) - p;
                s /= S;
                if (j < 0 || j >= D.N[q]) ok = false;
                else g[q] = greville(j, p, D.n[q]);
            }
            if (!ok) continue;
            const double v = vals[orow * ld + slot];
            m[0] += v;
            for (int q = 0; q < dim; ++q) m[1 + q] += v * g[q];
        }
        for (int q = 0; q <= dim; ++q) out[orow * (1 + dim) + q] = m[q];
    }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_checksum(int p, int dim, int64_t row_begin, int64_t rows, const double* vals, int64_t ld,
                           unsigned long long* out) {
    const int S = 2 * p + 1;
    int NS = 1;
    for (int q = 0; q < dim; ++q) NS *= S;
    unsigned long long h = 0;
    double s1 = 0.0, s2 = 0.0;
    const int64_t total = rows * NS;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t orow = t / NS;
        const int slot = (int)(t % NS);
        const double v = vals[orow * ld + slot];
        const unsigned long long key = (unsigned long long)(row_begin + orow) * (unsigned long long)NS + slot;
        h += mix64((unsigned long long)__double_as_longlong(v) ^ mix64(key));
        s1 += v;
        s2 += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        h += __shfl_xor_sync(0xffffffffu, h, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, h);
        atomicAdd((double*)(out + 1), s1);
        atomicAdd((double*)(out + 2), s2);
    }
}

unsigned grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

int64_t host_nnz_before(int64_t row, int p, const Dims& D) { return nnz_before(row, p, D); }

int launch_csr_structure(const wgq_rules_s* R, int64_t row_begin, int64_t row_end, int64_t* row_ptr, int32_t* col_idx,
                         void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = row_end - row_begin;
    k_row_ptr<<<grid_for(rows + 1), 256, 0, st>>>(R->p, R->dims, row_begin, rows, row_ptr);
    int NS = 1;
    for (int q = 0; q < R->dim; ++q) NS *= 2 * R->p + 1;
    if (rows > 0) k_col_idx<<<grid_for(rows * NS), 256, 0, st>>>(R->p, R->dims, row_begin, rows, row_ptr, col_idx);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

int launch_row_moments(const wgq_rules_s* R, const wgq_out_t* A, double* out, void* stream) {
    const int64_t rows = A->row_end - A->row_begin;
    if (rows <= 0) return WGQ_OK;
    k_row_moments<<<grid_for(rows), 256, 0, (cudaStream_t)stream>>>(R->p, R->dims, A->row_begin, rows, A->values,
                                                                     A->ld, out);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

int launch_checksum(const wgq_rules_s* R, const wgq_out_t* A, unsigned long long* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), st) != cudaSuccess) return WGQ_ECUDA;
    const int64_t rows = A->row_end - A->row_begin;
    if (rows <= 0) return WGQ_OK;
    int NS = 1;
    for (int q = 0; q < R->dim; ++q) NS *= 2 * R->p + 1;
    k_checksum<<<grid_for(rows * NS), 256, 0, st>>>(R->p, R->dim, A->row_begin, rows, A->values, A->ld, out);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

}  // namespace wgq
