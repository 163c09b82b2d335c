// End-to-end assembly from/to host memory (wgq_assemble_host): the coefficient slab is
// uploaded once, rows are assembled in chunks into double-buffered device staging on a
// compute stream, and each finished chunk is copied to the caller's host arrays on a copy
// stream while the next chunk is computed.  One cudaMemcpyAsync per copy (cudaMemcpy2DAsync
// into a padded host row stride: only the s^d structural slots of each host row are written).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

using namespace wgq;

extern "C" int wgq_assemble_mass_stiffness(wgq_rules_t, const wgq_coeff_t*, const wgq_out_t*, const wgq_out_t*, void*);
extern "C" int wgq_assemble_mass(wgq_rules_t, const wgq_coeff_t*, const wgq_out_t*, void*);
extern "C" int wgq_assemble_stiffness(wgq_rules_t, const wgq_coeff_t*, const wgq_out_t*, void*);

namespace {

struct Cleanup {
    void* dev[5] = {};
    cudaStream_t s[2] = {};
    cudaEvent_t e[4] = {};
    ~Cleanup() {
        for (void* p : dev)
            if (p) cudaFree(p);
        for (auto x : s)
            if (x) cudaStreamDestroy(x);
        for (auto x : e)
            if (x) cudaEventDestroy(x);
    }
};

}  // namespace

extern "C" int wgq_host_alloc(uint64_t bytes, void** ptr) {
    if (!ptr) return WGQ_EINVAL;
    return cudaHostAlloc(ptr, bytes, cudaHostAllocDefault) == cudaSuccess ? WGQ_OK : WGQ_ENOMEM;
}

extern "C" int wgq_host_free(void* ptr) { return cudaFreeHost(ptr) == cudaSuccess ? WGQ_OK : WGQ_ECUDA; }

extern "C" int wgq_assemble_host(wgq_rules_t R, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                                 double* M_host, double* K_host, int64_t ld, int64_t chunk_rows) {
    NvtxRange nvtx_("wgq_assemble_host");
    if (!R || !c || (!M_host && !K_host) || row_begin < 0 || row_end < row_begin) return WGQ_EINVAL;
    int64_t stencil = 1;
    for (int q = 0; q < R->dim; ++q) stencil *= 2 * R->p + 1;
    if (ld < stencil) return WGQ_ERANGE;
    if (row_end == row_begin) return WGQ_OK;
    // the descriptor must cover the whole range before anything is allocated or copied
    if (int rc0 = validate_coeff_range(R, c, row_begin, row_end)) return rc0;
    Cleanup cl;
    if (cudaStreamCreateWithFlags(&cl.s[0], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&cl.s[1], cudaStreamNonBlocking) != cudaSuccess)
        return WGQ_ECUDA;
    for (auto& e : cl.e)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return WGQ_ECUDA;
    cudaStream_t comp = cl.s[0], copy = cl.s[1];

    // coefficient: move a host GRID slab to the device once
    wgq_coeff_t dc = *c;
    if (c->kind == WGQ_COEF_GRID) {
        if (!c->grid) return WGQ_EINVAL;
        int64_t plane = 1;
        for (int q = 0; q < R->dim - 1; ++q) plane *= R->dims.n[q] + 1;
        const size_t bytes = (size_t)c->grid_planes * plane * sizeof(double);   // plane = 1 in 1D
        if (cudaMalloc(&cl.dev[0], bytes) != cudaSuccess) return WGQ_ECUDA;
        if (cudaMemcpyAsync(cl.dev[0], c->grid, bytes, cudaMemcpyHostToDevice, comp) != cudaSuccess) return WGQ_ECUDA;
        dc.grid = (const double*)cl.dev[0];
    }
    const int64_t rows = row_end - row_begin;
    // device staging holds compact rows (stride s^d); a padded host stride is written with 2D
    // copies, so the host slots [s^d, ld) are never written (as for the device ELL output)
    if (chunk_rows <= 0) chunk_rows = std::max<int64_t>(1, ((int64_t)1 << 27) / stencil);   // ~1 GiB per matrix
    chunk_rows = std::min(chunk_rows, rows);
    const size_t chunk_bytes = (size_t)chunk_rows * stencil * sizeof(double);
    const bool doM = M_host != nullptr, doK = K_host != nullptr;
    for (int b = 0; b < 2; ++b) {
        if (doM && cudaMalloc(&cl.dev[1 + b], chunk_bytes) != cudaSuccess) return WGQ_ECUDA;
        if (doK && cudaMalloc(&cl.dev[3 + b], chunk_bytes) != cudaSuccess) return WGQ_ECUDA;
    }
    cudaEvent_t computed[2] = {cl.e[0], cl.e[1]}, copied[2] = {cl.e[2], cl.e[3]};
    int rc = WGQ_OK;
    int64_t it = 0;
    for (int64_t lo = row_begin; lo < row_end; lo += chunk_rows, ++it) {
        const int64_t hi = std::min(row_end, lo + chunk_rows);
        const int b = (int)(it & 1);
        if (it >= 2) cudaStreamWaitEvent(comp, copied[b], 0);     // staging buffer b is free again
        wgq_out_t M{WGQ_ELL, lo, hi, (double*)cl.dev[1 + b], stencil, nullptr, nullptr};
        wgq_out_t K{WGQ_ELL, lo, hi, (double*)cl.dev[3 + b], stencil, nullptr, nullptr};
        if (doM && doK) rc = wgq_assemble_mass_stiffness(R, &dc, &M, &K, comp);
        else if (doM) rc = wgq_assemble_mass(R, &dc, &M, comp);
        else rc = wgq_assemble_stiffness(R, &dc, &K, comp);
        if (rc != WGQ_OK) break;
        cudaEventRecord(computed[b], comp);
        cudaStreamWaitEvent(copy, computed[b], 0);
        const size_t off = (size_t)(lo - row_begin) * ld;
        auto d2h = [&](double* dst, const void* src) {
            if (ld == stencil)
                return cudaMemcpyAsync(dst, src, (size_t)(hi - lo) * stencil * sizeof(double), cudaMemcpyDeviceToHost,
                                       copy);
            return cudaMemcpy2DAsync(dst, (size_t)ld * sizeof(double), src, (size_t)stencil * sizeof(double),
                                     (size_t)stencil * sizeof(double), (size_t)(hi - lo), cudaMemcpyDeviceToHost, copy);
        };
        if (doM && d2h(M_host + off, cl.dev[1 + b]) != cudaSuccess) {
            rc = WGQ_ECUDA;
            break;
        }
        if (doK && d2h(K_host + off, cl.dev[3 + b]) != cudaSuccess) {
            rc = WGQ_ECUDA;
            break;
        }
        cudaEventRecord(copied[b], copy);
    }
    if (cudaStreamSynchronize(comp) != cudaSuccess || cudaStreamSynchronize(copy) != cudaSuccess) rc = WGQ_ECUDA;
    (void)rows;
    return rc;
}
