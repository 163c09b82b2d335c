// Row-wise weighted-Gaussian assembly kernels for sm_100a.
//
// Generic kernel: one warp per row, any p in {2,3}, d in {1,2,3}, any coefficient kind
// and any row class.  For the row i = (i1,i2,i3) and each tensor term (M; K_x; K_y + K_z)
//   W[k1,k2,k3]  = c(x_k) * w1[k1] w2[k2] w3[k3]                      (a3, a4)
//   T1[k1,k2,o3] = sum_k3 W  A3[k3,o3]      z-stage                   (a5, eq:Decompo)
//   T2[k1,o2,o3] = sum_k2 T1 A2[k2,o2]      y-stage
//   R[o1,o2,o3] += sum_k1 T2 A1[k1,o1]      x-stage, lanes own output slots
// with A = B_{i+o}(x_k) (mass nodes) or B'_{i+o}(x_k) (stiffness nodes) from the per-row
// tables; the K_y and K_z terms share one x-stage (a6).  The staged W/T1/T2 live in the
// warp's shared-memory slice; lanes own the s^d output slots (slot = lane + 32 j), so the
// stores of a warp are contiguous 256-byte runs of the row (a7).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "coef.cuh"
#include "internal.h"

namespace wgq {
namespace {

constexpr int kMaxWarps = 8;

__device__ __constant__ double kOnes[kMaxStiffNodes * kMaxS] = {1.0};

// per-warp staging sizes (doubles) for the node counts of the rules at hand
struct Staging {
    int w, t1, t2, per_warp;
};

struct OutDev {
    double* values;
    int64_t ld;
    const int64_t* row_ptr;
    int layout;
};

struct GenericArgs {
    RowTables T;
    CoefDev coef;
    int64_t n, N;
    int64_t row_begin, row_end;
    OutDev M, K;
    int do_mass, do_stiff;
    Staging sg;
};

// per-direction operand of a tensor term
struct Dir {
    int m;             // nodes
    const double* x;   // [m]
    const double* w;   // [m]
    const double* A;   // [m][kMaxS]
};

template <int D>
__device__ __forceinline__ void stage_term(const GenericArgs& a, const Dir d1, const Dir d2, const Dir d3,
                                           int S1, int S2, int S3, double* W, double* T1, double* T2,
                                           bool accumulate, int lane) {
    const int n1 = d1.m, n2 = d2.m, n3 = d3.m;
    // a3-a4: weighted coefficient samples on the node tensor
    for (int e = lane; e < n1 * n2 * n3; e += 32) {
        const int k3 = e % n3, k2 = (e / n3) % n2, k1 = e / (n3 * n2);
        double x[3] = {d1.x[k1], d2.x[k2], d3.x[k3]};
        W[e] = coef_eval<D>(a.coef, a.n, x) * d1.w[k1] * d2.w[k2] * d3.w[k3];
    }
    __syncwarp();
    // z-stage
    for (int e = lane; e < n1 * n2 * S3; e += 32) {
        const int o3 = e % S3, k12 = e / S3;
        double s = 0.0;
        for (int k3 = 0; k3 < n3; ++k3) s = fma(W[k12 * n3 + k3], d3.A[k3 * kMaxS + o3], s);
        T1[e] = s;
    }
    __syncwarp();
    // y-stage: T2 is laid out [k1][o3][o2] so that o2 + S2*o3 is the slot's (o2,o3) part
    for (int e = lane; e < n1 * S2 * S3; e += 32) {
        const int o2 = e % S2, o3 = (e / S2) % S3, k1 = e / (S3 * S2);
        double s = accumulate ? T2[e] : 0.0;
        for (int k2 = 0; k2 < n2; ++k2) s = fma(T1[(k1 * n2 + k2) * S3 + o3], d2.A[k2 * kMaxS + o2], s);
        T2[e] = s;
    }
    __syncwarp();
}

template <int NJ>
__device__ __forceinline__ void x_stage(const Dir d1, int S1, int S2, int S3, const double* T2, double* acc, int lane) {
    const int NS = S1 * S2 * S3;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int slot = lane + 32 * j;
        if (slot < NS) {
            const int o1 = slot % S1, o23 = slot / S1;
            double s = acc[j];
            for (int k1 = 0; k1 < d1.m; ++k1) s = fma(T2[k1 * S2 * S3 + o23], d1.A[k1 * kMaxS + o1], s);
            acc[j] = s;
        }
    }
}

template <int P, int D>
__global__ void __launch_bounds__(kMaxWarps * 32) k_assemble_generic(const GenericArgs a) {
    constexpr int S = 2 * P + 1;
    constexpr int S1 = S, S2 = D >= 2 ? S : 1, S3 = D >= 3 ? S : 1;
    constexpr int NS = S1 * S2 * S3;
    constexpr int NJ = (NS + 31) / 32;
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    double* W = smem + warp * a.sg.per_warp;
    double* T1 = W + a.sg.w;
    double* T2 = T1 + a.sg.t1;
    double* T2b = T2 + a.sg.t2;
    const RowTables& T = a.T;
    const Dir ones = {1, kOnes, kOnes, kOnes};

    for (int64_t row = a.row_begin + (int64_t)blockIdx.x * warps + warp; row < a.row_end;
         row += (int64_t)gridDim.x * warps) {
        int64_t idx[3] = {0, 0, 0};
        int64_t rem = row;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            idx[q] = rem % a.N;
            rem /= a.N;
        }
        Dir dm[3], dk[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (q < D) {
                const int64_t r = idx[q];
                dm[q] = {T.mM[r], T.xM + r * kMaxMassNodes, T.wM + r * kMaxMassNodes, T.VM + r * kMaxMassNodes * kMaxS};
                dk[q] = {T.mK[r], T.xK + r * kMaxStiffNodes, T.wK + r * kMaxStiffNodes, T.DK + r * kMaxStiffNodes * kMaxS};
            } else {
                dm[q] = ones;
                dk[q] = ones;
            }
        }
        double accM[NJ], accK[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) accM[j] = accK[j] = 0.0;

        if (a.do_mass) {
            stage_term<D>(a, dm[0], dm[1], dm[2], S1, S2, S3, W, T1, T2, false, lane);
            x_stage<NJ>(dm[0], S1, S2, S3, T2, accM, lane);
        }
        if (a.do_stiff) {
            // K_x: stiffness nodes / derivative table in x
            stage_term<D>(a, dk[0], dm[1], dm[2], S1, S2, S3, W, T1, T2b, false, lane);
            x_stage<NJ>(dk[0], S1, S2, S3, T2b, accK, lane);
            __syncwarp();
            if (D >= 2) {
                stage_term<D>(a, dm[0], dk[1], dm[2], S1, S2, S3, W, T1, T2b, false, lane);   // K_y
                if (D >= 3) stage_term<D>(a, dm[0], dm[1], dk[2], S1, S2, S3, W, T1, T2b, true, lane);  // + K_z
                x_stage<NJ>(dm[0], S1, S2, S3, T2b, accK, lane);
            }
        }
        // a7: store (x + 0.0 turns a -0.0 from all-zero products into +0.0)
        const int64_t orow = row - a.row_begin;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int slot = lane + 32 * j;
            if (slot >= NS) continue;
            if (a.M.layout == WGQ_ELL) {
                if (a.do_mass) a.M.values[orow * a.M.ld + slot] = accM[j] + 0.0;
                if (a.do_stiff) a.K.values[orow * a.K.ld + slot] = accK[j] + 0.0;
            } else {
                // CSR: slot -> compacted position inside the box of valid offsets
                int o[3] = {slot % S1 - P, (slot / S1) % S2 - (D >= 2 ? P : 0), slot / (S1 * S2) - (D >= 3 ? P : 0)};
                int64_t pos = 0, stride = 1;
                bool ok = true;
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    const int64_t lo = idx[q] - P < 0 ? -idx[q] : -P;
                    const int64_t hi = idx[q] + P > a.N - 1 ? a.N - 1 - idx[q] : P;
                    if (o[q] < lo || o[q] > hi) ok = false;
                    pos += (o[q] - lo) * stride;
                    stride *= hi - lo + 1;
                }
                if (!ok) continue;
                if (a.do_mass) a.M.values[a.M.row_ptr[orow] + pos] = accM[j] + 0.0;
                if (a.do_stiff) a.K.values[a.K.row_ptr[orow] + pos] = accK[j] + 0.0;
            }
        }
        __syncwarp();
    }
}

template <int P, int D>
int launch_generic_pd(GenericArgs a, int maxM, int maxK, cudaStream_t st) {
    constexpr int S = 2 * P + 1;
    const int S2 = D >= 2 ? S : 1, S3 = D >= 3 ? S : 1;
    const int mx = maxM > maxK ? maxM : maxK;
    Staging sg;
    if (D == 3) {
        sg.w = mx * maxM * maxM;
        sg.t1 = mx * maxM * S3;
    } else if (D == 2) {
        sg.w = mx * maxM;
        sg.t1 = mx * maxM;
    } else {
        sg.w = mx;
        sg.t1 = mx;
    }
    sg.t2 = mx * S2 * S3;
    sg.per_warp = sg.w + sg.t1 + 2 * sg.t2;
    a.sg = sg;
    const size_t per_warp_bytes = (size_t)sg.per_warp * sizeof(double);
    int warps = (int)std::min<size_t>(kMaxWarps, (200 * 1024) / per_warp_bytes);
    warps = std::max(warps, 1);
    const size_t smem = warps * per_warp_bytes;
    if (cudaFuncSetAttribute(k_assemble_generic<P, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return WGQ_ECUDA;
    const int64_t rows = a.row_end - a.row_begin;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assemble_generic<P, D>, warps * 32, smem);
    int64_t blocks = (rows + warps - 1) / warps;
    blocks = std::min<int64_t>(blocks, (int64_t)sms * std::max(per_sm, 1) * 8);
    blocks = std::max<int64_t>(blocks, 1);
    k_assemble_generic<P, D><<<(unsigned)blocks, warps * 32, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

CoefDev make_coef(const wgq_coeff_t* c) {
    CoefDev d{};
    d.kind = c->kind;
    d.c0 = c->c0;
    d.amp = c->amp;
    for (int a = 0; a < 3; ++a) {
        d.trig[a] = c->trig[a];
        d.wavenum[a] = c->wavenum[a];
    }
    d.n_modes = c->kind == WGQ_COEF_FOURIER_LOGN ? c->n_modes : 0;
    for (int m = 0; m < d.n_modes; ++m)
        for (int q = 0; q < 5; ++q) d.modes[m][q] = c->modes[m * 5 + q];
    d.grid = c->grid;
    d.plane0 = c->grid_plane0;
    d.planes = c->grid_planes;
    return d;
}

}  // namespace

int launch_assemble(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const wgq_out_t* M,
                    const wgq_out_t* K, void* stream) {
    static const bool force_generic = [] {
        const char* e = getenv("WGQ_FORCE_GENERIC");
        return e && e[0] == '1';
    }();
    if (!force_generic && line_kernel_applies(R, c, M, K)) return launch_line(R, T, c, M, K, stream);
    GenericArgs a{};
    a.T = T;
    a.coef = make_coef(c);
    a.n = R->n;
    a.N = R->N;
    const wgq_out_t* any = M ? M : K;
    a.row_begin = any->row_begin;
    a.row_end = any->row_end;
    a.do_mass = M != nullptr;
    a.do_stiff = K != nullptr;
    if (M) a.M = {M->values, M->ld, M->row_ptr, M->layout};
    if (K) a.K = {K->values, K->ld, K->row_ptr, K->layout};
    if (!M) a.M.layout = K->layout;
    if (a.row_end <= a.row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int key = R->p * 10 + R->dim;
    switch (key) {
        case 21: return launch_generic_pd<2, 1>(a, T.maxM, T.maxK, st);
        case 22: return launch_generic_pd<2, 2>(a, T.maxM, T.maxK, st);
        case 23: return launch_generic_pd<2, 3>(a, T.maxM, T.maxK, st);
        case 31: return launch_generic_pd<3, 1>(a, T.maxM, T.maxK, st);
        case 32: return launch_generic_pd<3, 2>(a, T.maxM, T.maxK, st);
        case 33: return launch_generic_pd<3, 3>(a, T.maxM, T.maxK, st);
    }
    return WGQ_EUNSUPPORTED;
}

}  // namespace wgq
