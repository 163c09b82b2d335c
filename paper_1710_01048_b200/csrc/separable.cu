// Separable-coefficient fast path (SURVEY §8(a) a3-a7 for CONST and TRIG_SEP; C1, C2, C4).
//
// With c(x) = c0 + A prod_a f_a(x_a) (A = 0 for CONST), the row rule's sum factorises
// completely (eq:Decompo with the coefficient split into its two separable terms):
//
//   M_ij = c0 prod_a uM_a[o_a] + A prod_a vM_a[o_a]
//   K_ij = sum_a ( c0 uK_a[o_a] prod_{b!=a} uM_b[o_b] + A vK_a[o_a] prod_{b!=a} vM_b[o_b] )
//
// with, per direction a and 1D row r (nodes / effective weights of the row's rules, P:250,
// P:351):
//   uM[o] = sum_k wM_k B_{r+o}(xM_k)        vM[o] = sum_k wM_k f_a(xM_k) B_{r+o}(xM_k)
//   uK[o] = sum_k wK_k B'_{r+o}(xK_k)       vK[o] = sum_k wK_k f_a(xK_k) B'_{r+o}(xK_k)
//
// — the definition's sum, reordered; exact up to rounding.  A table kernel builds the 4 x s
// vectors of every 1D row; the assembly kernel is then a pure output stream: lanes own
// consecutive output elements of a warp's chunk of rows (coalesced stores), each element a
// few products of table entries (L1-resident).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <mutex>

#include "internal.h"

namespace wgq {
namespace {

struct SepArgs {
    const double* sep;     // [dim][N][4][kMaxS]: uM, vM, uK, vK
    int64_t N;
    int64_t row_begin, row_end;
    double c0, amp;
    double* Mv;
    double* Kv;
    int64_t ldM, ldK;
    const int64_t* rpM;    // CSR row pointers (slab-local), or null for ELL
    const int64_t* rpK;
    int layout;
};

__global__ void k_sep_tables(int dim, int p, RowTables T, int kind, int trig0, int trig1, int trig2, int wn0, int wn1,
                             int wn2, double* sep) {
    const int S = 2 * p + 1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = (tid / S) % T.N;
    const int a = (int)(tid / (S * T.N));
    const int o = (int)(tid % S);
    if (a >= dim) return;
    const int trig = a == 0 ? trig0 : (a == 1 ? trig1 : trig2);
    const int wn = a == 0 ? wn0 : (a == 1 ? wn1 : wn2);
    auto f = [&](double x) -> double {
        if (kind != WGQ_COEF_TRIG_SEP) return 0.0;
        const double arg = 2.0 * (double)wn * x;    // trig(pi * arg) = trig(2 pi k x)
        return trig == WGQ_TRIG_SIN ? sinpi(arg) : cospi(arg);
    };
    double uM = 0.0, vM = 0.0, uK = 0.0, vK = 0.0;
    for (int k = 0; k < T.mM[r]; ++k) {
        const double w = T.wM[r * kMaxMassNodes + k];
        const double b = T.VM[(r * kMaxMassNodes + k) * kMaxS + o];
        uM = fma(w, b, uM);
        vM = fma(w * f(T.xM[r * kMaxMassNodes + k]), b, vM);
    }
    for (int k = 0; k < T.mK[r]; ++k) {
        const double w = T.wK[r * kMaxStiffNodes + k];
        const double b = T.DK[(r * kMaxStiffNodes + k) * kMaxS + o];
        uK = fma(w, b, uK);
        vK = fma(w * f(T.xK[r * kMaxStiffNodes + k]), b, vK);
    }
    double* out = sep + ((int64_t)a * T.N + r) * 4 * kMaxS;
    out[0 * kMaxS + o] = uM;
    out[1 * kMaxS + o] = vM;
    out[2 * kMaxS + o] = uK;
    out[3 * kMaxS + o] = vK;
}

// position of slot (o - p per direction) inside the CSR row of (i1, i2, i3), or -1
template <int P, int D>
__device__ __forceinline__ int csr_pos(const int* o, const int64_t* idx, int64_t N) {
    int pos = 0, stride = 1;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        const int lo = idx[q] - P < 0 ? (int)-idx[q] : -P;
        const int hi = idx[q] + P > N - 1 ? (int)(N - 1 - idx[q]) : P;
        if (o[q] - P < lo || o[q] - P > hi) return -1;
        pos += (o[q] - P - lo) * stride;
        stride *= hi - lo + 1;
    }
    return pos;
}

// The value formulas, shared by both kernels so that ELL and CSR values are bitwise equal.
// y/z (line) constants of a slot: P = uM2 uM3, Q = vM2 vM3, PK = uK2 uM3 + uM2 uK3, QK likewise.
template <int D>
__device__ __forceinline__ void sep_consts(const double* f2, const double* f3, double& P, double& Q, double& PK,
                                           double& QK) {
    // f = {uM, vM, uK, vK} of direction 2 / 3 at the slot's offset
    if (D == 1) {
        P = Q = 1.0;
        PK = QK = 0.0;
    } else if (D == 2) {
        P = f2[0];
        Q = f2[1];
        PK = f2[2];
        QK = f2[3];
    } else {
        P = f2[0] * f3[0];
        Q = f2[1] * f3[1];
        PK = fma(f2[2], f3[0], f2[0] * f3[2]);
        QK = fma(f2[3], f3[1], f2[1] * f3[3]);
    }
}

__device__ __forceinline__ double sep_mass(double c0, double amp, double uM1, double vM1, double P, double Q) {
    return fma(amp, vM1 * Q, c0 * (uM1 * P)) + 0.0;
}

template <int D>
__device__ __forceinline__ double sep_stiff(double c0, double amp, double uM1, double vM1, double uK1, double vK1,
                                            double P, double Q, double PK, double QK) {
    const double su = D >= 2 ? fma(uK1, P, uM1 * PK) : uK1;
    const double sv = D >= 2 ? fma(vK1, Q, vM1 * QK) : vK1;
    return fma(amp, sv, c0 * su) + 0.0;
}

constexpr int kChunkRows = 32;

template <int P_, int D, int MODE>
__global__ void __launch_bounds__(256) k_sep(const SepArgs a) {
    constexpr int S = 2 * P_ + 1;
    constexpr int NS = D == 1 ? S : (D == 2 ? S * S : S * S * S);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t rows = a.row_end - a.row_begin;
    const uint64_t pol = pol_evict_first();
    for (int64_t c0row = warp * kChunkRows; c0row < rows; c0row += nwarps * kChunkRows) {
        const int64_t nrows = min((int64_t)kChunkRows, rows - c0row);
        const int64_t first = a.row_begin + c0row;
        // lane's first element: row first + lane / NS, slot lane % NS; indices advanced incrementally
        int rl = lane / NS, slot = lane % NS;
        int64_t idx[3] = {0, 0, 0};
        {
            int64_t rem = first + rl;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                idx[q] = rem % a.N;
                rem /= a.N;
            }
        }
        while (rl < nrows) {
            const int o[3] = {slot % S, (slot / S) % S, slot / (S * S)};
            double f[3][4];
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double* t = a.sep + ((int64_t)q * a.N + idx[q]) * 4 * kMaxS + o[q];
#pragma unroll
                for (int c = 0; c < 4; ++c) f[q][c] = (c < 2 || (MODE & 2)) ? __ldg(t + c * kMaxS) : 0.0;
            }
            double P, Q, PK, QK;
            sep_consts<D>(f[D >= 2 ? 1 : 0], f[D >= 3 ? 2 : 0], P, Q, PK, QK);
            const int64_t row = first + rl - a.row_begin;
            int cpos = 0;
            if (a.layout == WGQ_CSR) cpos = csr_pos<P_, D>(o, idx, a.N);
            if (MODE & 1) {
                const double m = sep_mass(a.c0, a.amp, f[0][0], f[0][1], P, Q);
                if (a.layout == WGQ_ELL) st_stream(a.Mv + row * a.ldM + slot, m, pol);
                else if (cpos >= 0) st_stream(a.Mv + a.rpM[row] + cpos, m, pol);
            }
            if (MODE & 2) {
                const double k = sep_stiff<D>(a.c0, a.amp, f[0][0], f[0][1], f[0][2], f[0][3], P, Q, PK, QK);
                if (a.layout == WGQ_ELL) st_stream(a.Kv + row * a.ldK + slot, k, pol);
                else if (cpos >= 0) st_stream(a.Kv + a.rpK[row] + cpos, k, pol);
            }
            // advance 32 elements: slot += 32, carrying whole rows into the row indices
            slot += 32;
            const int adv = slot / NS;
            slot -= adv * NS;
            rl += adv;
            idx[0] += adv;
#pragma unroll
            for (int q = 0; q + 1 < D; ++q) {
                while (idx[q] >= a.N) {
                    idx[q] -= a.N;
                    ++idx[q + 1];
                }
            }
        }
    }
}

// ELL fast variant (s^d <= 128): a warp walks a segment of one x-line.  Lane l owns the
// slots l + 32 j of every row (j < R); the y/z factors of those slots are line constants kept
// in registers (P = uM2 uM3, Q = vM2 vM3 and the stiffness combinations PK, QK), so a row
// costs each lane the four x-factors of its slots, a few FMAs and coalesced 256-byte stores.

constexpr int kSepSeg = 32;

template <int P, int D, int MODE>
__global__ void __launch_bounds__(256) k_sep_line(const SepArgs a) {
    constexpr int S = 2 * P + 1;
    constexpr int NS = D == 1 ? S : (D == 2 ? S * S : S * S * S);
    constexpr int R = (NS + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t N = a.N;
    const int64_t segs = (N + kSepSeg - 1) / kSepSeg;
    const int64_t line0 = a.row_begin / N, line1 = (a.row_end - 1) / N;
    const int64_t items = (line1 - line0 + 1) * segs;
    int o1[R];
#pragma unroll
    for (int j = 0; j < R; ++j) o1[j] = (lane + 32 * j) % S;
    const uint64_t pol = pol_evict_first();
    for (int64_t it = warp; it < items; it += nwarps) {
        const int64_t line = line0 + it / segs;
        const int64_t x0 = max((it % segs) * kSepSeg, a.row_begin - line * N);
        const int64_t x1 = min((it % segs) * kSepSeg + kSepSeg, min(N, a.row_end - line * N));
        if (x0 >= x1) continue;
        const int64_t i2 = D >= 2 ? line % N : 0, i3 = D >= 3 ? line / N : 0;
        // line constants per owned slot
        double cP[R], cQ[R], cPK[R], cQK[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int slot = min(lane + 32 * j, NS - 1);
            const int o23 = slot / S, o2 = o23 % S, o3 = o23 / S;
            double f2[4], f3[4];
            const double* t2 = a.sep + ((int64_t)1 * N + i2) * 4 * kMaxS + o2;
            const double* t3 = a.sep + ((int64_t)2 * N + i3) * 4 * kMaxS + o3;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                f2[c] = __ldg(t2 + c * kMaxS);
                f3[c] = D >= 3 ? __ldg(t3 + c * kMaxS) : 0.0;
            }
            sep_consts<D>(f2, f3, cP[j], cQ[j], cPK[j], cQK[j]);
        }
        // the x-direction vectors of the next row are loaded while the current row is stored
        double xu[R], xv[R], xuk[R], xvk[R];
        auto load_x = [&](int64_t i1) {
            const double* t1 = a.sep + i1 * 4 * kMaxS;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                xu[j] = __ldg(t1 + o1[j]);
                xv[j] = __ldg(t1 + kMaxS + o1[j]);
                if (MODE & 2) {
                    xuk[j] = __ldg(t1 + 2 * kMaxS + o1[j]);
                    xvk[j] = __ldg(t1 + 3 * kMaxS + o1[j]);
                }
            }
        };
        load_x(x0);
        for (int64_t i1 = x0; i1 < x1; ++i1) {
            const int64_t orow = line * N + i1 - a.row_begin;
            double cu[R], cv[R], cuk[R], cvk[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                cu[j] = xu[j];
                cv[j] = xv[j];
                cuk[j] = (MODE & 2) ? xuk[j] : 0.0;
                cvk[j] = (MODE & 2) ? xvk[j] : 0.0;
            }
            if (i1 + 1 < x1) load_x(i1 + 1);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int slot = lane + 32 * j;
                if (slot >= NS) continue;
                if (MODE & 1) st_stream(a.Mv + orow * a.ldM + slot, sep_mass(a.c0, a.amp, cu[j], cv[j], cP[j], cQ[j]), pol);
                if (MODE & 2)
                    st_stream(a.Kv + orow * a.ldK + slot, sep_stiff<D>(a.c0, a.amp, cu[j], cv[j], cuk[j], cvk[j], cP[j],
                                                                       cQ[j], cPK[j], cQK[j]), pol);
            }
        }
    }
}

template <int P, int D>
int launch_sep_pd(const SepArgs& a, int mode, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t chunks = (rows + kChunkRows - 1) / kChunkRows;
    int64_t blocks = (chunks + 7) / 8;
    blocks = std::min<int64_t>(blocks, (int64_t)sms * 16);
    blocks = std::max<int64_t>(blocks, 1);
    constexpr int NS = D == 1 ? 2 * P + 1 : (D == 2 ? (2 * P + 1) * (2 * P + 1) : (2 * P + 1) * (2 * P + 1) * (2 * P + 1));
    if constexpr (NS <= 128 && D == 3) {
      if (a.layout == WGQ_ELL) {
        const int64_t segs = (a.N + kSepSeg - 1) / kSepSeg;
        const int64_t items = ((a.row_end - 1) / a.N - a.row_begin / a.N + 1) * segs;
        // one warp per item, blocks dispatched in address order: the write stream stays one
        // front (a capped grid-stride lets warps drift apart; DESIGN.md roofline): 0.358 -> 0.350 ms
        const int64_t b2 = std::max<int64_t>(1, (items + 7) / 8);
        if (mode == 3) k_sep_line<P, D, 3><<<(unsigned)b2, 256, 0, st>>>(a);
        else if (mode == 1) k_sep_line<P, D, 1><<<(unsigned)b2, 256, 0, st>>>(a);
        else k_sep_line<P, D, 2><<<(unsigned)b2, 256, 0, st>>>(a);
        return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
      }
    }
    if (mode == 3) k_sep<P, D, 3><<<(unsigned)blocks, 256, 0, st>>>(a);
    else if (mode == 1) k_sep<P, D, 1><<<(unsigned)blocks, 256, 0, st>>>(a);
    else k_sep<P, D, 2><<<(unsigned)blocks, 256, 0, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

}  // namespace

bool sep_applies(const wgq_coeff_t* c) { return c->kind == WGQ_COEF_CONST || c->kind == WGQ_COEF_TRIG_SEP; }

// The 4 x s per-direction vectors of every 1D row (uM, vM, uK, vK); they depend on the rules and
// the factors f_a only (c0, amp enter the value formulas): built once per (device, kind, trig,
// wavenum) and cached in the rules handle.
int sep_vectors_for(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, cudaStream_t st, double** out) {
    const int S = 2 * R->p + 1;
    double* sep = nullptr;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        const bool trig = c->kind == WGQ_COEF_TRIG_SEP;
        const std::array<int, 8> key = {dev, c->kind, trig ? c->trig[0] : 0, trig ? c->trig[1] : 0, trig ? c->trig[2] : 0,
                                        trig ? c->wavenum[0] : 0, trig ? c->wavenum[1] : 0, trig ? c->wavenum[2] : 0};
        wgq_rules_s* Rm = const_cast<wgq_rules_s*>(R);
        std::lock_guard<std::mutex> lock(Rm->mu);
        auto it = Rm->sep_vectors.find(key);
        if (it == Rm->sep_vectors.end()) {
            const int64_t entries = (int64_t)R->dim * R->N * 4 * kMaxS;
            if (cudaMalloc((void**)&sep, (size_t)entries * sizeof(double)) != cudaSuccess) return WGQ_ENOMEM;
            const int64_t threads = (int64_t)R->dim * R->N * S;
            k_sep_tables<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(R->dim, R->p, T, c->kind, c->trig[0],
                                                                            c->trig[1], c->trig[2], c->wavenum[0],
                                                                            c->wavenum[1], c->wavenum[2], sep);
            // used from any stream afterwards: complete the one-time build now
            if (cudaStreamSynchronize(st) != cudaSuccess) return WGQ_ECUDA;
            Rm->sep_vectors.emplace(key, sep);
        } else {
            sep = it->second;
        }
    }
    *out = sep;
    return WGQ_OK;
}

int launch_sep(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const wgq_out_t* M,
               const wgq_out_t* K, void* stream) {
    const wgq_out_t* any = M ? M : K;
    if (any->row_end <= any->row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    double* sep = nullptr;
    {
        const int rc = sep_vectors_for(R, T, c, st, &sep);
        if (rc != WGQ_OK) return rc;
    }
    SepArgs a{};
    a.sep = sep;
    a.N = R->N;
    a.row_begin = any->row_begin;
    a.row_end = any->row_end;
    a.c0 = c->c0;
    a.amp = c->kind == WGQ_COEF_TRIG_SEP ? c->amp : 0.0;
    a.layout = any->layout;
    if (M) {
        a.Mv = M->values;
        a.ldM = M->ld;
        a.rpM = M->row_ptr;
    }
    if (K) {
        a.Kv = K->values;
        a.ldK = K->ld;
        a.rpK = K->row_ptr;
    }
    const int mode = (M ? 1 : 0) | (K ? 2 : 0);
    int rc = WGQ_EUNSUPPORTED;
    switch (R->p * 10 + R->dim) {
        case 21: rc = launch_sep_pd<2, 1>(a, mode, st); break;
        case 22: rc = launch_sep_pd<2, 2>(a, mode, st); break;
        case 23: rc = launch_sep_pd<2, 3>(a, mode, st); break;
        case 31: rc = launch_sep_pd<3, 1>(a, mode, st); break;
        case 32: rc = launch_sep_pd<3, 2>(a, mode, st); break;
        case 33: rc = launch_sep_pd<3, 3>(a, mode, st); break;
    }
    return rc;
}

// ---------------------------------------------------------------------------------------------
// Matrix-free y = M u, K u for the separable coefficients: with the row's
// per-direction vectors (uM, vM, uK, vK)_a, A_ij = c0 prod_a uM_a[o_a] + amp prod_a vM_a[o_a]
// (mass; stiffness as in sep_stiff), so y_i = sum_j A_ij u_j is contracted x -> y -> z per row:
// the same sum as the definition, reordered.  One thread per row; the x-direction vectors of the
// row live in registers, neighbouring threads read overlapping u windows (coalesced).
namespace {
template <int P, int D>
__global__ void __launch_bounds__(256) k_sep_apply(const double* sep, int64_t N, int64_t row_begin, int64_t row_end,
                                                   double c0, double amp, const double* u, int64_t u_row0, double* yM,
                                                   double* yK) {
    constexpr int S = 2 * P + 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t row = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < row_end; row += stride) {
        const int64_t i1 = row % N, i2 = D >= 2 ? (row / N) % N : 0, i3 = D >= 3 ? row / (N * N) : 0;
        const int lo1 = (int)max((int64_t)0, P - i1), hi1 = (int)min((int64_t)(2 * P), N - 1 - i1 + P);
        const int lo2 = D >= 2 ? (int)max((int64_t)0, P - i2) : 0, hi2 = D >= 2 ? (int)min((int64_t)(2 * P), N - 1 - i2 + P) : 0;
        const int lo3 = D >= 3 ? (int)max((int64_t)0, P - i3) : 0, hi3 = D >= 3 ? (int)min((int64_t)(2 * P), N - 1 - i3 + P) : 0;
        const double* t1 = sep + i1 * 4 * kMaxS;
        const double* t2 = sep + (N + i2) * 4 * kMaxS;
        const double* t3 = sep + (2 * N + i3) * 4 * kMaxS;
        double w1[4][S];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int o = 0; o < S; ++o) w1[c][o] = __ldg(t1 + c * kMaxS + o);
        double Mu = 0.0, Mv = 0.0, Ku = 0.0, Kv = 0.0;
        for (int o3 = lo3; o3 <= hi3; ++o3) {
            double Auu = 0.0, Avv = 0.0, Xu = 0.0, Xv = 0.0;    // Auu = sum uM2 (uM1 . u); X = K_x + K_y parts
            for (int o2 = lo2; o2 <= hi2; ++o2) {
                const int64_t base = D == 3 ? ((i3 - P + o3) * N + (i2 - P + o2)) * N : (D == 2 ? (i2 - P + o2) * N : 0);
                const double* ur = u + base + (i1 - P) - u_row0;
                double suM = 0.0, svM = 0.0, suK = 0.0, svK = 0.0;
#pragma unroll
                for (int o1 = 0; o1 < S; ++o1) {
                    if (o1 < lo1 || o1 > hi1) continue;
                    const double uv = __ldg(ur + o1);
                    suM = fma(w1[0][o1], uv, suM);
                    svM = fma(w1[1][o1], uv, svM);
                    suK = fma(w1[2][o1], uv, suK);
                    svK = fma(w1[3][o1], uv, svK);
                }
                if (D == 1) {
                    Mu = suM, Mv = svM, Ku = suK, Kv = svK;
                    continue;
                }
                const double uM2 = __ldg(t2 + o2), vM2 = __ldg(t2 + kMaxS + o2);
                const double uK2 = __ldg(t2 + 2 * kMaxS + o2), vK2 = __ldg(t2 + 3 * kMaxS + o2);
                Auu = fma(uM2, suM, Auu);
                Avv = fma(vM2, svM, Avv);
                Xu = fma(uM2, suK, fma(uK2, suM, Xu));             // uK1 uM2 + uM1 uK2
                Xv = fma(vM2, svK, fma(vK2, svM, Xv));
            }
            if (D == 1) break;
            if (D == 2) {
                Mu = Auu, Mv = Avv, Ku = Xu, Kv = Xv;
                break;
            }
            const double uM3 = __ldg(t3 + o3), vM3 = __ldg(t3 + kMaxS + o3);
            const double uK3 = __ldg(t3 + 2 * kMaxS + o3), vK3 = __ldg(t3 + 3 * kMaxS + o3);
            Mu = fma(uM3, Auu, Mu);
            Mv = fma(vM3, Avv, Mv);
            Ku = fma(uM3, Xu, fma(uK3, Auu, Ku));                  // (K_x + K_y) uM3 + uM1 uM2 uK3
            Kv = fma(vM3, Xv, fma(vK3, Avv, Kv));
        }
        const int64_t o = row - row_begin;
        if (yM) yM[o] = fma(amp, Mv, c0 * Mu);
        if (yK) yK[o] = fma(amp, Kv, c0 * Ku);
    }
}
}  // namespace

int launch_sep_apply(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const double* u, int64_t u_row0,
                     int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream) {
    if (row_end <= row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    double* sep = nullptr;
    int rc = sep_vectors_for(R, T, c, st, &sep);
    if (rc != WGQ_OK) return rc;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t rows = row_end - row_begin;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)sms * 16));
    const double amp = c->kind == WGQ_COEF_TRIG_SEP ? c->amp : 0.0;
    switch (R->p * 10 + R->dim) {
        case 21: k_sep_apply<2, 1><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        case 22: k_sep_apply<2, 2><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        case 23: k_sep_apply<2, 3><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        case 31: k_sep_apply<3, 1><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        case 32: k_sep_apply<3, 2><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        case 33: k_sep_apply<3, 3><<<blocks, 256, 0, st>>>(sep, R->N, row_begin, row_end, c->c0, amp, u, u_row0, yM, yK); break;
        default: return WGQ_EUNSUPPORTED;
    }
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

// Load vector for the separable coefficients: b_i = sum_k prod_a wM_a f(x_k)
// with f = c0 + amp prod_a f_a, and sum_o uM_a[o] = sum_k wM_k (partition of unity over the
// functions nonzero at each node; likewise vM with f_a), so b_i = c0 prod_a U_a + amp prod_a V_a.
namespace {
template <int D>
__global__ void __launch_bounds__(256) k_sep_load(const double* sep, int64_t N, int S, int64_t row_begin,
                                                  int64_t row_end, double c0, double amp, double* b) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t row = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < row_end; row += stride) {
        int64_t idx[3] = {row % N, D >= 2 ? (row / N) % N : 0, D >= 3 ? row / (N * N) : 0};
        double pu = 1.0, pv = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double* t = sep + ((int64_t)a * N + idx[a]) * 4 * kMaxS;
            double su = 0.0, sv = 0.0;
            for (int o = 0; o < S; ++o) {
                su += __ldg(t + o);
                sv += __ldg(t + kMaxS + o);
            }
            pu *= su;
            pv *= sv;
        }
        b[row - row_begin] = fma(amp, pv, c0 * pu);
    }
}
}  // namespace

int launch_sep_load(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                    double* b, void* stream) {
    if (row_end <= row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    double* sep = nullptr;
    int rc = sep_vectors_for(R, T, c, st, &sep);
    if (rc != WGQ_OK) return rc;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t rows = row_end - row_begin;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)sms * 16));
    const double amp = c->kind == WGQ_COEF_TRIG_SEP ? c->amp : 0.0;
    const int S = 2 * R->p + 1;
    if (R->dim == 1) k_sep_load<1><<<blocks, 256, 0, st>>>(sep, R->N, S, row_begin, row_end, c->c0, amp, b);
    else if (R->dim == 2) k_sep_load<2><<<blocks, 256, 0, st>>>(sep, R->N, S, row_begin, row_end, c->c0, amp, b);
    else k_sep_load<3><<<blocks, 256, 0, st>>>(sep, R->N, S, row_begin, row_end, c->c0, amp, b);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

}  // namespace wgq
