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

#include <cmath>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "coef.cuh"
#include "internal.h"

namespace wgq {
namespace {

constexpr int kMaxWarps = 8;

__device__ __constant__ double kOnes[kMaxStiffNodes * kMaxS] = {1.0};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// exp(x) for |x| < 700 in ~20 FP64 instructions: x = k ln2 + r (Cody-Waite, |r| <= ln2/2),
// e^r by its degree-13 Taylor polynomial (truncation < 2e-16 relative), times 2^k.  Within
// ~2 ulp of the correctly rounded value (the FOURIER_LOGN exponents are O(1), R13).
__constant__ double kExpTaylor[14] = {1.0,
                                      1.0,
                                      0.5,
                                      1.0 / 6.0,
                                      1.0 / 24.0,
                                      1.0 / 120.0,
                                      1.0 / 720.0,
                                      1.0 / 5040.0,
                                      1.0 / 40320.0,
                                      1.0 / 362880.0,
                                      1.0 / 3628800.0,
                                      1.0 / 39916800.0,
                                      1.0 / 479001600.0,
                                      1.0 / 6227020800.0};

__device__ __forceinline__ double exp_fast(double x) {
    // the Taylor coefficients come from the constant bank (DFMA operands), not 64-bit immediates
    // that the compiler would rebuild in uniform registers on every call
    const double k = rint(x * 1.4426950408889634);
    double r = fma(-k, 6.93147180369123816490e-01, x);
    r = fma(-k, 1.90821492927058770002e-10, r);
    double q = kExpTaylor[13];
#pragma unroll
    for (int i = 12; i >= 0; --i) q = fma(q, r, kExpTaylor[i]);
    return q * __longlong_as_double((long long)(1023 + (int)k) << 52);
}

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
    const double* ctab;    // per-direction coefficient factor tables (TRIG_SEP, FOURIER_LOGN) or null
    int cw;                // doubles per node in ctab
    const int64_t* rows_list;   // if set: assemble only these rows (global ids inside the range)
    int64_t nlist;
    // matrix-free mode (wgq_apply): instead of storing row i, y[i] = sum_j A_ij u[j - u_row0]
    int apply;
    const double* u;
    int64_t u_row0;
    double* yM;
    double* yK;
    // load-vector mode (wgq_assemble_load through k_fourier2d): b[i] = sum of the row's weighted mass samples
    int load;
    double* b;
    int64_t n, N;               // direction 0 (all directions on an isotropic mesh)
    RowTables T3[3];            // per-direction tables (= T when isotropic)
    Dims dims;                  // per-direction sizes
    int64_t ctabN;              // row stride of ctab (max N over the directions)
    int64_t row_begin, row_end;
    // k_fourier2d frame mode: skip the rows with both indices in [frame_lo, frame_hi] (done by
    // the interior kernel of fourier2d.cu); off when frame == 0
    int frame, frame_lo, frame_hi;
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
    const double* ct;  // [m][cw] coefficient factors at the nodes (ctab), or null
};

// Coefficient factor tables (a3 without per-sample transcendentals): for direction a, node
// kind (mass / stiffness), 1D row r and node k,
//   TRIG_SEP:     F = trig_a(2 pi k_a x)                                  (cw = 1)
//   FOURIER_LOGN: (C, S)_m = (cos, sin)(2 pi k_{m,a} x + [a = 0] theta_m) * ([a = 0] ? a_m : 1)
// so that c = c0 + amp prod_a F_a, resp. c = exp(sum_m Re prod_a (C + i S)_m): the angle-sum
// expansion of cos(2 pi k_m . x + theta_m) (R13), exact up to rounding.
// cos / sin of the mode phases theta_m, computed once on the host (they fold into direction 0's
// factors: a_m cos(2 pi k x + theta) = a_m (cos(2 pi k x) cos theta - sin(2 pi k x) sin theta))
struct PhaseTab {
    double c[WGQ_MAX_MODES], s[WGQ_MAX_MODES];
};

__global__ void k_coef_tables(const CoefDev c, const PhaseTab ph, int dim, const RowTables T3a, const RowTables T3b,
                              const RowTables T3c, int64_t ctabN, double* tab, int cw) {
    // one thread per (table entry, mode) (FOURIER; one per entry for TRIG_SEP): the modes of an
    // entry are independent, and a warp writes 32 consecutive 16-byte column pairs.  Every slot is
    // written (zeros for node slots beyond the rule and rows beyond the direction's count).
    const int nq = c.kind == WGQ_COEF_FOURIER_LOGN && c.n_modes > 0 ? c.n_modes : 1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t e = tid / nq;
    const int q = (int)(tid % nq);
    const int64_t per_ak = ctabN * kMaxNodes;
    const int64_t ak = e / per_ak;
    if (ak >= 2 * dim) return;
    const int a = (int)(ak / 2), kind = (int)(ak % 2);
    const RowTables& T = a == 0 ? T3a : (a == 1 ? T3b : T3c);     // direction a's rows
    const int64_t r = (e % per_ak) / kMaxNodes;
    const int k = (int)(e % kMaxNodes);
    const bool live = r < T.N && k < (kind == WGQ_MASS ? T.mM[r] : T.mK[r]);
    double* out = tab + e * cw;
    if (c.kind != WGQ_COEF_FOURIER_LOGN || c.n_modes == 0) {         // TRIG_SEP (cw = 1) or no modes
        double v = 0.0;
        if (live && c.kind == WGQ_COEF_TRIG_SEP) {
            const double arg = 2.0 * (double)c.wavenum[a] * (kind == WGQ_MASS ? T.xM : T.xK)[r * kMaxNodes + k];
            v = c.trig[a] == WGQ_TRIG_SIN ? sinpi(arg) : cospi(arg);       // trig(pi * arg)
        }
        out[0] = v;
        return;
    }
    double cp = 0.0, sp = 0.0;
    if (live) {
        const double x = (kind == WGQ_MASS ? T.xM : T.xK)[r * kMaxNodes + k];
        const double arg = 2.0 * c.modes[q][1 + a] * x;
        cp = cospi(arg), sp = sinpi(arg);
        if (a == 0) {
            const double ct = ph.c[q], st = ph.s[q];
            const double cc = cp * ct - sp * st, ss = sp * ct + cp * st;
            cp = c.modes[q][0] * cc;
            sp = c.modes[q][0] * ss;
        }
    }
    out[2 * q] = cp;
    out[2 * q + 1] = sp;
}

template <int D>
__device__ __forceinline__ double coef_from_tables(const CoefDev& c, const double* f1, const double* f2,
                                                   const double* f3) {
    if (c.kind == WGQ_COEF_TRIG_SEP) {
        double prod = f1[0];
        if (D > 1) prod *= f2[0];
        if (D > 2) prod *= f3[0];
        return c.c0 + c.amp * prod;
    }
    double s = 0.0;
    for (int q = 0; q < c.n_modes; ++q) {
        const double C1 = f1[2 * q], S1 = f1[2 * q + 1];
        if (D == 1) {
            s += C1;
        } else if (D == 2) {
            s += C1 * f2[2 * q] - S1 * f2[2 * q + 1];
        } else {
            const double C2 = f2[2 * q], S2 = f2[2 * q + 1], C3 = f3[2 * q], S3 = f3[2 * q + 1];
            s += C1 * (C2 * C3 - S2 * S3) - S1 * (S2 * C3 + C2 * S3);
        }
    }
    return exp(s);
}

template <int D>
__device__ __forceinline__ void stage_term(const GenericArgs& a, const Dir d1, const Dir d2, const Dir d3,
                                           int S1, int S2, int S3, double* W, double* T1, double* T2,
                                           bool accumulate, int lane) {
    const int n1 = d1.m, n2 = d2.m, n3 = d3.m;
    // a3-a4: weighted coefficient samples on the node tensor
    for (int e = lane; e < n1 * n2 * n3; e += 32) {
        const int k3 = e % n3, k2 = (e / n3) % n2, k1 = e / (n3 * n2);
        double cv;
        if (a.ctab) {
            cv = coef_from_tables<D>(a.coef, d1.ct + k1 * a.cw, d2.ct + k2 * a.cw, d3.ct + k3 * a.cw);
        } else {
            double x[3] = {d1.x[k1], d2.x[k2], d3.x[k3]};
            cv = coef_eval<D>(a.coef, a.dims.n, x);
        }
        W[e] = cv * d1.w[k1] * d2.w[k2] * d3.w[k3];
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
    const uint64_t pol = pol_evict_first();
    double* W = smem + warp * a.sg.per_warp;
    double* T1 = W + a.sg.w;
    double* T2 = T1 + a.sg.t1;
    double* T2b = T2 + a.sg.t2;
    const Dir ones = {1, kOnes, kOnes, kOnes, kOnes};

    const int64_t nwork = a.rows_list ? a.nlist : a.row_end - a.row_begin;
    for (int64_t w = (int64_t)blockIdx.x * warps + warp; w < nwork; w += (int64_t)gridDim.x * warps) {
        const int64_t row = a.rows_list ? a.rows_list[w] : a.row_begin + w;
        int64_t idx[3];
        a.dims.decode(row, idx);
        Dir dm[3], dk[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (q < D) {
                const RowTables& T = a.T3[q];
                const int64_t r = idx[q];
                const double* cm = a.ctab ? a.ctab + ((int64_t)(2 * q + WGQ_MASS) * a.ctabN + r) * kMaxNodes * a.cw : nullptr;
                const double* ck = a.ctab ? a.ctab + ((int64_t)(2 * q + WGQ_STIFFNESS) * a.ctabN + r) * kMaxNodes * a.cw : nullptr;
                dm[q] = {T.mM[r], T.xM + r * kMaxMassNodes, T.wM + r * kMaxMassNodes, T.VM + r * kMaxMassNodes * kMaxS, cm};
                dk[q] = {T.mK[r], T.xK + r * kMaxStiffNodes, T.wK + r * kMaxStiffNodes, T.DK + r * kMaxStiffNodes * kMaxS, ck};
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
        if (a.apply) {
            // matrix-free: dot the row with u over its structural columns, reduce over the warp
            double pm = 0.0, pk = 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int slot = lane + 32 * j;
                if (slot >= NS) continue;
                const int o[3] = {slot % S1 - P, (slot / S1) % S2 - (D >= 2 ? P : 0), slot / (S1 * S2) - (D >= 3 ? P : 0)};
                int64_t col = 0, stride = 1;
                bool ok = true;
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    const int64_t jq = idx[q] + o[q];
                    ok = ok && jq >= 0 && jq < a.dims.N[q];
                    col += jq * stride;
                    stride *= a.dims.N[q];
                }
                if (!ok) continue;
                const double uj = __ldg(a.u + (col - a.u_row0));
                pm = fma(accM[j], uj, pm);
                pk = fma(accK[j], uj, pk);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                pm += __shfl_xor_sync(0xffffffffu, pm, off);
                pk += __shfl_xor_sync(0xffffffffu, pk, off);
            }
            if (lane == 0) {
                if (a.yM) a.yM[orow] = pm;
                if (a.yK) a.yK[orow] = pk;
            }
            __syncwarp();
            continue;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int slot = lane + 32 * j;
            if (slot >= NS) continue;
            if (a.M.layout == WGQ_ELL) {
                if (a.do_mass) st_stream(a.M.values + orow * a.M.ld + slot, accM[j] + 0.0, pol);
                if (a.do_stiff) st_stream(a.K.values + orow * a.K.ld + slot, accK[j] + 0.0, pol);
            } else {
                // CSR: slot -> compacted position inside the box of valid offsets
                int o[3] = {slot % S1 - P, (slot / S1) % S2 - (D >= 2 ? P : 0), slot / (S1 * S2) - (D >= 3 ? P : 0)};
                int64_t pos = 0, stride = 1;
                bool ok = true;
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    const int64_t lo = idx[q] - P < 0 ? -idx[q] : -P;
                    const int64_t hi = idx[q] + P > a.dims.N[q] - 1 ? a.dims.N[q] - 1 - idx[q] : P;
                    if (o[q] < lo || o[q] > hi) ok = false;
                    pos += (o[q] - lo) * stride;
                    stride *= hi - lo + 1;
                }
                if (!ok) continue;
                if (a.do_mass) st_stream(a.M.values + a.M.row_ptr[orow] + pos, accM[j] + 0.0, pol);
                if (a.do_stiff) st_stream(a.K.values + a.K.row_ptr[orow] + pos, accK[j] + 0.0, pol);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// 2D FOURIER_LOGN fast path on the FP64 tensor cores (C3): one warp per row, ten DMMA m8n8k4.
//
// Row (i1, i2) samples c at its three node tensors (mass x mass for M; stiffness-x x mass-y and
// mass-x x stiffness-y for the two K terms).  With the factor tables (C, S)_m at the nodes
// (k_coef_tables), the exponent of every sample is a dot product over 2 n_modes:
//   E[x-node][y-node] = sum_m (C^x_m C^y_m - S^x_m S^y_m)          (the angle-sum expansion)
// computed for all 8 x-nodes (4 mass, 4 stiffness, interleaved: row 2k = mass node k, row
// 2k+1 = stiffness node k) against all 8 y-nodes (same interleave) in one 8 x 8 x 2n_modes
// DMMA chain.  Lane (g, t) then holds E for x-node g and y-nodes (mass t, stiffness t): with
// its weights it forms W_M (g even, mass y), W_Ky (g even, stiffness y) and W_Kx (g odd,
// mass y) — exactly the B fragment B[k = y-node t][n = x-node g] of the y-stage products
//   T^T_X = A2_X^T W_X^T      (A2 = B_{i2+o}(y) or B'_{i2+o}(y) at the y nodes)
// whose C fragment (lane (g, t): T^T[o2 = g][x-node column 2t (+1)]) is in turn exactly the B
// fragment of the x-stage products  M = A1^T T,  K = D1^T T_Kx + A1^T T_Ky  (a5, a6).
// Rows with more than 4 nodes in a direction (GL-fallback boundary classes, R1) are left to
// the generic kernel (shell pass).
constexpr int kF2dSeg = 32;   // rows of one x-line per work item (the y-side data is loaded once)

template <int P, int MODE, int KSMAX>
__global__ void __launch_bounds__(256) k_fourier2d(const GenericArgs a) {
    constexpr int S = 2 * P + 1;                        // KSMAX: k-steps of 4 over 2 n_modes
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const RowTables& T = a.T;
    const int cw = a.cw, J = 2 * a.coef.n_modes;
    const int N = (int)a.N;
    const bool gs = g & 1;                     // x-node of row g / y-node of column g: stiffness?
    const int kg = g >> 1;
    const int segs = (N + kF2dSeg - 1) / kF2dSeg;
    const int line0 = (int)(a.row_begin / N), line1 = (int)((a.row_end - 1) / N);
    // work items: (line, 32-row segment); in frame mode the lines with i2 in [frame_lo, frame_hi]
    // contribute only their two frame pieces x < frame_lo and x > frame_hi
    const int I0 = a.frame ? max(line0, a.frame_lo) : 1, I1 = a.frame ? min(line1, a.frame_hi) : 0;
    const int nI = I1 >= I0 ? I1 - I0 + 1 : 0;
    const int F0 = a.frame ? max(0, min(line1, a.frame_lo - 1) - line0 + 1) : line1 - line0 + 1;
    const int nF = line1 - line0 + 1 - nI;
    const int64_t items = (int64_t)nI * 2 + (int64_t)nF * segs;
    for (int64_t it = (int64_t)blockIdx.x * warps + warp; it < items; it += (int64_t)gridDim.x * warps) {
        int i2, x0, x1;
        if (it < (int64_t)nI * 2) {
            i2 = I0 + (int)(it >> 1);
            x0 = (it & 1) ? a.frame_hi + 1 : 0;
            x1 = (it & 1) ? N : a.frame_lo;
        } else {
            const int64_t f = (it - (int64_t)nI * 2) / segs;
            const int sg = (int)((it - (int64_t)nI * 2) % segs);
            i2 = f < F0 ? line0 + (int)f : max(line0, a.frame_hi + 1) + (int)(f - F0);
            x0 = sg * kF2dSeg;
            x1 = min(x0 + kF2dSeg, N);
        }
        x0 = max(x0, (int)(a.row_begin - (int64_t)i2 * N));
        x1 = min(x1, (int)min((int64_t)N, a.row_end - (int64_t)i2 * N));
        if (x0 >= x1) continue;
        // ---- y-side data of the line: counts, exponent B fragments, weights, y-stage A fragments
        const bool i2in = a.frame && a.frame_lo <= i2 && i2 <= a.frame_hi;
        const int nym = __ldg(T.mM + i2), nyk = __ldg(T.mK + i2);
        if (nym > 4 || nyk > 4) continue;                  // whole line in the generic shell pass
        const bool yv = kg < (gs ? nyk : nym);
        const double* Y = a.ctab + ((int64_t)(2 + (gs ? 1 : 0)) * N + i2) * kMaxNodes * cw + kg * cw;
        double yb[KSMAX];
#pragma unroll
        for (int s = 0; s < KSMAX; ++s) {
            const int j = 4 * s + t;
            double v = (yv && j < J) ? __ldg(Y + j) : 0.0;
            yb[s] = (j & 1) ? -v : v;
        }
        const double wym = t < nym ? __ldg(T.wM + i2 * kMaxNodes + t) : 0.0;
        const double wyk = t < nyk ? __ldg(T.wK + i2 * kMaxNodes + t) : 0.0;
        const double aVy = (g < S && t < nym) ? __ldg(T.VM + (i2 * kMaxNodes + t) * kMaxS + g) : 0.0;
        const double aDy = (g < S && t < nyk) ? __ldg(T.DK + (i2 * kMaxNodes + t) * kMaxS + g) : 0.0;
        const int64_t orow0 = (int64_t)i2 * N - a.row_begin;
        // x-side data of row i1, loaded one row ahead (the L2 latency of row i1+1's loads
        // overlaps row i1's tensor-core / exp chain)
        struct XData {
            int nxm, nxk;
            double xa[KSMAX], wx, aVx, aDx;
        };
        auto load_x = [&](int i1, XData& d) {
            d.nxm = __ldg(T.mM + i1);
            d.nxk = __ldg(T.mK + i1);
            const bool xv = kg < (gs ? d.nxk : d.nxm);
            const double* X = a.ctab + ((int64_t)(gs ? 1 : 0) * N + i1) * kMaxNodes * cw + kg * cw;
#pragma unroll
            for (int s = 0; s < KSMAX; ++s) {
                const int j = 4 * s + t;
                d.xa[s] = (4 * s < J && xv && j < J) ? __ldg(X + j) : 0.0;
            }
            d.wx = xv ? __ldg((gs ? T.wK : T.wM) + i1 * kMaxNodes + kg) : 0.0;
            d.aVx = (g < S && t < d.nxm) ? __ldg(T.VM + (i1 * kMaxNodes + t) * kMaxS + g) : 0.0;
            d.aDx = (g < S && t < d.nxk) ? __ldg(T.DK + (i1 * kMaxNodes + t) * kMaxS + g) : 0.0;
        };
        XData nx;
        if (x0 < x1) load_x(x0, nx);
        for (int i1 = x0; i1 < x1; ++i1) {
            const XData cx = nx;
            if (i1 + 1 < x1) load_x(i1 + 1, nx);
            if (cx.nxm > 4 || cx.nxk > 4) continue;        // generic shell pass
            if (i2in && i1 >= a.frame_lo && i1 <= a.frame_hi) continue;
            // ---- exponent GEMM: E[x-node g][y-node n] (B fragments of the line in yb) -------
            const bool xv = kg < (gs ? cx.nxk : cx.nxm);
            double e0 = 0.0, e1 = 0.0;
#pragma unroll
            for (int s = 0; s < KSMAX; ++s) {
                if (4 * s >= J) break;
                dmma(e0, e1, cx.xa[s], yb[s]);
            }
            if (a.load) {
                // load vector (eq:Load): the row's mass x mass samples, summed over the warp
                double v = (!gs && xv && t < nym) ? exp_fast(e0) * cx.wx * wym : 0.0;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) a.b[orow0 + i1] = v;
                continue;
            }
            // ---- weighted samples (lane (g, t): x-node g, y-nodes mass t / stiffness t) ----
            const double s0 = (xv && t < nym) ? exp_fast(e0) * cx.wx * wym : 0.0;
            const double s1 = (!gs && xv && t < nyk) ? exp_fast(e1) * cx.wx * wyk : 0.0;
            const double aVx = cx.aVx, aDx = cx.aDx;
            double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
            if (MODE & 1) {
                double tm0 = 0.0, tm1 = 0.0;
                dmma(tm0, tm1, aVy, gs ? 0.0 : s0);      // T_M^T: lane holds [o2 = g][x mass t] in tm0
                dmma(m0, m1, aVx, tm0);                   // M = A1^T T_M
            }
            if (MODE & 2) {
                double tx0 = 0.0, tx1 = 0.0, ty0 = 0.0, ty1 = 0.0;
                dmma(tx0, tx1, aVy, gs ? s0 : 0.0);      // T_Kx^T: [o2 = g][x stiffness t] in tx1
                dmma(ty0, ty1, aDy, gs ? 0.0 : s1);      // T_Ky^T: [o2 = g][x mass t] in ty0
                dmma(k0, k1, aDx, tx1);                   // K = D1^T T_Kx + A1^T T_Ky
                dmma(k0, k1, aVx, ty0);
            }
            // ---- store: lane holds (o1 = g, o2 = 2t + i) ---------------------------------------
            const int64_t orow = orow0 + i1;
            if (a.apply) {
                // matrix-free: y_i = sum over the lane's two columns of A_ij u_j, warp-reduced
                double pm = 0.0, pk = 0.0;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int o2 = 2 * t + i;
                    const int j1 = i1 + g - P, j2 = i2 + o2 - P;
                    if (g >= S || o2 >= S || j1 < 0 || j1 >= N || j2 < 0 || j2 >= N) continue;
                    const double uj = __ldg(a.u + ((int64_t)j2 * N + j1 - a.u_row0));
                    pm = fma(i ? m1 : m0, uj, pm);
                    pk = fma(i ? k1 : k0, uj, pk);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    pm += __shfl_xor_sync(0xffffffffu, pm, off);
                    pk += __shfl_xor_sync(0xffffffffu, pk, off);
                }
                if (lane == 0) {
                    if (MODE & 1) a.yM[orow] = pm;
                    if (MODE & 2) a.yK[orow] = pk;
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int o2 = 2 * t + i;
                if (g >= S || o2 >= S) continue;
                const double vm = (i ? m1 : m0) + 0.0, vk = (i ? k1 : k0) + 0.0;
                if (a.M.layout == WGQ_ELL) {
                    if (MODE & 1) a.M.values[orow * a.M.ld + g + S * o2] = vm;
                    if (MODE & 2) a.K.values[orow * a.K.ld + g + S * o2] = vk;
                } else {
                    const int lo1 = i1 - P < 0 ? -i1 : -P, hi1 = i1 + P > N - 1 ? N - 1 - i1 : P;
                    const int lo2 = i2 - P < 0 ? -i2 : -P, hi2 = i2 + P > N - 1 ? N - 1 - i2 : P;
                    if (g - P < lo1 || g - P > hi1 || o2 - P < lo2 || o2 - P > hi2) continue;
                    const int64_t pos = (g - P - lo1) + (int64_t)(o2 - P - lo2) * (hi1 - lo1 + 1);
                    if (MODE & 1) a.M.values[a.M.row_ptr[orow] + pos] = vm;
                    if (MODE & 2) a.K.values[a.K.row_ptr[orow] + pos] = vk;
                }
            }
        }
    }
}

template <int P>
int launch_fourier2d_p(const GenericArgs& a, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t segs = (a.N + kF2dSeg - 1) / kF2dSeg;
    const int64_t lines = (a.row_end - 1) / a.N - a.row_begin / a.N + 1;
    // (frame mode: most lines have only 2 short pieces; the grid only needs to cover the items)
    const int64_t items = a.frame ? std::min<int64_t>(lines * segs, 2 * lines + (int64_t)(a.N - (a.frame_hi - a.frame_lo + 1)) * segs)
                                  : lines * segs;
    int64_t blocks = std::min<int64_t>((items + 7) / 8, (int64_t)sms * 32);
    blocks = std::max<int64_t>(blocks, 1);
    const int mode = (a.do_mass ? 1 : 0) | (a.do_stiff ? 2 : 0);
    if (a.coef.n_modes <= 8) {
        if (mode == 3) k_fourier2d<P, 3, 4><<<(unsigned)blocks, 256, 0, st>>>(a);
        else if (mode == 1) k_fourier2d<P, 1, 4><<<(unsigned)blocks, 256, 0, st>>>(a);
        else k_fourier2d<P, 2, 4><<<(unsigned)blocks, 256, 0, st>>>(a);
    } else {
        if (mode == 3) k_fourier2d<P, 3, 8><<<(unsigned)blocks, 256, 0, st>>>(a);
        else if (mode == 1) k_fourier2d<P, 1, 8><<<(unsigned)blocks, 256, 0, st>>>(a);
        else k_fourier2d<P, 2, 8><<<(unsigned)blocks, 256, 0, st>>>(a);
    }
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
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
    const int64_t rows = a.rows_list ? a.nlist : a.row_end - a.row_begin;
    if (rows <= 0) return WGQ_OK;
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

// ---------------------------------------------------------------------------------------------
// Load vector (eq:Load): b_i = sum_k [prod_a w^M_{i_a,k_a}] f(x^M_k),
// row i's mass-kind rule applied to f.  One thread per row.
//  * GRID f (multilinear, R6): with PW[r][v] = sum_k w^M_k lambda_v(x_k) = sum_o PM[r][v][o]
//    (partition of unity), b_i = sum_v g[bz+vz][by+vy][bx+vx] prod_a PW_a[v_a] — the same sum
//    reordered (vertex projection, as in the line kernel).
//  * analytic f: the node-tensor sum with the coefficient factor tables (or c0).
// per-direction vertex weights PW (RowTables::PW, built with the row tables), passed as one
// pointer per direction
struct PW3 {
    const double* d[3];
};

template <int P, int D>
__global__ void __launch_bounds__(256) k_load(const GenericArgs a, const PW3 PW, double* b) {
    constexpr int V = P + 2;
    const int64_t rows = a.rows_list ? a.nlist : a.row_end - a.row_begin;   // rows_list: a shell pass
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = a.rows_list ? a.rows_list[t] : a.row_begin + t;
        int64_t idx[3];
        a.dims.decode(row, idx);
        double acc = 0.0;
        if (a.coef.kind == WGQ_COEF_GRID) {
            // vertex planes of (n_y+1) x (n_x+1)
            const int64_t nvx = a.dims.n[0] + 1, nvy = D >= 2 ? a.dims.n[1] + 1 : 1;
            const double* const* PWq = PW.d;
            int64_t base[3];
#pragma unroll
            for (int q = 0; q < D; ++q) base[q] = idx[q] - P > 0 ? idx[q] - P : 0;
            const int Vz = D >= 3 ? V : 1, Vy = D >= 2 ? V : 1;
            for (int vz = 0; vz < Vz; ++vz) {
                const double wz = D >= 3 ? PWq[2][idx[2] * kMaxV + vz] : 1.0;
                for (int vy = 0; vy < Vy; ++vy) {
                    const double wy = D >= 2 ? PWq[1][idx[1] * kMaxV + vy] : 1.0;
                    const int64_t zz = D >= 3 ? base[2] + vz : 0, yy = D >= 2 ? base[1] + vy : 0;
                    const int64_t zrow = D == 3 ? zz : (D == 2 ? yy : 0);
                    if (wz * wy == 0.0 || (D >= 3 && zz > a.dims.n[2]) || (D >= 2 && yy > a.dims.n[1])) continue;
                    double sx = 0.0;
#pragma unroll
                    for (int vx = 0; vx < V; ++vx) {
                        const int64_t xx = base[0] + vx;
                        const double wx = PWq[0][idx[0] * kMaxV + vx];
                        if (wx == 0.0 || xx > a.dims.n[0]) continue;
                        const double* g;
                        if (D == 1) g = a.coef.grid + (xx - a.coef.plane0);
                        else if (D == 2) g = a.coef.grid + (zrow - a.coef.plane0) * nvx + xx;
                        else g = a.coef.grid + ((zz - a.coef.plane0) * nvy + yy) * nvx + xx;
                        sx = fma(wx, __ldg(g), sx);
                    }
                    acc = fma(wz * wy, sx, acc);
                }
            }
        } else {
            const RowTables& T1 = a.T3[0];
            const RowTables& T2 = a.T3[1];
            const RowTables& T3 = a.T3[2];
            const int n1 = T1.mM[idx[0]], n2 = D >= 2 ? T2.mM[idx[1]] : 1, n3 = D >= 3 ? T3.mM[idx[2]] : 1;
            for (int k3 = 0; k3 < n3; ++k3) {
                const double w3 = D >= 3 ? T3.wM[idx[2] * kMaxMassNodes + k3] : 1.0;
                for (int k2 = 0; k2 < n2; ++k2) {
                    const double w2 = D >= 2 ? T2.wM[idx[1] * kMaxMassNodes + k2] : 1.0;
                    for (int k1 = 0; k1 < n1; ++k1) {
                        const double w1 = T1.wM[idx[0] * kMaxMassNodes + k1];
                        double cv = a.coef.c0;
                        if (a.ctab) {
                            const int64_t k[3] = {k1, k2, k3};
                            const double* f[3];
#pragma unroll
                            for (int q = 0; q < 3; ++q)
                                f[q] = q < D ? a.ctab + ((int64_t)(2 * q + WGQ_MASS) * a.ctabN + idx[q]) * kMaxNodes * a.cw +
                                                   k[q] * a.cw
                                             : nullptr;
                            cv = coef_from_tables<D>(a.coef, f[0], f[1], f[2]);
                        }
                        acc = fma(w1 * w2 * w3, cv, acc);
                    }
                }
            }
        }
        b[row - a.row_begin] = acc;
    }
}

// GRID load vector on the line structure (D = 2, 3): a warp takes 32 consecutive rows of one
// x-line; lane l first forms G[c] = sum_{vy,vz} g[bz+vz][by+vy][c] PWy[vy] PWz[vz] for the
// vertex planes c = c0 + l (+32) of the segment (coalesced loads along x), then row i1 = x0 + l
// gathers b = sum_vx PWx[i1][vx] G[bx+vx] from its neighbours' registers (warp shuffles).
template <int P, int D>
__global__ void __launch_bounds__(256) k_load_grid_line(const GenericArgs a, const PW3 PW3d, double* b) {
    const double* PW = PW3d.d[0];   // isotropic mesh (the launcher)
    constexpr int V = P + 2;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t N = a.N, nv = a.n + 1;
    const int64_t segs = (N + 31) / 32;
    const int64_t line0 = a.row_begin / N, line1 = (a.row_end - 1) / N;
    const int64_t items = (line1 - line0 + 1) * segs;
    for (int64_t it = warp; it < items; it += nwarps) {
        const int64_t line = line0 + it / segs;
        const int64_t x0 = (it % segs) * 32;
        const int64_t i2 = line % N, i3 = D >= 3 ? line / N : 0;
        const int64_t by = max((int64_t)0, i2 - P), bz = max((int64_t)0, i3 - P);
        const int64_t c0 = max((int64_t)0, x0 - P);
        double G[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = c0 + lane + 32 * h;
            double acc = 0.0;
            if (c <= a.n && (h == 0 || lane < V - 1)) {      // the segment's planes c0 .. c0+31+V-1
                // all V (x V) loads issued before the sums (fully unrolled, predicated)
                double gv[D >= 3 ? V : 1][V];
#pragma unroll
                for (int vz = 0; vz < (D >= 3 ? V : 1); ++vz) {
                    const int64_t z = bz + vz;
#pragma unroll
                    for (int vy = 0; vy < V; ++vy) {
                        const int64_t y = by + vy;
                        const bool ok = y <= a.n && (D < 3 || z <= a.n);
                        const double* g = D >= 3 ? a.coef.grid + ((z - a.coef.plane0) * nv + y) * nv + c
                                                 : a.coef.grid + (y - a.coef.plane0) * nv + c;
                        gv[vz][vy] = ok ? __ldg(g) : 0.0;
                    }
                }
#pragma unroll
                for (int vz = 0; vz < (D >= 3 ? V : 1); ++vz) {
                    double sy = 0.0;
#pragma unroll
                    for (int vy = 0; vy < V; ++vy) sy = fma(PW[i2 * kMaxV + vy], gv[vz][vy], sy);
                    acc = fma(D >= 3 ? PW[i3 * kMaxV + vz] : 1.0, sy, acc);
                }
            }
            G[h] = acc;
        }
        const int64_t i1 = x0 + lane;
        const int64_t row = line * N + i1;
        const bool mine = i1 < N && row >= a.row_begin && row < a.row_end;
        const int64_t bx = max((int64_t)0, i1 - P);
        double acc = 0.0;
#pragma unroll
        for (int vx = 0; vx < V; ++vx) {
            const int src = (int)(bx + vx - c0);                       // 0 .. 35
            const double g0 = __shfl_sync(0xffffffffu, G[0], src & 31);
            const double g1 = __shfl_sync(0xffffffffu, G[1], src & 31);
            const double wx = mine ? PW[i1 * kMaxV + vx] : 0.0;
            acc = fma(wx, src < 32 ? g0 : g1, acc);
        }
        if (mine) b[row - a.row_begin] = acc;
    }
}

// 3D GRID load vector, pencil kernel (round 2): the same sum b = sum PW_z PW_y PW_x g, contracted
// y -> z -> x with every stage in registers except the x halo.  A work column is kLPW lines i2
// (one per warp) x one x chunk of XO rows; a block slides along i3 through a contiguous range of
// output planes of one or two columns (the flattened (column, plane) range split evenly over a
// persistent grid, segments of at most kLPSEG planes).  Lane t owns R consecutive vertex columns
// c = x0 - P + R t + j (j < R) of its warp's line and the rows i1 = x0 + R t + j, each summed over
// its natural window, columns i1 - P .. i1 + 1:
//   y: q_z[j] = sum_vy PW_y[i2][vy] g[z][by + vy][c_j]     (vertex plane z from the smem ring)
//   z: s[j]   = sum_v Wn_z[i3][v] q_{i3-P+v}[j]            (a V-deep register ring, the z loop
//                                                            unrolled; i3 = z - 1 ends at plane z)
//   x: b[i1_j] = sum_v Wn_x[i1_j][v] s[j + v]              (the V - 1 columns past the lane's own
//                                                            come from lanes t + 1 .. by shuffles)
// Wn[r][v] = PW[r][v - sh], sh = max(0, P - r): a row r < P has window 0 .. V-1 (b_r = 0), but its
// basis function lives on elements 0 .. r, so PW[r][v] = 0 for v > r + 1 and the natural window
// r - P .. r + 1 (vertices < 0 read as zero) carries all of its terms.  The grid tile of each
// vertex plane (kLPW + V - 1 rows x 32 R columns; out-of-mesh elements zero-filled) streams
// through a shared-memory ring by 8-byte cp.async, 2 kLPA2 planes ahead; one block barrier per
// two vertex planes (their y stages and output planes are independent: ILP for the FP64 chains).
constexpr int kLPW = 8;        // warps (= lines) per block
constexpr int kLPR = 3;        // vertex columns / rows i1 per lane
constexpr int kLPA2 = 2;       // plane pairs in flight ahead (3: 0.084 ms at C5, 2: 0.081, 1: 0.083)
constexpr int kLPRR = 8;       // raw ring depth (power of two >= 2 kLPA2 + 2)
constexpr int kLPSEG = 96;     // output planes per segment (bounds the staged z weights)
static_assert(kLPRR >= 2 * kLPA2 + 2 && (kLPRR & (kLPRR - 1)) == 0, "load pencil raw ring depth");

template <int P>
struct LoadPencil {
    static constexpr int V = P + 2;
    static constexpr int R = kLPR;
    static constexpr int HL = (V - 1 + R - 1) / R;   // halo lanes
    static constexpr int XO = (32 - HL) * R;         // rows i1 per x chunk
    static constexpr int TW = 32 * R;                // tile columns
    static constexpr int TR = kLPW + V - 1;          // tile rows
    static constexpr int TILE = TR * TW;
    static constexpr int UN = V % 2 == 0 ? V : 2 * V; // z unroll: whole ring turns, whole plane pairs
    static constexpr size_t smem = (size_t)(kLPRR * TILE + kLPSEG * V) * sizeof(double);
};

template <int P>
__global__ void __launch_bounds__(kLPW * 32, 2) k_load_grid_pencil(const GenericArgs a, const PW3 PW, double* b,
                                                                   int dbg) {
    using LP = LoadPencil<P>;
    constexpr int V = LP::V, R = LP::R, HL = LP::HL, XO = LP::XO, TW = LP::TW, TR = LP::TR, TILE = LP::TILE,
                  UN = LP::UN;
    constexpr int NT = kLPW * 32, LPT = (TILE + NT - 1) / NT;
    extern __shared__ __align__(16) double lp_smem[];
    double* raw = lp_smem;                          // [kLPRR][TR][TW] vertex planes
    double* swz = raw + kLPRR * TILE;               // [kLPSEG][V] natural-window z weights of the segment
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // 32-bit indices: the launcher requires N^3 < 2^31
    const int N = (int)a.N, n = (int)a.n, nv = n + 1;
    const int64_t pr = (int64_t)N * N;
    const double* PWx = PW.d[0];
    const double* PWy = PW.d[1];
    const double* PWz = PW.d[2];
    const int zlo_all = (int)(a.row_begin / pr), zhi_all = (int)((a.row_end - 1) / pr);
    const int Zc = zhi_all - zlo_all + 1;
    const int nxc = (N + XO - 1) / XO, ncol = nxc * ((N + kLPW - 1) / kLPW);
    const int64_t total = (int64_t)ncol * Zc;
    const int64_t f1 = total * (blockIdx.x + 1) / gridDim.x;
    const int zg0 = (int)a.coef.plane0, zg1 = min((int)(a.coef.plane0 + a.coef.planes), n + 1);
    const int plane_el = nv * nv;
    const int64_t nrows = a.row_end - a.row_begin;
    for (int64_t f = total * blockIdx.x / gridDim.x; f < f1;) {
        // segment: column col, output planes [z_lo, z_hi)
        const int col = (int)(f / Zc);
        const int z_lo = zlo_all + (int)(f % Zc);
        const int z_hi = (int)min(min((int64_t)zlo_all + Zc, z_lo + (f1 - f)), (int64_t)z_lo + kLPSEG);
        f += z_hi - z_lo;
        const int x0 = (col % nxc) * XO, y0 = (col / nxc) * kLPW;
        const int by0 = max(0, y0 - P);
        const int zs = max(0, z_lo - P);
        const int zend = z_hi;                        // output i3 ends at plane i3 + 1
        for (int t = tid; t < (z_hi - z_lo) * V; t += NT) {
            const int i3 = z_lo + t / V, v = t % V, sh = max(0, P - i3);
            swz[t] = v >= sh ? __ldg(PWz + (int64_t)i3 * kMaxV + v - sh) : 0.0;
        }
        // load roles: tile element e = tid + NT m -> (row by0 + e / TW, column x0 - P + e % TW);
        // out-of-mesh elements are zero-filled (source size 0)
        int goff[LPT];
        uint32_t sdst[LPT];
#pragma unroll
        for (int m = 0; m < LPT; ++m) {
            const int e = tid + NT * m;
            const int y = by0 + e / TW, x = x0 - P + e % TW;
            const bool ok = e < TILE && y <= n && x >= 0 && x <= n;
            goff[m] = ok ? y * nv + x : -1;
            sdst[m] = (uint32_t)__cvta_generic_to_shared(raw + (e < TILE ? e : 0));
        }
        auto issue1 = [&](int z) {
            if (z <= zend) {
                const uint32_t so = (uint32_t)((z & (kLPRR - 1)) * TILE * sizeof(double));
                const bool have = z >= zg0 && z < zg1;
                const double* gz = a.coef.grid + (have ? (int64_t)(z - zg0) * plane_el : 0);
#pragma unroll
                for (int m = 0; m < LPT; ++m) {
                    if (TILE % NT != 0 && tid + NT * m >= TILE) break;
                    const bool ok = have && goff[m] >= 0;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sdst[m] + so),
                                 "l"(gz + (ok ? goff[m] : 0)), "r"(ok ? 8 : 0)
                                 : "memory");
                }
            }
        };
        auto issue2 = [&](int z) {                   // planes z, z + 1: one commit group (possibly empty)
            issue1(z);
            issue1(z + 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // this warp's line and the lane's rows
        const int i2 = y0 + warp;
        const bool lok = i2 < N;
        const int by = max(0, i2 - P);
        double wy[V];
#pragma unroll
        for (int v = 0; v < V; ++v) wy[v] = lok ? __ldg(PWy + (int64_t)i2 * kMaxV + v) : 0.0;
        double wx[R][V];
        bool xok[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int i1 = x0 + R * lane + j, sh = max(0, P - i1);
            xok[j] = lok && lane < 32 - HL && i1 < N;
#pragma unroll
            for (int v = 0; v < V; ++v) wx[j][v] = xok[j] && v >= sh ? __ldg(PWx + (int64_t)i1 * kMaxV + v - sh) : 0.0;
        }
        const double* rd = raw + (by - by0) * TW + R * lane;
        const int64_t rel0 = (int64_t)i2 * N + x0 + R * lane - a.row_begin;   // row (i3 = 0, i1 = x0 + R lane) - row_begin
        const bool all_in = (int64_t)z_lo * pr >= a.row_begin && (int64_t)z_hi * pr <= a.row_end;
        auto ystage = [&](double (&q)[R], int z) {
            const double* rz = rd + (z & (kLPRR - 1)) * TILE;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                q[j] = wy[0] * rz[j];
#pragma unroll
                for (int v = 1; v < V; ++v) q[j] = fma(wy[v], rz[v * TW + j], q[j]);
            }
        };
        // output plane i3 whose window ends at plane z = i3 + 1 (its V planes are the ring slots
        // (u + 1 + v) mod V, u = the slot of plane z)
        auto output = [&](const double (&qr)[V][R], int u, int i3) {
            const double* wz = swz + (i3 - z_lo) * V;
            double s[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                s[j] = wz[0] * qr[(u + 1) % V][j];
#pragma unroll
                for (int v = 1; v < V; ++v) s[j] = fma(wz[v], qr[(u + 1 + v) % V][j], s[j]);
            }
            double sl[R + V - 1];
#pragma unroll
            for (int j = 0; j < R; ++j) sl[j] = s[j];
#pragma unroll
            for (int k = 0; k < V - 1; ++k) sl[R + k] = __shfl_down_sync(0xffffffffu, s[k % R], 1 + k / R);
            double out[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                out[j] = wx[j][0] * sl[j];
#pragma unroll
                for (int v = 1; v < V; ++v) out[j] = fma(wx[j][v], sl[j + v], out[j]);
            }
            const int64_t rel = rel0 + (int64_t)i3 * pr;
            double* bo = b + rel;
            if (dbg & 1) {
                if (out[0] == 1.2345) bo[0] = out[1] + out[2];
            } else if (all_in) {
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (xok[j]) bo[j] = out[j];
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (xok[j] && rel + j >= 0 && rel + j < nrows) bo[j] = out[j];
            }
        };
        double qr[V][R];
#pragma unroll
        for (int u = 0; u < V; ++u)
#pragma unroll
            for (int j = 0; j < R; ++j) qr[u][j] = 0.0;
        for (int k = 0; k < kLPA2; ++k) issue2(zs + 2 * k);
        for (int zb = zs; zb <= zend; zb += UN) {
#pragma unroll
            for (int u = 0; u < UN; u += 2) {
                const int z = zb + u;
                if (z > zend) break;
                asm volatile("cp.async.wait_group %0;" ::"n"(kLPA2 - 1) : "memory");
                __syncthreads();                      // planes z, z+1 landed; the slots of z-2, z-1 are free
                issue2(z + 2 * kLPA2);
                if (dbg & 2) continue;
                // planes outside the grid slab are zero-filled; plane z + 1 > zend is never output.
                // Plane z + 1 takes the ring slot of plane z + 1 - V, the first plane of output
                // z - 1's window: that output is formed first.
                ystage(qr[u % V], z);
                if (z - 1 >= z_lo && z - 1 < z_hi) output(qr, u % V, z - 1);
                ystage(qr[(u + 1) % V], z + 1);
                if (z >= z_lo && z < z_hi) output(qr, (u + 1) % V, z);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();                              // the ring is reused by the next segment
    }
}

template <int P, int D>
int launch_load_pd(const GenericArgs& a, const PW3& PW, double* b, bool special, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t rows = a.row_end - a.row_begin;
    if (special && D == 3 && a.coef.kind == WGQ_COEF_GRID && a.N * a.N * a.N < ((int64_t)1 << 31)) {
        const int64_t pr = a.N * a.N;
        const int64_t planes = (a.row_end - 1) / pr - a.row_begin / pr + 1;
        {
            using LP = LoadPencil<P>;
            if (cudaFuncSetAttribute(k_load_grid_pencil<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)LP::smem) != cudaSuccess)
                return WGQ_ECUDA;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_load_grid_pencil<P>, kLPW * 32, LP::smem);
            const int64_t ncol = ((a.N + LP::XO - 1) / LP::XO) * ((a.N + kLPW - 1) / kLPW);
            const int64_t work = ncol * planes;
            // persistent: one wave, each block >= 16 output planes of work
            const int64_t nb = std::max<int64_t>(std::max<int64_t>(1, (work + kLPSEG - 1) / kLPSEG),
                                                 std::min<int64_t>((int64_t)std::max(per_sm, 1) * sms, work / 16));
            static const int dbg = [] {
                const char* e = getenv("WGQ_LOAD_DBG");
                return e ? atoi(e) : 0;
            }();
            static const int nb_env = [] {
                const char* e = getenv("WGQ_LOAD_NB");
                return e ? atoi(e) : 0;
            }();
            k_load_grid_pencil<P><<<(unsigned)(nb_env > 0 ? nb_env : nb), kLPW * 32, LP::smem, st>>>(a, PW, b, dbg);
            return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
        }
    }
    if (special && D >= 2 && a.coef.kind == WGQ_COEF_GRID) {
        const int64_t items = ((a.row_end - 1) / a.N - a.row_begin / a.N + 1) * ((a.N + 31) / 32);
        const int64_t b2 = std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, (int64_t)sms * 16));
        k_load_grid_line<P, D><<<(unsigned)b2, 256, 0, st>>>(a, PW, b);
        return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
    }
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)sms * 16));
    k_load<P, D><<<(unsigned)blocks, 256, 0, st>>>(a, PW, b);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

// coefficient factor tables for an analytic kind (stream-ordered scratch) or nullptr
// Coefficient factor tables (stream-ordered scratch the caller frees): [2 dim][ctabN][kMaxNodes][cw],
// unused node slots zero (written by k_coef_tables; the 2D kernels read 4 nodes per row and weigh
// the missing ones by 0).
int coef_tables(const wgq_rules_s* R, GenericArgs& a, const wgq_coeff_t* c, cudaStream_t st, double** tab) {
    *tab = nullptr;
    if (c->kind != WGQ_COEF_TRIG_SEP && c->kind != WGQ_COEF_FOURIER_LOGN) return WGQ_OK;
    a.cw = c->kind == WGQ_COEF_TRIG_SEP ? 1 : 2 * a.coef.n_modes;
    if (a.cw == 0) a.cw = 1;
    const int64_t entries = 2 * (int64_t)R->dim * a.ctabN * kMaxNodes;
    if (cudaMallocAsync((void**)tab, (size_t)entries * a.cw * sizeof(double), st) != cudaSuccess) return WGQ_ENOMEM;
    const int64_t threads = entries * (c->kind == WGQ_COEF_FOURIER_LOGN && a.coef.n_modes > 0 ? a.coef.n_modes : 1);
    PhaseTab ph{};
    for (int q = 0; q < a.coef.n_modes && q < WGQ_MAX_MODES; ++q) {
        ph.c[q] = std::cos(a.coef.modes[q][4]);
        ph.s[q] = std::sin(a.coef.modes[q][4]);
    }
    k_coef_tables<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a.coef, ph, R->dim, a.T3[0], a.T3[1], a.T3[2],
                                                                      a.ctabN, *tab, a.cw);
    a.ctab = *tab;
    return WGQ_OK;
}

int64_t max_rows_1d(const wgq_rules_s* R) {
    int64_t m = 0;
    for (int a = 0; a < R->dim; ++a) m = std::max<int64_t>(m, R->dims.N[a]);
    return m;
}

void set_dirs(GenericArgs& a, const wgq_rules_s* R, const Tables3& TT) {
    a.T = TT.t[0];
    for (int q = 0; q < 3; ++q) a.T3[q] = TT.t[q];
    a.dims = R->dims;
    a.ctabN = max_rows_1d(R);
    a.n = R->n;
    a.N = R->N;
}

GenericArgs base_args(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, int64_t row_begin,
                      int64_t row_end) {
    GenericArgs a{};
    set_dirs(a, R, TT);
    a.coef = make_coef(c);
    a.row_begin = row_begin;
    a.row_end = row_end;
    return a;
}

}  // namespace

// The 2D shell rows of [row_begin, row_end): rows whose line i2 or column i1 is a "wide" 1D row
// (a GL-fallback boundary class with more than 4 nodes, R1), in row order.  Per line l the rows
// are the whole line (wide l) or its wide columns; with the nw <= 2p sorted wide indices w_k the
// count and position of every row are closed forms, so the list is generated on the device into
// stream-ordered scratch (no per-range cache, no host copy: graph-capturable).
struct ShellDesc {
    int64_t N, rb, re, l0, l1;
    int nw;
    int64_t w[2 * kMaxP];
};

__host__ __device__ inline bool shell_is_wide(const ShellDesc& d, int64_t l) {
    for (int k = 0; k < d.nw; ++k)
        if (d.w[k] == l) return true;
    return false;
}
// rows of line l inside the range
__host__ __device__ inline int64_t shell_line_count(const ShellDesc& d, int64_t l) {
    const int64_t a = l * d.N > d.rb ? l * d.N : d.rb, b = (l + 1) * d.N < d.re ? (l + 1) * d.N : d.re;
    if (b <= a) return 0;
    if (shell_is_wide(d, l)) return b - a;
    int64_t c = 0;
    for (int k = 0; k < d.nw; ++k) c += (l * d.N + d.w[k] >= a && l * d.N + d.w[k] < b);
    return c;
}
// list position of line l's first row: count(l0) + full lines strictly between (N or nw rows)
__host__ __device__ inline int64_t shell_line_start(const ShellDesc& d, int64_t l) {
    if (l <= d.l0) return 0;
    int64_t wide_between = 0;
    for (int k = 0; k < d.nw; ++k) wide_between += (d.w[k] > d.l0 && d.w[k] < l);
    return shell_line_count(d, d.l0) + (l - d.l0 - 1) * d.nw + wide_between * (d.N - d.nw);
}

__global__ void k_shell_rows(const ShellDesc d, int64_t* out) {
    // one warp per line of the range
    const int64_t l = d.l0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (l > d.l1) return;
    const int64_t a = l * d.N > d.rb ? l * d.N : d.rb, b = (l + 1) * d.N < d.re ? (l + 1) * d.N : d.re;
    const int64_t base = shell_line_start(d, l);
    if (shell_is_wide(d, l)) {
        for (int64_t r = a + lane; r < b; r += 32) out[base + (r - a)] = r;
    } else if (lane == 0) {
        int64_t c = 0;
        for (int k = 0; k < d.nw; ++k) {
            const int64_t r = l * d.N + d.w[k];
            if (r >= a && r < b) out[base + c++] = r;
        }
    }
}

int shell_rows_2d(const wgq_rules_s* R, int64_t row_begin, int64_t row_end, cudaStream_t st, int64_t** rows,
                  int64_t* count) {
    *rows = nullptr;
    *count = 0;
    ShellDesc d{};
    d.N = R->N;
    d.rb = row_begin;
    d.re = row_end;
    for (int64_t r = 0; r < R->N; ++r) {
        const int cls = r < R->p ? (int)r : (r >= R->n ? (int)(R->n + R->p - 1 - r) : R->p);
        if ((R->rules[WGQ_MASS][cls].m > 4 || R->rules[WGQ_STIFFNESS][cls].m > 4) && d.nw < 2 * kMaxP) d.w[d.nw++] = r;
    }
    if (d.nw == 0 || row_end <= row_begin) return WGQ_OK;
    d.l0 = row_begin / R->N;
    d.l1 = (row_end - 1) / R->N;
    const int64_t total = d.l1 > d.l0 ? shell_line_start(d, d.l1) + shell_line_count(d, d.l1) : shell_line_count(d, d.l0);
    if (total == 0) return WGQ_OK;
    if (cudaMallocAsync((void**)rows, (size_t)total * sizeof(int64_t), st) != cudaSuccess) return WGQ_ENOMEM;
    const int64_t lines = d.l1 - d.l0 + 1;
    k_shell_rows<<<(unsigned)((lines * 32 + 255) / 256), 256, 0, st>>>(d, *rows);
    *count = total;
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

int launch_assemble(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const wgq_out_t* M,
                    const wgq_out_t* K, void* stream) {
    static const bool force_generic_env = [] {
        const char* e = getenv("WGQ_FORCE_GENERIC");
        return e && e[0] == '1';
    }();
    // the specialised kernels assume equal element counts in every direction
    const bool force_generic = force_generic_env || !R->iso;
    const RowTables& T = TT.t[0];
    // the GRID line kernel takes per-direction sizes itself
    if (!force_generic_env && line_kernel_applies(R, c, M, K)) return launch_line(R, TT, c, M, K, stream);
    if (!force_generic && sep_applies(c)) return launch_sep(R, T, c, M, K, stream);
    GenericArgs a{};
    set_dirs(a, R, TT);
    a.coef = make_coef(c);
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
    // analytic coefficients: factor tables at the nodes (stream-ordered scratch, freed after)
    double* tab = nullptr;
    int rc = coef_tables(R, a, c, st, &tab);
    if (rc != WGQ_OK) return rc;
    rc = WGQ_EUNSUPPORTED;
    const int key = R->p * 10 + R->dim;
    a.frame = 0;
    int64_t* shell = nullptr;            // 2D shell-row list (stream-ordered scratch)
    if (!force_generic && R->dim == 2 && c->kind == WGQ_COEF_FOURIER_LOGN && a.coef.n_modes > 0) {
        // p = 3: the fused interior / frame / shell launch of fourier2d.cu; otherwise the per-row
        // tensor-core kernel over the rows whose directions all have <= 4 nodes, then the generic
        // kernel over the remaining shell (GL-fallback classes, R1)
        static const bool interior_on = [] {
            const char* e = getenv("WGQ_F2D_INTERIOR");
            return !(e && e[0] == '0');
        }();
        if (interior_on && f2d_interior_applies(R, T, c)) {
            // class-I rows, the frame (per-row tables) and, when no rule has more than 8 nodes,
            // the shell rows (split into 4-node halves) in one launch (fourier2d.cu)
            int maxm = 0;
            for (int cl = 0; cl <= R->p; ++cl)
                maxm = std::max(maxm, std::max(R->rules[WGQ_MASS][cl].m, R->rules[WGQ_STIFFNESS][cl].m));
            int64_t nsh = 0;
            if (maxm <= 8) rc = shell_rows_2d(R, a.row_begin, a.row_end, st, &shell, &nsh);
            else rc = WGQ_OK;
            if (rc == WGQ_OK) rc = launch_f2d_interior(R, T, tab, a.cw, M, K, shell, nsh, st);
            if (rc != WGQ_OK || maxm <= 8) {          // done (the generic shell pass is not needed)
                if (shell) cudaFreeAsync(shell, st);
                cudaFreeAsync(tab, st);
                return rc;
            }
        } else {
            rc = R->p == 3 ? launch_fourier2d_p<3>(a, st) : launch_fourier2d_p<2>(a, st);
        }
        if (rc != WGQ_OK) {
            cudaFreeAsync(tab, st);
            return rc;
        }
        rc = shell_rows_2d(R, a.row_begin, a.row_end, st, &shell, &a.nlist);
        if (rc != WGQ_OK || a.nlist == 0) {
            cudaFreeAsync(tab, st);
            return rc;
        }
        a.rows_list = shell;
    }
    switch (key) {
        case 21: rc = launch_generic_pd<2, 1>(a, T.maxM, T.maxK, st); break;
        case 22: rc = launch_generic_pd<2, 2>(a, T.maxM, T.maxK, st); break;
        case 23: rc = launch_generic_pd<2, 3>(a, T.maxM, T.maxK, st); break;
        case 31: rc = launch_generic_pd<3, 1>(a, T.maxM, T.maxK, st); break;
        case 32: rc = launch_generic_pd<3, 2>(a, T.maxM, T.maxK, st); break;
        case 33: rc = launch_generic_pd<3, 3>(a, T.maxM, T.maxK, st); break;
    }
    if (shell) cudaFreeAsync(shell, st);
    if (tab) cudaFreeAsync(tab, st);
    return rc;
}

int launch_load(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                double* b, void* stream) {
    if (row_end <= row_begin) return WGQ_OK;
    static const bool force_generic_env = [] {
        const char* e = getenv("WGQ_FORCE_GENERIC");
        return e && e[0] == '1';
    }();
    const bool force_generic = force_generic_env || !R->iso;     // specialised kernels: equal counts
    const RowTables& T = TT.t[0];
    if (!force_generic && sep_applies(c)) return launch_sep_load(R, T, c, row_begin, row_end, b, stream);
    cudaStream_t st = (cudaStream_t)stream;
    GenericArgs a = base_args(R, TT, c, row_begin, row_end);
    double* tab = nullptr;
    const PW3 PW{{TT.t[0].PW, TT.t[1].PW, TT.t[2].PW}};
    int rc = coef_tables(R, a, c, st, &tab);
    if (rc != WGQ_OK) return rc;
    int64_t* shell = nullptr;            // 2D shell-row list (stream-ordered scratch)
    if (!force_generic && R->dim == 2 && c->kind == WGQ_COEF_FOURIER_LOGN && a.coef.n_modes > 0) {
        // the 2D tensor-core kernel in load mode (its exponent product and exp, no y / x stages),
        // then the generic per-row kernel over the shell rows (GL-fallback boundary classes)
        GenericArgs f = a;
        f.load = 1;
        f.b = b;
        f.do_mass = 1;
        f.do_stiff = 0;
        rc = R->p == 3 ? launch_fourier2d_p<3>(f, st) : launch_fourier2d_p<2>(f, st);
        if (rc == WGQ_OK) rc = shell_rows_2d(R, row_begin, row_end, st, &shell, &a.nlist);
        if (rc != WGQ_OK || a.nlist == 0) {
            if (tab) cudaFreeAsync(tab, st);
            return rc;
        }
        a.rows_list = shell;
    }
    rc = WGQ_EUNSUPPORTED;
    switch (R->p * 10 + R->dim) {
        case 21: rc = launch_load_pd<2, 1>(a, PW, b, !force_generic, st); break;
        case 22: rc = launch_load_pd<2, 2>(a, PW, b, !force_generic, st); break;
        case 23: rc = launch_load_pd<2, 3>(a, PW, b, !force_generic, st); break;
        case 31: rc = launch_load_pd<3, 1>(a, PW, b, !force_generic, st); break;
        case 32: rc = launch_load_pd<3, 2>(a, PW, b, !force_generic, st); break;
        case 33: rc = launch_load_pd<3, 3>(a, PW, b, !force_generic, st); break;
    }
    if (shell) cudaFreeAsync(shell, st);
    if (tab) cudaFreeAsync(tab, st);
    return rc;
}

int launch_apply(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const double* u, int64_t u_row0,
                 int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream) {
    if (row_end <= row_begin) return WGQ_OK;
    static const bool force_generic_env = [] {
        const char* e = getenv("WGQ_FORCE_GENERIC");
        return e && e[0] == '1';
    }();
    const bool force_generic = force_generic_env || !R->iso;     // specialised kernels: equal counts
    const RowTables& T = TT.t[0];
    if (!force_generic_env && line_apply_applies(R, c))
        return launch_line_apply(R, TT, c, u, u_row0, row_begin, row_end, yM, yK, stream);
    if (!force_generic && sep_applies(c))
        return launch_sep_apply(R, T, c, u, u_row0, row_begin, row_end, yM, yK, stream);
    cudaStream_t st = (cudaStream_t)stream;
    GenericArgs a = base_args(R, TT, c, row_begin, row_end);
    a.apply = 1;
    a.u = u;
    a.u_row0 = u_row0;
    a.yM = yM;
    a.yK = yK;
    a.do_mass = yM != nullptr;
    a.do_stiff = yK != nullptr;
    a.M.layout = WGQ_ELL;
    double* tab = nullptr;
    int rc = coef_tables(R, a, c, st, &tab);
    if (rc != WGQ_OK) return rc;
    int64_t* shell = nullptr;            // 2D shell-row list (stream-ordered scratch)
    if (!force_generic && R->dim == 2 && c->kind == WGQ_COEF_FOURIER_LOGN && a.coef.n_modes > 0) {
        // tensor-core rows, then the generic kernel over the shell rows (as for the assembly)
        rc = R->p == 3 ? launch_fourier2d_p<3>(a, st) : launch_fourier2d_p<2>(a, st);
        if (rc == WGQ_OK) rc = shell_rows_2d(R, row_begin, row_end, st, &shell, &a.nlist);
        if (rc != WGQ_OK || a.nlist == 0) {
            cudaFreeAsync(tab, st);
            return rc;
        }
        a.rows_list = shell;
    }
    rc = WGQ_EUNSUPPORTED;
    switch (R->p * 10 + R->dim) {
        case 21: rc = launch_generic_pd<2, 1>(a, T.maxM, T.maxK, st); break;
        case 22: rc = launch_generic_pd<2, 2>(a, T.maxM, T.maxK, st); break;
        case 23: rc = launch_generic_pd<2, 3>(a, T.maxM, T.maxK, st); break;
        case 31: rc = launch_generic_pd<3, 1>(a, T.maxM, T.maxK, st); break;
        case 32: rc = launch_generic_pd<3, 2>(a, T.maxM, T.maxK, st); break;
        case 33: rc = launch_generic_pd<3, 3>(a, T.maxM, T.maxK, st); break;
    }
    if (shell) cudaFreeAsync(shell, st);
    if (tab) cudaFreeAsync(tab, st);
    return rc;
}

}  // namespace wgq
