// 2D FOURIER_LOGN assembly of the interior rows (C3: p = 3, 2048^2, M + K), sm_100a.
//
// Row (i1, i2) samples the coefficient at three node tensors (a3): mass-x x mass-y (M),
// stiffness-x x mass-y (K_x term) and mass-x x stiffness-y (K_y term), 48 samples for p = 3,
// each an exp of a rank-2*n_modes exponent (R13: c = exp(sum_m a_m cos(2 pi k_m.x + theta_m)),
// expanded with the angle-sum identity into the factor tables of k_coef_tables):
//   E[x-node][y-node] = sum_m C^x_m C^y_m - S^x_m S^y_m.
// Rows whose index is in the interior class I in both directions (2p <= i_a <= N-1-2p) share
// one weighted 1D table per kind (w_k B_{i+o}(x_k), w_k B'_{i+o}(x_k); eq:GaussQuadSys P:249-252,
// eq:GaussQuadSysStiff P:350-353), so with Aw = w * B folded
//   M[o1][o2] = sum_{kx,ky} AwM[kx][o1] AwM[ky][o2] c(xM_kx, yM_ky)
//   K[o1][o2] = sum AwK[kx][o1] AwM[ky][o2] c(xK_kx, yM_ky) + AwM[kx][o1] AwK[ky][o2] c(xM_kx, yK_ky)
// which is the definition with the products regrouped, contracted y then x
// (eq:Decompo P:194-199).
//
// One warp owns a block of 2 x-lines (i2 = a, a+1) and walks pairs of rows (i1, i1+1):
//  * exponents on the FP64 tensor cores (DMMA m8n8k4): x-nodes of the pair form the 8 tile rows
//    (x-node g = (kx = g/2, row g%2)); tile A_a / A_b take the 8 y-nodes of line a / b
//    (y-node n = (ky = n/2, mass|stiffness)), tile B the stiffness x-nodes against the mass
//    y-nodes of both lines (n = (ky = n/2, line a|b)).  Every product is a used sample: 12 DMMA
//    per 4 rows, 6 samples per lane, lane-dense exp;
//  * exp by a 256-entry table of 2^(j/256) (16 lane-private copies, conflict-free) and a degree-4
//    polynomial on |r| <= ln2/512 (8 FP64 operations, remainder < 4e-17; the 64-entry table with a
//    degree-5 polynomial took 10 and the FP64 pipe, shared by the DMMAs, is the binding unit);
//  * y stage on DMMA: the exp'd accumulator fragment is the B operand of T^T = Aw_y^T W^T as is
//    (6 DMMA per 4 rows);
//  * x stage on DMMA: the y stage's output fragment is the B operand as is, the class-I Aw_x^T
//    fragment the y stage's A operand (12 DMMA per 4 rows);
//  * the rows are staged in shared memory (a bank-permuted slot layout, kF2iSlot: conflict-free
//    x-stage writes and run reads) and written as contiguous 16-byte runs with streaming stores.
// The frame rows (an index outside class I) and the split GL shell rows are extra items of the
// same launch (f2d_frame_item, f2d_shell_item).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "internal.h"

namespace wgq {
namespace {

constexpr int kF2iWarps = 8;
constexpr int kF2iMinBlocks = 2;
constexpr int kF2iChunk = 24;              // row pairs per work item (ticketed items: 16: 0.820 ms, 24: 0.797, 32: 0.844, 48: 0.805)
constexpr int kF2iRun = 112;                             // staging of one (line, matrix) run (56 16-byte slots)
// output staging of 2 lines x M, K
constexpr int kF2iWarpSmem = 4 * kF2iRun;

// Interior-kernel staging layout: element s (= run element + shift sh) of a (line, matrix) run
// lives in 16-byte slot kF2iSlot[sh][s >> 1], half s & 1.  The slots were searched
// (tools/staging_layout.py) so that, for either shift, every x-stage write (lane (g, t) ->
// elements g + 14 t + 7 j + 49 i + sh; 64-bit accesses are served per half-warp) hits 16 distinct
// 8-byte banks per half-warp and every 16-byte run read (lane -> pair lane + sh, lane + 32 + sh;
// served per quarter-warp) 8 distinct 16-byte bank groups per quarter-warp: 2 wavefronts per
// x-stage write (the natural layout took 4) and the minimum for the reads.
__constant__ int kF2iSlot[2][50] = {
    {5,  3,  2,  1,  6,  7,  0,  4,  14, 15, 13, 10, 11, 12, 9,  8,  19, 16, 20, 21, 17, 18, 23, 22, 28,
     25, 30, 31, 26, 24, 27, 29, 39, 34, 35, 37, 33, 36, 38, 32, 44, 40, 47, 46, 41, 42, 43, 45, 49, 48},
    {51, 7,  3,  1,  0,  2,  5,  6,  4,  8,  12, 15, 9,  11, 10, 13, 14, 23, 22, 19, 20, 16, 17, 18, 21,
     25, 28, 31, 26, 27, 24, 30, 29, 34, 37, 32, 33, 39, 36, 38, 35, 41, 46, 44, 42, 45, 40, 47, 43, 52}};
constexpr int kF2iEdge0 = 2 * 51 + 1;     // element 0 of a shifted run (s = 1): pair 0, high half
constexpr int kF2iEdge1 = 2 * 52;         // element 97 of a shifted run (s = 98): pair 49, low half

struct F2iArgs {
    const double* ctab;  // k_coef_tables layout: ((kind * N + r) * kMaxNodes + k) * cw + j
    unsigned long long* ticket;   // work-item counter (stream-ordered scratch, zeroed per launch)
    int cw;
    int64_t N, row_begin, row_end;
    int lo, hi;          // class-I index range [lo, hi] (both directions)
    int line0, line1;    // interior lines inside the row range
    double* Mv;
    double* Kv;
    int64_t ldM, ldK;
    const int64_t* rpM;
    const int64_t* rpK;
    int csr;
    int dbg;             // profiling switches (WGQ_F2D_DBG): 1 no global stores, 2 no exponent / exp
    double AwM[4][7], AwK[4][7];   // interior weighted tables w_k B_{i+o}(x_k), w_k B'_{i+o}(x_k)
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Taylor coefficients of e^r (degree 5) from the constant bank
__constant__ double kExp5[6] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0};

// exp(x), |x| < 700: x = k ln2/256 + r with k = rint(256 x / ln2) (the 1.5*2^52 shifter leaves k
// in the low word), |r| <= ln2/512 (Cody-Waite two-part ln2/256), e^x = 2^(k>>8) 2^((k&255)/256) e^r
// with e^r by its degree-4 Taylor polynomial (remainder < r^5/120 < 4e-17).
// tbl holds 2^(j/256) at [j * 16 + copy], tb = tbl + copy (copy = lane & 15): the 16 lanes of a
// half-warp read 16 different banks.
constexpr int kExpBits = 8;
__device__ __forceinline__ double exp_tab(double x, const double* tb) {
    const double s = fma(x, 369.32993046757462750, 6755399441055744.0);   // 256/ln2, 1.5*2^52
    const double kd = s - 6755399441055744.0;
    const int k = __double2loint(s);
    double r = fma(-kd, 6.93147180369123816490e-01 / 256.0, x);
    r = fma(-kd, 1.90821492927058770002e-10 / 256.0, r);
    double q = kExp5[4];
#pragma unroll
    for (int i = 3; i >= 0; --i) q = fma(q, r, kExp5[i]);
    const double t = tb[(k & 255) << 4];
    return q * __hiloint2double(__double2hiint(t) + ((k >> 8) << 20), __double2loint(t));
}

__device__ __forceinline__ void st_out(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ void st_out2(double* p, double v0, double v1, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v0), "d"(v1),
                 "l"(pol)
                 : "memory");
}

// The interior kernel's per-row store of one staged row pair (line Ln, rows i1, i1 + 1) of matrix
// mat when the pair is not part of a contiguous run (ragged ranges, padded ld): kept out of line
// so that its row checks and pointer arithmetic are not hoisted into the run path.
__device__ __noinline__ void store_pair_general(double* dst, const int64_t* rp, int64_t ld, int64_t N, int hi,
                                                int64_t row_begin, int64_t row_end, const double* src, int shv,
                                                const int* slot, int Ln, int i1, bool line_ok, int lane,
                                                uint64_t pol);

// ---------------------------------------------------------------------------------------------
// The frame: every 2D row with an index outside class I (and no GL-fallback wide direction),
// with the interior kernel's structure (2 lines x row pairs, DMMA exponent / y / x chain, table
// exp) but per-line y and per-row x weighted tables (RowTables::AW) as the A fragments, and
// per-row stores (a row is written only if it is in the frame: the interior kernel owns
// [lo, hi]^2).  Items: line pairs whose both lines are class I contribute their two frame row
// chunks [0, lo) and (hi, N); the other line pairs (the mesh's first and last lines) all their
// row chunks.
struct F2fArgs {
    int64_t items;            // frame work items (done before the interior items)
    const double* ctab;
    int cw;
    const double* AW;         // RowTables::AW [N][2][8][8]
    int64_t N, row_begin, row_end;
    int lo, hi;               // class-I range (the interior kernel's rows)
    int L0, nlp;              // first line of the pairing, number of line pairs
    int jA0, jA1;             // line pairs jA0 .. jA1 are interior (both lines class I)
    int nw;                   // wide 1D indices (GL-fallback classes, > 4 nodes): the shell rows
    int wide[2 * kMaxP];
    const int64_t* shell;     // shell rows done in this launch (<= 8 nodes per direction), or null
    int64_t nshell;
    double* Mv;
    double* Kv;
    int64_t ldM, ldK;
    const int64_t* rpM;
    const int64_t* rpK;
    int csr;
};

__device__ __forceinline__ bool f2f_wide(const F2fArgs& a, int64_t r) {
    bool w = false;
#pragma unroll
    for (int k = 0; k < 2 * kMaxP; ++k) w |= k < a.nw && a.wide[k] == r;
    return w;
}

template <int KS>
__device__ __forceinline__ void f2d_frame_item(const F2fArgs& a, int64_t it, const double* tbl, double* os, int lane,
                                               uint64_t pol) {
    constexpr int S = 7, P3 = 3;
    const int g = lane >> 2, t = lane & 3;
    const int copy = lane & 15;
    const int64_t N = a.N;
    const int cw = a.cw;
    const int64_t nstride = (int64_t)kMaxNodes * cw;
    const double ysg = (t & 1) ? -1.0 : 1.0;
    const int nA = a.jA1 >= a.jA0 ? a.jA1 - a.jA0 + 1 : 0;
    const int fullchunks = (int)((N + 2 * kF2iChunk - 1) / (2 * kF2iChunk));
    // A fragment of a weighted table, lane (g, t) = Aw^T[o = g][k = t] of 1D row r, kind
    auto afrag = [&](int64_t r, int kind) { return g < S ? __ldg(a.AW + r * 128 + kind * 64 + t * 8 + g) : 0.0; };
    int j, x0, npair;
    if (it < (int64_t)nA * 2) {
        j = a.jA0 + (int)(it >> 1);
        x0 = (it & 1) ? a.hi + 1 : 0;
        npair = (it & 1) ? (int)(N - 1 - a.hi + 1) / 2 : (a.lo + 1) / 2;
    } else {
        const int64_t f = it - (int64_t)nA * 2;
        const int jb = (int)(f / fullchunks);
        j = jb < a.jA0 ? jb : (nA > 0 ? jb + nA : jb);
        x0 = (int)(f % fullchunks) * 2 * kF2iChunk;
        npair = (int)min((int64_t)kF2iChunk, (N - x0 + 1) / 2);
    }
    const int La = a.L0 + 2 * j;
    const bool bval = La + 1 < N;
    const int Lb = bval ? La + 1 : La;
    double Ya[KS], Yb[KS], Yab[KS];
    {
        const int ky = g >> 1, hi = g & 1;
        const double* pa = a.ctab + ((int64_t)(2 + hi) * N + La) * nstride + ky * cw + t;
        const double* pb = a.ctab + ((int64_t)(2 + hi) * N + Lb) * nstride + ky * cw + t;
        const double* pab = a.ctab + ((int64_t)2 * N + (hi ? Lb : La)) * nstride + ky * cw + t;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const bool in = 4 * s + t < cw;
            Ya[s] = in ? ysg * __ldg(pa + 4 * s) : 0.0;
            Yb[s] = in ? ysg * __ldg(pb + 4 * s) : 0.0;
            Yab[s] = in ? ysg * __ldg(pab + 4 * s) : 0.0;
        }
    }
    const double aMa = afrag(La, 0), aKa = afrag(La, 1), aMb = afrag(Lb, 0), aKb = afrag(Lb, 1);
    const bool la_ok = !f2f_wide(a, La), lb_ok = bval && !f2f_wide(a, Lb);
    const bool la_in = La >= a.lo && La <= a.hi, lb_in = Lb >= a.lo && Lb <= a.hi;
    for (int pr = 0; pr < npair; ++pr) {
        const int i1 = x0 + 2 * pr;
        const int r0 = i1, r1 = i1 + 1 < N ? i1 + 1 : i1;
        // x-node g = (kx = g >> 1, row i1 + (g & 1))
        double XM[KS], XK[KS];
        {
            const int rr = (g & 1) ? r1 : r0;
            const double* pm = a.ctab + (int64_t)rr * nstride + (g >> 1) * cw + t;
            const double* pk = pm + N * nstride;
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const bool in = 4 * s + t < cw;
                XM[s] = in ? __ldg(pm + 4 * s) : 0.0;
                XK[s] = in ? __ldg(pk + 4 * s) : 0.0;
            }
        }
        double ea0 = 0.0, ea1 = 0.0, eb0 = 0.0, eb1 = 0.0, ek0 = 0.0, ek1 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            dmma(ea0, ea1, XM[s], Ya[s]);
            dmma(eb0, eb1, XM[s], Yb[s]);
            dmma(ek0, ek1, XK[s], Yab[s]);
        }
        const double wMa = exp_tab(ea0, tbl + copy), wKya = exp_tab(ea1, tbl + copy);
        const double wMb = exp_tab(eb0, tbl + copy), wKyb = exp_tab(eb1, tbl + copy);
        const double wKxa = exp_tab(ek0, tbl + copy), wKxb = exp_tab(ek1, tbl + copy);
        double tM[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, tKx[2][2] = {{0.0, 0.0}, {0.0, 0.0}},
               tKy[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        dmma(tM[0][0], tM[0][1], aMa, wMa);
        dmma(tKy[0][0], tKy[0][1], aKa, wKya);
        dmma(tKx[0][0], tKx[0][1], aMa, wKxa);
        dmma(tM[1][0], tM[1][1], aMb, wMb);
        dmma(tKy[1][0], tKy[1][1], aKb, wKyb);
        dmma(tKx[1][0], tKx[1][1], aMb, wKxb);
        const double aMx[2] = {afrag(r0, 0), afrag(r1, 0)}, aKx[2] = {afrag(r0, 1), afrag(r1, 1)};
#pragma unroll
        for (int L = 0; L < 2; ++L)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
                dmma(m0, m1, aMx[i], tM[L][i]);
                dmma(k0, k1, aKx[i], tKx[L][i]);
                dmma(k0, k1, aMx[i], tKy[L][i]);
                double* b = os + L * 2 * kF2iRun + i * 49 + g + 14 * t;
                if (g < S) {
                    b[0] = m0;
                    b[kF2iRun] = k0;
                    if (t < 3) {
                        b[7] = m1;
                        b[kF2iRun + 7] = k1;
                    }
                }
            }
        __syncwarp();
        // a7: per row (frame rows are partly outside the mesh: ELL slots of missing columns
        // hold +0.0, CSR rows are compacted to their valid columns, in slot order)
#pragma unroll
        for (int L = 0; L < 2; ++L) {
            const int i2 = L ? Lb : La;
            const bool lok = L ? lb_ok : la_ok, lin = L ? lb_in : la_in;
            const int lo2 = max(-P3, -i2), w2h = min(P3, (int)N - 1 - i2);
#pragma unroll
            for (int mat = 0; mat < 2; ++mat) {
                double* dst = mat ? a.Kv : a.Mv;
                if (!dst) continue;
                const double* src = os + (L * 2 + mat) * kF2iRun;
                for (int e = lane; e < 98; e += 32) {
                    const int i = e >= 49 ? 1 : 0, slot = e - 49 * i, r = i1 + i;
                    const int64_t grow = (int64_t)i2 * N + r;
                    if (!lok || r >= N || (lin && r >= a.lo && r <= a.hi) || f2f_wide(a, r) || grow < a.row_begin ||
                        grow >= a.row_end)
                        continue;
                    const int64_t orow = grow - a.row_begin;
                    const int o1 = slot % 7 - P3, o2 = slot / 7 - P3;
                    if (a.csr) {
                        const int lo1 = max(-P3, -r), hi1 = min(P3, (int)N - 1 - r);
                        if (o1 < lo1 || o1 > hi1 || o2 < lo2 || o2 > w2h) continue;
                        st_out(dst + (mat ? a.rpK : a.rpM)[orow] + (o1 - lo1) + (int64_t)(o2 - lo2) * (hi1 - lo1 + 1),
                               src[e], pol);
                    } else {
                        st_out(dst + orow * (mat ? a.ldK : a.ldM) + slot, src[e] + 0.0, pol);
                    }
                }
            }
        }
        __syncwarp();
    }
}

// A shell row (a direction with a GL-fallback rule of 5..8 nodes, R1): its nodes are split into
// two halves of 4 per direction (x: nodes 0-3 | 4-7, y likewise; a direction with <= 4 nodes
// has an empty second half: zero weights), the four (x half, y half) combinations are the 2 x 2
// rows of one step of the frame machinery, and the row is their sum: every sample of the
// definition appears in exactly one combination (the mass nodes all lie in the first half).
template <int KS>
__device__ __forceinline__ void f2d_shell_item(const F2fArgs& a, int64_t row, const double* tbl, double* os, int lane,
                                               uint64_t pol) {
    constexpr int S = 7, P3 = 3;
    const int g = lane >> 2, t = lane & 3;
    const int copy = lane & 15;
    const int64_t N = a.N;
    const int cw = a.cw;
    const int64_t nstride = (int64_t)kMaxNodes * cw;
    const double ysg = (t & 1) ? -1.0 : 1.0;
    const int i1 = (int)(row % N), i2 = (int)(row / N);
    auto afrag = [&](int64_t r, int kind, int k0) {
        return g < S ? __ldg(a.AW + r * 128 + kind * 64 + (k0 + t) * 8 + g) : 0.0;
    };
    // exponent B fragments: y-node (ky, type) of half L, mass y-nodes of both halves (tile B)
    double Ya[KS], Yb[KS], Yab[KS];
    {
        const int ky = g >> 1, hi = g & 1;
        const double* pa = a.ctab + ((int64_t)(2 + hi) * N + i2) * nstride + ky * cw + t;
        const double* pb = pa + 4 * cw;                                          // nodes 4..7
        const double* pab = a.ctab + ((int64_t)2 * N + i2) * nstride + (4 * hi + ky) * cw + t;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const bool in = 4 * s + t < cw;
            Ya[s] = in ? ysg * __ldg(pa + 4 * s) : 0.0;
            Yb[s] = in ? ysg * __ldg(pb + 4 * s) : 0.0;
            Yab[s] = in ? ysg * __ldg(pab + 4 * s) : 0.0;
        }
    }
    const double aMa = afrag(i2, 0, 0), aKa = afrag(i2, 1, 0), aMb = afrag(i2, 0, 4), aKb = afrag(i2, 1, 4);
    // x-node g = (kx = g >> 1, half g & 1): node 4 (g & 1) + kx of row i1
    double XM[KS], XK[KS];
    {
        const double* pm = a.ctab + (int64_t)i1 * nstride + (4 * (g & 1) + (g >> 1)) * cw + t;
        const double* pk = pm + N * nstride;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const bool in = 4 * s + t < cw;
            XM[s] = in ? __ldg(pm + 4 * s) : 0.0;
            XK[s] = in ? __ldg(pk + 4 * s) : 0.0;
        }
    }
    double ea0 = 0.0, ea1 = 0.0, eb0 = 0.0, eb1 = 0.0, ek0 = 0.0, ek1 = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        dmma(ea0, ea1, XM[s], Ya[s]);
        dmma(eb0, eb1, XM[s], Yb[s]);
        dmma(ek0, ek1, XK[s], Yab[s]);
    }
    const double wMa = exp_tab(ea0, tbl + copy), wKya = exp_tab(ea1, tbl + copy);
    const double wMb = exp_tab(eb0, tbl + copy), wKyb = exp_tab(eb1, tbl + copy);
    const double wKxa = exp_tab(ek0, tbl + copy), wKxb = exp_tab(ek1, tbl + copy);
    double tM[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, tKx[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, tKy[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    dmma(tM[0][0], tM[0][1], aMa, wMa);
    dmma(tKy[0][0], tKy[0][1], aKa, wKya);
    dmma(tKx[0][0], tKx[0][1], aMa, wKxa);
    dmma(tM[1][0], tM[1][1], aMb, wMb);
    dmma(tKy[1][0], tKy[1][1], aKb, wKyb);
    dmma(tKx[1][0], tKx[1][1], aMb, wKxb);
    const double aMx[2] = {afrag(i1, 0, 0), afrag(i1, 0, 4)}, aKx[2] = {afrag(i1, 1, 0), afrag(i1, 1, 4)};
#pragma unroll
    for (int L = 0; L < 2; ++L)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
            dmma(m0, m1, aMx[i], tM[L][i]);
            dmma(k0, k1, aKx[i], tKx[L][i]);
            dmma(k0, k1, aMx[i], tKy[L][i]);
            double* b = os + L * 2 * kF2iRun + i * 49 + g + 14 * t;
            if (g < S) {
                b[0] = m0;
                b[kF2iRun] = k0;
                if (t < 3) {
                    b[7] = m1;
                    b[kF2iRun + 7] = k1;
                }
            }
        }
    __syncwarp();
    if (row >= a.row_begin && row < a.row_end) {
        const int64_t orow = row - a.row_begin;
        const int lo1 = max(-P3, -i1), hi1 = min(P3, (int)N - 1 - i1);
        const int lo2 = max(-P3, -i2), hi2 = min(P3, (int)N - 1 - i2);
#pragma unroll
        for (int mat = 0; mat < 2; ++mat) {
            double* dst = mat ? a.Kv : a.Mv;
            if (!dst) continue;
            const double* src = os + mat * kF2iRun;
            for (int slot = lane; slot < 49; slot += 32) {
                const double v = src[slot] + src[49 + slot] + src[2 * kF2iRun + slot] + src[2 * kF2iRun + 49 + slot];
                const int o1 = slot % 7 - P3, o2 = slot / 7 - P3;
                if (a.csr) {
                    if (o1 < lo1 || o1 > hi1 || o2 < lo2 || o2 > hi2) continue;
                    st_out(dst + (mat ? a.rpK : a.rpM)[orow] + (o1 - lo1) + (int64_t)(o2 - lo2) * (hi1 - lo1 + 1), v,
                           pol);
                } else {
                    st_out(dst + orow * (mat ? a.ldK : a.ldM) + slot, v + 0.0, pol);
                }
            }
        }
    }
    __syncwarp();
}

__device__ __noinline__ void store_pair_general(double* dst, const int64_t* rp, int64_t ld, int64_t N, int hi,
                                                int64_t row_begin, int64_t row_end, const double* src, int shv,
                                                const int* slot, int Ln, int i1, bool line_ok, int lane,
                                                uint64_t pol) {
    double* d[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int64_t grow = (int64_t)Ln * N + i1 + i;
        const bool ok = line_ok && i1 + i <= hi && grow >= row_begin && grow < row_end;
        const int64_t orow = grow - row_begin;
        d[i] = !ok ? nullptr : dst + (rp ? rp[orow] : orow * ld);         // rp: CSR row starts
    }
    for (int e = lane; e < 98; e += 32) {             // src: the run's staging (slot layout)
        double* p = e < 49 ? d[0] : d[1];
        const int se = e + shv;
        if (p) st_out(p + (e < 49 ? e : e - 49), src[2 * slot[50 * shv + (se >> 1)] + (se & 1)], pol);
    }
}

// EXACT: cw == 4 KS (every k-step column is a table column, no predicated loads); DBG: the
// profiling switches (WGQ_F2D_DBG; 0 in production: no switch code in the hot loop)
template <int KS, bool EXACT, int DBG>
__global__ void __launch_bounds__(kF2iWarps * 32, kF2iMinBlocks) k_f2d_interior(const F2iArgs a, const F2fArgs fa) {
    constexpr int S = 7;
    __shared__ double tbl[(1 << kExpBits) * 16];
    __shared__ int slot_s[2 * 50];
    extern __shared__ double stage[];      // per warp: T staging, output staging
    for (int e = threadIdx.x; e < (1 << kExpBits) * 16; e += blockDim.x)
        tbl[e] = exp2((double)(e >> 4) * (1.0 / (1 << kExpBits)));
    if (threadIdx.x < 100) slot_s[threadIdx.x] = kF2iSlot[threadIdx.x / 50][threadIdx.x % 50];
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
    const double* tb = tbl + (lane & 15);
    double* ws = stage + warp * kF2iWarpSmem;
    double* os = ws;
    const uint64_t pol = pol_evict_first();
    const int64_t N = a.N;
    const int cw = EXACT ? 4 * KS : a.cw;
    const int64_t nstride = (int64_t)kMaxNodes * cw;                 // doubles per 1D row of ctab
    // y-stage A fragments (class-I lines): lane (g, t) = Aw^T[o2 = g][ky = t]
    double aMy = 0.0, aKy = 0.0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int oo = 0; oo < S; ++oo)
            if (kk == t && oo == g) {       // static parameter indices (no local-memory copy)
                aMy = a.AwM[kk][oo];
                aKy = a.AwK[kk][oo];
            }
    // the exponent tables of this lane's x-node (kx = g >> 1, row + (g & 1)) and y-nodes
    const int jt = t;
    const double ysg = (t & 1) ? -1.0 : 1.0;   // S components negated: E = sum C C - S S

    const int nlines = a.line1 - a.line0 + 1;
    const int lpairs = (nlines + 1) >> 1;
    const int rpairs = (a.hi - a.lo + 2) >> 1;
    const int chunks = (rpairs + kF2iChunk - 1) / kF2iChunk;
    const int64_t items = a.line1 >= a.line0 ? (int64_t)lpairs * chunks : 0;
    // the frame items first (their rows have per-row tables; a few per warp), then the interior
    // items are claimed from a ticket after the first one (frame, shell, then interior in
    // chunk-major order): a warp that finishes early takes the next item, no static tail
    const int64_t nwarps = (int64_t)gridDim.x * kF2iWarps;
    for (int64_t it0 = (int64_t)blockIdx.x * kF2iWarps + warp; it0 < fa.items + fa.nshell + items;) {
        if (it0 < fa.items) {
            f2d_frame_item<KS>(fa, it0, tbl, os, lane, pol);
        } else if (it0 < fa.items + fa.nshell) {
            f2d_shell_item<KS>(fa, fa.shell[it0 - fa.items], tbl, os, lane, pol);
        } else {
        const int64_t it = it0 - fa.items - fa.nshell;
        const int lp = (int)(it % lpairs), ch = (int)(it / lpairs);
        const int La = a.line0 + 2 * lp;
        const bool bval = La + 1 <= a.line1;
        // ---- line-pair data: exponent B fragments
        double Ya[KS], Yb[KS], Yab[KS];
        {
            const int ky = g >> 1, hi = g & 1;
            const double* pa = a.ctab + ((int64_t)(2 + hi) * N + La) * nstride + ky * cw + jt;
            const double* pb = pa + nstride;
            const double* pab = a.ctab + ((int64_t)2 * N + La + hi) * nstride + ky * cw + jt;
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const bool in = EXACT || 4 * s + jt < cw;
                Ya[s] = in ? ysg * __ldg(pa + 4 * s) : 0.0;
                Yb[s] = in ? ysg * __ldg(pb + 4 * s) : 0.0;
                Yab[s] = in ? ysg * __ldg(pab + 4 * s) : 0.0;
            }
        }
        const int p0 = ch * kF2iChunk, p1 = min(rpairs, p0 + kF2iChunk);
        // output runs: when every row of the chunk in line L is stored and consecutive rows are
        // 49 doubles apart (ELL ld = 49, or CSR: class-I rows have full stencils), the pair's
        // two rows are one 98-double run at base[L][mat] + 98 (pr - p0); sh[L] shifts the
        // staging by one double when the run starts 8 bytes off a 16-byte boundary
        bool full[2];
        int sh[2];
        double* base[2][2];
#pragma unroll
        for (int L = 0; L < 2; ++L) {
            const int64_t g0 = (int64_t)(La + L) * N + a.lo + 2 * p0;
            const int64_t g1 = g0 + 2 * (p1 - p0) - 1;
            full[L] = (L == 0 || bval) && a.lo + 2 * p1 - 1 <= a.hi && g0 >= a.row_begin && g1 < a.row_end &&
                      (a.csr || ((!a.Mv || a.ldM == 49) && (!a.Kv || a.ldK == 49)));
#pragma unroll
            for (int mat = 0; mat < 2; ++mat) {
                double* dst = mat ? a.Kv : a.Mv;
                base[L][mat] = nullptr;
                if (full[L] && dst) {
                    const int64_t orow = g0 - a.row_begin;
                    base[L][mat] = dst + (a.csr ? (mat ? a.rpK : a.rpM)[orow] : orow * 49);
                }
            }
            double* b0 = base[L][0] ? base[L][0] : base[L][1];
            sh[L] = b0 && (reinterpret_cast<uintptr_t>(b0) & 15) ? 1 : 0;
            // M and K runs must share the shift (equal alignment); else store line L per row
            if (base[L][0] && base[L][1] &&
                ((reinterpret_cast<uintptr_t>(base[L][0]) ^ reinterpret_cast<uintptr_t>(base[L][1])) & 15))
                full[L] = false, sh[L] = 0;
        }
        double* dl[2][2];                 // per lane: its 16-byte pair of the (L, mat) run of this step
        int woff[2][2][2];                // staging offsets of the lane's x-stage outputs [L][row i][o2 = 2t + j]
        int roff[2][2];                   // and of its 16-byte pairs lane + sh, lane + 32 + sh of line L's run
#pragma unroll
        for (int L = 0; L < 2; ++L) {
            const int r0 = L * 2 * kF2iRun;
#pragma unroll
            for (int mat = 0; mat < 2; ++mat) dl[L][mat] = base[L][mat] ? base[L][mat] + sh[L] + 2 * lane : nullptr;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int e = min(g + 14 * t + 7 * j + 49 * i + sh[L], 99);
                    woff[L][i][j] = r0 + 2 * slot_s[50 * sh[L] + (e >> 1)] + (e & 1);
                }
            const int q1 = lane + 32 + sh[L];
            roff[L][0] = r0 + 2 * slot_s[50 * sh[L] + lane + sh[L]];
            roff[L][1] = r0 + 2 * slot_s[50 * sh[L] + (q1 < 50 ? q1 : lane + sh[L])];
        }
        // x-node g of the pair = (kx = g >> 1, row i1 + (g & 1)); prefetched one pair ahead (the
        // last step re-reads its own pair: no branch in the loop)
        const double* pxm = a.ctab + (int64_t)(a.lo + 2 * p0 + (g & 1)) * nstride + (g >> 1) * cw + jt;
        const double* pxk = pxm + N * nstride;
        double XM[KS], XK[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const bool in = EXACT || 4 * s + jt < cw;
            XM[s] = in && p0 < p1 ? __ldg(pxm + 4 * s) : 0.0;
            XK[s] = in && p0 < p1 ? __ldg(pxk + 4 * s) : 0.0;
        }
        // FAST: both lines are full runs of both matrices (the common case): the store code is
        // straight-line (lane predicates only)
        auto steps = [&](auto fastc) {
            constexpr bool FAST = decltype(fastc)::value;
            for (int pr = p0; pr < p1; ++pr) {
                const int i1 = a.lo + 2 * pr;
                // ---- exponents (a3): three 8 x 8 x 2n_modes products
                double ea0 = 0.0, ea1 = 0.0, eb0 = 0.0, eb1 = 0.0, ek0 = 0.0, ek1 = 0.0;
                if constexpr (DBG & 2) {
                    ea0 = XM[0], ea1 = XM[1], eb0 = XM[2], eb1 = XM[3], ek0 = XK[0], ek1 = XK[1];
                } else {
#pragma unroll
                    for (int s = 0; s < KS; ++s) {
                        dmma(ea0, ea1, XM[s], Ya[s]);
                        dmma(eb0, eb1, XM[s], Yb[s]);
                        dmma(ek0, ek1, XK[s], Yab[s]);
                    }
                }
                const int64_t adv = pr + 1 < p1 ? 2 * nstride : 0;
                pxm += adv;
                pxk += adv;
#pragma unroll
                for (int s = 0; s < KS; ++s) {
                    const bool in = EXACT || 4 * s + jt < cw;
                    XM[s] = in ? __ldg(pxm + 4 * s) : 0.0;
                    XK[s] = in ? __ldg(pxk + 4 * s) : 0.0;
                }
                // ---- samples c = exp(E): lane (g, t) holds x-node g against y-node (ky = t, *)
                double wMa, wKya, wMb, wKyb, wKxa, wKxb;
                if constexpr (DBG & 2) {
                    wMa = ea0, wKya = ea1, wMb = eb0, wKyb = eb1, wKxa = ek0, wKxb = ek1;
                } else {
                    wMa = exp_tab(ea0, tb), wKya = exp_tab(ea1, tb);
                    wMb = exp_tab(eb0, tb), wKyb = exp_tab(eb1, tb);
                    wKxa = exp_tab(ek0, tb), wKxb = exp_tab(ek1, tb);
                }
                // ---- y stage (a5): T^T[o2][x-node] = Aw_y^T[o2][ky] W^T[ky][x-node]
                double tM[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, tKx[2][2] = {{0.0, 0.0}, {0.0, 0.0}},
                       tKy[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                dmma(tM[0][0], tM[0][1], aMy, wMa);
                dmma(tKy[0][0], tKy[0][1], aKy, wKya);
                dmma(tKx[0][0], tKx[0][1], aMy, wKxa);
                dmma(tM[1][0], tM[1][1], aMy, wMb);
                dmma(tKy[1][0], tKy[1][1], aKy, wKyb);
                dmma(tKx[1][0], tKx[1][1], aMy, wKxb);
                // lane (g, t) now holds T[line][row i][kx = t][o2 = g] in component i: exactly the B
                // fragment of the x stage of row i,
                // ---- x stage (a5, a6) on DMMA: M[o1][o2] = Aw_x^T[o1][kx] T[kx][o2] (the class-I A
                // operand Aw^T[o1 = g][kx = t] is the y stage's), K = AwK_x^T T_Kx + AwM_x^T T_Ky;
                // lane (g, t) receives M[o1 = g][o2 = 2t + j], staged at slot o1 + 7 o2 of its row
#pragma unroll
                for (int L = 0; L < 2; ++L)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
                        dmma(m0, m1, aMy, tM[L][i]);
                        dmma(k0, k1, aKy, tKx[L][i]);
                        dmma(k0, k1, aMy, tKy[L][i]);
                        if (g < S) {                     // (o1 = 7, o2 = 7: padding)
                            os[woff[L][i][0]] = m0;
                            os[woff[L][i][0] + kF2iRun] = k0;
                            if (t < 3) {
                                os[woff[L][i][1]] = m1;
                                os[woff[L][i][1] + kF2iRun] = k1;
                            }
                        }
                    }
                __syncwarp();
                // ---- a7: the two rows of each line (one 98-double run when full[L]: 16-byte
                // streaming stores, loads from the staging first), M and K
#pragma unroll
                for (int L = 0; L < 2; ++L) {
#pragma unroll
                    for (int mat = 0; mat < 2; ++mat) {
                        double* dst = mat ? a.Kv : a.Mv;
                        if constexpr (DBG & 1) continue;
                        if (FAST || full[L]) {
                            if (!FAST && !dst) continue;
                            // this lane's 16-byte pair(s) of the run; with sh = 1 lanes 0 / 1 also
                            // store the run's first / last element (offsets -1 / +94 from their pair)
                            const double* sp = os + mat * kF2iRun;
                            const double2 v0 = *reinterpret_cast<const double2*>(sp + roff[L][0]);
                            const bool two = lane + 32 < 49 - sh[L];
                            double2 v1 = make_double2(0.0, 0.0);
                            if (two) v1 = *reinterpret_cast<const double2*>(sp + roff[L][1]);
                            const bool edge = sh[L] && lane < 2;
                            const double ve = edge ? sp[L * 2 * kF2iRun + (lane ? kF2iEdge1 : kF2iEdge0)] : 0.0;
                            double* d = dl[L][mat];
                            st_out2(d, v0.x, v0.y, pol);
                            if (two) st_out2(d + 64, v1.x, v1.y, pol);
                            if (edge) st_out(d + (lane ? 94 : -1), ve, pol);
                            dl[L][mat] = d + 98;
                            continue;
                        }
                        if (!dst) continue;
                        store_pair_general(dst, a.csr ? (mat ? a.rpK : a.rpM) : nullptr, mat ? a.ldK : a.ldM, N,
                                           a.hi, a.row_begin, a.row_end, os + (L * 2 + mat) * kF2iRun, sh[L], slot_s,
                                           La + L, i1, L == 0 || bval, lane, pol);
                    }
                }
                __syncwarp();                         // the staging is rewritten by the next pair
            }
        };
        if (full[0] && full[1] && a.Mv && a.Kv) steps(std::true_type{});
        else steps(std::false_type{});
        }
        unsigned long long nx = 0;
        if (lane == 0) nx = atomicAdd(a.ticket, 1ull);
        it0 = nwarps + (int64_t)__shfl_sync(0xffffffffu, nx, 0);
    }
}

}  // namespace

bool f2d_interior_applies(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c) {
    if (R->p != 3 || R->dim != 2 || c->kind != WGQ_COEF_FOURIER_LOGN) return false;
    if (c->n_modes <= 0 || c->n_modes > 16 || !T.int_ok) return false;
    if (T.imM != 4 || T.imK != 4) return false;
    const int64_t lo = 2 * R->p, hi = R->N - 1 - 2 * R->p;
    if (hi < lo) return false;
    // the x stage skips the band's structural zeros: node k of a class-I row is nonzero on
    // columns o in [k, k + p] only (it lies in the support's element k)
    for (int kx = 0; kx < 4; ++kx)
        for (int o = 0; o < 7; ++o)
            if ((o < kx || o > kx + 3) && (T.iAwM[kx][o] != 0.0 || T.iAwK[kx][o] != 0.0)) return false;
    return true;
}

namespace {
F2fArgs frame_args(const wgq_rules_s* R, const RowTables& T, const double* ctab, int cw, const wgq_out_t* M,
                   const wgq_out_t* K) {
    const wgq_out_t* any = M ? M : K;
    F2fArgs a{};
    if (any->row_end <= any->row_begin) return a;
    a.ctab = ctab;
    a.cw = cw;
    a.AW = T.AW;
    a.N = R->N;
    a.row_begin = any->row_begin;
    a.row_end = any->row_end;
    a.lo = 2 * R->p;
    a.hi = (int)(R->N - 1 - 2 * R->p);
    const int64_t l0 = a.row_begin / R->N, l1 = (a.row_end - 1) / R->N;
    a.L0 = (int)l0;
    a.nlp = (int)((l1 - l0 + 2) / 2);
    // interior line pairs: both lines in [lo, hi] and inside the range
    a.jA0 = (int)std::max<int64_t>(0, (a.lo - l0 + 1) / 2);
    a.jA1 = -1;
    for (int j = a.nlp - 1; j >= a.jA0; --j)
        if (l0 + 2 * j + 1 <= std::min<int64_t>(a.hi, l1)) {
            a.jA1 = j;
            break;
        }
    if (a.jA1 < a.jA0) a.jA0 = a.nlp, a.jA1 = a.nlp - 1;     // none: every pair is a frame pair
    for (int64_t r = 0; r < R->N && a.nw < 2 * kMaxP; ++r) {
        const int cls = r < R->p ? (int)r : (r >= R->n ? (int)(R->n + R->p - 1 - r) : R->p);
        if (R->rules[WGQ_MASS][cls].m > 4 || R->rules[WGQ_STIFFNESS][cls].m > 4) a.wide[a.nw++] = r;
    }
    a.Mv = M ? M->values : nullptr;
    a.Kv = K ? K->values : nullptr;
    a.ldM = M ? M->ld : 0;
    a.ldK = K ? K->ld : 0;
    a.rpM = M ? M->row_ptr : nullptr;
    a.rpK = K ? K->row_ptr : nullptr;
    a.csr = any->layout == WGQ_CSR;
    const int nA = a.jA1 >= a.jA0 ? a.jA1 - a.jA0 + 1 : 0;
    const int64_t fullchunks = (R->N + 2 * kF2iChunk - 1) / (2 * kF2iChunk);
    a.items = (int64_t)nA * 2 + (int64_t)(a.nlp - nA) * fullchunks;
    return a;
}
}  // namespace

int launch_f2d_interior(const wgq_rules_s* R, const RowTables& T, const double* ctab, int cw, const wgq_out_t* M,
                        const wgq_out_t* K, const int64_t* shell, int64_t nshell, cudaStream_t st) {
    const wgq_out_t* any = M ? M : K;
    F2iArgs a{};
    a.ctab = ctab;
    a.cw = cw;
    a.N = R->N;
    a.row_begin = any->row_begin;
    a.row_end = any->row_end;
    a.lo = 2 * R->p;
    a.hi = (int)(R->N - 1 - 2 * R->p);
    const int64_t l0 = a.row_begin / R->N, l1 = (a.row_end - 1) / R->N;
    a.line0 = (int)std::max<int64_t>(l0, a.lo);
    a.line1 = (int)std::min<int64_t>(l1, a.hi);
    if (a.row_end <= a.row_begin) return WGQ_OK;
    F2fArgs fa = frame_args(R, T, ctab, cw, M, K);            // the frame rows, in the same launch
    fa.shell = shell;                                         // and the shell rows (<= 8 nodes)
    fa.nshell = shell ? nshell : 0;
    a.Mv = M ? M->values : nullptr;
    a.Kv = K ? K->values : nullptr;
    a.ldM = M ? M->ld : 0;
    a.ldK = K ? K->ld : 0;
    a.rpM = M ? M->row_ptr : nullptr;
    a.rpK = K ? K->row_ptr : nullptr;
    a.csr = any->layout == WGQ_CSR;
    static const int dbg = [] {
        const char* e = getenv("WGQ_F2D_DBG");
        return e ? atoi(e) : 0;
    }();
    a.dbg = dbg;
    for (int kx = 0; kx < 4; ++kx)
        for (int o = 0; o < 7; ++o) {
            a.AwM[kx][o] = T.iAwM[kx][o];
            a.AwK[kx][o] = T.iAwK[kx][o];
        }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t lpairs = (a.line1 - a.line0 + 2) / 2;
    const int64_t rpairs = (a.hi - a.lo + 2) / 2;
    const int64_t items = (a.line1 >= a.line0 ? lpairs * ((rpairs + kF2iChunk - 1) / kF2iChunk) : 0) + fa.items + fa.nshell;
    int64_t blocks = std::min<int64_t>((items + kF2iWarps - 1) / kF2iWarps, (int64_t)sms * kF2iMinBlocks);
    blocks = std::max<int64_t>(blocks, 1);
    const size_t smem = (size_t)kF2iWarps * kF2iWarpSmem * sizeof(double);
    if (cudaMallocAsync((void**)&a.ticket, sizeof(unsigned long long), st) != cudaSuccess) return WGQ_ENOMEM;
    cudaMemsetAsync(a.ticket, 0, sizeof(unsigned long long), st);
    auto go = [&](auto kern) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return WGQ_ECUDA;
        kern<<<(unsigned)blocks, kF2iWarps * 32, smem, st>>>(a, fa);
        return WGQ_OK;
    };
    int rc;
    if (cw == 16 && dbg == 1) rc = go(k_f2d_interior<4, true, 1>);
    else if (cw == 16 && dbg == 2) rc = go(k_f2d_interior<4, true, 2>);
    else if (cw == 16 && dbg == 3) rc = go(k_f2d_interior<4, true, 3>);
    else if (cw == 16) rc = go(k_f2d_interior<4, true, 0>);
    else if (cw < 16) rc = go(k_f2d_interior<4, false, 0>);
    else if (cw == 32) rc = go(k_f2d_interior<8, true, 0>);
    else rc = go(k_f2d_interior<8, false, 0>);
    cudaFreeAsync(a.ticket, st);
    if (rc != WGQ_OK) return rc;
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

}  // namespace wgq
