// Fast path for a multilinear (GRID) coefficient in 3D: line-blocked, sum-factorised
// assembly with TMA bulk stores (the C5 hot path).
//
// With the vertex field g interpolated multilinearly (R6), the coefficient at a node is
// sum_v g_v lambda_v(x), so the row rule collapses per direction into the vertex-projected
// tables P_r[v][o] = sum_k w_k A_k[o] lambda_v(x_k) (tables.cu).  For row (i1,i2,i3):
//
//   M[o1,o2,o3] = sum_{vx,vy,vz} g[bz+vz][by+vy][bx+vx] PMx[vx][o1] PMy[vy][o2] PMz[vz][o3]
//   K           = same with (PKx PMy PMz + PMx PKy PMz + PMx PMy PKz)
//
// i.e. eq:Decompo with the coefficient's vertex expansion folded into each direction.  All
// rows of one x-line (fixed i2, i3) share the y/z factors, so per vertex plane x = v
//   HM[v][o2,o3]  = sum_{vy,vz} g[..][..][v] PMy[vy][o2] PMz[vz][o3]
//   HK[v][o2,o3]  = sum_{vy,vz} g[..][..][v] (PKy PMz + PMy PKz)
// are computed once per line (phase A, ~1 plane per row) and each row finishes with
//   M[o1,o23] = sum_vx PMx[vx][o1] HM[bx+vx][o23],  K = sum_vx PKx HM + PMx HK     (phase B)
// Interior x-rows (class I) share one table P^ (times h resp. 1/h), passed as kernel
// parameters (constant bank, read through uniform registers); its zero pattern is structural
// (a node in element k touches planes k, k+1 and columns k..k+p), so phase B issues only the
// structurally nonzero FP64 FMAs.  A CTA (2 per SM) owns a line, walks it in tiles of TR = 12 rows (each thread
// finishes two consecutive rows of one (o2,o3) group from a 6-plane window, so the constant
// tables and index arithmetic are shared by both rows), prefetches the next tile's vertex
// patch with cp.async, stages the tile's M and K rows in shared memory and writes each tile
// with one cp.async.bulk per matrix; the bulk read of a tile overlaps the next tile's phase A.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace wgq {
namespace {


template <int P>
struct Cfg {
    static constexpr int S = 2 * P + 1;
    static constexpr int S2 = S * S;
    static constexpr int S3 = S2 * S;
    static constexpr int V = P + 2;
    static constexpr int TR = 12;                      // rows per tile
    static constexpr int RPT = 2;                      // consecutive rows per thread in phase B
    static constexpr int ITEMS = TR / RPT * S2;        // (row pair, o2 o3) items per tile
    static constexpr int NT = (ITEMS + 31) / 32 * 32;  // threads
    static constexpr int W = TR + V - 1;               // vertex planes of a tile's window
    static constexpr int RING = TR + P + 1 <= 16 ? 16 : TR + P + 1;   // H ring (>= W planes)
    static constexpr int SR = S3 + 1;                  // staging row stride for padded ld
    static constexpr int STAGE = TR * SR + 2;          // doubles per staging buffer per matrix
    static constexpr int PATCH = W * V * V;
#ifndef WGQ_LINE_PFD
#define WGQ_LINE_PFD 3
#endif
    static constexpr int PFD = WGQ_LINE_PFD;           // prefetch distance (tiles) = patch / Q buffers
    static constexpr int XB = 4 * P * 2 * V * S;       // x-boundary rows' vertex tables
    static constexpr int SMEM = 2 * STAGE + RING * 2 * S2 + PFD * 4 * V * S + PFD * PATCH + XB;
    static_assert(W <= RING, "ring too small");
};

// slot of vertex plane c in an H ring of RING planes (a mask when RING is a power of two)
template <int RING>
__device__ __forceinline__ int ring_slot(int c) {
    return (RING & (RING - 1)) == 0 ? (c & (RING - 1)) : c % RING;
}

struct LineArgs {
    RowTables T;                 // x-row tables (direction 0)
    RowTables Ty, Tz;            // line tables of directions 1, 2 (= T on an isotropic mesh)
    const double* grid;
    int plane0, planes;
    int n, N;                    // x: elements, rows per line
    int ny, nz, Ny, Nz;          // y, z: elements, rows (eq:Gmap3: each direction its own count)
    int row_begin, row_end;
    double* M;
    double* K;
    long long ld;
    double h, inv_h;
    // interior (class I) x-row vertex tables P^ in physical units: PMh = h * PM, PKi = PK / h
    // (kernel parameters: constant-bank operands, no global state shared between handles)
    double PMh[kMaxV][kMaxS], PKi[kMaxV][kMaxS];
    int dbg;   // profiling only (WGQ_LINE_DBG bits): 1 = skip compute, 2 = skip stores, 4 = skip loads,
               // 64 = skip phase A, 128 = skip phase B, 256 = random staging values (assembly)
    long long csr_base;   // CSR: global position of row_begin's first entry (closed form)
    // matrix-free application (k_line_apply): y = A u over the rows, u from global row u_row0
    const double* u;
    long long u_row0;
    double* yM;
    double* yK;
    // assembly: line tickets (stream-ordered scratch, zeroed per launch) or null for the static
    // round-robin line order
    unsigned long long* ticket;
};

// L2 policies: the assembled matrices stream through L2 once (evict_first), the vertex grid
// and row tables are re-read by neighbouring lines (evict_last), so the write stream does not
// evict the small read working set (each DRAM read inside the write stream costs bus
// turnarounds).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk_store(double* gdst, const double* ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
#ifdef WGQ_NO_L2_HINTS
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst), "r"(s),
                 "r"(bytes), "l"(policy_evict_first())
                 : "memory");
#endif
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
#ifdef WGQ_NO_L2_HINTS
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0) : "memory");
#else
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;" ::"r"(s), "l"(gsrc),
                 "r"(valid ? 8 : 0), "l"(policy_evict_last())
                 : "memory");
#endif
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Patch loading: thread tid owns vertex row (vz, vy) = divmod(tid / 8, V) of the patch and
// x-offsets j = tid % 8 (+ 8); the row's base pointer is refreshed only when the prefetched
// tile starts a new line, so issuing a tile costs each thread one or two cp.async.
struct PatchRow {
    const double* base;   // &g[z][y][0] of the thread's vertex row, or nullptr (outside grid/slab)
};

template <int P>
__device__ __forceinline__ void patch_row_init(const LineArgs& a, PatchRow& pr, int i2, int i3, int tid) {
    constexpr int V = P + 2;
    const int r = tid >> 3, vy = r % V, vz = r / V;
    const int y = max(0, i2 - P) + vy, z = max(0, i3 - P) + vz;
    const int nvx = a.n + 1, nvy = a.ny + 1;
    const bool ok = r < V * V && y <= a.ny && z <= a.nz && z - a.plane0 < a.planes;
    pr.base = ok ? a.grid + ((size_t)(z - a.plane0) * nvy + y) * nvx : nullptr;
}

// Issue the vertex patch of planes [c0, c0+nnew): patch[j][vz][vy]; out-of-range vertices
// are zero-filled (cp.async with source size 0).
template <int P>
__device__ __forceinline__ void load_patch(const LineArgs& a, const PatchRow& pr, double* patch, int c0, int nnew,
                                           int tid) {
    constexpr int V = P + 2;
    const int r = tid >> 3;
    if (r >= V * V) return;
    const int vy = r % V, vz = r / V;
    for (int j = tid & 7; j < nnew; j += 8) {
        const int x = c0 + j;
        const bool ok = pr.base != nullptr && x <= a.n;
        cp_async8(patch + (j * V + vz) * V + vy, ok ? pr.base + x : a.grid, ok);
    }
}

// two consecutive interior (class I) rows r, r+1 from the shared window hm/hk[0..V]: row r
// uses planes 0..V-1, row r+1 planes 1..V.  Only the structural nonzeros of P^ are issued
// (a node in element k touches planes k, k+1 and columns k..k+p), each constant-bank
// coefficient feeds both rows, and h / 1/h are folded into the tables.
template <int P, int MODE>
__device__ __forceinline__ void finish_pair_interior(const double* hm, const double* hk, double* dM, double* dK,
                                                     int SRr, bool second, const LineArgs& a) {
    constexpr int S = 2 * P + 1;
#pragma unroll
    for (int o1 = 0; o1 < S; ++o1) {
        double m0 = 0.0, k0 = 0.0, m1 = 0.0, k1 = 0.0;
#pragma unroll
        for (int v = (o1 - P > 0 ? o1 - P : 0); v <= (o1 + 1 < P + 1 ? o1 + 1 : P + 1); ++v) {
            const double pm = a.PMh[v][o1];
            if (MODE & 1) {
                m0 = fma(pm, hm[v], m0);
                m1 = fma(pm, hm[v + 1], m1);
            }
            if (MODE & 2) {
                const double pk = a.PKi[v][o1];
                k0 = fma(pk, hm[v], k0);
                k1 = fma(pk, hm[v + 1], k1);
                k0 = fma(pm, hk[v], k0);
                k1 = fma(pm, hk[v + 1], k1);
            }
        }
        if (MODE & 1) {
            dM[o1] = m0;
            if (second) dM[SRr + o1] = m1;
        }
        if (MODE & 2) {
            dK[o1] = k0;
            if (second) dK[SRr + o1] = k1;
        }
    }
}

// one interior row (P^ tables) from its window hm/hk[0..V)
template <int P, int MODE>
__device__ __forceinline__ void finish_interior(const double* hm, const double* hk, double* dM, double* dK,
                                                const LineArgs& a) {
    constexpr int S = 2 * P + 1;
#pragma unroll
    for (int o1 = 0; o1 < S; ++o1) {
        double m = 0.0, k = 0.0;
#pragma unroll
        for (int v = (o1 - P > 0 ? o1 - P : 0); v <= (o1 + 1 < P + 1 ? o1 + 1 : P + 1); ++v) {
            if (MODE & 1) m = fma(a.PMh[v][o1], hm[v], m);
            if (MODE & 2) {
                k = fma(a.PKi[v][o1], hm[v], k);
                k = fma(a.PMh[v][o1], hk[v], k);
            }
        }
        if (MODE & 1) dM[o1] = m;
        if (MODE & 2) dK[o1] = k;
    }
}

// a boundary-affected x-row: its own vertex tables (PM then PK, [v][o]), staged in shared
// memory once per CTA (the 4p such rows are the same for every line)
template <int P, int MODE>
__device__ __forceinline__ void finish_general(const double* pm, const double* hm, const double* hk, double* dM,
                                               double* dK, int lo1 = 0, int hi1 = 2 * P) {
    constexpr int S = 2 * P + 1, V = P + 2;
    const double* pk = pm + V * S;
#pragma unroll
    for (int o1 = 0; o1 < S; ++o1) {
        if (o1 < lo1 || o1 > hi1) continue;             // CSR: columns outside the mesh are not stored
        double s = 0.0, s1 = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double m = pm[v * S + o1];
            s = fma(m, hm[v], s);
            s1 = fma(pk[v * S + o1], hm[v], s1);
            s1 = fma(m, hk[v], s1);
        }
        if (MODE & 1) dM[o1] = s + 0.0;
        if (MODE & 2) dK[o1] = s1 + 0.0;
    }
}

// The apply's tiles carry little arithmetic, so its tile period is short and the vertex-patch /
// u-column loads need a longer lead than the assembly's: PFD tiles ahead, the u ring sized for
// the current window (<= TR + 2p columns) plus PFD tiles of new columns (<= TR + p each).
#ifndef WGQ_APPLY_PFD
#define WGQ_APPLY_PFD 3
#endif
struct ApplyCfg {
    static constexpr int PFD = WGQ_APPLY_PFD;
    static constexpr int URING = 16 + 11 * PFD;
    static_assert(PFD >= 2 && PFD <= 6, "desc ring holds tiles k .. k+PFD in 8 slots");
};

// Iterator over a CTA's tiles: lines first_line + blockIdx.x + m * gridDim.x, TR rows per
// tile.  Per-line quantities are refreshed only when the line changes, so the per-tile cost
// (paid by every thread of the CTA) is a few adds and compares.
struct TileIt {
    int line, i2, i3, x0, x1, t0;
    int nchg;    // line changes so far (ticketed order: which s_line slot the next line is in)
    bool pending;   // ticketed order: the next line is being fetched (resolved after a barrier)
    int qs;      // Q buffer of the line: line ordinal % PFD
    int ps;      // patch buffer of the tile: tile ordinal % PFD
    int lo, hi;  // vertex planes the tile adds to the line's H ring
    // basis columns X of u (matrix-free application): the line's columns occupy consecutive
    // positions of a ring, column X at lpos + X - X0 (mod the ring size)
    int X0, lpos, ulo, uhi;   // line's first column, its ring position, new columns [ulo, uhi]
};

template <int P, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ void it_planes(TileIt& t, int N) {
    constexpr int V = P + 2;
    t.lo = t.t0 == t.x0 ? max(0, t.x0 - P) : max(0, t.t0 - 1 - P) + V;
    t.hi = max(0, min(t.t0 + TR_, t.x1) - 1 - P) + V - 1;
    t.X0 = max(0, t.x0 - P);
    t.ulo = t.t0 == t.x0 ? t.X0 : min(N - 1, t.t0 - 1 + P) + 1;
    t.uhi = min(N - 1, min(t.t0 + TR_, t.x1) - 1 + P);
}

template <int P>
__device__ __forceinline__ void it_line(const LineArgs& a, TileIt& t) {
    t.i2 = t.line % a.Ny;
    t.i3 = t.line / a.Ny;
    t.x0 = max(a.row_begin, t.line * a.N) - t.line * a.N;
    t.x1 = min(a.row_end, t.line * a.N + a.N) - t.line * a.N;
    t.t0 = t.x0;
}

template <int P, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ void it_init(const LineArgs& a, TileIt& t) {
    t.line = a.row_begin / a.N + blockIdx.x;
    t.nchg = 0;
    t.pending = false;
    t.qs = 0;
    t.ps = 0;
    t.lpos = 0;
    it_line<P>(a, t);
    it_planes<P, TR_>(t, a.N);
}

template <int P, int PFD_ = Cfg<P>::PFD, int URING_ = ApplyCfg::URING, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ void it_next(const LineArgs& a, TileIt& t) {
    t.t0 += TR_;
    t.ps = t.ps == PFD_ - 1 ? 0 : t.ps + 1;
    if (t.t0 >= t.x1) {
        t.lpos = (t.lpos + min(a.N - 1, t.x1 - 1 + P) - t.X0 + 1) % URING_;   // finished line's columns
        t.line += gridDim.x;
        t.qs = t.qs == PFD_ - 1 ? 0 : t.qs + 1;
        it_line<P>(a, t);
    }
    it_planes<P, TR_>(t, a.N);
}

// Ticketed line order (assembly): the first line of CTA b is line b of the range, each further
// line is the next unclaimed one (a global atomic counter), so the lines in flight stay the
// ~gridDim most recent ones and the write stream advances through memory as one front (a static
// round-robin order lets the CTAs drift apart: 6.4 vs 7.3 TB/s for the same bulk stores,
// tools/write_probe3.cu).  Thread 0 claims the next line when the iterator leaves a line and
// publishes it in s_line[nchg & 1]; every thread picks it up after the next block barrier
// (it_resolve).  Two slots: a slot is rewritten two line changes later, after a barrier that
// every reader of its previous value has passed.
template <int P, int PFD_ = Cfg<P>::PFD, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ void it_next_ticket(const LineArgs& a, TileIt& t, int* s_line, int tid) {
    t.t0 += TR_;
    t.ps = t.ps == PFD_ - 1 ? 0 : t.ps + 1;
    if (t.t0 >= t.x1) {
        if (tid == 0)
            s_line[t.nchg & 1] = a.row_begin / a.N + (int)gridDim.x + (int)atomicAdd(a.ticket, 1ull);
        t.pending = true;
        t.qs = t.qs == PFD_ - 1 ? 0 : t.qs + 1;
    } else {
        it_planes<P, TR_>(t, a.N);
    }
}
template <int P, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ void it_resolve(const LineArgs& a, TileIt& t, const int* s_line) {
    if (!t.pending) return;
    t.line = s_line[t.nchg & 1];
    ++t.nchg;
    t.pending = false;
    it_line<P>(a, t);
    it_planes<P, TR_>(t, a.N);
}

// Issue (cp.async, one commit group) everything tile t reads from global memory: its new
// vertex planes into patch buffer t.ps and, for a line's first tile, the line's y/z vertex
// tables into Q buffer t.qs (and the thread's patch row).  An exhausted iterator commits an
// empty group.
template <int P, int NT = Cfg<P>::NT, int PATCH_ = Cfg<P>::PATCH>
__device__ __forceinline__ void tile_issue(const LineArgs& a, double* patches, double* qbufs, const TileIt& t,
                                           PatchRow& pr, int last_line, int tid) {
    using C = Cfg<P>;
    constexpr int V = C::V, S = C::S;
    if (t.line <= last_line) {
        if (t.t0 == t.x0) {
            patch_row_init<P>(a, pr, t.i2, t.i3, tid);
            double* Q = qbufs + t.qs * (4 * V * S);
            for (int e = tid; e < 4 * V * S; e += NT) {
                const int which = e / (V * S), v = (e / S) % V, o = e % S;
                const int r = which < 2 ? t.i2 : t.i3;
                const RowTables& TL = which < 2 ? a.Ty : a.Tz;
                cp_async8(Q + e, ((which & 1) ? TL.PK : TL.PM) + ((size_t)r * kMaxV + v) * kMaxS + o, true);
            }
        }
        load_patch<P>(a, pr, patches + t.ps * PATCH_, t.lo, t.hi - t.lo + 1, tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// CSR structure in closed form: a(r) = structural columns of 1D row r,
// A(r) = sum_{r' < r} a(r'), S = A(N); row (i1,i2,i3) starts at A(i3) S^2 + a(i3)(A(i2) S + a(i2) A(i1)).
__host__ __device__ __forceinline__ long long csr_a(long long r, int p, long long N) {
    return (r + p < N - 1 ? r + p : N - 1) - (r - p > 0 ? r - p : 0) + 1;
}
__host__ __device__ __forceinline__ long long csr_A(long long r, int p, long long N) {
    const long long m = r < p ? r : p, q = r - (N - p) > 0 ? r - (N - p) : 0;
    return (2 * p + 1) * r - (m * p - m * (m - 1) / 2) - q * (q + 1) / 2;
}
// per-direction sizes: S_a = A_a(N_a), start = A_z(i3) S_y S_x + a_z(i3) (A_y(i2) S_x + a_y(i2) A_x(i1))
__host__ __device__ __forceinline__ long long csr_start3(long long i1, long long i2, long long i3, int p, long long Nx,
                                                          long long Ny, long long Nz) {
    const long long Sx = csr_A(Nx, p, Nx), Sy = csr_A(Ny, p, Ny);
    return csr_A(i3, p, Nz) * Sy * Sx + csr_a(i3, p, Nz) * (csr_A(i2, p, Ny) * Sx + csr_a(i2, p, Ny) * csr_A(i1, p, Nx));
}
__host__ __device__ __forceinline__ long long csr_start(long long row, int p, long long Nx, long long Ny, long long Nz) {
    return csr_start3(row % Nx, (row / Nx) % Ny, row / (Nx * Ny), p, Nx, Ny, Nz);
}

// What every warp needs to know about a tile; written by thread 0 when the tile is prefetched.
struct TileDesc {
    int line;          // -1: past the CTA's last tile
    int t0, tr;        // first x-row, rows in the tile
    int lo, nnew;      // new vertex planes [lo, lo + nnew) for phase A
    int ps, qs;        // patch / Q buffers
    int pad;           // staging offset aligning the tile's first element
    long long orow0;   // output row of the tile's first row
    int Xlo, Xhi, upos;  // apply: the tile's u columns [Xlo, Xhi], ring position of Xlo
};

// CSR output only: slab-local position of the tile's first entry, entries per x-row unit
// (a2 a3), the y/z validity boxes (offset indices lo..hi of the 2p+1) and a2.  Kept apart
// from TileDesc so the ELL and apply kernels do not carry it.
struct TileCsr {
    long long cs0;
    int w23, lo2, hi2, lo3, hi3, a2;
};

template <int P>
__device__ __forceinline__ TileCsr make_csr(const LineArgs& a, const TileIt& t, int last_line) {
    TileCsr d{};
    if (t.line <= last_line) {
        d.cs0 = csr_start3(t.t0, t.i2, t.i3, P, a.N, a.Ny, a.Nz) - a.csr_base;   // no divisions on thread 0's path
        d.a2 = (int)csr_a(t.i2, P, a.Ny);
        d.w23 = d.a2 * (int)csr_a(t.i3, P, a.Nz);
        d.lo2 = max(0, P - t.i2);
        d.hi2 = min(2 * P, a.Ny - 1 - t.i2 + P);
        d.lo3 = max(0, P - t.i3);
        d.hi3 = min(2 * P, a.Nz - 1 - t.i3 + P);
    }
    return d;
}

template <int P, int URING_ = ApplyCfg::URING, int TR_ = Cfg<P>::TR>
__device__ __forceinline__ TileDesc make_desc(const LineArgs& a, const TileIt& t, int last_line, bool padded) {
    TileDesc d;
    d.line = t.line <= last_line ? t.line : -1;
    d.t0 = t.t0;
    d.tr = min(TR_, t.x1 - t.t0);
    d.lo = t.lo;
    d.nnew = t.hi - t.lo + 1;
    d.ps = t.ps;
    d.qs = t.qs;
    d.orow0 = (long long)t.line * a.N + t.t0 - a.row_begin;
    d.pad = padded ? 0 : (int)((d.orow0 * a.ld) & 1);
    d.Xlo = max(0, t.t0 - P);
    d.Xhi = t.uhi;
    d.upos = (t.lpos + d.Xlo - t.X0) % URING_;
    return d;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Phase A of tile t on the FP64 tensor cores (DMMA m8n8k4), one warp per new vertex plane c:
//   A1:  TT_X[o2][vz] = sum_vy Qy_X[vy][o2] g[bz+vz][by+vy][c]      (X = M, K)
//   A2:  HM[o2][o3]  = sum_vz TT_M[o2][vz] Qz_M[vz][o3]
//        HK[o2][o3]  = sum_vz TT_K[o2][vz] Qz_M[vz][o3] + TT_M[o2][vz] Qz_K[vz][o3]
// Fragments (lane = 4 g + t): A[g][t], B[t][g], C[g][2t+i].  The A1 output columns are
// permuted, column 2t+i <-> vz = t + 4i, so each lane ends A1 holding exactly its A2 A-fragment
// (TT[g][t], TT[g][t+4]): no shuffle or shared-memory round trip between the two products.
// Padding rows / columns (o2, o3 >= S, vy, vz >= V) carry zero coefficients.
template <int P, int NT = Cfg<P>::NT, int HS = Cfg<P>::S2, int RING = Cfg<P>::RING, int PATCH_ = Cfg<P>::PATCH>
__device__ __forceinline__ void phase_a(const LineArgs& a, const TileDesc& t, const double* patches,
                                        const double* qbufs, double* Hm, double* Hk, int tid) {
    using C = Cfg<P>;
    constexpr int V = C::V, S = C::S;
    constexpr int KS = (V + 3) / 4;                    // k-steps of 4 (p=3: 2, p=2: 1)
    constexpr int NW = NT / 32;
    const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, tq = lane & 3;
    const double* Q = qbufs + t.qs * (4 * V * S);
    double aYM[KS], aYK[KS], bZM[KS], bZK[KS];
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        const int v = tq + 4 * s;
        const bool ok = g < S && v < V;
        const int e = ok ? v * S + g : 0;
        aYM[s] = ok ? Q[e] : 0.0;
        aYK[s] = ok ? Q[V * S + e] : 0.0;
        bZM[s] = ok ? Q[2 * V * S + e] : 0.0;
        bZK[s] = ok ? Q[3 * V * S + e] : 0.0;
    }
    const double* patch = patches + t.ps * PATCH_;
    const int nnew = t.nnew;
    const int vzp = (g >> 1) + 4 * (g & 1);            // B column g of A1 <-> vz = pi(g)
    for (int j = NW - 1 - warp; j < ((a.dbg & 65) ? 0 : nnew); j += NW) {
        double tM0 = 0.0, tM1 = 0.0, tK0 = 0.0, tK1 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int vy = tq + 4 * s;
            const double b = (vzp < V && vy < V) ? patch[(j * V + vzp) * V + vy] : 0.0;
            dmma(tM0, tM1, aYM[s], b);
            dmma(tK0, tK1, aYK[s], b);
        }
        // lane holds TT_X[o2 = g][vz = tq] (x0) and TT_X[g][tq + 4] (x1)
        double hM0 = 0.0, hM1 = 0.0, hK0 = 0.0, hK1 = 0.0;
        dmma(hM0, hM1, tM0, bZM[0]);
        dmma(hK0, hK1, tK0, bZM[0]);
        dmma(hK0, hK1, tM0, bZK[0]);
        if (KS > 1) {
            dmma(hM0, hM1, tM1, bZM[KS - 1]);
            dmma(hK0, hK1, tK1, bZM[KS - 1]);
            dmma(hK0, hK1, tM1, bZK[KS - 1]);
        }
        const int slot = ring_slot<RING>(t.lo + j);
        const int o3 = 2 * tq;
        if (g < S) {
            double* hm = Hm + slot * HS + g;
            double* hk = Hk + slot * HS + g;
            if (o3 < S) {
                hm[S * o3] = hM0;
                hk[S * o3] = hK0;
            }
            if (o3 + 1 < S) {
                hm[S * (o3 + 1)] = hM1;
                hk[S * (o3 + 1)] = hK1;
            }
        }
    }
}

// Bulk store of a contiguous run of `total` values staged from st (st is offset so that the run's
// first element keeps its global 16-byte phase), by warp 0, without the commit.
__device__ __forceinline__ void store_run(double* out, const double* st, long long g0, int total, int lane) {
    const int head = (int)(g0 & 1);
    const int tail = (int)((g0 + total) & 1);
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (total - head - tail > 0) bulk_store(out + g0 + head, st + head, (uint32_t)(total - head - tail) * 8u);
    } else if (lane == 1 && head) {
        out[g0] = st[0];
    } else if (lane == 2 && tail && total > head) {
        out[g0 + total - 1] = st[total - 1];
    }
}

// Bulk store of one matrix of the staged tile (tr rows from output row orow0), by warp 0,
// without the commit: lane 0 issues the 16-byte aligned interior as one cp.async.bulk, lanes
// 1 / 2 the peeled odd end elements; padded even ld: one bulk copy per row (lane 0) and the
// rows' odd last elements (lanes 1..tr).
template <int P>
__device__ __forceinline__ void store_mat(const LineArgs& a, double* out, const double* st, long long orow0, int tr,
                                          int SRr, bool padded, int lane) {
    constexpr int S3 = Cfg<P>::S3;
    const long long g0 = orow0 * a.ld;
    if (!padded) {
        const int total = tr * S3;
        const int head = (int)(g0 & 1);
        const int tail = (int)((g0 + total) & 1);
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_store(out + g0 + head, st + head, (uint32_t)(total - head - tail) * 8u);
        } else if (lane == 1 && head) {
            out[g0] = st[0];
        } else if (lane == 2 && tail) {
            out[g0 + total - 1] = st[total - 1];
        }
    } else {
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int j = 0; j < tr; ++j) bulk_store(out + (orow0 + j) * a.ld, st + j * SRr, (uint32_t)(S3 - 1) * 8u);
        } else if (lane <= tr) {
            const int j = lane - 1;
            out[(orow0 + j) * a.ld + S3 - 1] = st[j * SRr + S3 - 1];
        }
    }
}

template <int P, int MODE, bool CSR>
__global__ void __launch_bounds__(Cfg<P>::NT, 2) k_line_grid3(const __grid_constant__ LineArgs a) {
    using C = Cfg<P>;
    constexpr int S = C::S, S2 = C::S2, S3 = C::S3, V = C::V, RING = C::RING;
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;                                   // [2 mat][STAGE] (single buffer)
    double* Hm = stage + 2 * C::STAGE;                    // [RING][S2]
    double* Hk = Hm + RING * S2;                          // [RING][S2]
    double* qbufs = Hk + RING * S2;                       // [PFD][QyM, QyK, QzM, QzK: [V][S] each]
    double* patches = qbufs + C::PFD * 4 * V * S;         // [PFD][W][V(z)][V(y)]
    double* xbt = patches + C::PFD * C::PATCH;            // [4P rows][PM, PK][V][S]

    __shared__ TileDesc desc[8];                          // tiles k .. k+PFD (ring)
    __shared__ TileCsr cdesc[CSR ? 8 : 1];
    __shared__ int s_line[2];                             // ticketed line order (it_next_ticket)
    constexpr int PFD = C::PFD;
    const int tid = threadIdx.x;
    const int n = a.n;
    const bool padded = a.ld != S3;
    const int SRr = padded ? C::SR : S3;
    const int last_line = (a.row_end - 1) / a.N;
    // fixed per-thread role in phase B: item (row pair q, o23)
    const int q = tid / S2, o23 = tid % S2;

    // Software pipeline, two barriers per tile:
    //   S1(k): phase B of tile k (H -> staging)
    //   S2(k): bulk store of tile k  +  phase A of tile k+1 (patch -> H ring)  +  prefetch k+PFD
    // The H ring holds a tile's window (W planes) and the next tile's new planes are written
    // only after that tile's phase B (S2 follows S1), so RING >= W suffices.  Global loads are
    // issued PFD tiles ahead: under saturated HBM writes their latency is several microseconds.
    // One tile iterator (the prefetch one) runs in every thread; thread 0 publishes each
    // prefetched tile's descriptor for phases A and B.
    // x-boundary rows r < 2P and r >= n-P: their vertex tables, once per CTA
    for (int e = tid; e < C::XB; e += C::NT) {
        const int i = e / (2 * V * S), rem = e % (2 * V * S), kind = rem / (V * S), v = (rem / S) % V, o = rem % S;
        const int r = i < 2 * P ? i : n - P + (i - 2 * P);
        xbt[e] = (kind ? a.T.PK : a.T.PM)[((size_t)r * kMaxV + v) * kMaxS + o];
    }
    if (a.dbg & 256) {      // profiling: staging holds fixed high-entropy values (with bit 1: stores only)
        for (int e = tid; e < 2 * C::STAGE; e += C::NT) {
            unsigned long long z = (unsigned long long)(e + 1) * 0x9E3779B97F4A7C15ull;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            stage[e] = 1.0 + (double)(z >> 11) * 0x1.0p-53;
        }
    }
    auto xb_row = [&](int r) -> const double* {
        return xbt + (r < 2 * P ? r : 2 * P + (r - (n - P))) * (2 * V * S);
    };
    TileIt itP;
    PatchRow prow;
    prow.base = nullptr;
    it_init<P>(a, itP);
    const bool ticketed = a.ticket != nullptr;
    auto advance = [&]() {
        if (itP.line > last_line) return;
        if (ticketed) it_next_ticket<P>(a, itP, s_line, tid);
        else it_next<P>(a, itP);
    };
    for (int k = 0; k < PFD; ++k) {
        tile_issue<P>(a, patches, qbufs, itP, prow, last_line, tid);
        if (tid == 0) desc[k] = make_desc<P>(a, itP, last_line, padded);
        if (CSR && tid == 0) cdesc[k & (CSR ? 7 : 0)] = make_csr<P>(a, itP, last_line);
        advance();
        if (ticketed) {
            __syncthreads();
            it_resolve<P>(a, itP, s_line);
        }
    }
    cp_async_wait<PFD - 1>();                             // tile 0 landed
    __syncthreads();
    {
        const TileDesc d0 = desc[0];
        if (d0.line >= 0) phase_a<P>(a, d0, patches, qbufs, Hm, Hk, tid);
    }
    cp_async_wait<PFD - 2>();                             // tile 1 landed
    __syncthreads();

    for (int k = 0;; ++k) {
        it_resolve<P>(a, itP, s_line);                    // the line claimed last iteration (ticketed)
        const TileDesc d = desc[k & 7];
        if (d.line < 0) break;
        const TileDesc dA = desc[(k + 1) & 7];
        TileCsr dc{};
        if (CSR) dc = cdesc[k & (CSR ? 7 : 0)];
        const int pad = CSR ? (int)(dc.cs0 & 1) : d.pad;
        double* stM = stage + pad;
        double* stK = stage + C::STAGE + pad;
        // ---- S1: phase B of tile k ---------------------------------------------------------
        if (tid < C::ITEMS && 2 * q < d.tr && !(a.dbg & 129)) {
            const int j = 2 * q, r = d.t0 + j;
            const int b0 = max(0, r - P);
            double hm[V + 1], hk[V + 1];
#pragma unroll
            for (int v = 0; v <= V; ++v) {             // planes b0 .. b0+V (the pair's union)
                const int slot = ring_slot<RING>(b0 + v);
                hm[v] = Hm[slot * S2 + o23];
                hk[v] = Hk[slot * S2 + o23];
            }
            const bool second = j + 1 < d.tr;
            const bool shift = r + 1 - P > 0;          // row r+1's window starts one plane later
            if (!CSR) {
                double* dM = stM + j * SRr + S * o23;
                double* dK = stK + j * SRr + S * o23;
                if (r >= 2 * P && r + 1 <= n - 1 - P) {   // both rows class I (the common case)
                    finish_pair_interior<P, MODE>(hm, hk, dM, dK, SRr, second, a);
                } else {
                    if (r >= 2 * P && r <= n - 1 - P) finish_interior<P, MODE>(hm, hk, dM, dK, a);
                    else finish_general<P, MODE>(xb_row(r), hm, hk, dM, dK);
                    if (second) {
                        double hm1[V], hk1[V];
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            hm1[v] = shift ? hm[v + 1] : hm[v];
                            hk1[v] = shift ? hk[v + 1] : hk[v];
                        }
                        if (r + 1 >= 2 * P && r + 1 <= n - 1 - P) finish_interior<P, MODE>(hm1, hk1, dM + SRr, dK + SRr, a);
                        else finish_general<P, MODE>(xb_row(r + 1), hm1, hk1, dM + SRr, dK + SRr);
                    }
                }
            } else {
                // CSR: row r's entries start at w23 (A(r) - A(t0)) in the tile; the thread's (o2, o3)
                // group sits at pos23 = (o2 - lo2) + a2 (o3 - lo3) if inside the mesh, its o1 at o1 - lo1(r)
                const int o2 = o23 % S, o3 = o23 / S;
                if (o2 >= dc.lo2 && o2 <= dc.hi2 && o3 >= dc.lo3 && o3 <= dc.hi3) {
                    const int pos23 = (o2 - dc.lo2) + dc.a2 * (o3 - dc.lo3);
                    if (r >= 2 * P && r + 1 <= n - 1 - P && d.t0 >= P) {
                        // both rows class I and every row from t0 on has a(.) = 2p+1 columns:
                        // A(r) - A(t0) = (2p+1)(r - t0), lo1 = 0
                        const int off0 = dc.w23 * S * (r - d.t0);
                        finish_pair_interior<P, MODE>(hm, hk, stM + off0 + S * pos23, stK + off0 + S * pos23, S * dc.w23,
                                                      second, a);
                    } else if (r >= 2 * P && r + 1 <= n - 1 - P) {
                        const int off0 = (int)(dc.w23 * (csr_A(r, P, a.N) - csr_A(d.t0, P, a.N)));
                        finish_pair_interior<P, MODE>(hm, hk, stM + off0 + S * pos23, stK + off0 + S * pos23, S * dc.w23,
                                                      second, a);
                    } else {
                        const long long At0 = csr_A(d.t0, P, a.N);
                        const int off0 = (int)(dc.w23 * (csr_A(r, P, a.N) - At0));
                        const int ar0 = (int)csr_a(r, P, a.N);
                        const int lo1 = max(0, P - r), hi1 = min(2 * P, a.N - 1 - r + P);
                        double* dM = stM + off0 + ar0 * pos23 - lo1;
                        double* dK = stK + off0 + ar0 * pos23 - lo1;
                        if (r >= 2 * P && r <= n - 1 - P) finish_interior<P, MODE>(hm, hk, dM, dK, a);
                        else finish_general<P, MODE>(xb_row(r), hm, hk, dM, dK, lo1, hi1);
                        if (second) {
                            const int r1 = r + 1;
                            double hm1[V], hk1[V];
#pragma unroll
                            for (int v = 0; v < V; ++v) {
                                hm1[v] = shift ? hm[v + 1] : hm[v];
                                hk1[v] = shift ? hk[v + 1] : hk[v];
                            }
                            const int off1 = (int)(dc.w23 * (csr_A(r1, P, a.N) - At0));
                            const int lo1b = max(0, P - r1), hi1b = min(2 * P, a.N - 1 - r1 + P);
                            double* dM1 = stM + off1 + (int)csr_a(r1, P, a.N) * pos23 - lo1b;
                            double* dK1 = stK + off1 + (int)csr_a(r1, P, a.N) * pos23 - lo1b;
                            if (r1 >= 2 * P && r1 <= n - 1 - P) finish_interior<P, MODE>(hm1, hk1, dM1, dK1, a);
                            else finish_general<P, MODE>(xb_row(r1), hm1, hk1, dM1, dK1, lo1b, hi1b);
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ---- S2: store tile k, phase A of tile k+1, prefetch tile k+3 --------------------
        if (tid < 32 && !(a.dbg & 2)) {
            if (CSR) {
                const long long total = (long long)dc.w23 * (csr_A(d.t0 + d.tr, P, a.N) - csr_A(d.t0, P, a.N));
                if (MODE & 1) store_run(a.M, stM, dc.cs0, (int)total, tid);
                if (MODE & 2) store_run(a.K, stK, dc.cs0, (int)total, tid);
            } else {
                if (MODE & 1) store_mat<P>(a, a.M, stM, d.orow0, d.tr, SRr, padded, tid);
                if (MODE & 2) store_mat<P>(a, a.K, stK, d.orow0, d.tr, SRr, padded, tid);
            }
            if (tid == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (dA.line >= 0) phase_a<P>(a, dA, patches, qbufs, Hm, Hk, tid);
        if (a.dbg & 4) asm volatile("cp.async.commit_group;" ::: "memory");
        else tile_issue<P>(a, patches, qbufs, itP, prow, last_line, tid);    // tile k+PFD
        if (tid == 0) desc[(k + PFD) & 7] = make_desc<P>(a, itP, last_line, padded);
        if (CSR && tid == 0) cdesc[(k + PFD) & (CSR ? 7 : 0)] = make_csr<P>(a, itP, last_line);
        advance();
        cp_async_wait<PFD - 2>();                                  // tile k+2 landed
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging free
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------
// Matrix-free application y = A u on the GRID line structure.
//
// Row i of M is sum_vx PMx[vx][o1] HM[bx+vx][o2,o3] (the assembly's phase B), so
//   y^M_i = sum_{vx,o1} PMx[vx][o1] D_M(bx+vx, i1-p+o1),   D_X(c, X) = sum_{o2,o3} H_X[c][o2,o3] u[X][i2-p+o2][i3-p+o3]
//   y^K_i = sum_{vx,o1} PKx[vx][o1] D_M(..) + PMx[vx][o1] D_K(..)
// — the definition y_i = sum_j A_ij u_j with the sums reordered.  Per tile of TRA rows (24:
// the per-tile iterator / descriptor / barrier cost is spread over three times the rows of the
// assembly's tiles, at 2 CTAs per SM) the D values for the (vertex plane c, column X) pairs of
// the tile's window are a banded (32 x 49) x (49 x 32) product per matrix on the FP64 tensor
// cores (the 10 of 16 8x8 blocks with |X - c| <= 1 block, DMMA m8n8k4 items of 13 k-steps);
// the H planes come from the assembly's phase A, the u columns X (49 values each) are
// prefetched with the vertex patches into a ring.  Nothing is stored but y.
// Band of the apply's D product on DFMA: D_X(c, X) = sum_k H_X[c][k] U[X][k] for the tile
// planes c = b0 + i (i = 8 pb + g) and the diagonals X - c = D0 .. D0 + ND - 1 (the structural
// band of the x-direction tables is X - c in [-1, p]: a node of element e touches vertex planes
// e, e+1 and columns e .. e+p).  Lane (g, t4) accumulates k = t4 (mod 4) — the operand rows are
// read in the DMMA fragment pattern, conflict-free — and the four partial sums are combined by
// shuffles.  Both matrices share the U operands.
template <int P, int D0, int ND, int HS, int RING, int URING>
__device__ __forceinline__ void d_band(const double* Hm, const double* Hk, const double* U, const double* zrow,
                                       double* Dm, double* Dk, int DC, int DR, int b0, int hi_plane, int Xhi,
                                       int upos0, int pb, int g, int t4) {
    constexpr int S2 = (2 * P + 1) * (2 * P + 1), KSD = (S2 + 3) / 4;
    const int i = 8 * pb + g, c = b0 + i;
    const bool cv = c <= hi_plane;
    const double* hm = (cv ? Hm + ring_slot<RING>(c) * HS : zrow) + t4;
    const double* hk = (cv ? Hk + ring_slot<RING>(c) * HS : zrow) + t4;
    const double* ur[ND];
#pragma unroll
    for (int q = 0; q < ND; ++q) {
        const int j = i + D0 + q;                          // X - Xlo (Xlo = b0)
        const bool xv = j >= 0 && b0 + j <= Xhi;
        int up = upos0 + j;
        up = up >= URING ? up - URING : up;
        ur[q] = (xv ? U + up * HS : zrow) + t4;
    }
    double am[ND], ak[ND];
#pragma unroll
    for (int q = 0; q < ND; ++q) am[q] = ak[q] = 0.0;
#pragma unroll
    for (int s = 0; s < KSD; ++s) {
        const double hmv = hm[4 * s], hkv = hk[4 * s];
#pragma unroll
        for (int q = 0; q < ND; ++q) {
            const double uv = ur[q][4 * s];
            am[q] = fma(hmv, uv, am[q]);
            ak[q] = fma(hkv, uv, ak[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < ND; ++q) {
        am[q] += __shfl_xor_sync(0xffffffffu, am[q], 1);
        ak[q] += __shfl_xor_sync(0xffffffffu, ak[q], 1);
        am[q] += __shfl_xor_sync(0xffffffffu, am[q], 2);
        ak[q] += __shfl_xor_sync(0xffffffffu, ak[q], 2);
        const int j = i + D0 + q;
        if (t4 == (q & 3) && i < DR && j >= 0 && j < DC) {
            Dm[i * DC + j] = am[q];
            Dk[i * DC + j] = ak[q];
        }
    }
}

// Tile geometry of the apply for TRA rows per tile: the vertex-plane window (TRA + p + 1 planes,
// H ring RING_A >= that), the D product's plane x column blocks of 8 (only blocks within the band
// |column - plane| <= 1 block carry nonzero P^ weights), the u ring (the next tile's window of
// TRA + 2p columns plus PFD - 1 further tiles of up to TRA + 2p new columns).
template <int P, int TRA>
struct ApplyGeom {
    static constexpr int V = P + 2, S = 2 * P + 1, S2 = S * S;
    static constexpr int W = TRA + V - 1;                              // planes of a tile's window
    static constexpr int RING = W <= 16 ? 16 : (W <= 32 ? 32 : 64);   // power of two >= W
    static constexpr int PATCH = W * V * V;
    static constexpr int PFD = ApplyCfg::PFD;
    static constexpr int DB = (W + 7) / 8;                             // plane blocks of D
    static constexpr int XBK = (TRA + 2 * P + 7) / 8;                  // column blocks of D
    // D extents; the row stride DC = 4 (mod 8) doubles keeps the finishing stage's reads (lanes
    // (row, vertex plane): consecutive rows step one column and one D row) conflict-free
    static constexpr int DR = DB * 8, DC = XBK * 8 + 4;
    static constexpr int UXMAX = (TRA + 2 * P + 7) / 8 * 8;            // new columns per tile (a slab's first
                                                                       // tile may start mid-line: TRA + 2p)
    // live columns when tile k+PFD is issued: tile k+1's window and the new columns of k+2..k+PFD
    // (at most TRA + 2p each: a tile that starts a slab inside a line)
    static constexpr int URING = TRA == 8 ? ApplyCfg::URING : PFD * (TRA + 2 * P) + 1;
    static constexpr int HS = (S2 + 3) / 4 * 4 + ((S2 + 3) / 4 % 2 == 0 ? 4 : 0);   // row stride = 4 (mod 8)
    static constexpr size_t smem_doubles() {
        return (size_t)2 * RING * HS + PFD * 4 * V * S + PFD * PATCH + 4 * P * 2 * V * S + (size_t)URING * HS +
               2 * DR * DC + 2 * V * S + HS;
    }
};

#ifndef WGQ_APPLY_THREADS
#define WGQ_APPLY_THREADS 256
#endif
constexpr int kApplyThreads = WGQ_APPLY_THREADS;

template <int P, int MODE, int TRA>
__global__ void __launch_bounds__(kApplyThreads, TRA == 8 ? 3 : 2) k_line_apply(const __grid_constant__ LineArgs a) {
    using C = Cfg<P>;
    using G = ApplyGeom<P, TRA>;
    constexpr int S = C::S, S2 = C::S2, V = C::V, RING = G::RING, URING = G::URING, PFD = G::PFD;
    constexpr int NT = kApplyThreads, NW = NT / 32;
    constexpr int HS = G::HS, DC = G::DC;
    extern __shared__ __align__(128) double sm[];
    double* Hm = sm;                                      // [RING][HS]
    double* Hk = Hm + RING * HS;
    double* qbufs = Hk + RING * HS;                       // [PFD][4][V][S]
    double* patches = qbufs + PFD * 4 * V * S;            // [PFD][W][V][V]
    double* xbt = patches + PFD * G::PATCH;               // [4P][2][V][S]
    double* U = xbt + C::XB;                              // [URING][HS]
    double* Dm = U + URING * HS;                          // [DR][DC]  D_M(c - b0, X - Xlo)
    double* Dk = Dm + G::DR * DC;
    double* pint = Dk + G::DR * DC;                       // [2][V][S]: interior P^ (h, 1/h folded)
    double* zrow = pint + 2 * V * S;                      // [HS] zeros: operand row of invalid planes / columns
    __shared__ TileDesc desc[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.n, N = a.N;
    const int last_line = (a.row_end - 1) / N;
    for (int e = tid; e < C::XB; e += NT) {
        const int i = e / (2 * V * S), rem = e % (2 * V * S), kind = rem / (V * S), v = (rem / S) % V, o = rem % S;
        const int r = i < 2 * P ? i : n - P + (i - 2 * P);
        xbt[e] = (kind ? a.T.PK : a.T.PM)[((size_t)r * kMaxV + v) * kMaxS + o];
    }
    for (int e = tid; e < 2 * V * S; e += NT) pint[e] = e < V * S ? a.PMh[e / S][e % S] : a.PKi[(e - V * S) / S][e % S];
    // zero rows and the padding columns [S2, HS) of the H and U rows: the D fragments then need no masks
    for (int e = tid; e < HS; e += NT) zrow[e] = 0.0;
    // D entries off the band are never written and stay zero (their x tables are structural zeros)
    for (int e = tid; e < 2 * G::DR * DC; e += NT) Dm[e] = 0.0;
    for (int e = tid; e < (2 * RING + URING) * (HS - S2); e += NT) {
        const int row = e / (HS - S2), col = S2 + e % (HS - S2);
        (row < 2 * RING ? Hm + row * HS : U + (row - 2 * RING) * HS)[col] = 0.0;
    }
    // u loads: thread tid owns elements e = tid + NT m (m < MU) of a tile's new columns, laid
    // out as [x-offset block][o23][x-offset & 7] so a warp reads contiguous runs along X; the
    // (o23, x-offset) of each element is fixed, its global row offset changes once per line
    constexpr int MU = (G::UXMAX * S2 + NT - 1) / NT;
    int uxo[MU], uo23[MU];
    long long ubase[MU];
#pragma unroll
    for (int m = 0; m < MU; ++m) {
        const int e = tid + NT * m;
        uxo[m] = (e & 7) + 8 * (e / (8 * S2));
        uo23[m] = (e >> 3) % S2;
        ubase[m] = -1;
    }
    auto issue = [&](const TileIt& t, PatchRow& pr) {
        if (t.line <= last_line) {
            if (t.t0 == t.x0) {                                // new line: the rows' global offsets
                const long long N2 = (long long)N * a.Ny;
#pragma unroll
                for (int m = 0; m < MU; ++m) {
                    const int o2 = uo23[m] % S, o3 = uo23[m] / S;
                    const int iy = t.i2 - P + o2, iz = t.i3 - P + o3;
                    ubase[m] = (iy >= 0 && iy < a.Ny && iz >= 0 && iz < a.Nz) ? (long long)iz * N2 + (long long)iy * N - a.u_row0
                                                                              : -1;
                }
            }
            const int nx = (a.dbg & 16) ? 0 : t.uhi - t.ulo + 1;
            const int p0 = (t.lpos + t.ulo - t.X0) % URING;            // ring position of column ulo
#pragma unroll
            for (int m = 0; m < MU; ++m) {
                if (uxo[m] >= nx || uxo[m] >= G::UXMAX) continue;
                const int X = t.ulo + uxo[m];
                const bool ok = ubase[m] >= 0;
                int pos = p0 + uxo[m];
                pos = pos >= URING ? pos - URING : pos;
                cp_async8(U + pos * HS + uo23[m], a.u + (ok ? ubase[m] + X : 0), ok);
            }
        }
        tile_issue<P, NT, G::PATCH>(a, patches, qbufs, t, pr, last_line, tid);     // commits the group
    };
    TileIt itP;
    PatchRow prow;
    prow.base = nullptr;
    it_init<P, TRA>(a, itP);
    for (int k = 0; k < PFD; ++k) {
        issue(itP, prow);
        if (tid == 0) desc[k] = make_desc<P, URING, TRA>(a, itP, last_line, false);
        if (itP.line <= last_line) it_next<P, PFD, URING, TRA>(a, itP);
    }
    cp_async_wait<PFD - 1>();
    __syncthreads();
    {
        const TileDesc d0 = desc[0];
        if (d0.line >= 0) phase_a<P, NT, HS, RING, G::PATCH>(a, d0, patches, qbufs, Hm, Hk, tid);
    }
    cp_async_wait<PFD - 2>();
    __syncthreads();
    const int g = lane >> 2, t4 = lane & 3;
    for (int k = 0;; ++k) {
        const TileDesc d = desc[k & 7];
        if (d.line < 0) break;
        const TileDesc dA = desc[(k + 1) & 7];
        const int b0 = max(0, d.t0 - P);
        const int hi_plane = max(0, d.t0 + d.tr - 1 - P) + V - 1;
        // ---- S1a: D_X = H_X (planes b0..) x U (columns Xlo..) on the band X - c in [-1, p] --
        // items (plane block of 8, diagonal half): diagonals -1 .. NDA - 2 and NDA - 1 .. p
        {
            constexpr int ND = P + 2, NDA = (ND + 1) / 2;
            for (int it = warp; it < 2 * G::DB; it += NW) {
                if (a.dbg & 8) break;
                if (it & 1)
                    d_band<P, NDA - 1, ND - NDA, HS, RING, URING>(Hm, Hk, U, zrow, Dm, Dk, DC, G::DR, b0, hi_plane,
                                                                   d.Xhi, d.upos, it >> 1, g, t4);
                else
                    d_band<P, -1, NDA, HS, RING, URING>(Hm, Hk, U, zrow, Dm, Dk, DC, G::DR, b0, hi_plane, d.Xhi,
                                                         d.upos, it >> 1, g, t4);
            }
        }
        __syncthreads();
        // ---- S1b: rows of tile k, phase A of tile k+1, prefetch tile k+PFD ------------------
        if (warp < (TRA + 7) / 8 && !(a.dbg & 32)) {
            // warp w finishes rows 8w..8w+7 of the tile: lane (j, vq) = row t0 + 8w + j, vertex
            // planes vx = vq (+4); y = sum_{vx,o1} P[vx][o1] D(b_r + vx, r - p + o1), over 4 lanes
            const int j = 8 * warp + (lane >> 2), vq = lane & 3;
            double ym = 0.0, yk = 0.0;
            if (j < d.tr) {
                const int r = d.t0 + j, br = max(0, r - P);
                const bool interior = r >= 2 * P && r <= n - 1 - P;
                const double* pm = interior ? pint : xbt + (r < 2 * P ? r : 2 * P + (r - (n - P))) * (2 * V * S);
                const double* pk = pm + V * S;
#pragma unroll
                for (int vv = 0; vv < 2; ++vv) {
                    const int vx = vq + 4 * vv;
                    if (vx >= V) break;
                    const double* dmr = Dm + (br + vx - b0) * DC - d.Xlo;
                    const double* dkr = Dk + (br + vx - b0) * DC - d.Xlo;
#pragma unroll
                    for (int o1 = 0; o1 < S; ++o1) {
                        const int X = r - P + o1;
                        if (X < 0 || X >= N) continue;
                        const double dm = dmr[X], cm = pm[vx * S + o1];
                        ym = fma(cm, dm, ym);
                        yk = fma(pk[vx * S + o1], dm, yk);
                        yk = fma(cm, dkr[X], yk);
                    }
                }
            }
            ym += __shfl_xor_sync(0xffffffffu, ym, 1);
            yk += __shfl_xor_sync(0xffffffffu, yk, 1);
            ym += __shfl_xor_sync(0xffffffffu, ym, 2);
            yk += __shfl_xor_sync(0xffffffffu, yk, 2);
            if (vq == 0 && j < d.tr) {
                if (MODE & 1) a.yM[d.orow0 + j] = ym;
                if (MODE & 2) a.yK[d.orow0 + j] = yk;
            }
        }
        if (dA.line >= 0) phase_a<P, NT, HS, RING, G::PATCH>(a, dA, patches, qbufs, Hm, Hk, tid);
        issue(itP, prow);                                            // tile k+PFD
        if (tid == NT - 1) desc[(k + PFD) & 7] = make_desc<P, URING, TRA>(a, itP, last_line, false);
        if (itP.line <= last_line) it_next<P, PFD, URING, TRA>(a, itP);
        cp_async_wait<PFD - 2>();                                    // tile k+2 landed
        __syncthreads();
    }
    cp_async_wait<0>();
}

#ifndef WGQ_APPLY_TR
#define WGQ_APPLY_TR 24
#endif

template <int P, int MODE>
int launch_apply_p(const LineArgs& a, cudaStream_t st) {
    constexpr int TRA = WGQ_APPLY_TR;
    using G = ApplyGeom<P, TRA>;
    const size_t smem = G::smem_doubles() * sizeof(double);
    auto kern = k_line_apply<P, MODE, TRA>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return WGQ_ECUDA;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kApplyThreads, smem);
    const int64_t lines = (a.row_end - 1) / a.N - a.row_begin / a.N + 1;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(lines, (int64_t)sms * std::max(per_sm, 1)));
    kern<<<(unsigned)blocks, kApplyThreads, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

template <int P, int MODE>
int launch_line_p(const LineArgs& a, cudaStream_t st) {
    using C = Cfg<P>;
    const size_t smem = (size_t)C::SMEM * sizeof(double);
    auto kern = a.csr_base >= 0 ? k_line_grid3<P, MODE, true> : k_line_grid3<P, MODE, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return WGQ_ECUDA;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, smem);
    const int64_t lines = (a.row_end - 1) / a.N - a.row_begin / a.N + 1;
    int64_t blocks = std::min<int64_t>(lines, (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)std::max<int64_t>(blocks, 1), C::NT, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

template <int P>
int launch_line_mode(const LineArgs& a, int mode, cudaStream_t st) {
    if (mode == 3) return launch_line_p<P, 3>(a, st);
    if (mode == 1) return launch_line_p<P, 1>(a, st);
    return launch_line_p<P, 2>(a, st);
}

}  // namespace

bool line_kernel_applies(const wgq_rules_s* R, const wgq_coeff_t* c, const wgq_out_t* M, const wgq_out_t* K) {
    const wgq_out_t* o = M ? M : K;
    if (c->kind != WGQ_COEF_GRID || R->dim != 3) return false;
    for (int d = 0; d < 3; ++d)
        if (R->dims.n[d] < R->p + 1) return false;
    if (o->layout == WGQ_CSR) {
        for (const wgq_out_t* x : {M, K})
            if (x && ((uintptr_t)x->values) % 16 != 0) return false;
        return true;
    }
    const int64_t S3 = (2 * R->p + 1) * (2 * R->p + 1) * (2 * R->p + 1);
    for (const wgq_out_t* x : {M, K}) {
        if (!x) continue;
        if (x->ld != S3 && (x->ld % 2) != 0) return false;
        if (((uintptr_t)x->values) % 16 != 0) return false;
    }
    if (M && K && M->ld != K->ld) return false;
    return true;
}

namespace {
void line_dims(LineArgs& a, const wgq_rules_s* R, const Tables3& TT) {
    a.T = TT.t[0];
    a.Ty = TT.t[1];
    a.Tz = TT.t[2];
    a.n = (int)R->dims.n[0];
    a.N = (int)R->dims.N[0];
    a.ny = (int)R->dims.n[1];
    a.Ny = (int)R->dims.N[1];
    a.nz = (int)R->dims.n[2];
    a.Nz = (int)R->dims.N[2];
}
}  // namespace

int launch_line(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const wgq_out_t* M,
                const wgq_out_t* K, void* stream) {
    const wgq_out_t* o = M ? M : K;
    LineArgs a{};
    line_dims(a, R, TT);
    a.grid = c->grid;
    a.plane0 = (int)c->grid_plane0;
    a.planes = (int)c->grid_planes;
    a.row_begin = (int)o->row_begin;
    a.row_end = (int)o->row_end;
    a.M = M ? M->values : nullptr;
    a.K = K ? K->values : nullptr;
    a.ld = o->layout == WGQ_CSR ? (2 * R->p + 1) * (2 * R->p + 1) * (2 * R->p + 1) : o->ld;
    a.csr_base = o->layout == WGQ_CSR ? csr_start(o->row_begin, R->p, a.N, a.Ny, a.Nz) : -1;
    const int mode = (M ? 1 : 0) | (K ? 2 : 0);
    a.h = 1.0 / (double)a.n;                  // x spacing: the interior x-row tables P^
    a.inv_h = (double)a.n;
    {
        double PM[kMaxV][kMaxS], PK[kMaxV][kMaxS];
        interior_vertex_tables(R->p, R->rules[WGQ_MASS][R->p], R->rules[WGQ_STIFFNESS][R->p], PM, PK);
        for (int v = 0; v < kMaxV; ++v)
            for (int o1 = 0; o1 < kMaxS; ++o1) {
                a.PMh[v][o1] = PM[v][o1] * a.h;
                a.PKi[v][o1] = PK[v][o1] * a.inv_h;
            }
    }
    if (const char* e = getenv("WGQ_LINE_DBG")) a.dbg = atoi(e);
    if (a.row_end <= a.row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    static const bool static_order = [] {
        const char* e = getenv("WGQ_LINE_STATIC");
        return e && e[0] == '1';
    }();
    if (!static_order) {
        if (cudaMallocAsync((void**)&a.ticket, sizeof(unsigned long long), st) != cudaSuccess) return WGQ_ENOMEM;
        cudaMemsetAsync(a.ticket, 0, sizeof(unsigned long long), st);
    }
    const int rc = R->p == 3 ? launch_line_mode<3>(a, mode, st) : launch_line_mode<2>(a, mode, st);
    if (a.ticket) cudaFreeAsync(a.ticket, st);
    return rc;
}

bool line_apply_applies(const wgq_rules_s* R, const wgq_coeff_t* c) {
    if (c->kind != WGQ_COEF_GRID || R->dim != 3) return false;
    for (int d = 0; d < 3; ++d)
        if (R->dims.n[d] < R->p + 1) return false;
    return true;
}

int launch_line_apply(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const double* u,
                      int64_t u_row0, int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream) {
    if (row_end <= row_begin) return WGQ_OK;
    LineArgs a{};
    line_dims(a, R, TT);
    a.grid = c->grid;
    a.plane0 = (int)c->grid_plane0;
    a.planes = (int)c->grid_planes;
    a.row_begin = (int)row_begin;
    a.row_end = (int)row_end;
    a.ld = 0;
    a.h = 1.0 / (double)a.n;
    a.inv_h = (double)a.n;
    double PM[kMaxV][kMaxS], PK[kMaxV][kMaxS];
    interior_vertex_tables(R->p, R->rules[WGQ_MASS][R->p], R->rules[WGQ_STIFFNESS][R->p], PM, PK);
    for (int v = 0; v < kMaxV; ++v)
        for (int o1 = 0; o1 < kMaxS; ++o1) {
            a.PMh[v][o1] = PM[v][o1] * a.h;
            a.PKi[v][o1] = PK[v][o1] * a.inv_h;
        }
    a.u = u;
    a.u_row0 = u_row0;
    a.yM = yM;
    a.yK = yK;
    if (const char* e = getenv("WGQ_LINE_DBG")) a.dbg = atoi(e);
    const int mode = (yM ? 1 : 0) | (yK ? 2 : 0);
    cudaStream_t st = (cudaStream_t)stream;
    if (R->p == 3) return mode == 3 ? launch_apply_p<3, 3>(a, st) : (mode == 1 ? launch_apply_p<3, 1>(a, st) : launch_apply_p<3, 2>(a, st));
    return mode == 3 ? launch_apply_p<2, 3>(a, st) : (mode == 1 ? launch_apply_p<2, 1>(a, st) : launch_apply_p<2, 2>(a, st));
}

}  // namespace wgq
