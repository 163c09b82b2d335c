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
// Interior x-rows (class I) share one table P^ (times h resp. 1/h) that lives in __constant__
// memory; its zero pattern is structural (a node in element k touches planes k, k+1 and
// columns k..k+p), so phase B issues only the structurally nonzero FP64 FMAs, with constant
// operands, plus 2 LDS per output group.  A CTA owns a set of lines and walks them in tiles of
// TR rows with two warp roles: 3 producer warps prefetch the next tile's vertex patch
// (cp.async) and build its new H planes into a plane ring; the consumer warps (one per 32
// output groups) finish the rows of the current tile into double-buffered shared-memory
// staging that one thread writes out with cp.async.bulk.  Producer and consumers hand tiles
// over through full/empty mbarriers, so neither role waits on a CTA-wide barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "internal.h"

namespace wgq {
namespace {

__constant__ double c_PM3[5][7], c_PK3[5][7];
__constant__ double c_PM2[4][5], c_PK2[4][5];

template <int P>
struct Cfg {
    static constexpr int S = 2 * P + 1;
    static constexpr int S2 = S * S;
    static constexpr int S3 = S2 * S;
    static constexpr int V = P + 2;
    static constexpr int TR = 8;                        // rows per tile
    static constexpr int ITEMS = TR * S2;               // (row, o2 o3) output groups per tile
    static constexpr int NC = (ITEMS + 31) / 32 * 32;   // consumer threads (one group each)
    static constexpr int NP = 96;                       // producer threads (3 warps)
    static constexpr int NT = NP + NC;
    static constexpr int W = TR + V - 1;                // vertex planes in a tile's window
    static constexpr int RING = 32;                     // H plane ring (>= 2 W), power of two
    static constexpr int DEPTH = 4;                     // tile-info / mbarrier ring
    static constexpr int SR = S3 + 1;                   // staging row stride for padded ld
    static constexpr int STAGE = TR * SR + 2;           // doubles per staging buffer per matrix
    static constexpr int PATCH = W * V * V;
    // doubles: staging, H ring (M, K), Q, 2 patches, TM, TK
    static constexpr int SMEM_D = 4 * STAGE + RING * 2 * S2 + 4 * V * S + 2 * PATCH + 2 * W * V * S;
    static constexpr int SMEM = SMEM_D * 8 + 2 * DEPTH * 8 + DEPTH * 32;
    static_assert(2 * W <= RING, "ring too small");
};

struct LineArgs {
    RowTables T;
    const double* grid;
    int plane0, planes;
    int n, N;
    int row_begin, row_end;
    double* M;
    double* K;
    long long ld;
    int do_mass, do_stiff;
    double h, inv_h;
};

// per-tile handoff record (producer -> consumers)
struct TileInfo {
    int line, t0, tr, lo_need, seq0;   // seq0 = ring sequence number of plane lo_need
};

__device__ __forceinline__ void bulk_store(double* gdst, const double* ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int P>
__device__ __forceinline__ double cPM(int v, int o) {
    if constexpr (P == 3) return c_PM3[v][o];
    else return c_PM2[v][o];
}
template <int P>
__device__ __forceinline__ double cPK(int v, int o) {
    if constexpr (P == 3) return c_PK3[v][o];
    else return c_PK2[v][o];
}

// Deterministic walk over this CTA's (line, tile) sequence, shared by both roles.
struct TileWalk {
    int line, t0, x0, x1;
    int last_line, stride, N, row_begin, row_end;
    __device__ void set_line() {
        x0 = max(row_begin, line * N) - line * N;
        x1 = min(row_end, line * N + N) - line * N;
        t0 = x0;
    }
    __device__ bool valid() const { return line <= last_line; }
    template <int TR>
    __device__ void next() {
        t0 += TR;
        if (t0 >= x1) {
            line += stride;
            if (line <= last_line) set_line();
        }
    }
};

template <int P>
__device__ __forceinline__ void issue_patch(const LineArgs& a, double* patch, int c0, int nnew, int by, int bz,
                                            int ptid) {
    using C = Cfg<P>;
    constexpr int V = C::V;
    const int nv = a.n + 1;
    for (int e = ptid; e < nnew * V * V; e += C::NP) {
        const int j = e % nnew, vy = (e / nnew) % V, vz = e / (nnew * V);
        const int x = c0 + j, y = by + vy, z = bz + vz;
        const bool ok = x <= a.n && y <= a.n && z <= a.n && z - a.plane0 < a.planes;
        const double* src = ok ? a.grid + ((size_t)(z - a.plane0) * nv + y) * nv + x : a.grid;
        cp_async8(patch + (j * V + vz) * V + vy, src, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int P>
__global__ void __launch_bounds__(Cfg<P>::NT, 1) k_line_grid3(const LineArgs a) {
    using C = Cfg<P>;
    constexpr int S = C::S, S2 = C::S2, S3 = C::S3, V = C::V, TR = C::TR, RING = C::RING, DEPTH = C::DEPTH;
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;                                   // [2 buf][2 mat][STAGE]
    double* Hm = stage + 4 * C::STAGE;                    // [RING][S2]
    double* Hk = Hm + RING * S2;                          // [RING][S2]
    double* Q = Hk + RING * S2;                           // QyM, QyK, QzM, QzK: [V][S] each
    double* patches = Q + 4 * V * S;                      // [2][W][V(z)][V(y)]
    double* TM = patches + 2 * C::PATCH;                  // [W][V(z)][S(o2)]
    double* TK = TM + C::W * V * S;
    uint64_t* full = (uint64_t*)(TK + C::W * V * S);      // [DEPTH]
    uint64_t* empty = full + DEPTH;                       // [DEPTH]
    TileInfo* info = (TileInfo*)(empty + DEPTH);          // [DEPTH]

    const int tid = threadIdx.x;
    const int N = a.N;
    TileWalk walk;
    walk.N = N;
    walk.row_begin = a.row_begin;
    walk.row_end = a.row_end;
    walk.last_line = (a.row_end - 1) / N;
    walk.stride = gridDim.x;
    walk.line = a.row_begin / N + blockIdx.x;
    if (walk.valid()) walk.set_line();

    if (tid == 0) {
        for (int k = 0; k < DEPTH; ++k) {
            mbar_init(&full[k], C::NP);
            mbar_init(&empty[k], C::NC / 32);
        }
    }
    __syncthreads();

    if (tid < C::NP) {
        // =============================== producer warps ===============================
        const int ptid = tid;
        const double* QyM = Q;
        const double* QyK = Q + V * S;
        const double* QzM = Q + 2 * V * S;
        const double* QzK = Q + 3 * V * S;
        int seq = 0;                 // ring sequence number of the next plane to produce
        int hcomp = -1, cur_line = -1, by = 0, bz = 0, lo_prev = 0, seq_lo_prev = 0;
        int t = 0;
        // patch for the first tile
        TileWalk nw = walk;
        auto tile_planes = [&](const TileWalk& w, int& lo_need, int& hi_need) {
            const int tr = min(TR, w.x1 - w.t0);
            lo_need = max(0, w.t0 - P);
            hi_need = max(0, w.t0 + tr - 1 - P) + V - 1;
        };
        if (walk.valid()) {
            int lo, hi;
            tile_planes(walk, lo, hi);
            const int i2 = walk.line % N, i3 = walk.line / N;
            issue_patch<P>(a, patches, lo, hi - lo + 1, max(0, i2 - P), max(0, i3 - P), ptid);
        }
        for (; walk.valid(); walk.next<TR>(), ++t) {
            const int i2 = walk.line % N, i3 = walk.line / N;
            int lo_need, hi_need;
            tile_planes(walk, lo_need, hi_need);
            const bool new_line = walk.line != cur_line;
            if (new_line) {
                named_sync(1, C::NP);                       // previous line's A2/A3 done with Q
                for (int e = ptid; e < 4 * V * S; e += C::NP) {
                    const int which = e / (V * S), v = (e / S) % V, o = e % S;
                    const int r = which < 2 ? i2 : i3;
                    const double* src = (which & 1) ? a.T.PK : a.T.PM;
                    Q[e] = src[((size_t)r * kMaxV + v) * kMaxS + o];
                }
                cur_line = walk.line;
                by = max(0, i2 - P);
                bz = max(0, i3 - P);
                hcomp = lo_need - 1;
            }
            const int c0 = hcomp + 1;
            const int nnew = hi_need - hcomp;
            const int seq_c0 = seq;                         // sequence number of plane c0
            // ring slots of this tile's new planes must no longer be read: tile t-2 consumed
            if (t >= 2) mbar_wait(&empty[(t - 2) % DEPTH], ((t - 2) / DEPTH) & 1);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            named_sync(1, C::NP);                           // patch + Q visible to the group
            const double* patch = patches + (t & 1) * C::PATCH;
            for (int e = ptid; e < nnew * V * S; e += C::NP) {
                const int o2 = e % S, vz = (e / S) % V, j = e / (S * V);
                const double* pr = patch + (j * V + vz) * V;
                double sm_ = 0.0, sk = 0.0;
#pragma unroll
                for (int vy = 0; vy < V; ++vy) {
                    sm_ = fma(pr[vy], QyM[vy * S + o2], sm_);
                    sk = fma(pr[vy], QyK[vy * S + o2], sk);
                }
                TM[(j * V + vz) * S + o2] = sm_;
                TK[(j * V + vz) * S + o2] = sk;
            }
            // prefetch the next tile's patch into the other buffer
            nw = walk;
            nw.next<TR>();
            if (nw.valid()) {
                int nlo, nhi;
                tile_planes(nw, nlo, nhi);
                const int ni2 = nw.line % N, ni3 = nw.line / N;
                const int nc0 = nw.line == walk.line ? hi_need + 1 : nlo;
                issue_patch<P>(a, patches + ((t + 1) & 1) * C::PATCH, nc0, nhi - nc0 + 1, max(0, ni2 - P),
                               max(0, ni3 - P), ptid);
            }
            named_sync(1, C::NP);                           // TM/TK complete
            for (int e = ptid; e < nnew * S2; e += C::NP) {
                const int o23 = e % S2, j = e / S2, o2 = o23 % S, o3 = o23 / S;
                const double* tm = TM + j * V * S + o2;
                const double* tk = TK + j * V * S + o2;
                double hm = 0.0, hk = 0.0;
#pragma unroll
                for (int vz = 0; vz < V; ++vz) {
                    hm = fma(tm[vz * S], QzM[vz * S + o3], hm);
                    hk = fma(tk[vz * S], QzM[vz * S + o3], hk);
                    hk = fma(tm[vz * S], QzK[vz * S + o3], hk);
                }
                const int slot = (seq_c0 + j) & (RING - 1);
                Hm[slot * S2 + o23] = hm;
                Hk[slot * S2 + o23] = hk;
            }
            seq += nnew;
            hcomp = hi_need;
            if (ptid == 0) {
                TileInfo ti;
                ti.line = walk.line;
                ti.t0 = walk.t0;
                ti.tr = min(TR, walk.x1 - walk.t0);
                ti.lo_need = lo_need;
                ti.seq0 = seq_c0 - (c0 - lo_need);          // planes lo_need..c0-1 were produced earlier
                info[t % DEPTH] = ti;
            }
            mbar_arrive(&full[t % DEPTH]);
            named_sync(1, C::NP);                           // TM/TK and patch buffer reuse guard
            (void)lo_prev;
            (void)seq_lo_prev;
        }
        return;
    }

    // ================================= consumer warps =================================
    const int ctid = tid - C::NP;
    const int n = a.n;
    const bool padded = a.ld != S3;
    const int SRr = padded ? C::SR : S3;
    for (int t = 0; walk.valid(); walk.next<TR>(), ++t) {
        mbar_wait(&full[t % DEPTH], (t / DEPTH) & 1);
        const TileInfo ti = info[t % DEPTH];
        const int j = ctid / S2, o23 = ctid % S2;
        const bool active = ctid < ti.tr * S2;
        const int r = ti.t0 + j;
        double hm[V], hk[V];
        if (active) {
            const int bx = max(0, r - P);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int slot = (ti.seq0 + (bx - ti.lo_need) + v) & (RING - 1);
                hm[v] = Hm[slot * S2 + o23];
                hk[v] = Hk[slot * S2 + o23];
            }
        }
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[t % DEPTH]);
        // staging buffer t&1 must have been read by the bulk copy of tile t-2
        const int buf = t & 1;
        if (t >= 2 && ctid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        named_sync(2, C::NC);
        const long long orow0 = (long long)ti.line * N + ti.t0 - a.row_begin;
        const long long g0 = orow0 * a.ld;
        const int pad = padded ? 0 : (int)(g0 & 1);
        double* stM = stage + (buf * 2 + 0) * C::STAGE + pad;
        double* stK = stage + (buf * 2 + 1) * C::STAGE + pad;
        if (active) {
            double* dM = stM + j * SRr + S * o23;
            double* dK = stK + j * SRr + S * o23;
            if (r >= 2 * P && r <= n - 1 - P) {           // class I: constant tables, structural zeros skipped
#pragma unroll
                for (int o1 = 0; o1 < S; ++o1) {
                    double s = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
                    for (int v = (o1 - P > 0 ? o1 - P : 0); v <= (o1 + 1 < P + 1 ? o1 + 1 : P + 1); ++v) {
                        s = fma(cPM<P>(v, o1), hm[v], s);
                        s1 = fma(cPK<P>(v, o1), hm[v], s1);
                        s2 = fma(cPM<P>(v, o1), hk[v], s2);
                    }
                    if (a.do_mass) dM[o1] = a.h * s + 0.0;
                    if (a.do_stiff) dK[o1] = fma(a.h, s2, s1 * a.inv_h) + 0.0;
                }
            } else {                                       // boundary-affected x-row: its own tables
                const double* pm = a.T.PM + (size_t)r * kMaxV * kMaxS;
                const double* pk = a.T.PK + (size_t)r * kMaxV * kMaxS;
#pragma unroll
                for (int o1 = 0; o1 < S; ++o1) {
                    double s = 0.0, s1 = 0.0;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const double m = __ldg(pm + v * kMaxS + o1);
                        s = fma(m, hm[v], s);
                        s1 = fma(__ldg(pk + v * kMaxS + o1), hm[v], s1);
                        s1 = fma(m, hk[v], s1);
                    }
                    if (a.do_mass) dM[o1] = s + 0.0;
                    if (a.do_stiff) dK[o1] = s1 + 0.0;
                }
            }
        }
        named_sync(2, C::NC);
        // ---- store the tile: bulk copies of the 16-byte aligned interior, peeled ends ----
        const int tr = ti.tr;
        if (!padded) {
            const int total = tr * S3;
            const int head = (int)(g0 & 1);
            const int tail = (int)((g0 + total) & 1);
            if (ctid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (a.do_mass) bulk_store(a.M + g0 + head, stM + head, (uint32_t)(total - head - tail) * 8u);
                if (a.do_stiff) bulk_store(a.K + g0 + head, stK + head, (uint32_t)(total - head - tail) * 8u);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            } else if (ctid == 32 && head) {
                if (a.do_mass) a.M[g0] = stM[0];
                if (a.do_stiff) a.K[g0] = stK[0];
            } else if (ctid == 64 && tail) {
                if (a.do_mass) a.M[g0 + total - 1] = stM[total - 1];
                if (a.do_stiff) a.K[g0 + total - 1] = stK[total - 1];
            }
        } else {                                           // even ld: rows start 16B-aligned
            if (ctid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                for (int jj = 0; jj < tr; ++jj) {
                    if (a.do_mass) bulk_store(a.M + (orow0 + jj) * a.ld, stM + jj * SRr, (uint32_t)(S3 - 1) * 8u);
                    if (a.do_stiff) bulk_store(a.K + (orow0 + jj) * a.ld, stK + jj * SRr, (uint32_t)(S3 - 1) * 8u);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (ctid >= 32 && ctid < 32 + tr) {
                const int jj = ctid - 32;
                if (a.do_mass) a.M[(orow0 + jj) * a.ld + S3 - 1] = stM[jj * SRr + S3 - 1];
                if (a.do_stiff) a.K[(orow0 + jj) * a.ld + S3 - 1] = stK[jj * SRr + S3 - 1];
            }
        }
    }
    if (ctid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int P>
int launch_line_p(const LineArgs& a, cudaStream_t st) {
    using C = Cfg<P>;
    const size_t smem = (size_t)C::SMEM;
    if (cudaFuncSetAttribute(k_line_grid3<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return WGQ_ECUDA;
    cudaFuncSetAttribute(k_line_grid3<P>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_line_grid3<P>, C::NT, smem);
    const int64_t lines = (a.row_end - 1) / a.N - a.row_begin / a.N + 1;
    int64_t blocks = std::min<int64_t>(lines, (int64_t)sms * std::max(per_sm, 1));
    k_line_grid3<P><<<(unsigned)std::max<int64_t>(blocks, 1), C::NT, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? WGQ_OK : WGQ_ECUDA;
}

std::mutex g_const_mu;
bool g_const_ready[64][4] = {};

int upload_constants(const wgq_rules_s* R) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_const_mu);
    if (dev < 64 && g_const_ready[dev][R->p]) return WGQ_OK;
    double PM[kMaxV][kMaxS], PK[kMaxV][kMaxS];
    interior_vertex_tables(R->p, R->rules[WGQ_MASS][R->p], R->rules[WGQ_STIFFNESS][R->p], PM, PK);
    cudaError_t e1, e2;
    if (R->p == 3) {
        double m[5][7], k[5][7];
        for (int v = 0; v < 5; ++v)
            for (int o = 0; o < 7; ++o) {
                m[v][o] = PM[v][o];
                k[v][o] = PK[v][o];
            }
        e1 = cudaMemcpyToSymbol(c_PM3, m, sizeof m);
        e2 = cudaMemcpyToSymbol(c_PK3, k, sizeof k);
    } else {
        double m[4][5], k[4][5];
        for (int v = 0; v < 4; ++v)
            for (int o = 0; o < 5; ++o) {
                m[v][o] = PM[v][o];
                k[v][o] = PK[v][o];
            }
        e1 = cudaMemcpyToSymbol(c_PM2, m, sizeof m);
        e2 = cudaMemcpyToSymbol(c_PK2, k, sizeof k);
    }
    if (e1 != cudaSuccess || e2 != cudaSuccess) return WGQ_ECUDA;
    if (dev < 64) g_const_ready[dev][R->p] = true;
    return WGQ_OK;
}

}  // namespace

bool line_kernel_applies(const wgq_rules_s* R, const wgq_coeff_t* c, const wgq_out_t* M, const wgq_out_t* K) {
    const wgq_out_t* o = M ? M : K;
    if (c->kind != WGQ_COEF_GRID || R->dim != 3 || o->layout != WGQ_ELL) return false;
    if (R->n < R->p + 1) return false;
    const int64_t S3 = (2 * R->p + 1) * (2 * R->p + 1) * (2 * R->p + 1);
    for (const wgq_out_t* x : {M, K}) {
        if (!x) continue;
        if (x->ld != S3 && (x->ld % 2) != 0) return false;
        if (((uintptr_t)x->values) % 16 != 0) return false;
    }
    if (M && K && M->ld != K->ld) return false;
    return true;
}

int launch_line(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const wgq_out_t* M,
                const wgq_out_t* K, void* stream) {
    int rc = upload_constants(R);
    if (rc != WGQ_OK) return rc;
    const wgq_out_t* o = M ? M : K;
    LineArgs a{};
    a.T = T;
    a.grid = c->grid;
    a.plane0 = (int)c->grid_plane0;
    a.planes = (int)c->grid_planes;
    a.n = (int)R->n;
    a.N = (int)R->N;
    a.row_begin = (int)o->row_begin;
    a.row_end = (int)o->row_end;
    a.M = M ? M->values : nullptr;
    a.K = K ? K->values : nullptr;
    a.ld = o->ld;
    a.do_mass = M != nullptr;
    a.do_stiff = K != nullptr;
    a.h = 1.0 / (double)R->n;
    a.inv_h = (double)R->n;
    if (a.row_end <= a.row_begin) return WGQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    return R->p == 3 ? launch_line_p<3>(a, st) : launch_line_p<2>(a, st);
}

}  // namespace wgq
