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
// Interior x-rows (class I) share one table P^ (scaled by h, 1/h) that lives in __constant__
// memory, so phase B is FP64 FMAs with constant operands plus two LDS per output group.
// A CTA owns a line, walks it in tiles of TR rows, stages the tile's M and K rows in shared
// memory (double-buffered) and writes each tile with one cp.async.bulk per matrix.
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
    static constexpr int TR = 8;                       // rows per tile
    static constexpr int ITEMS = TR * S2;              // (row, o2 o3) output groups per tile
    static constexpr int NT = (ITEMS + 31) / 32 * 32;  // threads
    static constexpr int MAXNEW = TR + V - 1;          // new vertex planes per tile (at most)
    static constexpr int RING = 16;                    // H ring (>= MAXNEW), power of two
    static constexpr int SR = S3 + 1;                  // staging row stride for padded ld
    static constexpr int STAGE = TR * SR + 2;          // doubles per staging buffer per matrix
    static constexpr int SMEM = 4 * STAGE + RING * 2 * S2 + 4 * V * S + MAXNEW * V * V + 2 * MAXNEW * V * S;
};

struct LineArgs {
    RowTables T;
    const double* grid;
    int64_t plane0, planes;
    int64_t n, N;
    int64_t row_begin, row_end;
    double* M;
    double* K;
    int64_t ld;
    int do_mass, do_stiff;
    double h, inv_h;
};

__device__ __forceinline__ void bulk_store(double* gdst, const double* ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
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

template <int P>
__global__ void __launch_bounds__(Cfg<P>::NT, 2) k_line_grid3(const LineArgs a) {
    using C = Cfg<P>;
    constexpr int S = C::S, S2 = C::S2, S3 = C::S3, V = C::V, TR = C::TR, RING = C::RING;
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;                                   // [2 buf][2 mat][STAGE]
    double* Hm = stage + 4 * C::STAGE;                    // [RING][S2]
    double* Hk = Hm + RING * S2;                          // [RING][S2]
    double* Q = Hk + RING * S2;                           // QyM, QyK, QzM, QzK: [V][S] each
    double* patch = Q + 4 * V * S;                        // [MAXNEW][V(z)][V(y)]
    double* TM = patch + C::MAXNEW * V * V;               // [MAXNEW][V(z)][S(o2)]
    double* TK = TM + C::MAXNEW * V * S;
    const double* QyM = Q;
    const double* QyK = Q + V * S;
    const double* QzM = Q + 2 * V * S;
    const double* QzK = Q + 3 * V * S;

    const int tid = threadIdx.x;
    const int64_t n = a.n, N = a.N, nv = n + 1;
    const bool padded = a.ld != S3;
    const int SRr = padded ? C::SR : S3;
    const int64_t first_line = a.row_begin / N, last_line = (a.row_end - 1) / N;
    int tiles = 0;

    for (int64_t line = first_line + blockIdx.x; line <= last_line; line += gridDim.x) {
        const int64_t i2 = line % N, i3 = line / N;
        const int64_t x0 = max(a.row_begin, line * N) - line * N;
        const int64_t x1 = min(a.row_end, line * N + N) - line * N;
        const int64_t by = i2 - P > 0 ? i2 - P : 0, bz = i3 - P > 0 ? i3 - P : 0;
        __syncthreads();                                   // previous line done with Q / H
        for (int e = tid; e < 4 * V * S; e += C::NT) {
            const int which = e / (V * S), v = (e / S) % V, o = e % S;
            const int64_t r = which < 2 ? i2 : i3;
            const double* src = (which & 1) ? a.T.PK : a.T.PM;
            Q[e] = src[(r * kMaxV + v) * kMaxS + o];
        }
        int64_t hcomp = -1;                                // vertex planes computed: (hcomp-RING, hcomp]
        for (int64_t t0 = x0; t0 < x1; t0 += TR) {
            const int tr = (int)min((int64_t)TR, x1 - t0);
            const int64_t lo_need = t0 - P > 0 ? t0 - P : 0;
            const int64_t last = t0 + tr - 1;
            const int64_t hi_need = (last - P > 0 ? last - P : 0) + V - 1;
            if (hcomp < lo_need - 1) hcomp = lo_need - 1;
            if (hcomp < hi_need) {
                // ---- phase A: new vertex planes c0..hi_need -> HM, HK --------------------
                const int64_t c0 = hcomp + 1;
                const int nnew = (int)(hi_need - hcomp);
                __syncthreads();                           // Q visible; ring slots free
                for (int e = tid; e < nnew * V * V; e += C::NT) {
                    const int j = e % nnew, vy = (e / nnew) % V, vz = e / (nnew * V);
                    const int64_t x = c0 + j, y = by + vy, z = bz + vz;
                    double g = 0.0;
                    if (x <= n && y <= n && z <= n && z - a.plane0 < a.planes)
                        g = __ldg(a.grid + ((z - a.plane0) * nv + y) * nv + x);
                    patch[(j * V + vz) * V + vy] = g;
                }
                __syncthreads();
                for (int e = tid; e < nnew * V * S; e += C::NT) {
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
                __syncthreads();
                for (int e = tid; e < nnew * S2; e += C::NT) {
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
                    const int slot = (int)((c0 + j) & (RING - 1));
                    Hm[slot * S2 + o23] = hm;
                    Hk[slot * S2 + o23] = hk;
                }
                hcomp = hi_need;
            }
            // ---- phase B: rows of the tile -> staging ------------------------------------
            const int buf = tiles & 1;
            if (tiles >= 2 && tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncthreads();                               // H ready; staging buffer free
            const int64_t orow0 = line * N + t0 - a.row_begin;     // output row of the tile
            const int64_t g0 = orow0 * a.ld;                       // first element (doubles)
            const int pad = padded ? 0 : (int)(g0 & 1);
            double* stM = stage + (buf * 2 + 0) * C::STAGE + pad;
            double* stK = stage + (buf * 2 + 1) * C::STAGE + pad;
            for (int it = tid; it < tr * S2; it += C::NT) {
                const int j = it / S2, o23 = it % S2;
                const int64_t r = t0 + j;
                const int64_t bx = r - P > 0 ? r - P : 0;
                double hm[V], hk[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int slot = (int)((bx + v) & (RING - 1));
                    hm[v] = Hm[slot * S2 + o23];
                    hk[v] = Hk[slot * S2 + o23];
                }
                double* dM = stM + j * SRr + S * o23;
                double* dK = stK + j * SRr + S * o23;
                if (r >= 2 * P && r <= n - 1 - P) {       // class I: constant tables
#pragma unroll
                    for (int o1 = 0; o1 < S; ++o1) {
                        double s = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            s = fma(cPM<P>(v, o1), hm[v], s);
                            s1 = fma(cPK<P>(v, o1), hm[v], s1);
                            s2 = fma(cPM<P>(v, o1), hk[v], s2);
                        }
                        if (a.do_mass) dM[o1] = a.h * s + 0.0;
                        if (a.do_stiff) dK[o1] = fma(a.h, s2, s1 * a.inv_h) + 0.0;
                    }
                } else {                                   // boundary-affected x-row: its own tables
                    const double* pm = a.T.PM + r * kMaxV * kMaxS;
                    const double* pk = a.T.PK + r * kMaxV * kMaxS;
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
            __syncthreads();
            // ---- store the tile: bulk copies of the 16-byte aligned interior, peeled ends ----
            for (int mat = 0; mat < 2; ++mat) {
                if (mat == 0 ? !a.do_mass : !a.do_stiff) continue;
                double* out = mat == 0 ? a.M : a.K;
                const double* st = mat == 0 ? stM : stK;
                if (!padded) {
                    const int total = tr * S3;
                    const int head = (int)(g0 & 1);
                    const int tail = (int)((g0 + total) & 1);
                    if (tid == 0) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        bulk_store(out + g0 + head, st + head, (uint32_t)(total - head - tail) * 8u);
                    } else if (tid == 32 && head) {
                        out[g0] = st[0];
                    } else if (tid == 64 && tail) {
                        out[g0 + total - 1] = st[total - 1];
                    }
                } else {                                   // even ld: rows start 16B-aligned
                    if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (tid == 0)
                        for (int j = 0; j < tr; ++j)
                            bulk_store(out + (orow0 + j) * a.ld, st + j * SRr, (uint32_t)(S3 - 1) * 8u);
                    if (tid >= 32 && tid < 32 + tr) {
                        const int j = tid - 32;
                        out[(orow0 + j) * a.ld + S3 - 1] = st[j * SRr + S3 - 1];
                    }
                }
            }
            if (tid == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            ++tiles;
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int P>
int launch_line_p(const LineArgs& a, cudaStream_t st) {
    using C = Cfg<P>;
    const size_t smem = (size_t)C::SMEM * sizeof(double);
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
    a.plane0 = c->grid_plane0;
    a.planes = c->grid_planes;
    a.n = R->n;
    a.N = R->N;
    a.row_begin = o->row_begin;
    a.row_end = o->row_end;
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
