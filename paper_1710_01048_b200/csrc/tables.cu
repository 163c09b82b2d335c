// Device construction of the per-1D-row tables: for every
// basis function r of one direction, its physical quadrature nodes, effective weights
// and the values B_{r+o}(x_k) / B'_{r+o}(x_k), o = -p..p, of the 2p+1 interacting
// functions at those nodes.  The tables depend on (p, n, rules) only and are built once
// per device and cached in the rules handle.
//
// Node placement (R1): row r < p uses the left boundary class j = r (x = h tau); row
// r >= n the mirrored class j = N-1-r (x = 1 - h tau); other rows the interior rule
// shifted to supp B_r = [(r-p)h, (r+1)h] (x = h (r - p + tau)), h = 1/n.  Weights
// scale by h (dx = h dtau); derivative values are physical.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace wgq {
namespace {

struct ClassArgs {
    int p;
    int64_t n;
    int64_t N;
    int m[2][kMaxP + 1];
    double tau[2][kMaxP + 1][kMaxStiffNodes];
    double omega[2][kMaxP + 1][kMaxStiffNodes];
};

// open uniform knot t_i on [0,1]: 0 for i <= p, (i-p)/n inside, 1 for i >= n+p (eq:Gmap3)
__device__ __forceinline__ double knot(int64_t i, int p, int64_t n) {
    int64_t k = i - p;
    k = k < 0 ? 0 : (k > n ? n : k);
    return (double)k / (double)n;
}

// Values and first derivatives of the p+1 nonzero B-splines on the span of x (Cox-de Boor
// triangle; vals[q] = B_{s-p+q}(x), ders[q] = B'_{s-p+q}(x)).  Returns the span s.
__device__ int64_t eval_span(double x, int p, int64_t n, double* vals, double* ders) {
    int64_t e = (int64_t)floor(x * (double)n);
    e = e < 0 ? 0 : (e > n - 1 ? n - 1 : e);
    const int64_t s = e + p;
    double lower[kMaxP + 1];           // degree p-1 values
    double N[kMaxP + 1];
    N[0] = 1.0;
    for (int deg = 1; deg <= p; ++deg) {
        if (deg == p)
            for (int q = 0; q < p; ++q) lower[q] = N[q];
        double next[kMaxP + 1];
        // functions B_{s-deg..s, deg}: q-th is B_{s-deg+q}
        for (int q = 0; q <= deg; ++q) {
            const int64_t i = s - deg + q;
            double v = 0.0;
            if (q >= 1) {                      // B_{i,deg-1} = N[q-1]
                double den = knot(i + deg, p, n) - knot(i, p, n);
                if (den > 0.0) v += (x - knot(i, p, n)) / den * N[q - 1];
            }
            if (q <= deg - 1) {                // B_{i+1,deg-1} = N[q]
                double den = knot(i + deg + 1, p, n) - knot(i + 1, p, n);
                if (den > 0.0) v += (knot(i + deg + 1, p, n) - x) / den * N[q];
            }
            next[q] = v;
        }
        for (int q = 0; q <= deg; ++q) N[q] = next[q];
    }
    for (int q = 0; q <= p; ++q) {
        vals[q] = N[q];
        const int64_t i = s - p + q;
        double d = 0.0;
        if (q >= 1) {
            double den = knot(i + p, p, n) - knot(i, p, n);
            if (den > 0.0) d += p / den * lower[q - 1];
        }
        if (q <= p - 1) {
            double den = knot(i + p + 1, p, n) - knot(i + 1, p, n);
            if (den > 0.0) d -= p / den * lower[q];
        }
        ders[q] = d;
    }
    return s;
}

__global__ void k_row_tables(ClassArgs A, RowTables T) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = tid / (2 * kMaxStiffNodes);
    const int kind = (int)((tid / kMaxStiffNodes) & 1);
    const int k = (int)(tid % kMaxStiffNodes);
    if (r >= A.N) return;
    const int p = A.p;
    const int64_t n = A.n, N = A.N;
    int cls;
    bool mirror = false;
    if (r < p) {
        cls = (int)r;
    } else if (r >= n) {
        cls = (int)(N - 1 - r);
        mirror = true;
    } else {
        cls = p;
    }
    const int m = A.m[kind][cls];
    const int maxn = kind == WGQ_MASS ? kMaxMassNodes : kMaxStiffNodes;
    if (k == 0) (kind == WGQ_MASS ? T.mM : T.mK)[r] = m;
    if (k >= maxn) return;
    double* X = kind == WGQ_MASS ? T.xM : T.xK;
    double* W = kind == WGQ_MASS ? T.wM : T.wK;
    double* V = kind == WGQ_MASS ? T.VM : T.DK;
    double* row = V + (r * maxn + k) * kMaxS;
    if (k >= m) {                         // unused node slot: zero weight, zero table
        X[r * maxn + k] = 0.0;
        W[r * maxn + k] = 0.0;
        for (int o = 0; o < kMaxS; ++o) row[o] = 0.0;
        return;
    }
    // x = h*(e0 + tau), omega_h = h*omega with h = 1/n, rounded exactly as written (no FMA
    // contraction) so that node coordinates are reproducible bit for bit (R14).
    const double h = 1.0 / (double)n;
    double x, om;
    if (cls == p) {
        x = __dmul_rn(h, __dadd_rn((double)(r - p), A.tau[kind][cls][k]));
        om = __dmul_rn(h, A.omega[kind][cls][k]);
    } else if (!mirror) {
        x = __dmul_rn(h, A.tau[kind][cls][k]);
        om = __dmul_rn(h, A.omega[kind][cls][k]);
    } else {
        x = __dsub_rn(1.0, __dmul_rn(h, A.tau[kind][cls][m - 1 - k]));
        om = __dmul_rn(h, A.omega[kind][cls][m - 1 - k]);
    }
    double vals[kMaxP + 1], ders[kMaxP + 1];
    const int64_t s = eval_span(x, p, n, vals, ders);
    const double* src = kind == WGQ_MASS ? vals : ders;
    for (int o = 0; o < kMaxS; ++o) {
        double v = 0.0;
        if (o <= 2 * p) {
            const int64_t i = r + o - p;
            if (i >= 0 && i < N && i >= s - p && i <= s) v = src[i - (s - p)];
        }
        row[o] = v;
    }
    X[r * maxn + k] = x;
    W[r * maxn + k] = om * row[p];        // omega * B_r(x) or omega * B'_r(x)
}

// Vertex-projected tables: one thread per (row, kind, v, o).
__global__ void k_vertex_tables(int p, int64_t n, RowTables T) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int per_row = 2 * kMaxV * kMaxS;
    const int64_t r = tid / per_row;
    if (r >= T.N) return;
    const int rem = (int)(tid % per_row);
    const int kind = rem / (kMaxV * kMaxS);
    const int v = (rem / kMaxS) % kMaxV;
    const int o = rem % kMaxS;
    const int m = kind == WGQ_MASS ? T.mM[r] : T.mK[r];
    const double* X = (kind == WGQ_MASS ? T.xM : T.xK) + r * kMaxNodes;
    const double* W = (kind == WGQ_MASS ? T.wM : T.wK) + r * kMaxNodes;
    const double* A = (kind == WGQ_MASS ? T.VM : T.DK) + r * kMaxNodes * kMaxS;
    const int64_t b = r - p > 0 ? r - p : 0;
    double acc = 0.0;
    for (int k = 0; k < m; ++k) {
        const double s = __dmul_rn(X[k], (double)n);
        int64_t e = (int64_t)floor(s);
        e = e < 0 ? 0 : (e > n - 1 ? n - 1 : e);
        const double f = s - (double)e;
        const int64_t rel = e - b;
        double lam = 0.0;
        if (rel == v) lam = 1.0 - f;
        else if (rel + 1 == v) lam = f;
        acc = fma(lam * W[k], A[k * kMaxS + o], acc);
    }
    (kind == WGQ_MASS ? T.PM : T.PK)[(r * kMaxV + v) * kMaxS + o] = acc;
}

// PW[r][v] = sum_o PM[r][v][o] (the row's 2p+1 neighbours; the load vector's vertex weights)
__global__ void k_vertex_weights(RowTables T, int p) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= T.N * kMaxV) return;
    double s = 0.0;
    for (int o = 0; o < 2 * p + 1; ++o) s += T.PM[e * kMaxS + o];
    T.PW[e] = s;
}

// AW[r][kind][k][o] = w_k A_k[o] for the first 8 nodes (fourier2d.cu): one thread per entry.
__global__ void k_weighted_tables(RowTables T) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= T.N * 128) return;
    const int64_t r = e / 128;
    const int kind = (int)(e / 64) % 2, k = (int)(e / 8) % 8, o = (int)(e % 8);
    const int m = kind == WGQ_MASS ? T.mM[r] : T.mK[r];
    double v = 0.0;
    if (k < m && o < kMaxS)
        v = kind == WGQ_MASS ? T.wM[r * kMaxMassNodes + k] * T.VM[(r * kMaxMassNodes + k) * kMaxS + o]
                             : T.wK[r * kMaxStiffNodes + k] * T.DK[(r * kMaxStiffNodes + k) * kMaxS + o];
    T.AW[e] = v;
}

}  // namespace

int build_row_tables(const wgq_rules_s* R, int64_t n_dir, RowTables* T, void* stream) {
    const int64_t N = n_dir + R->p;
    size_t bytes = 2 * N * sizeof(int) +
                   N * (kMaxMassNodes * (2 + kMaxS) + kMaxStiffNodes * (2 + kMaxS) + 2 * kMaxV * kMaxS) * sizeof(double);
    bytes += N * 128 * sizeof(double);         // AW
    bytes += N * kMaxV * sizeof(double);       // PW
    bytes += 256;
    void* base = nullptr;
    if (cudaMalloc(&base, bytes) != cudaSuccess) return WGQ_ECUDA;
    T->base = base;
    T->N = N;
    double* d = (double*)base;
    T->xM = d; d += N * kMaxMassNodes;
    T->wM = d; d += N * kMaxMassNodes;
    T->VM = d; d += N * kMaxMassNodes * kMaxS;
    T->xK = d; d += N * kMaxStiffNodes;
    T->wK = d; d += N * kMaxStiffNodes;
    T->DK = d; d += N * kMaxStiffNodes * kMaxS;
    T->PM = d; d += N * kMaxV * kMaxS;
    T->PK = d; d += N * kMaxV * kMaxS;
    T->AW = d; d += N * 128;
    T->PW = d; d += N * kMaxV;
    T->mM = (int*)d;
    T->mK = T->mM + N;
    T->maxM = T->maxK = 0;
    for (int c = 0; c <= R->p; ++c) {
        T->maxM = std::max(T->maxM, R->rules[WGQ_MASS][c].m);
        T->maxK = std::max(T->maxK, R->rules[WGQ_STIFFNESS][c].m);
    }
    ClassArgs A{};
    A.p = R->p;
    A.n = n_dir;
    A.N = N;
    for (int kind = 0; kind < 2; ++kind)
        for (int c = 0; c <= R->p; ++c) {
            A.m[kind][c] = R->rules[kind][c].m;
            for (int k = 0; k < kMaxStiffNodes; ++k) {
                A.tau[kind][c][k] = R->rules[kind][c].tau[k];
                A.omega[kind][c][k] = R->rules[kind][c].omega[k];
            }
        }
    const int64_t threads = N * 2 * kMaxStiffNodes;
    k_row_tables<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(A, *T);
    const int64_t vthreads = N * 2 * kMaxV * kMaxS;
    k_vertex_tables<<<(unsigned)((vthreads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(R->p, n_dir, *T);
    k_weighted_tables<<<(unsigned)((N * 128 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*T);
    k_vertex_weights<<<(unsigned)((N * kMaxV + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*T, R->p);
    if (cudaGetLastError() != cudaSuccess) return WGQ_ECUDA;
    return WGQ_OK;
}

int fetch_interior_tables(const wgq_rules_s* R, int64_t n_dir, RowTables* T) {
    T->int_ok = false;
    const int64_t r = 2 * R->p;                  // first class-I row (class I: 2p <= r <= n-1-p)
    if (r > n_dir - 1 - R->p) return WGQ_OK;     // no class-I rows on this mesh
    int m[2];
    double w[2][kMaxNodes], A[2][kMaxNodes * kMaxS];
    if (cudaMemcpy(&m[0], T->mM + r, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&m[1], T->mK + r, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(w[0], T->wM + r * kMaxMassNodes, sizeof(w[0]), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(w[1], T->wK + r * kMaxStiffNodes, sizeof(w[1]), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(A[0], T->VM + r * kMaxMassNodes * kMaxS, sizeof(A[0]), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(A[1], T->DK + r * kMaxStiffNodes * kMaxS, sizeof(A[1]), cudaMemcpyDeviceToHost) != cudaSuccess)
        return WGQ_ECUDA;
    if (m[0] > kMaxP + 1 || m[1] > kMaxP + 1) return WGQ_OK;
    T->imM = m[0];
    T->imK = m[1];
    for (int k = 0; k <= kMaxP; ++k)
        for (int o = 0; o < kMaxS; ++o) {
            T->iAwM[k][o] = k < m[0] ? w[0][k] * A[0][k * kMaxS + o] : 0.0;
            T->iAwK[k][o] = k < m[1] ? w[1][k] * A[1][k * kMaxS + o] : 0.0;
        }
    T->int_ok = true;
    return WGQ_OK;
}

void free_row_tables(RowTables* T) {
    if (T->base) cudaFree(T->base);
    T->base = nullptr;
}

}  // namespace wgq
