// Internal declarations shared by the host rule builder, the C-ABI layer and the CUDA
// kernels of libwgq.  Nothing here is part of the public ABI (include/wgq.h).
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <array>
#include <tuple>

#include "wgq.h"

#include <nvtx3/nvToolsExt.h>

#ifdef __CUDACC__
#define WGQ_HD __host__ __device__
#else
#define WGQ_HD
#endif

namespace wgq {

// NVTX range over a library call (SURVEY §5 tracing: rules, tables, grid generation, assembly,
// operators); header-only NVTX3, a no-op unless a tool (nsys / ncu) is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kMaxP = 3;

// Mesh sizes per direction (eq:Gmap3 P:113-120: every parameter direction has its own element
// count n_EL^i; eq:DimMulti P:134-136): n[a] elements and N[a] = n[a] + p basis functions in
// direction a < dim (entries past dim are 1).  Rows are lexicographic with x fastest:
// i = i_1 + N_1 (i_2 + N_2 i_3).
struct Dims {
    int dim = 1;
    int64_t n[3] = {1, 1, 1};
    int64_t N[3] = {1, 1, 1};
    WGQ_HD int64_t rows() const { return N[0] * N[1] * N[2]; }
    // rows of one slab unit along the slowest axis (a line in 2D, a plane in 3D)
    WGQ_HD int64_t plane_rows() const {
        int64_t r = 1;
        for (int a = 0; a < dim - 1; ++a) r *= N[a];
        return r;
    }
    WGQ_HD void decode(int64_t row, int64_t* idx) const {
        for (int a = 0; a < 3; ++a) {
            idx[a] = a < dim ? row % N[a] : 0;
            if (a < dim) row /= N[a];
        }
    }
    WGQ_HD bool iso() const {
        for (int a = 1; a < dim; ++a)
            if (n[a] != n[0]) return false;
        return true;
    }
};
constexpr int kMaxS = 2 * kMaxP + 1;   // stencil width per direction
constexpr int kMaxNodes = 12;          // per direction: GL(p+1) on up to p elements (R1, WGQ_BND_GL)
constexpr int kMaxMassNodes = kMaxNodes;
constexpr int kMaxStiffNodes = kMaxNodes;
constexpr int kMaxV = kMaxP + 2;       // vertex planes touched by one row's support

// One unit-spacing rule of a direction class (paper convention, P:250 / P:351).
struct ClassRule {
    int m = 0;
    double tau[kMaxStiffNodes] = {};
    double omega[kMaxStiffNodes] = {};
    double residual = 0.0;
};

// Per-1D-row tables produced on the device by the table kernel (tables.cu).
// Layout: struct of arrays over the N rows of one direction (all directions share it).
struct RowTables {
    int64_t N = 0;
    int maxM = 0, maxK = 0;    // largest node counts over all rows (sizes the kernels' staging)
    int* mM = nullptr;         // [N]   mass nodes of row r
    int* mK = nullptr;         // [N]   stiffness nodes of row r
    double* xM = nullptr;      // [N][kMaxMassNodes]   physical nodes
    double* wM = nullptr;      // [N][kMaxMassNodes]   effective weights omega*B_r(x)
    double* VM = nullptr;      // [N][kMaxMassNodes][kMaxS]  B_{r+o}(x_k), o = -p..p
    double* xK = nullptr;      // [N][kMaxStiffNodes]
    double* wK = nullptr;      // [N][kMaxStiffNodes]  omega*B'_r(x)
    double* DK = nullptr;      // [N][kMaxStiffNodes][kMaxS] B'_{r+o}(x_k)
    // Vertex-projected tables for a multilinear (GRID) coefficient: with b_r = max(0, r-p),
    //   PM[r][v][o] = sum_k wM[k] B_{r+o}(x_k) lambda_v(x_k),  PK likewise with wK, B',
    // lambda_v = the hat function of vertex plane b_r + v (v < p+2), i.e. the node's
    // interpolation weight on that vertex.  sum_v g_{b+v} PM[v][o] is the 1D rule applied
    // to c * B_{r+o} when c is the vertex field's linear interpolant (R6).
    double* PM = nullptr;      // [N][kMaxV][kMaxS]
    double* PK = nullptr;      // [N][kMaxV][kMaxS]
    // PW[r][v] = sum_o PM[r][v][o] = sum_k wM[k] lambda_v(x_k) (partition of unity): the mass
    // rule's weight on vertex plane b_r + v, the load vector's vertex projection
    double* PW = nullptr;      // [N][kMaxV]
    // Weighted 1D tables of the first 8 nodes, for the 2D FOURIER kernels (fourier2d.cu):
    // AW[r][kind][k][o] = w_k B_{r+o}(x_k) (kind 0, mass) / w_k B'_{r+o}(x_k) (kind 1), o < 7, zero
    // for k >= m and o = 7 (rows with more than 8 nodes are not read through it)
    double* AW = nullptr;      // [N][2][8][8]
    void* base = nullptr;      // single allocation
    // Host copies of one class-I (interior, 2p <= r <= N-1-2p) row's weighted tables
    // iAwM[k][o] = wM[k] VM[k][o], iAwK[k][o] = wK[k] DK[k][o] (shift-invariant up to rounding:
    // the interior kernels take them as kernel parameters), filled after the one-time build.
    bool int_ok = false;
    int imM = 0, imK = 0;
    double iAwM[kMaxP + 1][kMaxS] = {};
    double iAwK[kMaxP + 1][kMaxS] = {};
};

// The row tables of every direction (t[a] = t[0] on an isotropic mesh).
struct Tables3 {
    RowTables t[3];
};

}  // namespace wgq

struct wgq_rules_s {
    int p = 0;
    int dim = 0;
    int bnd = WGQ_BND_GAUSS;
    int64_t n = 0;             // direction 0 (every direction when the mesh is isotropic)
    int64_t N = 0;
    wgq::Dims dims;            // per-direction sizes
    bool iso = true;           // equal element counts in every direction (the specialised kernels)
    // rules[kind][cls]: cls 0..p-1 = left boundary weight j, cls p = interior
    wgq::ClassRule rules[2][wgq::kMaxP + 1];
    std::mutex mu;
    std::map<int, wgq::RowTables> tables;   // per CUDA device
    // separable-coefficient vectors (separable.cu), per (device, kind, trig[3], wavenum[3])
    std::map<std::array<int, 8>, double*> sep_vectors;
};

namespace wgq {

// rules.cpp (host)
int build_class_rules(int p, int bnd, ClassRule out[2][kMaxP + 1]);
// Unit-spacing vertex-projected tables of the interior (shift-invariant) rule:
// PM[v][o] = sum_k omega_k B(tau_k) B_o(tau_k) lambda_v(tau_k) (mass), PK with B' (stiffness).
void interior_vertex_tables(int p, const ClassRule& mass, const ClassRule& stiff, double PM[kMaxV][kMaxS],
                            double PK[kMaxV][kMaxS]);

// Basis-evaluation counts of the Gaussian and Newton-Cotes weighted schemes (E3).
void eval_counts(const wgq_rules_s* R, int kind, int64_t* gaussian, int64_t* newton_cotes);

// tables.cu
int build_row_tables(const wgq_rules_s* R, int64_t n, RowTables* T, void* stream);   // one direction, n elements
void free_row_tables(RowTables* T);

// assemble.cu
#ifdef __CUDACC__
// The 2D shell rows of [row_begin, row_end) (rows touching a GL-fallback boundary class), generated
// on the device into stream-ordered scratch the caller frees with cudaFreeAsync on the same stream.
int shell_rows_2d(const wgq_rules_s* R, int64_t row_begin, int64_t row_end, cudaStream_t st, int64_t** rows,
                  int64_t* count);
#endif
int launch_assemble(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c,
                    const wgq_out_t* M, const wgq_out_t* K, void* stream);
int launch_csr_structure(const wgq_rules_s* R, int64_t row_begin, int64_t row_end,
                         int64_t* row_ptr, int32_t* col_idx, void* stream);
int launch_row_moments(const wgq_rules_s* R, const wgq_out_t* A, double* out, void* stream);
int launch_checksum(const wgq_rules_s* R, const wgq_out_t* A, unsigned long long* out, void* stream);

// load vector / matrix-free application (assemble.cu)
int launch_load(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                double* b, void* stream);
int launch_apply(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const double* u, int64_t u_row0,
                 int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream);

// assemble_line.cu (GRID coefficient, d = 3, ELL)
bool line_kernel_applies(const wgq_rules_s* R, const wgq_coeff_t* c, const wgq_out_t* M, const wgq_out_t* K);
int launch_line(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const wgq_out_t* M,
                const wgq_out_t* K, void* stream);
bool line_apply_applies(const wgq_rules_s* R, const wgq_coeff_t* c);
int launch_sep_load(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                    double* b, void* stream);
int launch_sep_apply(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const double* u, int64_t u_row0,
                     int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream);
int launch_line_apply(const wgq_rules_s* R, const Tables3& TT, const wgq_coeff_t* c, const double* u,
                      int64_t u_row0, int64_t row_begin, int64_t row_end, double* yM, double* yK, void* stream);

// api.cpp: the coefficient descriptor check of the assembly calls, for a row range
int validate_coeff_range(const wgq_rules_s* R, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end);

// fourier2d.cu (2D FOURIER_LOGN, p = 3, rows of class I in both directions; C3)
bool f2d_interior_applies(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c);
#ifdef __CUDACC__
int launch_f2d_interior(const wgq_rules_s* R, const RowTables& T, const double* ctab, int cw, const wgq_out_t* M,
                        const wgq_out_t* K, const int64_t* shell, int64_t nshell, cudaStream_t st);
#endif
int fetch_interior_tables(const wgq_rules_s* R, int64_t n, RowTables* T);

// separable.cu (CONST, TRIG_SEP coefficients)
bool sep_applies(const wgq_coeff_t* c);
int launch_sep(const wgq_rules_s* R, const RowTables& T, const wgq_coeff_t* c, const wgq_out_t* M,
               const wgq_out_t* K, void* stream);

// grid.cu
int launch_generate_grid(const int64_t* n, int dim, uint64_t seed, double sigma, int64_t plane0,
                         int64_t planes, double* grid, void* stream);


#ifdef __CUDACC__
// Streaming output stores of the assembled values: no L1 allocation and L2 evict-first, so the
// write stream neither evicts the small per-row tables from L1 nor the coefficient data from L2
// (C4: 0.45 -> 0.36 ms).
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_stream(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
#endif

}  // namespace wgq
