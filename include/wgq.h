/*
 * wgq.h -- C-ABI of the B200-native weighted-Gaussian row-wise IGA assembly library
 *          (libwgq.so, built from paper_1710_01048_b200/csrc).
 *
 * Method: Barton, Puzyrev, Deng, Calo, "Efficient mass and stiffness matrix assembly via
 * weighted Gaussian quadrature rules for B-splines" (arXiv 1710.01048).  Citations are
 * PAPER.md line numbers (P:<line>) with the LaTeX equation label; Rn = DESIGN.md reading n.
 *
 * Discretisation: degree p in {2,3}, open uniform knot vector with n elements
 * per direction on [0,1] (eq:Gmap3), N = n + p basis functions per direction (eq:DimUni),
 * tensor-product basis in d in {1,2,3} directions (eq:Gmap2).  Global rows/columns are
 * lexicographic with x fastest: i = i1 + N*(i2 + N*i3).  Geometry is the identity (J = I),
 * so K_ij = int c grad B_i . grad B_j and M_ij = int c B_i B_j (eq:Stiffness P:159-163,
 * eq:Mass P:170-173), c a coefficient field (R4).
 *
 * Row i is integrated with its own tensor-product weighted Gaussian rule: per
 * direction, m nodes tau_k and weights omega_k with int f W = sum_k omega_k f(tau_k) W(tau_k)
 * exact for the 2p+1 interacting B-splines, W = B_i (mass, eq:GaussQuadSys P:249-252) or
 * W = B'_i (stiffness, eq:GaussQuadSysStiff P:350-353); boundary rows per R1.  The
 * contraction runs direction by direction (eq:Decompo P:194-199) in FP64 on the GPU.
 *
 * Conventions for every function:
 *  - Return 0 (WGQ_OK) or a negative WGQ_E* code; wgq_strerror() describes it.
 *  - Device pointers are CUDA device memory of the CURRENT device; host pointers are
 *    ordinary host memory.  The caller owns every buffer it passes and keeps it alive
 *    until the work enqueued on `stream` has completed.  The library never frees caller
 *    memory.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Kernels are enqueued
 *    asynchronously; no call synchronises except where stated.  Asynchronous CUDA faults
 *    surface at the caller's next synchronisation.
 *  - A rules handle is immutable after wgq_build_rules except for its per-device table
 *    cache, which is mutex-protected: one handle may be used from one thread per GPU.
 */
#ifndef WGQ_H
#define WGQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------------------- */
#define WGQ_OK            0
#define WGQ_EINVAL       -1   /* null/inconsistent descriptor, row range outside [0, N^d)  */
#define WGQ_EUNSUPPORTED -2   /* p not in {2,3}, dim not in {1,2,3}, n_elems < p           */
#define WGQ_ENOCONV      -3   /* a rule failed its Newton solve or residual check (>1e-13) */
#define WGQ_ECUDA        -4   /* CUDA launch/allocation error                              */
#define WGQ_ERANGE       -5   /* ld < (2p+1)^dim, or an index overflow                     */
#define WGQ_ENOMEM       -6   /* host allocation failure                                   */

/* ---- enums --------------------------------------------------------------------------- */
#define WGQ_BND_GAUSS 0       /* R1: minimal Gaussian boundary rules (default)              */
#define WGQ_BND_GL    1       /* R1 alternative: (p+1)-point Gauss-Legendre per element     */

#define WGQ_MASS      0
#define WGQ_STIFFNESS 1

#define WGQ_COEF_CONST        0   /* c = c0                                                    */
#define WGQ_COEF_TRIG_SEP     1   /* c = c0 + amp * prod_a trig_a(2 pi k_a x_a)   (C2, C4; R13) */
#define WGQ_COEF_FOURIER_LOGN 2   /* c = exp(sum_m a_m cos(2 pi k_m . x + theta_m)) (C3; R13)  */
#define WGQ_COEF_GRID         3   /* multilinear interpolation of vertex values (C5; R6)       */

#define WGQ_TRIG_SIN 0
#define WGQ_TRIG_COS 1
#define WGQ_MAX_MODES 16

#define WGQ_ELL 0
#define WGQ_CSR 1

typedef struct wgq_rules_s* wgq_rules_t;

/* Coefficient descriptor (passed by pointer, read during the call only).
 *  CONST        : c0.
 *  TRIG_SEP     : c0, amp, trig[a] (WGQ_TRIG_SIN/COS), wavenum[a] (integer k_a).
 *  FOURIER_LOGN : n_modes <= WGQ_MAX_MODES, modes = HOST array [n_modes][5] of
 *                 (a_m, kx_m, ky_m, kz_m, theta_m); copied by value into the launch.
 *  GRID         : grid = DEVICE array of vertex values, x fastest: d=3 [planes][n+1][n+1],
 *                 d=2 [planes][n+1], d=1 [n+1]; its slowest axis holds vertex planes
 *                 [grid_plane0, grid_plane0 + grid_planes).  Vertex (a,b,c) sits at (a,b,c)/n.
 *                 The planes must cover every element touched by the requested rows:
 *                 [max(0, z0 - p), min(n, z1 + 1)] where z0..z1 is the slowest row index range. */
typedef struct {
    int kind;
    double c0;
    double amp;
    int trig[3];
    int wavenum[3];
    int n_modes;
    const double* modes;
    const double* grid;
    int64_t grid_plane0;
    int64_t grid_planes;
} wgq_coeff_t;

/* Output descriptor.  Rows [row_begin, row_end) of the global matrix are written
 * (a slab; row_begin is output row 0).
 *  ELL: values = DEVICE array [row_end-row_begin][ld]; slot of column j in row i is
 *       (o1+p) + s*((o2+p) + s*(o3+p)), o_a = j_a - i_a, s = 2p+1 (only the first d
 *       offsets exist); slots whose column is outside [0, N) in some direction are +0.0.
 *       ld >= s^d; slots [s^d, ld) are not written.
 *  CSR: row_ptr = DEVICE int64 [rows+1] (slab-local, from 0), col_idx = DEVICE int32 [nnz]
 *       (ascending per row; == the ELL slot order), values = DEVICE [nnz].  row_ptr /
 *       col_idx are filled by wgq_csr_structure; the assembly writes values only. */
typedef struct {
    int layout;
    int64_t row_begin, row_end;
    double* values;
    int64_t ld;
    const int64_t* row_ptr;
    const int32_t* col_idx;
} wgq_out_t;

/* ---- library ------------------------------------------------------------------------- */
const char* wgq_strerror(int code);
const char* wgq_version(void);

/* ---- rules (host, setup) ---------------------------------------------------
 * Builds the interior rules (P:262-279 eq:QuadraticQuadrature, P:299-322 eq:CubicQuadrature,
 * P:372-389 eq:QuadraticQuadratureStiff, P:393-422 eq:CubicQuadratureStiff) and the boundary
 * classes (R1), verifies every rule against exact moments (residual < 1e-13,
 * else WGQ_ENOCONV).  No device work.  *out is owned by the caller: wgq_free_rules(). */
int wgq_build_rules(int p, int64_t n_elems, int dim, wgq_rules_t* out);
int wgq_build_rules_ex(int p, int64_t n_elems, int dim, int boundary_mode, wgq_rules_t* out);
/* Per-direction element counts (eq:Gmap3 P:113-120: each parameter direction has its own
 * knot vector with n_EL^i elements; eq:DimMulti P:134-136: N = prod_i (n_EL^i + p)).  HOST
 * n_elems[a], a < dim, each >= p (else WGQ_EUNSUPPORTED); rows are lexicographic with x
 * fastest, i = i1 + N1 (i2 + N2 i3), N_a = n_a + p; the product of the N_a must stay below 2^31
 * (WGQ_ERANGE).  wgq_build_rules_ex(p, n, ...) is wgq_build_rules_ex2 with n in every direction.
 * On an anisotropic mesh every call works; the specialised kernels (GRID line kernel,
 * separable, 2D FOURIER tensor-core kernels) require equal counts and the assembly, load and
 * apply calls use the generic per-row kernel there. */
int wgq_build_rules_ex2(int p, const int64_t* n_elems, int dim, int boundary_mode, wgq_rules_t* out);
void wgq_free_rules(wgq_rules_t rules);

/* Per-direction sizes: HOST n_elems[3] (0 past dim) and n_rows_dir[3] (N_a; 1 past dim), NULL skips. */
int wgq_rules_dims(wgq_rules_t rules, int64_t* n_elems, int64_t* n_rows_dir);

/* Sizes: N = n+p rows of direction 0 (every direction on an isotropic mesh), n_rows = the
 * product of the per-direction row counts, stencil = (2p+1)^dim (NULL skips). */
int wgq_rules_info(wgq_rules_t rules, int* p, int64_t* n_elems, int* dim,
                   int64_t* n_rows_1d, int64_t* n_rows, int* stencil);

/* Unit-spacing rule of a direction class: cls in [0, p) = left boundary weight j = cls,
 * cls == p = interior (shift-invariant) rule; right boundary classes are mirrors (R1).
 * kind = WGQ_MASS / WGQ_STIFFNESS.  Writes m (<= 12) nodes tau (from the left end of the
 * support), weights omega (paper convention) and the max exactness residual.
 * Nodes with zero effective weight (p=2 stiffness tau_2 = 3/2, R2) are omitted. */
int wgq_rules_query(wgq_rules_t rules, int cls, int kind, int* m,
                    double* tau, double* omega, double* max_residual);

/* Basis-evaluation counts (experiment E3).  For the full mesh of
 * the handle and kind = WGQ_MASS / WGQ_STIFFNESS: the number of evaluations of the 2p+1
 * interacting functions (B resp. B') that are nonzero at the points of every row's rule where
 * the weight B_i (B'_i) is nonzero, summed over rows (a tensor row costs the product over its
 * directions): *gaussian for this library's weighted Gaussian rules, *newton_cotes for the
 * knot-and-midpoint point sets of the weighted Newton-Cotes rules the paper compares against.
 * Host only; WGQ_EINVAL for bad arguments. */
int wgq_eval_counts(wgq_rules_t rules, int kind, int64_t* gaussian, int64_t* newton_cotes);

/* Structural nonzeros of rows [row_begin, row_end) (per matrix). */
int wgq_nnz(wgq_rules_t rules, int64_t row_begin, int64_t row_end, int64_t* nnz);

/* ---- assembly (device, the hot path) ---------------------------------------------------
 * Enqueue the assembly of rows [out.row_begin, out.row_end) of M and/or K on `stream`.
 * The fused call evaluates each row once for both matrices (M->row range must equal
 * K->row range).  Per-row arithmetic is independent of the slab/launch, so any split of
 * the rows gives bitwise-identical values. */
int wgq_assemble_mass(wgq_rules_t rules, const wgq_coeff_t* c, const wgq_out_t* M, void* stream);
int wgq_assemble_stiffness(wgq_rules_t rules, const wgq_coeff_t* c, const wgq_out_t* K, void* stream);
int wgq_assemble_mass_stiffness(wgq_rules_t rules, const wgq_coeff_t* c,
                                const wgq_out_t* M, const wgq_out_t* K, void* stream);

/* CSR structure of rows [row_begin, row_end): row_ptr (closed form, no scan) and col_idx
 * into caller-owned DEVICE arrays of sizes rows+1 and nnz (wgq_nnz). */
int wgq_csr_structure(wgq_rules_t rules, int64_t row_begin, int64_t row_end,
                      int64_t* row_ptr, int32_t* col_idx, void* stream);

/* ---- load vector (eq:Load) --------------------------------
 * b[i - row_begin] = sum_k [prod_a w^M_{i_a,k_a}] f(x^M_k) for rows [row_begin, row_end):
 * row i's own mass-kind weighted rule (the measure B_i, eq:GaussQuadSys P:249-252) applied
 * to f, a coefficient descriptor (GRID f must cover the rows' vertex planes as for the
 * assembly).  Exact when f lies in the row's spline space (constants, linear functions).
 * b: caller-owned DEVICE double[row_end - row_begin].  Enqueued on `stream`; errors as for
 * the assembly (WGQ_EINVAL for a null b / bad range / bad descriptor). */
int wgq_assemble_load(wgq_rules_t rules, const wgq_coeff_t* f, int64_t row_begin, int64_t row_end,
                      double* b, void* stream);

/* ---- matrix-free application (the consumer of the row-wise scheme)
 * y_M[i - row_begin] = sum_j M_ij u_j and y_K[i - row_begin] = sum_j K_ij u_j for rows
 * [row_begin, row_end), M and K exactly as wgq_assemble_* defines them for (rules, c): each
 * row is formed on the fly and contracted with u, nothing is stored.  u: DEVICE vector of
 * the global rows [u_row0, u_row0 + u_rows), which must contain every column of the rows
 * (slowest-axis planes z0-p .. z1+p of the slab, clipped to the mesh), else WGQ_ERANGE.
 * y_M, y_K: caller-owned DEVICE double[row_end - row_begin]; either may be NULL (not both). */
int wgq_apply(wgq_rules_t rules, const wgq_coeff_t* c, const double* u, int64_t u_row0, int64_t u_rows,
              int64_t row_begin, int64_t row_end, double* y_M, double* y_K, void* stream);

/* ---- end to end from/to HOST memory ---------------------------------------------------
 * Blocking convenience call for callers whose inputs and outputs live in host memory:
 * uploads the coefficient (for GRID, c->grid is a HOST pointer to the vertex planes
 * [c->grid_plane0, +grid_planes), which must cover the rows as for the device call),
 * assembles rows [row_begin, row_end) in chunks of `chunk_rows` (0 = automatic) on the
 * current device and streams each finished chunk into the HOST ELL arrays M_host / K_host
 * (row stride ld >= s^d, slots [s^d, ld) of each host row are not written; either array may
 * be NULL to skip that matrix) while the next chunk is
 * computed (two CUDA streams, double-buffered device staging that the call allocates and
 * frees).  Use page-locked host memory (wgq_host_alloc) for full PCIe bandwidth.  Returns
 * after all copies have completed. */
int wgq_assemble_host(wgq_rules_t rules, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end,
                      double* M_host, double* K_host, int64_t ld, int64_t chunk_rows);

/* Page-locked host memory (cudaHostAlloc / cudaFreeHost) for wgq_assemble_host. */
int wgq_host_alloc(uint64_t bytes, void** ptr);
int wgq_host_free(void* ptr);

/* ---- inputs / checks ------------------------------------------------------------------
 * Device generation of the seeded smoothed lognormal vertex field: vertex
 * planes [plane0, plane0+planes) of the (n+1)^dim field into grid (DEVICE, layout as in
 * wgq_coeff_t).  Every value depends only on its global vertex, so slabs of any split
 * agree with a global generation. */
int wgq_generate_grid(int64_t n_elems, int dim, uint64_t seed, double sigma,
                      int64_t plane0, int64_t planes, double* grid, void* stream);
/* The same field on a mesh with per-direction element counts (HOST n_elems[dim]; vertex planes
 * of (n_y+1) x (n_x+1) values, n_z+1 planes in 3D): white-noise keys
 * ((c+4)(n_y+9) + (b+4))(n_x+9) + (a+4) (SURVEY c.4 for equal counts). */
int wgq_generate_grid_ex(const int64_t* n_elems, int dim, uint64_t seed, double sigma,
                         int64_t plane0, int64_t planes, double* grid, void* stream);

/* Per-row products of an assembled ELL slab with the vectors 1 and g^a (Greville abscissae
 * of direction a, sum_j g_j B_j(x) = x): out = DEVICE [rows][1+dim] = (A 1, A g^1, ..).
 * These are the full-coverage identities of SURVEY §8(c) P9 (checks; not timed). */
int wgq_row_moments(wgq_rules_t rules, const wgq_out_t* A, double* out, void* stream);

/* Order-independent checksum of an ELL slab's structural entries: sum of a 64-bit mix of
 * (row, slot, value bits) mod 2^64, and the FP64 sums of v and v^2 (DEVICE out[3] as
 * uint64 / double / double, reduced with atomics: the hash is exact, the sums are not
 * bitwise-reproducible).  Used to compare slabs across GPUs. */
int wgq_checksum(wgq_rules_t rules, const wgq_out_t* A, unsigned long long* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WGQ_H */
