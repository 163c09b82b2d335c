// C-ABI of libwgq (include/wgq.h): argument validation, the per-device table cache and
// dispatch to the CUDA launchers.  No arithmetic of the method lives here.
#include <cuda_runtime.h>

#include <cstring>
#include <new>

#include "internal.h"

namespace wgq {
int64_t host_nnz_before(int64_t row, int p, const Dims& D);
}

using namespace wgq;

namespace {

int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

// Row tables of direction dir (per device; directions with the same element count share one).
int table_for(wgq_rules_s* R, int dir, RowTables* out, void* stream) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return WGQ_ECUDA;
    int src = dir;
    for (int a = 0; a < dir; ++a)
        if (R->dims.n[a] == R->dims.n[dir]) {
            src = a;
            break;
        }
    std::lock_guard<std::mutex> lock(R->mu);
    auto it = R->tables.find(dev * 4 + src);
    if (it == R->tables.end()) {
        NvtxRange nvtx_("wgq_row_tables (one-time build)");
        RowTables T;
        int rc = build_row_tables(R, R->dims.n[src], &T, stream);
        if (rc != WGQ_OK) return rc;
        // the cache is used from any stream afterwards: complete the one-time build now
        if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return WGQ_ECUDA;
        if (fetch_interior_tables(R, R->dims.n[src], &T) != WGQ_OK) return WGQ_ECUDA;
        // keep stream-ordered scratch (coefficient tables) in the device pool between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        it = R->tables.emplace(dev * 4 + src, T).first;
    }
    *out = it->second;
    return WGQ_OK;
}

int tables_for(wgq_rules_s* R, Tables3* out, void* stream) {
    for (int a = 0; a < 3; ++a) {
        const int d = a < R->dim ? a : 0;
        int rc = table_for(R, d, &out->t[a], stream);
        if (rc != WGQ_OK) return rc;
    }
    return WGQ_OK;
}

int check_out(const wgq_rules_s* R, const wgq_out_t* o) {
    if (!o) return WGQ_EINVAL;
    const int64_t total = R->dims.rows();
    if (o->row_begin < 0 || o->row_end < o->row_begin || o->row_end > total) return WGQ_EINVAL;
    if (o->layout != WGQ_ELL && o->layout != WGQ_CSR) return WGQ_EINVAL;
    if (o->row_end > o->row_begin && !o->values) return WGQ_EINVAL;
    if (o->layout == WGQ_ELL && o->ld < ipow(2 * R->p + 1, R->dim)) return WGQ_ERANGE;
    if (o->layout == WGQ_CSR && !o->row_ptr) return WGQ_EINVAL;
    return WGQ_OK;
}

int check_coeff(const wgq_rules_s* R, const wgq_coeff_t* c, const wgq_out_t* o) {
    if (!c) return WGQ_EINVAL;
    switch (c->kind) {
        case WGQ_COEF_CONST:
            return WGQ_OK;
        case WGQ_COEF_TRIG_SEP:
            for (int a = 0; a < R->dim; ++a)
                if (c->trig[a] != WGQ_TRIG_SIN && c->trig[a] != WGQ_TRIG_COS) return WGQ_EINVAL;
            return WGQ_OK;
        case WGQ_COEF_FOURIER_LOGN:
            if (c->n_modes < 0 || c->n_modes > WGQ_MAX_MODES || (c->n_modes > 0 && !c->modes)) return WGQ_EINVAL;
            return WGQ_OK;
        case WGQ_COEF_GRID: {
            if (!c->grid && o->row_end > o->row_begin) return WGQ_EINVAL;
            if (o->row_end <= o->row_begin) return WGQ_OK;
            const int64_t plane_rows = R->dims.plane_rows();
            const int64_t nz = R->dims.n[R->dim - 1];              // elements along the slowest axis
            const int64_t z0 = o->row_begin / plane_rows, z1 = (o->row_end - 1) / plane_rows;
            const int64_t need_lo = z0 - R->p > 0 ? z0 - R->p : 0;
            const int64_t need_hi = z1 + 1 < nz ? z1 + 1 : nz;
            if (c->grid_plane0 > need_lo || c->grid_plane0 + c->grid_planes - 1 < need_hi) return WGQ_EINVAL;
            return WGQ_OK;
        }
    }
    return WGQ_EINVAL;
}

int assemble(wgq_rules_t R, const wgq_coeff_t* c, const wgq_out_t* M, const wgq_out_t* K, void* stream) {
    if (!R) return WGQ_EINVAL;
    int rc;
    if (M && (rc = check_out(R, M)) != WGQ_OK) return rc;
    if (K && (rc = check_out(R, K)) != WGQ_OK) return rc;
    if (M && K && (M->row_begin != K->row_begin || M->row_end != K->row_end || M->layout != K->layout))
        return WGQ_EINVAL;
    const wgq_out_t* any = M ? M : K;
    if ((rc = check_coeff(R, c, any)) != WGQ_OK) return rc;
    if (any->row_end == any->row_begin) return WGQ_OK;
    Tables3 TT;
    if ((rc = tables_for(R, &TT, stream)) != WGQ_OK) return rc;
    return launch_assemble(R, TT, c, M, K, stream);
}

}  // namespace

namespace wgq {
int validate_coeff_range(const wgq_rules_s* R, const wgq_coeff_t* c, int64_t row_begin, int64_t row_end) {
    wgq_out_t range{WGQ_ELL, row_begin, row_end, nullptr, 0, nullptr, nullptr};
    return check_coeff(R, c, &range);
}
}  // namespace wgq

extern "C" {

const char* wgq_strerror(int code) {
    switch (code) {
        case WGQ_OK: return "ok";
        case WGQ_EINVAL: return "invalid argument (null or inconsistent descriptor, row range outside [0, N^d))";
        case WGQ_EUNSUPPORTED: return "unsupported: p must be 2 or 3, dim 1..3, n_elems >= p";
        case WGQ_ENOCONV: return "a quadrature rule failed its Newton solve or exactness check (residual > 1e-13)";
        case WGQ_ECUDA: return "CUDA launch or allocation error";
        case WGQ_ERANGE: return "ld < (2p+1)^dim or index overflow";
        case WGQ_ENOMEM: return "host allocation failure";
    }
    return "unknown error";
}

const char* wgq_version(void) { return "wgq 0.1 (sm_100a)"; }

int wgq_build_rules_ex2(int p, const int64_t* n_elems, int dim, int boundary_mode, wgq_rules_t* out) {
    NvtxRange nvtx_("wgq_build_rules");
    if (!out || !n_elems) return WGQ_EINVAL;
    *out = nullptr;
    if (p != 2 && p != 3) return WGQ_EUNSUPPORTED;
    if (dim < 1 || dim > 3) return WGQ_EUNSUPPORTED;
    Dims D;
    D.dim = dim;
    int64_t rows = 1;
    for (int a = 0; a < dim; ++a) {
        if (n_elems[a] < p) return WGQ_EUNSUPPORTED;
        if (n_elems[a] >= ((int64_t)1 << 31)) return WGQ_ERANGE;
        D.n[a] = n_elems[a];
        D.N[a] = n_elems[a] + p;
        rows *= D.N[a];
        if (rows >= ((int64_t)1 << 31)) return WGQ_ERANGE;   // int32 column ids
    }
    if (boundary_mode != WGQ_BND_GAUSS && boundary_mode != WGQ_BND_GL) return WGQ_EINVAL;
    wgq_rules_s* R = new (std::nothrow) wgq_rules_s();
    if (!R) return WGQ_ENOMEM;
    R->p = p;
    R->dim = dim;
    R->dims = D;
    R->iso = D.iso();
    R->n = D.n[0];
    R->N = D.N[0];
    R->bnd = boundary_mode;
    int rc = build_class_rules(p, boundary_mode, R->rules);
    if (rc != WGQ_OK) {
        delete R;
        return rc;
    }
    *out = R;
    return WGQ_OK;
}

int wgq_build_rules_ex(int p, int64_t n_elems, int dim, int boundary_mode, wgq_rules_t* out) {
    const int64_t n[3] = {n_elems, n_elems, n_elems};
    return wgq_build_rules_ex2(p, n, dim, boundary_mode, out);
}

int wgq_rules_dims(wgq_rules_t R, int64_t* n_elems, int64_t* n_rows_dir) {
    if (!R) return WGQ_EINVAL;
    for (int a = 0; a < 3; ++a) {
        if (n_elems) n_elems[a] = a < R->dim ? R->dims.n[a] : 0;
        if (n_rows_dir) n_rows_dir[a] = a < R->dim ? R->dims.N[a] : 1;
    }
    return WGQ_OK;
}

int wgq_build_rules(int p, int64_t n_elems, int dim, wgq_rules_t* out) {
    return wgq_build_rules_ex(p, n_elems, dim, WGQ_BND_GAUSS, out);
}

void wgq_free_rules(wgq_rules_t R) {
    if (!R) return;
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : R->tables) {
        cudaSetDevice(kv.first / 4);                 // key = device * 4 + direction
        free_row_tables(&kv.second);
    }
    for (auto& kv : R->sep_vectors) {
        cudaSetDevice(kv.first[0]);
        cudaFree(kv.second);
    }
    cudaSetDevice(cur);
    delete R;
}

int wgq_rules_info(wgq_rules_t R, int* p, int64_t* n_elems, int* dim, int64_t* n_rows_1d, int64_t* n_rows,
                   int* stencil) {
    if (!R) return WGQ_EINVAL;
    if (p) *p = R->p;
    if (n_elems) *n_elems = R->n;
    if (dim) *dim = R->dim;
    if (n_rows_1d) *n_rows_1d = R->N;
    if (n_rows) *n_rows = R->dims.rows();
    if (stencil) *stencil = (int)ipow(2 * R->p + 1, R->dim);
    return WGQ_OK;
}

int wgq_rules_query(wgq_rules_t R, int cls, int kind, int* m, double* tau, double* omega, double* max_residual) {
    if (!R || !m || cls < 0 || cls > R->p || (kind != WGQ_MASS && kind != WGQ_STIFFNESS)) return WGQ_EINVAL;
    const ClassRule& c = R->rules[kind][cls];
    *m = c.m;
    if (tau) std::memcpy(tau, c.tau, sizeof(double) * c.m);
    if (omega) std::memcpy(omega, c.omega, sizeof(double) * c.m);
    if (max_residual) *max_residual = c.residual;
    return WGQ_OK;
}

int wgq_nnz(wgq_rules_t R, int64_t row_begin, int64_t row_end, int64_t* nnz) {
    if (!R || !nnz) return WGQ_EINVAL;
    if (row_begin < 0 || row_end < row_begin || row_end > R->dims.rows()) return WGQ_EINVAL;
    *nnz = host_nnz_before(row_end, R->p, R->dims) - host_nnz_before(row_begin, R->p, R->dims);
    return WGQ_OK;
}

int wgq_assemble_mass(wgq_rules_t R, const wgq_coeff_t* c, const wgq_out_t* M, void* stream) {
    NvtxRange nvtx_("wgq_assemble_mass");
    if (!M) return WGQ_EINVAL;
    return assemble(R, c, M, nullptr, stream);
}

int wgq_assemble_stiffness(wgq_rules_t R, const wgq_coeff_t* c, const wgq_out_t* K, void* stream) {
    NvtxRange nvtx_("wgq_assemble_stiffness");
    if (!K) return WGQ_EINVAL;
    return assemble(R, c, nullptr, K, stream);
}

int wgq_assemble_mass_stiffness(wgq_rules_t R, const wgq_coeff_t* c, const wgq_out_t* M, const wgq_out_t* K,
                                void* stream) {
    NvtxRange nvtx_("wgq_assemble_mass_stiffness");
    if (!M || !K) return WGQ_EINVAL;
    return assemble(R, c, M, K, stream);
}

int wgq_assemble_load(wgq_rules_t R, const wgq_coeff_t* f, int64_t row_begin, int64_t row_end, double* b,
                      void* stream) {
    NvtxRange nvtx_("wgq_assemble_load");
    if (!R || row_begin < 0 || row_end < row_begin || row_end > R->dims.rows()) return WGQ_EINVAL;
    if (row_end > row_begin && !b) return WGQ_EINVAL;
    wgq_out_t range{};
    range.row_begin = row_begin;
    range.row_end = row_end;
    int rc;
    if ((rc = check_coeff(R, f, &range)) != WGQ_OK) return rc;
    if (row_end == row_begin) return WGQ_OK;
    Tables3 TT;
    if ((rc = tables_for(R, &TT, stream)) != WGQ_OK) return rc;
    return launch_load(R, TT, f, row_begin, row_end, b, stream);
}

int wgq_apply(wgq_rules_t R, const wgq_coeff_t* c, const double* u, int64_t u_row0, int64_t u_rows, int64_t row_begin,
              int64_t row_end, double* y_M, double* y_K, void* stream) {
    NvtxRange nvtx_("wgq_apply");
    if (!R || row_begin < 0 || row_end < row_begin || row_end > R->dims.rows()) return WGQ_EINVAL;
    if (row_end == row_begin) return WGQ_OK;
    if (!u || (!y_M && !y_K) || u_row0 < 0 || u_rows < 0) return WGQ_EINVAL;
    // u must hold every column of the rows: the slowest-axis planes z0-p .. z1+p (clipped)
    const int64_t plane_rows = R->dims.plane_rows();
    const int64_t Nz = R->dims.N[R->dim - 1];
    const int64_t z0 = row_begin / plane_rows, z1 = (row_end - 1) / plane_rows;
    const int64_t need_lo = (z0 - R->p > 0 ? z0 - R->p : 0) * plane_rows;
    const int64_t need_hi = (z1 + R->p + 1 < Nz ? z1 + R->p + 1 : Nz) * plane_rows;
    if (R->dim == 1) {
        if (u_row0 > (row_begin - R->p > 0 ? row_begin - R->p : 0) ||
            u_row0 + u_rows < (row_end + R->p < Nz ? row_end + R->p : Nz))
            return WGQ_ERANGE;
    } else if (u_row0 > need_lo || u_row0 + u_rows < need_hi) {
        return WGQ_ERANGE;
    }
    wgq_out_t range{};
    range.row_begin = row_begin;
    range.row_end = row_end;
    int rc;
    if ((rc = check_coeff(R, c, &range)) != WGQ_OK) return rc;
    Tables3 TT;
    if ((rc = tables_for(R, &TT, stream)) != WGQ_OK) return rc;
    return launch_apply(R, TT, c, u, u_row0, row_begin, row_end, y_M, y_K, stream);
}

int wgq_eval_counts(wgq_rules_t R, int kind, int64_t* gaussian, int64_t* newton_cotes) {
    if (!R || !gaussian || !newton_cotes || (kind != WGQ_MASS && kind != WGQ_STIFFNESS)) return WGQ_EINVAL;
    eval_counts(R, kind, gaussian, newton_cotes);
    return WGQ_OK;
}

int wgq_csr_structure(wgq_rules_t R, int64_t row_begin, int64_t row_end, int64_t* row_ptr, int32_t* col_idx,
                      void* stream) {
    NvtxRange nvtx_("wgq_csr_structure");
    if (!R || !row_ptr || row_begin < 0 || row_end < row_begin || row_end > R->dims.rows()) return WGQ_EINVAL;
    if (row_end > row_begin && !col_idx) return WGQ_EINVAL;
    return launch_csr_structure(R, row_begin, row_end, row_ptr, col_idx, stream);
}

int wgq_generate_grid_ex(const int64_t* n_elems, int dim, uint64_t seed, double sigma, int64_t plane0, int64_t planes,
                         double* grid, void* stream) {
    NvtxRange nvtx_("wgq_generate_grid");
    if (!grid || !n_elems || dim < 1 || dim > 3 || planes < 0 || plane0 < 0) return WGQ_EINVAL;
    for (int a = 0; a < dim; ++a)
        if (n_elems[a] < 1) return WGQ_EINVAL;
    const int64_t nz = n_elems[dim - 1];                        // the slowest axis
    if (dim == 1 && (plane0 != 0 || planes != nz + 1)) return WGQ_EINVAL;
    if (plane0 + planes > nz + 1) return WGQ_EINVAL;
    if (planes == 0) return WGQ_OK;
    return launch_generate_grid(n_elems, dim, seed, sigma, plane0, planes, grid, stream);
}

int wgq_generate_grid(int64_t n_elems, int dim, uint64_t seed, double sigma, int64_t plane0, int64_t planes,
                      double* grid, void* stream) {
    const int64_t n[3] = {n_elems, n_elems, n_elems};
    return wgq_generate_grid_ex(n, dim, seed, sigma, plane0, planes, grid, stream);
}

int wgq_row_moments(wgq_rules_t R, const wgq_out_t* A, double* out, void* stream) {
    NvtxRange nvtx_("wgq_row_moments");
    if (!R || !out) return WGQ_EINVAL;
    int rc = check_out(R, A);
    if (rc != WGQ_OK) return rc;
    if (A->layout != WGQ_ELL) return WGQ_EINVAL;
    return launch_row_moments(R, A, out, stream);
}

int wgq_checksum(wgq_rules_t R, const wgq_out_t* A, unsigned long long* out_dev, void* stream) {
    NvtxRange nvtx_("wgq_checksum");
    if (!R || !out_dev) return WGQ_EINVAL;
    int rc = check_out(R, A);
    if (rc != WGQ_OK) return rc;
    if (A->layout != WGQ_ELL) return WGQ_EINVAL;
    return launch_checksum(R, A, out_dev, stream);
}

}  // extern "C"
