// Host-side construction of the weighted Gaussian rules (setup, not the hot path).
//
// Paper: Sec. 3.  Every rule is stored in unit element spacing with nodes
// measured from the left end of the weight's support, in the paper's convention
//     int f W = sum_k omega_k f(tau_k) W(tau_k),   W = B_j (mass) or B'_j (stiffness)
// (eq:GaussQuadW P:242-244, eq:GaussQuadSys P:249-252, eq:GaussQuadSysStiff P:350-353).
//
//  interior p=2 mass : closed form of eq:QuadraticQuadrature: eliminating
//                      omega_1, omega_2 leaves 26 tau^2 - 48 tau + 21 = 0.
//  interior p=3 mass : damped Newton on the symmetric system eq:CubicQuadrature with the
//                      brackets tau_1 in (0,1), tau_2 in (1,2) of P:326 and multi-start.
//  interior p=2 stiff: tau = 3/4, 9/4, omega = 8/9 (eq:WQquadraticStiff P:383-388); the
//                      middle node has zero effective weight (R2) and is dropped.
//  interior p=3 stiff: omega_1 = 1, tau_1 = 1/2 - sqrt(225-30 sqrt 30)/30 (eq:CubicStiffTau1,
//                      P:412), (tau_2, omega_2) by Newton on lines 2 and 4 of
//                      eq:CubicQuadratureStiff (true signs R3).
//  boundary j < p    : reading R1 (remark P:438-440).
// Each rule is checked against exact moments over the full interacting set (< 1e-13).
// All of the setup arithmetic runs in x87 extended precision (long double, 64-bit mantissa)
// and each node/weight is rounded to double once, so the tables are correctly rounded
// (R14) instead of carrying the fp64 residual floor times the condition number.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "internal.h"

namespace wgq {
namespace {

using real = long double;

// ---------------------------------------------------------------------------------------
// B-splines on an explicit knot vector: all nonzero functions of a span and their
// derivatives (triangular de Boor table, Piegl & Tiller's algorithm A2.3).
// ---------------------------------------------------------------------------------------
struct Knots {
    std::vector<real> t;
    int p;
    int nfun() const { return (int)t.size() - p - 1; }
    int span(real x) const {
        int hi = nfun();                       // last valid span index is nfun()-1
        if (x >= t[hi]) return hi - 1;
        int s = p;
        while (s < hi - 1 && x >= t[s + 1]) ++s;
        return s;
    }
};

Knots unit_open_knots(int p, int n) {
    Knots k;
    k.p = p;
    for (int i = 0; i <= p; ++i) k.t.push_back(0.0L);
    for (int i = 1; i < n; ++i) k.t.push_back((real)i);
    for (int i = 0; i <= p; ++i) k.t.push_back((real)n);
    return k;
}

// ders[d][r] = d-th derivative of N_{s-p+r}(x), r = 0..p, d = 0..nd (nd <= 2)
void span_ders(const Knots& K, int s, real x, int nd, real ders[3][kMaxP + 1]) {
    const int p = K.p;
    const real* t = K.t.data();
    real ndu[kMaxP + 1][kMaxP + 1], left[kMaxP + 1], right[kMaxP + 1];
    ndu[0][0] = 1.0L;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - t[s + 1 - j];
        right[j] = t[s + j] - x;
        real saved = 0.0L;
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = right[r + 1] + left[j - r];
            real tmp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        ndu[j][j] = saved;
    }
    for (int r = 0; r <= p; ++r) ders[0][r] = ndu[r][p];
    for (int r = 0; r <= p; ++r) {
        real a[2][kMaxP + 1];
        int s1 = 0, s2 = 1;
        a[0][0] = 1.0L;
        for (int k = 1; k <= nd; ++k) {
            real d = 0.0L;
            int rk = r - k, pk = p - k;
            if (r >= k) {
                a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
                d = a[s2][0] * ndu[rk][pk];
            }
            int j1 = (rk >= -1) ? 1 : -rk;
            int j2 = (r - 1 <= pk) ? k - 1 : p - r;
            for (int j = j1; j <= j2; ++j) {
                a[s2][j] = (a[s1][j] - a[s1][j - 1]) / ndu[pk + 1][rk + j];
                d += a[s2][j] * ndu[rk + j][pk];
            }
            if (r <= pk) {
                a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
                d += a[s2][k] * ndu[r][pk];
            }
            ders[k][r] = d;
            std::swap(s1, s2);
        }
    }
    real f = p;
    for (int k = 1; k <= nd; ++k) {
        for (int r = 0; r <= p; ++r) ders[k][r] *= f;
        f *= (p - k);
    }
}

// value of the order-th derivative of B_i at x
real bval(const Knots& K, int i, real x, int order) {
    int s = K.span(x);
    if (i < s - K.p || i > s) return 0.0L;
    real ders[3][kMaxP + 1];
    span_ders(K, s, x, order, ders);
    return ders[order][i - (s - K.p)];
}

// ---------------------------------------------------------------------------------------
// Gauss-Legendre by Newton on the three-term recurrence.
// ---------------------------------------------------------------------------------------
void gauss_legendre(int m, std::vector<real>& x, std::vector<real>& w) {
    x.assign(m, 0.0L);
    w.assign(m, 0.0L);
    const real pi = 3.14159265358979323846264338327950288L;
    for (int i = 0; i < m; ++i) {
        real z = std::cos(pi * (i + 0.75L) / (m + 0.5L));
        real dp = 0.0L;
        for (int it = 0; it < 100; ++it) {
            real p0 = 1.0L, p1 = 0.0L;
            for (int k = 1; k <= m; ++k) {
                real p2 = p1;
                p1 = p0;
                p0 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p2) / k;
            }
            dp = m * (z * p0 - p1) / (z * z - 1.0L);
            real dz = p0 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-21L) break;
        }
        x[m - 1 - i] = z;                       // ascending
        w[m - 1 - i] = 2.0L / ((1.0L - z * z) * dp * dp);
    }
}

// int_{lo}^{hi} B_i^{(o)} B_j^{(o)} dx, exact by (p+2)-point GL on every knot span
real product_moment(const Knots& K, int i, int j, int order, real lo, real hi) {
    std::vector<real> gx, gw;
    gauss_legendre(K.p + 2, gx, gw);
    real sum = 0.0L;
    for (size_t s = 0; s + 1 < K.t.size(); ++s) {
        real a = K.t[s], b = K.t[s + 1];
        if (b <= a || a < lo || b > hi) continue;
        for (size_t q = 0; q < gx.size(); ++q) {
            real x = 0.5L * (a + b) + 0.5L * (b - a) * gx[q];
            sum += 0.5L * (b - a) * gw[q] * bval(K, i, x, order) * bval(K, j, x, order);
        }
    }
    return sum;
}

// exactness residual r_i = sum_k omega_k F_i(x_k) W(x_k) - mu_i
struct Exactness {
    Knots K;
    int j, order;
    real lo, hi;
    std::vector<int> rows;
    std::vector<real> mu;
    Exactness(int p, int j_, int order_, bool interior) : K(unit_open_knots(p, 4 * p + 2)), j(j_), order(order_) {
        lo = K.t[j];
        hi = K.t[j + p + 1];
        for (int i = j - p; i <= j + p; ++i)
            if (i >= 0 && i < K.nfun()) rows.push_back(i);
        (void)interior;
        for (int i : rows) mu.push_back(product_moment(K, i, j, order, lo, hi));
    }
    template <typename T>
    real residual(int row_index, int m, const T* tau, const T* om) const {
        real q = 0.0L;
        for (int k = 0; k < m; ++k) {
            real x = lo + (real)tau[k];
            q += (real)om[k] * bval(K, rows[row_index], x, order) * bval(K, j, x, order);
        }
        return q - mu[row_index];
    }
    double max_residual(int m, const double* tau, const double* om) const {
        real worst = 0.0L;
        for (size_t r = 0; r < rows.size(); ++r) worst = std::max(worst, std::fabs(residual((int)r, m, tau, om)));
        return (double)worst;
    }
};

// ---------------------------------------------------------------------------------------
// Damped Newton with finite-difference Jacobian, step halving and bracket projection.
// ---------------------------------------------------------------------------------------
using ResidualFn = std::function<void(const std::vector<real>& u, std::vector<real>& r)>;

bool solve_linear(std::vector<real> A, std::vector<real> b, int n, std::vector<real>& x) {
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
        if (std::fabs(A[piv * n + c]) < 1e-300L) return false;
        if (piv != c) {
            for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[piv * n + k]);
            std::swap(b[c], b[piv]);
        }
        for (int r = c + 1; r < n; ++r) {
            real f = A[r * n + c] / A[c * n + c];
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            b[r] -= f * b[c];
        }
    }
    x.assign(n, 0.0L);
    for (int r = n - 1; r >= 0; --r) {
        real s = b[r];
        for (int k = r + 1; k < n; ++k) s -= A[r * n + k] * x[k];
        x[r] = s / A[r * n + r];
    }
    return true;
}

real newton(const ResidualFn& F, std::vector<real>& u, const std::vector<std::pair<real, real>>& box) {
    const int n = (int)u.size();
    auto project = [&](std::vector<real>& v) {
        for (int i = 0; i < n; ++i) {
            real a = box[i].first, b = box[i].second;
            if (a < b) v[i] = std::min(std::max(v[i], a + 1e-12L * (b - a)), b - 1e-12L * (b - a));
        }
    };
    auto norm = [](const std::vector<real>& r) {
        real m = 0.0L;
        for (real v : r) m = std::max(m, std::fabs(v));
        return m;
    };
    project(u);
    std::vector<real> r(n), rp(n), rm(n), J(n * n), du, v;
    F(u, r);
    real nr = norm(r);
    for (int it = 0; it < 80 && nr > 1e-21L; ++it) {
        for (int c = 0; c < n; ++c) {
            real h = 1e-9L * std::max((real)1.0L, std::fabs(u[c]));
            std::vector<real> up = u, um = u;
            up[c] += h;
            um[c] -= h;
            F(up, rp);
            F(um, rm);
            for (int rr = 0; rr < n; ++rr) J[rr * n + c] = (rp[rr] - rm[rr]) / (2.0L * h);
        }
        if (!solve_linear(J, r, n, du)) break;
        real lam = 1.0L;
        bool ok = false;
        while (lam > 1e-6L) {
            v = u;
            for (int i = 0; i < n; ++i) v[i] -= lam * du[i];
            project(v);
            F(v, rp);
            real nv = norm(rp);
            if (std::isfinite((double)nv) && nv < nr) {
                u = v;
                r = rp;
                nr = nv;
                ok = true;
                break;
            }
            lam *= 0.5L;
        }
        if (!ok) break;
    }
    return nr;
}

// ---------------------------------------------------------------------------------------
// the rules
// ---------------------------------------------------------------------------------------
int finish(ClassRule& R, const Exactness& E) {
    R.residual = E.max_residual(R.m, R.tau, R.omega);
    return R.residual < 1e-13 ? WGQ_OK : WGQ_ENOCONV;
}

// round an extended-precision rule to the stored doubles
void store(ClassRule& R, int m, const real* tau, const real* om) {
    R.m = m;
    for (int k = 0; k < m; ++k) {
        R.tau[k] = (double)tau[k];
        R.omega[k] = (double)om[k];
    }
}

int interior_mass_p2(ClassRule& R) {
    Exactness E(2, 4, 0, true);
    const real t1 = (24.0L - std::sqrt(30.0L)) / 26.0L;   // root in (0,1) of 26t^2 - 48t + 21
    const real w1 = 1.0L / (30.0L * t1 * t1 * (1.0L - t1) * (1.0L - t1));
    const real w2 = (16.0L / 9.0L) * (11.0L / 20.0L - 0.5L * w1 * t1 * t1 * t1 * t1);
    const real tau[3] = {t1, 1.5L, 3.0L - t1}, om[3] = {w1, w2, w1};
    store(R, 3, tau, om);
    return finish(R, E);
}

int interior_mass_p3(ClassRule& R) {
    Exactness E(3, 6, 0, true);
    auto expand = [](const std::vector<real>& u, real* tau, real* om) {
        tau[0] = u[0]; tau[1] = u[1]; tau[2] = 4.0L - u[1]; tau[3] = 4.0L - u[0];
        om[0] = u[2]; om[1] = u[3]; om[2] = u[3]; om[3] = u[2];
    };
    ResidualFn F = [&](const std::vector<real>& u, std::vector<real>& r) {
        real tau[4], om[4];
        expand(u, tau, om);
        for (int k = 0; k < 4; ++k) r[k] = E.residual(k, 4, tau, om);   // offsets -3..0
    };
    const real s1[] = {0.5L, 0.3L, 0.7L, 0.15L, 0.85L}, s2[] = {1.5L, 1.3L, 1.7L, 1.15L, 1.85L};
    for (real a : s1)
        for (real b : s2) {
            std::vector<real> u = {a, b, 1.0L, 1.0L};
            real nr = newton(F, u, {{0.0L, 1.0L}, {1.0L, 2.0L}, {0.0L, 0.0L}, {0.0L, 0.0L}});
            if (nr < 1e-17L && u[0] > 0 && u[0] < 1 && u[1] > 1 && u[1] < 2 && u[2] > 0 && u[3] > 0) {
                real tau[4], om[4];
                expand(u, tau, om);
                store(R, 4, tau, om);
                return finish(R, E);
            }
        }
    return WGQ_ENOCONV;
}

int interior_stiff_p2(ClassRule& R) {
    Exactness E(2, 4, 1, true);
    // the middle node tau = 3/2 has B'_j = 0 (R2): dropped
    const real tau[2] = {0.75L, 2.25L}, om[2] = {8.0L / 9.0L, 8.0L / 9.0L};
    store(R, 2, tau, om);
    return finish(R, E);
}

int interior_stiff_p3(ClassRule& R) {
    Exactness E(3, 6, 1, true);
    const real w1 = 1.0L;
    const real t1 = 0.5L - std::sqrt(225.0L - 30.0L * std::sqrt(30.0L)) / 30.0L;
    auto expand = [&](const std::vector<real>& u, real* tau, real* om) {
        tau[0] = t1; tau[1] = u[0]; tau[2] = 4.0L - u[0]; tau[3] = 4.0L - t1;
        om[0] = w1; om[1] = u[1]; om[2] = u[1]; om[3] = w1;
    };
    ResidualFn F = [&](const std::vector<real>& u, std::vector<real>& r) {
        real tau[4], om[4];
        expand(u, tau, om);
        r[0] = E.residual(1, 4, tau, om);       // offset -2 (line 2)
        r[1] = E.residual(3, 4, tau, om);       // offset  0 (line 4)
    };
    for (real a : {1.5L, 1.3L, 1.7L, 1.15L, 1.85L}) {
        std::vector<real> u = {a, 1.0L};
        real nr = newton(F, u, {{1.0L, 2.0L}, {0.0L, 0.0L}});
        if (nr < 1e-17L && u[0] > 1 && u[0] < 2 && u[1] > 0) {
            real tau[4], om[4];
            expand(u, tau, om);
            store(R, 4, tau, om);
            return finish(R, E);
        }
    }
    return WGQ_ENOCONV;
}

void gl_per_element(int p, int j, ClassRule& R) {
    std::vector<real> gx, gw;
    gauss_legendre(p + 1, gx, gw);
    real tau[kMaxNodes], om[kMaxNodes];
    int m = 0;
    for (int e = 0; e <= j; ++e)
        for (int q = 0; q <= p; ++q) {
            tau[m] = e + 0.5L + 0.5L * gx[q];
            om[m] = 0.5L * gw[q];
            ++m;
        }
    store(R, m, tau, om);
}

// Reading R1: m = ceil(D/2) nodes; the last node is fixed at j + 1/2 when D is odd.
int boundary_rule(int p, int j, int kind, int bnd, ClassRule& R) {
    const int order = kind == WGQ_MASS ? 0 : 1;
    Exactness E(p, j, order, false);
    if (bnd == WGQ_BND_GL) {
        gl_per_element(p, j, R);
        return finish(R, E);
    }
    const int D = order == 0 ? p + j + 1 : p + j;
    const int m = (D + 1) / 2;
    const bool fixed = (D % 2) == 1;
    const int nfree = fixed ? m - 1 : m;
    const real L = j + 1.0L;
    const int neq = D;                         // stiffness: last constraint implied (sum B'_i = 0)
    auto expand = [&](const std::vector<real>& u, real* tau, real* om) {
        for (int k = 0; k < nfree; ++k) tau[k] = u[k];
        if (fixed) tau[m - 1] = j + 0.5L;
        for (int k = 0; k < m; ++k) om[k] = u[nfree + k];
    };
    ResidualFn F = [&](const std::vector<real>& u, std::vector<real>& r) {
        real tau[kMaxNodes], om[kMaxNodes];
        expand(u, tau, om);
        for (int e = 0; e < neq; ++e) r[e] = E.residual(e, m, tau, om);
    };
    std::vector<std::pair<real, real>> box;
    for (int k = 0; k < nfree; ++k) box.push_back({0.0L, L});
    for (int k = 0; k < m; ++k) box.push_back({0.0L, 0.0L});
    // deterministic multi-start: increasing tuples of a 9-point grid
    const int G = 9;
    std::vector<real> grid;
    for (int g = 0; g < G; ++g) grid.push_back(L * (0.05L + 0.9L * g / (G - 1)));
    std::vector<int> idx(nfree);
    std::function<bool(int, int)> rec = [&](int pos, int start) -> bool {
        if (pos == nfree) {
            std::vector<real> u;
            for (int k = 0; k < nfree; ++k) u.push_back(grid[idx[k]]);
            if (fixed && nfree > 0 && u.back() >= j + 0.5L) return false;
            for (int k = 0; k < m; ++k) u.push_back(1.0L / m);
            real nr = newton(F, u, box);
            if (nr > 1e-17L) return false;
            real tau[kMaxNodes], om[kMaxNodes];
            expand(u, tau, om);
            for (int k = 0; k < m; ++k) {
                if (!(tau[k] > 1e-9L && tau[k] < L - 1e-9L && om[k] > 0)) return false;
                if (k > 0 && !(tau[k] > tau[k - 1] + 1e-9L)) return false;
            }
            store(R, m, tau, om);
            return true;
        }
        for (int g = start; g < G; ++g) {
            idx[pos] = g;
            if (rec(pos + 1, g + 1)) return true;
        }
        return false;
    };
    if (!rec(0, 0)) gl_per_element(p, j, R);    // no admissible minimal rule -> GL (R1)
    return finish(R, E);
}

}  // namespace

void interior_vertex_tables(int p, const ClassRule& mass, const ClassRule& stiff, double PM[kMaxV][kMaxS],
                            double PK[kMaxV][kMaxS]) {
    // reference knots, cardinal weight j = 2p with support [p, 2p+1]; neighbours j+o
    Knots K = unit_open_knots(p, 4 * p + 2);
    const int j = 2 * p;
    real acc[2][kMaxV][kMaxS] = {};
    for (int kind = 0; kind < 2; ++kind) {
        const ClassRule& R = kind == 0 ? mass : stiff;
        for (int k = 0; k < R.m; ++k) {
            const real t = R.tau[k];
            const int e = (int)std::floor(t);                 // element of the node (inside it)
            const real f = t - e;
            const real x = p + t;
            const real w = (real)R.omega[k] * bval(K, j, x, kind);
            for (int o = -p; o <= p; ++o) {
                const real a = w * bval(K, j + o, x, kind);
                acc[kind][e][o + p] += (1.0L - f) * a;
                acc[kind][e + 1][o + p] += f * a;
            }
        }
    }
    for (int v = 0; v < kMaxV; ++v)
        for (int o = 0; o < kMaxS; ++o) {
            PM[v][o] = (double)acc[0][v][o];
            PK[v][o] = (double)acc[1][v][o];
        }
}

int build_class_rules(int p, int bnd, ClassRule out[2][kMaxP + 1]) {
    int rc;
    if (p == 2) {
        if ((rc = interior_mass_p2(out[WGQ_MASS][p])) != WGQ_OK) return rc;
        if ((rc = interior_stiff_p2(out[WGQ_STIFFNESS][p])) != WGQ_OK) return rc;
    } else if (p == 3) {
        if ((rc = interior_mass_p3(out[WGQ_MASS][p])) != WGQ_OK) return rc;
        if ((rc = interior_stiff_p3(out[WGQ_STIFFNESS][p])) != WGQ_OK) return rc;
    } else {
        return WGQ_EUNSUPPORTED;
    }
    for (int kind = 0; kind < 2; ++kind)
        for (int j = 0; j < p; ++j)
            if ((rc = boundary_rule(p, j, kind, bnd, out[kind][j])) != WGQ_OK) return rc;
    return WGQ_OK;
}

// Basis-evaluation counts (experiment E3): per 1D row, the number
// of the 2p+1 interacting functions (mass: B, stiffness: B') that are nonzero at each point of
// the row's rule where the weight B_r (B'_r) is nonzero — for the weighted Gaussian rules built
// here and for the weighted Newton-Cotes point set of Calabro et al. (the knots and element
// midpoints of supp B_r).  A tensor row costs the product over directions, so
// the n^d mesh costs (sum_r count(r))^d.
namespace {
void eval_counts_1d(const wgq_rules_s* R, int kind, int64_t n, int64_t* g_out, int64_t* nc_out) {
    const int p = R->p;
    const int64_t N = n + p;
    const int order = kind == WGQ_MASS ? 0 : 1;
    Knots K = unit_open_knots(p, (int)n);
    auto nonzero_at = [&](int64_t r, real x) {
        int c = 0;
        for (int o = -p; o <= p; ++o) {
            const int64_t j = r + o;
            if (j >= 0 && j < N && fabsl(bval(K, (int)j, x, order)) > 1e-12L) ++c;
        }
        return c;
    };
    int64_t g = 0, nc = 0;
    for (int64_t r = 0; r < N; ++r) {
        const int cls = r < p ? (int)r : (r >= n ? (int)(n + p - 1 - r) : p);
        const ClassRule& rule = R->rules[kind][cls];
        for (int k = 0; k < rule.m; ++k) {
            const real tau = (real)rule.tau[k];
            const real x = r < p ? tau : (r >= n ? (real)n - tau : (real)(r - p) + tau);
            if (fabsl(bval(K, (int)r, x, order)) > 1e-12L) g += nonzero_at(r, x);
        }
        const int64_t a = std::max<int64_t>(0, r - p), b = std::min<int64_t>(n, r + 1);   // supp B_r = [a, b]
        for (int64_t q = 2 * a; q <= 2 * b; ++q) {                  // knots (q even) and midpoints (q odd)
            const real x = (real)q / 2.0L;
            if (fabsl(bval(K, (int)r, x, order)) > 1e-12L) nc += nonzero_at(r, x);
        }
    }
    *g_out = g;
    *nc_out = nc;
}
}  // namespace

// A tensor row costs the product of its directions' counts: the mesh costs the product over
// directions of the per-direction sums (each direction with its own element count).
void eval_counts(const wgq_rules_s* R, int kind, int64_t* gaussian, int64_t* newton_cotes) {
    int64_t G = 1, C = 1;
    for (int a = 0; a < R->dim; ++a) {
        int64_t g = 0, nc = 0;
        eval_counts_1d(R, kind, R->dims.n[a], &g, &nc);
        G *= g;
        C *= nc;
    }
    *gaussian = G;
    *newton_cotes = C;
}

}  // namespace wgq
