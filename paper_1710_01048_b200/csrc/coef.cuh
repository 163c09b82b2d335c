// Coefficient fields c(x) evaluated on the device (readings R4, R6,
// R13).  The descriptor is copied by value into every launch.
#pragma once

#include <cuda_runtime.h>

#include "internal.h"

namespace wgq {

struct CoefDev {
    int kind;
    int n_modes;
    double c0, amp;
    int trig[3];
    int wavenum[3];
    double modes[WGQ_MAX_MODES][5];
    const double* grid;
    int64_t plane0, planes;
};

// Multilinear interpolation of the vertex field (R6).  The cell is the element that
// contains the point; the slowest axis is slab-local (plane0).
// n: elements per direction (vertex j of direction a at j / n[a]; planes of (n[1]+1) x (n[0]+1))
template <int D>
__device__ __forceinline__ double grid_eval(const CoefDev& c, const int64_t* n, const double* x) {
    int64_t e[3];
    double f[3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double s = __dmul_rn(x[a], (double)n[a]);
        int64_t k = (int64_t)floor(s);
        k = k < 0 ? 0 : (k > n[a] - 1 ? n[a] - 1 : k);
        e[a] = k;
        f[a] = s - (double)k;
    }
    const int64_t nvx = n[0] + 1, nvy = D >= 2 ? n[1] + 1 : 1;
    double out = 0.0;
    if (D == 1) {
        const double* g = c.grid + (e[0] - c.plane0);
        out = (1.0 - f[0]) * g[0] + f[0] * g[1];
    } else if (D == 2) {
        const double* g = c.grid + (e[1] - c.plane0) * nvx + e[0];
        out = (1.0 - f[1]) * ((1.0 - f[0]) * g[0] + f[0] * g[1]) + f[1] * ((1.0 - f[0]) * g[nvx] + f[0] * g[nvx + 1]);
    } else {
        const double* g = c.grid + ((e[2] - c.plane0) * nvy + e[1]) * nvx + e[0];
        const int64_t sy = nvx, sz = nvx * nvy;
        double c00 = (1.0 - f[0]) * g[0] + f[0] * g[1];
        double c10 = (1.0 - f[0]) * g[sy] + f[0] * g[sy + 1];
        double c01 = (1.0 - f[0]) * g[sz] + f[0] * g[sz + 1];
        double c11 = (1.0 - f[0]) * g[sz + sy] + f[0] * g[sz + sy + 1];
        out = (1.0 - f[2]) * ((1.0 - f[1]) * c00 + f[1] * c10) + f[2] * ((1.0 - f[1]) * c01 + f[1] * c11);
    }
    return out;
}

template <int D>
__device__ __forceinline__ double coef_eval(const CoefDev& c, const int64_t* n, const double* x) {
    switch (c.kind) {
        case WGQ_COEF_CONST:
            return c.c0;
        case WGQ_COEF_TRIG_SEP: {
            double prod = 1.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                double arg = 2.0 * (double)c.wavenum[a] * x[a];   // trig(pi * arg)
                prod *= c.trig[a] == WGQ_TRIG_SIN ? sinpi(arg) : cospi(arg);
            }
            return c.c0 + c.amp * prod;
        }
        case WGQ_COEF_FOURIER_LOGN: {
            double s = 0.0;
            for (int m = 0; m < c.n_modes; ++m) {
                double arg = c.modes[m][1] * x[0];
                if (D > 1) arg += c.modes[m][2] * x[1];
                if (D > 2) arg += c.modes[m][3] * x[2];
                // cos(2 pi arg + theta): reduce 2*arg exactly with cospi/sinpi
                double cp = cospi(2.0 * arg), sp = sinpi(2.0 * arg);
                double ct, st;
                sincos(c.modes[m][4], &st, &ct);
                s += c.modes[m][0] * (cp * ct - sp * st);
            }
            return exp(s);
        }
        default:
            return grid_eval<D>(c, n, x);
    }
}

}  // namespace wgq
