"""The five BASELINE.json workloads (SURVEY.md §8(d) "Synthetic inputs").

A coefficient descriptor is a plain dict:
  {"kind": "const", "c0": c}
  {"kind": "trig_sep", "c0": c0, "amp": A, "trig": ("sin"|"cos", ...), "wavenum": (k1, ...)}
      c = c0 + A * prod_a trig_a(2 pi k_a x_a)
  {"kind": "fourier_logn", "modes": [M, 5] array of (a, kx, ky, kz, theta)}
      c = exp(sum_m a_m cos(2 pi (kx x + ky y + kz z) + theta_m))
  {"kind": "grid", "seed": s, "sigma": sig}   (vertex field, see gen.lognormal_grid)
"""
from .gen import SEED, fourier_modes

CONFIGS = {
    "C1": dict(name="1d_p2_n64_mass_const", p=2, n=64, dim=1, kinds=("mass",),
               coeff={"kind": "const", "c0": 1.0}),
    "C2": dict(name="2d_p2_n512_mk_trig", p=2, n=512, dim=2, kinds=("mass", "stiffness"),
               coeff={"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos"), "wavenum": (1, 1)}),
    "C3": dict(name="2d_p3_n2048_mk_fourier", p=3, n=2048, dim=2, kinds=("mass", "stiffness"),
               coeff={"kind": "fourier_logn", "seed": SEED, "n_modes": 8, "amp": 0.3}),
    "C4": dict(name="3d_p2_n128_mass_trig", p=2, n=128, dim=3, kinds=("mass",),
               coeff={"kind": "trig_sep", "c0": 1.0, "amp": 0.3, "trig": ("sin", "sin", "sin"), "wavenum": (1, 1, 1)}),
    "C5": dict(name="3d_p3_n256_mk_grid", p=3, n=256, dim=3, kinds=("mass", "stiffness"),
               coeff={"kind": "grid", "seed": SEED, "sigma": 0.5}),
}


def config(name, n=None):
    """A copy of config ``name`` (optionally with a different element count n)."""
    c = dict(CONFIGS[name])
    c["coeff"] = dict(c["coeff"])
    if n is not None:
        c["n"] = n
    return c


def coefficient(desc, dim):
    """Materialise the seeded parameters of a descriptor (FOURIER modes)."""
    d = dict(desc)
    if d["kind"] == "fourier_logn" and "modes" not in d:
        d["modes"] = fourier_modes(d.get("seed", SEED), d.get("n_modes", 8), d.get("amp", 0.3), dim)
    return d
