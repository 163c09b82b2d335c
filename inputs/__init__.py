"""Seeded synthetic inputs shared by the tests, the bench and the oracle.

This module holds NONE of the method's arithmetic (no B-splines, no quadrature
rules, no assembly).  It only synthesises the coefficient fields and row samples
the paper-shaped workloads need:

* ``splitmix64`` / ``u53``      -- the counter-based generator of c.4.
* ``fourier_modes``             -- FOURIER_LOGN parameters (C3), c.4.
* ``lognormal_grid``            -- the smoothed lognormal vertex grid (C5), c.4.
* ``configs``                   -- the five BASELINE.json workloads.

The CUDA library implements the same GRID generator independently on the device
(``wgq_generate_grid``); tests compare the two.
"""
from .gen import splitmix64, u53, fourier_modes, lognormal_grid, GRID_NORM, SEED  # noqa: F401
from .configs import CONFIGS, config, coefficient  # noqa: F401
