"""Seeded input generators (inputs/) -- shared by oracle and CUDA tests (no GPU)."""
import math

import numpy as np

import inputs


def test_splitmix64_known_values():
    # splitmix64 finaliser of 0 is 0; of 1 the standard mix constant chain
    assert int(inputs.splitmix64(0)) == 0
    z = 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
    z ^= z >> 31
    assert int(inputs.splitmix64(1)) == z
    assert 0.0 <= float(inputs.u53(inputs.splitmix64(12345))) < 1.0


def test_fourier_modes_spec():
    m = inputs.fourier_modes(inputs.SEED, 8, 0.3, 2)
    assert m.shape == (8, 5)
    assert list(m[:, 1]) == list(range(1, 9))
    assert sorted(m[:, 2]) == list(range(1, 9))
    assert abs(np.linalg.norm(m[:, 0]) - 0.3 * math.sqrt(8)) < 1e-14
    assert np.all((m[:, 4] >= 0) & (m[:, 4] < 2 * math.pi))
    assert np.array_equal(m, inputs.fourier_modes(inputs.SEED, 8, 0.3, 2))


def test_grid_slab_equals_global():
    n = 12
    g = inputs.lognormal_grid(n, seed=5)
    s = inputs.lognormal_grid(n, seed=5, plane0=4, planes=3)
    assert g.shape == (n + 1, n + 1, n + 1)
    assert np.array_equal(g[4:7], s)
    g2 = inputs.lognormal_grid(n, seed=5, dim=2)
    assert g2.shape == (n + 1, n + 1)


def test_grid_statistics():
    g = inputs.lognormal_grid(48, seed=inputs.SEED)
    lg = np.log(g) / 0.5
    assert abs(lg.std() - 1.0) < 0.1
    assert np.all(g > 0)
