"""CPU tests of the C-ABI library's host side (no GPU, no compute kernels).

The library loads, exports every symbol include/wgq.h declares, validates arguments,
and its independently implemented host rule builder reproduces the paper's constants and
agrees with the oracle's rules (reading R1 for the boundary classes).
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1710_01048_b200 import build, wgq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return wgq.lib()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "wgq.h")).read()
    return sorted(set(re.findall(r"\b(wgq_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(L):
    decl = declared_symbols()
    assert len(decl) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", wgq.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (wgq_\w+)", out))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    assert sorted(wgq.exported_symbols()) == decl
    for s in decl:
        getattr(L, s)


def test_sm100a_code_present(L):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", wgq.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_strerror_and_errors(L):
    assert L.wgq_strerror(0) == b"ok"
    h = ctypes.c_void_p()
    assert L.wgq_build_rules(4, 10, 2, ctypes.byref(h)) == wgq.WGQ_EUNSUPPORTED
    assert L.wgq_build_rules(3, 2, 2, ctypes.byref(h)) == wgq.WGQ_EUNSUPPORTED   # n < p
    assert L.wgq_build_rules(2, 10, 4, ctypes.byref(h)) == wgq.WGQ_EUNSUPPORTED
    assert L.wgq_build_rules(2, 10, 2, None) == wgq.WGQ_EINVAL
    assert L.wgq_build_rules_ex(2, 10, 2, 7, ctypes.byref(h)) == wgq.WGQ_EINVAL
    assert L.wgq_build_rules(3, 2000, 3, ctypes.byref(h)) == wgq.WGQ_ERANGE      # > 2^31 rows
    r = wgq.Rules(3, 8, 3)
    # descriptor validation happens before any device work
    c = wgq.make_coeff({"kind": "const", "c0": 1.0})
    o = wgq.wgq_out_t()
    o.layout, o.row_begin, o.row_end, o.values, o.ld = wgq.WGQ_ELL, 0, r.n_rows + 1, 8, 343
    assert L.wgq_assemble_mass(r.handle, ctypes.byref(c), ctypes.byref(o), None) == wgq.WGQ_EINVAL
    o.row_end, o.ld = 10, 300
    assert L.wgq_assemble_mass(r.handle, ctypes.byref(c), ctypes.byref(o), None) == wgq.WGQ_ERANGE
    o.ld = 343
    c.kind = 9
    assert L.wgq_assemble_mass(r.handle, ctypes.byref(c), ctypes.byref(o), None) == wgq.WGQ_EINVAL
    g = wgq.make_coeff({"kind": "const", "c0": 1.0})
    g.kind, g.grid, g.grid_plane0, g.grid_planes = wgq.WGQ_COEF_GRID, 8, 3, 2   # planes do not cover rows
    assert L.wgq_assemble_mass(r.handle, ctypes.byref(g), ctypes.byref(o), None) == wgq.WGQ_EINVAL


def test_rules_info_and_nnz(L):
    r = wgq.Rules(3, 256, 3)
    assert (r.N, r.n_rows, r.stencil) == (259, 17373979, 343)
    # C5 has 5,841,725,401 structural nonzeros per matrix
    assert wgq.wgq_nnz(r, 0, r.n_rows) == 5841725401
    r2 = wgq.Rules(2, 512, 2)
    assert wgq.wgq_nnz(r2, 0, r2.n_rows) == 6574096
    # additivity over slabs, brute force on a small mesh
    r3 = wgq.Rules(2, 3, 3)
    N = r3.N
    brute = 0
    for row in range(r3.n_rows):
        i = [(row // N ** a) % N for a in range(3)]
        w = 1
        for a in range(3):
            w *= min(i[a] + 2, N - 1) - max(i[a] - 2, 0) + 1
        brute += w
        if row % 17 == 0:
            assert wgq.wgq_nnz(r3, 0, row + 1) == brute
    assert wgq.wgq_nnz(r3, 0, r3.n_rows) == brute


def test_library_rules_match_paper_and_oracle(L):
    from oracle import rules as orules
    paper = {("mass", 2): ([0.71241440095955149482, 1.5], [0.79410713110801847176, 0.79595121334251753503]),
             ("mass", 3): ([0.72289886179270511319, 1.58789880583487289415], [0.88863704203309628490, 0.83494225417405959060]),
             ("stiffness", 3): ([0.24033518882038592858, 1.16015740029939774803], [1.0, 0.86030876544418464920])}
    for p in (2, 3):
        for mode in (wgq.WGQ_BND_GAUSS, wgq.WGQ_BND_GL):
            r = wgq.Rules(p, 12, 2, mode)
            ocr = orules.class_rules(p, "gauss" if mode == wgq.WGQ_BND_GAUSS else "gl")
            for kind, kc in (("mass", wgq.WGQ_MASS), ("stiffness", wgq.WGQ_STIFFNESS)):
                for cls in range(p + 1):
                    tau, om, res = wgq.wgq_rules_query(r, cls, kc)
                    assert res < 1e-13
                    o = ocr[kind]["interior" if cls == p else cls]
                    ot, oo = o.tau, o.omega
                    if kind == "stiffness" and p == 2 and cls == p:   # R2: zero-weight middle node dropped
                        ot, oo = ot[[0, 2]], oo[[0, 2]]
                    # both sides are correctly rounded (R14): at most 1 ulp apart
                    assert np.all(np.abs(tau - ot) <= np.spacing(ot)), (p, kind, cls, tau, ot)
                    assert np.all(np.abs(om - oo) <= np.spacing(oo)), (p, kind, cls, om, oo)
                    if cls == p and (kind, p) in paper:
                        pt, po = paper[(kind, p)]
                        assert np.allclose(tau[:len(pt)], pt, atol=1e-14) and np.allclose(om[:len(po)], po, atol=1e-14)


def test_operator_argument_errors(L):
    """wgq_assemble_load / wgq_apply validate before any device work (no GPU needed)."""
    r = wgq.Rules(3, 6, 3)
    c = wgq.make_coeff({"kind": "const", "c0": 1.0})
    assert L.wgq_assemble_load(r.handle, ctypes.byref(c), 0, 10, None, None) == wgq.WGQ_EINVAL
    assert L.wgq_assemble_load(r.handle, ctypes.byref(c), 5, 4, 8, None) == wgq.WGQ_EINVAL
    assert L.wgq_assemble_load(r.handle, ctypes.byref(c), 0, r.n_rows + 1, 8, None) == wgq.WGQ_EINVAL
    assert L.wgq_assemble_load(r.handle, ctypes.byref(c), 3, 3, None, None) == wgq.WGQ_OK      # empty range
    N = r.N
    z0, z1 = 4, 6                                              # rows of planes 4, 5: need u planes 1..8
    rb, re_ = z0 * N * N, z1 * N * N
    # no outputs / no u
    assert L.wgq_apply(r.handle, ctypes.byref(c), 8, 0, r.n_rows, rb, re_, None, None, None) == wgq.WGQ_EINVAL
    assert L.wgq_apply(r.handle, ctypes.byref(c), None, 0, r.n_rows, rb, re_, 8, None, None) == wgq.WGQ_EINVAL
    # u must cover planes z0-p .. z1+p-1 (clipped): one plane short on either side is an error
    lo, hi = (z0 - 3) * N * N, min(N, z1 + 3) * N * N
    assert L.wgq_apply(r.handle, ctypes.byref(c), 8, lo + N * N, hi - lo - N * N, rb, re_, 8, None, None) == wgq.WGQ_ERANGE
    assert L.wgq_apply(r.handle, ctypes.byref(c), 8, lo, hi - lo - N * N, rb, re_, 8, None, None) == wgq.WGQ_ERANGE
    assert L.wgq_apply(r.handle, ctypes.byref(c), 8, lo, hi - lo, 7, 7, 8, None, None) == wgq.WGQ_OK   # empty range


def test_rules_json_export(L):
    """rule tables exportable as JSON {kind, degree, nodes[], weights[], residual_max}."""
    import json

    from paper_1710_01048_b200 import api
    for p in (2, 3):
        r = wgq.Rules(p, 10, 1)
        doc = json.loads(api.rules_json(r))
        assert len(doc) == 2 * (p + 1)
        for entry in doc:
            assert set(entry) == {"kind", "degree", "class", "nodes", "weights", "residual_max"}
            assert entry["degree"] == p and entry["residual_max"] < 1e-13
            kc = wgq.WGQ_MASS if entry["kind"] == "mass" else wgq.WGQ_STIFFNESS
            cls = p if entry["class"] == "interior" else entry["class"]
            tau, om, _ = wgq.wgq_rules_query(r, cls, kc)
            assert entry["nodes"] == list(tau) and entry["weights"] == list(om)   # 17 digits round-trip exactly
