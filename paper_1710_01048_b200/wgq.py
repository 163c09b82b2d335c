"""Thin ctypes binding of libwgq (include/wgq.h): argument marshalling only.

Every function has the name of the C entry point it calls.  Tensors are passed by
``data_ptr()``; streams by ``torch.cuda.Stream.cuda_stream``.  Nothing here computes any
part of the method: the product path is the CUDA library, and it fails loudly (ImportError
/ WgqError) when the library is missing or a call fails -- there is no CPU fallback.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WGQ_LIB") or os.path.join(_HERE, "libwgq.so")   # WGQ_LIB: kernel experiments

WGQ_OK, WGQ_EINVAL, WGQ_EUNSUPPORTED, WGQ_ENOCONV, WGQ_ECUDA, WGQ_ERANGE, WGQ_ENOMEM = 0, -1, -2, -3, -4, -5, -6
WGQ_BND_GAUSS, WGQ_BND_GL = 0, 1
WGQ_MASS, WGQ_STIFFNESS = 0, 1
WGQ_COEF_CONST, WGQ_COEF_TRIG_SEP, WGQ_COEF_FOURIER_LOGN, WGQ_COEF_GRID = 0, 1, 2, 3
WGQ_TRIG_SIN, WGQ_TRIG_COS = 0, 1
WGQ_MAX_MODES = 16
WGQ_ELL, WGQ_CSR = 0, 1


class WgqError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {code} ({_lib.wgq_strerror(code).decode()})")
        self.code = code


class wgq_coeff_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("c0", ctypes.c_double), ("amp", ctypes.c_double),
                ("trig", ctypes.c_int * 3), ("wavenum", ctypes.c_int * 3), ("n_modes", ctypes.c_int),
                ("modes", ctypes.POINTER(ctypes.c_double)), ("grid", ctypes.c_void_p),
                ("grid_plane0", ctypes.c_int64), ("grid_planes", ctypes.c_int64)]


class wgq_out_t(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("values", ctypes.c_void_p), ("ld", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libwgq.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1710_01048_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c_int, c_i64, vp, dp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
    sig = {
        "wgq_strerror": (ctypes.c_char_p, [c_int]),
        "wgq_version": (ctypes.c_char_p, []),
        "wgq_build_rules": (c_int, [c_int, c_i64, c_int, ctypes.POINTER(vp)]),
        "wgq_build_rules_ex": (c_int, [c_int, c_i64, c_int, c_int, ctypes.POINTER(vp)]),
        "wgq_build_rules_ex2": (c_int, [c_int, ctypes.POINTER(c_i64), c_int, c_int, ctypes.POINTER(vp)]),
        "wgq_rules_dims": (c_int, [vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
        "wgq_free_rules": (None, [vp]),
        "wgq_rules_info": (c_int, [vp, ctypes.POINTER(c_int), ctypes.POINTER(c_i64), ctypes.POINTER(c_int),
                                   ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), ctypes.POINTER(c_int)]),
        "wgq_rules_query": (c_int, [vp, c_int, c_int, ctypes.POINTER(c_int), dp, dp, dp]),
        "wgq_nnz": (c_int, [vp, c_i64, c_i64, ctypes.POINTER(c_i64)]),
        "wgq_eval_counts": (c_int, [vp, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
        "wgq_assemble_mass": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), ctypes.POINTER(wgq_out_t), vp]),
        "wgq_assemble_stiffness": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), ctypes.POINTER(wgq_out_t), vp]),
        "wgq_assemble_mass_stiffness": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), ctypes.POINTER(wgq_out_t),
                                                ctypes.POINTER(wgq_out_t), vp]),
        "wgq_csr_structure": (c_int, [vp, c_i64, c_i64, vp, vp, vp]),
        "wgq_assemble_load": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), c_i64, c_i64, vp, vp]),
        "wgq_apply": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), vp, c_i64, c_i64, c_i64, c_i64, vp, vp, vp]),
        "wgq_generate_grid": (c_int, [c_i64, c_int, ctypes.c_uint64, ctypes.c_double, c_i64, c_i64, vp, vp]),
        "wgq_generate_grid_ex": (c_int, [ctypes.POINTER(c_i64), c_int, ctypes.c_uint64, ctypes.c_double, c_i64, c_i64,
                                         vp, vp]),
        "wgq_row_moments": (c_int, [vp, ctypes.POINTER(wgq_out_t), vp, vp]),
        "wgq_checksum": (c_int, [vp, ctypes.POINTER(wgq_out_t), vp, vp]),
        "wgq_assemble_host": (c_int, [vp, ctypes.POINTER(wgq_coeff_t), c_i64, c_i64, vp, vp, c_i64, c_i64]),
        "wgq_host_alloc": (c_int, [ctypes.c_uint64, ctypes.POINTER(vp)]),
        "wgq_host_free": (c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols():
    return ["wgq_strerror", "wgq_version", "wgq_build_rules", "wgq_build_rules_ex", "wgq_build_rules_ex2",
            "wgq_rules_dims", "wgq_generate_grid_ex", "wgq_free_rules",
            "wgq_rules_info", "wgq_rules_query", "wgq_nnz", "wgq_eval_counts", "wgq_assemble_mass", "wgq_assemble_stiffness",
            "wgq_assemble_mass_stiffness", "wgq_csr_structure", "wgq_assemble_load", "wgq_apply",
            "wgq_generate_grid", "wgq_row_moments",
            "wgq_checksum", "wgq_assemble_host", "wgq_host_alloc", "wgq_host_free"]


def _check(fn, rc):
    if rc != WGQ_OK:
        raise WgqError(fn, rc)


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


# ---------------------------------------------------------------------------------------
# rules
# ---------------------------------------------------------------------------------------
class Rules:
    """Owns a wgq_rules_t handle (wgq_build_rules_ex2 / wgq_free_rules).

    n_elems: elements per direction, an int (every direction) or one count per direction
    (eq:Gmap3 P:113-120).  Attributes: ns / Ns (per-direction elements / rows), n / N (those of
    direction 0, the value of every direction on an isotropic mesh), n_rows, stencil."""

    def __init__(self, p, n_elems, dim, boundary_mode=WGQ_BND_GAUSS):
        ns = [int(n_elems)] * dim if np.ndim(n_elems) == 0 else [int(v) for v in n_elems]
        if len(ns) != dim:
            raise ValueError(f"n_elems: expected {dim} counts, got {len(ns)}")
        h = ctypes.c_void_p()
        arr = (ctypes.c_int64 * 3)(*(ns + [1] * (3 - dim)))
        _check("wgq_build_rules_ex2", lib().wgq_build_rules_ex2(p, arr, dim, boundary_mode, ctypes.byref(h)))
        self.handle = h
        self.p, self.dim = p, dim
        self.ns = tuple(ns)
        self.Ns = tuple(v + p for v in ns)
        self.iso = all(v == ns[0] for v in ns)
        self.n = ns[0]
        info = wgq_rules_info(self)
        self.N, self.n_rows, self.stencil = info["n_rows_1d"], info["n_rows"], info["stencil"]

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.wgq_free_rules(self.handle)
            self.handle = None


def wgq_build_rules(p, n_elems, dim, boundary_mode=WGQ_BND_GAUSS):
    return Rules(p, n_elems, dim, boundary_mode)


def wgq_rules_info(rules):
    p, d, st = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    n, N, nr = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check("wgq_rules_info", lib().wgq_rules_info(rules.handle, ctypes.byref(p), ctypes.byref(n), ctypes.byref(d),
                                                  ctypes.byref(N), ctypes.byref(nr), ctypes.byref(st)))
    return {"p": p.value, "n_elems": n.value, "dim": d.value, "n_rows_1d": N.value, "n_rows": nr.value,
            "stencil": st.value}


def wgq_rules_query(rules, cls, kind):
    m = ctypes.c_int()
    tau = (ctypes.c_double * 12)()
    om = (ctypes.c_double * 12)()
    res = ctypes.c_double()
    _check("wgq_rules_query", lib().wgq_rules_query(rules.handle, cls, kind, ctypes.byref(m), tau, om, ctypes.byref(res)))
    return np.array(tau[:m.value]), np.array(om[:m.value]), res.value


def wgq_eval_counts(rules, kind):
    """(Gaussian, Newton-Cotes) basis-evaluation counts of the handle's mesh (E3)."""
    g, c = ctypes.c_int64(), ctypes.c_int64()
    _check("wgq_eval_counts", lib().wgq_eval_counts(rules.handle, kind, ctypes.byref(g), ctypes.byref(c)))
    return g.value, c.value


def wgq_nnz(rules, row_begin, row_end):
    out = ctypes.c_int64()
    _check("wgq_nnz", lib().wgq_nnz(rules.handle, row_begin, row_end, ctypes.byref(out)))
    return out.value


# ---------------------------------------------------------------------------------------
# argument checks (the C-ABI takes raw pointers: a wrong dtype, a host tensor or a
# non-contiguous view would be read or written out of bounds, so refuse them here)
# ---------------------------------------------------------------------------------------
def _need(t, name, dtype="float64", numel=None, device=True):
    import torch
    want = {"float64": torch.float64, "int64": torch.int64, "int32": torch.int32}[dtype]
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if t.dtype != want:
        raise TypeError(f"{name}: expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    if device and not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name}: needs at least {numel} elements, has {t.numel()}")
    return t


# ---------------------------------------------------------------------------------------
# descriptors
# ---------------------------------------------------------------------------------------
def make_coeff(desc, grid=None, plane0=0):
    """wgq_coeff_t from a descriptor dict (inputs/configs.py); grid = device tensor."""
    c = wgq_coeff_t()
    kind = desc["kind"]
    keep = []
    if kind == "const":
        c.kind = WGQ_COEF_CONST
        c.c0 = float(desc["c0"])
    elif kind == "trig_sep":
        c.kind = WGQ_COEF_TRIG_SEP
        c.c0 = float(desc["c0"])
        c.amp = float(desc["amp"])
        for a, (tr, k) in enumerate(zip(desc["trig"], desc["wavenum"])):
            c.trig[a] = WGQ_TRIG_SIN if tr == "sin" else WGQ_TRIG_COS
            c.wavenum[a] = int(k)
    elif kind == "fourier_logn":
        c.kind = WGQ_COEF_FOURIER_LOGN
        modes = np.ascontiguousarray(desc["modes"], dtype=np.float64)
        c.n_modes = modes.shape[0]
        buf = (ctypes.c_double * modes.size)(*modes.reshape(-1))
        keep.append(buf)
        c.modes = ctypes.cast(buf, ctypes.POINTER(ctypes.c_double))
    elif kind == "grid":
        c.kind = WGQ_COEF_GRID
        if grid is None:
            raise ValueError("grid coefficient needs a device grid tensor")
        if not hasattr(grid, "arr"):                   # bench's host-array adapter is checked by the library
            _need(grid, "grid")
        c.grid = grid.data_ptr()
        keep.append(grid)                  # the descriptor holds a raw pointer: keep the tensor alive
        c.grid_plane0 = int(plane0)
        c.grid_planes = int(grid.shape[0])
    else:
        raise ValueError(kind)
    c._keep = keep
    return c


def make_out(values, row_begin, row_end, ld=None, layout=WGQ_ELL, row_ptr=None):
    o = wgq_out_t()
    o.layout = layout
    o.row_begin, o.row_end = int(row_begin), int(row_end)
    if values is not None:
        rows = max(0, int(row_end) - int(row_begin))
        if layout == WGQ_ELL:
            lde = int(ld if ld is not None else (values.shape[1] if values.dim() == 2 else 0))
            _need(values, "values", numel=rows * lde)
        else:
            _need(values, "values")
    if row_ptr is not None:
        _need(row_ptr, "row_ptr", "int64", numel=max(0, int(row_end) - int(row_begin)) + 1)
    o.values = values.data_ptr() if values is not None else None
    o.ld = int(ld if ld is not None else (values.shape[1] if values is not None and values.dim() == 2 else 0))
    o.row_ptr = row_ptr.data_ptr() if row_ptr is not None else None
    o.col_idx = None
    return o


# ---------------------------------------------------------------------------------------
# assembly / inputs / checks
# ---------------------------------------------------------------------------------------
def wgq_assemble_mass(rules, coeff, M, stream=None):
    _check("wgq_assemble_mass", lib().wgq_assemble_mass(rules.handle, ctypes.byref(coeff), ctypes.byref(M), _stream(stream)))


def wgq_assemble_stiffness(rules, coeff, K, stream=None):
    _check("wgq_assemble_stiffness",
           lib().wgq_assemble_stiffness(rules.handle, ctypes.byref(coeff), ctypes.byref(K), _stream(stream)))


def wgq_assemble_mass_stiffness(rules, coeff, M, K, stream=None):
    _check("wgq_assemble_mass_stiffness",
           lib().wgq_assemble_mass_stiffness(rules.handle, ctypes.byref(coeff), ctypes.byref(M), ctypes.byref(K),
                                             _stream(stream)))


def wgq_csr_structure(rules, row_begin, row_end, row_ptr, col_idx, stream=None):
    _need(row_ptr, "row_ptr", "int64", numel=max(0, row_end - row_begin) + 1)
    if col_idx is not None:
        _need(col_idx, "col_idx", "int32", numel=wgq_nnz(rules, row_begin, row_end))
    _check("wgq_csr_structure", lib().wgq_csr_structure(rules.handle, row_begin, row_end, row_ptr.data_ptr(),
                                                        col_idx.data_ptr() if col_idx is not None else None,
                                                        _stream(stream)))


def wgq_assemble_load(rules, f, row_begin, row_end, b, stream=None):
    _need(b, "b", numel=max(0, row_end - row_begin))
    _check("wgq_assemble_load", lib().wgq_assemble_load(rules.handle, ctypes.byref(f), row_begin, row_end, b.data_ptr(),
                                                        _stream(stream)))


def wgq_apply(rules, coeff, u, u_row0, row_begin, row_end, yM=None, yK=None, stream=None):
    ptr = (lambda t: t.data_ptr() if t is not None else None)
    _need(u, "u")
    for name, y in (("yM", yM), ("yK", yK)):
        if y is not None:
            _need(y, name, numel=max(0, row_end - row_begin))
    _check("wgq_apply", lib().wgq_apply(rules.handle, ctypes.byref(coeff), u.data_ptr(), u_row0, u.numel(), row_begin,
                                        row_end, ptr(yM), ptr(yK), _stream(stream)))


def wgq_generate_grid(n_elems, dim, seed, sigma, plane0, planes, grid, stream=None):
    """n_elems: an int (every direction) or one count per direction (wgq_generate_grid_ex)."""
    ns = [int(n_elems)] * dim if np.ndim(n_elems) == 0 else [int(v) for v in n_elems]
    plane = int(np.prod([v + 1 for v in ns[:dim - 1]])) if dim > 1 else 1
    _need(grid, "grid", numel=planes * plane if dim > 1 else ns[0] + 1)
    arr = (ctypes.c_int64 * 3)(*(ns + [1] * (3 - dim)))
    _check("wgq_generate_grid_ex", lib().wgq_generate_grid_ex(arr, dim, seed, sigma, plane0, planes, grid.data_ptr(),
                                                              _stream(stream)))


def wgq_row_moments(rules, A, out, stream=None):
    _need(out, "out", numel=max(0, A.row_end - A.row_begin) * (1 + rules.dim))
    _check("wgq_row_moments", lib().wgq_row_moments(rules.handle, ctypes.byref(A), out.data_ptr(), _stream(stream)))


def wgq_checksum(rules, A, out, stream=None):
    if out.element_size() != 8 or out.numel() < 3 or not out.is_cuda or not out.is_contiguous():
        raise ValueError("out: expected a contiguous CUDA tensor of >= 3 8-byte elements")
    _check("wgq_checksum", lib().wgq_checksum(rules.handle, ctypes.byref(A), out.data_ptr(), _stream(stream)))


def _need_host(a, name, numel, writeable=True):
    if a is None:
        return
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: expected a numpy array")
    if a.dtype != np.float64:
        raise TypeError(f"{name}: expected dtype float64, got {a.dtype}")
    if not a.flags["C_CONTIGUOUS"] or (writeable and not a.flags["WRITEABLE"]):
        raise ValueError(f"{name}: expected a {'writeable ' if writeable else ''}C-contiguous array")
    if a.size < numel:
        raise ValueError(f"{name}: needs at least {numel} elements, has {a.size}")


def wgq_assemble_host(rules, coeff, row_begin, row_end, M_host, K_host, ld, chunk_rows=0):
    """Blocking end-to-end call; M_host / K_host are numpy arrays (or None) [rows][ld]."""
    rows = max(0, int(row_end) - int(row_begin))
    _need_host(M_host, "M_host", rows * int(ld))
    _need_host(K_host, "K_host", rows * int(ld))
    g = coeff._keep[0] if coeff.kind == WGQ_COEF_GRID and coeff._keep else None
    if g is not None and hasattr(g, "arr"):          # host grid slab: [grid_planes][plane]
        plane = (rules.n + 1) ** (rules.dim - 1)
        _need_host(g.arr, "grid", coeff.grid_planes * plane, writeable=False)
    ptr = (lambda a: a.ctypes.data if a is not None else None)
    _check("wgq_assemble_host", lib().wgq_assemble_host(rules.handle, ctypes.byref(coeff), row_begin, row_end,
                                                        ptr(M_host), ptr(K_host), ld, chunk_rows))


class HostGrid:
    """A host (numpy, float64, C-contiguous) GRID slab [planes][...] for wgq_assemble_host,
    which copies it to the device itself; pass it to make_coeff in place of a device tensor."""

    def __init__(self, arr):
        self.arr = arr
        self.shape = arr.shape

    def data_ptr(self):
        return self.arr.ctypes.data


class PinnedArray:
    """numpy view of page-locked host memory from wgq_host_alloc (freed on close/del)."""

    def __init__(self, shape, dtype=np.float64):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        _check("wgq_host_alloc", lib().wgq_host_alloc(max(nbytes, 8), ctypes.byref(p)))
        self._ptr = p
        buf = (ctypes.c_char * max(nbytes, 8)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def close(self):
        if getattr(self, "_ptr", None) is not None and _lib is not None:
            self.array = None
            _lib.wgq_host_free(self._ptr)
            self._ptr = None

    def __del__(self):
        self.close()
