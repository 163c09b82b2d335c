"""The GPU-vs-oracle comparison every parity test uses (north_star; R12).

Bar: relative Frobenius <= 1e-12 and max entrywise relative <= 1e-10.  The entrywise
denominator is max(|o|, 1e-14 max_row |o|, F) with F = 64 eps / 1e-10 * sum_k |term_k| (the
oracle's absolute-value assembly, ``scale``): an entry smaller than the rounding scale of its
own terms (cancellation) is held to that rounding scale.

Every call records, besides pass/fail, the RAW max entrywise relative error (denominator
max(|o|, 1e-14 max_row |o|), no rounding-scale floor) and how many entries only pass because
of the floor (raw error > 1e-10).  ``pytest_terminal_summary`` in conftest.py prints the
totals, and, if WGQ_PARITY_REPORT names a file, every record is written there as JSON.
"""
import numpy as np

REL_F = 1e-12
REL_E = 1e-10
EPS = np.finfo(np.float64).eps
FLOOR = 64 * EPS / REL_E

RECORDS = []


def compare(gpu, ref, what="", scale=None, rowwise=True):
    """Assert parity; returns (rel_frobenius, max floored entrywise relative error).

    rowwise: the 1e-14 structural-zero floor is relative to each row's maximum (matrices);
    otherwise to the vector's maximum (load vectors, y = A u)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    nrm = np.linalg.norm(ref)
    relf = float(np.linalg.norm(gpu - ref) / (nrm if nrm > 0 else 1.0))
    if rowwise and ref.ndim == 2:
        rowmax = np.max(np.abs(ref), axis=1, keepdims=True)
    else:
        rowmax = np.max(np.abs(ref)) if ref.size else 0.0
    err = np.abs(gpu - ref)
    den_raw = np.maximum(np.abs(ref), 1e-14 * rowmax)
    den = den_raw if scale is None else np.maximum(den_raw, FLOOR * np.asarray(scale))
    raw = err / np.where(den_raw > 0, den_raw, 1.0)
    fl = err / np.where(den > 0, den, 1.0)
    rele = float(fl.max()) if fl.size else 0.0
    raw_max = float(raw.max()) if raw.size else 0.0
    floored = int(np.count_nonzero((raw > REL_E) & (fl <= REL_E)))
    RECORDS.append({"what": str(what), "entries": int(ref.size), "rel_frobenius": relf, "max_rel": rele,
                    "max_rel_raw": raw_max, "entries_needing_floor": floored,
                    "max_abs_err_over_max_abs": float(err.max() / max(np.abs(ref).max(), 1e-300)) if ref.size else 0.0})
    assert relf <= REL_F, (what, relf)
    assert rele <= REL_E, (what, rele, "raw", raw_max, "floored entries", floored)
    return relf, rele
