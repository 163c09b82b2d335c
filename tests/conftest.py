import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; runs the CUDA path through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session")
def cuda_lib():
    """The built C-ABI library (GPU tests only; fails loudly if it is missing)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1710_01048_b200 import wgq
    return wgq.lib()


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Parity summary (tests/parity.py): raw vs floored entrywise error over every comparison."""
    try:
        import parity
    except Exception:
        return
    recs = parity.RECORDS
    if not recs:
        return
    import json
    worst = max(recs, key=lambda r: r["max_rel_raw"])
    need = [r for r in recs if r["entries_needing_floor"]]
    tr = terminalreporter
    tr.write_line(f"parity: {len(recs)} comparisons, {sum(r['entries'] for r in recs)} entries; "
                  f"max rel-Frobenius {max(r['rel_frobenius'] for r in recs):.2e}; "
                  f"max entrywise (floored) {max(r['max_rel'] for r in recs):.2e}; "
                  f"max entrywise RAW {worst['max_rel_raw']:.2e} ({worst['what']}); "
                  f"{sum(r['entries_needing_floor'] for r in recs)} entries in {len(need)} comparisons need the R12 floor")
    for r in sorted(need, key=lambda r: -r["entries_needing_floor"])[:12]:
        tr.write_line(f"  floor used: {r['what']}: {r['entries_needing_floor']} of {r['entries']} entries, "
                      f"raw {r['max_rel_raw']:.2e}, floored {r['max_rel']:.2e}")
    path = os.environ.get("WGQ_PARITY_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(recs, f, indent=0)
