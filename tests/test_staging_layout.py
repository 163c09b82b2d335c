"""The C3 interior kernel's bank-permuted staging layout (fourier2d.cu, kF2iSlot) is a valid,
conflict-free slot assignment: for either run shift the 50 pairs map to distinct 16-byte slots of
the 112-double run, every x-stage write phase costs the minimum 2 wavefronts, the run reads the
minimum, and the shifted-run edge offsets kF2iEdge0/1 point at elements 0 and 97.  The tables are
parsed from the CUDA source so the kernel and tools/staging_layout.py cannot drift apart.
(Host logic only: a wrong table would silently corrupt the staged rows; the GPU parity tests
catch that too, this pins the performance property.)"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import staging_layout as sl  # noqa: E402


def _source_tables():
    src = open(os.path.join(ROOT, "paper_1710_01048_b200", "csrc", "fourier2d.cu")).read()
    body = re.search(r"kF2iSlot\[2\]\[50\]\s*=\s*\{(.*?)\};", src, re.S).group(1)
    nums = [int(x) for x in re.findall(r"\d+", body)]
    assert len(nums) == 100
    edges = {k: v for k, v in re.findall(r"constexpr int (kF2iEdge[01]) = ([0-9 *+]+);", src)}
    run = int(re.search(r"constexpr int kF2iRun = (\d+);", src).group(1))
    return [nums[:50], nums[50:]], {k: eval(v) for k, v in edges.items()}, run


def test_source_matches_tool():
    tabs, _, _ = _source_tables()
    assert tabs == sl.COMMITTED


def test_slots_are_a_bijection_inside_the_run():
    tabs, _, run = _source_tables()
    for sh in (0, 1):
        assert len(set(tabs[sh])) == 50
        assert max(tabs[sh]) * 2 + 1 < run            # 16-byte slots inside the run's staging


def test_wavefronts_are_minimal():
    tabs, _, _ = _source_tables()
    for sh in (0, 1):
        writes, r1, r2 = sl.cost(tabs[sh], sh)
        assert writes == [2, 2, 2, 2]                   # 28 / 21 lanes x 8 bytes: 2 half-warp phases
        assert r1 == 4                                   # 32 lanes x 16 bytes: 4 quarter-warp phases
        assert r2 == (3 if sh == 0 else 2)               # lanes 0..16-sh: 3 / 2 phases
    # the natural layout (round 1) pays 4 wavefronts per write: the property is not vacuous
    assert sl.cost(list(range(50)), 0)[0] == [4, 4, 4, 4]


def test_edge_offsets():
    tabs, edges, _ = _source_tables()
    # shifted run: element e lives at staging element s = e + 1 -> slot[s >> 1], half s & 1
    assert edges["kF2iEdge0"] == 2 * tabs[1][0] + 1     # element 0 (s = 1)
    assert edges["kF2iEdge1"] == 2 * tabs[1][49]        # element 97 (s = 98)
