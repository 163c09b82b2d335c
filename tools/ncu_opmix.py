"""Dynamic instruction mix of an ncu report: executed warp instructions per SASS opcode
(and per opcode class), from the source page's per-instruction counts.

    python tools/ncu_opmix.py report.ncu-rep [units]      # units: divide counts by this (e.g. rows)
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter()
stall = collections.Counter()
for r in rows[2:]:
    try:
        ex = float(r[idx["Instructions Executed"]].replace(",", "") or 0)
        st = float(r[idx["Warp Stall Sampling (All Samples)"]].replace(",", "") or 0)
    except (ValueError, IndexError):
        continue
    src = r[idx["Source"]].strip()
    tok = src.split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
    op = op.split(".")[0]
    ops[op] += ex
    stall[op] += st
tot = sum(ops.values())
ts = sum(stall.values()) or 1
print(f"total {tot:.4g} warp instructions ({tot / units:.1f} per unit)")
for op, n in ops.most_common(40):
    print(f"{op:10s} {n / units:9.2f} per unit  {100 * n / tot:5.1f}% inst  {100 * stall[op] / ts:5.1f}% stall")
