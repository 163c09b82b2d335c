"""Per-CUDA-source-line stall samples and executed instructions of an ncu report
(`--page source --print-source sass,cuda`), top lines first.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ist, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > iex and r[0] not in ("", "Line No"):
        try:
            lines.append((float(r[ist] or 0), float(r[iex] or 0), r[0], r[1]))
        except ValueError:
            pass
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print("samples", ts, "instructions", ti)
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print("%5.1f%% stall %5.1f%% inst  L%-4s %s" % (100 * s / ts, 100 * i / ti, ln, src.strip()[:80]))
