"""Per-CUDA-source-line instructions / stall samples / shared-memory bank conflicts of an ncu
report (source page, sass+cuda view: the rows with a line number are the CUDA lines).

    python tools/ncu_lines2.py REPORT FILE_SUBSTRING [first_line last_line]
"""
import csv
import io
import subprocess
import sys

rep, fsub = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10 ** 9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, res = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or not r[0].isdigit() or hdr is None or cur is None or fsub not in cur:
        continue
    ln = int(r[0])
    if not lo <= ln <= hi:
        continue

    def f(k):
        try:
            return float(r[hdr.index(k)].replace(",", "") or 0)
        except (ValueError, IndexError):
            return 0.0
    conf = [h for h in hdr if "Wavefronts Shared Excessive" in h]
    res.append((ln, f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"),
                f(conf[0]) if conf else 0.0, r[1][:80]))
ti = sum(x[1] for x in res) or 1
ts = sum(x[2] for x in res) or 1
tc = sum(x[3] for x in res) or 1
for ln, i, s, c, src in res:
    if i / ti > 0.004 or s / ts > 0.004 or c / tc > 0.02:
        print(f"{ln:5d} inst {100 * i / ti:5.1f}% stall {100 * s / ts:5.1f}% conf {100 * c / tc:5.1f}%  {src}")
