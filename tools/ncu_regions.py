"""Instructions / stall samples of an ncu report grouped by source function (line ranges of
assemble_line.cu are found by scanning the source for the function headers)."""
import csv
import io
import re
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
rows_per_launch = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
heads = []
for i, l in enumerate(open(src), 1):
    m = re.match(r"^(?:__device__|__global__|template|struct|int |bool ).*?\b(\w+)\s*\(", l)
    if m and not l.startswith("template"):
        heads.append((i, m.group(1)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = {}
for r in rows:
    if len(r) > ie and r[0] not in ("", "Line No"):
        try:
            ln, ins, st = int(r[0]), float(r[ie] or 0), float(r[ist] or 0)
        except ValueError:
            continue
        name = "?"
        for hl, hn in heads:
            if hl <= ln:
                name = hn
        a = agg.setdefault(name, [0.0, 0.0])
        a[0] += ins
        a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print("%-24s inst %5.1f%% (%7.1f/row)  stall %5.1f%%" % (k, 100 * i / ti, i / rows_per_launch, 100 * s / ts))
