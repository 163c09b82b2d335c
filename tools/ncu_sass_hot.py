"""Top SASS instructions of an ncu report by stall samples / executed count / smem excess."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def num(r, k):
    try:
        return float(r[idx[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


tot = sum(num(r, key) for r in data) or 1
print("total", key, tot)
for r in sorted(data, key=lambda r: -num(r, key))[:top]:
    print("%6.2f%% %s %-60s exec=%d smemX=%d" % (100 * num(r, key) / tot, r[idx["Address"]], r[idx["Source"]][:60],
                                                  num(r, "Instructions Executed"),
                                                  num(r, "L1 Wavefronts Shared Excessive")))
