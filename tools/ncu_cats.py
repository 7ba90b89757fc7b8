"""Executed instructions and stall samples of one ncu capture, grouped by
source region (join.cu line ranges given on the command line as name:lo-hi)."""
import csv, subprocess, sys
from collections import defaultdict

rep, anchors = sys.argv[1], float(sys.argv[2])
ranges = []
for a in sys.argv[3:]:
    name, rng = a.split(":")
    lo, hi = (int(v) for v in rng.split("-"))
    ranges.append((lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0])
fname = hdr = None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    ln = int(r[0])
    cat = fname
    if fname == "join.cu":
        cat = next((n for lo, hi, n in ranges if lo <= ln < hi), "join.cu other")
    agg[cat][0] += int(r[4] or 0)
    agg[cat][1] += int(r[ie] or 0)
S = sum(v[0] for v in agg.values())
E = sum(v[1] for v in agg.values())
for c, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{c:28s} samples {100 * s / S:5.1f}%  instr {100 * e / E:5.1f}%  {e / anchors:7.0f}/anchor")
