"""Aggregate ncu stall samples and executed instructions per CUDA source line."""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
extra = sys.argv[3:]  # e.g. --launch-skip 1 --launch-count 1; "--col stall_no_inst" ranks by one stall reason
col = None
if "--col" in extra:
    i = extra.index("--col")
    col = extra[i + 1]
    extra = extra[:i] + extra[i + 2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", *extra],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: [0, 0, ""])
fname = None
hdr = None
tot = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_s = hdr.index(col) if col else 4
        i_ex = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    s = int(r[i_s] or 0)
    e = int(r[i_ex] or 0)
    key = (fname, int(r[0]))
    agg[key][0] += s
    agg[key][1] += e
    agg[key][2] = r[1][:70]
    tot += s
top = sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
print("total samples", tot)
for (f, ln), (s, e, src) in top:
    print(f"{100 * s / tot:5.1f}% {e / 1e6:8.1f}M {f}:{ln:<4d} {src}")
