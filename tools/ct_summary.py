"""Aggregate gpurun_out/class_timing.log (KNND_CLASS_TIMING=1 runs of tools/class_timing.sh) per size class."""
import collections
import re
import sys

cur = None
agg = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0.0, 0]))
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/class_timing.log"):
    if l.startswith("=="):
        cur = l.strip()
        continue
    m = re.match(r"knnd class (\d+) kind (\d+) logH (\d+): (\d+) anchors, (\d+) comparisons, ([\d.]+) ms", l)
    if m:
        k = (int(m[1]), int(m[2]), int(m[3]))
        a = agg[cur][k]
        a[2] += 1
        if a[2] == 1 and k[0] != 0:
            continue  # the first launch of a kernel pays its module load: not a rate
        a[0] += int(m[5])
        a[1] += float(m[6])
    if l.startswith("rep 1"):
        print(cur, l.strip())
for c, d in agg.items():
    print(c)
    tot = sum(v[1] for v in d.values())
    for k, v in sorted(d.items()):
        print("  class %d kind %d logH %d: %.3e comps %.2f ms (%.0f%%) %.3e/s" % (*k, v[0], v[1], 100 * v[1] / tot, v[0] / max(v[1], 1e-9) * 1e3))
    print("  total ms %.2f" % tot)
