"""Copy the judged evidence from gpurun_out/ into profiles/ (round-tagged).

  profiles/<tag>_bench_c3.json            bench.py JSON line (B200 arm)
  profiles/<tag>_bench_reference_c3.json  bench.py --impl reference JSON line
  profiles/<tag>_bench_c{2,4,5}.json      bench.py --config c2/c4/c5 JSON lines
  profiles/<tag>_ncu_launches_c3.json     per-launch gpu__time_duration of one bench step (ncu, cold cache)
  profiles/<tag>_ncu_join_w1_summary.txt  ncu --set full summary of one W1 local-join launch
  profiles/<tag>_ncu_join_w1_lines.txt    per-source-line stall samples / instructions of that launch
  profiles/ncu_join_c3.json               dram bytes per launch of that capture (bench.py roofline.traffic)
"""
import csv, json, os, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
SKIP = 9  # the ncu capture's -s (W1 launches skipped)
G = "gpurun_out"
P = "profiles"
os.makedirs(P, exist_ok=True)
for src, dst in (("bench.log", "bench_c3.json"), ("bench_ref.log", "bench_reference_c3.json"),
                 ("bench_c2.log", "bench_c2.json"), ("bench_c4.log", "bench_c4.json"), ("bench_c5.log", "bench_c5.json")):
    p = os.path.join(G, src)
    if os.path.exists(p):
        line = open(p).readline().strip()
        json.loads(line)
        open(os.path.join(P, f"{tag}_{dst}"), "w").write(line + "\n")
p = os.path.join(G, "bench_launches.csv")
if os.path.exists(p):
    rows = list(csv.reader(open(p)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iK, iV, iG, iB = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
    launches = [{"kernel": r[iK][:100], "grid": r[iG], "block": r[iB], "ns": float(r[iV])} for r in rows[start + 1:]
                if len(r) > iV]
    tot = sum(x["ns"] for x in launches)
    ours = [x for x in launches if "knnd::" in x["kernel"]]
    join = sum(x["ns"] for x in ours if "join" in x["kernel"] or "classify" in x["kernel"])
    by = {}
    for x in launches:
        k = x["kernel"].split("(")[0]
        by[k] = by.get(k, 0) + x["ns"]
    json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 1 "
                          "--warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks",
               "note": "cold-cache, serialised launches (warm-up + 1 timed step): compare shares, not absolutes",
               "total_ms": tot / 1e6, "local_join_share_of_gpu_time": join / tot,
               "ms_by_kernel": {k: v / 1e6 for k, v in sorted(by.items(), key=lambda t: -t[1])},
               "n_launches": len(launches), "n_knnd_launches": len(ours), "launches": launches},
              open(os.path.join(P, f"{tag}_ncu_launches_c3.json"), "w"), indent=1)
rep = os.path.join(G, "bench_w1.ncu-rep")
if os.path.exists(rep):
    s = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
    open(os.path.join(P, f"{tag}_ncu_join_w1_summary.txt"), "w").write(s)
    s = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "40"], capture_output=True, text=True).stdout
    open(os.path.join(P, f"{tag}_ncu_join_w1_lines.txt"), "w").write(s)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2]
    def metric(name):
        i = h.index(name)
        return float(v[i].replace(",", "")), rows[1][i]
    rd, ru = metric("dram__bytes_read.sum")
    wr, wu = metric("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = rd * scale.get(ru, 1) + wr * scale.get(wu, 1)
    dur, du = metric("gpu__time_duration.sum")
    # the captured launch's comparisons: the ncu command ran with KNND_CLASS_TIMING=1,
    # which prints one line per class launch; the capture is the (skip+1)-th W1 line
    comps = None
    logp = os.path.join(G, "ncu_bench_full.log")
    if os.path.exists(logp):
        w1 = [int(l.split(" anchors, ")[1].split(" ")[0]) for l in open(logp) if " kind 0 " in l and "anchors," in l]
        if len(w1) > SKIP:
            comps = w1[SKIP]
    out = {"capture": f"{tag}: ncu --set full, one W1 join_warp_kernel launch of a C3 bench step "
                      f"(launch index {SKIP}: round 3 of the second descent)",
           "dram_bytes_per_launch": dram, "duration": [dur, du]}
    if comps:
        out.update({"comparisons": comps, "algorithmic_bytes_per_launch": 80 * comps,
                    "dram_over_algorithmic": dram / (80 * comps)})
    json.dump(out, open(os.path.join(P, "ncu_join_c3.json"), "w"), indent=1)
print(sorted(os.listdir(P)))
