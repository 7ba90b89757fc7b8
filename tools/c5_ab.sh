# C5 bench line with the Q15 screen (default there) and with the Q23 screen
for e in "KNND_Q23=0" "KNND_Q23=1"; do
  echo "== $e" >> gpurun_out/c5_ab.log
  env $e timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-recall >> gpurun_out/c5_ab.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/c5_ab.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value %.4e ms/step %.2f frac %.3f join %.4e/s clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["comparisons_per_s"], d["clocks"]))
    else:
        print(l.rstrip()[:200])
PY
