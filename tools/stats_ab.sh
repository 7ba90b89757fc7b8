# bench lines at C3 and C2 (value only) for the current tree
for c in c3 c2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-recall > gpurun_out/bench_$c.q.log 2>&1
  python - <<PY
import json
for l in open("gpurun_out/bench_$c.q.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("$c value %.4e ms/step %.3f e2e %.4e frac %.3f join %.4e/s share %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["comparisons_per_s"], d["roofline"]["share_of_step"]))
PY
done
