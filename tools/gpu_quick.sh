# parity (all GPU tests) then a bench line; prints the headline numbers
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --e2e-steps 2 --no-cpu-baseline --no-recall ${BENCH_ARGS:-} > gpurun_out/bench_q.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_q.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value %.4e ms/step %.2f e2e %.4e frac %.3f join %.4e/s" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["comparisons_per_s"]))
    else:
        print(l.rstrip()[:300])
PY
