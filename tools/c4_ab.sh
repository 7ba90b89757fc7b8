# C4 (d = 50, K = 30) with the fp32 rows and with 160-byte Q23 rows, after the parity tests
timeout 900 python -m pytest tests/test_q23.py tests/test_gpu.py -m "gpu" -x -q -p no:cacheprovider -k "q23 or size_classes or c4" > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c4.log
tail -3 gpurun_out/pytest_c4.log
rm -f gpurun_out/c4_ab.log
for e in "KNND_Q23=0" "KNND_Q23=1"; do
  echo "== $e" >> gpurun_out/c4_ab.log
  env $e timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-recall >> gpurun_out/c4_ab.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/c4_ab.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value %.4e ms/step %.2f frac %.3f join %.4e/s clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["comparisons_per_s"], d["clocks"]))
    else:
        print(l.rstrip()[:200])
PY
