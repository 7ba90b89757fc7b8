# A/B of the join-fused CSR in-degree count (KNND_FUSED_COUNT), C3 bench lines alternated
timeout 900 python -m pytest tests/test_gpu.py tests/test_fuzz_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -3 gpurun_out/pytest_ab.log
for i in 1 2 3; do
  for v in 0 1; do
    KNND_FUSED_COUNT=$v timeout 600 python bench.py --e2e-steps 1 --no-cpu-baseline --no-recall > gpurun_out/ab_$v.log 2>&1
    python - "$v" <<'PY'
import json, sys
for l in open(f"gpurun_out/ab_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("fused=%s value %.4e ms/step %.2f e2e %.4e" % (sys.argv[1], d["value"], d["ms_per_step"], d["e2e"]["value"]))
PY
  done
done
