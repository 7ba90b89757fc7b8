# try size-class plans on the C3 probe (rounds time + per-round join ms)
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for plan in default "w11,w12,b256:14" "w11,b128:12,b256:14" "w11,b128:12,b128:13,b256:15" "b128:11,b128:12,b256:14" "w11,b128:13,b256:15" "w11,b256:12,b256:14"; do
  if [ "$plan" = default ]; then unset KNND_PLAN; else export KNND_PLAN="$plan"; fi
  echo "== $plan" >> gpurun_out/tune.log
  timeout 120 python tools/probe.py 1000000 20 20 2 2>&1 | tail -8 >> gpurun_out/tune.log
done
unset KNND_PLAN
tail -1 gpurun_out/pytest_gpu.log
