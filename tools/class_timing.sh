# per-class join timing (KNND_CLASS_TIMING) at C3 for the given env settings; usage: bash tools/class_timing.sh "ENV=.." ...
rm -f gpurun_out/class_timing.log
for e in "$@"; do
  echo "== $e" >> gpurun_out/class_timing.log
  env $e KNND_CLASS_TIMING=1 timeout 120 python tools/probe.py 1000000 20 20 1 >> gpurun_out/class_timing.log 2>&1
  echo "-- untimed" >> gpurun_out/class_timing.log
  env $e timeout 120 python tools/probe.py 1000000 20 20 2 2>&1 | tail -8 >> gpurun_out/class_timing.log
done
