# try size-class plans on the C3 probe (rounds time); usage: bash tools/tune_plan.sh "plan1" "plan2" ...
rm -f gpurun_out/tune.log
for plan in "$@"; do
  if [ "$plan" = default ]; then unset KNND_PLAN; else export KNND_PLAN="$plan"; fi
  echo "== $plan" >> gpurun_out/tune.log
  timeout 120 python tools/probe.py 1000000 20 20 2 2>&1 | tail -8 >> gpurun_out/tune.log
done
