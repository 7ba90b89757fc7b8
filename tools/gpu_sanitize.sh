#!/bin/bash
# compute-sanitizer over tools/sanitize_workload.py (every libknnd kernel, checked
# against the C oracle).  ONE tool per invocation (and per gpurun call: running
# several tools in one call has left B200s unusable on this pool).
#   usage: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck [outdir]
set -u
tool=${1:-memcheck}
out=${2:-gpurun_out}
mkdir -p "$out"
extra=""
[ "$tool" = memcheck ] && extra="--leak-check no"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --error-exitcode 9 --print-limit 100 \
  python tools/sanitize_workload.py > "$out/sanitize_$tool.log" 2>&1
rc=$?
tail -3 "$out/sanitize_$tool.log"
echo "sanitize $tool rc=$rc"
exit $rc
