# A/B of the Q23 screen at C3 (per-class timings + untimed descents), after its parity tests
timeout 600 python -m pytest tests/test_q23.py -x -q -p no:cacheprovider > gpurun_out/q23_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q23_tests.log
tail -5 gpurun_out/q23_tests.log
bash tools/class_timing.sh "KNND_Q23=0" "KNND_Q23=1"
grep -E "==|class|untimed|rep|  r[0-9]" gpurun_out/class_timing.log | cut -c1-150
