# quick parity subset (q23 + fuzz + core gpu tests, not slow) then class timing at C3
timeout 900 python -m pytest tests/test_q23.py tests/test_fuzz_gpu.py tests/test_gpu.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
bash tools/class_timing.sh "${1:-KNND_Q23=1}"
