# Euclidean scorer: parity tests, then the n = 1M, d = 20, K = 20 descent with the fp32 rows and the Q23 rows
timeout 900 python -m pytest tests/test_l2.py tests/test_fuzz_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_l2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_l2.log
tail -4 gpurun_out/pytest_l2.log
for e in "KNND_Q23=0" "KNND_Q23=1"; do echo "== $e"; env $e timeout 600 python tools/l2_probe.py 1000000 20 20 2>&1 | tail -3; done
