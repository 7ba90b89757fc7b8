# exact K-NN: parity tests + C3 timing (sample and full graph)
timeout 900 python -m pytest tests/test_exact.py tests/test_l2.py -x -q -p no:cacheprovider > gpurun_out/pytest_exact.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_exact.log
tail -5 gpurun_out/pytest_exact.log
timeout 300 python tools/exact_probe.py 1000000 20 20 10000 2>&1 | tail -2
timeout 600 python tools/exact_probe.py 1000000 20 20 all 2>&1 | tail -2
timeout 300 python tools/exact_probe.py 1000000 50 30 10000 2>&1 | tail -2
