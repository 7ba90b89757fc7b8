# parity tests + C3 probe + per-launch list (ncu) of one C3 run
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py 1000000 20 20 2 > gpurun_out/probe_c3.log 2>&1
python tools/probe.py 1000000 20 20 1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/probe.py 1000000 20 20 1 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
