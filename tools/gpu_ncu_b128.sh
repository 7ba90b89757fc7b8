python tools/probe.py 1000000 20 20 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:^join_kernel -s 6 -c 4 -o gpurun_out/${1:-b128} python tools/probe.py 1000000 20 20 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
