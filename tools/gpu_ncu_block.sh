python tools/probe.py 1000000 20 20 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:^join_kernel -s 4 -c 3 -o gpurun_out/${1:-block_c3} python tools/probe.py 1000000 20 20 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
