# full ncu capture of a late-round W1 local-join launch at C3 (launch index 5 = round 6; after a plain run)
python tools/probe.py 1000000 20 20 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:join_warp_kernel -s ${2:-5} -c 1 -o gpurun_out/${1:-warp_c3_late} python tools/probe.py 1000000 20 20 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
