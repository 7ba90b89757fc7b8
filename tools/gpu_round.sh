bash tools/gpu_full.sh
python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall > gpurun_out/bench_short.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall > gpurun_out/ncu_bench.log 2>&1
KNND_CLASS_TIMING=1 ncu --set full --clock-control none --import-source on -k regex:join_warp_kernel -s 9 -c 1 -o gpurun_out/bench_w1 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall > gpurun_out/ncu_bench_full.log 2>&1
tail -1 gpurun_out/bench.log
