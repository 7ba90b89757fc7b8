# Round evidence (one call): all GPU tests + smoke + the bench lines (C3 both arms,
# C2/C4/C5), the launch list of one C3 step and the ncu --set full capture of one W1
# join launch (the block-class / C5 / exact K-NN captures: tools/gpu_ncu_blocks.sh,
# summarised on the box — gpurun_out holds 64 MiB).
bash tools/gpu_full.sh
for c in c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall"
$B > gpurun_out/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv $B > gpurun_out/ncu_bench.log 2>&1
KNND_CLASS_TIMING=1 $B > gpurun_out/bench_short_ct.log 2>&1 && \
  KNND_CLASS_TIMING=1 ncu --set full --clock-control none --import-source on -k regex:join_warp_kernel -s 9 -c 1 \
    -o gpurun_out/bench_w1 $B > gpurun_out/ncu_bench_full.log 2>&1
timeout 300 python tools/exact_probe.py 1000000 20 20 all > gpurun_out/exact_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; ls gpurun_out
