# full ncu capture of one 2^12 block-class join launch of a C3 bench step; the report is kept (51 MB)
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall"
rm -f gpurun_out/*.ncu-rep
$B > gpurun_out/bench_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:join_kernel<\(int\)128, \(int\)4, \(int\)1, \(bool\)0, \(bool\)0' -s 9 -c 1 -o gpurun_out/bench_b128 $B > gpurun_out/ncu_bench_b128.log 2>&1
ls -la gpurun_out/*.ncu-rep
