# ncu --set full captures of one B128 (2^12), one B256 join launch of a C3 bench step and
# one C5 W1 launch; summarised on the box (evidence text), reports deleted (gpurun_out <= 64 MiB)
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall"
summ() {  # report label
  python tools/ncu_evidence.py gpurun_out/$1.ncu-rep "$2" > gpurun_out/$1_evidence.txt 2>&1
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/$1.ncu-rep 30 > gpurun_out/$1_lines.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
KNND_CLASS_TIMING=1 $B > gpurun_out/bench_short_ct.log 2>&1 && \
KNND_CLASS_TIMING=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:join_kernel<\(int\)128, \(int\)4, \(int\)1, \(bool\)0, \(bool\)0' -s 9 -c 1 -o gpurun_out/bench_b128 $B > gpurun_out/ncu_bench_b128.log 2>&1
summ bench_b128 "B128 (2^12 table) join launch, C3 bench step"
KNND_CLASS_TIMING=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:join_kernel<\(int\)256' -s 4 -c 1 -o gpurun_out/bench_b256 $B > gpurun_out/ncu_bench_b256.log 2>&1
summ bench_b256 "B256 (2^14 table) join launch, C3 bench step"
C5="python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks --no-recall"
$C5 > gpurun_out/bench_c5_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:join_warp_kernel -s 2 -c 1 -o gpurun_out/bench_c5_w1 $C5 > gpurun_out/ncu_c5.log 2>&1
summ bench_c5_w1 "C5 W1 join launch (Q23 screen), bench step"
python tools/exact_probe.py 1000000 20 20 100000 > gpurun_out/exact_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:exact_tc -s 1 -c 1 -o gpurun_out/exact_tc \
    python tools/exact_probe.py 1000000 20 20 100000 > gpurun_out/ncu_exact.log 2>&1
summ exact_tc "tensor-core exact K-NN screen, 100k queries x 1M points (C3)"
ls -la gpurun_out
