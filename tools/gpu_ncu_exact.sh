# ncu capture of the tensor-core exact K-NN screen (10k queries x 1M points, C3)
python tools/exact_probe.py 1000000 20 20 ${Q:-10000} > gpurun_out/exact_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:exact_tc -s 2 -c 1 -o gpurun_out/exact_tc \
  python tools/exact_probe.py 1000000 20 20 ${Q:-10000} > gpurun_out/ncu_exact.log 2>&1
tail -3 gpurun_out/ncu_exact.log
