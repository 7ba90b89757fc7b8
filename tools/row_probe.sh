# random-row gather rate by row size and occupancy (tools/row_probe.cu)
rm -f gpurun_out/row_probe.txt
for n in 1000000 10000000; do
  for ld in 4 8 12 16 20; do
    for b in 4 8; do
      ./tools/row_probe$ld $n 256 $b >> gpurun_out/row_probe.txt 2>&1
    done
  done
done
cat gpurun_out/row_probe.txt
