mkdir -p gpurun_out
./tools/codelet_probe 1034 654 1176 > gpurun_out/codelet_probe.txt 2>&1
cat gpurun_out/codelet_probe.txt
