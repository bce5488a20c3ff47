# ncu --set full of one K2 launch at C1 (R = 1): per-item epilogue overhead
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_corr_pfa" -s 1 -c 1 -o gpurun_out/prof_c1 -f python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/prof_c1.log 2>&1
tail -2 gpurun_out/prof_c1.log
