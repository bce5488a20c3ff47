mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacq_corr -s 2 -c 1 -o gpurun_out/prof_tc -f python bench.py --steps 3 --warmup 3 --batch 64 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/prof_tc.log 2>&1
tail -3 gpurun_out/prof_tc.log
