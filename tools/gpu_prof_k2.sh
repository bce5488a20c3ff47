mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_corr_pfa" -s 1 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 3 --warmup 3 --batch 64 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/prof_k2.log 2>&1
tail -2 gpurun_out/prof_k2.log | cut -c1-300
