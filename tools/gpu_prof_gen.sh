mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_gen_corr" -s 1 -c 1 -o gpurun_out/prof_gen -f python bench.py --config g8 --steps 2 --warmup 3 --batch 8 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/prof_gen.log 2>&1
