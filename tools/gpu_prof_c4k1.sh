mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_fwd_pfa" -s 1 -c 1 -o gpurun_out/prof_c4k1 -f python bench.py --config c4 --steps 2 --warmup 3 --batch 4 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/prof_c4k1.log 2>&1
