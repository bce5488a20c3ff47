# Bench pass: C3 bench line, reference arm, ncu launch list (args: tag)
mkdir -p gpurun_out
T=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gacq_ -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/${T}_b_ncu.log 2>&1
tail -3 gpurun_out/${T}_bench_c3.err
