# ncu --set full capture of the generic correlation kernel (args: tag [config], default g5)
mkdir -p gpurun_out
T=${1:-gen}; C=${2:-g5}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_gen_corr" -s 1 -c 1 -o gpurun_out/${T}_prof_gen -f python bench.py --config $C --steps 2 --warmup 3 --batch 16 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/${T}_prof_gen.log 2>&1
tail -2 gpurun_out/${T}_prof_gen.log
