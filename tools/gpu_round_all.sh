bash tools/gpu_round.sh
for c in c1 c2 c4 d8 g5 g8; do timeout 600 python bench.py --config $c --steps 10 --tracking-epochs 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
