# generic path, warp-split correlation: parity subset, G5/G8 timing with it on and off, one ncu capture (args: tag)
mkdir -p gpurun_out
T=${1:-ws}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_configs.py -q -x -k "golden or generic or power_of_two or random" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for cf in g5 g8; do
  timeout 600 python tools/k2_ab.py --config $cf --batch 64 default 2>&1 | cut -c1-150
  GACQ_GEN_WS=0 timeout 600 python tools/k2_ab.py --config $cf --batch 64 default 2>&1 | cut -c1-150
done
timeout 800 ncu --set full --clock-control none --import-source on -k regex:"gacq_gen_corr" -s 1 -c 1 -o gpurun_out/${T}_prof_gen -f python bench.py --config g5 --steps 3 --warmup 3 --batch 8 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/${T}_prof_gen.log 2>&1
