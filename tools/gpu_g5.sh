mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k generic > gpurun_out/pytest_generic.log 2>&1
timeout 600 python bench.py --config g5 --steps 5 --tracking-epochs 1 > gpurun_out/bench_g5.json 2> gpurun_out/bench_g5.err
timeout 600 python bench.py --steps 5 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/bench_c3q.json 2>&1
