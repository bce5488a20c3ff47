mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c3}; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/q_$c.json 2>&1; done
