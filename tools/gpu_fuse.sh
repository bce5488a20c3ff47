mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_iffile.py -q -x > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
timeout 300 python bench.py --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/ab_fused.json 2>&1
GACQ_FUSE=0 timeout 300 python bench.py --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/ab_nofuse.json 2>&1
timeout 300 python bench.py --config c1 --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/ab_fused_c1.json 2>&1
