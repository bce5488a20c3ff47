mkdir -p gpurun_out
timeout 600 python tools/k2_ab.py --config c3 --batch 256 new > gpurun_out/k2ab.log 2>&1
cat gpurun_out/k2ab.log | cut -c1-250
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
