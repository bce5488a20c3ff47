mkdir -p gpurun_out
GACQ_LIB=exp/libgacq_rader.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_rader.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rader.log
bash tools/gpu_ab.sh direct rader
